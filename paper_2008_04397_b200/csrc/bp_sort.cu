// On-device cell sort (particles.sort_by_cell, particles.py:157-167) and the
// exact periodic fold of int64 moment grids (fields.fold_periodic,
// fields.py:28-47).
//
// Sort: key kernel (geometry.cell_index_of semantics, geometry.py:152-159:
// f64 arithmetic, truncation, clamp of the upper face, x fastest), a stable
// LSD radix sort of (key, index) pairs over ceil(log2(n_cells)) bits, then a
// gather-permute of the 8 particle arrays through one scratch array.
#include <cub/device/device_radix_sort.cuh>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "bp_launch.h"

namespace bp {

namespace {

// int(t / d) exactly as the reference's f64 division then truncation
// (geometry.py:152-159), without the division in the common case: t * (1/d)
// is within 2 ulp of the rounded quotient, so its truncation can only differ
// when the quotient lies within a few ulp of an integer — then divide.
__device__ __forceinline__ int64_t cell_trunc(double t, double d, double rd) {
  double q = t * rd;
  if (fabs(q - rint(q)) <= 8.0 * 2.220446049250313e-16 * fmax(fabs(q), 1.0)) q = t / d;
  return (int64_t)q;
}

// four consecutive particles per thread: 16-byte loads and stores (f32 only)
__global__ void cell_key4_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                 const float* __restrict__ z, int64_t n, double ox, double oy,
                                 double oz, double dx, double dy, double dz, int64_t nx,
                                 int64_t ny, int64_t nz, uint32_t* keys32, uint32_t* idx,
                                 int* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double rx = 1.0 / dx, ry = 1.0 / dy, rz = 1.0 / dz;
  const int64_t n4 = n / 4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += stride) {
    const float4 X = __ldcs(reinterpret_cast<const float4*>(x) + t);
    const float4 Y = __ldcs(reinterpret_cast<const float4*>(y) + t);
    const float4 Z = __ldcs(reinterpret_cast<const float4*>(z) + t);
    const float xs[4] = {X.x, X.y, X.z, X.w}, ys[4] = {Y.x, Y.y, Y.z, Y.w};
    const float zs[4] = {Z.x, Z.y, Z.z, Z.w};
    uint32_t kk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int64_t i = cell_trunc((double)xs[e] - ox, dx, rx);
      int64_t j = cell_trunc((double)ys[e] - oy, dy, ry);
      int64_t k = cell_trunc((double)zs[e] - oz, dz, rz);
      i = i < nx - 1 ? i : nx - 1;
      j = j < ny - 1 ? j : ny - 1;
      k = k < nz - 1 ? k : nz - 1;
      if (i < 0 || j < 0 || k < 0) {
        *bad = 1;
        i = j = k = 0;
      }
      kk[e] = (uint32_t)(i + nx * (j + ny * k));
    }
    __stcs(reinterpret_cast<uint4*>(keys32) + t, make_uint4(kk[0], kk[1], kk[2], kk[3]));
    const uint32_t b = (uint32_t)(4 * t);
    __stcs(reinterpret_cast<uint4*>(idx) + t, make_uint4(b, b + 1, b + 2, b + 3));
  }
}

template <typename P>
__global__ void cell_key_kernel(const P* __restrict__ x, const P* __restrict__ y,
                                const P* __restrict__ z, int64_t n, double ox, double oy,
                                double oz, double dx, double dy, double dz, int64_t nx,
                                int64_t ny, int64_t nz, uint32_t* keys32, int64_t* keys64,
                                uint32_t* idx, int* bad, uint32_t idx0) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double rx = 1.0 / dx, ry = 1.0 / dy, rz = 1.0 / dz;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    int64_t i = cell_trunc((double)x[p] - ox, dx, rx);
    int64_t j = cell_trunc((double)y[p] - oy, dy, ry);
    int64_t k = cell_trunc((double)z[p] - oz, dz, rz);
    i = i < nx - 1 ? i : nx - 1;
    j = j < ny - 1 ? j : ny - 1;
    k = k < nz - 1 ? k : nz - 1;
    if (i < 0 || j < 0 || k < 0) {
      *bad = 1;
      i = j = k = 0;
    }
    const int64_t key = i + nx * (j + ny * k);
    if (keys32) keys32[p] = (uint32_t)key;
    if (keys64) keys64[p] = key;
    if (idx) idx[p] = idx0 + (uint32_t)p;
  }
}

template <typename T>
__global__ void gather_perm(const T* __restrict__ src, const uint32_t* __restrict__ order,
                            T* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
    dst[r] = src[order[r]];
}

// 16-byte-aligned store of four consecutive elements (streaming)
__device__ __forceinline__ void store4(float* d, float a, float b, float c, float e) {
  __stcs(reinterpret_cast<float4*>(d), make_float4(a, b, c, e));
}
__device__ __forceinline__ void store4(double* d, double a, double b, double c, double e) {
  __stcs(reinterpret_cast<double2*>(d), make_double2(a, b));
  __stcs(reinterpret_cast<double2*>(d) + 1, make_double2(c, e));
}

// all eight particle arrays gathered through one read of the order: the
// sorted copy lands in separate destination arrays (no copy back).  Four
// consecutive destinations per thread: 16-byte order loads and stores.
template <typename T>
__global__ void gather_perm8(const T* __restrict__ x, const T* __restrict__ y,
                             const T* __restrict__ z, const T* __restrict__ u,
                             const T* __restrict__ v, const T* __restrict__ w,
                             const T* __restrict__ q, const long long* __restrict__ id,
                             const uint32_t* __restrict__ order, T* __restrict__ ox,
                             T* __restrict__ oy, T* __restrict__ oz, T* __restrict__ ou,
                             T* __restrict__ ov, T* __restrict__ ow, T* __restrict__ oq,
                             long long* __restrict__ oid, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;
  const T* src[7] = {x, y, z, u, v, w, q};
  T* dst[7] = {ox, oy, oz, ou, ov, ow, oq};
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += stride) {
    const uint4 j = __ldcs(reinterpret_cast<const uint4*>(order) + t);
#pragma unroll
    for (int a = 0; a < 7; ++a) {
      if (a == 6 && !q) break;
      const T* sa = src[a];
      store4(dst[a] + 4 * t, sa[j.x], sa[j.y], sa[j.z], sa[j.w]);
    }
    if (id) {
      longlong2* di = reinterpret_cast<longlong2*>(oid + 4 * t);
      __stcs(di, make_longlong2(id[j.x], id[j.y]));
      __stcs(di + 1, make_longlong2(id[j.z], id[j.w]));
    }
  }
  for (int64_t r = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint32_t j = order[r];
#pragma unroll
    for (int a = 0; a < 7; ++a) {
      if (a == 6 && !q) break;
      dst[a][r] = src[a][j];
    }
    if (id) oid[r] = id[j];
  }
}

// One group of the gather: up to 4 same-type arrays and optionally the ids,
// one block per 1024 destinations with no grid stride, so resident blocks
// sweep the destination in order and the sources they touch (a particle
// moves at most a few cells between sorts) stay in a window of about three
// z-planes of the source arrays.  Gathering the arrays in groups keeps that
// window (bytes per particle of the group x plane size) inside L2; all eight
// arrays at once overflow it and every moved particle costs a full sector.
template <typename T>
struct GatherGroup {
  const T* src[4];
  T* dst[4];
  int na;
  const long long* sid;
  long long* did;
};

__device__ __forceinline__ uint64_t keep_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float ld_keep(const float* a, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ long long ld_keep(const long long* a, uint64_t pol) {
  long long v;
  asm volatile("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) gather_group(GatherGroup<T> g,
                                                    const uint32_t* __restrict__ order,
                                                    int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r0 = 4 * t;
  if (r0 + 4 <= n) {
    const uint4 j = __ldcs(reinterpret_cast<const uint4*>(order) + t);
    const uint64_t pol = keep_policy();
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (a >= g.na) break;
      const T* sa = g.src[a];
      store4(g.dst[a] + r0, ld_keep(sa + j.x, pol), ld_keep(sa + j.y, pol),
             ld_keep(sa + j.z, pol), ld_keep(sa + j.w, pol));
    }
    if (g.sid) {
      longlong2* di = reinterpret_cast<longlong2*>(g.did + r0);
      __stcs(di, make_longlong2(ld_keep(g.sid + j.x, pol), ld_keep(g.sid + j.y, pol)));
      __stcs(di + 1, make_longlong2(ld_keep(g.sid + j.z, pol), ld_keep(g.sid + j.w, pol)));
    }
  } else {
    for (int64_t r = r0; r < n; ++r) {
      const uint32_t j = order[r];
      for (int a = 0; a < g.na; ++a) g.dst[a][r] = g.src[a][j];
      if (g.sid) g.did[r] = g.sid[j];
    }
  }
}

int check(cudaError_t e, const char* what);

// the eight arrays in `groups` passes (1: all at once through gather_perm8)
template <typename T>
int gather_grouped(const void* const* src, const void* src_ids, void* const* dst, void* dst_ids,
                   const uint32_t* order, int64_t n, int groups, cudaStream_t s) {
  // arrays 0..6 (q may be null) then ids
  static const int kSplit2[] = {0, 4, 7};
  static const int kSplit3[] = {0, 3, 6, 7};
  const int* cut = groups == 2 ? kSplit2 : kSplit3;
  const int ng = groups == 2 ? 2 : 3;
  const unsigned blocks = (unsigned)((n + 1023) / 1024);
  for (int gi = 0; gi < ng; ++gi) {
    GatherGroup<T> g{};
    g.na = 0;
    for (int a = cut[gi]; a < cut[gi + 1]; ++a) {
      if (!src[a]) continue;
      g.src[g.na] = static_cast<const T*>(src[a]);
      g.dst[g.na] = static_cast<T*>(dst[a]);
      ++g.na;
    }
    if (gi == ng - 1 && src_ids) {
      g.sid = static_cast<const long long*>(src_ids);
      g.did = static_cast<long long*>(dst_ids);
    }
    if (!g.na && !g.sid) continue;
    gather_group<T><<<blocks, 256, 0, s>>>(g, order, n);
    note_launch();
    const int rc = check(cudaGetLastError(), "gather_group");
    if (rc) return rc;
  }
  return 0;
}

int gather_groups_env() {
  static int g = [] {
    const char* e = getenv("BP_GATHER_GROUPS");
    const int v = e ? atoi(e) : 3;
    return v == 1 || v == 2 ? v : 3;
  }();
  return g;
}

// fold one periodic axis of a (rows, NX, NY, NZ) grid: first += last; last = first
__global__ void fold_axis(long long* a, int64_t rows, int NX, int NY, int NZ, int axis) {
  const int n1 = axis == 0 ? NY : NX;
  const int n2 = axis == 2 ? NY : NZ;
  const int64_t plane = (int64_t)n1 * n2;
  const int64_t total = rows * plane;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t r = t / plane;
    const int64_t rem = t - r * plane;
    const int a1 = (int)(rem / n2), a2 = (int)(rem % n2);
    int64_t first, last;
    const int64_t base = r * (int64_t)NX * NY * NZ;
    if (axis == 0) {
      first = base + ((int64_t)0 * NY + a1) * NZ + a2;
      last = base + ((int64_t)(NX - 1) * NY + a1) * NZ + a2;
    } else if (axis == 1) {
      first = base + ((int64_t)a1 * NY + 0) * NZ + a2;
      last = base + ((int64_t)a1 * NY + (NY - 1)) * NZ + a2;
    } else {
      first = base + ((int64_t)a1 * NY + a2) * NZ + 0;
      last = base + ((int64_t)a1 * NY + a2) * NZ + (NZ - 1);
    }
    const long long s = a[first] + a[last];
    a[first] = s;
    a[last] = s;
  }
}

int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (int)b;
}

int check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

template <typename P>
int keys_launch(const void* xs, const void* ys, const void* zs, int64_t n, const double* o,
                const double* d, const int64_t* c, uint32_t* k32, int64_t* k64, uint32_t* idx,
                int* bad, cudaStream_t s, uint32_t idx0) {
  cell_key_kernel<P><<<blocks_for(n), 256, 0, s>>>((const P*)xs, (const P*)ys, (const P*)zs, n,
                                                   o[0], o[1], o[2], d[0], d[1], d[2], c[0],
                                                   c[1], c[2], k32, k64, idx, bad, idx0);
  note_launch();
  return check(cudaGetLastError(), "cell_key_kernel");
}

int keys_any(int pbytes, const void* xs, const void* ys, const void* zs, int64_t n,
             const double* o, const double* d, const int64_t* c, uint32_t* k32, int64_t* k64,
             uint32_t* idx, int* bad, cudaStream_t s, uint32_t idx0 = 0) {
  if (pbytes == 8) return keys_launch<double>(xs, ys, zs, n, o, d, c, k32, k64, idx, bad, s, idx0);
  if (pbytes == 4) return keys_launch<float>(xs, ys, zs, n, o, d, c, k32, k64, idx, bad, s, idx0);
  set_error("unsupported particle dtype (%d bytes)", pbytes);
  return -1;
}

template <typename T>
int permute_one(void* arr, const uint32_t* order, void* tmp, int64_t n, cudaStream_t s) {
  gather_perm<T><<<blocks_for(n), 256, 0, s>>>((const T*)arr, order, (T*)tmp, n);
  note_launch();
  int rc = check(cudaGetLastError(), "gather_perm");
  if (rc) return rc;
  return check(cudaMemcpyAsync(arr, tmp, n * sizeof(T), cudaMemcpyDeviceToDevice, s),
               "permute copy");
}

}  // namespace

int cell_keys(int pbytes, const void* xs, const void* ys, const void* zs, int64_t n,
              const double* origin, const double* spacing, const int64_t* counts,
              int64_t* keys, cudaStream_t s) {
  if (n <= 0) return 0;
  int* bad = nullptr;
  int rc = check(cudaMallocAsync((void**)&bad, sizeof(int), s), "alloc");
  if (rc) return rc;
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  rc = keys_any(pbytes, xs, ys, zs, n, origin, spacing, counts, nullptr, keys, nullptr, bad, s);
  int hbad = 0;
  if (!rc) rc = check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  if (!rc) rc = check(cudaStreamSynchronize(s), "sync");
  cudaFreeAsync(bad, s);
  if (rc) return rc;
  return hbad ? 3 : 0;
}

// Grow-only sort workspaces (keys, indices, permutation scratch, CUB temp
// storage), so periodic sorts do not re-allocate ~40 B/particle.  A sort
// leases an idle workspace of its device for the whole call, so sorts of
// different species on different streams (and host threads) run
// concurrently; the pool grows to the number of concurrent sorts.
struct SortWs {
  void* base = nullptr;
  size_t bytes = 0;
  int dev = -1;
  bool busy = false;
};
static std::mutex g_sort_mu;
static std::vector<SortWs*> g_sort_pool;

class WsLease {
 public:
  // *rc = 0 and ws() >= need bytes on success
  WsLease(size_t need, cudaStream_t s, int* rc) : s_(s) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lock(g_sort_mu);
      for (SortWs* w : g_sort_pool)
        if (w->dev == dev && !w->busy && (!w_ || w->bytes > w_->bytes)) w_ = w;
      if (!w_) {
        w_ = new SortWs;
        w_->dev = dev;
        g_sort_pool.push_back(w_);
      }
      w_->busy = true;
    }
    *rc = 0;
    if (w_->bytes < need) {
      if (w_->base) {
        cudaStreamSynchronize(s);
        cudaFree(w_->base);  // also waits for the device's other streams
        w_->base = nullptr;
        w_->bytes = 0;
      }
      *rc = check(cudaMalloc(&w_->base, need), "sort workspace");
      if (!*rc) w_->bytes = need;
    }
  }
  ~WsLease() {
    cudaStreamSynchronize(s_);  // (early error returns may leave work queued)
    std::lock_guard<std::mutex> lock(g_sort_mu);
    w_->busy = false;
  }
  void* base() const { return w_->base; }

 private:
  SortWs* w_ = nullptr;
  cudaStream_t s_;
};

int sort_by_cell(int pbytes, void* xs, void* ys, void* zs, void* us, void* vs, void* ws,
                 void* qs, int64_t* ids, int64_t n, const double* origin,
                 const double* spacing, const int64_t* counts, cudaStream_t s) {
  if (n <= 1) return 0;
  if (n > 0xffffffffLL) {
    set_error("sort_by_cell: %lld particles exceed the 32-bit index space", (long long)n);
    return -1;
  }
  const int64_t ncell = counts[0] * counts[1] * counts[2];
  int end_bit = 1;
  while (end_bit < 32 && (1LL << end_bit) < ncell) ++end_bit;
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, end_bit, s);
  auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t nb = up((size_t)n * sizeof(uint32_t));
  const size_t need = 4 * nb + up(sizeof(int)) + up((size_t)n * 8) + up(cub_bytes);
  int lrc = 0;
  WsLease lease(need, s, &lrc);
  if (lrc) return lrc;
  char* p = static_cast<char*>(lease.base());
  uint32_t* k_in = (uint32_t*)p; p += nb;
  uint32_t* k_out = (uint32_t*)p; p += nb;
  uint32_t* i_in = (uint32_t*)p; p += nb;
  uint32_t* i_out = (uint32_t*)p; p += nb;
  int* bad = (int*)p; p += up(sizeof(int));
  void* tmp = p; p += up((size_t)n * 8);
  void* cub_tmp = p;
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  int rc = keys_any(pbytes, xs, ys, zs, n, origin, spacing, counts, k_in, nullptr, i_in, bad, s);
  int hbad = 0;
  if (!rc) rc = check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  if (!rc) rc = check(cudaStreamSynchronize(s), "sync");
  if (!rc && !hbad) {
    rc = check(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k_in, k_out, i_in, i_out, n,
                                               0, end_bit, s),
               "radix sort");
    void* parr[7] = {xs, ys, zs, us, vs, ws, qs};
    for (int a = 0; a < 7 && !rc; ++a) {
      if (!parr[a]) continue;
      rc = pbytes == 8 ? permute_one<double>(parr[a], i_out, tmp, n, s)
                       : permute_one<float>(parr[a], i_out, tmp, n, s);
    }
    if (!rc && ids) rc = permute_one<long long>(ids, i_out, tmp, n, s);
    if (!rc) rc = check(cudaStreamSynchronize(s), "sync");
  }
  if (rc) return rc;
  return hbad ? 3 : 0;
}

// Sorted copy of src into dst (eight arrays each; q / ids optional), one
// host synchronisation at the end.  On BP_ERR_DOMAIN dst is unspecified and
// src untouched.
int sort_by_cell_into(int pbytes, void* const* src, int64_t* src_ids, void* const* dst,
                      int64_t* dst_ids, int64_t n, const double* origin, const double* spacing,
                      const int64_t* counts, cudaStream_t s) {
  if (n <= 0) return 0;
  if (n > 0xffffffffLL) {
    set_error("sort_by_cell: %lld particles exceed the 32-bit index space", (long long)n);
    return -1;
  }
  const int64_t ncell = counts[0] * counts[1] * counts[2];
  int end_bit = 1;
  while (end_bit < 32 && (1LL << end_bit) < ncell) ++end_bit;
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, end_bit, s);
  auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t nb = up((size_t)n * sizeof(uint32_t));
  const size_t need = 4 * nb + up(sizeof(int)) + up((size_t)n * 8) + up(cub_bytes);
  int lrc = 0;
  WsLease lease(need, s, &lrc);
  if (lrc) return lrc;
  char* p = static_cast<char*>(lease.base());
  uint32_t* k_in = (uint32_t*)p; p += nb;
  uint32_t* k_out = (uint32_t*)p; p += nb;
  uint32_t* i_in = (uint32_t*)p; p += nb;
  uint32_t* i_out = (uint32_t*)p; p += nb;
  int* bad = (int*)p; p += up(sizeof(int));
  p += up((size_t)n * 8);
  void* cub_tmp = p;
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  int rc = 0;
  // the vector kernels need 16-byte-aligned arrays (a shard view such as
  // x[start:] may not be); otherwise the scalar kernels run
  auto a16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool vkeys = pbytes == 4 && a16(src[0]) && a16(src[1]) && a16(src[2]);
  bool vgather = !dst_ids || a16(dst_ids);
  for (int a = 0; a < 7; ++a)
    if (dst[a] && !a16(dst[a])) vgather = false;
  const int64_t n4 = vkeys ? n / 4 * 4 : 0;
  if (n4) {
    cell_key4_kernel<<<blocks_for(n4 / 4), 256, 0, s>>>(
        (const float*)src[0], (const float*)src[1], (const float*)src[2], n4, origin[0],
        origin[1], origin[2], spacing[0], spacing[1], spacing[2], counts[0], counts[1],
        counts[2], k_in, i_in, bad);
    note_launch();
    rc = check(cudaGetLastError(), "cell_key4_kernel");
  }
  if (!rc && n4 < n) {
    // the tail (and f64 particles): one particle per thread, indices offset
    rc = keys_any(pbytes, (const char*)src[0] + n4 * pbytes, (const char*)src[1] + n4 * pbytes,
                  (const char*)src[2] + n4 * pbytes, n - n4, origin, spacing, counts,
                  k_in + n4, nullptr, i_in + n4, bad, s, (uint32_t)n4);
  }
  if (!rc)
    rc = check(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k_in, k_out, i_in, i_out, n,
                                               0, end_bit, s),
               "radix sort");
  const int groups = gather_groups_env();
  if (!rc && !vgather) {
    for (int a = 0; a < 7 && !rc; ++a) {
      if (!src[a]) continue;
      if (pbytes == 8)
        gather_perm<double><<<blocks_for(n), 256, 0, s>>>((const double*)src[a], i_out,
                                                          (double*)dst[a], n);
      else
        gather_perm<float><<<blocks_for(n), 256, 0, s>>>((const float*)src[a], i_out,
                                                         (float*)dst[a], n);
      note_launch();
      rc = check(cudaGetLastError(), "gather_perm");
    }
    if (!rc && src_ids) {
      gather_perm<long long><<<blocks_for(n), 256, 0, s>>>((const long long*)src_ids, i_out,
                                                           (long long*)dst_ids, n);
      note_launch();
      rc = check(cudaGetLastError(), "gather_perm");
    }
  } else if (!rc && groups > 1) {
    rc = pbytes == 8 ? gather_grouped<double>(src, src_ids, dst, dst_ids, i_out, n, groups, s)
                     : gather_grouped<float>(src, src_ids, dst, dst_ids, i_out, n, groups, s);
  } else if (!rc) {
    if (pbytes == 8)
      gather_perm8<double><<<blocks_for(n), 256, 0, s>>>(
          (const double*)src[0], (const double*)src[1], (const double*)src[2],
          (const double*)src[3], (const double*)src[4], (const double*)src[5],
          (const double*)src[6], (const long long*)src_ids, i_out, (double*)dst[0],
          (double*)dst[1], (double*)dst[2], (double*)dst[3], (double*)dst[4], (double*)dst[5],
          (double*)dst[6], (long long*)dst_ids, n);
    else
      gather_perm8<float><<<blocks_for(n), 256, 0, s>>>(
          (const float*)src[0], (const float*)src[1], (const float*)src[2],
          (const float*)src[3], (const float*)src[4], (const float*)src[5],
          (const float*)src[6], (const long long*)src_ids, i_out, (float*)dst[0],
          (float*)dst[1], (float*)dst[2], (float*)dst[3], (float*)dst[4], (float*)dst[5],
          (float*)dst[6], (long long*)dst_ids, n);
    note_launch();
    rc = check(cudaGetLastError(), "gather_perm8");
  }
  int hbad = 0;
  if (!rc) rc = check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  if (!rc) rc = check(cudaStreamSynchronize(s), "sync");
  if (rc) return rc;
  return hbad ? 3 : 0;
}

int fold_periodic_i64(int64_t* acc, int64_t rows, const int64_t* geo_i, cudaStream_t s) {
  const int NX = (int)geo_i[0] + 1, NY = (int)geo_i[1] + 1, NZ = (int)geo_i[2] + 1;
  for (int axis = 0; axis < 3; ++axis) {
    if (geo_i[3 + axis] != 0) continue;  // reflecting
    const int n1 = axis == 0 ? NY : NX;
    const int n2 = axis == 2 ? NY : NZ;
    fold_axis<<<blocks_for(rows * n1 * n2), 256, 0, s>>>((long long*)acc, rows, NX, NY, NZ, axis);
    note_launch();
    int rc = check(cudaGetLastError(), "fold_axis");
    if (rc) return rc;
  }
  return 0;
}

}  // namespace bp
