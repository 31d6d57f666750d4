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
#include <mutex>

#include "bp_launch.h"

namespace bp {

namespace {

template <typename P>
__global__ void cell_key_kernel(const P* __restrict__ x, const P* __restrict__ y,
                                const P* __restrict__ z, int64_t n, double ox, double oy,
                                double oz, double dx, double dy, double dz, int64_t nx,
                                int64_t ny, int64_t nz, uint32_t* keys32, int64_t* keys64,
                                uint32_t* idx, int* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    int64_t i = (int64_t)(((double)x[p] - ox) / dx);
    int64_t j = (int64_t)(((double)y[p] - oy) / dy);
    int64_t k = (int64_t)(((double)z[p] - oz) / dz);
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
    if (idx) idx[p] = (uint32_t)p;
  }
}

template <typename T>
__global__ void gather_perm(const T* __restrict__ src, const uint32_t* __restrict__ order,
                            T* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
    dst[r] = src[order[r]];
}

// all eight particle arrays gathered through one read of the order: the
// sorted copy lands in separate destination arrays (no copy back)
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
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const uint32_t j = __ldcs(order + r);
    ox[r] = x[j]; oy[r] = y[j]; oz[r] = z[j];
    ou[r] = u[j]; ov[r] = v[j]; ow[r] = w[j];
    if (q) oq[r] = q[j];
    if (id) oid[r] = id[j];
  }
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
                int* bad, cudaStream_t s) {
  cell_key_kernel<P><<<blocks_for(n), 256, 0, s>>>((const P*)xs, (const P*)ys, (const P*)zs, n,
                                                   o[0], o[1], o[2], d[0], d[1], d[2], c[0],
                                                   c[1], c[2], k32, k64, idx, bad);
  note_launch();
  return check(cudaGetLastError(), "cell_key_kernel");
}

int keys_any(int pbytes, const void* xs, const void* ys, const void* zs, int64_t n,
             const double* o, const double* d, const int64_t* c, uint32_t* k32, int64_t* k64,
             uint32_t* idx, int* bad, cudaStream_t s) {
  if (pbytes == 8) return keys_launch<double>(xs, ys, zs, n, o, d, c, k32, k64, idx, bad, s);
  if (pbytes == 4) return keys_launch<float>(xs, ys, zs, n, o, d, c, k32, k64, idx, bad, s);
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

// Grow-only sort workspace per device (keys, indices, permutation scratch,
// CUB temp storage), so periodic sorts do not re-allocate ~40 B/particle.
struct SortWs {
  void* base = nullptr;
  size_t bytes = 0;
};
static std::mutex g_sort_mu;
static SortWs g_sort_ws[64];

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
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_sort_mu);
  SortWs& W = g_sort_ws[dev & 63];
  if (W.bytes < need) {
    if (W.base) {
      cudaStreamSynchronize(s);
      cudaFree(W.base);
      W.base = nullptr;
      W.bytes = 0;
    }
    int rc = check(cudaMalloc(&W.base, need), "sort workspace");
    if (rc) return rc;
    W.bytes = need;
  }
  char* p = static_cast<char*>(W.base);
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
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_sort_mu);
  SortWs& W = g_sort_ws[dev & 63];
  if (W.bytes < need) {
    if (W.base) {
      cudaStreamSynchronize(s);
      cudaFree(W.base);
      W.base = nullptr;
      W.bytes = 0;
    }
    int rc = check(cudaMalloc(&W.base, need), "sort workspace");
    if (rc) return rc;
    W.bytes = need;
  }
  char* p = static_cast<char*>(W.base);
  uint32_t* k_in = (uint32_t*)p; p += nb;
  uint32_t* k_out = (uint32_t*)p; p += nb;
  uint32_t* i_in = (uint32_t*)p; p += nb;
  uint32_t* i_out = (uint32_t*)p; p += nb;
  int* bad = (int*)p; p += up(sizeof(int));
  p += up((size_t)n * 8);
  void* cub_tmp = p;
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  int rc = keys_any(pbytes, src[0], src[1], src[2], n, origin, spacing, counts, k_in, nullptr,
                    i_in, bad, s);
  if (!rc)
    rc = check(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k_in, k_out, i_in, i_out, n,
                                               0, end_bit, s),
               "radix sort");
  if (!rc) {
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
