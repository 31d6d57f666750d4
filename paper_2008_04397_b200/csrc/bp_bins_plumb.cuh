// Cell-binned layout: the types and the record-moving kernels shared by the
// f32 path (bp_bins.cu) and the f64 path (bp_bins64.cu), templated on the
// particle scalar S.  A slot is one particle record of two 4-vectors of S,
// x y z u | v w q 0 (32 bytes for f32, 64 for f64), plus an int64 id; bin c
// owns slots [start[c], start[c + 1]), the first count[c] live.
//
// Kernels here: leaver migration, cell keys / capacities / stable scatter of
// the build, export to flat arrays, and the re-slack copy.  The push and the
// deposit, which differ per precision, live in the two translation units.
#pragma once
#include <cstdint>

#include "bp_common.cuh"

namespace bp {
namespace bins {

template <typename S>
struct V4;
template <>
struct V4<float> {
  typedef float4 type;
};
template <>
struct V4<double> {
  typedef double4 type;
};

template <typename S>
__device__ __forceinline__ typename V4<S>::type mk4(S a, S b, S c, S d) {
  typedef typename V4<S>::type V;
  V v;
  v.x = a; v.y = b; v.z = c; v.w = d;
  return v;
}

// a leaver in transit: the record, its id; b.w carries the destination cell
// (int bits for f32, int64 bits for f64; < 0: no particle).  48 / 80 bytes.
template <typename S>
struct __align__(16) LeaverT {
  typename V4<S>::type a;  // x y z u
  typename V4<S>::type b;  // v w q, destination cell
  long long id;
  long long pad;
};

__device__ __forceinline__ int dest_of(float w) { return __float_as_int(w); }
__device__ __forceinline__ int dest_of(double w) { return (int)__double_as_longlong(w); }
template <typename S>
__device__ __forceinline__ S dest_bits(int c);
template <>
__device__ __forceinline__ float dest_bits<float>(int c) { return __int_as_float(c); }
template <>
__device__ __forceinline__ double dest_bits<double>(int c) {
  return __longlong_as_double((long long)c);
}

enum {
  ST_LEAVERS = 0,    // leaver slots claimed this cycle
  ST_OVERFLOW = 1,   // leavers that found their bin full
  ST_MISPLACED = 2,  // particles left in a bin that is not their cell
  ST_LOST = 3,       // overflow / late list full: particles dropped (fatal)
  ST_WORK_MOVE = 4,  // work counters
  ST_WORK_DEP = 5,
  ST_LATE = 6,       // misplaced particles the deposit listed for deposit_list
  ST_N = 8
};

template <typename S>
struct BinsT {
  typedef typename V4<S>::type V;
  V* rec;  // 2 per slot: x y z u | v w q 0
  long long* id;
  const long long* start;  // [ncell + 1]
  int* count;              // [ncell]
  int ncell;
  int move_claim;  // bins per mover claim
  int dep_rounds;  // deposit rounds per claim
  LeaverT<S>* lv;
  long long lv_cap;
  LeaverT<S>* ov;
  long long ov_cap;
  LeaverT<S>* late;  // the deposit's misplaced particles (deposited by deposit_list)
  long long late_cap;
  unsigned long long* stat;  // [ST_N]
};

// one full record with 256-bit stores (sm_100 st.global .v8.f32 / .v4.f64)
__device__ __forceinline__ void st_rec(float4* p, const float4& a, const float4& b) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.x),
               "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}
__device__ __forceinline__ void st_rec(double4* p, const double4& a, const double4& b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(a.z),
               "d"(a.w)
               : "memory");
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 1), "d"(b.x), "d"(b.y),
               "d"(b.z), "d"(b.w)
               : "memory");
}

// one record copied with streaming (evict-first) accesses
__device__ __forceinline__ void copy_rec_stream(float4* d, const float4* s) {
  __stcs(d, __ldcs(s));
  __stcs(d + 1, __ldcs(s + 1));
}
__device__ __forceinline__ void copy_rec_stream(double4* d, const double4* s) {
  const double2* s2 = reinterpret_cast<const double2*>(s);
  double2* d2 = reinterpret_cast<double2*>(d);
#pragma unroll
  for (int k = 0; k < 4; ++k) __stcs(d2 + k, __ldcs(s2 + k));
}

// the cell geometry of the bin keys: the fast arithmetic's
// gx = x * (1/dx) - ox/dx, cell = min(trunc(gx), n - 1), x fastest
template <typename S>
struct KeyGeo {
  S idx[3], ogs[3];
  int nx, ny, nz;
};

// ---------------------------------------------------------------------------
// Migration: every listed leaver claims a slot at the end of its new bin.
// A warp's 32 leavers come from one or two source bins, so they go to a few
// neighbouring cells: lanes with the same destination are grouped
// (__match_any_sync) and claim their slots with one atomic per group.
template <typename S>
__global__ void __launch_bounds__(256) migrate_bins(const __grid_constant__ BinsT<S> b) {
  const long long nl = min((long long)b.stat[ST_LEAVERS], b.lv_cap);
  const unsigned lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < nl;
       i0 += stride) {
    const long long i = i0 + lane;
    LeaverT<S> L{};
    int dest = -1;
    if (i < nl) {
      L = b.lv[i];
      dest = dest_of(L.b.w);
    }
    const bool ok = dest >= 0 && dest < b.ncell;
    const unsigned grp = __match_any_sync(0xffffffffu, ok ? dest : -1);
    const int leader = __ffs(grp) - 1;
    int pos = 0;
    if (ok && (int)lane == leader) pos = atomicAdd(&b.count[dest], __popc(grp));
    pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(grp & lt);
    if (!ok) continue;
    const long long s = b.start[dest];
    if (pos < b.start[dest + 1] - s) {
      const long long d = s + pos;
      // whole 32-byte sectors (no partial-sector read-modify-write)
      st_rec(b.rec + 2 * d, L.a, mk4<S>(L.b.x, L.b.y, L.b.z, S(0)));
      b.id[d] = L.id;
    } else {
      const unsigned long long o = atomicAdd(&b.stat[ST_OVERFLOW], 1ULL);
      if ((long long)o < b.ov_cap) b.ov[o] = L;
      else atomicAdd(&b.stat[ST_LOST], 1ULL);
    }
  }
}

// ---------------------------------------------------------------------------
// Build: cell keys, histogram, capacities, stable scatter.
template <typename S>
__global__ void bin_keys(const KeyGeo<S> g, const S* __restrict__ x, const S* __restrict__ y,
                         const S* __restrict__ z, long long n, unsigned* keys, unsigned* idx,
                         int* hist, int* bad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const S gx = fma(x[p], g.idx[0], -g.ogs[0]);
    const S gy = fma(y[p], g.idx[1], -g.ogs[1]);
    const S gz = fma(z[p], g.idx[2], -g.ogs[2]);
    int c = 0;
    if (!(gx > S(-1) && gy > S(-1) && gz > S(-1))) {
      *bad = 1;
    } else {
      const int i = min((int)gx, g.nx - 1), j = min((int)gy, g.ny - 1),
                k = min((int)gz, g.nz - 1);
      c = i + g.nx * j + g.nx * g.ny * k;
    }
    if (keys) keys[p] = (unsigned)c;
    if (idx) idx[p] = (unsigned)p;
    if (hist) atomicAdd(hist + c, 1);
  }
}

static __global__ void bin_caps(const int* __restrict__ cnt, int ncell, float frac, int smin,
                                long long* cap) {
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= ncell; c += stride) {
    if (c == ncell) {
      cap[c] = 0;
      continue;
    }
    const int n = cnt[c];
    // multiples of 8 slots: every bin starts on a 32-byte sector
    cap[c] = ((long long)n + max(smin, (int)ceilf(frac * (float)n)) + 7) & ~7LL;
  }
}

// sorted position r -> slot start[key] + (r - first[key]); first = exclusive
// scan of the counts
template <typename S>
__global__ void bin_scatter(const unsigned* __restrict__ skeys,
                            const unsigned* __restrict__ sidx, long long n,
                            const long long* __restrict__ start,
                            const long long* __restrict__ first, const S* const* src,
                            const long long* __restrict__ sid,
                            typename V4<S>::type* __restrict__ drec, long long* __restrict__ did) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const unsigned k = skeys[r], j = sidx[r];
    const long long d = start[k] + (r - first[k]);
    drec[2 * d] = mk4<S>(src[0][j], src[1][j], src[2][j], src[3][j]);
    drec[2 * d + 1] = mk4<S>(src[4][j], src[5][j], src[6][j], S(0));
    did[d] = sid[j];
  }
}

// export: bin c's live particles to flat[off[c] ...]
template <typename S>
__global__ void bin_export(const __grid_constant__ BinsT<S> b, const long long* __restrict__ off,
                           S* const* dst, long long* __restrict__ did) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long c = gw; c < b.ncell; c += nw) {
    const long long s0 = b.start[c];
    const int n = (int)min((long long)b.count[c], b.start[c + 1] - s0);
    const long long o = off[c];
    for (int r = lane; r < n; r += 32) {
      const auto x = b.rec[2 * (s0 + r)], y = b.rec[2 * (s0 + r) + 1];
      dst[0][o + r] = x.x; dst[1][o + r] = x.y; dst[2][o + r] = x.z; dst[3][o + r] = x.w;
      dst[4][o + r] = y.x; dst[5][o + r] = y.y; dst[6][o + r] = y.z;
      did[o + r] = b.id[s0 + r];
    }
  }
}

// the overflow list appended after the bins' particles
template <typename S>
__global__ void list_export(const __grid_constant__ BinsT<S> b, long long o0, S* const* dst,
                            long long* __restrict__ did) {
  const long long n = min((long long)b.stat[ST_OVERFLOW], b.ov_cap);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const LeaverT<S> L = b.ov[i];
    const long long d = o0 + i;
    dst[0][d] = L.a.x; dst[1][d] = L.a.y; dst[2][d] = L.a.z; dst[3][d] = L.a.w;
    dst[4][d] = L.b.x; dst[5][d] = L.b.y; dst[6][d] = L.b.z;
    did[d] = L.id;
  }
}

static __global__ void clamp_counts(int* cnt, const long long* start, int ncell) {
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += stride) {
    const long long cap = start[c + 1] - start[c];
    if (cnt[c] > cap) cnt[c] = (int)cap;
  }
}

// ---------------------------------------------------------------------------
// Re-slack (the cheap rebuild after an overflow): new capacities from the
// live counts plus the overflow list's arrivals, then every bin is copied to
// its new place and the overflow list appended (no sort: the bins are
// already in cell order).
template <typename S>
__global__ void reslack_counts(const __grid_constant__ BinsT<S> b, int* __restrict__ ncount) {
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < b.ncell; c += stride)
    ncount[c] = (int)min((long long)b.count[c], b.start[c + 1] - b.start[c]);
}
template <typename S>
__global__ void reslack_hist(const __grid_constant__ BinsT<S> b, int* __restrict__ ncount) {
  const long long no = min((long long)b.stat[ST_OVERFLOW], b.ov_cap);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < no; i += stride) {
    const int dest = dest_of(b.ov[i].b.w);
    if (dest >= 0 && dest < b.ncell) atomicAdd(ncount + dest, 1);
  }
}
// warp per bin: live particles to the new layout; ncount = live count
template <typename S>
__global__ void reslack_copy(const __grid_constant__ BinsT<S> b,
                             const long long* __restrict__ nstart, int* __restrict__ ncount,
                             typename V4<S>::type* __restrict__ drec,
                             long long* __restrict__ did) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long c = gw; c < b.ncell; c += nw) {
    const long long s0 = b.start[c];
    const int n = (int)min((long long)b.count[c], b.start[c + 1] - s0);
    const long long d0 = nstart[c];
    for (int r = lane; r < n; r += 32) {
      copy_rec_stream(drec + 2 * (d0 + r), b.rec + 2 * (s0 + r));
      __stcs(did + d0 + r, __ldcs(b.id + s0 + r));
    }
    if (lane == 0) ncount[c] = n;
  }
}
template <typename S>
__global__ void reslack_place(const __grid_constant__ BinsT<S> b,
                              const long long* __restrict__ nstart, int* __restrict__ ncount,
                              typename V4<S>::type* __restrict__ drec,
                              long long* __restrict__ did) {
  const long long no = min((long long)b.stat[ST_OVERFLOW], b.ov_cap);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < no; i += stride) {
    const LeaverT<S> L = b.ov[i];
    const int dest = dest_of(L.b.w);
    if (dest < 0 || dest >= b.ncell) continue;
    const long long d = nstart[dest] + atomicAdd(ncount + dest, 1);
    drec[2 * d] = L.a;
    drec[2 * d + 1] = mk4<S>(L.b.x, L.b.y, L.b.z, S(0));
    did[d] = L.id;
  }
}

}  // namespace bins
}  // namespace bp
