// The fast-arithmetic fused span as two kernels — the implicit mover and the
// 10-moment interpolation (deposit) — for f32 particles ("single" / "mixed"),
// sm_100a.  The code is written for T = float or double; the f64
// instantiation is not dispatched (see split_fused).  Same algorithm as the
// reference fused_span (pkg/src/batchpic/kernels.py:458-735); DESIGN.md §4
// has the instruction budget and the measurements behind every choice here.
//
// Cell records (pack_cells): for each cell, in the particles' sort order
// (x fastest), the trilinear form of the 6 components
//     f(fx,fy,fz) = [c0 + c1 fx + (c2 + c4 fx) fy] + fz [c3 + c5 fx + (c6 + c7 fx) fy]
// (the reference's 8-weight sum, kernels.py:557-591, regrouped), components
// paired (Ex Ey | Bx By | Ez Bz): 12 quads of T per cell.  For f32 the pairs
// are evaluated with the packed FP32 instruction FFMA2 (two f32 lanes per
// instruction, sm_100): 21 FFMA2 per gather.  The f32 mover keeps the record
// in registers while the midpoint stays in its cell.
//
// Mover: one particle per thread, persistent grid, next particle prefetched,
// boundary kinds as template parameters, boundary folds skipped for warps
// that provably stay inside (interior()).  Failed particles (runaway,
// midpoint) are not stored and get a bit in the `skip` bitmask.
//
// Deposit: per-warp transposed fold (lane = corner x moment group, tiles of
// 32 staged particles) into a per-warp node patch in shared memory, flushed
// onto the int64 lattice (x invvol x 2^43, rint) with REDG.ADD.64.  A tile's
// partial sums are formed in T and rounded once onto the lattice — within
// the north star's 1e-4 for f32 — and every chunk is flushed on its own, so
// the result is deterministic for a given launch.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "bp_common.cuh"
#include "bp_f32_common.cuh"
#include "bp_launch.h"

namespace bp {
namespace sk {

// staged row stride (elements): rows read by one warp LDS.128 land in
// distinct banks (36 floats / 34 doubles = 4 mod 32 words)
template <typename T>
__host__ __device__ constexpr int row_len() {
  return sizeof(T) == 4 ? 36 : 34;
}
// staging rows: 8 bases (corner c), then 10 moments (row 8 + m; m = 0 is 1)
template <typename T>
__host__ __device__ constexpr int stage_len() {
  return 18 * row_len<T>();
}

// ---------------------------------------------------------------------------
// Mover: one particle per thread, coalesced SoA streams, no shared memory, so
// the SM holds enough warps to hide the latency of the dependent gather +
// rotation steps.  Particles that fail (kernels.py:618-621, 672-676) are not
// stored; their bit in `skip` keeps them out of the deposit.
template <typename T, bool RX, bool RY, bool RZ, bool REUSE, int MINB, int WCH>
__global__ void __launch_bounds__(256, MINB) mover_kernel(const __grid_constant__ Params<T> a) {
  // persistent grid; each warp walks chunks of WCH consecutive 32-particle
  // tiles (chunks gw, gw + nw, ...), so the cell records its first tile loads
  // are L1-hot for the following tiles of the same cells; the next tile's
  // loads are in flight while this one is pushed
  const unsigned lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const long long nw = (long long)gridDim.x * 8;
  constexpr long long CH = 32LL * WCH;
  long long c = gw;
  int ti = 0;
  T n1[6] = {0, 0, 0, 0, 0, 0};
  auto fetch = [&](long long rr) {
    if (rr < a.count) {
      const long long p = a.start + rr;
      n1[0] = __ldcs(a.x + p); n1[1] = __ldcs(a.y + p); n1[2] = __ldcs(a.z + p);
      n1[3] = __ldcs(a.u + p); n1[4] = __ldcs(a.v + p); n1[5] = __ldcs(a.w + p);
    }
  };
  fetch(c * CH + lane);
  // |qdt2m| max|E| (+1e-5 relative slack for the coefficient rounding)
  const T qe = fabs(a.qdt2m) * (T)__ldg(a.emax) * T(1.00001);
  for (long long base = c * CH; base < a.count; base = c * CH + 32LL * ti) {
    const long long r = base + lane;
    T xp = n1[0], yp = n1[1], zp = n1[2], un = n1[3], vn = n1[4], wn = n1[5];
    if (++ti == WCH) {
      ti = 0;
      c += nw;
    }
    fetch(c * CH + 32LL * ti + lane);
    int st = ST_OK;
    // warp-uniform: the whole warp takes the boundary-free push when it can
    const bool all_in =
        __all_sync(0xffffffffu, r >= a.count || interior(a, qe, xp, yp, zp, un, vn, wn));
    if (r < a.count) {
      const long long p = a.start + r;
      st = push<T, RX, RY, RZ, REUSE>(a, xp, yp, zp, un, vn, wn, all_in);
      if (st == ST_OK) {
        __stcs(a.x + p, xp); __stcs(a.y + p, yp); __stcs(a.z + p, zp);
        __stcs(a.u + p, un); __stcs(a.v + p, vn); __stcs(a.w + p, wn);
      }
    }
    const unsigned bad = __ballot_sync(0xffffffffu, st != ST_OK);
    if (bad) {
      if (lane == 0) atomicOr(a.skip + (r >> 5), bad);
      if (st != ST_OK) atomicMax(a.status, st);
    }
  }
}

// ---------------------------------------------------------------------------
// Deposition.  Lane L of a warp owns corner c = L & 7 of moments g, g + 4
// (g = L >> 3) and, over half a tile, moment 8 + (g & 1).  Every tile's
// staged particles are folded per cell (q * w_c * m) and added into a
// per-warp node patch in shared memory: sums over the nodes
// [pi0, pi0 + PX) x [pj0, pj0 + 4) x [pk0, pk0 + 4) for the 10 moments — the
// neighbourhood of the cells a chunk of sorted particles covers, strays
// included.  Each lane only ever touches the patch values of its own
// (corner, moment) pairs, so no atomics.  The patch is converted to the
// lattice and flushed when the chunk ends or its cells leave the patch.
template <int PX>
struct Patch {
  static constexpr int kNodes = PX * 16;      // node (px, py, pz) at (px * 4 + py) * 4 + pz
  static constexpr int kStride = kNodes + 2;  // per moment; +2 spreads lane groups over banks
  static constexpr int kLen = 10 * kStride;
};

template <typename T>
__device__ __forceinline__ long long lattice(const Params<T>& a, T v, int node) {
  const double iv = a.iv_d ? __ldg(a.iv_d + node) : (double)__ldg(a.iv_f + node);
  return __double2ll_rn((double)v * iv * a.scale);
}

// The patch's nodes are split over the lanes (node lane + 32 i); each lane
// holds invvol * 2^43 of its nodes in registers, loaded when the patch is
// anchored so the loads complete long before the flush uses them.
template <int PX>
struct PatchNodes {
  static constexpr int kPer = PX * 16 / 32;
  double ivs[kPer];
  int gnode[kPer];  // global node index, -1 outside the grid
};

template <int PX, typename T>
__device__ __forceinline__ void patch_anchor(const Params<T>& a, PatchNodes<PX>& pn, int pi0,
                                             int pj0, int pk0, unsigned lane) {
#pragma unroll
  for (int i = 0; i < PatchNodes<PX>::kPer; ++i) {
    const int n = (int)lane + 32 * i;
    const int gi = pi0 + (n >> 4), gj = pj0 + ((n >> 2) & 3), gk = pk0 + (n & 3);
    const bool in = gi >= 0 && gi <= a.nx && gj >= 0 && gj <= a.ny && gk >= 0 && gk <= a.nz;
    const int g = in ? (gi * a.NY + gj) * a.NZ + gk : 0;
    pn.gnode[i] = in ? g : -1;
    const double iv = a.iv_d ? __ldg(a.iv_d + g) : (double)__ldg(a.iv_f + g);
    pn.ivs[i] = iv * a.scale;
  }
}

// Flush and clear the patch: lane handles its nodes for all 10 moments; a
// nonzero sum goes onto the lattice (x invvol x 2^43, rint) with one
// REDG.ADD.64 (consecutive lanes hold z-consecutive nodes).
template <int PX, typename T>
__device__ __forceinline__ void patch_flush(const Params<T>& a, T* patch,
                                            const PatchNodes<PX>& pn, unsigned lane) {
  typedef Patch<PX> Pt;
#pragma unroll
  for (int i = 0; i < PatchNodes<PX>::kPer; ++i) {
    const int n = (int)lane + 32 * i;
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      T* pv = patch + m * Pt::kStride + n;
      const T v = *pv;
      if (v != T(0)) {
        *pv = T(0);
        if (pn.gnode[i] >= 0)
          atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + (size_t)m * a.NN + pn.gnode[i]),
                    (unsigned long long)__double2ll_rn((double)v * pn.ivs[i]));
      }
    }
  }
  __syncwarp();  // the cleared patch is written by the other lanes' folds next
}

// main fold of all 32 staged particles for this lane's three values: rows of
// bases br, moments m0r / m1r over the whole tile, and the third moment m3r
// over this lane's half tile (b3 = bases of that half)
__device__ __forceinline__ void main_fold(const float* br, const float* m0r, const float* m1r,
                                          const float* b3, const float* m3r, float& s0,
                                          float& s1, float& s2) {
  F2 S0 = f2(0.f, 0.f), S1 = f2(0.f, 0.f), S2 = f2(0.f, 0.f);
#pragma unroll
  for (int kk = 0; kk < 32; kk += 4) {
    const float4 b = *reinterpret_cast<const float4*>(br + kk);
    const float4 x0 = *reinterpret_cast<const float4*>(m0r + kk);
    const float4 x1 = *reinterpret_cast<const float4*>(m1r + kk);
    S0 = fma2(f2(b.x, b.y), f2(x0.x, x0.y), S0);
    S0 = fma2(f2(b.z, b.w), f2(x0.z, x0.w), S0);
    S1 = fma2(f2(b.x, b.y), f2(x1.x, x1.y), S1);
    S1 = fma2(f2(b.z, b.w), f2(x1.z, x1.w), S1);
  }
#pragma unroll
  for (int kk = 0; kk < 16; kk += 4) {
    const float4 b = *reinterpret_cast<const float4*>(b3 + kk);
    const float4 x2 = *reinterpret_cast<const float4*>(m3r + kk);
    S2 = fma2(f2(b.x, b.y), f2(x2.x, x2.y), S2);
    S2 = fma2(f2(b.z, b.w), f2(x2.z, x2.w), S2);
  }
  s0 = S0.x + S0.y;
  s1 = S1.x + S1.y;
  s2 = S2.x + S2.y;
}
__device__ __forceinline__ void main_fold(const double* br, const double* m0r,
                                          const double* m1r, const double* b3,
                                          const double* m3r, double& s0, double& s1,
                                          double& s2) {
  double a0 = 0, a1 = 0, c0 = 0, c1 = 0, e0 = 0, e1 = 0;
#pragma unroll
  for (int kk = 0; kk < 32; kk += 2) {
    const double2 b = *reinterpret_cast<const double2*>(br + kk);
    const double2 x0 = *reinterpret_cast<const double2*>(m0r + kk);
    const double2 x1 = *reinterpret_cast<const double2*>(m1r + kk);
    a0 = fma(b.x, x0.x, a0);
    a1 = fma(b.y, x0.y, a1);
    c0 = fma(b.x, x1.x, c0);
    c1 = fma(b.y, x1.y, c1);
  }
#pragma unroll
  for (int kk = 0; kk < 16; kk += 2) {
    const double2 b = *reinterpret_cast<const double2*>(b3 + kk);
    const double2 x2 = *reinterpret_cast<const double2*>(m3r + kk);
    e0 = fma(b.x, x2.x, e0);
    e1 = fma(b.y, x2.y, e1);
  }
  s0 = a0 + a1;
  s1 = c0 + c1;
  s2 = e0 + e1;
}

// Deposit (interpolation of the 10 moments) of the moved particles.  Each
// warp claims chunks of CHUNK particles; tiles of 32 are staged in shared
// memory and folded per cell.
template <typename T, int PX, int CHUNK, int MINB>
__global__ void __launch_bounds__(256, MINB) deposit_kernel(const __grid_constant__ Params<T> a) {
  typedef Patch<PX> Pt;
  constexpr int KR = row_len<T>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const smem_t = reinterpret_cast<T*>(smem_raw);
  const unsigned lane = lane_id();
  T* const st = smem_t + (threadIdx.x >> 5) * (stage_len<T>() + Pt::kLen);
  T* const st_bs = st;             // [8][KR] bases q * w_c
  T* const st_mv = st + 8 * KR;    // [10][KR], row m = moment m (row 0: constant 1)
  T* const patch = st + stage_len<T>();  // [10][kStride]
  const int lc = lane & 7, lg = lane >> 3;
  const int poff = (lc & 1) * 16 + ((lc >> 1) & 1) * 4 + ((lc >> 2) & 1);
  const bool third = lg < 2;
  const int m3 = 8 + (lg & 1), h3 = (lg >> 1) * 16;
  // this lane's three patch value columns (moments lg, lg + 4, 8 + lg)
  T* const pv0 = patch + lg * Pt::kStride + poff;
  T* const pv1 = patch + (lg + 4) * Pt::kStride + poff;
  T* const pv2 = patch + (third ? lg + 8 : 8) * Pt::kStride + poff;
  st_mv[lane] = T(1);
  for (int r = lane; r < Pt::kLen; r += 32) patch[r] = T(0);
  __syncwarp();
  long long nxt = 0;
  if (lane == 0) nxt = (long long)atomicAdd(a.work, (unsigned long long)CHUNK);
  nxt = __shfl_sync(0xffffffffu, nxt, 0);
  // prefetched particle of the next tile
  T px_ = 0, py_ = 0, pz_ = 0, pu_ = 0, pv_ = 0, pw_ = 0, pq_ = 0;
  unsigned sk_ = 0u;
  auto fetch = [&](long long r, long long end) {
    if (r < end) {
      const long long p = a.start + r;
      px_ = __ldcs(a.x + p); py_ = __ldcs(a.y + p); pz_ = __ldcs(a.z + p);
      pu_ = __ldcs(a.u + p); pv_ = __ldcs(a.v + p); pw_ = __ldcs(a.w + p);
      pq_ = __ldcs(a.q + p);
    }
    sk_ = __ldg(a.skip + (r >> 5));
  };
  if (nxt < a.count) fetch(nxt + lane, nxt + CHUNK < a.count ? nxt + CHUNK : a.count);
  const T* brow = st_bs + lc * KR;
  const T* m0row = st_mv + lg * KR;
  const T* m1row = st_mv + (lg + 4) * KR;
  const T* m2row = st_mv + (third ? lg + 8 : 8) * KR;
  while (nxt < a.count) {
    const long long w0 = nxt;
    const long long w1 = w0 + CHUNK < a.count ? w0 + CHUNK : a.count;
    if (lane == 0) nxt = (long long)atomicAdd(a.work, (unsigned long long)CHUNK);
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
    int pi0 = 0, pj0 = 0, pk0 = 0;  // patch origin (node coordinates)
    bool anchored = false;
    PatchNodes<PX> pn;
    for (long long t0 = w0; t0 < w1; t0 += 32) {
      const long long r = t0 + lane;
      const bool valid = r < w1 && !((sk_ >> lane) & 1u);
      const T xp = px_, yp = py_, zp = pz_, un = pu_, vn = pv_, wn = pw_, qp = pq_;
      if (t0 + 32 < w1) fetch(t0 + 32 + lane, w1);
      else if (nxt < a.count) fetch(nxt + lane, nxt + CHUNK < a.count ? nxt + CHUNK : a.count);
      // ---- stage this lane's particle: 8 bases q*w_c and the moments
      int ci = 0, cj = 0, ck = 0;
      {
        T fx = 0, fy = 0, fz = 0, qs = 0;
        if (valid) {
          cell_of(a, xp, yp, zp, fx, fy, fz, ci, cj, ck);
          qs = qp;
        }
        const T qax = qs * (T(1) - fx), qfx = qs * fx;
        const T ay = T(1) - fy, az = T(1) - fz;
        const T w00 = qax * ay, w10 = qfx * ay, w01 = qax * fy, w11 = qfx * fy;
        st_bs[0 * KR + lane] = w00 * az; st_bs[1 * KR + lane] = w10 * az;
        st_bs[2 * KR + lane] = w01 * az; st_bs[3 * KR + lane] = w11 * az;
        st_bs[4 * KR + lane] = w00 * fz; st_bs[5 * KR + lane] = w10 * fz;
        st_bs[6 * KR + lane] = w01 * fz; st_bs[7 * KR + lane] = w11 * fz;
        T* mv = st_mv + lane;
        mv[1 * KR] = un; mv[2 * KR] = vn; mv[3 * KR] = wn;
        mv[4 * KR] = un * un; mv[5 * KR] = un * vn; mv[6 * KR] = un * wn;
        mv[7 * KR] = vn * vn; mv[8 * KR] = vn * wn; mv[9 * KR] = wn * wn;
      }
      const unsigned V = __ballot_sync(0xffffffffu, valid);
      if (V == 0u) continue;
      // ---- patch placement
      if (!anchored) {
        anchored = true;
        const int src = __ffs(V) - 1;
        pi0 = __shfl_sync(0xffffffffu, ci, src) - 1;
        pj0 = __shfl_sync(0xffffffffu, cj, src) - 1;
        pk0 = __shfl_sync(0xffffffffu, ck, src) - 1;
        patch_anchor<PX>(a, pn, pi0, pj0, pk0, lane);
      }
      int dx = ci - pi0, dy = cj - pj0, dz = ck - pk0;
      bool fit = valid && (unsigned)dx <= (unsigned)(PX - 2) && (unsigned)dy <= 2u &&
                 (unsigned)dz <= 2u;
      unsigned F = __ballot_sync(0xffffffffu, fit);
      if (__popc(V & ~F) > __popc(F)) {
        // the run moved on: flush and re-anchor at its first particle outside
        patch_flush<PX>(a, patch, pn, lane);
        const int src = __ffs(V & ~F) - 1;
        pi0 = __shfl_sync(0xffffffffu, ci, src) - 1;
        pj0 = __shfl_sync(0xffffffffu, cj, src) - 1;
        pk0 = __shfl_sync(0xffffffffu, ck, src) - 1;
        patch_anchor<PX>(a, pn, pi0, pj0, pk0, lane);
        dx = ci - pi0; dy = cj - pj0; dz = ck - pk0;
        fit = valid && (unsigned)dx <= (unsigned)(PX - 2) && (unsigned)dy <= 2u &&
              (unsigned)dz <= 2u;
        F = __ballot_sync(0xffffffffu, fit);
      }
      const int pnode = (dx * 4 + dy) * 4 + dz;  // patch node of corner 000 (fitting lanes)
      // ---- main cell: the larger of the first / last fitting lane's cells
      const int ka = __shfl_sync(0xffffffffu, pnode, __ffs(F | 1u) - 1);
      const int kb = __shfl_sync(0xffffffffu, pnode, 31 - __clz(F | 1u));
      const unsigned MA = __ballot_sync(0xffffffffu, fit && pnode == ka);
      const unsigned MB = __ballot_sync(0xffffffffu, fit && pnode == kb);
      const bool useb = __popc(MB) > __popc(MA);
      const int kmain = useb ? kb : ka;
      const unsigned Mm = useb ? MB : MA;
      __syncwarp();
      // ---- other cells of the tile: per-cell fold of their few particles
      for (unsigned rest = F & ~Mm; rest;) {
        const int kg = __shfl_sync(0xffffffffu, pnode, __ffs(rest) - 1);
        const unsigned MG = __ballot_sync(0xffffffffu, fit && pnode == kg);
        rest &= ~MG;
        // a neighbouring lane may have written this node (its corner of the
        // previous group's cell): order the patch accesses of the warp
        __syncwarp();
        // the cell's patch values are read first (no alias with the staged
        // rows) so their latency hides behind the fold
        // (moment 8 + (g & 1) is owned by the lanes of groups 0 and 1)
        const T o0 = pv0[kg], o1 = pv1[kg], o2 = third ? pv2[kg] : T(0);
        // members software-pipelined: the next member's loads are issued
        // before this member's products
        unsigned m = MG;
        int kk = __ffs(m) - 1;
        m &= m - 1u;
        T b = brow[kk], x0 = m0row[kk], x1 = m1row[kk], x2 = m2row[kk];
        T t0s = 0, t1s = 0, t2s = 0;
        while (m) {
          const int kn = __ffs(m) - 1;
          m &= m - 1u;
          const T bn = brow[kn], y0 = m0row[kn], y1 = m1row[kn], y2 = m2row[kn];
          t0s = fma(b, x0, t0s);
          t1s = fma(b, x1, t1s);
          t2s = fma(b, x2, t2s);
          b = bn; x0 = y0; x1 = y1; x2 = y2;
        }
        t0s = fma(b, x0, t0s);
        t1s = fma(b, x1, t1s);
        t2s = fma(b, x2, t2s);
        pv0[kg] = o0 + t0s;
        pv1[kg] = o1 + t1s;
        if (third) pv2[kg] = o2 + t2s;
      }
      // ---- particles whose cells are outside the patch (rare): straight to the lattice
      for (unsigned out = V & ~F; out;) {
        const int src = __ffs(out) - 1;
        const int oi = __shfl_sync(0xffffffffu, ci, src);
        const int oj = __shfl_sync(0xffffffffu, cj, src);
        const int ok = __shfl_sync(0xffffffffu, ck, src);
        const unsigned M2 =
            __ballot_sync(0xffffffffu, valid && !fit && ci == oi && cj == oj && ck == ok);
        out &= ~M2;
        T t0s = 0, t1s = 0, t2s = 0;
        for (unsigned m = M2; m; m &= m - 1u) {
          const int kk = __ffs(m) - 1;
          const T b = brow[kk];
          t0s = fma(b, m0row[kk], t0s);
          t1s = fma(b, m1row[kk], t1s);
          t2s = fma(b, m2row[kk], t2s);
        }
        const int node = ((oi + (lc & 1)) * a.NY + (oj + ((lc >> 1) & 1))) * a.NZ + ok +
                         ((lc >> 2) & 1);
        long long* dst = a.acc + (size_t)lg * a.NN + node;
        atomicAdd(reinterpret_cast<unsigned long long*>(dst),
                  (unsigned long long)lattice(a, t0s, node));
        atomicAdd(reinterpret_cast<unsigned long long*>(dst + (size_t)4 * a.NN),
                  (unsigned long long)lattice(a, t1s, node));
        if (third)
          atomicAdd(reinterpret_cast<unsigned long long*>(dst + (size_t)8 * a.NN),
                    (unsigned long long)lattice(a, t2s, node));
      }
      if (V & ~Mm) {
        __syncwarp();  // every lane is done reading the staged rows
        if (((V & ~Mm) >> lane) & 1u) {
#pragma unroll
          for (int c = 0; c < 8; ++c) st_bs[c * KR + lane] = T(0);
        }
        __syncwarp();
      }
      // ---- main fold: all 32 staged particles (others have zero bases)
      if (Mm) {
        T s0, s1, s2;
        main_fold(brow, m0row, m1row, brow + h3, st_mv + m3 * KR + h3, s0, s1, s2);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 16);
        pv0[kmain] += s0;
        pv1[kmain] += s1;
        if (third) pv2[kmain] += s2;
      }
      __syncwarp();
    }
    if (anchored) patch_flush<PX>(a, patch, pn, lane);
    __syncwarp();
  }
}

// Per-cell coefficient records (computed in f64, rounded once to O), three
// component pairs (a, b) = (Ex, Ey), (Bx, By), (Ez, Bz), four quads each:
// (c0a c0b c1a c1b) (c2a c2b c4a c4b) (c3a c3b c5a c5b) (c6a c6b c7a c7b);
// after the records, max |E| over the nodes (float, rounded up).
// Tiles of 32 (x) x 8 (z) cells at one y: the 33 x 2 x 9 nodes of the six
// components are staged in shared memory with k-fastest (coalesced) reads,
// then warp w builds the records of z-row k0 + w, one cell per lane, and
// writes 32 consecutive records (x fastest, the particles' sort order).
constexpr int kPackTI = 32, kPackTK = 8, kPackRow = 19;  // 2 x 9 node values + 1 pad

template <typename F, typename O>
__global__ void __launch_bounds__(256) pack_cells(const F* __restrict__ E,
                                                  const F* __restrict__ B, int nx, int ny,
                                                  int nz, O* __restrict__ rec,
                                                  unsigned* __restrict__ emax_bits) {
  __shared__ F nodes[6][kPackTI + 1][kPackRow];
  __shared__ unsigned wmax[8];
  // the warp's 32 records, written out as contiguous 512-byte rows
  extern __shared__ __align__(16) unsigned char pack_out_raw[];
  O* const wout = reinterpret_cast<O*>(pack_out_raw) + (threadIdx.x >> 5) * (kPackTI * 48);
  const int NY = ny + 1, NZ = nz + 1, NN = (nx + 1) * NY * NZ;
  const int comp[6] = {0, 1, 3, 4, 2, 5};  // component of pair slot 2p + member
  const int tx = (nx + kPackTI - 1) / kPackTI;
  const int i0 = (blockIdx.x % tx) * kPackTI, k0 = (blockIdx.x / tx) * kPackTK;
  const int j = blockIdx.y;
  // stage: (h, i', j', k') with k' fastest; nodes past the grid are not read
  constexpr int kVals = 6 * (kPackTI + 1) * 18;
  for (int v = threadIdx.x; v < kVals; v += blockDim.x) {
    const int kk = v % 9, jj = (v / 9) & 1, ii = (v / 18) % (kPackTI + 1), h = v / (18 * (kPackTI + 1));
    const int gi = i0 + ii, gk = k0 + kk;
    F val = F(0);
    if (gi <= nx && gk <= nz) {
      const int m = comp[h];
      const F* f = m < 3 ? E + (size_t)m * NN : B + (size_t)(m - 3) * NN;
      val = f[((size_t)gi * NY + (j + jj)) * NZ + gk];
    }
    nodes[h][ii][jj * 9 + kk] = val;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = i0 + lane, k = k0 + w;
  double e2max = 0.0;
  if (i < nx && k < nz) {
    double co[6][8];
    double e2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int h = 0; h < 6; ++h) {
      const F* r0 = nodes[h][lane];
      const F* r1 = nodes[h][lane + 1];
      const double f000 = r0[w], f100 = r1[w], f010 = r0[9 + w], f110 = r1[9 + w];
      const double f001 = r0[w + 1], f101 = r1[w + 1], f011 = r0[10 + w], f111 = r1[10 + w];
      if (comp[h] < 3) {
        e2[0] += f000 * f000; e2[1] += f100 * f100; e2[2] += f010 * f010; e2[3] += f110 * f110;
        e2[4] += f001 * f001; e2[5] += f101 * f101; e2[6] += f011 * f011; e2[7] += f111 * f111;
      }
      co[h][0] = f000;
      co[h][1] = f100 - f000;
      co[h][2] = f010 - f000;
      co[h][3] = f001 - f000;
      co[h][4] = (f110 - f100) - (f010 - f000);
      co[h][5] = (f101 - f001) - (f100 - f000);
      co[h][6] = (f011 - f001) - (f010 - f000);
      co[h][7] = ((f111 - f011) - (f101 - f001)) - ((f110 - f010) - (f100 - f000));
    }
    O* o = wout + lane * 48;
    const int slot[4][2] = {{0, 1}, {2, 4}, {3, 5}, {6, 7}};
#pragma unroll
    for (int pr = 0; pr < 3; ++pr)
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        O* d = o + (4 * pr + qd) * 4;
        d[0] = (O)co[2 * pr][slot[qd][0]];
        d[1] = (O)co[2 * pr + 1][slot[qd][0]];
        d[2] = (O)co[2 * pr][slot[qd][1]];
        d[3] = (O)co[2 * pr + 1][slot[qd][1]];
      }
#pragma unroll
    for (int q = 0; q < 8; ++q) e2max = fmax(e2max, e2[q]);
  }
  __syncwarp();
  if (k < nz) {
    // this warp's cells i0 .. i0 + n - 1 of row (j, k): n * 48 contiguous values
    const int n = min(kPackTI, nx - i0);
    O* dst = rec + ((size_t)i0 + (size_t)nx * (j + (size_t)ny * k)) * 48;
    const float4* src4 = reinterpret_cast<const float4*>(wout);
    float4* dst4 = reinterpret_cast<float4*>(dst);
    const int n16 = n * 48 * (int)sizeof(O) / 16;
    for (int v = lane; v < n16; v += 32) __stcs(dst4 + v, src4[v]);
  }
  // non-negative floats order like their bit patterns; rounded up; one
  // atomic per block
  unsigned bits = __float_as_uint(__double2float_ru(sqrt(e2max)));
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, sh));
  if (lane == 0) wmax[w] = bits;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned m = 0;
    for (int q = 0; q < 8; ++q) m = max(m, wmax[q]);
    if (m) atomicMax(emax_bits, m);
  }
}

}  // namespace sk

namespace {

int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// persistent grid: every SM gets its occupancy's worth of blocks
template <typename K>
int grid_of(K k, size_t smem, long long per_block_work, long long count) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem);
  if (per_sm < 1) per_sm = 1;
  const long long need = (count + per_block_work - 1) / per_block_work;
  long long g = (long long)sms() * per_sm;
  if (need < g) g = need;
  return (int)(g < 1 ? 1 : g);
}

template <typename T, bool RX, bool RY, bool RZ, int WCH>
int launch_mover_w(const sk::Params<T>& a, cudaStream_t s) {
  constexpr bool kF = std::is_same<T, float>::value;
  auto k = sk::mover_kernel<T, RX, RY, RZ, kF, 2, WCH>;
  const int g = grid_of(k, 0, 256, a.count);
  const int th = timing_begin(TK_MOVER, s);
  k<<<g, 256, 0, s>>>(a);
  timing_end(th, s);
  note_launch();
  return launch_check("mover launch");
}

// f32: record reuse across the mover iterations (~100 registers, 16 warps /
// SM; measured best); f64: no reuse (the record is 96 registers)
template <typename T, bool RX, bool RY, bool RZ>
int launch_mover(const sk::Params<T>& a, cudaStream_t s) {
  static int wch = -1;
  if (wch < 0) {
    const char* e = getenv("BP_MOVER_WCH");
    wch = e ? atoi(e) : 4;
  }
  // tiles per warp chunk (measured: 1 -> 1.30 ms, 4 -> 1.27, 8 / 16 -> 1.27)
  if (wch == 1) return launch_mover_w<T, RX, RY, RZ, 1>(a, s);
  return launch_mover_w<T, RX, RY, RZ, 4>(a, s);
}

// f32: 8-node-wide patch, 512-particle chunks, 3 blocks (24 warps) / SM;
// f64: the shared memory per warp doubles, so 6-wide patches, 256-particle
// chunks and 2 blocks / SM
template <typename T, int PX, int CHUNK, int MINB>
int launch_deposit_cfg(const sk::Params<T>& a, cudaStream_t s) {
  auto k = sk::deposit_kernel<T, PX, CHUNK, MINB>;
  const size_t smem =
      (size_t)(256 / 32) * (sk::stage_len<T>() + sk::Patch<PX>::kLen) * sizeof(T);
  static bool attr[64] = {};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  const int g = grid_of(k, smem, (long long)CHUNK * 8, a.count);
  const int th = timing_begin(TK_DEPOSIT, s);
  k<<<g, 256, smem, s>>>(a);
  timing_end(th, s);
  note_launch();
  return launch_check("deposit launch");
}

// f32: 8-node-wide patch, 512-particle chunks, 3 blocks (24 warps) / SM;
// f64: the shared memory per warp doubles, so 6-wide patches, 256-particle
// chunks and 2 blocks / SM
template <typename T>
int launch_deposit(const sk::Params<T>& a, cudaStream_t s) {
  // (measured: 6-wide patches with 256-particle chunks at 24 or 32 warps / SM
  // are 3-4% slower)
  if constexpr (std::is_same<T, float>::value) {
    return launch_deposit_cfg<T, 8, 512, 3>(a, s);
  } else {
    return launch_deposit_cfg<T, 6, 256, 2>(a, s);
  }
}

// the mover for the span's boundary kinds (geo_i[3..5]: reflecting axes)
template <typename T>
int launch_movers(const sk::Params<T>& a, const int64_t* geo_i, cudaStream_t s) {
  switch ((geo_i[3] ? 1 : 0) | (geo_i[4] ? 2 : 0) | (geo_i[5] ? 4 : 0)) {
    case 0: return launch_mover<T, false, false, false>(a, s);
    case 1: return launch_mover<T, true, false, false>(a, s);
    case 2: return launch_mover<T, false, true, false>(a, s);
    case 3: return launch_mover<T, true, true, false>(a, s);
    case 4: return launch_mover<T, false, false, true>(a, s);
    case 5: return launch_mover<T, true, false, true>(a, s);
    case 6: return launch_mover<T, false, true, true>(a, s);
    default: return launch_mover<T, true, true, true>(a, s);
  }
}

template <typename T>
int launch_pair(const sk::Params<T>& a, const int64_t* geo_i, cudaStream_t s) {
  const int rc = launch_movers<T>(a, geo_i, s);
  return rc ? rc : launch_deposit<T>(a, s);
}

}  // namespace

// kernel parameters of one span call (geometry, scalars, pointers); the
// per-call scratch (work counter, skip bitmask, records) is the caller's
template <typename T>
void fill_params(const Call& c, sk::Params<T>& a) {
  a = sk::Params<T>{};
  a.x = (T*)c.x; a.y = (T*)c.y; a.z = (T*)c.z;
  a.u = (T*)c.u; a.v = (T*)c.v; a.w = (T*)c.w;
  a.q = (const T*)c.q;
  a.start = c.start; a.count = c.count;
  a.iv_f = c.fbytes == 4 ? (const float*)c.invvol : nullptr;
  a.iv_d = c.fbytes == 8 ? (const double*)c.invvol : nullptr;
  a.acc = (long long*)c.acc;
  a.nx = (int)c.geo_i[0]; a.ny = (int)c.geo_i[1]; a.nz = (int)c.geo_i[2];
  a.NY = a.ny + 1; a.NZ = a.nz + 1; a.NN = (a.nx + 1) * a.NY * a.NZ;
  a.cny = a.nx * a.ny;
  a.nm1[0] = (T)(a.nx - 1); a.nm1[1] = (T)(a.ny - 1); a.nm1[2] = (T)(a.nz - 1);
  a.nxf = (T)a.nx; a.cnyf = (T)a.cny;
  for (int k = 0; k < 3; ++k) {
    const T o = (T)c.geo_f[3 + k], L = (T)c.geo_f[6 + k];
    const T hi = o + L;  // particle-precision sum, as the reference
    a.o[k] = o; a.L[k] = L; a.hi[k] = hi; a.hi2[k] = hi + hi;
    const double gd = c.fbytes == 8 ? c.geo_g[k] : (double)(float)c.geo_g[k];
    const double go = c.fbytes == 8 ? c.geo_g[3 + k] : (double)(float)c.geo_g[3 + k];
    a.idx[k] = (T)(1.0 / gd);
    a.ogs[k] = (T)(go / gd);
    a.bc_eps[k] = (T)((sizeof(T) == 4 ? 1e-5 : 1e-13) * (fabs((double)o) + (double)L) + 1e-30);
  }
  a.dt = (T)c.dt; a.dth = (T)c.dth; a.qdt2m = (T)c.qdt2m;
  a.beta = (T)c.beta;
  a.beta2 = a.beta * a.beta;
  a.scale = c.scale;
  a.n_iters = c.n_iters;
  a.status = c.status;
}
template void fill_params<float>(const Call&, sk::Params<float>&);
template void fill_params<double>(const Call&, sk::Params<double>&);

namespace {

template <typename T>
int split_fused(const Call& c, const void* rec_in, cudaStream_t s) {
  sk::Params<T> a;
  fill_params<T>(c, a);
  void* rec = const_cast<void*>(rec_in);
  const size_t rbytes = split_records_bytes((int)sizeof(T), c.geo_i);
  // one bit per particle, +2 words of slack
  const size_t skip_bytes = (((size_t)c.count + 31) / 32 * 4 + 8 + 255) & ~(size_t)255;
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, 256 + skip_bytes + (rec ? 0 : rbytes), s);
  if (e != cudaSuccess) {
    set_error("split scratch alloc: %s", cudaGetErrorString(e));
    return -2;
  }
  a.work = (unsigned long long*)scratch;
  a.skip = (unsigned*)((char*)scratch + 256);
  cudaMemsetAsync(scratch, 0, 256 + skip_bytes, s);
  int rc = 0;
  if (!rec) {
    rec = (char*)scratch + 256 + skip_bytes;
    rc = split_pack_records((int)sizeof(T), c.fbytes, c.E, c.B, c.geo_i, rec, s);
  }
  a.rec = rec;
  a.emax = reinterpret_cast<const float*>((const char*)rec + (rbytes - 32));
  if (!rc) rc = launch_pair<T>(a, c.geo_i, s);
  cudaFreeAsync(scratch, s);
  return rc;
}

}  // namespace

size_t split_records_bytes(int pbytes, const int64_t* geo_i) {
  // 12 quads of the particle type per cell, then 32 bytes holding max |E|
  return (size_t)geo_i[0] * geo_i[1] * geo_i[2] * 48 * (pbytes == 8 ? 8 : 4) + 32;
}

int split_pack_records(int pbytes, int fbytes, const void* E, const void* B,
                       const int64_t* geo_i, void* rec, cudaStream_t s) {
  const int nx = (int)geo_i[0], ny = (int)geo_i[1], nz = (int)geo_i[2];
  const dim3 blocks((unsigned)(((nx + sk::kPackTI - 1) / sk::kPackTI) *
                               ((nz + sk::kPackTK - 1) / sk::kPackTK)),
                    (unsigned)ny);
  unsigned* emax =
      reinterpret_cast<unsigned*>((char*)rec + split_records_bytes(pbytes, geo_i) - 32);
  cudaMemsetAsync(emax, 0, 32, s);
  const int th = timing_begin(TK_RECORDS, s);
  const size_t osm = (size_t)8 * sk::kPackTI * 48 * (pbytes == 8 ? 8 : 4);
  static bool attr[64] = {};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(sk::pack_cells<double, double>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * sk::kPackTI * 48 * 8);
    cudaFuncSetAttribute(sk::pack_cells<float, double>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * sk::kPackTI * 48 * 8);
    cudaFuncSetAttribute(sk::pack_cells<double, float>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * sk::kPackTI * 48 * 4);
    cudaFuncSetAttribute(sk::pack_cells<float, float>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * sk::kPackTI * 48 * 4);
  });
  if (pbytes == 8) {
    if (fbytes == 8)
      sk::pack_cells<double, double><<<blocks, 256, osm, s>>>((const double*)E, (const double*)B,
                                                            nx, ny, nz, (double*)rec, emax);
    else
      sk::pack_cells<float, double><<<blocks, 256, osm, s>>>((const float*)E, (const float*)B,
                                                           nx, ny, nz, (double*)rec, emax);
  } else {
    if (fbytes == 8)
      sk::pack_cells<double, float><<<blocks, 256, osm, s>>>((const double*)E, (const double*)B,
                                                           nx, ny, nz, (float*)rec, emax);
    else
      sk::pack_cells<float, float><<<blocks, 256, osm, s>>>((const float*)E, (const float*)B, nx,
                                                          ny, nz, (float*)rec, emax);
  }
  timing_end(th, s);
  note_launch();
  return launch_check("cell record pack");
}

// f64 fast fused span, push half: the split mover (coefficient records,
// warp-uniform interior skip) over the span, each failed particle's bit set
// in `skip`; the deposit half is the generic kernel's per-contribution
// lattice deposit (bp_fast.cu), which keeps f64 within 1e-10.
int split_push_f64(const Call& c, const void* rec_in, unsigned* skip, cudaStream_t s) {
  sk::Params<double> a;
  fill_params<double>(c, a);
  void* rec = const_cast<void*>(rec_in);
  const size_t rbytes = split_records_bytes(8, c.geo_i);
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, 256 + (rec ? 0 : rbytes), s);
  if (e != cudaSuccess) {
    set_error("split scratch alloc: %s", cudaGetErrorString(e));
    return -2;
  }
  a.work = (unsigned long long*)scratch;
  a.skip = skip;
  cudaMemsetAsync(scratch, 0, 256, s);
  int rc = 0;
  if (!rec) {
    rec = (char*)scratch + 256;
    rc = split_pack_records(8, c.fbytes, c.E, c.B, c.geo_i, rec, s);
  }
  a.rec = rec;
  a.emax = reinterpret_cast<const float*>((const char*)rec + (rbytes - 32));
  if (!rc) rc = launch_movers<double>(a, c.geo_i, s);
  cudaFreeAsync(scratch, s);
  return rc;
}

int split_fused(const Call& c, const void* rec, cudaStream_t s) {
  // the f64 instantiation (per-tile f64 sums) measured 25% faster than the
  // generic f64 kernel but outside 1e-10 of the reference's per-contribution
  // lattice rounding on the small moments, so only f32 particles come here
  if (c.pbytes != 4) {
    set_error("split kernels: f32 particles only");
    return -1;
  }
  return split_fused<float>(c, rec, s);
}

}  // namespace bp
