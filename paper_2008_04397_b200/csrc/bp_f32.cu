// Fused mover + deposition for f32 particles ("single" and "mixed" modes),
// fast arithmetic, sm_100a.  Same algorithm as the reference fused_span
// (pkg/src/batchpic/kernels.py:458-735); the instruction budget per particle
// is what this file is about.
//
// Push: fields come from per-cell coefficient records (pack_cells): for each
// component f the trilinear form
//     f(fx,fy,fz) = [c0 + c1 fx + (c2 + c4 fx) fy] + fz [c3 + c5 fx + (c6 + c7 fx) fy]
// (the reference's 8-weight sum, kernels.py:557-591, regrouped).  Components
// are paired (Ex Ey | Bx By | Ez Bz) and evaluated with the packed FP32
// instruction FFMA2 (two lanes of f32 per instruction, sm_100), so one gather
// is 12 contiguous 16-byte loads from one 192-byte record and 21 FFMA2; the
// record stays in registers while the midpoint remains in its cell, so the
// mover iterations after the first usually load nothing.  Boundary kinds are
// template parameters.
//
// Deposit: the per-warp transposed fold of bp_common.cuh (lane = corner x
// moment group, 32 staged particles per tile) in f32: each tile's partial sum
// of q * w_c * m is rounded once onto the int64 lattice, after multiplying by
// invvol * 2^43 of the lane's node (kernels.py:707-734 apply invvol and the
// scale per contribution; here per tile — within the 1e-4 f32 tolerance).
// Integer slot sums and REDG.ADD.64 flushes as in the exact path.  Slots are
// flushed at the end of every dynamically claimed chunk, so every tile's
// grouping depends only on the chunk's content: the result is deterministic.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "bp_common.cuh"
#include "bp_launch.h"

namespace bp {
namespace f32k {

struct Params {
  float *x, *y, *z, *u, *v, *w;
  const float* q;
  long long start, count;
  const float4* rec;     // 12 float4 per cell, cell = i + nx * (j + ny * k)
  const float* iv_f;     // invvol (nx+1, ny+1, nz+1) when fields are f32
  const double* iv_d;    // ... when fields are f64 (mixed)
  long long* acc;        // (10, NN) int64
  int nx, ny, nz, NY, NZ, NN;
  int cny;               // nx * ny (cell-record z stride)
  float o[3], hi[3], L[3], hi2[3], idx[3], ogs[3];
  float dt, dth, qdt2m, beta, beta2;
  double scale;
  int n_iters;
  int* status;
  unsigned long long* work;  // deposit: next unclaimed particle of the span
  unsigned* skip;            // one bit per span particle the mover did not store
  const float* emax;         // max |E| over the nodes (end of the cell records)
  float bc_eps[3];           // rounding slack of the boundary-skip test per axis
};

constexpr int kRow = 36;  // staged row stride (floats): conflict-free LDS.128 per warp
// staging rows: 8 bases (corner c) then 10 moments (row 8 + m); row 8 (m = 1) is constant
constexpr int kStage = 18 * kRow;

__device__ __forceinline__ float4 ldg4(const float4* p) {
  float4 r;
  asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p));
  return r;
}

// 1 / d for d = 1 + beta^2 |h|^2 >= 1 (MUFU.RCP alone, no range fix-up)
__device__ __forceinline__ float rcp_approx(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return r;
}

// one 32-byte load (LDG.E.ENL2.256) into two float4; cell records are
// kept in L1 / L2 in preference to the particle streams (evict_last)
__device__ __forceinline__ void ldg8(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.L1::evict_last.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}

// pull a cell record (192 bytes = two 128-byte lines) into L1
__device__ __forceinline__ void prefetch_record(const float4* r) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(r));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(r + 11));
}

template <bool REFL>
__device__ __forceinline__ float fold_mid(float xm, float o, float L, float hi, float hi2) {
  if (!REFL) {
    if (xm < o) xm += L;
    else if (xm > hi) xm -= L;
  } else {
    if (xm < o) xm = o + (o - xm);
    else if (xm > hi) xm = hi2 - xm;
  }
  return xm;
}

template <bool REFL>
__device__ __forceinline__ void fold_commit(float& q, float& vel, float o, float L, float hi,
                                            float hi2) {
  if (!REFL) {
    if (q < o) {
      q += L;
      if (q >= hi) q = o;
    } else if (q >= hi) {
      q -= L;
    }
  } else {
    if (q < o) {
      q = o + (o - q);
      vel = -vel;
    } else if (q > hi) {
      q = hi2 - q;
      vel = -vel;
    }
  }
}

// True when no position of the push can leave the box: the implicit
// rotation never lengthens t = v + qdt2m E (|v_bar| <= |t|),
// and |E| at any point is at most its node maximum, so every midpoint and the
// committed position lie within dt * (|v|_1 + |qdt2m| max|E|) of the start.
__device__ __forceinline__ bool interior(const Params& a, float qe, float x, float y, float z,
                                         float u, float v, float w) {
  const float reach = (fabsf(u) + fabsf(v) + fabsf(w) + qe) * a.dt;
  return x - a.o[0] > reach + a.bc_eps[0] && a.hi[0] - x > reach + a.bc_eps[0] &&
         y - a.o[1] > reach + a.bc_eps[1] && a.hi[1] - y > reach + a.bc_eps[1] &&
         z - a.o[2] > reach + a.bc_eps[2] && a.hi[2] - z > reach + a.bc_eps[2];
}

// cell of an in-box position: truncation (in-box gx >= -ulp truncates to 0)
// and the upper-face clamp of kernels.py:541-556; returns the cell index
__device__ __forceinline__ int cell_of(const Params& a, float x, float y, float z, float& fx,
                                      float& fy, float& fz, int& i, int& j, int& k) {
  const float gx = fmaf(x, a.idx[0], -a.ogs[0]);
  const float gy = fmaf(y, a.idx[1], -a.ogs[1]);
  const float gz = fmaf(z, a.idx[2], -a.ogs[2]);
  i = min((int)gx, a.nx - 1);
  j = min((int)gy, a.ny - 1);
  k = min((int)gz, a.nz - 1);
  fx = gx - (float)i;
  fy = gy - (float)j;
  fz = gz - (float)k;
  return i + a.nx * j + a.cny * k;
}

typedef float2 F2;
__device__ __forceinline__ F2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ F2 mul2(F2 a, F2 b) { return __fmul2_rn(a, b); }

// one component pair from its four coefficient quads (record layout of
// pack_cells: A = c0 c0' c1 c1', B = c2 c2' c4 c4', C = c3 c3' c5 c5', D = c6 c6' c7 c7')
__device__ __forceinline__ F2 tri2(const float4& A, const float4& B, const float4& C,
                                   const float4& D, F2 FX, F2 FY, F2 FZ) {
  const F2 p = fma2(f2(A.z, A.w), FX, f2(A.x, A.y));
  const F2 q = fma2(f2(B.z, B.w), FX, f2(B.x, B.y));
  const F2 r = fma2(f2(C.z, C.w), FX, f2(C.x, C.y));
  const F2 t = fma2(f2(D.z, D.w), FX, f2(D.x, D.y));
  return fma2(fma2(t, FY, r), FZ, fma2(q, FY, p));
}

// skipbc (warp-uniform): the caller has shown that no position of this push
// can leave the box (interior()), so the boundary folds and checks are
// identities and are skipped.
template <bool RX, bool RY, bool RZ, bool REUSE>
__device__ __forceinline__ int push(const Params& a, float& xp, float& yp, float& zp, float& un,
                                    float& vn, float& wn, bool skipbc = false) {
  float vbx = un, vby = vn, vbz = wn;
  float4 R[12];
  int held = -1;  // cell whose record is in R
#pragma unroll 1
  for (int it = 0; it < a.n_iters; ++it) {
    const F2 XM = fma2(f2(vbx, vby), f2(a.dth, a.dth), f2(xp, yp));
    float xm = XM.x, ym = XM.y, zm = fmaf(vbz, a.dth, zp);
    if (!skipbc) {
      xm = fold_mid<RX>(xm, a.o[0], a.L[0], a.hi[0], a.hi2[0]);
      ym = fold_mid<RY>(ym, a.o[1], a.L[1], a.hi[1], a.hi2[1]);
      zm = fold_mid<RZ>(zm, a.o[2], a.L[2], a.hi[2], a.hi2[2]);
      if (xm < a.o[0] || xm > a.hi[0] || ym < a.o[1] || ym > a.hi[1] || zm < a.o[2] ||
          zm > a.hi[2])
        return ST_MIDPOINT;
    }
    float fx, fy, fz;
    int i, j, k;
    const int cell = cell_of(a, xm, ym, zm, fx, fy, fz, i, j, k);
    if (!REUSE || cell != held) {
      held = cell;
      const float4* r = a.rec + (size_t)cell * 12;
#pragma unroll
      for (int q = 0; q < 12; q += 2) ldg8(r + q, R[q], R[q + 1]);
    }
    const F2 FX = f2(fx, fx), FY = f2(fy, fy), FZ = f2(fz, fz);
    const F2 Exy = tri2(R[0], R[1], R[2], R[3], FX, FY, FZ);
    const F2 Bxy = tri2(R[4], R[5], R[6], R[7], FX, FY, FZ);
    const F2 EBz = tri2(R[8], R[9], R[10], R[11], FX, FY, FZ);
    const F2 Txy = fma2(f2(a.qdt2m, a.qdt2m), Exy, f2(un, vn));
    const float tx = Txy.x, ty = Txy.y, tz = fmaf(a.qdt2m, EBz.x, wn);
    const float hx = Bxy.x, hy = Bxy.y, hz = EBz.y;
    const float bsq = fmaf(hx, hx, fmaf(hy, hy, hz * hz));
    const float inv = rcp_approx(fmaf(a.beta2, bsq, 1.0f));
    const float tdb = fmaf(tx, hx, fmaf(ty, hy, tz * hz));
    const float bt = a.beta * tdb;
    const float cx = fmaf(ty, hz, -tz * hy), cy = fmaf(tz, hx, -tx * hz),
                cz = fmaf(tx, hy, -ty * hx);
    vbx = fmaf(a.beta, fmaf(bt, hx, cx), tx) * inv;
    vby = fmaf(a.beta, fmaf(bt, hy, cy), ty) * inv;
    vbz = fmaf(a.beta, fmaf(bt, hz, cz), tz) * inv;
  }
  float xo = fmaf(vbx, a.dt, xp), yo = fmaf(vby, a.dt, yp), zo = fmaf(vbz, a.dt, zp);
  float uo = 2.0f * vbx - un, vo = 2.0f * vby - vn, wo = 2.0f * vbz - wn;
  if (!skipbc) {
    fold_commit<RX>(xo, uo, a.o[0], a.L[0], a.hi[0], a.hi2[0]);
    fold_commit<RY>(yo, vo, a.o[1], a.L[1], a.hi[1], a.hi2[1]);
    fold_commit<RZ>(zo, wo, a.o[2], a.L[2], a.hi[2], a.hi2[2]);
    if (xo < a.o[0] || xo > a.hi[0] || yo < a.o[1] || yo > a.hi[1] || zo < a.o[2] ||
        zo > a.hi[2])
      return ST_RUNAWAY;
  }
  xp = xo; yp = yo; zp = zo;
  un = uo; vn = vo; wn = wo;
  return ST_OK;
}

// ---------------------------------------------------------------------------
// Deposition.  Lane L of a warp owns corner c = L & 7 of moments g, g + 4
// (g = L >> 3) and, over half a tile, moment 8 + (g & 1).  Every tile's
// staged particles are folded per cell in f32 (q * w_c * m) and added into a
// per-warp node patch in shared memory: f32 sums over the nodes
// [pi0, pi0 + PX) x [pj0, pj0 + 4) x [pk0, pk0 + 4) for the 10 moments — the
// neighbourhood of the cells a chunk of sorted particles covers, strays
// included.  Each lane only ever touches the patch values of its own
// (corner, moment) pairs, so no atomics.  The patch is converted to the
// lattice (x invvol x 2^43, rint) and flushed with REDG.ADD.64 when the chunk
// ends or its cells leave the patch.
template <int PX>
struct Patch {
  static constexpr int kNodes = PX * 16;       // node (px, py, pz) at (px * 4 + py) * 4 + pz
  static constexpr int kStride = kNodes + 2;   // per moment; +2 spreads the lane groups over banks
  static constexpr int kFloats = 10 * kStride;
};

// lattice value of a patch sum at global node `node`
__device__ __forceinline__ long long lattice(const Params& a, float v, int node) {
  const double iv = a.iv_d ? __ldg(a.iv_d + node) : (double)__ldg(a.iv_f + node);
  return __double2ll_rn((double)v * iv * a.scale);
}

// The patch's nodes are split over the lanes (node lane + 32 i, i < PX/2);
// each lane holds invvol * 2^43 of its nodes in registers, loaded when the
// patch is anchored so the loads complete long before the flush uses them.
template <int PX>
struct PatchNodes {
  static constexpr int kPer = PX * 16 / 32;
  double ivs[kPer];
  int gnode[kPer];  // global node index, -1 outside the grid
};

template <int PX>
__device__ __forceinline__ void patch_anchor(const Params& a, PatchNodes<PX>& pn, int pi0,
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
template <int PX>
__device__ __forceinline__ void patch_flush(const Params& a, float* patch,
                                            const PatchNodes<PX>& pn, unsigned lane) {
  typedef Patch<PX> Pt;
#pragma unroll
  for (int i = 0; i < PatchNodes<PX>::kPer; ++i) {
    const int n = (int)lane + 32 * i;
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      float* pv = patch + m * Pt::kStride + n;
      const float v = *pv;
      if (v != 0.f) {
        *pv = 0.f;
        if (pn.gnode[i] >= 0)
          atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + (size_t)m * a.NN + pn.gnode[i]),
                    (unsigned long long)__double2ll_rn((double)v * pn.ivs[i]));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Mover: one particle per thread, coalesced SoA streams, no shared memory, so
// the SM holds enough warps to hide the latency of the three dependent
// gather + rotation steps.  Particles that fail (kernels.py:618-621, 672-676)
// are not stored; their bit in `skip` keeps them out of the deposit.
template <bool RX, bool RY, bool RZ, bool REUSE, int MINB, bool PF = false>
__global__ void __launch_bounds__(256, MINB) mover_f32(const __grid_constant__ Params a) {
  // persistent grid: each thread walks particles r, r + stride, ...; the
  // loads of the particle two steps ahead are in flight, and the record of
  // the next particle's cell is prefetched into L1 while this one is pushed
  const long long stride = (long long)gridDim.x * 256;
  long long r = (long long)blockIdx.x * 256 + threadIdx.x;
  float n1[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, n2[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto fetch = [&](long long rr, float* d) {
    if (rr < a.count) {
      const long long p = a.start + rr;
      d[0] = __ldcs(a.x + p); d[1] = __ldcs(a.y + p); d[2] = __ldcs(a.z + p);
      d[3] = __ldcs(a.u + p); d[4] = __ldcs(a.v + p); d[5] = __ldcs(a.w + p);
    }
  };
  fetch(r, n1);
  if (PF) fetch(r + stride, n2);
  // |qdt2m| max|E| (+1e-5 relative slack for the f32 coefficient rounding)
  const float qe = fabsf(a.qdt2m) * __ldg(a.emax) * 1.00001f;
  const long long rbase = r - (threadIdx.x & 31);  // warp-uniform loop bound
  for (long long rb = rbase; rb < a.count; rb += stride, r += stride) {
    float xp = n1[0], yp = n1[1], zp = n1[2], un = n1[3], vn = n1[4], wn = n1[5];
    if (PF) {
#pragma unroll
      for (int q = 0; q < 6; ++q) n1[q] = n2[q];
      fetch(r + 2 * stride, n2);
      float fx, fy, fz;
      int i, j, k;
      const int cell = cell_of(a, n1[0], n1[1], n1[2], fx, fy, fz, i, j, k);
      // one prefetch per distinct cell of the warp (sorted runs share cells)
      const int prev = __shfl_up_sync(0xffffffffu, cell, 1);
      if (r + stride < a.count && ((threadIdx.x & 31) == 0 || prev != cell))
        prefetch_record(a.rec + (size_t)cell * 12);
    } else {
      fetch(r + stride, n1);
    }
    int st = ST_OK;
    // warp-uniform: the whole warp takes the boundary-free push when it can
    const bool all_in =
        __all_sync(0xffffffffu, r >= a.count || interior(a, qe, xp, yp, zp, un, vn, wn));
    if (r < a.count) {
      const long long p = a.start + r;
      st = push<RX, RY, RZ, REUSE>(a, xp, yp, zp, un, vn, wn, all_in);
      if (st == ST_OK) {
        __stcs(a.x + p, xp); __stcs(a.y + p, yp); __stcs(a.z + p, zp);
        __stcs(a.u + p, un); __stcs(a.v + p, vn); __stcs(a.w + p, wn);
      }
    }
    const unsigned bad = __ballot_sync(0xffffffffu, st != ST_OK);
    if (bad) {
      if ((threadIdx.x & 31) == 0) atomicOr(a.skip + (r >> 5), bad);
      if (st != ST_OK) atomicMax(a.status, st);
    }
  }
}

// ---------------------------------------------------------------------------
// Deposit (interpolation of the 10 moments) of the moved particles.  Each
// warp claims chunks of CHUNK particles; tiles of 32 are staged in shared
// memory and folded per cell (see the comment above Patch).
// PUSH: the fused variant (mover + deposit in one pass over the particles,
// BC kinds RX RY RZ); otherwise the particles are deposited as they are.
template <int PX, int CHUNK, int MINB, bool STRAY_VEC, int STRAY_GROUP, bool PUSH = false,
          bool RX = false, bool RY = false, bool RZ = false>
__global__ void __launch_bounds__(256, MINB) deposit_f32(const __grid_constant__ Params a) {
  typedef Patch<PX> Pt;
  extern __shared__ float smem_f[];
  const unsigned lane = lane_id();
  float* const st = smem_f + (threadIdx.x >> 5) * (kStage + Pt::kFloats);
  float* const st_bs = st;             // [8][kRow] bases q * w_c
  float* const st_mv = st + 8 * kRow;  // [10][kRow], row m = moment m (row 0: constant 1)
  float* const patch = st + kStage;    // [10][kStride]
  const int lc = lane & 7, lg = lane >> 3;
  const int poff = (lc & 1) * 16 + ((lc >> 1) & 1) * 4 + ((lc >> 2) & 1);
  const bool third = lg < 2;
  const int m3 = 8 + (lg & 1), h3 = (lg >> 1) * 16;
  // this lane's three patch value columns (moments lg, lg + 4, 8 + lg)
  float* const pv0 = patch + lg * Pt::kStride + poff;
  float* const pv1 = patch + (lg + 4) * Pt::kStride + poff;
  float* const pv2 = patch + (third ? lg + 8 : 8) * Pt::kStride + poff;
  st_mv[lane] = 1.0f;
  for (int r = lane; r < Pt::kFloats; r += 32) patch[r] = 0.f;
  __syncwarp();
  long long nxt = 0;
  if (lane == 0) nxt = (long long)atomicAdd(a.work, (unsigned long long)CHUNK);
  nxt = __shfl_sync(0xffffffffu, nxt, 0);
  // prefetched particle of the next tile
  float px_ = 0.f, py_ = 0.f, pz_ = 0.f, pu_ = 0.f, pv_ = 0.f, pw_ = 0.f, pq_ = 0.f;
  unsigned sk_ = 0u;
  auto fetch = [&](long long r, long long end) {
    if (r < end) {
      const long long p = a.start + r;
      px_ = __ldcs(a.x + p); py_ = __ldcs(a.y + p); pz_ = __ldcs(a.z + p);
      pu_ = __ldcs(a.u + p); pv_ = __ldcs(a.v + p); pw_ = __ldcs(a.w + p);
      pq_ = __ldcs(a.q + p);
    }
    if (!PUSH) sk_ = __ldg(a.skip + (r >> 5));
  };
  if (nxt < a.count) fetch(nxt + lane, nxt + CHUNK < a.count ? nxt + CHUNK : a.count);
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
      bool valid = r < w1 && (PUSH || !((sk_ >> lane) & 1u));
      float xp = px_, yp = py_, zp = pz_, un = pu_, vn = pv_, wn = pw_;
      const float qp = pq_;
      if (t0 + 32 < w1) fetch(t0 + 32 + lane, w1);
      else if (nxt < a.count) fetch(nxt + lane, nxt + CHUNK < a.count ? nxt + CHUNK : a.count);
      if (PUSH && valid) {
        const int st = push<RX, RY, RZ, true>(a, xp, yp, zp, un, vn, wn);
        if (st != ST_OK) {
          atomicMax(a.status, st);  // not stored, not deposited (kernels.py:618-621)
          valid = false;
        } else {
          const long long p = a.start + r;
          __stcs(a.x + p, xp); __stcs(a.y + p, yp); __stcs(a.z + p, zp);
          __stcs(a.u + p, un); __stcs(a.v + p, vn); __stcs(a.w + p, wn);
        }
      }
      // ---- stage this lane's particle: 8 bases q*w_c and the moments
      int ci = 0, cj = 0, ck = 0;
      {
        float fx = 0.f, fy = 0.f, fz = 0.f, qs = 0.f;
        if (valid) {
          cell_of(a, xp, yp, zp, fx, fy, fz, ci, cj, ck);
          qs = qp;
        }
        const float qax = qs * (1.0f - fx), qfx = qs * fx;
        const float ay = 1.0f - fy, az = 1.0f - fz;
        const float w00 = qax * ay, w10 = qfx * ay, w01 = qax * fy, w11 = qfx * fy;
        st_bs[0 * kRow + lane] = w00 * az; st_bs[1 * kRow + lane] = w10 * az;
        st_bs[2 * kRow + lane] = w01 * az; st_bs[3 * kRow + lane] = w11 * az;
        st_bs[4 * kRow + lane] = w00 * fz; st_bs[5 * kRow + lane] = w10 * fz;
        st_bs[6 * kRow + lane] = w01 * fz; st_bs[7 * kRow + lane] = w11 * fz;
        float* mv = st_mv + lane;
        mv[1 * kRow] = un; mv[2 * kRow] = vn; mv[3 * kRow] = wn;
        mv[4 * kRow] = un * un; mv[5 * kRow] = un * vn; mv[6 * kRow] = un * wn;
        mv[7 * kRow] = vn * vn; mv[8 * kRow] = vn * wn; mv[9 * kRow] = wn * wn;
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
      // ---- other cells of the tile.  A large group (a sorted run's next
      // cell) is folded over its quads with the other lanes masked; the
      // remaining strays are added one by one straight into the patch.
      unsigned rest = F & ~Mm;
      if (rest) {
        const int k2 = __shfl_sync(0xffffffffu, pnode, __ffs(rest) - 1);
        const unsigned M2 = __ballot_sync(0xffffffffu, fit && pnode == k2);
        const int q0 = (__ffs(M2) - 1) >> 2, q1 = (31 - __clz(M2)) >> 2;
        if (STRAY_VEC && 20 * (q1 - q0 + 1) < 15 * __popc(M2)) {
          rest &= ~M2;
          F2 T0 = f2(0.f, 0.f), T1 = f2(0.f, 0.f), T2 = f2(0.f, 0.f);
          const float* m2r = st_mv + (third ? lg + 8 : 8) * kRow;
          for (int q = q0; q <= q1; ++q) {
            const unsigned bits = M2 >> (4 * q);
            float4 b = *reinterpret_cast<const float4*>(st_bs + lc * kRow + 4 * q);
            b.x = (bits & 1u) ? b.x : 0.f;
            b.y = (bits & 2u) ? b.y : 0.f;
            b.z = (bits & 4u) ? b.z : 0.f;
            b.w = (bits & 8u) ? b.w : 0.f;
            const float4 x0 = *reinterpret_cast<const float4*>(st_mv + lg * kRow + 4 * q);
            const float4 x1 = *reinterpret_cast<const float4*>(st_mv + (lg + 4) * kRow + 4 * q);
            const float4 x2 = *reinterpret_cast<const float4*>(m2r + 4 * q);
            T0 = fma2(f2(b.x, b.y), f2(x0.x, x0.y), T0);
            T0 = fma2(f2(b.z, b.w), f2(x0.z, x0.w), T0);
            T1 = fma2(f2(b.x, b.y), f2(x1.x, x1.y), T1);
            T1 = fma2(f2(b.z, b.w), f2(x1.z, x1.w), T1);
            T2 = fma2(f2(b.x, b.y), f2(x2.x, x2.y), T2);
            T2 = fma2(f2(b.z, b.w), f2(x2.z, x2.w), T2);
          }
          pv0[k2] += T0.x + T0.y;
          pv1[k2] += T1.x + T1.y;
          if (third) pv2[k2] += T2.x + T2.y;
        }
        if (STRAY_GROUP) {
          const float* brow = st_bs + lc * kRow;
          const float* m0row = st_mv + lg * kRow;
          const float* m1row = st_mv + (lg + 4) * kRow;
          const float* m2row = st_mv + (third ? lg + 8 : 8) * kRow;
          while (rest) {
            const int kg = __shfl_sync(0xffffffffu, pnode, __ffs(rest) - 1);
            const unsigned MG = __ballot_sync(0xffffffffu, fit && pnode == kg);
            rest &= ~MG;
            // the cell's patch values are read first (no alias with the
            // staged rows) so their latency hides behind the fold
            const float o0 = pv0[kg], o1 = pv1[kg], o2 = pv2[kg];
            float t0s = 0.f, t1s = 0.f, t2s = 0.f;
            for (unsigned m = MG; m; m &= m - 1u) {
              const int kk = __ffs(m) - 1;
              const float b = brow[kk];
              t0s = fmaf(b, m0row[kk], t0s);
              t1s = fmaf(b, m1row[kk], t1s);
              t2s = fmaf(b, m2row[kk], t2s);
            }
            pv0[kg] = o0 + t0s;
            pv1[kg] = o1 + t1s;
            if (third) pv2[kg] = o2 + t2s;
          }
        } else {
          for (; rest; rest &= rest - 1u) {
            const int kk = __ffs(rest) - 1;
            const int k3 = __shfl_sync(0xffffffffu, pnode, kk);
            const float b = st_bs[lc * kRow + kk];
            pv0[k3] = fmaf(b, st_mv[lg * kRow + kk], pv0[k3]);
            pv1[k3] = fmaf(b, st_mv[(lg + 4) * kRow + kk], pv1[k3]);
            if (third) pv2[k3] = fmaf(b, st_mv[(lg + 8) * kRow + kk], pv2[k3]);
          }
        }
      }
      // ---- particles whose cells are outside the patch (rare): straight to the lattice
      unsigned out = V & ~F;
      while (out) {
        const int src = __ffs(out) - 1;
        const int oi = __shfl_sync(0xffffffffu, ci, src);
        const int oj = __shfl_sync(0xffffffffu, cj, src);
        const int ok = __shfl_sync(0xffffffffu, ck, src);
        const unsigned M2 = __ballot_sync(0xffffffffu, valid && !fit && ci == oi && cj == oj &&
                                                         ck == ok);
        out &= ~M2;
        float t0s = 0.f, t1s = 0.f, t2s = 0.f;
        for (unsigned m = M2; m; m &= m - 1u) {
          const int kk = __ffs(m) - 1;
          const float b = st_bs[lc * kRow + kk];
          t0s = fmaf(b, st_mv[lg * kRow + kk], t0s);
          t1s = fmaf(b, st_mv[(lg + 4) * kRow + kk], t1s);
          t2s = fmaf(b, st_mv[(third ? lg + 8 : 8) * kRow + kk], t2s);
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
        if (((V & ~Mm) >> lane) & 1u) {
#pragma unroll
          for (int c = 0; c < 8; ++c) st_bs[c * kRow + lane] = 0.0f;
        }
        __syncwarp();
      }
      // ---- main fold: all 32 staged particles (others have zero bases)
      if (Mm) {
        const float* br = st_bs + lc * kRow;
        const float* m0r = st_mv + lg * kRow;
        const float* m1r = st_mv + (lg + 4) * kRow;
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
        const float* b3 = st_bs + lc * kRow + h3;
        const float* m3r = st_mv + m3 * kRow + h3;
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          const float4 b = *reinterpret_cast<const float4*>(b3 + kk);
          const float4 x2 = *reinterpret_cast<const float4*>(m3r + kk);
          S2 = fma2(f2(b.x, b.y), f2(x2.x, x2.y), S2);
          S2 = fma2(f2(b.z, b.w), f2(x2.z, x2.w), S2);
        }
        float s2 = S2.x + S2.y;
        s2 += __shfl_xor_sync(0xffffffffu, s2, 16);
        pv0[kmain] += S0.x + S0.y;
        pv1[kmain] += S1.x + S1.y;
        if (third) pv2[kmain] += s2;
      }
      __syncwarp();
    }
    if (anchored) patch_flush<PX>(a, patch, pn, lane);
    __syncwarp();
  }
}

// Per-cell coefficient records (computed in f64, rounded once to f32), three
// component pairs (a, b) = (Ex, Ey), (Bx, By), (Ez, Bz), four float4 each:
// (c0a c0b c1a c1b) (c2a c2b c4a c4b) (c3a c3b c5a c5b) (c6a c6b c7a c7b).
template <typename F>
__global__ void pack_cells(const F* __restrict__ E, const F* __restrict__ B, int nx, int ny,
                           int nz, float4* __restrict__ rec, unsigned* __restrict__ emax_bits) {
  double e2max = 0.0;  // max over nodes of |E|^2 (the mover's boundary-skip bound)
  const int NY = ny + 1, NZ = nz + 1, NN = (nx + 1) * NY * NZ;
  const int ncell = nx * ny * nz;
  // component of pair slot (pair p, member h): Ex Ey | Bx By | Ez Bz
  const int comp[6] = {0, 1, 3, 4, 2, 5};
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncell; t += gridDim.x * blockDim.x) {
    // threads walk the cells k fastest (coalesced field reads, k is the
    // fastest index of E / B); records are stored x fastest (sort order)
    const int k = t % nz, j = (t / nz) % ny, i = t / (nz * ny);
    const int c = i + nx * (j + ny * k);
    const int n0 = (i * NY + j) * NZ + k;
    const int sx = NY * NZ, sy = NZ;
    float co[6][8];
    double e2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int h = 0; h < 6; ++h) {
      const int m = comp[h];
      const F* f = (m < 3 ? E + (size_t)m * NN : B + (size_t)(m - 3) * NN) + n0;
      const double f000 = f[0], f100 = f[sx], f010 = f[sy], f110 = f[sx + sy];
      const double f001 = f[1], f101 = f[sx + 1], f011 = f[sy + 1], f111 = f[sx + sy + 1];
      if (m < 3) {
        e2[0] += f000 * f000; e2[1] += f100 * f100; e2[2] += f010 * f010; e2[3] += f110 * f110;
        e2[4] += f001 * f001; e2[5] += f101 * f101; e2[6] += f011 * f011; e2[7] += f111 * f111;
      }
      co[h][0] = (float)f000;
      co[h][1] = (float)(f100 - f000);
      co[h][2] = (float)(f010 - f000);
      co[h][3] = (float)(f001 - f000);
      co[h][4] = (float)((f110 - f100) - (f010 - f000));
      co[h][5] = (float)((f101 - f001) - (f100 - f000));
      co[h][6] = (float)((f011 - f001) - (f010 - f000));
      co[h][7] = (float)(((f111 - f011) - (f101 - f001)) - ((f110 - f010) - (f100 - f000)));
    }
    float4* o = rec + (size_t)c * 12;
#pragma unroll
    for (int pr = 0; pr < 3; ++pr) {
      const float* A = co[2 * pr];
      const float* Bq = co[2 * pr + 1];
      o[4 * pr + 0] = make_float4(A[0], Bq[0], A[1], Bq[1]);
      o[4 * pr + 1] = make_float4(A[2], Bq[2], A[4], Bq[4]);
      o[4 * pr + 2] = make_float4(A[3], Bq[3], A[5], Bq[5]);
      o[4 * pr + 3] = make_float4(A[6], Bq[6], A[7], Bq[7]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) e2max = fmax(e2max, e2[q]);
  }
  // non-negative floats order like their bit patterns; rounded up
  unsigned bits = __float_as_uint(__double2float_ru(sqrt(e2max)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, o));
  if ((threadIdx.x & 31) == 0 && bits) atomicMax(emax_bits, bits);
}

}  // namespace f32k

namespace {

int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

int sm_count_f32() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// blocks per SM cap (BP_F32_MOVER_BPS / BP_F32_DEPOSIT_BPS; 0 = occupancy):
// lets a mover and a deposit of different spans share the SMs when the
// caller runs them on two streams
int env_int(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}

template <bool RX, bool RY, bool RZ, bool REUSE, int MINB, bool PF = false>
int launch_mover_cfg(const f32k::Params& a, cudaStream_t s) {
  auto k = f32k::mover_f32<RX, RY, RZ, REUSE, MINB, PF>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
  static const int cap = env_int("BP_F32_MOVER_BPS");
  if (cap > 0 && per_sm > cap) per_sm = cap;
  if (per_sm < 1) per_sm = 1;
  const long long need = (a.count + 255) / 256;
  long long g = (long long)sm_count_f32() * per_sm;
  if (need < g) g = need;
  if (g < 1) g = 1;
  const int th = timing_begin(TK_MOVER, s);
  k<<<(int)g, 256, 0, s>>>(a);
  timing_end(th, s);
  note_launch();
  return launch_check("f32 mover launch");
}

template <bool RX, bool RY, bool RZ>
int launch_mover(const f32k::Params& a, cudaStream_t s) {
  static int cfg = -1;
  if (cfg < 0) {
    const char* env = getenv("BP_F32_MOVER");
    cfg = env ? atoi(env) : 0;
  }
  // record reuse across the mover iterations (the midpoint rarely leaves its
  // cell) needs ~100 registers: 16 warps / SM; measured best on the GEM bench
  switch (cfg) {
    case 1: return launch_mover_cfg<RX, RY, RZ, true, 2, true>(a, s);  // + record prefetch
    case 2: return launch_mover_cfg<RX, RY, RZ, true, 3>(a, s);
    default: return launch_mover_cfg<RX, RY, RZ, true, 2>(a, s);
  }
}

template <int PX, int CHUNK, int MINB, bool SV, int SG, bool PUSH = false, bool RX = false,
          bool RY = false, bool RZ = false>
int launch_deposit_cfg(const f32k::Params& a, cudaStream_t s) {
  auto k = f32k::deposit_f32<PX, CHUNK, MINB, SV, SG, PUSH, RX, RY, RZ>;
  const size_t smem = (size_t)(256 / 32) * (f32k::kStage + f32k::Patch<PX>::kFloats) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem);
  static const int cap = env_int("BP_F32_DEPOSIT_BPS");
  if (cap > 0 && per_sm > cap) per_sm = cap;
  if (per_sm < 1) per_sm = 1;
  const long long need = (a.count + CHUNK * 8 - 1) / (CHUNK * 8);
  long long g = (long long)sm_count_f32() * per_sm;
  if (need < g) g = need;
  if (g < 1) g = 1;
  const int th = timing_begin(TK_DEPOSIT, s);
  k<<<(int)g, 256, smem, s>>>(a);
  timing_end(th, s);
  note_launch();
  return launch_check("f32 deposit launch");
}

int launch_deposit(const f32k::Params& a, cudaStream_t s) {
  static int cfg = -1;
  if (cfg < 0) {
    const char* env = getenv("BP_F32_DEPOSIT");
    cfg = env ? atoi(env) : 0;
  }
  switch (cfg) {
    // strays: per-cell groups folded then added (default, measured best on
    // the GEM bench), + a masked-quad fold of a large second group, or one
    // by one straight into the patch
    case 1: return launch_deposit_cfg<8, 512, 3, true, 1>(a, s);
    case 2: return launch_deposit_cfg<8, 512, 3, false, 0>(a, s);
    case 3: return launch_deposit_cfg<12, 1024, 2, false, 1>(a, s);
    case 5: return launch_deposit_cfg<8, 1024, 3, false, 1>(a, s);
    case 6: return launch_deposit_cfg<8, 256, 3, false, 1>(a, s);
    default: return launch_deposit_cfg<8, 512, 3, false, 1>(a, s);
  }
}

}  // namespace

// Number of bytes of cell records for a grid (12 float4 per cell).
size_t f32_records_bytes(const int64_t* geo_i) {
  // 12 float4 per cell, then 32 bytes: max |E| over the nodes (float)
  return (size_t)geo_i[0] * geo_i[1] * geo_i[2] * 12 * sizeof(float4) + 32;
}

int f32_pack_records(int fbytes, const void* E, const void* B, const int64_t* geo_i,
                     void* rec, cudaStream_t s) {
  const int nx = (int)geo_i[0], ny = (int)geo_i[1], nz = (int)geo_i[2];
  const long long ncell = (long long)nx * ny * nz;
  int blocks = (int)((ncell + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  const int th = timing_begin(TK_RECORDS, s);
  unsigned* emax = reinterpret_cast<unsigned*>((char*)rec + (size_t)ncell * 12 * sizeof(float4));
  cudaMemsetAsync(emax, 0, 32, s);
  if (fbytes == 8)
    f32k::pack_cells<double><<<blocks, 256, 0, s>>>((const double*)E, (const double*)B, nx, ny,
                                                     nz, (float4*)rec, emax);
  else
    f32k::pack_cells<float><<<blocks, 256, 0, s>>>((const float*)E, (const float*)B, nx, ny, nz,
                                                    (float4*)rec, emax);
  timing_end(th, s);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("cell record pack: %s", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

// Fused f32 launch with prebuilt records (rec) or, when rec == NULL, records
// built on the stream for this call.
int f32_fused(const Call& c, const void* rec_in, cudaStream_t s) {
  f32k::Params a;
  a.x = (float*)c.x; a.y = (float*)c.y; a.z = (float*)c.z;
  a.u = (float*)c.u; a.v = (float*)c.v; a.w = (float*)c.w;
  a.q = (const float*)c.q;
  a.start = c.start; a.count = c.count;
  a.iv_f = c.fbytes == 4 ? (const float*)c.invvol : nullptr;
  a.iv_d = c.fbytes == 8 ? (const double*)c.invvol : nullptr;
  a.acc = (long long*)c.acc;
  a.nx = (int)c.geo_i[0]; a.ny = (int)c.geo_i[1]; a.nz = (int)c.geo_i[2];
  a.NY = a.ny + 1; a.NZ = a.nz + 1; a.NN = (a.nx + 1) * a.NY * a.NZ;
  a.cny = a.nx * a.ny;
  for (int k = 0; k < 3; ++k) {
    const float o = (float)c.geo_f[3 + k], L = (float)c.geo_f[6 + k];
    const float hi = o + L;  // f32 sum, as the reference's single/mixed modes
    a.o[k] = o; a.L[k] = L; a.hi[k] = hi; a.hi2[k] = hi + hi;
    const double gd = (double)(c.fbytes == 8 ? c.geo_g[k] : (double)(float)c.geo_g[k]);
    const double go = (double)(c.fbytes == 8 ? c.geo_g[3 + k] : (double)(float)c.geo_g[3 + k]);
    a.idx[k] = (float)(1.0 / gd);
    a.ogs[k] = (float)(go / gd);
    a.bc_eps[k] = (float)(1e-5 * (fabs((double)o) + (double)L) + 1e-30);
  }
  a.dt = (float)c.dt; a.dth = (float)c.dth; a.qdt2m = (float)c.qdt2m;
  a.beta = (float)c.beta;
  a.beta2 = a.beta * a.beta;
  a.scale = c.scale;
  a.n_iters = c.n_iters;
  a.status = c.status;
  void* rec = const_cast<void*>(rec_in);
  const size_t rbytes = f32_records_bytes(c.geo_i);
  // one bit per particle, +2 words so a round's second tile may read past the end
  const size_t skip_bytes = (((size_t)c.count + 31) / 32 * 4 + 8 + 255) & ~(size_t)255;
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, 256 + skip_bytes + (rec ? 0 : rbytes), s);
  if (e != cudaSuccess) {
    set_error("f32 scratch alloc: %s", cudaGetErrorString(e));
    return -2;
  }
  a.work = (unsigned long long*)scratch;
  a.skip = (unsigned*)((char*)scratch + 256);
  cudaMemsetAsync(scratch, 0, 256 + skip_bytes, s);
  int rc = 0;
  if (!rec) {
    rec = (char*)scratch + 256 + skip_bytes;
    rc = f32_pack_records(c.fbytes, c.E, c.B, c.geo_i, rec, s);
  }
  a.rec = (const float4*)rec;
  a.emax = reinterpret_cast<const float*>((const char*)rec + (f32_records_bytes(c.geo_i) - 32));
  static int fusedk = -1;
  if (fusedk < 0) {
    const char* env = getenv("BP_F32_FUSED");
    fusedk = (env && env[0] == '1') ? 1 : 0;
  }
  if (!rc && fusedk) {
    // one-pass variant (dev comparison): mover + deposit in one kernel
    const int m = (c.geo_i[3] ? 1 : 0) | (c.geo_i[4] ? 2 : 0) | (c.geo_i[5] ? 4 : 0);
    if (m == 2) rc = launch_deposit_cfg<8, 512, 2, false, 1, true, false, true, false>(a, s);
    else if (m == 0) rc = launch_deposit_cfg<8, 512, 2, false, 1, true, false, false, false>(a, s);
    else { set_error("fused f32 variant: only P/R/P and periodic boxes"); rc = -1; }
    cudaFreeAsync(scratch, s);
    return rc;
  }
  if (!rc) {
    const int m = (c.geo_i[3] ? 1 : 0) | (c.geo_i[4] ? 2 : 0) | (c.geo_i[5] ? 4 : 0);
    switch (m) {
      case 0: rc = launch_mover<false, false, false>(a, s); break;
      case 1: rc = launch_mover<true, false, false>(a, s); break;
      case 2: rc = launch_mover<false, true, false>(a, s); break;
      case 3: rc = launch_mover<true, true, false>(a, s); break;
      case 4: rc = launch_mover<false, false, true>(a, s); break;
      case 5: rc = launch_mover<true, false, true>(a, s); break;
      case 6: rc = launch_mover<false, true, true>(a, s); break;
      default: rc = launch_mover<true, true, true>(a, s); break;
    }
  }
  if (!rc) rc = launch_deposit(a, s);
  cudaFreeAsync(scratch, s);
  return rc;
}

}  // namespace bp
