// Fused implicit mover + moment deposition, sm_100a.
//
// Semantics follow the reference batchpic kernels (pkg/src/batchpic/kernels.py):
//   push block   fused_span :489-682 (== push_span :112-306)
//   deposit      fused_span :683-734 (== deposit_span :327-381)
//   gather       gather_span :385-455
// Arithmetic contract ("parity" build, this header compiled with -fmad=false):
// numba's typing — every f32(op)f64 / f32(op)i64 is f64,
// f32(op)f32 stays f32, no FMA, IEEE division, rint half-even.  P is the
// particle storage type and F the field storage type.
//
// Layout in HBM (the reference data contract, unchanged):
//   particles  SoA x y z u v w q, one contiguous array each (P)
//   E, B       (3, nx+1, ny+1, nz+1) C order, k fastest (F)
//   acc        (10, nx+1, ny+1, nz+1) int64 fixed point (rho Jx Jy Jz Pxx Pxy
//              Pxz Pyy Pyz Pzz), quantum 2^-43 (fields.py:20-25)
//   invvol     (nx+1, ny+1, nz+1) (F)
//
// Deposition is exact integer arithmetic, so contributions may be summed in
// any grouping: per-cell sums are kept in registers spread over a warp and
// flushed with one REDG.ADD.64 per (node, moment) when the cell changes; the
// result is bit-identical to the reference's sequential `acc[...] += rint(...)`.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bp {

typedef long long i64;

// ST_DOMAIN: a deposit/gather position outside the box (the reference does
// not check; the GPU refuses to index out of bounds).
enum { ST_OK = 0, ST_RUNAWAY = 1, ST_MIDPOINT = 2, ST_DOMAIN = 3 };

// Raw geometry exactly as the reference packs it (make_geo_arrays,
// kernels.py:57-67): geo_f / geo_g = dx dy dz ox oy oz Lx Ly Lz, geo_i =
// nx ny nz bcx bcy bcz (bc 0 periodic, 1 reflecting).  Doubles hold the P/F
// values exactly.
struct RawGeo {
  double f[9];
  double g[9];
  i64 i[6];
};

template <typename P, typename F>
struct SpanParams {
  P *x, *y, *z, *u, *v, *w;
  const P* q;
  i64 start, count;
  const F* E;
  const F* B;
  i64* acc;
  const F* invvol;
  // boundary arithmetic (particle precision), hi = (P)(o + L), hi2 = (P)(hi + hi)
  P ox, oy, oz, Lx, Ly, Lz, hx, hy, hz, hx2, hy2, hz2;
  // cell location (field precision)
  F gdx, gdy, gdz, gox, goy, goz;
  int nx, ny, nz, bcx, bcy, bcz;
  int NY, NZ, NN;  // node extents (y, z) and node count
  P dt, dth, qdt2m, beta, one, two, beta2;
  F scale;
  // the same scalars widened to double once on the host (exact), so the
  // kernel never re-converts them per particle
  struct Wide {
    double o[3], L[3], hi[3], hi2[3], gd[3], go[3];
    double dt, dth, qdt2m, beta, one, two, beta2, scale;
  } d;
  int n_iters, mixed, apply_bc;
  int* status;
  P* gather_out;  // gather only: (count, 6)
  // Node-interleaved copy of E, B and invvol widened to double, 8 doubles
  // per node: Ex Ey Ez Bx By Bz invvol 0 (built by pack_nodes per call).
  const double* fnode;
};

// E, B, invvol -> one 64-byte record per node (exact widening to double), so a
// corner of the gather is three 16-byte loads from one record.
template <typename F>
__global__ void pack_nodes(const F* __restrict__ E, const F* __restrict__ B,
                           const F* __restrict__ invvol, int NN, double* __restrict__ out) {
  const int stride = gridDim.x * blockDim.x;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < NN; n += stride) {
    double4 lo, hi;
    lo.x = E ? (double)E[n] : 0.0;
    lo.y = E ? (double)E[NN + n] : 0.0;
    lo.z = E ? (double)E[2 * NN + n] : 0.0;
    lo.w = B ? (double)B[n] : 0.0;
    hi.x = B ? (double)B[NN + n] : 0.0;
    hi.y = B ? (double)B[2 * NN + n] : 0.0;
    hi.z = invvol ? (double)invvol[n] : 0.0;
    hi.w = 0.0;
    reinterpret_cast<double4*>(out)[2 * n] = lo;
    reinterpret_cast<double4*>(out)[2 * n + 1] = hi;
  }
}

__device__ __forceinline__ unsigned lane_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

// midpoint fold, kernels.py:505-534
// o, L, hi = (P)(o+L), hi2 = (P)(hi+hi) are particle-precision values widened
__device__ __forceinline__ double fold_mid(double xm, double o, double L, double hi,
                                           double hi2, int bc) {
  if (bc == 0) {
    if (xm < o) xm = xm + L;
    else if (xm > hi) xm = xm - L;
  } else {
    if (xm < o) xm = o + (o - xm);
    else if (xm > hi) xm = hi2 - xm;
  }
  return xm;
}

// commit boundary, kernels.py:629-671
__device__ __forceinline__ void fold_commit(double& q, double& vel, double o, double L,
                                            double hi, double hi2, int bc) {
  if (bc == 0) {
    if (q < o) {
      q = q + L;
      if (q >= hi) q = o;
    } else if (q >= hi) {
      q = q - L;
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

template <typename F>
__device__ __forceinline__ double ldf(const F* p) {
  return (double)__ldg(p);
}

// 6-component trilinear gather, left-to-right corner order (kernels.py:568-591)
template <typename P, typename F>
__device__ __forceinline__ void gather6(const SpanParams<P, F>& a, int n000, const double w[8],
                                        double out[6]) {
  const int sx = a.NY * a.NZ, sy = a.NZ;
  const int off[8] = {0, sx, sy, sx + sy, 1, sx + 1, sy + 1, sx + sy + 1};
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const F* A = (c < 3 ? a.E : a.B) + (size_t)(c % 3) * a.NN + n000;
    double s = w[0] * ldf(A + off[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) s = s + w[k] * ldf(A + off[k]);
    out[c] = s;
  }
}

// Same gather from the packed node records.  The first corner initialises
// the sum (0.0 + w*F would turn a -0.0 product into +0.0).
__device__ __forceinline__ void gather_packed(const double* __restrict__ fn, int n000, int sx,
                                              int sy, const double w[8], double s[6]) {
  const int off[8] = {0, sx, sy, sx + sy, 1, sx + 1, sy + 1, sx + sy + 1};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2* r = reinterpret_cast<const double2*>(fn + (size_t)(n000 + off[k]) * 8);
    const double2 a0 = __ldg(r), a1 = __ldg(r + 1), a2 = __ldg(r + 2);
    if (k == 0) {
      s[0] = w[0] * a0.x; s[1] = w[0] * a0.y; s[2] = w[0] * a1.x;
      s[3] = w[0] * a1.y; s[4] = w[0] * a2.x; s[5] = w[0] * a2.y;
    } else {
      s[0] = s[0] + w[k] * a0.x; s[1] = s[1] + w[k] * a0.y; s[2] = s[2] + w[k] * a1.x;
      s[3] = s[3] + w[k] * a1.y; s[4] = s[4] + w[k] * a2.x; s[5] = s[5] + w[k] * a2.y;
    }
  }
}

__device__ __forceinline__ void weights8(double fx, double fy, double fz, double ax, double ay,
                                         double az, double w[8]) {
  w[0] = ax * ay * az; w[1] = fx * ay * az; w[2] = ax * fy * az; w[3] = fx * fy * az;
  w[4] = ax * ay * fz; w[5] = fx * ay * fz; w[6] = ax * fy * fz; w[7] = fx * fy * fz;
}

// Push block for one particle.  On ST_OK, xo..wo hold the committed state in
// double (already exactly representable after the caller rounds to P).
template <typename P, typename F>
__device__ __forceinline__ int push_one(const SpanParams<P, F>& a, P xp, P yp, P zp, P vnx,
                                        P vny, P vnz, double& xo, double& yo, double& zo,
                                        double& uo, double& vo, double& wo) {
  const auto& d = a.d;
  double vbx = (double)vnx, vby = (double)vny, vbz = (double)vnz;
  for (int it = 0; it < a.n_iters; ++it) {
    double xm = (double)xp + vbx * d.dth;
    double ym = (double)yp + vby * d.dth;
    double zm = (double)zp + vbz * d.dth;
    xm = fold_mid(xm, d.o[0], d.L[0], d.hi[0], d.hi2[0], a.bcx);
    ym = fold_mid(ym, d.o[1], d.L[1], d.hi[1], d.hi2[1], a.bcy);
    zm = fold_mid(zm, d.o[2], d.L[2], d.hi[2], d.hi2[2], a.bcz);
    if (xm < d.o[0] || xm > d.hi[0] || ym < d.o[1] || ym > d.hi[1] || zm < d.o[2] ||
        zm > d.hi[2])
      return ST_MIDPOINT;
    const double gx = (xm - d.go[0]) / d.gd[0];
    const double gy = (ym - d.go[1]) / d.gd[1];
    const double gz = (zm - d.go[2]) / d.gd[2];
    int i = (int)(i64)gx, j = (int)(i64)gy, k = (int)(i64)gz;
    if (i > a.nx - 1) i = a.nx - 1;
    if (j > a.ny - 1) j = a.ny - 1;
    if (k > a.nz - 1) k = a.nz - 1;
    const double fx = gx - (double)i, fy = gy - (double)j, fz = gz - (double)k;
    const double ax = d.one - fx, ay = d.one - fy, az = d.one - fz;
    double w[8];
    weights8(fx, fy, fz, ax, ay, az, w);
    double s[6];
    gather_packed(a.fnode, (i * a.NY + j) * a.NZ + k, a.NY * a.NZ, a.NZ, w, s);
    double tx, ty, tz, hx, hy, hz;
    if (a.mixed) {
      // sample rounded once to P, t = v + qdt2m*sample in P (kernels.py:592-604)
      const P sx = (P)s[0], sy = (P)s[1], sz = (P)s[2];
      tx = (double)(P)(vnx + (P)(a.qdt2m * sx));
      ty = (double)(P)(vny + (P)(a.qdt2m * sy));
      tz = (double)(P)(vnz + (P)(a.qdt2m * sz));
      hx = (double)(P)s[3]; hy = (double)(P)s[4]; hz = (double)(P)s[5];
    } else {
      tx = (double)vnx + d.qdt2m * s[0];
      ty = (double)vny + d.qdt2m * s[1];
      tz = (double)vnz + d.qdt2m * s[2];
      hx = s[3]; hy = s[4]; hz = s[5];
    }
    // rotation, kernels.py:606-617; beta*beta was formed in P on the host
    const double bsq = hx * hx + hy * hy + hz * hz;
    const double denom = d.one + d.beta2 * bsq;
    const double tdb = tx * hx + ty * hy + tz * hz;
    const double be = d.beta;
    vbx = (tx + be * ((ty * hz - tz * hy) + be * tdb * hx)) / denom;
    vby = (ty + be * ((tz * hx - tx * hz) + be * tdb * hy)) / denom;
    vbz = (tz + be * ((tx * hy - ty * hx) + be * tdb * hz)) / denom;
  }
  // commit, kernels.py:622-628
  xo = (double)xp + vbx * d.dt;
  yo = (double)yp + vby * d.dt;
  zo = (double)zp + vbz * d.dt;
  uo = d.two * vbx - (double)vnx;
  vo = d.two * vby - (double)vny;
  wo = d.two * vbz - (double)vnz;
  if (a.apply_bc) {
    fold_commit(xo, uo, d.o[0], d.L[0], d.hi[0], d.hi2[0], a.bcx);
    fold_commit(yo, vo, d.o[1], d.L[1], d.hi[1], d.hi2[1], a.bcy);
    fold_commit(zo, wo, d.o[2], d.L[2], d.hi[2], d.hi2[2], a.bcz);
    if (xo < d.o[0] || xo > d.hi[0] || yo < d.o[1] || yo > d.hi[1] || zo < d.o[2] ||
        zo > d.hi[2])
      return ST_RUNAWAY;
  }
  return ST_OK;
}

// Cell + weights of the deposit block; gx in promote(P, F) (f32 only when
// both are f32 — the reloaded f32 position against f32 geometry).
template <typename P, typename F>
__device__ __forceinline__ int deposit_cell(const SpanParams<P, F>& a, P xp, P yp, P zp,
                                            double& fx, double& fy, double& fz) {
  typedef decltype(P() - F()) G;
  const G gx = ((G)xp - (G)a.gox) / (G)a.gdx;
  const G gy = ((G)yp - (G)a.goy) / (G)a.gdy;
  const G gz = ((G)zp - (G)a.goz) / (G)a.gdz;
  if (!(gx >= (G)0 && gy >= (G)0 && gz >= (G)0 && gx < (G)2147483647 && gy < (G)2147483647 &&
        gz < (G)2147483647))
    return -1;  // outside the box or NaN
  int i = (int)(i64)gx, j = (int)(i64)gy, k = (int)(i64)gz;
  if (i > a.nx - 1) i = a.nx - 1;
  if (j > a.ny - 1) j = a.ny - 1;
  if (k > a.nz - 1) k = a.nz - 1;
  fx = (double)gx - (double)i;
  fy = (double)gy - (double)j;
  fz = (double)gz - (double)k;
  return (i * a.NY + j) * a.NZ + k;
}

// --------------------------------------------------------------------------
// Deposition.  Contribution (moment m, corner c) of one particle is
//   rint((base_c * m) * scale),  base_c = (q * (wx*wy*wz)) * invvol_c
// (kernels.py:707-734), m in {1, u, v, w, uu, uv, uw, vv, vw, ww} with the
// dyads formed in particle precision.  With scale a power of two,
// (base*m)*scale == (base*scale)*m exactly, so bases are pre-scaled once per
// particle (PRESCALE); otherwise the reference expression is evaluated as is.
//
// Accumulation is exact int64, so any grouping gives the reference's bits.
// Each warp walks a contiguous run of (cell-sorted) particles; the 80 sums
// of the cell currently being filled live in registers spread over the 32
// lanes: lane L owns corner c = L & 7 of moments g, g+4, g+8 (g = L >> 3).
// Per particle the owning lane stages its 8 bases and 10 moment values in
// shared memory, then all lanes fold that particle into their 2-3
// accumulators — no cross-lane reduction at all.  A second slot keeps the
// sums of the last "stray" cell, so a particle that crossed into a
// neighbour cell does not force a flush of the main cell.  Sums are flushed
// with one REDG.ADD.64 per (slot, value) when a slot is evicted.

__device__ __forceinline__ void red_add(i64* p, i64 v) {
  if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// shared-memory staging of one warp (doubles): bases [32][8] and moments
// [32][4][4] laid out so lane group g reads (m_g, m_g+4) with one 16-byte
// load and m_g+8 (zero for g >= 2) with a second
constexpr int kStageBs = 32 * 8;
constexpr int kStageMv = 32 * 16;
constexpr int kWarpStage = kStageBs + kStageMv + 16;  // + 32 int keys

// Exact rint without the conversion pipe: for |t| < 2^51, t + 1.5*2^52 lands
// in [2^52, 2^53) where the ulp is 1, so the FP add rounds t half-to-even
// exactly like cvt.rni and the low mantissa bits hold rint(t) in two's
// complement: bits(t + M) = bits(M) + rint(t).  Slots accumulate raw bit
// patterns and subtract n * bits(M) when flushed.  Tiles whose values could
// leave the range take the cvt path instead (checked per particle).
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr i64 kMagicBits = 0x4338000000000000LL;
constexpr double kMagicLimit = 1125899906842624.0;  // 2^50

typedef unsigned long long u64;  // modular sums of biased bit patterns

struct Slot {
  int key;
  int n;  // folded particles since the last flush (bit-pattern bias count)
  u64 s0, s1, s2;
};

__device__ __forceinline__ void slot_flush(const Slot& sl, i64* __restrict__ acc, int NN,
                                           int m0, int coff, bool third) {
  if (sl.key < 0) return;
  const u64 bias = (u64)sl.n * (u64)kMagicBits;
  i64* p = acc + (size_t)m0 * NN + sl.key + coff;
  red_add(p, (i64)(sl.s0 - bias));
  red_add(p + (size_t)4 * NN, (i64)(sl.s1 - bias));
  if (third) red_add(p + (size_t)8 * NN, (i64)(sl.s2 - bias));
}


// Fold staged particle k into a slot: this lane's corner lc of moments
// lg, lg+4, lg+8.
// quantised value as a biased bit pattern: bits(M) + rint(t)
template <bool PRESCALE, bool MAGIC>
__device__ __forceinline__ u64 qbits(double b, double m, double sc) {
  const double t = PRESCALE ? b * m : b * m * sc;
  return MAGIC ? (u64)__double_as_longlong(t + kMagic)
               : (u64)__double2ll_rn(t) + (u64)kMagicBits;
}

template <bool PRESCALE, bool MAGIC>
__device__ __forceinline__ void fold_vals(u64& s0, u64& s1, u64& s2, const double* st_bs,
                                          const double* st_mv, int k, int lc, int lg,
                                          double sc) {
  const double b = st_bs[k * 8 + lc];
  const double2 m01 = *reinterpret_cast<const double2*>(st_mv + k * 16 + lg * 4);
  const double m2 = st_mv[k * 16 + lg * 4 + 2];
  s0 += qbits<PRESCALE, MAGIC>(b, m01.x, sc);
  s1 += qbits<PRESCALE, MAGIC>(b, m01.y, sc);
  s2 += qbits<PRESCALE, MAGIC>(b, m2, sc);  // m2 == 0 for lane groups 2, 3
}

template <bool PRESCALE, bool MAGIC>
__device__ __forceinline__ void fold_one(Slot& S, const double* st_bs, const double* st_mv,
                                         int k, int lc, int lg, double sc) {
  fold_vals<PRESCALE, MAGIC>(S.s0, S.s1, S.s2, st_bs, st_mv, k, lc, lg, sc);
  S.n += 1;
}

// all 32 staged particles into S, two interleaved chains
template <bool PRESCALE, bool MAGIC>
__device__ __forceinline__ void fold_tile(Slot& S, const double* st_bs, const double* st_mv,
                                          int lc, int lg, double sc) {
  u64 t0 = 0, t1 = 0, t2 = 0;
#pragma unroll 8
  for (int k = 0; k < 32; k += 2) {
    fold_vals<PRESCALE, MAGIC>(S.s0, S.s1, S.s2, st_bs, st_mv, k, lc, lg, sc);
    fold_vals<PRESCALE, MAGIC>(t0, t1, t2, st_bs, st_mv, k + 1, lc, lg, sc);
  }
  S.s0 += t0; S.s1 += t1; S.s2 += t2;
  S.n += 32;
}

// One kernel body for fused / push-only / deposit-only.  Each warp owns a
// contiguous run of the span and walks it 32 particles at a time (coalesced
// SoA loads/stores); every lane of a warp runs the same trip count so warp
// collectives always see 32 lanes.
template <typename P, typename F, bool DO_PUSH, bool DO_DEPOSIT, bool PRESCALE>
__global__ void __launch_bounds__(256, 2) span_kernel(SpanParams<P, F> a) {
  extern __shared__ double stage_all[];
  const unsigned lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const i64 nwarps = (i64)gridDim.x * (blockDim.x >> 5);
  const i64 gw = (i64)blockIdx.x * (blockDim.x >> 5) + wib;
  const i64 per = ((a.count + nwarps - 1) / nwarps + 31) & ~(i64)31;
  const i64 w0 = gw * per;
  const i64 w1 = w0 + per < a.count ? w0 + per : a.count;
  double* const st_bs = stage_all + (size_t)wib * kWarpStage;
  double* const st_mv = st_bs + kStageBs;
  int* const st_key = reinterpret_cast<int*>(st_mv + kStageMv);
  const int sx = a.NY * a.NZ, sy = a.NZ;
  // this lane's share of the 80 sums
  const int lc = lane & 7, lg = lane >> 3;
  const int coff = (lc & 1) * sx + ((lc >> 1) & 1) * sy + ((lc >> 2) & 1);
  const bool third = lg < 2;
  const double sc = a.d.scale;
  Slot A{-1, 0, 0, 0, 0}, Bs{-1, 0, 0, 0, 0};
  int worst = ST_OK;
  for (i64 t0 = w0; t0 < w1; t0 += 32) {
    const i64 r = t0 + lane;
    bool valid = r < w1;
    const i64 p = a.start + r;
    P xp = 0, yp = 0, zp = 0, un = 0, vn = 0, wn = 0, qp = 0;
    if (valid) {
      xp = a.x[p]; yp = a.y[p]; zp = a.z[p];
      un = a.u[p]; vn = a.v[p]; wn = a.w[p];
      if (DO_DEPOSIT) qp = a.q[p];
    }
    if (DO_PUSH && valid) {
      double xo, yo, zo, uo, vo, wo;
      const int st = push_one<P, F>(a, xp, yp, zp, un, vn, wn, xo, yo, zo, uo, vo, wo);
      if (st != ST_OK) {
        worst = st > worst ? st : worst;
        valid = false;
      } else {
        xp = (P)xo; yp = (P)yo; zp = (P)zo;
        un = (P)uo; vn = (P)vo; wn = (P)wo;
        a.x[p] = xp; a.y[p] = yp; a.z[p] = zp;
        a.u[p] = un; a.v[p] = vn; a.w[p] = wn;
      }
    }
    if (DO_DEPOSIT) {
      // ---- owner lane: cell, 8 bases, 10 moment values -> shared memory
      double fx = 0, fy = 0, fz = 0;
      int n000 = -1;
      bool big = false;
      if (valid) {
        n000 = deposit_cell<P, F>(a, xp, yp, zp, fx, fy, fz);
        if (n000 < 0) worst = ST_DOMAIN > worst ? ST_DOMAIN : worst;
      }
      {
        // invalid particles stage zero bases: folding them adds exact zeros
        const double q = n000 >= 0 ? (double)qp : 0.0;
        const int nb = n000 >= 0 ? n000 : 0;
        const double ax = a.d.one - fx, ay = a.d.one - fy, az = a.d.one - fz;
        const int off[8] = {0, sx, sy, sx + sy, 1, sx + 1, sy + 1, sx + sy + 1};
        double bs[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double wx = (c & 1) ? fx : ax, wy = (c & 2) ? fy : ay, wz = (c & 4) ? fz : az;
          const double iv = __ldg(a.fnode + (size_t)(nb + off[c]) * 8 + 6);
          const double base = q * (wx * wy * wz) * iv;
          bs[c] = PRESCALE ? base * sc : base;
        }
        double2* b2 = reinterpret_cast<double2*>(st_bs + lane * 8);
#pragma unroll
        for (int c = 0; c < 4; ++c) b2[c] = make_double2(bs[2 * c], bs[2 * c + 1]);
        const P pxx = un * un, pxy = un * vn, pxz = un * wn;
        const P pyy = vn * vn, pyz = vn * wn, pzz = wn * wn;
        {
          // |value| < 2^50 for every (corner, moment) keeps the magic rint exact
          double mb = 0.0;
#pragma unroll
          for (int c = 0; c < 8; ++c) mb = fmax(mb, fabs(bs[c]));
          double mm = fmax(1.0, fmax(fabs((double)un), fmax(fabs((double)vn), fabs((double)wn))));
          mm = fmax(mm, fmax(fabs((double)pxx), fmax(fabs((double)pyy), fabs((double)pzz))));
          const double lim = PRESCALE ? kMagicLimit : kMagicLimit / sc;
          big = n000 >= 0 && !(mb * mm < lim);
        }
        // moments m0..m9 = 1 u v w uu uv uw vv vw ww, grouped (g, g+4, g+8)
        double2* m2 = reinterpret_cast<double2*>(st_mv + lane * 16);
        m2[0] = make_double2(1.0, (double)pxx);
        m2[1] = make_double2((double)pyz, 0.0);
        m2[2] = make_double2((double)un, (double)pxy);
        m2[3] = make_double2((double)pzz, 0.0);
        m2[4] = make_double2((double)vn, (double)pxz);
        m2[5] = make_double2(0.0, 0.0);
        m2[6] = make_double2((double)wn, (double)pyy);
        m2[7] = make_double2(0.0, 0.0);
      }
      st_key[lane] = n000;
      __syncwarp();
      // ---- all lanes: fold the 32 staged particles into the slot sums.
      // Lanes are grouped by cell with ballots: the group of the main slot's
      // cell (usually almost the whole warp) and, one by one, the few other
      // cells present (particles that crossed into a neighbour cell, or the
      // next cell of the sort) which go through the stray slot.
      const bool has = n000 >= 0;
      const unsigned V = __ballot_sync(0xffffffffu, has);
      const bool magic = __ballot_sync(0xffffffffu, big) == 0u;
      if (V) {
        unsigned MA = __ballot_sync(0xffffffffu, has && n000 == A.key);
        if (MA == 0u) {
          const int knew = __shfl_sync(0xffffffffu, n000, __ffs(V) - 1);
          if (knew == Bs.key) {
            const Slot t = A;
            A = Bs;
            Bs = t;
          } else {
            slot_flush(Bs, a.acc, a.NN, lg, coff, third);
            Bs = A;
            A.key = knew;
            A.n = 0;
            A.s0 = A.s1 = A.s2 = 0;
          }
          MA = __ballot_sync(0xffffffffu, has && n000 == A.key);
        }
        const unsigned strays = V & ~MA;
        unsigned rest = strays;
        while (rest) {
          const int k2 = __shfl_sync(0xffffffffu, n000, __ffs(rest) - 1);
          const unsigned M2 = __ballot_sync(0xffffffffu, has && n000 == k2);
          rest &= ~M2;
          if (k2 != Bs.key) {
            slot_flush(Bs, a.acc, a.NN, lg, coff, third);
            Bs.key = k2;
            Bs.n = 0;
            Bs.s0 = Bs.s1 = Bs.s2 = 0;
          }
          if (magic) {
            for (unsigned m = M2; m; m &= m - 1u)
              fold_one<PRESCALE, true>(Bs, st_bs, st_mv, __ffs(m) - 1, lc, lg, sc);
          } else {
            for (unsigned m = M2; m; m &= m - 1u)
              fold_one<PRESCALE, false>(Bs, st_bs, st_mv, __ffs(m) - 1, lc, lg, sc);
          }
        }
        if (strays) {
          // folded already: neutralise their bases for the unmasked main fold
          if ((strays >> lane) & 1u) {
            double2* b2 = reinterpret_cast<double2*>(st_bs + lane * 8);
#pragma unroll
            for (int c = 0; c < 4; ++c) b2[c] = make_double2(0.0, 0.0);
          }
          __syncwarp();
        }
        // invalid lanes staged zero bases, so the whole tile folds unmasked
        if (magic)
          fold_tile<PRESCALE, true>(A, st_bs, st_mv, lc, lg, sc);
        else
          fold_tile<PRESCALE, false>(A, st_bs, st_mv, lc, lg, sc);
      }
      __syncwarp();
    }
  }
  if (DO_DEPOSIT) {
    slot_flush(A, a.acc, a.NN, lg, coff, third);
    slot_flush(Bs, a.acc, a.NN, lg, coff, third);
  }
  if (worst != ST_OK) atomicMax(a.status, worst);
}

template <typename P, typename F>
__global__ void __launch_bounds__(256) gather_kernel(SpanParams<P, F> a) {
  const i64 nthreads = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < a.count; r += nthreads) {
    const i64 p = a.start + r;
    double fx, fy, fz;
    const int n000 = deposit_cell<P, F>(a, a.x[p], a.y[p], a.z[p], fx, fy, fz);
    if (n000 < 0) {
#pragma unroll
      for (int c = 0; c < 6; ++c) a.gather_out[r * 6 + c] = (P)0;
      atomicMax(a.status, (int)ST_DOMAIN);
      continue;
    }
    const double ax = 1.0 - fx, ay = 1.0 - fy, az = 1.0 - fz;
    double w[8];
    weights8(fx, fy, fz, ax, ay, az, w);
    double s[6];
    gather6(a, n000, w, s);
#pragma unroll
    for (int c = 0; c < 6; ++c) a.gather_out[r * 6 + c] = (P)s[c];
  }
}

}  // namespace bp
