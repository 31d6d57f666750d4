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
// Deposition is exact integer arithmetic, so contributions may be reduced in
// any order: lanes of a warp that share a cell are summed with a transposed
// shuffle reduction before one REDG.ADD.64 per (node, moment); the result is
// bit-identical to the reference's sequential `acc[...] += rint(...)`.
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
  int n_iters, mixed, apply_bc;
  int* status;
  P* gather_out;  // gather only: (count, 6)
};

__device__ __forceinline__ unsigned lane_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

// midpoint fold, kernels.py:505-534
template <typename P>
__device__ __forceinline__ double fold_mid(double xm, P o, P L, P hi, P hi2, int bc) {
  if (bc == 0) {
    if (xm < (double)o) xm = xm + (double)L;
    else if (xm > (double)hi) xm = xm - (double)L;
  } else {
    if (xm < (double)o) xm = (double)o + ((double)o - xm);
    else if (xm > (double)hi) xm = (double)hi2 - xm;
  }
  return xm;
}

// commit boundary, kernels.py:629-671
template <typename P>
__device__ __forceinline__ void fold_commit(double& q, double& vel, P o, P L, P hi, P hi2,
                                            int bc) {
  if (bc == 0) {
    if (q < (double)o) {
      q = q + (double)L;
      if (q >= (double)hi) q = (double)o;
    } else if (q >= (double)hi) {
      q = q - (double)L;
    }
  } else {
    if (q < (double)o) {
      q = (double)o + ((double)o - q);
      vel = -vel;
    } else if (q > (double)hi) {
      q = (double)hi2 - q;
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
  double vbx = (double)vnx, vby = (double)vny, vbz = (double)vnz;
  for (int it = 0; it < a.n_iters; ++it) {
    double xm = (double)xp + vbx * (double)a.dth;
    double ym = (double)yp + vby * (double)a.dth;
    double zm = (double)zp + vbz * (double)a.dth;
    xm = fold_mid<P>(xm, a.ox, a.Lx, a.hx, a.hx2, a.bcx);
    ym = fold_mid<P>(ym, a.oy, a.Ly, a.hy, a.hy2, a.bcy);
    zm = fold_mid<P>(zm, a.oz, a.Lz, a.hz, a.hz2, a.bcz);
    if (xm < (double)a.ox || xm > (double)a.hx || ym < (double)a.oy || ym > (double)a.hy ||
        zm < (double)a.oz || zm > (double)a.hz)
      return ST_MIDPOINT;
    const double gx = (xm - (double)a.gox) / (double)a.gdx;
    const double gy = (ym - (double)a.goy) / (double)a.gdy;
    const double gz = (zm - (double)a.goz) / (double)a.gdz;
    int i = (int)(i64)gx, j = (int)(i64)gy, k = (int)(i64)gz;
    if (i > a.nx - 1) i = a.nx - 1;
    if (j > a.ny - 1) j = a.ny - 1;
    if (k > a.nz - 1) k = a.nz - 1;
    const double fx = gx - (double)i, fy = gy - (double)j, fz = gz - (double)k;
    const double ax = (double)a.one - fx, ay = (double)a.one - fy, az = (double)a.one - fz;
    double w[8];
    weights8(fx, fy, fz, ax, ay, az, w);
    double s[6];
    gather6(a, (i * a.NY + j) * a.NZ + k, w, s);
    double tx, ty, tz, hx, hy, hz;
    if (a.mixed) {
      const P sx = (P)s[0], sy = (P)s[1], sz = (P)s[2];
      tx = (double)(P)(vnx + (P)(a.qdt2m * sx));
      ty = (double)(P)(vny + (P)(a.qdt2m * sy));
      tz = (double)(P)(vnz + (P)(a.qdt2m * sz));
      hx = (double)(P)s[3]; hy = (double)(P)s[4]; hz = (double)(P)s[5];
    } else {
      tx = (double)vnx + (double)a.qdt2m * s[0];
      ty = (double)vny + (double)a.qdt2m * s[1];
      tz = (double)vnz + (double)a.qdt2m * s[2];
      hx = s[3]; hy = s[4]; hz = s[5];
    }
    const double bsq = hx * hx + hy * hy + hz * hz;
    const double denom = (double)a.one + (double)a.beta2 * bsq;
    const double tdb = tx * hx + ty * hy + tz * hz;
    const double be = (double)a.beta;
    vbx = (tx + be * ((ty * hz - tz * hy) + be * tdb * hx)) / denom;
    vby = (ty + be * ((tz * hx - tx * hz) + be * tdb * hy)) / denom;
    vbz = (tz + be * ((tx * hy - ty * hx) + be * tdb * hz)) / denom;
  }
  xo = (double)xp + vbx * (double)a.dt;
  yo = (double)yp + vby * (double)a.dt;
  zo = (double)zp + vbz * (double)a.dt;
  uo = (double)a.two * vbx - (double)vnx;
  vo = (double)a.two * vby - (double)vny;
  wo = (double)a.two * vbz - (double)vnz;
  if (a.apply_bc) {
    fold_commit<P>(xo, uo, a.ox, a.Lx, a.hx, a.hx2, a.bcx);
    fold_commit<P>(yo, vo, a.oy, a.Ly, a.hy, a.hy2, a.bcy);
    fold_commit<P>(zo, wo, a.oz, a.Lz, a.hz, a.hz2, a.bcz);
    if (xo < (double)a.ox || xo > (double)a.hx || yo < (double)a.oy || yo > (double)a.hy ||
        zo < (double)a.oz || zo > (double)a.hz)
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
// Per-particle deposit inputs; contribution idx = corner*10 + moment is
// rint(q*(wx*wy*wz)*invvol * m * scale) in the reference's expression order
// ((base*m)*scale, kernels.py:707-734).
template <typename P>
struct DepIn {
  double fx, fy, fz, ax, ay, az, q;
  P u, v, w, pxx, pxy, pxz, pyy, pyz, pzz;
  double iv[8];
};

template <typename P, typename F>
__device__ __forceinline__ void dep_inputs(const SpanParams<P, F>& a, bool valid, int n000,
                                           double fx, double fy, double fz, P vnx, P vny,
                                           P vnz, P q, DepIn<P>& d) {
  d.fx = fx; d.fy = fy; d.fz = fz;
  d.ax = (double)a.one - fx; d.ay = (double)a.one - fy; d.az = (double)a.one - fz;
  d.q = (double)q;
  d.u = vnx; d.v = vny; d.w = vnz;
  d.pxx = vnx * vnx; d.pxy = vnx * vny; d.pxz = vnx * vnz;
  d.pyy = vny * vny; d.pyz = vny * vnz; d.pzz = vnz * vnz;
  const int sx = a.NY * a.NZ, sy = a.NZ;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int ci = c & 1, cj = (c >> 1) & 1, ck = (c >> 2) & 1;
    d.iv[c] = valid ? ldf(a.invvol + n000 + ci * sx + cj * sy + ck) : 0.0;
  }
}

template <typename P>
__device__ __forceinline__ i64 contrib(const DepIn<P>& d, double sc, int idx) {
  const int c = idx / 10, m = idx % 10;
  const int ci = c & 1, cj = (c >> 1) & 1, ck = (c >> 2) & 1;
  const double wx = ci ? d.fx : d.ax, wy = cj ? d.fy : d.ay, wz = ck ? d.fz : d.az;
  const double base = d.q * (wx * wy * wz) * d.iv[c];
  double mv;
  switch (m) {
    case 0: return __double2ll_rn(base * sc);
    case 1: mv = (double)d.u; break;
    case 2: mv = (double)d.v; break;
    case 3: mv = (double)d.w; break;
    case 4: mv = (double)d.pxx; break;
    case 5: mv = (double)d.pxy; break;
    case 6: mv = (double)d.pxz; break;
    case 7: mv = (double)d.pyy; break;
    case 8: mv = (double)d.pyz; break;
    default: mv = (double)d.pzz; break;
  }
  return __double2ll_rn(base * mv * sc);
}

__device__ __forceinline__ void red_add(i64* p, i64 v) {
  if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

__device__ __forceinline__ i64* acc_addr(i64* acc, int NN, int n000, int sx, int sy, int idx) {
  const int c = idx / 10, m = idx - 10 * (idx / 10);
  const int ci = c & 1, cj = (c >> 1) & 1, ck = (c >> 2) & 1;
  return acc + (size_t)m * NN + n000 + ci * sx + cj * sy + ck;
}

// Shared-memory scratch of one warp: 32 contributions x 32 lanes, row
// stride 33 (conflict-free column reads).
constexpr int kWarpScratch = 32 * 33;

// Exact warp-segmented deposit.  Each lane stages a chunk of its 80 int64
// contributions in shared memory; lane L then walks the 32 source lanes in
// order and sums contribution L over every run of lanes sharing a cell
// (particles are cell-sorted, so a warp holds one or two runs), issuing one
// REDG.ADD.64 per (run, contribution).  Unsorted input degenerates to one
// atomic per contribution.  Integer sums make the result order-free.
template <typename P>
__device__ __forceinline__ void warp_deposit(i64* acc, int NN, int sx, int sy, bool valid,
                                             int n000, const DepIn<P>& d, double sc,
                                             i64* sv) {
  const unsigned lane = lane_id();
  const int key = valid ? n000 : -1;
  const int prev = __shfl_up_sync(0xffffffffu, key, 1);
  const unsigned brk = __ballot_sync(0xffffffffu, lane == 0 || key != prev);
  if (__ballot_sync(0xffffffffu, valid) == 0) return;
#pragma unroll
  for (int chunk = 0; chunk < 3; ++chunk) {
    const int nv = chunk < 2 ? 32 : 16;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < nv; ++i) sv[i * 33 + lane] = valid ? contrib(d, sc, chunk * 32 + i) : 0;
    __syncwarp();
    int cur = __shfl_sync(0xffffffffu, key, 0);
    i64 sum = 0;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      if (k > 0 && ((brk >> k) & 1u)) {
        if (cur >= 0 && lane < nv) red_add(acc_addr(acc, NN, cur, sx, sy, chunk * 32 + lane), sum);
        cur = __shfl_sync(0xffffffffu, key, k);
        sum = 0;
      }
      if (lane < nv) sum += sv[lane * 33 + k];
    }
    if (cur >= 0 && lane < nv) red_add(acc_addr(acc, NN, cur, sx, sy, chunk * 32 + lane), sum);
  }
}

// --------------------------------------------------------------------------
// One kernel body for fused / push-only / deposit-only.  Every warp iterates
// the same number of times so warp collectives see all 32 lanes.
template <typename P, typename F, bool DO_PUSH, bool DO_DEPOSIT>
__global__ void __launch_bounds__(256) span_kernel(SpanParams<P, F> a) {
  extern __shared__ i64 sv[];
  const i64 nthreads = (i64)gridDim.x * blockDim.x;
  const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 warp_base = tid - lane_id();
  int worst = ST_OK;
  for (i64 wb = warp_base; wb < a.count; wb += nthreads) {
    const i64 r = wb + lane_id();
    bool valid = r < a.count;
    const i64 p = a.start + r;
    P xp = 0, yp = 0, zp = 0, un = 0, vn = 0, wn = 0;
    if (valid) {
      xp = a.x[p]; yp = a.y[p]; zp = a.z[p];
      un = a.u[p]; vn = a.v[p]; wn = a.w[p];
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
      double fx = 0, fy = 0, fz = 0;
      int n000 = 0;
      P q = 0;
      if (valid) {
        n000 = deposit_cell<P, F>(a, xp, yp, zp, fx, fy, fz);
        if (n000 < 0) {
          worst = ST_DOMAIN > worst ? ST_DOMAIN : worst;
          valid = false;
          n000 = 0;
        } else {
          q = a.q[p];
        }
      }
      DepIn<P> d;
      dep_inputs<P, F>(a, valid, n000, fx, fy, fz, un, vn, wn, q, d);
      warp_deposit<P>(a.acc, a.NN, a.NY * a.NZ, a.NZ, valid, n000, d, (double)a.scale,
                      sv + (threadIdx.x >> 5) * kWarpScratch);
    }
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
