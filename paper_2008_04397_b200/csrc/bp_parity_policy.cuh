// Parity arithmetic: bit for bit the reference numba kernels.
//
// Compile with -fmad=false (no contraction) and IEEE division.  numba's
// typing (pinned by the golden vectors of
// tests/golden/make_golden.py): every f32(op)f64 and f32(op)i64 is f64,
// f32(op)f32 stays f32, rint is half-to-even.  Concretely, in "single" and
// "mixed" modes the midpoint, cell, weights, gather sums and rotation are f64
// arithmetic on f32-stored values; ox+Lx, (ox+Lx)+(ox+Lx), beta*beta, the
// mixed-mode t = v + qdt2m*sample and the pressure dyads are f32; the deposit
// cell index in "single" is computed in f32 (reloaded f32 position against
// f32 geometry).
#pragma once
#include "bp_common.cuh"

namespace bp {

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

// commit boundary, kernels.py:629-671 (`>=` wrap with snap-to-origin)
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

__device__ __forceinline__ void weights8(double fx, double fy, double fz, double ax, double ay,
                                         double az, double w[8]) {
  w[0] = ax * ay * az; w[1] = fx * ay * az; w[2] = ax * fy * az; w[3] = fx * fy * az;
  w[4] = ax * ay * fz; w[5] = fx * ay * fz; w[6] = ax * fy * fz; w[7] = fx * fy * fz;
}

// 6-component gather from the double node records, left-to-right corner order
// (kernels.py:568-591).  The first corner initialises the sum (0.0 + w*F
// would turn a -0.0 product into +0.0).
__device__ __forceinline__ void gather_records(const double* __restrict__ fn, int n000, int sx,
                                               int sy, const double w[8], double s[6]) {
  const int off[8] = {0, sx, sy, sx + sy, 1, sx + 1, sy + 1, sx + sy + 1};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double* rec = fn + (size_t)(n000 + off[k]) * 8;
    double q4[4];
    ldg256(rec, q4);
    const double2 a0 = make_double2(q4[0], q4[1]), a1 = make_double2(q4[2], q4[3]);
    const double2 a2 = __ldg(reinterpret_cast<const double2*>(rec) + 2);
    if (k == 0) {
      s[0] = w[0] * a0.x; s[1] = w[0] * a0.y; s[2] = w[0] * a1.x;
      s[3] = w[0] * a1.y; s[4] = w[0] * a2.x; s[5] = w[0] * a2.y;
    } else {
      s[0] = s[0] + w[k] * a0.x; s[1] = s[1] + w[k] * a0.y; s[2] = s[2] + w[k] * a1.x;
      s[3] = s[3] + w[k] * a1.y; s[4] = s[4] + w[k] * a2.x; s[5] = s[5] + w[k] * a2.y;
    }
  }
}

template <typename P_, typename F_>
struct ParityPolicy {
  typedef P_ P;
  typedef F_ F;
  typedef double NodeT;
  static constexpr bool kFmaFold = false;
  struct Consts {
    double iv_max;
    __device__ __forceinline__ explicit Consts(const SpanParams<P, F>& a)
        : iv_max(a.iv_max ? __ldg(a.iv_max) : 0.0) {}
  };

  // Push block for one particle (kernels.py:489-682), in place on OK.
  static __device__ __forceinline__ int push(const SpanParams<P, F>& a, const Consts&, P& xp,
                                             P& yp, P& zp, P& vnx, P& vny, P& vnz) {
    const auto& d = a.d;
    const double* fn = static_cast<const double*>(a.fnode);
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
      gather_records(fn, (i * a.NY + j) * a.NZ + k, a.NY * a.NZ, a.NZ, w, s);
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
    double xo = (double)xp + vbx * d.dt;
    double yo = (double)yp + vby * d.dt;
    double zo = (double)zp + vbz * d.dt;
    double uo = d.two * vbx - (double)vnx;
    double vo = d.two * vby - (double)vny;
    double wo = d.two * vbz - (double)vnz;
    if (a.apply_bc) {
      fold_commit(xo, uo, d.o[0], d.L[0], d.hi[0], d.hi2[0], a.bcx);
      fold_commit(yo, vo, d.o[1], d.L[1], d.hi[1], d.hi2[1], a.bcy);
      fold_commit(zo, wo, d.o[2], d.L[2], d.hi[2], d.hi2[2], a.bcz);
      if (xo < d.o[0] || xo > d.hi[0] || yo < d.o[1] || yo > d.hi[1] || zo < d.o[2] ||
          zo > d.hi[2])
        return ST_RUNAWAY;
    }
    xp = (P)xo; yp = (P)yo; zp = (P)zo;
    vnx = (P)uo; vny = (P)vo; vnz = (P)wo;
    return ST_OK;
  }

  // Cell of the deposit block; gx in promote(P, F) (f32 only when both are f32).
  static __device__ __forceinline__ int cell(const SpanParams<P, F>& a, P xp, P yp, P zp,
                                             double& fx, double& fy, double& fz) {
    typedef decltype(P() - F()) G;
    const G gx = ((G)xp - (G)a.gox) / (G)a.gdx;
    const G gy = ((G)yp - (G)a.goy) / (G)a.gdy;
    const G gz = ((G)zp - (G)a.goz) / (G)a.gdz;
    if (!(gx >= (G)0 && gy >= (G)0 && gz >= (G)0 && gx < (G)2147483647 &&
          gy < (G)2147483647 && gz < (G)2147483647))
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

  // Deposit values of one particle (kernels.py:683-734), staged as doubles.
  template <bool PRESCALE>
  static __device__ __forceinline__ int stage(const SpanParams<P, F>& a, const Consts& K,
                                              bool valid, P xp, P yp, P zp, P un, P vn, P wn,
                                              P qp, double* st_bs, double* st_mv, bool& big) {
    double fx = 0, fy = 0, fz = 0;
    int key = valid ? cell(a, xp, yp, zp, fx, fy, fz) : -1;
    // invalid particles stage zero bases: folding them adds exact zeros
    const double q = key >= 0 ? (double)qp : 0.0;
    const int nb = key >= 0 ? key : 0;
    const double* fn = static_cast<const double*>(a.fnode);
    const int sx = a.NY * a.NZ, sy = a.NZ;
    const int off[8] = {0, sx, sy, sx + sy, 1, sx + 1, sy + 1, sx + sy + 1};
    const double ax = a.d.one - fx, ay = a.d.one - fy, az = a.d.one - fz;
    double bs[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double wx = (c & 1) ? fx : ax, wy = (c & 2) ? fy : ay, wz = (c & 4) ? fz : az;
      const double iv = __ldg(fn + (size_t)(nb + off[c]) * 8 + 6);
      const double base = q * (wx * wy * wz) * iv;
      bs[c] = PRESCALE ? base * a.d.scale : base;
    }
    stage_bases(st_bs, bs);
    // dyads in particle precision (kernels.py:701-706)
    const P pxx = un * un, pxy = un * vn, pxz = un * wn;
    const P pyy = vn * vn, pyz = vn * wn, pzz = wn * wn;
    stage_moments(st_mv, (double)un, (double)vn, (double)wn, (double)pxx, (double)pxy,
                  (double)pxz, (double)pyy, (double)pyz, (double)pzz);
    big = key >= 0 && magic_unsafe(q * K.iv_max * (PRESCALE ? a.d.scale : 1.0), (double)pxx,
                                   (double)pyy, (double)pzz,
                                   PRESCALE ? kMagicLimit : kMagicLimit / a.d.scale);
    return key;
  }
};

// gather_span (kernels.py:385-455): E/B at in-domain points, rounded once to P
template <typename P, typename F>
__global__ void __launch_bounds__(256) gather_kernel(SpanParams<P, F> a) {
  typedef ParityPolicy<P, F> Pol;
  const i64 nthreads = (i64)gridDim.x * blockDim.x;
  const double* fn = static_cast<const double*>(a.fnode);
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < a.count; r += nthreads) {
    const i64 p = a.start + r;
    double fx, fy, fz;
    const int n000 = Pol::cell(a, a.x[p], a.y[p], a.z[p], fx, fy, fz);
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
    gather_records(fn, n000, a.NY * a.NZ, a.NZ, w, s);
#pragma unroll
    for (int c = 0; c < 6; ++c) a.gather_out[r * 6 + c] = (P)s[c];
  }
}

}  // namespace bp
