// Fast arithmetic: the same algorithm (kernels.py:458-735) in the particle
// precision T = P with fused multiply-adds and reciprocal multiplies —
// sputniPIC's native single / double precision.  Mixed mode (f32 particles,
// f64 fields) rounds the fields to f32 once, in the node records.
//
// Differences from the reference arithmetic (all bounded):
//   gx = x * (1/dx) - ox/dx instead of (x - ox) / dx; trilinear sums and the
//   rotation use FMA; 1/denom is multiplied instead of dividing; f32 particles
//   compute in f32 (the reference promotes most of the algebra to f64); the
//   deposit rounds fma(base, m, 1.5*2^52) (the exact product) to the lattice.
// The moment lattice itself (int64, quantum 2^-43, one rint per contribution)
// is unchanged, so deposits stay exact and batch/order independent.
#pragma once
#include "bp_common.cuh"

namespace bp {

// Per-thread constants of the fast arithmetic.  f32: read from the host-
// rounded parameter copy (no per-particle conversions); f64: the wide copy.
template <typename T>
struct FastScalars;

template <>
struct FastScalars<float> {
  const NarrowScalars& f;
  double qlim;  // |q * scale| bound for the magic-rint guard
  template <typename P, typename F>
  __device__ __forceinline__ explicit FastScalars(const SpanParams<P, F>& a)
      : f(a.f), qlim((a.iv_max ? __ldg(a.iv_max) : 0.0) * 1.0000001) {}
  __device__ __forceinline__ float o(int k) const { return f.o[k]; }
  __device__ __forceinline__ float L(int k) const { return f.L[k]; }
  __device__ __forceinline__ float hi(int k) const { return f.hi[k]; }
  __device__ __forceinline__ float hi2(int k) const { return f.hi2[k]; }
  __device__ __forceinline__ float idx(int k) const { return f.idx[k]; }
  __device__ __forceinline__ float ogs(int k) const { return f.ogs[k]; }
  __device__ __forceinline__ float dt() const { return f.dt; }
  __device__ __forceinline__ float dth() const { return f.dth; }
  __device__ __forceinline__ float qdt2m() const { return f.qdt2m; }
  __device__ __forceinline__ float beta() const { return f.beta; }
  __device__ __forceinline__ float beta2() const { return f.beta2; }
  __device__ __forceinline__ float scale() const { return f.scale; }
};

template <>
struct FastScalars<double> {
  const WideScalars& d;
  double qlim;
  template <typename P, typename F>
  __device__ __forceinline__ explicit FastScalars(const SpanParams<P, F>& a)
      : d(a.d), qlim(a.iv_max ? __ldg(a.iv_max) : 0.0) {}
  __device__ __forceinline__ double o(int k) const { return d.o[k]; }
  __device__ __forceinline__ double L(int k) const { return d.L[k]; }
  __device__ __forceinline__ double hi(int k) const { return d.hi[k]; }
  __device__ __forceinline__ double hi2(int k) const { return d.hi2[k]; }
  __device__ __forceinline__ double idx(int k) const { return d.inv_gd[k]; }
  __device__ __forceinline__ double ogs(int k) const { return d.go_s[k]; }
  __device__ __forceinline__ double dt() const { return d.dt; }
  __device__ __forceinline__ double dth() const { return d.dth; }
  __device__ __forceinline__ double qdt2m() const { return d.qdt2m; }
  __device__ __forceinline__ double beta() const { return d.beta; }
  __device__ __forceinline__ double beta2() const { return d.beta2; }
  __device__ __forceinline__ double scale() const { return d.scale; }
};

template <typename T>
__device__ __forceinline__ T fold_mid_t(T xm, T o, T L, T hi, T hi2, int bc) {
  if (bc == 0) {
    if (xm < o) xm = xm + L;
    else if (xm > hi) xm = xm - L;
  } else {
    if (xm < o) xm = o + (o - xm);
    else if (xm > hi) xm = hi2 - xm;
  }
  return xm;
}

template <typename T>
__device__ __forceinline__ void fold_commit_t(T& q, T& vel, T o, T L, T hi, T hi2, int bc) {
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

// 1 / denom with denom = 1 + beta^2 |h|^2 >= 1: MUFU.RCP (2 ulp) is ample
// against the 1e-4 tolerance of the f32 path
__device__ __forceinline__ float fast_rcp(float x) { return __fdividef(1.0f, x); }
__device__ __forceinline__ double fast_rcp(double x) { return __drcp_rn(x); }

// one node record (8 T) -> E, B (two 16-byte loads: measured faster here
// than one 32-byte LDG.256)
__device__ __forceinline__ void load_record(const float* r8, float e[6]) {
  const float4* r = reinterpret_cast<const float4*>(r8);
  const float4 a = __ldg(r), b = __ldg(r + 1);
  e[0] = a.x; e[1] = a.y; e[2] = a.z; e[3] = a.w; e[4] = b.x; e[5] = b.y;
}
__device__ __forceinline__ void load_record(const double* r8, double e[6]) {
  const double2* r = reinterpret_cast<const double2*>(r8);
  const double2 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2);
  e[0] = a.x; e[1] = a.y; e[2] = b.x; e[3] = b.y; e[4] = c.x; e[5] = c.y;
}

template <typename P_, typename F_>
struct FastPolicy {
  typedef P_ P;
  typedef F_ F;
  typedef P_ T;
  typedef P_ NodeT;
  static constexpr bool kFmaFold = true;
  typedef FastScalars<P_> Consts;

  static __device__ __forceinline__ int cell_t(const SpanParams<P, F>& a,
                                               const FastScalars<T>& s, T x, T y, T z, T& fx,
                                               T& fy, T& fz) {
    const T gx = fma(x, s.idx(0), -s.ogs(0));
    const T gy = fma(y, s.idx(1), -s.ogs(1));
    const T gz = fma(z, s.idx(2), -s.ogs(2));
    int i = (int)gx, j = (int)gy, k = (int)gz;
    // callers pass in-box positions: gx >= -ulp truncates to 0, only the upper
    // face needs the clamp (kernels.py:541-552)
    i = min(i, a.nx - 1);
    j = min(j, a.ny - 1);
    k = min(k, a.nz - 1);
    fx = gx - (T)i; fy = gy - (T)j; fz = gz - (T)k;
    return (i * a.NY + j) * a.NZ + k;
  }

  static __device__ __forceinline__ int push(const SpanParams<P, F>& a, const Consts& s, P& xp,
                                             P& yp, P& zp, P& vnx, P& vny, P& vnz) {
    const T* fn = static_cast<const T*>(a.fnode);
    const int sx = a.NY * a.NZ, sy = a.NZ;
    T vbx = vnx, vby = vny, vbz = vnz;
    for (int it = 0; it < a.n_iters; ++it) {
      T xm = fma(vbx, s.dth(), xp), ym = fma(vby, s.dth(), yp), zm = fma(vbz, s.dth(), zp);
      xm = fold_mid_t(xm, s.o(0), s.L(0), s.hi(0), s.hi2(0), a.bcx);
      ym = fold_mid_t(ym, s.o(1), s.L(1), s.hi(1), s.hi2(1), a.bcy);
      zm = fold_mid_t(zm, s.o(2), s.L(2), s.hi(2), s.hi2(2), a.bcz);
      if (xm < s.o(0) || xm > s.hi(0) || ym < s.o(1) || ym > s.hi(1) || zm < s.o(2) ||
          zm > s.hi(2))
        return ST_MIDPOINT;
      T fx, fy, fz;
      const int n000 = cell_t(a, s, xm, ym, zm, fx, fy, fz);
      const T ax = T(1) - fx, ay = T(1) - fy, az = T(1) - fz;
      const T wxy[4] = {ax * ay, fx * ay, ax * fy, fx * fy};
      // four record pointers (i/i+1, j/j+1); the k+1 corner is the next record
      const T* r00 = fn + (size_t)n000 * 8;
      const T* rr[4] = {r00, r00 + (size_t)sx * 8, r00 + (size_t)sy * 8,
                        r00 + (size_t)(sx + sy) * 8};
      T e[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const T wc = wxy[c & 3] * ((c & 4) ? fz : az);
        T r[6];
        load_record(rr[c & 3] + ((c & 4) ? 8 : 0), r);
#pragma unroll
        for (int m = 0; m < 6; ++m) e[m] = fma(wc, r[m], e[m]);
      }
      const T tx = fma(s.qdt2m(), e[0], vnx), ty = fma(s.qdt2m(), e[1], vny),
              tz = fma(s.qdt2m(), e[2], vnz);
      const T hx = e[3], hy = e[4], hz = e[5];
      const T bsq = fma(hx, hx, fma(hy, hy, hz * hz));
      const T inv = fast_rcp(fma(s.beta2(), bsq, T(1)));
      const T tdb = fma(tx, hx, fma(ty, hy, tz * hz));
      const T bt = s.beta() * tdb;
      const T cx = fma(ty, hz, -tz * hy), cy = fma(tz, hx, -tx * hz), cz = fma(tx, hy, -ty * hx);
      vbx = fma(s.beta(), fma(bt, hx, cx), tx) * inv;
      vby = fma(s.beta(), fma(bt, hy, cy), ty) * inv;
      vbz = fma(s.beta(), fma(bt, hz, cz), tz) * inv;
    }
    T xo = fma(vbx, s.dt(), xp), yo = fma(vby, s.dt(), yp), zo = fma(vbz, s.dt(), zp);
    T uo = T(2) * vbx - vnx, vo = T(2) * vby - vny, wo = T(2) * vbz - vnz;
    if (a.apply_bc) {
      fold_commit_t(xo, uo, s.o(0), s.L(0), s.hi(0), s.hi2(0), a.bcx);
      fold_commit_t(yo, vo, s.o(1), s.L(1), s.hi(1), s.hi2(1), a.bcy);
      fold_commit_t(zo, wo, s.o(2), s.L(2), s.hi(2), s.hi2(2), a.bcz);
      if (xo < s.o(0) || xo > s.hi(0) || yo < s.o(1) || yo > s.hi(1) || zo < s.o(2) ||
          zo > s.hi(2))
        return ST_RUNAWAY;
    }
    xp = xo; yp = yo; zp = zo;
    vnx = uo; vny = vo; vnz = wo;
    return ST_OK;
  }

  template <bool PRESCALE>
  static __device__ __forceinline__ int stage(const SpanParams<P, F>& a, const Consts& s,
                                              bool valid, P xp, P yp, P zp, P un, P vn, P wn,
                                              P qp, double* st_bs, double* st_mv, bool& big) {
    const T* fn = static_cast<const T*>(a.fnode);
    const int sx = a.NY * a.NZ, sy = a.NZ;
    int key = -1;
    T fx = 0, fy = 0, fz = 0;
    if (valid) {
      // domain check as in the reference deposit (positions are in the box
      // after the push; a deposit-only call may hand us anything)
      if (xp >= s.o(0) && xp <= s.hi(0) && yp >= s.o(1) && yp <= s.hi(1) && zp >= s.o(2) &&
          zp <= s.hi(2))
        key = cell_t(a, s, xp, yp, zp, fx, fy, fz);
    }
    const int nb = key >= 0 ? key : 0;
    const T qs = key >= 0 ? qp * s.scale() : T(0);  // the lattice scale is folded in once
    const T ax = T(1) - fx, ay = T(1) - fy, az = T(1) - fz;
    const T wxy[4] = {ax * ay, fx * ay, ax * fy, fx * fy};
    const T* r00 = fn + (size_t)nb * 8 + 6;
    const T* rr[4] = {r00, r00 + (size_t)sx * 8, r00 + (size_t)sy * 8,
                      r00 + (size_t)(sx + sy) * 8};
    double bs[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const T iv = __ldg(rr[c & 3] + ((c & 4) ? 8 : 0));
      bs[c] = (double)(qs * (wxy[c & 3] * ((c & 4) ? fz : az)) * iv);
    }
    stage_bases(st_bs, bs);
    const T pxx = un * un, pxy = un * vn, pxz = un * wn;
    const T pyy = vn * vn, pyz = vn * wn, pzz = wn * wn;
    stage_moments(st_mv, (double)un, (double)vn, (double)wn, (double)pxx, (double)pxy,
                  (double)pxz, (double)pyy, (double)pyz, (double)pzz);
    big = key >= 0 && magic_unsafe((double)qs * s.qlim, (double)pxx, (double)pyy, (double)pzz,
                                   kMagicLimit);
    return key;
  }
};

}  // namespace bp
