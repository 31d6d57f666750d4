// Device helpers shared by the f32 fast kernels: the flat split kernels
// (bp_split.cu) and the cell-binned kernels (bp_bins.cu).  Arithmetic as the
// reference fused_span (pkg/src/batchpic/kernels.py:458-735) in native f32
// with FMA; DESIGN.md §4.
#pragma once
#include <cstdint>
#include <type_traits>

#include "bp_common.cuh"

namespace bp {
namespace sk {

template <typename T>
struct Params {
  T *x, *y, *z, *u, *v, *w;
  const T* q;
  long long start, count;
  const void* rec;     // 12 quads of T per cell, cell = i + nx * (j + ny * k)
  const float* iv_f;   // invvol (nx+1, ny+1, nz+1) when fields are f32
  const double* iv_d;  // ... when fields are f64
  long long* acc;      // (10, NN) int64
  int nx, ny, nz, NY, NZ, NN;
  int cny;  // nx * ny (cell-record z stride)
  T o[3], hi[3], L[3], hi2[3], idx[3], ogs[3];
  T dt, dth, qdt2m, beta, beta2;
  double scale;
  int n_iters;
  int* status;
  unsigned long long* work;  // deposit: next unclaimed particle of the span
  unsigned* skip;            // one bit per span particle the mover did not store
  const float* emax;         // max |E| over the nodes (after the cell records)
  T bc_eps[3];               // rounding slack of the boundary-skip test per axis
  T nm1[3];                  // cell counts - 1, and nx, nx * ny, in T (float cell index)
  T nxf, cnyf;
};

// record quad of T
template <typename T>
struct Quad;
template <>
struct Quad<float> {
  typedef float4 type;
};
template <>
struct Quad<double> {
  typedef double4 type;
};

__device__ __forceinline__ float rcp_fast(float d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));  // d >= 1: MUFU.RCP alone
  return r;
}
__device__ __forceinline__ double rcp_fast(double d) { return __drcp_rn(d); }

// record loads (kept in L1 / L2 in preference to the particle streams)
__device__ __forceinline__ void ldg_pair(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.L1::evict_last.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void ldg_pair(const double4* p, double4& a, double4& b) {
  asm("ld.global.nc.L1::evict_last.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(a.z), "=d"(a.w)
      : "l"(p));
  asm("ld.global.nc.L1::evict_last.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(b.x), "=d"(b.y), "=d"(b.z), "=d"(b.w)
      : "l"(p + 1));
}

template <bool REFL, typename T>
__device__ __forceinline__ T fold_mid(T xm, T o, T L, T hi, T hi2) {
  if (!REFL) {
    if (xm < o) xm += L;
    else if (xm > hi) xm -= L;
  } else {
    if (xm < o) xm = o + (o - xm);
    else if (xm > hi) xm = hi2 - xm;
  }
  return xm;
}

template <bool REFL, typename T>
__device__ __forceinline__ void fold_commit(T& q, T& vel, T o, T L, T hi, T hi2) {
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
template <typename T>
__device__ __forceinline__ bool interior(const Params<T>& a, T qe, T x, T y, T z, T u, T v,
                                         T w) {
  const T reach = (fabs(u) + fabs(v) + fabs(w) + qe) * a.dt;
  return x - a.o[0] > reach + a.bc_eps[0] && a.hi[0] - x > reach + a.bc_eps[0] &&
         y - a.o[1] > reach + a.bc_eps[1] && a.hi[1] - y > reach + a.bc_eps[1] &&
         z - a.o[2] > reach + a.bc_eps[2] && a.hi[2] - z > reach + a.bc_eps[2];
}

// cell of an in-box position: truncation (in-box gx >= -ulp truncates to 0)
// and the upper-face clamp of kernels.py:541-556; returns the cell index
template <typename T>
__device__ __forceinline__ int cell_of(const Params<T>& a, T x, T y, T z, T& fx, T& fy, T& fz,
                                       int& i, int& j, int& k) {
  const T gx = fma(x, a.idx[0], -a.ogs[0]);
  const T gy = fma(y, a.idx[1], -a.ogs[1]);
  const T gz = fma(z, a.idx[2], -a.ogs[2]);
  i = min((int)gx, a.nx - 1);
  j = min((int)gy, a.ny - 1);
  k = min((int)gz, a.nz - 1);
  fx = gx - (T)i;
  fy = gy - (T)j;
  fz = gz - (T)k;
  return i + a.nx * j + a.cny * k;
}

typedef float2 F2;
__device__ __forceinline__ F2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) { return __ffma2_rn(a, b, c); }

// one component pair (a, b) from its four quads: A = c0a c0b c1a c1b,
// B = c2a c2b c4a c4b, C = c3a c3b c5a c5b, D = c6a c6b c7a c7b
__device__ __forceinline__ void tri_pair(const float4& A, const float4& B, const float4& C,
                                         const float4& D, float fx, float fy, float fz,
                                         float& ra, float& rb) {
  const F2 FX = f2(fx, fx), FY = f2(fy, fy), FZ = f2(fz, fz);
  const F2 p = fma2(f2(A.z, A.w), FX, f2(A.x, A.y));
  const F2 q = fma2(f2(B.z, B.w), FX, f2(B.x, B.y));
  const F2 r = fma2(f2(C.z, C.w), FX, f2(C.x, C.y));
  const F2 t = fma2(f2(D.z, D.w), FX, f2(D.x, D.y));
  const F2 o = fma2(fma2(t, FY, r), FZ, fma2(q, FY, p));
  ra = o.x;
  rb = o.y;
}
__device__ __forceinline__ void tri_pair(const double4& A, const double4& B, const double4& C,
                                         const double4& D, double fx, double fy, double fz,
                                         double& ra, double& rb) {
  ra = fma(fma(fma(D.z, fx, D.x), fy, fma(C.z, fx, C.x)), fz,
           fma(fma(B.z, fx, B.x), fy, fma(A.z, fx, A.x)));
  rb = fma(fma(fma(D.w, fx, D.y), fy, fma(C.w, fx, C.y)), fz,
           fma(fma(B.w, fx, B.y), fy, fma(A.w, fx, A.y)));
}


// The implicit push of the fast kernels (kernels.py:498-676) on the per-cell
// coefficient records: the flat split mover (bp_split.cu, f32) and the f64
// binned mover (bp_bins64.cu).
// skipbc (warp-uniform): the caller has shown that no position of this push
// can leave the box (interior()), so the boundary folds and checks are
// identities and are skipped.
template <typename T, bool RX, bool RY, bool RZ, bool REUSE>
__device__ __forceinline__ int push(const Params<T>& a, T& xp, T& yp, T& zp, T& un, T& vn,
                                    T& wn, bool skipbc) {
  typedef typename Quad<T>::type Q;
  T vbx = un, vby = vn, vbz = wn;
  Q R[12];
  int held = -1;  // cell whose record is in R
#pragma unroll 1
  for (int it = 0; it < a.n_iters; ++it) {
    T xm, ym;
    if constexpr (std::is_same<T, float>::value) {
      const F2 XM = fma2(f2(vbx, vby), f2(a.dth, a.dth), f2(xp, yp));
      xm = XM.x;
      ym = XM.y;
    } else {
      xm = fma(vbx, a.dth, xp);
      ym = fma(vby, a.dth, yp);
    }
    T zm = fma(vbz, a.dth, zp);
    if (!skipbc) {
      xm = fold_mid<RX>(xm, a.o[0], a.L[0], a.hi[0], a.hi2[0]);
      ym = fold_mid<RY>(ym, a.o[1], a.L[1], a.hi[1], a.hi2[1]);
      zm = fold_mid<RZ>(zm, a.o[2], a.L[2], a.hi[2], a.hi2[2]);
      if (xm < a.o[0] || xm > a.hi[0] || ym < a.o[1] || ym > a.hi[1] || zm < a.o[2] ||
          zm > a.hi[2])
        return ST_MIDPOINT;
    }
    T fx, fy, fz;
    int i, j, k;
    const int cell = cell_of(a, xm, ym, zm, fx, fy, fz, i, j, k);
    if (!REUSE || cell != held) {
      held = cell;
      const Q* r = static_cast<const Q*>(a.rec) + (size_t)cell * 12;
#pragma unroll
      for (int q = 0; q < 12; q += 2) ldg_pair(r + q, R[q], R[q + 1]);
    }
    T ex, ey, hx, hy, ez, hz;
    tri_pair(R[0], R[1], R[2], R[3], fx, fy, fz, ex, ey);
    tri_pair(R[4], R[5], R[6], R[7], fx, fy, fz, hx, hy);
    tri_pair(R[8], R[9], R[10], R[11], fx, fy, fz, ez, hz);
    T tx, ty;
    if constexpr (std::is_same<T, float>::value) {
      const F2 Txy = fma2(f2(a.qdt2m, a.qdt2m), f2(ex, ey), f2(un, vn));
      tx = Txy.x;
      ty = Txy.y;
    } else {
      tx = fma(a.qdt2m, ex, un);
      ty = fma(a.qdt2m, ey, vn);
    }
    const T tz = fma(a.qdt2m, ez, wn);
    const T bsq = fma(hx, hx, fma(hy, hy, hz * hz));
    const T inv = rcp_fast(fma(a.beta2, bsq, T(1)));
    const T tdb = fma(tx, hx, fma(ty, hy, tz * hz));
    const T bt = a.beta * tdb;
    const T cx = fma(ty, hz, -tz * hy), cy = fma(tz, hx, -tx * hz), cz = fma(tx, hy, -ty * hx);
    vbx = fma(a.beta, fma(bt, hx, cx), tx) * inv;
    vby = fma(a.beta, fma(bt, hy, cy), ty) * inv;
    vbz = fma(a.beta, fma(bt, hz, cz), tz) * inv;
  }
  T xo = fma(vbx, a.dt, xp), yo = fma(vby, a.dt, yp), zo = fma(vbz, a.dt, zp);
  T uo = T(2) * vbx - un, vo = T(2) * vby - vn, wo = T(2) * vbz - wn;
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

}  // namespace sk

struct Call;
// Params of one span call (bp_split.cu): geometry, scalars and pointers of
// `c`; the per-call scratch fields (work, skip, rec, emax) are left null.
template <typename T>
void fill_params(const Call& c, sk::Params<T>& a);

}  // namespace bp
