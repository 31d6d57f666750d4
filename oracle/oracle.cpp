// SPDX-License-Identifier: MIT
//
// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT PATH.
//
// CPU restatement of the reference hot path (batchpic `kernels.py`), used
//   * by tests/ as the parity checker for the CUDA kernels,
//   * by __graft_entry__.smoke() as the checker of one small launch,
//   * by bench.py's `cpu_baseline` leg and `--impl reference` arm as the CPU
//     implementation timed beside the GPU ("kind": "port").
// Nothing under paper_2008_04397_b200/ may load this library.
//
// Parity pinning: this file is checked bitwise against golden vectors made
// by the reference package itself (tests/golden/make_golden.py imports
// /root/reference/pkg/src/batchpic and runs its numba kernels), see
// tests/test_oracle_golden.py.
//
// Arithmetic contract (reference numba 0.65 typing):
//   P = particle storage type, F = field storage type, D = double.
//   numba types every f32 (op) int64 / f32 (op) f64 expression as f64, keeps
//   f32 (op) f32 as f32, emits no FMA and IEEE division.  The template below
//   spells out every promotion explicitly.  Compile with -ffp-contract=off.
//
// Reference line map (pkg/src/batchpic/kernels.py):
//   push block ........ fused_span :489-682  (== push_span :112-306)
//   deposit block ..... fused_span :683-734  (== deposit_span :327-381)
//   gather ............ gather_span :385-455
//   make_geo_arrays ... :57-67 (geo layout dx dy dz ox oy oz Lx Ly Lz; nx ny nz bcx bcy bcz)
//   sort key .......... geometry.py:152-159 cell_index_of, particles.py:157-167

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <thread>

typedef int64_t i64;
typedef double D;

enum { OR_OK = 0, OR_ERR_RUNAWAY = 1, OR_ERR_MIDPOINT = 2, OR_ERR_ARGS = -1 };

namespace {

template <typename P, typename F>
struct Geo {
  // geo_f (particle precision): boundary arithmetic
  P ox, oy, oz, Lx, Ly, Lz;
  // geo_g (field precision): cell location
  F gdx, gdy, gdz, gox, goy, goz;
  i64 nx, ny, nz, bcx, bcy, bcz;
  i64 NX, NY, NZ;  // node extents
  Geo(const D* gf, const D* gg, const i64* gi) {
    ox = (P)gf[3]; oy = (P)gf[4]; oz = (P)gf[5];
    Lx = (P)gf[6]; Ly = (P)gf[7]; Lz = (P)gf[8];
    gdx = (F)gg[0]; gdy = (F)gg[1]; gdz = (F)gg[2];
    gox = (F)gg[3]; goy = (F)gg[4]; goz = (F)gg[5];
    nx = gi[0]; ny = gi[1]; nz = gi[2];
    bcx = gi[3]; bcy = gi[4]; bcz = gi[5];
    NX = nx + 1; NY = ny + 1; NZ = nz + 1;
  }
  inline i64 node(i64 i, i64 j, i64 k) const { return (i * NY + j) * NZ + k; }
};

// midpoint boundary fold, kernels.py:505-534 (`>` on the upper face)
template <typename P>
static inline D fold_mid(D xm, P o, P L, i64 bc) {
  const P hi = (P)(o + L);  // ox + Lx in particle precision
  if (bc == 0) {
    if (xm < (D)o) xm = xm + (D)L;
    else if (xm > (D)hi) xm = xm - (D)L;
  } else {
    if (xm < (D)o) xm = (D)o + ((D)o - xm);
    else if (xm > (D)hi) xm = (D)(P)(hi + hi) - xm;
  }
  return xm;
}

// cell + fractional offset along one axis (gx is D in the push block)
static inline void cell1(D g, i64 n, i64& i, D& f) {
  i = (i64)g;
  if (i > n - 1) i = n - 1;
  f = g - (D)i;
}

template <typename P, typename F>
static inline D tri(const F* A, const Geo<P, F>& g, i64 i, i64 j, i64 k,
                    const D w[8]) {
  const i64 i1 = i + 1, j1 = j + 1, k1 = k + 1;
  // strictly left-to-right, kernels.py:568-591
  D s = w[0] * (D)A[g.node(i, j, k)];
  s = s + w[1] * (D)A[g.node(i1, j, k)];
  s = s + w[2] * (D)A[g.node(i, j1, k)];
  s = s + w[3] * (D)A[g.node(i1, j1, k)];
  s = s + w[4] * (D)A[g.node(i, j, k1)];
  s = s + w[5] * (D)A[g.node(i1, j, k1)];
  s = s + w[6] * (D)A[g.node(i, j1, k1)];
  s = s + w[7] * (D)A[g.node(i1, j1, k1)];
  return s;
}

static inline void weights8(D fx, D fy, D fz, D ax, D ay, D az, D w[8]) {
  w[0] = ax * ay * az; w[1] = fx * ay * az; w[2] = ax * fy * az; w[3] = fx * fy * az;
  w[4] = ax * ay * fz; w[5] = fx * ay * fz; w[6] = ax * fy * fz; w[7] = fx * fy * fz;
}

// One particle through the push block.  Returns status; on OK writes the
// committed position/velocity (already rounded to P) into out[6].
template <typename P, typename F>
static int push_one(P xp, P yp, P zp, P vnx, P vny, P vnz, const F* E, const F* B,
                    const Geo<P, F>& g, P dt, P dth, P qdt2m, P beta, P one,
                    int n_iters, int apply_bc, int mixed, P out[6]) {
  const i64 NN = g.NX * g.NY * g.NZ;
  D vbx = (D)vnx, vby = (D)vny, vbz = (D)vnz;
  for (int it = 0; it < n_iters; ++it) {
    D xm = (D)xp + vbx * (D)dth;
    D ym = (D)yp + vby * (D)dth;
    D zm = (D)zp + vbz * (D)dth;
    xm = fold_mid<P>(xm, g.ox, g.Lx, g.bcx);
    ym = fold_mid<P>(ym, g.oy, g.Ly, g.bcy);
    zm = fold_mid<P>(zm, g.oz, g.Lz, g.bcz);
    const P hx_ = (P)(g.ox + g.Lx), hy_ = (P)(g.oy + g.Ly), hz_ = (P)(g.oz + g.Lz);
    if (xm < (D)g.ox || xm > (D)hx_ || ym < (D)g.oy || ym > (D)hy_ ||
        zm < (D)g.oz || zm > (D)hz_)
      return OR_ERR_MIDPOINT;
    const D gx = (xm - (D)g.gox) / (D)g.gdx;
    const D gy = (ym - (D)g.goy) / (D)g.gdy;
    const D gz = (zm - (D)g.goz) / (D)g.gdz;
    i64 i, j, k;
    D fx, fy, fz;
    cell1(gx, g.nx, i, fx);
    cell1(gy, g.ny, j, fy);
    cell1(gz, g.nz, k, fz);
    const D ax = (D)one - fx, ay = (D)one - fy, az = (D)one - fz;
    D w[8];
    weights8(fx, fy, fz, ax, ay, az, w);
    const D epx = tri(E, g, i, j, k, w);
    const D epy = tri(E + NN, g, i, j, k, w);
    const D epz = tri(E + 2 * NN, g, i, j, k, w);
    const D bpx = tri(B, g, i, j, k, w);
    const D bpy = tri(B + NN, g, i, j, k, w);
    const D bpz = tri(B + 2 * NN, g, i, j, k, w);
    D tx, ty, tz, hx, hy, hz;
    if (mixed) {
      // sample rounded once through the P-typed scratch; t in P (:592-604)
      const P sx = (P)epx, sy = (P)epy, sz = (P)epz;
      tx = (D)(P)(vnx + (P)(qdt2m * sx));
      ty = (D)(P)(vny + (P)(qdt2m * sy));
      tz = (D)(P)(vnz + (P)(qdt2m * sz));
      hx = (D)(P)bpx; hy = (D)(P)bpy; hz = (D)(P)bpz;
    } else {
      tx = (D)vnx + (D)qdt2m * epx;
      ty = (D)vny + (D)qdt2m * epy;
      tz = (D)vnz + (D)qdt2m * epz;
      hx = bpx; hy = bpy; hz = bpz;
    }
    // rotation, kernels.py:606-617; beta*beta stays in P
    const D bsq = hx * hx + hy * hy + hz * hz;
    const D denom = (D)one + (D)(P)(beta * beta) * bsq;
    const D tdb = tx * hx + ty * hy + tz * hz;
    vbx = (tx + (D)beta * ((ty * hz - tz * hy) + (D)beta * tdb * hx)) / denom;
    vby = (ty + (D)beta * ((tz * hx - tx * hz) + (D)beta * tdb * hy)) / denom;
    vbz = (tz + (D)beta * ((tx * hy - ty * hx) + (D)beta * tdb * hz)) / denom;
  }
  // commit, kernels.py:622-628
  D x = (D)xp + vbx * (D)dt;
  D y = (D)yp + vby * (D)dt;
  D z = (D)zp + vbz * (D)dt;
  const P two = (P)(one + one);
  D u = (D)two * vbx - (D)vnx;
  D v = (D)two * vby - (D)vny;
  D w = (D)two * vbz - (D)vnz;
  if (apply_bc) {
    // kernels.py:629-676 (`>=` wrap with snap-to-origin on periodic axes)
    P o3[3] = {g.ox, g.oy, g.oz};
    P L3[3] = {g.Lx, g.Ly, g.Lz};
    i64 bc3[3] = {g.bcx, g.bcy, g.bcz};
    D* q3[3] = {&x, &y, &z};
    D* v3[3] = {&u, &v, &w};
    for (int a = 0; a < 3; ++a) {
      const P o = o3[a], L = L3[a];
      const P hi = (P)(o + L);
      D& q = *q3[a];
      if (bc3[a] == 0) {
        if (q < (D)o) {
          q = q + (D)L;
          if (q >= (D)hi) q = (D)o;
        } else if (q >= (D)hi) {
          q = q - (D)L;
        }
      } else {
        if (q < (D)o) {
          q = (D)o + ((D)o - q);
          *v3[a] = -*v3[a];
        } else if (q > (D)hi) {
          q = (D)(P)(hi + hi) - q;
          *v3[a] = -*v3[a];
        }
      }
    }
    if (x < (D)g.ox || x > (D)(P)(g.ox + g.Lx) || y < (D)g.oy ||
        y > (D)(P)(g.oy + g.Ly) || z < (D)g.oz || z > (D)(P)(g.oz + g.Lz))
      return OR_ERR_RUNAWAY;
  }
  out[0] = (P)x; out[1] = (P)y; out[2] = (P)z;
  out[3] = (P)u; out[4] = (P)v; out[5] = (P)w;
  return OR_OK;
}

// deposit block, kernels.py:683-734 / deposit_span :327-381.
// gx is computed in promote(P, F): f32 in single mode, f64 otherwise.
template <typename P, typename F>
static inline void deposit_one(P xp, P yp, P zp, P vnx, P vny, P vnz, P q,
                               i64* acc, const F* invvol, const Geo<P, F>& g,
                               P one, F scale) {
  typedef decltype(P() - F()) G;
  const G gx = ((G)xp - (G)g.gox) / (G)g.gdx;
  const G gy = ((G)yp - (G)g.goy) / (G)g.gdy;
  const G gz = ((G)zp - (G)g.goz) / (G)g.gdz;
  i64 i = (i64)gx, j = (i64)gy, k = (i64)gz;
  if (i > g.nx - 1) i = g.nx - 1;
  if (j > g.ny - 1) j = g.ny - 1;
  if (k > g.nz - 1) k = g.nz - 1;
  const D fx = (D)gx - (D)i, fy = (D)gy - (D)j, fz = (D)gz - (D)k;
  const D ax = (D)one - fx, ay = (D)one - fy, az = (D)one - fz;
  const P pxx = vnx * vnx, pxy = vnx * vny, pxz = vnx * vnz;
  const P pyy = vny * vny, pyz = vny * vnz, pzz = vnz * vnz;
  const i64 NN = g.NX * g.NY * g.NZ;
  const D sc = (D)scale;
  for (int c = 0; c < 8; ++c) {
    const int ci = c & 1, cj = (c >> 1) & 1, ck = (c >> 2) & 1;
    const i64 n = g.node(i + ci, j + cj, k + ck);
    const D wx = ci ? fx : ax, wy = cj ? fy : ay, wz = ck ? fz : az;
    const D base = (D)q * (wx * wy * wz) * (D)invvol[n];
    acc[0 * NN + n] += (i64)std::nearbyint(base * sc);
    acc[1 * NN + n] += (i64)std::nearbyint(base * (D)vnx * sc);
    acc[2 * NN + n] += (i64)std::nearbyint(base * (D)vny * sc);
    acc[3 * NN + n] += (i64)std::nearbyint(base * (D)vnz * sc);
    acc[4 * NN + n] += (i64)std::nearbyint(base * (D)pxx * sc);
    acc[5 * NN + n] += (i64)std::nearbyint(base * (D)pxy * sc);
    acc[6 * NN + n] += (i64)std::nearbyint(base * (D)pxz * sc);
    acc[7 * NN + n] += (i64)std::nearbyint(base * (D)pyy * sc);
    acc[8 * NN + n] += (i64)std::nearbyint(base * (D)pyz * sc);
    acc[9 * NN + n] += (i64)std::nearbyint(base * (D)pzz * sc);
  }
}

template <typename P, typename F>
static int fused_t(void* xs_, void* ys_, void* zs_, void* us_, void* vs_, void* ws_,
                   const void* qs_, i64 start, i64 count, const void* E_,
                   const void* B_, i64* acc, const void* invvol_, const D* gf,
                   const D* gg, const i64* gi, D dt, D dth, D qdt2m, D beta, D one,
                   int n_iters, D scale, int mixed, int do_push, int do_deposit,
                   int apply_bc) {
  P* xs = (P*)xs_; P* ys = (P*)ys_; P* zs = (P*)zs_;
  P* us = (P*)us_; P* vs = (P*)vs_; P* ws = (P*)ws_;
  const P* qs = (const P*)qs_;
  const F* E = (const F*)E_;
  const F* B = (const F*)B_;
  const F* invvol = (const F*)invvol_;
  Geo<P, F> g(gf, gg, gi);
  int worst = OR_OK;
  for (i64 p = start; p < start + count; ++p) {
    if (do_push) {
      P out[6];
      int st = push_one<P, F>(xs[p], ys[p], zs[p], us[p], vs[p], ws[p], E, B, g,
                              (P)dt, (P)dth, (P)qdt2m, (P)beta, (P)one, n_iters,
                              apply_bc, mixed, out);
      if (st != OR_OK) {
        if (st > worst) worst = st;
        continue;
      }
      xs[p] = out[0]; ys[p] = out[1]; zs[p] = out[2];
      us[p] = out[3]; vs[p] = out[4]; ws[p] = out[5];
    }
    if (do_deposit)
      deposit_one<P, F>(xs[p], ys[p], zs[p], us[p], vs[p], ws[p], qs[p], acc,
                        invvol, g, (P)one, (F)scale);
  }
  return worst;
}

template <typename P, typename F>
static int gather_t(const void* xs_, const void* ys_, const void* zs_, i64 start,
                    i64 count, const void* E_, const void* B_, const D* gg,
                    const i64* gi, void* out_) {
  const P* xs = (const P*)xs_; const P* ys = (const P*)ys_; const P* zs = (const P*)zs_;
  const F* E = (const F*)E_;
  const F* B = (const F*)B_;
  P* out = (P*)out_;
  D gf[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  Geo<P, F> g(gf, gg, gi);
  const i64 NN = g.NX * g.NY * g.NZ;
  typedef decltype(P() - F()) G;
  for (i64 p = start; p < start + count; ++p) {
    const G gx = ((G)xs[p] - (G)g.gox) / (G)g.gdx;
    const G gy = ((G)ys[p] - (G)g.goy) / (G)g.gdy;
    const G gz = ((G)zs[p] - (G)g.goz) / (G)g.gdz;
    i64 i = (i64)gx, j = (i64)gy, k = (i64)gz;
    if (i > g.nx - 1) i = g.nx - 1;
    if (j > g.ny - 1) j = g.ny - 1;
    if (k > g.nz - 1) k = g.nz - 1;
    const D fx = (D)gx - (D)i, fy = (D)gy - (D)j, fz = (D)gz - (D)k;
    const D ax = 1.0 - fx, ay = 1.0 - fy, az = 1.0 - fz;
    D w[8];
    weights8(fx, fy, fz, ax, ay, az, w);
    P* o = out + (p - start) * 6;
    o[0] = (P)tri(E, g, i, j, k, w);
    o[1] = (P)tri(E + NN, g, i, j, k, w);
    o[2] = (P)tri(E + 2 * NN, g, i, j, k, w);
    o[3] = (P)tri(B, g, i, j, k, w);
    o[4] = (P)tri(B + NN, g, i, j, k, w);
    o[5] = (P)tri(B + 2 * NN, g, i, j, k, w);
  }
  return OR_OK;
}

}  // namespace

extern "C" {

// pbytes / fbytes: 8 = float64, 4 = float32 (particle / field storage).
// Supported pairs: (8,8) double, (4,4) single, (4,8) mixed.
int or_span(int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us, void* vs,
            void* ws, const void* qs, i64 start, i64 count, const void* E,
            const void* B, i64* acc, const void* invvol, const D* geo_f,
            const D* geo_g, const i64* geo_i, D dt, D dth, D qdt2m, D beta, D one,
            int n_iters, D scale, int mixed, int do_push, int do_deposit,
            int apply_bc) {
#define OR_ARGS                                                                   \
  xs, ys, zs, us, vs, ws, qs, start, count, E, B, acc, invvol, geo_f, geo_g, geo_i, \
      dt, dth, qdt2m, beta, one, n_iters, scale, mixed, do_push, do_deposit, apply_bc
  if (pbytes == 8 && fbytes == 8) return fused_t<double, double>(OR_ARGS);
  if (pbytes == 4 && fbytes == 4) return fused_t<float, float>(OR_ARGS);
  if (pbytes == 4 && fbytes == 8) return fused_t<float, double>(OR_ARGS);
#undef OR_ARGS
  return OR_ERR_ARGS;
}

int or_gather(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs,
              i64 start, i64 count, const void* E, const void* B, const D* geo_g,
              const i64* geo_i, void* out) {
  if (pbytes == 8 && fbytes == 8)
    return gather_t<double, double>(xs, ys, zs, start, count, E, B, geo_g, geo_i, out);
  if (pbytes == 4 && fbytes == 4)
    return gather_t<float, float>(xs, ys, zs, start, count, E, B, geo_g, geo_i, out);
  if (pbytes == 4 && fbytes == 8)
    return gather_t<float, double>(xs, ys, zs, start, count, E, B, geo_g, geo_i, out);
  return OR_ERR_ARGS;
}

// Fused pass split over nthreads host threads, one private int64 grid per
// thread merged at the end (the reference pipeline's per-batch accumulator +
// integer merge, pipeline.py:178-268).  Used as the timed CPU baseline.
int or_fused_parallel(int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us,
                      void* vs, void* ws, const void* qs, i64 start, i64 count,
                      const void* E, const void* B, i64* acc, const void* invvol,
                      const D* geo_f, const D* geo_g, const i64* geo_i, D dt, D dth,
                      D qdt2m, D beta, D one, int n_iters, D scale, int mixed,
                      int nthreads) {
  const i64 nn = (geo_i[0] + 1) * (geo_i[1] + 1) * (geo_i[2] + 1) * 10;
  if (nthreads < 1) nthreads = 1;
  std::vector<int> st(nthreads, 0);
  std::vector<std::vector<i64>> priv(nthreads);
  std::vector<std::thread> pool;
  const i64 per = (count + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    pool.emplace_back([&, t]() {
      priv[t].assign(nn, 0);
      const i64 s = start + per * t;
      const i64 e = (s + per < start + count) ? s + per : start + count;
      if (s < e)
        st[t] = or_span(pbytes, fbytes, xs, ys, zs, us, vs, ws, qs, s, e - s, E, B,
                        priv[t].data(), invvol, geo_f, geo_g, geo_i, dt, dth, qdt2m,
                        beta, one, n_iters, scale, mixed, 1, 1, 1);
    });
  }
  for (auto& th : pool) th.join();
  int worst = 0;
  for (int t = 0; t < nthreads; ++t) {
    if (st[t] < 0) return st[t];
    if (st[t] > worst) worst = st[t];
    for (i64 n = 0; n < nn; ++n) acc[n] += priv[t][n];
  }
  return worst;
}

// Linear cell index, x fastest, computed in f64 (geometry.py:152-159).
// origin/spacing are the geometry's python floats (f64).  Returns -1 if a
// position lies below the origin (reference raises DomainError).
int or_cell_keys(int pbytes, const void* xs, const void* ys, const void* zs, i64 n,
                 const D* origin, const D* spacing, const i64* counts, i64* keys) {
  for (i64 p = 0; p < n; ++p) {
    D x, y, z;
    if (pbytes == 8) {
      x = ((const D*)xs)[p]; y = ((const D*)ys)[p]; z = ((const D*)zs)[p];
    } else {
      x = ((const float*)xs)[p]; y = ((const float*)ys)[p]; z = ((const float*)zs)[p];
    }
    i64 i = (i64)((x - origin[0]) / spacing[0]);
    i64 j = (i64)((y - origin[1]) / spacing[1]);
    i64 k = (i64)((z - origin[2]) / spacing[2]);
    if (i > counts[0] - 1) i = counts[0] - 1;
    if (j > counts[1] - 1) j = counts[1] - 1;
    if (k > counts[2] - 1) k = counts[2] - 1;
    if (i < 0 || j < 0 || k < 0) return -1;
    keys[p] = i + counts[0] * (j + counts[1] * k);
  }
  return 0;
}

// Stable counting sort of keys in [0, nkeys): order[r] = source index of the
// r-th particle (np.argsort(kind="stable") semantics, particles.py:164).
int or_stable_order(const i64* keys, i64 n, i64 nkeys, i64* order) {
  std::vector<i64> off(nkeys + 1, 0);
  for (i64 p = 0; p < n; ++p) {
    if (keys[p] < 0 || keys[p] >= nkeys) return -1;
    off[keys[p] + 1]++;
  }
  for (i64 c = 0; c < nkeys; ++c) off[c + 1] += off[c];
  for (i64 p = 0; p < n; ++p) order[off[keys[p]]++] = p;
  return 0;
}

}  // extern "C"
