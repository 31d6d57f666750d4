// Cell-binned fast path for f32 particles (DeviceSimulation layout "bins").
//
// The reference keeps every species as one flat SoA and restores cell order
// with a stable sort every sort_period cycles (particles.py:157-167,
// pipeline.py:300-304); between sorts the particles drift out of order, and
// on a GPU every out-of-order particle costs the mover a field-record fetch
// and the deposit a cross-lane regrouping.  Here a species lives in per-cell
// bins instead: cell c owns slots [start[c], start[c + 1]) of the SoA arrays
// (x y z u v w q + int64 ids, the reference's ParticleBuffer columns), the
// first count[c] of them live.  Every cycle, per species:
//
//   mover_bins    one warp per bin: the bin's cell record (bp_split.cu's
//                 trilinear coefficient form) is loaded ONCE into registers
//                 and serves every midpoint gather inside the cell; the push
//                 is the reference's (kernels.py:498-676) in native f32.
//                 Particles whose new cell differs ("leavers") are written
//                 to a leaver list and their slots are refilled from the
//                 bin's tail, so a bin stays dense.
//   migrate_bins  every leaver is appended to its new cell's bin.
//   deposit_bins  a quarter-warp (8 lanes) per bin: all of a bin's particles
//                 share one cell, so each lane accumulates the 80 products
//                 (10 moments x 8 corners, kernels.py:689-734) of its
//                 particles in registers with FFMA2; one shared-memory
//                 transpose per bin reduces the 8 lanes, and each lane adds
//                 one corner's 10 sums onto the int64 lattice (x invvol x
//                 2^43, rint; fields.py:20-25) with REDG.ADD.64.
//
// So the particles are cell-sorted at every cycle, not every tenth, and
// neither kernel does per-particle regrouping.  Bins have slack (the build
// sizes them count + max(min, frac x count)); a leaver that finds its bin
// full goes to an overflow list, deposited on its own, and the host rebuilds
// the species' bins at the end of the cycle.  Particles that could not be
// listed as leavers stay in their old bin ("misplaced"): both kernels test
// each particle's cell and handle those on a slow path, and the host
// rebuilds too.  Arithmetic: as bp_split.cu (fast f32, within the north
// star's 1e-4 of the reference); the f32 per-bin sums are rounded once onto
// the lattice.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "bp_f32_common.cuh"
#include "bp_bins_plumb.cuh"
#include "bp_launch.h"

namespace bp {
namespace bins {

using sk::F2;
using sk::f2;
using sk::fma2;
typedef sk::Params<float> P;

typedef BinsT<float> Bins;
typedef LeaverT<float> Leaver;

// one 32-byte particle record per thread: a single 256-bit access (sm_100
// ld/st .v8), so the lanes of a warp cover whole sectors with one instruction
__device__ __forceinline__ void ld_rec_stream(const float4* p, float4& a, float4& b) {
  asm volatile("ld.global.L1::evict_first.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void ld_rec_ro(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void st_rec_stream(float4* p, const float4& a, const float4& b) {
  asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}
// slot q's record (2 float4): one 32 x 32 -> 64-bit multiply-add (the f32
// mover keeps slot indices in 32 bits; bins_plan refuses layouts of 2^31 or
// more slots)
__device__ __forceinline__ float4* slot_rec(float4* rec, int q) {
  return reinterpret_cast<float4*>(reinterpret_cast<char*>(rec) + (size_t)(unsigned)q * 32u);
}

constexpr int kHoleCap = 256;    // leavers per bin per cycle tracked for the refill (more: misplaced, rebuild)
constexpr int kMoveClaim = 8;    // bins per mover work claim (at most; Bins::move_claim)
constexpr int kLvChunk = 128;    // leaver slots per warp reservation
constexpr int kDepClaim = 16;    // bins per deposit work claim, 4 rounds of 4 (at most)
// deposit flush rows: lane L's 80 sums corner-major (10 moments + 2 pad per
// corner), rows 100 floats apart so the 8 lanes of a quarter write 4 banks
// apart and a reader's corner is 3 contiguous float4
constexpr int kCornerS = 12;
constexpr int kRowS = 8 * kCornerS + 4;
constexpr int kWarpSm = 32 * kRowS;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Grid-unit box of cell (i, j, k): cell_of (bp_f32_common.cuh) puts gx in
// cell i iff min(trunc(gx), n - 1) == i, i.e. gx in [lo, hi) with lo = i (the
// largest float above -1 for i = 0: trunc maps (-1, 1) to 0) and hi = i + 1
// (+inf for the last cell); fx = gx - i exactly as cell_of.
struct Box {
  float lo[3], hi[3], cf[3];
};
struct Ijk {
  int i, j, k;
};
__device__ __forceinline__ Ijk ijk_of(const P& a, int c) {
  return Ijk{c % a.nx, (c / a.nx) % a.ny, c / a.cny};
}
// the cell t positions further in x-fastest order
__device__ __forceinline__ Ijk ijk_advance(const P& a, Ijk q, int t) {
  q.i += t;
  while (q.i >= a.nx) {
    q.i -= a.nx;
    if (++q.j == a.ny) {
      q.j = 0;
      ++q.k;
    }
  }
  return q;
}
__device__ __forceinline__ Box cell_box(const P& a, Ijk q) {
  Box b;
  const int idx[3] = {q.i, q.j, q.k};
  const int n[3] = {a.nx, a.ny, a.nz};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    b.cf[d] = (float)idx[d];
    b.lo[d] = idx[d] == 0 ? __int_as_float(0xbf7fffff) : b.cf[d];
    b.hi[d] = idx[d] == n[d] - 1 ? __int_as_float(0x7f800000) : b.cf[d] + 1.f;
  }
  return b;
}

__device__ __forceinline__ bool in_box(const Box& b, float gx, float gy, float gz) {
  return gx >= b.lo[0] && gx < b.hi[0] && gy >= b.lo[1] && gy < b.hi[1] && gz >= b.lo[2] &&
         gz < b.hi[2];
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void load_record(const P& a, int cell, float4 (&R)[12]) {
  const float4* r = static_cast<const float4*>(a.rec) + (size_t)cell * 12;
#pragma unroll
  for (int q = 0; q < 12; q += 2) sk::ldg_pair(r + q, R[q], R[q + 1]);
}

// The implicit push (bp_split.cu push(), kernels.py:498-676 in native f32)
// with the lane's record R of cell `held` kept across particles: a bin's
// particles start in the bin's cell, so R (the bin's record, staged in shared
// memory) serves nearly every midpoint, and only a lane whose midpoint lies
// in another cell reloads it.  Every lane of the warp runs the whole push
// (no early return: a failing particle keeps a safe position and reports
// its status), so the reload is a warp-uniform branch.
// The shared-memory field window of a mover claim of nb <= 8 bins along x
// (cells c0 .. c0 + nb - 1 at (i0 .. i0 + nb - 1, j, k)): slots 0..9 the x
// run c0 - 1 .. c0 + nb (the home records at 1 .. nb), 10..17 / 18..25 the
// same x range at j - 1 / j + 1, 26..33 / 34..41 at k - 1 / k + 1, each
// present when inside the grid (flags) — staged by TMA bulk copies, so a
// midpoint that moved to a face neighbour reloads from shared memory.
constexpr int kWinRecs = 10 + 4 * kMoveClaim;
enum { WIN_XLO = 1, WIN_XHI = 2, WIN_YM = 4, WIN_YP = 8, WIN_ZM = 16, WIN_ZP = 32 };
struct Win {
  const float4* base;
  int i0, j, k, nb, fl;
};
// window slot of cell (i, j, k), or -1 (global memory)
__device__ __forceinline__ int win_slot(const Win& W, int i, int j, int k) {
  const int di = i - W.i0;
  if (j == W.j && k == W.k) {
    if (di >= 0 && di < W.nb) return di + 1;
    if (di == -1 && (W.fl & WIN_XLO)) return 0;
    if (di == W.nb && (W.fl & WIN_XHI)) return W.nb + 1;
    return -1;
  }
  if (di < 0 || di >= W.nb) return -1;
  if (k == W.k) {
    if (j == W.j - 1 && (W.fl & WIN_YM)) return 10 + di;
    if (j == W.j + 1 && (W.fl & WIN_YP)) return 18 + di;
  } else if (j == W.j) {
    if (k == W.k - 1 && (W.fl & WIN_ZM)) return 26 + di;
    if (k == W.k + 1 && (W.fl & WIN_ZP)) return 34 + di;
  }
  return -1;
}

// NIT > 0: the iteration count as a compile-time constant (fully unrolled);
// NIT == 0: a.n_iters at run time
// FC (grids below 2^24 cells): the midpoint's cell index and fractions in
// float — trunc, clamp and the x-fastest index are exact there, fx = gx - i
// bitwise as cell_of — so the per-iteration reload test needs no F2I / I2F
// round trip; `held` / `home` are then float cell indices.
template <bool FC>
using HeldT = typename std::conditional<FC, float, int>::type;

template <bool RX, bool RY, bool RZ, int NIT, bool FC>
__device__ __forceinline__ int push_bin(const P& a, float4 (&R)[12], HeldT<FC>& held, HeldT<FC> home,
                                        const float4* home_rec, const Win& W, float& xp,
                                        float& yp, float& zp, float& un, float& vn, float& wn,
                                        bool skipbc) {
  float vbx = un, vby = vn, vbz = wn;
  int st = ST_OK;
  const int nit = NIT > 0 ? NIT : a.n_iters;
#pragma unroll
  for (int it = 0; it < nit; ++it) {
    const F2 XM = fma2(f2(vbx, vby), f2(a.dth, a.dth), f2(xp, yp));
    float xm = XM.x, ym = XM.y;
    float zm = fmaf(vbz, a.dth, zp);
    if (!skipbc) {
      xm = sk::fold_mid<RX>(xm, a.o[0], a.L[0], a.hi[0], a.hi2[0]);
      ym = sk::fold_mid<RY>(ym, a.o[1], a.L[1], a.hi[1], a.hi2[1]);
      zm = sk::fold_mid<RZ>(zm, a.o[2], a.L[2], a.hi[2], a.hi2[2]);
      if (xm < a.o[0] || xm > a.hi[0] || ym < a.o[1] || ym > a.hi[1] || zm < a.o[2] ||
          zm > a.hi[2]) {
        st = ST_MIDPOINT;  // (kernels.py:535-538) carried on at a safe position
        xm = xp; ym = yp; zm = zp;
      }
    }
    float fx, fy, fz;
    int i = 0, j = 0, k = 0;
    HeldT<FC> cell;
    if constexpr (FC) {
      const F2 G = fma2(f2(xm, ym), f2(a.idx[0], a.idx[1]), f2(-a.ogs[0], -a.ogs[1]));
      const float gz = fmaf(zm, a.idx[2], -a.ogs[2]);
      const float tx = fminf(truncf(G.x), a.nm1[0]), ty = fminf(truncf(G.y), a.nm1[1]);
      const float tz = fminf(truncf(gz), a.nm1[2]);
      fx = G.x - tx;
      fy = G.y - ty;
      fz = gz - tz;
      cell = fmaf(tz, a.cnyf, fmaf(ty, a.nxf, tx));
    } else {
      cell = sk::cell_of(a, xm, ym, zm, fx, fy, fz, i, j, k);
    }
    float ex, ey, hx, hy, ez, hz;
    const bool need = cell != held;
    if (__any_sync(0xffffffffu, need)) {
      if (need) {
        held = cell;
        if (cell == home) {  // back in the bin's cell: its record is in shared memory
#pragma unroll
          for (int q = 0; q < 12; ++q) R[q] = home_rec[q];
        } else {
#if BP_MOVER_WINDOW
          const int sl = win_slot(W, i, j, k);
          if (sl >= 0) {
#pragma unroll
            for (int q = 0; q < 12; ++q) R[q] = W.base[sl * 12 + q];
          } else {
            load_record(a, cell, R);
          }
#else
          load_record(a, (int)cell, R);
#endif
        }
      }
    }
    sk::tri_pair(R[0], R[1], R[2], R[3], fx, fy, fz, ex, ey);
    sk::tri_pair(R[4], R[5], R[6], R[7], fx, fy, fz, hx, hy);
    sk::tri_pair(R[8], R[9], R[10], R[11], fx, fy, fz, ez, hz);
    const F2 Txy = fma2(f2(a.qdt2m, a.qdt2m), f2(ex, ey), f2(un, vn));
    const float tx = Txy.x, ty = Txy.y;
    const float tz = fmaf(a.qdt2m, ez, wn);
    const float bsq = fmaf(hx, hx, fmaf(hy, hy, hz * hz));
    const float inv = sk::rcp_fast(fmaf(a.beta2, bsq, 1.f));
    const float tdb = fmaf(tx, hx, fmaf(ty, hy, tz * hz));
    const float bt = a.beta * tdb;
    const float cx = fmaf(ty, hz, -tz * hy), cy = fmaf(tz, hx, -tx * hz),
                cz = fmaf(tx, hy, -ty * hx);
    vbx = fmaf(a.beta, fmaf(bt, hx, cx), tx) * inv;
    vby = fmaf(a.beta, fmaf(bt, hy, cy), ty) * inv;
    vbz = fmaf(a.beta, fmaf(bt, hz, cz), tz) * inv;
  }
  if (st != ST_OK) return st;
  float xo = fmaf(vbx, a.dt, xp), yo = fmaf(vby, a.dt, yp), zo = fmaf(vbz, a.dt, zp);
  float uo = 2.f * vbx - un, vo = 2.f * vby - vn, wo = 2.f * vbz - wn;
  if (!skipbc) {
    sk::fold_commit<RX>(xo, uo, a.o[0], a.L[0], a.hi[0], a.hi2[0]);
    sk::fold_commit<RY>(yo, vo, a.o[1], a.L[1], a.hi[1], a.hi2[1]);
    sk::fold_commit<RZ>(zo, wo, a.o[2], a.L[2], a.hi[2], a.hi2[2]);
    if (xo < a.o[0] || xo > a.hi[0] || yo < a.o[1] || yo > a.hi[1] || zo < a.o[2] ||
        zo > a.hi[2])
      return ST_RUNAWAY;
  }
  xp = xo; yp = yo; zp = zo;
  un = uo; vn = vo; wn = wo;
  return ST_OK;
}

// Speed bound below which no position of a push from cell q can leave the
// box (interior() of bp_f32_common.cuh, per bin instead of per particle): a
// particle of cell (i, j, k) lies at least min(i, n - 1 - i) cells from the
// faces of each axis, and every midpoint and the committed position lie
// within dt (|v|_1 + |qdt2m| max|E|) of the start; 1e-4 of the distance
// (hmin = 0.9999 x the smallest spacing) and bc_eps cover the rounding.  A
// bin touching a face gets a negative bound: every push there checks.
__device__ __forceinline__ float bin_speed_bound(const P& a, Ijk q, float qe, float hmin,
                                                 float epsmax) {
  const int cells = min(min(min(q.i, a.nx - 1 - q.i), min(q.j, a.ny - 1 - q.j)),
                        min(q.k, a.nz - 1 - q.k));
  return __fdividef(fmaf((float)cells, hmin, -epsmax), a.dt) - qe;
}

// ---------------------------------------------------------------------------
// Mover: one warp per bin.  A warp claims kMoveClaim consecutive bins; their
// cell records (contiguous: records are in cell order) are staged in shared
// memory by one TMA bulk copy per claim, one claim ahead (double buffer,
// mbarrier completion).  Stayers are written back in place; each leaver is
// listed (x..w, q, id, new cell) and leaves a hole; after the bin's last tile
// the holes below the new count are refilled with the bin's trailing stayers
// (about as many particle copies as leavers).  The next tile's particles
// (across bins of the claim) are loaded while the current tile is pushed.
#ifndef BP_MOVER_WINDOW
#define BP_MOVER_WINDOW 0  // 1: face-neighbour field window staged per claim
#endif
#ifndef BP_MOVER_TPB
#define BP_MOVER_TPB 128  // threads per block of mover_bins (measured: 128 x 5 > 256 x 2)
#endif
#ifndef BP_MOVER_MINB
#define BP_MOVER_MINB 5   // resident blocks per SM it is compiled for (<= 102 registers)
#endif
#ifndef BP_MOVER_SMP
#define BP_MOVER_SMP 1    // next particle staged in shared memory by cp.async (0: registers)
#endif
#ifndef BP_MOVER_FCELL
#define BP_MOVER_FCELL 1  // float midpoint cell index where exact (< 2^24 cells)
#endif
#if BP_MOVER_WINDOW && BP_MOVER_FCELL
#error "the field window needs the integer cell coordinates (build with -DBP_MOVER_FCELL=0)"
#endif
#ifndef BP_MOVER_IDPF
#define BP_MOVER_IDPF 1   // L2 prefetch of each bin's ids at the bin's start
#endif
constexpr int kMoverWarps = BP_MOVER_TPB / 32;

__device__ __forceinline__ void prefetch_l2(uintptr_t p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <bool RX, bool RY, bool RZ, int NIT, bool FC>
__global__ void __launch_bounds__(BP_MOVER_TPB, BP_MOVER_MINB) mover_bins(const __grid_constant__ P a,
                                                     const __grid_constant__ Bins b) {
#if BP_MOVER_WINDOW
  __shared__ __align__(128) float4 win_s[kMoverWarps][kWinRecs * 12];
#else
  __shared__ __align__(128) float4 recs_s[kMoverWarps][2][kMoveClaim * 12];
#endif
  __shared__ __align__(8) unsigned long long bars_s[kMoverWarps][2];
  // hole slots within the bin (< 65536) and the leavers' list slots (< 2^31:
  // the list holds a quarter of the species + 1M)
#if BP_MOVER_SMP
  __shared__ __align__(16) float4 pst_s[kMoverWarps][64];  // next particle of each lane
#endif
  __shared__ unsigned short holes_s[kMoverWarps][kHoleCap];
  __shared__ int lvslot_s[kMoverWarps][kHoleCap];
  const int wid = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  unsigned short* const holes = holes_s[wid];
  int* const lvslot = lvslot_s[wid];
  unsigned long long* const bars = bars_s[wid];
  const unsigned lt = lanemask_lt();
  const float qe = fabsf(a.qdt2m) * __ldg(a.emax) * 1.00001f;
  const float hmin = 0.9999f * fminf(fminf(a.L[0] / (float)a.nx, a.L[1] / (float)a.ny),
                                     a.L[2] / (float)a.nz);
  const float epsmax = fmaxf(fmaxf(a.bc_eps[0], a.bc_eps[1]), a.bc_eps[2]);
  const float4* const rec_g = static_cast<const float4*>(a.rec);
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  fence_proxy_async();
  __syncwarp();
#if BP_MOVER_WINDOW
  // claim up to 8 bins and stage their field window (single buffer: the
  // next claim's copies start when this claim is done)
  Win W{win_s[wid], 0, 0, 0, 0, 0};
  auto claim_win = [&]() -> int {
    unsigned long long cc = 0;
    if (lane == 0) cc = atomicAdd(&b.stat[ST_WORK_MOVE], (unsigned long long)b.move_claim);
    const int c = (int)min(__shfl_sync(0xffffffffu, cc, 0), (unsigned long long)b.ncell);
    if (c >= b.ncell) return c;
    const int nb = min(b.move_claim, b.ncell - c);
    W.i0 = c % a.nx;
    W.j = (c / a.nx) % a.ny;
    W.k = c / a.cny;
    W.nb = nb;
    // a claim crossing an x row stages its home records only
    const bool row = W.i0 + nb <= a.nx;
    W.fl = row ? ((W.i0 > 0 ? WIN_XLO : 0) | (W.i0 + nb < a.nx ? WIN_XHI : 0) |
                  (W.j > 0 ? WIN_YM : 0) | (W.j < a.ny - 1 ? WIN_YP : 0) |
                  (W.k > 0 ? WIN_ZM : 0) | (W.k < a.nz - 1 ? WIN_ZP : 0))
               : 0;
    if (!row) W.i0 = -1000;  // no cell matches the window geometry
    if (lane == 0) {
      const unsigned rb = 12u * 16u;
      const int xa = (W.fl & WIN_XLO) ? c - 1 : c;
      const int xb = (W.fl & WIN_XHI) ? c + nb : c + nb - 1;
      unsigned bytes = (unsigned)(xb - xa + 1) * rb;
      const int runs[4] = {c - a.nx, c + a.nx, c - a.cny, c + a.cny};
      const int rfl[4] = {WIN_YM, WIN_YP, WIN_ZM, WIN_ZP};
      for (int q = 0; q < 4; ++q)
        if (W.fl & rfl[q]) bytes += (unsigned)nb * rb;
      fence_proxy_async();
      mbar_expect_tx(&bars[0], bytes);
      bulk_load(win_s[wid] + (xa - (c - 1)) * 12, rec_g + (size_t)xa * 12,
                (unsigned)(xb - xa + 1) * rb, &bars[0]);
      for (int q = 0; q < 4; ++q)
        if (W.fl & rfl[q])
          bulk_load(win_s[wid] + (10 + 8 * q) * 12, rec_g + (size_t)runs[q] * 12,
                    (unsigned)nb * rb, &bars[0]);
    }
    return c;
  };
#else
  const Win W{nullptr, 0, 0, 0, 0, 0};  // (unused)
  // claim kMoveClaim bins and stage their records into buffer `bf`
  auto claim = [&](int bf) -> int {
    unsigned long long c = 0;
    if (lane == 0) {
      c = atomicAdd(&b.stat[ST_WORK_MOVE], (unsigned long long)b.move_claim);
      if (c < (unsigned long long)b.ncell) {
        const int nb = min(b.move_claim, b.ncell - (int)c);
        const unsigned bytes = (unsigned)nb * 12u * 16u;
        fence_proxy_async();
        mbar_expect_tx(&bars[bf], bytes);
        bulk_load(recs_s[wid][bf], rec_g + (size_t)c * 12, bytes, &bars[bf]);
      }
    }
    return (int)min(__shfl_sync(0xffffffffu, c, 0), (unsigned long long)b.ncell);
  };
#endif
  int st_worst = ST_OK;  // the lane's worst push status (ST_OK = 0 < errors)
  // the warp's current chunk of leaver slots [lv_base, lv_base + kLvChunk),
  // lv_used of them taken (starts "full": the first leaver claims a chunk)
  int lv_base = 0, lv_next = 0;
  int lv_used = kLvChunk;
  // mbarrier phase parity of buffer k in bit k (a register: an array indexed
  // by bf would live in local memory)
  unsigned phases = 0u;
  int bf = 0;
#if BP_MOVER_WINDOW
  int c0 = claim_win();
#else
  int c0 = claim(0);
#endif
  // prefetched particle (one per lane) and the slot it came from
  float4 n1a = make_float4(0.f, 0.f, 0.f, 0.f), n1b = n1a;
  // streaming loads (read once per cycle): the 32-byte record of slot q, or
  // (lanes past the end of the tile's bin) of the tile's first slot q0 — a
  // broadcast in lane 0's sector — so those lanes push a copy of lane 0's
  // particle (not stored) and the whole warp runs the push
#if BP_MOVER_SMP
  // the next particle goes global -> shared (cp.async, no registers held
  // across the push), read back at the next tile's top
  float4* const pmine = pst_s[wid] + 2 * lane;
  auto fetch = [&](int q, bool ok, int q0) {
    const float4* g = slot_rec(b.rec, ok ? q : q0);
    cp_async16(pmine, g);
    cp_async16(pmine + 1, g + 1);
  };
#else
  auto fetch = [&](int q, bool ok, int q0) { ld_rec_stream(slot_rec(b.rec, ok ? q : q0), n1a, n1b); };
#endif
  float4 R[12];
  while (c0 < b.ncell) {
    const int c1 = min(c0 + b.move_claim, b.ncell);
#if BP_MOVER_WINDOW
    mbar_wait(&bars[0], phases & 1u);
    phases ^= 1u;
#else
    const int cn = claim(bf ^ 1);  // the next claim's records load meanwhile
    mbar_wait(&bars[bf], (phases >> bf) & 1u);
    phases ^= 1u << bf;
#endif
    int s0 = (int)b.start[c0];
    int n = min(b.count[c0], (int)b.start[c0 + 1] - s0);
    if (n > 0) fetch(s0 + lane, (int)lane < n, s0);
    bool pf_ok = true;  // (warp-uniform) n1 holds this bin's first tile
    Ijk q3 = ijk_of(a, c0);
    for (int c = c0; c < c1; ++c, q3 = ijk_advance(a, q3, 1)) {
      // metadata of the next bin of the claim (its first tile is prefetched
      // during this bin's last tile)
      int s1 = 0;
      int n_1 = 0;
      if (c + 1 < c1) {
        s1 = (int)b.start[c + 1];
        n_1 = min(b.count[c + 1], (int)b.start[c + 2] - s1);
      }
      if (n > 0) {
        if (!pf_ok) fetch(s0 + lane, (int)lane < n, s0);
#if BP_MOVER_IDPF
        {
          // the bin's ids are read only by the refill at the bin's end (the
          // leavers' ids and the trailing stayers'): bring their lines from
          // DRAM into L2 now, one 128-byte line per lane (bins up to 512)
          const uintptr_t i0 = reinterpret_cast<uintptr_t>(b.id + s0);
          const uintptr_t ln = (i0 & ~(uintptr_t)127) + ((uintptr_t)lane << 7);
          if (ln <= reinterpret_cast<uintptr_t>(b.id + s0 + n - 1)) prefetch_l2(ln);
        }
#endif
#if BP_MOVER_WINDOW
        const float4* rs = win_s[wid] + (1 + c - c0) * 12;
#else
        const float4* rs = recs_s[wid][bf] + (c - c0) * 12;
#endif
#pragma unroll
        for (int q = 0; q < 12; ++q) R[q] = rs[q];
        const float vmax = bin_speed_bound(a, q3, qe, hmin, epsmax);
        HeldT<FC> held = (HeldT<FC>)c;
        const HeldT<FC> homec = (HeldT<FC>)c;
        int nh = 0;
#pragma unroll 1
        for (int t0 = 0; t0 < n; t0 += 32) {
          const int r = t0 + (int)lane;
          const bool valid = r < n;
          const int p = s0 + r;
#if BP_MOVER_SMP
          cp_async_wait_all();
          n1a = pmine[0];
          n1b = pmine[1];
#endif
          float xp = n1a.x, yp = n1a.y, zp = n1a.z, un = n1a.w, vn = n1b.x, wn = n1b.y;
          const float qp = n1b.z;
#if !BP_MOVER_SMP
          if (t0 + 32 < n) fetch(p + 32, r + 32 < n, s0 + t0 + 32);
          else if (n_1 > 0) fetch(s1 + lane, (int)lane < n_1, s1);
#endif
          const bool all_in =
              __all_sync(0xffffffffu, fabsf(un) + fabsf(vn) + fabsf(wn) < vmax);
#if BP_MOVER_SMP
          // the lane's slot is refilled only after the vote has consumed its
          // particle (both shared loads have returned)
          if (t0 + 32 < n) fetch(p + 32, r + 32 < n, s0 + t0 + 32);
          else if (n_1 > 0) fetch(s1 + lane, (int)lane < n_1, s1);
#endif
          const int st =
              push_bin<RX, RY, RZ, NIT, FC>(a, R, held, homec, rs, W, xp, yp, zp, un, vn, wn,
                                            all_in);
          int dest = c;
          if (st == ST_OK) {
            // the new cell (cell_of's formula, bp_f32_common.cuh)
            const float gx = fmaf(xp, a.idx[0], -a.ogs[0]);
            const float gy = fmaf(yp, a.idx[1], -a.ogs[1]);
            const float gz = fmaf(zp, a.idx[2], -a.ogs[2]);
            const int i = min((int)gx, a.nx - 1), j = min((int)gy, a.ny - 1),
                      k = min((int)gz, a.nz - 1);
            dest = i + a.nx * j + a.cny * k;
          } else if (valid) {
            // not stored (kernels.py:618-621); the cycle raises.  Reported
            // once per lane at the end: no atomic path in the tile loop
            st_worst = max(st_worst, st);
          }
        const bool leave = valid && st == ST_OK && dest != c;
        const unsigned L = __ballot_sync(0xffffffffu, leave);
        bool listed = false;
        if (L) {
          // leaver slots from the warp's private chunk of the list (one
          // global atomic per kLvChunk slots, not one per tile)
          const int nl = __popc(L);
          const int rank = __popc(L & lt);
          if (lv_used + nl > kLvChunk) {
            // the rest of the current chunk, then a fresh chunk
            unsigned long long nb = 0;
            if (lane == 0) nb = atomicAdd(&b.stat[ST_LEAVERS], (unsigned long long)kLvChunk);
            nb = __shfl_sync(0xffffffffu, nb, 0);
            lv_next = (int)min(nb, (unsigned long long)0x7fffff00);
          }
          const int room = kLvChunk - lv_used;  // slots left in the current chunk
          const int slot = rank < room ? lv_base + lv_used + rank : lv_next + (rank - room);
          // accepted leavers are a prefix in rank order (hole index grows
          // with the rank), so their hole indices stay contiguous
          listed = leave && slot < b.lv_cap && nh + rank < kHoleCap && r < 65536;
          if (listed) {
            // the id is added at the end of the bin (one load latency per
            // bin instead of per tile)
            float4* rec = reinterpret_cast<float4*>(b.lv + slot);
            rec[0] = make_float4(xp, yp, zp, un);
            rec[1] = make_float4(vn, wn, qp, __int_as_float(dest));
            holes[nh + rank] = (unsigned short)r;
            lvslot[nh + rank] = slot;
          } else if (leave) {
            // stays here as a misplaced particle (slow paths; host rebuilds)
            atomicAdd(&b.stat[ST_MISPLACED], 1ULL);
            if (slot < b.lv_cap) b.lv[slot].b.w = __int_as_float(-1);
          }
          nh += __popc(__ballot_sync(0xffffffffu, listed));
          if (lv_used + nl > kLvChunk) {
            lv_base = lv_next;
            lv_used = nl - room;
          } else {
            lv_used += nl;
          }
        }
        // every lane of the tile stores (a listed leaver's slot becomes a
        // hole, refilled below or past the new count), so whole sectors are
        // written; write-back stores, so the refill and the migration find
        // the bin's lines in L2
        if (valid && st == ST_OK) {
          st_rec_stream(slot_rec(b.rec, p), make_float4(xp, yp, zp, un),
                        make_float4(vn, wn, qp, 0.f));
        }
      }
        __syncwarp();
        if (nh > 0) {
          // leavers' ids into their records; refill: the holes below the
          // new count take the trailing stayers (holes are ascending; the
          // k-th trailing stayer is the k-th slot >= n_stay that is not a
          // hole).  All loads are issued before any store: the refill writes
          // into leaver slots.
          const int n_stay = n - nh;
          int nlow = 0;
          for (int k0 = 0; k0 < nh; k0 += 32) {
            const int k = k0 + (int)lane;
            nlow += __popc(__ballot_sync(0xffffffffu, k < nh && (int)holes[k] < n_stay));
          }
          for (int k0 = 0; k0 < nh; k0 += 32) {
            const int k = k0 + (int)lane;
            // this lane's leaver (k < nh) and refill pair (k < nlow)
            long long lid = 0;
            if (k < nh) lid = b.id[s0 + holes[k]];
            int src = 0, dst = 0;
            float4 ra = make_float4(0.f, 0.f, 0.f, 0.f), rb = ra;
            long long rid = 0;
            if (k < nlow) {
              int t = n_stay + k;
              for (int j = nlow; j < nh; ++j) {
                if ((int)holes[j] <= t) ++t;
                else break;
              }
              src = s0 + t;
              dst = s0 + holes[k];
              ra = slot_rec(b.rec, src)[0];
              rb = slot_rec(b.rec, src)[1];
              rid = b.id[src];
            }
            if (k < nh) b.lv[lvslot[k]].id = lid;
            __syncwarp();
            if (k < nlow) {
              slot_rec(b.rec, dst)[0] = ra;
              slot_rec(b.rec, dst)[1] = rb;
              b.id[dst] = rid;
            }
          }
        if (lane == 0) b.count[c] = n_stay;
        }
        __syncwarp();
      }
      pf_ok = n > 0 && n_1 > 0;
      s0 = s1;
      n = n_1;
    }
    __syncwarp();  // every lane is done with buffer bf before it is refilled
#if BP_MOVER_WINDOW
    c0 = claim_win();
#else
    c0 = cn;
    bf ^= 1;
#endif
  }
  // unused slots of the last leaver chunk carry no particle
  for (int k = lv_used + (int)lane; k < kLvChunk; k += 32)
    if (lv_base + k < b.lv_cap) b.lv[lv_base + k].b.w = __int_as_float(-1);
  if (st_worst != ST_OK) atomicMax(a.status, st_worst);
}

// ---------------------------------------------------------------------------
// Deposit of the overflow list and of the particles the deposit found
// misplaced: one particle straight onto the lattice with the reference's
// per-contribution rounding (kernels.py:689-734).  Rare.
__device__ __forceinline__ void deposit_one(const P& a, float x, float y, float z, float u,
                                            float v, float w, float q) {
  float fx, fy, fz;
  int i, j, k;
  sk::cell_of(a, x, y, z, fx, fy, fz, i, j, k);
  const float wx[2] = {1.f - fx, fx}, wy[2] = {1.f - fy, fy}, wz[2] = {1.f - fz, fz};
  const float mv[10] = {1.f, u, v, w, u * u, u * v, u * w, v * v, v * w, w * w};
  for (int c = 0; c < 8; ++c) {
    const int node = ((i + (c & 1)) * a.NY + (j + ((c >> 1) & 1))) * a.NZ + k + ((c >> 2) & 1);
    const double iv =
        (a.iv_d ? __ldg(a.iv_d + node) : (double)__ldg(a.iv_f + node)) * a.scale;
    const float base = q * wx[c & 1] * wy[(c >> 1) & 1] * wz[(c >> 2) & 1];
    for (int m = 0; m < 10; ++m) {
      const long long l = __double2ll_rn((double)(base * mv[m]) * iv);
      if (l) atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + (size_t)m * a.NN + node),
                       (unsigned long long)l);
    }
  }
}

__global__ void __launch_bounds__(256) deposit_list(const __grid_constant__ P a,
                                                    const __grid_constant__ Bins b) {
  const long long no = min((long long)b.stat[ST_OVERFLOW], b.ov_cap);
  const long long nl = min((long long)b.stat[ST_LATE], b.late_cap);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < no + nl;
       i += stride) {
    const Leaver L = i < no ? b.ov[i] : b.late[i - no];
    deposit_one(a, L.a.x, L.a.y, L.a.z, L.a.w, L.b.x, L.b.y, L.b.z);
  }
}

// ---------------------------------------------------------------------------
// Deposit: quarter-warp q (8 lanes) per bin, four bins per warp round.
// Lane l accumulates for its particles the 80 products q w_c m_k in
// registers: A[k][cp] holds corners (2cp, 2cp + 1) of moment k, so one FFMA2
// multiplies a corner pair of bases by a broadcast moment value.  The flush
// writes each lane's 80 sums as a corner-major row of shared memory (24 x
// STS.128), and lane (q, l) then adds corner l's 10 moments over its
// quarter's 8 rows (3 x LDS.128 and 5 FADD2 per row; against 80 scalar LDS
// and 80 FADD in [moment][corner] rows: 0.509 -> 0.505 ms at C3).
// The next particle of each lane (same bin, or the next round's bin) is
// loaded while the current one is accumulated.
// measured (scripts/build_variants.sh): 4 particles per lane in flight at
// 128 x 3 (12 warps, 168 registers) 0.53 ms; 1 at 256 x 2: 0.76 ms; 2: 0.69;
// 3: 0.56; 6 or 8 spill
#ifndef BP_DEP_TPB
#define BP_DEP_TPB 128  // threads per block of deposit_bins
#endif
#ifndef BP_DEP_MINB
#define BP_DEP_MINB 3
#endif
#ifndef BP_DEP_UNR
#define BP_DEP_UNR 4    // particles per lane and iteration (loads in flight)
#endif
// CHK: some particle may sit in a bin that is not its cell (the mover
// counted misplaced ones this cycle): test each against the bin's cell box.
// Without misplaced particles the test — and the per-bin box it needs, which
// the register allocator otherwise rematerialises per particle — is skipped.
template <bool CHK>
__device__ __forceinline__ void deposit_bins_body(const P& a, const Bins& b, float* dsm) {
  const unsigned lane = threadIdx.x & 31;
  const int qd = (int)(lane >> 3), l = (int)(lane & 7);
  float* const ws = dsm + (threadIdx.x >> 5) * kWarpSm;
  float* const myrow = ws + lane * kRowS;
  const float* const rd = ws + (8 * qd) * kRowS + l * kCornerS;
  const int ci_off = l & 1, cj_off = (l >> 1) & 1, ck_off = (l >> 2) & 1;
  constexpr int U = BP_DEP_UNR;
  float n1[U][7];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < 7; ++k) n1[u][k] = 0.f;
  // the U particles q, q + 8, ... of this lane (those < lim): one 256-bit
  // read-only load each
  auto fetch = [&](int q0, int i0, int lim) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + 8 * u < lim) {
        float4 ra, rb;
        ld_rec_ro(slot_rec(b.rec, q0 + 8 * u), ra, rb);
        n1[u][0] = ra.x; n1[u][1] = ra.y; n1[u][2] = ra.z; n1[u][3] = ra.w;
        n1[u][4] = rb.x; n1[u][5] = rb.y; n1[u][6] = rb.z;
      }
    }
  };
  for (;;) {
    unsigned long long cc = 0;
    if (lane == 0) cc = atomicAdd(&b.stat[ST_WORK_DEP], (unsigned long long)(4 * b.dep_rounds));
    cc = __shfl_sync(0xffffffffu, cc, 0);
    if (cc >= (unsigned long long)b.ncell) break;
    const int c0 = (int)cc;
    // this quarter's bin of round 0 and its cell coordinates
    int c = c0 + qd;
    Ijk q3 = ijk_of(a, min(c, b.ncell - 1));
    int s0 = 0;
    int n = 0;
    if (c < b.ncell) {
      s0 = (int)b.start[c];
      n = min(b.count[c], (int)b.start[c + 1] - s0);
    }
    fetch(s0 + l, l, n);
#pragma unroll 1
    for (int rnd = 0; rnd < b.dep_rounds; ++rnd) {
      if (c0 + 4 * rnd >= b.ncell) break;
      const bool okb = c < b.ncell;
      // next round's bin of this quarter
      const int cn = c + 4;
      int s1 = 0;
      int n_1 = 0;
      if (rnd + 1 < b.dep_rounds && cn < b.ncell) {
        s1 = (int)b.start[cn];
        n_1 = min(b.count[cn], (int)b.start[cn + 1] - s1);
      }
      const int nit =
          (int)__reduce_max_sync(0xffffffffu, (unsigned)((n + 8 * U - 1) / (8 * U)));
      if (nit == 0) fetch(s1 + l, l, n_1);  // (the loop below prefetches otherwise)
      const float cfx = (float)q3.i, cfy = (float)q3.j, cfz = (float)q3.k;
      F2 A[10][4];
#pragma unroll
      for (int k = 0; k < 10; ++k)
#pragma unroll
        for (int cp = 0; cp < 4; ++cp) A[k][cp] = f2(0.f, 0.f);
#pragma unroll 1
      for (int it = 0; it < nit; ++it) {
        const int pi = it * 8 * U + l;
        float cur[U][7];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < 7; ++k) cur[u][k] = n1[u][k];
        if (it + 1 < nit) fetch(s0 + pi + 8 * U, pi + 8 * U, n);
        else fetch(s1 + l, l, n_1);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bool valid = pi + 8 * u < n;
          const float xp = cur[u][0], yp = cur[u][1], zp = cur[u][2], un = cur[u][3],
                      vn = cur[u][4], wn = cur[u][5], qp = cur[u][6];
          const float gx = fmaf(xp, a.idx[0], -a.ogs[0]);
          const float gy = fmaf(yp, a.idx[1], -a.ogs[1]);
          const float gz = fmaf(zp, a.idx[2], -a.ogs[2]);
          if (CHK && valid && !in_box(cell_box(a, q3), gx, gy, gz)) {
            // misplaced (a leaver the mover could not list): the late list
            const unsigned long long o = atomicAdd(&b.stat[ST_LATE], 1ULL);
            if ((long long)o < b.late_cap) {
              Leaver L;
              L.a = make_float4(xp, yp, zp, un);
              L.b = make_float4(vn, wn, qp, 0.f);
              L.id = 0;
              L.pad = 0;
              b.late[o] = L;
            } else {
              atomicAdd(&b.stat[ST_LOST], 1ULL);
            }
            valid = false;
          }
          const float qs = valid ? qp : 0.f;
          const float fx = gx - cfx, fy = gy - cfy, fz = gz - cfz;
          const F2 Q = f2(qs - qs * fx, qs * fx);  // q (1 - fx), q fx
          const F2 Qy0 = __fmul2_rn(Q, f2(1.f - fy, 1.f - fy));
          const F2 Qy1 = __fmul2_rn(Q, f2(fy, fy));
          const float az = 1.f - fz;
          F2 Bc[4];
          Bc[0] = __fmul2_rn(Qy0, f2(az, az));
          Bc[1] = __fmul2_rn(Qy1, f2(az, az));
          Bc[2] = __fmul2_rn(Qy0, f2(fz, fz));
          Bc[3] = __fmul2_rn(Qy1, f2(fz, fz));
          const float mv[10] = {1.f,     un,      vn,      wn,      un * un,
                                un * vn, un * wn, vn * vn, vn * wn, wn * wn};
#pragma unroll
          for (int cp = 0; cp < 4; ++cp) A[0][cp] = __fadd2_rn(A[0][cp], Bc[cp]);
#pragma unroll
          for (int k = 1; k < 10; ++k)
#pragma unroll
            for (int cp = 0; cp < 4; ++cp) A[k][cp] = fma2(Bc[cp], f2(mv[k], mv[k]), A[k][cp]);
        }
      }
      if (nit > 0) {
        // ---- flush: transpose through shared memory (corner-major rows),
        // then lane (q, l) sums corner l's 10 moments over its quarter's rows
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float v[10];
#pragma unroll
          for (int k = 0; k < 10; ++k) v[k] = (c & 1) ? A[k][c >> 1].y : A[k][c >> 1].x;
          float4* o = reinterpret_cast<float4*>(myrow + c * kCornerS);
          o[0] = make_float4(v[0], v[1], v[2], v[3]);
          o[1] = make_float4(v[4], v[5], v[6], v[7]);
          o[2] = make_float4(v[8], v[9], 0.f, 0.f);
        }
        __syncwarp();
        F2 s2[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) s2[k] = f2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float4* q = reinterpret_cast<const float4*>(rd + r * kRowS);
          const float4 x0 = q[0], x1 = q[1], x2 = q[2];
          s2[0] = __fadd2_rn(s2[0], f2(x0.x, x0.y));
          s2[1] = __fadd2_rn(s2[1], f2(x0.z, x0.w));
          s2[2] = __fadd2_rn(s2[2], f2(x1.x, x1.y));
          s2[3] = __fadd2_rn(s2[3], f2(x1.z, x1.w));
          s2[4] = __fadd2_rn(s2[4], f2(x2.x, x2.y));
        }
        __syncwarp();
        const float sm[10] = {s2[0].x, s2[0].y, s2[1].x, s2[1].y, s2[2].x,
                              s2[2].y, s2[3].x, s2[3].y, s2[4].x, s2[4].y};
        if (okb && n > 0) {
          const int node = ((q3.i + ci_off) * a.NY + (q3.j + cj_off)) * a.NZ + q3.k + ck_off;
          const double iv =
              (a.iv_d ? __ldg(a.iv_d + node) : (double)__ldg(a.iv_f + node)) * a.scale;
          unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.acc + node);
#pragma unroll
          for (int m = 0; m < 10; ++m) {
            if (sm[m] != 0.f)
              atomicAdd(dst + (size_t)m * a.NN,
                        (unsigned long long)__double2ll_rn((double)sm[m] * iv));
          }
        }
      }
      c = cn;
      q3 = ijk_advance(a, q3, 4);
      s0 = s1;
      n = n_1;
    }
  }
}

// Both variants are launched; the one the mover's misplaced count (this
// stream, an earlier kernel) does not select returns at once — separate
// kernels keep the checked variant's registers out of the common one.
template <bool CHK>
__global__ void __launch_bounds__(BP_DEP_TPB, BP_DEP_MINB) deposit_bins(const __grid_constant__ P a,
                                                                        const __grid_constant__ Bins b) {
  extern __shared__ __align__(16) float dsm[];
  if ((__ldg(b.stat + ST_MISPLACED) != 0ULL) != CHK) return;
  deposit_bins_body<CHK>(a, b, dsm);
}

}  // namespace bins

namespace {

int bcheck(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

int nsm() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <typename K>
int resident_grid(K k, size_t smem, int threads = 256) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
  return nsm() * (per_sm < 1 ? 1 : per_sm);
}

template <bool RX, bool RY, bool RZ>
int launch_mover_bins(const bins::P& a, const bins::Bins& b, cudaStream_t s) {
  // the reference's default of 3 midpoint iterations unrolled
#if BP_MOVER_FCELL
  // float cell indices are exact below 2^24 cells
  auto k = a.n_iters != 3                  ? bins::mover_bins<RX, RY, RZ, 0, false>
           : (long long)a.cny * a.nz < (1 << 24) ? bins::mover_bins<RX, RY, RZ, 3, true>
                                                 : bins::mover_bins<RX, RY, RZ, 3, false>;
#else
  auto k = a.n_iters == 3 ? bins::mover_bins<RX, RY, RZ, 3, false>
                          : bins::mover_bins<RX, RY, RZ, 0, false>;
#endif
  const int g = resident_grid(k, 0, BP_MOVER_TPB);
  // claims of up to 8 bins, fewer on small grids so that every warp gets
  // several claims (the dynamic claiming then balances the tail)
  bins::Bins bb = b;
  const long long warps = (long long)g * (BP_MOVER_TPB / 32);
  bb.move_claim = (int)std::max(1LL, std::min((long long)bins::kMoveClaim, b.ncell / (6 * warps)));
  const int th = timing_begin(TK_MOVER, s);
  k<<<g, BP_MOVER_TPB, 0, s>>>(a, bb);
  timing_end(th, s);
  note_launch();
  return bcheck("mover_bins launch");
}

int launch_mover_bins_any(const bins::P& a, const bins::Bins& b, const int64_t* geo_i,
                          cudaStream_t s) {
  switch ((geo_i[3] ? 1 : 0) | (geo_i[4] ? 2 : 0) | (geo_i[5] ? 4 : 0)) {
    case 0: return launch_mover_bins<false, false, false>(a, b, s);
    case 1: return launch_mover_bins<true, false, false>(a, b, s);
    case 2: return launch_mover_bins<false, true, false>(a, b, s);
    case 3: return launch_mover_bins<true, true, false>(a, b, s);
    case 4: return launch_mover_bins<false, false, true>(a, b, s);
    case 5: return launch_mover_bins<true, false, true>(a, b, s);
    case 6: return launch_mover_bins<false, true, true>(a, b, s);
    default: return launch_mover_bins<true, true, true>(a, b, s);
  }
}

}  // namespace

// One cycle of one species on the binned layout: mover, migration, deposit
// (+ the overflow and late lists).  The stat words are zeroed here; the host
// reads them after the cycle (overflow / misplaced -> rebuild, lost -> error).
int bins_cycle(const Call& c, const BinsArgs& ba, cudaStream_t s) {
  if (c.pbytes == 8) return bins_cycle64(c, ba, s);
  bins::P a;
  fill_params<float>(c, a);
  a.rec = c.records;
  a.emax = reinterpret_cast<const float*>(
      (const char*)c.records + (split_records_bytes(4, c.geo_i) - 32));
  bins::Bins b;
  b.rec = (float4*)ba.rec;
  b.id = (long long*)ba.ids;
  b.start = (const long long*)ba.start;
  b.count = ba.count;
  b.ncell = (int)ba.ncell;
  b.lv = (bins::Leaver*)ba.leavers;
  b.lv_cap = ba.leaver_cap;
  b.ov = (bins::Leaver*)ba.overflow;
  b.ov_cap = ba.overflow_cap;
  b.late = (bins::Leaver*)ba.late;
  b.late_cap = ba.late_cap;
  b.stat = (unsigned long long*)ba.stat;
  cudaMemsetAsync(b.stat, 0, bins::ST_N * sizeof(unsigned long long), s);
  int rc = launch_mover_bins_any(a, b, c.geo_i, s);
  if (rc) return rc;
  bins::migrate_bins<float><<<nsm() * 8, 256, 0, s>>>(b);
  note_launch();
  if ((rc = bcheck("migrate_bins launch"))) return rc;
  const size_t smem = (size_t)(BP_DEP_TPB / 32) * bins::kWarpSm * sizeof(float);
  static bool attr[64] = {};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(bins::deposit_bins<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(bins::deposit_bins<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  });
  const int g = resident_grid(bins::deposit_bins<false>, smem, BP_DEP_TPB);
  b.dep_rounds = (int)std::max(
      1LL, std::min((long long)bins::kDepClaim / 4,
                    (long long)b.ncell / (24LL * g * (BP_DEP_TPB / 32))));
  const int th = timing_begin(TK_DEPOSIT, s);
  bins::deposit_bins<false><<<g, BP_DEP_TPB, smem, s>>>(a, b);
  bins::deposit_bins<true><<<g, BP_DEP_TPB, smem, s>>>(a, b);
  timing_end(th, s);
  note_launch();
  note_launch();
  if ((rc = bcheck("deposit_bins launch"))) return rc;
  bins::deposit_list<<<nsm(), 256, 0, s>>>(a, b);
  note_launch();
  return bcheck("deposit_list launch");
}

namespace {

// the fast arithmetic's cell keys (fill_params / make_params: 1/d and o/d of
// the field-precision spacing, rounded to S)
template <typename S>
bins::KeyGeo<S> key_geo(const Call& c) {
  bins::KeyGeo<S> g;
  for (int k = 0; k < 3; ++k) {
    const double gd = c.fbytes == 8 ? c.geo_g[k] : (double)(float)c.geo_g[k];
    const double go = c.fbytes == 8 ? c.geo_g[3 + k] : (double)(float)c.geo_g[3 + k];
    g.idx[k] = (S)(1.0 / gd);
    g.ogs[k] = (S)(go / gd);
  }
  g.nx = (int)c.geo_i[0];
  g.ny = (int)c.geo_i[1];
  g.nz = (int)c.geo_i[2];
  return g;
}

template <typename S>
bins::BinsT<S> bins_of(const BinsArgs& ba, const void* src_rec) {
  bins::BinsT<S> b{};
  b.rec = (typename bins::V4<S>::type*)const_cast<void*>(src_rec);
  b.id = (long long*)ba.ids;
  b.start = (const long long*)ba.start;
  b.count = ba.count;
  b.ncell = (int)ba.ncell;
  b.ov = (bins::LeaverT<S>*)ba.overflow;
  b.ov_cap = ba.overflow_cap;
  b.stat = (unsigned long long*)ba.stat;
  return b;
}

// Build step 1: cell histogram and bin layout (start = exclusive scan of the
// capacities); returns the total slot count through *total (synchronises).
template <typename S>
int plan_t(const Call& c, int* count, int64_t* start, double frac, int smin, int64_t* total,
           cudaStream_t s) {
  const bins::KeyGeo<S> g = key_geo<S>(c);
  const int ncell = g.nx * g.ny * g.nz;
  const long long n = c.count;
  cudaMemsetAsync(count, 0, (size_t)ncell * sizeof(int), s);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (long long*)nullptr, (long long*)nullptr,
                                ncell + 1, s);
  int* bad = nullptr;
  long long* caps = nullptr;
  void* tmp = nullptr;
  if (cudaMallocAsync(&bad, 16, s) != cudaSuccess ||
      cudaMallocAsync(&caps, (size_t)(ncell + 1) * 8, s) != cudaSuccess ||
      cudaMallocAsync(&tmp, tmp_bytes + 16, s) != cudaSuccess) {
    set_error("bins_plan: scratch allocation failed");
    return -2;
  }
  cudaMemsetAsync(bad, 0, 16, s);
  if (n > 0) {
    bins::bin_keys<S><<<nsm() * 8, 256, 0, s>>>(g, (const S*)c.x + c.start,
                                                (const S*)c.y + c.start,
                                                (const S*)c.z + c.start, n, nullptr, nullptr,
                                                count, bad);
    note_launch();
  }
  bins::bin_caps<<<nsm() * 4, 256, 0, s>>>(count, ncell, (float)frac, smin, caps);
  note_launch();
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, caps, (long long*)start, ncell + 1, s);
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(total, start + ncell, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(bad, s);
  cudaFreeAsync(caps, s);
  cudaFreeAsync(tmp, s);
  int rc = bcheck("bins_plan");
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = bcheck("bins_plan sync");
  if (rc) return rc;
  return hbad ? 3 : 0;
}

// Build step 2: stable scatter of the flat span into the planned bins.
template <typename S>
int fill_t(const Call& c, const int64_t* src_ids, const int64_t* start, void* dst_rec,
           int64_t* dst_ids, cudaStream_t s) {
  const bins::KeyGeo<S> g = key_geo<S>(c);
  const int ncell = g.nx * g.ny * g.nz;
  const long long n = c.count;
  if (n <= 0) return 0;
  if (n > 0xffffffffLL) {
    set_error("bins_fill: %lld particles exceed the 32-bit index space", n);
    return -1;
  }
  int end_bit = 1;
  while (end_bit < 32 && (1LL << end_bit) < ncell) ++end_bit;
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (unsigned*)nullptr, (unsigned*)nullptr,
                                  (unsigned*)nullptr, (unsigned*)nullptr, n, 0, end_bit, s);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int*)nullptr, (long long*)nullptr, ncell,
                                s);
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t nb = up((size_t)n * 4);
  const size_t need = 4 * nb + up((size_t)ncell * 4) + up((size_t)ncell * 8) + up(16) +
                      up(sort_bytes) + up(scan_bytes) + up(16 * sizeof(void*));
  char* ws = nullptr;
  if (cudaMallocAsync(&ws, need, s) != cudaSuccess) {
    set_error("bins_fill: scratch allocation failed");
    return -2;
  }
  char* p = ws;
  unsigned* k_in = (unsigned*)p; p += nb;
  unsigned* k_out = (unsigned*)p; p += nb;
  unsigned* i_in = (unsigned*)p; p += nb;
  unsigned* i_out = (unsigned*)p; p += nb;
  int* hist = (int*)p; p += up((size_t)ncell * 4);
  long long* first = (long long*)p; p += up((size_t)ncell * 8);
  int* bad = (int*)p; p += up(16);
  void* sort_tmp = p; p += up(sort_bytes);
  void* scan_tmp = p; p += up(scan_bytes);
  void** ptrs = (void**)p;
  cudaMemsetAsync(hist, 0, (size_t)ncell * 4, s);
  cudaMemsetAsync(bad, 0, 16, s);
  bins::bin_keys<S><<<nsm() * 8, 256, 0, s>>>(g, (const S*)c.x + c.start,
                                              (const S*)c.y + c.start, (const S*)c.z + c.start,
                                              n, k_in, i_in, hist, bad);
  note_launch();
  cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, k_in, k_out, i_in, i_out, n, 0, end_bit,
                                  s);
  cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, hist, first, ncell, s);
  const void* hp[16] = {(const S*)c.x + c.start, (const S*)c.y + c.start,
                        (const S*)c.z + c.start, (const S*)c.u + c.start,
                        (const S*)c.v + c.start, (const S*)c.w + c.start,
                        (const S*)c.q + c.start, nullptr, nullptr, nullptr, nullptr,
                        nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaMemcpyAsync(ptrs, hp, sizeof(hp), cudaMemcpyHostToDevice, s);
  bins::bin_scatter<S><<<nsm() * 8, 256, 0, s>>>(
      k_out, i_out, n, (const long long*)start, first, (const S* const*)ptrs,
      (const long long*)src_ids + c.start, (typename bins::V4<S>::type*)dst_rec,
      (long long*)dst_ids);
  note_launch();
  cudaFreeAsync(ws, s);
  int rc = bcheck("bins_fill");
  // the host array hp must outlive the async copy
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = bcheck("bins_fill sync");
  return rc;
}

// Live-particle offsets of the bins (exclusive scan of the clamped counts)
// and the flat copy; the overflow list follows at the end.  Returns the
// particle total through *total (synchronises).
template <typename S>
int export_t(const BinsArgs& ba, const void* src_rec, int64_t* offsets, void* const* dst,
             int64_t* dst_ids, int64_t* total, cudaStream_t s) {
  const bins::BinsT<S> b = bins_of<S>(ba, src_rec);
  const int ncell = b.ncell;
  bins::clamp_counts<<<nsm() * 4, 256, 0, s>>>(ba.count, b.start, ncell);
  note_launch();
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int*)nullptr, (long long*)nullptr,
                                ncell + 1, s);
  void* tmp = nullptr;
  int* cnt1 = nullptr;
  if (cudaMallocAsync(&tmp, scan_bytes + 16, s) != cudaSuccess ||
      cudaMallocAsync(&cnt1, (size_t)(ncell + 1) * 4, s) != cudaSuccess) {
    set_error("bins_export: scratch allocation failed");
    return -2;
  }
  cudaMemsetAsync(cnt1 + ncell, 0, 4, s);
  cudaMemcpyAsync(cnt1, ba.count, (size_t)ncell * 4, cudaMemcpyDeviceToDevice, s);
  cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, cnt1, (long long*)offsets, ncell + 1, s);
  long long nb = 0;
  unsigned long long st[bins::ST_N] = {};
  cudaMemcpyAsync(&nb, offsets + ncell, 8, cudaMemcpyDeviceToHost, s);
  if (ba.stat) cudaMemcpyAsync(st, ba.stat, sizeof(st), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return bcheck("bins_export sync");
  const long long nov =
      ba.overflow ? std::min((long long)st[bins::ST_OVERFLOW], (long long)ba.overflow_cap) : 0LL;
  *total = nb + nov;
  if (!dst) {
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(cnt1, s);
    return bcheck("bins_export");
  }
  void** ptrs = nullptr;
  cudaMallocAsync(&ptrs, 8 * sizeof(void*), s);
  cudaMemcpyAsync(ptrs, dst, 7 * sizeof(void*), cudaMemcpyHostToDevice, s);
  bins::bin_export<S><<<nsm() * 8, 256, 0, s>>>(b, (const long long*)offsets, (S* const*)ptrs,
                                                (long long*)dst_ids);
  note_launch();
  if (nov > 0) {
    bins::list_export<S><<<nsm(), 256, 0, s>>>(b, nb, (S* const*)ptrs, (long long*)dst_ids);
    note_launch();
  }
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(cnt1, s);
  cudaFreeAsync(ptrs, s);
  int rc = bcheck("bins_export");
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = bcheck("bins_export sync");
  return rc;
}

template <typename S>
int reslack_plan_t(const BinsArgs& ba, const void* src_rec, int* ncount, int64_t* nstart,
                   double frac, int smin, int64_t* total, cudaStream_t s) {
  const bins::BinsT<S> b = bins_of<S>(ba, src_rec);
  const int ncell = b.ncell;
  bins::reslack_counts<S><<<nsm() * 4, 256, 0, s>>>(b, ncount);
  note_launch();
  bins::reslack_hist<S><<<nsm() * 2, 256, 0, s>>>(b, ncount);
  note_launch();
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (long long*)nullptr, (long long*)nullptr,
                                ncell + 1, s);
  long long* caps = nullptr;
  void* tmp = nullptr;
  if (cudaMallocAsync(&caps, (size_t)(ncell + 1) * 8, s) != cudaSuccess ||
      cudaMallocAsync(&tmp, tmp_bytes + 16, s) != cudaSuccess) {
    set_error("bins_reslack_plan: scratch allocation failed");
    return -2;
  }
  bins::bin_caps<<<nsm() * 4, 256, 0, s>>>(ncount, ncell, (float)frac, smin, caps);
  note_launch();
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, caps, (long long*)nstart, ncell + 1, s);
  cudaMemcpyAsync(total, nstart + ncell, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(caps, s);
  cudaFreeAsync(tmp, s);
  int rc = bcheck("bins_reslack_plan");
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = bcheck("bins_reslack_plan sync");
  return rc;
}

template <typename S>
int reslack_copy_t(const BinsArgs& ba, const void* src_rec, const int64_t* nstart, int* ncount,
                   void* dst_rec, int64_t* dst_ids, cudaStream_t s) {
  typedef typename bins::V4<S>::type V;
  const bins::BinsT<S> b = bins_of<S>(ba, src_rec);
  bins::reslack_copy<S><<<nsm() * 8, 256, 0, s>>>(b, (const long long*)nstart, ncount,
                                                  (V*)dst_rec, (long long*)dst_ids);
  note_launch();
  bins::reslack_place<S><<<nsm() * 2, 256, 0, s>>>(b, (const long long*)nstart, ncount,
                                                   (V*)dst_rec, (long long*)dst_ids);
  note_launch();
  int rc = bcheck("bins_reslack_copy");
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = bcheck("bins_reslack_copy sync");
  return rc;
}

}  // namespace

int bins_leaver_bytes(int pbytes) {
  return pbytes == 8 ? (int)sizeof(bins::LeaverT<double>) : (int)sizeof(bins::LeaverT<float>);
}

// the f32 mover indexes slots in 32 bits
static int check_f32_slots(int pbytes, int rc, const int64_t* total) {
  if (!rc && pbytes == 4 && *total >= 0x7fffffffLL) {
    set_error("binned layout of %lld slots: the f32 bins hold < 2^31 (use a smaller slack or "
              "the flat layout)", (long long)*total);
    return -1;
  }
  return rc;
}

int bins_plan(const Call& c, int* count, int64_t* start, double frac, int smin, int64_t* total,
              cudaStream_t s) {
  const int rc = c.pbytes == 8 ? plan_t<double>(c, count, start, frac, smin, total, s)
                               : plan_t<float>(c, count, start, frac, smin, total, s);
  return check_f32_slots(c.pbytes, rc, total);
}

int bins_fill(const Call& c, const int64_t* src_ids, const int64_t* start, void* dst_rec,
              int64_t* dst_ids, cudaStream_t s) {
  return c.pbytes == 8 ? fill_t<double>(c, src_ids, start, dst_rec, dst_ids, s)
                       : fill_t<float>(c, src_ids, start, dst_rec, dst_ids, s);
}

int bins_export(const BinsArgs& ba, const void* src_rec, int64_t* offsets, void* const* dst,
                int64_t* dst_ids, int64_t* total, cudaStream_t s) {
  return ba.pbytes == 8 ? export_t<double>(ba, src_rec, offsets, dst, dst_ids, total, s)
                        : export_t<float>(ba, src_rec, offsets, dst, dst_ids, total, s);
}

// Re-slack plan: ncount = live + overflow arrivals per bin, nstart = exclusive
// scan of the padded capacities; *total = nstart[ncell] (synchronises).
int bins_reslack_plan(const BinsArgs& ba, const void* src_rec, int* ncount, int64_t* nstart,
                      double frac, int smin, int64_t* total, cudaStream_t s) {
  const int rc =
      ba.pbytes == 8 ? reslack_plan_t<double>(ba, src_rec, ncount, nstart, frac, smin, total, s)
                     : reslack_plan_t<float>(ba, src_rec, ncount, nstart, frac, smin, total, s);
  return check_f32_slots(ba.pbytes, rc, total);
}

// Re-slack copy into dst (nstart from the plan); ncount ends as the new
// live counts (synchronises).
int bins_reslack_copy(const BinsArgs& ba, const void* src_rec, const int64_t* nstart,
                      int* ncount, void* dst_rec, int64_t* dst_ids, cudaStream_t s) {
  return ba.pbytes == 8
             ? reslack_copy_t<double>(ba, src_rec, nstart, ncount, dst_rec, dst_ids, s)
             : reslack_copy_t<float>(ba, src_rec, nstart, ncount, dst_rec, dst_ids, s);
}

}  // namespace bp
