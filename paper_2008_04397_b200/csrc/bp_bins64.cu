// Cell-binned fast path for f64 particles (DeviceSimulation layout "bins",
// precision "double", arithmetic "fast").  Same layout and cycle as the f32
// path (bp_bins.cu; bins in cell order, sorted after every cycle, no sort
// phase), with the f64 fast arithmetic of the flat path, so that the result
// is BITWISE the flat f64 fast path's (bp_fast.cu f64_split_fused: the split
// mover, then the generic FastPolicy<double, double> deposit):
//
//   mover_bins64    one warp per bin (claims of consecutive bins); each lane
//                   pushes its particle with the split kernels' push
//                   (sk::push<double>, kernels.py:498-676: the cell's
//                   coefficient record, 42 DFMA per gather, implicit
//                   rotation), boundary folds skipped for a warp below the
//                   bin's speed bound — a bin's particles share one cell, so
//                   its record stays in L1; leavers are listed and the holes
//                   refilled exactly as in the f32 mover.
//   migrate_bins    (bp_bins_plumb.cuh) every leaver to its new bin.
//   deposit_bins64  one warp per bin, 32-particle tiles staged in shared memory
//                   (cell check, fractions, moment values once per particle);
//                   lane (q, l) owns corner l and folds the staged particles
//                   q, q + 4, ... — for each, the ten contributions
//                   rint(base_l * m_k) onto the int64 lattice
//                   (fields.py:20-25) as the generic deposit forms them
//                   (bp_fast_policy.cuh stage(), bp_common.cuh qbits: the
//                   exact product base * m rounded once), summed in
//                   registers as integers; the four quarters' sums are added
//                   with shuffles and lanes 0-7 issue the REDG.ADD.64.
//                   Integer sums are order-free, so the lattice equals the
//                   flat path's (which deposits per contribution, in another
//                   grouping) bit for bit — the per-contribution rounding
//                   that keeps f64 within 1e-10 of the reference.
//   deposit_list64  the overflow and misplaced particles (rare), one at a time.
//
// Field records: the split kernels' per-cell coefficient records in f64
// (bp_field_records_build, pbytes 8; max |E| in the last 32 bytes).  The
// deposit reads invvol itself; max |invvol| (the magic-rint range guard's
// bound) is reduced into the spare stat word 7 at the start of the cycle.
#include <algorithm>
#include <cstdint>

#include "bp_bins_plumb.cuh"
#include "bp_f32_common.cuh"
#include "bp_fast_policy.cuh"
#include "bp_launch_impl.cuh"

namespace bp {
namespace bins64 {

typedef SpanParams<double, double> SP;
typedef FastPolicy<double, double> Pol;
typedef bins::BinsT<double> Bins;
typedef bins::LeaverT<double> Leaver;
using bins::ST_LATE;
using bins::ST_LEAVERS;
using bins::ST_LOST;
using bins::ST_MISPLACED;
using bins::ST_OVERFLOW;
using bins::ST_WORK_DEP;
using bins::ST_WORK_MOVE;

constexpr int kHoleCap = 256;   // leavers per bin per cycle tracked for the refill
constexpr int kMoveClaim = 8;   // bins per mover work claim (at most)
constexpr int kLvChunk = 128;   // leaver slots per warp reservation
constexpr int kTpb = 128;       // threads per block of both kernels
constexpr int kWarps = kTpb / 32;

// 64-byte particle records: two 256-bit accesses
__device__ __forceinline__ void ld_rec_stream(const double4* p, double4& a, double4& b) {
  asm volatile("ld.global.L1::evict_first.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(a.z), "=d"(a.w)
               : "l"(p));
  asm volatile("ld.global.L1::evict_first.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(b.x), "=d"(b.y), "=d"(b.z), "=d"(b.w)
               : "l"(p + 1));
}
__device__ __forceinline__ void ld_rec_ro(const double4* p, double4& a, double4& b) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(a.z), "=d"(a.w)
      : "l"(p));
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(b.x), "=d"(b.y), "=d"(b.z), "=d"(b.w)
      : "l"(p + 1));
}
__device__ __forceinline__ void st_rec_stream(double4* p, const double4& a, const double4& b) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x),
               "d"(a.y), "d"(a.z), "d"(a.w)
               : "memory");
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 1), "d"(b.x),
               "d"(b.y), "d"(b.z), "d"(b.w)
               : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// the bin (x-fastest cell index) of an in-box position: sk::cell_of's
// arithmetic (gx = x * (1/dx) - ox/dx, min(trunc(gx), n - 1)), which is also
// FastPolicy::cell_t's
__device__ __forceinline__ int bin_of(const sk::Params<double>& a, double x, double y,
                                      double z) {
  const int i = min((int)fma(x, a.idx[0], -a.ogs[0]), a.nx - 1);
  const int j = min((int)fma(y, a.idx[1], -a.ogs[1]), a.ny - 1);
  const int k = min((int)fma(z, a.idx[2], -a.ogs[2]), a.nz - 1);
  return i + a.nx * j + a.cny * k;
}

// ---------------------------------------------------------------------------
// Mover: one warp per bin.  Stayers are written back in place; each leaver is
// listed (x..w, q, id, new cell) and leaves a hole; after the bin's last tile
// the holes below the new count take the bin's trailing stayers.  The next
// tile's records (or the next bin's first tile) load during the push.
#ifndef BP_MOV64_MINB
#define BP_MOV64_MINB 5  // resident 128-thread blocks per SM (measured at C2: 4 -> 0.248 ms, 5 -> 0.242, 6 -> 0.256)
#endif
template <bool RX, bool RY, bool RZ>
__global__ void __launch_bounds__(kTpb, BP_MOV64_MINB) mover_bins64(
    const __grid_constant__ sk::Params<double> a, const __grid_constant__ Bins b) {
  __shared__ unsigned short holes_s[kWarps][kHoleCap];
  __shared__ int lvslot_s[kWarps][kHoleCap];
  const int wid = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  unsigned short* const holes = holes_s[wid];
  int* const lvslot = lvslot_s[wid];
  const unsigned lt = lanemask_lt();
  // the per-bin speed bound below which no position of a push leaves the box
  // (bp_bins.cu bin_speed_bound, in f64)
  const double qe = fabs(a.qdt2m) * (double)__ldg(a.emax) * 1.00001;
  const double hmin = 0.9999 * fmin(fmin(a.L[0] / a.nx, a.L[1] / a.ny), a.L[2] / a.nz);
  const double epsmax = fmax(fmax(a.bc_eps[0], a.bc_eps[1]), a.bc_eps[2]);
  long long lv_base = 0, lv_next = 0;
  int lv_used = kLvChunk;
  double4 na = make_double4(0, 0, 0, 0), nb = na;
  for (;;) {
    unsigned long long cc = 0;
    if (lane == 0) cc = atomicAdd(&b.stat[ST_WORK_MOVE], (unsigned long long)b.move_claim);
    const int c0 = (int)min(__shfl_sync(0xffffffffu, cc, 0), (unsigned long long)b.ncell);
    if (c0 >= b.ncell) break;
    const int c1 = min(c0 + b.move_claim, b.ncell);
    long long s0 = b.start[c0];
    int n = (int)min((long long)b.count[c0], b.start[c0 + 1] - s0);
    if ((int)lane < n) ld_rec_stream(b.rec + 2 * (s0 + lane), na, nb);
    bool pf_ok = true;  // (warp-uniform) na/nb hold this bin's first tile
    for (int c = c0; c < c1; ++c) {
      long long s1 = 0;
      int n_1 = 0;
      if (c + 1 < c1) {
        s1 = b.start[c + 1];
        n_1 = (int)min((long long)b.count[c + 1], b.start[c + 2] - s1);
      }
      if (n > 0) {
        if (!pf_ok && (int)lane < n) ld_rec_stream(b.rec + 2 * (s0 + lane), na, nb);
        const int ci = c % a.nx, cj = (c / a.nx) % a.ny, ck = c / a.cny;
        const int cells = min(min(min(ci, a.nx - 1 - ci), min(cj, a.ny - 1 - cj)),
                              min(ck, a.nz - 1 - ck));
        const double vmax = (cells * hmin - epsmax) / a.dt - qe;
        int nh = 0;
#pragma unroll 1
        for (int t0 = 0; t0 < n; t0 += 32) {
          const int r = t0 + (int)lane;
          const bool valid = r < n;
          const long long p = s0 + r;
          double xp = na.x, yp = na.y, zp = na.z, un = na.w, vn = nb.x, wn = nb.y;
          const double qp = nb.z;
          if (t0 + 32 < n) {
            if (r + 32 < n) ld_rec_stream(b.rec + 2 * (p + 32), na, nb);
          } else if (n_1 > 0 && (int)lane < n_1) {
            ld_rec_stream(b.rec + 2 * (s1 + lane), na, nb);
          }
          int st = ST_OK;
          int dest = c;
          const bool all_in =
              __all_sync(0xffffffffu, !valid || fabs(un) + fabs(vn) + fabs(wn) < vmax);
          if (valid) {
            st = sk::push<double, RX, RY, RZ, false>(a, xp, yp, zp, un, vn, wn, all_in);
            if (st == ST_OK) dest = bin_of(a, xp, yp, zp);
            else atomicMax(a.status, st);  // not stored (kernels.py:618-621); the cycle raises
          }
          const bool leave = valid && st == ST_OK && dest != c;
          const unsigned L = __ballot_sync(0xffffffffu, leave);
          if (L) {
            // leaver slots from the warp's private chunk of the list
            const int nl = __popc(L);
            const int rank = __popc(L & lt);
            if (lv_used + nl > kLvChunk) {
              unsigned long long c2 = 0;
              if (lane == 0) c2 = atomicAdd(&b.stat[ST_LEAVERS], (unsigned long long)kLvChunk);
              lv_next = (long long)__shfl_sync(0xffffffffu, c2, 0);
            }
            const int room = kLvChunk - lv_used;
            const long long slot =
                rank < room ? lv_base + lv_used + rank : lv_next + (rank - room);
            const bool listed = leave && slot < b.lv_cap && nh + rank < kHoleCap && r < 65536;
            if (listed) {
              double4* rec = reinterpret_cast<double4*>(b.lv + slot);
              rec[0] = make_double4(xp, yp, zp, un);
              rec[1] = make_double4(vn, wn, qp, bins::dest_bits<double>(dest));
              holes[nh + rank] = (unsigned short)r;
              lvslot[nh + rank] = (int)slot;
            } else if (leave) {
              // stays here as a misplaced particle (slow paths; host rebuilds)
              atomicAdd(&b.stat[ST_MISPLACED], 1ULL);
              if (slot < b.lv_cap) b.lv[slot].b.w = bins::dest_bits<double>(-1);
            }
            nh += __popc(__ballot_sync(0xffffffffu, listed));
            if (lv_used + nl > kLvChunk) {
              lv_base = lv_next;
              lv_used = nl - room;
            } else {
              lv_used += nl;
            }
          }
          if (valid && st == ST_OK)
            st_rec_stream(b.rec + 2 * p, make_double4(xp, yp, zp, un),
                          make_double4(vn, wn, qp, 0.0));
        }
        __syncwarp();
        if (nh > 0) {
          // leavers' ids into their records; the holes below the new count
          // take the trailing stayers (all loads before any store: the refill
          // writes into leaver slots)
          const int n_stay = n - nh;
          int nlow = 0;
          for (int k0 = 0; k0 < nh; k0 += 32) {
            const int k = k0 + (int)lane;
            nlow += __popc(__ballot_sync(0xffffffffu, k < nh && (int)holes[k] < n_stay));
          }
          for (int k0 = 0; k0 < nh; k0 += 32) {
            const int k = k0 + (int)lane;
            long long lid = 0;
            if (k < nh) lid = b.id[s0 + holes[k]];
            long long dst = 0;
            double4 ra = make_double4(0, 0, 0, 0), rb = ra;
            long long rid = 0;
            if (k < nlow) {
              int t = n_stay + k;
              for (int j = nlow; j < nh; ++j) {
                if ((int)holes[j] <= t) ++t;
                else break;
              }
              const long long src = s0 + t;
              dst = s0 + holes[k];
              ra = b.rec[2 * src];
              rb = b.rec[2 * src + 1];
              rid = b.id[src];
            }
            if (k < nh) b.lv[lvslot[k]].id = lid;
            __syncwarp();
            if (k < nlow) {
              bins::st_rec(b.rec + 2 * dst, ra, rb);
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
  }
  // unused slots of the last leaver chunk carry no particle
  for (int k = lv_used + (int)lane; k < kLvChunk; k += 32)
    if (lv_base + k < b.lv_cap) b.lv[lv_base + k].b.w = bins::dest_bits<double>(-1);
}

// ---------------------------------------------------------------------------
// One contribution as a biased bit pattern: bits(M) + rint(base * m) (the
// generic deposit's qbits with FMA: the exact product rounded once), or the
// conversion path for a particle the magic range guard rejects.
__device__ __forceinline__ u64 qb(double b, double m, bool magic) {
  if (magic) return (u64)__double_as_longlong(__fma_rn(b, m, kMagic));
  return (u64)__double2ll_rn(b * m) + (u64)kMagicBits;
}

// The particle's in-box check and corner-000 cell as FastPolicy::stage (-1:
// outside the box, not deposited).
__device__ __forceinline__ int stage_cell(const SP& a, const FastScalars<double>& s, double x,
                                          double y, double z, double& fx, double& fy,
                                          double& fz) {
  fx = fy = fz = 0.0;
  if (!(x >= s.o(0) && x <= s.hi(0) && y >= s.o(1) && y <= s.hi(1) && z >= s.o(2) &&
        z <= s.hi(2)))
    return -1;
  return Pol::cell_t(a, s, x, y, z, fx, fy, fz);
}

// corner l of node key: +x (bit 0), +y (bit 1), +z (bit 2), as stage()'s rr[]
__device__ __forceinline__ int corner_node(const SP& a, int key, int l) {
  return key + ((l & 1) ? a.NY * a.NZ : 0) + ((l & 2) ? a.NZ : 0) + ((l & 4) ? 1 : 0);
}

// base of corner l: (q scale (w_xy w_z)) invvol — stage()'s expression order
__device__ __forceinline__ double corner_base(double qs, double fx, double fy, double fz, int l,
                                              double iv) {
  const double ax = 1.0 - fx, ay = 1.0 - fy, az = 1.0 - fz;
  const double wx = (l & 1) ? fx : ax, wy = (l & 2) ? fy : ay;
  return qs * (wx * wy * ((l & 4) ? fz : az)) * iv;
}

__global__ void __launch_bounds__(256) deposit_list64(const __grid_constant__ SP a,
                                                      const __grid_constant__ Bins b) {
  const FastScalars<double> s(a);
  const long long no = min((long long)b.stat[ST_OVERFLOW], b.ov_cap);
  const long long nl = min((long long)b.stat[ST_LATE], b.late_cap);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < no + nl;
       i += stride) {
    const Leaver L = i < no ? b.ov[i] : b.late[i - no];
    double fx, fy, fz;
    const int key = stage_cell(a, s, L.a.x, L.a.y, L.a.z, fx, fy, fz);
    if (key < 0) {
      atomicMax(a.status, ST_DOMAIN);
      continue;
    }
    const double u = L.a.w, v = L.b.x, w = L.b.y;
    const double qs = L.b.z * s.scale();
    const double mv[10] = {1.0, u, v, w, u * u, u * v, u * w, v * v, v * w, w * w};
    const bool magic = !magic_unsafe(qs * s.qlim, mv[4], mv[7], mv[9], kMagicLimit);
    for (int l = 0; l < 8; ++l) {
      const int node = corner_node(a, key, l);
      const double bs = corner_base(qs, fx, fy, fz, l, __ldg(a.invvol + node));
      for (int m = 0; m < 10; ++m) {
        const long long v64 = (long long)(qb(bs, mv[m], magic) - (u64)kMagicBits);
        if (v64) atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + (size_t)m * a.NN + node),
                           (unsigned long long)v64);
      }
    }
  }
}

// Deposit: one warp per bin (claims of dep_rounds bins), 32-particle tiles.
// Stage: lane j takes particle j of the tile — cell check (a misplaced one,
// a leaver the mover could not list, goes to the late list), fractions, q
// scale and the moment values — into its shared-memory row (zeros for an
// empty or misplaced slot, whose contributions are then exactly 0).  Fold:
// lane (q, l) owns corner l and folds rows q, q + 8, ... paired with rows
// q + 4, q + 12, ...: per pair, two bases and the ten contributions of each,
// added two at a time (one 3-input 64-bit add per moment).  The magic-rint
// range guard is decided per tile (warp-uniform), as the generic deposit
// does.
constexpr int kRowD = 18;  // doubles per staged row (14 used): LDS.128 of 4 rows hit 16 banks

__device__ __forceinline__ void fold_pair(u64 (&S)[10], const double* ra, const double* rb,
                                          int l, double iv, bool magic) {
  const double2 a0 = *reinterpret_cast<const double2*>(ra);
  const double2 a1 = *reinterpret_cast<const double2*>(ra + 2);
  const double2 b0 = *reinterpret_cast<const double2*>(rb);
  const double2 b1 = *reinterpret_cast<const double2*>(rb + 2);
  // rows: fx fy | fz qs | u v | w uu | uv uw | vv vw | ww 0
  const double ba = corner_base(a1.y, a0.x, a0.y, a1.x, l, iv);
  const double bb = corner_base(b1.y, b0.x, b0.y, b1.x, l, iv);
  double ma[10], mb[10];
  ma[0] = 1.0;
  mb[0] = 1.0;
#pragma unroll
  for (int k = 0; k < 9; k += 2) {
    const double2 x = *reinterpret_cast<const double2*>(ra + 4 + k);
    const double2 y = *reinterpret_cast<const double2*>(rb + 4 + k);
    ma[1 + k] = x.x;
    mb[1 + k] = y.x;
    if (k + 1 < 9) {
      ma[2 + k] = x.y;
      mb[2 + k] = y.y;
    }
  }
  if (magic) {
#pragma unroll
    for (int m = 0; m < 10; ++m) S[m] += qb(ba, ma[m], true) + qb(bb, mb[m], true);
  } else {
#pragma unroll
    for (int m = 0; m < 10; ++m) S[m] += qb(ba, ma[m], false) + qb(bb, mb[m], false);
  }
}

__global__ void __launch_bounds__(kTpb) deposit_bins64(const __grid_constant__ SP a,
                                                       const __grid_constant__ Bins b) {
  __shared__ __align__(16) double st_s[kWarps][32 * kRowD];
  const unsigned lane = threadIdx.x & 31;
  const int qd = (int)(lane >> 3), l = (int)(lane & 7);
  double* const st = st_s[threadIdx.x >> 5];
  double* const myrow = st + lane * kRowD;
  const FastScalars<double> s(a);
  for (;;) {
    unsigned long long cc = 0;
    if (lane == 0) cc = atomicAdd(&b.stat[ST_WORK_DEP], (unsigned long long)b.dep_rounds);
    const int c0 = (int)min(__shfl_sync(0xffffffffu, cc, 0), (unsigned long long)b.ncell);
    if (c0 >= b.ncell) break;
    const int c1 = min(c0 + b.dep_rounds, b.ncell);
    for (int c = c0; c < c1; ++c) {
      const long long s0 = b.start[c];
      const int n = (int)min((long long)b.count[c], b.start[c + 1] - s0);
      if (n == 0) continue;
      const int ci = c % a.nx, cj = (c / a.nx) % a.ny, ck = c / (a.nx * a.ny);
      const int key = (ci * a.NY + cj) * a.NZ + ck;
      const int node = corner_node(a, key, l);
      const double iv = __ldg(a.invvol + node);
      u64 S[10];
#pragma unroll
      for (int m = 0; m < 10; ++m) S[m] = 0;
      int nf = 0;  // folded rows (each adds bits(M) once per value)
      double4 ra = make_double4(0, 0, 0, 0), rb = ra;
      if ((int)lane < n) ld_rec_ro(b.rec + 2 * (s0 + lane), ra, rb);
#pragma unroll 1
      for (int t0 = 0; t0 < n; t0 += 32) {
        const int nt = min(32, n - t0);
        const double4 ca = ra, cb = rb;
        if (t0 + 32 + (int)lane < n) ld_rec_ro(b.rec + 2 * (s0 + t0 + 32 + lane), ra, rb);
        // ---- stage this lane's particle
        bool ok = (int)lane < nt;
        double fx = 0, fy = 0, fz = 0;
        if (ok) {
          const int k2 = stage_cell(a, s, ca.x, ca.y, ca.z, fx, fy, fz);
          if (k2 != key) {
            // misplaced: the late list (its deposit checks the box)
            ok = false;
            const unsigned long long o = atomicAdd(&b.stat[ST_LATE], 1ULL);
            if ((long long)o < b.late_cap) {
              Leaver Lv;
              Lv.a = ca;
              Lv.b = make_double4(cb.x, cb.y, cb.z, 0.0);
              Lv.id = 0;
              Lv.pad = 0;
              b.late[o] = Lv;
            } else {
              atomicAdd(&b.stat[ST_LOST], 1ULL);
            }
          }
        }
        const double u = ok ? ca.w : 0.0, v = ok ? cb.x : 0.0, w = ok ? cb.y : 0.0;
        const double qs = ok ? cb.z * s.scale() : 0.0;
        if (!ok) fx = fy = fz = 0.0;
        const double uu = u * u, vv = v * v, ww = w * w;
        const bool magic = !magic_unsafe(qs * s.qlim, uu, vv, ww, kMagicLimit);
        double2* r2 = reinterpret_cast<double2*>(myrow);
        r2[0] = make_double2(fx, fy);
        r2[1] = make_double2(fz, qs);
        r2[2] = make_double2(u, v);
        r2[3] = make_double2(w, uu);
        r2[4] = make_double2(u * v, u * w);
        r2[5] = make_double2(vv, v * w);
        r2[6] = make_double2(ww, 0.0);
        const bool all_magic = __all_sync(0xffffffffu, magic);
        __syncwarp();
        // ---- fold: rows qd + 8i paired with qd + 8i + 4 (rows >= nt are zero)
        for (int j = qd; j < nt; j += 8) {
          fold_pair(S, st + j * kRowD, st + (j + 4) * kRowD, l, iv, all_magic);
          nf += 2;
        }
        __syncwarp();
      }
      const u64 bias = (u64)nf * (u64)kMagicBits;
#pragma unroll
      for (int m = 0; m < 10; ++m) {
        u64 v = S[m] - bias;
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        S[m] = v;
      }
      if (qd == 0) {
#pragma unroll
        for (int m = 0; m < 10; ++m)
          if (S[m]) atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + (size_t)m * a.NN + node),
                              (unsigned long long)S[m]);
      }
    }
  }
}

// max |invvol| as the bits of a non-negative double (they order like the
// values) into *out: the magic-rint guard's bound (pack_nodes computes the same)
__global__ void __launch_bounds__(256) invvol_max(const double* __restrict__ iv, int NN,
                                                  unsigned long long* out) {
  double m = 0.0;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < NN; n += gridDim.x * blockDim.x)
    m = fmax(m, fabs(iv[n]));
  unsigned long long bits = (unsigned long long)__double_as_longlong(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = v > bits ? v : bits;
  }
  if ((threadIdx.x & 31) == 0 && bits) atomicMax(out, bits);
}

}  // namespace bins64

namespace {

int check64(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

template <typename K>
int resident_blocks(K k, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0);
  return sm_count() * (per_sm < 1 ? 1 : per_sm);
}

}  // namespace

// One cycle of one f64 species on the binned layout (c.records: the f64
// coefficient records of bp_field_records_build for the current E/B).
template <bool RX, bool RY, bool RZ>
int launch_mover64(const sk::Params<double>& ap, const bins64::Bins& b, cudaStream_t s) {
  auto k = bins64::mover_bins64<RX, RY, RZ>;
  const int g = resident_blocks(k, bins64::kTpb);
  bins64::Bins bb = b;
  // claims sized so that every warp gets several (dynamic claiming balances
  // the tail)
  const long long w = (long long)g * bins64::kWarps;
  bb.move_claim = (int)std::max(1LL, std::min((long long)bins64::kMoveClaim, b.ncell / (6 * w)));
  const int th = timing_begin(TK_MOVER, s);
  k<<<g, bins64::kTpb, 0, s>>>(ap, bb);
  timing_end(th, s);
  note_launch();
  return check64("mover_bins64 launch");
}

int bins_cycle64(const Call& c0, const BinsArgs& ba, cudaStream_t s) {
  Call c = c0;
  c.apply_bc = 1;
  bins64::SP a = make_params<double, double>(c);
  sk::Params<double> ap;
  fill_params<double>(c, ap);
  ap.rec = c.records;
  ap.emax = reinterpret_cast<const float*>((const char*)c.records +
                                           split_records_bytes(8, c.geo_i) - 32);
  bins64::Bins b{};
  b.rec = (double4*)ba.rec;
  b.id = (long long*)ba.ids;
  b.start = (const long long*)ba.start;
  b.count = ba.count;
  b.ncell = (int)ba.ncell;
  b.lv = (bins64::Leaver*)ba.leavers;
  b.lv_cap = ba.leaver_cap;
  b.ov = (bins64::Leaver*)ba.overflow;
  b.ov_cap = ba.overflow_cap;
  b.late = (bins64::Leaver*)ba.late;
  b.late_cap = ba.late_cap;
  b.stat = (unsigned long long*)ba.stat;
  cudaMemsetAsync(b.stat, 0, bins::ST_N * sizeof(unsigned long long), s);
  // stat word 7: max |invvol| for the deposit's range guard
  a.iv_max = reinterpret_cast<const double*>(b.stat + 7);
  bins64::invvol_max<<<std::min((a.NN + 255) / 256, 1024), 256, 0, s>>>(
      (const double*)c.invvol, a.NN, b.stat + 7);
  note_launch();
  int rc;
  switch ((c.geo_i[3] ? 1 : 0) | (c.geo_i[4] ? 2 : 0) | (c.geo_i[5] ? 4 : 0)) {
    case 0: rc = launch_mover64<false, false, false>(ap, b, s); break;
    case 1: rc = launch_mover64<true, false, false>(ap, b, s); break;
    case 2: rc = launch_mover64<false, true, false>(ap, b, s); break;
    case 3: rc = launch_mover64<true, true, false>(ap, b, s); break;
    case 4: rc = launch_mover64<false, false, true>(ap, b, s); break;
    case 5: rc = launch_mover64<true, false, true>(ap, b, s); break;
    case 6: rc = launch_mover64<false, true, true>(ap, b, s); break;
    default: rc = launch_mover64<true, true, true>(ap, b, s); break;
  }
  if (rc) return rc;
  bins::migrate_bins<double><<<sm_count() * 8, 256, 0, s>>>(b);
  note_launch();
  if ((rc = check64("migrate_bins launch"))) return rc;
  const int gd = resident_blocks(bins64::deposit_bins64, bins64::kTpb);
  const long long wd = (long long)gd * bins64::kWarps;
  b.dep_rounds = (int)std::max(1LL, std::min(8LL, b.ncell / (6 * wd)));
  const int th = timing_begin(TK_DEPOSIT, s);
  bins64::deposit_bins64<<<gd, bins64::kTpb, 0, s>>>(a, b);
  timing_end(th, s);
  note_launch();
  if ((rc = check64("deposit_bins64 launch"))) return rc;
  bins64::deposit_list64<<<sm_count(), 256, 0, s>>>(a, b);
  note_launch();
  return check64("deposit_list64 launch");
}

}  // namespace bp
