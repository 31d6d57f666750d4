// Fused implicit mover + moment deposition, sm_100a — shared machinery.
//
// Semantics follow the reference batchpic kernels (pkg/src/batchpic/kernels.py):
//   push block   fused_span :489-682 (== push_span :112-306)
//   deposit      fused_span :683-734 (== deposit_span :327-381)
//   gather       gather_span :385-455
// The arithmetic of the push block and of the per-particle deposit values is
// a policy: bp_parity_policy.cuh (bitwise the reference, compiled with
// -fmad=false) or bp_fast_policy.cuh (FMA, reciprocals, native f32).  The
// kernel body, the field records and the exact deposition are shared here.
//
// Layout in HBM (the reference data contract, unchanged):
//   particles  SoA x y z u v w q, one contiguous array each (P)
//   E, B       (3, nx+1, ny+1, nz+1) C order, k fastest (F)
//   acc        (10, nx+1, ny+1, nz+1) int64 fixed point (rho Jx Jy Jz Pxx Pxy
//              Pxz Pyy Pyz Pzz), quantum 2^-43 (fields.py:20-25)
//   invvol     (nx+1, ny+1, nz+1) (F)
// plus one per-call scratch array of node records (pack_nodes).
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
typedef unsigned long long u64;  // modular sums of biased bit patterns

// ST_DOMAIN: a deposit/gather position outside the box (the reference does
// not check; the GPU refuses to index out of bounds).
enum { ST_OK = 0, ST_RUNAWAY = 1, ST_MIDPOINT = 2, ST_DOMAIN = 3 };

// Scalars widened to double once on the host (exact), so kernels never
// re-convert them per particle; inv_gd / go_s serve the fast arithmetic
// only (gx = x * (1/d) - o/d).
struct WideScalars {
  double o[3], L[3], hi[3], hi2[3], gd[3], go[3], inv_gd[3], go_s[3];
  double dt, dth, qdt2m, beta, one, two, beta2, scale;
};

// The fast arithmetic's constants rounded once to f32 on the host, read
// straight from the parameter bank by FFMA/FSETP.
struct NarrowScalars {
  float o[3], L[3], hi[3], hi2[3], idx[3], ogs[3];
  float dt, dth, qdt2m, beta, beta2, scale;
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
  WideScalars d;
  NarrowScalars f;
  int n_iters, mixed, apply_bc;
  int* status;
  P* gather_out;  // gather only: (count, 6)
  // per-call node records (pack_nodes), element type Policy::NodeT:
  // Ex Ey Ez Bx By Bz invvol 0 for every node
  const void* fnode;
  // max |invvol| (written by pack_nodes): bounds every staged base for the
  // magic-rint range guard
  const double* iv_max;
  // every full 32-particle tile of the span is 16-byte aligned in all arrays:
  // tiles stream through shared memory with TMA bulk copies
  int bulk;
  // dynamic work distribution: next unclaimed particle of the span
  unsigned long long* work;
  // two-pass fused span (push-only then deposit-only launch): one bit per
  // span particle whose push failed — set by the push pass, skipped by the
  // deposit pass (NULL: not used)
  unsigned* skip;
};

// particles per dynamically claimed chunk (32 tiles of a warp)
constexpr int kChunk = 1024;

// ---- TMA bulk copies and mbarriers (sm_90+ PTX, UBLKCP in SASS) ----------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ unsigned lane_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

// 32-byte read-only loads (LDG.E.ENL2.256, sm_100+): one node record of
// floats, or half a record of doubles, per instruction
__device__ __forceinline__ void ldg256(const float* p, float r[8]) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7])
      : "l"(p));
}
__device__ __forceinline__ void ldg256(const double* p, double r[4]) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
      : "l"(p));
}

// one node record as 16-byte vector stores
__device__ __forceinline__ void store_record(float* o, const float* r) {
  reinterpret_cast<float4*>(o)[0] = make_float4(r[0], r[1], r[2], r[3]);
  reinterpret_cast<float4*>(o)[1] = make_float4(r[4], r[5], r[6], r[7]);
}
__device__ __forceinline__ void store_record(double* o, const double* r) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    reinterpret_cast<double2*>(o)[k] = make_double2(r[2 * k], r[2 * k + 1]);
}

// E, B, invvol -> one 8-element record per node, so one corner of a gather is
// a couple of 16-byte loads from one record and the deposit's control volume
// comes from the same line.  T = double (parity: exact widening) or the fast
// policy's compute type.
template <typename F, typename T>
__global__ void pack_nodes(const F* __restrict__ E, const F* __restrict__ B,
                           const F* __restrict__ invvol, int NN, T* __restrict__ out,
                           unsigned long long* iv_max) {
  const int stride = gridDim.x * blockDim.x;
  double vmax = 0.0;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < NN; n += stride) {
    if (invvol) vmax = fmax(vmax, fabs((double)invvol[n]));
    T r[8];
    r[0] = E ? (T)E[n] : T(0);
    r[1] = E ? (T)E[NN + n] : T(0);
    r[2] = E ? (T)E[2 * NN + n] : T(0);
    r[3] = B ? (T)B[n] : T(0);
    r[4] = B ? (T)B[NN + n] : T(0);
    r[5] = B ? (T)B[2 * NN + n] : T(0);
    r[6] = invvol ? (T)invvol[n] : T(0);
    r[7] = T(0);
    store_record(out + (size_t)n * 8, r);
  }
  // one same-address atomic per warp, not per thread (a per-thread atomicMax
  // serialised ~NN updates in one L2 slice); non-negative doubles order like
  // their bit patterns
  unsigned long long bits = (unsigned long long)__double_as_longlong(vmax);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = b > bits ? b : bits;
  }
  if (iv_max && bits != 0ull && (threadIdx.x & 31) == 0) atomicMax(iv_max, bits);
}

// --------------------------------------------------------------------------
// Deposition.  Contribution (moment m, corner c) of one particle is
//   rint((base_c * m) * scale),  base_c = (q * (wx*wy*wz)) * invvol_c
// (kernels.py:707-734), m in {1, u, v, w, uu, uv, uw, vv, vw, ww}.  The
// policy stages per particle the 8 bases (pre-multiplied by scale when that
// is exact — PRESCALE) and the 10 moment values as doubles.
//
// Each warp walks a contiguous run of (cell-sorted) particles; the 80 sums
// of the cell currently being filled live in registers spread over the 32
// lanes: lane L owns corner c = L & 7 of moments g, g+4, g+8 (g = L >> 3).
// Per tile of 32 particles the owning lanes stage their values in shared
// memory, then all lanes fold every particle into their 2-3 accumulators —
// no cross-lane reduction at all.  A second slot keeps the sums of the last
// "stray" cell (a particle that crossed into a neighbour cell, or the next
// cell of the sort) so it does not force a flush of the main cell.  Sums are
// flushed with one REDG.ADD.64 per (slot, value) when a slot is evicted.

__device__ __forceinline__ void red_add(i64* p, i64 v) {
  if (v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// Shared-memory staging of one warp (doubles), particle-minor so a lane reads
// the values of two consecutive particles with one 16-byte load:
//   bases   [corner c][particle]            8 rows
//   moments [group g][slot j][particle]     12 rows: slot j of group g holds
//           moment g + 4j (zero for g + 4j >= 10)
// Rows are padded to 34 doubles (272 B) so the 8 corner rows / 4 group rows
// read by one warp instruction fall in distinct banks.
constexpr int kRow = 34;
constexpr int kStageBs = 8 * kRow;
constexpr int kStageMv = 12 * kRow;
constexpr int kWarpStage = kStageBs + kStageMv;
// particle tiles: 2 stages x 7 arrays x 32 particles of P, + 2 mbarriers
template <typename P>
__host__ __device__ constexpr int warp_smem_doubles() {
  return kWarpStage + (2 * 7 * 32 * (int)sizeof(P)) / 8 + 2;
}

// Exact rint without the conversion pipe: for |t| < 2^51, t + 1.5*2^52 lands
// in [2^52, 2^53) where the ulp is 1, so the FP add rounds t half-to-even
// exactly like cvt.rni and the low mantissa bits hold rint(t) in two's
// complement: bits(t + M) = bits(M) + rint(t).  Slots accumulate raw bit
// patterns and subtract n * bits(M) when flushed.  Tiles whose values could
// leave the range take the cvt path instead (checked per particle).
// FMA = true (fast policy only) rounds the exact product b*m instead of
// RN(b*m) — one rounding less, not bitwise the reference.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr i64 kMagicBits = 0x4338000000000000LL;
constexpr double kMagicLimit = 1125899906842624.0;  // 2^50

struct Slot {
  int key;
  int n;  // folded particles since the last flush (bit-pattern bias count)
  u64 s0, s1, s2;
};

__device__ __forceinline__ void red_add_always(i64* p, i64 v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// Flush a slot: one REDG.ADD.64 per value, issued unconditionally (a zero
// add is cheaper than the branch around it); lanes of groups 2-3 own only
// two values.
__device__ __forceinline__ void slot_flush(const Slot& sl, i64* __restrict__ acc, int NN,
                                           int m0, int coff, bool third) {
  if (sl.key < 0) return;
  const u64 bias = (u64)sl.n * (u64)kMagicBits;
  i64* p = acc + ((size_t)m0 * NN + (size_t)(sl.key + coff));
  const size_t st4 = (size_t)4 * NN;
  red_add_always(p, (i64)(sl.s0 - bias));
  red_add_always(p + st4, (i64)(sl.s1 - bias));
  if (third) red_add_always(p + 2 * st4, (i64)(sl.s2 - bias));
}

// quantised value as a biased bit pattern: bits(M) + rint(t)
template <bool PRESCALE, bool MAGIC, bool FMA>
__device__ __forceinline__ u64 qbits(double b, double m, double sc) {
  if (MAGIC) {
    if (FMA) return (u64)__double_as_longlong(__fma_rn(b, m, kMagic));
    const double t = PRESCALE ? b * m : b * m * sc;
    return (u64)__double_as_longlong(t + kMagic);
  }
  const double t = PRESCALE ? b * m : b * m * sc;
  return (u64)__double2ll_rn(t) + (u64)kMagicBits;
}

// staged particle k into S: this lane's corner lc of moments lg, lg+4, lg+8
template <bool PRESCALE, bool MAGIC, bool FMA>
__device__ __forceinline__ void fold_one(Slot& S, const double* st_bs, const double* st_mv,
                                         int k, int lc, int lg, double sc) {
  const double b = st_bs[lc * kRow + k];
  const double* mv = st_mv + lg * 3 * kRow + k;
  S.s0 += qbits<PRESCALE, MAGIC, FMA>(b, mv[0], sc);
  S.s1 += qbits<PRESCALE, MAGIC, FMA>(b, mv[kRow], sc);
  S.s2 += qbits<PRESCALE, MAGIC, FMA>(b, mv[2 * kRow], sc);  // 0 for lane groups 2, 3
  S.n += 1;
}

// All 32 staged particles into S, two particles per step: one 16-byte load
// per staged row, and the two contributions of a value summed with one
// 3-input 64-bit add (IADD3 + IADD3.X).
template <bool PRESCALE, bool MAGIC, bool FMA>
__device__ __forceinline__ void fold_tile(Slot& S, const double* st_bs, const double* st_mv,
                                          int lc, int lg, bool third, double sc) {
  const double* br = st_bs + lc * kRow;
  const double* mr = st_mv + lg * 3 * kRow;
#pragma unroll 4
  for (int k = 0; k < 32; k += 2) {
    const double2 b = *reinterpret_cast<const double2*>(br + k);
    const double2 m0 = *reinterpret_cast<const double2*>(mr + k);
    const double2 m1 = *reinterpret_cast<const double2*>(mr + kRow + k);
    S.s0 += qbits<PRESCALE, MAGIC, FMA>(b.x, m0.x, sc) + qbits<PRESCALE, MAGIC, FMA>(b.y, m0.y, sc);
    S.s1 += qbits<PRESCALE, MAGIC, FMA>(b.x, m1.x, sc) + qbits<PRESCALE, MAGIC, FMA>(b.y, m1.y, sc);
    if (third) {
      // lane groups 2-3 own two values: their third row is not read
      const double2 m2 = *reinterpret_cast<const double2*>(mr + 2 * kRow + k);
      S.s2 += qbits<PRESCALE, MAGIC, FMA>(b.x, m2.x, sc) + qbits<PRESCALE, MAGIC, FMA>(b.y, m2.y, sc);
    }
  }
  S.n += 32;
}

// Stage the moment values m0..m9 = 1 u v w uu uv uw vv vw ww of one particle
// into its column (mv = st_mv + lane): row g*3 + j holds moment g + 4j.
__device__ __forceinline__ void stage_moments(double* mv, double u, double v, double w,
                                              double uu, double uv, double uw, double vv,
                                              double vw, double ww) {
  const double r[12] = {1.0, uu, vw, u, uv, ww, v, uw, 0.0, w, vv, 0.0};
#pragma unroll
  for (int i = 0; i < 12; ++i) mv[i * kRow] = r[i];
}

__device__ __forceinline__ void stage_bases(double* st, const double bs[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) st[c * kRow] = bs[c];
}

// |base_c * m| < 2^50 for every (corner, moment) keeps the magic rint exact.
// |base_c| <= |q| * iv_max (weights <= 1) and |m| <= max(1, u^2, v^2, w^2)
// (|uv| <= max(u^2, v^2)), so one bound per particle suffices; the bound
// is slightly loose, a failing tile just takes the cvt path.
__device__ __forceinline__ bool magic_unsafe(double qbound, double uu, double vv, double ww,
                                             double lim) {
  const double mm = fmax(1.0, fmax(uu, fmax(vv, ww)));
  return !(fabs(qbound) * mm < lim);
}

// Fold one staged tile into the slots.  Lanes are grouped by cell with
// ballots: the group of the main slot's cell (usually almost the whole warp)
// and, one by one, the few other cells present, which go through the stray
// slot; strays then have their bases zeroed so the main fold runs unmasked
// over all 32 (invalid lanes staged zero bases too).
template <bool PRESCALE, bool FMA>
__device__ __forceinline__ void deposit_tile(Slot& A, Slot& Bs, i64* __restrict__ acc, int NN,
                                             int key, bool big, double* st_bs,
                                             const double* st_mv, unsigned lane, int lc,
                                             int lg, int coff, bool third, double sc) {
  const bool has = key >= 0;
  const unsigned V = __ballot_sync(0xffffffffu, has);
  const bool magic = __ballot_sync(0xffffffffu, big) == 0u;
  if (V == 0u) return;
  unsigned MA = __ballot_sync(0xffffffffu, has && key == A.key);
  if (MA == 0u) {
    const int knew = __shfl_sync(0xffffffffu, key, __ffs(V) - 1);
    if (knew == Bs.key) {
      const Slot t = A;
      A = Bs;
      Bs = t;
    } else {
      slot_flush(Bs, acc, NN, lg, coff, third);
      Bs = A;
      A.key = knew;
      A.n = 0;
      A.s0 = A.s1 = A.s2 = 0;
    }
    MA = __ballot_sync(0xffffffffu, has && key == A.key);
  } else if (MA != V) {
    // a sorted run crossing into its next cell: once the new cell holds
    // the majority of the tile, make it the main slot
    const int kc = __shfl_sync(0xffffffffu, key, 31 - __clz(V));
    const unsigned MC = __ballot_sync(0xffffffffu, has && key == kc);
    if (__popc(MC) > __popc(MA)) {
      if (kc == Bs.key) {
        const Slot t = A;
        A = Bs;
        Bs = t;
      } else {
        slot_flush(Bs, acc, NN, lg, coff, third);
        Bs = A;
        A.key = kc;
        A.n = 0;
        A.s0 = A.s1 = A.s2 = 0;
      }
      MA = MC;
    }
  }
  const unsigned strays = V & ~MA;
  unsigned rest = strays;
  while (rest) {
    const int k2 = __shfl_sync(0xffffffffu, key, __ffs(rest) - 1);
    const unsigned M2 = __ballot_sync(0xffffffffu, has && key == k2);
    rest &= ~M2;
    if (k2 != Bs.key) {
      slot_flush(Bs, acc, NN, lg, coff, third);
      Bs.key = k2;
      Bs.n = 0;
      Bs.s0 = Bs.s1 = Bs.s2 = 0;
    }
    if (magic) {
      for (unsigned m = M2; m; m &= m - 1u)
        fold_one<PRESCALE, true, FMA>(Bs, st_bs, st_mv, __ffs(m) - 1, lc, lg, sc);
    } else {
      for (unsigned m = M2; m; m &= m - 1u)
        fold_one<PRESCALE, false, FMA>(Bs, st_bs, st_mv, __ffs(m) - 1, lc, lg, sc);
    }
  }
  if (strays) {
    __syncwarp();  // every lane is done reading the staged rows
    if ((strays >> lane) & 1u) {
#pragma unroll
      for (int c = 0; c < 8; ++c) st_bs[c * kRow + lane] = 0.0;
    }
    __syncwarp();
  }
  if (magic)
    fold_tile<PRESCALE, true, FMA>(A, st_bs, st_mv, lc, lg, third, sc);
  else
    fold_tile<PRESCALE, false, FMA>(A, st_bs, st_mv, lc, lg, third, sc);
}

// --------------------------------------------------------------------------
// One kernel body for fused / push-only / deposit-only.  Each warp owns a
// contiguous run of the span and walks it 32 particles at a time (coalesced
// SoA loads/stores); every lane of a warp runs the same trip count so warp
// collectives always see 32 lanes.
//
// Policy provides:  P, F, NodeT, Consts (per-thread constants built from the
// params once), kFmaFold,
//   static int push(const Params&, const Consts&, P& x, P& y, P& z, P& u, P& v, P& w)
//   static int stage(const Params&, const Consts&, bool valid, P x, P y, P z,
//                    P u, P v, P w, P q, double* st_bs_lane, double* st_mv_lane,
//                    bool& big)
//     -> cell key (node index of corner 000) or -1 when outside the box.
#ifndef BP_MIN_BLOCKS
#define BP_MIN_BLOCKS 3
#endif
template <class Pol, bool DO_PUSH, bool DO_DEPOSIT, bool PRESCALE>
__global__ void __launch_bounds__(256, BP_MIN_BLOCKS)
    span_kernel(SpanParams<typename Pol::P, typename Pol::F> a) {
  typedef typename Pol::P P;
  extern __shared__ double stage_all[];
  const unsigned lane = lane_id();
  const int wib = threadIdx.x >> 5;
  // per-warp shared memory: deposit staging [+ particle tile stages when bulk]
  double* const st_bs =
      stage_all + (size_t)wib * (a.bulk ? warp_smem_doubles<P>() : kWarpStage);
  double* const st_mv = st_bs + kStageBs;
  // particle tile stages [2][7][32] of P, then the 2 mbarriers
  P* const tiles = reinterpret_cast<P*>(st_bs + kWarpStage);
  unsigned long long* const bars = reinterpret_cast<unsigned long long*>(
      st_bs + kWarpStage + (2 * 7 * 32 * (int)sizeof(P)) / 8);
  const int sx = a.NY * a.NZ, sy = a.NZ;
  // this lane's share of the 80 sums
  const int lc = lane & 7, lg = lane >> 3;
  const int coff = (lc & 1) * sx + ((lc >> 1) & 1) * sy + ((lc >> 2) & 1);
  const bool third = lg < 2;
  const double sc = a.d.scale;
  const typename Pol::Consts K(a);  // per-thread constants of the policy
  Slot A{-1, 0, 0, 0, 0}, Bs{-1, 0, 0, 0, 0};
  int worst = ST_OK;
  // Particle SoA streams: full tiles move HBM <-> shared memory with TMA bulk
  // copies (one elected lane, 128/256-byte transfers per array, the next
  // tile's load in flight while this one is computed); a ragged last tile or
  // an unaligned span uses plain coalesced loads/stores.
  P* const arr[7] = {a.x, a.y, a.z, a.u, a.v, a.w, const_cast<P*>(a.q)};
  const int narr = DO_DEPOSIT ? 7 : 6;
  const unsigned tile_bytes = 32 * sizeof(P);
  if (a.bulk && lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    fence_proxy_async();
  }
  __syncwarp();
  unsigned phase = 0;  // bit s: parity of stage s's next completion
  // Warps claim contiguous chunks of the span from a global counter (no tail
  // of idle SMs, no imbalance from uneven disorder); slot sums persist across
  // chunks — any grouping of the integer sums is exact.
  for (;;) {
  i64 w0 = 0;
  if (lane == 0) w0 = (i64)atomicAdd(a.work, (unsigned long long)kChunk);
  w0 = __shfl_sync(0xffffffffu, w0, 0);
  if (w0 >= a.count) break;
  const i64 w1 = w0 + kChunk < a.count ? w0 + kChunk : a.count;
  auto full = [&](i64 t) { return a.bulk && t + 32 <= w1; };
  auto issue = [&](i64 t, int stg) {
    if (lane == 0) {
      mbar_expect_tx(bars + stg, narr * tile_bytes);
      for (int k = 0; k < narr; ++k)
        bulk_load(tiles + (stg * 7 + k) * 32, arr[k] + a.start + t, tile_bytes, bars + stg);
    }
  };
  if (full(w0)) {
    // stage 0 may still feed the previous chunk's last bulk store
    if (DO_PUSH && lane == 0) bulk_wait_read_all();
    __syncwarp();
    issue(w0, 0);
  }
  int it = 0;
  for (i64 t0 = w0; t0 < w1; t0 += 32, ++it) {
    const int stg = it & 1;
    const i64 r = t0 + lane;
    bool valid = r < w1;
    if (!DO_PUSH && a.skip) valid = valid && !((__ldg(a.skip + (t0 >> 5)) >> lane) & 1u);
    const i64 p = a.start + r;
    const bool cur_full = full(t0);
    if (full(t0 + 32)) {
      // the other stage held tile it-1: its bulk store must have read it
      if (DO_PUSH && lane == 0) bulk_wait_read_all();
      __syncwarp();
      issue(t0 + 32, stg ^ 1);
    }
    P xp = 0, yp = 0, zp = 0, un = 0, vn = 0, wn = 0, qp = 0;
    P* const cur = tiles + stg * 7 * 32;
    if (cur_full) {
      mbar_wait(bars + stg, (phase >> stg) & 1u);
      phase ^= 1u << stg;
      xp = cur[0 * 32 + lane]; yp = cur[1 * 32 + lane]; zp = cur[2 * 32 + lane];
      un = cur[3 * 32 + lane]; vn = cur[4 * 32 + lane]; wn = cur[5 * 32 + lane];
      if (DO_DEPOSIT) qp = cur[6 * 32 + lane];
    } else if (valid) {
      // streamed once: evict-first so the field records keep L1
      xp = __ldcs(a.x + p); yp = __ldcs(a.y + p); zp = __ldcs(a.z + p);
      un = __ldcs(a.u + p); vn = __ldcs(a.v + p); wn = __ldcs(a.w + p);
      if (DO_DEPOSIT) qp = __ldcs(a.q + p);
    }
    bool failed = false;
    if (DO_PUSH) {
      if (valid) {
        const int st = Pol::push(a, K, xp, yp, zp, un, vn, wn);
        if (st != ST_OK) {
          // not stored, not deposited (kernels.py:618-621, 672-676); a bulk
          // store writes the tile's loaded values back unchanged
          worst = st > worst ? st : worst;
          valid = false;
          failed = true;
        } else if (cur_full) {
          cur[0 * 32 + lane] = xp; cur[1 * 32 + lane] = yp; cur[2 * 32 + lane] = zp;
          cur[3 * 32 + lane] = un; cur[4 * 32 + lane] = vn; cur[5 * 32 + lane] = wn;
        } else {
          __stcs(a.x + p, xp); __stcs(a.y + p, yp); __stcs(a.z + p, zp);
          __stcs(a.u + p, un); __stcs(a.v + p, vn); __stcs(a.w + p, wn);
        }
      }
      if (cur_full) {
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          for (int k = 0; k < 6; ++k)
            bulk_store(arr[k] + a.start + t0, cur + k * 32, tile_bytes);
          bulk_commit();
        }
      }
      if (a.skip) {
        const unsigned fb = __ballot_sync(0xffffffffu, failed);
        if (fb && lane == 0) atomicOr(a.skip + (t0 >> 5), fb);
      }
    }
    if (DO_DEPOSIT) {
      bool big = false;
      const int key = Pol::template stage<PRESCALE>(a, K, valid, xp, yp, zp, un, vn, wn, qp,
                                                    st_bs + lane, st_mv + lane, big);
      if (valid && key < 0) worst = ST_DOMAIN > worst ? ST_DOMAIN : worst;
      __syncwarp();
      deposit_tile<PRESCALE, Pol::kFmaFold>(A, Bs, a.acc, a.NN, key, big, st_bs, st_mv, lane,
                                            lc, lg, coff, third, sc);
      __syncwarp();
    }
  }
  }  // chunks
  if (DO_DEPOSIT) {
    slot_flush(A, a.acc, a.NN, lg, coff, third);
    slot_flush(Bs, a.acc, a.NN, lg, coff, third);
  }
  if (DO_PUSH && a.bulk && lane == 0) bulk_wait_all();
  if (worst != ST_OK) atomicMax(a.status, worst);
}

}  // namespace bp
