// Host-side launch plumbing shared by the parity and fast translation units:
// Call -> SpanParams, per-call node records, grid sizing, dispatch over the
// supported (particle, field) dtype pairs.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "bp_common.cuh"
#include "bp_launch.h"

namespace bp {
namespace {

template <typename P, typename F>
SpanParams<P, F> make_params(const Call& c) {
  SpanParams<P, F> a;
  a.x = (P*)c.x; a.y = (P*)c.y; a.z = (P*)c.z;
  a.u = (P*)c.u; a.v = (P*)c.v; a.w = (P*)c.w;
  a.q = (const P*)c.q;
  a.start = c.start; a.count = c.count;
  a.E = (const F*)c.E; a.B = (const F*)c.B;
  a.acc = (i64*)c.acc;
  a.invvol = (const F*)c.invvol;
  a.ox = (P)c.geo_f[3]; a.oy = (P)c.geo_f[4]; a.oz = (P)c.geo_f[5];
  a.Lx = (P)c.geo_f[6]; a.Ly = (P)c.geo_f[7]; a.Lz = (P)c.geo_f[8];
  // ox + Lx and (ox+Lx) + (ox+Lx) in particle precision (kernels.py:507-533)
  a.hx = (P)(a.ox + a.Lx); a.hy = (P)(a.oy + a.Ly); a.hz = (P)(a.oz + a.Lz);
  a.hx2 = (P)(a.hx + a.hx); a.hy2 = (P)(a.hy + a.hy); a.hz2 = (P)(a.hz + a.hz);
  a.gdx = (F)c.geo_g[0]; a.gdy = (F)c.geo_g[1]; a.gdz = (F)c.geo_g[2];
  a.gox = (F)c.geo_g[3]; a.goy = (F)c.geo_g[4]; a.goz = (F)c.geo_g[5];
  a.nx = (int)c.geo_i[0]; a.ny = (int)c.geo_i[1]; a.nz = (int)c.geo_i[2];
  a.bcx = (int)c.geo_i[3]; a.bcy = (int)c.geo_i[4]; a.bcz = (int)c.geo_i[5];
  a.NY = a.ny + 1; a.NZ = a.nz + 1;
  a.NN = (a.nx + 1) * a.NY * a.NZ;
  a.dt = (P)c.dt; a.dth = (P)c.dth; a.qdt2m = (P)c.qdt2m; a.beta = (P)c.beta;
  a.one = (P)c.one;
  a.two = (P)(a.one + a.one);
  a.beta2 = (P)(a.beta * a.beta);  // f32*f32 stays f32 (kernels.py:615)
  a.scale = (F)c.scale;
  a.n_iters = c.n_iters; a.mixed = c.mixed; a.apply_bc = c.apply_bc;
  a.status = c.status;
  a.gather_out = (P*)c.out;
  a.fnode = nullptr;
  const P o3[3] = {a.ox, a.oy, a.oz}, L3[3] = {a.Lx, a.Ly, a.Lz};
  const P h3[3] = {a.hx, a.hy, a.hz}, h23[3] = {a.hx2, a.hy2, a.hz2};
  const F gd3[3] = {a.gdx, a.gdy, a.gdz}, go3[3] = {a.gox, a.goy, a.goz};
  for (int k = 0; k < 3; ++k) {
    a.d.o[k] = (double)o3[k]; a.d.L[k] = (double)L3[k];
    a.d.hi[k] = (double)h3[k]; a.d.hi2[k] = (double)h23[k];
    a.d.gd[k] = (double)gd3[k]; a.d.go[k] = (double)go3[k];
    a.d.inv_gd[k] = 1.0 / a.d.gd[k];
    a.d.go_s[k] = a.d.go[k] / a.d.gd[k];
  }
  a.d.dt = (double)a.dt; a.d.dth = (double)a.dth; a.d.qdt2m = (double)a.qdt2m;
  a.d.beta = (double)a.beta; a.d.one = (double)a.one; a.d.two = (double)a.two;
  a.d.beta2 = (double)a.beta2; a.d.scale = (double)a.scale;
  a.iv_max = nullptr;
  a.work = nullptr;
  a.skip = c.skip;
  {
    // TMA bulk tiles need every full tile 16-byte aligned in all 7 arrays
    const void* ptrs[7] = {c.x, c.y, c.z, c.u, c.v, c.w, c.q};
    bool ok = ((c.start * (int64_t)sizeof(P)) % 16) == 0;
    for (int k = 0; k < 7; ++k)
      if (ptrs[k] && ((uintptr_t)ptrs[k] % 16) != 0) ok = false;
    if (!c.x || !c.u || (c.op != OP_PUSH && !c.q)) ok = false;
    // opt-in: measured slower on B200 at C3 (its shared memory is taken from
    // the L1 that serves the field gathers), see DESIGN.md
    const char* env = getenv("BP_TMA_STREAM");
    a.bulk = (ok && env && env[0] == '1') ? 1 : 0;
  }
  for (int k = 0; k < 3; ++k) {
    a.f.o[k] = (float)a.d.o[k]; a.f.L[k] = (float)a.d.L[k];
    a.f.hi[k] = (float)a.d.hi[k]; a.f.hi2[k] = (float)a.d.hi2[k];
    a.f.idx[k] = (float)a.d.inv_gd[k]; a.f.ogs[k] = (float)a.d.go_s[k];
  }
  a.f.dt = (float)a.d.dt; a.f.dth = (float)a.d.dth; a.f.qdt2m = (float)a.d.qdt2m;
  a.f.beta = (float)a.d.beta; a.f.beta2 = (float)a.d.beta2; a.f.scale = (float)a.d.scale;
  return a;
}

constexpr int kThreads = 256;

inline int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <typename K>
int grid_for(K kernel, size_t smem, int64_t count, int per_block) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (count + per_block - 1) / per_block;
  const int64_t full = (int64_t)sm_count() * per_sm;
  int64_t g = need < full ? need : full;
  return (int)(g < 1 ? 1 : g);
}

inline bool is_pow2(double v) {
  int e;
  return v > 0.0 && std::isfinite(v) && std::frexp(v, &e) == 0.5;
}

inline int launch_error(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

template <class Pol, bool PUSH, bool DEP, bool PRE>
int launch_span(const SpanParams<typename Pol::P, typename Pol::F>& a, int64_t count,
                cudaStream_t s) {
  auto k = span_kernel<Pol, PUSH, DEP, PRE>;
  // deposit staging always; the particle tile stages only on the TMA path
  // (the rest of the SM's shared memory stays L1 for the field gathers)
  constexpr size_t kFull =
      (size_t)(kThreads / 32) * warp_smem_doubles<typename Pol::P>() * sizeof(double);
  constexpr size_t kStageOnly = (size_t)(kThreads / 32) * kWarpStage * sizeof(double);
  // a push-only launch without TMA tiles touches no shared memory
  const size_t smem = a.bulk ? kFull : (DEP ? kStageOnly : 0);
  static bool attr[64] = {};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFull);
  });
  // one wave of resident blocks; every warp walks a contiguous run of >= 32
  const int grid = grid_for(k, smem, count, kThreads);
  const int th = timing_begin(TK_SPAN, s);
  k<<<grid, kThreads, smem, s>>>(a);
  timing_end(th, s);
  note_launch();
  return launch_error("span kernel launch");
}

// Build the node records on the stream, run, release (stream-ordered).
template <class Pol, bool PUSH, bool DEP>
int run_span(const Call& c, bool prescale_ok, cudaStream_t s) {
  typedef typename Pol::P P;
  typedef typename Pol::F F;
  typedef typename Pol::NodeT T;
  auto a = make_params<P, F>(c);
  T* fn = nullptr;
  const size_t rec_bytes = ((size_t)a.NN * 8 * sizeof(T) + 255) & ~(size_t)255;
  cudaError_t e = cudaMallocAsync((void**)&fn, rec_bytes + 256, s);
  if (e != cudaSuccess) {
    set_error("node record alloc: %s", cudaGetErrorString(e));
    return -2;
  }
  unsigned long long* ivm = reinterpret_cast<unsigned long long*>((char*)fn + rec_bytes);
  cudaMemsetAsync(ivm, 0, 2 * sizeof(unsigned long long), s);  // iv_max, work counter
  a.work = ivm + 1;
  const int pb = (a.NN + 255) / 256 < 4096 ? (a.NN + 255) / 256 : 4096;
  pack_nodes<F, T><<<pb, 256, 0, s>>>(PUSH ? a.E : nullptr, PUSH ? a.B : nullptr,
                                      DEP ? a.invvol : nullptr, a.NN, fn, ivm);
  a.iv_max = reinterpret_cast<const double*>(ivm);
  note_launch();
  a.fnode = fn;
  int rc;
  if (DEP && prescale_ok)
    rc = launch_span<Pol, PUSH, DEP, true>(a, c.count, s);
  else
    rc = launch_span<Pol, PUSH, DEP, false>(a, c.count, s);
  cudaFreeAsync(fn, s);
  return rc;
}

// Fused span as two launches of the generic kernel — push-only (high
// occupancy, no deposit staging) then deposit-only — with a bitmask of the
// particles whose push failed so they are not deposited (kernels.py:618-621).
// Same arithmetic as the one-pass kernel, and the deposit's exact integer sums
// make the moments identical.
template <class Pol>
int run_two_pass(const Call& c0, bool prescale_ok, cudaStream_t s) {
  Call c = c0;
  const size_t skip_bytes = (((size_t)c.count + 31) / 32 * 4 + 8 + 255) & ~(size_t)255;
  unsigned* skip = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&skip, skip_bytes, s);
  if (e != cudaSuccess) {
    set_error("skip bitmask alloc: %s", cudaGetErrorString(e));
    return -2;
  }
  cudaMemsetAsync(skip, 0, skip_bytes, s);
  c.skip = skip;
  c.apply_bc = 1;
  int rc = run_span<Pol, true, false>(c, prescale_ok, s);
  if (!rc) rc = run_span<Pol, false, true>(c, prescale_ok, s);
  cudaFreeAsync(skip, s);
  return rc;
}

// default on (measured at C3: parity single +1%, f64 fast +4%);
// BP_GENERIC_TWO_PASS=0 selects the one-pass fused kernel
inline bool two_pass_requested() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BP_GENERIC_TWO_PASS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

}  // namespace
}  // namespace bp
