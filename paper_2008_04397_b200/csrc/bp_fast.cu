// Fast build of the span kernels: FMA contraction, reciprocal multiplies and
// native particle-precision arithmetic (bp_fast_policy.cuh).  Deposits keep
// the exact int64 lattice.
#include "bp_fast_policy.cuh"
#include "bp_launch_impl.cuh"

namespace bp {
namespace {

template <typename P, typename F>
int dispatch(const Call& c, cudaStream_t s) {
  typedef FastPolicy<P, F> Pol;
  switch (c.op) {
    case OP_FUSED:
      return two_pass_requested() ? run_two_pass<Pol>(c, true, s)
                                  : run_span<Pol, true, true>(c, true, s);
    case OP_PUSH: return run_span<Pol, true, false>(c, true, s);
    case OP_DEPOSIT: return run_span<Pol, false, true>(c, true, s);
  }
  set_error("op %d has no fast arithmetic variant", c.op);
  return -1;
}

// f64 fused span: the split mover (coefficient records, interior skip;
// bp_split.cu) then the generic per-contribution deposit over the particles
// whose push succeeded — the arithmetic of the f64 binned path
// (bp_bins64.cu), which is bitwise this one
int f64_split_fused(const Call& c0, cudaStream_t s) {
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
  int rc = split_push_f64(c, c.records, skip, s);
  if (!rc) rc = run_span<FastPolicy<double, double>, false, true>(c, true, s);
  cudaFreeAsync(skip, s);
  return rc;
}

}  // namespace

int launch_fast(const Call& c, cudaStream_t s) {
  // f32 particles, fused: the mover + deposit kernels of bp_split.cu; f64,
  // fused: the split mover + the generic deposit, whose per-contribution rint
  // keeps the moments within 1e-10 of the reference's lattice (per-tile f64
  // sums do not: the reference's own rounding noise is ~1e-10 of the small
  // pressure moments).  BP_FAST_GENERIC=1 selects the generic policy kernel
  // for both.
  const char* env = getenv("BP_FAST_GENERIC");
  const bool generic = env && env[0] == '1';
  if (c.op == OP_FUSED && c.pbytes == 4 && !generic) return split_fused(c, c.records, s);
  if (c.op == OP_FUSED && c.pbytes == 8 && c.fbytes == 8 && !generic)
    return f64_split_fused(c, s);
  if (c.pbytes == 8 && c.fbytes == 8) return dispatch<double, double>(c, s);
  if (c.pbytes == 4 && c.fbytes == 4) return dispatch<float, float>(c, s);
  if (c.pbytes == 4 && c.fbytes == 8) return dispatch<float, double>(c, s);
  set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", c.pbytes,
            c.fbytes);
  return -1;
}

}  // namespace bp
