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

}  // namespace

int launch_fast(const Call& c, cudaStream_t s) {
  // f32 particles, fused: the mover + deposit kernels of bp_split.cu
  // (BP_FAST_GENERIC=1 selects the generic policy kernel instead).  f64 stays
  // on the generic kernel: its per-contribution rint keeps the moments within
  // 1e-10 of the reference's lattice, which per-tile f64 sums do not (the
  // reference's own rounding noise is ~1e-10 of the small pressure moments).
  if (c.op == OP_FUSED && c.pbytes == 4) {
    const char* env = getenv("BP_FAST_GENERIC");
    if (!(env && env[0] == '1')) return split_fused(c, c.records, s);
  }
  if (c.pbytes == 8 && c.fbytes == 8) return dispatch<double, double>(c, s);
  if (c.pbytes == 4 && c.fbytes == 4) return dispatch<float, float>(c, s);
  if (c.pbytes == 4 && c.fbytes == 8) return dispatch<float, double>(c, s);
  set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", c.pbytes,
            c.fbytes);
  return -1;
}

}  // namespace bp
