// Parity build of the span kernels: compiled with -fmad=false and IEEE
// division so every particle follows the reference numba arithmetic bit for
// bit (kernels.py:458-735).
#include "bp_launch_impl.cuh"
#include "bp_parity_policy.cuh"

namespace bp {
namespace {

template <typename P, typename F>
int run_gather(const Call& c, cudaStream_t s) {
  auto a = make_params<P, F>(c);
  double* fn = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&fn, (size_t)a.NN * 8 * sizeof(double), s);
  if (e != cudaSuccess) {
    set_error("node record alloc: %s", cudaGetErrorString(e));
    return -2;
  }
  const int pb = (a.NN + 255) / 256 < 4096 ? (a.NN + 255) / 256 : 4096;
  pack_nodes<F, double><<<pb, 256, 0, s>>>(a.E, a.B, (const F*)nullptr, a.NN, fn, nullptr);
  note_launch();
  a.fnode = fn;
  const int grid = grid_for(gather_kernel<P, F>, 0, c.count, kThreads);
  gather_kernel<P, F><<<grid, kThreads, 0, s>>>(a);
  note_launch();
  const int rc = launch_error("gather kernel launch");
  cudaFreeAsync(fn, s);
  return rc;
}

template <typename P, typename F>
int dispatch(const Call& c, cudaStream_t s) {
  typedef ParityPolicy<P, F> Pol;
  // (base*m)*scale == (base*scale)*m exactly only for a power-of-two scale
  const bool pre = is_pow2(c.scale);
  switch (c.op) {
    case OP_FUSED:
      return two_pass_requested() ? run_two_pass<Pol>(c, pre, s)
                                  : run_span<Pol, true, true>(c, pre, s);
    case OP_PUSH: return run_span<Pol, true, false>(c, pre, s);
    case OP_DEPOSIT: return run_span<Pol, false, true>(c, pre, s);
    case OP_GATHER: return run_gather<P, F>(c, s);
  }
  set_error("unknown op %d", c.op);
  return -1;
}

}  // namespace

int launch_parity(const Call& c, cudaStream_t s) {
  if (c.pbytes == 8 && c.fbytes == 8) return dispatch<double, double>(c, s);
  if (c.pbytes == 4 && c.fbytes == 4) return dispatch<float, float>(c, s);
  if (c.pbytes == 4 && c.fbytes == 8) return dispatch<float, double>(c, s);
  set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", c.pbytes,
            c.fbytes);
  return -1;
}

}  // namespace bp
