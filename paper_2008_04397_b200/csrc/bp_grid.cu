// Device-side phase 4 of the cycle: the immediate
// consumers of the deposited moments, so the host solve receives ready
// inputs without a per-species host pass.
//   total          exact int64 sum over species   (fields.total_moments, fields.py:170-179)
//   susceptibility (theta dt^2 / 2) max(0, sum_s 4 pi rho_s qom_s)
//                                                  (maxwell.plasma_susceptibility,
//                                                   maxwell.py:163-179)
// Compiled with -fmad=false: the susceptibility is bitwise the reference's
// numpy expression order.
#include <cstdint>

#include "bp_launch.h"

namespace bp {
namespace {

constexpr int kMaxSpecies = 16;

struct SpeciesRows {
  const long long* rho[kMaxSpecies];  // row 0 (rho) of each species' accumulator
  double qom[kMaxSpecies];
};

__global__ void total_kernel(SpeciesRows s, int ns, int64_t n, long long* total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    long long t = 0;
    for (int k = 0; k < ns; ++k) t += s.rho[k][i];
    total[i] = t;
  }
}

// rho = acc * (1 / 2^43) in float64 (int64 -> double rounds to nearest),
// rounded to f32 and back when the fields are single (MomentGrid.to_float);
// chi accumulates (4 pi * rho) * qom species by species, is clipped at 0
// and scaled by ((0.5 * theta) * dt) * dt.
__global__ void chi_kernel(SpeciesRows s, int ns, int single, double factor, int64_t n,
                           double* chi) {
  const double four_pi = 4.0 * 3.141592653589793;
  const double inv_scale = 1.0 / 8796093022208.0;  // 2^-43
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double c = 0.0;
    for (int k = 0; k < ns; ++k) {
      double rho = __ll2double_rn(s.rho[k][i]) * inv_scale;
      if (single) rho = (double)__double2float_rn(rho);
      c = c + four_pi * rho * s.qom[k];
    }
    if (c < 0.0) c = 0.0;
    chi[i] = c * factor;
  }
}

int blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

int fill(SpeciesRows& s, const long long* const* accs, const double* qom, int ns) {
  if (ns < 1 || ns > kMaxSpecies) {
    set_error("species count %d outside 1..%d", ns, kMaxSpecies);
    return -1;
  }
  for (int k = 0; k < ns; ++k) {
    s.rho[k] = accs[k];
    s.qom[k] = qom ? qom[k] : 0.0;
  }
  return 0;
}

}  // namespace

int moments_total(const long long* const* rows, int ns, int64_t n, long long* total,
                  cudaStream_t st) {
  SpeciesRows s;
  if (fill(s, rows, nullptr, ns)) return -1;
  total_kernel<<<blocks(n), 256, 0, st>>>(s, ns, n, total);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("total_kernel: %s", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

int susceptibility(const long long* const* rho_rows, const double* qom, int ns, int single,
                   double factor, int64_t n, double* chi, cudaStream_t st) {
  SpeciesRows s;
  if (fill(s, rho_rows, qom, ns)) return -1;
  chi_kernel<<<blocks(n), 256, 0, st>>>(s, ns, single, factor, n, chi);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("chi_kernel: %s", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

}  // namespace bp
