// Internal interface between the C ABI (bp_capi.cu) and the kernel
// translation units (bp_parity.cu: -fmad=false, bp_fast.cu: FMA).
#pragma once
#include <mutex>
#include <cstdint>
#include <cuda_runtime.h>

namespace bp {

enum Op { OP_FUSED = 0, OP_PUSH = 1, OP_DEPOSIT = 2, OP_GATHER = 3 };

// One span call, reference argument meaning (kernels.py:82,310,385,458).
struct Call {
  int op;
  int pbytes, fbytes;
  void *x, *y, *z, *u, *v, *w;
  const void* q;
  int64_t start, count;
  const void* E;
  const void* B;
  int64_t* acc;
  const void* invvol;
  double geo_f[9], geo_g[9];
  int64_t geo_i[6];
  double dt, dth, qdt2m, beta, one, scale;
  int n_iters, mixed, apply_bc;
  void* out;    // gather rows
  int* status;  // device int, atomicMax
  const void* records;  // prebuilt cell records (bp_field_records_build) or NULL
  unsigned* skip;       // two-pass fused span: failed-push bitmask (internal)
};

// Return 0 on a successful enqueue, else a negative BP_E* code.
int launch_parity(const Call& c, cudaStream_t s);
int launch_fast(const Call& c, cudaStream_t s);

void set_error(const char* fmt, ...);

// Fast arithmetic, fused op, as the mover + deposit kernel pair of
// bp_split.cu (f32 particles with f32 or f64 fields, and f64 / f64): per-cell
// coefficient records `rec` (split_records_bytes, particle precision) built
// by split_pack_records, or NULL to build them on the stream for this call.
size_t split_records_bytes(int pbytes, const int64_t* geo_i);
int split_pack_records(int pbytes, int fbytes, const void* E, const void* B,
                       const int64_t* geo_i, void* rec, cudaStream_t s);
int split_fused(const Call& c, const void* rec, cudaStream_t s);
// the f64 fast fused span's mover pass (bp_split.cu) with the failed-push bitmask
int split_push_f64(const Call& c, const void* rec, unsigned* skip, cudaStream_t s);

// Cell-binned f32 fast path (bp_bins.cu): the bin layout of one species
struct BinsArgs {
  void* rec;             // particle records x y z u | v w q 0 per slot (2 x 4 scalars)
  int64_t* ids;
  const int64_t* start;  // [ncell + 1] slot offsets
  int* count;            // [ncell] live particles per bin
  int64_t ncell;
  void* leavers;         // leaver list (bins_leaver_bytes() each)
  int64_t leaver_cap;
  void* overflow;        // overflow list (same records)
  int64_t overflow_cap;
  uint64_t* stat;        // [8] counters (bp_b200.h BP_BINS_STAT_*)
  void* late;            // misplaced particles met by the deposit (same records)
  int64_t late_cap;
  int pbytes = 4;        // particle scalar: 4 (32-byte records) or 8 (64-byte)
};
int bins_leaver_bytes(int pbytes);
int bins_cycle(const Call& c, const BinsArgs& ba, cudaStream_t s);
int bins_cycle64(const Call& c, const BinsArgs& ba, cudaStream_t s);  // bp_bins64.cu

int bins_plan(const Call& c, int* count, int64_t* start, double frac, int smin, int64_t* total,
              cudaStream_t s);
int bins_fill(const Call& c, const int64_t* src_ids, const int64_t* start, void* dst_rec,
              int64_t* dst_ids, cudaStream_t s);
int bins_export(const BinsArgs& ba, const void* src_rec, int64_t* offsets, void* const* dst,
                int64_t* dst_ids, int64_t* total, cudaStream_t s);
int bins_reslack_plan(const BinsArgs& ba, const void* src_rec, int* ncount, int64_t* nstart,
                      double frac, int smin, int64_t* total, cudaStream_t s);
int bins_reslack_copy(const BinsArgs& ba, const void* src_rec, const int64_t* nstart,
                      int* ncount, void* dst_rec, int64_t* dst_ids, cudaStream_t s);

// Bit-exact device loader (bp_init.cu): one species of the reference's
// init_maxwellian on the cell range [c0, c0 + nc)
struct InitArgs {
  int pbytes;
  uint64_t seed, species_id;
  int64_t n_cells, nx, ny;
  int ppc;
  int64_t c0, nc;
  double origin[3], spacing[3], drift[3], vth[3];
  const double* q_cell;  // [nc] device
  void* arr[7];          // x y z u v w q (device, nc * ppc each)
  int64_t* ids;
  int64_t* tail_k;       // tail-strip normals: 2 * ordinal + sign
  double* tail_u;        // ... and the accepted uniform
  int64_t tail_cap;
  int64_t* n_tail;       // host
  int skip_velocities;
};
int init_maxwellian(const InitArgs& A, cudaStream_t s);

// count of kernels this library launched (bp_kernel_launches)
void note_launch(int n = 1);

// device timing per kernel class (bp_timing_*): begin returns a handle or -1
enum { TK_MOVER = 0, TK_DEPOSIT = 1, TK_RECORDS = 2, TK_SPAN = 3, TK_COUNT = 4 };
int timing_begin(int cls, cudaStream_t s);
void timing_end(int handle, cudaStream_t s);

// keep the default stream-ordered pool's memory mapped between calls
void ensure_pool();

// Runs `set` once per device for this flag array (kernel attributes such as
// the dynamic shared memory limit are per device, so a process driving two
// GPUs must set them on each).  Thread-safe: a concurrent caller returns only
// after `set` has run (the host pipeline is called from thread pools).
template <class F>
inline void once_per_device(bool (&flags)[64], F&& set) {
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    set();
    return;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!flags[dev]) {
    set();
    flags[dev] = true;
  }
}

}  // namespace bp
