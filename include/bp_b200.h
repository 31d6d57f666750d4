/*
 * bp_b200.h — C ABI of the B200-native particle mover + moment deposition.
 *
 * Drop-in boundary for the reference package's compiled-kernel seam,
 * `batchpic.kernels` (/root/reference/pkg/src/batchpic/kernels.py).  Every
 * caller of that path (mover.py:85,135,154,179,194,221, pipeline.py:206 and
 * the acceptance tests) resolves `kernels.<name>` at call time, so binding
 * these entry points under those names replaces the path.  Arguments keep the
 * reference's positional order and meaning; only the dtype is made explicit
 * (pbytes / fbytes = 8 for float64, 4 for float32; supported pairs (8,8)
 * "double", (4,4) "single", (4,8) "mixed", as config.py:19-52 allows).
 *
 * Pointers
 *   Particle arrays, E, B, acc, invvol, out: DEVICE pointers (cudaMalloc /
 *   torch CUDA tensors), C-contiguous in the reference layout:
 *     particles  1-D, one array per component          (particles.py:23-81)
 *     E, B       (3, nx+1, ny+1, nz+1), k fastest      (fields.py:76-105)
 *     acc        (10, nx+1, ny+1, nz+1) int64, +=      (fields.py:108-162)
 *     invvol     (nx+1, ny+1, nz+1)                    (geometry.py:186-203)
 *   geo_f / geo_g / geo_i: HOST arrays, the reference's make_geo_arrays
 *   packs (kernels.py:57-67) with the P / F values widened to double.
 *   The *_host entry points take HOST particle/field/acc arrays instead and
 *   stream them through the device in batches (pinned staging, CUDA streams);
 *   that is the reference-facing call for populations held in host memory.
 *
 * Status (kernels.py:45-47, plus one GPU-only code)
 *   0 BP_OK, 1 BP_ERR_RUNAWAY, 2 BP_ERR_MIDPOINT, 3 BP_ERR_DOMAIN (a deposit
 *   or gather position outside the box; the reference indexes without
 *   checking, the GPU refuses).  As in the reference, a failing particle is
 *   neither stored nor deposited and processing continues.
 *   Negative returns are call errors: BP_EINVAL (bad arguments / unsupported
 *   dtype pair), BP_ECUDA (CUDA launch or runtime failure; see
 *   bp_last_error()).
 *
 * Synchrony
 *   d_status == NULL: the call synchronises `stream` and returns the worst
 *   particle status (reference semantics: the int the numba kernel returns).
 *   d_status != NULL: launch only; the worst status is atomicMax-ed into the
 *   device int *d_status and the call returns BP_OK once enqueued.
 *   `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Arithmetic ("arith" argument of the *_ex entry points)
 *   BP_ARITH_PARITY: bitwise the reference numba kernels (no FMA, IEEE
 *   division, numba's f32->f64 promotions).  BP_ARITH_FAST: FMA, reciprocal
 *   multiplies and native f32 arithmetic for f32 particles; agrees with the
 *   reference within 1e-10 (f64) / 1e-4 (f32) relative to the array maximum.
 *   The moment lattice (int64, quantum 2^-43, per-contribution rint) is the
 *   same in both, so deposits stay exact and order independent.
 */
#ifndef BP_B200_H
#define BP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_OK 0
#define BP_ERR_RUNAWAY 1
#define BP_ERR_MIDPOINT 2
#define BP_ERR_DOMAIN 3
#define BP_EINVAL (-1)
#define BP_ECUDA (-2)

#define BP_ARITH_PARITY 0
#define BP_ARITH_FAST 1

/* Library version, e.g. 100 for 0.1.0. */
int bp_version(void);

/* Last error message of the calling thread ("" if none). */
const char* bp_last_error(void);

/* Number of CUDA kernels this library has launched in this process (all
 * threads): the evidence behind a benchmark's "gpu_launches". */
long long bp_kernel_launches(void);

/* Device timing of this library's kernels (benchmark evidence): while
 * enabled, every mover / deposit / record-build / generic span launch is
 * bracketed by CUDA events on its stream.  bp_timing_read() waits for them
 * and returns per class (0 mover, 1 deposit, 2 record build, 3 generic span
 * kernel) the summed milliseconds and launch counts since the last read,
 * then resets; returns the number of classes. */
int bp_timing_enable(int on);
int bp_timing_read(double* ms, long long* counts, int n);

/* Replaces kernels.fused_span (kernels.py:458-735): implicit mover with
 * boundary folding, then deposition of the 10 moments at the new state. */
int bp_fused_span(int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us, void* vs,
                  void* ws, const void* qs, int64_t start, int64_t count, const void* E,
                  const void* B, int64_t* acc, const void* invvol, const double* geo_f,
                  const double* geo_g, const int64_t* geo_i, double dt, double dth,
                  double qdt2m, double beta, double one, int n_iters, double scale, int mixed,
                  int* d_status, void* stream);

/* Replaces kernels.push_span (kernels.py:82-307). */
int bp_push_span(int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us, void* vs,
                 void* ws, int64_t start, int64_t count, const void* E, const void* B,
                 const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                 double dth, double qdt2m, double beta, double one, int n_iters, int apply_bc,
                 int mixed, int* d_status, void* stream);

/* Replaces kernels.deposit_span (kernels.py:310-382). fbytes = invvol dtype. */
int bp_deposit_span(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs,
                    const void* us, const void* vs, const void* ws, const void* qs,
                    int64_t start, int64_t count, int64_t* acc, const void* invvol,
                    const double* geo_g, const int64_t* geo_i, double one, double scale,
                    int* d_status, void* stream);

/* Replaces kernels.gather_span (kernels.py:385-455); out is (count, 6) in the
 * particle dtype, rounded once. */
int bp_gather_span(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs,
                   int64_t start, int64_t count, const void* E, const void* B,
                   const double* geo_g, const int64_t* geo_i, double one, void* out,
                   int* d_status, void* stream);

/* As bp_fused_span / bp_push_span with an explicit arithmetic mode. */
int bp_fused_span_ex(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us,
                     void* vs, void* ws, const void* qs, int64_t start, int64_t count,
                     const void* E, const void* B, int64_t* acc, const void* invvol,
                     const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                     double dth, double qdt2m, double beta, double one, int n_iters,
                     double scale, int mixed, int* d_status, void* stream);

/* Per-cell field records of the fast kernels (csrc/bp_split.cu): for every
 * cell the trilinear coefficients of Ex Ey Ez Bx By Bz (48 values in the
 * particle precision).  The fused call builds them from E / B on its stream
 * unless the caller passes records built once per field update:
 * bp_field_records_bytes() gives the size of the (32-byte aligned) device
 * buffer for particles of pbytes, bp_field_records_build() fills it from E,
 * B, and bp_fused_span_rec() is bp_fused_span_ex() with a `records` argument
 * (NULL = build per call; ignored by the parity kernels).  The records must
 * describe the E, B passed to the call. */
int64_t bp_field_records_bytes(int pbytes, const int64_t* geo_i);
int bp_field_records_build(int pbytes, int fbytes, const void* E, const void* B,
                           const int64_t* geo_i, void* records, void* stream);
int bp_fused_span_rec(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us,
                      void* vs, void* ws, const void* qs, int64_t start, int64_t count,
                      const void* E, const void* B, int64_t* acc, const void* invvol,
                      const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                      double dth, double qdt2m, double beta, double one, int n_iters,
                      double scale, int mixed, const void* records, int* d_status,
                      void* stream);

/* Host-memory variant of bp_fused_span: particle arrays, E, B, acc and invvol
 * are HOST pointers (pinned or pageable).  The span is streamed through the
 * device in batches of at most batch_particles (0 = automatic) with
 * double-buffered H2D / kernel / D2H overlap; acc receives the exact integer
 * sum.  Synchronous; returns the worst status. */
int bp_fused_span_host(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs,
                       void* us, void* vs, void* ws, const void* qs, int64_t start,
                       int64_t count, const void* E, const void* B, int64_t* acc,
                       const void* invvol, const double* geo_f, const double* geo_g,
                       const int64_t* geo_i, double dt, double dth, double qdt2m, double beta,
                       double one, int n_iters, double scale, int mixed,
                       int64_t batch_particles);

/* Replaces particles.sort_by_cell (particles.py:157-167) on device: keys are
 * geometry.cell_index_of (geometry.py:152-159, f64 arithmetic, x fastest,
 * upper faces clamped); a stable sort; then x y z u v w q (pbytes each) and
 * ids (int64) are permuted in place.  Returns BP_ERR_DOMAIN if a position is
 * below the origin (reference: DomainError), leaving the buffer unchanged.
 * Synchronous on `stream`. */
int bp_sort_by_cell(int pbytes, void* xs, void* ys, void* zs, void* us, void* vs, void* ws,
                    void* qs, int64_t* ids, int64_t n, const double* origin,
                    const double* spacing, const int64_t* counts, void* stream);

/* Sorted copy: src[0..6] = x y z u v w q (q may be NULL), src_ids (may be
 * NULL) are read, their cell-sorted permutation (same order as
 * bp_sort_by_cell) is written to the distinct arrays dst / dst_ids — one
 * fused gather pass and no copy back, for callers that keep a spare buffer
 * set and swap.  On BP_ERR_DOMAIN, dst is unspecified and src untouched. */
int bp_sort_by_cell_into(int pbytes, void* const* src, int64_t* src_ids, void* const* dst,
                         int64_t* dst_ids, int64_t n, const double* origin,
                         const double* spacing, const int64_t* counts, void* stream);

/* Linear cell key per particle (geometry.cell_index_of) into keys[n] (device
 * int64).  Returns BP_ERR_DOMAIN on positions below the origin. */
int bp_cell_keys(int pbytes, const void* xs, const void* ys, const void* zs, int64_t n,
                 const double* origin, const double* spacing, const int64_t* counts,
                 int64_t* keys, void* stream);

/* Exact int64 sum over species of n-element grids (fields.total_moments,
 * fields.py:170-179): total[i] = sum_s accs[s][i].  Device pointers. */
int bp_moments_total(const int64_t* const* accs, int nspecies, int64_t n, int64_t* total,
                     void* stream);

/* Scalar implicit plasma response (maxwell.plasma_susceptibility,
 * maxwell.py:163-179), bitwise: chi[i] = (0.5 theta dt^2) *
 * max(0, sum_s (4 pi rho_s[i]) qom_s) with rho_s = acc_s * 2^-43 (rounded to
 * f32 and back when single != 0).  rho_rows[s] = row 0 of species s's
 * accumulator (device); qom is a host array. */
int bp_susceptibility(const int64_t* const* rho_rows, const double* qom, int nspecies,
                      int single, double theta, double dt, int64_t n, double* chi,
                      void* stream);

/* Exact merge of duplicated periodic node planes of a (rows, nx+1, ny+1,
 * nz+1) int64 grid (fields.fold_periodic, fields.py:28-47). */
int bp_fold_periodic_i64(int64_t* acc, int64_t rows, const int64_t* geo_i, void* stream);

/* ------------------------------------------------------------------------
 * Cell-binned layout (fast arithmetic; f32 particles with f32 or f64 fields,
 * or f64 particles with f64 fields) — the device-resident cycle path
 * (pipeline.DeviceSimulation layout "bins").  It replaces the
 * reference's phase 3 + phase 6 pair, run_cycle's per-batch fused_span calls
 * (pipeline.py:178-268, kernels.py:458-735) and the periodic stable cell sort
 * (pipeline.py:300-304, particles.py:157-167), for one species at a time:
 * the particles are records of 8 scalars of pbytes each (x y z u | v w q 0:
 * 32 bytes for f32, 64 for f64; 32-byte aligned; rec) with an int64 id
 * array; cell c owns slots [start[c],
 * start[c+1]), the first count[c] live; every bp_bins_cycle leaves each
 * particle in its cell's bin, so the order is cell-sorted every cycle.
 * Records, ids, start, count, the leaver / overflow lists, stat, field
 * records, acc, invvol: DEVICE pointers.
 *
 * bp_bins_plan   histogram of the flat arrays' cells (the fast kernels' cell
 *                formula in the particle precision) into count[ncell]; start[ncell + 1] = exclusive
 *                scan of count + max(slack_min, ceil(slack_frac * count));
 *                *total = start[ncell] (host int64; the call synchronises).
 *                Returns 3 (BP_ERR_DOMAIN) for positions below the origin.
 * bp_bins_fill   stable scatter of the flat arrays (x y z u v w q, ids) into
 *                the records dst_rec / dst_ids of start[ncell] slots
 *                (synchronises).
 * bp_bins_cycle  mover + leaver migration + 10-moment deposit of the bins
 *                into acc (+=); leavers / overflow / late are lists of
 *                bp_bins_leaver_bytes(pbytes) records (the leaver list is scratch
 *                of the call, the overflow list feeds the rebuild, the late
 *                list holds misplaced particles met by the deposit; it may alias the
 *                leaver list, which the migration has drained by then), with
 *                `records` = the per-cell records of bp_field_records_build
 *                in the particle precision (pbytes) — the f64 cycle is
 *                bitwise the flat f64 fast path's (particles and lattice);
 *                asynchronous; the worst
 *                particle status goes to *d_status (atomicMax).  stat[8]
 *                (uint64) counts leavers (0), overflowed leavers (1),
 *                misplaced particles (2) and lost particles (3): after the
 *                cycle, (1) or (2) non-zero asks for a rebuild (export +
 *                plan + fill: the overflow list is part of the export), (3)
 *                non-zero is fatal (overflow list too small).
 * bp_bins_reslack  the cheap rebuild after an overflow (no sort: the bins are
 *                in cell order): with dst == NULL, new_count = live +
 *                overflow arrivals per bin and new_start = the padded layout,
 *                *total = new_start[ncell] (synchronises); with dst, the
 *                bins and the overflow list are copied into dst_rec / dst_ids
 *                (new_count becomes the new live counts; synchronises).
 * bp_bins_export the live particles in cell order, then the overflow list,
 *                to the flat (reference SoA) arrays dst[7] / dst_ids
 *                (dst == NULL: count only; dst itself is a host table);
 *                offsets[ncell + 1] = exclusive scan of the clamped counts;
 *                *total = particles (synchronises).
 */
#define BP_BINS_STAT_LEAVERS 0
#define BP_BINS_STAT_OVERFLOW 1
#define BP_BINS_STAT_MISPLACED 2
#define BP_BINS_STAT_LOST 3
int bp_bins_leaver_bytes(int pbytes);
int bp_bins_plan(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs, int64_t n,
                 const double* geo_f, const double* geo_g, const int64_t* geo_i,
                 double slack_frac, int slack_min, int32_t* count, int64_t* start,
                 int64_t* total, void* stream);
int bp_bins_fill(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs, const void* us,
                 const void* vs, const void* ws, const void* qs, const int64_t* ids, int64_t n,
                 const double* geo_f, const double* geo_g, const int64_t* geo_i,
                 const int64_t* start, void* dst_rec, int64_t* dst_ids, void* stream);
int bp_bins_cycle(int pbytes, int fbytes, void* rec, int64_t* ids, const int64_t* start, int32_t* count,
                  int64_t ncell,
                  void* leavers, int64_t leaver_cap, void* overflow, int64_t overflow_cap,
                  void* late, int64_t late_cap, uint64_t* stat, const void* records,
                  int64_t* acc, const void* invvol,
                  const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                  double dth, double qdt2m, double beta, double one, int n_iters, double scale,
                  int* d_status, void* stream);
int bp_bins_reslack(int pbytes, const void* rec, int64_t* ids, const int64_t* start, int32_t* count,
                    int64_t ncell, const void* overflow, int64_t overflow_cap, uint64_t* stat,
                    double slack_frac, int slack_min, int32_t* new_count, int64_t* new_start,
                    void* dst_rec, int64_t* dst_ids, int64_t* total, void* stream);
int bp_bins_export(int pbytes, const void* rec, int64_t* ids, const int64_t* start, int32_t* count,
                   int64_t ncell, const void* overflow, int64_t overflow_cap, uint64_t* stat,
                   int64_t* offsets, void* const* dst, int64_t* dst_ids, int64_t* total,
                   void* stream);

/* ------------------------------------------------------------------------
 * Bit-exact device loader: one species of the reference's init_maxwellian
 * (pkg/src/batchpic/particles.py:177-241, _species_rng :173-175) generated in
 * HBM for the cells [c0, c0 + nc) (x fastest, ppc particles each: the rank's
 * shard).  Positions o + d (cell index) + d U and velocities drift + vth N
 * with U / N numpy's Generator(Philox(key=[seed, species_id])).random /
 * .standard_normal draws (jitter (3, n_p) first, normals (3, n_p) next),
 * cast to the particle dtype (pbytes); q = q_cell[cell - c0] (the caller's
 * species.charge * density(cell centre) * cell volume / ppc); ids = the
 * global particle index.  All outputs, q_cell, tail_k / tail_u: DEVICE;
 * geo_i, origin[3], spacing[3], drift[3], vth[3], n_tail: host.  Normals of
 * the ziggurat's tail strip (~0.03%) are bit-exact only with the host libm's
 * log1p: each is listed as tail_k = 2 * ordinal + sign, tail_u = its
 * uniform, and the caller finishes it as +-(r - log1p(-u) / r)
 * (numpy random_standard_normal; paper_2008_04397_b200/gem.py does).
 * Synchronises; *n_tail = listed tail normals (> tail_cap: error).
 */
int bp_init_maxwellian(int pbytes, uint64_t seed, uint64_t species_id, const int64_t* geo_i,
                       const double* origin, const double* spacing, int ppc,
                       const double* drift, const double* vth, const double* q_cell,
                       int64_t c0, int64_t nc, void* xs, void* ys, void* zs, void* us,
                       void* vs, void* ws, void* qs, int64_t* ids, int64_t* tail_k,
                       double* tail_u, int64_t tail_cap, int64_t* n_tail, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BP_B200_H */
