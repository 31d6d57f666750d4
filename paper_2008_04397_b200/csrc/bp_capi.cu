// C ABI (include/bp_b200.h): argument checking, status handling, and the
// host-memory streaming pipeline.  Kernels live in bp_parity.cu (bitwise
// reference arithmetic) and bp_fast.cu (FMA / native f32 arithmetic).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/bp_b200.h"
#include "bp_launch.h"

namespace bp {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Optional device timing per kernel class (bp_timing_enable / bp_timing_read):
// an event pair on the launching stream around each launch, resolved when
// the caller reads the totals.
namespace {
struct TimedSpan {
  int cls;
  cudaEvent_t a, b;
};
std::mutex g_tmu;
std::atomic<bool> g_timing{false};
std::vector<TimedSpan> g_spans;
std::vector<cudaEvent_t> g_free_events;
double g_tms[TK_COUNT] = {};
long long g_tcnt[TK_COUNT] = {};

cudaEvent_t take_event() {
  if (!g_free_events.empty()) {
    cudaEvent_t e = g_free_events.back();
    g_free_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

int timing_begin(int cls, cudaStream_t s) {
  if (!g_timing.load(std::memory_order_relaxed)) return -1;
  std::lock_guard<std::mutex> lock(g_tmu);
  TimedSpan t{cls, take_event(), take_event()};
  cudaEventRecord(t.a, s);
  g_spans.push_back(t);
  return (int)g_spans.size() - 1;
}

void timing_end(int idx, cudaStream_t s) {
  if (idx < 0) return;
  std::lock_guard<std::mutex> lock(g_tmu);
  if (idx < (int)g_spans.size()) cudaEventRecord(g_spans[idx].b, s);
}

// Scratch (node records, sort buffers) comes from the device's default
// stream-ordered pool; keep its memory mapped between calls instead of
// returning it to the driver at every synchronisation (release threshold 0
// by default), which otherwise costs a re-map of hundreds of MB per call.
void ensure_pool() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long keep = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cell_keys(int pbytes, const void* xs, const void* ys, const void* zs, int64_t n,
              const double* origin, const double* spacing, const int64_t* counts,
              int64_t* keys, cudaStream_t s);
int sort_by_cell(int pbytes, void* xs, void* ys, void* zs, void* us, void* vs, void* ws,
                 void* qs, int64_t* ids, int64_t n, const double* origin,
                 const double* spacing, const int64_t* counts, cudaStream_t s);
int fold_periodic_i64(int64_t* acc, int64_t rows, const int64_t* geo_i, cudaStream_t s);
int sort_by_cell_into(int pbytes, void* const* src, int64_t* src_ids, void* const* dst,
                      int64_t* dst_ids, int64_t n, const double* origin, const double* spacing,
                      const int64_t* counts, cudaStream_t s);
int moments_total(const long long* const* rows, int ns, int64_t n, long long* total,
                  cudaStream_t st);
int susceptibility(const long long* const* rho_rows, const double* qom, int ns, int single,
                   double factor, int64_t n, double* chi, cudaStream_t st);

namespace {

int cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return BP_ECUDA;
  }
  return BP_OK;
}

bool valid_pair(int pb, int fb) {
  return (pb == 8 && fb == 8) || (pb == 4 && fb == 4) || (pb == 4 && fb == 8);
}

int check_geo(const double* geo_g, const int64_t* geo_i) {
  if (!geo_g || !geo_i) {
    set_error("geometry arrays are required");
    return BP_EINVAL;
  }
  for (int a = 0; a < 3; ++a) {
    if (geo_i[a] < 1) {
      set_error("cell counts must be >= 1");
      return BP_EINVAL;
    }
    if (geo_i[3 + a] != 0 && geo_i[3 + a] != 1) {
      set_error("boundary codes must be 0 (periodic) or 1 (reflecting)");
      return BP_EINVAL;
    }
    if (!(geo_g[a] > 0.0)) {
      set_error("grid spacings must be positive");
      return BP_EINVAL;
    }
  }
  const int64_t nn = (geo_i[0] + 1) * (geo_i[1] + 1) * (geo_i[2] + 1);
  if (nn * 10 >= (int64_t)1 << 31) {
    set_error("grid of %lld nodes exceeds the 32-bit node index space", (long long)nn);
    return BP_EINVAL;
  }
  return BP_OK;
}

// Per-thread status slot for the synchronous (d_status == NULL) form.
struct StatusSlot {
  int* d = nullptr;
  int* h = nullptr;
  int dev = -1;
};
static thread_local StatusSlot g_slot;

int* sync_slot(cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_slot.d == nullptr || g_slot.dev != dev) {
    if (cudaMalloc((void**)&g_slot.d, sizeof(int)) != cudaSuccess) return nullptr;
    if (cudaMallocHost((void**)&g_slot.h, sizeof(int)) != cudaSuccess) return nullptr;
    g_slot.dev = dev;
  }
  cudaMemsetAsync(g_slot.d, 0, sizeof(int), s);
  return g_slot.d;
}

int finish(int rc, bool sync, cudaStream_t s) {
  if (rc != BP_OK || !sync) return rc;
  rc = cuda_check(cudaMemcpyAsync(g_slot.h, g_slot.d, sizeof(int), cudaMemcpyDeviceToHost, s),
                  "status copy");
  if (rc) return rc;
  rc = cuda_check(cudaStreamSynchronize(s), "kernel execution");
  if (rc) return rc;
  return *g_slot.h;
}

int run(Call& c, int arith, int* d_status, cudaStream_t s) {
  if (c.count < 0 || c.start < 0) {
    set_error("negative span (%lld, %lld)", (long long)c.start, (long long)c.count);
    return BP_EINVAL;
  }
  const bool sync = d_status == nullptr;
  if (c.count == 0) return BP_OK;
  ensure_pool();
  c.status = sync ? sync_slot(s) : d_status;
  if (!c.status) {
    set_error("status slot allocation failed");
    return BP_ECUDA;
  }
  int rc;
  if (arith == BP_ARITH_PARITY) rc = launch_parity(c, s);
  else if (arith == BP_ARITH_FAST) rc = launch_fast(c, s);
  else {
    set_error("unknown arithmetic mode %d", arith);
    rc = BP_EINVAL;
  }
  return finish(rc, sync, s);
}

void fill_geo(Call& c, const double* geo_f, const double* geo_g, const int64_t* geo_i) {
  for (int k = 0; k < 9; ++k) {
    c.geo_f[k] = geo_f ? geo_f[k] : 0.0;
    c.geo_g[k] = geo_g[k];
  }
  for (int k = 0; k < 6; ++k) c.geo_i[k] = geo_i[k];
}

int fused_call(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us,
               void* vs, void* ws, const void* qs, int64_t start, int64_t count, const void* E,
               const void* B, int64_t* acc, const void* invvol, const double* geo_f,
               const double* geo_g, const int64_t* geo_i, double dt, double dth, double qdt2m,
               double beta, double one, int n_iters, double scale, int mixed, int* d_status,
               cudaStream_t s, const void* records = nullptr) {
  if (!valid_pair(pbytes, fbytes)) {
    set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", pbytes, fbytes);
    return BP_EINVAL;
  }
  int rc = check_geo(geo_g, geo_i);
  if (rc) return rc;
  if (!geo_f || n_iters < 0) {
    set_error("geo_f required and n_iters >= 0");
    return BP_EINVAL;
  }
  Call c{};
  c.op = OP_FUSED;
  c.pbytes = pbytes; c.fbytes = fbytes;
  c.x = xs; c.y = ys; c.z = zs; c.u = us; c.v = vs; c.w = ws; c.q = qs;
  c.start = start; c.count = count;
  c.E = E; c.B = B; c.acc = acc; c.invvol = invvol;
  fill_geo(c, geo_f, geo_g, geo_i);
  c.dt = dt; c.dth = dth; c.qdt2m = qdt2m; c.beta = beta; c.one = one; c.scale = scale;
  c.n_iters = n_iters; c.mixed = mixed; c.apply_bc = 1;
  c.records = records;
  return run(c, arith, d_status, s);
}

// ---------------------------------------------------------------------------
// Host-memory streaming pipeline (bp_fused_span_host).
constexpr int kSlots = 3;  // batches in flight: H2D of one, kernels, D2H of another

struct HostCtx {
  int dev = -1;
  cudaStream_t st[kSlots] = {};
  cudaEvent_t ready[kSlots];
  void* slot[kSlots][7] = {};
  size_t slot_bytes = 0;
  void* rec = nullptr;  // f32 cell records, built once per call
  size_t rec_bytes = 0;
  void* dE = nullptr;
  void* dB = nullptr;
  void* dinv = nullptr;
  int64_t* dacc = nullptr;
  size_t field_bytes = 0, acc_bytes = 0;
  int* dstatus = nullptr;
  int* hstatus = nullptr;
};
// One pipeline (streams, slots, field and accumulator buffers) per concurrent
// call: the reference calls fused_span concurrently from a thread pool on
// disjoint spans with private accumulators (pipeline.py:164-165, 255-257), and
// those calls then overlap on the device — one call's pipeline fill and drain
// under another's steady state.  A call borrows a free pipeline (or makes
// one) and returns it; pipelines live for the process, like the runtime's
// own pools, so no CUDA call runs at thread or process exit.
static std::mutex g_host_mu;
static std::vector<HostCtx*> g_host_free;
struct HostLease {
  HostCtx* h;
  HostLease() {
    std::lock_guard<std::mutex> lock(g_host_mu);
    if (g_host_free.empty()) {
      h = new HostCtx();
    } else {
      h = g_host_free.back();
      g_host_free.pop_back();
    }
  }
  ~HostLease() {
    std::lock_guard<std::mutex> lock(g_host_mu);
    g_host_free.push_back(h);
  }
};

int host_ctx_reserve(HostCtx& h, size_t slot_bytes, size_t field_bytes, size_t acc_bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (h.dev != dev) {
    h = HostCtx();
    h.dev = dev;
    for (int k = 0; k < kSlots; ++k) {
      if (cudaStreamCreateWithFlags(&h.st[k], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&h.ready[k], cudaEventDisableTiming) != cudaSuccess)
        return cuda_check(cudaGetLastError(), "stream create");
    }
    if (cudaMalloc((void**)&h.dstatus, sizeof(int)) != cudaSuccess ||
        cudaMallocHost((void**)&h.hstatus, sizeof(int)) != cudaSuccess)
      return cuda_check(cudaGetLastError(), "status alloc");
  }
  if (slot_bytes > h.slot_bytes) {
    for (int k = 0; k < kSlots; ++k)
      for (int a = 0; a < 7; ++a) {
        if (h.slot[k][a]) cudaFree(h.slot[k][a]);
        if (cudaMalloc(&h.slot[k][a], slot_bytes) != cudaSuccess)
          return cuda_check(cudaGetLastError(), "slot alloc");
      }
    h.slot_bytes = slot_bytes;
  }
  if (field_bytes > h.field_bytes) {
    if (h.dE) { cudaFree(h.dE); cudaFree(h.dB); cudaFree(h.dinv); }
    if (cudaMalloc(&h.dE, field_bytes) != cudaSuccess || cudaMalloc(&h.dB, field_bytes) != cudaSuccess ||
        cudaMalloc(&h.dinv, field_bytes / 3 + 64) != cudaSuccess)
      return cuda_check(cudaGetLastError(), "field alloc");
    h.field_bytes = field_bytes;
  }
  if (acc_bytes > h.acc_bytes) {
    if (h.dacc) cudaFree(h.dacc);
    if (cudaMalloc((void**)&h.dacc, acc_bytes) != cudaSuccess)
      return cuda_check(cudaGetLastError(), "acc alloc");
    h.acc_bytes = acc_bytes;
  }
  return BP_OK;
}

}  // namespace
}  // namespace bp

using namespace bp;

extern "C" {

int bp_version(void) { return 100; }

int bp_timing_enable(int on) {
  std::lock_guard<std::mutex> lock(g_tmu);
  g_timing.store(on != 0);
  return BP_OK;
}

int bp_timing_read(double* ms, long long* counts, int n) {
  std::lock_guard<std::mutex> lock(g_tmu);
  for (auto& t : g_spans) {
    float v = 0.f;
    if (cudaEventSynchronize(t.b) == cudaSuccess && cudaEventElapsedTime(&v, t.a, t.b) == cudaSuccess) {
      g_tms[t.cls] += v;
      g_tcnt[t.cls] += 1;
    }
    g_free_events.push_back(t.a);
    g_free_events.push_back(t.b);
  }
  g_spans.clear();
  for (int k = 0; k < n && k < TK_COUNT; ++k) {
    if (ms) ms[k] = g_tms[k];
    if (counts) counts[k] = g_tcnt[k];
  }
  for (int k = 0; k < TK_COUNT; ++k) {
    g_tms[k] = 0.0;
    g_tcnt[k] = 0;
  }
  return TK_COUNT;
}

long long bp_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* bp_last_error(void) { return g_err; }

int bp_fused_span(int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us, void* vs,
                  void* ws, const void* qs, int64_t start, int64_t count, const void* E,
                  const void* B, int64_t* acc, const void* invvol, const double* geo_f,
                  const double* geo_g, const int64_t* geo_i, double dt, double dth,
                  double qdt2m, double beta, double one, int n_iters, double scale, int mixed,
                  int* d_status, void* stream) {
  return fused_call(BP_ARITH_PARITY, pbytes, fbytes, xs, ys, zs, us, vs, ws, qs, start, count,
                    E, B, acc, invvol, geo_f, geo_g, geo_i, dt, dth, qdt2m, beta, one, n_iters,
                    scale, mixed, d_status, (cudaStream_t)stream);
}

int bp_fused_span_ex(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us,
                     void* vs, void* ws, const void* qs, int64_t start, int64_t count,
                     const void* E, const void* B, int64_t* acc, const void* invvol,
                     const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                     double dth, double qdt2m, double beta, double one, int n_iters,
                     double scale, int mixed, int* d_status, void* stream) {
  return fused_call(arith, pbytes, fbytes, xs, ys, zs, us, vs, ws, qs, start, count, E, B, acc,
                    invvol, geo_f, geo_g, geo_i, dt, dth, qdt2m, beta, one, n_iters, scale,
                    mixed, d_status, (cudaStream_t)stream);
}

int64_t bp_field_records_bytes(int pbytes, const int64_t* geo_i) {
  if (pbytes != 4 && pbytes != 8) {
    set_error("particle dtype must be 4 or 8 bytes");
    return BP_EINVAL;
  }
  if (!geo_i || geo_i[0] < 1 || geo_i[1] < 1 || geo_i[2] < 1) {
    set_error("cell counts must be >= 1");
    return BP_EINVAL;
  }
  return (int64_t)split_records_bytes(pbytes, geo_i);
}

int bp_field_records_build(int pbytes, int fbytes, const void* E, const void* B,
                           const int64_t* geo_i, void* records, void* stream) {
  if (!valid_pair(pbytes, fbytes)) {
    set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", pbytes, fbytes);
    return BP_EINVAL;
  }
  if (!E || !B || !records || !geo_i) {
    set_error("E, B, geo_i and records are required");
    return BP_EINVAL;
  }
  if (geo_i[0] < 1 || geo_i[1] < 1 || geo_i[2] < 1) {
    set_error("cell counts must be >= 1");
    return BP_EINVAL;
  }
  if (((uintptr_t)records % 32) != 0) {
    set_error("records must be 32-byte aligned");
    return BP_EINVAL;
  }
  return split_pack_records(pbytes, fbytes, E, B, geo_i, records, (cudaStream_t)stream)
             ? BP_ECUDA
             : BP_OK;
}

int bp_fused_span_rec(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us,
                      void* vs, void* ws, const void* qs, int64_t start, int64_t count,
                      const void* E, const void* B, int64_t* acc, const void* invvol,
                      const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                      double dth, double qdt2m, double beta, double one, int n_iters,
                      double scale, int mixed, const void* records, int* d_status,
                      void* stream) {
  if (records && ((uintptr_t)records % 32) != 0) {
    set_error("records must be 32-byte aligned");
    return BP_EINVAL;
  }
  return fused_call(arith, pbytes, fbytes, xs, ys, zs, us, vs, ws, qs, start, count, E, B, acc,
                    invvol, geo_f, geo_g, geo_i, dt, dth, qdt2m, beta, one, n_iters, scale,
                    mixed, d_status, (cudaStream_t)stream, records);
}

int bp_push_span(int pbytes, int fbytes, void* xs, void* ys, void* zs, void* us, void* vs,
                 void* ws, int64_t start, int64_t count, const void* E, const void* B,
                 const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                 double dth, double qdt2m, double beta, double one, int n_iters, int apply_bc,
                 int mixed, int* d_status, void* stream) {
  if (!valid_pair(pbytes, fbytes)) {
    set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", pbytes, fbytes);
    return BP_EINVAL;
  }
  int rc = check_geo(geo_g, geo_i);
  if (rc) return rc;
  if (!geo_f) {
    set_error("geo_f required");
    return BP_EINVAL;
  }
  Call c{};
  c.op = OP_PUSH;
  c.pbytes = pbytes; c.fbytes = fbytes;
  c.x = xs; c.y = ys; c.z = zs; c.u = us; c.v = vs; c.w = ws;
  c.start = start; c.count = count;
  c.E = E; c.B = B;
  fill_geo(c, geo_f, geo_g, geo_i);
  c.dt = dt; c.dth = dth; c.qdt2m = qdt2m; c.beta = beta; c.one = one;
  c.n_iters = n_iters; c.mixed = mixed; c.apply_bc = apply_bc ? 1 : 0;
  return run(c, BP_ARITH_PARITY, d_status, (cudaStream_t)stream);
}

int bp_deposit_span(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs,
                    const void* us, const void* vs, const void* ws, const void* qs,
                    int64_t start, int64_t count, int64_t* acc, const void* invvol,
                    const double* geo_g, const int64_t* geo_i, double one, double scale,
                    int* d_status, void* stream) {
  if (!valid_pair(pbytes, fbytes)) {
    set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", pbytes, fbytes);
    return BP_EINVAL;
  }
  int rc = check_geo(geo_g, geo_i);
  if (rc) return rc;
  Call c{};
  c.op = OP_DEPOSIT;
  c.pbytes = pbytes; c.fbytes = fbytes;
  c.x = (void*)xs; c.y = (void*)ys; c.z = (void*)zs;
  c.u = (void*)us; c.v = (void*)vs; c.w = (void*)ws; c.q = qs;
  c.start = start; c.count = count;
  c.acc = acc; c.invvol = invvol;
  fill_geo(c, nullptr, geo_g, geo_i);
  c.one = one; c.scale = scale;
  return run(c, BP_ARITH_PARITY, d_status, (cudaStream_t)stream);
}

int bp_gather_span(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs,
                   int64_t start, int64_t count, const void* E, const void* B,
                   const double* geo_g, const int64_t* geo_i, double one, void* out,
                   int* d_status, void* stream) {
  if (!valid_pair(pbytes, fbytes)) {
    set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", pbytes, fbytes);
    return BP_EINVAL;
  }
  int rc = check_geo(geo_g, geo_i);
  if (rc) return rc;
  Call c{};
  c.op = OP_GATHER;
  c.pbytes = pbytes; c.fbytes = fbytes;
  c.x = (void*)xs; c.y = (void*)ys; c.z = (void*)zs;
  c.start = start; c.count = count;
  c.E = E; c.B = B; c.out = out;
  fill_geo(c, nullptr, geo_g, geo_i);
  c.one = one;
  return run(c, BP_ARITH_PARITY, d_status, (cudaStream_t)stream);
}

int bp_fused_span_host(int arith, int pbytes, int fbytes, void* xs, void* ys, void* zs,
                       void* us, void* vs, void* ws, const void* qs, int64_t start,
                       int64_t count, const void* E, const void* B, int64_t* acc,
                       const void* invvol, const double* geo_f, const double* geo_g,
                       const int64_t* geo_i, double dt, double dth, double qdt2m, double beta,
                       double one, int n_iters, double scale, int mixed,
                       int64_t batch_particles) {
  if (!valid_pair(pbytes, fbytes)) {
    set_error("unsupported dtype pair (particles %d bytes, fields %d bytes)", pbytes, fbytes);
    return BP_EINVAL;
  }
  int rc = check_geo(geo_g, geo_i);
  if (rc) return rc;
  if (count < 0 || start < 0) {
    set_error("negative span");
    return BP_EINVAL;
  }
  if (count == 0) return BP_OK;
  HostLease lease;
  HostCtx& h = *lease.h;
  const int64_t nn = (geo_i[0] + 1) * (geo_i[1] + 1) * (geo_i[2] + 1);
  int64_t batch = batch_particles > 0 ? batch_particles : ((int64_t)1 << 21);
  if (batch > count) batch = count;
  rc = host_ctx_reserve(h, (size_t)batch * pbytes, (size_t)3 * nn * fbytes,
                        (size_t)10 * nn * sizeof(int64_t));
  if (rc) return rc;
  cudaStream_t s0 = h.st[0];
  // fields, invvol and the caller's accumulator go up once
  rc |= cuda_check(cudaMemcpyAsync(h.dE, E, 3 * nn * fbytes, cudaMemcpyHostToDevice, s0), "E h2d");
  rc |= cuda_check(cudaMemcpyAsync(h.dB, B, 3 * nn * fbytes, cudaMemcpyHostToDevice, s0), "B h2d");
  rc |= cuda_check(cudaMemcpyAsync(h.dinv, invvol, nn * fbytes, cudaMemcpyHostToDevice, s0), "invvol h2d");
  rc |= cuda_check(cudaMemcpyAsync(h.dacc, acc, 10 * nn * 8, cudaMemcpyHostToDevice, s0), "acc h2d");
  rc |= cuda_check(cudaMemsetAsync(h.dstatus, 0, sizeof(int), s0), "status");
  // fast path (f32, or f64 with f64 fields): the cell records of E/B once
  // for all batches
  const bool f32rec = arith == BP_ARITH_FAST && (pbytes == 4 || fbytes == 8);
  if (f32rec && !rc) {
    const size_t rb = split_records_bytes(pbytes, geo_i) + 256;
    if (rb > h.rec_bytes) {
      if (h.rec) cudaFree(h.rec);
      h.rec = nullptr;
      h.rec_bytes = 0;
      rc = cuda_check(cudaMalloc(&h.rec, rb), "records alloc");
      if (!rc) h.rec_bytes = rb;
    }
    if (!rc) rc = split_pack_records(pbytes, fbytes, h.dE, h.dB, geo_i, h.rec, s0) ? BP_ECUDA : BP_OK;
  }
  rc |= cuda_check(cudaEventRecord(h.ready[0], s0), "event");
  if (rc) return rc < 0 ? rc : BP_ECUDA;
  for (int k = 1; k < kSlots; ++k)
    rc |= cuda_check(cudaStreamWaitEvent(h.st[k], h.ready[0], 0), "wait");
  char* host[7] = {(char*)xs, (char*)ys, (char*)zs, (char*)us, (char*)vs, (char*)ws, (char*)qs};
  int64_t b = 0;
  for (int64_t off = 0; off < count && !rc; off += batch, ++b) {
    const int k = (int)(b % kSlots);
    cudaStream_t s = h.st[k];
    const int64_t n = (count - off < batch) ? count - off : batch;
    const size_t bytes = (size_t)n * pbytes;
    const size_t hoff = (size_t)(start + off) * pbytes;
    for (int a = 0; a < 7 && !rc; ++a)
      rc = cuda_check(cudaMemcpyAsync(h.slot[k][a], host[a] + hoff, bytes,
                                      cudaMemcpyHostToDevice, s), "batch h2d");
    if (rc) break;
    Call c{};
    c.op = OP_FUSED;
    c.pbytes = pbytes; c.fbytes = fbytes;
    c.x = h.slot[k][0]; c.y = h.slot[k][1]; c.z = h.slot[k][2];
    c.u = h.slot[k][3]; c.v = h.slot[k][4]; c.w = h.slot[k][5]; c.q = h.slot[k][6];
    c.start = 0; c.count = n;
    c.E = h.dE; c.B = h.dB; c.acc = h.dacc; c.invvol = h.dinv;
    fill_geo(c, geo_f, geo_g, geo_i);
    c.dt = dt; c.dth = dth; c.qdt2m = qdt2m; c.beta = beta; c.one = one; c.scale = scale;
    c.n_iters = n_iters; c.mixed = mixed; c.apply_bc = 1;
    c.status = h.dstatus;
    c.records = f32rec ? h.rec : nullptr;
    rc = arith == BP_ARITH_FAST ? launch_fast(c, s) : launch_parity(c, s);
    if (rc) break;
    for (int a = 0; a < 6 && !rc; ++a)
      rc = cuda_check(cudaMemcpyAsync(host[a] + hoff, h.slot[k][a], bytes,
                                      cudaMemcpyDeviceToHost, s), "batch d2h");
  }
  // join the streams, bring the accumulator and status back
  for (int k = 1; k < kSlots; ++k) {
    cudaEventRecord(h.ready[k], h.st[k]);
    cudaStreamWaitEvent(s0, h.ready[k], 0);
  }
  if (!rc) rc = cuda_check(cudaMemcpyAsync(acc, h.dacc, 10 * nn * 8, cudaMemcpyDeviceToHost, s0), "acc d2h");
  if (!rc) rc = cuda_check(cudaMemcpyAsync(h.hstatus, h.dstatus, sizeof(int), cudaMemcpyDeviceToHost, s0), "status d2h");
  int rc2 = cuda_check(cudaStreamSynchronize(s0), "pipeline");
  if (rc) return rc;
  if (rc2) return rc2;
  return *h.hstatus;
}

int bp_sort_by_cell(int pbytes, void* xs, void* ys, void* zs, void* us, void* vs, void* ws,
                    void* qs, int64_t* ids, int64_t n, const double* origin,
                    const double* spacing, const int64_t* counts, void* stream) {
  if (pbytes != 4 && pbytes != 8) {
    set_error("unsupported particle dtype (%d bytes)", pbytes);
    return BP_EINVAL;
  }
  ensure_pool();
  return sort_by_cell(pbytes, xs, ys, zs, us, vs, ws, qs, ids, n, origin, spacing, counts,
                      (cudaStream_t)stream);
}

int bp_sort_by_cell_into(int pbytes, void* const* src, int64_t* src_ids, void* const* dst,
                         int64_t* dst_ids, int64_t n, const double* origin,
                         const double* spacing, const int64_t* counts, void* stream) {
  if (pbytes != 4 && pbytes != 8) {
    set_error("unsupported particle dtype (%d bytes)", pbytes);
    return BP_EINVAL;
  }
  if (!src || !dst) {
    set_error("src and dst arrays are required");
    return BP_EINVAL;
  }
  for (int k = 0; k < 7; ++k) {
    // x..w are required, q (k = 6) is optional but must then be given on both sides
    if (k < 6 && (!src[k] || !dst[k])) {
      set_error("sort_by_cell_into needs x, y, z, u, v, w on both sides");
      return BP_EINVAL;
    }
    if ((src[k] == nullptr) != (dst[k] == nullptr) || (src[k] && src[k] == dst[k])) {
      set_error("sort_by_cell_into needs distinct source and destination arrays");
      return BP_EINVAL;
    }
  }
  if ((src_ids == nullptr) != (dst_ids == nullptr) || (src_ids && src_ids == dst_ids)) {
    set_error("sort_by_cell_into needs distinct source and destination id arrays");
    return BP_EINVAL;
  }
  ensure_pool();
  return sort_by_cell_into(pbytes, src, src_ids, dst, dst_ids, n, origin, spacing, counts,
                           (cudaStream_t)stream);
}

int bp_cell_keys(int pbytes, const void* xs, const void* ys, const void* zs, int64_t n,
                 const double* origin, const double* spacing, const int64_t* counts,
                 int64_t* keys, void* stream) {
  ensure_pool();
  return cell_keys(pbytes, xs, ys, zs, n, origin, spacing, counts, keys, (cudaStream_t)stream);
}

int bp_moments_total(const int64_t* const* accs, int nspecies, int64_t n, int64_t* total,
                     void* stream) {
  if (!accs || !total || n < 0) {
    set_error("bp_moments_total: null arrays or negative size");
    return BP_EINVAL;
  }
  if (n == 0) return BP_OK;
  return moments_total(reinterpret_cast<const long long* const*>(accs), nspecies, n,
                       reinterpret_cast<long long*>(total), (cudaStream_t)stream);
}

int bp_susceptibility(const int64_t* const* rho_rows, const double* qom, int nspecies,
                      int single, double theta, double dt, int64_t n, double* chi,
                      void* stream) {
  if (!rho_rows || !qom || !chi || n < 0) {
    set_error("bp_susceptibility: null arrays or negative size");
    return BP_EINVAL;
  }
  if (n == 0) return BP_OK;
  const double factor = 0.5 * theta * dt * dt;  // maxwell.py:178, left to right
  return susceptibility(reinterpret_cast<const long long* const*>(rho_rows), qom, nspecies,
                        single, factor, n, chi, (cudaStream_t)stream);
}

int bp_fold_periodic_i64(int64_t* acc, int64_t rows, const int64_t* geo_i, void* stream) {
  return fold_periodic_i64(acc, rows, geo_i, (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Cell-binned fast path (bp_bins.cu f32, bp_bins64.cu f64)
namespace {
int bins_call(Call& c, int pbytes, int fbytes, const void* xs, const void* ys, const void* zs,
              const void* us, const void* vs, const void* ws, const void* qs, int64_t start,
              int64_t count, const double* geo_f, const double* geo_g, const int64_t* geo_i) {
  // f32 particles with f32 or f64 fields; f64 particles with f64 fields
  if (!((pbytes == 4 && (fbytes == 4 || fbytes == 8)) || (pbytes == 8 && fbytes == 8))) {
    set_error("unsupported dtype pair for the binned layout (particles %d, fields %d bytes)",
              pbytes, fbytes);
    return BP_EINVAL;
  }
  int rc = check_geo(geo_g, geo_i);
  if (rc) return rc;
  if (!geo_f) {
    set_error("geo_f required");
    return BP_EINVAL;
  }
  c.op = OP_FUSED;
  c.pbytes = pbytes; c.fbytes = fbytes;
  c.x = const_cast<void*>(xs); c.y = const_cast<void*>(ys); c.z = const_cast<void*>(zs);
  c.u = const_cast<void*>(us); c.v = const_cast<void*>(vs); c.w = const_cast<void*>(ws);
  c.q = qs;
  c.start = start; c.count = count;
  fill_geo(c, geo_f, geo_g, geo_i);
  ensure_pool();
  return BP_OK;
}
}  // namespace

int bp_bins_leaver_bytes(int pbytes) {
  if (pbytes != 4 && pbytes != 8) {
    set_error("particle dtype must be 4 or 8 bytes");
    return BP_EINVAL;
  }
  return bp::bins_leaver_bytes(pbytes);
}

int bp_bins_plan(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs, int64_t n,
                 const double* geo_f, const double* geo_g, const int64_t* geo_i,
                 double slack_frac, int slack_min, int32_t* count, int64_t* start,
                 int64_t* total, void* stream) {
  Call c{};
  int rc = bins_call(c, pbytes, fbytes, xs, ys, zs, nullptr, nullptr, nullptr, nullptr, 0, n, geo_f,
                     geo_g, geo_i);
  if (rc) return rc;
  if (!count || !start || !total || n < 0 || slack_frac < 0 || slack_min < 0) {
    set_error("bins_plan: bad arguments");
    return BP_EINVAL;
  }
  return bins_plan(c, count, start, slack_frac, slack_min, total, (cudaStream_t)stream);
}

int bp_bins_fill(int pbytes, int fbytes, const void* xs, const void* ys, const void* zs, const void* us,
                 const void* vs, const void* ws, const void* qs, const int64_t* ids, int64_t n,
                 const double* geo_f, const double* geo_g, const int64_t* geo_i,
                 const int64_t* start, void* dst_rec, int64_t* dst_ids, void* stream) {
  Call c{};
  int rc = bins_call(c, pbytes, fbytes, xs, ys, zs, us, vs, ws, qs, 0, n, geo_f, geo_g, geo_i);
  if (rc) return rc;
  if (!ids || !start || !dst_rec || ((uintptr_t)dst_rec % 16) != 0 || !dst_ids || !us || !vs ||
      !ws || !qs) {
    set_error("bins_fill: bad arguments (16-byte aligned records)");
    return BP_EINVAL;
  }
  return bins_fill(c, ids, start, dst_rec, dst_ids, (cudaStream_t)stream);
}

int bp_bins_cycle(int pbytes, int fbytes, void* rec, int64_t* ids, const int64_t* start, int32_t* count,
                  int64_t ncell,
                  void* leavers, int64_t leaver_cap, void* overflow, int64_t overflow_cap,
                  void* late, int64_t late_cap, uint64_t* stat, const void* records,
                  int64_t* acc, const void* invvol,
                  const double* geo_f, const double* geo_g, const int64_t* geo_i, double dt,
                  double dth, double qdt2m, double beta, double one, int n_iters, double scale,
                  int* d_status, void* stream) {
  Call c{};
  int rc = bins_call(c, pbytes, fbytes, rec, rec, rec, rec, rec, rec, rec, 0, 0, geo_f, geo_g,
                     geo_i);
  if (rc) return rc;
  // 256-bit record accesses: 32-byte aligned slots
  if (!rec || ((uintptr_t)rec % 32) != 0 || !records || ((uintptr_t)records % 32) != 0 ||
      !acc || !invvol || !ids || !start ||
      !count || !stat || !leavers || !overflow || !late || leaver_cap < 0 ||
      leaver_cap > 0x7fffff00LL ||
      overflow_cap < 0 || late_cap < 0 ||
      n_iters < 0 || !d_status) {
    set_error("bins_cycle: bad arguments (rec and records 32-byte aligned, buffers, d_status "
              "required)");
    return BP_EINVAL;
  }
  if (ncell != geo_i[0] * geo_i[1] * geo_i[2]) {
    set_error("bins_cycle: ncell does not match geo_i");
    return BP_EINVAL;
  }
  c.acc = acc; c.invvol = invvol;
  c.dt = dt; c.dth = dth; c.qdt2m = qdt2m; c.beta = beta; c.one = one; c.scale = scale;
  c.n_iters = n_iters; c.mixed = pbytes != fbytes; c.apply_bc = 1;
  c.records = records;
  c.status = d_status;
  BinsArgs ba{rec,     ids,      start,        count, ncell, leavers,
              leaver_cap, overflow, overflow_cap, stat,  late,  late_cap, pbytes};
  return bins_cycle(c, ba, (cudaStream_t)stream);
}

int bp_bins_export(int pbytes, const void* rec, int64_t* ids, const int64_t* start, int32_t* count,
                   int64_t ncell, const void* overflow, int64_t overflow_cap, uint64_t* stat,
                   int64_t* offsets, void* const* dst, int64_t* dst_ids, int64_t* total,
                   void* stream) {
  if ((pbytes != 4 && pbytes != 8) || !rec || ((uintptr_t)rec % 16) != 0 || !ids || !start ||
      !count || !offsets || !total || ncell <= 0) {
    set_error("bins_export: bad arguments");
    return BP_EINVAL;
  }
  ensure_pool();
  BinsArgs ba{nullptr, ids,  start, count, ncell, nullptr, 0, const_cast<void*>(overflow),
              overflow ? overflow_cap : 0, stat, nullptr, 0, pbytes};
  return bins_export(ba, rec, offsets, dst, dst_ids, total, (cudaStream_t)stream);
}

int bp_bins_reslack(int pbytes, const void* rec, int64_t* ids, const int64_t* start, int32_t* count,
                    int64_t ncell, const void* overflow, int64_t overflow_cap, uint64_t* stat,
                    double slack_frac, int slack_min, int32_t* new_count, int64_t* new_start,
                    void* dst_rec, int64_t* dst_ids, int64_t* total, void* stream) {
  if ((pbytes != 4 && pbytes != 8) || !rec || ((uintptr_t)rec % 16) != 0 || !ids || !start ||
      !count || !new_count ||
      !new_start || !total || ncell <= 0 || slack_frac < 0 || slack_min < 0 ||
      (overflow && !stat)) {
    set_error("bins_reslack: bad arguments");
    return BP_EINVAL;
  }
  ensure_pool();
  BinsArgs ba{nullptr, ids,  start, count, ncell, nullptr, 0, const_cast<void*>(overflow),
              overflow ? overflow_cap : 0, stat, nullptr, 0, pbytes};
  if (!dst_rec)
    return bins_reslack_plan(ba, rec, new_count, new_start, slack_frac, slack_min,
                             total, (cudaStream_t)stream);
  if (!dst_ids || ((uintptr_t)dst_rec % 16) != 0) {
    set_error("bins_reslack: dst_ids required with dst_rec (16-byte aligned)");
    return BP_EINVAL;
  }
  return bins_reslack_copy(ba, rec, new_start, new_count, dst_rec, dst_ids,
                           (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Bit-exact device loader (bp_init.cu)
int bp_init_maxwellian(int pbytes, uint64_t seed, uint64_t species_id, const int64_t* geo_i,
                       const double* origin, const double* spacing, int ppc,
                       const double* drift, const double* vth, const double* q_cell,
                       int64_t c0, int64_t nc, void* xs, void* ys, void* zs, void* us,
                       void* vs, void* ws, void* qs, int64_t* ids, int64_t* tail_k,
                       double* tail_u, int64_t tail_cap, int64_t* n_tail, void* stream) {
  if ((pbytes != 4 && pbytes != 8) || !geo_i || !origin || !spacing || !drift || !vth ||
      !q_cell || ppc < 1 || c0 < 0 || nc < 0 || !xs || !ys || !zs || !us || !vs || !ws ||
      !qs || !ids || !n_tail || tail_cap < 0 || (tail_cap > 0 && (!tail_k || !tail_u))) {
    set_error("init_maxwellian: bad arguments");
    return BP_EINVAL;
  }
  const int64_t n_cells = geo_i[0] * geo_i[1] * geo_i[2];
  if (n_cells <= 0 || c0 + nc > n_cells || n_cells * (int64_t)ppc > ((int64_t)1 << 40)) {
    set_error("init_maxwellian: cell range outside the grid");
    return BP_EINVAL;
  }
  ensure_pool();
  InitArgs A{};
  A.pbytes = pbytes;
  A.seed = seed;
  A.species_id = species_id;
  A.n_cells = n_cells;
  A.nx = geo_i[0];
  A.ny = geo_i[1];
  A.ppc = ppc;
  A.c0 = c0;
  A.nc = nc;
  for (int a = 0; a < 3; ++a) {
    A.origin[a] = origin[a];
    A.spacing[a] = spacing[a];
    A.drift[a] = drift[a];
    A.vth[a] = vth[a];
  }
  A.q_cell = q_cell;
  void* arr[7] = {xs, ys, zs, us, vs, ws, qs};
  for (int k = 0; k < 7; ++k) A.arr[k] = arr[k];
  A.ids = ids;
  A.tail_k = tail_k;
  A.tail_u = tail_u;
  A.tail_cap = tail_cap;
  A.n_tail = n_tail;
  *n_tail = 0;
  return init_maxwellian(A, (cudaStream_t)stream);
}
