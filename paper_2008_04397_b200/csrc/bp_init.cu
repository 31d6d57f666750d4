// Bit-exact device particle loader: the reference's init_maxwellian
// (pkg/src/batchpic/particles.py:177-241) generated in HBM.
//
// The reference draws, per species, from numpy's
// Generator(Philox(key=[seed, species_id])): first random((3, n_p)) — the
// cell jitter of x, y, z, one u64 per value — then standard_normal((3, n_p))
// — numpy's 256-layer ziggurat (random_standard_normal), which consumes a
// variable number of u64 per normal (rectangle: 1, wedge: 2 or more, tail
// strip: 3 or more).  The u64 stream is counter based: u64 m is word m % 4 of
// the Philox4x64-10 block with counter m / 4 + 1 (numpy increments before
// use), so every jitter value is computed independently.  The normals are
// resolved in four passes over the stream positions p (relative to the first
// normal's u64, 3 n_p):
//   zig_len      per position, the u64 count of a normal starting there
//                (rectangle test inline, one Philox block per thread);
//   zig_chunks   per chunk of kChunk positions and entry offset e < kEntries,
//                the exit offset into the next chunk and the normal count
//                when the chain of normals enters the chunk at e;
//   zig_resolve  one thread walks the chunks: the true entry of each chunk
//                and the ordinal of its first normal;
//   zig_emit     per chunk, the chain from its entry: normal k goes to
//                component k / n_p, particle k % n_p (when on this shard).
// Arithmetic as numpy's (no contraction: __dmul_rn / __dadd_rn).  The tail
// strip's value -(1/r) log1p(-U) depends on the host libm's log1p, which is
// not correctly rounded and has no bit-exact device twin: those normals
// (~0.03% of draws) are listed (ordinal, U, sign) and finished by the host
// caller with its libm (paper_2008_04397_b200/gem.py).  The wedge and tail
// acceptance tests use the device exp / log1p: they can differ from the
// host's only for a draw within an ulp of the acceptance boundary.
#include <cstdint>
#include <cstdio>

#include "bp_launch.h"
#include "bp_ziggurat_tables.h"

namespace bp {
namespace init {

constexpr unsigned long long kM0 = 0xD2E7470EE14C6C93ULL, kM1 = 0xCA5A826395121157ULL;
constexpr unsigned long long kW0 = 0x9E3779B97F4A7C15ULL, kW1 = 0xBB67AE8584CAA73BULL;
constexpr double kZR = 3.6541528853610087963519472518;    // ziggurat_nor_r
constexpr double kZIR = 0.27366123732975827203338247596;  // ziggurat_nor_inv_r
constexpr int kChunk = 16384;
constexpr int kEntries = 8;

struct U4 {
  unsigned long long v[4];
};

// Philox4x64-10 (Random123 / numpy philox.h) of counter (c0, 0, 0, 0)
__device__ __forceinline__ U4 philox(unsigned long long c0, unsigned long long k0,
                                     unsigned long long k1) {
  unsigned long long c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kW0;
      k1 += kW1;
    }
    const unsigned long long lo0 = kM0 * c0, hi0 = __umul64hi(kM0, c0);
    const unsigned long long lo1 = kM1 * c2, hi1 = __umul64hi(kM1, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  return U4{{c0, c1, c2, c3}};
}

// the species' u64 stream with a one-block cache
struct Stream {
  unsigned long long k0, k1;
  long long blk;
  U4 buf;
  __device__ Stream(unsigned long long a, unsigned long long b) : k0(a), k1(b), blk(-1) {}
  __device__ __forceinline__ unsigned long long at(long long m) {
    const long long b = m >> 2;
    if (b != blk) {
      blk = b;
      buf = philox((unsigned long long)b + 1ULL, k0, k1);
    }
    return buf.v[m & 3];
  }
};

__device__ __forceinline__ double next_double(unsigned long long r) {
  return __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0);
}

struct Normal {
  double val;
  int len;       // u64 consumed
  int tail;      // 1: tail strip (value finished by the host)
  double tail_u;  // the accepted tail iteration's first uniform
  int sign;
};

// random_standard_normal (numpy distributions.c) from stream position m0
__device__ Normal normal_at(Stream& S, long long m0) {
  long long m = m0;
  for (;;) {
    unsigned long long r = S.at(m++);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, __ldg(zig::kWi + idx));
    if (sign) x = -x;
    if (rabs < __ldg(zig::kKi + idx)) return Normal{x, (int)(m - m0), 0, 0.0, 0};
    if (idx == 0) {
      for (;;) {
        const double u1 = next_double(S.at(m++));
        const double u2 = next_double(S.at(m++));
        const double xx = __dmul_rn(-kZIR, log1p(-u1));
        const double yy = -log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          const int neg = (int)((rabs >> 8) & 1);
          const double v = __dadd_rn(kZR, xx);
          return Normal{neg ? -v : v, (int)(m - m0), 1, u1, neg};
        }
      }
    } else {
      const double fa = __ldg(zig::kFi + idx - 1), fb = __ldg(zig::kFi + idx);
      const double u = next_double(S.at(m++));
      if (__dadd_rn(__dmul_rn(__dsub_rn(fa, fb), u), fb) < exp(__dmul_rn(__dmul_rn(-0.5, x), x)))
        return Normal{x, (int)(m - m0), 0, 0.0, 0};
    }
  }
}

struct Load {
  unsigned long long k0, k1;  // Philox key (seed, species id)
  long long n_p;              // particles of the species (all cells)
  int ppc, nx, ny;
  long long p0, p1;           // this shard's particles [p0, p1)
  double o[3], d[3];          // origin, spacings
  double drift[3], vth[3];
  const double* q_cell;       // [shard cells] charge weight per cell
  int pbytes;
  void* arr[7];               // x y z u v w q of the shard
  long long* ids;
  long long base;             // first u64 of the normals: 3 n_p
  long long M;                // stream positions examined
  long long N;                // normals needed: 3 n_p
  unsigned short* len;        // [M]
  int* exits;                 // [nchunk][kEntries]
  int* counts;
  int* entry;                 // [nchunk]
  long long* kfirst;          // [nchunk]
  int* status;                // [0] error bits, [1] last chunk + 1
  long long* tail_k;          // ordinal * 2 + sign
  double* tail_u;
  unsigned long long* n_tail;
  long long tail_cap;
};

__device__ __forceinline__ void put(const Load& L, int a, long long i, double v) {
  if (L.pbytes == 4)
    static_cast<float*>(L.arr[a])[i] = __double2float_rn(v);
  else
    static_cast<double*>(L.arr[a])[i] = v;
}

// x = (o + d ci) + d U, the reference's expression order (particles.py:211-216)
__global__ void jitter(const __grid_constant__ Load L) {
  const long long nb = (L.p1 - L.p0 + 3) / 4 + 1;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < 3 * nb;
       t += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(t / nb);
    // u64 m = a n_p + p; blocks of 4 aligned on m
    const long long mlo = a * L.n_p + L.p0;
    const long long b = (mlo >> 2) + (t % nb);
    const U4 w = philox((unsigned long long)b + 1ULL, L.k0, L.k1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long p = 4 * b + j - a * L.n_p;
      if (p < L.p0 || p >= L.p1) continue;
      const long long cell = p / L.ppc;
      const long long ci = a == 0 ? cell % L.nx : (a == 1 ? (cell / L.nx) % L.ny
                                                           : cell / ((long long)L.nx * L.ny));
      const double corner = __dadd_rn(L.o[a], __dmul_rn(L.d[a], (double)ci));
      put(L, a, p - L.p0, __dadd_rn(corner, __dmul_rn(L.d[a], next_double(w.v[j]))));
    }
  }
}

__global__ void charge_ids(const __grid_constant__ Load L) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L.p1 - L.p0;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = L.p0 + i;
    put(L, 6, i, L.q_cell[p / L.ppc - L.p0 / L.ppc]);
    L.ids[i] = p;
  }
}

// u64 count of the normal starting at each stream position (one Philox
// block of 4 positions per thread; the rectangle test inline)
__global__ void zig_len(const __grid_constant__ Load L) {
  const long long b0 = L.base >> 2, b1 = (L.base + L.M + 3) >> 2;
  for (long long b = b0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; b < b1;
       b += (long long)gridDim.x * blockDim.x) {
    Stream S(L.k0, L.k1);
    S.blk = b;
    S.buf = philox((unsigned long long)b + 1ULL, L.k0, L.k1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long m = 4 * b + j, p = m - L.base;
      if (p < 0 || p >= L.M) continue;
      const unsigned long long r = S.buf.v[j];
      const int idx = (int)(r & 0xff);
      const unsigned long long rabs = (r >> 9) & 0x000fffffffffffffULL;
      int n = 1;
      if (rabs >= __ldg(zig::kKi + idx)) {
        Stream T(L.k0, L.k1);
        n = normal_at(T, m).len;
      }
      L.len[p] = (unsigned short)min(n, 65535);
    }
  }
}

// chunk tables: chain entering chunk j at offset e -> exit offset, count
__global__ void zig_chunks(const __grid_constant__ Load L, long long nchunk) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nchunk * kEntries;
       t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / kEntries;
    const int e = (int)(t % kEntries);
    const long long end = min((j + 1) * (long long)kChunk, L.M);
    long long p = j * (long long)kChunk + e;
    int cnt = 0;
    while (p < end) {
      const int n = L.len[p];
      if (n == 65535) {
        atomicOr(L.status, 2);  // a normal longer than the length field
        break;
      }
      p += n;
      ++cnt;
    }
    L.exits[t] = (int)(p - (j + 1) * (long long)kChunk);
    L.counts[t] = cnt;
  }
}

// one thread: the true entry of every chunk and its first normal's ordinal
__global__ void zig_resolve(const __grid_constant__ Load L, long long nchunk) {
  if (blockIdx.x || threadIdx.x) return;
  long long k = 0;
  int e = 0;
  long long j = 0;
  for (; j < nchunk && k < L.N; ++j) {
    L.entry[j] = e;
    L.kfirst[j] = k;
    int ex, cn;
    if (e < kEntries) {
      ex = L.exits[j * kEntries + e];
      cn = L.counts[j * kEntries + e];
    } else {  // a long normal overshot the table: walk this chunk directly
      const long long end = min((j + 1) * (long long)kChunk, L.M);
      long long p = j * (long long)kChunk + e;
      cn = 0;
      while (p < end) {
        p += L.len[p];
        ++cn;
      }
      ex = (int)(p - (j + 1) * (long long)kChunk);
    }
    k += cn;
    e = ex;
  }
  L.status[1] = (int)j;
  if (k < L.N) atomicOr(L.status, 1);  // stream window too short
}

__global__ void zig_emit(const __grid_constant__ Load L) {
  const long long nch = L.status[1];
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < nch;
       j += (long long)gridDim.x * blockDim.x) {
    // normals k of this chunk: [kfirst[j], kfirst[j + 1]); skip the chunk
    // unless it holds a normal of the shard (k mod n_p in [p0, p1))
    const long long klo = L.kfirst[j], khi = j + 1 < nch ? L.kfirst[j + 1] : L.N;
    bool hit = false;
    for (int a = 0; a < 3 && !hit; ++a)
      hit = klo < a * L.n_p + L.p1 && khi > a * L.n_p + L.p0;
    if (!hit) continue;
    Stream S(L.k0, L.k1);
    const long long end = min((j + 1) * (long long)kChunk, L.M);
    long long p = j * (long long)kChunk + L.entry[j];
    long long k = klo;
    while (p < end && k < L.N) {
      const Normal nm = normal_at(S, L.base + p);
      if (nm.len != (int)L.len[p]) atomicOr(L.status, 4);
      const int a = (int)(k / L.n_p);
      const long long pp = k % L.n_p;
      if (pp >= L.p0 && pp < L.p1) {
        put(L, 3 + a, pp - L.p0, __dadd_rn(L.drift[a], __dmul_rn(L.vth[a], nm.val)));
        if (nm.tail) {
          const unsigned long long o = atomicAdd(L.n_tail, 1ULL);
          if ((long long)o < L.tail_cap) {
            L.tail_k[o] = 2 * k + nm.sign;
            L.tail_u[o] = nm.tail_u;
          } else {
            atomicOr(L.status, 8);
          }
        }
      }
      p += nm.len;
      ++k;
    }
  }
}

}  // namespace init

namespace {
int icheck(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -2;
  }
  return 0;
}
int nsm_init() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}
}  // namespace

// See bp_b200.h bp_init_maxwellian.
int init_maxwellian(const InitArgs& A, cudaStream_t s) {
  init::Load L{};
  L.k0 = A.seed;
  L.k1 = A.species_id;
  L.n_p = A.n_cells * A.ppc;
  L.ppc = A.ppc;
  L.nx = (int)A.nx;
  L.ny = (int)A.ny;
  L.p0 = A.c0 * A.ppc;
  L.p1 = (A.c0 + A.nc) * A.ppc;
  for (int a = 0; a < 3; ++a) {
    L.o[a] = A.origin[a];
    L.d[a] = A.spacing[a];
    L.drift[a] = A.drift[a];
    L.vth[a] = A.vth[a];
  }
  L.q_cell = A.q_cell;
  L.pbytes = A.pbytes;
  for (int k = 0; k < 7; ++k) L.arr[k] = A.arr[k];
  L.ids = (long long*)A.ids;
  L.base = 3 * L.n_p;
  L.N = 3 * L.n_p;
  // expected u64 per normal ~1.02 (numpy's ziggurat): 1/16 margin + slack
  L.M = L.N + L.N / 16 + 4 * init::kChunk;
  const long long nchunk = (L.M + init::kChunk - 1) / init::kChunk;
  L.tail_k = (long long*)A.tail_k;
  L.tail_u = A.tail_u;
  L.tail_cap = A.tail_cap;
  const int g = nsm_init() * 8;
  if (L.p1 > L.p0) {
    init::jitter<<<g, 256, 0, s>>>(L);
    init::charge_ids<<<g, 256, 0, s>>>(L);
    note_launch(2);
  }
  if (A.skip_velocities) return icheck("init jitter");
  size_t bytes = (size_t)L.M * 2 + (size_t)nchunk * init::kEntries * 8 + (size_t)nchunk * 12 +
                 64 + 1024;
  char* ws = nullptr;
  if (cudaMallocAsync(&ws, bytes, s) != cudaSuccess) {
    set_error("init_maxwellian: scratch allocation of %zu bytes failed", bytes);
    return -2;
  }
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  char* p = ws;
  L.len = (unsigned short*)p; p += up((size_t)L.M * 2);
  L.exits = (int*)p; p += up((size_t)nchunk * init::kEntries * 4);
  L.counts = (int*)p; p += up((size_t)nchunk * init::kEntries * 4);
  L.entry = (int*)p; p += up((size_t)nchunk * 4);
  L.kfirst = (long long*)p; p += up((size_t)nchunk * 8);
  L.status = (int*)p; p += 64;
  L.n_tail = (unsigned long long*)p;
  cudaMemsetAsync(L.status, 0, 64 + 8, s);
  init::zig_len<<<g, 256, 0, s>>>(L);
  init::zig_chunks<<<g, 256, 0, s>>>(L, nchunk);
  init::zig_resolve<<<1, 32, 0, s>>>(L, nchunk);
  init::zig_emit<<<(int)((nchunk + 127) / 128), 128, 0, s>>>(L);
  note_launch(4);
  int st[2] = {0, 0};
  unsigned long long nt = 0;
  cudaMemcpyAsync(st, L.status, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&nt, L.n_tail, 8, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(ws, s);
  int rc = icheck("init_maxwellian");
  if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = icheck("init_maxwellian sync");
  if (rc) return rc;
  if (st[0]) {
    set_error("init_maxwellian: normal stream resolution failed (flags %d)", st[0]);
    return -2;
  }
  *A.n_tail = (int64_t)nt;
  return 0;
}

}  // namespace bp
