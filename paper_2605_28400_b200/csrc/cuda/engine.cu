// engine.cu — host engine + C-ABI (include/trioalign_capi.h).
//
// Replaces the reference batch path: plan_partition/run_batch/run_worker
// (/root/reference/proj/src/dispatch.cpp:29-162) and the engine entry points
// align / oracle_align (tiled.cpp:62-71, oracle.cpp:182-190).  One call:
//   host ASCII -> H2D -> 2-bit pack (device) -> length buckets -> persistent
//   wavefront kernels (K1, or K2 + K3 walker for rows) -> D2H results.
// There is no CPU fallback: every alignment is computed by the kernels in
// wavefront.cuh; a missing/failed device is reported as TA_ERR_CUDA.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a profiler attaches

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <tuple>
#include <thread>
#include <utility>
#include <vector>

#include "../../../include/trioalign_capi.h"
#include "kernels.h"
#include "kernels_aff.h"

namespace {
// NVTX range for the host phases of the engine (visible in Nsight Systems /
// Compute timelines: ta/create, ta/plan, ta/launch, ta/rows, ...)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define TA_CK(expr)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(TA_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// device buffers

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
  cudaError_t reserve(size_t n) {
    if (n <= cap && ptr) return cudaSuccess;
    release();
    const size_t want = std::max<size_t>(n, 1);
    cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
};

struct WaveRound {
  int ctas = 0;
  int soff_at = 0;   // this round's stream offsets start at soff[soff_at]
  int steps_at = 0;  // and its per-CTA step counts at steps[steps_at]
};

struct BucketLaunch {
  int grid = 0, lanes = 0, mode = 0;
  bool wave = false;
  ta::KernelEntry ke;
  int ctas = 0;
  DevBuf<int4> items;
  DevBuf<int32_t> soff, steps;
  DevBuf<int32_t> faces;
  DevBuf<int64_t> face_off;
  DevBuf<int64_t> wave_base;  // wave mode: per triplet id, face area in 8-byte entries
  std::vector<WaveRound> rounds;  // wave mode: launches in dependency order
  int64_t face_bytes = 0;
  uint32_t epoch = 0;         // wave mode: tag epoch of the last launch
  int64_t padded = 0;
};


// ---------------------------------------------------------------------------
// kernels around the wavefront

// One warp per sequence: ASCII -> 2-bit codes, 16 bases per word.
__global__ void pack_kernel(const char* __restrict__ ascii, const int64_t* __restrict__ src_off,
                            const int32_t* __restrict__ len, const uint32_t* __restrict__ dst_word,
                            int64_t nseq, uint32_t* __restrict__ seq, int32_t* __restrict__ bad) {
  const int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nseq) return;
  const char* src = ascii + src_off[s];
  const int L = len[s];
  const int nw = (L + 15) >> 4;
  bool badc = false;
  for (int w = lane; w < nw; w += 32) {
    uint32_t word = 0;
    const int base = w * 16;
    const int cnt = min(16, L - base);
    for (int q = 0; q < cnt; ++q) {
      const char ch = src[base + q];
      uint32_t code;
      switch (ch) {
        case 'A': code = 0; break;
        case 'C': code = 1; break;
        case 'G': code = 2; break;
        case 'T': code = 3; break;
        default: code = 0; badc = true; break;
      }
      word |= code << (2 * q);
    }
    seq[dst_word[s] + w] = word;
  }
  if (__any_sync(0xFFFFFFFFu, badc) && lane == 0) bad[s / 3] = 1;
}

// (value, lexicographic index) keys -> score and end coordinates.
__global__ void decode_keys_kernel(const unsigned long long* __restrict__ key,
                                   const ta::TripletDesc* __restrict__ desc,
                                   const int32_t* __restrict__ ids, int64_t n,
                                   int32_t* __restrict__ score, int32_t* __restrict__ end) {
  const int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int32_t id = ids[x];
  const unsigned long long k = key[id];
  const ta::TripletDesc d = desc[id];
  const unsigned long long lin = ta::key_lin(k);
  const unsigned long long plane = static_cast<unsigned long long>(d.b + 1) * static_cast<unsigned long long>(d.c + 1);
  const unsigned long long i = lin / plane;
  const unsigned long long rem = lin - i * plane;
  const unsigned long long j = rem / static_cast<unsigned long long>(d.c + 1);
  const unsigned long long kk = rem - j * static_cast<unsigned long long>(d.c + 1);
  score[id] = ta::key_value(k);
  end[3 * id] = static_cast<int32_t>(i);
  end[3 * id + 1] = static_cast<int32_t>(j);
  end[3 * id + 2] = static_cast<int32_t>(kk);
}

__device__ __forceinline__ char base_char(const uint32_t* seq, uint32_t w, int pos) {
  const uint32_t code = (seq[w + (pos >> 4)] >> ((pos & 15) * 2)) & 3u;
  return "ACGT"[code];
}

// K3: traceback walker over the direction cube (oracle.cpp:98-180).  One
// thread per triplet: walk from `end` choosing the recorded first-max term;
// stop at (0,0,0) (global), an axis cell (semi) or a floor cell (local);
// emit rows with semi-global free prefix / suffix columns.
__global__ void walker_kernel(const ta::TripletDesc* __restrict__ desc,
                              const uint32_t* __restrict__ seq, const int32_t* __restrict__ ids,
                              int n, const uint32_t* __restrict__ dirs,
                              const int64_t* __restrict__ dir_off, int grid, int mode,
                              const int32_t* __restrict__ end, int32_t* __restrict__ begin,
                              char* __restrict__ rows, const int64_t* __restrict__ row_off,
                              int32_t* __restrict__ row_len, int32_t* __restrict__ status,
                              int32_t* __restrict__ len_ord) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int id = ids[x];
  const ta::TripletDesc d = desc[id];
  constexpr int N = ta::kTileN;
  const int T = grid * grid;
  const uint32_t* base = dirs + dir_off[id];
  const int GN = grid * N;
  const int Bk = (d.c + 1 + GN - 1) / GN;
  // record layout (wavefront.cuh, kDirWords): [block][slice][word][thread],
  // thread = anti-diagonal index of the tile, word/bit = sweep-order index of the cell
  auto code_at = [&](int i, int j, int k) -> uint32_t {
    const int blk = (j / GN) * Bk + (k / GN);
    const int jj = j % GN, kk = k % GN;
    const int t = ta::antidiag_index(jj / N, kk / N, grid);
    const int cs = ta::antidiag_index(jj % N, kk % N, N);
    const int m = cs % 10;
    const uint32_t w = base[((int64_t(blk) * (d.a + 1) + i) * ta::kDirWords + cs / 10) * T + t];
    return (w >> (m < 5 ? 3 * m : 16 + 3 * (m - 5))) & 7u;
  };
  auto stop_at = [&](int i, int j, int k, uint32_t code) {
    if (mode == ta::kGlobal) return i == 0 && j == 0 && k == 0;
    if (mode == ta::kSemi) return (j == 0 && k == 0) || (i == 0 && k == 0) || (i == 0 && j == 0);
    return code == ta::kTagStop;
  };
  const int ei = end[3 * id], ej = end[3 * id + 1], ek = end[3 * id + 2];
  // pass 1: path length and begin
  int i = ei, j = ej, k = ek, steps = 0;
  const int limit = d.a + d.b + d.c + 1;
  bool ok = true;
  for (;;) {
    const uint32_t code = (mode == ta::kLocal) ? code_at(i, j, k) : 0u;
    if (stop_at(i, j, k, code)) break;
    const uint32_t c = (mode == ta::kLocal) ? code : code_at(i, j, k);
    int di, dj, dk;
    switch (c) {
      case ta::kTagT1: di = 1, dj = 1, dk = 1; break;
      case ta::kTagT2: di = 1, dj = 1, dk = 0; break;
      case ta::kTagT3: di = 1, dj = 0, dk = 1; break;
      case ta::kTagT4: di = 0, dj = 1, dk = 1; break;
      case ta::kTagT5: di = 1, dj = 0, dk = 0; break;
      case ta::kTagT6: di = 0, dj = 1, dk = 0; break;
      case ta::kTagT7: di = 0, dj = 0, dk = 1; break;
      default: di = dj = dk = -1; break;
    }
    if (di < 0 || i - di < 0 || j - dj < 0 || k - dk < 0 || ++steps > limit) {
      ok = false;
      break;
    }
    i -= di, j -= dj, k -= dk;
  }
  if (!ok) {
    status[id] = TA_ERR_LOGIC;
    row_len[id] = 0;
    if (len_ord) len_ord[x] = 0;
    return;
  }
  begin[3 * id] = i, begin[3 * id + 1] = j, begin[3 * id + 2] = k;
  const int bi = i, bj = j, bk = k;
  const bool semi = mode == ta::kSemi;
  const int prefix = semi ? (bi + bj + bk) : 0;
  const int suffix = semi ? ((d.a - ei) + (d.b - ej) + (d.c - ek)) : 0;
  const int len = prefix + steps + suffix;
  row_len[id] = len;
  if (len_ord) len_ord[x] = len;
  const int64_t cap = int64_t(d.a) + d.b + d.c;
  char* r0 = rows + row_off[id];
  char* r1 = r0 + cap;
  char* r2 = r1 + cap;
  int pos = 0;
  if (semi) {
    for (int p = 0; p < bi; ++p, ++pos) r0[pos] = base_char(seq, d.w0, p), r1[pos] = '-', r2[pos] = '-';
    for (int p = 0; p < bj; ++p, ++pos) r0[pos] = '-', r1[pos] = base_char(seq, d.w1, p), r2[pos] = '-';
    for (int p = 0; p < bk; ++p, ++pos) r0[pos] = '-', r1[pos] = '-', r2[pos] = base_char(seq, d.w2, p);
  }
  // pass 2: write the path columns back to front
  i = ei, j = ej, k = ek;
  for (int s = steps - 1; s >= 0; --s) {
    const uint32_t c = code_at(i, j, k);
    const int at = prefix + s;
    const bool u0 = c == ta::kTagT1 || c == ta::kTagT2 || c == ta::kTagT3 || c == ta::kTagT5;
    const bool u1 = c == ta::kTagT1 || c == ta::kTagT2 || c == ta::kTagT4 || c == ta::kTagT6;
    const bool u2 = c == ta::kTagT1 || c == ta::kTagT3 || c == ta::kTagT4 || c == ta::kTagT7;
    r0[at] = u0 ? base_char(seq, d.w0, i - 1) : '-';
    r1[at] = u1 ? base_char(seq, d.w1, j - 1) : '-';
    r2[at] = u2 ? base_char(seq, d.w2, k - 1) : '-';
    i -= u0, j -= u1, k -= u2;
  }
  pos = prefix + steps;
  if (semi) {
    for (int p = ei; p < d.a; ++p, ++pos) r0[pos] = base_char(seq, d.w0, p), r1[pos] = '-', r2[pos] = '-';
    for (int p = ej; p < d.b; ++p, ++pos) r0[pos] = '-', r1[pos] = base_char(seq, d.w1, p), r2[pos] = '-';
    for (int p = ek; p < d.c; ++p, ++pos) r0[pos] = '-', r1[pos] = '-', r2[pos] = base_char(seq, d.w2, p);
  }
}

// K3a: traceback walker of the affine path (SPEC-AFFINE.md).  Each cell
// record (affine.cuh) holds the 3-bit tags of V1's source (7 = start), of
// B's argmax and of the predecessor type of every V_t; tag = 7 - type.
__global__ void affine_walker_kernel(const ta::TripletDesc* __restrict__ desc, const uint32_t* __restrict__ seq,
                                     const int32_t* __restrict__ ids, int n, const uint32_t* __restrict__ dirs,
                                     const int64_t* __restrict__ dir_off, int mode, const int32_t* __restrict__ end,
                                     int32_t* __restrict__ begin, char* __restrict__ rows,
                                     const int64_t* __restrict__ row_off, int32_t* __restrict__ row_len,
                                     int32_t* __restrict__ status) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int id = ids[x];
  const ta::TripletDesc d = desc[id];
  constexpr int N = ta::kAffN, G = ta::kAffG, T = G * G, GN = G * N;
  const uint32_t* base = dirs + dir_off[id] * 4;
  const int Bk = (d.c + 1 + GN - 1) / GN;
  auto rec_at = [&](int i, int j, int k) -> uint32_t {
    const int blk = (j / GN) * Bk + (k / GN);
    const int jj = j % GN, kk = k % GN;
    const int t = (jj / N) * G + (kk / N);
    const int cell = (jj % N) * N + (kk % N);
    return base[((int64_t(blk) * (d.a + 1) + i) * T + t) * ta::kAffRec + cell];
  };
  static constexpr int kMaskOf[8] = {0, 7, 3, 5, 6, 1, 2, 4};
  const int ei = end[3 * id], ej = end[3 * id + 1], ek = end[3 * id + 2];
  // pass 1: path length and begin
  int i = ei, j = ej, k = ek, steps = 0;
  int ty = 7 - int((rec_at(i, j, k) >> 3) & 7u);
  const int t_end = ty;
  const int limit = d.a + d.b + d.c + 1;
  bool ok = true;
  for (;;) {
    const uint32_t rc = rec_at(i, j, k);
    if (ty == 1 && (rc & 7u) == 7u) break;  // a start
    const uint32_t tag = ty == 1 ? (rc & 7u) : (rc >> (6 + 3 * (ty - 2))) & 7u;
    const int m = kMaskOf[ty];
    const int di = m & 1, dj = (m >> 1) & 1, dk = (m >> 2) & 1;
    if (tag == 7u || i - di < 0 || j - dj < 0 || k - dk < 0 || ++steps > limit) {
      ok = false;
      break;
    }
    i -= di, j -= dj, k -= dk;
    ty = 7 - int(tag);
  }
  if (!ok) {
    status[id] = TA_ERR_LOGIC;
    row_len[id] = 0;
    return;
  }
  begin[3 * id] = i, begin[3 * id + 1] = j, begin[3 * id + 2] = k;
  const int bi = i, bj = j, bk = k;
  const bool semi = mode == ta::kSemi;
  const int prefix = semi ? (bi + bj + bk) : 0;
  const int suffix = semi ? ((d.a - ei) + (d.b - ej) + (d.c - ek)) : 0;
  row_len[id] = prefix + steps + suffix;
  const int64_t cap = int64_t(d.a) + d.b + d.c;
  char* r0 = rows + row_off[id];
  char* r1 = r0 + cap;
  char* r2 = r1 + cap;
  int pos = 0;
  if (semi) {
    for (int p = 0; p < bi; ++p, ++pos) r0[pos] = base_char(seq, d.w0, p), r1[pos] = '-', r2[pos] = '-';
    for (int p = 0; p < bj; ++p, ++pos) r0[pos] = '-', r1[pos] = base_char(seq, d.w1, p), r2[pos] = '-';
    for (int p = 0; p < bk; ++p, ++pos) r0[pos] = '-', r1[pos] = '-', r2[pos] = base_char(seq, d.w2, p);
  }
  // pass 2: the path columns back to front
  i = ei, j = ej, k = ek, ty = t_end;
  for (int s = steps - 1; s >= 0; --s) {
    const uint32_t rc = rec_at(i, j, k);
    const uint32_t tag = ty == 1 ? (rc & 7u) : (rc >> (6 + 3 * (ty - 2))) & 7u;
    const int m = kMaskOf[ty];
    const int u0 = m & 1, u1 = (m >> 1) & 1, u2 = (m >> 2) & 1;
    const int at = prefix + s;
    r0[at] = u0 ? base_char(seq, d.w0, i - 1) : '-';
    r1[at] = u1 ? base_char(seq, d.w1, j - 1) : '-';
    r2[at] = u2 ? base_char(seq, d.w2, k - 1) : '-';
    i -= u0, j -= u1, k -= u2;
    ty = 7 - int(tag);
  }
  pos = prefix + steps;
  if (semi) {
    for (int p = ei; p < d.a; ++p, ++pos) r0[pos] = base_char(seq, d.w0, p), r1[pos] = '-', r2[pos] = '-';
    for (int p = ej; p < d.b; ++p, ++pos) r0[pos] = '-', r1[pos] = base_char(seq, d.w1, p), r2[pos] = '-';
    for (int p = ek; p < d.c; ++p, ++pos) r0[pos] = '-', r1[pos] = '-', r2[pos] = base_char(seq, d.w2, p);
  }
}

// ---------------------------------------------------------------------------
// per-device context (stream + events), created lazily

template <class T>
struct PinnedBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  ~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
  cudaError_t reserve(size_t n) {
    if (n <= cap && ptr) return cudaSuccess;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n + n / 4, 1024);
    cudaError_t e = cudaHostAlloc(&ptr, want * sizeof(T), cudaHostAllocDefault);
    if (e == cudaSuccess) cap = want;
    return e;
  }
};

struct DeviceCtx {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // H2D of the pipelined path
  cudaStream_t d2h = nullptr;   // D2H of the pipelined path (never queues ahead of an H2D)
  int sms = 0;
  std::mutex mu;                // one pipelined call at a time per device
  // cached buffers of the pipelined score path (grow-only)
  PinnedBuf<uint32_t> h_words[2];
  PinnedBuf<ta::TripletDesc> h_desc;
  PinnedBuf<int32_t> h_out;     // score, end (3), per triplet
  DevBuf<uint32_t> d_words;
  DevBuf<ta::TripletDesc> d_desc;
  DevBuf<int32_t> d_score, d_end;
  DevBuf<unsigned long long> d_key;
  std::vector<std::unique_ptr<BucketLaunch>> plan_pool;  // pipelined path launch plans (grow-only)
  ta_batch* oneshot = nullptr;  // reused batch object of the one-shot rows / affine path (never freed)
  ta_stats last_stats{};        // of the last ta_align_batch call (ta_last_stats)
  PinnedBuf<char> h_rows[2];    // rows path: double-buffered D2H staging of row chunks
  PinnedBuf<int32_t> h_len[2];
};

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DeviceCtx>> g_ctx;

int get_ctx(int device, DeviceCtx** out) {
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    return fail(TA_ERR_CUDA, std::string("no CUDA device available: ") +
                                 (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                                 " (the trioalign B200 engine has no CPU fallback)");
  }
  if (device < 0 || device >= count) return fail(TA_ERR_CUDA, "device index out of range");
  if (g_ctx.size() < size_t(count)) g_ctx.resize(size_t(count));
  if (!g_ctx[device]) {
    auto ctx = std::make_unique<DeviceCtx>();
    ctx->device = device;
    TA_CK(cudaSetDevice(device));
    TA_CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    TA_CK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    TA_CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    TA_CK(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device));
    g_ctx[device] = std::move(ctx);
  }
  TA_CK(cudaSetDevice(device));
  *out = g_ctx[device].get();
  return TA_OK;
}

// Host packing threads of one pipelined call: TA_HOST_THREADS if set (e.g.
// cores / ranks when several processes share the host), else the cores
// divided by the calls in flight in this process (run_batch runs one call
// per worker thread and device), so concurrent workers do not oversubscribe.
std::atomic<int> g_calls_in_flight{0};
int host_threads() {
  if (const char* e = std::getenv("TA_HOST_THREADS")) {
    const int v = std::atoi(e);
    if (v > 0) return v;
  }
  const int hw = int(std::max(1u, std::thread::hardware_concurrency()));
  return std::max(1, hw / std::max(1, g_calls_in_flight.load()));
}

// ---------------------------------------------------------------------------
// scheme / option validation with reference semantics

int validate_scheme(const ta_scheme& s) {
  // core.cpp:10-18
  if (s.match <= 0) return fail(TA_ERR_INVALID_ARGUMENT, "match score must be positive");
  if (s.mismatch > 0) return fail(TA_ERR_INVALID_ARGUMENT, "mismatch score must be <= 0");
  if (s.gap > 0) return fail(TA_ERR_INVALID_ARGUMENT, "gap score must be <= 0");
  if (std::abs(s.match) > 1024 || std::abs(s.mismatch) > 1024 || std::abs(s.gap) > 1024)
    return fail(TA_ERR_INVALID_ARGUMENT, "score magnitudes must be <= 1024");
  // affine extension (SPEC-AFFINE.md)
  if (s.gap_open > 0) return fail(TA_ERR_INVALID_ARGUMENT, "gap open score must be <= 0");
  if (std::abs(s.gap_open) > 1024) return fail(TA_ERR_INVALID_ARGUMENT, "score magnitudes must be <= 1024");
  return TA_OK;
}

int validate_options(const ta_options& o) {
  // tiled.cpp:8-15
  if (o.tile_size < 1 || o.tile_size > 4096)
    return fail(TA_ERR_CONFIG, "tile size must be in [1, 4096], got " + std::to_string(o.tile_size));
  if (o.team_width < 0) return fail(TA_ERR_CONFIG, "team width must be >= 0");
  if (o.team_threads < 1) return fail(TA_ERR_CONFIG, "team threads must be >= 1");
  if (o.cell_budget == 0) return fail(TA_ERR_CONFIG, "cell budget must be positive");
  if (o.mode < 0 || o.mode > 2) return fail(TA_ERR_INVALID_ARGUMENT, "unknown alignment mode");
  return TA_OK;
}

int32_t derive_team_width(int32_t tile_size, int32_t b, int32_t c) {
  const int32_t need = std::max(b, c);
  if (need <= 0) return 1;
  return (need + tile_size - 1) / tile_size;
}

// ---------------------------------------------------------------------------
// lane choice: s16x2 is used only when every value provably fits (exact)

struct LanePlan {
  bool packed16 = false;
};

// Largest in-grid cell value (gap-shifted, >= 0) a triplet can produce, incl.
// padding cells and idle slices: (match + |g2|) * (slices + j extent + k extent).
int64_t lane_bound(const ta_scheme& s, int32_t a, int32_t b, int32_t c, int grid, int tile_n = ta::kTileN) {
  const int g2 = 2 * s.gap;
  const int64_t gn = int64_t(grid) * tile_n;
  const int64_t ej = ((b + 1 + gn - 1) / gn) * gn, ek = ((c + 1 + gn - 1) / gn) * gn;
  const int64_t slices = std::max<int64_t>(a + 1, grid + 2 + (grid * grid + 31) / 32);
  return int64_t(s.match - g2) * (slices + ej + ek);
}

bool s16_ok(const ta_scheme& s, int64_t max_bound) {
  const int g2 = 2 * s.gap;
  const int mp = s.match - g2, mm = s.mismatch - g2;
  if (mm < 0 || mp > 127) return false;  // carry-free packed adds + byte tables
  // values in [0, bound]; unreachable terms stay below 0 from NEG = -16384
  return max_bound + 3 * 127 + int64_t(-g2) * 2 * ta::kTileN <= 32000;
}

// TRACE kernels scale values by 8 (3-bit direction tags in the low bits):
// s16x2 lanes need the scaled bound to fit as well.
bool trace16_ok(const ta_scheme& s, int64_t max_bound) {
  const int g2 = 2 * s.gap;
  const int mp = s.match - g2, mm = s.mismatch - g2;
  if (mm < 0 || mp > 127) return false;
  return (max_bound + 3 * 127 + int64_t(-g2) * 2 * ta::kTileN) * 8 + 64 <= 32000;
}

// Semi-global / local best-cell keys (ta::best_key) hold 36 bits of cell
// index and 28 bits of biased value: the triplet's tensor must have at most
// 2^36 cells and every value must stay within +-2^27 (|M| <= (a+b+c) times
// the largest per-column score, packed_score_bound's argument, plus opening
// penalties for affine gaps).
bool key_fits(int32_t a, int32_t b, int32_t c, const ta_scheme& s) {
  const uint64_t cells = uint64_t(a + 1) * uint64_t(b + 1) * uint64_t(c + 1);
  if (cells > (uint64_t(1) << ta::kKeyLinBits)) return false;
  const int64_t per = 3 * (std::max({std::abs(int64_t(s.match)), std::abs(int64_t(s.mismatch)),
                                     std::abs(int64_t(s.gap))}) + std::abs(int64_t(s.gap_open)));
  return (int64_t(a) + b + c + 1) * per < (int64_t(1) << 27) - 4096;
}

// Smallest tile grid whose plane holds the triplet; longer triplets use the
// largest grid as a sequence of blocks.
int pick_grid(int32_t b, int32_t c) {
  const int ext = std::max(b, c) + 1;
  for (int g : ta::kGridSizes)
    if (g * ta::kTileN >= ext) return g;
  return ta::kGridSizes[ta::kNumGrid - 1];
}

}  // namespace

// ---------------------------------------------------------------------------
// the batch object

struct ta_batch {
  int device = 0;
  DeviceCtx* ctx = nullptr;
  int64_t n = 0;
  std::vector<int32_t> a, b, c;
  std::vector<ta::TripletDesc> desc;
  std::vector<int32_t> pre_status;   // parse errors
  std::vector<int32_t> status;       // last run
  DevBuf<uint32_t> seq;
  DevBuf<ta::TripletDesc> d_desc;
  DevBuf<int32_t> d_score, d_end, d_begin, d_status, d_rowlen;
  DevBuf<unsigned long long> d_key;
  DevBuf<int32_t> d_items, d_soff, d_steps, d_ids;
  DevBuf<uint4> d_dirs;
  DevBuf<int64_t> d_diroff, d_rowoff;
  DevBuf<char> d_rows;
  DevBuf<int32_t> d_lenord;            // rows path: row length per position of the chunk order
  bool rows_scattered = false;         // rows path: the pipeline already wrote the caller's row planes
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evw0 = nullptr, evw1 = nullptr;
  cudaEvent_t evk[2] = {nullptr, nullptr}, evc[2] = {nullptr, nullptr};
  ta_stats stats{};
  // score-path launch plans of the last run (reused while the bucket
  // contents, lanes and mode are unchanged)
  std::vector<std::unique_ptr<BucketLaunch>> plan_cache;
  std::vector<ta::AffEntry> aff_cache;  // affine path: kernel per cached plan
  std::vector<std::unique_ptr<BucketLaunch>> rows_pool;  // rows path: per-chunk launch plans (grow-only)
  // staging of ta_batch_create (kept so a reused batch allocates nothing)
  DevBuf<char> s_ascii;
  DevBuf<int64_t> s_src;
  DevBuf<int32_t> s_len, s_bad;
  DevBuf<uint32_t> s_dst;
  std::string plan_key;
  // front cache of the linear score path: per-triplet validation, buckets and
  // the plan key of the last run, reused while scheme and options are
  // unchanged (the batch is immutable), so a repeated run does no O(n) host work
  std::string front_key;
  std::vector<int32_t> front_status, front_all_ok;
  bool status_is_front = false;  // status still equals front_status
  int64_t front_cells = 0;
  int last_mode = -1;
  bool last_rows = false;
  ~ta_batch() {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (evw0) cudaEventDestroy(evw0);
    if (evw1) cudaEventDestroy(evw1);
    for (auto e : evk)
      if (e) cudaEventDestroy(e);
    for (auto e : evc)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

struct StreamPlan {
  std::vector<int4> items;
  std::vector<int32_t> soff, steps;
  std::vector<int64_t> face_off;
  int64_t face_words = 0;
  int64_t padded_slices = 0;  // sum over items of slices * blocks (for stats)
};

struct Blocks {
  int bj = 1, bk = 1;
};

inline Blocks blocks_of(int32_t b, int32_t c, int grid, int tile_n = ta::kTileN) {
  const int gn = grid * tile_n;
  return Blocks{(b + 1 + gn - 1) / gn, (c + 1 + gn - 1) / gn};
}

// slices one block item occupies in a stream: a+1, padded for multi-block
// triplets so that a block's faces are written well before the next block's
// edge tiles prefetch them: G+1 steps in lockstep, plus the largest drift
// between warps under per-warp synchronisation (warps - 1 steps), which is
// also the length of the mbarrier release/acquire chain that makes the
// face stores visible to the prefetching warp.
inline int item_len(int32_t a, const Blocks& bl, int grid) {
  const int warps = (grid * grid + 31) / 32;
  return (bl.bj * bl.bk > 1) ? std::max(a + 1, grid + 2 + warps) : a + 1;
}

// Greedy least-loaded assignment of triplets to CTA lane streams (the
// "dynamic" rule of plan_partition, dispatch.cpp:46-56, applied to slices);
// a long triplet contributes its Bj*Bk blocks as consecutive items.
void plan_streams(const std::vector<int32_t>& ids, const std::vector<int32_t>& a,
                  const std::vector<int32_t>& b, const std::vector<int32_t>& c, int ctas, int lanes, int grid,
                  StreamPlan* out, int tile_n = ta::kTileN, bool affine = false) {
  const int S = ctas * lanes;
  const int gn = grid * tile_n;
  std::vector<std::vector<int32_t>> lists(static_cast<size_t>(S));
  std::vector<int64_t> load(static_cast<size_t>(S), 0), face(static_cast<size_t>(S), 0);
  using Load = std::pair<int64_t, int32_t>;
  auto cost = [&](int32_t id) {
    const Blocks bl = blocks_of(b[size_t(id)], c[size_t(id)], grid, tile_n);
    return int64_t(item_len(a[size_t(id)], bl, grid)) * bl.bj * bl.bk;
  };
  auto put = [&](int s, int32_t id) {
    lists[size_t(s)].push_back(id);
    load[size_t(s)] += cost(id);
    const Blocks bl = blocks_of(b[size_t(id)], c[size_t(id)], grid, tile_n);
    if (bl.bj * bl.bk > 1)
      face[size_t(s)] = std::max(face[size_t(s)], (affine ? ta::aff_face_words(a[size_t(id)], bl.bk, gn) : ta::face_words(a[size_t(id)], bl.bk, gn)));
  };
  std::vector<int32_t> singles;
  if (lanes == 2) {
    // Pair triplets with identical stream items (slices, Bj, Bk) into the two
    // lanes of one CTA so both lanes switch triplets in the same step (one
    // combined table build instead of two divergent ones).  Pairs first,
    // unpaired triplets at the stream tails.
    std::vector<int32_t> order(ids);
    auto key = [&](int32_t id) {
      const Blocks bl = blocks_of(b[size_t(id)], c[size_t(id)], grid, tile_n);
      return std::make_tuple(item_len(a[size_t(id)], bl, grid), bl.bj, bl.bk);
    };
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return key(x) < key(y); });
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
    for (int cta = 0; cta < ctas; ++cta) heap.push({0, cta});
    size_t i = 0;
    while (i < order.size()) {
      if (i + 1 < order.size() && key(order[i]) == key(order[i + 1])) {
        Load top = heap.top();
        heap.pop();
        put(top.second * 2, order[i]);
        put(top.second * 2 + 1, order[i + 1]);
        top.first += cost(order[i]);
        heap.push(top);
        i += 2;
      } else {
        singles.push_back(order[i]);
        i += 1;
      }
    }
  } else {
    singles = ids;
  }
  {
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
    for (int s = 0; s < S; ++s) heap.push({load[size_t(s)], s});
    for (int32_t id : singles) {
      Load top = heap.top();
      heap.pop();
      put(top.second, id);
      top.first = load[size_t(top.second)];
      heap.push(top);
    }
  }
  out->items.clear();
  out->soff.assign(size_t(S) + 1, 0);
  out->steps.assign(size_t(ctas), 0);
  out->face_off.assign(size_t(S), 0);
  out->face_words = 0;
  out->padded_slices = 0;
  for (int s = 0; s < S; ++s) {
    out->soff[size_t(s)] = int32_t(out->items.size());
    out->face_off[size_t(s)] = out->face_words;
    out->face_words += face[size_t(s)];
    for (int32_t id : lists[size_t(s)]) {
      const Blocks bl = blocks_of(b[size_t(id)], c[size_t(id)], grid, tile_n);
      const int len = item_len(a[size_t(id)], bl, grid);
      for (int J = 0; J < bl.bj; ++J)
        for (int K = 0; K < bl.bk; ++K) out->items.push_back(make_int4(id, (J << 16) | K, len, (bl.bj << 16) | bl.bk));
      out->padded_slices += int64_t(len) * bl.bj * bl.bk;
    }
  }
  out->soff[size_t(S)] = int32_t(out->items.size());
  for (int cta = 0; cta < ctas; ++cta) {
    int64_t mx = 0;
    for (int l = 0; l < lanes; ++l) mx = std::max(mx, load[size_t(cta * lanes + l)]);
    out->steps[size_t(cta)] = int32_t(mx + 2 * (grid - 1));
  }
}

// Wave mode: the blocks of long triplets are spread over all CTAs instead of
// running as one CTA's item sequence.  Blocks are ordered by anti-diagonal
// d = J + K (a block depends only on blocks of diagonal d - 1), dealt
// round-robin to the CTAs, and - with two lanes - paired only with a block it
// cannot depend on (same diagonal, or another triplet) and of equal length, so
// both lanes switch together.  With every CTA resident, the lowest unfinished
// diagonal can always progress: no deadlock.  Faces travel through per-block
// tagged rings (wavefront.cuh, WAVE).
struct WavePlan {
  std::vector<int4> items;
  std::vector<int32_t> soff, steps;
  std::vector<WaveRound> rounds;
  std::vector<int64_t> base;  // per triplet id (only wave triplets set)
  int64_t entries = 0;
  int64_t padded_slices = 0;
};

void plan_wave(const std::vector<int32_t>& ids, const std::vector<int32_t>& a, const std::vector<int32_t>& b,
               const std::vector<int32_t>& c, int max_ctas, int lanes, int grid, int64_t n, WavePlan* out,
               int* ctas_out, int tile_n = ta::kTileN, bool affine = false) {
  struct Blk {
    int d, id, J, K;
  };
  std::vector<Blk> blks;
  out->base.assign(size_t(n), 0);
  out->entries = 0;
  for (int32_t id : ids) {
    const Blocks bl = blocks_of(b[size_t(id)], c[size_t(id)], grid, tile_n);
    out->base[size_t(id)] = out->entries;
    out->entries += int64_t(bl.bj) * bl.bk *
                    (affine ? ta::aff_wave_block_entries(a[size_t(id)], grid) : ta::wave_block_entries(a[size_t(id)], grid));
    for (int J = 0; J < bl.bj; ++J)
      for (int K = 0; K < bl.bk; ++K) blks.push_back(Blk{J + K, id, J, K});
  }
  std::stable_sort(blks.begin(), blks.end(), [](const Blk& x, const Blk& y) { return x.d < y.d; });
  auto rec = [&](const Blk& x) {
    const Blocks bl = blocks_of(b[size_t(x.id)], c[size_t(x.id)], grid, tile_n);
    return make_int4(x.id, (x.J << 16) | x.K, a[size_t(x.id)] + 1, (bl.bj << 16) | bl.bk);
  };
  std::vector<std::pair<int4, int4>> pairs;  // (lane 0, lane 1); lane 1 may be a null item
  // Pairing halves the CTAs but doubles every face CTA's per-step face work
  // (the step is latency bound on the face warp): pair only when the blocks
  // outnumber the resident CTAs (TA_WAVE_PAIR=1 forces pairing: dev A/B knob).
  static const bool force_pair = [] {
    const char* e = std::getenv("TA_WAVE_PAIR");
    return e && std::atoi(e) == 1;
  }();
  const bool pair = force_pair || blks.size() > size_t(std::max(1, max_ctas));
  for (size_t i = 0; i < blks.size();) {
    const int4 x = rec(blks[i]);
    if (lanes == 2 && pair && i + 1 < blks.size()) {
      const Blk& u = blks[i];
      const Blk& v = blks[i + 1];
      const bool independent = u.id != v.id || u.d == v.d;
      if (independent && a[size_t(u.id)] == a[size_t(v.id)]) {
        pairs.push_back({x, rec(v)});
        i += 2;
        continue;
      }
    }
    pairs.push_back({x, make_int4(-1, 0, x.z, 0x00010001)});
    i += 1;
  }
  // One pair per CTA and launch: a CTA that held two wave items would start
  // the second (its front tiles) while its back tiles still finish the first,
  // and a wait in the second could then block producers others wait on.  So
  // pairs beyond the resident CTA count go to a later launch (round); faces
  // of earlier rounds are complete and tagged when a round starts.
  const size_t C = size_t(std::max(1, max_ctas));
  out->items.clear();
  out->soff.clear();
  out->steps.clear();
  out->rounds.clear();
  out->padded_slices = 0;
  for (size_t k0 = 0; k0 < pairs.size(); k0 += C) {
    const size_t k1 = std::min(pairs.size(), k0 + C);
    WaveRound rd;
    rd.ctas = int(k1 - k0);
    rd.soff_at = int(out->soff.size());
    rd.steps_at = int(out->steps.size());
    for (size_t k = k0; k < k1; ++k) {
      out->soff.push_back(int32_t(out->items.size()));
      out->items.push_back(pairs[k].first);
      if (lanes == 2) {
        out->soff.push_back(int32_t(out->items.size()));
        out->items.push_back(pairs[k].second);
      }
      if (pairs[k].first.x >= 0) out->padded_slices += pairs[k].first.z;
      if (lanes == 2 && pairs[k].second.x >= 0) out->padded_slices += pairs[k].second.z;
      out->steps.push_back(int32_t(pairs[k].first.z + 2 * (grid - 1)));
    }
    out->soff.push_back(int32_t(out->items.size()));
    out->rounds.push_back(rd);
  }
  *ctas_out = out->rounds.empty() ? 0 : out->rounds[0].ctas;
}

// Long triplets go to wave mode when there are too few of them to fill the
// CTA lane streams (e.g. a single 1000-2000 bp triplet, config C5).
bool wave_eligible(int32_t a, int32_t b, int32_t c, int grid) {
  const Blocks bl = blocks_of(b, c, grid);
  return grid == ta::kGridSizes[ta::kNumGrid - 1] && bl.bj * bl.bk > 1 && a + 1 < 65535;
}

void split_wave(const std::vector<int32_t>& ids, const std::vector<int32_t>& a, const std::vector<int32_t>& b,
                const std::vector<int32_t>& c, int grid, int lane_streams, std::vector<int32_t>* wave,
                std::vector<int32_t>* rest) {
  wave->clear();
  rest->clear();
  std::vector<int32_t> cand;
  for (int32_t id : ids)
    (wave_eligible(a[size_t(id)], b[size_t(id)], c[size_t(id)], grid) ? cand : *rest).push_back(id);
  if (int64_t(cand.size()) * 2 <= lane_streams) {
    *wave = cand;
  } else {
    rest->insert(rest->end(), cand.begin(), cand.end());
    std::sort(rest->begin(), rest->end());
  }
}

// Multi-block triplets of the largest grid whose (j, k) extents pad less in
// 128-wide blocks (8 x 8 tiles) than in 160-wide ones, weighting a 128-block
// cell by the measured per-cell cost ratio of the two kernels (smaller tiles
// amortise the per-step work over 64 instead of 100 cells).  Example: 250 bp
// (extent 251) pads to 2 x 2 blocks either way: 65536 vs 102400 cells/slice.
double t8_cost_ratio() {
  static const double r = [] {
    const char* e = std::getenv("TA_T8_COST");
    return e ? std::atof(e) : 1.2;  // measured: 2247 vs 2686 padded-cell GCUPS (C3)
  }();
  return r;
}

bool prefer_t8(int32_t b, int32_t c) {
  const Blocks b10 = blocks_of(b, c, 16);
  if (b10.bj * b10.bk <= 1) return false;
  const Blocks b8 = blocks_of(b, c, 16, ta::kSmallTileN);
  const double g10 = 16.0 * ta::kTileN, g8 = 16.0 * ta::kSmallTileN;
  return double(b8.bj * b8.bk) * g8 * g8 * t8_cost_ratio() < double(b10.bj * b10.bk) * g10 * g10;
}

// Splits the largest grid's bucket into wave triplets, 128-wide-block
// triplets (prefer_t8, with their own lane choice) and the rest.
void split_largest(const std::vector<int32_t>& bucket, const std::vector<int32_t>& a, const std::vector<int32_t>& b,
                   const std::vector<int32_t>& c, const ta_scheme& scheme, int lane_streams,
                   std::vector<int32_t>* wave, std::vector<int32_t>* rest, std::vector<int32_t>* t8, int* lanes8) {
  const int g = ta::kGridSizes[ta::kNumGrid - 1];
  split_wave(bucket, a, b, c, g, lane_streams, wave, rest);
  std::vector<int32_t> keep;
  int64_t bound8 = 0;
  t8->clear();
  for (int32_t id : *rest) {
    if (prefer_t8(b[size_t(id)], c[size_t(id)])) {
      t8->push_back(id);
      bound8 = std::max(bound8, lane_bound(scheme, a[size_t(id)], b[size_t(id)], c[size_t(id)], g, ta::kSmallTileN));
    } else {
      keep.push_back(id);
    }
  }
  rest->swap(keep);
  *lanes8 = s16_ok(scheme, bound8) ? 2 : 1;
}

// Wave launches of `ids` with tile side n: one block pair per resident CTA and
// round, rounds run one after another (plan_wave); smaller tiles make more
// blocks, so they pay only while they need no more rounds.
int64_t wave_rounds(const ta_batch* bt, const std::vector<int32_t>& ids, int grid, int n, int lanes) {
  int64_t blocks = 0;
  for (int32_t id : ids) {
    const Blocks bl = blocks_of(bt->b[size_t(id)], bt->c[size_t(id)], grid, n);
    blocks += int64_t(bl.bj) * bl.bk;
  }
  const int64_t per_round = int64_t(std::max(1, bt->ctx->sms)) * lanes;
  return (blocks + per_round - 1) / per_round;
}

// Tile side of score-only wave buckets: a wave step is latency bound per
// thread, so the 8 x 8 tiles (64 cells per tile-step instead of 100) shorten
// every step of a long triplet's critical path.  TA_WAVE_TILE=10 selects the
// 10 x 10 kernels (dev-only A/B knob).
int wave_tile_n() {
  static const int n = [] {
    const char* e = std::getenv("TA_WAVE_TILE");
    return e && std::atoi(e) == ta::kTileN ? ta::kTileN : ta::kSmallTileN;
  }();
  return n;
}

// Host planning + upload for one bucket (outside any timed region).
int prepare_bucket(ta_batch* bt, const std::vector<int32_t>& ids, int grid, int lanes, int mode,
                   bool trace, cudaStream_t st, BucketLaunch* bl, bool wave = false, int tile_n = ta::kTileN) {
  bl->grid = grid;
  bl->lanes = lanes;
  bl->mode = mode;
  bl->wave = wave;
  if (wave) {
    // the lane width was proven for 160-wide blocks: keep 8 x 8 tiles only
    // while no triplet's 128-padded extents exceed its 160-padded ones (the
    // value bound grows with them, lane_bound)
    for (int32_t id : ids) {
      if (tile_n == ta::kTileN) break;
      auto ext = [&](int n) {
        const int64_t gn = int64_t(grid) * n;
        return ((bt->b[size_t(id)] + gn) / gn + (bt->c[size_t(id)] + gn) / gn) * gn;
      };
      if (ext(tile_n) > ext(ta::kTileN)) tile_n = ta::kTileN;
    }
    if (tile_n != ta::kTileN && wave_rounds(bt, ids, grid, tile_n, lanes) > wave_rounds(bt, ids, grid, ta::kTileN, lanes))
      tile_n = ta::kTileN;
    // blocks that fit one per resident CTA run unpaired (plan_wave): the
    // int32-lane kernel then carries no idle partner lane
    static const bool lanes1 = [] {
      const char* e = std::getenv("TA_WAVE_LANES1");
      return !(e && std::atoi(e) == 0);
    }();
    if (lanes1 && lanes == 2 && wave_rounds(bt, ids, grid, tile_n, 1) <= 1) bl->lanes = lanes = 1;
    if (tile_n != ta::kTileN && (grid != 16 || trace))
      return fail(TA_ERR_LOGIC, "8 x 8-tile wave kernels exist for score items of grid 16 only");
    bl->ke = tile_n != ta::kTileN ? ta::kernel_g16_t8_wave(lanes, mode) : ta::lookup_kernel(grid, lanes, mode, trace, 2);
    const ta::KernelEntry& ke = bl->ke;
    if (!ke.fn) return fail(TA_ERR_LOGIC, "no wave kernel instantiation for grid " + std::to_string(grid));
    TA_CK(cudaFuncSetAttribute(ke.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ke.smem)));
    int per_sm = 0;
    TA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ke.fn, ke.threads, ke.smem));
    if (per_sm < 1) return fail(TA_ERR_CUDA, "wavefront kernel does not fit on an SM");
    WavePlan plan;
    int ctas = 0;
    plan_wave(ids, bt->a, bt->b, bt->c, per_sm * bt->ctx->sms, lanes, grid, int64_t(bt->a.size()), &plan, &ctas, tile_n);
    bl->ctas = ctas;
    bl->rounds = plan.rounds;
    TA_CK(bl->items.reserve(plan.items.size()));
    TA_CK(bl->soff.reserve(plan.soff.size()));
    TA_CK(bl->steps.reserve(plan.steps.size()));
    TA_CK(bl->faces.reserve(size_t(plan.entries) * 2 + 4));
    TA_CK(bl->wave_base.reserve(plan.base.size()));
    TA_CK(bl->face_off.reserve(1));
    bl->face_bytes = plan.entries * 8;
    TA_CK(cudaMemsetAsync(bl->faces.ptr, 0, size_t(bl->face_bytes), st));  // no stale tags
    bl->epoch = 0;
    TA_CK(cudaMemcpyAsync(bl->wave_base.ptr, plan.base.data(), plan.base.size() * 8, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bl->items.ptr, plan.items.data(), plan.items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bl->soff.ptr, plan.soff.data(), plan.soff.size() * 4, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bl->steps.ptr, plan.steps.data(), plan.steps.size() * 4, cudaMemcpyHostToDevice, st));
    bl->padded = plan.padded_slices * grid * grid * tile_n * tile_n;
    return TA_OK;
  }
  bool multi = false;
  for (int32_t id : ids) {
    const Blocks b = blocks_of(bt->b[size_t(id)], bt->c[size_t(id)], grid, tile_n);
    if (b.bj * b.bk > 1) {
      multi = true;
      break;
    }
  }
  if (tile_n != ta::kTileN && (grid != 16 || trace || !multi))
    return fail(TA_ERR_LOGIC, "8 x 8 tiles exist for multi-block score items of grid 16 only");
  bl->ke = tile_n != ta::kTileN ? ta::kernel_g16_t8(lanes, mode) : ta::lookup_kernel(grid, lanes, mode, trace, multi ? 1 : 0);
  const ta::KernelEntry& ke = bl->ke;
  if (!ke.fn) return fail(TA_ERR_LOGIC, "no kernel instantiation for grid " + std::to_string(grid));
  TA_CK(cudaFuncSetAttribute(ke.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ke.smem)));
  int per_sm = 0;
  TA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ke.fn, ke.threads, ke.smem));
  if (per_sm < 1) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, ke.fn);
    return fail(TA_ERR_CUDA, "wavefront kernel does not fit on an SM (grid " + std::to_string(grid) + ", " +
                                 std::to_string(ke.threads) + " threads, " + std::to_string(fa.numRegs) + " regs, " +
                                 std::to_string(ke.smem) + " B dynamic smem, max threads " +
                                 std::to_string(fa.maxThreadsPerBlock) + ")");
  }
  const int64_t want = (int64_t(ids.size()) + lanes - 1) / lanes;
  bl->ctas = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(per_sm) * bt->ctx->sms, want)));
  StreamPlan plan;
  plan_streams(ids, bt->a, bt->b, bt->c, bl->ctas, lanes, grid, &plan, tile_n);
  if (plan.face_words > (int64_t(1) << 31)) return fail(TA_ERR_CAPACITY, "block-face scratch exceeds 2^31 words");
  TA_CK(bl->items.reserve(plan.items.size()));
  TA_CK(bl->soff.reserve(plan.soff.size()));
  TA_CK(bl->steps.reserve(plan.steps.size()));
  TA_CK(bl->faces.reserve(size_t(plan.face_words) + 1));
  TA_CK(bl->face_off.reserve(plan.face_off.size()));
  TA_CK(cudaMemcpyAsync(bl->face_off.ptr, plan.face_off.data(), plan.face_off.size() * 8, cudaMemcpyHostToDevice, st));
  TA_CK(cudaMemcpyAsync(bl->items.ptr, plan.items.data(), plan.items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  TA_CK(cudaMemcpyAsync(bl->soff.ptr, plan.soff.data(), plan.soff.size() * 4, cudaMemcpyHostToDevice, st));
  TA_CK(cudaMemcpyAsync(bl->steps.ptr, plan.steps.data(), plan.steps.size() * 4, cudaMemcpyHostToDevice, st));
  bl->padded = plan.padded_slices * grid * grid * tile_n * tile_n;
  return TA_OK;
}

int launch_prepared(BucketLaunch* bl, const ta::WaveArgs& base, cudaStream_t st, int64_t* launches) {
  ta::WaveArgs args = base;
  args.items = bl->items.ptr;
  args.stream_off = bl->soff.ptr;
  args.cta_steps = bl->steps.ptr;
  args.faces = bl->faces.ptr;
  args.face_off = bl->face_off.ptr;
  if (bl->wave) {
    if (++bl->epoch >= 65536u) {  // tags would repeat: clear the rings
      TA_CK(cudaMemsetAsync(bl->faces.ptr, 0, size_t(bl->face_bytes), st));
      bl->epoch = 1;
    }
    args.wave_base = bl->wave_base.ptr;
    args.epoch = bl->epoch;
    for (const WaveRound& rd : bl->rounds) {
      ta::WaveArgs ra = args;
      ra.stream_off = bl->soff.ptr + rd.soff_at;
      ra.cta_steps = bl->steps.ptr + rd.steps_at;
      // CTAs of a wave round wait on each other's faces: the cooperative
      // launch guarantees they are co-resident (or fails loudly), whatever
      // else runs on the device
      void* kargs[] = {&ra};
      TA_CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(bl->ke.fn), dim3(rd.ctas), dim3(bl->ke.threads),
                                        kargs, bl->ke.smem, st));
      *launches += 1;
    }
    return TA_OK;
  }
  bl->ke.fn<<<bl->ctas, bl->ke.threads, bl->ke.smem, st>>>(args);
  TA_CK(cudaGetLastError());
  *launches += 1;
  return TA_OK;
}

// One launch plan per call from the batch's pool (grow-only buffers).
BucketLaunch* rows_plan(ta_batch* bt, size_t* used) {
  if (*used == bt->rows_pool.size()) bt->rows_pool.push_back(std::make_unique<BucketLaunch>());
  BucketLaunch* bl = bt->rows_pool[(*used)++].get();
  bl->wave = false;
  bl->rounds.clear();
  return bl;
}

int launch_bucket(ta_batch* bt, const std::vector<int32_t>& ids, int grid, int lanes, int mode,
                  bool trace, const ta::WaveArgs& base, cudaStream_t st, int64_t* launches, size_t* used) {
  // few long triplets of the largest grid run in wave mode (their blocks
  // spread over all CTAs, direction records in the same layout), the rest
  // as sequential block items of one stream
  std::vector<int32_t> wave, rest;
  if (grid == ta::kGridSizes[ta::kNumGrid - 1]) {
    split_wave(ids, bt->a, bt->b, bt->c, grid, bt->ctx->sms * lanes, &wave, &rest);
  } else {
    rest = ids;
  }
  for (int w = 0; w < 2; ++w) {
    const std::vector<int32_t>& part = w ? wave : rest;
    if (part.empty()) continue;
    BucketLaunch* bl = rows_plan(bt, used);
    if (int rc = prepare_bucket(bt, part, grid, lanes, mode, trace, st, bl, w == 1)) return rc;
    if (int rc = launch_prepared(bl, base, st, launches)) return rc;
    bt->stats.padded_cells += bl->padded;
  }
  return TA_OK;
}

// ---------------------------------------------------------------------------
// Affine path (SPEC-AFFINE.md): one 16 x 16 grid of 5 x 5 tiles; triplets
// wider than 80 cells run as block items (faces of 4 values per position).

// Largest biased, gap-shifted value: -8 open + (match - 2 gap) * (slices + extents).
int64_t aff_lane_bound(const ta_scheme& s, int32_t a, int32_t b, int32_t c, int tile_n = ta::kAffN) {
  const int g2 = 2 * s.gap;
  const int64_t gn = int64_t(ta::kAffG) * tile_n;
  const int64_t ej = ((b + 1 + gn - 1) / gn) * gn, ek = ((c + 1 + gn - 1) / gn) * gn;
  const int warps = (ta::kAffG * ta::kAffG + 31) / 32;
  const int64_t slices = std::max<int64_t>(a + 1, ta::kAffG + 2 + warps);
  return -10 * int64_t(s.gap_open) + int64_t(s.match - g2) * (slices + ej + ek);
}

bool aff_s16_ok(const ta_scheme& s, int64_t max_bound) {
  const int g2 = 2 * s.gap;
  const int mp = s.match - g2, mm = s.mismatch - g2;
  if (mm < 0 || mp > 127) return false;
  return max_bound + 3 * 127 + int64_t(-g2) * 2 * ta::kAffN + 2 * int64_t(-s.gap_open) <= 32000;
}

// Block items that pad less in 64-wide blocks (4 x 4 tiles) than in 80-wide
// ones, weighting a 64-block cell by the per-cell cost ratio of the kernels.
// Example: 250 bp (extent 251) = 4 x 4 blocks either way: 65536 vs 102400.
bool prefer_aff4(int32_t b, int32_t c) {
  static const double ratio = [] {
    const char* e = std::getenv("TA_AFF4_COST");
    return e ? std::atof(e) : 1.3;
  }();
  const Blocks b5 = blocks_of(b, c, ta::kAffG, ta::kAffN);
  const Blocks b4 = blocks_of(b, c, ta::kAffG, ta::kAffSmallN);
  const double g5 = double(ta::kAffG) * ta::kAffN, g4 = double(ta::kAffG) * ta::kAffSmallN;
  return double(b4.bj * b4.bk) * g4 * g4 * ratio < double(b5.bj * b5.bk) * g5 * g5;
}

// Tile side of affine score-only wave buckets (see wave_tile_n): 4 x 4 tiles,
// TA_AFF_WAVE_TILE=5 selects the 5 x 5 kernels (dev-only A/B knob).
int aff_wave_tile_n() {
  static const int n = [] {
    const char* e = std::getenv("TA_AFF_WAVE_TILE");
    return e && std::atoi(e) == ta::kAffN ? ta::kAffN : ta::kAffSmallN;
  }();
  return n;
}

int aff_prepare(ta_batch* bt, const std::vector<int32_t>& ids, int lanes, int mode, bool trace, int blk,
                cudaStream_t st, BucketLaunch* bl, ta::AffEntry* ae, int tile_n = ta::kAffN) {
  if (blk == 2) {
    // the lane width was proven for 80-wide blocks: keep 4 x 4 tiles only while
    // no triplet's 64-padded extents exceed its 80-padded ones (aff_lane_bound)
    for (int32_t id : ids) {
      if (tile_n == ta::kAffN) break;
      auto ext = [&](int n) {
        const int64_t gn = int64_t(ta::kAffG) * n;
        return ((bt->b[size_t(id)] + gn) / gn + (bt->c[size_t(id)] + gn) / gn) * gn;
      };
      if (ext(tile_n) > ext(ta::kAffN)) tile_n = ta::kAffN;
    }
    if (tile_n != ta::kAffN && wave_rounds(bt, ids, ta::kAffG, tile_n, lanes) > wave_rounds(bt, ids, ta::kAffG, ta::kAffN, lanes))
      tile_n = ta::kAffN;
  }
  if (tile_n != ta::kAffN && (blk == 0 || trace))
    return fail(TA_ERR_LOGIC, "4 x 4 affine tiles exist for block / wave score items only");
  *ae = tile_n == ta::kAffN ? ta::lookup_affine(lanes, mode, trace, blk)
        : blk == 2          ? ta::affine_kernel_wave4(lanes, mode)
                            : ta::affine_kernel_blocks4(lanes, mode);
  if (!ae->fn) return fail(TA_ERR_LOGIC, "no affine kernel instantiation");
  TA_CK(cudaFuncSetAttribute(ae->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ae->smem)));
  int per_sm = 0;
  TA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ae->fn, ae->threads, ae->smem));
  if (per_sm < 1) return fail(TA_ERR_CUDA, "affine kernel does not fit on an SM");
  bl->wave = blk == 2;
  bl->rounds.clear();
  if (blk == 2) {  // wave mode: blocks spread over all CTAs, tagged rings (see plan_wave)
    WavePlan plan;
    int ctas = 0;
    plan_wave(ids, bt->a, bt->b, bt->c, per_sm * bt->ctx->sms, lanes, ta::kAffG, int64_t(bt->a.size()), &plan, &ctas,
              tile_n, true);
    bl->grid = ta::kAffG;
    bl->lanes = lanes;
    bl->mode = mode;
    bl->ctas = ctas;
    bl->rounds = plan.rounds;
    TA_CK(bl->items.reserve(plan.items.size()));
    TA_CK(bl->soff.reserve(plan.soff.size()));
    TA_CK(bl->steps.reserve(plan.steps.size()));
    TA_CK(bl->faces.reserve(size_t(plan.entries) * 2 + 4));
    TA_CK(bl->wave_base.reserve(plan.base.size()));
    TA_CK(bl->face_off.reserve(1));
    bl->face_bytes = plan.entries * 8;
    TA_CK(cudaMemsetAsync(bl->faces.ptr, 0, size_t(bl->face_bytes), st));
    bl->epoch = 0;
    TA_CK(cudaMemcpyAsync(bl->wave_base.ptr, plan.base.data(), plan.base.size() * 8, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bl->items.ptr, plan.items.data(), plan.items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bl->soff.ptr, plan.soff.data(), plan.soff.size() * 4, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bl->steps.ptr, plan.steps.data(), plan.steps.size() * 4, cudaMemcpyHostToDevice, st));
    bl->padded = plan.padded_slices * ta::kAffG * ta::kAffG * tile_n * tile_n;
    return TA_OK;
  }
  const int64_t want = (int64_t(ids.size()) + lanes - 1) / lanes;
  bl->grid = ta::kAffG;
  bl->lanes = lanes;
  bl->mode = mode;
  bl->ctas = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(per_sm) * bt->ctx->sms, want)));
  StreamPlan plan;
  plan_streams(ids, bt->a, bt->b, bt->c, bl->ctas, lanes, ta::kAffG, &plan, tile_n, true);
  if (plan.face_words > (int64_t(1) << 31)) return fail(TA_ERR_CAPACITY, "block-face scratch exceeds 2^31 words");
  TA_CK(bl->items.reserve(plan.items.size()));
  TA_CK(bl->soff.reserve(plan.soff.size()));
  TA_CK(bl->steps.reserve(plan.steps.size()));
  TA_CK(bl->faces.reserve(size_t(plan.face_words) + 4));
  TA_CK(bl->face_off.reserve(plan.face_off.size()));
  TA_CK(cudaMemcpyAsync(bl->face_off.ptr, plan.face_off.data(), plan.face_off.size() * 8, cudaMemcpyHostToDevice, st));
  TA_CK(cudaMemcpyAsync(bl->items.ptr, plan.items.data(), plan.items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  TA_CK(cudaMemcpyAsync(bl->soff.ptr, plan.soff.data(), plan.soff.size() * 4, cudaMemcpyHostToDevice, st));
  TA_CK(cudaMemcpyAsync(bl->steps.ptr, plan.steps.data(), plan.steps.size() * 4, cudaMemcpyHostToDevice, st));
  bl->padded = plan.padded_slices * ta::kAffG * ta::kAffG * tile_n * tile_n;
  return TA_OK;
}

int aff_launch(BucketLaunch* bl, const ta::AffEntry& ae, const ta::AffArgs& base, cudaStream_t st,
               int64_t* launches) {
  ta::AffArgs args = base;
  args.items = bl->items.ptr;
  args.stream_off = bl->soff.ptr;
  args.cta_steps = bl->steps.ptr;
  args.faces = bl->faces.ptr;
  args.face_off = bl->face_off.ptr;
  if (bl->wave) {
    if (++bl->epoch >= 65536u) {  // tags would repeat: clear the rings
      TA_CK(cudaMemsetAsync(bl->faces.ptr, 0, size_t(bl->face_bytes), st));
      bl->epoch = 1;
    }
    args.face_off = bl->wave_base.ptr;  // wave: ring base per triplet (AffArgs)
    if (args.dirs) {
      // TRACE (dir_off shares the epoch's slot): the kernel tags with epoch 1,
      // so a traceback plan is launched once, on rings zeroed by aff_prepare
      if (bl->epoch != 1) return fail(TA_ERR_LOGIC, "affine traceback wave plan launched twice");
    } else {
      args.epoch = bl->epoch;
    }
    for (const WaveRound& rd : bl->rounds) {
      ta::AffArgs ra = args;
      ra.stream_off = bl->soff.ptr + rd.soff_at;
      ra.cta_steps = bl->steps.ptr + rd.steps_at;
      void* kargs[] = {&ra};  // co-resident CTAs (see launch_prepared)
      TA_CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(ae.fn), dim3(rd.ctas), dim3(ae.threads), kargs,
                                        ae.smem, st));
      *launches += 1;
    }
    return TA_OK;
  }
  ae.fn<<<bl->ctas, ae.threads, ae.smem, st>>>(args);
  TA_CK(cudaGetLastError());
  *launches += 1;
  return TA_OK;
}

int run_affine(ta_batch* bt, const ta_scheme& scheme, const ta_options& opt, cudaStream_t st,
               const std::vector<int32_t>& all_ok, bool rows) {
  NvtxRange nv(rows ? "ta/affine_rows" : "ta/affine");
  const int64_t n = bt->n;
  std::vector<int32_t> single, multi, wave;
  int64_t maxb = 0;
  for (int32_t id : all_ok) {
    const int32_t B = bt->b[size_t(id)], C = bt->c[size_t(id)];
    (std::max(B, C) + 1 <= ta::kAffExtent ? single : multi).push_back(id);
    maxb = std::max(maxb, aff_lane_bound(scheme, bt->a[size_t(id)], B, C));
  }
  const int lanes = (!rows && aff_s16_ok(scheme, maxb)) ? 2 : 1;
  // few long triplets: spread their blocks over all CTAs (wave mode)
  if (!multi.empty() && int64_t(multi.size()) * 2 <= int64_t(bt->ctx->sms) * lanes) {
    bool ok = true;
    for (int32_t id : multi) ok &= bt->a[size_t(id)] + 1 < 65535;
    if (ok) wave.swap(multi);
  }
  // block items that pad less in 64-wide blocks (score path), own lane choice
  std::vector<int32_t> multi4;
  int lanes4 = 1;
  if (!rows && !multi.empty()) {
    std::vector<int32_t> keep;
    int64_t maxb4 = 0;
    for (int32_t id : multi) {
      const int32_t B = bt->b[size_t(id)], C = bt->c[size_t(id)];
      if (prefer_aff4(B, C)) {
        multi4.push_back(id);
        maxb4 = std::max(maxb4, aff_lane_bound(scheme, bt->a[size_t(id)], B, C, ta::kAffSmallN));
      } else {
        keep.push_back(id);
      }
    }
    multi.swap(keep);
    lanes4 = aff_s16_ok(scheme, maxb4) ? 2 : 1;
  }
  ta::AffArgs base{};
  base.seq = bt->seq.ptr;
  base.desc = bt->d_desc.ptr;
  base.out_score = bt->d_score.ptr;
  base.out_end = bt->d_end.ptr;
  base.out_key = bt->d_key.ptr;
  base.g2 = 2 * scheme.gap;
  base.match_p = scheme.match - base.g2;
  base.mismatch_p = scheme.mismatch - base.g2;
  base.open = scheme.gap_open;
  base.bias = -10 * scheme.gap_open;
  base.one = 1u;
  if (!bt->ev0) TA_CK(cudaEventCreate(&bt->ev0));
  if (!bt->ev1) TA_CK(cudaEventCreate(&bt->ev1));
  if (opt.mode != TA_GLOBAL) TA_CK(cudaMemsetAsync(bt->d_key.ptr, 0, size_t(n) * 8, st));
  int64_t launches = 0;
  int nbuckets = 0;
  float ms = 0.f;
  auto decode = [&](const std::vector<int32_t>& ids) -> int {
    if (opt.mode == TA_GLOBAL || ids.empty()) return TA_OK;
    TA_CK(bt->d_ids.reserve(ids.size()));
    TA_CK(cudaMemcpyAsync(bt->d_ids.ptr, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, st));
    const int64_t m = int64_t(ids.size());
    decode_keys_kernel<<<unsigned((m + 255) / 256), 256, 0, st>>>(bt->d_key.ptr, bt->d_desc.ptr, bt->d_ids.ptr, m,
                                                                bt->d_score.ptr, bt->d_end.ptr);
    TA_CK(cudaGetLastError());
    ++launches;
    return TA_OK;
  };
  if (!rows) {
    std::string key = "aff:" + std::to_string(opt.mode) + ":" + std::to_string(lanes) + ":" +
                      std::to_string(scheme.gap_open) + ":" + std::to_string(all_ok.size()) + ":" +
                      std::to_string(multi4.size()) + ":" + std::to_string(lanes4);
    uint64_t h = 1469598103934665603ull;
    for (int32_t id : all_ok) h = (h ^ uint64_t(id)) * 1099511628211ull;
    key += ":" + std::to_string(h);
    if (key != bt->plan_key) {
      bt->plan_cache.clear();
      bt->aff_cache.clear();
      bt->plan_key.clear();
      for (int w = 0; w < 4; ++w) {
        const std::vector<int32_t>& part = w == 3 ? multi4 : w == 2 ? wave : w ? multi : single;
        if (part.empty()) continue;
        bt->plan_cache.push_back(std::make_unique<BucketLaunch>());
        bt->aff_cache.emplace_back();
        if (int rc = aff_prepare(bt, part, w == 3 ? lanes4 : lanes, opt.mode, false, w == 3 ? 1 : w, st,
                                 bt->plan_cache.back().get(), &bt->aff_cache.back(),
                                 w == 3 ? ta::kAffSmallN : w == 2 ? aff_wave_tile_n() : ta::kAffN))
          return rc;
      }
      bt->plan_key = key;
    }
    if (opt.mode != TA_GLOBAL && !all_ok.empty()) {
      TA_CK(bt->d_ids.reserve(all_ok.size()));
      TA_CK(cudaMemcpyAsync(bt->d_ids.ptr, all_ok.data(), all_ok.size() * 4, cudaMemcpyHostToDevice, st));
    }
    TA_CK(cudaEventRecord(bt->ev0, st));
    for (size_t x = 0; x < bt->plan_cache.size(); ++x) {
      if (int rc = aff_launch(bt->plan_cache[x].get(), bt->aff_cache[x], base, st, &launches)) return rc;
      bt->stats.padded_cells += bt->plan_cache[x]->padded;
      ++nbuckets;
    }
    if (opt.mode != TA_GLOBAL && !all_ok.empty()) {
      const int64_t m = int64_t(all_ok.size());
      decode_keys_kernel<<<unsigned((m + 255) / 256), 256, 0, st>>>(bt->d_key.ptr, bt->d_desc.ptr, bt->d_ids.ptr, m,
                                                                  bt->d_score.ptr, bt->d_end.ptr);
      TA_CK(cudaGetLastError());
      ++launches;
    }
    TA_CK(cudaEventRecord(bt->ev1, st));
    TA_CK(cudaEventSynchronize(bt->ev1));
    TA_CK(cudaEventElapsedTime(&ms, bt->ev0, bt->ev1));
  } else {
    // records: (a+1) * blocks * T tile-slices of kAffRec words per triplet, chunked by free HBM
    size_t free_b = 0, total_b = 0;
    TA_CK(cudaMemGetInfo(&free_b, &total_b));
    const size_t budget = std::max<size_t>(size_t(1) << 28, size_t(double(free_b + bt->d_dirs.cap * 16) * 0.5));
    size_t pool_used = 0;
    bt->plan_key.clear();
    TA_CK(cudaEventRecord(bt->ev0, st));
    for (int w = 0; w < 3; ++w) {
      const std::vector<int32_t>& ids = w == 2 ? wave : w ? multi : single;
      if (ids.empty()) continue;
      ++nbuckets;
      size_t pos = 0;
      while (pos < ids.size()) {
        std::vector<int32_t> chunk;
        std::vector<int64_t> diroff(static_cast<size_t>(n), 0);
        size_t used = 0;  // uint4 units
        while (pos < ids.size()) {
          const int32_t id = ids[pos];
          const Blocks blk = blocks_of(bt->b[size_t(id)], bt->c[size_t(id)], ta::kAffG, ta::kAffN);
          const size_t need = size_t(blk.bj) * blk.bk * size_t(bt->a[size_t(id)] + 1) * ta::kAffG * ta::kAffG *
                              (ta::kAffRec / 4);
          if (!chunk.empty() && (used + need) * 16 > budget) break;
          diroff[size_t(id)] = int64_t(used);
          used += need;
          chunk.push_back(id);
          ++pos;
        }
        TA_CK(bt->d_dirs.reserve(used));
        TA_CK(bt->d_diroff.reserve(size_t(n)));
        TA_CK(cudaMemcpyAsync(bt->d_diroff.ptr, diroff.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
        ta::AffArgs args = base;
        args.dirs = reinterpret_cast<uint32_t*>(bt->d_dirs.ptr);
        args.dir_off = bt->d_diroff.ptr;
        BucketLaunch* bl = rows_plan(bt, &pool_used);
        ta::AffEntry ae;
        if (int rc = aff_prepare(bt, chunk, 1, opt.mode, true, w, st, bl, &ae)) return rc;
        if (int rc = aff_launch(bl, ae, args, st, &launches)) return rc;
        bt->stats.padded_cells += bl->padded;
        if (int rc = decode(chunk)) return rc;
        TA_CK(bt->d_ids.reserve(chunk.size()));
        TA_CK(cudaMemcpyAsync(bt->d_ids.ptr, chunk.data(), chunk.size() * 4, cudaMemcpyHostToDevice, st));
        const int m = int(chunk.size());
        affine_walker_kernel<<<unsigned((m + 127) / 128), 128, 0, st>>>(
            bt->d_desc.ptr, bt->seq.ptr, bt->d_ids.ptr, m, reinterpret_cast<const uint32_t*>(bt->d_dirs.ptr),
            bt->d_diroff.ptr, opt.mode, bt->d_end.ptr, bt->d_begin.ptr, bt->d_rows.ptr, bt->d_rowoff.ptr,
            bt->d_rowlen.ptr, bt->d_status.ptr);
        TA_CK(cudaGetLastError());
        ++launches;
        TA_CK(cudaStreamSynchronize(st));  // bl's buffers die here
      }
    }
    TA_CK(cudaEventRecord(bt->ev1, st));
    TA_CK(cudaEventSynchronize(bt->ev1));
    TA_CK(cudaEventElapsedTime(&ms, bt->ev0, bt->ev1));
  }
  int64_t cells = 0;
  for (int32_t id : all_ok) cells += int64_t(bt->a[size_t(id)]) * bt->b[size_t(id)] * bt->c[size_t(id)];
  bt->stats.kernel_ms = ms;
  bt->stats.wavefront_ms = ms;
  bt->stats.cells = cells;
  bt->stats.launches = launches;
  bt->stats.lanes = lanes;
  bt->stats.buckets = nbuckets;
  bt->last_mode = opt.mode;
  bt->last_rows = rows;
  return TA_OK;
}

int run_impl(ta_batch* bt, const ta_scheme& scheme, const ta_options& opt, cudaStream_t st,
             ta_results* rows_out) {
  NvtxRange nv(opt.with_rows ? "ta/run_rows" : "ta/run");
  const int64_t n = bt->n;
  bt->stats = ta_stats{};
  const bool rows = opt.with_rows != 0;
  if (int rc = validate_scheme(scheme)) return rc;
  if (opt.mode < 0 || opt.mode > 2) return fail(TA_ERR_INVALID_ARGUMENT, "unknown alignment mode");
  // Per-triplet engine errors, exactly where the reference raises them:
  // EngineConfig::validate + make_layout (tiled.cpp:8-15, 37-58) on the
  // score path, the tensor budget (oracle.cpp:16-20) on the rows path.
  const int cfg_rc = rows ? TA_OK : validate_options(opt);
  const std::string cfg_msg = cfg_rc ? g_err : std::string();
  std::vector<std::vector<int32_t>> buckets(ta::kNumGrid);
  std::vector<int32_t> all_ok;
  int64_t max_bound_bucket[ta::kNumGrid] = {0};
  const bool front_ok = !rows && !cfg_rc && scheme.gap_open == 0 && opt.gap_model != 1;
  std::string fkey;
  if (front_ok) {
    fkey = std::to_string(scheme.match) + "," + std::to_string(scheme.mismatch) + "," + std::to_string(scheme.gap) +
           "|" + std::to_string(opt.mode) + "," + std::to_string(opt.tile_size) + "," +
           std::to_string(opt.team_width) + "," + std::to_string(opt.team_threads) + "," +
           std::to_string(opt.lane_mode) + "," + std::to_string(opt.cell_budget);
  }
  const bool front_hit = front_ok && fkey == bt->front_key && !bt->plan_key.empty();
  if (!front_hit) bt->front_key.clear();
  if (front_hit) {
    // a repeated run: status and the valid ids are the cached ones (status is
    // copied back only if another run changed it since)
    if (!bt->status_is_front) bt->status = bt->front_status;
  } else {
  bt->status_is_front = false;
  bt->status = bt->pre_status;
  all_ok.reserve(size_t(n));
  for (int64_t t = 0; t < n; ++t) {
    if (bt->status[size_t(t)] != TA_OK) continue;
    const int32_t A = bt->a[size_t(t)], B = bt->b[size_t(t)], C = bt->c[size_t(t)];
    if (!rows) {
      if (cfg_rc) {
        bt->status[size_t(t)] = cfg_rc;
        continue;
      }
      const uint64_t cells = uint64_t(A) * uint64_t(B) * uint64_t(C);
      if (cells > opt.cell_budget) {
        bt->status[size_t(t)] = TA_ERR_CAPACITY;
        continue;
      }
      const int32_t width = opt.team_width > 0 ? opt.team_width : derive_team_width(opt.tile_size, B, C);
      if (int64_t(width) * opt.tile_size < std::max(B, C)) {
        bt->status[size_t(t)] = TA_ERR_CONFIG;
        continue;
      }
    } else {
      const uint64_t total = uint64_t(A + 1) * uint64_t(B + 1) * uint64_t(C + 1);
      if (total > opt.cell_budget) {
        bt->status[size_t(t)] = TA_ERR_CAPACITY;
        continue;
      }
    }
    if (opt.mode != TA_GLOBAL && !key_fits(A, B, C, scheme)) {
      bt->status[size_t(t)] = TA_ERR_CAPACITY;
      continue;
    }
    const int g = pick_grid(B, C);
    int gi = 0;
    while (ta::kGridSizes[gi] != g) ++gi;
    buckets[size_t(gi)].push_back(int32_t(t));
    max_bound_bucket[gi] = std::max(max_bound_bucket[gi], lane_bound(scheme, A, B, C, g));
    all_ok.push_back(int32_t(t));
  }
  }
  if (cfg_rc) g_err = cfg_msg;
  if (scheme.gap_open != 0 || opt.gap_model == 1) return run_affine(bt, scheme, opt, st, all_ok, rows);

  ta::WaveArgs base{};
  base.seq = bt->seq.ptr;
  base.desc = bt->d_desc.ptr;
  base.out_score = bt->d_score.ptr;
  base.out_end = bt->d_end.ptr;
  base.out_key = bt->d_key.ptr;
  base.g2 = 2 * scheme.gap;
  base.match_p = scheme.match - base.g2;
  base.mismatch_p = scheme.mismatch - base.g2;
  base.one = 1u;

  if (!bt->ev0) TA_CK(cudaEventCreate(&bt->ev0));
  if (!bt->ev1) TA_CK(cudaEventCreate(&bt->ev1));
  if (opt.mode != TA_GLOBAL) TA_CK(cudaMemsetAsync(bt->d_key.ptr, 0, size_t(n) * 8, st));

  int64_t launches = 0;
  int lanes_used = 1;
  int nbuckets = 0;
  float ms_total = 0.f;
  if (!rows) {
    // plan key: mode + per-bucket (grid, lanes, ids) fingerprint
    std::string key = std::to_string(opt.mode);
    std::vector<int> lanes_of(ta::kNumGrid, 1);
    if (!front_hit) {
    // largest grid: wave triplets, 128-wide-block triplets (prefer_t8), the rest
    const int gl = ta::kNumGrid - 1;
    std::vector<int32_t> wave_ids, rest_ids, t8_ids;
    int lanes8 = 1;
    if (!buckets[size_t(gl)].empty()) {
      const int l = s16_ok(scheme, max_bound_bucket[gl]) ? 2 : 1;
      split_largest(buckets[size_t(gl)], bt->a, bt->b, bt->c, scheme, bt->ctx->sms * l, &wave_ids, &rest_ids, &t8_ids,
                    &lanes8);
      key += "|t8:" + std::to_string(t8_ids.size()) + ":" + std::to_string(lanes8);
    }
    for (int gi = 0; gi < ta::kNumGrid; ++gi) {
      if (buckets[size_t(gi)].empty()) continue;
      lanes_of[size_t(gi)] = s16_ok(scheme, max_bound_bucket[gi]) ? 2 : 1;
      uint64_t h = 1469598103934665603ull;
      for (int32_t id : buckets[size_t(gi)]) h = (h ^ uint64_t(id)) * 1099511628211ull;
      key += "|" + std::to_string(ta::kGridSizes[gi]) + ":" + std::to_string(lanes_of[size_t(gi)]) + ":" +
             std::to_string(buckets[size_t(gi)].size()) + ":" + std::to_string(h);
    }
    if (key != bt->plan_key) {
      bt->plan_cache.clear();
      bt->plan_key.clear();
      for (int gi = 0; gi < ta::kNumGrid; ++gi) {
        if (buckets[size_t(gi)].empty()) continue;
        if (gi != gl) {
          bt->plan_cache.push_back(std::make_unique<BucketLaunch>());
          if (int rc = prepare_bucket(bt, buckets[size_t(gi)], ta::kGridSizes[gi], lanes_of[size_t(gi)], opt.mode,
                                      false, st, bt->plan_cache.back().get()))
            return rc;
          continue;
        }
        for (int w = 0; w < 3; ++w) {
          const std::vector<int32_t>& part = w == 2 ? t8_ids : w ? wave_ids : rest_ids;
          if (part.empty()) continue;
          bt->plan_cache.push_back(std::make_unique<BucketLaunch>());
          if (int rc = prepare_bucket(bt, part, ta::kGridSizes[gi], w == 2 ? lanes8 : lanes_of[size_t(gi)], opt.mode,
                                      false, st, bt->plan_cache.back().get(), w == 1,
                                      w == 2 ? ta::kSmallTileN : w == 1 ? wave_tile_n() : ta::kTileN))
            return rc;
        }
      }
      bt->plan_key = key;
    }
    }  // !front_hit
    for (auto& bl : bt->plan_cache) {
      lanes_used = std::max(lanes_used, bl->lanes);
      ++nbuckets;
    }
    const std::vector<int32_t>& ok_ids = front_hit ? bt->front_all_ok : all_ok;
    if (opt.mode != TA_GLOBAL && !ok_ids.empty()) {
      TA_CK(bt->d_ids.reserve(ok_ids.size()));
      TA_CK(cudaMemcpyAsync(bt->d_ids.ptr, ok_ids.data(), ok_ids.size() * 4, cudaMemcpyHostToDevice, st));
    }
    TA_CK(cudaEventRecord(bt->ev0, st));
    for (auto& bl : bt->plan_cache) {
      if (int rc = launch_prepared(bl.get(), base, st, &launches)) return rc;
      bt->stats.padded_cells += bl->padded;
    }
    if (opt.mode != TA_GLOBAL && !ok_ids.empty()) {
      const int64_t m = int64_t(ok_ids.size());
      decode_keys_kernel<<<unsigned((m + 255) / 256), 256, 0, st>>>(bt->d_key.ptr, bt->d_desc.ptr, bt->d_ids.ptr, m,
                                                                  bt->d_score.ptr, bt->d_end.ptr);
      TA_CK(cudaGetLastError());
      ++launches;
    }
    TA_CK(cudaEventRecord(bt->ev1, st));
    TA_CK(cudaEventSynchronize(bt->ev1));
    TA_CK(cudaEventElapsedTime(&ms_total, bt->ev0, bt->ev1));
  } else {
    // Direction-record chunks: (a+1) * G^2 tile-slices of 40 B per triplet,
    // sized to half the free HBM and - when rows go back to a host caller -
    // to at most 1/8 of the batch, so the D2H of chunk k's rows and their
    // scatter into the caller's row planes overlap chunk k+1's kernels.  All
    // chunk plans are made up front (one upload of record offsets, ids and
    // row offsets); chunks run back to back on the stream.
    size_t free_b = 0, total_b = 0;
    TA_CK(cudaMemGetInfo(&free_b, &total_b));
    const size_t budget = std::max<size_t>(size_t(1) << 28, size_t(double(free_b + bt->d_dirs.cap * 16) * 0.5));
    const bool scatter = rows_out && rows_out->rows0 && rows_out->rows1 && rows_out->rows2 && rows_out->row_offsets;
    const size_t pipe_max = scatter ? std::max<size_t>(4096, (all_ok.size() + 7) / 8) : SIZE_MAX;
    struct Chunk {
      int g;
      size_t lo, hi;
      int lanes;
      int64_t rlo, rhi;  // device row bytes of the chunk
    };
    std::vector<Chunk> chunks;
    std::vector<int32_t> order;
    order.reserve(all_ok.size());
    std::vector<int64_t> diroff(static_cast<size_t>(n), 0), roff(static_cast<size_t>(n), 0);
    size_t max_used = 0;
    int64_t rtot = 0, max_rbytes = 0;
    size_t max_chunk = 0;
    for (int gi = 0; gi < ta::kNumGrid; ++gi) {
      const std::vector<int32_t>& ids = buckets[size_t(gi)];
      if (ids.empty()) continue;
      ++nbuckets;
      const int g = ta::kGridSizes[gi];
      size_t pos = 0;
      while (pos < ids.size()) {
        const size_t lo = order.size();
        const int64_t rlo = rtot;
        size_t used = 0;  // 32-bit words
        while (pos < ids.size() && order.size() - lo < pipe_max) {
          const int32_t id = ids[pos];
          const Blocks blk = blocks_of(bt->b[size_t(id)], bt->c[size_t(id)], g);
          const size_t need = size_t(blk.bj) * blk.bk * size_t(bt->a[size_t(id)] + 1) * size_t(g) * g * ta::kDirWords;
          if (order.size() > lo && (used + need) * 4 > budget) break;
          diroff[size_t(id)] = int64_t(used);
          used += need;
          roff[size_t(id)] = rtot;
          rtot += 3 * (int64_t(bt->a[size_t(id)]) + bt->b[size_t(id)] + bt->c[size_t(id)]);
          order.push_back(id);
          ++pos;
        }
        chunks.push_back(Chunk{g, lo, order.size(), trace16_ok(scheme, max_bound_bucket[gi]) ? 2 : 1, rlo, rtot});
        max_used = std::max(max_used, used);
        max_rbytes = std::max(max_rbytes, rtot - rlo);
        max_chunk = std::max(max_chunk, order.size() - lo);
        bt->stats.dir_bytes += int64_t(used) * 4;
      }
    }
    TA_CK(bt->d_dirs.reserve(max_used / 4 + 1));
    TA_CK(bt->d_diroff.reserve(size_t(n) + 1));
    TA_CK(bt->d_ids.reserve(order.size() + 1));
    TA_CK(bt->d_lenord.reserve(order.size() + 1));
    TA_CK(bt->d_rows.reserve(size_t(rtot) + 1));
    TA_CK(bt->d_rowoff.reserve(size_t(n) + 1));
    if (!bt->evw0) TA_CK(cudaEventCreate(&bt->evw0));
    if (!bt->evw1) TA_CK(cudaEventCreate(&bt->evw1));
    for (int k = 0; k < 2; ++k) {
      if (!bt->evk[k]) TA_CK(cudaEventCreateWithFlags(&bt->evk[k], cudaEventDisableTiming));
      if (!bt->evc[k]) TA_CK(cudaEventCreateWithFlags(&bt->evc[k], cudaEventDisableTiming));
    }
    DeviceCtx* ctx = bt->ctx;
    if (scatter) {
      for (int k = 0; k < 2 && chunks.size() > size_t(k); ++k) {
        TA_CK(ctx->h_rows[k].reserve(size_t(max_rbytes) + 1));
        TA_CK(ctx->h_len[k].reserve(max_chunk + 1));
      }
    }
    if (n) {
      TA_CK(cudaMemcpyAsync(bt->d_diroff.ptr, diroff.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
      TA_CK(cudaMemcpyAsync(bt->d_rowoff.ptr, roff.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
    }
    if (!order.empty())
      TA_CK(cudaMemcpyAsync(bt->d_ids.ptr, order.data(), order.size() * 4, cudaMemcpyHostToDevice, st));
    // host side of the pipeline: copy chunk c's rows out of its staging slot
    auto scatter_chunk = [&](size_t c) -> int {
      const Chunk& ch = chunks[c];
      TA_CK(cudaEventSynchronize(bt->evc[c & 1]));
      const char* src = ctx->h_rows[c & 1].ptr;
      const int32_t* len = ctx->h_len[c & 1].ptr;
      auto copy_range = [&](size_t x0, size_t x1) {
        for (size_t x = x0; x < x1; ++x) {
          const int32_t id = order[ch.lo + x];
          const int64_t cap = int64_t(bt->a[size_t(id)]) + bt->b[size_t(id)] + bt->c[size_t(id)];
          const char* r = src + (roff[size_t(id)] - ch.rlo);
          const int64_t o = rows_out->row_offsets[id];
          const size_t L = size_t(len[x]);
          std::memcpy(rows_out->rows0 + o, r, L);
          std::memcpy(rows_out->rows1 + o, r + cap, L);
          std::memcpy(rows_out->rows2 + o, r + 2 * cap, L);
        }
      };
      const size_t m = ch.hi - ch.lo;
      const int nt = int(std::min<size_t>(size_t(std::max(1, host_threads() / 2)), m / 4096 + 1));
      std::vector<std::thread> pool;
      for (int w = 1; w < nt; ++w) pool.emplace_back(copy_range, m * size_t(w) / size_t(nt), m * size_t(w + 1) / size_t(nt));
      copy_range(0, m / size_t(nt));
      for (auto& th : pool) th.join();
      return TA_OK;
    };
    size_t pool_used = 0;
    float walker_ms = 0.f;
    TA_CK(cudaEventRecord(bt->ev0, st));
    for (size_t c = 0; c < chunks.size(); ++c) {
      const Chunk& ch = chunks[c];
      const std::vector<int32_t> chunk(order.begin() + std::ptrdiff_t(ch.lo), order.begin() + std::ptrdiff_t(ch.hi));
      const int32_t* d_chunk = bt->d_ids.ptr + ch.lo;
      const int64_t m = int64_t(chunk.size());
      ta::WaveArgs args = base;
      args.dirs = reinterpret_cast<uint32_t*>(bt->d_dirs.ptr);
      args.dir_off = bt->d_diroff.ptr;
      if (int rc = launch_bucket(bt, chunk, ch.g, ch.lanes, opt.mode, true, args, st, &launches, &pool_used)) return rc;
      lanes_used = std::max(lanes_used, ch.lanes);
      if (opt.mode != TA_GLOBAL) {
        decode_keys_kernel<<<unsigned((m + 255) / 256), 256, 0, st>>>(bt->d_key.ptr, bt->d_desc.ptr, d_chunk, m,
                                                                    bt->d_score.ptr, bt->d_end.ptr);
        TA_CK(cudaGetLastError());
        ++launches;
      }
      const bool timed = chunks.size() == 1;  // per-chunk event sync would serialise the host
      if (timed) TA_CK(cudaEventRecord(bt->evw0, st));
      walker_kernel<<<unsigned((m + 127) / 128), 128, 0, st>>>(
          bt->d_desc.ptr, bt->seq.ptr, d_chunk, int(m), reinterpret_cast<const uint32_t*>(bt->d_dirs.ptr),
          bt->d_diroff.ptr, ch.g, opt.mode, bt->d_end.ptr, bt->d_begin.ptr, bt->d_rows.ptr, bt->d_rowoff.ptr,
          bt->d_rowlen.ptr, bt->d_status.ptr, bt->d_lenord.ptr + ch.lo);
      TA_CK(cudaGetLastError());
      ++launches;
      if (timed) TA_CK(cudaEventRecord(bt->evw1, st));
      if (scatter) {
        // chunk c-1's rows were queued for copy behind its kernels: scatter
        // them now (the GPU already has chunk c), then queue chunk c's copy
        // into the slot chunk c-2 used (already scattered)
        if (c > 0)
          if (int rc = scatter_chunk(c - 1)) return rc;
        TA_CK(cudaEventRecord(bt->evk[c & 1], st));
        TA_CK(cudaStreamWaitEvent(ctx->d2h, bt->evk[c & 1], 0));
        TA_CK(cudaMemcpyAsync(ctx->h_rows[c & 1].ptr, bt->d_rows.ptr + ch.rlo, size_t(ch.rhi - ch.rlo),
                              cudaMemcpyDeviceToHost, ctx->d2h));
        TA_CK(cudaMemcpyAsync(ctx->h_len[c & 1].ptr, bt->d_lenord.ptr + ch.lo, size_t(m) * 4, cudaMemcpyDeviceToHost,
                              ctx->d2h));
        TA_CK(cudaEventRecord(bt->evc[c & 1], ctx->d2h));
      }
    }
    TA_CK(cudaEventRecord(bt->ev1, st));
    if (scatter && !chunks.empty())
      if (int rc = scatter_chunk(chunks.size() - 1)) return rc;
    TA_CK(cudaEventSynchronize(bt->ev1));
    TA_CK(cudaEventElapsedTime(&ms_total, bt->ev0, bt->ev1));
    if (chunks.size() == 1) TA_CK(cudaEventElapsedTime(&walker_ms, bt->evw0, bt->evw1));
    bt->stats.walker_ms = walker_ms;
    bt->rows_scattered = scatter;
  }
  (void)rows_out;
  int64_t cells = 0;
  if (front_hit) {
    cells = bt->front_cells;
  } else {
    for (int32_t id : all_ok) cells += int64_t(bt->a[size_t(id)]) * bt->b[size_t(id)] * bt->c[size_t(id)];
    if (front_ok) {
      bt->front_key = fkey;
      bt->front_status = bt->status;
      bt->status_is_front = true;
      bt->front_all_ok = all_ok;
      bt->front_cells = cells;
    }
  }
  bt->stats.kernel_ms = ms_total;
  bt->stats.wavefront_ms = ms_total - bt->stats.walker_ms;
  bt->stats.cells = cells;
  bt->stats.launches = launches;
  bt->stats.lanes = lanes_used;
  bt->stats.buckets = nbuckets;
  bt->last_mode = opt.mode;
  bt->last_rows = rows;
  return TA_OK;
}


// ---------------------------------------------------------------------------
// Pipelined one-shot score path (ta_align_batch without rows).
//
// The batch is cut into contiguous chunks.  For chunk k the host packs ASCII
// -> 2-bit words with all cores straight into pinned memory, the copy stream
// moves them (4x fewer bytes than ASCII) while the compute stream still runs
// chunk k-1, and chunk k's results come back asynchronously: host packing,
// planning and both copies hide behind the kernels.

struct Lut {
  uint8_t v[256];
  Lut() {
    for (int i = 0; i < 256; ++i) v[i] = 0xFF;
    v['A'] = 0;
    v['C'] = 1;
    v['G'] = 2;
    v['T'] = 3;
  }
};

// Packs the sequences of triplets [lo, hi) (their words are contiguous,
// starting at global word `wbase`) into dst; flags non-ACGT triplets.
void host_pack(const char* seqs, const int64_t* offs, int64_t lo, int64_t hi, const std::vector<uint32_t>& wofs,
               uint32_t wbase, uint32_t* dst, std::vector<int32_t>& status, int threads) {
  static const Lut lut;
  auto work = [&](int64_t a0, int64_t a1) {
    for (int64_t t = a0; t < a1; ++t) {
      uint8_t orv = 0;
      for (int d = 0; d < 3; ++d) {
        const int64_t s0 = offs[3 * t + d], L = offs[3 * t + d + 1] - s0;
        const unsigned char* src = reinterpret_cast<const unsigned char*>(seqs + s0);
        uint32_t* out = dst + (wofs[size_t(3 * t + d)] - wbase);
        const int64_t nw = (L + 15) >> 4;
        for (int64_t w = 0; w < nw; ++w) {
          const int64_t base = w * 16, cnt = std::min<int64_t>(16, L - base);
          uint32_t word = 0;
          for (int64_t q = 0; q < cnt; ++q) {
            const uint8_t code = lut.v[src[base + q]];
            orv |= code;
            word |= uint32_t(code & 3u) << (2 * q);
          }
          out[w] = word;
        }
      }
      if (orv > 3) status[size_t(t)] = TA_ERR_PARSE;
    }
  };
  const int64_t n = hi - lo;
  const int nt = int(std::max<int64_t>(1, std::min<int64_t>(threads, n / 256)));
  if (nt == 1) {
    work(lo, hi);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w) pool.emplace_back(work, lo + n * w / nt, lo + n * (w + 1) / nt);
  for (auto& th : pool) th.join();
}

int align_scores_pipelined(DeviceCtx* ctx, const char* seqs, const int64_t* offsets, int64_t n,
                           const ta_scheme& scheme, const ta_options& opt, ta_results* out, cudaStream_t st) {
  NvtxRange nv("ta/align_pipelined");
  std::lock_guard<std::mutex> lock(ctx->mu);
  const auto tq0 = std::chrono::steady_clock::now();
  if (int rc = validate_scheme(scheme)) return rc;
  if (opt.mode < 0 || opt.mode > 2) return fail(TA_ERR_INVALID_ARGUMENT, "unknown alignment mode");
  const int cfg_rc = validate_options(opt);
  const std::string cfg_msg = cfg_rc ? g_err : std::string();
  const size_t nn = size_t(n);
  std::vector<int32_t> a(nn), b(nn), c(nn), status(nn, TA_OK);
  std::vector<uint32_t> wofs(3 * nn);
  uint64_t words = 0;
  int64_t total_cells = 0;
  // The only O(n) host pass before the first chunk launches (the GPU idles
  // meanwhile): lengths, packed-word offsets and cells.  Per-triplet checks and
  // descriptors are made chunk by chunk, behind the previous chunk's kernels.
  // two parallel passes: per-range lengths / words / cells, then the word
  // offsets from the ranges' prefix sums
  {
    const int nt = int(std::max<size_t>(1, std::min<size_t>(size_t(host_threads()), nn / 32768)));
    std::vector<uint64_t> rw(size_t(nt) + 1, 0);
    std::vector<int64_t> rc_(size_t(nt), 0), bad(size_t(nt), -1);
    auto pass1 = [&](int w) {
      const size_t t0 = nn * size_t(w) / size_t(nt), t1 = nn * size_t(w + 1) / size_t(nt);
      uint64_t wd = 0;
      int64_t cl = 0;
      for (size_t t = t0; t < t1; ++t) {
        for (int d = 0; d < 3; ++d) {
          const int64_t L = offsets[3 * t + d + 1] - offsets[3 * t + d];
          if ((L < 0 || L > (int64_t(1) << 24)) && bad[size_t(w)] < 0) bad[size_t(w)] = int64_t(t);
          wd += uint64_t((std::max<int64_t>(L, 0) + 15) / 16);
        }
        a[t] = int32_t(offsets[3 * t + 1] - offsets[3 * t]);
        b[t] = int32_t(offsets[3 * t + 2] - offsets[3 * t + 1]);
        c[t] = int32_t(offsets[3 * t + 3] - offsets[3 * t + 2]);
        cl += int64_t(a[t]) * b[t] * c[t];
      }
      rw[size_t(w) + 1] = wd;
      rc_[size_t(w)] = cl;
    };
    auto pass2 = [&](int w) {
      const size_t t0 = nn * size_t(w) / size_t(nt), t1 = nn * size_t(w + 1) / size_t(nt);
      uint64_t wd = rw[size_t(w)];
      for (size_t t = t0; t < t1; ++t)
        for (int d = 0; d < 3; ++d) {
          wofs[3 * t + d] = uint32_t(wd);
          wd += uint64_t((std::max<int64_t>(offsets[3 * t + d + 1] - offsets[3 * t + d], 0) + 15) / 16);
        }
    };
    auto run_all = [&](auto&& f) {
      std::vector<std::thread> pool;
      for (int w = 1; w < nt; ++w) pool.emplace_back(f, w);
      f(0);
      for (auto& th : pool) th.join();
    };
    run_all(pass1);
    for (int w = 0; w < nt; ++w) {
      if (bad[size_t(w)] >= 0)
        return fail(TA_ERR_INVALID_ARGUMENT, "bad sequence offsets for triplet " + std::to_string(bad[size_t(w)]));
      rw[size_t(w) + 1] += rw[size_t(w)];
      total_cells += rc_[size_t(w)];
    }
    words = rw[size_t(nt)];
    if (words > 0xFFFFFFF0ull) return fail(TA_ERR_CAPACITY, "batch exceeds 2^32 packed words");
    run_all(pass2);
  }
  // the batch shim lends lengths and the SM count to plan_streams / prepare_bucket
  ta_batch shim;
  shim.ctx = ctx;
  // engine errors per triplet, where the reference raises them (tiled.cpp:8-15, 37-58)
  auto check = [&](int64_t t0, int64_t t1) {
    for (int64_t t = t0; t < t1; ++t) {
      if (cfg_rc) {
        status[size_t(t)] = cfg_rc;
        continue;
      }
      const int32_t A = shim.a[size_t(t)], B = shim.b[size_t(t)], C = shim.c[size_t(t)];
      if (uint64_t(A) * uint64_t(B) * uint64_t(C) > opt.cell_budget) {
        status[size_t(t)] = TA_ERR_CAPACITY;
        continue;
      }
      const int32_t width = opt.team_width > 0 ? opt.team_width : derive_team_width(opt.tile_size, B, C);
      if (int64_t(width) * opt.tile_size < std::max(B, C)) {
        status[size_t(t)] = TA_ERR_CONFIG;
        continue;
      }
      if (opt.mode != TA_GLOBAL && !key_fits(A, B, C, scheme)) status[size_t(t)] = TA_ERR_CAPACITY;
    }
  };
  TA_CK(ctx->d_words.reserve(size_t(words) + 2));
  TA_CK(ctx->d_desc.reserve(nn));
  TA_CK(ctx->d_score.reserve(nn));
  TA_CK(ctx->d_end.reserve(3 * nn));
  TA_CK(ctx->d_key.reserve(nn));
  TA_CK(ctx->h_desc.reserve(nn));
  TA_CK(ctx->h_out.reserve(4 * nn));
  // chunks: contiguous triplet ranges of ~equal cells
  // Chunk boundaries by cells: the first chunks are small (1/64, 1/64, 1/32,
  // 1/16 of the batch) so the GPU starts early; the rest are equal.
  const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(16, n / 20000));
  std::vector<double> frac;  // cumulative cell fractions at the cuts
  if (nchunks >= 8) {
    double at = 0;
    for (double f : {1.0 / 64, 1.0 / 64, 1.0 / 32, 1.0 / 16}) frac.push_back(at += f);
    for (int64_t k = 1; k < nchunks - 1; ++k) frac.push_back(at + (1.0 - at) * double(k) / double(nchunks - 1));
  } else {
    for (int64_t k = 1; k < nchunks; ++k) frac.push_back(double(k) / double(nchunks));
  }
  std::vector<int64_t> cut{0};
  {
    int64_t acc = 0;
    size_t k = 0;
    for (int64_t t = 0; t < n; ++t) {
      acc += int64_t(a[size_t(t)]) * b[size_t(t)] * c[size_t(t)];
      if (k < frac.size() && double(acc) >= frac[k] * double(total_cells) && t + 1 < n) {
        cut.push_back(t + 1);
        ++k;
      }
    }
    cut.push_back(n);
  }
  const int threads = host_threads();
  const bool prof = std::getenv("TA_PROFILE_PIPELINE") != nullptr;
  const int g2 = 2 * scheme.gap;
  ta::WaveArgs base{};
  base.seq = ctx->d_words.ptr;
  base.desc = ctx->d_desc.ptr;
  base.out_score = ctx->d_score.ptr;
  base.out_end = ctx->d_end.ptr;
  base.out_key = ctx->d_key.ptr;
  base.g2 = g2;
  base.match_p = scheme.match - g2;
  base.mismatch_p = scheme.mismatch - g2;
  base.one = 1u;
  cudaEvent_t slot_free[2], h2d_done, kdone;
  for (auto& e : slot_free) TA_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TA_CK(cudaEventCreateWithFlags(&h2d_done, cudaEventDisableTiming));
  TA_CK(cudaEventCreateWithFlags(&kdone, cudaEventDisableTiming));
  shim.a.swap(a);
  shim.b.swap(b);
  shim.c.swap(c);
  // Launch plans come from a per-device pool that outlives the call: no
  // cudaMalloc / cudaFree (which can stall the host or the device) inside the
  // pipeline, and repeated calls reuse the buffers.
  size_t pool_used = 0;
  auto take_plan = [&]() -> BucketLaunch* {
    if (pool_used == ctx->plan_pool.size()) ctx->plan_pool.push_back(std::make_unique<BucketLaunch>());
    BucketLaunch* bl = ctx->plan_pool[pool_used++].get();
    bl->wave = false;
    bl->rounds.clear();
    return bl;
  };
  int64_t launches = 0;
  int rc = TA_OK;
  const auto tq1 = std::chrono::steady_clock::now();
  for (size_t k = 0; k + 1 < cut.size() && rc == TA_OK; ++k) {
    const int64_t lo = cut[k], hi = cut[k + 1];
    if (hi <= lo) continue;
    const uint32_t w0 = wofs[3 * size_t(lo)];
    const uint32_t w1 = hi < n ? wofs[3 * size_t(hi)] : uint32_t(words);
    PinnedBuf<uint32_t>& slot = ctx->h_words[k & 1];
    const auto tp0 = std::chrono::steady_clock::now();
    TA_CK(cudaEventSynchronize(slot_free[k & 1]));  // the previous H2D from this slot is done
    TA_CK(slot.reserve(size_t(w1 - w0) + 2));
    const auto tp1 = std::chrono::steady_clock::now();
    check(lo, hi);
    for (int64_t t = lo; t < hi; ++t)
      ctx->h_desc.ptr[t] = ta::TripletDesc{shim.a[size_t(t)], shim.b[size_t(t)], shim.c[size_t(t)], 0,
                                           wofs[3 * size_t(t)], wofs[3 * size_t(t) + 1], wofs[3 * size_t(t) + 2], 0};
    TA_CK(cudaMemcpyAsync(ctx->d_desc.ptr + lo, ctx->h_desc.ptr + lo, size_t(hi - lo) * sizeof(ta::TripletDesc),
                          cudaMemcpyHostToDevice, ctx->copy));
    host_pack(seqs, offsets, lo, hi, wofs, w0, slot.ptr, status, threads);
    const auto tp2 = std::chrono::steady_clock::now();
    TA_CK(cudaMemcpyAsync(ctx->d_words.ptr + w0, slot.ptr, size_t(w1 - w0) * 4, cudaMemcpyHostToDevice, ctx->copy));
    TA_CK(cudaEventRecord(slot_free[k & 1], ctx->copy));
    std::vector<std::vector<int32_t>> buckets(ta::kNumGrid);
    int64_t max_bound[ta::kNumGrid] = {0};
    std::vector<int32_t> ok_ids;
    for (int64_t t = lo; t < hi; ++t) {
      if (status[size_t(t)] != TA_OK) continue;
      const int32_t A = shim.a[size_t(t)], B = shim.b[size_t(t)], C = shim.c[size_t(t)];
      const int g = pick_grid(B, C);
      int gi = 0;
      while (ta::kGridSizes[gi] != g) ++gi;
      buckets[size_t(gi)].push_back(int32_t(t));
      max_bound[gi] = std::max(max_bound[gi], lane_bound(scheme, A, B, C, g));
      ok_ids.push_back(int32_t(t));
    }
    std::vector<BucketLaunch*> launch_now;
    for (int gi = 0; gi < ta::kNumGrid && rc == TA_OK; ++gi) {
      if (buckets[size_t(gi)].empty()) continue;
      const int lanes = s16_ok(scheme, max_bound[gi]) ? 2 : 1;
      std::vector<int32_t> wave_ids, rest_ids, t8_ids;
      int lanes8 = 1;
      if (gi == ta::kNumGrid - 1)
        split_largest(buckets[size_t(gi)], shim.a, shim.b, shim.c, scheme, ctx->sms * lanes, &wave_ids, &rest_ids,
                      &t8_ids, &lanes8);
      else
        rest_ids = buckets[size_t(gi)];
      for (int w = 0; w < 3 && rc == TA_OK; ++w) {
        const std::vector<int32_t>& part = w == 2 ? t8_ids : w ? wave_ids : rest_ids;
        if (part.empty()) continue;
        BucketLaunch* bl = take_plan();
        rc = prepare_bucket(&shim, part, ta::kGridSizes[gi], w == 2 ? lanes8 : lanes, opt.mode, false, ctx->copy, bl,
                            w == 1, w == 2 ? ta::kSmallTileN : w == 1 ? wave_tile_n() : ta::kTileN);
        launch_now.push_back(bl);
      }
    }
    if (rc != TA_OK) break;
    DevBuf<int32_t>* ids_buf = nullptr;
    if (opt.mode != TA_GLOBAL && !ok_ids.empty()) {
      ids_buf = &take_plan()->soff;
      TA_CK(ids_buf->reserve(ok_ids.size()));
      TA_CK(cudaMemcpyAsync(ids_buf->ptr, ok_ids.data(), ok_ids.size() * 4, cudaMemcpyHostToDevice, ctx->copy));
      TA_CK(cudaMemsetAsync(ctx->d_key.ptr + lo, 0, size_t(hi - lo) * 8, ctx->copy));
    }
    TA_CK(cudaEventRecord(h2d_done, ctx->copy));
    TA_CK(cudaStreamWaitEvent(st, h2d_done, 0));
    for (BucketLaunch* bl : launch_now) {
      rc = launch_prepared(bl, base, st, &launches);
      if (rc != TA_OK) break;
    }
    if (rc != TA_OK) break;
    if (ids_buf) {
      const int64_t m = int64_t(ok_ids.size());
      decode_keys_kernel<<<unsigned((m + 255) / 256), 256, 0, st>>>(ctx->d_key.ptr, ctx->d_desc.ptr, ids_buf->ptr, m,
                                                                  ctx->d_score.ptr, ctx->d_end.ptr);
      TA_CK(cudaGetLastError());
    }
    TA_CK(cudaEventRecord(kdone, st));
    TA_CK(cudaStreamWaitEvent(ctx->d2h, kdone, 0));
    if (prof) {
      const auto tp3 = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "[ta pipeline] chunk %zu: wait %.2f ms  pack %.2f ms  plan+launch %.2f ms\n", k,
                   ms(tp0, tp1), ms(tp1, tp2), ms(tp2, tp3));
    }
    TA_CK(cudaMemcpyAsync(ctx->h_out.ptr + lo, ctx->d_score.ptr + lo, size_t(hi - lo) * 4, cudaMemcpyDeviceToHost,
                          ctx->d2h));
    TA_CK(cudaMemcpyAsync(ctx->h_out.ptr + nn + 3 * size_t(lo), ctx->d_end.ptr + 3 * lo, size_t(hi - lo) * 12,
                          cudaMemcpyDeviceToHost, ctx->d2h));
  }
  const auto tq2 = std::chrono::steady_clock::now();
  cudaError_t e1 = cudaStreamSynchronize(ctx->copy);
  if (e1 == cudaSuccess) e1 = cudaStreamSynchronize(ctx->d2h);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  const auto tq3 = std::chrono::steady_clock::now();
  for (auto& e : slot_free) cudaEventDestroy(e);
  cudaEventDestroy(h2d_done);
  cudaEventDestroy(kdone);
  if (rc != TA_OK) return rc;
  TA_CK(e1);
  TA_CK(e2);
  auto deliver = [&](size_t t0, size_t t1) {
    for (size_t t = t0; t < t1; ++t) {
      const bool ok = status[t] == TA_OK;
      if (out->scores) out->scores[t] = ok ? ctx->h_out.ptr[t] : 0;
      if (out->ends)
        for (int d = 0; d < 3; ++d) out->ends[3 * t + d] = ok ? ctx->h_out.ptr[nn + 3 * t + d] : 0;
      if (out->status) out->status[t] = status[t];
    }
  };
  {
    const int nt = int(std::max<size_t>(1, std::min<size_t>(size_t(threads), nn / 65536)));
    std::vector<std::thread> pool;
    for (int w = 1; w < nt; ++w) pool.emplace_back(deliver, nn * size_t(w) / size_t(nt), nn * size_t(w + 1) / size_t(nt));
    deliver(0, nn / size_t(nt));
    for (auto& th : pool) th.join();
  }
  if (prof) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[ta pipeline] prologue %.2f ms  chunks %.2f ms  drain %.2f ms  epilogue %.2f ms\n",
                 ms(tq0, tq1), ms(tq1, tq2), ms(tq2, tq3), ms(tq3, std::chrono::steady_clock::now()));
  }
  if (cfg_rc) g_err = cfg_msg;
  ctx->last_stats = ta_stats{};
  ctx->last_stats.launches = launches;
  return TA_OK;
}

}  // namespace

// ===========================================================================
// C-ABI

extern "C" {

const char* ta_last_error(void) { return g_err.c_str(); }

const char* ta_version(void) { return "trioalign-b200 0.1 (sm_100a)"; }

int ta_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) c = 0;
  *count = c;
  return TA_OK;
}

// (Re)initialises a batch object with new inputs; device buffers are reused
// (grow-only), so a batch object kept by the caller allocates nothing.
static int batch_init(ta_batch* bt, DeviceCtx* ctx, int device, const char* seqs, const int64_t* offsets, int64_t n,
               cudaStream_t st) {
  bt->plan_cache.clear();
  bt->aff_cache.clear();
  bt->plan_key.clear();
  bt->front_key.clear();
  bt->stats = ta_stats{};
  bt->device = device;
  bt->ctx = ctx;
  bt->n = n;
  bt->a.resize(size_t(n));
  bt->b.resize(size_t(n));
  bt->c.resize(size_t(n));
  bt->desc.resize(size_t(n));
  bt->pre_status.assign(size_t(n), TA_OK);
  std::vector<int64_t> src_off(static_cast<size_t>(3 * n));
  std::vector<int32_t> len(static_cast<size_t>(3 * n));
  std::vector<uint32_t> dst_word(static_cast<size_t>(3 * n));
  uint64_t words = 0;
  for (int64_t t = 0; t < n; ++t) {
    for (int d = 0; d < 3; ++d) {
      const int64_t lo = offsets[3 * t + d], hi = offsets[3 * t + d + 1];
      if (hi < lo || hi - lo > (int64_t(1) << 24))
        return fail(TA_ERR_INVALID_ARGUMENT, "bad sequence offsets for triplet " + std::to_string(t));
      src_off[size_t(3 * t + d)] = lo;
      len[size_t(3 * t + d)] = int32_t(hi - lo);
      dst_word[size_t(3 * t + d)] = uint32_t(words);
      words += uint64_t((hi - lo + 15) / 16);
    }
    ta::TripletDesc& ds = bt->desc[size_t(t)];
    ds.a = bt->a[size_t(t)] = len[size_t(3 * t)];
    ds.b = bt->b[size_t(t)] = len[size_t(3 * t + 1)];
    ds.c = bt->c[size_t(t)] = len[size_t(3 * t + 2)];
    ds.flags = 0;
    ds.w0 = dst_word[size_t(3 * t)];
    ds.w1 = dst_word[size_t(3 * t + 1)];
    ds.w2 = dst_word[size_t(3 * t + 2)];
    ds.pad = 0;
  }
  if (words > 0xFFFFFFF0ull) return fail(TA_ERR_CAPACITY, "batch exceeds 2^32 packed words");
  const int64_t first = n ? offsets[0] : 0;
  const int64_t bytes = n ? offsets[3 * n] - first : 0;
  for (auto& o : src_off) o -= first;
  TA_CK(bt->seq.reserve(size_t(words) + 1));
  TA_CK(bt->d_desc.reserve(size_t(n)));
  TA_CK(bt->d_score.reserve(size_t(n)));
  TA_CK(bt->d_end.reserve(size_t(3 * n)));
  TA_CK(bt->d_status.reserve(size_t(n)));
  TA_CK(bt->d_key.reserve(size_t(n)));
  if (n > 0) {
    DevBuf<char>& ascii = bt->s_ascii;
    DevBuf<int64_t>& d_src = bt->s_src;
    DevBuf<int32_t>& d_len = bt->s_len;
    DevBuf<int32_t>& d_bad = bt->s_bad;
    DevBuf<uint32_t>& d_dst = bt->s_dst;
    TA_CK(ascii.reserve(size_t(bytes) + 1));
    TA_CK(d_src.reserve(size_t(3 * n)));
    TA_CK(d_len.reserve(size_t(3 * n)));
    TA_CK(d_dst.reserve(size_t(3 * n)));
    TA_CK(d_bad.reserve(size_t(n)));
    TA_CK(cudaMemcpyAsync(ascii.ptr, seqs + first, size_t(bytes), cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(d_src.ptr, src_off.data(), size_t(3 * n) * 8, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(d_len.ptr, len.data(), size_t(3 * n) * 4, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(d_dst.ptr, dst_word.data(), size_t(3 * n) * 4, cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemcpyAsync(bt->d_desc.ptr, bt->desc.data(), size_t(n) * sizeof(ta::TripletDesc),
                          cudaMemcpyHostToDevice, st));
    TA_CK(cudaMemsetAsync(d_bad.ptr, 0, size_t(n) * 4, st));
    const int64_t nseq = 3 * n;
    const int64_t threads = nseq * 32;
    pack_kernel<<<unsigned((threads + 255) / 256), 256, 0, st>>>(ascii.ptr, d_src.ptr, d_len.ptr, d_dst.ptr,
                                                               nseq, bt->seq.ptr, d_bad.ptr);
    TA_CK(cudaGetLastError());
    std::vector<int32_t> bad(static_cast<size_t>(n));
    TA_CK(cudaMemcpyAsync(bad.data(), d_bad.ptr, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
    TA_CK(cudaStreamSynchronize(st));
    for (int64_t t = 0; t < n; ++t)
      if (bad[size_t(t)]) bt->pre_status[size_t(t)] = TA_ERR_PARSE;
  }
  return TA_OK;
}

int ta_batch_create(int device, const char* seqs, const int64_t* offsets, int64_t n,
                    ta_batch** out, void* stream) {
  NvtxRange nv("ta/batch_create");
  *out = nullptr;
  if (n < 0) return fail(TA_ERR_INVALID_ARGUMENT, "negative triplet count");
  DeviceCtx* ctx = nullptr;
  if (int rc = get_ctx(device, &ctx)) return rc;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  auto bt = std::make_unique<ta_batch>();
  if (int rc = batch_init(bt.get(), ctx, device, seqs, offsets, n, st)) return rc;
  *out = bt.release();
  return TA_OK;
}

int ta_batch_run(ta_batch* b, const ta_scheme* scheme, const ta_options* opt, void* stream) {
  if (!b || !scheme || !opt) return fail(TA_ERR_INVALID_ARGUMENT, "null argument");
  TA_CK(cudaSetDevice(b->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : b->ctx->stream;
  if (opt->with_rows) {
    // rows need the row buffers; use ta_align_batch for the rows path
    return fail(TA_ERR_INVALID_ARGUMENT, "ta_batch_run computes scores; rows go through ta_align_batch");
  }
  std::lock_guard<std::mutex> lock(b->ctx->mu);  // one engine run per device at a time
  return run_impl(b, *scheme, *opt, st, nullptr);
}

int ta_batch_fetch(ta_batch* b, ta_results* out, void* stream) {
  NvtxRange nv("ta/batch_fetch");
  if (!b || !out) return fail(TA_ERR_INVALID_ARGUMENT, "null argument");
  TA_CK(cudaSetDevice(b->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : b->ctx->stream;
  const size_t n = size_t(b->n);
  if (n == 0) return TA_OK;
  if (out->scores) TA_CK(cudaMemcpyAsync(out->scores, b->d_score.ptr, n * 4, cudaMemcpyDeviceToHost, st));
  if (out->ends) TA_CK(cudaMemcpyAsync(out->ends, b->d_end.ptr, n * 12, cudaMemcpyDeviceToHost, st));
  TA_CK(cudaStreamSynchronize(st));
  if (out->status) std::memcpy(out->status, b->status.data(), n * 4);
  for (size_t t = 0; t < n; ++t) {
    if (b->status[t] != TA_OK) {
      if (out->scores) out->scores[t] = 0;
      if (out->ends) out->ends[3 * t] = out->ends[3 * t + 1] = out->ends[3 * t + 2] = 0;
    }
  }
  return TA_OK;
}

int ta_last_stats(int device, ta_stats* out) {
  if (!out) return fail(TA_ERR_INVALID_ARGUMENT, "null argument");
  DeviceCtx* ctx = nullptr;
  if (int rc = get_ctx(device, &ctx)) return rc;
  std::lock_guard<std::mutex> lock(ctx->mu);
  *out = ctx->last_stats;
  return TA_OK;
}

int ta_batch_stats(const ta_batch* b, ta_stats* out) {
  if (!b || !out) return fail(TA_ERR_INVALID_ARGUMENT, "null argument");
  *out = b->stats;
  return TA_OK;
}

void ta_batch_destroy(ta_batch* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  delete b;
}

int ta_align_batch(int device, const char* seqs, const int64_t* offsets, int64_t n,
                   const ta_scheme* scheme, const ta_options* opt, ta_results* out, void* stream) {
  if (!scheme || !opt || !out) return fail(TA_ERR_INVALID_ARGUMENT, "null argument");
  if (n < 0) return fail(TA_ERR_INVALID_ARGUMENT, "negative triplet count");
  const bool affine = scheme->gap_open != 0 || opt->gap_model == 1;
  if (!opt->with_rows && n > 0 && !affine) {
    DeviceCtx* ctx = nullptr;
    if (int rc = get_ctx(device, &ctx)) return rc;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    struct InFlight {
      InFlight() { ++g_calls_in_flight; }
      ~InFlight() { --g_calls_in_flight; }
    } in_flight;
    return align_scores_pipelined(ctx, seqs, offsets, n, *scheme, *opt, out, st);
  }
  // One cached batch object per device: its device buffers (sequences,
  // results, direction records, launch plans) are reused call after call.
  DeviceCtx* ctx = nullptr;
  if (int rc = get_ctx(device, &ctx)) return rc;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (!ctx->oneshot) ctx->oneshot = new ta_batch();
  ta_batch* bt = ctx->oneshot;
  if (int rc = batch_init(bt, ctx, device, seqs, offsets, n, st)) return rc;
  if (!opt->with_rows) {
    if (int rc = run_impl(bt, *scheme, *opt, st, nullptr)) return rc;
    ctx->last_stats = bt->stats;
    return ta_batch_fetch(bt, out, stream);
  }
  // rows path: device row buffers sized a+b+c per row
  const size_t nn = size_t(n);
  std::vector<int64_t> roff(nn);
  int64_t total = 0;
  for (size_t t = 0; t < nn; ++t) {
    roff[t] = total;
    total += 3 * (int64_t(bt->a[t]) + bt->b[t] + bt->c[t]);
  }
  TA_CK(bt->d_rows.reserve(size_t(total) + 1));
  TA_CK(bt->d_rowoff.reserve(nn));
  TA_CK(bt->d_rowlen.reserve(nn));
  TA_CK(bt->d_begin.reserve(3 * nn));
  TA_CK(cudaMemsetAsync(bt->d_rowlen.ptr, 0, nn * 4, st));
  TA_CK(cudaMemsetAsync(bt->d_begin.ptr, 0, nn * 12, st));
  TA_CK(cudaMemsetAsync(bt->d_status.ptr, 0, nn * 4, st));
  if (nn) TA_CK(cudaMemcpyAsync(bt->d_rowoff.ptr, roff.data(), nn * 8, cudaMemcpyHostToDevice, st));
  bt->rows_scattered = false;
  if (int rc = run_impl(bt, *scheme, *opt, st, out)) return rc;
  ctx->last_stats = bt->stats;
  if (nn == 0) return TA_OK;
  std::vector<int32_t> dstat(nn), rlen(nn), beg(3 * nn);
  std::vector<char> rows(bt->rows_scattered ? 1 : size_t(total) + 1);
  TA_CK(cudaMemcpyAsync(dstat.data(), bt->d_status.ptr, nn * 4, cudaMemcpyDeviceToHost, st));
  TA_CK(cudaMemcpyAsync(rlen.data(), bt->d_rowlen.ptr, nn * 4, cudaMemcpyDeviceToHost, st));
  TA_CK(cudaMemcpyAsync(beg.data(), bt->d_begin.ptr, nn * 12, cudaMemcpyDeviceToHost, st));
  if (!bt->rows_scattered)
    TA_CK(cudaMemcpyAsync(rows.data(), bt->d_rows.ptr, size_t(total), cudaMemcpyDeviceToHost, st));
  TA_CK(cudaStreamSynchronize(st));
  bt->status_is_front = false;
  for (size_t t = 0; t < nn; ++t)
    if (bt->status[t] == TA_OK && dstat[t] != TA_OK) bt->status[t] = dstat[t];
  if (int rc = ta_batch_fetch(bt, out, stream)) return rc;
  for (size_t t = 0; t < nn; ++t) {
    const bool ok = bt->status[t] == TA_OK;
    if (out->begins) {
      for (int d = 0; d < 3; ++d) out->begins[3 * t + d] = ok ? beg[3 * t + d] : 0;
    }
    if (out->row_lens) out->row_lens[t] = ok ? rlen[t] : 0;
    if (ok && out->rows0 && out->row_offsets && !bt->rows_scattered) {
      const int64_t cap = int64_t(bt->a[t]) + bt->b[t] + bt->c[t];
      const char* src = rows.data() + roff[t];
      std::memcpy(out->rows0 + out->row_offsets[t], src, size_t(rlen[t]));
      std::memcpy(out->rows1 + out->row_offsets[t], src + cap, size_t(rlen[t]));
      std::memcpy(out->rows2 + out->row_offsets[t], src + 2 * cap, size_t(rlen[t]));
    }
  }
  return TA_OK;
}

int64_t ta_packed_score_bound(int64_t a, int64_t b, int64_t c, const ta_scheme* s) {
  const int64_t per = std::max({3 * std::abs(int64_t(s->match)), 3 * std::abs(int64_t(s->mismatch)),
                                2 * std::abs(int64_t(s->gap))});
  return (a + b + c) * per;
}

int32_t ta_derive_team_width(int32_t tile_size, int32_t b, int32_t c) {
  return derive_team_width(tile_size, b, c);
}

int ta_validate_scheme(const ta_scheme* s) { return validate_scheme(*s); }

int ta_validate_options(const ta_options* o) { return validate_options(*o); }

int ta_plan_partition(const uint64_t* cells, int64_t n, int32_t strategy, int32_t workers,
                      int32_t* assignment) {
  // dispatch.cpp:29-60
  if (workers < 1) return fail(TA_ERR_CONFIG, "worker count must be >= 1");
  if (n <= 0) return fail(TA_ERR_CONFIG, "cannot partition an empty dataset");
  switch (strategy) {
    case 0: {
      const int64_t chunk = (n + workers - 1) / workers;
      for (int64_t i = 0; i < n; ++i) assignment[i] = int32_t(i / chunk);
      break;
    }
    case 1:
      for (int64_t i = 0; i < n; ++i) assignment[i] = int32_t(i % workers);
      break;
    case 2: {
      std::vector<uint64_t> load(static_cast<size_t>(workers), 0);
      for (int64_t i = 0; i < n; ++i) {
        int32_t best = 0;
        for (int32_t w = 1; w < workers; ++w)
          if (load[size_t(w)] < load[size_t(best)]) best = w;
        assignment[i] = best;
        load[size_t(best)] += cells[i];
      }
      break;
    }
    default:
      return fail(TA_ERR_PARSE, "unknown partition strategy");
  }
  return TA_OK;
}

}  // extern "C"
