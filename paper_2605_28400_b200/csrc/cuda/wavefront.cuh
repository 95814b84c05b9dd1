// wavefront.cuh — the sm_100a 3-way DP wavefront kernel (K1 score / K2
// direction cube) for batched exact 3-way Needleman-Wunsch alignment.
//
// Replaces the reference tiled engine's hot loop: tile_step / run_team
// (/root/reference/proj/include/trioalign/tiled.hpp:200-516) and, with
// TRACE=true, the full-tensor fill that feeds traceback
// (/root/reference/proj/src/oracle.cpp:11-65,98-180).
//
// Design:
//  * One CTA is a G x G grid of threads; thread (r, c) owns the N x N tile
//    j in [rN, rN+N), k in [cN, cN+N) of the (j, k) plane (the plane
//    includes the j = 0 / k = 0 faces, so every cell runs the same code).
//    The tile lives in registers and is updated in place (slice i - 1 until
//    the sweep of slice i overwrites a cell).
//  * Anti-diagonal pipeline (tiled.hpp:386-388): thread (r, c) computes
//    stream position s - LAG (r + c) at step s (LAG = 2 for single-plane
//    kernels, see WaveSmem).  Each CTA owns LANES independent
//    "slice streams" (the concatenated slices of the triplets assigned to
//    it), so the pipeline fills once per CTA, not once per triplet.
//  * LANES = 2 packs two independent triplet streams into s16x2 registers:
//    one VIADDMNMX.S16x2 / VIMNMX3.S16x2 advances two triplets.
//  * Scores are computed in a gap-shifted space M' = M - g2*(i+j+k)
//    (g2 = 2*gap), which zeroes the weight of the three single-residue
//    terms.  The tile is updated in place (no previous-slice copy); per cell
//    2 VIADDMNMX + 2 VIMNMX3 + 2 packed adds (IMAD), sigma12' folded out of
//    max(t1, t4).
//  * Neighbour boundaries (right column / down row + corner) go through a
//    shared-memory mailbox ring of LAG + 1 buffers, synchronised by
//    mbarriers (split arrive / wait, no __syncthreads in the loop).
//  * Exactness: all arithmetic is integer; lane width is chosen by the host
//    from a proven bound, so results are bit-identical to the reference.
#pragma once

#include <climits>
#include <cstdint>
#include <type_traits>

#ifndef TA_MBAR_SUSPEND_NS
#define TA_MBAR_SUSPEND_NS 0
#endif

namespace ta {

constexpr int kGlobal = 0;
constexpr int kSemi = 1;
constexpr int kLocal = 2;

// Direction tags carried in the 3 low bits of TRACE values (values scaled by
// 8, so both int32 and s16x2 lanes trace).  Larger tag wins ties, so the max
// selects the FIRST term of Eq. 1 in listed order (oracle.cpp:124-144).
// 7 = local-mode floor (stop, oracle.cpp:109-110).
constexpr uint32_t kTagT1 = 6, kTagT2 = 5, kTagT3 = 4, kTagT4 = 3;
constexpr uint32_t kTagT5 = 2, kTagT6 = 1, kTagT7 = 0, kTagStop = 7;
// Direction records: per (lane triplet, block, slice, tile) kDirWords 32-bit
// words, stored [word][thread] so a warp's stores are 128 B contiguous.  Word
// w holds the 3-bit codes of sweep-order cells 10w .. 10w+9: cell m < 5 at
// bit 3m, cell m >= 5 at bit 16 + 3(m - 5) (two 15-bit halves).
constexpr int kDirWords = 10;
// Sweep-order index of cell (p, q) of an n x n tile visited by anti-diagonals
// (d = p + q, p ascending); with n = G it is the thread index of tile (r, c)
// under the kernel's anti-diagonal thread map.
__host__ __device__ inline int antidiag_index(int p, int q, int n) {
  const int d = p + q;
  const int before = d <= n - 1 ? d * (d + 1) / 2 : n * (n + 1) / 2 + (n * (n - 1) - (2 * n - d) * (2 * n - d - 1)) / 2;
  return before + p - (d > n - 1 ? d - (n - 1) : 0);
}

// Semi-global / local best-cell key (optimal_score, oracle.cpp:67-88): one
// 64-bit word that orders by larger value, then smaller lexicographic (i, j, k)
// = smaller linear index lin = (i (b+1) + j)(c+1) + k.  28 bits of biased
// value above 36 bits of ~lin, so triplets of up to 2^36 cells (a 2000 bp
// triplet has 8e9 > 2^32) keep exact tie-breaks; the host rejects a triplet
// whose cell count or score bound does not fit (CapacityError).  Key 0 = none.
constexpr int kKeyLinBits = 36;
constexpr unsigned long long kKeyLinMask = (1ull << kKeyLinBits) - 1ull;
constexpr int kKeyValBias = 1 << 27;
__host__ __device__ __forceinline__ unsigned long long best_key(int mval, unsigned long long lin) {
  return (static_cast<unsigned long long>(static_cast<uint32_t>(mval + kKeyValBias)) << kKeyLinBits) |
         (kKeyLinMask - lin);
}
__host__ __device__ __forceinline__ int key_value(unsigned long long key) {
  return static_cast<int>(static_cast<uint32_t>(key >> kKeyLinBits)) - kKeyValBias;
}
__host__ __device__ __forceinline__ unsigned long long key_lin(unsigned long long key) {
  return kKeyLinMask - (key & kKeyLinMask);
}

struct TripletDesc {
  int32_t a, b, c, flags;
  uint32_t w0, w1, w2, pad;  // word offsets of s0/s1/s2 in the packed array
};

struct WaveArgs {
  const uint32_t* __restrict__ seq;        // 2-bit packed, 16 bases per word
  const TripletDesc* __restrict__ desc;
  const int4* __restrict__ items;          // stream items {tid, J<<16|K, slices, Bj<<16|Bk}
  const int32_t* __restrict__ stream_off;  // [gridDim.x * LANES + 1]
  const int32_t* __restrict__ cta_steps;   // [gridDim.x]
  int32_t* __restrict__ out_score;
  int32_t* __restrict__ out_end;           // 3 per triplet
  unsigned long long* __restrict__ out_key;  // semi/local (value, lex index)
  uint32_t* __restrict__ dirs;             // TRACE: direction records (kDirWords per tile-slice)
  const int64_t* __restrict__ dir_off;     // TRACE: per triplet, in 32-bit words
  int32_t match_p;                         // sigma' of equal residues   (match - g2)
  int32_t mismatch_p;                      // sigma' of unequal residues (mismatch - g2)
  int32_t g2;                              // 2 * gap (<= 0)
  uint32_t one;                            // == 1; keeps packed adds on the FMA pipe (IMAD)
  int32_t* __restrict__ faces;             // block-boundary faces of long triplets (int32 lane values)
  const int64_t* __restrict__ face_off;    // per stream, in words
  const int64_t* __restrict__ wave_base;   // WAVE: per triplet, its face area in 8-byte entries
  uint32_t epoch;                          // WAVE: launch epoch, high half of every face tag
};

// Wave mode (one long triplet spread over many CTAs): every block has its own
// down / right face rings in global memory, [a + 1][G][kSegE] entries of
// (value, tag) written with single 8-byte stores; tag = epoch << 16 | i + 1.
// A consumer checks the tags it staged and re-reads (L2) until they match, so
// cross-CTA block dependencies need no fences or flags (8-byte store
// atomicity, as in NCCL's LL protocol).
constexpr int kSegE = 12;  // entries per face segment (N + 1 <= 11 used), 96 B = 6 x 16 B
__host__ __device__ inline int64_t wave_block_entries(int a, int g) { return int64_t(2) * (a + 1) * g * kSegE; }

// Long triplets are split into row-major G*N x G*N blocks of the (j, k)
// plane; block (J, K) receives its top face (row J*GN - 1, GN + 1 values
// incl. the corner) and its left face (column K*GN - 1, GN values) per slice
// from global memory.  Per stream and triplet the face buffer holds
//   Fdown  [Bk][a + 1][GN + 1]   written by block (J, K), read by (J + 1, K)
//   Fright [a + 1][GN]           written by block (J, K), read by (J, K + 1)
__host__ __device__ inline int64_t face_words(int a, int bk, int gn) {
  return int64_t(bk) * (a + 1) * (gn + 1) + int64_t(a + 1) * gn;
}

template <int LANES>
struct LaneOps;

template <>
struct LaneOps<1> {
  static constexpr uint32_t kNeg = 0xE0000000u;  // -2^29
  static constexpr uint32_t kOne = 1u;
  __device__ __forceinline__ static uint32_t addmax(uint32_t a, uint32_t b, uint32_t c) {
    return static_cast<uint32_t>(__viaddmax_s32(static_cast<int>(a), static_cast<int>(b), static_cast<int>(c)));
  }
  __device__ __forceinline__ static uint32_t max3(uint32_t a, uint32_t b, uint32_t c) {
    return static_cast<uint32_t>(__vimax3_s32(static_cast<int>(a), static_cast<int>(b), static_cast<int>(c)));
  }
  __device__ __forceinline__ static uint32_t max2(uint32_t a, uint32_t b) {
    return static_cast<uint32_t>(max(static_cast<int>(a), static_cast<int>(b)));
  }
  __device__ __forceinline__ static int lane(uint32_t v, int) { return static_cast<int>(v); }
  __device__ __forceinline__ static uint32_t splat(int v) { return static_cast<uint32_t>(v); }
  __device__ __forceinline__ static uint32_t mask(int) { return 0xFFFFFFFFu; }
};

template <>
struct LaneOps<2> {
  static constexpr uint32_t kNeg = 0xC000C000u;  // -16384 per lane
  static constexpr uint32_t kOne = 0x00010001u;
  __device__ __forceinline__ static uint32_t addmax(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmax_s16x2(a, b, c);
  }
  __device__ __forceinline__ static uint32_t max3(uint32_t a, uint32_t b, uint32_t c) {
    return __vimax3_s16x2(a, b, c);
  }
  __device__ __forceinline__ static uint32_t max2(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }
  __device__ __forceinline__ static int lane(uint32_t v, int l) {
    return static_cast<int>(static_cast<int16_t>(l ? (v >> 16) : (v & 0xFFFFu)));
  }
  __device__ __forceinline__ static uint32_t splat(int v) {
    return (static_cast<uint32_t>(v) & 0xFFFFu) * 0x00010001u;
  }
  __device__ __forceinline__ static uint32_t mask(int l) { return l ? 0xFFFF0000u : 0x0000FFFFu; }
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

// d = a * one + c on the FMA pipe (one == 1 at run time): the packed lane add
// of the t1 partial sum leaves the ALU pipe, which bounds the recurrence.
__device__ __forceinline__ uint32_t fma_add(uint32_t a, uint32_t one, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(c));
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar, uint32_t count) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared.b64 st, [%0], %1;\n}" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count)
               : "memory");
}

// One aggregated arrival per converged group of threads (every thread is
// counted exactly once, whichever branch it is in).
__device__ __forceinline__ void mbar_arrive_group(uint64_t* bar) {
  const uint32_t m = __activemask();
  __syncwarp(m);
  if ((threadIdx.x & 31) == static_cast<uint32_t>(__ffs(m) - 1)) mbar_arrive(bar, __popc(m));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
#if TA_MBAR_SUSPEND_NS > 0
  // suspend (up to the hint) instead of spinning: a waiting warp does not
  // steal issue slots from the warps still computing the step
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1, %2;\n @!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity), "n"(TA_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
#endif
}

// Wave-mode face entries: (value, tag) as ONE 64-bit word, published and
// re-read with single-copy-atomic relaxed gpu-scope accesses, so a consumer
// that sees the new tag also sees the new value (PTX memory model).
__device__ __forceinline__ void st_face(void* p, uint32_t value, uint32_t tag) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p),
               "l"((static_cast<unsigned long long>(tag) << 32) | value)
               : "memory");
}
__device__ __forceinline__ uint2 ld_face(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
}

__device__ __forceinline__ uint32_t lop_sel(uint32_t a, uint32_t b, uint32_t m) {
  return (a & ~m) | (b & m);  // one LOP3
}

// Base codes of a 2-bit packed sequence: positions [pos, pos + n), n <= 16;
// out-of-range positions (pos < 0 or >= len) yield 0.
__device__ __forceinline__ int base_at(const uint32_t* __restrict__ seq, uint32_t w, int pos,
                                       int len) {
  if (pos < 0 || pos >= len) return 0;
  return static_cast<int>((__ldg(seq + w + (pos >> 4)) >> ((pos & 15) * 2)) & 3u);
}

#ifdef TA_WAVE_CLOCK
// dev-only (variant builds): per wave CTA and step, globaltimer at the step
// start, after the faces were taken and at the mailbox arrival (thread 0)
static __device__ unsigned long long g_wave_clock[4096][256][8];  // CTA 1 only, every thread
#endif

template <int N, int G, int LANES, int BLK = 1>
struct WaveSmem {
  static constexpr int T = G * G;
  static constexpr int NN = N * N;
  // Pipeline lag: tile (r, c) runs stream position s - LAG (r + c) at step s,
  // so the halos it reads at step s were published LAG steps earlier.  With
  // LAG = 2 (single-plane kernels) a warp waits only for step s - 2 before it
  // reads and for step s - 1 before it overwrites a mailbox buffer (NB = 3):
  // warps drift up to one step apart instead of meeting at every step, so the
  // tail of one warp's step overlaps the start of the next step of the others.
  // Block kernels keep LAG = 1 (their face timing is derived for it).
  static constexpr int LAG = BLK == 0 ? 2 : 1;
  static constexpr int NB = LAG + 1;  // mailbox buffers
  // Mailbox slot per tile: the down row (N + 1 values incl. the corner) at
  // words [0, DR), the right column (N values) at [DR, DR + RC), 16-byte
  // aligned for vector loads / stores; with two buffers an odd number of
  // vectors per slot keeps 8 slots of one LDS.128 phase on distinct banks
  // (three buffers do not fit with the padding: 2-way conflicts instead).
  static constexpr int DR = (N + 1 + 3) / 4 * 4;
  static constexpr int RC = (N + 3) / 4 * 4;
  static constexpr int XV = (((DR + RC) / 4) % 2 || NB > 2) ? (DR + RC) / 4 : (DR + RC) / 4 + 1;  // vectors per slot
  static constexpr int XW = 4 * XV;
  static constexpr size_t kSig = size_t(NN) * T * 4;      // sigma12 per cell
  static constexpr size_t kTab = size_t(N) * T * 8;       // per table (8 B per (row, thread))
  static constexpr size_t kX = size_t(NB) * XW * (T + 1) * 4;
  // cold per-lane state: single-plane kernels keep no block geometry, wave
  // kernels also the ring base (kWSeg)
  static constexpr int kLaneFields = BLK == 2 ? 11 : BLK ? 10 : 6;
  static constexpr size_t kLane = size_t(LANES) * kLaneFields * T * 4;
  // prefetched block faces (either layout); single-plane kernels have none
  static constexpr size_t kStage = BLK ? size_t(LANES) * 2 * G * kSegE * 8 : 0;
  static constexpr size_t kBar = 48;                       // NB <= 4 mbarriers + per-lane stream ends
  static constexpr int kSlots = 64;                        // open stream items per lane (ring)
  static constexpr size_t kBest = size_t(LANES) * kSlots * 12;  // per-item best key + finish count
  static constexpr size_t bytes = kSig + 2 * kTab + kX + kLane + kStage + kBar + kBest;
  static_assert(bytes <= 232448, "shared memory");
  static_assert(kSlots > 2 * LAG * (G - 1), "open items per lane exceed the ring");
};


// Cold per-lane fields kept in shared memory ([lane][field][thread]); the
// block geometry (kOrgJ ..) is stored by block kernels only (constants else).
enum LaneField { kItem = 0, kTid, kLenB, kLenC, kW0, kLen, kOrgJ, kOrgK, kBk, kBj, kIEnd, kWSeg = kIEnd };
// kIEnd: affine kernel only; kWSeg: linear wave kernels only - the block's own ring base in kSegE-entry
// segments, so face addresses need no dependent global load of wave_base per step

// ---------------------------------------------------------------------------
template <int N, int G, int LANES, int MODE, bool TRACE, int BLK>
__global__ void __launch_bounds__(G * G, 1) wavefront_kernel(const WaveArgs args) {
  // BLK: 0 = every triplet fits one plane; 1 = long triplets as consecutive
  // block items of one stream (faces via a per-stream buffer); 2 = wave mode
  // (blocks of a triplet on different CTAs, tagged faces).
  constexpr bool BLOCKS = BLK != 0;
  constexpr bool WAVE = BLK == 2;
  static_assert(N + 1 <= kSegE, "face segment too small");
  static_assert((N * N) % 4 == 0, "tile cells must group by 4");
  static_assert(!TRACE || N * N == 10 * kDirWords, "direction records hold 10 cells per word");
  using Ops = LaneOps<LANES>;
  using SM = WaveSmem<N, G, LANES, BLK>;
  constexpr int T = SM::T;
  [[maybe_unused]] constexpr int NN = SM::NN;
  constexpr int XW = SM::XW;
  constexpr int LAG = SM::LAG, NB = SM::NB;
  constexpr int SH = TRACE ? 3 : 0;  // value scale 2^SH (tags in low bits)
  constexpr uint32_t NEG = (TRACE && LANES == 1) ? 0xF0000000u : Ops::kNeg;
  constexpr uint32_t kOneL = Ops::kOne;  // 1 per lane
  constexpr uint32_t kDone = 1u, kOwner = 2u;
  constexpr uint32_t kInTop = 8u, kInLeft = 16u, kOutDown = 32u, kOutRight = 64u;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4* const s12v = reinterpret_cast<uint4*>(smem_raw);                     // [NN/4][T]
  uint32_t* const s12w = reinterpret_cast<uint32_t*>(smem_raw);
  unsigned char* const tab1 = smem_raw + SM::kSig;                            // 8 B per (row, thread)
  unsigned char* const tab2 = tab1 + SM::kTab;
  uint32_t* const xbuf = reinterpret_cast<uint32_t*>(tab2 + SM::kTab);        // [2][T+1][XW]
  int32_t* const lst = reinterpret_cast<int32_t*>(tab2 + SM::kTab + SM::kX);  // [LANES][8][T]
  int32_t* const stage = reinterpret_cast<int32_t*>(tab2 + SM::kTab + SM::kX + SM::kLane);  // [LANES][2G][N+1]
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(tab2 + SM::kTab + SM::kX + SM::kLane + SM::kStage);
  // Best (value, cell) of every open stream item, shared by the CTA's threads:
  // key = best_key(value, lin) (larger value, then smaller (i, j, k));
  // bcnt counts threads that finished the item (the last one flushes).
  int32_t* const iend_s = reinterpret_cast<int32_t*>(mbar + 4);                          // [LANES] stream ends
  unsigned long long* const bkey = reinterpret_cast<unsigned long long*>(mbar + 6);     // [LANES][kSlots]
  uint32_t* const bcnt = reinterpret_cast<uint32_t*>(bkey + LANES * SM::kSlots);         // [LANES][kSlots]

  constexpr int GN = G * N;

  const int t = threadIdx.x;
  // Thread -> tile map in anti-diagonal order: a warp spans only 2-3
  // pipeline skews (r + c), so per-triplet work at lane switches is not
  // replayed by many divergent subsets of the warp.
  int r, cc;
  {
    int rem = t, d = 0;
    for (; d < 2 * G - 1; ++d) {
      const int cnt = min(d, 2 * G - 2 - d) + 1;
      if (rem < cnt) break;
      rem -= cnt;
    }
    r = max(0, d - (G - 1)) + rem;
    cc = d - r;
  }
  const int tile = r * G + cc;

  const int j0 = r * N;
  const int k0 = cc * N;
  const int left = cc ? tile - 1 : T;
  const int up = r ? tile - G : T;
  const int skew = LAG * (r + cc);
  const int g2 = args.g2;
  const int ag2 = -g2;
  const uint32_t one = args.one;
  // TRACE: run-time powers of two and -1 keep the record packing on the FMA pipe
  [[maybe_unused]] const uint32_t mone = 0u - one;
  [[maybe_unused]] const uint32_t pw[5] = {one, one << 3, one << 6, one << 9, one << 12};
  // single-plane kernels: origin 0, one block (constants the compiler folds)
  [[maybe_unused]] int32_t cst[LANES][4];
#pragma unroll
  for (int l = 0; l < LANES; ++l) cst[l][0] = cst[l][1] = 0, cst[l][2] = cst[l][3] = 1;
  auto LS = [&](int l, int f) -> int32_t& {
    if constexpr (!BLOCKS) {
      if (f >= kOrgJ) return cst[l][f - kOrgJ];
    }
    return lst[(l * SM::kLaneFields + f) * T + t];
  };

  for (int w = t; w < NB * XW; w += T) xbuf[((w / XW) * (T + 1) + T) * XW + w % XW] = NEG;
  for (int w = t; w < LANES * SM::kSlots; w += T) {
    bkey[w] = 0ull;
    bcnt[w] = 0u;
  }
  if (t == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&mbar[b], T);
  }

  // hot per-lane state in registers
  int si[LANES], la[LANES];
  // semi: best M value of this tile's face row (0) / column (1) in the open
  // item and where: slice * 16 + first maximal cell of the line (-1: none);
  // offered once, when the item ends
  [[maybe_unused]] int fbv[LANES][2], fbs[LANES][2];
#pragma unroll
  for (int l = 0; l < LANES; ++l) fbs[l][0] = fbs[l][1] = -1, fbv[l][0] = fbv[l][1] = INT_MIN;
  uint32_t s0word[LANES], flags[LANES];

  // 2-bit codes of the N bases at positions [pos, pos + N) of a sequence of
  // length len (packed at word w), slot s -> bits 2s; out of range -> 0.
  auto load_codes = [&](uint32_t w, int pos, int len) -> uint32_t {
    const int p0 = pos < 0 ? 0 : pos;
    if (p0 >= len) return 0u;
    const uint32_t* src = args.seq + w + (p0 >> 4);
    const unsigned long long both =
        static_cast<unsigned long long>(__ldg(src)) | (static_cast<unsigned long long>(__ldg(src + 1)) << 32);
    uint32_t codes = static_cast<uint32_t>(both >> (2 * (p0 & 15)));
    if (pos < 0) codes <<= 2;
    const int nvalid = len - pos;
    if (nvalid < 16) codes &= (1u << (2 * nvalid)) - 1u;
    return codes;
  };

  struct LaneLoad {
    uint32_t c1, c2;  // 2-bit codes of the tile's N s1 / s2 characters
    uint32_t v1, v2;  // bit p: position p holds a real s1 / s2 residue (else padding: sigma' = 0)
    int mp, mm;       // sigma' of equal / unequal residues (0, 0 for the null item)
  };
  // positions p in [0, N) with 0 <= g - 1 + p < len
  auto valid_bits = [](int g, int len) -> uint32_t {
    const int lo = g == 0 ? 1 : 0;
    const int hi = max(0, min(N, len - g + 1));
    return hi > lo ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
  };

  // Loads stream item `it` of lane l (or the null item when it >= end: all
  // zero weights, which keeps an idle lane's values bounded): lengths, block
  // origin and flags; returns the tile's characters for the sigma tables.
  auto fetch = [&](int l, int it, int iend) -> LaneLoad {
    int id = -1, a_ = 0, b_ = -1, c_ = -1, len = 0x3FFFFFFF, J = 0, K = 0, Bj = 1, Bk = 1;
    uint32_t ww0 = 0, ww1 = 0, ww2 = 0;
    int4 rec = make_int4(-1, 0, 0x3FFFFFFF, 0x00010001);
    if (it < iend) rec = __ldg(args.items + it);
    if (rec.x < 0 && it < iend) len = rec.z;  // null item: the lane idles for len slices
    if (rec.x >= 0) {
      id = rec.x;
      if constexpr (BLOCKS) {
        J = rec.y >> 16;
        K = rec.y & 0xFFFF;
        Bj = rec.w >> 16;
        Bk = rec.w & 0xFFFF;
      }
      len = rec.z;
      const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(args.desc + id));
      const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(args.desc + id) + 1);
      a_ = static_cast<int>(d0.x);
      b_ = static_cast<int>(d0.y);
      c_ = static_cast<int>(d0.z);
      ww0 = d1.x;
      ww1 = d1.y;
      ww2 = d1.z;
    }
    la[l] = a_;
    LS(l, kTid) = id;
    LS(l, kLenB) = b_;
    LS(l, kLenC) = c_;
    LS(l, kW0) = static_cast<int32_t>(ww0);
    LS(l, kOrgJ) = J * GN;
    LS(l, kOrgK) = K * GN;
    LS(l, kLen) = len;
    LS(l, kBk) = Bk;
    LS(l, kBj) = Bj;
    if constexpr (WAVE) {
      // ring bases are multiples of kSegE entries (wave_block_entries); 2^32
      // segments of 96 B exceed the device memory
      LS(l, kWSeg) = id >= 0 ? static_cast<int32_t>(static_cast<uint32_t>(
                                   args.wave_base[id] / kSegE + int64_t(J * Bk + K) * 2 * (a_ + 1) * G))
                             : 0;
    }
    const int gj0 = J * GN + j0, gk0 = K * GN + k0;
    uint32_t f = (id >= 0 || it < iend) ? 0u : kDone;  // a null item keeps the lane alive
    if (id >= 0 && b_ / N == gj0 / N && c_ / N == gk0 / N && b_ >= gj0 && c_ >= gk0) f |= kOwner;
    if (id >= 0 && J > 0) f |= kInTop;
    if (id >= 0 && K > 0) f |= kInLeft;
    if (id >= 0 && J + 1 < Bj) f |= kOutDown;
    if (id >= 0 && K + 1 < Bk) f |= kOutRight;
    flags[l] = f;
    return LaneLoad{load_codes(ww1, gj0 - 1, b_), load_codes(ww2, gk0 - 1, c_), valid_bits(gj0, b_),
                    valid_bits(gk0, c_), id >= 0 ? args.match_p : 0, id >= 0 ? args.mismatch_p : 0};
  };

  // sigma tables of one lane (the other lane's halves are left untouched)
  auto tables_lane = [&](int l, const LaneLoad& ld) {
    const uint32_t c1 = ld.c1, c2 = ld.c2;
    const int mp = ld.mp, mm = ld.mm;
    if constexpr (LANES == 1) {
      // int16 tables: 4 values (s0 code 0..3) per row, 8 B per (row, thread)
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const uint32_t x1 = (c1 >> (2 * p)) & 3u, x2 = (c2 >> (2 * p)) & 3u;
        uint32_t v1[4], v2[4];
#pragma unroll
        for (int code = 0; code < 4; ++code) {
          v1[code] = ((ld.v1 >> p) & 1u) ? static_cast<uint32_t>(code == int(x1) ? mp : mm) & 0xFFFFu : 0u;
          v2[code] = ((ld.v2 >> p) & 1u) ? static_cast<uint32_t>(code == int(x2) ? mp : mm) & 0xFFFFu : 0u;
        }
        reinterpret_cast<uint2*>(tab1)[p * T + t] = make_uint2(v1[0] | (v1[1] << 16), v1[2] | (v1[3] << 16));
        reinterpret_cast<uint2*>(tab2)[p * T + t] = make_uint2(v2[0] | (v2[1] << 16), v2[2] | (v2[3] << 16));
      }
      const int sc = TRACE ? 8 : 1;
      const int tg = TRACE ? static_cast<int>(kTagT4) : 0;
      // sigma12' in the sweep's anti-diagonal cell order, 4 cells per STS.128
      uint32_t v[4];
      int k = 0;
#pragma unroll
      for (int d = 0; d <= 2 * N - 2; ++d)
#pragma unroll
        for (int p = 0; p < N; ++p) {
          const int q = d - p;
          if (q < 0 || q >= N) continue;
          const int sv = ((ld.v1 >> p) & (ld.v2 >> q) & 1u) ? ((((c1 >> (2 * p)) & 3u) == ((c2 >> (2 * q)) & 3u)) ? mp : mm) : 0;
          v[k & 3] = static_cast<uint32_t>(sv * sc + tg);
          if ((k & 3) == 3) s12v[(k >> 2) * T + t] = make_uint4(v[0], v[1], v[2], v[3]);
          ++k;
        }
    } else {
      // byte tables: sigma'(code, x) = mm + (mp - mm) * [code == x], byte `code`
      const uint32_t mm8 = static_cast<uint32_t>(mm) * 0x01010101u;
      const uint32_t dm = static_cast<uint32_t>(mp - mm);
      uint32_t t2w[N];
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const uint32_t x1 = (c1 >> (2 * p)) & 3u, x2 = (c2 >> (2 * p)) & 3u;
        reinterpret_cast<uint32_t*>(tab1)[(p * T + t) * 2 + l] = ((ld.v1 >> p) & 1u) ? mm8 + (dm << (8 * x1)) : 0u;
        t2w[p] = ((ld.v2 >> p) & 1u) ? mm8 + (dm << (8 * x2)) : 0u;
        reinterpret_cast<uint32_t*>(tab2)[(p * T + t) * 2 + l] = t2w[p];
      }
      uint16_t* s12h = reinterpret_cast<uint16_t*>(s12w);
      int k = 0;
#pragma unroll
      for (int d = 0; d <= 2 * N - 2; ++d)
#pragma unroll
        for (int p = 0; p < N; ++p) {
          const int q = d - p;
          if (q < 0 || q >= N) continue;
          const uint32_t x1 = (c1 >> (2 * p)) & 3u;
          const uint32_t sel = x1 | ((x1 | 8u) << 4);
          const uint32_t sv = ((ld.v1 >> p) & 1u) ? (prmt(t2w[q], 0u, sel) & 0xFFFFu) : 0u;
          s12h[((size_t(k >> 2) * T + t) * 4 + (k & 3)) * 2 + l] = static_cast<uint16_t>(TRACE ? sv * 8u + kTagT4 : sv);
          ++k;
        }
    }
  };

  // sigma tables of both s16x2 lanes at once (paired lane switch): one PRMT
  // per cell builds the packed word, written 4 cells per STS.128.
  auto tables_both = [&](const LaneLoad& l0, const LaneLoad& l1) {
    const uint32_t m0 = static_cast<uint32_t>(l0.mm) * 0x01010101u, d0 = static_cast<uint32_t>(l0.mp - l0.mm);
    const uint32_t m1 = static_cast<uint32_t>(l1.mm) * 0x01010101u, d1 = static_cast<uint32_t>(l1.mp - l1.mm);
    uint32_t t2a[N], t2b[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
      const uint32_t x10 = (l0.c1 >> (2 * p)) & 3u, x20 = (l0.c2 >> (2 * p)) & 3u;
      const uint32_t x11 = (l1.c1 >> (2 * p)) & 3u, x21 = (l1.c2 >> (2 * p)) & 3u;
      reinterpret_cast<uint2*>(tab1)[p * T + t] =
          make_uint2(((l0.v1 >> p) & 1u) ? m0 + (d0 << (8 * x10)) : 0u, ((l1.v1 >> p) & 1u) ? m1 + (d1 << (8 * x11)) : 0u);
      t2a[p] = ((l0.v2 >> p) & 1u) ? m0 + (d0 << (8 * x20)) : 0u;
      t2b[p] = ((l1.v2 >> p) & 1u) ? m1 + (d1 << (8 * x21)) : 0u;
      reinterpret_cast<uint2*>(tab2)[p * T + t] = make_uint2(t2a[p], t2b[p]);
    }
    uint32_t sel[N], pm[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
      const uint32_t x10 = (l0.c1 >> (2 * p)) & 3u, x11 = ((l1.c1 >> (2 * p)) & 3u) + 4u;
      sel[p] = x10 | ((x10 | 8u) << 4) | (x11 << 8) | ((x11 | 8u) << 12);
      pm[p] = (((l0.v1 >> p) & 1u) ? 0x0000FFFFu : 0u) | (((l1.v1 >> p) & 1u) ? 0xFFFF0000u : 0u);
    }
    uint32_t v[4];
    int k = 0;
#pragma unroll
    for (int d = 0; d <= 2 * N - 2; ++d)
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const int q = d - p;
        if (q < 0 || q >= N) continue;
        v[k & 3] = prmt(t2a[q], t2b[q], sel[p]) & pm[p];
        if constexpr (TRACE) v[k & 3] = v[k & 3] * 8u + kTagT4 * kOneL;
        if ((k & 3) == 3) s12v[(k >> 2) * T + t] = make_uint4(v[0], v[1], v[2], v[3]);
        ++k;
      }
  };

  auto setup = [&](int l, int it, int iend) { tables_lane(l, fetch(l, it, iend)); };

  const int sbase = blockIdx.x * LANES;
  LaneLoad first[LANES];
#pragma unroll
  for (int l = 0; l < LANES; ++l) {
    const int it = args.stream_off[sbase + l];
    const int ie = args.stream_off[sbase + l + 1];
    LS(l, kItem) = it;
    if (t == 0) iend_s[l] = ie;
    si[l] = 0;
    s0word[l] = 0;
    first[l] = fetch(l, it, ie);
  }
  if constexpr (LANES == 2) {
    tables_both(first[0], first[1]);
  } else {
    tables_lane(0, first[0]);
  }
  // Paired lanes (sequential block items): both lanes hold block items with the
  // same slices and block grid in lockstep (the host pairs equal-shape
  // triplets), so their block faces travel as packed words through lane 0's
  // face buffer: one store / prefetch / load per position instead of a
  // per-lane extract, splat and masked merge (see affine.cuh).
  constexpr bool kPackFaces = LANES == 2 && BLK == 1;
  auto lockstep = [&]() -> bool {
    if constexpr (!kPackFaces) {
      return false;
    } else {
      return !(flags[0] & kDone) && !(flags[1] & kDone) && LS(0, kTid) >= 0 && LS(1, kTid) >= 0 &&
             si[0] == si[1] && la[0] == la[1] && LS(0, kBj) == LS(1, kBj) && LS(0, kBk) == LS(1, kBk) &&
             LS(0, kOrgJ) == LS(1, kOrgJ) && LS(0, kOrgK) == LS(1, kOrgK) && LS(0, kLen) == LS(1, kLen);
    }
  };
  bool paired = lockstep();

  // the tile in registers (row / column 0: the halos), updated in place:
  // slice i - 1 until the sweep of slice i overwrites it cell by cell
  uint32_t Cu[N + 1][N + 1];
#pragma unroll
  for (int P = 0; P <= N; ++P)
#pragma unroll
    for (int Q = 0; Q <= N; ++Q) Cu[P][Q] = NEG;

  __syncthreads();

  // Mailbox protocol: step s publishes into xbuf[s % NB] and arrives on
  // mbar[s % NB]; step s + LAG waits for that phase before it reads.  LAG = 1:
  // a thread publishing at step s+1 has waited for every thread's step-s
  // arrival, which follows that thread's step-s reads of the same buffer.
  // LAG = 2: a thread reads at step s what its neighbours published at step
  // s - 2 (waits for phase s - 2), and before it overwrites buffer s % 3 -
  // read by its neighbours at step s - 1 - it waits for phase s - 1.  Either
  // way the ring is race-free without __syncthreads, and the per-step tail
  // work (extraction, lane switches, prefetch) overlaps the slowest warp.
  // The host's step count covers a LAG = 1 pipeline; the extra fill is added here.
  const int nsteps = args.cta_steps[blockIdx.x] + (LAG - 1) * 2 * (G - 1);
  // phase of step q: the (q / NB)-th completion of mbar[q % NB]
  auto wait_step = [&](int q) { mbar_wait(&mbar[q % NB], static_cast<uint32_t>(q / NB) & 1u); };
  // LAG = 2: before a thread publishes (or arrives) at step s, the buffer
  // readers of step s - 1 are done (this also orders its arrivals per mbarrier)
  auto wait_free = [&](int s_) {
    if constexpr (LAG > 1) {
      if (s_ >= 1) wait_step(s_ - 1);
    }
  };
  // Wave mode: segment `idx` of slice `sl` of ring `ring` (0 down, 1 right) of
  // the block at offset `dblk` from this lane's (0 own, -1 left, -Bk top)
  [[maybe_unused]] auto ring_seg = [&](int l, int dblk, int ring, int sl, int idx) -> uint64_t* {
    const int a1 = la[l] + 1;
    const int64_t seg = int64_t(static_cast<uint32_t>(LS(l, kWSeg))) + ((int64_t(dblk) * 2 + ring) * a1 + sl) * G + idx;
    return reinterpret_cast<uint64_t*>(args.faces) + seg * kSegE;
  };
  // Wave mode: stage the (value, tag) face segments of slice `sl` of lane l
  // (cp.async, no registers held).  A step issues the next slice's segments
  // right after it has read this slice's, so the L2 round trip from the
  // producer CTA overlaps the whole sweep instead of the next step's start.
  [[maybe_unused]] auto wave_prefetch = [&](int l, int sl) {
    if (LS(l, kTid) < 0 || !(flags[l] & (kInTop | kInLeft))) return;
    auto fetch_seg = [&](int seg, const uint64_t* src) {
      uint64_t* dst = reinterpret_cast<uint64_t*>(stage) + (l * 2 * G + seg) * kSegE;
#pragma unroll
      for (int v = 0; v < kSegE / 2; ++v)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(dst + 2 * v))),
                     "l"(src + 2 * v)
                     : "memory");
    };
    if (r == 0 && (flags[l] & kInTop))  // down ring of block (J - 1, K), segment cc
      fetch_seg(cc, ring_seg(l, -LS(l, kBk), 0, sl, cc));
    if (cc == 0 && (flags[l] & kInLeft))  // right ring of block (J, K - 1), segment r
      fetch_seg(G + r, ring_seg(l, -1, 1, sl, r));
  };
  for (int s = 0; s < nsteps; ++s) {
    const int buf = s % NB;
    [[maybe_unused]] bool early[LANES];
#pragma unroll
    for (int l = 0; l < LANES; ++l) early[l] = false;
    const int rbuf = (s + 1) % NB;  // == (s - LAG) mod NB
    bool any = false;
#pragma unroll
    for (int l = 0; l < LANES; ++l) any |= !(flags[l] & kDone);
    const bool active = s >= skew && any;
    // Every thread (active or idle) waits for the previous phase before it
    // arrives again: no thread can arrive on mbar[b] twice within one phase.
#ifdef TA_WAVE_CLOCK
    auto wclock = [&](int k) {
      if (WAVE && blockIdx.x == 1 && s < 4096 && T <= 256) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        g_wave_clock[s][r * G + cc][k] = g;
      }
    };
    wclock(0);
    unsigned long long wrereads = 0;
#endif
    if (s >= LAG) wait_step(s - LAG);
#ifdef TA_WAVE_CLOCK
    wclock(3);
#endif
    // A tile that holds no real cell of any live lane this step (padding
    // beyond b / c, or the padded slices of a block item) skips the sweep: its
    // values only ever feed other padding, and its warp's issue slots go to
    // the tiles doing real work.
    // (Measured per mode: +64% for local, -4..7% for the others, whose
    // register allocation it perturbs; so only local mode skips.)
    constexpr bool kSkipPadding = MODE == kLocal;
    bool work = !kSkipPadding;
    if constexpr (kSkipPadding) {
#pragma unroll
      for (int l = 0; l < LANES; ++l)
        work |= !(flags[l] & kDone) && si[l] <= la[l] && LS(l, kLenB) - LS(l, kOrgJ) - j0 >= 0 &&
                LS(l, kLenC) - LS(l, kOrgK) - k0 >= 0;
    }
    if (active) {
     if (work) {
      // ---- 1. per-slice sigma row / column tables -----------------------
      uint32_t sel = 0;  // LANES == 2: PRMT selector; LANES == 1: code
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        const int pos = si[l] - 1;
        const uint32_t code = (pos >= 0 && (!BLOCKS || pos < la[l])) ? (s0word[l] >> ((pos & 15) * 2)) & 3u : 0u;
        if constexpr (LANES == 1) {
          sel = code;
        } else {
          const uint32_t b = code + 4u * l;
          sel |= (b | ((b | 8u) << 4)) << (8 * l);
        }
      }
      auto sig_row = [&](const unsigned char* tab, int p) -> uint32_t {
        if constexpr (LANES == 1) {
          return static_cast<uint32_t>(static_cast<int>(
              reinterpret_cast<const int16_t*>(tab)[(size_t(p) * T + t) * 4 + sel]));
        } else {
          const uint2 e = reinterpret_cast<const uint2*>(tab)[p * T + t];
          return prmt(e.x, e.y, sel);
        }
      };
      uint32_t s02[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        s02[q] = sig_row(tab2, q);
        if constexpr (TRACE) s02[q] = s02[q] * 8u + kTagT3 * kOneL;
      }
      // TRACE: t1's column term sigma02' with tag 4 - 6 (lane-exact), so that
      // t1 = W + a2c + sg carries tag 5 + 4 - 6 + 3 = 6
      [[maybe_unused]] uint32_t a2c[TRACE ? N : 1];
      if constexpr (TRACE) {
#pragma unroll
        for (int q = 0; q < N; ++q) a2c[q] = Ops::addmax(s02[q], Ops::splat(-6), NEG);
      }
      uint32_t a1v[N];
#pragma unroll
      for (int p = 0; p < N; ++p) {
        a1v[p] = sig_row(tab1, p);
        if constexpr (TRACE) a1v[p] = a1v[p] * 8u + kTagT2 * kOneL;
      }

      // ---- 2. previous-slice terms of the halo, then the new halos -------
      // The tile is updated in place: Cu[P][Q] holds M'(i - 1) until the
      // sweep overwrites it with M'(i).  Two partial sums of a previous-slice
      // value are formed before it is overwritten (packed adds on the FMA
      // pipe, carry-free: values >= 0 or NEG-derived, weights >= 0):
      //   W[P][Q] = M'(i-1, P-1, Q) + sigma01'(P)  (t2 of (P, Q); t1 of (P, Q+1))
      //   Z[P][Q] = M'(i-1, P, Q-1) + sigma02'(Q)  (t3 of (P, Q))
      // so the recurrence needs 2 DPX + 2 three-way max per cell and no
      // previous-slice copy.  The halo row / column feed W[1][*], W[*][0] and
      // Z[*][1] before this slice's halos replace them.
      uint32_t W[N + 1][N + 1], Z[N + 1][N + 1];
#pragma unroll
      for (int Q = 0; Q <= N; ++Q) W[1][Q] = fma_add(Cu[0][Q], one, a1v[0]);
#pragma unroll
      for (int P = 2; P <= N; ++P) W[P][0] = fma_add(Cu[P - 1][0], one, a1v[P - 1]);
#pragma unroll
      for (int P = 1; P <= N; ++P) Z[P][1] = fma_add(Cu[P][0], one, s02[0]);

      // new halos (published by the neighbours LAG steps earlier)
      {
        const uint4* xu = reinterpret_cast<const uint4*>(xbuf + (rbuf * (T + 1) + up) * XW);
        const uint4* xl = reinterpret_cast<const uint4*>(xbuf + (rbuf * (T + 1) + left) * XW + SM::DR);
#pragma unroll
        for (int v = 0; v < SM::DR / 4; ++v) {
          const uint4 e = xu[v];
          const uint32_t w4[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (4 * v + u <= N) Cu[0][4 * v + u] = w4[u];
        }
#pragma unroll
        for (int v = 0; v < SM::RC / 4; ++v) {
          if (4 * v + 2 >= N) {  // the last pair (N % 4 == 2): one 8-byte load
            const uint2 e = reinterpret_cast<const uint2*>(xl + v)[0];
            Cu[4 * v + 1][0] = e.x;
            if (4 * v + 1 < N) Cu[4 * v + 2][0] = e.y;
            continue;
          }
          const uint4 e = xl[v];
          const uint32_t w4[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (4 * v + u < N) Cu[4 * v + u + 1][0] = w4[u];
        }
      }
      if (BLOCKS && (r == 0 || cc == 0)) {
        bool top = false, lft = false;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          top |= r == 0 && (flags[l] & kInTop) && si[l] <= la[l];
          lft |= cc == 0 && (flags[l] & kInLeft) && si[l] <= la[l];
        }
        if (top || lft) {
          asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef TA_WAVE_CLOCK
          wclock(5);
#endif
          if (kPackFaces && paired) {
            if (r == 0 && (flags[0] & kInTop) && si[0] <= la[0]) {
              const uint32_t* st = reinterpret_cast<const uint32_t*>(stage) + cc * (N + 1);
#pragma unroll
              for (int q = 0; q <= N; ++q) Cu[0][q] = st[q];
            }
            if (cc == 0 && (flags[0] & kInLeft) && si[0] <= la[0]) {
              const uint32_t* st = reinterpret_cast<const uint32_t*>(stage) + (G + r) * (N + 1);
#pragma unroll
              for (int p = 0; p < N; ++p) Cu[p + 1][0] = st[p];
            }
          } else
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            const bool ok = si[l] <= la[l];
            if constexpr (WAVE) {
              if (LS(l, kTid) < 0) continue;  // a null item (idle partner lane) has no faces
              const uint32_t want = (args.epoch << 16) + static_cast<uint32_t>(si[l]) + 1u;
              // the staged (value, tag) entries [0, CNT) of segment seg: one
              // branch when every tag is fresh (the common case); otherwise
              // each stale entry is re-read from L2 until its tag matches
              auto take_seg = [&](int seg, const uint64_t* src, auto cnt, int32_t (&out)[N + 1]) {
                constexpr int CNT = decltype(cnt)::value;
                const uint2* sv = reinterpret_cast<const uint2*>(stage) + (l * 2 * G + seg) * kSegE;
                uint2 v[CNT];
                bool fresh = true;
#pragma unroll
                for (int e = 0; e < CNT; ++e) {
                  v[e] = sv[e];
                  fresh &= v[e].y == want;
                }
                if (!fresh) {
#pragma unroll
                  for (int e = 0; e < CNT; ++e) {
                    uint2 w = v[e];
                    while (w.y != want) {
                      w = ld_face(src + e);
#ifdef TA_WAVE_CLOCK
                      ++wrereads;
#endif
                    }
                    out[e] = static_cast<int32_t>(w.x);
                  }
                } else {
#pragma unroll
                  for (int e = 0; e < CNT; ++e) out[e] = static_cast<int32_t>(v[e].x);
                }
              };
              // only a lane for which this tile holds real cells waits for its
              // faces: padding producers of the other lane skip their sweep
              const bool real = LS(l, kLenB) - LS(l, kOrgJ) - j0 >= 0 && LS(l, kLenC) - LS(l, kOrgK) - k0 >= 0;
              if (r == 0 && (flags[l] & kInTop) && ok && real) {
                int32_t fv[N + 1];
                take_seg(cc, ring_seg(l, -LS(l, kBk), 0, si[l], cc), std::integral_constant<int, N + 1>{}, fv);
#pragma unroll
                for (int q = 0; q <= N; ++q) Cu[0][q] = lop_sel(Cu[0][q], Ops::splat(fv[q] << SH), Ops::mask(l));
              }
              if (cc == 0 && (flags[l] & kInLeft) && ok && real) {
                int32_t fv[N + 1];
                take_seg(G + r, ring_seg(l, -1, 1, si[l], r), std::integral_constant<int, N>{}, fv);
#pragma unroll
                for (int p = 0; p < N; ++p) Cu[p + 1][0] = lop_sel(Cu[p + 1][0], Ops::splat(fv[p] << SH), Ops::mask(l));
              }
              // this lane's staged segments are consumed: stage the next slice
              if (!(flags[l] & kDone) && si[l] + 1 <= la[l]) {
#ifdef TA_WAVE_CLOCK
                wclock(6);
#endif
                wave_prefetch(l, si[l] + 1);
#ifdef TA_WAVE_CLOCK
                wclock(7);
#endif
                early[l] = true;
              }
              continue;
            }
            if (r == 0 && (flags[l] & kInTop) && ok) {
              const int32_t* st = stage + (l * 2 * G + cc) * (N + 1);
#pragma unroll
              for (int q = 0; q <= N; ++q) Cu[0][q] = lop_sel(Cu[0][q], Ops::splat(st[q] << SH), Ops::mask(l));
            }
            if (cc == 0 && (flags[l] & kInLeft) && ok) {
              const int32_t* st = stage + (l * 2 * G + G + r) * (N + 1);
#pragma unroll
              for (int p = 0; p < N; ++p) Cu[p + 1][0] = lop_sel(Cu[p + 1][0], Ops::splat(st[p] << SH), Ops::mask(l));
            }
          }
        }
      }

#ifdef TA_WAVE_CLOCK
      wclock(1);
      {
        if (WAVE && blockIdx.x == 1 && s < 4096 && T <= 256) g_wave_clock[s][r * G + cc][4] = wrereads;
      }
#endif
      // ---- 3. forced cells (reference initialisation, oracle.cpp:30-39) --
      // global: M(0,0,0) = 0; semi: axis cells are 0 in M-space.
      uint32_t fcorner = NEG;
      // semi slice-0 axis cells: row P = 1 / column Q = 1 start values as a
      // packed base plus a per-cell step (NEG base and 0 step in lanes that
      // force nothing), folded into the one sweep (no second copy of the tile
      // loop: the semi kernel was instruction-cache bound)
      uint32_t frb = NEG, fcb = NEG, frs = 0u, fcs = 0u;
      uint32_t flbase = 0;
      bool force = false;  // semi: this step computes slice-0 axis cells of a lane
      if constexpr (MODE == kSemi) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          const int oj = LS(l, kOrgJ), ok = LS(l, kOrgK);
          force |= !(flags[l] & kDone) && si[l] == 0 && ((r == 0 && oj == 0) || (cc == 0 && ok == 0));
        }
      }
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        const bool live = !(flags[l] & kDone);
        if constexpr (MODE == kGlobal) {
          if (t == 0 && live && si[l] == 0 && LS(l, kOrgJ) == 0 && LS(l, kOrgK) == 0)
            fcorner = lop_sel(fcorner, 0u, Ops::mask(l));
        } else if constexpr (MODE == kSemi) {
          const int oj = LS(l, kOrgJ), ok = LS(l, kOrgK);
          if (t == 0 && live && oj == 0 && ok == 0 && si[l] <= la[l])
            fcorner = lop_sel(fcorner, Ops::splat((ag2 * si[l]) << SH), Ops::mask(l));
          if (force && live && si[l] == 0) {
            if (r == 0 && oj == 0) {
              frb = lop_sel(frb, Ops::splat((ag2 * (ok + k0)) << SH), Ops::mask(l));
              frs = lop_sel(frs, Ops::splat(ag2 << SH), Ops::mask(l));
            }
            if (cc == 0 && ok == 0) {
              fcb = lop_sel(fcb, Ops::splat((ag2 * (oj + j0)) << SH), Ops::mask(l));
              fcs = lop_sel(fcs, Ops::splat(ag2 << SH), Ops::mask(l));
            }
          }
        } else {
          // local floor base: |g2| * (i + j + k) at the tile origin
          flbase = lop_sel(flbase, Ops::splat((ag2 * (si[l] + LS(l, kOrgJ) + LS(l, kOrgK) + j0 + k0)) << SH),
                           Ops::mask(l));
        }
      }

      // ---- 4. the tile: 2 DPX + 2 three-way max + 2 packed adds per cell --
      // TRACE: direction records of this step, one pointer per live lane
      [[maybe_unused]] uint32_t* dptr[LANES];
      [[maybe_unused]] bool dok[LANES];
      if constexpr (TRACE) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          dok[l] = !(flags[l] & kDone) && si[l] <= la[l] && LS(l, kTid) >= 0;
          dptr[l] = args.dirs;
          if (dok[l]) {
            const int blk = (LS(l, kOrgJ) / GN) * LS(l, kBk) + LS(l, kOrgK) / GN;
            dptr[l] = args.dirs + args.dir_off[LS(l, kTid)] +
                      (static_cast<int64_t>(blk) * (la[l] + 1) + si[l]) * (kDirWords * T) + t;
          }
        }
      }
      [[maybe_unused]] uint32_t accA = 0, accB = 0;
      // local floor |g2| * (i + j + k) of the current cell, stepped along the
      // row on the FMA pipe (values >= 0: packed adds never carry)
      const uint32_t ag2s = Ops::splat(ag2 * (1 << SH));
      uint32_t flrow = flbase + (TRACE ? kTagStop * kOneL : 0u);
      auto sweep_tile = [&]() {
      // Cells in anti-diagonal order (d = P + Q): consecutive cells are
      // independent, so the row / column dependencies of the recurrence are
      // ~N instructions apart instead of back to back.  sigma12' is stored in
      // the same order (4 cells per LDS.128).
      uint4 sg4 = make_uint4(0, 0, 0, 0);
      [[maybe_unused]] uint32_t fd = flrow;  // local floor of diagonal d (depends on P + Q only)
      [[maybe_unused]] uint32_t frv = frb, fcv = fcb;  // semi: start of the next row-1 / column-1 cell
      int k = 0;
#pragma unroll
      for (int d = 0; d <= 2 * N - 2; ++d) {
        if constexpr (MODE == kLocal) {
          if (d > 0) fd = fma_add(fd, one, ag2s);
        }
#pragma unroll
        for (int P0 = 0; P0 < N; ++P0) {
          const int Q0 = d - P0;
          if (Q0 < 0 || Q0 >= N) continue;
          const int P = P0 + 1, Q = Q0 + 1;
          if ((k & 3) == 0) sg4 = s12v[(k >> 2) * T + t];
          const uint32_t sg = (k & 3) == 0 ? sg4.x : (k & 3) == 1 ? sg4.y : (k & 3) == 2 ? sg4.z : sg4.w;
          [[maybe_unused]] const int ks = k;  // sweep-order index of this cell
          ++k;
          // the previous-slice value of this cell feeds (P + 1, Q) and (P, Q + 1);
          // its last use is the cell's own final max (t5), so the new value can
          // take its register (no permutation moves at the loop back edge)
          const uint32_t old = Cu[P][Q];
          if (P < N) W[P + 1][Q] = fma_add(old, one, a1v[P]);
          if (Q < N) Z[P][Q + 1] = fma_add(old, one, s02[Q]);
          uint32_t x;
          if constexpr (!TRACE) {
            const uint32_t c = Ops::addmax(W[P][Q - 1], s02[Q - 1], Cu[P - 1][Q - 1]);  // max(t1, t4) - sg
            x = Ops::addmax(c, sg, Z[P][Q]);                                           // t1, t4 vs t3
            x = Ops::max3(x, W[P][Q], old);                                            // t2, t5
            x = Ops::max3(x, Cu[P - 1][Q], Cu[P][Q - 1]);                              // t6, t7
          } else {
            // tags: W, Z, sg carry 5, 4, 3; t1 = 5 + (4 - 6) + 3 = 6; t5, t6, t7: 2, 1, 0
            const uint32_t c = Ops::addmax(W[P][Q - 1], a2c[Q - 1], Cu[P - 1][Q - 1]);  // tags 3 / 0
            x = Ops::addmax(c, sg, Z[P][Q]);                                            // t1 6, t4 3, t3 4
            x = Ops::max3(x, W[P][Q], Cu[P][Q - 1]);                                    // t2 5, t7 0
            x = Ops::addmax(old, kTagT5 * kOneL, x);                                    // t5
            x = Ops::addmax(Cu[P - 1][Q], kTagT6 * kOneL, x);                           // t6
          }
          if constexpr (MODE == kLocal) x = Ops::addmax(fd, one ^ 1u, x);  // floor 0 (oracle.cpp:59), fused form
          if constexpr (MODE == kGlobal || MODE == kSemi) {
            if (P == 1 && Q == 1) x = Ops::max2(x, fcorner);
          }
          if constexpr (MODE == kSemi) {
            // row-1 cells are visited with Q increasing, column-1 cells with P
            if (P == 1) {
              x = Ops::max2(x, frv);
              if (Q < N) frv = fma_add(frv, one, frs);
            }
            if (Q == 1) {
              x = Ops::max2(x, fcv);
              if (P < N) fcv = fma_add(fcv, one, fcs);
            }
          }
          if constexpr (TRACE) {
            // tag -> record (IMAD accumulation on the FMA pipe), value := x - tag
            const uint32_t code = x & (7u * kOneL);
            x = fma_add(code, mone, x);
            const int m = ks % 10;
            if (m == 0) accA = code;
            else if (m < 5) accA = fma_add(code, pw[m], accA);
            else if (m == 5) accB = code;
            else accB = fma_add(code, pw[m - 5], accB);
            if (m == 9) {
              const int w = ks / 10;
              if (dok[0]) dptr[0][w * T] = prmt(accA, accB, 0x5410u);
              if constexpr (LANES == 2) {
                if (dok[LANES - 1]) dptr[LANES - 1][w * T] = prmt(accA, accB, 0x7632u);
              }
            }
          }
          Cu[P][Q] = x;
        }
      }
      };
      sweep_tile();

      // ---- 5. publish right column / down row (+ corner) ----------------
      wait_free(s);
      {
        uint4* xo = reinterpret_cast<uint4*>(xbuf + (buf * (T + 1) + tile) * XW);
#pragma unroll
        for (int v = 0; v < SM::DR / 4; ++v) {
          uint32_t w4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) w4[u] = 4 * v + u <= N ? Cu[N][4 * v + u] : 0u;
          xo[v] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
#pragma unroll
        for (int v = 0; v < SM::RC / 4; ++v) {
          uint32_t w4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) w4[u] = 4 * v + u < N ? Cu[4 * v + u + 1][N] : 0u;
          if (4 * v + 2 >= N) {
            reinterpret_cast<uint2*>(xo + SM::DR / 4 + v)[0] = make_uint2(w4[0], w4[1]);
          } else {
            xo[SM::DR / 4 + v] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
          }
        }
      }
      if (BLOCKS && (r == G - 1 || cc == G - 1)) {
        bool wrote = false;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (si[l] > la[l]) continue;
          const bool dn = r == G - 1 && (flags[l] & kOutDown);
          const bool rt = cc == G - 1 && (flags[l] & kOutRight);
          if (!dn && !rt) continue;
          const int a1 = la[l] + 1;
          if constexpr (WAVE) {
            const uint32_t tag = (args.epoch << 16) + static_cast<uint32_t>(si[l]) + 1u;
            if (dn) {  // down ring of this block: segment cc, entries q = 0..N (q = 0 is the corner)
              uint2* d = reinterpret_cast<uint2*>(ring_seg(l, 0, 0, si[l], cc));
#pragma unroll
              for (int q = 0; q <= N; ++q) st_face(d + q, static_cast<uint32_t>(Ops::lane(Cu[N][q], l) >> SH), tag);
            }
            if (rt) {  // right ring: segment r, entries p = 0..N-1
              uint2* d = reinterpret_cast<uint2*>(ring_seg(l, 0, 1, si[l], r));
#pragma unroll
              for (int p = 0; p < N; ++p) st_face(d + p, static_cast<uint32_t>(Ops::lane(Cu[p + 1][N], l) >> SH), tag);
            }
            continue;
          }
          if (kPackFaces && paired) {  // lane 0's buffer, both lanes packed; once
            if (l != 0) continue;
            uint32_t* fb = reinterpret_cast<uint32_t*>(args.faces + args.face_off[sbase]);
            if (dn) {
              uint32_t* d = fb + (int64_t(LS(0, kOrgK) / GN) * a1 + si[0]) * (GN + 1) + cc * N;
#pragma unroll
              for (int q = 0; q <= N; ++q) d[q] = Cu[N][q];
            }
            if (rt) {
              uint32_t* d = fb + int64_t(LS(0, kBk)) * a1 * (GN + 1) + int64_t(si[0]) * GN + r * N;
#pragma unroll
              for (int p = 0; p < N; ++p) d[p] = Cu[p + 1][N];
            }
            wrote = true;
            continue;
          }
          int32_t* fb = args.faces + args.face_off[sbase + l];
          if (dn) {  // Fdown[K][i][cN + q], q = 0 is the corner (k = cN - 1)
            int32_t* d = fb + (int64_t(LS(l, kOrgK) / GN) * a1 + si[l]) * (GN + 1) + cc * N;
#pragma unroll
            for (int q = 0; q <= N; ++q) d[q] = Ops::lane(Cu[N][q], l) >> SH;
          }
          if (rt) {  // Fright[i][rN + p]
            int32_t* d = fb + int64_t(LS(l, kBk)) * a1 * (GN + 1) + int64_t(si[l]) * GN + r * N;
#pragma unroll
            for (int p = 0; p < N; ++p) d[p] = Ops::lane(Cu[p + 1][N], l) >> SH;
          }
          wrote = true;
        }
        if (wrote) __threadfence_block();
      }
#ifdef TA_WAVE_CLOCK
      wclock(2);
#endif
      mbar_arrive_group(&mbar[buf]);

      // ---- 7. score extraction ------------------------------------------
      if constexpr (MODE == kGlobal) {
        // M[a, b, c] (tiled.hpp:495-502): the owner tile, last slice
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if ((flags[l] & kOwner) && si[l] == la[l]) {
            const int B = LS(l, kLenB), C = LS(l, kLenC), id = LS(l, kTid);
            const int want = (B - LS(l, kOrgJ) - j0 + 1) * (N + 1) + (C - LS(l, kOrgK) - k0 + 1);
            uint32_t v = 0;
#pragma unroll
            for (int P = 1; P <= N; ++P)
#pragma unroll
              for (int Q = 1; Q <= N; ++Q)
                if (P * (N + 1) + Q == want) v = Cu[P][Q];
            args.out_score[id] = (Ops::lane(v, l) >> SH) + g2 * (la[l] + B + C);
            args.out_end[3 * id] = la[l];
            args.out_end[3 * id + 1] = B;
            args.out_end[3 * id + 2] = C;
          }
        }
      } else {
        // Best tracking (oracle.cpp:67-88, tiled.hpp:129-144, 222-228): max
        // value, ties to the lexicographically smallest (i, j, k).
        // Candidates: local = every real cell; semi = i == a || j == b || k == c.
        //
        // Padding cells need no masks: their sigma' is 0 (tables), which
        // makes every padded cell (i, j, k) <= the real cell
        // (i, min(j, b), min(k, c)) of the same tile, and that cell comes
        // first in row-major (= lexicographic) order, so it wins every tie.
        // Tiles that hold no real cell of a lane are skipped for that lane.
        constexpr int SC = 1 << SH;
        const uint32_t g2s = Ops::splat(g2 * SC);
        int rb[LANES], cb[LANES];
        bool full[LANES], face[LANES];
        bool anyfull = false, anyface = false;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          rb[l] = LS(l, kLenB) - LS(l, kOrgJ) - j0;  // rows P-1 <= rb are real
          cb[l] = LS(l, kLenC) - LS(l, kOrgK) - k0;
          const bool inside = !(flags[l] & kDone) && si[l] <= la[l] && rb[l] >= 0 && cb[l] >= 0;
          full[l] = inside && (MODE == kLocal || si[l] == la[l]);
          face[l] = MODE == kSemi && inside && !full[l] && (rb[l] < N || cb[l] < N);
          anyfull |= full[l];
          anyface |= face[l];
        }
        auto key_of = [](int mval, unsigned long long lin) -> unsigned long long { return best_key(mval, lin); };
        auto lin_of = [&](int l, int P, int Q) -> unsigned long long {
          const uint32_t j = LS(l, kOrgJ) + j0 + P - 1, k = LS(l, kOrgK) + k0 + Q - 1;
          return (static_cast<unsigned long long>(static_cast<uint32_t>(si[l])) * static_cast<uint32_t>(LS(l, kLenB) + 1) + j) *
                     static_cast<uint32_t>(LS(l, kLenC) + 1) + k;
        };
        // Only a tile that can beat the item's best so far (its max value with
        // the tile's smallest cell index) searches for its first maximal cell.
        auto may_beat = [&](int l, int mval) -> bool {
          const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(
              &bkey[l * SM::kSlots + (LS(l, kItem) & (SM::kSlots - 1))]);
          return key_of(mval, lin_of(l, 1, 1)) > cur;
        };
        // The offer is a fire-and-forget 64-bit max in global memory (native
        // RED.MAX.64; a 64-bit shared-memory atomicMax is a CAS spin loop that
        // the face threads of a step contend on).  The shared slot keeps only a
        // filter hint: a plain store of an offered key, so it never exceeds
        // the true best (a racing lower store only lets later offers through).
        auto offer = [&](int l, int mval, int P, int Q) {
          const unsigned long long key = key_of(mval, lin_of(l, P, Q));
          atomicMax(args.out_key + LS(l, kTid), key);
          volatile unsigned long long* hint = &bkey[l * SM::kSlots + (LS(l, kItem) & (SM::kSlots - 1))];
          if (key > *hint) *hint = key;
        };
        // max over Q of Cu[P][Q] + g2 * (Q - 1) (Horner, one VIADDMNMX per cell)
        auto row_max = [&](int P) -> uint32_t {
          uint32_t acc = Cu[P][N];
#pragma unroll
          for (int Q = N - 1; Q >= 1; --Q) acc = Ops::addmax(acc, g2s, Cu[P][Q]);
          return acc;
        };
        // fr[Q - 1] = Cu[p + 1][Q] / fc[P - 1] = Cu[P][q + 1] for a run-time p / q in [0, N)
        auto select_row = [&](int p, uint32_t (&fr)[N]) {
#pragma unroll
          for (int Q = 1; Q <= N; ++Q) {
            uint32_t v = Cu[1][Q];
#pragma unroll
            for (int P = 2; P <= N; ++P) v = p == P - 1 ? Cu[P][Q] : v;
            fr[Q - 1] = v;
          }
        };
        auto select_col = [&](int q, uint32_t (&fc)[N]) {
#pragma unroll
          for (int P = 1; P <= N; ++P) {
            uint32_t v = Cu[P][1];
#pragma unroll
            for (int Q = 2; Q <= N; ++Q) v = q == Q - 1 ? Cu[P][Q] : v;
            fc[P - 1] = v;
          }
        };
        if (anyfull) {
          uint32_t stepmax = row_max(N);
#pragma unroll
          for (int P = N - 1; P >= 1; --P) stepmax = Ops::addmax(stepmax, g2s, row_max(P));
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            if (!full[l]) continue;
            const int sm = Ops::lane(stepmax, l);  // scaled by SC, relative to the tile origin
            const int mval = (sm >> SH) + g2 * (si[l] + LS(l, kOrgJ) + LS(l, kOrgK) + j0 + k0);
            if (may_beat(l, mval)) {
              // first row, then first cell of that row, attaining the maximum;
              // the row is selected into fr (one SEL per cell) so the scan
              // below exists once, not once per row (code size: the semi /
              // local loops were instruction-cache bound)
              int fp = 0;
#pragma unroll
              for (int P = N; P >= 1; --P)
                if (Ops::lane(row_max(P), l) + g2 * SC * (P - 1) == sm) fp = P;
              uint32_t fr[N];
              select_row(fp - 1, fr);
              int fq = 0;
#pragma unroll
              for (int Q = N; Q >= 1; --Q)
                if (Ops::lane(fr[Q - 1], l) + g2 * SC * (fp - 1 + Q - 1) == sm) fq = Q;
              offer(l, mval, fp, fq);
            }
          }
        }
        if constexpr (MODE == kSemi) {
          if (anyface) {
            // faces j == b (tile row rb) and k == c (tile column cb): per step
            // only the line's maximum (in M units) is compared with the best
            // of earlier slices (strictly greater: the earliest slice wins
            // ties, oracle.cpp:74-85); the winning line is saved and its first
            // maximal cell is resolved once, when the item ends
#pragma unroll
            for (int l = 0; l < LANES; ++l) {
              if (!face[l]) continue;
              const int base = g2 * (si[l] + LS(l, kOrgJ) + LS(l, kOrgK) + j0 + k0);
              const int rbl = rb[l], cbl = cb[l];
              if (rbl < N) {
                uint32_t fr[N];
                if (rbl == 0) {  // lengths that are multiples of N: no select
#pragma unroll
                  for (int Q = 1; Q <= N; ++Q) fr[Q - 1] = Cu[1][Q];
                } else {
                  select_row(rbl, fr);
                }
                uint32_t acc = fr[N - 1];
#pragma unroll
                for (int Q = N - 1; Q >= 1; --Q) acc = Ops::addmax(acc, g2s, fr[Q - 1]);
                const int hv = (Ops::lane(acc, l) >> SH) + g2 * rbl + base;
                if (hv > fbv[l][0]) {
                  int at = 0;
#pragma unroll
                  for (int x = N; x >= 1; --x)
                    if ((Ops::lane(fr[x - 1], l) >> SH) + g2 * (rbl + x - 1) + base == hv) at = x;
                  fbv[l][0] = hv;
                  fbs[l][0] = si[l] * 16 + at;
                }
              }
              if (cbl < N) {
                uint32_t fc[N];
                if (cbl == 0) {
#pragma unroll
                  for (int P = 1; P <= N; ++P) fc[P - 1] = Cu[P][1];
                } else {
                  select_col(cbl, fc);
                }
                uint32_t acc = fc[N - 1];
#pragma unroll
                for (int P = N - 1; P >= 1; --P) acc = Ops::addmax(acc, g2s, fc[P - 1]);
                const int hv = (Ops::lane(acc, l) >> SH) + g2 * cbl + base;
                if (hv > fbv[l][1]) {
                  int at = 0;
#pragma unroll
                  for (int x = N; x >= 1; --x)
                    if ((Ops::lane(fc[x - 1], l) >> SH) + g2 * (cbl + x - 1) + base == hv) at = x;
                  fbv[l][1] = hv;
                  fbs[l][1] = si[l] * 16 + at;
                }
              }
            }
          }
        }
      }

     } else {
      wait_free(s);
      mbar_arrive_group(&mbar[buf]);
     }

      // ---- 9. advance the lanes (switch triplets at the end of a stream item)
      bool sw[LANES];
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        sw[l] = false;
        if (flags[l] & kDone) continue;
        si[l] += 1;
        sw[l] = BLOCKS ? si[l] >= LS(l, kLen) : si[l] > la[l];
        if (sw[l]) {
          if constexpr (MODE == kSemi) {
            // offer this tile's face bests of the finished item (one 64-bit key each)
#pragma unroll
            for (int f = 0; f < 2; ++f) {
              if (fbs[l][f] < 0) continue;
              const int oj = LS(l, kOrgJ), ok = LS(l, kOrgK);
              const int line = f ? LS(l, kLenC) - ok - k0 : LS(l, kLenB) - oj - j0;  // rb or cb
              const int sl = fbs[l][f] >> 4, at = fbs[l][f] & 15;
              const uint32_t j = oj + j0 + (f ? at - 1 : line), k = ok + k0 + (f ? line : at - 1);
              const unsigned long long lin =
                  (static_cast<unsigned long long>(static_cast<uint32_t>(sl)) * static_cast<uint32_t>(LS(l, kLenB) + 1) + j) *
                      static_cast<uint32_t>(LS(l, kLenC) + 1) + k;
              atomicMax(args.out_key + LS(l, kTid), best_key(fbv[l][f], lin));
              fbs[l][f] = -1;
              fbv[l][f] = INT_MIN;
            }
          }
          if constexpr (MODE != kGlobal) {
            // the last thread to leave the item publishes its best and frees the slot
            const int slot = l * SM::kSlots + (LS(l, kItem) & (SM::kSlots - 1));
            __threadfence_block();
            if (atomicAdd(&bcnt[slot], 1u) == static_cast<uint32_t>(T - 1)) {
              __threadfence_block();
              const unsigned long long key = atomicExch(&bkey[slot], 0ull);
              if (key) atomicMax(args.out_key + LS(l, kTid), key);
              bcnt[slot] = 0u;
            }
          }
        }
      }
      if (LANES == 2 && sw[0] && sw[LANES - 1]) {
        // paired switch (the host aligns equal-length items in both lanes)
        const int it0 = LS(0, kItem) + 1, it1 = LS(LANES - 1, kItem) + 1;
        LS(0, kItem) = it0;
        LS(LANES - 1, kItem) = it1;
        const LaneLoad l0 = fetch(0, it0, iend_s[0]);
        const LaneLoad l1 = fetch(LANES - 1, it1, iend_s[LANES - 1]);
        if constexpr (LANES == 2) tables_both(l0, l1);
#pragma unroll
        for (int l = 0; l < LANES; ++l) si[l] = 0;
#pragma unroll
        for (int P = 0; P <= N; ++P)
#pragma unroll
          for (int Q = 0; Q <= N; ++Q) Cu[P][Q] = NEG;
        if constexpr (kPackFaces) paired = lockstep();
      } else {
        [[maybe_unused]] bool switched = false;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (!sw[l]) continue;
          const int it = LS(l, kItem) + 1;
          LS(l, kItem) = it;
          setup(l, it, iend_s[l]);
          si[l] = 0;
          switched = true;
#pragma unroll
          for (int P = 0; P <= N; ++P)
#pragma unroll
            for (int Q = 0; Q <= N; ++Q) Cu[P][Q] = lop_sel(Cu[P][Q], NEG, Ops::mask(l));
        }
        if (kPackFaces && switched) paired = lockstep();
      }
    } else {
      wait_free(s);
      mbar_arrive_group(&mbar[buf]);
    }
    // next slice's s0 word (consumed after the barrier: latency hidden)
#pragma unroll
    for (int l = 0; l < LANES; ++l) {
      const int pos = si[l] - 1;
      s0word[l] = (!(flags[l] & kDone) && pos >= 0 && (!BLOCKS || pos < la[l]))
                      ? __ldg(args.seq + static_cast<uint32_t>(LS(l, kW0)) + (pos >> 4))
                      : 0u;
    }
    // next slice's block faces -> shared staging (cp.async: no registers held)
    if (BLOCKS && (r == 0 || cc == 0)) {
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if ((flags[l] & kDone) || si[l] > la[l]) continue;
        const int a1 = la[l] + 1;
        if constexpr (WAVE) {
          if (!early[l]) wave_prefetch(l, si[l]);  // else issued right after this step's halos
          continue;
        }
        if (kPackFaces && paired && l != 0) continue;  // packed faces: lane 0's buffer only
        const int32_t* fb = args.faces + args.face_off[sbase + l];
        if (r == 0 && (flags[l] & kInTop)) {
          const int32_t* src = fb + (int64_t(LS(l, kOrgK) / GN) * a1 + si[l]) * (GN + 1) + cc * N;
          int32_t* dst = stage + (l * 2 * G + cc) * (N + 1);
#pragma unroll
          for (int q = 0; q <= N; ++q)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(dst + q))),
                         "l"(src + q)
                         : "memory");
        }
        if (cc == 0 && (flags[l] & kInLeft)) {
          const int32_t* src = fb + int64_t(LS(l, kBk)) * a1 * (GN + 1) + int64_t(si[l]) * GN + r * N;
          int32_t* dst = stage + (l * 2 * G + G + r) * (N + 1);
#pragma unroll
          for (int p = 0; p < N; ++p)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(dst + p))),
                         "l"(src + p)
                         : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
}

}  // namespace ta
