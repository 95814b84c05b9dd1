// affine.cuh — the sm_100a wavefront kernel for the AFFINE-gap 3-way
// alignment of SPEC-AFFINE.md (the reference has linear gaps only:
// SPEC.md:99,241; this path is pinned against the builder's own oracle,
// oracle/affine_oracle.c).
//
// Same machine as the linear kernel (wavefront.cuh): a CTA is a G x G grid
// of threads, thread (r, c) owns an N x N tile of the (j, k) plane, tiles
// run an anti-diagonal pipeline over the i-slices of LANES independent
// streams, neighbours exchange boundaries through a double-buffered shared
// mailbox with split mbarrier arrive/wait, long triplets run as sequences
// of block items with faces in global memory.  What changes is the cell:
// seven column-type states instead of one value.  Per cell and slice
//
//   V1 = max(B'(i-1,j-1,k-1) + sop', start)   V2 = E2'(i-1,j-1,k) + s01'
//   V3 = E3'(i-1,j,k-1) + s02'                 V4 = E4(i,j-1,k-1) + s12'
//   V5 = E5'(i-1,j,k)   V6 = E6(i,j-1,k)       V7 = E7(i,j,k-1)
//   B  = max(V1..V7)
//   Et = max(Vt, open + max(Va, Vb), 2 open + B)   ({a,b} = n(t',t) = 1 types)
//
// (primes: previous slice).  A thread keeps B, E2, E3, E5 of its tile for the
// next slice and E4, E6, E7 for the cells to its right / below; the mailbox
// carries (B, E3, E4, E7) of the right column and (B, E4, E2, E6) of the bottom
// row.  14 ALU-pipe (VIADDMNMX / VIMNMX3) + 8 FMA-pipe (IMAD) instructions
// per cell; values are gap-shifted (-2 gap (i+j+k)) and biased by -10 open so
// that every real value is >= 0 and packed s16x2 adds on the FMA pipe are
// exact.  TRACE: values carry a 3-bit type tag (7 - t) in their low bits, the
// maxima select the smallest type on ties (SPEC-AFFINE.md traceback rule), and
// each cell records the tags of V1's source, B and E2..E7 (24 bits).
#pragma once

#include "wavefront.cuh"

namespace ta {

struct AffArgs {
  const uint32_t* __restrict__ seq;
  const TripletDesc* __restrict__ desc;
  const int4* __restrict__ items;
  const int32_t* __restrict__ stream_off;
  const int32_t* __restrict__ cta_steps;
  int32_t* __restrict__ out_score;
  int32_t* __restrict__ out_end;
  unsigned long long* __restrict__ out_key;
  uint32_t* __restrict__ dirs;              // TRACE: per-cell records
  union {
    const int64_t* __restrict__ dir_off;    // TRACE: per triplet, in uint4
    uint64_t epoch;                         // wave mode, score kernels: launch epoch, the high half of the tags
                                            // (TRACE wave launches run once per freshly zeroed plan: epoch 1)
  };
  int32_t match_p, mismatch_p, g2;          // sigma' (= sigma - 2 gap) and 2 gap
  int32_t open;                             // gap_open (<= 0)
  int32_t bias;                             // -8 open
  uint32_t one;
  int32_t* __restrict__ faces;              // block faces, 4 values per position
  const int64_t* __restrict__ face_off;     // blocks: per stream, in words; wave: per triplet, its rings in
                                            // 8-byte entries (the parameter block is kept at its pre-wave size:
                                            // two more fields cost the block kernel 4.5% through ptxas scheduling)
};

constexpr int kAffN = 5;  // tile side of the affine kernel
constexpr int kAffRec = 28;  // TRACE record words per tile-slice (25 cells, padded to 16 B)

// Block faces per stream and triplet (sequential block items):
//   Fdown [Bk][a + 1][GN + 1][4]  (B, E2, E4, E6) of row J*GN - 1, position k + 1
//   Fright[a + 1][GN][4]          (B, E3, E4, E7) of column K*GN - 1, position j
__host__ __device__ inline int64_t aff_face_words(int a, int bk, int gn) {
  return (int64_t(bk) * (a + 1) * (gn + 1) + int64_t(a + 1) * gn) * 4;
}

// Wave mode (blocks of a long triplet on different CTAs, wavefront.cuh's
// scheme): per block a down and a right ring [a + 1][G][kAffSegE] of (value,
// tag) 8-byte entries; a segment holds N + 1 positions x 4 values.
constexpr int kAffSegE = 24;  // 4 x (kAffN + 1) entries = 192 B = 12 x 16 B
__host__ __device__ inline int64_t aff_wave_block_entries(int a, int g) { return int64_t(2) * (a + 1) * g * kAffSegE; }

template <int N, int G, int LANES, int BLK>
struct AffSmem {
  static constexpr int T = G * G;
  static constexpr int NN = N * N;
  // mailbox slot per tile: the right column as (B, E3, E4, E7) per row, then
  // the bottom row as (B, E4, E2, E6) per column (one 16-byte vector per
  // position), padded to 11 vectors so 8 consecutive slots hit distinct banks
  static constexpr int XW = 8 * N + 4;  // 2N + 1 vectors (odd: 8 consecutive slots are bank-conflict free)
  static constexpr size_t kSig = size_t(NN) * T * 4;
  static constexpr size_t kTab = size_t(N) * T * 8;
  static constexpr size_t kX = size_t(2) * XW * (T + 1) * 4;
  static constexpr int kLaneFields = 12;
  static constexpr size_t kLane = size_t(LANES) * kLaneFields * T * 4;
  // prefetched faces: int4 per position (sequential blocks) or tagged ring
  // segments (wave); sized per variant so the L1 carve-out stays as large as
  // possible (the face prefetch of sequential blocks goes through L1)
  static constexpr size_t kStage = BLK == 2 ? size_t(LANES) * 2 * G * kAffSegE * 8 : size_t(LANES) * 2 * G * (N + 1) * 16;
  static constexpr size_t kBar = 16;
  static constexpr int kSlots = 64;
  static constexpr size_t kBest = size_t(LANES) * kSlots * 12;
  static constexpr size_t bytes = kSig + 2 * kTab + kX + kLane + kStage + kBar + kBest;
};

template <int N, int G, int LANES, int MODE, bool TRACE, int BLK>
__global__ void __launch_bounds__(G * G, 1) affine_kernel(const AffArgs args) {
  // BLK: 0 single block, 1 sequential block items, 2 wave mode (tagged rings)
  constexpr bool BLOCKS = BLK != 0;
  constexpr bool WAVE = BLK == 2;
  static_assert(4 * (N + 1) <= kAffSegE, "ring segment too small");
  static_assert(!TRACE || LANES == 1, "TRACE uses int32 lanes");
  using Ops = LaneOps<LANES>;
  using SM = AffSmem<N, G, LANES, BLK>;
  constexpr int T = SM::T;
  constexpr int NN = SM::NN;
  constexpr int XW = SM::XW;
  constexpr int SH = TRACE ? 3 : 0;  // value scale 2^SH (type tags in the low bits)
  constexpr int SC = 1 << SH;
  constexpr uint32_t NEG = TRACE ? 0xF0000000u : Ops::kNeg;
  constexpr uint32_t kDone = 1u, kOwner = 2u;
  constexpr uint32_t kInTop = 8u, kInLeft = 16u, kOutDown = 32u, kOutRight = 64u;
  constexpr int GN = G * N;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* const s12w = reinterpret_cast<uint32_t*>(smem_raw);  // [NN][T]
  unsigned char* const tab1 = smem_raw + SM::kSig;
  unsigned char* const tab2 = tab1 + SM::kTab;
  uint32_t* const xbuf = reinterpret_cast<uint32_t*>(tab2 + SM::kTab);  // [2][T+1][XW]
  int32_t* const lst = reinterpret_cast<int32_t*>(tab2 + SM::kTab + SM::kX);
  int32_t* const stage = reinterpret_cast<int32_t*>(tab2 + SM::kTab + SM::kX + SM::kLane);  // [LANES][2G][N+1][4]
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(tab2 + SM::kTab + SM::kX + SM::kLane + SM::kStage);
  unsigned long long* const bkey = reinterpret_cast<unsigned long long*>(mbar + 2);
  uint32_t* const bcnt = reinterpret_cast<uint32_t*>(bkey + LANES * SM::kSlots);

  const int t = threadIdx.x;
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
  const int skew = r + cc;
  const int g2 = args.g2;
  const int ag2 = -g2;
  const uint32_t one = args.one;
  const uint32_t op1 = Ops::splat(args.open * SC);      // + open   (lane-safe ALU adds)
  // + open / + 2 open as plain 32-bit adds on the FMA pipe: the bias (-10 open)
  // keeps every real V >= 2 |open| and B >= 4 |open|, so subtracting never
  // borrows across the s16x2 lanes (NEG = -16384 per lane stays negative).
  const uint32_t osub1 = LANES == 2 ? 0u - static_cast<uint32_t>(-args.open * SC) * 0x00010001u
                                    : static_cast<uint32_t>(args.open * SC);
  const uint32_t osub2 = LANES == 2 ? 0u - static_cast<uint32_t>(-2 * args.open * SC) * 0x00010001u
                                    : static_cast<uint32_t>(2 * args.open * SC);
  auto LS = [&](int l, int f) -> int32_t& { return lst[(l * SM::kLaneFields + f) * T + t]; };

  for (int w = t; w < 2 * XW; w += T) xbuf[((w / XW) * (T + 1) + T) * XW + w % XW] = NEG;
  for (int w = t; w < LANES * SM::kSlots; w += T) {
    bkey[w] = 0ull;
    bcnt[w] = 0u;
  }
  if (t == 0) {
    mbar_init(&mbar[0], T);
    mbar_init(&mbar[1], T);
  }

  int si[LANES], la[LANES];
  uint32_t s0word[LANES], flags[LANES];

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
    uint32_t c1, c2;
    int mp, mm;
  };

  auto fetch = [&](int l, int it, int iend) -> LaneLoad {
    int id = -1, a_ = 0, b_ = -1, c_ = -1, len = 0x3FFFFFFF, J = 0, K = 0, Bj = 1, Bk = 1;
    uint32_t ww0 = 0, ww1 = 0, ww2 = 0;
    if (it < iend) {
      const int4 rec = __ldg(args.items + it);
      if (WAVE && rec.x < 0) {
        len = rec.z;  // null item (wave partner): idle for len slices
      } else {
      id = rec.x;
      J = rec.y >> 16;
      K = rec.y & 0xFFFF;
      len = rec.z;
      Bj = rec.w >> 16;
      Bk = rec.w & 0xFFFF;
      const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(args.desc + id));
      const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(args.desc + id) + 1);
      a_ = static_cast<int>(d0.x);
      b_ = static_cast<int>(d0.y);
      c_ = static_cast<int>(d0.z);
      ww0 = d1.x;
      ww1 = d1.y;
      ww2 = d1.z;
      }
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
    const int gj0 = J * GN + j0, gk0 = K * GN + k0;
    uint32_t f = (id >= 0 || (WAVE && it < iend)) ? 0u : kDone;
    if (id >= 0 && b_ / N == gj0 / N && c_ / N == gk0 / N && b_ >= gj0 && c_ >= gk0) f |= kOwner;
    if (id >= 0 && J > 0) f |= kInTop;
    if (id >= 0 && K > 0) f |= kInLeft;
    if (id >= 0 && J + 1 < Bj) f |= kOutDown;
    if (id >= 0 && K + 1 < Bk) f |= kOutRight;
    flags[l] = f;
    return LaneLoad{load_codes(ww1, gj0 - 1, b_), load_codes(ww2, gk0 - 1, c_), id >= 0 ? args.match_p : 0,
                    id >= 0 ? args.mismatch_p : 0};
  };

  // sigma' tables of lane l: tab1 / tab2 rows keyed by the s0 code, s12 per cell
  auto tables_lane = [&](int l, const LaneLoad& ld) {
    const uint32_t c1 = ld.c1, c2 = ld.c2;
    const int mp = ld.mp, mm = ld.mm;
    if constexpr (LANES == 1) {
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const uint32_t x1 = (c1 >> (2 * p)) & 3u, x2 = (c2 >> (2 * p)) & 3u;
        uint32_t v1[4], v2[4];
#pragma unroll
        for (int code = 0; code < 4; ++code) {
          v1[code] = static_cast<uint32_t>(code == int(x1) ? mp : mm) & 0xFFFFu;
          v2[code] = static_cast<uint32_t>(code == int(x2) ? mp : mm) & 0xFFFFu;
        }
        reinterpret_cast<uint2*>(tab1)[p * T + t] = make_uint2(v1[0] | (v1[1] << 16), v1[2] | (v1[3] << 16));
        reinterpret_cast<uint2*>(tab2)[p * T + t] = make_uint2(v2[0] | (v2[1] << 16), v2[2] | (v2[3] << 16));
      }
#pragma unroll
      for (int cell = 0; cell < NN; ++cell) {
        const int p = cell / N, q = cell % N;
        s12w[cell * T + t] =
            static_cast<uint32_t>((((c1 >> (2 * p)) & 3u) == ((c2 >> (2 * q)) & 3u) ? mp : mm) * SC);
      }
    } else {
      const uint32_t mm8 = static_cast<uint32_t>(mm) * 0x01010101u;
      const uint32_t dm = static_cast<uint32_t>(mp - mm);
      uint32_t t2w[N];
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const uint32_t x1 = (c1 >> (2 * p)) & 3u, x2 = (c2 >> (2 * p)) & 3u;
        reinterpret_cast<uint32_t*>(tab1)[(p * T + t) * 2 + l] = mm8 + (dm << (8 * x1));
        t2w[p] = mm8 + (dm << (8 * x2));
        reinterpret_cast<uint32_t*>(tab2)[(p * T + t) * 2 + l] = t2w[p];
      }
      uint16_t* s12h = reinterpret_cast<uint16_t*>(s12w);
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const uint32_t x1 = (c1 >> (2 * p)) & 3u;
        const uint32_t sel = x1 | ((x1 | 8u) << 4);
#pragma unroll
        for (int q = 0; q < N; ++q) s12h[(size_t((p * N + q)) * T + t) * 2 + l] = static_cast<uint16_t>(prmt(t2w[q], 0u, sel));
      }
    }
  };

  const int sbase = blockIdx.x * LANES;
#pragma unroll
  for (int l = 0; l < LANES; ++l) {
    const int it = args.stream_off[sbase + l];
    const int ie = args.stream_off[sbase + l + 1];
    LS(l, kItem) = it;
    LS(l, kIEnd) = ie;
    si[l] = 0;
    s0word[l] = 0;
    tables_lane(l, fetch(l, it, ie));
  }
  // Paired lanes (sequential block items only): both lanes hold block items of
  // identical geometry in lockstep (the host pairs equal-shape triplets), so
  // their block faces travel as packed s16x2 words through lane 0's face
  // buffer: one store / prefetch / load per position instead of a per-lane
  // extract, splat and masked merge.  Holds for all blocks of a triplet pair.
  constexpr bool kPackFaces = LANES == 2 && BLK == 1;
  auto lockstep = [&]() -> bool {
    if constexpr (!kPackFaces) {
      return false;
    } else {
      return !(flags[0] & kDone) && !(flags[1] & kDone) && LS(0, kTid) >= 0 && LS(1, kTid) >= 0 &&
             // same slices and block grid: every later block of the two
             // triplets lines up too, so producer and consumer agree on the packing
             si[0] == si[1] && la[0] == la[1] && LS(0, kBj) == LS(1, kBj) && LS(0, kBk) == LS(1, kBk) &&
             LS(0, kOrgJ) == LS(1, kOrgJ) && LS(0, kOrgK) == LS(1, kOrgK) && LS(0, kLen) == LS(1, kLen);
    }
  };
  bool paired = lockstep();

  // B, E2, E3, E5 of the tile (incl. the halo row / column), updated in
  // place: slice i - 1 until the sweep of slice i overwrites a cell (the
  // slice i-1 terms a later cell needs are formed first, see the sweep)
  uint32_t cB[N + 1][N + 1], cE2[N + 1][N + 1], cE3[N + 1][N + 1], cE5[N + 1][N + 1];
#pragma unroll
  for (int P = 0; P <= N; ++P)
#pragma unroll
    for (int Q = 0; Q <= N; ++Q) cB[P][Q] = cE2[P][Q] = cE3[P][Q] = cE5[P][Q] = NEG;

  __syncthreads();

  const int nsteps = args.cta_steps[blockIdx.x];
  for (int s = 0; s < nsteps; ++s) {
    const int buf = s & 1;
    bool any = false;
#pragma unroll
    for (int l = 0; l < LANES; ++l) any |= !(flags[l] & kDone);
    const bool active = s >= skew && any;
    if (s > 0) mbar_wait(&mbar[buf ^ 1], static_cast<uint32_t>((s - 1) >> 1) & 1u);
    if (active) {
      uint32_t cE4[N + 1][N + 1], cE6[N + 1][N + 1], cE7[N + 1][N + 1];
      uint32_t rec[TRACE ? NN : 1];
      // ---- 2. sigma' of this slice's s0 residue against the tile's s1 / s2
      uint32_t sel = 0;
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
          return static_cast<uint32_t>(
              static_cast<int>(reinterpret_cast<const int16_t*>(tab)[(size_t(p) * T + t) * 4 + sel]) * SC);
        } else {
          const uint2 e = reinterpret_cast<const uint2*>(tab)[p * T + t];
          return prmt(e.x, e.y, sel);
        }
      };
      uint32_t s02[N], a1v[N];
#pragma unroll
      for (int q = 0; q < N; ++q) s02[q] = sig_row(tab2, q);
#pragma unroll
      for (int p = 0; p < N; ++p) a1v[p] = sig_row(tab1, p);
      // slice i-1 partial sums of the halo (before this slice's halos replace
      // it): Y[P][Q] = B'(P-1, Q-1) + s01' + s02' (V1), V2[P][Q] = E2'(P-1, Q)
      // + s01', V3[P][Q] = E3'(P, Q-1) + s02'; the sweep forms the interior ones
      uint32_t Y[N + 1][N + 1], V2[N + 1][N + 1], V3[N + 1][N + 1];
#pragma unroll
      for (int Q = 1; Q <= N; ++Q) {
        Y[1][Q] = fma_add(fma_add(cB[0][Q - 1], one, a1v[0]), one, s02[Q - 1]);
        V2[1][Q] = fma_add(cE2[0][Q], one, a1v[0]);
      }
#pragma unroll
      for (int P = 1; P <= N; ++P) {
        if (P > 1) Y[P][1] = fma_add(fma_add(cB[P - 1][0], one, a1v[P - 1]), one, s02[0]);
        V3[P][1] = fma_add(cE3[P][0], one, s02[0]);
      }


      // ---- 1. halos of this slice (published by the neighbours at step s-1)
      const uint4* xin = reinterpret_cast<const uint4*>(xbuf + (buf ^ 1) * XW * (T + 1));
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const uint4 v = xin[up * (XW / 4) + N + q];
        cB[0][q] = v.x;
        cE4[0][q] = v.y;
        cE2[0][q + 1] = v.z;
        cE6[0][q + 1] = v.w;
      }
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const uint4 v = xin[left * (XW / 4) + p];
        cB[p + 1][0] = v.x;
        cE3[p + 1][0] = v.y;
        cE4[p + 1][0] = v.z;
        cE7[p + 1][0] = v.w;
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
          if (kPackFaces && paired) {
            if (r == 0 && (flags[0] & kInTop) && si[0] <= la[0]) {
              const uint4* st = reinterpret_cast<const uint4*>(stage) + cc * (N + 1);
#pragma unroll
              for (int q = 0; q <= N; ++q) {
                const uint4 v = st[q];  // packed (B, E2, E4, E6) at k = cN + q - 1
                if (q < N) {
                  cB[0][q] = v.x;
                  cE4[0][q] = v.z;
                }
                if (q > 0) {
                  cE2[0][q] = v.y;
                  cE6[0][q] = v.w;
                }
              }
            }
            if (cc == 0 && (flags[0] & kInLeft) && si[0] <= la[0]) {
              const uint4* st = reinterpret_cast<const uint4*>(stage) + (G + r) * (N + 1);
#pragma unroll
              for (int p = 0; p < N; ++p) {
                const uint4 v = st[p];  // packed (B, E3, E4, E7) at j = rN + p
                cB[p + 1][0] = v.x;
                cE3[p + 1][0] = v.y;
                cE4[p + 1][0] = v.z;
                cE7[p + 1][0] = v.w;
              }
            }
          } else
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            const bool ok = si[l] <= la[l];
            const uint32_t m = Ops::mask(l);
            if constexpr (WAVE) {
              // tagged rings: only a lane with real cells in this tile waits
              const bool real = LS(l, kTid) >= 0 && LS(l, kLenB) - LS(l, kOrgJ) - j0 >= 0 &&
                                LS(l, kLenC) - LS(l, kOrgK) - k0 >= 0;
              if (!ok || !real) continue;
              const uint32_t want = ((TRACE ? 1u : static_cast<uint32_t>(args.epoch)) << 16) + static_cast<uint32_t>(si[l]) + 1u;
              const uint64_t* fb = reinterpret_cast<const uint64_t*>(args.faces) + args.face_off[LS(l, kTid)];
              const int a1 = la[l] + 1;
              const int blk = (LS(l, kOrgJ) / GN) * LS(l, kBk) + LS(l, kOrgK) / GN;
              const uint2* sv = reinterpret_cast<const uint2*>(stage) + l * 2 * G * kAffSegE;
              // staged entry e of segment seg, re-read from L2 until its tag is fresh
              auto take = [&](int seg, const uint64_t* src, int e) -> int32_t {
                uint2 v = sv[seg * kAffSegE + e];
                while (v.y != want) {
                  v = ld_face(src + e);
                }
                return static_cast<int32_t>(v.x);
              };
              // entries a segment's consumer reads: top (B, E4) at q < N, (E2, E6) at q > 0; left all 4N
              auto used = [](bool top, int e) { return !top || (e % 2 == 0 ? e < 4 * N : e >= 4); };
              // one branch when every used tag is fresh (the common case: see wavefront.cuh)
              auto fresh = [&](int seg, bool top) {
                bool f = true;
#pragma unroll
                for (int e = 0; e < 4 * N + 4; ++e)
                  if (e < (top ? 4 * N + 4 : 4 * N) && used(top, e)) f &= sv[seg * kAffSegE + e].y == want;
                return f;
              };
              auto put_top = [&](auto get) {
#pragma unroll
                for (int q = 0; q <= N; ++q) {  // (B, E2, E4, E6) at k = cN + q - 1
                  if (q < N) {
                    cB[0][q] = lop_sel(cB[0][q], Ops::splat(get(4 * q)), m);
                    cE4[0][q] = lop_sel(cE4[0][q], Ops::splat(get(4 * q + 2)), m);
                  }
                  if (q > 0) {
                    cE2[0][q] = lop_sel(cE2[0][q], Ops::splat(get(4 * q + 1)), m);
                    cE6[0][q] = lop_sel(cE6[0][q], Ops::splat(get(4 * q + 3)), m);
                  }
                }
              };
              auto put_left = [&](auto get) {
#pragma unroll
                for (int p = 0; p < N; ++p) {  // (B, E3, E4, E7) at j = rN + p
                  cB[p + 1][0] = lop_sel(cB[p + 1][0], Ops::splat(get(4 * p)), m);
                  cE3[p + 1][0] = lop_sel(cE3[p + 1][0], Ops::splat(get(4 * p + 1)), m);
                  cE4[p + 1][0] = lop_sel(cE4[p + 1][0], Ops::splat(get(4 * p + 2)), m);
                  cE7[p + 1][0] = lop_sel(cE7[p + 1][0], Ops::splat(get(4 * p + 3)), m);
                }
              };
              if (r == 0 && (flags[l] & kInTop)) {
                const uint64_t* src = fb + ((int64_t(blk - LS(l, kBk)) * 2 * a1 + si[l]) * G + cc) * kAffSegE;
                if (fresh(cc, true))
                  put_top([&](int e) { return static_cast<int32_t>(sv[cc * kAffSegE + e].x); });
                else
                  put_top([&](int e) { return take(cc, src, e); });
              }
              if (cc == 0 && (flags[l] & kInLeft)) {
                const uint64_t* src = fb + (((int64_t(blk - 1) * 2 + 1) * a1 + si[l]) * G + r) * kAffSegE;
                if (fresh(G + r, false))
                  put_left([&](int e) { return static_cast<int32_t>(sv[(G + r) * kAffSegE + e].x); });
                else
                  put_left([&](int e) { return take(G + r, src, e); });
              }
              continue;
            }
            if (r == 0 && (flags[l] & kInTop) && ok) {
              const int4* st = reinterpret_cast<const int4*>(stage) + (l * 2 * G + cc) * (N + 1);
#pragma unroll
              for (int q = 0; q <= N; ++q) {
                const int4 v = st[q];  // (B, E2, E4, E6) at k = cN + q - 1
                if (q < N) {
                  cB[0][q] = lop_sel(cB[0][q], Ops::splat(v.x), m);
                  cE4[0][q] = lop_sel(cE4[0][q], Ops::splat(v.z), m);
                }
                if (q > 0) {
                  cE2[0][q] = lop_sel(cE2[0][q], Ops::splat(v.y), m);
                  cE6[0][q] = lop_sel(cE6[0][q], Ops::splat(v.w), m);
                }
              }
            }
            if (cc == 0 && (flags[l] & kInLeft) && ok) {
              const int4* st = reinterpret_cast<const int4*>(stage) + (l * 2 * G + G + r) * (N + 1);
#pragma unroll
              for (int p = 0; p < N; ++p) {
                const int4 v = st[p];  // (B, E3, E4, E7) at j = rN + p
                cB[p + 1][0] = lop_sel(cB[p + 1][0], Ops::splat(v.x), m);
                cE3[p + 1][0] = lop_sel(cE3[p + 1][0], Ops::splat(v.y), m);
                cE4[p + 1][0] = lop_sel(cE4[p + 1][0], Ops::splat(v.z), m);
                cE7[p + 1][0] = lop_sel(cE7[p + 1][0], Ops::splat(v.w), m);
              }
            }
          }
        }
      }

      // ---- 3. starts (SPEC-AFFINE.md): global origin, semi axis cells, local every cell
      // biased, gap-shifted value of M = 0 at (i, j, k): bias + |g2| (i + j + k)
      uint32_t stbase = NEG;  // local: start value of the tile's cell (1, 1)
      uint32_t fcorner = NEG;
      bool force = false;
      // semi slice-0 axis starts of row P = 1 / column Q = 1: packed base +
      // per-cell step (NEG / 0 in lanes that force nothing), folded into the
      // one sweep (see wavefront.cuh)
      uint32_t frb = NEG, fcb = NEG, frs = 0u, fcs = 0u;
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        const bool live = !(flags[l] & kDone);
        const int oj = LS(l, kOrgJ), ok = LS(l, kOrgK);
        if constexpr (MODE == kGlobal) {
          if (t == 0 && live && si[l] == 0 && oj == 0 && ok == 0)
            fcorner = lop_sel(fcorner, Ops::splat(args.bias * SC + (SC - 1)), Ops::mask(l));
        } else if constexpr (MODE == kSemi) {
          if (t == 0 && live && oj == 0 && ok == 0 && si[l] <= la[l])
            fcorner = lop_sel(fcorner, Ops::splat((args.bias + ag2 * si[l]) * SC + (SC - 1)), Ops::mask(l));
          force |= live && si[l] == 0 && ((r == 0 && oj == 0) || (cc == 0 && ok == 0));
        } else {
          stbase = lop_sel(stbase, Ops::splat((args.bias + ag2 * (si[l] + oj + ok + j0 + k0)) * SC + (SC - 1)),
                           Ops::mask(l));
        }
      }
      if constexpr (MODE == kSemi) {
        if (force) {
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            const int oj = LS(l, kOrgJ), ok = LS(l, kOrgK);
            if ((flags[l] & kDone) || si[l] != 0) continue;
            if (r == 0 && oj == 0) {
              frb = lop_sel(frb, Ops::splat((args.bias + ag2 * (ok + k0)) * SC + (SC - 1)), Ops::mask(l));
              frs = lop_sel(frs, Ops::splat(ag2 * SC), Ops::mask(l));
            }
            if (cc == 0 && ok == 0) {
              fcb = lop_sel(fcb, Ops::splat((args.bias + ag2 * (oj + j0)) * SC + (SC - 1)), Ops::mask(l));
              fcs = lop_sel(fcs, Ops::splat(ag2 * SC), Ops::mask(l));
            }
          }
        }
      }
      const uint32_t ag2s = Ops::splat(ag2 * SC);

      // ---- 4. the tile -------------------------------------------------------
      // Cells in anti-diagonal order (d = P + Q), as in the linear sweep:
      // consecutive cells are independent, so the E7 -> B -> E7 chain along a
      // row and E6 along a column are several cells apart in the schedule.
      auto sweep = [&]() {
        [[maybe_unused]] uint32_t sd = stbase;  // local: start value of diagonal d (depends on P + Q only)
        [[maybe_unused]] uint32_t frv = frb, fcv = fcb;  // semi: row-1 cells come with Q, column-1 cells with P increasing
#pragma unroll
        for (int d = 0; d <= 2 * N - 2; ++d) {
          if constexpr (MODE == kLocal) {
            if (d > 0) sd = fma_add(sd, one, ag2s);
          }
#pragma unroll
          for (int P0 = 0; P0 < N; ++P0) {
            const int Q0 = d - P0;
            if (Q0 < 0 || Q0 >= N) continue;
            const int P = P0 + 1, Q = Q0 + 1;
            const int cell = (P - 1) * N + (Q - 1);
            const uint32_t sg = s12w[cell * T + t];
            // start value of this cell (NEG where no alignment may start)
            uint32_t start = NEG;
            if constexpr (MODE == kLocal) {
              start = sd;
            } else {
              if (P == 1 && Q == 1) start = fcorner;
              if constexpr (MODE == kSemi) {
                if (P == 1) {
                  start = Ops::max2(start, frv);
                  if (Q < N) frv = fma_add(frv, one, frs);
                }
                if (Q == 1) {
                  start = Ops::max2(start, fcv);
                  if (P < N) fcv = fma_add(fcv, one, fcs);
                }
              }
            }
            // slice i-1 values of this cell: form the partial sums the later
            // cells need, so the cell can be overwritten in place
            const uint32_t oB = cB[P][Q], oE2 = cE2[P][Q], oE3 = cE3[P][Q];
            if (P < N && Q < N) Y[P + 1][Q + 1] = fma_add(fma_add(oB, one, a1v[P]), one, s02[Q]);
            if (P < N) V2[P + 1][Q] = fma_add(oE2, one, a1v[P]);
            if (Q < N) V3[P][Q + 1] = fma_add(oE3, one, s02[Q]);
            // no start possible here (global: all but the origin cell; semi:
            // off row / column 1): V1 is a plain packed add on the FMA pipe
            // (Y >= NEG-derived, sg >= 0: the clamp at NEG never binds)
            const bool no_start = MODE == kGlobal ? (P > 1 || Q > 1) : MODE == kSemi ? (P > 1 && Q > 1) : false;
            uint32_t v1 = no_start ? fma_add(Y[P][Q], one, sg) : Ops::addmax(Y[P][Q], sg, start);
            uint32_t v2 = V2[P][Q];
            uint32_t v3 = V3[P][Q];
            uint32_t v4 = fma_add(cE4[P - 1][Q - 1], one, sg);
            uint32_t v5 = cE5[P][Q];
            uint32_t v6 = cE6[P - 1][Q];
            uint32_t v7 = cE7[P][Q - 1];
            [[maybe_unused]] uint32_t rc = 0;
            if constexpr (TRACE) {
              // record the source tags, then re-tag every V_t with its own type
              rc = (v1 & 7u) | ((v2 & 7u) << 6) | ((v3 & 7u) << 9) | ((v4 & 7u) << 12) | ((v5 & 7u) << 15) |
                   ((v6 & 7u) << 18) | ((v7 & 7u) << 21);
              v1 = (v1 & ~7u) | 6u;
              v2 = (v2 & ~7u) | 5u;
              v3 = (v3 & ~7u) | 4u;
              v4 = (v4 & ~7u) | 3u;
              v5 = (v5 & ~7u) | 2u;
              v6 = (v6 & ~7u) | 1u;
              v7 = v7 & ~7u;
            }
            const uint32_t b = Ops::max3(Ops::max3(Ops::max3(v1, v2, v3), v4, v5), v6, v7);
            // E_t = max(V_t, open + V_a, open + V_b, 2 open + B) ({a, b}: the
            // n = 1 types of t).  Every E_t takes b2, and every open + V_a
            // appears in two E_t, so four of them are fused with b2 once
            // (p_a = max(V_a + open, b2), one VIADDMNMX) and each E_t is one
            // VIMNMX3 of three shared terms: 10 ALU + 2 FMA for the six E_t
            // instead of 12 + 4; the candidate sets, hence the (tagged)
            // maxima, are unchanged.
            const uint32_t b2 = fma_add(b, one, osub2);
            const uint32_t p2 = Ops::addmax(v2, op1, b2), p4 = Ops::addmax(v4, op1, b2);
            const uint32_t p5 = Ops::addmax(v5, op1, b2), p7 = Ops::addmax(v7, op1, b2);
            const uint32_t w3 = fma_add(v3, one, osub1), w6 = fma_add(v6, one, osub1);
            cB[P][Q] = b;
            cE2[P][Q] = Ops::max3(v2, p5, w6);  // v2, open + v5, open + v6, b2
            cE3[P][Q] = Ops::max3(v3, p5, p7);  // v3, open + v5, open + v7, b2
            cE4[P][Q] = Ops::max3(v4, w6, p7);  // v4, open + v6, open + v7, b2
            cE5[P][Q] = Ops::max3(v5, p2, w3);  // v5, open + v2, open + v3, b2
            cE6[P][Q] = Ops::max3(v6, p2, p4);  // v6, open + v2, open + v4, b2
            cE7[P][Q] = Ops::max3(v7, w3, p4);  // v7, open + v3, open + v4, b2
            if constexpr (TRACE) rec[cell] = rc | ((b & 7u) << 3);
          }
        }
      };
      sweep();

      // ---- 5. publish right column / bottom row -----------------------------
      uint4* xout = reinterpret_cast<uint4*>(xbuf + buf * XW * (T + 1)) + tile * (XW / 4);
#pragma unroll
      for (int p = 0; p < N; ++p) xout[p] = make_uint4(cB[p + 1][N], cE3[p + 1][N], cE4[p + 1][N], cE7[p + 1][N]);
#pragma unroll
      for (int q = 0; q < N; ++q) xout[N + q] = make_uint4(cB[N][q], cE4[N][q], cE2[N][q + 1], cE6[N][q + 1]);
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
            const uint32_t tag = ((TRACE ? 1u : static_cast<uint32_t>(args.epoch)) << 16) + static_cast<uint32_t>(si[l]) + 1u;
            uint2* fb = reinterpret_cast<uint2*>(reinterpret_cast<uint64_t*>(args.faces) + args.face_off[LS(l, kTid)]);
            const int blk = (LS(l, kOrgJ) / GN) * LS(l, kBk) + LS(l, kOrgK) / GN;
            auto put = [&](uint2* d, int e, uint32_t v) { st_face(d + e, static_cast<uint32_t>(Ops::lane(v, l)), tag); };
            if (dn) {  // segment cc: q = 0 is the corner (this tile's halo), q = 1..N its bottom row
              uint2* d = fb + ((int64_t(blk) * 2 * a1 + si[l]) * G + cc) * kAffSegE;
              put(d, 0, cB[N][0]);
              put(d, 2, cE4[N][0]);
#pragma unroll
              for (int q = 1; q <= N; ++q) {
                put(d, 4 * q, cB[N][q]);
                put(d, 4 * q + 1, cE2[N][q]);
                put(d, 4 * q + 2, cE4[N][q]);
                put(d, 4 * q + 3, cE6[N][q]);
              }
            }
            if (rt) {  // segment r: positions p = 0..N-1 of this tile's right column
              uint2* d = fb + (((int64_t(blk) * 2 + 1) * a1 + si[l]) * G + r) * kAffSegE;
#pragma unroll
              for (int p = 0; p < N; ++p) {
                put(d, 4 * p, cB[p + 1][N]);
                put(d, 4 * p + 1, cE3[p + 1][N]);
                put(d, 4 * p + 2, cE4[p + 1][N]);
                put(d, 4 * p + 3, cE7[p + 1][N]);
              }
            }
            continue;
          }
          if (kPackFaces && paired) {  // lane 0's buffer, both lanes packed; once
            if (l != 0) continue;
            uint4* fb = reinterpret_cast<uint4*>(args.faces + args.face_off[sbase]);
            if (dn) {
              uint4* d = fb + (int64_t(LS(0, kOrgK) / GN) * a1 + si[0]) * (GN + 1) + cc * N;
              if (cc == 0) d[0] = make_uint4(cB[N][0], 0u, cE4[N][0], 0u);
#pragma unroll
              for (int q = 1; q <= N; ++q) d[q] = make_uint4(cB[N][q], cE2[N][q], cE4[N][q], cE6[N][q]);
            }
            if (rt) {
              uint4* d = fb + int64_t(LS(0, kBk)) * a1 * (GN + 1) + int64_t(si[0]) * GN + r * N;
#pragma unroll
              for (int p = 0; p < N; ++p) d[p] = make_uint4(cB[p + 1][N], cE3[p + 1][N], cE4[p + 1][N], cE7[p + 1][N]);
            }
            wrote = true;
            continue;
          }
          int4* fb = reinterpret_cast<int4*>(args.faces + args.face_off[sbase + l]);
          if (dn) {  // own cells Q = 1..N at positions cN + Q; tile 0 also the corner (its halo)
            int4* d = fb + (int64_t(LS(l, kOrgK) / GN) * a1 + si[l]) * (GN + 1) + cc * N;
            if (cc == 0)
              d[0] = make_int4(Ops::lane(cB[N][0], l), 0, Ops::lane(cE4[N][0], l), 0);
#pragma unroll
            for (int q = 1; q <= N; ++q)
              d[q] = make_int4(Ops::lane(cB[N][q], l), Ops::lane(cE2[N][q], l), Ops::lane(cE4[N][q], l),
                               Ops::lane(cE6[N][q], l));
          }
          if (rt) {
            int4* d = fb + int64_t(LS(l, kBk)) * a1 * (GN + 1) + int64_t(si[l]) * GN + r * N;
#pragma unroll
            for (int p = 0; p < N; ++p)
              d[p] = make_int4(Ops::lane(cB[p + 1][N], l), Ops::lane(cE3[p + 1][N], l), Ops::lane(cE4[p + 1][N], l),
                               Ops::lane(cE7[p + 1][N], l));
          }
          wrote = true;
        }
        if (wrote) __threadfence_block();
      }
      mbar_arrive_group(&mbar[buf]);

      // ---- 6. traceback records (int32 lanes) --------------------------------
      if constexpr (TRACE) {
        if (!(flags[0] & kDone) && si[0] <= la[0]) {
          const int a1 = la[0] + 1;
          const int blk = (LS(0, kOrgJ) / GN) * LS(0, kBk) + LS(0, kOrgK) / GN;
          uint4* dst = reinterpret_cast<uint4*>(args.dirs) + args.dir_off[LS(0, kTid)] +
                       ((size_t(blk) * a1 + si[0]) * T + tile) * (kAffRec / 4);
#pragma unroll
          for (int v = 0; v < kAffRec / 4; ++v)
            dst[v] = make_uint4(rec[min(4 * v, NN - 1)], 4 * v + 1 < NN ? rec[4 * v + 1] : 0u,
                                4 * v + 2 < NN ? rec[4 * v + 2] : 0u, 4 * v + 3 < NN ? rec[4 * v + 3] : 0u);
        }
      }

      // ---- 7. score extraction -------------------------------------------------
      // M = (value >> SH) - bias + g2 (i + j + k)
      if constexpr (MODE == kGlobal) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if ((flags[l] & kOwner) && si[l] == la[l]) {
            const int Bn = LS(l, kLenB), Cn = LS(l, kLenC), id = LS(l, kTid);
            const int want = (Bn - LS(l, kOrgJ) - j0 + 1) * (N + 1) + (Cn - LS(l, kOrgK) - k0 + 1);
            uint32_t v = 0;
#pragma unroll
            for (int P = 1; P <= N; ++P)
#pragma unroll
              for (int Q = 1; Q <= N; ++Q)
                if (P * (N + 1) + Q == want) v = cB[P][Q];
            args.out_score[id] = (Ops::lane(v, l) >> SH) - args.bias + g2 * (la[l] + Bn + Cn);
            args.out_end[3 * id] = la[l];
            args.out_end[3 * id + 1] = Bn;
            args.out_end[3 * id + 2] = Cn;
          }
        }
      } else {
        // candidates: local every real cell, semi the faces i == a, j == b, k == c;
        // padding cells (j > b or k > c) are masked (the affine opens break the
        // linear kernel's "padding never wins" argument)
        const uint32_t g2s = Ops::splat(g2 * SC);
        int rb[LANES], cb[LANES];
        bool full[LANES], face[LANES];
        bool anyfull = false, anyface = false, edge = false;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          rb[l] = LS(l, kLenB) - LS(l, kOrgJ) - j0;
          cb[l] = LS(l, kLenC) - LS(l, kOrgK) - k0;
          const bool inside = !(flags[l] & kDone) && si[l] <= la[l] && rb[l] >= 0 && cb[l] >= 0;
          full[l] = inside && (MODE == kLocal || si[l] == la[l]);
          face[l] = MODE == kSemi && inside && !full[l] && (rb[l] < N || cb[l] < N);
          anyfull |= full[l];
          anyface |= face[l];
          edge |= full[l] && (rb[l] < N - 1 || cb[l] < N - 1);
        }
        auto key_of = [](int mval, unsigned long long lin) -> unsigned long long { return best_key(mval, lin); };
        auto lin_of = [&](int l, int P, int Q) -> unsigned long long {
          const uint32_t j = LS(l, kOrgJ) + j0 + P - 1, k = LS(l, kOrgK) + k0 + Q - 1;
          return (static_cast<unsigned long long>(static_cast<uint32_t>(si[l])) * static_cast<uint32_t>(LS(l, kLenB) + 1) + j) *
                     static_cast<uint32_t>(LS(l, kLenC) + 1) + k;
        };
        auto slot_of = [&](int l) { return l * SM::kSlots + (LS(l, kItem) & (SM::kSlots - 1)); };
        auto may_beat = [&](int l, int mval) -> bool {
          const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(&bkey[slot_of(l)]);
          return key_of(mval, lin_of(l, 1, 1)) > cur;
        };
        // global RED.MAX.64 + shared filter hint (see wavefront.cuh)
        auto offer = [&](int l, int mval, int P, int Q) {
          const unsigned long long key = key_of(mval, lin_of(l, P, Q));
          atomicMax(args.out_key + LS(l, kTid), key);
          volatile unsigned long long* hint = &bkey[slot_of(l)];
          if (key > *hint) *hint = key;
        };
        // value of cell (P, Q) for the scans: padding masked to NEG
        auto cellv = [&](int P, int Q) -> uint32_t {
          uint32_t m = 0xFFFFFFFFu;
          if (edge) {
            m = 0;
#pragma unroll
            for (int l = 0; l < LANES; ++l)
              if (P - 1 <= rb[l] && Q - 1 <= cb[l]) m |= Ops::mask(l);
          }
          return lop_sel(NEG, cB[P][Q], m);
        };
        if (anyfull) {
          uint32_t stepmax = NEG, rowacc[N];
#pragma unroll
          for (int P = N; P >= 1; --P) {
            uint32_t acc = cellv(P, N);
#pragma unroll
            for (int Q = N - 1; Q >= 1; --Q) acc = Ops::addmax(acc, g2s, cellv(P, Q));
            rowacc[P - 1] = acc;
            stepmax = P == N ? acc : Ops::addmax(stepmax, g2s, acc);
          }
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            if (!full[l]) continue;
            const int sm = Ops::lane(stepmax, l) >> SH;
            const int mval = sm - args.bias + g2 * (si[l] + LS(l, kOrgJ) + LS(l, kOrgK) + j0 + k0);
            if (may_beat(l, mval)) {
              // first row attaining the maximum (its masked row max), then the
              // first real cell of that row (selected with a SEL chain)
              int fp = 0;
#pragma unroll
              for (int P = N; P >= 1; --P)
                if ((Ops::lane(rowacc[P - 1], l) >> SH) + g2 * (P - 1) == sm) fp = P;
              int fq = 0;
#pragma unroll
              for (int Q = N; Q >= 1; --Q) {
                uint32_t v = cB[1][Q];
#pragma unroll
                for (int P = 2; P <= N; ++P) v = fp == P ? cB[P][Q] : v;
                if (Q - 1 <= cb[l] && (Ops::lane(v, l) >> SH) + g2 * (fp - 1 + Q - 1) == sm) fq = Q;
              }
              offer(l, mval, fp, fq);
            }
          }
        }
        if constexpr (MODE == kSemi) {
          if (anyface) {
#pragma unroll
            for (int l = 0; l < LANES; ++l) {
              if (!face[l]) continue;
              const int base = -args.bias + g2 * (si[l] + LS(l, kOrgJ) + LS(l, kOrgK) + j0 + k0);
              const int rbl = rb[l], cbl = cb[l];
              // the face row (P = rb + 1, real cells Q - 1 <= cb) and column
              // (Q = cb + 1, P - 1 <= rb), selected with SEL chains and scanned
              // once: row first, then the column cells that come earlier in
              // row-major order win ties
              uint32_t fr[N], fc[N];
#pragma unroll
              for (int x = 1; x <= N; ++x) {
                uint32_t vr = cB[1][x], vc = cB[x][1];
#pragma unroll
                for (int y = 2; y <= N; ++y) {
                  vr = rbl == y - 1 ? cB[y][x] : vr;
                  vc = cbl == y - 1 ? cB[x][y] : vc;
                }
                fr[x - 1] = vr;
                fc[x - 1] = vc;
              }
              int bv = 0, bp = 0, bq = 0;
              bool have = false;
              if (rbl < N) {
#pragma unroll
                for (int Q = 1; Q <= N; ++Q) {
                  const int v = (Ops::lane(fr[Q - 1], l) >> SH) + g2 * (rbl + Q - 1);
                  if (Q - 1 <= cbl && (!have || v > bv)) bv = v, bp = rbl + 1, bq = Q, have = true;
                }
              }
              if (cbl < N) {
#pragma unroll
                for (int P = 1; P <= N; ++P) {
                  const int v = (Ops::lane(fc[P - 1], l) >> SH) + g2 * (P - 1 + cbl);
                  if (P - 1 <= rbl && (!have || v > bv || (v == bv && P < bp))) bv = v, bp = P, bq = cbl + 1, have = true;
                }
              }
              if (have && may_beat(l, bv + base)) offer(l, bv + base, bp, bq);
            }
          }
        }
      }

      // ---- 9. advance the lanes ---------------------------------------------------
      [[maybe_unused]] bool switched = false;
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if (flags[l] & kDone) continue;
        si[l] += 1;
        const bool sw = BLOCKS ? si[l] >= LS(l, kLen) : si[l] > la[l];
        if (!sw) continue;
        if constexpr (MODE != kGlobal) {
          const int slot = l * SM::kSlots + (LS(l, kItem) & (SM::kSlots - 1));
          __threadfence_block();
          if (atomicAdd(&bcnt[slot], 1u) == static_cast<uint32_t>(T - 1)) {
            __threadfence_block();
            const unsigned long long key = atomicExch(&bkey[slot], 0ull);
            if (key) atomicMax(args.out_key + LS(l, kTid), key);
            bcnt[slot] = 0u;
          }
        }
        const int it = LS(l, kItem) + 1;
        LS(l, kItem) = it;
        tables_lane(l, fetch(l, it, LS(l, kIEnd)));
        si[l] = 0;
        switched = true;
#pragma unroll
        for (int P = 0; P <= N; ++P)
#pragma unroll
          for (int Q = 0; Q <= N; ++Q) {
            cB[P][Q] = lop_sel(cB[P][Q], NEG, Ops::mask(l));
            cE2[P][Q] = lop_sel(cE2[P][Q], NEG, Ops::mask(l));
            cE3[P][Q] = lop_sel(cE3[P][Q], NEG, Ops::mask(l));
            cE5[P][Q] = lop_sel(cE5[P][Q], NEG, Ops::mask(l));
          }
      }
      if (kPackFaces && switched) paired = lockstep();
    } else {
      mbar_arrive_group(&mbar[buf]);
    }
    // next slice's s0 word
#pragma unroll
    for (int l = 0; l < LANES; ++l) {
      const int pos = si[l] - 1;
      s0word[l] = (!(flags[l] & kDone) && pos >= 0 && (!BLOCKS || pos < la[l]))
                      ? __ldg(args.seq + static_cast<uint32_t>(LS(l, kW0)) + (pos >> 4))
                      : 0u;
    }
    // next slice's block faces -> shared staging (16 B per position)
    if (BLOCKS && (r == 0 || cc == 0)) {
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if ((flags[l] & kDone) || si[l] > la[l]) continue;
        const int a1 = la[l] + 1;
        if constexpr (WAVE) {
          if (LS(l, kTid) < 0 || !(flags[l] & (kInTop | kInLeft))) continue;
          const uint64_t* fw = reinterpret_cast<const uint64_t*>(args.faces) + args.face_off[LS(l, kTid)];
          const int blk = (LS(l, kOrgJ) / GN) * LS(l, kBk) + LS(l, kOrgK) / GN;
          auto fetch_seg = [&](int seg, const uint64_t* src) {
            uint64_t* dst = reinterpret_cast<uint64_t*>(stage) + (l * 2 * G + seg) * kAffSegE;
#pragma unroll
            for (int v = 0; v < kAffSegE / 2; ++v)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                               static_cast<uint32_t>(__cvta_generic_to_shared(dst + 2 * v))),
                           "l"(src + 2 * v)
                           : "memory");
          };
          if (r == 0 && (flags[l] & kInTop))
            fetch_seg(cc, fw + ((int64_t(blk - LS(l, kBk)) * 2 * a1 + si[l]) * G + cc) * kAffSegE);
          if (cc == 0 && (flags[l] & kInLeft))
            fetch_seg(G + r, fw + (((int64_t(blk - 1) * 2 + 1) * a1 + si[l]) * G + r) * kAffSegE);
          continue;
        }
        if (kPackFaces && paired && l != 0) continue;  // packed faces: lane 0's buffer only
        const int4* fb = reinterpret_cast<const int4*>(args.faces + args.face_off[sbase + l]);
        if (r == 0 && (flags[l] & kInTop)) {
          const int4* src = fb + (int64_t(LS(l, kOrgK) / GN) * a1 + si[l]) * (GN + 1) + cc * N;
          int4* dst = reinterpret_cast<int4*>(stage) + (l * 2 * G + cc) * (N + 1);
#pragma unroll
          for (int q = 0; q <= N; ++q)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(dst + q))),
                         "l"(src + q)
                         : "memory");
        }
        if (cc == 0 && (flags[l] & kInLeft)) {
          const int4* src = fb + int64_t(LS(l, kBk)) * a1 * (GN + 1) + int64_t(si[l]) * GN + r * N;
          int4* dst = reinterpret_cast<int4*>(stage) + (l * 2 * G + G + r) * (N + 1);
#pragma unroll
          for (int p = 0; p < N; ++p)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
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
