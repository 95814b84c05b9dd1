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
//    The tile lives in registers; the previous i-slice is kept alongside.
//  * Anti-diagonal pipeline (tiled.hpp:386-388): thread (r, c) computes
//    stream position s - r - c at step s.  Each CTA owns LANES independent
//    "slice streams" (the concatenated slices of the triplets assigned to
//    it), so the pipeline fills once per CTA, not once per triplet.
//  * LANES = 2 packs two independent triplet streams into s16x2 registers:
//    one VIADDMNMX.S16x2 / VIMNMX3.S16x2 advances two triplets.
//  * Scores are computed in a gap-shifted space M' = M - g2*(i+j+k)
//    (g2 = 2*gap), which zeroes the weight of the three single-residue
//    terms: 6 instructions per cell (IADD3 + 4 VIADDMNMX + VIMNMX3).
//  * Neighbour boundaries (right column / down row + corner) go through a
//    double-buffered shared-memory mailbox, one __syncthreads per step.
//  * Exactness: all arithmetic is integer; lane width is chosen by the host
//    from a proven bound, so results are bit-identical to the reference.
#pragma once

#include <cstdint>

namespace ta {

constexpr int kGlobal = 0;
constexpr int kSemi = 1;
constexpr int kLocal = 2;

// Direction tags carried in the 4 low bits of TRACE values.  Larger tag wins
// ties, so the max selects the FIRST term of Eq. 1 in listed order
// (oracle.cpp:124-144).  15 = local-mode floor (stop, oracle.cpp:109-110).
constexpr uint32_t kTagT1 = 12, kTagT2 = 5, kTagT3 = 4, kTagT4 = 3;
constexpr uint32_t kTagT5 = 2, kTagT6 = 1, kTagT7 = 0, kTagStop = 15;

struct TripletDesc {
  int32_t a, b, c, flags;
  uint32_t w0, w1, w2, pad;  // word offsets of s0/s1/s2 in the packed array
};

struct WaveArgs {
  const uint32_t* __restrict__ seq;        // 2-bit packed, 16 bases per word
  const TripletDesc* __restrict__ desc;
  const int32_t* __restrict__ items;       // stream item lists (triplet ids)
  const int32_t* __restrict__ stream_off;  // [gridDim.x * LANES + 1]
  const int32_t* __restrict__ cta_steps;   // [gridDim.x]
  int32_t* __restrict__ out_score;
  int32_t* __restrict__ out_end;           // 3 per triplet
  unsigned long long* __restrict__ out_key;  // semi/local (value, lex index)
  uint4* __restrict__ dirs;                // TRACE: direction cube
  const int64_t* __restrict__ dir_off;     // TRACE: per triplet, in uint4
  int32_t match_p;                         // sigma' of equal residues   (match - g2)
  int32_t mismatch_p;                      // sigma' of unequal residues (mismatch - g2)
  int32_t g2;                              // 2 * gap (<= 0)
};

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

template <int N, int G, int LANES>
struct WaveSmem {
  static constexpr int T = G * G;
  static constexpr int NN = N * N;
  static constexpr int XW = 2 * N + 1;
  static constexpr size_t kSig = size_t(NN) * T * 4;      // sigma12 per cell
  static constexpr size_t kTab = size_t(N) * T * 8;       // per table (8 B per (row, thread))
  static constexpr size_t kX = size_t(2) * XW * (T + 1) * 4;
  static constexpr size_t bytes = kSig + 2 * kTab + kX;
};

// ---------------------------------------------------------------------------
template <int N, int G, int LANES, int MODE, bool TRACE>
__global__ void __launch_bounds__(G * G, 1) wavefront_kernel(const WaveArgs args) {
  static_assert(!TRACE || LANES == 1, "direction cube uses int32 lanes");
  static_assert((N * N) % 4 == 0, "tile cells must group by 4");
  static_assert(!TRACE || (N * N) <= 128, "direction slot is 64 B per tile-slice");
  using Ops = LaneOps<LANES>;
  using SM = WaveSmem<N, G, LANES>;
  constexpr int T = SM::T;
  constexpr int NN = SM::NN;
  constexpr int XW = SM::XW;
  constexpr int SH = TRACE ? 4 : 0;  // value scale 2^SH (tags in low bits)
  constexpr uint32_t NEG = TRACE ? 0xF0000000u : Ops::kNeg;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4* const s12v = reinterpret_cast<uint4*>(smem_raw);                         // [NN/4][T]
  uint32_t* const s12w = reinterpret_cast<uint32_t*>(smem_raw);
  unsigned char* const tab1 = smem_raw + SM::kSig;                                // 8 B per (p, t)
  unsigned char* const tab2 = tab1 + SM::kTab;
  uint32_t* const xbuf = reinterpret_cast<uint32_t*>(tab2 + SM::kTab);            // [2][XW][T+1]

  const int t = threadIdx.x;
  const int r = t / G;
  const int cc = t - r * G;
  const int j0 = r * N;
  const int k0 = cc * N;
  const int left = cc ? t - 1 : T;
  const int up = r ? t - G : T;
  const int skew = r + cc;
  const int g2 = args.g2;
  const int ag2 = -g2;

  for (int w = t; w < 2 * XW; w += T) xbuf[w * (T + 1) + T] = NEG;

  // ---- per-lane stream state ---------------------------------------------
  int item[LANES], iend[LANES], tid[LANES], si[LANES], la[LANES], lb[LANES], lc[LANES];
  uint32_t w0[LANES], s0word[LANES];
  bool done[LANES];
  int bestv[LANES];
  uint32_t bestlin[LANES];
  bool bestok[LANES];

  // Builds this thread's sigma tables for lane l (triplet id, or -1 = null
  // lane with all-zero weights, which keeps an idle lane bounded).
  auto setup = [&](int l, int id) {
    int a_ = 0x3FFFFFFF, b_ = -1, c_ = -1;
    uint32_t ww1 = 0, ww2 = 0;
    if (id >= 0) {
      const TripletDesc d = args.desc[id];
      a_ = d.a;
      b_ = d.b;
      c_ = d.c;
      w0[l] = d.w0;
      ww1 = d.w1;
      ww2 = d.w2;
    }
    la[l] = a_;
    lb[l] = b_;
    lc[l] = c_;
    const int mp = id >= 0 ? args.match_p : 0;
    const int mm = id >= 0 ? args.mismatch_p : 0;
    int x1[N], x2[N];
#pragma unroll
    for (int p = 0; p < N; ++p) x1[p] = base_at(args.seq, ww1, j0 + p - 1, b_);
#pragma unroll
    for (int q = 0; q < N; ++q) x2[q] = base_at(args.seq, ww2, k0 + q - 1, c_);
#pragma unroll
    for (int p = 0; p < N; ++p) {
#pragma unroll
      for (int code = 0; code < 4; ++code) {
        const int v1 = code == x1[p] ? mp : mm;
        const int v2 = code == x2[p] ? mp : mm;
        if constexpr (LANES == 1) {
          reinterpret_cast<int16_t*>(tab1)[(p * 4 + code) * T + t] = static_cast<int16_t>(v1);
          reinterpret_cast<int16_t*>(tab2)[(p * 4 + code) * T + t] = static_cast<int16_t>(v2);
        } else {
          tab1[(size_t(p) * T + t) * 8 + l * 4 + code] = static_cast<unsigned char>(v1);
          tab2[(size_t(p) * T + t) * 8 + l * 4 + code] = static_cast<unsigned char>(v2);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < N; ++p) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const int cell = p * N + q;
        const int v = x1[p] == x2[q] ? mp : mm;
        const size_t word = size_t(cell >> 2) * T * 4 + size_t(t) * 4 + (cell & 3);
        if constexpr (LANES == 1) {
          s12w[word] = static_cast<uint32_t>(TRACE ? (v * 16 + static_cast<int>(kTagT4)) : v);
        } else {
          reinterpret_cast<uint16_t*>(s12w)[word * 2 + l] = static_cast<uint16_t>(v);
        }
      }
    }
  };

  const int sbase = blockIdx.x * LANES;
#pragma unroll
  for (int l = 0; l < LANES; ++l) {
    item[l] = args.stream_off[sbase + l];
    iend[l] = args.stream_off[sbase + l + 1];
    si[l] = 0;
    bestok[l] = false;
    bestv[l] = 0;
    bestlin[l] = 0;
    s0word[l] = 0;
    w0[l] = 0;
    if (item[l] < iend[l]) {
      tid[l] = args.items[item[l]];
      done[l] = false;
      setup(l, tid[l]);
    } else {
      tid[l] = -1;
      done[l] = true;
      setup(l, -1);
    }
  }

  uint32_t Pv[N + 1][N + 1];
#pragma unroll
  for (int P = 0; P <= N; ++P)
#pragma unroll
    for (int Q = 0; Q <= N; ++Q) Pv[P][Q] = NEG;

  // column constants
  uint32_t colc[N];   // local floor: |g2| * (Q-1)        (x 2^SH)
  uint32_t cold[N];   // best tracking: g2 * (Q-1)       (x 2^SH)
#pragma unroll
  for (int q = 0; q < N; ++q) {
    colc[q] = Ops::splat((ag2 * q) << SH);
    cold[q] = Ops::splat((g2 * q) << SH);
  }

  __syncthreads();

  const int nsteps = args.cta_steps[blockIdx.x];
  for (int s = 0; s < nsteps; ++s) {
    const int buf = s & 1;
    bool any = false;
#pragma unroll
    for (int l = 0; l < LANES; ++l) any |= !done[l];
    if (s >= skew && any) {
      // ---- 1. new halos (published by neighbours at step s-1) ----------
      uint32_t Cu[N + 1][N + 1];
      const uint32_t* xin = xbuf + (buf ^ 1) * XW * (T + 1);
#pragma unroll
      for (int q = 0; q <= N; ++q) Cu[0][q] = xin[(N + q) * (T + 1) + up];
#pragma unroll
      for (int p = 0; p < N; ++p) Cu[p + 1][0] = xin[p * (T + 1) + left];

      // ---- 2. per-slice sigma rows/cols ---------------------------------
      int code[LANES];
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        const int i = si[l];
        code[l] = 0;
        if (i >= 1 && !done[l]) {
          const int pos = i - 1;
          if ((pos & 15) == 0) s0word[l] = __ldg(args.seq + w0[l] + (pos >> 4));
          code[l] = static_cast<int>((s0word[l] >> ((pos & 15) * 2)) & 3u);
        }
      }
      uint32_t s01[N], s02[N];
      if constexpr (LANES == 1) {
        const int16_t* t1 = reinterpret_cast<const int16_t*>(tab1) + code[0] * T + t;
        const int16_t* t2 = reinterpret_cast<const int16_t*>(tab2) + code[0] * T + t;
#pragma unroll
        for (int p = 0; p < N; ++p) {
          const int v1 = t1[p * 4 * T];
          const int v2 = t2[p * 4 * T];
          if constexpr (TRACE) {
            s01[p] = static_cast<uint32_t>(v1 * 16 + static_cast<int>(kTagT2));
            s02[p] = static_cast<uint32_t>(v2 * 16 + static_cast<int>(kTagT3));
          } else {
            s01[p] = static_cast<uint32_t>(v1);
            s02[p] = static_cast<uint32_t>(v2);
          }
        }
      } else {
        const uint32_t c0 = static_cast<uint32_t>(code[0]);
        const uint32_t c1 = static_cast<uint32_t>(code[1]) + 4u;
        const uint32_t sel = c0 | ((c0 | 8u) << 4) | (c1 << 8) | ((c1 | 8u) << 12);
        const uint2* t1 = reinterpret_cast<const uint2*>(tab1) + t;
        const uint2* t2 = reinterpret_cast<const uint2*>(tab2) + t;
#pragma unroll
        for (int p = 0; p < N; ++p) {
          const uint2 e1 = t1[p * T];
          const uint2 e2 = t2[p * T];
          s01[p] = prmt(e1.x, e1.y, sel);
          s02[p] = prmt(e2.x, e2.y, sel);
        }
      }

      // ---- 3. forced cells (reference initialisation, oracle.cpp:30-39) --
      // global: M(0,0,0) = 0; semi: axis cells are 0 in M-space.
      uint32_t fcorner = NEG;
      uint32_t frow[N], fcol[N];  // semi slice-0 faces (row j=0 / col k=0)
      bool semi0 = false;
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        const bool live = !done[l];
        if constexpr (MODE == kGlobal) {
          if (t == 0 && live && si[l] == 0) fcorner = lop_sel(fcorner, 0u, Ops::mask(l));
        } else if constexpr (MODE == kSemi) {
          if (t == 0 && live)
            fcorner = lop_sel(fcorner, Ops::splat((ag2 * si[l]) << SH), Ops::mask(l));
          semi0 |= live && si[l] == 0 && (r == 0 || cc == 0);
        }
      }
      if constexpr (MODE == kSemi) {
#pragma unroll
        for (int q = 0; q < N; ++q) frow[q] = fcol[q] = NEG;
        if (semi0) {
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            if (!done[l] && si[l] == 0) {
#pragma unroll
              for (int q = 0; q < N; ++q) {
                if (r == 0) frow[q] = lop_sel(frow[q], Ops::splat((ag2 * (k0 + q)) << SH), Ops::mask(l));
                if (cc == 0) fcol[q] = lop_sel(fcol[q], Ops::splat((ag2 * (j0 + q)) << SH), Ops::mask(l));
              }
            }
          }
        }
      }
      // local floor base per lane: |g2| * (i + j0 + k0)
      uint32_t flbase = 0;
      if constexpr (MODE == kLocal) {
#pragma unroll
        for (int l = 0; l < LANES; ++l)
          flbase = lop_sel(flbase, Ops::splat((ag2 * (si[l] + j0 + k0)) << SH), Ops::mask(l));
      }

      // ---- 4. the tile: 6 integer instructions per cell -----------------
      constexpr int NW = (NN + 7) / 8;
      uint32_t dirw[TRACE ? NW : 1];
      if constexpr (TRACE) {
#pragma unroll
        for (int w = 0; w < NW; ++w) dirw[w] = 0;
      }
      uint4 sg4 = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int P = 1; P <= N; ++P) {
        uint32_t flrow = 0;
        if constexpr (MODE == kLocal) {
          flrow = flbase + Ops::splat((ag2 * (P - 1)) << SH) + (TRACE ? kTagStop : 0u);
        }
#pragma unroll
        for (int Q = 1; Q <= N; ++Q) {
          const int cell = (P - 1) * N + (Q - 1);
          if ((cell & 3) == 0) sg4 = s12v[(cell >> 2) * T + t];
          const uint32_t sg = (cell & 3) == 0 ? sg4.x : (cell & 3) == 1 ? sg4.y : (cell & 3) == 2 ? sg4.z : sg4.w;
          const uint32_t a1 = s01[P - 1];
          const uint32_t a2 = s02[Q - 1];
          uint32_t x;
          if constexpr (!TRACE) {
            const uint32_t y = Pv[P - 1][Q - 1] + a1 + a2;         // t1 partial (IADD3)
            x = Ops::addmax(Pv[P - 1][Q], a1, Pv[P][Q]);             // max(t2, t5)
            x = Ops::addmax(Pv[P][Q - 1], a2, x);                    // t3
            x = Ops::addmax(y, sg, x);                               // t1
            x = Ops::addmax(Cu[P - 1][Q - 1], sg, x);                // t4
            x = Ops::max3(x, Cu[P - 1][Q], Cu[P][Q - 1]);            // t6, t7
          } else {
            // tags: t1 = 5+4+3 = 12 (a1, a2, sg carry 5, 4, 3)
            const uint32_t y = Pv[P - 1][Q - 1] + a1 + a2;
            x = Ops::addmax(Pv[P - 1][Q], a1, Cu[P][Q - 1]);         // max(t2, t7)
            x = Ops::addmax(Pv[P][Q - 1], a2, x);                    // t3
            x = Ops::addmax(y, sg, x);                               // t1
            x = Ops::addmax(Cu[P - 1][Q - 1], sg, x);                // t4
            x = Ops::addmax(Pv[P][Q], kTagT5, x);                    // t5
            x = Ops::addmax(Cu[P - 1][Q], kTagT6, x);                // t6
          }
          if constexpr (MODE == kLocal) x = Ops::addmax(flrow, colc[Q - 1], x);  // floor 0
          if constexpr (MODE == kGlobal || MODE == kSemi) {
            if (P == 1 && Q == 1) x = Ops::max2(x, fcorner);
          }
          if constexpr (MODE == kSemi) {
            if (P == 1) x = Ops::max2(x, frow[Q - 1]);
            if (Q == 1) x = Ops::max2(x, fcol[P - 1]);
          }
          if constexpr (TRACE) {
            dirw[cell >> 3] |= (x & 15u) << ((cell & 7) * 4);
            x &= ~15u;
          }
          Cu[P][Q] = x;
        }
      }

      // ---- 5. publish right column / down row (+ corner) ----------------
      uint32_t* xout = xbuf + buf * XW * (T + 1) + t;
#pragma unroll
      for (int p = 0; p < N; ++p) xout[p * (T + 1)] = Cu[p + 1][N];
#pragma unroll
      for (int q = 0; q <= N; ++q) xout[(N + q) * (T + 1)] = Cu[N][q];

      // ---- 6. direction cube slot (64 B per tile-slice) -----------------
      if constexpr (TRACE) {
        if (!done[0]) {
          uint4* dst = args.dirs + args.dir_off[tid[0]] + (size_t(si[0]) * T + t) * 4;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (v * 4 < NW) {
              dst[v] = make_uint4(dirw[v * 4], v * 4 + 1 < NW ? dirw[(v * 4 + 1) % NW] : 0u,
                                  v * 4 + 2 < NW ? dirw[(v * 4 + 2) % NW] : 0u,
                                  v * 4 + 3 < NW ? dirw[(v * 4 + 3) % NW] : 0u);
            }
          }
        }
      }

      // ---- 7. score extraction ------------------------------------------
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if (done[l]) continue;
        const int i = si[l];
        if constexpr (MODE == kGlobal) {
          // reads M[a, b, c] (tiled.hpp:495-502): the owner tile, last slice
          if (i == la[l] && (lb[l] / N) == r && (lc[l] / N) == cc) {
            const int want = (lb[l] - j0 + 1) * (N + 1) + (lc[l] - k0 + 1);
            uint32_t v = 0;
#pragma unroll
            for (int P = 1; P <= N; ++P)
#pragma unroll
              for (int Q = 1; Q <= N; ++Q)
                if (P * (N + 1) + Q == want) v = Cu[P][Q];
            const int mv = Ops::lane(v, l) >> SH;
            const int id = tid[l];
            args.out_score[id] = mv + g2 * (la[l] + lb[l] + lc[l]);
            args.out_end[3 * id] = la[l];
            args.out_end[3 * id + 1] = lb[l];
            args.out_end[3 * id + 2] = lc[l];
          }
        }
      }
      if constexpr (MODE != kGlobal) {
        // Best tracking (oracle.cpp:67-88, tiled.hpp:129-144, 222-228):
        // max value, ties to the lexicographically smallest (i, j, k).
        // Candidates: local = every real cell; semi = cells with
        // i == a || j == b || k == c.  Non-candidates are masked out.
        uint32_t rin[N], cin[N], rf[N], cf[N];
        bool cand[LANES];
        bool anyc = false;
#pragma unroll
        for (int p = 0; p < N; ++p) rin[p] = cin[p] = rf[p] = cf[p] = 0;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          cand[l] = false;
          if (done[l]) continue;
          const bool lastslice = si[l] == la[l];
#pragma unroll
          for (int p = 0; p < N; ++p) {
            const int j = j0 + p, k = k0 + p;
            if (j <= lb[l]) rin[p] |= Ops::mask(l);
            if (k <= lc[l]) cin[p] |= Ops::mask(l);
            if (MODE == kSemi && (j == lb[l] || lastslice)) rf[p] |= Ops::mask(l);
            if (MODE == kSemi && k == lc[l]) cf[p] |= Ops::mask(l);
          }
          const bool inside = j0 <= lb[l] && k0 <= lc[l];
          if (MODE == kLocal) {
            cand[l] = inside;
          } else {
            cand[l] = inside && (lastslice || (lb[l] - j0) < N || (lc[l] - k0) < N);
          }
          anyc |= cand[l];
        }
        auto masked = [&](int P, int Q) -> uint32_t {
          if constexpr (MODE == kLocal) {
            return Cu[P][Q] & rin[P - 1] & cin[Q - 1];
          } else {
            const uint32_t keep = (rf[P - 1] & rin[P - 1] & cin[Q - 1]) | (rin[P - 1] & cf[Q - 1]);
            return lop_sel(NEG, Cu[P][Q], keep);
          }
        };
        if (anyc) {
          uint32_t stepmax = NEG;
#pragma unroll
          for (int P = 1; P <= N; ++P) {
            uint32_t rowacc = NEG;
#pragma unroll
            for (int Q = 1; Q <= N; ++Q) rowacc = Ops::addmax(masked(P, Q), cold[Q - 1], rowacc);
            stepmax = Ops::addmax(rowacc, Ops::splat((g2 * (P - 1)) << SH), stepmax);
          }
#pragma unroll
          for (int l = 0; l < LANES; ++l) {
            if (!cand[l]) continue;
            const int sm = Ops::lane(stepmax, l);
            const int base = (g2 * (si[l] + j0 + k0)) << SH;
            const int mval = (sm + base) >> SH;
            if (!bestok[l] || mval > bestv[l]) {
              // first cell (row-major = lexicographic) attaining the maximum
              int fp = 0, fq = 0;
              bool found = false;
#pragma unroll
              for (int P = 1; P <= N; ++P)
#pragma unroll
                for (int Q = 1; Q <= N; ++Q) {
                  const int v = Ops::lane(masked(P, Q), l) + ((g2 * (P - 1 + Q - 1)) << SH);
                  if (!found && v == sm) {
                    found = true;
                    fp = P - 1;
                    fq = Q - 1;
                  }
                }
              const uint32_t j = j0 + fp, k = k0 + fq;
              bestv[l] = mval;
              bestlin[l] = (static_cast<uint32_t>(si[l]) * static_cast<uint32_t>(lb[l] + 1) + j) *
                               static_cast<uint32_t>(lc[l] + 1) + k;
              bestok[l] = true;
            }
          }
        }
      }

      // ---- 8. previous slice := this slice ------------------------------
#pragma unroll
      for (int P = 0; P <= N; ++P)
#pragma unroll
        for (int Q = 0; Q <= N; ++Q) Pv[P][Q] = Cu[P][Q];

      // ---- 9. advance the lanes -----------------------------------------
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if (done[l]) continue;
        si[l] += 1;
        if (si[l] > la[l]) {
          if constexpr (MODE != kGlobal) {
            if (bestok[l]) {
              const unsigned long long key =
                  (static_cast<unsigned long long>(static_cast<uint32_t>(bestv[l]) ^ 0x80000000u) << 32) |
                  static_cast<unsigned long long>(0xFFFFFFFFu - bestlin[l]);
              atomicMax(args.out_key + tid[l], key);
            }
            bestok[l] = false;
          }
          item[l] += 1;
          if (item[l] < iend[l]) {
            tid[l] = args.items[item[l]];
            setup(l, tid[l]);
          } else {
            done[l] = true;
            setup(l, -1);
          }
          si[l] = 0;
#pragma unroll
          for (int P = 0; P <= N; ++P)
#pragma unroll
            for (int Q = 0; Q <= N; ++Q) Pv[P][Q] = lop_sel(Pv[P][Q], NEG, Ops::mask(l));
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace ta
