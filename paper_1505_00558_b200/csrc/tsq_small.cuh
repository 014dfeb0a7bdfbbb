// tsq_small.cuh -- on-chip sort of a small segment: an LSD radix sort over
// the segment's own key range.  This is the role insertion_sort plays in the
// reference (smallsort.py:12-47) for ranges of <= insertion_threshold keys
// (core.py:1652-1658); here, segments of <= small_t keys.
//
// By the time the recursion hands a segment to the on-chip sort, its keys lie
// between two ancestor pivots, so their encoded range is narrow (uniform int32
// at 2^26: ~21 bits for a 32K-key segment).  One CTA per segment:
//
//   1. coalesced load into shared memory, encode, CTA-wide min / max; the
//      active threads (ceil(len / KPT)) read KPT consecutive keys each back
//      ("blocked") and form items = key - min (records: the local index
//      packed below it while both fit, else in a 16-bit side array);
//   2. stable counting passes of <= DB-bit digits, each:
//        count  every thread bumps its own 16-bit counter (digit, thread) for
//               each of its items, in position order;
//        scan   one exclusive scan over the counters in (digit, thread) order
//               gives every (digit, thread) its first output slot;
//        rank   the same sweep again now hands out slots: each item goes to
//               its slot in shared memory; the next pass reads them back
//               blocked.
//      Thread order = position order inside a digit, so every pass is stable
//      and the LSD passes leave the items in key order.  A range wider than
//      TPASS * DB bits is sorted on its leading bits only, then finished by
//      odd-even exchange rounds over the full items (radix_run);
//   3. keys written back as min + item (caller's encoding, coalesced);
//      record payloads gathered by local index.
//
// Measured alternatives (B200, uniform int32 2^26, DESIGN.md section 9;
// several are still here behind the TSQ_S_* switches): warp-collective
// ranking with __match_any_sync runs on the ADU pipe at ~2 SM-cycles per
// distinct digit in the warp (60 per 8-bit match, scripts/micro/match_tp.cu)
// -- 2.3 ms for the on-chip sort; ballot-based peer masks take ~9
// instructions per digit bit; shared-memory atomics run at 2 cycles per lane;
// 256 threads x 128 keys with 7-bit digits cannot hide the counter
// read-modify-write chain (8 warps per SM); the segment brought in by bulk
// copy and read as 16-byte chunks costs more instructions than the coalesced
// loads it replaces; paired / quad counter steps with kept ranks add more
// instructions than the latency they hide at 16 warps; counters overlaying
// the item buffer (7-bit digits at 512 threads) double the zero + scan work.
// The round-1 warp bitonic + merge-path sort took 0.95 ms at ~320
// instructions per key; 1024 threads x 32 keys with 5-bit digits 0.68 ms at
// ~176; this geometry (512 x 80, 6-bit digits, 40960 slots) 0.59 ms at ~130,
// shared-memory wavefronts at 62 % of peak.
#pragma once

#include "tsq_bitonic.cuh"

namespace tsq {

// phase clocks of CTA 0 (profiling builds only: -DTSQ_S_CLOCK; printed at kernel end)
#ifdef TSQ_S_CLOCK
__device__ long long g_ph[16];
__device__ long long g_ph_last;
#define TSQ_PH(i)                                   \
  do {                                              \
    if (blockIdx.x == 0 && threadIdx.x == 0) {      \
      const long long c_ = clock64();               \
      g_ph[i] += c_ - g_ph_last;                    \
      g_ph_last = c_;                               \
    }                                               \
  } while (0)
#else
#define TSQ_PH(i) ((void)0)
#endif

template <typename U>
__device__ __forceinline__ void warp_minmax(U &mn, U &mx) {
  if constexpr (sizeof(U) == 4) {
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const U a = __shfl_xor_sync(0xffffffffu, mn, o);
      const U b = __shfl_xor_sync(0xffffffffu, mx, o);
      mn = a < mn ? a : mn;
      mx = b > mx ? b : mx;
    }
  }
}

// Class geometry: threads, item slots, digit bits.  A class takes segments
// of up to SLOTS - kSmallSlack keys (the bulk copy brings the 16-byte aligned
// window around a segment: up to 3 + 3 foreign keys).  Class 2 of bare
// 4-byte keys keeps its keys in registers, up to KPT = SLOTS / NT per thread
// in steps of 32 (so every thread takes part whatever the segment's length).
#ifndef TSQ_S2_NT
#define TSQ_S2_NT 512
#endif
#ifndef TSQ_S2_DB
#define TSQ_S2_DB 6
#endif
// feature switches (experiment builds, scripts/variants.py)
#ifndef TSQ_S_TMA
#define TSQ_S_TMA 0    // bare keys arrive by bulk copy (else coalesced loads)
#endif
#ifndef TSQ_S_VAR
#define TSQ_S_VAR 1    // items per thread chosen per segment
#endif
#ifndef TSQ_S_LOUT
#define TSQ_S_LOUT 1   // sorted bare keys leave by bulk copy
#endif
#ifndef TSQ_S_ALIAS
#define TSQ_S_ALIAS 0  // class 2 of bare 4-byte keys: the counters overlay the item buffer
#endif
#ifndef TSQ_S_TRUNC
#define TSQ_S_TRUNC 1  // wide ranges: leading bits first, then exchange rounds
#endif
#ifndef TSQ_S_TPASS6W
#define TSQ_S_TPASS6W 3 // same, 8-byte keys
#endif
#ifndef TSQ_S_TPASS6
#define TSQ_S_TPASS6 4 // leading-bit passes of a 6-bit class
#endif
#ifndef TSQ_S_PREFETCH
#define TSQ_S_PREFETCH 1  // the next segment's keys prefetched into L2 during the current sort
#endif
#ifndef TSQ_S_QUAD
#define TSQ_S_QUAD 0   // four counters per step, ranks kept from the count sweep
#endif
#ifndef TSQ_S2P_NT
#define TSQ_S2P_NT 1024   // class 2 of records
#endif
#ifndef TSQ_S2P_DB
#define TSQ_S2P_DB 5
#endif
#ifndef TSQ_S2W_NT
#define TSQ_S2W_NT 512    // class 2 of bare 8-byte keys
#endif
#ifndef TSQ_S2W_DB
#define TSQ_S2W_DB 6
#endif
template <int KB, bool PAY, int CLS>
struct SmallClass {
  static constexpr bool BARE4 = KB == 4 && !PAY;
  static constexpr bool BARE8 = KB == 8 && !PAY;
  static constexpr int NT = CLS == 0 ? kThreads : (CLS == 1 ? 2 * kThreads : (BARE4 ? TSQ_S2_NT : (BARE8 ? TSQ_S2W_NT : TSQ_S2P_NT)));
  static constexpr int SLOTS = CLS == 0   ? kSmallT
                               : CLS == 1 ? (BARE4 ? kSmallHuge : kSmallMax)
                                          : (BARE4 ? kSmallGiant : kSmallHuge);
  static constexpr int DB = (CLS == 2 && BARE4) ? TSQ_S2_DB : ((CLS == 2 && BARE8) ? TSQ_S2W_DB : (CLS == 2 ? TSQ_S2P_DB : 5));
  static constexpr int MINB = CLS == 0 ? 4 : (CLS == 1 ? 2 : 1);
  // the counters overlay the item buffer: the items stay in registers from
  // the pass's first read to its scatter, the ranks are taken into registers
  // before the first scatter store
  static constexpr bool ALIAS = CLS == 2 && BARE4 && TSQ_S_ALIAS;
};

// Shared-memory geometry of one item form (T = u32 / u64 items, IDX =
// separate 16-bit local-index array).  Item slot r lives at r + r / kpt (one
// pad per thread's run of kpt slots; kpt = 16: one per 32), so the blocked
// reads (thread stride kpt + 1) and the striped ones both spread over the
// banks.  Counters: R (digit) rows of NT 16-bit counters (radix_cnt_byte).
template <int NT, int SLOTS, int DB, typename T, bool PAY, bool IDX, int KB, bool ALIAS = false>
struct RadixForm {
  static constexpr int KPT = SLOTS / NT;
  static constexpr int CAPP = SLOTS + (KPT >= 32 ? NT : SLOTS / 32);   // padded item slots
  static constexpr int DBMAX = (KB == 8 && sizeof(T) == 8 && IDX) ? DB - 1 : DB;
  static constexpr int RMAX = 1 << DBMAX;
  // misc: min/max exchange [0, 512), warp totals [512, 640), mbarrier [640, 648), ticket [656, 660)
  static constexpr size_t MISC = 1024;
  static constexpr size_t OFF_BUF = MISC;
  static constexpr size_t OFF_IBUF = OFF_BUF + (size_t)CAPP * sizeof(T);
  static constexpr size_t OFF_CNT0 = (OFF_IBUF + (IDX ? (size_t)CAPP * 2 : 0) + 15) & ~(size_t)15;
  static constexpr size_t OFF_CNT = ALIAS ? OFF_BUF : OFF_CNT0;
  static constexpr size_t END0 = OFF_CNT + (size_t)RMAX * NT * 2;
  static constexpr size_t END = ALIAS && OFF_CNT0 > END0 ? OFF_CNT0 : END0;
};

// Counter (digit d, thread t) layout.  Threads form groups of 64, m = t / 64;
// a row (digit) is NT/2 32-bit words, a group 32 of them: lane l = t % 32 of
// the group's first warp owns the low half of word l, the same lane of its
// second warp the high half.  So a warp's bumps touch 32 distinct banks
// whatever digits its lanes hold (rows are a multiple of 32 words apart).
template <int NT>
__device__ __forceinline__ uint32_t radix_cnt_byte(int t) {
  const int m = t >> 6, h = (t >> 5) & 1, l = t & 31;
  return (uint32_t)((m * 32 + l) * 4 + 2 * h);
}

template <class C, bool PAY, int CLS>
struct RadixGeo {
  typedef typename C::U U;
  typedef SmallClass<(int)sizeof(U), PAY, CLS> K;
  static constexpr int KB = (int)sizeof(U);
  static constexpr int NT = K::NT, SLOTS = K::SLOTS, DB = K::DB;
  static constexpr int CAP = SLOTS - kSmallSlack;   // keys a segment of this class may have
  static constexpr int NW = NT / 32;
  static constexpr int CLASS = CLS;
  static constexpr int KPT = SLOTS / NT;
  static constexpr int VN = 16 / KB;        // keys per 16-byte chunk
  static constexpr int G = 8 * VN;          // keys per thread come in steps of G when KPT > G
  static constexpr bool LIN = !PAY && TSQ_S_TMA;   // bulk-copied linear window (bare keys)
  static constexpr bool VAR = KPT > G && LIN && TSQ_S_VAR;
  static constexpr bool ALIAS = K::ALIAS;
  static constexpr size_t S32 = RadixForm<NT, SLOTS, DB, uint32_t, PAY, PAY, KB, ALIAS>::END;
  static constexpr size_t S32p = RadixForm<NT, SLOTS, DB, uint32_t, PAY, false, KB, ALIAS>::END;
  static constexpr size_t S64a = KB == 8 ? RadixForm<NT, SLOTS, DB, u64, PAY, PAY, KB>::END : 0;
  static constexpr size_t S64b = KB == 8 ? RadixForm<NT, SLOTS, DB, u64, PAY, false, KB>::END : 0;
  static constexpr size_t SLIN = RadixForm<NT, SLOTS, DB, U, PAY, false, KB>::OFF_BUF + (size_t)SLOTS * KB + 16;
  static constexpr size_t m2(size_t a, size_t b) { return a > b ? a : b; }
  static constexpr size_t SMEM = m2(m2(m2(S32, S32p), m2(S64a, S64b)), SLIN);
  static_assert(KPT * NT == SLOTS, "a whole number of items per thread");
  static_assert(KPT >= 16 && KPT % 16 == 0 && (KPT >= 32 || KPT == 16), "items per thread");
  static_assert(!VAR || KPT % G == 0, "variable items per thread: whole granules");
  static_assert(2 * NW * sizeof(U) <= 512 && NW <= 32, "misc region");
  static_assert(SMEM <= 227 * 1024, "shared memory per CTA");
  static_assert(SLOTS < 65536, "16-bit counters");
};

// Exclusive scan of the R x NT counters in (digit, thread) order.  In that
// order a block (digit d, group m) is 64 consecutive counters: the 32 low
// halves (threads 64m .. 64m+31) then the 32 high halves.  Scan thread t
// takes the BPT consecutive blocks from t * BPT on.  It reads a block's eight
// 16-byte chunks starting at chunk t % 8 and wrapping round, so the eight
// lanes of a quarter warp touch eight different bank groups (every block
// starts at bank 0).  The packed sum P of a block's 32 words is two 16-bit
// totals (no carries: a segment has < 2^16 items); PH = the part summed
// before the wrap (chunks t % 8 .. 7).  With s0 = the block's exclusive
// prefix, chunk 0 starts at the packed (s0, s0 + lo(P)), and the thread's
// first chunk at that plus P - PH.
template <int NT, int RMAX>
__device__ __forceinline__ void radix_scan(uint16_t *cnt, uint32_t *wt, int R) {
  constexpr int NW = NT / 32;
  constexpr int GPR = NT / 64;  // blocks per row
  constexpr int BPT = (RMAX * GPR + NT - 1) / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = R * GPR;
  const int rot = tid & 7;
  uint4 *blk0 = reinterpret_cast<uint4 *>(cnt) + (size_t)tid * BPT * 8;
  uint32_t P[BPT], PH[BPT];
  uint32_t sum = 0;
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    P[b] = 0;
    PH[b] = 0;
    if (tid * BPT + b < nblk) {
      const uint4 *blk = blk0 + b * 8;
      uint32_t acc = 0, hi = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = (c + rot) & 7;
        const uint4 v = blk[j];
        acc += v.x + v.y + v.z + v.w;
        if (j == 7) hi = acc;
      }
      P[b] = acc;
      PH[b] = hi;
      sum += (acc & 0xffffu) + (acc >> 16);
    }
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wt[warp] = inc;
  __syncthreads();
  uint32_t s0 = inc - sum;
#pragma unroll
  for (int i = 0; i < NW; ++i)
    if (i < warp) s0 += wt[i];
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    if (tid * BPT + b < nblk) {
      uint4 *blk = blk0 + b * 8;
      const uint32_t start = s0 | ((s0 + (P[b] & 0xffffu)) << 16);
      uint32_t run = start + (P[b] - PH[b]);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = (c + rot) & 7;
        const uint4 v = blk[j];
        uint4 o;
        o.x = run; run += v.x;
        o.y = run; run += v.y;
        o.z = run; run += v.z;
        o.w = run; run += v.w;
        blk[j] = o;
        if (j == 7) run = start;
      }
      s0 += (P[b] & 0xffffu) + (P[b] >> 16);
    }
  }
}

// element e of a 16-byte chunk of keys
template <int e> __device__ __forceinline__ uint32_t chunk_get(const uint4 &v) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}
template <int e> __device__ __forceinline__ u64 chunk_get(const ulonglong2 &v) {
  return e == 0 ? v.x : v.y;
}

// Item slot of rank r: one pad slot per thread's run of kpt slots (kpt a
// per-segment multiple of G when VAR: r / kpt as a multiply-shift, exact for
// r < 2^16 and the kpt in use -- tests/test_api_cpu.py checks the constants).
template <int KPT, bool VAR>
struct SlotMap {
  uint32_t inv;
  __device__ __forceinline__ explicit SlotMap(int kpt) : inv((4194304u + (uint32_t)kpt - 1u) / (uint32_t)kpt) {}
  __device__ __forceinline__ int operator()(int r) const {
    if constexpr (VAR) return r + (int)(((uint32_t)r * inv) >> 22);
    else if constexpr (KPT >= 32) return r + (int)((uint32_t)r / (uint32_t)KPT);
    else return r + (r >> 5);
  }
};

// What the kernel reads from Params once.
template <typename U>
struct SmallEnv {
  const U *keys0, *keys1;      // the caller's buffer (also the destination), the workspace partner
  uint32_t *pay0;
  const uint32_t *pay1;
  bool raw0, raw1;             // buffer holds the caller's encoding
  bool aligned;                // both key buffers 16-byte aligned
  long long n;
  __device__ __forceinline__ const U *keys(int b) const { return b ? keys1 : keys0; }
  __device__ __forceinline__ const uint32_t *pay(int b) const { return b ? pay1 : pay0; }
  __device__ __forceinline__ bool raw(int b) const { return b ? raw1 : raw0; }
  __device__ __forceinline__ U *dst() const { return const_cast<U *>(keys0); }
};

// Radix passes over items T whose digits occupy bits [b0, b0 + bits); IDX:
// the local index travels in a 16-bit side array (else it is packed below
// b0 for records, or absent).  Bare keys (LIN): the encoded keys arrive in
// registers (kr, invalid window positions as all-ones), kpt per thread; the
// sorted keys leave through the linear window image when items are as wide
// as keys.  Records: the encoded keys sit in shared memory at slot
// rpad(i) of a U-typed array; the first pass turns them into items as it
// reads them back blocked.  `lo` is their minimum.
template <class C, bool PAY, int CLS, typename T, bool IDX>
__device__ __forceinline__ void radix_run(const SmallEnv<typename C::U> &E, const SmallSeg &sm,
                                          unsigned char *smem, typename C::U lo, int b0, int bits,
                                          typename C::U (&kr)[RadixGeo<C, PAY, CLS>::LIN ? RadixGeo<C, PAY, CLS>::KPT : 1],
                                          int head, int kpt) {
  typedef typename C::U U;
  typedef RadixGeo<C, PAY, CLS> G;
  typedef RadixForm<G::NT, G::SLOTS, G::DB, T, PAY, IDX, G::KB, G::ALIAS> F;
  constexpr int KPT = G::KPT, NT = G::NT;
  constexpr bool ALIAS = G::ALIAS;
  constexpr bool LIN = G::LIN, VAR = G::VAR;
  constexpr bool LOUT = LIN && sizeof(T) == sizeof(U) && TSQ_S_LOUT;
  constexpr bool QUAD = TSQ_S_QUAD != 0;
  constexpr bool PACKED = PAY && !IDX;
  constexpr int GK = VAR ? G::G : KPT;   // items per guarded block
  const int tid = threadIdx.x;
  const int len = sm.len;
  const int sup = head + len;            // window positions in use
  // active threads hold kpt consecutive positions each; pads (window
  // positions outside the segment, the last thread's tail) carry the largest
  // digit in every pass
  const int NA = (sup + kpt - 1) / kpt;
  const bool act = tid < NA;
  const SlotMap<KPT, VAR> slot(kpt);
  T *buf = reinterpret_cast<T *>(smem + F::OFF_BUF);
  uint16_t *ibuf = reinterpret_cast<uint16_t *>(smem + F::OFF_IBUF);
  uint16_t *cnt = reinterpret_cast<uint16_t *>(smem + F::OFF_CNT);
  uint32_t *wt = reinterpret_cast<uint32_t *>(smem) + 128;
  // this thread's counter of digit 0; rows are NT * 2 bytes apart
  unsigned char *mycb = reinterpret_cast<unsigned char *>(cnt) + radix_cnt_byte<NT>(tid);
  // this thread's slots: slot(t*kpt + k) = slot(t*kpt) + k
  T *mine = buf + slot(tid * kpt);
  uint16_t *imine = ibuf + slot(tid * kpt);
  T it[KPT];
  uint16_t ix[IDX ? KPT : 1];
  uint32_t lr[QUAD ? KPT / 4 : 1];   // each item's rank among the thread's items of its digit
  static_assert(KPT <= 256 && KPT % 8 == 0, "8-bit ranks inside a thread");
  static_assert(!ALIAS || (!QUAD && !LIN && !IDX && sizeof(T) == 4), "overlay: plain 32-bit items only");
  // A wide range (float64 keys: ~45 bits in an 8K-key segment of 2^26 normal
  // keys) is first sorted on its leading TB bits only -- TPASS digit passes
  // instead of ceil(bits / DB) -- which leaves only items with equal leading
  // bits possibly out of order: for keys spread over the range, a few
  // adjacent pairs.  Odd-even exchange rounds over the full items put them
  // right; if they have not settled after kFixRounds (keys clustered inside
  // few leading-bit buckets), the full LSD passes run after all.
#ifdef TSQ_S_TPASS
  constexpr int TPASS = TSQ_S_TPASS;
#else
  constexpr int TPASS = F::DBMAX >= 6 ? (sizeof(U) == 8 ? TSQ_S_TPASS6W : TSQ_S_TPASS6) : (F::DBMAX == 5 ? 3 : 4);
#endif
  constexpr int TB = TPASS * F::DBMAX;
  constexpr int kFixRounds = 12;
  const bool trunc = TSQ_S_TRUNC && !LIN && bits > TB;
#pragma unroll 1
  for (int attempt = 0; attempt < 2; ++attempt) {
  const bool tr = trunc && attempt == 0;
  const int tbits = tr ? TB : bits;          // key bits this attempt's passes cover
  const int shift0 = bits - tbits;
#ifdef TSQ_S_MAXPASS   // timing experiments only: the output is not sorted
  const int passes0 = (tbits + F::DBMAX - 1) / F::DBMAX;
  const int passes = passes0 < TSQ_S_MAXPASS ? passes0 : TSQ_S_MAXPASS;
  const int db = (tbits + passes0 - 1) / passes0;
#else
  const int passes = (tbits + F::DBMAX - 1) / F::DBMAX;   // bits >= 1
  const int db = (tbits + passes - 1) / passes;
#endif
  const uint32_t mask = (1u << db) - 1u;
  const int R = 1 << db;
  const int wbits = b0 + passes * db;
  const T padv = wbits >= (int)(8 * sizeof(T)) ? ~T(0) : (T)((T(1) << wbits) - 1);
#pragma unroll 1
  for (int ps = 0; ps < passes; ++ps) {
    const int sh = b0 + shift0 + db * ps;
    const bool last = ps == passes - 1 && !tr;
    const bool first = ps == 0 && attempt == 0;
    if (!first || !LIN) __syncthreads();   // previous scatter (or the key load) complete
    TSQ_PH(ps == 0 ? 2 : 8);
    if (first) {
      if constexpr (LIN) {
        // items from the keys in registers; a pad (all-ones key) clamps to padv
        const U padu = (U)padv;
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
          const U d = kr[k] - lo;
          it[k] = (T)(d < padu ? d : padu);
        }
      } else {
        const U *rmine = reinterpret_cast<const U *>(smem + F::OFF_BUF) + slot(tid * kpt);
        if (act) {
#pragma unroll
          for (int k = 0; k < KPT; ++k) {
            const int p = tid * KPT + k;
            it[k] = p < len ? (((T)(rmine[k] - lo) << b0) | (PACKED ? (T)p : (T)0)) : ~T(0);
            if (IDX) ix[k] = (uint16_t)p;
          }
        }
      }
      // keys wider than items: the key array overlaps the counters
      if (sizeof(U) > sizeof(T) || LIN) __syncthreads();
    } else if (act) {
#pragma unroll
      for (int k0 = 0; k0 < KPT; k0 += GK) {
        if (k0 < kpt) {
#pragma unroll
          for (int k = k0; k < k0 + GK; ++k) {
            it[k] = mine[k];
            if (IDX) ix[k] = imine[k];
          }
        }
      }
    }
    if (ALIAS && !(first && (sizeof(U) > sizeof(T) || LIN))) __syncthreads();   // every item is in registers
    TSQ_PH(first ? 3 : 4);
    {
      uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
      const int n4 = R * NT / 8;
      for (int i = tid; i < n4; i += NT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    TSQ_PH(5);
    // count: this thread's items, in position order, four per step: the
    // four counters are read together, each item's rank among the thread's
    // items of its digit (counter + equal digits earlier in the step) is
    // kept (8 bits), and the counters are written back in order -- a quarter
    // of the dependent shared-memory round trips
    if (act && QUAD) {
#pragma unroll
      for (int k0 = 0; k0 < KPT; k0 += GK) {
        if (k0 < kpt) {
#pragma unroll
          for (int k = k0; k < k0 + GK; k += 4) {
            const uint32_t o0 = ((uint32_t)(it[k] >> sh) & mask) * (2 * NT);
            const uint32_t o1 = ((uint32_t)(it[k + 1] >> sh) & mask) * (2 * NT);
            const uint32_t o2 = ((uint32_t)(it[k + 2] >> sh) & mask) * (2 * NT);
            const uint32_t o3 = ((uint32_t)(it[k + 3] >> sh) & mask) * (2 * NT);
            const uint32_t c0 = *reinterpret_cast<uint16_t *>(mycb + o0);
            const uint32_t c1 = *reinterpret_cast<uint16_t *>(mycb + o1);
            const uint32_t c2 = *reinterpret_cast<uint16_t *>(mycb + o2);
            const uint32_t c3 = *reinterpret_cast<uint16_t *>(mycb + o3);
            const uint32_t l1 = c1 + (o1 == o0 ? 1u : 0u);
            const uint32_t l2 = c2 + (o2 == o0 ? 1u : 0u) + (o2 == o1 ? 1u : 0u);
            const uint32_t l3 = c3 + (o3 == o0 ? 1u : 0u) + (o3 == o1 ? 1u : 0u) + (o3 == o2 ? 1u : 0u);
            *reinterpret_cast<uint16_t *>(mycb + o0) = (uint16_t)(c0 + 1u);
            *reinterpret_cast<uint16_t *>(mycb + o1) = (uint16_t)(l1 + 1u);
            *reinterpret_cast<uint16_t *>(mycb + o2) = (uint16_t)(l2 + 1u);
            *reinterpret_cast<uint16_t *>(mycb + o3) = (uint16_t)(l3 + 1u);
            lr[k >> 2] = c0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
          }
        }
      }
    }
    if (act && !QUAD) {
#pragma unroll
      for (int k0 = 0; k0 < KPT; k0 += GK) {
        if (k0 < kpt) {
#pragma unroll
          for (int k = k0; k < k0 + GK; ++k) {
            uint16_t *a = reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k] >> sh) & mask) * (2 * NT));
            *a = (uint16_t)(*a + 1u);
          }
        }
      }
    }
    __syncthreads();
    TSQ_PH(6);
    radix_scan<NT, F::RMAX>(cnt, wt, R);
    __syncthreads();
    TSQ_PH(7);
    // rank + scatter: an item's slot = its (digit, thread) prefix + its rank
    // in the thread; the prefixes of eight items are read before the first
    // scatter store
    if (act && QUAD) {
      U *out = reinterpret_cast<U *>(smem + F::OFF_BUF) + head;
#pragma unroll
      for (int k0 = 0; k0 < KPT; k0 += GK) {
        if (k0 < kpt) {
#pragma unroll
          for (int k8 = k0; k8 < k0 + GK; k8 += 8) {
            uint32_t r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              r[j] = *reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k8 + j] >> sh) & mask) * (2 * NT));
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int k = k8 + j;
              r[j] += (lr[k >> 2] >> (8 * (k & 3))) & 0xffu;
              TSQ_CHECK(r[j] < (uint32_t)(NA * kpt));
              if (LOUT && last) {
                // the sorted keys, decoded, at their place in the window image
                const U kv = lo + (U)it[k];
                if (r[j] < (uint32_t)len) out[r[j]] = E.raw0 ? C::dec(kv) : kv;
              } else {
                buf[slot((int)r[j])] = it[k];
                if (IDX) ibuf[slot((int)r[j])] = ix[k];
              }
            }
          }
        }
      }
    }
    if (!QUAD && ALIAS) {
      // ranks into registers (two 16-bit ranks per word), then -- the
      // counters are dead -- the scatter over them
      uint32_t rk[KPT / 2];
      if (act) {
#pragma unroll
        for (int k = 0; k < KPT; k += 2) {
          uint16_t *a0 = reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k] >> sh) & mask) * (2 * NT));
          const uint32_t r0 = *a0;
          *a0 = (uint16_t)(r0 + 1u);
          uint16_t *a1 = reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k + 1] >> sh) & mask) * (2 * NT));
          const uint32_t r1 = *a1;
          *a1 = (uint16_t)(r1 + 1u);
          rk[k >> 1] = r0 | (r1 << 16);
        }
      }
      __syncthreads();
      if (act) {
#pragma unroll
        for (int k = 0; k < KPT; k += 2) {
          const uint32_t r0 = rk[k >> 1] & 0xffffu, r1 = rk[k >> 1] >> 16;
          TSQ_CHECK(r0 < (uint32_t)(NA * kpt) && r1 < (uint32_t)(NA * kpt));
          buf[slot((int)r0)] = it[k];
          buf[slot((int)r1)] = it[k + 1];
        }
      }
    }
    if (act && !QUAD && !ALIAS) {
      U *out = reinterpret_cast<U *>(smem + F::OFF_BUF) + head;
#pragma unroll
      for (int k0 = 0; k0 < KPT; k0 += GK) {
        if (k0 < kpt) {
#pragma unroll
          for (int k = k0; k < k0 + GK; ++k) {
            uint16_t *a = reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k] >> sh) & mask) * (2 * NT));
            const uint32_t r = *a;
            *a = (uint16_t)(r + 1u);
            TSQ_CHECK(r < (uint32_t)(NA * kpt));
            if (LOUT && last) {
              const U kv = lo + (U)it[k];
              if (r < (uint32_t)len) out[r] = E.raw0 ? C::dec(kv) : kv;
            } else {
              buf[slot((int)r)] = it[k];
              if (IDX) ibuf[slot((int)r)] = ix[k];
            }
          }
        }
      }
    }
  }
  if (!tr) break;
  // odd-even exchange rounds over the full items (slots [0, len))
  __syncthreads();
  bool settled = false;
#pragma unroll 1
  for (int round = 0; round < kFixRounds && !settled; ++round) {
    bool swapped = false;
#pragma unroll
    for (int ph = 0; ph < 2; ++ph) {
      for (int i = 2 * tid + ph; i + 1 < len; i += 2 * NT) {
        const int sa = slot(i), sb = slot(i + 1);
        TSQ_CHECK(sa >= 0 && sb < F::CAPP);
        const T a = buf[sa], b = buf[sb];
        if (a > b) {
          buf[sa] = b;
          buf[sb] = a;
          if (IDX) {
            const uint16_t ia = ibuf[sa];
            ibuf[sa] = ibuf[sb];
            ibuf[sb] = ia;
          }
          swapped = true;
        }
      }
      __syncthreads();
    }
    settled = !__syncthreads_or(swapped);
  }
  if (settled) break;
  }
  U *dst = E.dst() + sm.begin;
  if constexpr (LOUT) {
    // the window image leaves as bulk copies (whole 16-byte chunks of the
    // destination), its ragged ends as scalar stores
    constexpr int VN = G::VN;
    const U *out = reinterpret_cast<const U *>(smem + F::OFF_BUF) + head;
    fence_proxy_async_smem();
    __syncthreads();
    if (E.aligned) {
      int r1 = (VN - head) & (VN - 1);
      r1 = r1 < len ? r1 : len;
      const int r2 = r1 + (len - r1) / VN * VN;
      if (tid < 32) {
        constexpr uint32_t PIECE = 4096;
        const uint32_t bytes = (uint32_t)(r2 - r1) * sizeof(U);
        for (uint32_t o = (uint32_t)tid * PIECE; o < bytes; o += 32 * PIECE) {
          const uint32_t b = bytes - o < PIECE ? bytes - o : PIECE;
          bulk_store(reinterpret_cast<char *>(dst + r1) + o,
                     reinterpret_cast<const char *>(out + r1) + o, b);
        }
        bulk_commit();
      } else if (tid < 32 + VN) {
        const int i = tid - 32;
        if (i < r1) dst[i] = out[i];
        if (r2 + i < len) dst[r2 + i] = out[r2 + i];
      }
    } else {
      for (int i = tid; i < len; i += NT) dst[i] = out[i];
    }
    return;
  }
  __syncthreads();
  TSQ_PH(8);
  // buf[0, len) holds the sorted items
  const bool dst_raw = E.raw0;
  if (PAY) {
    // payloads gathered by local index from the source (an L1/L2-resident
    // window) into registers, all before any is written (the source may be
    // buffer 0 itself)
    const uint32_t *ps = E.pay(sm.buf) + sm.begin;
    uint32_t pv[KPT];
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
      const int i = tid + q * NT;
      pv[q] = i < len ? ps[IDX ? (uint32_t)ibuf[slot(i)]
                               : (uint32_t)(buf[slot(i)] & (T)((1u << b0) - 1u))]
                      : 0u;
    }
    __syncthreads();
    uint32_t *pd = E.pay0 + sm.begin;
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
      const int i = tid + q * NT;
      if (i < len) pd[i] = pv[q];
    }
  }
#pragma unroll 4
  for (int q = 0; q < KPT; ++q) {
    const int i = tid + q * NT;
    if (i < len) {
      const U k = lo + (U)(buf[slot(i)] >> b0);
      dst[i] = dst_raw ? C::dec(k) : k;
    }
  }
}

// Sort one queued segment (all threads of the CTA).  `phase`: parity of the
// load barrier's next completion.
template <class C, bool PAY, int CLS, class AfterLoad>
__device__ __forceinline__ void radix_sort_seg(const SmallEnv<typename C::U> &E, const SmallSeg &sm,
                                               unsigned char *smem, uint32_t &phase,
                                               AfterLoad after_load) {
  typedef typename C::U U;
  typedef RadixGeo<C, PAY, CLS> G;
  constexpr int KPT = G::KPT, NW = G::NW, NT = G::NT, VN = G::VN;
  constexpr bool LIN = G::LIN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int len = sm.len;
  const U *src = E.keys(sm.buf) + sm.begin;
  const bool raw = E.raw(sm.buf);
  TSQ_CHECK(len >= 1 && len <= G::CAP && sm.begin >= 0 && sm.begin + len <= E.n);
  U mn = KeyMax<U>::v, mx = U(0);
  U kr[LIN ? KPT : 1];
  int head = 0, kpt = KPT;
  if constexpr (LIN) {
    // the 16-byte aligned window [begin - head, ...) around the segment, as
    // bulk copies of its whole chunks (the ragged end by scalar loads); any
    // earlier bulk stores have finished reading the same shared memory
    typedef typename Vec<U>::K KV;
    U *lin = reinterpret_cast<U *>(smem + 1024);
    u64 *bar = reinterpret_cast<u64 *>(smem + 640);
    head = E.aligned ? (int)(sm.begin & (VN - 1)) : 0;
    const int sup = head + len;
    if (G::VAR) kpt = G::G * ((sup + NT * G::G - 1) / (NT * G::G));
    TSQ_CHECK(kpt <= KPT && NT * kpt >= sup);
    if (E.aligned) {
      const int whole = sup / VN * VN;
      if (tid < 32) {
        constexpr uint32_t PIECE = 4096;
        const uint32_t bytes = (uint32_t)whole * sizeof(U);
        bulk_wait_read0();
        if (tid == 0) mbar_arrive_expect_tx(bar, bytes);
        __syncwarp();
        for (uint32_t o = (uint32_t)tid * PIECE; o < bytes; o += 32 * PIECE) {
          const uint32_t b = bytes - o < PIECE ? bytes - o : PIECE;
          bulk_load(reinterpret_cast<char *>(lin) + o,
                    reinterpret_cast<const char *>(src - head) + o, b, bar);
        }
      } else if (tid < 32 + VN) {
        const int i = whole + tid - 32;
        if (i < sup) lin[i] = ldcg(src - head + i);
      }
      __syncthreads();
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
      for (int i = tid; i < len; i += NT) lin[i] = ldcg(src + i);
      __syncthreads();
    }
    // this thread's window positions [tid * kpt, tid * kpt + kpt) as 16-byte
    // chunks, taken in rotated order (chunk jj + rot, wrapping): a quarter
    // warp's eight threads read eight different bank groups
    constexpr int NCH = KPT / VN;
    const int nch = kpt / VN;
    const int rot = NCH >= 8 ? (tid & 7) : ((tid * NCH) >> 3) & (NCH - 1);
    const KV *chunks = reinterpret_cast<const KV *>(lin) + (size_t)tid * nch;
#pragma unroll
    for (int jj = 0; jj < NCH; ++jj) {
      if ((jj & 7) != 0 || jj < nch) {   // whole granules of 8 chunks
        int c = jj + rot;
        if (c >= nch) c -= nch;
        const KV v = chunks[c];
        const int j0 = tid * kpt + c * VN;
        const bool whole_in = j0 >= head && j0 + VN <= sup;
        U ve[VN];
        ve[0] = chunk_get<0>(v);
        ve[1] = chunk_get<1>(v);
        if constexpr (VN == 4) {
          ve[2] = chunk_get<2>(v);
          ve[3] = chunk_get<3>(v);
        }
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          const bool ok = whole_in || (j0 + e >= head && j0 + e < sup);
          const U x = raw ? C::enc(ve[e]) : ve[e];
          kr[jj * VN + e] = ok ? x : KeyMax<U>::v;
          mn = ok && x < mn ? x : mn;
          mx = ok && x > mx ? x : mx;
        }
      } else {
        break;
      }
    }
  } else {
    // coalesced load of the encoded keys into shared memory (slot rpad(i)),
    // taking the min / max on the way (explicit global loads, a batch in
    // flight before the first shared store: a generic load could alias the
    // shared array and would be serialised)
    const SlotMap<KPT, false> slot(KPT);
    U *kbuf = reinterpret_cast<U *>(smem + 1024);
#ifdef TSQ_S_LB
    constexpr int LB = (KPT % TSQ_S_LB == 0 && KPT >= 64) ? TSQ_S_LB : ((sizeof(U) == 8 || KPT < 16) ? 8 : 16);
#else
    constexpr int LB = (sizeof(U) == 8 || KPT < 16) ? 8 : 16;   // loads in flight per batch
#endif
#pragma unroll 1
    for (int q0 = 0; q0 < KPT; q0 += LB) {
      if (q0 * NT >= len) break;
      U v[LB];
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        const int i = tid + (q0 + q) * NT;
        v[q] = i < len ? ldcg(src + i) : U(0);
      }
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        const int i = tid + (q0 + q) * NT;
        if (i < len) {
          const U x = raw ? C::enc(v[q]) : v[q];
          kbuf[slot(i)] = x;
          mn = x < mn ? x : mn;
          mx = x > mx ? x : mx;
        }
      }
    }
  }
  TSQ_PH(1);
  warp_minmax<U>(mn, mx);
  U *s_mm = reinterpret_cast<U *>(smem);
  if (lane == 0) {
    s_mm[warp] = mn;
    s_mm[NW + warp] = mx;
  }
  __syncthreads();
  after_load();   // the segment's keys are on chip
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const U a = s_mm[w], b = s_mm[NW + w];
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  const U range = mx - mn;
  if (range == 0) {
    // every key equal: already in order
    U *dst = E.dst() + sm.begin;
    const U k = E.raw0 ? C::dec(mn) : mn;
    if (PAY && sm.buf != 0) {
      const uint32_t *ps = E.pay(sm.buf) + sm.begin;
      uint32_t *pd = E.pay0 + sm.begin;
      for (int i = tid; i < len; i += NT) pd[i] = ps[i];
    }
    for (int i = tid; i < len; i += NT) dst[i] = k;
    return;
  }
  const int bits = sizeof(U) == 4 ? 32 - __clz((uint32_t)range) : 64 - __clzll((long long)range);
  // item form: 32-bit items whenever the range fits (records: index packed
  // below the key offset while both fit in 32 bits), else 64-bit items
  if (PAY && bits <= 18) {
    radix_run<C, PAY, CLS, uint32_t, false>(E, sm, smem, mn, 14, bits, kr, head, kpt);
  } else if (sizeof(U) == 4 || bits <= 32) {
    radix_run<C, PAY, CLS, uint32_t, PAY>(E, sm, smem, mn, 0, bits, kr, head, kpt);
  } else if constexpr (sizeof(U) == 8) {
    if (PAY && bits <= 50) radix_run<C, PAY, CLS, u64, false>(E, sm, smem, mn, 14, bits, kr, head, kpt);
    else radix_run<C, PAY, CLS, u64, PAY>(E, sm, smem, mn, 0, bits, kr, head, kpt);
  }
}

// One CTA per queued segment (tickets), one kernel per class (SmallClass).
template <class C, bool PAY, int CLS>
__global__ void __launch_bounds__(RadixGeo<C, PAY, CLS>::NT, RadixGeo<C, PAY, CLS>::K::MINB)
    small_sort_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t *s_ticket = reinterpret_cast<uint32_t *>(smem_raw + 656);
  u64 *bar = reinterpret_cast<u64 *>(smem_raw + 640);
  Ctl *ctl = P->ctl;
  constexpr int cls = CLS;
  const uint32_t n_q = ctl->sq_count[cls];
  const uint32_t cap = P->sq_cap[cls];
  const uint32_t count = n_q < cap ? n_q : cap;
  const SmallSeg *q = P->sq[cls];
  uint32_t *ticket = &ctl->sq_ticket[cls];
  SmallEnv<U> E;
  E.keys0 = reinterpret_cast<const U *>(P->keys[0]);
  E.keys1 = reinterpret_cast<const U *>(P->keys[1]);
  E.pay0 = P->pay[0];
  E.pay1 = P->pay[1];
  E.raw0 = P->raw[0] != 0;
  E.raw1 = P->raw[1] != 0;
  E.aligned = P->aligned[0] != 0 && P->aligned[1] != 0;
  E.n = P->n;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
#ifdef TSQ_S_CLOCK
  if (blockIdx.x == 0 && threadIdx.x == 0) g_ph_last = clock64();
#endif
  uint32_t phase = 0;
  uint64_t elems = 0;
  // tickets are claimed one segment ahead: while a segment is sorted, the
  // next one's keys are on their way into L2 (bulk prefetch)
  if (threadIdx.x == 0) *s_ticket = atomicAdd(ticket, 1u);
  __syncthreads();
  uint32_t t = *s_ticket;
  while (t < count) {
    const SmallSeg sm = q[t];
    __syncthreads();   // everyone has read the ticket
    TSQ_PH(0);
    if (threadIdx.x == 0) *s_ticket = atomicAdd(ticket, 1u);
    auto prefetch_next = [&]() {
#if TSQ_S_PREFETCH
      if (threadIdx.x < 32) {
        const uint32_t tn = *s_ticket;   // written before the barrier just passed
        if (tn < count) {
          const SmallSeg nx = q[tn];
          const char *p0 = reinterpret_cast<const char *>(E.keys(nx.buf) + nx.begin);
          const char *p1 = p0 + (size_t)nx.len * sizeof(U);
          const char *a0 = reinterpret_cast<const char *>(((uintptr_t)p0 + 15) & ~(uintptr_t)15);
          const char *a1 = reinterpret_cast<const char *>((uintptr_t)p1 & ~(uintptr_t)15);
          if (a1 > a0) {
            const size_t per = (((size_t)(a1 - a0) / 32) + 15) & ~(size_t)15;
            const char *b0 = a0 + per * threadIdx.x;
            if (b0 < a1) {
              const size_t nb = (size_t)(a1 - b0) < per ? (size_t)(a1 - b0) : per;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0), "r"((uint32_t)nb)
                           : "memory");
            }
          }
        }
      }
#endif
    };
    radix_sort_seg<C, PAY, CLS>(E, sm, smem_raw, phase, prefetch_next);
    elems += (uint64_t)sm.len;
    __syncthreads();
    TSQ_PH(9);
    t = *s_ticket;
  }
#ifdef TSQ_S_CLOCK
  if (blockIdx.x == 0 && threadIdx.x == 0 && elems) {
    printf("class %d phases (cycles, CTA 0, %llu keys): ticket %lld load %lld minmax+sync %lld items0 %lld reload %lld "
           "zero %lld count %lld scan %lld rank+scatter %lld output %lld\n", CLS, (unsigned long long)elems,
           g_ph[0], g_ph[1], g_ph[2], g_ph[3], g_ph[4], g_ph[5], g_ph[6], g_ph[7], g_ph[8], g_ph[9]);
    for (int i = 0; i < 16; ++i) g_ph[i] = 0;
  }
#endif
  if (RadixGeo<C, PAY, CLS>::LIN && threadIdx.x < 32) bulk_wait0();
  if (threadIdx.x == 0 && elems) {
    atomicAdd(&ctl->small_elements, (u64)elems);
    atomicAdd(&ctl->bytes_small, 2ull * (u64)elems * (sizeof(U) + (PAY ? 4 : 0)));
    atomicAdd(&ctl->writes0, (u64)elems);
  }
}

}  // namespace tsq
