// tsq_small.cuh -- on-chip sort of a small segment: an LSD radix sort over
// the segment's own key range.  This is the role insertion_sort plays in the
// reference (smallsort.py:12-47) for ranges of <= insertion_threshold keys
// (core.py:1652-1658); here, segments of <= small_t keys.
//
// By the time the recursion hands a segment to the on-chip sort, its keys lie
// between two ancestor pivots, so their encoded range is narrow (uniform int32
// at 2^26: ~20 bits for a 16K-key segment).  One CTA per segment:
//
//   1. coalesced load into shared memory, encode, CTA-wide min / max; the
//      active threads (ceil(len / KPT)) read KPT consecutive keys each back
//      ("blocked") and form items = key - min (records: the local index
//      packed below it while both fit, else in a 16-bit side array);
//   2. ceil(bits(range) / 5) stable counting passes of <= 5-bit digits, each:
//        count  every thread bumps its own 16-bit counter (digit, thread) for
//               each of its items, in position order;
//        scan   one exclusive scan over the counters in (digit, thread) order
//               gives every (digit, thread) its first output slot;
//        rank   the same sweep again now hands out slots: each item goes to
//               its slot in shared memory; the next pass reads them back
//               blocked.
//      Thread order = position order inside a digit, so every pass is stable
//      and the LSD passes leave the items in key order.
//   3. keys written back as min + item (caller's encoding, coalesced);
//      record payloads gathered by local index.
//
// Measured alternatives (B200, uniform int32 2^26, profiles/r02*): warp-
// collective ranking with __match_any_sync runs on the ADU pipe at ~2
// SM-cycles per distinct digit in the warp (60 per 8-bit match,
// scripts/micro/match_tp.cu) -- 2.3 ms for the on-chip sort; ballot-based
// peer masks take ~9 instructions per digit bit; per-thread counters cost 6
// instructions per bump.  Blocked global loads straight into registers
// (no shared-memory transpose) were 1.6x slower (32 lines per load
// instruction); two-at-a-time counter bumps cut the shared-memory latency
// stalls but added 10 % instructions (net +4 %).  The round-1 warp bitonic +
// merge-path sort took 0.95 ms at ~320 instructions per key; this one 0.68 ms
// at ~176.
#pragma once

#include "tsq_bitonic.cuh"

namespace tsq {

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

// item slot i -> shared-memory word: one pad word per 32, so both the
// striped (consecutive) and the blocked (stride KE) accesses spread over the
// banks
__device__ __forceinline__ int rpad(int i) { return i + (i >> 5); }

// Shared-memory geometry of one item form (T = u32 / u64 items, IDX =
// separate 16-bit local-index array).  Counters: R (digit) rows of NT 16-bit
// counters (see radix_cnt_byte for the layout), RMAX * NT * 2 bytes.
template <int NT, int CAP, typename T, bool IDX>
struct RadixForm {
  static constexpr int CAPP = CAP + CAP / 32;              // padded item slots
  static constexpr int DBMAX = (sizeof(T) == 8 && IDX) ? 4 : 5;
  static constexpr int RMAX = 1 << DBMAX;
  static constexpr size_t MISC = 1024;  // min/max exchange [0, 512), warp totals [512, 640)
  static constexpr size_t OFF_BUF = MISC;
  static constexpr size_t OFF_IBUF = OFF_BUF + (size_t)CAPP * sizeof(T);
  static constexpr size_t OFF_CNT = (OFF_IBUF + (IDX ? (size_t)CAPP * 2 : 0) + 15) & ~(size_t)15;
  static constexpr size_t END = OFF_CNT + (size_t)RMAX * NT * 2;
};

// Counter (digit d, thread t) layout.  Threads form groups of 64, m = t / 64;
// a row (digit) is NT/2 32-bit words, a group 32 of them: lane l = t % 32 of
// the group's first warp owns the low half of one word, the same lane of its
// second warp the high half.  So a warp's bumps touch 32 distinct words of
// one block per row -- conflict-free whatever digits its lanes hold (rows are
// a multiple of 32 words apart).  Inside a block the 16-byte chunks are
// XOR-swizzled by m, so the scan threads (one per block) read their blocks
// with conflict-free 16-byte vectors: lane l sits in chunk (l/4) ^ (m % 8).
template <int NT>
__device__ __forceinline__ uint32_t radix_cnt_byte(int t) {
  const int m = t >> 6, h = (t >> 5) & 1, l = t & 31;
  const int word = m * 32 + ((((l >> 2) ^ (m & 7)) << 2) | (l & 3));
  return (uint32_t)(word * 4 + 2 * h);
}

template <class C, bool PAY, int NT>
struct RadixGeo {
  typedef typename C::U U;
  static constexpr int NW = NT / 32;
  static constexpr int CLASS = NT == kThreads ? 0 : (NT == 2 * kThreads ? 1 : 2);
  static constexpr int CAP = CLASS == 0   ? kSmallT
                             : CLASS == 1 ? ((!PAY && sizeof(U) == 4) ? kSmallHuge : kSmallMax)
                                          : ((!PAY && sizeof(U) == 4) ? kSmallGiant : kSmallHuge);
  static constexpr int KPT = CAP / NT;
  static constexpr size_t S32 = RadixForm<NT, CAP, uint32_t, PAY>::END;
  static constexpr size_t S64a = sizeof(U) == 8 ? RadixForm<NT, CAP, u64, PAY>::END : 0;
  static constexpr size_t S64b = sizeof(U) == 8 ? RadixForm<NT, CAP, u64, false>::END : 0;
  static constexpr size_t S64 = S64a > S64b ? S64a : S64b;
  static constexpr size_t SMEM = S32 > S64 ? S32 : S64;
  static_assert(KPT * NT == CAP, "capacity is a whole number of items per thread");
  static_assert(2 * NW * sizeof(U) <= 512 && NW <= 32, "misc region");
};

// Exclusive scan of the R x NT counters in (digit, thread) order.  In that
// order a block (digit d, group m) is 64 consecutive counters: the 32 low
// halves (threads 64m .. 64m+31) then the 32 high halves.  Scan thread g
// takes block g = d * (NT/64) + m: the packed sum P of its 32 words is two
// 16-bit totals (no carries: a segment has < 2^16 items), and with s0 = the
// block's exclusive prefix, word j becomes (s0 | (s0 + lo(P)) << 16) plus the
// packed running sum of the words before it.
template <int NT>
__device__ __forceinline__ void radix_scan(uint16_t *cnt, uint32_t *wt, int R) {
  constexpr int NW = NT / 32;
  constexpr int GPR = NT / 64;  // blocks per row
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool own = tid < R * GPR;
  const int sw = (tid % GPR) & 7;
  const uint4 *blk = reinterpret_cast<const uint4 *>(cnt) + tid * 8;
  uint32_t packed = 0;
  if (own) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 v = blk[c ^ sw];
      packed += v.x + v.y + v.z + v.w;
    }
  }
  const uint32_t sum = (packed & 0xffffu) + (packed >> 16);
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
  if (own) {
    uint32_t run = s0 | ((s0 + (packed & 0xffffu)) << 16);
    uint4 *wb = reinterpret_cast<uint4 *>(cnt) + tid * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint4 v = wb[c ^ sw];
      uint4 o;
      o.x = run; run += v.x;
      o.y = run; run += v.y;
      o.z = run; run += v.z;
      o.w = run; run += v.w;
      wb[c ^ sw] = o;
    }
  }
}

// Radix passes over items T whose digits occupy bits [b0, b0 + bits); IDX:
// the local index travels in a 16-bit side array (else it is packed below
// b0 for records, or absent).  On entry the encoded keys (U) sit in shared
// memory at slot rpad(i) of a U-typed array over the same region; the first
// pass turns them into items as it reads them back blocked.  `lo` is their
// minimum.
template <class C, bool PAY, int NT, typename T, bool IDX>
__device__ __forceinline__ void radix_run(const Params *P, const SmallSeg &sm,
                                          unsigned char *smem, typename C::U lo, int b0,
                                          int bits) {
  typedef typename C::U U;
  typedef RadixGeo<C, PAY, NT> G;
  typedef RadixForm<NT, G::CAP, T, IDX> F;
  constexpr int KPT = G::KPT;
  constexpr bool PACKED = PAY && !IDX;
  const int tid = threadIdx.x;
  const int len = sm.len;
  // active threads hold KPT consecutive positions each (t*KPT .. t*KPT +
  // KPT - 1); pads past len (the last thread's tail) sort last (all ones)
  const int NA = (len + KPT - 1) / KPT;
  const bool act = tid < NA;
  T *buf = reinterpret_cast<T *>(smem + F::OFF_BUF);
  uint16_t *ibuf = reinterpret_cast<uint16_t *>(smem + F::OFF_IBUF);
  uint16_t *cnt = reinterpret_cast<uint16_t *>(smem + F::OFF_CNT);
  uint32_t *wt = reinterpret_cast<uint32_t *>(smem) + 128;
  // this thread's counter of digit 0; rows are NT * 2 bytes apart
  unsigned char *mycb = reinterpret_cast<unsigned char *>(cnt) + radix_cnt_byte<NT>(tid);
  // this thread's slots: rpad(t*KPT + k) = rpad(t*KPT) + k (KPT divides 32)
  T *mine = buf + rpad(tid * KPT);
  uint16_t *imine = ibuf + rpad(tid * KPT);
  const int passes = (bits + F::DBMAX - 1) / F::DBMAX;   // bits >= 1
  const int db = (bits + passes - 1) / passes;
  const uint32_t mask = (1u << db) - 1u;
  const int R = 1 << db;
  const U *rmine = reinterpret_cast<const U *>(smem + F::OFF_BUF) + rpad(tid * KPT);
  T it[KPT];
  uint16_t ix[IDX ? KPT : 1];
#pragma unroll 1
  for (int ps = 0; ps < passes; ++ps) {
    const int sh = b0 + db * ps;
    __syncthreads();   // previous scatter (or the key load) complete
    if (ps == 0) {
      if (act) {
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
          const int p = tid * KPT + k;
          it[k] = p < len ? (((T)(rmine[k] - lo) << b0) | (PACKED ? (T)p : (T)0)) : ~T(0);
          if (IDX) ix[k] = (uint16_t)p;
        }
      }
      // 64-bit keys in 32-bit items: the key array overlaps the counters
      if (sizeof(U) > sizeof(T)) __syncthreads();
    } else if (act) {
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        it[k] = mine[k];
        if (IDX) ix[k] = imine[k];
      }
    }
    {
      uint4 *c4 = reinterpret_cast<uint4 *>(cnt);
      const int n4 = R * NT / 8;
      for (int i = tid; i < n4; i += NT) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    // count: this thread's items, in position order
    if (act) {
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        uint16_t *a = reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k] >> sh) & mask) * (2 * NT));
        *a = (uint16_t)(*a + 1u);
      }
    }
    __syncthreads();
    radix_scan<NT>(cnt, wt, R);
    __syncthreads();
    // rank + scatter, same order
    if (act) {
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        uint16_t *a = reinterpret_cast<uint16_t *>(mycb + ((uint32_t)(it[k] >> sh) & mask) * (2 * NT));
        const uint32_t r = *a;
        *a = (uint16_t)(r + 1u);
        TSQ_CHECK(r < (uint32_t)(NA * KPT));
        buf[rpad((int)r)] = it[k];
        if (IDX) ibuf[rpad((int)r)] = ix[k];
      }
    }
  }
  __syncthreads();
  // buf[0, len) holds the sorted items
  U *dst = reinterpret_cast<U *>(P->keys[0]) + sm.begin;
  const bool dst_raw = P->raw[0] != 0;
  if (PAY) {
    // payloads gathered by local index from the source (an L1/L2-resident
    // window) into registers, all before any is written (the source may be
    // buffer 0 itself)
    const uint32_t *ps = P->pay[sm.buf] + sm.begin;
    uint32_t pv[KPT];
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
      const int i = tid + q * NT;
      pv[q] = i < len ? ps[IDX ? (uint32_t)ibuf[rpad(i)]
                               : (uint32_t)(buf[rpad(i)] & (T)((1u << b0) - 1u))]
                      : 0u;
    }
    __syncthreads();
    uint32_t *pd = P->pay[0] + sm.begin;
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
      const int i = tid + q * NT;
      if (i < len) pd[i] = pv[q];
    }
  }
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int i = tid + q * NT;
    if (i < len) {
      const U k = lo + (U)(buf[rpad(i)] >> b0);
      dst[i] = dst_raw ? C::dec(k) : k;
    }
  }
}

// Sort one queued segment (all threads of the CTA).
template <class C, bool PAY, int NT>
__device__ __forceinline__ void radix_sort_seg(const Params *P, const SmallSeg &sm,
                                               unsigned char *smem) {
  typedef typename C::U U;
  typedef RadixGeo<C, PAY, NT> G;
  constexpr int KPT = G::KPT, NW = G::NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int len = sm.len;
  const U *src = reinterpret_cast<const U *>(P->keys[sm.buf]) + sm.begin;
  const bool raw = P->raw[sm.buf] != 0;
  TSQ_CHECK(len >= 1 && len <= G::CAP && sm.begin >= 0 && sm.begin + len <= P->n);
  // coalesced load of the encoded keys into shared memory (slot rpad(i)),
  // taking the min / max on the way (explicit global loads, a batch in
  // flight before the first shared store: a generic load could alias the
  // shared array and would be serialised)
  U *kbuf = reinterpret_cast<U *>(smem + RadixForm<NT, G::CAP, U, false>::OFF_BUF);
  U mn = KeyMax<U>::v, mx = U(0);
  constexpr int LB = (sizeof(U) == 8 || KPT < 16) ? 8 : 16;   // loads in flight per batch
#pragma unroll
  for (int q0 = 0; q0 < KPT; q0 += LB) {
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
        kbuf[rpad(i)] = x;
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
      }
    }
  }
  warp_minmax<U>(mn, mx);
  U *s_mm = reinterpret_cast<U *>(smem);
  if (lane == 0) {
    s_mm[warp] = mn;
    s_mm[NW + warp] = mx;
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const U a = s_mm[w], b = s_mm[NW + w];
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  const U range = mx - mn;
  if (range == 0) {
    // every key equal: already in order
    U *dst = reinterpret_cast<U *>(P->keys[0]) + sm.begin;
    const U k = P->raw[0] ? C::dec(mn) : mn;
    if (PAY && sm.buf != 0) {
      const uint32_t *ps = P->pay[sm.buf] + sm.begin;
      uint32_t *pd = P->pay[0] + sm.begin;
      for (int i = tid; i < len; i += NT) pd[i] = ps[i];
    }
    for (int i = tid; i < len; i += NT) dst[i] = k;
    return;
  }
  const int bits = sizeof(U) == 4 ? 32 - __clz((uint32_t)range) : 64 - __clzll((long long)range);
  // item form: 32-bit items whenever the range fits (records: index packed
  // below the key offset while both fit in 32 bits), else 64-bit items
  if (PAY && bits <= 18) {
    radix_run<C, PAY, NT, uint32_t, false>(P, sm, smem, mn, 14, bits);
  } else if (sizeof(U) == 4 || bits <= 32) {
    radix_run<C, PAY, NT, uint32_t, PAY>(P, sm, smem, mn, 0, bits);
  } else if constexpr (sizeof(U) == 8) {
    if (PAY && bits <= 50) radix_run<C, PAY, NT, u64, false>(P, sm, smem, mn, 14, bits);
    else radix_run<C, PAY, NT, u64, PAY>(P, sm, smem, mn, 0, bits);
  }
}

// One CTA per queued segment (tickets), one kernel per class: NT = 256 takes
// the queue of segments of <= kSmallT keys, NT = 512 kSmallT+1 .. its
// capacity, NT = 1024 (4-byte keys only) the rest up to kSmallGiant.
template <class C, bool PAY, int NT>
__global__ void __launch_bounds__(NT, NT == kThreads ? 4 : (NT == 2 * kThreads ? 2 : 1))
    small_sort_kernel(const Params *__restrict__ P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_ticket;
  Ctl *ctl = P->ctl;
  constexpr int cls = RadixGeo<C, PAY, NT>::CLASS;
  const uint32_t n_q = ctl->sq_count[cls];
  const uint32_t cap = P->sq_cap[cls];
  const uint32_t count = n_q < cap ? n_q : cap;
  const SmallSeg *q = P->sq[cls];
  uint32_t *ticket = &ctl->sq_ticket[cls];
  uint64_t elems = 0;
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t t = s_ticket;
    __syncthreads();
    if (t >= count) break;
    const SmallSeg sm = q[t];
    radix_sort_seg<C, PAY, NT>(P, sm, smem_raw);
    elems += (uint64_t)sm.len;
    __syncthreads();
  }
  if (threadIdx.x == 0 && elems) {
    typedef typename C::U U;
    atomicAdd(&ctl->small_elements, (u64)elems);
    atomicAdd(&ctl->bytes_small, 2ull * (u64)elems * (sizeof(U) + (PAY ? 4 : 0)));
    atomicAdd(&ctl->writes0, (u64)elems);
  }
}

}  // namespace tsq
