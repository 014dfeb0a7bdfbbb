// tsq_consume.cuh -- counter and consumer warps, and the partition kernel
// entry.  Included by tsq_partition.cuh after the producer and look-back
// warps.
//
//   counter warps (4)  all take every tile as soon as it lands, each
//                      counting two consumer warps' keys: per consumer
//                      thread the (<, >, valid) counts and their exclusive
//                      lane prefix; the last one to finish combines the tile
//                      aggregate and hands the stage to the look-back warps.
//                      Verification tiles (sorted / reversed fast paths) are
//                      checked here too.
//   consumers (8)      once the tile's offsets are known: keys to registers,
//                      then (after a named barrier) restaged in place -- each
//                      to its thread's next < slot or > slot, aligned like
//                      the destination -- and written with cp.async.bulk
//                      stores (scalar stores for the <= 3 unaligned keys at
//                      each end); the stage is released once the stores
//                      have read it
#pragma once

namespace tsq {

// Write one staged run: element j of the run (global index D + j) sits at
// R[(D & 3) + j]; the 16B-aligned body goes out as one bulk store issued by
// `issuer`, the <= 3 keys at each ragged end as scalar stores by lanes < 8
// of warp `scal_warp`.
template <typename T>
__device__ __forceinline__ void emit_run(T *g, long long D, long long L, const T *R,
                                         bool issuer, int scal_warp) {
  if (L <= 0) return;
  const long long b0 = (D + kAlign - 1) & ~(long long)(kAlign - 1);
  const long long b1 = (D + L) & ~(long long)(kAlign - 1);
  const long long base = D & ~(long long)(kAlign - 1);
  const bool body = b1 > b0;
  TSQ_CHECK(!body || ((reinterpret_cast<uintptr_t>(g + b0) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(R + (b0 - base)) & 15) == 0));
  if (body && issuer)
    bulk_store(g + b0, R + (b0 - base), (uint32_t)((b1 - b0) * (long long)sizeof(T)));
  if ((int)(threadIdx.x >> 5) == scal_warp) {
    const int lane = threadIdx.x & 31;
    const long long h = body ? (b0 - D) : L;   // head count (all if no body)
    const long long ts = body ? (b1 - D) : L;  // tail start
    const long long e = lane < h ? lane : ts + (lane - h);
    if (lane < 8 && (lane < h || e < L)) g[D + e] = R[(D - base) + e];
  }
}

// per-stage counts of each consumer warp's keys (<, ==, >) and, per
// consumer thread, the (<, >, valid) counts of the lanes before it in its
// warp, packed 10 bits each
struct StageCounts {
  uint32_t w[kConsumerWarps][3];
  uint32_t t[kConsumers];
  u64 x[kConsumerWarps];  // per consumer warp: exclusive (<, ==, >) prefix, 21 bits each
  u64 tot;                // the tile's (<, ==, >) totals, same packing
};

// One key against the pivot: two compares and two predicated increments.
// (The compiler's code for `lt += x < piv` is an add plus a predicated move
// per side in one serial chain per counter; a counter lane counts 48 keys of
// a tile, and the counter warps' 1.7 us per tile -- per-tile timeline,
// scripts/trace_level.py -- is the longest stage of a pass whose data comes
// from L2.)  Callers keep one pair of counters per vector element, so the
// dependent chains are a quarter as long.
template <bool SIGNED>
__device__ __forceinline__ void count_key(uint32_t &lt, uint32_t &gt, uint32_t x, uint32_t piv) {
  if (SIGNED)
    asm("{\n\t.reg .pred pl, pg;\n\tsetp.lt.s32 pl, %2, %3;\n\tsetp.gt.s32 pg, %2, %3;\n\t"
        "@pl add.u32 %0, %0, 1;\n\t@pg add.u32 %1, %1, 1;\n\t}"
        : "+r"(lt), "+r"(gt) : "r"(x), "r"(piv));
  else
    asm("{\n\t.reg .pred pl, pg;\n\tsetp.lt.u32 pl, %2, %3;\n\tsetp.gt.u32 pg, %2, %3;\n\t"
        "@pl add.u32 %0, %0, 1;\n\t@pg add.u32 %1, %1, 1;\n\t}"
        : "+r"(lt), "+r"(gt) : "r"(x), "r"(piv));
}
template <bool SIGNED>
__device__ __forceinline__ void count_key(uint32_t &lt, uint32_t &gt, u64 x, u64 piv) {
  if (SIGNED)
    asm("{\n\t.reg .pred pl, pg;\n\tsetp.lt.s64 pl, %2, %3;\n\tsetp.gt.s64 pg, %2, %3;\n\t"
        "@pl add.u32 %0, %0, 1;\n\t@pg add.u32 %1, %1, 1;\n\t}"
        : "+r"(lt), "+r"(gt) : "l"(x), "l"(piv));
  else
    asm("{\n\t.reg .pred pl, pg;\n\tsetp.lt.u64 pl, %2, %3;\n\tsetp.gt.u64 pg, %2, %3;\n\t"
        "@pl add.u32 %0, %0, 1;\n\t@pg add.u32 %1, %1, 1;\n\t}"
        : "+r"(lt), "+r"(gt) : "l"(x), "l"(piv));
}

// one consumer warp's keys of a stage, counted by a counter lane in the
// order the consumer will rank them; FULL: the whole tile is the segment's
// RAWCMP: the stage holds the caller's encoding of a kRawOrder key type --
// compare natively against the decoded pivot, no per-key re-encoding.
template <class C, bool PAY, bool FULL, bool RAWCMP>
__device__ __forceinline__ uint32_t count_slice(const typename C::U *sk, int w, int lane, bool raw,
                                                typename C::U piv, int rlo, int rhi) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  uint32_t lt = 0, gt = 0, va = 0;
#ifdef TSQ_EXP_OLD_COUNT
  constexpr bool kLean = false;
#else
  constexpr bool kLean = FULL;
#endif
  if constexpr (kLean) {
    uint32_t l4[G::VN], g4[G::VN];
#pragma unroll
    for (int q = 0; q < G::VN; ++q) l4[q] = g4[q] = 0;
#pragma unroll
    for (int v = 0; v < G::VPT; ++v) {
      const int e0 = (v * kConsumers + w * 32 + lane) * G::VN;
      U key[G::VN];
      unpack(*reinterpret_cast<const typename Vec<U>::K *>(sk + e0), key);
#pragma unroll
      for (int q = 0; q < G::VN; ++q) {
        const U x = RAWCMP ? key[q] : (raw ? C::enc(key[q]) : key[q]);
        count_key<RAWCMP && C::kSigned>(l4[q], g4[q], x, piv);
      }
    }
#pragma unroll
    for (int q = 0; q < G::VN; ++q) { lt += l4[q]; gt += g4[q]; }
    va = G::IPT;
  } else {
#pragma unroll
    for (int v = 0; v < G::VPT; ++v) {
      const int e0 = (v * kConsumers + w * 32 + lane) * G::VN;
      U key[G::VN];
      unpack(*reinterpret_cast<const typename Vec<U>::K *>(sk + e0), key);
#pragma unroll
      for (int q = 0; q < G::VN; ++q) {
        const U x = RAWCMP ? key[q] : (raw ? C::enc(key[q]) : key[q]);
        const bool below = RAWCMP ? C::rlt(x, piv) : x < piv;
        const bool above = RAWCMP ? C::rlt(piv, x) : x > piv;
        if (FULL) {
          lt += below ? 1u : 0u;
          gt += above ? 1u : 0u;
        } else {
          const int idx = e0 + q;
          const bool valid = idx >= rlo && idx < rhi;
          lt += (valid && below) ? 1u : 0u;
          gt += (valid && above) ? 1u : 0u;
          va += valid ? 1u : 0u;
        }
      }
    }
    if (FULL) va = G::IPT;
  }
  return lt | (gt << 10) | (va << 20);
}

// Per-stage scratch of the counter warps: how many are done with the stage.
struct CounterShare {
  uint32_t finished;
};

// Counter warps: all kCounterWarps warps take every tile, warp cw counting
// the slices of consumer warps [cw * kSlices, (cw + 1) * kSlices) -- a tile
// is counted in a quarter of the time one warp would take.  The warp that
// finishes a tile last combines the shares into the tile's aggregate (and
// in reproducible mode publishes it for the decoupled look-back) and hands
// the stage to the look-back warps, which turn it into the tile's offsets.
template <class C, bool PAY>
__device__ __forceinline__ void counter_loop(const Params *P, int cur, const typename C::U *in_k,
                                             u64 *full, u64 *aggr, u64 *empty, StageMeta *meta,
                                             StageCounts *sc, CounterShare *cs,
                                             int cw) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  constexpr int kSlices = kConsumerWarps / kCounterWarps;
  const int lane = threadIdx.x & 31;
  const bool reproducible = P->reproducible != 0;
  const uint32_t level = P->ctl->level;
  (void)level;
  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % G::STAGES);
    wait_full_consumer(&full[s], (it / G::STAGES) & 1u);
    StageMeta &m = meta[s];
    if (m.kind == KIND_DONE) {
      // out of tiles: the last counter warp here passes the marker on
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&cs[s].finished, 1u) == kCounterWarps - 1) mbar_arrive(&aggr[s]);
      }
      return;
    }
    const uint32_t t = m.t;
    if (lane == 0 && cw == 0) TSQ_MARK(level, t, 2);
    const U *sk = in_k + (size_t)s * G::SLOT;
    const bool raw = P->raw[m.buf] != 0;
    const bool rawcmp = C::kRawOrder && raw;
    const int rlo = (int)(m.lo - m.tstart), rhi = (int)(m.hi - m.tstart);
    const bool part = m.kind == KIND_PARTITION;
    if (!part) {
      // verification: every pair (i, i+1) of the segment's keys in this tile,
      // the last one against the first key of the next tile
      bool bad = false;
      if (!m.skip && rlo == 0 && rhi == G::TILE) {
        // whole tile: 16-byte vectors, each checked against its successor
        const bool asc = m.kind == KIND_VERIFY_ASC;
        constexpr int VN = G::VN;
        constexpr int NV = G::TILE / VN;  // vectors per tile
        const U *gk = reinterpret_cast<const U *>(P->keys[m.buf]);
#pragma unroll 4
        for (int v = cw * (NV / kCounterWarps) + lane; v < (cw + 1) * (NV / kCounterWarps);
             v += 32) {
          U k[VN + 1];
          unpack(*reinterpret_cast<const typename Vec<U>::K *>(sk + v * VN), k);
          bool have = true;
          if (v + 1 < NV) k[VN] = sk[(v + 1) * VN];
          else if (m.has_next) k[VN] = gk[m.hi];
          else { have = false; k[VN] = k[VN - 1]; }
          if (rawcmp) {
#pragma unroll
            for (int q = 0; q < VN; ++q)
              if (q + 1 < VN || have)
                bad |= asc ? C::rlt(k[q + 1], k[q]) : C::rlt(k[q], k[q + 1]);
          } else {
#pragma unroll
            for (int q = 0; q <= VN; ++q)
              if (raw) k[q] = C::enc(k[q]);
#pragma unroll
            for (int q = 0; q < VN; ++q)
              if (q + 1 < VN || have) bad |= asc ? (k[q] > k[q + 1]) : (k[q] < k[q + 1]);
          }
        }
      } else if (!m.skip) {
        const bool asc = m.kind == KIND_VERIFY_ASC;
        for (int i = rlo + cw * 32 + lane; i < rhi; i += 32 * kCounterWarps) {
          U a = sk[i], b = a;
          bool have = true;
          if (i + 1 < rhi) b = sk[i + 1];
          else if (m.has_next) b = reinterpret_cast<const U *>(P->keys[m.buf])[m.hi];
          else have = false;
          if (rawcmp) {
            if (have) bad |= asc ? C::rlt(b, a) : C::rlt(a, b);
          } else {
            if (raw) {
              a = C::enc(a);
              b = C::enc(b);
            }
            if (have) bad |= asc ? (a > b) : (a < b);
          }
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&P->segs[cur][m.sid].fail, 1u);
    } else {
      // this warp's consumer slices, in the order the consumers rank them;
      // all counted first, then their lane scans interleaved
      const U piv = (U)m.pivot;
      uint32_t own[kSlices], inc[kSlices];
      const bool whole = rlo == 0 && rhi == G::TILE;
      if (rawcmp) {
        const U pr = C::dec(piv);  // the pivot in the caller's encoding
        if (whole) {
#pragma unroll
          for (int j = 0; j < kSlices; ++j)
            own[j] = count_slice<C, PAY, true, true>(sk, cw * kSlices + j, lane, raw, pr, rlo, rhi);
        } else {
#pragma unroll
          for (int j = 0; j < kSlices; ++j)
            own[j] = count_slice<C, PAY, false, true>(sk, cw * kSlices + j, lane, raw, pr, rlo, rhi);
        }
      } else if (whole) {
#pragma unroll
        for (int j = 0; j < kSlices; ++j)
          own[j] = count_slice<C, PAY, true, false>(sk, cw * kSlices + j, lane, raw, piv, rlo, rhi);
      } else {
#pragma unroll
        for (int j = 0; j < kSlices; ++j)
          own[j] = count_slice<C, PAY, false, false>(sk, cw * kSlices + j, lane, raw, piv, rlo, rhi);
      }
      // at most 32 * IPT = 512 per class: three 10-bit counts, scanned
      // across the lanes; each consumer thread gets its exclusive prefix
#pragma unroll
      for (int j = 0; j < kSlices; ++j) inc[j] = own[j];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int j = 0; j < kSlices; ++j) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc[j], o);
          if (lane >= o) inc[j] += y;
        }
      }
#pragma unroll
      for (int j = 0; j < kSlices; ++j) {
        const int w = cw * kSlices + j;
        sc[s].t[w * 32 + lane] = inc[j] - own[j];
        const uint32_t pk = __shfl_sync(0xffffffffu, inc[j], 31);
        const uint32_t lt = pk & 0x3ffu, gt = (pk >> 10) & 0x3ffu, va = pk >> 20;
        if (lane == 0) {
          sc[s].w[w][0] = lt;
          sc[s].w[w][1] = va - lt - gt;
          sc[s].w[w][2] = gt;
        }
      }
    }
    __syncwarp();
    // the last counter warp done with the stage hands it on
    uint32_t last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(&cs[s].finished, 1u) == kCounterWarps - 1 ? 1u : 0u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      if (part) {
        // consumer warps' (<, ==, >) counts -> exclusive prefixes and the
        // tile totals (lanes 0..7, 21-bit fields), so a consumer thread
        // reads its warp's offsets instead of summing the others'
        u64 pk = 0;
        if (lane < kConsumerWarps)
          pk = (u64)ld_volatile32(&sc[s].w[lane][0]) |
               ((u64)ld_volatile32(&sc[s].w[lane][1]) << 21) |
               ((u64)ld_volatile32(&sc[s].w[lane][2]) << 42);
        u64 inc = pk;
#pragma unroll
        for (int o = 1; o < kConsumerWarps; o <<= 1) {
          const u64 y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        if (lane < kConsumerWarps) sc[s].x[lane] = inc - pk;
        const u64 tot = __shfl_sync(0xffffffffu, inc, kConsumerWarps - 1);
        if (lane == 0) {
          sc[s].tot = tot;
          const uint32_t tl = (uint32_t)(tot & 0x1fffffull), tq = (uint32_t)((tot >> 21) & 0x1fffffull);
          const uint32_t tg = (uint32_t)(tot >> 42);
          const u64 agg = ((u64)tl << 31) | (u64)tg;
          m.agg = agg;
          m.eq_excl = tq;  // (the look-back warp turns it into a slot)
          if (reproducible)
            st_volatile(&P->lookback[cur][t], (m.k == 0 ? kFlagInc : kFlagAgg) | agg);
          TSQ_MARK(level, t, 3);
        }
      }
      if (lane == 0) {
        cs[s].finished = 0;
        // the look-back warps turn the aggregate into the tile's offsets
        mbar_arrive(&aggr[s]);
      }
    }
    if (lane == 0) mbar_arrive(&empty[s]);  // done reading the stage
  }
}

// One consumer thread's keys (and payloads) of a stage, into registers.
template <class C, bool PAY>
__device__ __forceinline__ void load_keys(const typename C::U *sk, const uint32_t *sp, int tid,
                                          typename C::U *key, uint32_t *pay) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
#pragma unroll
  for (int v = 0; v < G::VPT; ++v) {
    const int e0 = (v * kConsumers + tid) * G::VN;
    unpack(*reinterpret_cast<const typename Vec<U>::K *>(sk + e0), key + v * G::VN);
    if (PAY) unpack(*reinterpret_cast<const typename Vec<U>::P *>(sp + e0), pay + v * G::VN);
  }
}

// One key of a whole keys-only tile into its run: two compares, one
// predicated store at the selected side's slot (a second, predicated-off
// store per key measured 2 % slower per sort) and a predicated step per side
// (the compiler's own code for the same
// loop re-derives each slot address from the rank and repeats the compares,
// ~12 instructions per key).  a_lt / a_gt: shared-window byte addresses of the
// thread's next < slot and next > slot; s_lt / s_gt: the (signed) byte steps
// to the slot after it.
template <bool SIGNED>
__device__ __forceinline__ void place_key(uint32_t &a_lt, uint32_t &a_gt, uint32_t s_lt,
                                          uint32_t s_gt, uint32_t x, uint32_t piv, uint32_t y) {
  if (SIGNED)
    asm volatile(
        "{\n\t.reg .pred pl, pg, pe;\n\t.reg .u32 a;\n\t"
        "setp.lt.s32 pl, %2, %3;\n\tsetp.gt.s32 pg, %2, %3;\n\t"
        "selp.u32 a, %0, %1, pl;\n\tor.pred pe, pl, pg;\n\t@pe st.shared.u32 [a], %4;\n\t"
        "@pl add.u32 %0, %0, %5;\n\t@pg add.u32 %1, %1, %6;\n\t}"
        : "+r"(a_lt), "+r"(a_gt)
        : "r"(x), "r"(piv), "r"(y), "r"(s_lt), "r"(s_gt)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred pl, pg, pe;\n\t.reg .u32 a;\n\t"
        "setp.lt.u32 pl, %2, %3;\n\tsetp.gt.u32 pg, %2, %3;\n\t"
        "selp.u32 a, %0, %1, pl;\n\tor.pred pe, pl, pg;\n\t@pe st.shared.u32 [a], %4;\n\t"
        "@pl add.u32 %0, %0, %5;\n\t@pg add.u32 %1, %1, %6;\n\t}"
        : "+r"(a_lt), "+r"(a_gt)
        : "r"(x), "r"(piv), "r"(y), "r"(s_lt), "r"(s_gt)
        : "memory");
}
template <bool SIGNED>
__device__ __forceinline__ void place_key(uint32_t &a_lt, uint32_t &a_gt, uint32_t s_lt,
                                          uint32_t s_gt, u64 x, u64 piv, u64 y) {
  if (SIGNED)
    asm volatile(
        "{\n\t.reg .pred pl, pg, pe;\n\t.reg .u32 a;\n\t"
        "setp.lt.s64 pl, %2, %3;\n\tsetp.gt.s64 pg, %2, %3;\n\t"
        "selp.u32 a, %0, %1, pl;\n\tor.pred pe, pl, pg;\n\t@pe st.shared.u64 [a], %4;\n\t"
        "@pl add.u32 %0, %0, %5;\n\t@pg add.u32 %1, %1, %6;\n\t}"
        : "+r"(a_lt), "+r"(a_gt)
        : "l"(x), "l"(piv), "l"(y), "r"(s_lt), "r"(s_gt)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred pl, pg, pe;\n\t.reg .u32 a;\n\t"
        "setp.lt.u64 pl, %2, %3;\n\tsetp.gt.u64 pg, %2, %3;\n\t"
        "selp.u32 a, %0, %1, pl;\n\tor.pred pe, pl, pg;\n\t@pe st.shared.u64 [a], %4;\n\t"
        "@pl add.u32 %0, %0, %5;\n\t@pg add.u32 %1, %1, %6;\n\t}"
        : "+r"(a_lt), "+r"(a_gt)
        : "l"(x), "l"(piv), "l"(y), "r"(s_lt), "r"(s_gt)
        : "memory");
}

// Stage one consumer thread's keys back into the stage, in output order:
// each key goes to the thread's next < slot (counting up) or next > slot
// (counting down); records also stage the == payloads.  MODE 0: both
// buffers hold encoded keys, 1: source raw, 2: destination raw, 3: both raw.
// plt / pgt / peq: the thread's first < slot, first > slot (its runs' last)
// and first == payload slot; st_lt / st_gt: slots between two consecutive
// keys of the thread in a run (whole keys-only tiles; 1 otherwise).
template <class C, bool PAY, bool FULL, int MODE>
__device__ __forceinline__ void stage_keys(const typename C::U *key, const uint32_t *pay, int tid,
                                           typename C::U piv, int rlo, int rhi, uint32_t plt,
                                           uint32_t pgt, uint32_t peq, uint32_t st_lt,
                                           uint32_t st_gt, typename C::U *ok, uint32_t *op) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  // MODE 3 with a raw-order codec: native compare against the decoded pivot
  constexpr bool RC = MODE == 3 && C::kRawOrder;
  constexpr bool LEAN = !PAY && FULL;
  uint32_t a_lt = 0, a_gt = 0, s_lt = 0, s_gt = 0;
  if (LEAN) {
    a_lt = smem_u32(ok + plt);
    a_gt = smem_u32(ok + pgt);
    s_lt = st_lt * (uint32_t)sizeof(U);
    s_gt = 0u - st_gt * (uint32_t)sizeof(U);
  }
#pragma unroll
  for (int v = 0; v < G::VPT; ++v) {
    const int e0 = (v * kConsumers + tid) * G::VN;
#pragma unroll
    for (int q = 0; q < G::VN; ++q) {
      const U kq = key[v * G::VN + q];
      const U x = RC ? kq : ((MODE & 1) ? C::enc(kq) : kq);
      const U y = MODE == 2 ? C::dec(kq) : (MODE == 1 ? x : kq);
      if (LEAN) {
        place_key<RC && C::kSigned>(a_lt, a_gt, s_lt, s_gt, x, piv, y);
        continue;
      }
      const bool valid = FULL || (e0 + q >= rlo && e0 + q < rhi);
      const bool is_lt = valid && (RC ? C::rlt(x, piv) : x < piv);
      const bool is_gt = valid && (RC ? C::rlt(piv, x) : x > piv);
      if (PAY) {
        const uint32_t pos = is_lt ? plt : (is_gt ? pgt : peq);
        if (is_lt || is_gt) ok[pos] = y;
        if (valid) op[pos] = pay[v * G::VN + q];
        peq += (valid && !is_lt && !is_gt) ? 1u : 0u;
      } else {
        const uint32_t pos = is_lt ? plt : pgt;
        if (is_lt || is_gt) ok[pos] = y;
      }
      plt += is_lt ? 1u : 0u;
      pgt -= is_gt ? 1u : 0u;
    }
  }
}

// Emit one tile: its offsets (reserved by the counters or resolved by the
// look-back), every consumer's keys into registers, then -- once all are
// loaded -- back into the same stage in output order, aligned like their
// destinations, and out with bulk stores.  The stage goes back to the
// producer once those stores have read it: thread 0 releases the previous
// tile's stage after committing this one's (`pend`).
template <class C, bool PAY>
__device__ __forceinline__ void emit_tile(const Params *P, uint32_t it, typename C::U *in_k,
                                          uint32_t *in_p, u64 *empty, StageMeta *meta,
                                          const StageCounts *sc, int &pend) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int s = (int)(it % G::STAGES);
  const StageMeta &m = meta[s];
  const uint32_t level = P->ctl->level;
  (void)level;
  if (m.kind != KIND_PARTITION) {
    // verified by the counters: nothing to write.  Every consumer warp must
    // have read this stage's meta before the stage goes back to the
    // producer (which rewrites it for a later tile): a warp that lagged
    // would otherwise take the next tile's kind for this one and leave the
    // consumers' named barriers out of step.  The stage the last partition
    // tile's bulk stores were reading is released here too -- otherwise a
    // run of verification tiles after a partition tile would leave it held
    // until the next partition tile, and the producer, wrapping around the
    // ring onto it, would stall the pipeline for good.
    named_sync(1, kConsumers);
    if (tid == 0) {
      if (pend >= 0) {
        bulk_wait_read0();
        mbar_arrive(&empty[pend]);
        pend = -1;
      }
      mbar_arrive(&empty[s]);
    }
    return;
  }
  const uint32_t t = m.t;
  (void)t;
  if (tid == 0) TSQ_MARK(level, t, 6);
  U *sk = in_k + (size_t)s * G::SLOT;
  uint32_t *sp = PAY ? in_p + (size_t)s * G::SLOT : nullptr;
  U key[G::IPT];
  uint32_t pay[G::IPT];
  load_keys<C, PAY>(sk, sp, tid, key, pay);
  const StageCounts &c = sc[s];
  const u64 xw = c.x[warp], tt = c.tot;
  const uint32_t w_lt = (uint32_t)(xw & 0x1fffffull), w_eq = (uint32_t)((xw >> 21) & 0x1fffffull),
                 w_gt = (uint32_t)(xw >> 42);
  const uint32_t t_lt = (uint32_t)(tt & 0x1fffffull), t_eq = (uint32_t)((tt >> 21) & 0x1fffffull),
                 t_gt = (uint32_t)(tt >> 42);
  const u64 ex = m.excl;
  const int sb = (int)m.buf, db = sb ^ 1;
  const bool src_raw = P->raw[sb] != 0, dst_raw = P->raw[db] != 0;
  const long long begin = m.begin, lo = m.lo;
  const long long ex_lt = (long long)(ex >> 31), ex_gt = (long long)(ex & 0x7fffffffull);
  const long long D_lt = begin + ex_lt;                    // first slot of this tile's < run
  const long long D_gt = m.end - ex_gt - (long long)t_gt;  // first slot of its > run
  TSQ_CHECK(D_lt >= begin && D_lt + (long long)t_lt <= D_gt && D_gt >= begin &&
            D_gt + (long long)t_gt <= m.end && m.end <= P->n);
  // records: the tile's first == payload slot in the side buffer
  const long long D_eq = P->reproducible ? lo - ex_lt - ex_gt : begin + (long long)m.eq_excl;
  const int o_lt = (int)(D_lt & (kAlign - 1));
  const int g_base = (o_lt + (int)t_lt + kAlign - 1) & ~(kAlign - 1);
  const int o_gt = g_base + (int)(D_gt & (kAlign - 1));
  const int e_base = (o_gt + (int)t_gt + kAlign - 1) & ~(kAlign - 1);
  const int o_eq = e_base + (int)(D_eq & (kAlign - 1));
  const U piv = (U)m.pivot;
  const int rlo = (int)(lo - m.tstart), rhi = (int)(m.hi - m.tstart);
  // this thread's first slots: warp offset + the counter's per-lane prefix
  const uint32_t pre = c.t[tid];
  const uint32_t e_lt = pre & 0x3ffu, e_gt = (pre >> 10) & 0x3ffu, e_va = pre >> 20;
  uint32_t plt = (uint32_t)o_lt + w_lt + e_lt;              // next < slot
  uint32_t pgt = (uint32_t)o_gt + t_gt - 1u - w_gt - e_gt;  // next > slot (backwards)
  uint32_t peq = (uint32_t)o_eq + w_eq + (e_va - e_lt - e_gt);
  const bool full = rlo == 0 && rhi == G::TILE;
  // A warp whose lanes all place the same number c of < keys (sorted or
  // blockwise-sorted input: whole tiles on one side of the pivot) would store
  // to slots c apart in every step -- gcd(c, 32)-way bank conflicts, 8-way at
  // c = 24 (measured: such passes ran 0.125 ms against 0.094 at 2^26).  Its
  // 32 c slots are dealt column-wise instead: lane l takes slots l, l + 32,
  // ... of the warp's part of the run (a bijection exactly because the counts
  // are equal; the order of a run's keys is free).  Same for the > side.
  uint32_t st_lt = 1, st_gt = 1;
  if (!PAY && full) {
    const uint32_t lane = (uint32_t)tid & 31u;
    const uint32_t wl = c.w[warp][0], wg = c.w[warp][2];
    const bool ul = __all_sync(0xffffffffu, e_lt == (wl >> 5) * lane) && (wl & 31u) == 0;
    const bool ug = __all_sync(0xffffffffu, e_gt == (wg >> 5) * lane) && (wg & 31u) == 0;
    if (ul) { plt = (uint32_t)o_lt + w_lt + lane; st_lt = 32; }
    if (ug) { pgt = (uint32_t)o_gt + t_gt - 1u - w_gt - lane; st_gt = 32; }
  }
#ifdef TSQ_DEBUG_CHECKS
  if (!PAY && full) {
    // this thread's slots (first, step, count per side) lie inside the runs
    uint32_t nl = 0, ng = 0;
    const bool rr = src_raw && dst_raw && C::kRawOrder;
    const U pq = rr ? C::dec(piv) : piv;
#pragma unroll
    for (int i = 0; i < G::IPT; ++i) {
      const U x = rr ? key[i] : (src_raw ? C::enc(key[i]) : key[i]);
      nl += (rr ? C::rlt(x, pq) : x < pq) ? 1u : 0u;
      ng += (rr ? C::rlt(pq, x) : x > pq) ? 1u : 0u;
    }
    TSQ_CHECK(nl == 0 || (plt >= (uint32_t)o_lt && plt + (nl - 1) * st_lt < (uint32_t)o_lt + t_lt));
    TSQ_CHECK(ng == 0 || (pgt < (uint32_t)o_gt + t_gt && pgt >= (uint32_t)o_gt + (ng - 1) * st_gt));
  }
#endif
  named_sync(1, kConsumers);  // every consumer holds its keys: restage in place
#if defined(TSQ_EXP_COPY) && !defined(TSQ_EXP_STAGE)
  if (full) {  // experiment: pipeline ceiling -- the tile goes out unpartitioned
    fence_proxy_async_smem();
    named_sync(1, kConsumers);
    if (tid == 0) {
      bulk_store(reinterpret_cast<U *>(P->keys[db]) + m.tstart, sk, G::TILE * sizeof(U));
      bulk_commit();
      bulk_wait_read1();
      if (pend >= 0) mbar_arrive(&empty[pend]);
      pend = s;
    }
    return;
  }
#endif
#define TSQ_STAGE stage_keys
  if (src_raw && dst_raw) {
    // raw-order codecs compare in the caller's encoding: the decoded pivot
    const U pv3 = C::kRawOrder ? C::dec(piv) : piv;
    if (full) TSQ_STAGE<C, PAY, true, 3>(key, pay, tid, pv3, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
    else TSQ_STAGE<C, PAY, false, 3>(key, pay, tid, pv3, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
  } else if (src_raw) {
    if (full) TSQ_STAGE<C, PAY, true, 1>(key, pay, tid, piv, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
    else TSQ_STAGE<C, PAY, false, 1>(key, pay, tid, piv, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
  } else if (dst_raw) {
    if (full) TSQ_STAGE<C, PAY, true, 2>(key, pay, tid, piv, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
    else TSQ_STAGE<C, PAY, false, 2>(key, pay, tid, piv, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
  } else {
    if (full) TSQ_STAGE<C, PAY, true, 0>(key, pay, tid, piv, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
    else TSQ_STAGE<C, PAY, false, 0>(key, pay, tid, piv, rlo, rhi, plt, pgt, peq, st_lt, st_gt, sk, sp);
  }
#undef TSQ_STAGE
  fence_proxy_async_smem();
  named_sync(1, kConsumers);
#ifdef TSQ_EXP_STAGE
  if (full) {  // experiment: restaged, then out as one contiguous store
    if (tid == 0) {
      bulk_store(reinterpret_cast<U *>(P->keys[db]) + m.tstart, sk, G::TILE * sizeof(U));
      bulk_commit();
      bulk_wait_read1();
      if (pend >= 0) mbar_arrive(&empty[pend]);
      pend = s;
    }
    return;
  }
#endif
  U *dst = reinterpret_cast<U *>(P->keys[db]);
  const bool issuer = tid == 0;
  emit_run<U>(dst, D_lt, t_lt, sk, issuer, 1);
  emit_run<U>(dst, D_gt, t_gt, sk + g_base, issuer, 2);
  if (PAY) {
    uint32_t *dpay = P->pay[db];
    emit_run<uint32_t>(dpay, D_lt, t_lt, sp, issuer, 3);
    emit_run<uint32_t>(dpay, D_gt, t_gt, sp + g_base, issuer, 4);
    emit_run<uint32_t>(P->side_pay, D_eq, t_eq, sp + e_base, issuer, 5);
  }
  if (issuer) {
    bulk_commit();
    TSQ_MARK(level, t, 7);
    // the previous tile's stores have read their stage: hand it back
    bulk_wait_read1();
    if (pend >= 0) mbar_arrive(&empty[pend]);
    pend = s;
  }
}

template <class C, bool PAY>
__global__ void __launch_bounds__(kPartThreads, 2) partition_kernel(const Params *__restrict__ Pg,
                                                                    Ctl *ctl) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  // every role reads the launch parameters per tile: keep a copy on chip
  // (the global copy misses L1, which the shared-memory carve-out squeezes)
  __shared__ __align__(16) Params sparams;
  static_assert(sizeof(Params) % 8 == 0, "Params copy granularity");
  if (threadIdx.x < sizeof(Params) / 8)
    reinterpret_cast<u64 *>(&sparams)[threadIdx.x] = reinterpret_cast<const u64 *>(Pg)[threadIdx.x];
  const Params *P = &sparams;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  U *in_k = reinterpret_cast<U *>(smem_raw);
  uint32_t *in_p = reinterpret_cast<uint32_t *>(in_k + (size_t)G::STAGES * G::SLOT);
  __shared__ __align__(8) u64 full[G::STAGES], aggr[G::STAGES], ready[G::STAGES], empty[G::STAGES];
  __shared__ StageMeta meta[G::STAGES];
  __shared__ StageCounts sc[G::STAGES];
  __shared__ CounterShare cshare[G::STAGES];

  // (ctl by value: its read runs beside the copy of the parameter block,
  // which is complete after the barrier below)
#ifdef TSQ_EXP_CTL_FROM_PARAMS
  ctl = Pg->ctl;
#endif
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u);
  const uint32_t ntiles = ctl->cur_ntiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::STAGES; ++s) cshare[s].finished = 0;
    for (int s = 0; s < G::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&aggr[s], 1);
      mbar_init(&ready[s], 1);
      mbar_init(&empty[s], 1 + kCounterWarps);  // consumers (thread 0) + counters
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp == kProducerWarp) {
    producer_loop<C, PAY>(P, cur, ntiles, in_k, in_p, full, aggr, empty, meta);
    return;
  }
  if (warp >= kCounterWarp) {
    counter_loop<C, PAY>(P, cur, in_k, full, aggr, empty, meta, sc, cshare,
                         warp - kCounterWarp);
    return;
  }
  if (warp >= kLookbackWarp) {
    lookback_loop<PAY, G::STAGES>(P, cur, aggr, ready, meta, warp - kLookbackWarp);
    return;
  }
  int pend = -1;  // (thread 0) the stage the last bulk stores may still be reading
  for (uint32_t k = 0;; ++k) {
    const int s = (int)(k % G::STAGES);
    wait_ready_consumer(&ready[s], (k / G::STAGES) & 1u);
    if (meta[s].kind == KIND_DONE) break;
    emit_tile<C, PAY>(P, k, in_k, in_p, empty, meta, sc, pend);
  }
  if (threadIdx.x == 0) {
    bulk_wait0();
    if (pend >= 0) mbar_arrive(&empty[pend]);
  }
}

}  // namespace tsq
