// tsq_partition.cuh -- the multi-block three-way partition pass (one
// recursion level over every live segment).  Included by tsq_kernels.cuh.
//
// The stage it performs is the one _run_machine performs for one segment
// (/root/reference/pkg/src/tsqsort/core.py:198-984): afterwards every key
// < p sits at the segment front, every key > p at the back, and the == p
// block (retired, never compared again) in between (core.py:944-967).
//
// Persistent CTAs, warp-specialised (320 threads):
//   warp 8  producer   claims a tile (one atomic ticket) as soon as a stage of
//                      the 4-deep shared-memory ring is free, resolves its
//                      segment, and streams it in with cp.async.bulk (TMA
//                      engine) completing on the stage's mbarrier
//   warp 9  look-back  for each stage in order: once the consumers published
//                      the tile's (<, >) aggregate, resolves the tile's
//                      exclusive prefix in its segment by decoupled look-back
//                      over the segment's earlier tiles and publishes the
//                      inclusive prefix
//   warps 0-7 consumers  software-pipelined by one tile: classify tile k+1
//                      (every key against the pivot, ranked in its class with
//                      __ballot_sync / __popc) and publish its aggregate,
//                      then stage tile k's < run and > run (and, for records,
//                      its == payloads) in shared memory aligned like their
//                      destinations and write them with cp.async.bulk stores
//                      (scalar stores for the <= 3 unaligned keys at each end)
// The one-tile skew gives every look-back a full tile of consumer work to
// complete in, so the consumers rarely wait for offsets.
#pragma once

namespace tsq {

// ---------------------------------------------------------------------------
// Producer warp.

template <class C, bool PAY>
__device__ __forceinline__ void producer_loop(const Params *P, int cur, uint32_t ntiles,
                                              typename C::U *in_k, uint32_t *in_p, u64 *full,
                                              u64 *empty, StageMeta *meta) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int lane = threadIdx.x & 31;
  Ctl *ctl = P->ctl;
  const uint32_t level = ctl->level;
  (void)level;
  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % kStages);
    const uint32_t j = it / kStages;
    // claim a tile only once a stage is free for it, so claim order tracks
    // processing order across CTAs (the look-back waits on predecessors)
    if (j > 0) wait_empty_producer(&empty[s], (j - 1) & 1u);
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(&ctl->tile_ticket, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    StageMeta &m = meta[s];
    if (t >= ntiles) {
      if (lane == 0) {
        m.t = kDone;
        mbar_arrive(&full[s]);
      }
      return;
    }
    TSQ_MARK(level, t, 0);
    const uint32_t sid = P->tilemap[cur][t];
    const Seg *sgp = &P->segs[cur][sid];
    const long long begin = sgp->begin, end = sgp->end;
    const uint32_t tile_base = sgp->tile_base, kind = sgp->kind, buf = sgp->buf;
    const u64 pivot = sgp->pivot;
    const uint32_t k = t - tile_base;
    const long long tstart = (begin / G::TILE + k) * (long long)G::TILE;
    const long long lo = tstart > begin ? tstart : begin;
    const long long hi = (tstart + G::TILE) < end ? (tstart + G::TILE) : end;
    const U *src = reinterpret_cast<const U *>(P->keys[buf]);
    const uint32_t *psrc = PAY ? P->pay[buf] : nullptr;
    uint32_t skip = 0;
    if (kind != KIND_PARTITION) skip = ld_volatile32(&sgp->fail) != 0 ? 1u : 0u;
    U *dk = in_k + (size_t)s * G::TILE;
    uint32_t *dp = PAY ? in_p + (size_t)s * G::TILE : nullptr;
    uint32_t tx = 0;
    long long a0 = 0, a1 = 0;
    if (!skip) {
      if (P->aligned[buf]) {
        a0 = lo & ~(long long)(kAlign - 1);
        a1 = (hi + kAlign - 1) & ~(long long)(kAlign - 1);
        const long long cap = P->n & ~(long long)(kAlign - 1);  // never read past n
        if (a1 > cap) a1 = cap;
        if (a1 < a0) a1 = a0;
        for (long long i = a1 + lane; i < hi; i += 32) {  // ragged end of the array
          dk[i - tstart] = src[i];
          if (PAY) dp[i - tstart] = psrc[i];
        }
        tx = (uint32_t)((a1 - a0) * (long long)(sizeof(U) + (PAY ? 4 : 0)));
      } else {
        for (long long i = lo + lane; i < hi; i += 32) {
          dk[i - tstart] = src[i];
          if (PAY) dp[i - tstart] = psrc[i];
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      m.tstart = tstart; m.lo = lo; m.hi = hi; m.begin = begin; m.end = end;
      m.pivot = pivot;
      m.t = t; m.k = k; m.kind = kind; m.buf = buf; m.tile_base = tile_base; m.sid = sid;
      m.skip = skip;
      m.has_next = 0;
      if (kind != KIND_PARTITION && !skip && hi < end) {
        U v = src[hi];
        if (P->raw[buf]) v = C::enc(v);
        m.next_key = (u64)v;
        m.has_next = 1;
      }
      TSQ_MARK(level, t, 1);
      if (tx) {
        mbar_arrive_expect_tx(&full[s], tx);
        bulk_load(dk + (a0 - tstart), src + a0, (uint32_t)((a1 - a0) * sizeof(U)), &full[s]);
        if (PAY) bulk_load(dp + (a0 - tstart), psrc + a0, (uint32_t)((a1 - a0) * 4), &full[s]);
      } else {
        mbar_arrive(&full[s]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Look-back warp.

// Decoupled look-back of one tile: the exclusive (<, >) prefix of tile
// `base + 1` over the tiles [stop, base] of its segment.  Each round trip
// reads a window of 32 * kLbPerLane descriptors (lane l holds distances
// l*kLbPerLane .. l*kLbPerLane + kLbPerLane - 1, nearest first), stops at
// the nearest inclusive prefix and only re-reads when a descriptor nearer
// than that one is not yet published; tiles before `stop` count as an
// inclusive zero (segment start).
constexpr int kLbPerLane = 8;

__device__ __forceinline__ u64 lookback_window(u64 *lb, long long base, long long stop) {
  const int lane = threadIdx.x & 31;
  u64 excl = 0;
  for (;;) {
    u64 d[kLbPerLane];
#pragma unroll
    for (int e = 0; e < kLbPerLane; ++e) {
      const long long idx = base - (lane * kLbPerLane + e);
      d[e] = idx >= stop ? ld_volatile(&lb[idx]) : kFlagInc;
    }
    int first_inc = kLbPerLane, first_zero = kLbPerLane;
#pragma unroll
    for (int e = kLbPerLane - 1; e >= 0; --e) {
      const u64 f = d[e] >> 62;
      if (f == 2) first_inc = e;
      if (f == 0) first_zero = e;
    }
    const uint32_t inc_mask = __ballot_sync(0xffffffffu, first_inc < kLbPerLane);
    const int L = inc_mask ? __ffs(inc_mask) - 1 : 32;
    const int e_inc = __shfl_sync(0xffffffffu, first_inc, L & 31);
    // a descriptor nearer than the nearest inclusive one is still unpublished:
    // spin on the nearest such descriptor alone, then re-read the window
    const bool gap = (lane < L && first_zero < kLbPerLane) || (lane == L && first_zero < e_inc);
    const uint32_t gap_mask = __ballot_sync(0xffffffffu, gap);
    if (gap_mask) {
      const int gl = __ffs(gap_mask) - 1;
      if (lane == gl) {
        const u64 *p = &lb[base - (gl * kLbPerLane + first_zero)];
        unsigned ns = 32;
        while ((ld_volatile(p) >> 62) == 0) {
          __nanosleep(ns);
          ns = ns < 256 ? ns * 2 : ns;
        }
      }
      __syncwarp();
      continue;
    }
    u64 sum = 0;
#pragma unroll
    for (int e = 0; e < kLbPerLane; ++e)
      if (lane < L || (lane == L && e <= e_inc)) sum += d[e] & kValMask;
    excl += warp_sum64(sum);
    if (inc_mask) return excl;
    base -= 32 * kLbPerLane;
  }
}

__device__ __forceinline__ void lookback_loop(const Params *P, int cur, u64 *aggr, u64 *ready,
                                              StageMeta *meta, int lw) {
  const int lane = threadIdx.x & 31;
  u64 *lb = P->lookback[cur];
  const uint32_t level = P->ctl->level;
  (void)level;
  // look-back warp lw owns every kLookbackWarps-th tile of this CTA, so a
  // slow walk back delays only its own tiles
  for (uint32_t it = (uint32_t)lw;; it += kLookbackWarps) {
    const int s = (int)(it % kStages);
    wait_aggr_lookback(&aggr[s], (it / kStages) & 1u);
    StageMeta &m = meta[s];
    const uint32_t t = m.t;
    if (t == kDone) return;
    if (m.kind == KIND_PARTITION && m.k > 0) {
      const u64 agg = m.agg;
      const u64 excl = lookback_window(lb, (long long)t - 1, (long long)m.tile_base);
      if (lane == 0) {
        st_volatile(&lb[t], kFlagInc | (excl + agg));
        TSQ_MARK(level, t, 4);
        m.excl = excl;
      }
    } else if (lane == 0) {
      m.excl = 0;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ready[s]);
  }
}

// ---------------------------------------------------------------------------
// Consumers.

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

// What the consumers carry from classifying a tile to emitting it.
template <int IPT>
struct TileState {
  int s;
  uint32_t par;
  uint32_t partition;  // 0 for a verification tile
  uint32_t t_lt, t_gt, t_eq, w_lt, w_gt, w_eq;
  uint32_t cls[IPT];   // class (0 <, 1 ==, 2 >, 3 none) << 16 | rank in class
};

// one verification tile: every adjacent pair inside the tile and the pair
// that crosses into the next tile must be ordered; a violation marks the
// segment failed (its later tiles are skipped by the producer)
template <class C, bool PAY>
__device__ __forceinline__ void verify_tile(const Params *P, int cur, const StageMeta &m,
                                            const typename C::U *sk, uint32_t *s_flag) {
  typedef typename C::U U;
  const int tid = threadIdx.x;
  const bool raw = P->raw[m.buf] != 0;
  const bool asc = m.kind == KIND_VERIFY_ASC;
  const long long rlo = m.lo - m.tstart, rhi = m.hi - m.tstart;
  bool bad = false;
  if (!m.skip) {
    for (long long i = rlo + tid; i < rhi; i += kConsumers) {
      U a = sk[i];
      U b;
      bool have = true;
      if (i + 1 < rhi) b = sk[i + 1];
      else if (m.has_next) b = (U)m.next_key;
      else have = false;
      if (raw) {
        a = C::enc(a);
        if (i + 1 < rhi) b = C::enc(b);
      }
      if (have) bad |= asc ? (a > b) : (a < b);
    }
  }
  if (tid == 0) *s_flag = 0;
  named_sync(1, kConsumers);
  if (bad) *s_flag = 1;
  named_sync(1, kConsumers);
  if (tid == 0 && *s_flag) atomicOr(&P->segs[cur][m.sid].fail, 1u);
}

// Phase A of tile `it`: classify and rank every key, publish the aggregate.
// Returns false at the end-of-level marker.
template <class C, bool PAY>
__device__ __forceinline__ bool classify_tile(const Params *P, int cur, uint32_t it,
                                              const typename C::U *in_k, u64 *full, u64 *aggr,
                                              StageMeta *meta, uint32_t (*wcnt)[3],
                                              uint32_t *s_flag, TileState<Geo<C, PAY>::IPT> &ts) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  ts.s = (int)(it % kStages);
  ts.par = (it / kStages) & 1u;
  wait_full_consumer(&full[ts.s], ts.par);
  const StageMeta &m = meta[ts.s];
  const uint32_t t = m.t;
  // Every path through here ends with a consumer barrier that thread 0
  // (the bulk-store issuer) reaches only after the previous tile's bulk
  // stores finished reading the out buffer, which the next emit restages.
  if (t == kDone) {
    if (tid == 0) {
      // every look-back warp must see an end marker: this stage's and, for
      // the others, the next ones (their last fills were emitted already)
      mbar_arrive(&aggr[ts.s]);
      for (uint32_t e = 1; e < (uint32_t)kLookbackWarps; ++e) {
        const int se = (int)((it + e) % kStages);
        meta[se].t = kDone;
        mbar_arrive(&aggr[se]);
      }
      bulk_wait_read0();
    }
    named_sync(1, kConsumers);
    return false;
  }
  const U *sk = in_k + (size_t)ts.s * G::TILE;
  const uint32_t level = P->ctl->level;
  (void)level;
  if (tid == 0) TSQ_MARK(level, t, 2);
  if (m.kind != KIND_PARTITION) {
    ts.partition = 0;
    if (tid == 0) bulk_wait_read0();
    verify_tile<C, PAY>(P, cur, m, sk, s_flag);
    if (tid == 0) mbar_arrive(&aggr[ts.s]);
    return true;
  }
  ts.partition = 1;
  const bool src_raw = P->raw[m.buf] != 0;
  const U piv = (U)m.pivot;
  const int rlo = (int)(m.lo - m.tstart), rhi = (int)(m.hi - m.tstart);
  const bool full_tile = rlo == 0 && rhi == G::TILE;
#pragma unroll
  for (int v = 0; v < G::VPT; ++v) {
    const int e0 = (v * kConsumers + tid) * G::VN;
    U key[G::VN];
    unpack(*reinterpret_cast<const typename Vec<U>::K *>(sk + e0), key);
#pragma unroll
    for (int q = 0; q < G::VN; ++q) {
      const int idx = e0 + q;
      const U x = src_raw ? C::enc(key[q]) : key[q];
      const uint32_t valid = (full_tile || (idx >= rlo && idx < rhi)) ? 1u : 0u;
      // 0 <, 1 ==, 2 >, 3 outside the segment (branch-free)
      const uint32_t c = ((uint32_t)(x >= piv) + (uint32_t)(x > piv)) | ((valid ^ 1u) * 3u);
      ts.cls[v * G::VN + q] = c;
    }
  }
  // warp-level ranks per class, ordered by (item, lane); masks select the
  // class's ballot and running count without branches
  const uint32_t lmask = (1u << lane) - 1u;
  uint32_t lt_run = 0, gt_run = 0, eq_run = 0;
#pragma unroll
  for (int i = 0; i < G::IPT; ++i) {
    const uint32_t c = ts.cls[i];
    const uint32_t blt = __ballot_sync(0xffffffffu, c == 0);
    const uint32_t bgt = __ballot_sync(0xffffffffu, c == 2);
    const uint32_t beq = PAY ? __ballot_sync(0xffffffffu, c == 1) : 0u;
    const uint32_t mlt = 0u - (uint32_t)(c == 0), mgt = 0u - (uint32_t)(c == 2);
    const uint32_t meq = PAY ? 0u - (uint32_t)(c == 1) : 0u;
    const uint32_t bm = (blt & mlt) | (bgt & mgt) | (beq & meq);
    const uint32_t base = (lt_run & mlt) | (gt_run & mgt) | (eq_run & meq);
    ts.cls[i] = (c << 16) | (base + __popc(bm & lmask));
    lt_run += __popc(blt);
    gt_run += __popc(bgt);
    if (PAY) eq_run += __popc(beq);
  }
  uint32_t(*wc)[3] = wcnt + (it & 1u) * kConsumerWarps;
  if (lane == 0) {
    wc[warp][0] = lt_run;
    wc[warp][1] = eq_run;
    wc[warp][2] = gt_run;
  }
  // the previous tile's bulk stores must have finished reading the out
  // buffer before the tile after this barrier restages it
  if (tid == 0) bulk_wait_read0();
  named_sync(1, kConsumers);
  uint32_t w_lt = 0, w_eq = 0, w_gt = 0, t_lt = 0, t_eq = 0, t_gt = 0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) {
    const uint32_t a = wc[w][0], b = wc[w][1], c = wc[w][2];
    if (w < warp) { w_lt += a; w_eq += b; w_gt += c; }
    t_lt += a; t_eq += b; t_gt += c;
  }
  ts.w_lt = w_lt; ts.w_eq = w_eq; ts.w_gt = w_gt;
  ts.t_lt = t_lt; ts.t_eq = t_eq; ts.t_gt = t_gt;
  if (tid == 0) {
    const u64 agg = ((u64)t_lt << 31) | (u64)t_gt;
    StageMeta &mw = meta[ts.s];
    mw.agg = agg;
    st_volatile(&P->lookback[cur][t], (m.k == 0 ? kFlagInc : kFlagAgg) | agg);
    TSQ_MARK(level, t, 3);
    mbar_arrive(&aggr[ts.s]);
  }
  return true;
}

// Phase B of a tile: wait for its offsets, stage its runs, write them out.
template <class C, bool PAY>
__device__ __forceinline__ void emit_tile(const Params *P, const typename C::U *in_k,
                                          const uint32_t *in_p, u64 *ready, u64 *empty,
                                          StageMeta *meta, typename C::U *ok, uint32_t *op,
                                          const TileState<Geo<C, PAY>::IPT> &ts) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (!ts.partition) {
    // the look-back warp still walks this stage's meta: wait for it (this
    // also keeps the aggr / ready phases of a stage from running ahead)
    wait_ready_consumer(&ready[ts.s], ts.par);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ts.s]);
    return;
  }
  const StageMeta &m = meta[ts.s];
  const uint32_t level = P->ctl->level;
  (void)level;
  if (tid == 0) TSQ_MARK(level, m.t, 5);
  wait_ready_consumer(&ready[ts.s], ts.par);
  if (tid == 0) TSQ_MARK(level, m.t, 6);
  const u64 ex = m.excl;
  const int sb = (int)m.buf, db = sb ^ 1;
  const bool src_raw = P->raw[sb] != 0, dst_raw = P->raw[db] != 0;
  const long long begin = m.begin, end = m.end, lo = m.lo;
  const long long ex_lt = (long long)(ex >> 31), ex_gt = (long long)(ex & 0x7fffffffull);
  const long long D_lt = begin + ex_lt;                      // first slot of this tile's < run
  const long long D_gt = end - ex_gt - (long long)ts.t_gt;   // first slot of its > run
  const long long D_eq = begin + (lo - begin) - ex_lt - ex_gt;  // records: side-buffer slot
  const int o_lt = (int)(D_lt & (kAlign - 1));
  const int g_base = (o_lt + (int)ts.t_lt + kAlign - 1) & ~(kAlign - 1);
  const int o_gt = g_base + (int)(D_gt & (kAlign - 1));
  const int e_base = (o_gt + (int)ts.t_gt + kAlign - 1) & ~(kAlign - 1);
  const int o_eq = e_base + (int)(D_eq & (kAlign - 1));
  const U *sk = in_k + (size_t)ts.s * G::TILE;
  const uint32_t *sp = PAY ? in_p + (size_t)ts.s * G::TILE : nullptr;
  const uint32_t lt0 = (uint32_t)o_lt + ts.w_lt;
  const uint32_t gt0 = (uint32_t)o_gt + ts.t_gt - 1u - ts.w_gt;
  const uint32_t eq0 = (uint32_t)o_eq + ts.w_eq;
#pragma unroll
  for (int v = 0; v < G::VPT; ++v) {
    const int e0 = (v * kConsumers + tid) * G::VN;
    U key[G::VN];
    uint32_t pay[G::VN];
    unpack(*reinterpret_cast<const typename Vec<U>::K *>(sk + e0), key);
    if (PAY) unpack(*reinterpret_cast<const typename Vec<U>::P *>(sp + e0), pay);
#pragma unroll
    for (int q = 0; q < G::VN; ++q) {
      // branch-free: select the slot, predicate the stores
      const uint32_t cr = ts.cls[v * G::VN + q];
      const uint32_t c = cr >> 16, rk = cr & 0xffffu;
      const uint32_t p_lt = lt0 + rk;
      const uint32_t p_gt = gt0 - rk;  // > run fills backwards
      uint32_t pos = c == 0u ? p_lt : p_gt;
      if (PAY) pos = c == 1u ? eq0 + rk : pos;
      U x = key[q];
      if (src_raw != dst_raw) x = src_raw ? C::enc(x) : C::dec(x);
      if ((c & 1u) == 0u) ok[pos] = x;   // c == 0 or c == 2
      if (PAY && c != 3u) op[pos] = pay[q];
    }
  }
  const uint32_t t = m.t;
  (void)t;
  // the stage is no longer needed: hand it back to the producer
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[ts.s]);
  fence_proxy_async_smem();
  named_sync(1, kConsumers);
  U *dst = reinterpret_cast<U *>(P->keys[db]);
  const bool issuer = tid == 0;
  emit_run<U>(dst, D_lt, ts.t_lt, ok, issuer, 1);
  emit_run<U>(dst, D_gt, ts.t_gt, ok + g_base, issuer, 2);
  if (PAY) {
    uint32_t *dpay = P->pay[db];
    emit_run<uint32_t>(dpay, D_lt, ts.t_lt, op, issuer, 3);
    emit_run<uint32_t>(dpay, D_gt, ts.t_gt, op + g_base, issuer, 4);
    emit_run<uint32_t>(P->side_pay, D_eq, ts.t_eq, op + e_base, issuer, 5);
  }
  if (issuer) {
    bulk_commit();
    TSQ_MARK(level, t, 7);
  }
}

template <class C, bool PAY>
__global__ void __launch_bounds__(kPartThreads, 2) partition_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  U *in_k = reinterpret_cast<U *>(smem_raw);
  uint32_t *in_p = reinterpret_cast<uint32_t *>(in_k + (size_t)kStages * G::TILE);
  U *out_k = reinterpret_cast<U *>(smem_raw + (size_t)kStages * G::STAGE_BYTES);
  uint32_t *out_p = reinterpret_cast<uint32_t *>(smem_raw + (size_t)kStages * G::STAGE_BYTES +
                                                 G::OUT_K);
  __shared__ __align__(8) u64 full[kStages], aggr[kStages], ready[kStages], empty[kStages];
  __shared__ StageMeta meta[kStages];
  __shared__ uint32_t wcnt[2 * kConsumerWarps][3];
  __shared__ uint32_t s_flag;

  Ctl *ctl = P->ctl;
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u);
  const uint32_t ntiles = ctl->cur_ntiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&aggr[s], 1);
      mbar_init(&ready[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp == kProducerWarp) {
    producer_loop<C, PAY>(P, cur, ntiles, in_k, in_p, full, empty, meta);
    return;
  }
  if (warp >= kLookbackWarp) {
    lookback_loop(P, cur, aggr, ready, meta, warp - kLookbackWarp);
    return;
  }
  TileState<G::IPT> a, b;
  bool more = classify_tile<C, PAY>(P, cur, 0, in_k, full, aggr, meta, wcnt, &s_flag, a);
  for (uint32_t it = 1; more; ++it) {
    // classify the next tile before emitting this one: its aggregate is
    // published while this tile's look-back completes
    const bool next = classify_tile<C, PAY>(P, cur, it, in_k, full, aggr, meta, wcnt, &s_flag, b);
    emit_tile<C, PAY>(P, in_k, in_p, ready, empty, meta, out_k, out_p, a);
    if (!next) break;
    a = b;
  }
  if (threadIdx.x == 0) bulk_wait0();
}

}  // namespace tsq
