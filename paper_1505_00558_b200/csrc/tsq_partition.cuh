// tsq_partition.cuh -- the multi-block three-way partition pass (one
// recursion level over every live segment).  Included by tsq_kernels.cuh.
//
// The stage it performs is the one _run_machine performs for one segment
// (/root/reference/pkg/src/tsqsort/core.py:198-984): afterwards every key
// < p sits at the segment front, every key > p at the back, and the == p
// block (retired, never compared again) in between (core.py:944-967).
//
// Persistent CTAs (2 per SM), warp-specialised (480 threads):
//   warp 8       producer: deals tiles round-robin, resolves their segments
//                32 at a time, streams each into a 4- or 6-deep shared-memory ring (Geo)
//                with cp.async.bulk (TMA engine) completing on the stage's
//                mbarrier; a DONE marker ends the ring
//   warps 11-14  counters (tsq_consume.cuh): per consumer thread the (<, >)
//                counts of its keys and their lane prefixes; tile aggregate
//   warps 9-10   look-back: the tile's output offsets in its segment -- one
//                atomic range reservation, or (reproducible mode) decoupled
//                look-back over the segment's earlier tiles
//   warps 0-7    consumers (tsq_consume.cuh): restage the tile in place in
//                output order and write the < and > runs with cp.async.bulk
#pragma once

namespace tsq {

// ---------------------------------------------------------------------------
// Producer warp.

// The fields of a tile's segment the producer needs, resolved for a batch
// of 32 upcoming tiles at a time (one per lane) so their dependent global
// loads overlap instead of serialising the producer tile by tile.
struct TileSeg {
  long long begin, end;
  u64 pivot;
  uint32_t sid, tile_base, kind, buf, fail;
};

__device__ __forceinline__ TileSeg resolve_tile(const Params *P, int cur, uint32_t t,
                                                uint32_t ntiles) {
  TileSeg r;
  r.begin = r.end = 0; r.pivot = 0; r.sid = r.tile_base = r.kind = r.buf = r.fail = 0;
  if (t < ntiles) {
    r.sid = P->tilemap[cur][t];
    const Seg *sg = &P->segs[cur][r.sid];
    r.begin = sg->begin; r.end = sg->end; r.pivot = sg->pivot;
    r.tile_base = sg->tile_base; r.kind = sg->kind; r.buf = sg->buf;
    // a verification that already failed elsewhere needs no more data (a
    // hint: a stale 0 only costs the load)
    r.fail = r.kind != KIND_PARTITION ? ld_volatile32(&sg->fail) : 0u;
  }
  return r;
}

template <typename T>
__device__ __forceinline__ T bcast(T v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// Tiles are claimed in "guided" chunks from the level's ticket: while many
// remain a CTA takes up to 32 consecutive tiles at a time (their segments
// resolved one lane each, so the dependent loads overlap), near the end
// single tiles -- the pass ends within a tile or two on every CTA instead of
// the ~12 us spread of a static round-robin deal.  Claims go out in
// increasing tile order, so a look-back (reproducible mode) only ever waits
// on tiles already claimed; the next chunk is claimed before the current one
// runs out, so the claim's round trip stays off the producer's path.
__device__ __forceinline__ uint32_t guided_chunk(uint32_t claimed, uint32_t ntiles, uint32_t grid,
                                                 bool single) {
  // reproducible mode: one tile per claim -- a chunk's first tile would wait
  // in its look-back for the whole chunk of the CTA before it (measured:
  // 11.7 ms instead of 0.12 ms per level at 2^26 with 32-tile chunks)
  if (single) return 1u;
  const uint32_t left = claimed < ntiles ? ntiles - claimed : 0u;
  uint32_t c = left / (4u * grid);
  return c < 1u ? 1u : (c > 32u ? 32u : c);
}

template <class C, bool PAY>
__device__ __forceinline__ void producer_loop(const Params *P, int cur, uint32_t ntiles,
                                              typename C::U *in_k, uint32_t *in_p, u64 *full,
                                              u64 *aggr, u64 *empty, StageMeta *meta) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int lane = threadIdx.x & 31;
  const uint32_t level = P->ctl->level;
  (void)level;
  uint32_t *ticket = &P->ctl->tile_ticket;
  const uint32_t grid = gridDim.x;
  TileSeg mine;  // lane j: the tile c0 + j of the current chunk
  // current chunk [c0, c0 + cn) at position ci; the next one, claimed ahead.
  // Tile b of the level is CTA b's without a claim (the ticket counts from
  // tile G), so a level of <= G tiles takes no atomic at all.
  uint32_t c0 = 0, cn = 0, ci = 0, n0 = blockIdx.x, nn = 1;
  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % G::STAGES);
    const uint32_t j = it / G::STAGES;
    if (ci == cn) {
      // move to the claimed chunk; claim the one after it right away
      c0 = __shfl_sync(0xffffffffu, n0, 0);
      cn = __shfl_sync(0xffffffffu, nn, 0);
      ci = 0;
      if (lane == 0 && c0 < ntiles && grid < ntiles) {
        nn = guided_chunk(c0 + cn > grid ? c0 + cn : grid, ntiles, grid, P->reproducible != 0);
        n0 = grid + atomicAdd(ticket, nn);
      } else if (lane == 0) {
        n0 = ntiles;  // nothing left to claim
      }
      const uint32_t tl = c0 + (uint32_t)lane;
      mine = resolve_tile(P, cur, (lane < (int)cn && tl < ntiles) ? tl : ntiles, ntiles);
    }
    const u64 t64 = (u64)c0 + ci;
    const int src_lane = (int)ci;
    ++ci;
    if (j > 0) wait_empty_producer(&empty[s], (j - 1) & 1u);
    if (t64 >= ntiles) {
      // out of tiles: a DONE marker in the next stage stops every role.  The
      // look-back warps take alternate stages, so each gets a marker of its
      // own (the later ones straight on `aggr`).
      const int markers = kLookbackWarps;
      for (int e = 0; e < markers; ++e) {
        const uint32_t ie = it + (uint32_t)e;
        const int se = (int)(ie % G::STAGES);
        if (e > 0 && ie >= (uint32_t)G::STAGES)
          wait_empty_producer(&empty[se], (ie / G::STAGES - 1) & 1u);
        if (lane == 0) {
          meta[se].kind = KIND_DONE;
          meta[se].k = (uint32_t)e;
          mbar_arrive(e == 0 ? &full[se] : &aggr[se]);
        }
      }
      return;
    }
    const uint32_t t = (uint32_t)t64;
    const long long begin = bcast(mine.begin, src_lane), end = bcast(mine.end, src_lane);
    const u64 pivot = bcast(mine.pivot, src_lane);
    const uint32_t sid = bcast(mine.sid, src_lane), tile_base = bcast(mine.tile_base, src_lane);
    const uint32_t kind = bcast(mine.kind, src_lane), buf = bcast(mine.buf, src_lane);
    const uint32_t skip = bcast(mine.fail, src_lane) != 0 ? 1u : 0u;
    StageMeta &m = meta[s];
    TSQ_MARK(level, t, 0);
    const uint32_t k = t - tile_base;
    // tiles on a grid anchored at the segment's (bulk-copy aligned) start:
    // a segment of L keys takes ceil(L / TILE) tiles (+1 only when its
    // alignment slack crosses a boundary), not the extra partial tile an
    // absolute grid costs it (-1.2 % per sort at 2^26, measured)
    const long long tstart = (begin & ~(long long)(kAlign - 1)) + (long long)k * G::TILE;
    const long long lo = tstart > begin ? tstart : begin;
    const long long hi = (tstart + G::TILE) < end ? (tstart + G::TILE) : end;
    TSQ_CHECK(lo < hi && hi <= P->n && lo - tstart >= 0 && hi - tstart <= G::TILE);
    const U *src = reinterpret_cast<const U *>(P->keys[buf]);
    const uint32_t *psrc = PAY ? P->pay[buf] : nullptr;
    U *dk = in_k + (size_t)s * G::SLOT;
    uint32_t *dp = PAY ? in_p + (size_t)s * G::SLOT : nullptr;
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
      m.has_next = hi < end ? 1u : 0u;  // verification: the counters read key hi
      TSQ_MARK(level, t, 1);
      if (tx) {
        TSQ_CHECK((reinterpret_cast<uintptr_t>(src + a0) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dk + (a0 - tstart)) & 15) == 0 &&
                  a0 >= tstart - kAlign && a1 - tstart <= G::SLOT);
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

// Look-back warps: take alternate stages once counted and give each tile its
// offsets in its segment -- by decoupled look-back over the segment's earlier
// tiles (reproducible mode), or by reserving its < and > ranges with one
// atomic on the segment's fill word (the first tile's descriptor slot; the
// records' == payload slots on the segment's eq_fill).  Either way the
// counters never wait on a global round trip.
template <bool PAY, int NS>
__device__ __forceinline__ void lookback_loop(const Params *P, int cur, u64 *aggr, u64 *ready,
                                              StageMeta *meta, int lw) {
  const int lane = threadIdx.x & 31;
  u64 *lb = P->lookback[cur];
  const bool reproducible = P->reproducible != 0;
  const uint32_t level = P->ctl->level;
  (void)level;
  for (uint32_t it = (uint32_t)lw;; it += kLookbackWarps) {
    const int s = (int)(it % NS);
    wait_aggr_lookback(&aggr[s], (it / NS) & 1u);
    StageMeta &m = meta[s];
    if (m.kind == KIND_DONE) {
      // the first marker goes on to the consumers; later ones only stop
      // the other look-back warps
      __syncwarp();
      if (lane == 0 && m.k == 0) mbar_arrive(&ready[s]);
      return;
    }
    const uint32_t t = m.t;
    (void)t;
    if (m.kind != KIND_PARTITION) {
      // verified by the counters: nothing to place
    } else if (!reproducible) {
      if (lane == 0) {
        const u64 ex = atomicAdd(
            reinterpret_cast<unsigned long long *>(&P->segs[cur][m.sid].fill), m.agg);
        const uint32_t eqx = PAY ? atomicAdd(&P->segs[cur][m.sid].eq_fill, m.eq_excl) : 0u;
        m.excl = ex;
        m.eq_excl = eqx;
        TSQ_MARK(level, t, 4);
      }
    } else if (m.k > 0) {
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

}  // namespace tsq

#include "tsq_consume.cuh"
