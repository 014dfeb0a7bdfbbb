// tsq_schedule.cuh -- the per-segment bookkeeping between two partition
// passes (the tail of one Sorter._range stage and the head of the next,
// /root/reference/pkg/src/tsqsort/core.py:1705-1728).  Included by
// tsq_kernels.cuh.
//
// For every segment of the level just partitioned: retire the == p block
// (never compared again), then queue each child -- the < part and the > part
// -- either for the on-chip sort (<= small_t keys) or for the next level
// with its pivot sampled now (select_pivot's role, pivot.py:205-248).
//   few, large segments   one CTA per (segment, child), 1023-key samples sorted by a
//                         register bitonic network across the CTA
//   many, small segments  one warp per (segment, child), <= 127-key samples
//                         sorted in the warp's registers; the queue slots of all of a
//                         CTA's segments are claimed with one atomic per
//                         queue per round (the queues are single hot words)
#pragma once

namespace tsq {

// phase stamps of CTA 0 / warp 0 (profiling builds only: -DTSQ_SCHED_CLOCK;
// printed at kernel end for level TSQ_SCHED_CLOCK)
#ifdef TSQ_SCHED_CLOCK
#include <cstdio>
__device__ unsigned long long g_sc[16];
#define TSQ_SC(i)                                                         \
  do {                                                                    \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                            \
      unsigned long long t_;                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
      g_sc[i] = t_;                                                       \
    }                                                                     \
  } while (0)
#else
#define TSQ_SC(i) ((void)0)
#endif

// per-CTA statistics: one slice per warp, written by that warp's leader lane
// alone (plain updates: 64-bit shared-memory atomics are compare-and-swap
// loops, ~0.7 us of the segment head), summed into one global flush per CTA
enum SchedStat {
  ST_STAGES, ST_SORTED, ST_REVERSED, ST_DEPTH, ST_BYTES_PART, ST_BYTES_RETIRE, ST_W0, ST_W1,
  ST_FALLBACK, ST_PARTITIONED, ST_EQ_RUNS, ST_EQ_ELEMS, ST_BISECTED, ST_COUNT
};

// Key bounds of a segment's children (encoded keys): < child [klo, p - 1],
// > child [p + 1, khi].  An empty side never gets scheduled, so the clamps
// only keep the arithmetic in range.
__device__ __forceinline__ void child_bounds(const Seg &sg, int c, u64 *lo, u64 *hi) {
  if (c == 0) {
    *lo = sg.klo;
    *hi = sg.pivot > sg.klo ? sg.pivot - 1 : sg.klo;
  } else {
    *lo = sg.pivot < sg.khi ? sg.pivot + 1 : sg.khi;
    *hi = sg.khi;
  }
}

// Beyond the depth guard: split at the midpoint of the key bound.  Every
// such level halves the bound, so a segment ends within key-bits levels
// (all keys equal once klo == khi: one == p run).
__device__ __forceinline__ u64 bisect_pivot(u64 lo, u64 hi) { return lo + ((hi - lo) >> 1); }

#ifndef TSQ_WARP_SAMPLES
#define TSQ_WARP_SAMPLES 127
#endif
#ifndef TSQ_CTA_SCHED_MIN
#define TSQ_CTA_SCHED_MIN (1ll << 20)
#endif
constexpr int kWarpSampleMax = TSQ_WARP_SAMPLES;  // warp-mode sample cap (4 per lane)
// Segments of at least this many keys (on average) are scheduled by a whole
// CTA per child; below it one warp per child.
constexpr long long kCtaScheduleMin = TSQ_CTA_SCHED_MIN;

__device__ __forceinline__ void append_small(const Params *P, long long begin, long long len,
                                             uint32_t buf) {
  Ctl *ctl = P->ctl;
  const int c = small_class(P, len);
  TSQ_CHECK(len > 0 && len <= P->sq_lim[c] && begin >= 0 && begin + len <= P->n);
  const uint32_t slot = atomicAdd(&ctl->sq_count[c], 1u);
  if (slot < P->sq_cap[c]) {
    SmallSeg s;
    s.begin = begin; s.len = (int)len; s.buf = (int)buf;
    P->sq[c][slot] = s;
  } else {
    atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
  }
}

template <class C, bool PAY>
__device__ __forceinline__ uint32_t tiles_of(long long begin, long long end) {
  const long long T = Geo<C, PAY>::TILE;
  // segment-anchored tile grid (producer_loop, tsq_partition.cuh)
  return (uint32_t)(((end - 1) - (begin & ~(long long)(kAlign - 1))) / T + 1);
}

__device__ __forceinline__ uint32_t chunks_of(uint32_t kind, long long len, uint32_t buf) {
  if (kind == RUN_REVERSED && buf == 0) return (uint32_t)(((len >> 1) + kRunChunk - 1) / kRunChunk);
  return (uint32_t)((len + kRunChunk - 1) / kRunChunk);
}

// ---- sample sorting networks (all-ascending bitonic, as in tsq_small.cuh) --

// warp: 32 * Q keys, lane l holds l*Q .. l*Q+Q-1
template <typename U, int Q>
__device__ __forceinline__ void warp_bitonic(U (&v)[Q]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * Q; k <<= 1) {
    if (k <= Q) {
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        const int p = r ^ (k - 1);
        if (r < p) { const U a = v[r], b = v[p]; v[r] = a < b ? a : b; v[p] = a < b ? b : a; }
      }
    } else {
      const int m = k / Q - 1;
      const bool lower = (lane & (k / (2 * Q))) == 0;
      U y[Q];
#pragma unroll
      for (int r = 0; r < Q; ++r) y[r] = __shfl_xor_sync(0xffffffffu, v[Q - 1 - r], m);
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        const U mn = v[r] < y[r] ? v[r] : y[r], mx = v[r] < y[r] ? y[r] : v[r];
        v[r] = lower ? mn : mx;
      }
    }
#pragma unroll
    for (int j = k >> 2; j >= 1; j >>= 1) {
      if (j >= Q) {
        const int m = j / Q;
        const bool lower = (lane & m) == 0;
#pragma unroll
        for (int r = 0; r < Q; ++r) {
          const U y = __shfl_xor_sync(0xffffffffu, v[r], m);
          const U mn = v[r] < y ? v[r] : y, mx = v[r] < y ? y : v[r];
          v[r] = lower ? mn : mx;
        }
      } else {
#pragma unroll
        for (int r = 0; r < Q; ++r)
          if (!(r & j)) { const U a = v[r], b = v[r | j]; v[r] = a < b ? a : b; v[r | j] = a < b ? b : a; }
      }
    }
  }
}

// Load the S strided samples of [begin, begin+len) in position order into
// v (blocked, padded with +max to `slots` entries).  The first, middle and
// last positions are fixed anchors; interior positions shift by the
// MitigationRng jitter (dran, pivot.py:223-237).
template <class C, int Q>
__device__ __forceinline__ void load_samples(const typename C::U *data, bool encoded_src,
                                             long long begin, long long len, int S, double dran,
                                             int mitigation, int owner, typename C::U (&v)[Q]) {
  typedef typename C::U U;
  const int midi = S >> 1;
  const long long span = len - 1;
  long long shift = 0;
  const double step = (double)span / (double)(S - 1);
  if (mitigation) shift = (long long)floor((dran - 1.0) * step * 0.5);
  // positions first (clamped into the segment so every load is valid), then
  // all Q loads back to back so their latencies overlap
  const U *ptr[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = min(owner * Q + q, S - 1);
    long long pos = (i == S - 1) ? begin + span : begin + (long long)((double)i * step);
    if (i != 0 && i != midi && i != S - 1) {
      pos += shift;
      pos = pos < begin ? begin : (pos > begin + span ? begin + span : pos);
    }
    ptr[q] = data + pos;
  }
  U x[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) x[q] = ldcg(ptr[q]);
#pragma unroll
  for (int q = 0; q < Q; ++q)
    v[q] = owner * Q + q < S ? (encoded_src ? x[q] : C::enc(x[q])) : KeyMax<U>::v;
}

// order flag of the samples in position order (+1 nondecreasing, -1
// nonincreasing, 0) for a warp holding them blocked
template <typename U, int Q>
__device__ __forceinline__ int warp_order_flag(const U (&v)[Q], int S) {
  const int lane = threadIdx.x & 31;
  bool asc = true, desc = true;
#pragma unroll
  for (int q = 0; q + 1 < Q; ++q) {
    if (lane * Q + q + 1 < S) {
      asc &= v[q] <= v[q + 1];
      desc &= v[q] >= v[q + 1];
    }
  }
  const U nxt = __shfl_down_sync(0xffffffffu, v[0], 1);
  if (lane < 31 && (lane + 1) * Q < S) {
    asc &= v[Q - 1] <= nxt;
    desc &= v[Q - 1] >= nxt;
  }
  asc = __all_sync(0xffffffffu, asc);
  desc = __all_sync(0xffffffffu, desc);
  return asc ? 1 : (desc ? -1 : 0);
}

template <typename U, int Q>
__device__ __forceinline__ U warp_pick(const U (&v)[Q], int idx) {
  U x = v[0];
#pragma unroll
  for (int q = 1; q < Q; ++q)
    if ((idx % Q) == q) x = v[q];
  return __shfl_sync(0xffffffffu, x, idx / Q);
}

// warp pivot sampling: S <= kWarpSampleMax
template <class C, int Q>
__device__ __forceinline__ typename C::U warp_pivot_q(const typename C::U *data, bool enc_src,
                                                      long long begin, long long len, int S,
                                                      double dran, int mitigation, int *flag) {
  typedef typename C::U U;
  // reconverge first: after lane-0-only bookkeeping the warp may still run
  // split, and the network's shuffles would take the divergent slow path
  __syncwarp();
  U v[Q];
  load_samples<C, Q>(data, enc_src, begin, len, S, dran, mitigation, threadIdx.x & 31, v);
  *flag = warp_order_flag<U, Q>(v, S);
  warp_bitonic<U, Q>(v);
  return warp_pick<U, Q>(v, S >> 1);
}

template <class C>
__device__ typename C::U warp_select_pivot(const typename C::U *data, bool enc_src,
                                           long long begin, long long len, double dran,
                                           int mitigation, int *flag) {
  int S = sample_count(len);
  if (S > kWarpSampleMax) S = kWarpSampleMax;
  if (S <= 32) return warp_pivot_q<C, 1>(data, enc_src, begin, len, S, dran, mitigation, flag);
  if (S <= 64) return warp_pivot_q<C, 2>(data, enc_src, begin, len, S, dran, mitigation, flag);
  if (S <= 128) return warp_pivot_q<C, 4>(data, enc_src, begin, len, S, dran, mitigation, flag);
  return warp_pivot_q<C, 8>(data, enc_src, begin, len, S, dran, mitigation, flag);
}

// CTA pivot sampling: S <= 1023 samples, 4 per thread, register bitonic with
// shuffle and shared-memory stages (block_bitonic from tsq_small.cuh)
template <class C>
__device__ typename C::U cta_select_pivot_fast(const typename C::U *data, bool enc_src,
                                               long long begin, long long len, double dran,
                                               int mitigation, typename C::U *xk,
                                               volatile uint32_t *bc, int *flag) {
  typedef typename C::U U;
  constexpr int Q = 4;  // 256 * 4 = 1024 slots
  const int S = sample_count(len);
  const int tid = threadIdx.x;
  U raw[Q];
  load_samples<C, Q>(data, enc_src, begin, len, S, dran, mitigation, tid, raw);
  // order flag over position order
  bool asc = true, desc = true;
#pragma unroll
  for (int q = 0; q + 1 < Q; ++q)
    if (tid * Q + q + 1 < S) {
      asc &= raw[q] <= raw[q + 1];
      desc &= raw[q] >= raw[q + 1];
    }
  xk[tid] = raw[0];
  __syncthreads();
  if (tid < kThreads - 1 && (tid + 1) * Q < S) {
    asc &= raw[Q - 1] <= xk[tid + 1];
    desc &= raw[Q - 1] >= xk[tid + 1];
  }
  asc = __syncthreads_and(asc);
  desc = __syncthreads_and(desc);
  *flag = asc ? 1 : (desc ? -1 : 0);
  SortItem<U, false> v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) v[q].k = raw[q];
  block_bitonic<U, false, Q>(v, xk, nullptr);
  const int midi = S >> 1;
  __syncthreads();
  if (tid == midi / Q) {
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (q == midi % Q) xk[0] = v[q].k;
  }
  __syncthreads();
  const U piv = xk[0];
  __syncthreads();
  (void)bc;
  return piv;
}

// ---------------------------------------------------------------------------
// Segment head: statistics, verification outcome, == p retirement.  Returns
// the child layout in *lt / *gt, or false when the segment produced no
// children to schedule (verified run, failed verification re-queued, single
// stage).  Executed by a whole group; queue appends here are rare (runs).

template <class C, bool PAY, bool CTA>
__device__ bool segment_head(const Params *P, int nxt, const Seg &sg, int cur, u64 *st,
                             long long *lt_out, long long *gt_out, uint32_t *requeue,
                             bool bookkeep = true) {
  typedef typename C::U U;
  const int r = CTA ? (int)threadIdx.x : (int)(threadIdx.x & 31);
  const int gsize = CTA ? kThreads : 32;
  const bool leader = r == 0;
  Ctl *ctl = P->ctl;
  const long long len = sg.end - sg.begin;
  const int kb = (int)sizeof(U);
  *requeue = 0;
  if (sg.kind != KIND_PARTITION) {
    if (!bookkeep) return false;
    if (sg.fail == 0) {
      const uint32_t rk = sg.kind == KIND_VERIFY_ASC ? RUN_SORTED : RUN_REVERSED;
      if (leader) {
        st[ST_STAGES] += 1ull;
        st[rk == RUN_SORTED ? ST_SORTED : ST_REVERSED] += 1ull;
        st[ST_DEPTH] = st[ST_DEPTH] > (u64)sg.depth ? st[ST_DEPTH] : (u64)sg.depth;
        st[ST_BYTES_PART] += (u64)len * kb;  // the verify read
        if (!(rk == RUN_SORTED && sg.buf == 0)) {
          st[ST_BYTES_RETIRE] += 2ull * (u64)len * (u64)(kb + (PAY ? 4 : 0));
          st[ST_W0] += (u64)len;
        }
      }
    } else {
      if (leader) st[ST_FALLBACK] += 1ull;
      *requeue = 1;
    }
    return false;
  }
  // the segment's (<, >) totals: the last tile's inclusive descriptor, or
  // the record's fill word all its tiles reserved from
  const u64 inc = P->reproducible ? P->lookback[cur][sg.tile_base + sg.ntiles - 1] : sg.fill;
  const long long lt = (long long)((inc >> 31) & 0x7fffffffull);
  const long long gt = (long long)(inc & 0x7fffffffull);
  const long long eq = len - lt - gt;
  *lt_out = lt;
  *gt_out = gt;
  if (!bookkeep) return !P->single_stage;
  if (leader) {
    st[ST_STAGES] += 1ull;
    st[ST_PARTITIONED] += (u64)len;
    st[ST_DEPTH] = st[ST_DEPTH] > (u64)sg.depth ? st[ST_DEPTH] : (u64)sg.depth;
    u64 bytes = (u64)len * kb + (u64)(lt + gt) * kb;
    if (PAY) bytes += (u64)len * 8ull;
    st[ST_BYTES_PART] += bytes;
    st[sg.buf == 0 ? ST_W1 : ST_W0] += (u64)(lt + gt);
    if (PAY) st[ST_W1] += (u64)eq;
    if (eq > 0) {
      st[ST_EQ_RUNS] += 1ull;
      st[ST_EQ_ELEMS] += (u64)eq;
      st[ST_BYTES_RETIRE] += (u64)eq * (kb + (PAY ? 8 : 0));
      st[ST_W0] += (u64)eq;
    }
    if (P->single_stage) {
      ctl->stage_lt = (u64)lt;
      ctl->stage_gt = (u64)gt;
    }
  }
  if (eq > 0 && PAY) {
    // Records: the == p payloads sit at side_pay[begin ...], a range the
    // children reuse at the next level, so they move to their final place
    // now (nothing else touches [begin+lt, end-gt) of buffer 0).
    const uint32_t *side = P->side_pay + sg.begin;
    uint32_t *p0 = P->pay[0] + sg.begin + lt;
    U *k0 = reinterpret_cast<U *>(P->keys[0]) + sg.begin + lt;
    const U v = P->raw[0] ? C::dec((U)sg.pivot) : (U)sg.pivot;
    for (long long i = r; i < eq; i += gsize) {
      p0[i] = side[i];
      k0[i] = v;
    }
  }
  *lt_out = lt;
  *gt_out = gt;
  return !P->single_stage;
}

// ---------------------------------------------------------------------------
// Appends aggregated over one round of the CTA's warps.

struct ReqLevel {  // a child queued for the next level
  long long begin, end;
  u64 pivot, klo, khi;
  uint32_t buf, kind, depth, noverify, ntiles, valid;
};
struct ReqRun {
  long long begin, len, src;
  u64 pivot;
  uint32_t kind, buf, nchunks, valid;
};
struct ReqSmall {
  long long begin, len;
  uint32_t buf, valid;
};

struct RoundShared {
  ReqLevel lv[kThreads / 32][2];
  ReqRun run[kThreads / 32];
  ReqSmall sm[kThreads / 32][2];
  uint32_t lv_slot0, lv_tile0, run_slot0, run_chunk0, sq_slot0[kSmallClasses];
};

// Warp mode: one task per warp, task = (segment, child); the child-0 warp
// also does the segment's bookkeeping (statistics, == p run, verified runs,
// re-queued verifications), so the two pivot samplings of a segment run on
// two warps side by side.
template <class C, bool PAY>
__device__ void schedule_round_warp(const Params *P, int cur, int nxt, uint32_t task, bool have,
                                    u64 *st, RoundShared &rs) {
  typedef typename C::U U;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarpQ = (kWarpSampleMax + 32) / 32;   // samples per lane (4 for 127)
  U sv[kWarpQ];
  int S = 0;   // > 0: this warp's child awaits its pivot (samples in sv)
  if (lane == 0) {
    rs.lv[warp][0].valid = rs.lv[warp][1].valid = 0;
    rs.sm[warp][0].valid = rs.sm[warp][1].valid = 0;
    rs.run[warp].valid = 0;
  }
  __syncwarp();
  if (have) {
    const uint32_t sid = task >> 1;
    const int c = (int)(task & 1u);
    const Seg sg = P->segs[cur][sid];
#ifdef TSQ_SCHED_CLOCK
    if (sg.end < 0) return;  // (never: keeps the stamp behind the load)
#endif
    TSQ_SC(2);
    long long lt = 0, gt = 0;
    uint32_t requeue = 0;
    const bool kids =
        segment_head<C, PAY, false>(P, nxt, sg, cur, st, &lt, &gt, &requeue, c == 0);
    TSQ_SC(3);
    const long long len = sg.end - sg.begin;
    if (lane == 0 && c == 0) {
      if (sg.kind != KIND_PARTITION) {
        if (requeue) {
          ReqLevel &q = rs.lv[warp][0];
          q.begin = sg.begin; q.end = sg.end; q.pivot = sg.pivot; q.buf = sg.buf;
          q.klo = sg.klo; q.khi = sg.khi;
          q.kind = KIND_PARTITION; q.depth = sg.depth; q.noverify = 1;
          q.ntiles = tiles_of<C, PAY>(sg.begin, sg.end); q.valid = 1;
        } else if (sg.fail == 0) {
          const uint32_t rk = sg.kind == KIND_VERIFY_ASC ? RUN_SORTED : RUN_REVERSED;
          if (!(rk == RUN_SORTED && sg.buf == 0)) {
            ReqRun &q = rs.run[warp];
            q.begin = sg.begin; q.len = len; q.src = sg.begin; q.pivot = 0; q.kind = rk;
            q.buf = sg.buf; q.nchunks = chunks_of(rk, len, sg.buf); q.valid = 1;
          }
        }
      } else {
        const long long eq = len - lt - gt;
        if (eq > 0 && !PAY) {
          ReqRun &q = rs.run[warp];
          q.begin = sg.begin + lt; q.len = eq; q.src = sg.begin; q.pivot = sg.pivot;
          q.kind = RUN_EQ; q.buf = sg.buf; q.nchunks = chunks_of(RUN_EQ, eq, sg.buf); q.valid = 1;
        }
      }
    }
    const long long cb = c == 0 ? sg.begin : sg.end - gt;
    TSQ_CHECK(lt >= 0 && gt >= 0 && lt + gt <= sg.end - sg.begin);
    const long long cl = c == 0 ? lt : gt;
    if (kids && cl > 0) {
      const uint32_t db = sg.buf ^ 1u;
      const uint32_t depth = sg.depth + 1;
      if (cl <= P->small_t) {
        if (lane == 0) {
          ReqSmall &q = rs.sm[warp][0];
          q.begin = cb; q.len = cl; q.buf = db; q.valid = 1;
          st[ST_DEPTH] = st[ST_DEPTH] > (u64)depth ? st[ST_DEPTH] : (u64)depth;
        }
      } else {
        u64 klo, khi;
        child_bounds(sg, c, &klo, &khi);
        int flag = 0;
        u64 piv;
        if ((int)depth > P->max_depth) {  // depth guard: bisect the key bound
          piv = bisect_pivot(klo, khi);
          if (lane == 0) st[ST_BISECTED] += 1ull;
        } else {
          // the samples are only loaded here; they are sorted after the
          // round's queue claims, whose round trip their loads overlap
          S = sample_count(cl);
          if (S > kWarpSampleMax) S = kWarpSampleMax;
          __syncwarp();
          load_samples<C, kWarpQ>(reinterpret_cast<const U *>(P->keys[db]), !P->raw[db], cb, cl, S,
                                  P->dran, P->mitigation, lane, sv);
          piv = 0;
        }
        if (lane == 0) {
          uint32_t kind = KIND_PARTITION;
          if (P->fast_paths)
            kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
          ReqLevel &q = rs.lv[warp][0];
          q.klo = klo; q.khi = khi;
          q.begin = cb; q.end = cb + cl; q.pivot = piv; q.buf = db; q.kind = kind;
          q.depth = depth; q.noverify = 0; q.ntiles = tiles_of<C, PAY>(cb, cb + cl); q.valid = 1;
        }
      }
    }
  }
  TSQ_SC(4);
  __syncthreads();
  TSQ_SC(5);
  // one claim per queue for the whole round, the queues' atomics issued by
  // separate lanes of warp 0 so their round trips overlap
  if (threadIdx.x < 2 + kSmallClasses) {
    uint32_t nl = 0, nt = 0, nr = 0, nc = 0, nq = 0;
    const int q = (int)threadIdx.x - 2;
    for (int w = 0; w < kThreads / 32; ++w) {
      for (int c = 0; c < 2; ++c) {
        if (rs.lv[w][c].valid) { ++nl; nt += rs.lv[w][c].ntiles; }
        if (rs.sm[w][c].valid && q >= 0 && small_class(P, rs.sm[w][c].len) == q) ++nq;
      }
      if (rs.run[w].valid) { ++nr; nc += rs.run[w].nchunks; }
    }
    Ctl *ctl = P->ctl;
    if (threadIdx.x == 0 && nl) {
      const u64 old = atomicAdd(&ctl->next_packed, ((u64)nl << 32) | nt);
      rs.lv_slot0 = (uint32_t)(old >> 32);
      rs.lv_tile0 = (uint32_t)old;
      if (rs.lv_slot0 + nl > P->seg_cap || (u64)rs.lv_tile0 + nt > P->tile_cap) {
        atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
        rs.lv_slot0 = kDone;
      }
    } else if (threadIdx.x == 1 && nr) {
      const u64 old = atomicAdd(&ctl->run_packed, ((u64)nr << 32) | nc);
      rs.run_slot0 = (uint32_t)(old >> 32);
      rs.run_chunk0 = (uint32_t)old;
      if (rs.run_slot0 + nr > P->run_cap || (u64)rs.run_chunk0 + nc > P->chunk_cap) {
        atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
        rs.run_slot0 = kDone;
      }
    } else if (q >= 0 && nq) {
      rs.sq_slot0[q] = atomicAdd(&ctl->sq_count[q], nq);
      if (rs.sq_slot0[q] + nq > P->sq_cap[q]) {
        atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
        rs.sq_slot0[q] = kDone;
      }
    }
  }
  __syncthreads();
  TSQ_SC(6);
  if (S > 0) {
    // the pivot: median of the sorted samples; the order flag picks the
    // verification fast paths
    const int flag = warp_order_flag<U, kWarpQ>(sv, S);
    warp_bitonic<U, kWarpQ>(sv);
    const u64 piv = (u64)warp_pick<U, kWarpQ>(sv, S >> 1);
    if (lane == 0) {
      ReqLevel &q = rs.lv[warp][0];
      q.pivot = piv;
      if (P->fast_paths)
        q.kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    }
    __syncwarp();
  }
  TSQ_SC(7);
  // each warp writes its records at its offsets
  uint32_t lslot = rs.lv_slot0, ltile = rs.lv_tile0, rslot = rs.run_slot0;
  uint32_t rchunk = rs.run_chunk0;
  uint32_t qslot[kSmallClasses];
#pragma unroll
  for (int q = 0; q < kSmallClasses; ++q) qslot[q] = rs.sq_slot0[q];
  for (int w = 0; w < warp; ++w) {
    for (int c = 0; c < 2; ++c) {
      if (rs.lv[w][c].valid) { ++lslot; ltile += rs.lv[w][c].ntiles; }
      if (rs.sm[w][c].valid) ++qslot[small_class(P, rs.sm[w][c].len)];
    }
    if (rs.run[w].valid) { ++rslot; rchunk += rs.run[w].nchunks; }
  }
  for (int c = 0; c < 2; ++c) {
    const ReqLevel &q = rs.lv[warp][c];
    if (q.valid) {
      if (rs.lv_slot0 != kDone) {
        if (lane == 0) {
          Seg s;
          s.begin = q.begin; s.end = q.end; s.pivot = q.pivot;
          s.klo = q.klo; s.khi = q.khi;
          s.tile_base = ltile; s.ntiles = q.ntiles;
          s.buf = q.buf; s.kind = q.kind; s.depth = q.depth; s.noverify = q.noverify;
          s.eq_fill = 0; s.fail = 0; s.fill = 0;
          P->segs[nxt][lslot] = s;
        }
        uint32_t *tm = P->tilemap[nxt] + ltile;
        for (uint32_t i = lane; i < q.ntiles; i += 32) tm[i] = lslot;
      }
      ++lslot;
      ltile += q.ntiles;
    }
    const ReqSmall &m = rs.sm[warp][c];
    if (m.valid) {
      const int q = small_class(P, m.len);
      if (rs.sq_slot0[q] != kDone && lane == 0) {
        SmallSeg s;
        s.begin = m.begin; s.len = (int)m.len; s.buf = (int)m.buf;
        P->sq[q][qslot[q]] = s;
      }
      ++qslot[q];
    }
  }
  const ReqRun &q = rs.run[warp];
  if (q.valid && rs.run_slot0 != kDone) {
    if (lane == 0) {
      Run r;
      r.begin = q.begin; r.len = q.len; r.pivot = q.pivot; r.src = q.src;
      r.kind = q.kind; r.buf = q.buf; r.chunk_base = rchunk; r.nchunks = q.nchunks;
      P->runs[rslot] = r;
    }
    uint32_t *cm = P->chunkmap + rchunk;
    for (uint32_t i = lane; i < q.nchunks; i += 32) cm[i] = rslot;
  }
  __syncthreads();  // the round's shared requests are consumed
  TSQ_SC(8);
}

// CTA-wide appends (CTA mode: few segments, no contention to aggregate)
template <class C, bool PAY>
__device__ void cta_append_level(const Params *P, int nxt, long long begin, long long end,
                                 uint32_t buf, u64 pivot, u64 klo, u64 khi, uint32_t kind,
                                 uint32_t depth, uint32_t noverify, volatile uint32_t *bc) {
  const uint32_t ntiles = tiles_of<C, PAY>(begin, end);
  if (threadIdx.x == 0) {
    Ctl *ctl = P->ctl;
    const u64 old = atomicAdd(&ctl->next_packed, (1ull << 32) | ntiles);
    uint32_t slot = (uint32_t)(old >> 32);
    const uint32_t tbase = (uint32_t)old;
    if (slot < P->seg_cap && (u64)tbase + ntiles <= P->tile_cap) {
      Seg s;
      s.begin = begin; s.end = end; s.pivot = pivot;
      s.klo = klo; s.khi = khi;
      s.tile_base = tbase; s.ntiles = ntiles;
      s.buf = buf; s.kind = kind; s.depth = depth; s.noverify = noverify;
      s.eq_fill = 0; s.fail = 0; s.fill = 0;
      P->segs[nxt][slot] = s;
    } else {
      atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
      slot = kDone;
    }
    bc[0] = slot;
    bc[1] = tbase;
  }
  __syncthreads();
  const uint32_t slot = bc[0], tbase = bc[1];
  if (slot != kDone) {
    uint32_t *tm = P->tilemap[nxt] + tbase;
    for (uint32_t i = threadIdx.x; i < ntiles; i += kThreads) tm[i] = slot;
  }
  __syncthreads();
}

__device__ void cta_append_run(const Params *P, uint32_t kind, long long begin, long long len,
                               uint32_t buf, u64 pivot, long long src, volatile uint32_t *bc) {
  const uint32_t nchunks = chunks_of(kind, len, buf);
  if (nchunks == 0) return;
  if (threadIdx.x == 0) {
    Ctl *ctl = P->ctl;
    const u64 old = atomicAdd(&ctl->run_packed, (1ull << 32) | nchunks);
    uint32_t slot = (uint32_t)(old >> 32);
    const uint32_t cbase = (uint32_t)old;
    if (slot < P->run_cap && (u64)cbase + nchunks <= P->chunk_cap) {
      Run r;
      r.begin = begin; r.len = len; r.pivot = pivot; r.src = src;
      r.kind = kind; r.buf = buf; r.chunk_base = cbase; r.nchunks = nchunks;
      P->runs[slot] = r;
    } else {
      atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
      slot = kDone;
    }
    bc[0] = slot;
    bc[1] = cbase;
  }
  __syncthreads();
  const uint32_t slot = bc[0], cbase = bc[1];
  if (slot != kDone) {
    uint32_t *cm = P->chunkmap + cbase;
    for (uint32_t i = threadIdx.x; i < nchunks; i += kThreads) cm[i] = slot;
  }
  __syncthreads();
}

// CTA mode: one CTA per (segment, child); the child-0 CTA also does the
// segment's bookkeeping.
template <class C, bool PAY>
__device__ void schedule_segment_cta(const Params *P, int cur, int nxt, uint32_t task,
                                     typename C::U *xk, u64 *st, volatile uint32_t *bc) {
  typedef typename C::U U;
  const uint32_t sid = task >> 1;
  const int only = (int)(task & 1u);
  const Seg sg = P->segs[cur][sid];
  long long lt = 0, gt = 0;
  uint32_t requeue = 0;
  const bool kids =
      segment_head<C, PAY, true>(P, nxt, sg, cur, st, &lt, &gt, &requeue, only == 0);
  __syncthreads();
  const long long len = sg.end - sg.begin;
  if (only == 1) {
    if (!kids) return;
  } else if (sg.kind != KIND_PARTITION) {
    if (requeue) {
      cta_append_level<C, PAY>(P, nxt, sg.begin, sg.end, sg.buf, sg.pivot, sg.klo, sg.khi,
                               KIND_PARTITION, sg.depth, 1, bc);
    } else {
      const uint32_t rk = sg.kind == KIND_VERIFY_ASC ? RUN_SORTED : RUN_REVERSED;
      if (!(rk == RUN_SORTED && sg.buf == 0))
        cta_append_run(P, rk, sg.begin, len, sg.buf, 0ull, sg.begin, bc);
    }
    return;
  }
  const long long eq = len - lt - gt;
  if (only == 0 && eq > 0 && !PAY)
    cta_append_run(P, RUN_EQ, sg.begin + lt, eq, sg.buf, sg.pivot, sg.begin, bc);
  if (!kids) return;
  const uint32_t db = sg.buf ^ 1u;
  const uint32_t depth = sg.depth + 1;
  {
    const int c = only;
    const long long cb = c == 0 ? sg.begin : sg.end - gt;
    TSQ_CHECK(lt >= 0 && gt >= 0 && lt + gt <= sg.end - sg.begin);
    const long long cl = c == 0 ? lt : gt;
    if (cl <= 0) return;
    if (cl <= P->small_t) {
      if (threadIdx.x == 0) {
        append_small(P, cb, cl, db);
        st[ST_DEPTH] = st[ST_DEPTH] > (u64)depth ? st[ST_DEPTH] : (u64)depth;
      }
      return;
    }
    u64 klo, khi;
    child_bounds(sg, c, &klo, &khi);
    int flag = 0;
    u64 piv;
    if ((int)depth > P->max_depth) {  // depth guard: bisect the key bound
      piv = bisect_pivot(klo, khi);
      if (threadIdx.x == 0) st[ST_BISECTED] += 1ull;
    } else {
      piv = (u64)cta_select_pivot_fast<C>(reinterpret_cast<const U *>(P->keys[db]), !P->raw[db],
                                          cb, cl, P->dran, P->mitigation, xk, bc, &flag);
    }
    uint32_t kind = KIND_PARTITION;
    if (P->fast_paths)
      kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    cta_append_level<C, PAY>(P, nxt, cb, cb + cl, db, piv, klo, khi, kind, depth, 0, bc);
  }
}

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) schedule_kernel(const Params *__restrict__ P,
                                                            Ctl *ctl) {
  typedef typename C::U U;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ u64 st_all[kThreads / 32][ST_COUNT];
  __shared__ uint32_t bcast[2];
  __shared__ RoundShared rs;
  // the parameter block on chip (read all over the scheduling; its global
  // copy costs a round trip at first touch), fetched beside the level state
  __shared__ __align__(16) Params sparams;
  static_assert(sizeof(Params) / 8 <= kThreads, "Params copy");
  if (threadIdx.x < sizeof(Params) / 8)
    reinterpret_cast<u64 *>(&sparams)[threadIdx.x] = reinterpret_cast<const u64 *>(P)[threadIdx.x];
  P = &sparams;  // (complete after the barrier below)
  u64 *st = st_all[threadIdx.x >> 5];
  // (ctl by value: this read does not wait for the parameter block's)
#ifdef TSQ_EXP_CTL_FROM_PARAMS
  ctl = P->ctl;
#endif
  TSQ_SC(0);
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u), nxt = cur ^ 1;
  const uint32_t nseg = ctl->cur_nseg;
  for (int i = threadIdx.x; i < (kThreads / 32) * ST_COUNT; i += kThreads) (&st_all[0][0])[i] = 0ull;
  __syncthreads();
  if (P->reproducible) {  // the next level's look-back descriptors
    u64 *lbn = P->lookback[nxt];
    const uint32_t cap = P->tile_cap;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < cap; i += gridDim.x * kThreads)
      lbn[i] = 0ull;
  }
#ifdef TSQ_SCHED_CLOCK
  if (level == 0xffffffffu) return;  // (never: keeps the stamp behind the read)
#endif
  TSQ_SC(1);
  const long long avg = nseg ? ((long long)ctl->cur_ntiles * Geo<C, PAY>::TILE) / nseg : 0;
  if (avg >= kCtaScheduleMin) {
    U *xk = reinterpret_cast<U *>(smem_raw);
    for (uint32_t task = blockIdx.x; task < 2 * nseg; task += gridDim.x)
      schedule_segment_cta<C, PAY>(P, cur, nxt, task, xk, st, bcast);
  } else {
    const uint32_t per_round = gridDim.x * (kThreads / 32);
    const uint32_t ntask = 2 * nseg;
    for (uint32_t base = blockIdx.x * (kThreads / 32); base < ntask; base += per_round) {
      const uint32_t task = base + (threadIdx.x >> 5);
      schedule_round_warp<C, PAY>(P, cur, nxt, task, task < ntask, st, rs);
    }
  }
  __syncthreads();
  TSQ_SC(9);
  u64 tot = 0;
  if (threadIdx.x < ST_COUNT) {
    for (int w = 0; w < kThreads / 32; ++w) {
      const u64 v = st_all[w][threadIdx.x];
      tot = threadIdx.x == ST_DEPTH ? (tot > v ? tot : v) : tot + v;
    }
  }
  if (threadIdx.x < ST_COUNT && tot) {
    u64 *dst[ST_COUNT] = {&ctl->stages, &ctl->sorted_bypass, &ctl->reversed_bypass,
                          &ctl->max_depth, &ctl->bytes_partition, &ctl->bytes_retire,
                          &ctl->writes0, &ctl->writes1, &ctl->verify_fallbacks,
                          &ctl->partitioned_elements, &ctl->eq_runs, &ctl->eq_elements,
                          &ctl->bisected};
    if (threadIdx.x == ST_DEPTH) atomicMax(dst[ST_DEPTH], tot);
    else atomicAdd(dst[threadIdx.x], tot);
  }
  if (threadIdx.x == 0) {
    // one acquire-release counter bump per CTA (after the CTA barrier above
    // it publishes every thread's queue writes and, for the CTA that finds
    // itself last, makes all the others' visible)
    uint32_t d;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(d)
                 : "l"(&ctl->ctas_done)
                 : "memory");
    TSQ_SC(10);
    if (d == gridDim.x - 1) {
      // the queue state the decision needs, read side by side with the
      // exchange of the append cursor
      const uint32_t err0 = ld_volatile32(&ctl->error);
      const u64 runp = ld_volatile(&ctl->run_packed);
      const uint32_t sq0 = ld_volatile32(&ctl->sq_count[0]);
      const u64 packed = atomicExch(&ctl->next_packed, 0ull);
      const uint32_t ns = (uint32_t)(packed >> 32), nt = (uint32_t)packed;
      ctl->cur_nseg = ns;
      ctl->cur_ntiles = nt;
      ctl->tile_ticket = 0;
      ctl->ctas_done = 0;
      ctl->level = level + 1;
      ctl->levels += 1;
      bool more = ns > 0;
      uint32_t err = err0;
      if (more && level + 1 >= (uint32_t)kMaxLevels) {
        atomicOr(&ctl->error, (uint32_t)ERR_LEVELS);
        err |= (uint32_t)ERR_LEVELS;
      }
      if (err) more = false;
      // drain the on-chip and run queues before a level could overflow them:
      // one level appends at most 2 * seg_cap small segments and seg_cap runs
      // (the large on-chip class cannot overflow: its segments are disjoint
      // and longer than the small class's capacity, sq_cap[1] > n / that)
      const uint32_t runs = (uint32_t)(runp >> 32);
      const bool flush = more && (sq0 + 2u * P->seg_cap > P->sq_cap[0] ||
                                  runs + P->seg_cap > P->run_cap);
      ctl->flush = flush ? 1u : 0u;
      // (the kernel boundary orders these writes before the next kernel)
      if (P->use_cond) cudaGraphSetConditional(P->cond, (more && !flush) ? 1u : 0u);
#ifdef TSQ_SCHED_CLOCK
      {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        if (level == TSQ_SCHED_CLOCK) {
          printf("sched level %u nseg %u last-cta %u: ", level, nseg, blockIdx.x);
          for (int i = 1; i <= 10; ++i) printf("%d:%lld ", i, (long long)(g_sc[i] - g_sc[0]));
          printf("end:%lld ns\n", (long long)(t_ - g_sc[0]));
        }
      }
#endif
    }
  }
}

}  // namespace tsq
