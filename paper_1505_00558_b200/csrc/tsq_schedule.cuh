// tsq_schedule.cuh -- the per-segment bookkeeping between two partition
// passes (the tail of one Sorter._range stage and the head of the next,
// /root/reference/pkg/src/tsqsort/core.py:1705-1728).  Included by
// tsq_kernels.cuh.
//
// For every segment of the level just partitioned: retire the == p block
// (never compared again), then queue each child -- the < part and the > part
// -- either for the on-chip sort (<= small_t keys) or for the next level
// with its pivot sampled now (select_pivot's role, pivot.py:205-248).  A
// group of threads owns one segment: a whole CTA while segments are large
// (few segments, 1023-key samples), one warp per segment once they are small
// (thousands of segments, 31..255-key samples).
#pragma once

namespace tsq {

// per-CTA statistics (shared-memory atomics, one global flush per CTA)
enum SchedStat {
  ST_STAGES, ST_SORTED, ST_REVERSED, ST_DEPTH, ST_BYTES_PART, ST_BYTES_RETIRE, ST_W0, ST_W1,
  ST_FALLBACK, ST_PARTITIONED, ST_EQ_RUNS, ST_EQ_ELEMS, ST_COUNT
};

// A cooperating group: one warp, or the whole CTA.
template <bool CTA>
struct Group {
  static constexpr int SIZE = CTA ? kThreads : 32;
  static __device__ __forceinline__ int rank() { return CTA ? (int)threadIdx.x : (int)(threadIdx.x & 31); }
  static __device__ __forceinline__ void sync() {
    if (CTA) __syncthreads(); else __syncwarp();
  }
};

// Queue a segment for the next level: the leader claims the slot and its
// tile range with one packed atomic, the group fills the tile map.
template <class C, bool PAY, bool CTA>
__device__ void group_append_level(const Params *P, int nxt, long long begin, long long end,
                                   uint32_t buf, u64 pivot, uint32_t kind, uint32_t depth,
                                   uint32_t noverify, volatile uint32_t *bc) {
  typedef Group<CTA> G;
  const long long T = Geo<C, PAY>::TILE;
  const uint32_t ntiles = (uint32_t)((end - 1) / T - begin / T + 1);
  if (G::rank() == 0) {
    Ctl *ctl = P->ctl;
    const u64 old = atomicAdd(&ctl->next_packed, (1ull << 32) | ntiles);
    uint32_t slot = (uint32_t)(old >> 32);
    const uint32_t tbase = (uint32_t)old;
    if (slot < P->seg_cap && (u64)tbase + ntiles <= P->tile_cap) {
      Seg s;
      s.begin = begin; s.end = end; s.pivot = pivot;
      s.tile_base = tbase; s.ntiles = ntiles;
      s.buf = buf; s.kind = kind; s.depth = depth; s.noverify = noverify;
      s.done = 0; s.fail = 0;
      P->segs[nxt][slot] = s;
    } else {
      atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
      slot = kDone;
    }
    bc[0] = slot;
    bc[1] = tbase;
  }
  G::sync();
  const uint32_t slot = bc[0], tbase = bc[1];
  if (slot != kDone) {
    uint32_t *tm = P->tilemap[nxt] + tbase;
    for (uint32_t i = G::rank(); i < ntiles; i += G::SIZE) tm[i] = slot;
  }
  G::sync();
}

template <bool CTA>
__device__ void group_append_run(const Params *P, uint32_t kind, long long begin, long long len,
                                 uint32_t buf, u64 pivot, long long src, volatile uint32_t *bc) {
  typedef Group<CTA> G;
  uint32_t nchunks;
  if (kind == RUN_REVERSED && buf == 0)
    nchunks = (uint32_t)(((len >> 1) + kRunChunk - 1) / kRunChunk);
  else
    nchunks = (uint32_t)((len + kRunChunk - 1) / kRunChunk);
  if (nchunks == 0) return;
  if (G::rank() == 0) {
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
  G::sync();
  const uint32_t slot = bc[0], cbase = bc[1];
  if (slot != kDone) {
    uint32_t *cm = P->chunkmap + cbase;
    for (uint32_t i = G::rank(); i < nchunks; i += G::SIZE) cm[i] = slot;
  }
  G::sync();
}

__device__ __forceinline__ void append_small(const Params *P, long long begin, long long len,
                                             uint32_t buf) {
  Ctl *ctl = P->ctl;
  const uint32_t slot = atomicAdd(&ctl->small_count, 1u);
  if (slot < P->small_cap) {
    SmallSeg s;
    s.begin = begin; s.len = (int)len; s.buf = (int)buf;
    P->smalls[slot] = s;
  } else {
    atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
  }
}

// ---- group pivot sampling (select_pivot analogue, pivot.py:205-248) --------
// Median of S = sample_count(len) strided samples; the first, middle and
// last positions are fixed anchors and interior positions shift by the
// MitigationRng jitter (dran, pivot.py:223-237).  *flag gets the order flag
// of the samples in position order (+1 nondecreasing, -1 nonincreasing).
// `s` is the group's scratch of kMaxSample + 1 keys.
template <class C, bool CTA>
__device__ typename C::U group_select_pivot(const typename C::U *data, bool encoded_src,
                                            long long begin, long long len, double dran,
                                            int mitigation, typename C::U *s, int *flag,
                                            volatile uint32_t *bc) {
  typedef typename C::U U;
  typedef Group<CTA> G;
  constexpr int Q = (kMaxSample + 1) / G::SIZE;
  const int r = G::rank();
  const int S = sample_count(len);
  const int P2 = S + 1;
  const int midi = S >> 1;
  const long long span = len - 1;
  long long shift = 0;
  if (mitigation) {
    const double stride = (double)span / (double)(S - 1);
    shift = (long long)floor((dran - 1.0) * stride * 0.5);
  }
  const double step = (double)span / (double)(S - 1);
  // all of a thread's sample loads are issued before any is consumed
  U vals[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = r + G::SIZE * q;
    vals[q] = KeyMax<U>::v;
    if (i < S) {
      long long pos = (i == S - 1) ? begin + span : begin + (long long)((double)i * step);
      if (i != 0 && i != midi && i != S - 1) {
        pos += shift;
        pos = pos < begin ? begin : (pos > begin + span ? begin + span : pos);
      }
      vals[q] = ldcg(data + pos);
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = r + G::SIZE * q;
    if (i < P2) s[i] = (i < S && !encoded_src) ? C::enc(vals[q]) : vals[q];
  }
  G::sync();
  bool asc = true, desc = true;
  for (int i = r; i < S - 1; i += G::SIZE) {
    const U a = s[i], b = s[i + 1];
    asc &= (a <= b);
    desc &= (a >= b);
  }
  if (CTA) {
    asc = __syncthreads_and(asc);
    desc = __syncthreads_and(desc);
  } else {
    asc = __all_sync(0xffffffffu, asc);
    desc = __all_sync(0xffffffffu, desc);
  }
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = r; i < (P2 >> 1); i += G::SIZE) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo + j;
        const bool up = (lo & k) == 0;
        const U a = s[lo], b = s[hi];
        if ((a > b) == up) {
          s[lo] = b;
          s[hi] = a;
        }
      }
      G::sync();
    }
  }
  *flag = asc ? 1 : (desc ? -1 : 0);
  const U piv = s[midi];
  G::sync();
  return piv;
}

// ---------------------------------------------------------------------------

template <class C, bool PAY, bool CTA>
__device__ void schedule_segment(const Params *P, int cur, int nxt, uint32_t sid,
                                 typename C::U *scratch, u64 *st, volatile uint32_t *bc) {
  typedef typename C::U U;
  typedef Group<CTA> G;
  const int r = G::rank();
  const bool leader = r == 0;
  Ctl *ctl = P->ctl;
  const Seg sg = P->segs[cur][sid];
  const long long len = sg.end - sg.begin;
  const int kb = (int)sizeof(U);
  if (sg.kind != KIND_PARTITION) {
    const bool failed = sg.fail != 0;
    if (!failed) {
      const uint32_t rk = sg.kind == KIND_VERIFY_ASC ? RUN_SORTED : RUN_REVERSED;
      const bool moves = !(rk == RUN_SORTED && sg.buf == 0);
      if (leader) {
        atomicAdd(&st[ST_STAGES], 1ull);
        atomicAdd(&st[rk == RUN_SORTED ? ST_SORTED : ST_REVERSED], 1ull);
        atomicMax(&st[ST_DEPTH], (u64)sg.depth);
        atomicAdd(&st[ST_BYTES_PART], (u64)len * kb);  // the verify read
        if (moves) {
          atomicAdd(&st[ST_BYTES_RETIRE], 2ull * (u64)len * (u64)(kb + (PAY ? 4 : 0)));
          atomicAdd(&st[ST_W0], (u64)len);
        }
      }
      if (moves) group_append_run<CTA>(P, rk, sg.begin, len, sg.buf, 0ull, sg.begin, bc);
    } else {
      if (leader) atomicAdd(&st[ST_FALLBACK], 1ull);
      group_append_level<C, PAY, CTA>(P, nxt, sg.begin, sg.end, sg.buf, sg.pivot,
                                      KIND_PARTITION, sg.depth, 1, bc);
    }
    return;
  }
  const u64 inc = P->lookback[cur][sg.tile_base + sg.ntiles - 1];
  const long long lt = (long long)((inc >> 31) & 0x7fffffffull);
  const long long gt = (long long)(inc & 0x7fffffffull);
  const long long eq = len - lt - gt;
  if (leader) {
    atomicAdd(&st[ST_STAGES], 1ull);
    atomicAdd(&st[ST_PARTITIONED], (u64)len);
    atomicMax(&st[ST_DEPTH], (u64)sg.depth);
    u64 bytes = (u64)len * kb + (u64)(lt + gt) * kb;
    if (PAY) bytes += (u64)len * 8ull;
    atomicAdd(&st[ST_BYTES_PART], bytes);
    atomicAdd(&st[sg.buf == 0 ? ST_W1 : ST_W0], (u64)(lt + gt));
    if (PAY) atomicAdd(&st[ST_W1], (u64)eq);
    if (eq > 0) {
      atomicAdd(&st[ST_EQ_RUNS], 1ull);
      atomicAdd(&st[ST_EQ_ELEMS], (u64)eq);
      atomicAdd(&st[ST_BYTES_RETIRE], (u64)eq * (kb + (PAY ? 8 : 0)));
      atomicAdd(&st[ST_W0], (u64)eq);
    }
    if (P->single_stage) {
      ctl->stage_lt = (u64)lt;
      ctl->stage_gt = (u64)gt;
    }
  }
  if (eq > 0) {
    if (PAY) {
      // Records: the == p payloads sit at side_pay[begin ...], a range the
      // children reuse at the next level, so they move to their final place
      // now (nothing else touches [begin+lt, end-gt) of buffer 0).
      const uint32_t *side = P->side_pay + sg.begin;
      uint32_t *p0 = P->pay[0] + sg.begin + lt;
      U *k0 = reinterpret_cast<U *>(P->keys[0]) + sg.begin + lt;
      const U v = P->raw[0] ? C::dec((U)sg.pivot) : (U)sg.pivot;
      for (long long i = r; i < eq; i += G::SIZE) {
        p0[i] = side[i];
        k0[i] = v;
      }
    } else {
      group_append_run<CTA>(P, RUN_EQ, sg.begin + lt, eq, sg.buf, sg.pivot, sg.begin, bc);
    }
  }
  if (P->single_stage) return;
  const uint32_t db = sg.buf ^ 1u;
  const uint32_t depth = sg.depth + 1;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const long long cb = c == 0 ? sg.begin : sg.end - gt;
    const long long cl = c == 0 ? lt : gt;
    if (cl <= 0) continue;
    if (cl <= P->small_t) {
      if (leader) {
        append_small(P, cb, cl, db);
        atomicMax(&st[ST_DEPTH], (u64)depth);
      }
      continue;
    }
    if ((int)depth > P->max_depth) {
      if (leader) atomicOr(&ctl->error, (uint32_t)ERR_DEPTH);
      continue;
    }
    int flag = 0;
    const U piv = group_select_pivot<C, CTA>(reinterpret_cast<const U *>(P->keys[db]),
                                             !P->raw[db], cb, cl, P->dran, P->mitigation,
                                             scratch, &flag, bc);
    uint32_t kind = KIND_PARTITION;
    if (P->fast_paths)
      kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    group_append_level<C, PAY, CTA>(P, nxt, cb, cb + cl, db, (u64)piv, kind, depth, 0, bc);
  }
}

// Segments of at least this many keys (on average) are scheduled by a whole
// CTA each; below it one warp per segment.
constexpr long long kCtaScheduleMin = 1ll << 17;

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) schedule_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ u64 st[ST_COUNT];
  __shared__ uint32_t bcast[kThreads / 32][2];
  Ctl *ctl = P->ctl;
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u), nxt = cur ^ 1;
  const uint32_t nseg = ctl->cur_nseg;
  const int warp = threadIdx.x >> 5;
  {
    u64 *lbn = P->lookback[nxt];
    const uint32_t cap = P->tile_cap;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < cap; i += gridDim.x * kThreads)
      lbn[i] = 0ull;
  }
  if (threadIdx.x < ST_COUNT) st[threadIdx.x] = 0ull;
  __syncthreads();
  const long long avg = nseg ? ((long long)ctl->cur_ntiles * Geo<C, PAY>::TILE) / nseg : 0;
  if (avg >= kCtaScheduleMin) {
    U *scratch = reinterpret_cast<U *>(smem_raw);
    for (uint32_t sid = blockIdx.x; sid < nseg; sid += gridDim.x)
      schedule_segment<C, PAY, true>(P, cur, nxt, sid, scratch, st, bcast[0]);
  } else {
    U *scratch = reinterpret_cast<U *>(smem_raw) + warp * (kMaxSample + 1);
    const uint32_t nwarps = gridDim.x * (kThreads / 32);
    for (uint32_t sid = blockIdx.x * (kThreads / 32) + warp; sid < nseg; sid += nwarps)
      schedule_segment<C, PAY, false>(P, cur, nxt, sid, scratch, st, bcast[warp]);
  }
  __syncthreads();
  if (threadIdx.x < ST_COUNT && st[threadIdx.x]) {
    u64 *dst[ST_COUNT] = {&ctl->stages, &ctl->sorted_bypass, &ctl->reversed_bypass,
                          &ctl->max_depth, &ctl->bytes_partition, &ctl->bytes_retire,
                          &ctl->writes0, &ctl->writes1, &ctl->verify_fallbacks,
                          &ctl->partitioned_elements, &ctl->eq_runs, &ctl->eq_elements};
    if (threadIdx.x == ST_DEPTH) atomicMax(dst[ST_DEPTH], st[ST_DEPTH]);
    else atomicAdd(dst[threadIdx.x], st[threadIdx.x]);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t d = atomicAdd(&ctl->ctas_done, 1u);
    if (d == gridDim.x - 1) {
      __threadfence();
      const u64 packed = atomicExch(&ctl->next_packed, 0ull);
      const uint32_t ns = (uint32_t)(packed >> 32), nt = (uint32_t)packed;
      ctl->cur_nseg = ns;
      ctl->cur_ntiles = nt;
      ctl->tile_ticket = 0;
      ctl->ctas_done = 0;
      ctl->level = level + 1;
      ctl->levels += 1;
      bool more = ns > 0;
      if (more && level + 1 >= (uint32_t)kMaxLevels) {
        atomicOr(&ctl->error, (uint32_t)ERR_LEVELS);
        more = false;
      }
      if (ctl->error) more = false;
      __threadfence();
      if (P->use_cond) cudaGraphSetConditional(P->cond, more ? 1u : 0u);
    }
  }
}

}  // namespace tsq
