// tsq_kernels.cuh -- the kernels of the B200 three-way partition sort.
//
//   init_kernel        root stage: pivot sampling of [0, n) and the level-0
//                      queue (Sorter.sort_with_stats -> _range entry,
//                      core.py:1599-1607)
//   partition_kernel   one recursion level over every live segment: the
//                      multi-block three-way partition (the stage that
//                      _run_machine performs, core.py:198-984).  Persistent,
//                      warp-specialised: a producer warp claims tiles and
//                      streams them into a 3-deep shared-memory ring with
//                      bulk copies (TMA engine, cp.async.bulk + mbarrier);
//                      8 consumer warps classify keys with __ballot_sync /
//                      __popc, publish per-tile (<, >) counts and resolve
//                      their offsets by decoupled look-back, then write the
//                      < run from the segment front and the > run from the
//                      back.  Segments whose samples looked sorted/reversed
//                      are verified instead (core.py:1678-1698 fast paths).
//   schedule_kernel    one warp per segment of the level: retires the ==p
//                      run, samples the children's pivots (pivot.py:205-248)
//                      and queues them for the next level or the on-chip
//                      sort (core.py:1711-1728); the last CTA advances the
//                      level and sets the CUDA-graph loop condition
//   small_sort_kernel  on-chip sorting network for segments <= small_t
//                      (insertion_sort's role, smallsort.py:12-47)
//   retire_kernel      writes ==p runs and verified runs into buffer 0
//
// Buffers: keys[0] is the caller's array (raw encoding), keys[1] the
// workspace partner (order-preserving unsigned encoding).  A partition pass
// reads a segment from buffer b and writes it to buffer b^1; every finished
// piece (==p run, on-chip-sorted segment, verified run) lands in buffer 0.
#pragma once

#include "tsq_device.cuh"

namespace tsq {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;   // 256
constexpr int kPartThreads = kConsumers + 32;     // + 1 producer warp
constexpr int kStages = 3;                        // input ring depth
constexpr int kAlign = 4;                         // bulk-copy element alignment
constexpr uint32_t kDone = 0xffffffffu;

template <class C, bool PAY>
struct Geo {
  typedef typename C::U U;
  static constexpr int VN = Vec<U>::N;     // keys per 16-byte vector
  static constexpr int VPT = 4;            // vectors per thread per tile
  static constexpr int IPT = VN * VPT;     // keys per thread per tile
  static constexpr int TILE = kConsumers * IPT;
  static constexpr size_t KB = sizeof(U);
  static constexpr size_t STAGE_BYTES = (size_t)TILE * (KB + (PAY ? 4 : 0));
  static constexpr size_t SMEM = (size_t)(kStages + 1) * STAGE_BYTES;
};

__device__ __forceinline__ void unpack(const uint4 &v, uint32_t *o) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void unpack(const ulonglong2 &v, u64 *o) {
  o[0] = v.x; o[1] = v.y;
}
__device__ __forceinline__ void unpack(const uint2 &v, uint32_t *o) {
  o[0] = v.x; o[1] = v.y;
}

// Tile descriptor handed from the producer warp to the consumers.
struct StageMeta {
  long long tstart, lo, hi, begin, end;
  u64 pivot, next_key;
  uint32_t t, k, kind, buf, tile_base, sid, skip, has_next;
};

// ---------------------------------------------------------------------------
// Warp-level queue appends (lane 0 claims the slot; the warp fills the map).

template <class C, bool PAY>
__device__ void warp_append_level(const Params *P, int nxt, long long begin, long long end,
                                  uint32_t buf, u64 pivot, uint32_t kind, uint32_t depth,
                                  uint32_t noverify) {
  const int lane = threadIdx.x & 31;
  const long long T = Geo<C, PAY>::TILE;
  const uint32_t ntiles = (uint32_t)((end - 1) / T - begin / T + 1);
  uint32_t slot = kDone, tbase = 0;
  if (lane == 0) {
    Ctl *ctl = P->ctl;
    const u64 old = atomicAdd(&ctl->next_packed, (1ull << 32) | ntiles);
    slot = (uint32_t)(old >> 32);
    tbase = (uint32_t)old;
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
  }
  slot = __shfl_sync(0xffffffffu, slot, 0);
  tbase = __shfl_sync(0xffffffffu, tbase, 0);
  if (slot != kDone) {
    uint32_t *tm = P->tilemap[nxt] + tbase;
    for (uint32_t i = lane; i < ntiles; i += 32) tm[i] = slot;
  }
}

__device__ void warp_append_run(const Params *P, uint32_t kind, long long begin, long long len,
                                uint32_t buf, u64 pivot, long long src) {
  const int lane = threadIdx.x & 31;
  uint32_t nchunks;
  if (kind == RUN_REVERSED && buf == 0)
    nchunks = (uint32_t)(((len >> 1) + kRunChunk - 1) / kRunChunk);
  else
    nchunks = (uint32_t)((len + kRunChunk - 1) / kRunChunk);
  if (nchunks == 0) return;
  uint32_t slot = kDone, cbase = 0;
  if (lane == 0) {
    Ctl *ctl = P->ctl;
    const u64 old = atomicAdd(&ctl->run_packed, (1ull << 32) | nchunks);
    slot = (uint32_t)(old >> 32);
    cbase = (uint32_t)old;
    if (slot < P->run_cap && (u64)cbase + nchunks <= P->chunk_cap) {
      Run r;
      r.begin = begin; r.len = len; r.pivot = pivot; r.src = src;
      r.kind = kind; r.buf = buf; r.chunk_base = cbase; r.nchunks = nchunks;
      P->runs[slot] = r;
    } else {
      atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
      slot = kDone;
    }
  }
  slot = __shfl_sync(0xffffffffu, slot, 0);
  cbase = __shfl_sync(0xffffffffu, cbase, 0);
  if (slot != kDone) {
    uint32_t *cm = P->chunkmap + cbase;
    for (uint32_t i = lane; i < nchunks; i += 32) cm[i] = slot;
  }
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

// ---- warp-level pivot sampling (select_pivot analogue, pivot.py:205-248) ---
// Same sample positions as cta_select_pivot; `s` is this warp's scratch of
// kMaxSample + 1 keys.  Returns the pivot; *flag gets the order flag.
template <class C>
__device__ typename C::U warp_select_pivot(const typename C::U *data, bool encoded_src,
                                           long long begin, long long len, double dran,
                                           int mitigation, typename C::U *s, int *flag) {
  typedef typename C::U U;
  const int lane = threadIdx.x & 31;
  const int S = sample_count(len);
  const int P2 = S + 1;
  const int midi = S >> 1;
  const long long span = len - 1;
  long long shift = 0;
  if (mitigation) {
    const double stride = (double)span / (double)(S - 1);
    shift = (long long)floor((dran - 1.0) * stride * 0.5);
  }
  for (int i = lane; i < P2; i += 32) {
    U v = KeyMax<U>::v;
    if (i < S) {
      long long pos = begin + ((long long)i * span) / (S - 1);
      if (i != 0 && i != midi && i != S - 1) {
        pos += shift;
        pos = pos < begin ? begin : (pos > begin + span ? begin + span : pos);
      }
      v = ldcg(data + pos);
      if (!encoded_src) v = C::enc(v);
    }
    s[i] = v;
  }
  __syncwarp();
  bool asc = true, desc = true;
  for (int i = lane; i < S - 1; i += 32) {
    const U a = s[i], b = s[i + 1];
    asc &= (a <= b);
    desc &= (a >= b);
  }
  asc = __all_sync(0xffffffffu, asc);
  desc = __all_sync(0xffffffffu, desc);
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < (P2 >> 1); i += 32) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo + j;
        const bool up = (lo & k) == 0;
        const U a = s[lo], b = s[hi];
        if ((a > b) == up) {
          s[lo] = b;
          s[hi] = a;
        }
      }
      __syncwarp();
    }
  }
  *flag = asc ? 1 : (desc ? -1 : 0);
  const U piv = s[midi];
  __syncwarp();
  return piv;
}

// ---------------------------------------------------------------------------
// Partition kernel: producer warp.

template <class C, bool PAY>
__device__ __forceinline__ void producer_loop(const Params *P, int cur, uint32_t ntiles,
                                              typename C::U *in_k, uint32_t *in_p, u64 *full,
                                              u64 *empty, StageMeta *meta) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int lane = threadIdx.x & 31;
  Ctl *ctl = P->ctl;
  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % kStages);
    const uint32_t j = it / kStages;
    if (j > 0) mbar_wait(&empty[s], (j - 1) & 1u);
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
    const uint32_t sid = P->tilemap[cur][t];
    const Seg *sgp = &P->segs[cur][sid];
    const long long begin = sgp->begin, end = sgp->end;
    const uint32_t tile_base = sgp->tile_base, kind = sgp->kind, buf = sgp->buf;
    const uint32_t k = t - tile_base;
    const long long tstart = (begin / G::TILE + k) * (long long)G::TILE;
    const long long lo = tstart > begin ? tstart : begin;
    const long long hi = (tstart + G::TILE) < end ? (tstart + G::TILE) : end;
    const U *src = reinterpret_cast<const U *>(P->keys[buf]);
    const uint32_t *psrc = PAY ? P->pay[buf] : nullptr;
    U *dk = in_k + (size_t)s * G::TILE;
    uint32_t *dp = PAY ? in_p + (size_t)s * G::TILE : nullptr;
    uint32_t skip = 0;
    if (kind != KIND_PARTITION) skip = ld_volatile32(&sgp->fail) != 0 ? 1u : 0u;
    uint32_t tx = 0;
    long long a0 = 0, a1 = 0;
    if (!skip) {
      if (P->aligned[buf]) {
        a0 = lo & ~(long long)(kAlign - 1);
        a1 = (hi + kAlign - 1) & ~(long long)(kAlign - 1);
        const long long cap = P->n & ~(long long)(kAlign - 1);  // never read past n
        if (a1 > cap) a1 = cap;
        if (a1 < a0) a1 = a0;
        // ragged tail of the caller's array: plain loads
        for (long long i = a1 + lane; i < hi; i += 32) {
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
      m.pivot = sgp->pivot;
      m.t = t; m.k = k; m.kind = kind; m.buf = buf; m.tile_base = tile_base; m.sid = sid;
      m.skip = skip;
      m.has_next = 0;
      if (kind != KIND_PARTITION && !skip && hi < end) {
        U v = src[hi];
        if (P->raw[buf]) v = C::enc(v);
        m.next_key = (u64)v;
        m.has_next = 1;
      }
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
// Partition kernel: one tile on the consumer warps.

template <class C, bool PAY>
__device__ __forceinline__ void consume_partition(const Params *P, int cur, const StageMeta &m,
                                                  const typename C::U *sk,
                                                  const uint32_t *sp, u64 *empty_s,
                                                  typename C::U *ok, uint32_t *op,
                                                  uint32_t (*wcnt)[3], u64 *s_excl) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int sb = (int)m.buf, db = sb ^ 1;
  const bool src_raw = P->raw[sb] != 0, dst_raw = P->raw[db] != 0;
  const U piv = (U)m.pivot;
  const long long rlo = m.lo - m.tstart, rhi = m.hi - m.tstart;

  U key[G::IPT];
  uint32_t pay[PAY ? G::IPT : 1];
  uint32_t cls[G::IPT];
#pragma unroll
  for (int v = 0; v < G::VPT; ++v) {
    const int e0 = (v * kConsumers + tid) * G::VN;
    typename Vec<U>::K kv = *reinterpret_cast<const typename Vec<U>::K *>(sk + e0);
    unpack(kv, key + v * G::VN);
    if (PAY) {
      typename Vec<U>::P pv = *reinterpret_cast<const typename Vec<U>::P *>(sp + e0);
      unpack(pv, pay + v * G::VN);
    }
#pragma unroll
    for (int q = 0; q < G::VN; ++q) {
      const int idx = e0 + q;
      cls[v * G::VN + q] = (idx >= rlo && idx < rhi) ? 0u : 3u;
    }
  }
  // the stage is in registers: hand it back to the producer
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_s);
#pragma unroll
  for (int i = 0; i < G::IPT; ++i) {
    if (src_raw) key[i] = C::enc(key[i]);
    if (cls[i] == 0) cls[i] = key[i] < piv ? 0u : (key[i] == piv ? 1u : 2u);
  }
  // warp-level ranks per class, ordered by (item, lane)
  const uint32_t lmask = (1u << lane) - 1u;
  uint32_t lt_run = 0, gt_run = 0, eq_run = 0;
  uint32_t rank[G::IPT];
#pragma unroll
  for (int i = 0; i < G::IPT; ++i) {
    const uint32_t blt = __ballot_sync(0xffffffffu, cls[i] == 0);
    const uint32_t bgt = __ballot_sync(0xffffffffu, cls[i] == 2);
    const uint32_t beq = PAY ? __ballot_sync(0xffffffffu, cls[i] == 1) : 0u;
    uint32_t r;
    if (cls[i] == 0) r = lt_run + __popc(blt & lmask);
    else if (cls[i] == 2) r = gt_run + __popc(bgt & lmask);
    else r = eq_run + __popc(beq & lmask);
    rank[i] = r;
    lt_run += __popc(blt);
    gt_run += __popc(bgt);
    eq_run += __popc(beq);
  }
  if (lane == 0) {
    wcnt[warp][0] = lt_run;
    wcnt[warp][1] = eq_run;
    wcnt[warp][2] = gt_run;
  }
  named_sync(1, kConsumers);
  uint32_t w_lt = 0, w_eq = 0, w_gt = 0, t_lt = 0, t_eq = 0, t_gt = 0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) {
    const uint32_t a = wcnt[w][0], b = wcnt[w][1], c = wcnt[w][2];
    if (w < warp) { w_lt += a; w_eq += b; w_gt += c; }
    t_lt += a; t_eq += b; t_gt += c;
  }
  const u64 agg = ((u64)t_lt << 31) | (u64)t_gt;
  u64 *lb = P->lookback[cur];
  if (tid == 0) st_volatile(&lb[m.t], (m.k == 0 ? kFlagInc : kFlagAgg) | agg);

  // stage the tile as [< | > | == (payload only)]
  const uint32_t nlg = t_lt + t_gt;
#pragma unroll
  for (int i = 0; i < G::IPT; ++i) {
    const uint32_t c = cls[i];
    if (c == 3u) continue;
    uint32_t pos;
    if (c == 0u) pos = w_lt + rank[i];
    else if (c == 2u) pos = t_lt + w_gt + rank[i];
    else {
      if (!PAY) continue;
      pos = nlg + w_eq + rank[i];
    }
    if (c != 1u) ok[pos] = key[i];
    if (PAY) op[pos] = pay[i];
  }

  // decoupled look-back (warp 0), bounded by the segment's first tile
  if (warp == 0) {
    u64 excl = 0;
    if (m.k > 0) {
      long long base = (long long)m.t - 1;
      const long long stop = (long long)m.tile_base;
      for (;;) {
        const long long idx = base - lane;
        u64 d = kFlagInc;
        if (idx >= stop) {
          do {
            d = ld_volatile(&lb[idx]);
          } while ((d >> 62) == 0);
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (d >> 62) == 2);
        if (inc) {
          const int first = __ffs(inc) - 1;
          excl += warp_sum64(lane <= first ? (d & kValMask) : 0ull);
          break;
        }
        excl += warp_sum64(d & kValMask);
        base -= 32;
      }
      if (lane == 0) st_volatile(&lb[m.t], kFlagInc | (excl + agg));
    }
    if (lane == 0) *s_excl = excl;
  }
  named_sync(1, kConsumers);

  const u64 ex = *s_excl;
  const long long ex_lt = (long long)(ex >> 31), ex_gt = (long long)(ex & 0x7fffffffull);
  U *dst = reinterpret_cast<U *>(P->keys[db]);
  uint32_t *dpay = PAY ? P->pay[db] : nullptr;
  const long long lt_base = m.begin + ex_lt;
  const long long gt_base = m.end - 1 - ex_gt;
  for (uint32_t i = tid; i < nlg; i += kConsumers) {
    const long long d = (i < t_lt) ? (lt_base + i) : (gt_base - (long long)(i - t_lt));
    U v = ok[i];
    if (dst_raw) v = C::dec(v);
    dst[d] = v;
    if (PAY) dpay[d] = op[i];
  }
  if (PAY) {
    const long long ex_eq = (m.lo - m.begin) - ex_lt - ex_gt;
    uint32_t *side = P->side_pay + m.begin + ex_eq;
    for (uint32_t i = tid; i < t_eq; i += kConsumers) side[i] = op[nlg + i];
  }
}

// one verification tile: every adjacent pair inside the tile and the pair
// that crosses into the next tile must be ordered; a violation marks the
// segment failed (its later tiles are skipped by the producer)
template <class C, bool PAY>
__device__ __forceinline__ void consume_verify(const Params *P, int cur, const StageMeta &m,
                                               const typename C::U *sk, u64 *empty_s,
                                               uint32_t *s_flag) {
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
  __syncwarp();
  if ((tid & 31) == 0) mbar_arrive(empty_s);
  named_sync(1, kConsumers);
  if (tid == 0 && *s_flag) atomicOr(&P->segs[cur][m.sid].fail, 1u);
}

template <class C, bool PAY>
__global__ void __launch_bounds__(kPartThreads, PAY ? 2 : 3)
    partition_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  U *in_k = reinterpret_cast<U *>(smem_raw);
  uint32_t *in_p = reinterpret_cast<uint32_t *>(in_k + (size_t)kStages * G::TILE);
  U *out_k = reinterpret_cast<U *>(smem_raw + (size_t)kStages * G::STAGE_BYTES);
  uint32_t *out_p = reinterpret_cast<uint32_t *>(out_k + G::TILE);
  __shared__ __align__(8) u64 full[kStages], empty[kStages];
  __shared__ StageMeta meta[kStages];
  __shared__ uint32_t wcnt[kConsumerWarps][3];
  __shared__ u64 s_excl;
  __shared__ uint32_t s_flag;

  Ctl *ctl = P->ctl;
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u);
  const uint32_t ntiles = ctl->cur_ntiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x >= kConsumers) {
    producer_loop<C, PAY>(P, cur, ntiles, in_k, in_p, full, empty, meta);
    return;
  }
  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % kStages);
    mbar_wait(&full[s], (it / kStages) & 1u);
    const StageMeta m = meta[s];
    if (m.t == kDone) break;
    const U *sk = in_k + (size_t)s * G::TILE;
    if (m.kind == KIND_PARTITION) {
      consume_partition<C, PAY>(P, cur, m, sk, in_p + (size_t)s * G::TILE, &empty[s], out_k,
                                out_p, wcnt, &s_excl);
    } else {
      consume_verify<C, PAY>(P, cur, m, sk, &empty[s], &s_flag);
    }
  }
}

// ---------------------------------------------------------------------------
// Schedule kernel: one warp per segment of the level just partitioned.

template <class C, bool PAY>
__device__ void schedule_segment(const Params *P, int cur, int nxt, uint32_t sid,
                                 typename C::U *scratch) {
  typedef typename C::U U;
  const int lane = threadIdx.x & 31;
  Ctl *ctl = P->ctl;
  const Seg sg = P->segs[cur][sid];
  const long long len = sg.end - sg.begin;
  const int kb = (int)sizeof(U);
  if (sg.kind != KIND_PARTITION) {
    const bool failed = sg.fail != 0;
    if (!failed) {
      const uint32_t rk = sg.kind == KIND_VERIFY_ASC ? RUN_SORTED : RUN_REVERSED;
      const bool moves = !(rk == RUN_SORTED && sg.buf == 0);
      if (lane == 0) {
        atomicAdd(&ctl->stages, 1ull);
        atomicAdd(rk == RUN_SORTED ? &ctl->sorted_bypass : &ctl->reversed_bypass, 1ull);
        atomicMax(&ctl->max_depth, (u64)sg.depth);
        atomicAdd(&ctl->bytes_partition, (u64)len * kb);  // the verify read
        if (moves) {
          atomicAdd(&ctl->bytes_retire, 2ull * (u64)len * (u64)(kb + (PAY ? 4 : 0)));
          atomicAdd(&ctl->writes0, (u64)len);
        }
      }
      if (moves) warp_append_run(P, rk, sg.begin, len, sg.buf, 0ull, sg.begin);
    } else {
      if (lane == 0) atomicAdd(&ctl->verify_fallbacks, 1ull);
      warp_append_level<C, PAY>(P, nxt, sg.begin, sg.end, sg.buf, sg.pivot, KIND_PARTITION,
                                sg.depth, 1);
    }
    return;
  }
  const u64 inc = P->lookback[cur][sg.tile_base + sg.ntiles - 1];
  const long long lt = (long long)((inc >> 31) & 0x7fffffffull);
  const long long gt = (long long)(inc & 0x7fffffffull);
  const long long eq = len - lt - gt;
  if (lane == 0) {
    atomicAdd(&ctl->stages, 1ull);
    atomicAdd(&ctl->partitioned_elements, (u64)len);
    atomicMax(&ctl->max_depth, (u64)sg.depth);
    u64 bytes = (u64)len * kb + (u64)(lt + gt) * kb;
    if (PAY) bytes += (u64)len * 8ull;
    atomicAdd(&ctl->bytes_partition, bytes);
    atomicAdd(sg.buf == 0 ? &ctl->writes1 : &ctl->writes0, (u64)(lt + gt));
    if (PAY) atomicAdd(&ctl->writes1, (u64)eq);
    if (eq > 0) {
      atomicAdd(&ctl->eq_runs, 1ull);
      atomicAdd(&ctl->eq_elements, (u64)eq);
      atomicAdd(&ctl->bytes_retire, (u64)eq * (kb + (PAY ? 8 : 0)));
      atomicAdd(&ctl->writes0, (u64)eq);
    }
    if (P->single_stage) {
      ctl->stage_lt = (u64)lt;
      ctl->stage_gt = (u64)gt;
    }
  }
  if (eq > 0) {
    if (PAY) {
      // Records: the ==p payloads sit at side_pay[begin ...], a range the
      // children reuse at the next level, so they move to their final place
      // now (nothing else touches [begin+lt, end-gt) of buffer 0).
      const uint32_t *side = P->side_pay + sg.begin;
      uint32_t *p0 = P->pay[0] + sg.begin + lt;
      U *k0 = reinterpret_cast<U *>(P->keys[0]) + sg.begin + lt;
      const U v = P->raw[0] ? C::dec((U)sg.pivot) : (U)sg.pivot;
      for (long long i = lane; i < eq; i += 32) {
        p0[i] = side[i];
        k0[i] = v;
      }
    } else {
      warp_append_run(P, RUN_EQ, sg.begin + lt, eq, sg.buf, sg.pivot, sg.begin);
    }
  }
  if (P->single_stage) return;
  const uint32_t db = sg.buf ^ 1u;
  const long long cb[2] = {sg.begin, sg.end - gt};
  const long long cl[2] = {lt, gt};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (cl[c] <= 0) continue;
    const uint32_t depth = sg.depth + 1;
    if (cl[c] <= P->small_t) {
      if (lane == 0) {
        append_small(P, cb[c], cl[c], db);
        atomicMax(&ctl->max_depth, (u64)depth);
      }
      continue;
    }
    if ((int)depth > P->max_depth) {
      if (lane == 0) atomicOr(&ctl->error, (uint32_t)ERR_DEPTH);
      continue;
    }
    int flag = 0;
    const U piv = warp_select_pivot<C>(reinterpret_cast<const U *>(P->keys[db]), !P->raw[db],
                                       cb[c], cl[c], P->dran, P->mitigation, scratch, &flag);
    uint32_t kind = KIND_PARTITION;
    if (P->fast_paths)
      kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    warp_append_level<C, PAY>(P, nxt, cb[c], cb[c] + cl[c], db, (u64)piv, kind, depth, 0);
  }
}

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) schedule_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  U *scratch = reinterpret_cast<U *>(smem_raw) + (threadIdx.x >> 5) * (kMaxSample + 1);
  Ctl *ctl = P->ctl;
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u), nxt = cur ^ 1;
  const uint32_t nseg = ctl->cur_nseg;
  {
    u64 *lbn = P->lookback[nxt];
    const uint32_t cap = P->tile_cap;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < cap; i += gridDim.x * kThreads)
      lbn[i] = 0ull;
  }
  const uint32_t nwarps = gridDim.x * (kThreads / 32);
  for (uint32_t sid = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); sid < nseg;
       sid += nwarps)
    schedule_segment<C, PAY>(P, cur, nxt, sid, scratch);
  __syncthreads();
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

// ---------------------------------------------------------------------------

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) init_kernel(Params pv, Params *P) {
  typedef typename C::U U;
  __shared__ __align__(16) U s_scr[kMaxSample + 1];
  Ctl *ctl = pv.ctl;
  if (threadIdx.x == 0) {
    *P = pv;
    u64 *z = reinterpret_cast<u64 *>(ctl);
    for (unsigned i = 0; i < sizeof(Ctl) / sizeof(u64); ++i) z[i] = 0ull;
  }
  for (uint32_t i = threadIdx.x; i < pv.tile_cap; i += kThreads) pv.lookback[0][i] = 0ull;
  __syncthreads();
  const long long n = pv.n;
  const long long T = Geo<C, PAY>::TILE;
  bool more = false;
  if (pv.single_stage || n > pv.small_t) {
    u64 piv = pv.given_pivot;
    uint32_t kind = KIND_PARTITION, buf = pv.single_stage ? 1u : 0u;
    if (!pv.single_stage) {
      __shared__ U s_piv;
      __shared__ int s_flag;
      cta_select_pivot<C>(reinterpret_cast<const U *>(pv.keys[0]), !pv.raw[0], 0, n, pv.dran,
                          pv.mitigation, s_scr, &s_piv, &s_flag);
      piv = (u64)s_piv;
      if (pv.fast_paths)
        kind = s_flag > 0 ? KIND_VERIFY_ASC : (s_flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    }
    const uint32_t ntiles = (uint32_t)((n - 1) / T + 1);
    if (threadIdx.x == 0) {
      Seg s;
      s.begin = 0; s.end = n; s.pivot = piv;
      s.tile_base = 0; s.ntiles = ntiles;
      s.buf = buf; s.kind = kind; s.depth = 1; s.noverify = 0; s.done = 0; s.fail = 0;
      pv.segs[0][0] = s;
      ctl->cur_nseg = 1;
      ctl->cur_ntiles = ntiles;
    }
    for (uint32_t i = threadIdx.x; i < ntiles; i += kThreads) pv.tilemap[0][i] = 0;
    more = true;
  } else if (n > 1) {
    if (threadIdx.x == 0) {
      append_small(&pv, 0, n, 0);
      ctl->max_depth = 1;
    }
  }
  if (threadIdx.x == 0 && pv.use_cond) cudaGraphSetConditional(pv.cond, more ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// On-chip sort of segments <= small_t: bitonic sorting network in shared
// memory (records sort (key, local index) pairs so equal keys keep distinct
// payloads; padding sorts last).  Output always lands in buffer 0.

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) small_sort_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  U *s_k = reinterpret_cast<U *>(smem_raw);
  uint32_t *s_p = reinterpret_cast<uint32_t *>(s_k + kSmallT);
  uint16_t *s_i = reinterpret_cast<uint16_t *>(s_p + (PAY ? kSmallT : 0));
  __shared__ uint32_t s_ticket;
  Ctl *ctl = P->ctl;
  const uint32_t count = ctl->small_count < P->small_cap ? ctl->small_count : P->small_cap;
  U *dst = reinterpret_cast<U *>(P->keys[0]);
  const bool dst_raw = P->raw[0] != 0;
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->small_ticket, 1u);
    __syncthreads();
    const uint32_t t = s_ticket;
    __syncthreads();
    if (t >= count) break;
    const SmallSeg sm = P->smalls[t];
    const U *src = reinterpret_cast<const U *>(P->keys[sm.buf]);
    const bool raw = P->raw[sm.buf] != 0;
    const int len = sm.len;
    int P2 = 1;
    while (P2 < len) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += kThreads) {
      U v = KeyMax<U>::v;
      if (i < len) {
        v = src[sm.begin + i];
        if (raw) v = C::enc(v);
        if (PAY) s_p[i] = P->pay[sm.buf][sm.begin + i];
      }
      s_k[i] = v;
      if (PAY) s_i[i] = (uint16_t)i;
    }
    __syncthreads();
    for (int kk = 2; kk <= P2; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < (P2 >> 1); i += kThreads) {
          const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
          const int hi = lo + j;
          const bool up = (lo & kk) == 0;
          const U a = s_k[lo], b = s_k[hi];
          if (PAY) {
            const uint16_t ia = s_i[lo], ib = s_i[hi];
            const bool gt = (a > b) || (a == b && ia > ib);
            if (gt == up) {
              s_k[lo] = b; s_k[hi] = a;
              s_i[lo] = ib; s_i[hi] = ia;
            }
          } else {
            if ((a > b) == up) {
              s_k[lo] = b;
              s_k[hi] = a;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < len; i += kThreads) {
      U v = s_k[i];
      if (dst_raw) v = C::dec(v);
      dst[sm.begin + i] = v;
      if (PAY) P->pay[0][sm.begin + i] = s_p[s_i[i]];
    }
    if (threadIdx.x == 0) {
      atomicAdd(&ctl->small_elements, (u64)len);
      atomicAdd(&ctl->bytes_small, 2ull * (u64)len * (sizeof(U) + (PAY ? 4 : 0)));
      atomicAdd(&ctl->writes0, (u64)len);
    }
    __syncthreads();
  }
}

// Retire finished runs into buffer 0, chunk by chunk.
template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) retire_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  __shared__ uint32_t s_ticket;
  Ctl *ctl = P->ctl;
  const uint32_t total = (uint32_t)ctl->run_packed;
  U *k0 = reinterpret_cast<U *>(P->keys[0]);
  uint32_t *p0 = PAY ? P->pay[0] : nullptr;
  const bool raw0 = P->raw[0] != 0;
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->run_ticket, 1u);
    __syncthreads();
    const uint32_t c = s_ticket;
    __syncthreads();
    if (c >= total || c >= P->chunk_cap) break;
    const Run r = P->runs[P->chunkmap[c]];
    const long long cc = (long long)(c - r.chunk_base);
    const long long lo = cc * kRunChunk;
    if (r.kind == RUN_EQ) {
      const long long hi = (lo + kRunChunk) < r.len ? (lo + kRunChunk) : r.len;
      const U v = raw0 ? C::dec((U)r.pivot) : (U)r.pivot;
      for (long long i = lo + threadIdx.x; i < hi; i += kThreads) {
        k0[r.begin + i] = v;
        if (PAY) p0[r.begin + i] = P->side_pay[r.src + i];
      }
    } else if (r.kind == RUN_SORTED) {
      const long long hi = (lo + kRunChunk) < r.len ? (lo + kRunChunk) : r.len;
      const U *kb = reinterpret_cast<const U *>(P->keys[r.buf]);
      const bool rawb = P->raw[r.buf] != 0;
      for (long long i = lo + threadIdx.x; i < hi; i += kThreads) {
        U v = kb[r.begin + i];
        if (rawb != raw0) v = rawb ? C::enc(v) : C::dec(v);
        k0[r.begin + i] = v;
        if (PAY) p0[r.begin + i] = P->pay[r.buf][r.begin + i];
      }
    } else {  // RUN_REVERSED
      if (r.buf == 0) {
        const long long half = r.len >> 1;
        const long long hi = (lo + kRunChunk) < half ? (lo + kRunChunk) : half;
        for (long long i = lo + threadIdx.x; i < hi; i += kThreads) {
          const long long a = r.begin + i, b = r.begin + r.len - 1 - i;
          const U x = k0[a], y = k0[b];
          k0[a] = y;
          k0[b] = x;
          if (PAY) {
            const uint32_t px = p0[a], py = p0[b];
            p0[a] = py;
            p0[b] = px;
          }
        }
      } else {
        const long long hi = (lo + kRunChunk) < r.len ? (lo + kRunChunk) : r.len;
        const U *kb = reinterpret_cast<const U *>(P->keys[r.buf]);
        const bool rawb = P->raw[r.buf] != 0;
        for (long long i = lo + threadIdx.x; i < hi; i += kThreads) {
          const long long s = r.begin + r.len - 1 - i;
          U v = kb[s];
          if (rawb != raw0) v = rawb ? C::enc(v) : C::dec(v);
          k0[r.begin + i] = v;
          if (PAY) p0[r.begin + i] = P->pay[r.buf][s];
        }
      }
    }
  }
}

// Pivot-sampling entry for tsq_select_pivot: one CTA over keys[0..n) of
// buffer 0; writes (pivot, flag) into the control block.
template <class C>
__global__ void __launch_bounds__(kThreads) select_pivot_kernel(Params pv) {
  typedef typename C::U U;
  __shared__ __align__(16) U s_scr[kMaxSample + 1];
  __shared__ U s_piv;
  __shared__ int s_flag;
  cta_select_pivot<C>(reinterpret_cast<const U *>(pv.keys[0]), !pv.raw[0], 0, pv.n, pv.dran,
                      pv.mitigation, s_scr, &s_piv, &s_flag);
  if (threadIdx.x == 0) {
    pv.ctl->stage_lt = (u64)(C::dec(s_piv));
    pv.ctl->stage_gt = (u64)(long long)s_flag;
  }
}

}  // namespace tsq
