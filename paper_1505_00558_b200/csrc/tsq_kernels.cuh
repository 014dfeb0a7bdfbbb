// tsq_kernels.cuh -- the four kernels of the B200 three-way partition sort.
//
//   init_kernel        root stage: pivot sampling of [0, n) and the level-0
//                      queue (Sorter.sort_with_stats -> _range entry,
//                      core.py:1599-1607)
//   level_kernel       one recursion level over every live segment: the
//                      multi-block three-way partition (the _run_machine
//                      stage, core.py:198-984) with decoupled look-back,
//                      the sorted / reversed verification fast paths
//                      (core.py:1678-1698), and, in the CTA that finishes a
//                      segment, the next level's bookkeeping: ==p run
//                      retirement, child pivot sampling (pivot.py:205-248)
//                      and queue appends (core.py:1711-1728)
//   small_sort_kernel  on-chip sorting network for segments <= kSmallT
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

template <class C, bool PAY>
struct Geo {
  typedef typename C::U U;
  static constexpr int VN = Vec<U>::N;     // keys per 16-byte vector
  static constexpr int VPT = 4;            // vectors per thread per tile
  static constexpr int IPT = VN * VPT;     // keys per thread per tile
  static constexpr int TILE = kThreads * IPT;
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

struct Shared {
  uint32_t wcnt[kThreads / 32][3];
  u64 excl;
  uint32_t ticket, last, bc0, bc1;
  u64 piv;
  int flag;
};

// ---------------------------------------------------------------------------
// Queue appends (cooperative: every thread of the CTA calls).

template <class C, bool PAY>
__device__ void append_level(const Params *P, Shared &sh, int nxt, long long begin,
                             long long end, uint32_t buf, u64 pivot, uint32_t kind,
                             uint32_t depth, uint32_t noverify) {
  const long long T = Geo<C, PAY>::TILE;
  const uint32_t ntiles = (uint32_t)((end - 1) / T - begin / T + 1);
  if (threadIdx.x == 0) {
    Ctl *ctl = P->ctl;
    u64 old = atomicAdd(&ctl->next_packed, (1ull << 32) | ntiles);
    uint32_t slot = (uint32_t)(old >> 32), tbase = (uint32_t)old;
    bool ok = slot < P->seg_cap && (u64)tbase + ntiles <= P->tile_cap;
    if (ok) {
      Seg s;
      s.begin = begin; s.end = end; s.pivot = pivot;
      s.tile_base = tbase; s.ntiles = ntiles;
      s.buf = buf; s.kind = kind; s.depth = depth; s.noverify = noverify;
      s.done = 0; s.fail = 0;
      P->segs[nxt][slot] = s;
    } else {
      atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
    }
    sh.bc0 = ok ? slot : 0xffffffffu;
    sh.bc1 = tbase;
  }
  __syncthreads();
  const uint32_t slot = sh.bc0, tbase = sh.bc1;
  if (slot != 0xffffffffu) {
    uint32_t *tm = P->tilemap[nxt] + tbase;
    for (uint32_t i = threadIdx.x; i < ntiles; i += kThreads) tm[i] = slot;
  }
  __syncthreads();
}

__device__ void append_run(const Params *P, Shared &sh, uint32_t kind, long long begin,
                           long long len, uint32_t buf, u64 pivot, long long src) {
  uint32_t nchunks;
  if (kind == RUN_REVERSED && buf == 0)
    nchunks = (uint32_t)(((len >> 1) + kRunChunk - 1) / kRunChunk);
  else
    nchunks = (uint32_t)((len + kRunChunk - 1) / kRunChunk);
  if (nchunks == 0) return;  // uniform across the CTA
  if (threadIdx.x == 0) {
    Ctl *ctl = P->ctl;
    u64 old = atomicAdd(&ctl->run_packed, (1ull << 32) | nchunks);
    uint32_t slot = (uint32_t)(old >> 32), cbase = (uint32_t)old;
    bool ok = slot < P->run_cap && (u64)cbase + nchunks <= P->chunk_cap;
    if (ok) {
      Run r;
      r.begin = begin; r.len = len; r.pivot = pivot; r.src = src;
      r.kind = kind; r.buf = buf; r.chunk_base = cbase; r.nchunks = nchunks;
      P->runs[slot] = r;
    } else {
      atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
    }
    sh.bc0 = ok ? slot : 0xffffffffu;
    sh.bc1 = cbase;
  }
  __syncthreads();
  const uint32_t slot = sh.bc0, cbase = sh.bc1;
  if (slot != 0xffffffffu) {
    uint32_t *cm = P->chunkmap + cbase;
    for (uint32_t i = threadIdx.x; i < nchunks; i += kThreads) cm[i] = slot;
  }
  __syncthreads();
}

__device__ __forceinline__ void append_small(const Params *P, long long begin, long long len,
                                             uint32_t buf) {
  // thread 0 only
  Ctl *ctl = P->ctl;
  uint32_t slot = atomicAdd(&ctl->small_count, 1u);
  if (slot < P->small_cap) {
    SmallSeg s;
    s.begin = begin; s.len = (int)len; s.buf = (int)buf;
    P->smalls[slot] = s;
  } else {
    atomicOr(&ctl->error, (uint32_t)ERR_CAPACITY);
  }
}

// choose the next stage for a segment of > kSmallT keys living in `buf`
template <class C, bool PAY>
__device__ void schedule_child(const Params *P, Shared &sh, typename C::U *scratch, int nxt,
                               long long begin, long long len, uint32_t buf, uint32_t depth) {
  typedef typename C::U U;
  if ((int)depth > P->max_depth) {
    if (threadIdx.x == 0) atomicOr(&P->ctl->error, (uint32_t)ERR_DEPTH);
    __syncthreads();
    return;
  }
  U piv;
  int flag;
  {
    __shared__ U s_piv;
    __shared__ int s_flag;
    cta_select_pivot<C>(reinterpret_cast<const U *>(P->keys[buf]), !P->raw[buf], begin, len,
                        P->dran, P->mitigation, scratch, &s_piv, &s_flag);
    piv = s_piv;
    flag = s_flag;
    __syncthreads();
  }
  uint32_t kind = KIND_PARTITION;
  if (P->fast_paths) kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
  append_level<C, PAY>(P, sh, nxt, begin, begin + len, buf, (u64)piv, kind, depth, 0);
}

// ---------------------------------------------------------------------------
// One partition tile: classify every key against the pivot (ballot/popc
// ranks), publish the tile's (<, >) counts, find its offsets by decoupled
// look-back over the segment's earlier tiles, then write the < keys from the
// segment front and the > keys from the segment back.

template <class C, bool PAY>
__device__ __forceinline__ void partition_tile(const Params *P, Shared &sh, const Seg &sg,
                                               uint32_t t, uint32_t k, int cur,
                                               typename C::U *s_keys, uint32_t *s_pay) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sb = (int)sg.buf, db = sb ^ 1;
  const U *src = reinterpret_cast<const U *>(P->keys[sb]);
  U *dst = reinterpret_cast<U *>(P->keys[db]);
  const bool src_raw = P->raw[sb] != 0, dst_raw = P->raw[db] != 0;
  const bool vec_ok = P->aligned[sb] != 0;
  const long long tstart = (sg.begin / G::TILE + k) * (long long)G::TILE;
  const long long lo = tstart > sg.begin ? tstart : sg.begin;
  const long long hi = (tstart + G::TILE) < sg.end ? (tstart + G::TILE) : sg.end;
  const U piv = (U)sg.pivot;

  U key[G::IPT];
  uint32_t pay[PAY ? G::IPT : 1];
  uint32_t cls[G::IPT];
#pragma unroll
  for (int v = 0; v < G::VPT; ++v) {
    const long long e0 = tstart + (long long)(v * kThreads + threadIdx.x) * G::VN;
    if (vec_ok && e0 >= lo && e0 + G::VN <= hi) {
      typename Vec<U>::K kv = __ldcs(reinterpret_cast<const typename Vec<U>::K *>(src + e0));
      unpack(kv, key + v * G::VN);
      if (PAY) {
        typename Vec<U>::P pv = __ldcs(reinterpret_cast<const typename Vec<U>::P *>(P->pay[sb] + e0));
        unpack(pv, pay + v * G::VN);
      }
#pragma unroll
      for (int q = 0; q < G::VN; ++q) cls[v * G::VN + q] = 0;
    } else {
#pragma unroll
      for (int q = 0; q < G::VN; ++q) {
        const long long idx = e0 + q;
        const bool ok = idx >= lo && idx < hi;
        key[v * G::VN + q] = ok ? src[idx] : (U)0;
        if (PAY) pay[v * G::VN + q] = ok ? P->pay[sb][idx] : 0u;
        cls[v * G::VN + q] = ok ? 0u : 3u;
      }
    }
  }
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
    sh.wcnt[warp][0] = lt_run;
    sh.wcnt[warp][1] = eq_run;
    sh.wcnt[warp][2] = gt_run;
  }
  __syncthreads();
  uint32_t w_lt = 0, w_eq = 0, w_gt = 0, t_lt = 0, t_eq = 0, t_gt = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const uint32_t a = sh.wcnt[w][0], b = sh.wcnt[w][1], c = sh.wcnt[w][2];
    if (w < warp) { w_lt += a; w_eq += b; w_gt += c; }
    t_lt += a; t_eq += b; t_gt += c;
  }
  const u64 agg = ((u64)t_lt << 31) | (u64)t_gt;
  u64 *lb = P->lookback[cur];
  if (threadIdx.x == 0) st_volatile(&lb[t], (k == 0 ? kFlagInc : kFlagAgg) | agg);

  // stage the tile in shared memory as [< | > | == (payload only)]
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
    if (c != 1u) s_keys[pos] = key[i];
    if (PAY) s_pay[pos] = pay[i];
  }

  // decoupled look-back (warp 0), bounded by the segment's first tile
  if (warp == 0) {
    u64 excl = 0;
    if (k > 0) {
      long long base = (long long)t - 1;
      const long long stop = (long long)sg.tile_base;
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
      if (lane == 0) st_volatile(&lb[t], kFlagInc | (excl + agg));
    }
    if (lane == 0) sh.excl = excl;
  }
  __syncthreads();

  const u64 ex = sh.excl;
  const long long ex_lt = (long long)(ex >> 31), ex_gt = (long long)(ex & 0x7fffffffull);
  uint32_t *dpay = PAY ? P->pay[db] : nullptr;
  for (uint32_t i = threadIdx.x; i < nlg; i += kThreads) {
    const long long d = (i < t_lt) ? (sg.begin + ex_lt + i)
                                   : (sg.end - 1 - (ex_gt + (long long)(i - t_lt)));
    U v = s_keys[i];
    if (dst_raw) v = C::dec(v);
    dst[d] = v;
    if (PAY) dpay[d] = s_pay[i];
  }
  if (PAY) {
    const long long ex_eq = (lo - sg.begin) - ex_lt - ex_gt;
    uint32_t *side = P->side_pay + sg.begin + ex_eq;
    for (uint32_t i = threadIdx.x; i < t_eq; i += kThreads) side[i] = s_pay[nlg + i];
  }
}

// One verification tile of a segment whose samples looked sorted (+1) or
// reversed (-1): checks every adjacent pair including the one that crosses
// into the next tile.  Any violation marks the segment failed; later tiles
// of a failed segment skip their reads.
template <class C, bool PAY>
__device__ __forceinline__ void verify_tile(const Params *P, Shared &sh, Seg *sgp, const Seg &sg,
                                            uint32_t k, typename C::U *s_keys) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  if (threadIdx.x == 0) sh.bc0 = ld_volatile32(&sgp->fail);
  __syncthreads();
  if (sh.bc0) return;
  const int sb = (int)sg.buf;
  const U *src = reinterpret_cast<const U *>(P->keys[sb]);
  const bool raw = P->raw[sb] != 0;
  const long long tstart = (sg.begin / G::TILE + k) * (long long)G::TILE;
  const long long lo = tstart > sg.begin ? tstart : sg.begin;
  const long long hi = (tstart + G::TILE) < sg.end ? (tstart + G::TILE) : sg.end;
  const int cnt = (int)(hi - lo) + (hi < sg.end ? 1 : 0);
  for (int i = threadIdx.x; i < cnt; i += kThreads) {
    U v = src[lo + i];
    s_keys[i] = raw ? C::enc(v) : v;
  }
  __syncthreads();
  const bool asc = sg.kind == KIND_VERIFY_ASC;
  bool ok = true;
  for (int i = threadIdx.x; i + 1 < cnt; i += kThreads) {
    const U a = s_keys[i], b = s_keys[i + 1];
    ok &= asc ? (a <= b) : (a >= b);
  }
  ok = __syncthreads_and(ok);
  if (!ok && threadIdx.x == 0) atomicOr(&sgp->fail, 1u);
}

// The CTA that completes a segment's last tile runs the rest of the stage:
// ==p retirement, children scheduling (smaller / larger order is irrelevant
// on the device: both children are queued for the next level).
template <class C, bool PAY>
__device__ void finalize_segment(const Params *P, Shared &sh, Seg *sgp, int cur, int nxt,
                                 typename C::U *scratch) {
  typedef typename C::U U;
  Ctl *ctl = P->ctl;
  const Seg sg = *sgp;
  const long long len = sg.end - sg.begin;
  const int key_bytes = (int)sizeof(U);
  if (sg.kind != KIND_PARTITION) {
    const bool failed = ld_volatile32(&sgp->fail) != 0;
    if (!failed) {
      const uint32_t rk = sg.kind == KIND_VERIFY_ASC ? RUN_SORTED : RUN_REVERSED;
      if (threadIdx.x == 0) {
        atomicAdd(&ctl->stages, 1ull);
        atomicAdd(rk == RUN_SORTED ? &ctl->sorted_bypass : &ctl->reversed_bypass, 1ull);
        atomicMax(&ctl->max_depth, (u64)sg.depth);
        u64 moved = (rk == RUN_SORTED && sg.buf == 0) ? 0ull : 2ull * (u64)len;
        atomicAdd(&ctl->bytes_retire, moved * (u64)(key_bytes + (PAY ? 4 : 0)));
        if (moved) atomicAdd(&ctl->writes0, (u64)len);
        atomicAdd(&ctl->bytes_partition, (u64)len * key_bytes);  // the verify read
      }
      if (!(rk == RUN_SORTED && sg.buf == 0))
        append_run(P, sh, rk, sg.begin, len, sg.buf, 0ull, sg.begin);
    } else {
      if (threadIdx.x == 0) atomicAdd(&ctl->verify_fallbacks, 1ull);
      append_level<C, PAY>(P, sh, nxt, sg.begin, sg.end, sg.buf, sg.pivot, KIND_PARTITION,
                           sg.depth, 1);
    }
    return;
  }
  const u64 inc = ld_volatile(&P->lookback[cur][sg.tile_base + sg.ntiles - 1]);
  const long long lt = (long long)((inc >> 31) & 0x7fffffffull);
  const long long gt = (long long)(inc & 0x7fffffffull);
  const long long eq = len - lt - gt;
  if (threadIdx.x == 0) {
    atomicAdd(&ctl->stages, 1ull);
    atomicAdd(&ctl->partitioned_elements, (u64)len);
    atomicMax(&ctl->max_depth, (u64)sg.depth);
    u64 bytes = (u64)len * key_bytes + (u64)(lt + gt) * key_bytes;
    if (PAY) bytes += (u64)len * 8ull;
    atomicAdd(&ctl->bytes_partition, bytes);
    atomicAdd(sg.buf == 0 ? &ctl->writes1 : &ctl->writes0, (u64)(lt + gt));
    if (PAY) atomicAdd(&ctl->writes1, (u64)eq);
    if (eq > 0) {
      atomicAdd(&ctl->eq_runs, 1ull);
      atomicAdd(&ctl->eq_elements, (u64)eq);
      atomicAdd(&ctl->bytes_retire, (u64)eq * (key_bytes + (PAY ? 8 : 0)));
      atomicAdd(&ctl->writes0, (u64)eq);
    }
    if (P->single_stage) {
      ctl->stage_lt = (u64)lt;
      ctl->stage_gt = (u64)gt;
    }
  }
  if (eq > 0) {
    if (PAY) {
      // Records: the ==p payloads were staged at side_pay[begin ...], a
      // range the children reuse at the next level, so they move to their
      // final place now.  Nothing else touches [begin+lt, end-gt) of
      // buffer 0 during this level: the segment's reads are complete and
      // its < / > writes land outside the ==p block.
      const uint32_t *side = P->side_pay + sg.begin;
      uint32_t *p0 = P->pay[0] + sg.begin + lt;
      U *k0 = reinterpret_cast<U *>(P->keys[0]) + sg.begin + lt;
      const U v = P->raw[0] ? C::dec((U)sg.pivot) : (U)sg.pivot;
      for (long long i = threadIdx.x; i < eq; i += kThreads) {
        p0[i] = __ldcg(side + i);
        k0[i] = v;
      }
    } else {
      append_run(P, sh, RUN_EQ, sg.begin + lt, eq, sg.buf, sg.pivot, sg.begin);
    }
  }
  if (P->single_stage) return;
  const uint32_t db = sg.buf ^ 1u;
  const long long cb[2] = {sg.begin, sg.end - gt};
  const long long cl[2] = {lt, gt};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (cl[c] <= 0) continue;
    if (cl[c] <= P->small_t) {
      if (threadIdx.x == 0) {
        append_small(P, cb[c], cl[c], db);
        atomicMax(&ctl->max_depth, (u64)sg.depth + 1);
      }
    } else {
      schedule_child<C, PAY>(P, sh, scratch, nxt, cb[c], cl[c], db, sg.depth + 1);
    }
  }
}

// ---------------------------------------------------------------------------

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) init_kernel(Params pv, Params *P) {
  typedef typename C::U U;
  __shared__ __align__(16) U s_scr[kMaxSample + 1];
  __shared__ Shared sh;
  Ctl *ctl = pv.ctl;
  if (threadIdx.x == 0) {
    *P = pv;
    u64 *z = reinterpret_cast<u64 *>(ctl);
    for (unsigned i = 0; i < sizeof(Ctl) / sizeof(u64); ++i) z[i] = 0ull;
  }
  for (uint32_t i = threadIdx.x; i < pv.tile_cap; i += kThreads) pv.lookback[0][i] = 0ull;
  __syncthreads();
  const long long n = pv.n;
  bool more = false;
  if (pv.single_stage) {
    // tsq_partition_segment: one given-pivot stage over buffer 1
    if (threadIdx.x == 0) {
      const long long T = Geo<C, PAY>::TILE;
      Seg s;
      s.begin = 0; s.end = n; s.pivot = pv.given_pivot;
      s.tile_base = 0; s.ntiles = (uint32_t)((n - 1) / T + 1);
      s.buf = 1; s.kind = KIND_PARTITION; s.depth = 1; s.noverify = 1; s.done = 0; s.fail = 0;
      pv.segs[0][0] = s;
      ctl->cur_nseg = 1;
      ctl->cur_ntiles = s.ntiles;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < ctl->cur_ntiles; i += kThreads) pv.tilemap[0][i] = 0;
    more = true;
  } else if (n > pv.small_t) {
    U piv;
    int flag;
    {
      __shared__ U s_piv;
      __shared__ int s_flag;
      cta_select_pivot<C>(reinterpret_cast<const U *>(pv.keys[0]), !pv.raw[0], 0, n, pv.dran,
                          pv.mitigation, s_scr, &s_piv, &s_flag);
      piv = s_piv;
      flag = s_flag;
    }
    uint32_t kind = KIND_PARTITION;
    if (pv.fast_paths) kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    const long long T = Geo<C, PAY>::TILE;
    const uint32_t ntiles = (uint32_t)((n - 1) / T + 1);
    if (threadIdx.x == 0) {
      Seg s;
      s.begin = 0; s.end = n; s.pivot = (u64)piv;
      s.tile_base = 0; s.ntiles = ntiles;
      s.buf = 0; s.kind = kind; s.depth = 1; s.noverify = 0; s.done = 0; s.fail = 0;
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

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) level_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  typedef Geo<C, PAY> G;
  __shared__ __align__(16) U s_keys[G::TILE + 8];
  __shared__ __align__(16) uint32_t s_pay[PAY ? G::TILE : 1];
  __shared__ Shared sh;
  Ctl *ctl = P->ctl;
  const uint32_t level = ctl->level;
  const int cur = (int)(level & 1u), nxt = cur ^ 1;
  const uint32_t ntiles = ctl->cur_ntiles;
  {
    u64 *lbn = P->lookback[nxt];
    const uint32_t cap = P->tile_cap;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < cap; i += gridDim.x * kThreads)
      lbn[i] = 0ull;
  }
  for (;;) {
    if (threadIdx.x == 0) sh.ticket = atomicAdd(&ctl->tile_ticket, 1u);
    __syncthreads();
    const uint32_t t = sh.ticket;
    if (t >= ntiles) break;
    const uint32_t sid = P->tilemap[cur][t];
    Seg *sgp = &P->segs[cur][sid];
    Seg sg;
    sg.begin = sgp->begin; sg.end = sgp->end; sg.pivot = sgp->pivot;
    sg.tile_base = sgp->tile_base; sg.ntiles = sgp->ntiles;
    sg.buf = sgp->buf; sg.kind = sgp->kind; sg.depth = sgp->depth; sg.noverify = sgp->noverify;
    const uint32_t k = t - sg.tile_base;
    if (sg.kind == KIND_PARTITION)
      partition_tile<C, PAY>(P, sh, sg, t, k, cur, s_keys, s_pay);
    else
      verify_tile<C, PAY>(P, sh, sgp, sg, k, s_keys);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t old = atomicAdd(&sgp->done, 1u);
      sh.last = (old == sg.ntiles - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (sh.last) {
      __threadfence();
      finalize_segment<C, PAY>(P, sh, sgp, cur, nxt, s_keys);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t d = atomicAdd(&ctl->ctas_done, 1u);
    if (d == gridDim.x - 1) {
      __threadfence();
      const u64 packed = atomicExch(&ctl->next_packed, 0ull);
      const uint32_t nseg = (uint32_t)(packed >> 32), nt = (uint32_t)packed;
      ctl->cur_nseg = nseg;
      ctl->cur_ntiles = nt;
      ctl->tile_ticket = 0;
      ctl->ctas_done = 0;
      ctl->level = level + 1;
      ctl->levels += 1;
      bool more = nseg > 0;
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
// On-chip sort of segments <= kSmallT: bitonic sorting network in shared
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
          const int lo = ((i / j) * 2 * j) + (i % j);
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
