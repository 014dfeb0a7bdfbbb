// tsq_kernels.cuh -- the kernels of the B200 three-way partition sort.
//
//   init_kernel        root stage: pivot sampling of [0, n) and the level-0
//                      queue (Sorter.sort_with_stats -> _range entry,
//                      core.py:1599-1607)
//   partition_kernel   one recursion level over every live segment: the
//                      multi-block three-way partition (the stage that
//                      _run_machine performs, core.py:198-984).  Persistent,
//                      warp-specialised (tsq_partition.cuh): a producer warp
//                      streams 24 KB tiles into a 4- or 6-deep shared-memory ring with
//                      cp.async.bulk (TMA engine) + mbarriers; counter warps
//                      count each consumer thread's < / > keys; look-back
//                      warps turn tile counts into output offsets; consumer
//                      warps restage each tile in output order and write the
//                      < run from the segment front and the > run from the
//                      back.  Segments whose samples looked sorted/reversed
//                      are verified instead (core.py:1678-1698 fast paths).
//   schedule_kernel    one warp (or CTA) per child of each segment of the
//                      level: retires the ==p run, samples the children's
//                      pivots (pivot.py:205-248) and queues them for the next
//                      level or the on-chip sort (core.py:1711-1728); the last
//                      CTA advances the level and sets the CUDA-graph loop
//                      condition
//   small_sort_kernel  on-chip sort of segments <= small_t (insertion_sort's
//                      role, smallsort.py:12-47): LSD radix sort over the
//                      segment's key range
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
constexpr int kProducerWarp = kConsumerWarps;     // warp 8: tile claims + bulk loads
constexpr int kLookbackWarp = kConsumerWarps + 1; // warps 9, 10: decoupled look-back
#ifndef TSQ_LB_WARPS
#define TSQ_LB_WARPS 2
#endif
constexpr int kLookbackWarps = TSQ_LB_WARPS;      // alternate stages between them
constexpr int kCounterWarp = kLookbackWarp + kLookbackWarps;  // warps 11-14: counts
constexpr int kCounterWarps = 4;
constexpr int kPartThreads = kConsumers + 32 * (1 + kLookbackWarps + kCounterWarps);
// stage ring depth: records 6 (24 KB tiles), keys only TSQ_STAGES (see Geo)
#ifndef TSQ_STAGES
#define TSQ_STAGES 4
#endif
constexpr int kStages = 8;                        // upper bound on any ring depth
constexpr int kAlign = 4;                         // bulk-copy element alignment
constexpr int kOutPad = 16;                       // alignment slack of a restaged tile
constexpr uint32_t kDone = 0xffffffffu;

template <class C, bool PAY>
struct Geo {
  typedef typename C::U U;
  static constexpr int VN = Vec<U>::N;     // keys per 16-byte vector
#ifndef TSQ_VPT
#define TSQ_VPT 6
#endif
  // Tile geometry (measured on B200, scripts/variants.py): a tile costs a
  // fixed share of pipeline work besides its bytes, so keys-only tiles are
  // 24 KB -- 6 vectors per thread (6144 int32 / 3072 64-bit keys) in a
  // 4-deep ring, 2 CTAs/SM -- like the 64-bit-key records' 2048-key tiles
  // (16 KB keys + 8 KB payloads, 4-deep ring).  16 KB int32 tiles ran the
  // pass 9.5 % slower, 32 KB tiles need a 3-deep ring and lose more;
  // 64-bit records 5 % slower with the 6-deep ring (1 CTA/SM); 32-bit
  // records (32 KB stages) are best with 6 (8 % faster than 4).  The
  // counters' 10-bit lane-scan fields hold a warp slice of up to 1023 keys
  // (32 * IPT).
  static constexpr int VPT = PAY ? 4 : TSQ_VPT;
  static constexpr int STAGES = PAY ? (sizeof(U) == 8 ? 4 : 6) : TSQ_STAGES;
  static constexpr int IPT = VN * VPT;     // keys per thread per tile
  static constexpr int TILE = kConsumers * IPT;
  // a stage holds a tile as loaded and then, restaged in place, its output
  // runs, each aligned like its destination (<= 3 slots of padding per run)
  static constexpr int SLOT = TILE + kOutPad;
  static constexpr size_t KB = sizeof(U);
  static constexpr size_t STAGE_BYTES = (size_t)SLOT * (KB + (PAY ? 4 : 0));
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES;
  static_assert(STAGES <= kStages, "stage ring deeper than the barrier arrays");
  static_assert(32 * IPT <= 1023, "counter lane-scan fields are 10 bits");
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

// Tile descriptor handed from the producer warp to the counter and consumer
// warps; `agg` (the tile's (<, >) counts) is filled in by the consumers and
// `excl` (its exclusive prefix in its segment) by the look-back warp.
struct StageMeta {
  long long tstart, lo, hi, begin, end;
  u64 pivot, agg, excl;
  uint32_t t, k, kind, buf, tile_base, sid, skip, has_next;
  uint32_t eq_excl;  // records, atomic placement: this tile's first == side slot
};

}  // namespace tsq

#include "tsq_partition.cuh"
#include "tsq_small.cuh"
#include "tsq_schedule.cuh"
#include "tsq_gather.cuh"

namespace tsq {

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
  if (pv.reproducible)
    for (uint32_t i = threadIdx.x; i < pv.tile_cap; i += kThreads) pv.lookback[0][i] = 0ull;
  __syncthreads();
  const long long n = pv.n;
  const long long T = Geo<C, PAY>::TILE;
  bool more = false;
  if (pv.single_stage || n > pv.small_t) {
    u64 piv = pv.given_pivot;
    uint32_t kind = KIND_PARTITION, buf = pv.single_stage ? 1u : 0u;
    if (!pv.single_stage) {
      // the register bitonic network of the schedule kernel's CTA mode
      __shared__ uint32_t s_bc[2];
      int flag = 0;
      piv = (u64)cta_select_pivot_fast<C>(reinterpret_cast<const U *>(pv.keys[0]), !pv.raw[0], 0,
                                          n, pv.dran, pv.mitigation, s_scr, s_bc, &flag);
      if (pv.fast_paths)
        kind = flag > 0 ? KIND_VERIFY_ASC : (flag < 0 ? KIND_VERIFY_DESC : KIND_PARTITION);
    }
    const uint32_t ntiles = (uint32_t)((n - 1) / T + 1);
    if (threadIdx.x == 0) {
      Seg s;
      s.begin = 0; s.end = n; s.pivot = piv;
      s.klo = 0; s.khi = (u64)KeyMax<U>::v;  // the whole (encoded) key space
      s.tile_base = 0; s.ntiles = ntiles;
      s.buf = buf; s.kind = kind; s.depth = 1; s.noverify = 0; s.eq_fill = 0; s.fail = 0;
      s.fill = 0;
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

// End of a drain round (after the on-chip sort and retire kernels have
// consumed the queues): reset the queues, and resume the level loop if
// segments remain (a flush paused it) or end the sort.
__global__ void drain_kernel(const Params *__restrict__ P) {
  Ctl *ctl = P->ctl;
  if (threadIdx.x != 0) return;
  for (int c = 0; c < kSmallClasses; ++c) {
    ctl->small_segs_done += (u64)ctl->sq_count[c];
    ctl->sq_count[c] = 0;
    ctl->sq_ticket[c] = 0;
  }
  ctl->run_packed = 0;
  ctl->run_ticket = 0;
  const bool more = ctl->cur_nseg > 0 && ctl->error == 0;
  if (more) ctl->flushes += 1;
  ctl->flush = 0;
  __threadfence();
  if (P->use_cond) {
    cudaGraphSetConditional(P->cond, more ? 1u : 0u);
    cudaGraphSetConditional(P->cond_outer, more ? 1u : 0u);
  }
}

// Stage export (stage_hook / trace mode, host-driven levels): between a
// level's partition pass and its scheduling, write every segment's
// post-stage contents into the caller's buffers (the view) and its record --
// the state the reference's hook sees after each stage (core.py:1705-1710).
// One CTA per segment; debug path, plain loads and stores.
template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) export_level_kernel(const Params *__restrict__ P) {
  typedef typename C::U U;
  __shared__ u64 s_cnt[2];
  const Ctl *ctl = P->ctl;
  const int cur = (int)(ctl->level & 1u);
  const uint32_t nseg = ctl->cur_nseg;
  U *vk = reinterpret_cast<U *>(P->view_keys);
  uint32_t *vp = P->view_pay;
  for (uint32_t sid = blockIdx.x; sid < nseg; sid += gridDim.x) {
    const Seg sg = P->segs[cur][sid];
    const long long b = sg.begin, e = sg.end, len = e - b;
    const U praw = C::dec((U)sg.pivot);
    StageRecord rec;
    rec.a = b;
    rec.b = e - 1;
    rec.pivot = (u64)praw;
    rec.depth = (int32_t)sg.depth;
    rec.new_l = -1;
    rec.new_r = -1;
    if (sg.kind == KIND_PARTITION) {
      const u64 inc =
          P->reproducible ? P->lookback[cur][sg.tile_base + sg.ntiles - 1] : sg.fill;
      const long long lt = (long long)((inc >> 31) & 0x7fffffffull);
      const long long gt = (long long)(inc & 0x7fffffffull);
      const int db = (int)sg.buf ^ 1;
      const U *src = reinterpret_cast<const U *>(P->keys[db]);
      const bool raw = P->raw[db] != 0;
      for (long long i = threadIdx.x; i < len; i += kThreads) {
        const bool mid = i >= lt && i < len - gt;
        vk[b + i] = mid ? praw : (raw ? src[b + i] : C::dec(src[b + i]));
        if (PAY) vp[b + i] = mid ? P->side_pay[b + (i - lt)] : P->pay[db][b + i];
      }
      rec.kind = TSQ_STAGE_PARTITION;
      rec.new_l = b + lt - 1;
      rec.new_r = e - gt;
    } else if (sg.fail) {
      rec.kind = TSQ_STAGE_HANDLER_FALLBACK;
      rec.new_l = sg.kind == KIND_VERIFY_ASC ? TSQ_STAGE_SORTED : TSQ_STAGE_REVERSED;
    } else {
      // verified: the segment is sorted (or reversed) where it lies
      const bool desc = sg.kind == KIND_VERIFY_DESC;
      const U *src = reinterpret_cast<const U *>(P->keys[sg.buf]);
      const bool raw = P->raw[sg.buf] != 0;
      if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
      __syncthreads();
      u64 lt = 0, gt = 0;
      for (long long i = threadIdx.x; i < len; i += kThreads) {
        const long long s = desc ? e - 1 - i : b + i;
        const U x = src[s];
        const U ex = raw ? C::enc(x) : x;
        lt += ex < (U)sg.pivot ? 1 : 0;
        gt += ex > (U)sg.pivot ? 1 : 0;
        vk[b + i] = raw ? x : C::dec(x);
        if (PAY) vp[b + i] = P->pay[sg.buf][s];
      }
      atomicAdd(&s_cnt[0], lt);
      atomicAdd(&s_cnt[1], gt);
      __syncthreads();
      rec.kind = desc ? TSQ_STAGE_REVERSED : TSQ_STAGE_SORTED;
      rec.new_l = b + (long long)s_cnt[0] - 1;
      rec.new_r = e - (long long)s_cnt[1];
    }
    if (threadIdx.x == 0) P->stage_out[sid] = rec;
    __syncthreads();
  }
}

__device__ __forceinline__ uint4 reversed(const uint4 &v) { return make_uint4(v.w, v.z, v.y, v.x); }
__device__ __forceinline__ uint2 reversed(const uint2 &v) { return make_uint2(v.y, v.x); }
__device__ __forceinline__ ulonglong2 reversed(const ulonglong2 &v) {
  return make_ulonglong2(v.y, v.x);
}

// Retire finished runs into buffer 0, chunk by chunk.
constexpr int kRB = 8;  // loads in flight per thread

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
    TSQ_CHECK(r.begin >= 0 && r.begin + r.len <= P->n && c >= r.chunk_base &&
              c < r.chunk_base + r.nchunks);
    const long long cc = (long long)(c - r.chunk_base);
    const long long lo = cc * kRunChunk;
    // every loop below issues kRB loads per thread before its stores, so
    // the loads overlap (the buffers may alias: no reordering otherwise)
    if (r.kind == RUN_EQ) {
      const long long hi = (lo + kRunChunk) < r.len ? (lo + kRunChunk) : r.len;
      const U v = raw0 ? C::dec((U)r.pivot) : (U)r.pivot;
      for (long long i = lo + threadIdx.x; i < hi; i += kThreads) {
        k0[r.begin + i] = v;
        if (PAY) p0[r.begin + i] = P->side_pay[r.src + i];
      }
    } else if (r.kind == RUN_SORTED || r.buf != 0) {
      // copy (sorted run) or reversed copy from the workspace into buffer 0
      const bool rev = r.kind == RUN_REVERSED;
      const long long hi = (lo + kRunChunk) < r.len ? (lo + kRunChunk) : r.len;
      const U *kb = reinterpret_cast<const U *>(P->keys[r.buf]);
      const uint32_t *pb = PAY ? P->pay[r.buf] : nullptr;
      const bool rawb = P->raw[r.buf] != 0;
      for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += (long long)kThreads * kRB) {
        U v[kRB];
        uint32_t pv[kRB];
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const long long i = i0 + (long long)q * kThreads;
          if (i < hi) {
            const long long s = rev ? r.begin + r.len - 1 - i : r.begin + i;
            v[q] = kb[s];
            if (PAY) pv[q] = pb[s];
          }
        }
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const long long i = i0 + (long long)q * kThreads;
          if (i < hi) {
            U x = v[q];
            if (rawb != raw0) x = rawb ? C::enc(x) : C::dec(x);
            k0[r.begin + i] = x;
            if (PAY) p0[r.begin + i] = pv[q];
          }
        }
      }
    } else if (P->aligned[0] && (r.begin & (Vec<U>::N - 1)) == 0 &&
               (r.len & (2 * Vec<U>::N - 1)) == 0) {
      // RUN_REVERSED in buffer 0, vector-aligned (the root of a descending
      // input): mirror pairs of 16-byte vectors, each reversed in registers
      constexpr int VN = Vec<U>::N;
      typedef typename Vec<U>::K KV;
      typedef typename Vec<U>::P PV;
      const long long half = r.len >> 1;
      const long long hi = (lo + kRunChunk) < half ? (lo + kRunChunk) : half;
      KV *kv = reinterpret_cast<KV *>(k0 + r.begin);
      PV *pvv = PAY ? reinterpret_cast<PV *>(p0 + r.begin) : nullptr;
      const long long nv = r.len / VN;  // vectors in the run; vector j mirrors nv - 1 - j
      constexpr int RBV = 4;
      for (long long j0 = lo / VN + threadIdx.x; j0 < hi / VN; j0 += (long long)kThreads * RBV) {
        KV x[RBV], y[RBV];
        PV px[RBV], py[RBV];
#pragma unroll
        for (int q = 0; q < RBV; ++q) {
          const long long j = j0 + (long long)q * kThreads;
          if (j < hi / VN) {
            x[q] = kv[j];
            y[q] = kv[nv - 1 - j];
            if (PAY) { px[q] = pvv[j]; py[q] = pvv[nv - 1 - j]; }
          }
        }
#pragma unroll
        for (int q = 0; q < RBV; ++q) {
          const long long j = j0 + (long long)q * kThreads;
          if (j < hi / VN) {
            kv[j] = reversed(y[q]);
            kv[nv - 1 - j] = reversed(x[q]);
            if (PAY) { pvv[j] = reversed(py[q]); pvv[nv - 1 - j] = reversed(px[q]); }
          }
        }
      }
    } else {  // RUN_REVERSED in buffer 0: swap the two halves' mirror pairs
      const long long half = r.len >> 1;
      const long long hi = (lo + kRunChunk) < half ? (lo + kRunChunk) : half;
      for (long long i0 = lo + threadIdx.x; i0 < hi; i0 += (long long)kThreads * kRB) {
        U x[kRB], y[kRB];
        uint32_t px[kRB], py[kRB];
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const long long i = i0 + (long long)q * kThreads;
          if (i < hi) {
            const long long a = r.begin + i, b = r.begin + r.len - 1 - i;
            x[q] = k0[a];
            y[q] = k0[b];
            if (PAY) { px[q] = p0[a]; py[q] = p0[b]; }
          }
        }
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const long long i = i0 + (long long)q * kThreads;
          if (i < hi) {
            const long long a = r.begin + i, b = r.begin + r.len - 1 - i;
            k0[a] = y[q];
            k0[b] = x[q];
            if (PAY) { p0[a] = py[q]; p0[b] = px[q]; }
          }
        }
      }
    }
  }
}

// Copy the control block to mapped host memory (read_ctl).
__global__ void publish_ctl_kernel(const Ctl *ctl, Ctl *host) {
  const u64 *s = reinterpret_cast<const u64 *>(ctl);
  volatile u64 *d = reinterpret_cast<volatile u64 *>(host);
  for (unsigned i = threadIdx.x; i < sizeof(Ctl) / sizeof(u64); i += blockDim.x) d[i] = s[i];
  __threadfence_system();
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
