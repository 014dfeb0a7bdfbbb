// tsq_device.cuh -- device-side building blocks of the B200 three-way
// partition sort: key codecs, queue records, the control block, and the
// CTA-wide pivot-sampling / sorting-network / look-back helpers.
//
// Reference path being accelerated (tsqsort 0.1.0,
// /root/reference/pkg/src/tsqsort): Sorter._range (core.py:1643-1728),
// select_pivot (pivot.py:205-248), _run_machine (core.py:198-984) and
// insertion_sort (smallsort.py:12-47).  See DESIGN.md for the mapping.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/tsq.h"

namespace tsq {

typedef unsigned long long u64;

constexpr int kThreads = 256;        // every kernel: 8 warps per CTA
constexpr int kSmallT = 4096;        // on-chip sort, 256-thread class (<= this)
constexpr int kSmallMax = 8192;      // on-chip sort, 512-thread class, 8-byte items
constexpr int kSmallHuge = 16384;    // on-chip sort, 512-thread class, 4-byte keys only
#ifndef TSQ_S2_SLOTS
#define TSQ_S2_SLOTS 40960
#endif
constexpr int kSmallGiant = TSQ_S2_SLOTS;   // on-chip sort, class 2 of bare 4-byte keys
constexpr int kSmallClasses = 3;
constexpr int kSmallSlack = 8;       // a class of S item slots takes segments of <= S - 8 keys
constexpr int kMaxSample = 1023;     // pivot sample size cap (2^10 - 1)
constexpr int kRunChunk = 8192;      // elements per retire work item
constexpr int kMaxLevels = 512;      // hard stop for the level loop (never reached: the
                                     // depth guard bisects key bounds, see Seg::klo)

constexpr u64 kFlagAgg = 1ull << 62;  // look-back: tile aggregate published
constexpr u64 kFlagInc = 2ull << 62;  // look-back: inclusive prefix published
constexpr u64 kValMask = (1ull << 62) - 1;

enum SegKind : uint32_t {
  KIND_PARTITION = 0,
  KIND_VERIFY_ASC = 1,
  KIND_VERIFY_DESC = 2,
  KIND_DONE = 3  // stage marker: the partition pass ran out of tiles
};
enum RunKind : uint32_t { RUN_EQ = 0, RUN_SORTED = 1, RUN_REVERSED = 2 };
enum ErrFlag : uint32_t { ERR_DEPTH = 1u, ERR_CAPACITY = 2u, ERR_LEVELS = 4u };

// A live segment of one level: [begin, end) of buffer `buf` (0 = the
// caller's keys, 1 = the workspace partner), partitioned around `pivot`
// (an encoded key) or verified sorted / reversed.  [klo, khi] bounds its
// encoded keys: the root's is the whole key space, a < child's is
// [klo, pivot - 1] and a > child's [pivot + 1, khi].  Beyond the depth
// guard a segment is split at the bound's midpoint instead of a sampled
// pivot, which halves the bound every level -- the recursion always ends
// (the reference's _range always finishes, core.py:1643-1728).
struct Seg {
  long long begin, end;
  u64 pivot;
  u64 klo, khi;
  // atomic placement: the (<, >) ranges its tiles have reserved so far, and
  // after the pass the segment's totals -- read with the record by the
  // scheduling (no further round trip); look-back placement keeps its
  // descriptors in lookback[]
  u64 fill;
  uint32_t tile_base, ntiles;
  uint32_t buf, kind, depth, noverify;
  uint32_t eq_fill;  // records, atomic placement: == payload slots reserved so far
  uint32_t fail;
};

// A segment of <= kSmallHuge elements waiting for the on-chip sort.
struct SmallSeg {
  long long begin;
  int len;
  int buf;
};

// A finished run: an ==p block (fill / payload copy from the side buffer),
// or a verified sorted / reversed segment that only needs moving to buffer 0.
struct Run {
  long long begin, len;
  u64 pivot;
  long long src;          // ==p runs: payload offset in side_pay
  uint32_t kind, buf;
  uint32_t chunk_base, nchunks;
};

// Control block (device memory; zeroed by the init kernel every sort).
struct Ctl {
  u64 next_packed;        // (segments << 32) | tiles appended for next level
  u64 run_packed;         // (runs << 32) | chunks appended
  uint32_t cur_nseg, cur_ntiles;
  uint32_t level, tile_ticket;
  uint32_t ctas_done, run_ticket;
  uint32_t error, pad0;
  // on-chip sort queues, one per class (256 / 512 threads): appended
  // segments, work tickets
  uint32_t sq_count[kSmallClasses], sq_ticket[kSmallClasses];
  u64 stages, max_depth, levels, eq_runs, eq_elements;
  u64 sorted_bypass, reversed_bypass, verify_fallbacks;
  u64 partitioned_elements, small_elements;
  u64 bytes_partition, bytes_small, bytes_retire;
  u64 stage_lt, stage_gt;   // single-stage / select-pivot results
  u64 writes0, writes1;     // element writes into buffer 0 / workspace
  // queue flushes: when the small-sort or run queues could not take one more
  // level's appends, the level loop pauses, the on-chip sort and retire
  // kernels drain them, and the loop resumes (so they never overflow)
  uint32_t flush, flushes;
  u64 small_segs_done;      // on-chip segments of earlier flush rounds
  u64 bisected;             // segments split at their key-bound midpoint
};

// Everything a kernel needs; lives in device memory, written by the init
// kernel from its by-value argument so the captured graph can be reused.
struct Params {
  void *keys[2];          // [0] caller's keys, [1] workspace partner
  uint32_t *pay[2];       // same for the uint32 payload (records)
  uint32_t *side_pay;     // ==p payloads staged during a partition pass
  long long n;
  double dran;
  int mitigation, fast_paths, max_depth, use_cond;
  int raw[2];             // buffer holds the caller's encoding (else ordered)
  int aligned[2];         // buffer's key / payload pointers are 16B aligned
  int single_stage;       // tsq_partition_segment: one given-pivot stage
  int small_t;            // segments <= small_t go to the on-chip sort
  int reproducible;       // look-back placement (else atomic range reservation)
  u64 given_pivot;        // encoded pivot for single_stage
  Seg *segs[2];
  uint32_t *tilemap[2];
  u64 *lookback[2];
  SmallSeg *sq[kSmallClasses];  // on-chip sort queues, one per class
  int sq_lim[kSmallClasses];    // largest segment of each class
  Run *runs;
  uint32_t *chunkmap;
  uint32_t sq_cap[kSmallClasses];
  uint32_t seg_cap, tile_cap, run_cap, chunk_cap;
  Ctl *ctl;
  cudaGraphConditionalHandle cond;        // inner loop: one recursion level per pass
  cudaGraphConditionalHandle cond_outer;  // outer loop: levels, then a queue drain
  // stage export (stage_hook / trace mode, host-driven levels only): after
  // each level, every segment's post-stage contents are written into the
  // caller's buffers (view_*) -- the sort itself runs in an aligned copy --
  // and a per-segment record into `stage_out`
  void *view_keys;
  uint32_t *view_pay;
  struct StageRecord *stage_out;
};

// One stage of a host-driven level, as reported to stage_hook / trace
// (tsq_stage_record in include/tsq.h; core.py:1705-1710).
struct StageRecord {
  long long a, b, new_l, new_r;
  u64 pivot;          // caller's encoding (raw bits)
  int32_t kind;       // TSQ_STAGE_* (include/tsq.h)
  int32_t depth;
};

// ---- invariant checks (debug builds only: -DTSQ_DEBUG_CHECKS) ---------------
// compute-sanitizer is not available on the GPU pool; a debug build checks
// the invariants every bulk copy, queue append and scatter relies on, and
// traps (a sticky launch error the host reports) on the first violation.
#ifdef TSQ_DEBUG_CHECKS
#include <cstdio>
#define TSQ_CHECK(cond)                                                                       \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("TSQ_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                              \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define TSQ_CHECK(cond) ((void)0)
#endif

// ---- optional per-tile timeline (profiling builds only: -DTSQ_TRACE) -------
#ifdef TSQ_TRACE
constexpr int kTraceTiles = 65536;
__device__ u64 g_trace[kTraceTiles * 8];
__device__ int g_trace_level;
__device__ __forceinline__ void trace_mark(uint32_t level, uint32_t t, int slot) {
  if ((int)level == g_trace_level && t < (uint32_t)kTraceTiles) {
    u64 ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    g_trace[(size_t)t * 8 + slot] = ns;
  }
}
#define TSQ_MARK(level, t, slot) trace_mark((level), (t), (slot))
#else
#define TSQ_MARK(level, t, slot) ((void)0)
#endif

// ---- order-preserving key codecs (native order -> unsigned order) ----------
template <int DT> struct Codec;
// kRawOrder: the caller's bits compare natively (signed / unsigned integer
// compare), so both ping-pong buffers keep the caller's encoding and the
// partition pass compares with rlt() -- no per-key re-encoding.  Floats
// keep the order-preserving unsigned encoding in the workspace buffer.
template <> struct Codec<TSQ_I32> {
  typedef uint32_t U;
  static constexpr bool kSigned = true;  // rlt is a signed compare
  static constexpr bool kRawOrder = true;
  static __device__ __forceinline__ bool rlt(U a, U b) { return (int32_t)a < (int32_t)b; }
  static __device__ __forceinline__ U enc(U x) { return x ^ 0x80000000u; }
  static __device__ __forceinline__ U dec(U x) { return x ^ 0x80000000u; }
};
template <> struct Codec<TSQ_U32> {
  typedef uint32_t U;
  static constexpr bool kSigned = false;  // rlt is a signed compare
  static constexpr bool kRawOrder = true;
  static __device__ __forceinline__ bool rlt(U a, U b) { return a < b; }
  static __device__ __forceinline__ U enc(U x) { return x; }
  static __device__ __forceinline__ U dec(U x) { return x; }
};
template <> struct Codec<TSQ_F32> {
  typedef uint32_t U;
  static constexpr bool kSigned = false;  // rlt is a signed compare
  static constexpr bool kRawOrder = false;
  static __device__ __forceinline__ bool rlt(U a, U b) { return enc(a) < enc(b); }
  static __device__ __forceinline__ U enc(U x) {
    return x ^ ((0u - (x >> 31)) | 0x80000000u);
  }
  static __device__ __forceinline__ U dec(U x) {
    return x ^ (((x >> 31) - 1u) | 0x80000000u);
  }
};
template <> struct Codec<TSQ_I64> {
  typedef u64 U;
  static constexpr bool kSigned = true;  // rlt is a signed compare
  static constexpr bool kRawOrder = true;
  static __device__ __forceinline__ bool rlt(U a, U b) { return (long long)a < (long long)b; }
  static __device__ __forceinline__ U enc(U x) { return x ^ 0x8000000000000000ull; }
  static __device__ __forceinline__ U dec(U x) { return x ^ 0x8000000000000000ull; }
};
template <> struct Codec<TSQ_U64> {
  typedef u64 U;
  static constexpr bool kSigned = false;  // rlt is a signed compare
  static constexpr bool kRawOrder = true;
  static __device__ __forceinline__ bool rlt(U a, U b) { return a < b; }
  static __device__ __forceinline__ U enc(U x) { return x; }
  static __device__ __forceinline__ U dec(U x) { return x; }
};
template <> struct Codec<TSQ_F64> {
  typedef u64 U;
  static constexpr bool kSigned = false;  // rlt is a signed compare
  static constexpr bool kRawOrder = false;
  static __device__ __forceinline__ bool rlt(U a, U b) { return enc(a) < enc(b); }
  static __device__ __forceinline__ U enc(U x) {
    return x ^ ((0ull - (x >> 63)) | 0x8000000000000000ull);
  }
  static __device__ __forceinline__ U dec(U x) {
    return x ^ (((x >> 63) - 1ull) | 0x8000000000000000ull);
  }
};

template <typename U> struct KeyMax;
template <> struct KeyMax<uint32_t> { static constexpr uint32_t v = 0xffffffffu; };
template <> struct KeyMax<u64> { static constexpr u64 v = ~0ull; };

// 16-byte vector of keys / matching payload vector
template <typename U> struct Vec;
template <> struct Vec<uint32_t> {
  static constexpr int N = 4;
  typedef uint4 K;
  typedef uint4 P;
};
template <> struct Vec<u64> {
  static constexpr int N = 2;
  typedef ulonglong2 K;
  typedef uint2 P;
};

__device__ __forceinline__ uint32_t ldcg(const uint32_t *p) { return __ldcg(p); }
__device__ __forceinline__ u64 ldcg(const u64 *p) { return __ldcg(p); }

__device__ __forceinline__ u64 ld_volatile(const u64 *p) {
  return *reinterpret_cast<const volatile u64 *>(p);
}
__device__ __forceinline__ void st_volatile(u64 *p, u64 v) {
  *reinterpret_cast<volatile u64 *>(p) = v;
}
__device__ __forceinline__ uint32_t ld_volatile32(const uint32_t *p) {
  return *reinterpret_cast<const volatile uint32_t *>(p);
}

// ---- mbarrier + bulk-copy (TMA engine) PTX wrappers -----------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u64 *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(u64 *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(u64 *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TSQ_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TSQ_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Waits: probe the barrier; while it is not there yet, back off with a
// short sleep.  (The suspend hint of try_wait alone wakes on every barrier
// event of the CTA, so idle warps would spin and take issue slots from the
// working ones.)  Distinct copies per role so profiles attribute the waits.
#ifndef TSQ_SLEEP_NS
#define TSQ_SLEEP_NS 32
#endif
#ifndef TSQ_SLEEP_PRODUCER_NS
#define TSQ_SLEEP_PRODUCER_NS 64
#endif
__device__ __forceinline__ bool mbar_test(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
template <int NS>
__device__ __forceinline__ void mbar_wait_sleep(u64 *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_test(a, parity)) {
    if (NS > 0) __nanosleep(NS);
  }
}
#ifndef TSQ_SLEEP_COUNTER_NS
#define TSQ_SLEEP_COUNTER_NS TSQ_SLEEP_NS
#endif
#ifndef TSQ_SLEEP_LB_NS
#define TSQ_SLEEP_LB_NS TSQ_SLEEP_NS
#endif
#ifndef TSQ_SLEEP_CONSUMER_NS
#define TSQ_SLEEP_CONSUMER_NS TSQ_SLEEP_NS
#endif
__device__ __forceinline__ void wait_full_consumer(u64 *bar, uint32_t parity) {
  mbar_wait_sleep<TSQ_SLEEP_COUNTER_NS>(bar, parity);
}
__device__ __forceinline__ void wait_aggr_lookback(u64 *bar, uint32_t parity) {
  mbar_wait_sleep<TSQ_SLEEP_LB_NS>(bar, parity);
}
__device__ __forceinline__ void wait_ready_consumer(u64 *bar, uint32_t parity) {
  mbar_wait_sleep<TSQ_SLEEP_CONSUMER_NS>(bar, parity);
}
__device__ __forceinline__ void wait_empty_producer(u64 *bar, uint32_t parity) {
  mbar_wait_sleep<TSQ_SLEEP_PRODUCER_NS>(bar, parity);
}


// 1-D bulk copy global -> shared, completing `bytes` on the mbarrier
// (cp.async.bulk: SASS UBLKCP); dst/src 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gsrc, uint32_t bytes,
                                          u64 *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy shared -> global (bulk-group completion)
__device__ __forceinline__ void bulk_store(void *gdst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all but the most recent bulk-store group have finished reading smem
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// generic-proxy smem writes -> visible to the async (bulk copy) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ u64 warp_sum64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// on-chip class of a segment of len keys
__device__ __forceinline__ int small_class(const Params *P, long long len) {
  return len <= P->sq_lim[0] ? 0 : (len <= P->sq_lim[1] ? 1 : 2);
}

// ---- pivot sample size: ~sqrt(len), 2^k - 1 with k in [5, 10] -------------
__device__ __forceinline__ int sample_count(long long len) {
  int bits = 64 - __clzll((long long)len);
  int k = (bits + 1) >> 1;
  k = k < 5 ? 5 : (k > 10 ? 10 : k);
  return (1 << k) - 1;
}

// ---- CTA-wide bitonic sorting network over s[0, P2) (P2 power of two) -------
template <typename U>
__device__ __forceinline__ void cta_bitonic(U *s, int P2) {
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (P2 >> 1); i += blockDim.x) {
        int lo = ((i / j) * 2 * j) + (i % j);
        int hi = lo + j;
        bool up = (lo & k) == 0;
        U a = s[lo], b = s[hi];
        if ((a > b) == up) {
          s[lo] = b;
          s[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// ---- device pivot sampling (select_pivot analogue, pivot.py:205-248) --------
// Median of S = sample_count(len) strided samples; the first, middle and last
// positions are fixed anchors and interior positions are shifted by the
// MitigationRng jitter (dran, pivot.py:223-237).  Also returns the order flag
// of the samples in position order (+1 nondecreasing, -1 nonincreasing).
// All threads of the CTA must call; `s` holds >= 1024 U of shared memory.
template <class C>
__device__ void cta_select_pivot(const typename C::U *data, bool encoded_src,
                                 long long begin, long long len, double dran,
                                 int mitigation, typename C::U *s,
                                 typename C::U *pivot_out, int *flag_out) {
  typedef typename C::U U;
  const int S = sample_count(len);
  const int P2 = S + 1;
  const int midi = S >> 1;
  const long long span = len - 1;
  long long shift = 0;
  if (mitigation) {
    const double stride = (double)span / (double)(S - 1);
    shift = (long long)floor((dran - 1.0) * stride * 0.5);
  }
  for (int i = threadIdx.x; i < P2; i += blockDim.x) {
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
  __syncthreads();
  bool asc = true, desc = true;
  for (int i = threadIdx.x; i < S - 1; i += blockDim.x) {
    U a = s[i], b = s[i + 1];
    asc &= (a <= b);
    desc &= (a >= b);
  }
  asc = __syncthreads_and(asc);
  desc = __syncthreads_and(desc);
  cta_bitonic(s, P2);
  if (threadIdx.x == 0) {
    *pivot_out = s[midi];
    *flag_out = asc ? 1 : (desc ? -1 : 0);
  }
  __syncthreads();
}

}  // namespace tsq
