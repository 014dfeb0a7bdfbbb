// tsq_small.cuh -- on-chip sort of the segments the recursion leaves behind
// (<= small_t keys): the role insertion_sort plays for ranges of at most
// insertion_threshold keys in the reference (smallsort.py:12-47,
// core.py:1652-1658), done as a bitonic sorting network.
//
// One CTA (256 threads) per segment, the segment padded to N = 256 * E keys
// (E = 1 .. 16 per thread) with +max sentinels.  Keys live in registers in
// blocked order (thread t holds elements t*E .. t*E+E-1), so the stages of
// the network map to three exchange mechanisms:
//   j <  E        both keys in the same thread's registers (IMNMX)
//   j <  32 E     partner thread in the same warp (__shfl_xor_sync)
//   j >= 32 E     partner thread in another warp: one shared-memory round
//                 trip in register-major order (conflict-free)
// Records sort (key, local index) pairs so equal keys keep their own
// payloads and sentinels sort after every real key; payloads are gathered
// by index at the end.  Output always lands in buffer 0.
#pragma once

namespace tsq {

template <typename U, bool PAY>
struct SortItem {
  U k;
  uint32_t i;  // local index (records only)
};

// "a sorts before b"
template <typename U, bool PAY>
__device__ __forceinline__ bool item_less(const SortItem<U, PAY> &a, const SortItem<U, PAY> &b) {
  if (PAY) return a.k < b.k || (a.k == b.k && a.i < b.i);
  return a.k < b.k;
}

// keep the smaller (keep_min) or larger of (x, y) in x
template <typename U, bool PAY>
__device__ __forceinline__ void keep(SortItem<U, PAY> &x, const SortItem<U, PAY> &y,
                                     bool keep_min) {
  const bool take = item_less<U, PAY>(y, x) == keep_min;
  if (PAY) {
    x.k = take ? y.k : x.k;
    x.i = take ? y.i : x.i;
  } else {
    x.k = take ? y.k : x.k;
  }
}

template <typename U>
__device__ __forceinline__ U shfl_xor_u(U v, int m);
template <>
__device__ __forceinline__ uint32_t shfl_xor_u<uint32_t>(uint32_t v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
template <>
__device__ __forceinline__ u64 shfl_xor_u<u64>(u64 v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Bitonic sort of N = 256 * E items held as v[E] per thread (blocked).
// xk / xi: shared scratch of >= N keys / indices for cross-warp stages.
template <typename U, bool PAY, int E>
__device__ __forceinline__ void block_bitonic(SortItem<U, PAY> (&v)[E], U *xk, uint32_t *xi) {
  constexpr int N = kThreads * E;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  // merge size k and cross-thread strides are runtime loops (small code);
  // in-thread strides are unrolled so register indices stay compile-time
#pragma unroll 1
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j >= E; j >>= 1) {
      if (j < 32 * E) {
        // partner thread tid ^ (j / E) in the same warp, same register
        const int m = j / E;
        const bool lower = (lane & m) == 0;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int i = tid * E + r;
          const bool up = (i & k) == 0;
          SortItem<U, PAY> y;
          y.k = shfl_xor_u<U>(v[r].k, m);
          if (PAY) y.i = __shfl_xor_sync(0xffffffffu, v[r].i, m);
          keep<U, PAY>(v[r], y, lower == up);
        }
      } else {
        // partner thread tid ^ (j / E) in another warp: register-major
        // exchange through shared memory (lanes touch consecutive words)
        const int m = j / E;
        const bool lower = (tid & m) == 0;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) {
          xk[r * kThreads + tid] = v[r].k;
          if (PAY) xi[r * kThreads + tid] = v[r].i;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int i = tid * E + r;
          const bool up = (i & k) == 0;
          SortItem<U, PAY> y;
          y.k = xk[r * kThreads + (tid ^ m)];
          if (PAY) y.i = xi[r * kThreads + (tid ^ m)];
          keep<U, PAY>(v[r], y, lower == up);
        }
      }
    }
    // both partners in this thread: strides E/2 .. 1 (those below k)
#pragma unroll
    for (int j = E / 2; j >= 1; j >>= 1) {
      if (j >= k) continue;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (r & j) continue;
        const int i = tid * E + r;
        const bool up = (i & k) == 0;
        SortItem<U, PAY> a = v[r], b = v[r | j];
        const bool sw = item_less<U, PAY>(b, a) == up;
        v[r] = sw ? b : a;
        v[r | j] = sw ? a : b;
      }
    }
  }
}

template <class C, bool PAY, int E>
__device__ __forceinline__ void small_sort_one(const Params *P, const SmallSeg &sm,
                                               unsigned char *smem) {
  typedef typename C::U U;
  constexpr int N = kThreads * E;
  U *xk = reinterpret_cast<U *>(smem);
  uint32_t *xi = reinterpret_cast<uint32_t *>(xk + N);
  uint32_t *sp = xi + (PAY ? N : 0);  // staged payloads (records)
  const int tid = threadIdx.x;
  const U *src = reinterpret_cast<const U *>(P->keys[sm.buf]) + sm.begin;
  const bool raw = P->raw[sm.buf] != 0;
  const int len = sm.len;
  SortItem<U, PAY> v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = tid * E + r;
    U x = KeyMax<U>::v;
    if (i < len) {
      x = src[i];
      if (raw) x = C::enc(x);
    }
    v[r].k = x;
    v[r].i = (uint32_t)i;
  }
  if (PAY) {
    const uint32_t *ps = P->pay[sm.buf] + sm.begin;
    for (int i = tid; i < len; i += kThreads) sp[i] = ps[i];
  }
  block_bitonic<U, PAY, E>(v, xk, xi);
  __syncthreads();  // every key was loaded before any is stored (in place)
  U *dst = reinterpret_cast<U *>(P->keys[0]) + sm.begin;
  const bool dst_raw = P->raw[0] != 0;
  uint32_t *pd = PAY ? P->pay[0] + sm.begin : nullptr;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = tid * E + r;
    if (i < len) {
      dst[i] = dst_raw ? C::dec(v[r].k) : v[r].k;
      if (PAY) pd[i] = sp[v[r].i];
    }
  }
}

template <class C, bool PAY>
__global__ void __launch_bounds__(kThreads) small_sort_kernel(const Params *__restrict__ P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_ticket;
  Ctl *ctl = P->ctl;
  const uint32_t count = ctl->small_count < P->small_cap ? ctl->small_count : P->small_cap;
  uint64_t elems = 0;
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->small_ticket, 1u);
    __syncthreads();
    const uint32_t t = s_ticket;
    __syncthreads();
    if (t >= count) break;
    const SmallSeg sm = P->smalls[t];
    const int len = sm.len;
    if (len <= kThreads) small_sort_one<C, PAY, 1>(P, sm, smem_raw);
    else if (len <= 2 * kThreads) small_sort_one<C, PAY, 2>(P, sm, smem_raw);
    else if (len <= 4 * kThreads) small_sort_one<C, PAY, 4>(P, sm, smem_raw);
    else if (len <= 8 * kThreads) small_sort_one<C, PAY, 8>(P, sm, smem_raw);
    else small_sort_one<C, PAY, 16>(P, sm, smem_raw);
    elems += (uint64_t)len;
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
