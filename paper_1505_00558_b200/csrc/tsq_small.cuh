// tsq_small.cuh -- on-chip sort of the segments the recursion leaves behind
// (<= small_t keys): the role insertion_sort plays for ranges of at most
// insertion_threshold keys in the reference (smallsort.py:12-47,
// core.py:1652-1658), done as a bitonic sorting network.
//
// One CTA (256 threads) per segment, padded to N = 256 * E keys (E = 1 .. 16
// per thread) with +max sentinels.  Keys live in registers in blocked order
// (thread t holds elements t*E .. t*E+E-1).  The network is the all-ascending
// bitonic formulation: merge k starts with a "flip" stage (i against
// i ^ (k-1)) followed by half-cleaners (i against i ^ j), and every
// comparator puts the minimum at the lower index -- no direction logic, one
// min/max pair per comparator.  Stages exchange data three ways:
//   stride <  E      both keys in the thread's registers
//   stride <  32 E   partner thread in the same warp (__shfl_xor_sync)
//   stride >= 32 E   partner in another warp: one shared-memory round trip
//                    in register-major order (conflict-free)
// Global I/O is staged through shared memory (padded rows) so it coalesces.
// Records sort (key, local index) pairs so equal keys keep their own payloads
// and sentinels sort after every real key; payloads are gathered by index.
// Output always lands in buffer 0.
#pragma once

namespace tsq {

template <typename U, bool PAY>
struct SortItem {
  U k;
  uint32_t i;  // local index (records only)
};

template <typename U, bool PAY>
__device__ __forceinline__ bool item_less(const SortItem<U, PAY> &a, const SortItem<U, PAY> &b) {
  if (PAY) return a.k < b.k || (a.k == b.k && a.i < b.i);
  return a.k < b.k;
}

// comparator: a <- min, b <- max
template <typename U, bool PAY>
__device__ __forceinline__ void cmpx(SortItem<U, PAY> &a, SortItem<U, PAY> &b) {
  if (PAY) {
    const bool sw = item_less<U, PAY>(b, a);
    const SortItem<U, PAY> x = a;
    a.k = sw ? b.k : a.k;
    a.i = sw ? b.i : a.i;
    b.k = sw ? x.k : b.k;
    b.i = sw ? x.i : b.i;
  } else {
    const U x = a.k, y = b.k;
    a.k = x < y ? x : y;
    b.k = x < y ? y : x;
  }
}

// x <- min(x, y) if keep_min else max(x, y)
template <typename U, bool PAY>
__device__ __forceinline__ void keep(SortItem<U, PAY> &x, const SortItem<U, PAY> &y,
                                     bool keep_min) {
  if (PAY) {
    const bool take = item_less<U, PAY>(y, x) == keep_min;
    x.k = take ? y.k : x.k;
    x.i = take ? y.i : x.i;
  } else {
    const U mn = x.k < y.k ? x.k : y.k;
    const U mx = x.k < y.k ? y.k : x.k;
    x.k = keep_min ? mn : mx;
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

// Exchange with thread tid ^ m: y[r] = partner's v[rev ? E-1-r : r].
template <typename U, bool PAY, int E>
__device__ __forceinline__ void exchange(const SortItem<U, PAY> (&v)[E], SortItem<U, PAY> (&y)[E],
                                         int m, bool rev, U *xk, uint32_t *xi) {
  const int tid = threadIdx.x;
  if (m < 32) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const SortItem<U, PAY> &s = rev ? v[E - 1 - r] : v[r];
      y[r].k = shfl_xor_u<U>(s.k, m);
      if (PAY) y[r].i = __shfl_xor_sync(0xffffffffu, s.i, m);
    }
  } else {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < E; ++r) {
      xk[r * kThreads + tid] = v[r].k;
      if (PAY) xi[r * kThreads + tid] = v[r].i;
    }
    __syncthreads();
    const int p = tid ^ m;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int rr = rev ? E - 1 - r : r;
      y[r].k = xk[rr * kThreads + p];
      if (PAY) y[r].i = xi[rr * kThreads + p];
    }
  }
}

// in-thread half-cleaners with strides E/2 .. 1 (compile-time indices)
template <typename U, bool PAY, int E>
__device__ __forceinline__ void half_clean_regs(SortItem<U, PAY> (&v)[E]) {
#pragma unroll
  for (int j = E / 2; j >= 1; j >>= 1) {
#pragma unroll
    for (int r = 0; r < E; ++r)
      if (!(r & j)) cmpx<U, PAY>(v[r], v[r | j]);
  }
}

// Bitonic sort of N = 256 * E items held as v[E] per thread (blocked).
template <typename U, bool PAY, int E>
__device__ __forceinline__ void block_bitonic(SortItem<U, PAY> (&v)[E], U *xk, uint32_t *xi) {
  constexpr int N = kThreads * E;
  const int tid = threadIdx.x;
  // merges of size 2 .. E: entirely inside each thread
#pragma unroll
  for (int k = 2; k <= E; k <<= 1) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int p = r ^ (k - 1);
      if (r < p) cmpx<U, PAY>(v[r], v[p]);
    }
#pragma unroll
    for (int j = k >> 2; j >= 1; j >>= 1) {
#pragma unroll
      for (int r = 0; r < E; ++r)
        if (!(r & j)) cmpx<U, PAY>(v[r], v[r | j]);
    }
  }
  // merges of size 2E .. N: cross-thread strides first, then in registers
#pragma unroll 1
  for (int k = 2 * E; k <= N; k <<= 1) {
    SortItem<U, PAY> y[E];
    {
      // flip: element (tid, r) against (tid ^ (k/E - 1), E-1-r)
      const int m = k / E - 1;
      const bool lower = (tid & (k / (2 * E))) == 0;
      exchange<U, PAY, E>(v, y, m, true, xk, xi);
#pragma unroll
      for (int r = 0; r < E; ++r) keep<U, PAY>(v[r], y[r], lower);
    }
#pragma unroll 1
    for (int j = k >> 2; j >= E; j >>= 1) {
      const int m = j / E;
      const bool lower = (tid & m) == 0;
      exchange<U, PAY, E>(v, y, m, false, xk, xi);
#pragma unroll
      for (int r = 0; r < E; ++r) keep<U, PAY>(v[r], y[r], lower);
    }
    half_clean_regs<U, PAY, E>(v);
  }
}

template <class C, bool PAY, int E>
__device__ __forceinline__ void small_sort_one(const Params *P, const SmallSeg &sm,
                                               unsigned char *smem) {
  typedef typename C::U U;
  constexpr int N = kThreads * E;
  constexpr int ROW = E + 1;  // padded row per thread for blocked access
  // smem: keys [kThreads * ROW] | indices [kThreads * ROW] | payloads [N]
  U *xk = reinterpret_cast<U *>(smem);
  uint32_t *xi = reinterpret_cast<uint32_t *>(xk + kThreads * ROW);
  uint32_t *sp = xi + (PAY ? kThreads * ROW : 0);
  const int tid = threadIdx.x;
  const U *src = reinterpret_cast<const U *>(P->keys[sm.buf]) + sm.begin;
  const bool raw = P->raw[sm.buf] != 0;
  const int len = sm.len;
  // coalesced load into padded rows: element i -> row i / E, column i % E
  for (int i = tid; i < N; i += kThreads) {
    U x = KeyMax<U>::v;
    if (i < len) {
      x = src[i];
      if (raw) x = C::enc(x);
    }
    xk[(i / E) * ROW + (i % E)] = x;
  }
  if (PAY) {
    const uint32_t *ps = P->pay[sm.buf] + sm.begin;
    for (int i = tid; i < len; i += kThreads) sp[i] = ps[i];
  }
  __syncthreads();
  SortItem<U, PAY> v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    v[r].k = xk[tid * ROW + r];
    v[r].i = (uint32_t)(tid * E + r);
  }
  block_bitonic<U, PAY, E>(v, xk, xi);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < E; ++r) xk[tid * ROW + r] = v[r].k;
  if (PAY) {
    __syncthreads();  // xi (the exchange scratch) becomes the index row buffer
#pragma unroll
    for (int r = 0; r < E; ++r) xi[tid * ROW + r] = v[r].i;
  }
  __syncthreads();
  U *dst = reinterpret_cast<U *>(P->keys[0]) + sm.begin;
  const bool dst_raw = P->raw[0] != 0;
  uint32_t *pd = PAY ? P->pay[0] + sm.begin : nullptr;
  for (int i = tid; i < len; i += kThreads) {
    const U x = xk[(i / E) * ROW + (i % E)];
    dst[i] = dst_raw ? C::dec(x) : x;
    if (PAY) pd[i] = sp[xi[(i / E) * ROW + (i % E)]];
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
