// tsq_bitonic.cuh -- CTA-wide bitonic sorting network over register-held
// items (the schedule kernel's CTA-mode pivot sample sort, pivot.py:205-248:
// the median of up to 1023 samples).
//
// One CTA (256 threads) sorts N = 256 * E items, padded with +max sentinels.
// Items live in registers in blocked order (thread t holds elements t*E ..
// t*E+E-1).  The network is the all-ascending bitonic formulation: merge k
// starts with a "flip" stage (i against i ^ (k-1)) followed by half-cleaners
// (i against i ^ j), and every comparator puts the minimum at the lower index
// -- no direction logic, one min/max pair per comparator.  Stages exchange
// data three ways:
//   stride <  E      both keys in the thread's registers
//   stride <  32 E   partner thread in the same warp (__shfl_xor_sync)
//   stride >= 32 E   partner in another warp: one shared-memory round trip
//                    in register-major order (conflict-free)
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

}  // namespace tsq
