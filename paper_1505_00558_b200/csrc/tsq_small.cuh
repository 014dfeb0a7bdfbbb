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

// ---------------------------------------------------------------------------
// The on-chip sort proper: every warp sorts 512 items (16 per lane) with a
// bitonic network in registers and shuffles, then log2(len/512) rounds merge
// pairs of sorted runs through shared memory along merge paths -- each
// thread binary-searches where its 16 outputs start and merges them
// sequentially.  Padding only to a multiple of 512 (merge runs are clamped to
// the segment length).
//
// Sort item: keys only -> the key; records with 32-bit keys -> key << 32 |
// local index in one u64; records with 64-bit keys -> (key, index) pairs in
// two arrays.  The index breaks ties (every item distinct) and gathers the
// payloads at the end.

constexpr int kVT = 16;     // items per thread
constexpr int kLogVT = 4;

template <class C, bool PAY>
struct MergeTraits {
  typedef typename C::U U;
  static constexpr bool kPack = PAY && sizeof(U) == 4;   // (key, index) in one u64
  static constexpr bool kIdx = PAY && sizeof(U) == 8;    // separate index array
  typedef typename std::conditional<kPack, u64, U>::type K;
};

__device__ __forceinline__ int pidx(int i) { return i + (i >> kLogVT); }  // padded rows

template <typename K, bool IDX>
__device__ __forceinline__ bool mless(K a, uint32_t ia, K b, uint32_t ib) {
  return IDX ? (a < b || (a == b && ia < ib)) : a < b;
}

template <typename K, bool IDX>
__device__ __forceinline__ void mcmpx(K &a, uint32_t &ia, K &b, uint32_t &ib) {
  if (IDX) {
    const bool sw = mless<K, IDX>(b, ib, a, ia);
    const K x = a; const uint32_t ix = ia;
    a = sw ? b : a; ia = sw ? ib : ia;
    b = sw ? x : b; ib = sw ? ix : ib;
  } else {
    const K x = a, y = b;
    a = x < y ? x : y;
    b = x < y ? y : x;
  }
}

// in-register bitonic sort of kVT items (all-ascending formulation)
template <typename K, bool IDX>
__device__ __forceinline__ void sort_thread(K (&v)[kVT], uint32_t (&vi)[kVT]) {
#pragma unroll
  for (int k = 2; k <= kVT; k <<= 1) {
#pragma unroll
    for (int r = 0; r < kVT; ++r) {
      const int p = r ^ (k - 1);
      if (r < p) mcmpx<K, IDX>(v[r], vi[r], v[p], vi[p]);
    }
#pragma unroll
    for (int j = k >> 2; j >= 1; j >>= 1) {
#pragma unroll
      for (int r = 0; r < kVT; ++r)
        if (!(r & j)) mcmpx<K, IDX>(v[r], vi[r], v[r | j], vi[r | j]);
    }
  }
}

template <typename K>
__device__ __forceinline__ K shfl_xor_k(K v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// x <- min(x, y) if keep_min else max(x, y)
template <typename K, bool IDX>
__device__ __forceinline__ void mkeep(K &x, uint32_t &ix, K y, uint32_t iy, bool keep_min) {
  if (IDX) {
    const bool take = mless<K, IDX>(y, iy, x, ix) == keep_min;
    x = take ? y : x;
    ix = take ? iy : ix;
  } else {
    const K mn = x < y ? x : y, mx = x < y ? y : x;
    x = keep_min ? mn : mx;
  }
}

// Bitonic sort of the warp's 32 * kVT items, lane l holding l*kVT ..
// l*kVT + kVT - 1: in-thread merges first, then merges of 32 .. 32 kVT with
// shuffle stages for the cross-lane strides.
template <typename K, bool IDX>
__device__ __forceinline__ void warp_sort(K (&v)[kVT], uint32_t (&vi)[kVT]) {
  const int lane = threadIdx.x & 31;
  sort_thread<K, IDX>(v, vi);
#pragma unroll 1
  for (int k = 2 * kVT; k <= 32 * kVT; k <<= 1) {
    {
      const int m = k / kVT - 1;
      const bool lower = (lane & (k / (2 * kVT))) == 0;
      K y[kVT];
      uint32_t yi[kVT];
#pragma unroll
      for (int r = 0; r < kVT; ++r) {
        y[r] = shfl_xor_k<K>(v[kVT - 1 - r], m);
        yi[r] = IDX ? __shfl_xor_sync(0xffffffffu, vi[kVT - 1 - r], m) : 0u;
      }
#pragma unroll
      for (int r = 0; r < kVT; ++r) mkeep<K, IDX>(v[r], vi[r], y[r], yi[r], lower);
    }
#pragma unroll 1
    for (int j = k >> 2; j >= kVT; j >>= 1) {
      const int m = j / kVT;
      const bool lower = (lane & m) == 0;
#pragma unroll
      for (int r = 0; r < kVT; ++r) {
        const K y = shfl_xor_k<K>(v[r], m);
        const uint32_t yi = IDX ? __shfl_xor_sync(0xffffffffu, vi[r], m) : 0u;
        mkeep<K, IDX>(v[r], vi[r], y, yi, lower);
      }
    }
#pragma unroll
    for (int j = kVT / 2; j >= 1; j >>= 1) {
#pragma unroll
      for (int r = 0; r < kVT; ++r)
        if (!(r & j)) mcmpx<K, IDX>(v[r], vi[r], v[r | j], vi[r | j]);
    }
  }
}

// One merge step for the thread whose outputs start at `o`: runs of length R
// (clamped to len) in (S, SI), kVT outputs into registers.
template <typename K, bool IDX>
__device__ __forceinline__ int merge_thread(const K *S, const uint32_t *SI, int o, int R, int len,
                                            K (&out)[kVT], uint32_t (&oi)[kVT]) {
  const int base = o & ~(2 * R - 1);
  const int a0 = base, na = min(R, len - base);
  const int b0 = base + na, nb = max(0, min(R, len - base - R));
  const int diag = o - base;
  int lo = max(0, diag - nb), hi = min(diag, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int pa = pidx(a0 + mid), pb = pidx(b0 + diag - 1 - mid);
    const K ka = S[pa], kb = S[pb];
    const uint32_t ja = IDX ? SI[pa] : 0u, jb = IDX ? SI[pb] : 0u;
    if (mless<K, IDX>(kb, jb, ka, ja)) hi = mid;
    else lo = mid + 1;
  }
  int ia = a0 + lo, ib = b0 + (diag - lo);
  const int ae = a0 + na, be = b0 + nb;
  // an exhausted run reads as the sentinel (greater than every item)
  const K SENT = ~K(0);
  K ka = ia < ae ? S[pidx(ia)] : SENT, kb = ib < be ? S[pidx(ib)] : SENT;
  uint32_t ja = IDX ? (ia < ae ? SI[pidx(ia)] : 0xffffffffu) : 0u;
  uint32_t jb = IDX ? (ib < be ? SI[pidx(ib)] : 0xffffffffu) : 0u;
  const int cnt = min(kVT, na + nb - diag);
#pragma unroll
  for (int r = 0; r < kVT; ++r) {
    const bool ta = !mless<K, IDX>(kb, jb, ka, ja);
    out[r] = ta ? ka : kb;
    if (IDX) oi[r] = ta ? ja : jb;
    const int nx = ta ? ++ia : ++ib;
    const bool ok = nx < (ta ? ae : be);
    const K kn = ok ? S[pidx(nx)] : SENT;
    const uint32_t jn = IDX ? (ok ? SI[pidx(nx)] : 0xffffffffu) : 0u;
    if (ta) { ka = kn; ja = jn; } else { kb = kn; jb = jn; }
  }
  return cnt;
}

// Class geometry.  MULT: 16-key output chunks per thread in a merge round
// (the 512-thread class takes up to 16384 four-byte keys with two).
// Single-buffer classes hold every merge round's outputs in registers and
// write them back over the input after a barrier, so they need one padded
// buffer instead of two -- that is what fits the two-chunk class and 8-byte
// sort items into the 512-thread class's shared memory at 2 CTAs per SM.
template <class C, bool PAY, int NT>
struct SmallGeo {
  typedef MergeTraits<C, PAY> M;
  typedef typename M::K K;
  static constexpr int CLASS = NT == kThreads ? 0 : 1;
  static constexpr int MULT = (CLASS == 1 && !PAY && sizeof(typename C::U) == 4) ? 2 : 1;
  static constexpr int CAP = NT * kVT * MULT;       // keys
  static constexpr int NP = CAP + CAP / kVT;         // padded capacity (rows of kVT + 1)
  static constexpr bool SINGLE =
      NT == 2 * kThreads && (MULT > 1 || (sizeof(K) + (M::kIdx ? 4 : 0)) > 4);
  static constexpr size_t SMEM = (SINGLE ? 1 : 2) * (size_t)NP * (sizeof(K) + (M::kIdx ? 4 : 0));
};

// Sort items: keys only -> the key; records with 32-bit keys -> key << 32 |
// local index; records with 64-bit keys -> (key - lo) << 14 | local index
// when the segment's keys span less than 2^50 (PK64: one u64 compare per
// step, like the 32-bit case), else (key, index) pairs in two arrays.
template <class C, bool PAY, int NT, bool PK64>
__device__ __forceinline__ void small_sort_one(const Params *P, const SmallSeg &sm,
                                               unsigned char *smem, u64 lo) {
  typedef typename C::U U;
  typedef MergeTraits<C, PAY> M;
  typedef typename M::K K;
  typedef SmallGeo<C, PAY, NT> SG;
  constexpr bool IDX = M::kIdx && !PK64;
  constexpr bool PACK = M::kPack || PK64;   // (key, index) packed in one u64
  constexpr int SH = M::kPack ? 32 : 14;    // index bits below the key
  constexpr bool SINGLE = SG::SINGLE;
  constexpr int NP = SG::NP;
  constexpr int MULT = SG::MULT;
  constexpr int LPT = kVT * MULT;  // keys per thread
  // smem: buffers A, B [NP] of K | (records, 64-bit keys) index A, B [NP];
  // single-buffer classes: A only
  K *ka = reinterpret_cast<K *>(smem), *kb = SINGLE ? ka : ka + NP;  // current / other buffer
  uint32_t *ia = reinterpret_cast<uint32_t *>(ka + (SINGLE ? NP : 2 * NP));
  uint32_t *ib = SINGLE ? ia : ia + (IDX ? NP : 0);
  const int tid = threadIdx.x;
  const int len = sm.len;
  // threads holding items: whole warps (the warp sort covers 32 * kVT)
  const int rows = ((len + 32 * kVT - 1) / (32 * kVT)) * 32;
  const U *src = reinterpret_cast<const U *>(P->keys[sm.buf]) + sm.begin;
  const bool raw = P->raw[sm.buf] != 0;
  // coalesced load into padded rows (sentinels complete the last rows): all
  // of a thread's loads issued before any is used, so their latencies overlap
  U raw_k[LPT];
#pragma unroll
  for (int q = 0; q < LPT; ++q) {
    const int i = tid + q * NT;
    raw_k[q] = i < len ? src[i] : U(0);
  }
#pragma unroll
  for (int q = 0; q < LPT; ++q) {
    const int i = tid + q * NT;
    if (i < rows * kVT) {
      K x;
      if (i < len) {
        const U k = raw ? C::enc(raw_k[q]) : raw_k[q];
        x = PACK ? (K)((((u64)k - lo) << SH) | (u64)i) : (K)k;
      } else {
        x = ~K(0);
      }
      ka[pidx(i)] = x;
      if (IDX) ia[pidx(i)] = i < len ? (uint32_t)i : 0xffffffffu;
    }
  }
  __syncthreads();
  // every warp sorts runs of 32 rows (row = tid, tid + NT, ...: warp-uniform)
#pragma unroll 1
  for (int row = tid; row < rows; row += NT) {
    K v[kVT];
    uint32_t vi[kVT];
#pragma unroll
    for (int r = 0; r < kVT; ++r) {
      v[r] = ka[row * (kVT + 1) + r];
      vi[r] = IDX ? ia[row * (kVT + 1) + r] : 0u;
    }
    warp_sort<K, IDX>(v, vi);
#pragma unroll
    for (int r = 0; r < kVT; ++r) {
      ka[row * (kVT + 1) + r] = v[r];
      if (IDX) ia[row * (kVT + 1) + r] = vi[r];
    }
  }
  // merge rounds: output chunk m of a thread is row tid + m * NT
  for (int R = 32 * kVT; R < len; R <<= 1) {
    __syncthreads();
    K out[MULT][kVT];
    uint32_t oi[MULT][kVT];
    int cnt[MULT];
#pragma unroll
    for (int m = 0; m < MULT; ++m) {
      const int o = (tid + m * NT) * kVT;
      cnt[m] = o < len ? merge_thread<K, IDX>(ka, ia, o, R, len, out[m], oi[m]) : 0;
    }
    if (SINGLE) __syncthreads();  // every thread has read its inputs
#pragma unroll
    for (int m = 0; m < MULT; ++m) {
      const int row = tid + m * NT;
#pragma unroll
      for (int r = 0; r < kVT; ++r)
        if (r < cnt[m]) {
          kb[row * (kVT + 1) + r] = out[m][r];
          if (IDX) ib[row * (kVT + 1) + r] = oi[m][r];
        }
    }
    if (!SINGLE) {
      K *tk = ka; ka = kb; kb = tk;
      uint32_t *ti = ia; ia = ib; ib = ti;
    }
  }
  __syncthreads();
  U *dst = reinterpret_cast<U *>(P->keys[0]) + sm.begin;
  const bool dst_raw = P->raw[0] != 0;
  if (PAY && SINGLE) {
    // payloads gathered by local index straight from the source (an L1/L2
    // resident window) into registers, all before any is written (the
    // source may be buffer 0 itself)
    const uint32_t *ps = P->pay[sm.buf] + sm.begin;
    uint32_t pv[LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int i = tid + q * NT;
      pv[q] = i < len ? ps[PACK ? (uint32_t)((u64)ka[pidx(i)] & ((1ull << SH) - 1)) : ia[pidx(i)]]
                      : 0u;
    }
    __syncthreads();
    uint32_t *pd = P->pay[0] + sm.begin;
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int i = tid + q * NT;
      if (i < len) pd[i] = pv[q];
    }
  } else if (PAY) {
    // the same through the free merge buffer
    const uint32_t *ps = P->pay[sm.buf] + sm.begin;
    uint32_t *stage = reinterpret_cast<uint32_t *>(kb);
    for (int i = tid; i < len; i += NT)
      stage[i] = ps[PACK ? (uint32_t)((u64)ka[pidx(i)] & ((1ull << SH) - 1)) : ia[pidx(i)]];
    __syncthreads();
    uint32_t *pd = P->pay[0] + sm.begin;
    for (int i = tid; i < len; i += NT) pd[i] = stage[i];
  }
  for (int i = tid; i < len; i += NT) {
    const K x = ka[pidx(i)];
    const U k = PACK ? (U)(lo + ((u64)x >> SH)) : (U)x;
    dst[i] = dst_raw ? C::dec(k) : k;
  }
}

// One CTA per queued segment (tickets).  NT = 256: the queue of segments of
// <= kSmallT keys; NT = 512: kSmallT+1 .. the class capacity.
template <class C, bool PAY, int NT>
__global__ void __launch_bounds__(NT, NT == kThreads ? (PAY ? 2 : 3) : (PAY ? 1 : 2))
    small_sort_kernel(const Params *__restrict__ P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_ticket;
  __shared__ u64 s_range[2];
  Ctl *ctl = P->ctl;
  constexpr int cls = SmallGeo<C, PAY, NT>::CLASS;
  const uint32_t n_q = ctl->sq_count[cls];
  const uint32_t cap = P->sq_cap[cls];
  const uint32_t count = n_q < cap ? n_q : cap;
  const SmallSeg *q = P->sq[cls];
  uint32_t *ticket = &ctl->sq_ticket[cls];
  uint64_t elems = 0;
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t t = s_ticket;
    __syncthreads();
    if (t >= count) break;
    const SmallSeg sm = q[t];
    if constexpr (MergeTraits<C, PAY>::kIdx) {
      // 64-bit keys with payloads: the segment's key range decides the item
      // form (one u64 when it spans < 2^50, else key + index arrays)
      typedef typename C::U U;
      const U *src = reinterpret_cast<const U *>(P->keys[sm.buf]) + sm.begin;
      const bool raw = P->raw[sm.buf] != 0;
      u64 mn = ~0ull, mx = 0ull;
      for (int i = threadIdx.x; i < sm.len; i += NT) {
        const u64 k = (u64)(raw ? C::enc(src[i]) : src[i]);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
      }
      if (threadIdx.x == 0) { s_range[0] = ~0ull; s_range[1] = 0ull; }
      __syncthreads();
      atomicMin(&s_range[0], mn);
      atomicMax(&s_range[1], mx);
      __syncthreads();
      const u64 lo = s_range[0], hi = s_range[1];
      __syncthreads();
      if (((hi - lo) >> 50) == 0) small_sort_one<C, PAY, NT, true>(P, sm, smem_raw, lo);
      else small_sort_one<C, PAY, NT, false>(P, sm, smem_raw, 0ull);
    } else {
      small_sort_one<C, PAY, NT, false>(P, sm, smem_raw, 0ull);
    }
    elems += (uint64_t)sm.len;
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
