// select_dev.cuh -- CTA-level selection primitives (radix select, bitonic sort)
// shared by select.cu (K5) and ivf.cu (probe selection).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace seldev {

constexpr int SEL_MAX_WARPS = 32;

static __device__ __forceinline__ bool match_above(uint64_t v, uint64_t prefix, int s) {
  return s >= 64 ? true : ((v ^ prefix) >> s) == 0;
}

struct SelShared {
  unsigned int hist[256];
  unsigned long long red_min[SEL_MAX_WARPS];
  unsigned long long red_max[SEL_MAX_WARPS];
  unsigned long long vmin, vmax;
  unsigned long long prefix;
  unsigned long long k;
  unsigned long long less;
  unsigned long long eq;
  int digit;
  int out_cnt;
  long long M;
  long long r_eff;
};

// Block reduce of min/max over valid values.  Returns via sh.vmin/vmax.
template <class Get>
__device__ __forceinline__ void block_minmax(int64_t M, Get get, SelShared& sh) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    uint64_t v;
    if (get(i, v)) {
      lo = v < lo ? v : lo;
      hi = v > hi ? v : hi;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh.red_min[w] = lo;
    sh.red_max[w] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = ~0ull, b = 0ull;
    for (int i = 0; i < nw; ++i) {
      a = sh.red_min[i] < a ? sh.red_min[i] : a;
      b = sh.red_max[i] > b ? sh.red_max[i] : b;
    }
    sh.vmin = a;
    sh.vmax = b;
  }
  __syncthreads();
}

// MSD radix select: k-th smallest (0-based) among valid values produced by get.
// Requires k < number of valid values.  Leaves sh.prefix = value,
// sh.less = #valid < value, sh.eq = #valid == value.
template <class Get>
__device__ void block_radix_select(int64_t M, Get get, unsigned long long k, SelShared& sh) {
  block_minmax(M, get, sh);
  const unsigned long long vmin = sh.vmin, vmax = sh.vmax;
  if (vmin == vmax) {
    // all valid values equal
    if (threadIdx.x == 0) {
      sh.prefix = vmin;
      sh.less = 0;
      sh.eq = 0;  // filled below
      sh.k = k;
    }
    __syncthreads();
    // count valid
    if (threadIdx.x == 0) sh.hist[0] = 0;
    __syncthreads();
    unsigned int local = 0;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      uint64_t v;
      if (get(i, v)) ++local;
    }
    atomicAdd(&sh.hist[0], local);
    __syncthreads();
    if (threadIdx.x == 0) sh.eq = sh.hist[0];
    __syncthreads();
    return;
  }
  const int hib = 63 - __clzll((long long)(vmin ^ vmax));
  int shift = (hib / 8) * 8;
  if (threadIdx.x == 0) {
    const int s = shift + 8;
    sh.prefix = s >= 64 ? 0ull : (vmin >> s) << s;
    sh.k = k;
    sh.less = 0;
  }
  __syncthreads();
  for (; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sh.prefix;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      uint64_t v;
      if (get(i, v) && match_above(v, prefix, shift + 8)) atomicAdd(&sh.hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // each lane owns 8 consecutive bins
      const int lane = threadIdx.x;
      unsigned long long s8 = 0;
      for (int b = 0; b < 8; ++b) s8 += sh.hist[lane * 8 + b];
      unsigned long long incl = s8;
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const unsigned long long excl = incl - s8;
      const unsigned long long kk = sh.k;
      if (kk >= excl && kk < incl) {
        unsigned long long c = excl;
        int d = lane * 8;
        for (int b = 0; b < 8; ++b) {
          const unsigned int h = sh.hist[lane * 8 + b];
          if (kk < c + h) {
            d = lane * 8 + b;
            break;
          }
          c += h;
        }
        sh.digit = d;
        sh.k = kk - c;
        sh.less += c;
        sh.eq = sh.hist[d];
        sh.prefix = prefix | ((unsigned long long)d << shift);
      }
    }
    __syncthreads();
  }
}

static __device__ __forceinline__ bool pair_less(uint64_t ka, int64_t ia, uint64_t kb, int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

static __device__ __forceinline__ void bitonic_step(uint64_t* K, int64_t* I, int t, int size, int stride) {
  const int lo = 2 * t - (t & (stride - 1));
  const int hi = lo + stride;
  const bool up = ((lo & size) == 0);
  const uint64_t ka = K[lo], kb = K[hi];
  const int64_t ia = I[lo], ib = I[hi];
  const bool sw = up ? pair_less(kb, ib, ka, ia) : pair_less(ka, ia, kb, ib);
  if (sw) {
    K[lo] = kb;
    K[hi] = ka;
    I[lo] = ib;
    I[hi] = ia;
  }
}

// Sort P (power of two) (key, id) pairs in shared memory ascending.  Small
// arrays are sorted by warp 0 alone (warp-level syncs instead of ~log^2 P
// block barriers); every thread of the block must call this.
static __device__ void bitonic_sort(uint64_t* K, int64_t* I, int P) {
  if (P <= 1024) {
    if (threadIdx.x < 32) {
      for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int t = threadIdx.x; t < P / 2; t += 32) bitonic_step(K, I, t, size, stride);
          __syncwarp();
        }
      }
    }
    __syncthreads();
    return;
  }
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) bitonic_step(K, I, t, size, stride);
      __syncthreads();
    }
  }
}


// ---------------------------------------------------------------------------
// k-th smallest (0-based) of the valid u32 keys of a block: get(i, v) -> bool
// (valid) for i < M.  MSD radix select with 8-bit digits starting at the
// highest bit where the keys differ (min/max pass), warp-aggregated shared
// histogram updates (__match_any_sync: a skewed digit costs one atomic per
// warp, not 32) into 8 sub-histograms, lane-parallel digit search.  Requires
// k < number of valid keys; every thread of the block must call it.
struct KthU32Shared {
  unsigned int wh[8][256];
  unsigned int red[SEL_MAX_WARPS][2];
  unsigned int prefix, k, vmin, vmax;
};

template <class Get>
__device__ unsigned int block_kth_u32(int64_t M, Get get, unsigned int k, KthU32Shared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned int lo = 0xFFFFFFFFu, hi = 0u;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    unsigned int v;
    if (get(i, v)) {
      lo = min(lo, v);
      hi = max(hi, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    sh.red[warp][0] = lo;
    sh.red[warp][1] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int a = 0xFFFFFFFFu, b = 0u;
    for (int w = 0; w < nw; ++w) {
      a = min(a, sh.red[w][0]);
      b = max(b, sh.red[w][1]);
    }
    sh.vmin = a;
    sh.vmax = b;
    sh.k = k;
  }
  __syncthreads();
  const unsigned int vmin = sh.vmin, vmax = sh.vmax;
  if (vmin == vmax) return vmin;
  const int hib = 31 - __clz((int)(vmin ^ vmax));
  int shift = (hib / 8) * 8;
  if (threadIdx.x == 0) sh.prefix = shift + 8 >= 32 ? 0u : (vmin >> (shift + 8)) << (shift + 8);
  __syncthreads();
  for (; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh.wh[0][0])[i] = 0;
    __syncthreads();
    const unsigned int prefix = sh.prefix;
    unsigned int* h = sh.wh[warp & 7];
    for (int64_t base = 0; base < M; base += blockDim.x) {
      const int64_t i = base + threadIdx.x;
      unsigned int v = 0;
      bool ok = i < M && get(i, v);
      ok = ok && (shift + 8 >= 32 || ((v ^ prefix) >> (shift + 8)) == 0);
      const unsigned int d = ok ? (v >> shift) & 255u : 256u;
      const unsigned int grp = __match_any_sync(0xffffffffu, d);
      if (ok && lane == __ffs(grp) - 1) atomicAdd(&h[d], (unsigned int)__popc(grp));
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // lane-parallel digit search: each lane owns 8 bins
      unsigned int c8[8], s8 = 0;
#pragma unroll
      for (int bb = 0; bb < 8; ++bb) {
        unsigned int t = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += sh.wh[w][lane * 8 + bb];
        c8[bb] = t;
        s8 += t;
      }
      unsigned int incl = s8;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const unsigned int kk = sh.k, excl = incl - s8;
      if (kk >= excl && kk < incl) {
        unsigned int cc = excl;
        int d = lane * 8;
        for (int bb = 0; bb < 8; ++bb) {
          if (kk < cc + c8[bb]) {
            d = lane * 8 + bb;
            break;
          }
          cc += c8[bb];
        }
        sh.k = kk - cc;
        sh.prefix = prefix | ((unsigned int)d << shift);
      }
    }
    __syncthreads();
  }
  return sh.prefix;
}

}  // namespace seldev
