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
  // digits of up to 8 bits from the highest differing bit down: the first
  // digit spans the top 8 varying bits, so all 256 bins are in use (no
  // hot-bin atomics); bits above hib are common to every key (the prefix)
  int top = hib + 1;
  if (threadIdx.x == 0) {
    sh.prefix = top >= 64 ? 0ull : (vmin >> top) << top;
    sh.k = k;
    sh.less = 0;
  }
  __syncthreads();
  while (top > 0) {
    const int width = top < 8 ? top : 8, shift = top - width;
    const unsigned long long dmask = (1ull << width) - 1ull;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sh.prefix;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      uint64_t v;
      if (get(i, v) && match_above(v, prefix, top)) atomicAdd(&sh.hist[(v >> shift) & dmask], 1u);
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
    top = shift;
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


}  // namespace seldev
