// ivf.cu -- IVFADC query (K7 probes, K8 list-major scan).
//
// Reference: query_ivf kernel='adc' (ivf.py:148-196): probe the ma nearest
// coarse cells by fp64 (distance, index) (nearest_k, _dist.py:42-67), scan
// each cell's list against the tables of the fp64 residual q - coarse[c]
// (ivf.py:179-183), merge all per-list top-r by (distance, id).
//
// B200 design:
//  K7  probes: probe.cu (tcgen05 kind::tf32 GEMM with the key and the
//      certified candidate filter fused into its epilogue, exact fp64
//      re-score) -> identical probe sets and order to nearest_k.
//  K8  the residual tables are never materialised per (query, list): with
//      PQ sub-spaces disjoint, sum_j T_j = ||q-c||^2 + sum_j U_q[j][code_j]
//      + V[code] where U_q[j][i] = ||C_ji||^2 - 2<q_j, C_ji> (per query) and
//      V = 2 sum_j <c_j, C_j[code_j]> (per stored code, at index build).
//      The list-major kernel (one CTA per inverted list, all queries probing
//      it) adds those in fp32 as a certified filter; survivors are re-scored
//      exactly (residual tables in fp64, scan.py:45-56 + 77-81 order) in the
//      select kernel.  The filter threshold per query comes from a sample
//      (the first 64 codes of every probed list).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "pqs_common.cuh"
#include "select_dev.cuh"
#include "tc_common.cuh"

namespace {

using namespace seldev;


// ------------------------------------------------------------ index build
__global__ void cnorm_kernel(const float* __restrict__ coarse, int64_t K, int d, double* __restrict__ cnorm,
                             float* __restrict__ gnorm, float* __restrict__ cnormf) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= K) return;
  double s = 0.0;
  for (int t = 0; t < d; ++t) {
    const double v = (double)coarse[c * d + t];
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  cnorm[c] = s;
  gnorm[c] = (float)sqrt(s);
  cnormf[c] = (float)s;
}

// index build: nearest of P pivot cells for every cell (fp32; only orders the
// list scan so that lists probed by nearby queries run close in time)
__global__ void pivot_assign_kernel(const float* __restrict__ coarse, int64_t K, int d, int P, int* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= K) return;
  const float* x = coarse + c * d;
  float best = __int_as_float(0x7f800000);
  int arg = 0;
  for (int p = 0; p < P; ++p) {
    const float* y = coarse + ((int64_t)p * K / P) * d;
    float s = 0.f;
    for (int t = 0; t < d; ++t) {
      const float df = x[t] - __ldg(y + t);
      s = fmaf(df, df, s);
    }
    if (s < best) {
      best = s;
      arg = p;
    }
  }
  out[c] = arg;
}

// V[pos] = 2 sum_j <g_cj, C_j[code_j]>, fp64 -> fp32; one CTA per list
__global__ void v_kernel(const float* __restrict__ coarse, const float* __restrict__ books,
                         const int64_t* __restrict__ offsets, const uint8_t* __restrict__ codes, int m, int k,
                         int dsub, int d, float* __restrict__ V, float* __restrict__ vmax_out) {
  const int64_t c = blockIdx.x;
  const int64_t b = offsets[c], e = offsets[c + 1];
  const float* g = coarse + c * (int64_t)d;
  float vmax = 0.f;
  for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) {
      const float* cb = books + ((int64_t)j * k + codes[p * m + j]) * dsub;
      for (int t = 0; t < dsub; ++t) s += (double)g[j * dsub + t] * (double)cb[t];
    }
    const float v = (float)(2.0 * s);
    V[p] = v;
    vmax = fmaxf(vmax, fabsf(v));
  }
  for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  if ((threadIdx.x & 31) == 0) atomicMax((int*)vmax_out, __float_as_int(vmax));
}

// per-query tables U[q][i][j] = ||C_ji||^2 - 2 <q_j, C_ji> (fp64 -> fp32),
// entry-major ([i * m + j]): the list scan's shared-memory row of (entry i,
// component j) then sits in bank window j mod 4 (see ivf_list_kernel).
// One CTA per UQ queries, thread = entry i: each codebook row is loaded once
// per CTA, the UQ tables are built in shared memory and written out with
// coalesced 16-byte stores.
constexpr int UQ = 8;
__global__ void __launch_bounds__(256) utables_kernel(QVec queries,
                                                      const float* __restrict__ books, int64_t nq, int m, int k,
                                                      int dsub, float* __restrict__ U) {
  extern __shared__ __align__(16) float usm[];  // [UQ][k * m] tables, then [UQ][d] fp64 queries
  const int d = m * dsub, mk = m * k;
  double* sq = reinterpret_cast<double*>(usm + (size_t)UQ * mk + ((size_t)UQ * mk & 1));
  const int64_t q0 = (int64_t)blockIdx.x * UQ;
  const int nqb = (int)min((int64_t)UQ, nq - q0);
  for (int t = threadIdx.x; t < nqb * d; t += blockDim.x) sq[t] = queries.at(q0 * d + t);
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    for (int j = 0; j < m; ++j) {
      const float* cb = books + ((int64_t)j * k + i) * dsub;
      double nn = 0.0;
      double dot[UQ];
#pragma unroll
      for (int u = 0; u < UQ; ++u) dot[u] = 0.0;
      for (int s2 = 0; s2 < dsub; ++s2) {
        const double cv = (double)__ldg(cb + s2);
        nn += cv * cv;
#pragma unroll
        for (int u = 0; u < UQ; ++u) dot[u] += sq[u * d + j * dsub + s2] * cv;
      }
#pragma unroll
      for (int u = 0; u < UQ; ++u) usm[u * mk + i * m + j] = (float)(nn - 2.0 * dot[u]);
    }
  }
  __syncthreads();
  float* out = U + q0 * mk;
  if ((mk & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(usm);
    float4* o4 = reinterpret_cast<float4*>(out);
    for (int t = threadIdx.x; t < nqb * mk / 4; t += blockDim.x) o4[t] = s4[t];
  } else {
    for (int t = threadIdx.x; t < nqb * mk; t += blockDim.x) out[t] = usm[t];
  }
}

// per query: E_q = certified bound of |filter distance - exact distance|
__global__ void ivf_bound_kernel(const float* __restrict__ U, const double* __restrict__ pdist, int64_t nq, int ma,
                                 int m, int k, const float* __restrict__ vmax, float* __restrict__ aerr) {
  const int64_t q = blockIdx.x;
  __shared__ double part[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double s = 0.0;
  for (int j = warp; j < m; j += nw) {
    float mx = 0.f;
    for (int i = lane; i < k; i += 32) mx = fmaxf(mx, fabsf(U[(q * k + i) * (int64_t)m + j]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    s += (double)mx;
  }
  if (lane == 0) part[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double usum = 0.0;
    for (int i = 0; i < nw; ++i) usum += part[i];
    double amax = 0.0;
    for (int p = 0; p < ma; ++p) amax = fmax(amax, pdist[q * ma + p]);
    const double B = amax + (double)vmax[0] + usum;
    const double u = 5.9604644775390625e-08;
    aerr[q] = (float)((m + 6) * u * 1.05 * B + 1e-30);
  }
}

// ------------------------------------------------------------ K8 helpers
// Filter threshold per query from a sample -- the first spl codes of every
// probed list -- computed and selected in one CTA: theta = (r-th smallest
// sampled filter distance) + 2 * aerr, rounded up (a certified upper bound
// of the r-th smallest exact distance over the probed lists); +inf when the
// sample holds fewer than r codes.
constexpr int THETA_THREADS = 512;
constexpr int THETA_SAMPLE_CAP = 16384;

__global__ void __launch_bounds__(THETA_THREADS) ivf_theta_kernel(
    const float* __restrict__ U, const int64_t* __restrict__ cells, const double* __restrict__ pdist,
    const int64_t* __restrict__ offsets, const uint8_t* __restrict__ codes, const float* __restrict__ V, int ma_row,
    int ma, int spl, int m, int k, int r, const float* __restrict__ aerr, float* __restrict__ theta) {
  // ma_row: probes per query (row stride of cells / pdist); ma: the nearest probes that are sampled
  extern __shared__ __align__(16) unsigned char tsm[];
  float* su = (float*)tsm;                                   // [m][k] (lanes read random entries of one row)
  unsigned int* keys = (unsigned int*)(su + (size_t)m * k);  // [ma*spl]
  __shared__ unsigned int hist[256];
  __shared__ unsigned int s_prefix, s_k, s_valid, s_kmin, s_kmax, s_cnt2;
  const int64_t q = blockIdx.x;
  for (int i = threadIdx.x; i < m * k; i += blockDim.x) {
    const int e = i / m, j = i - e * m;
    su[j * k + e] = U[q * (int64_t)m * k + i];
  }
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_k = (unsigned)(r - 1);
    s_valid = 0;
    s_kmin = 0xFFFFFFFFu;
    s_kmax = 0u;
  }
  __syncthreads();
  const int ns = ma * spl;
  // list bases / lengths / probe distances of the ma probes: one dependent
  // load chain per probe (not per sample), so the sample loop below issues
  // independent loads only
  int64_t* s_b = reinterpret_cast<int64_t*>(keys + ns + (ns & 1));  // [ma]
  int* s_len = reinterpret_cast<int*>(s_b + ma);                    // [ma]
  float* s_pd = reinterpret_cast<float*>(s_len + ma);               // [ma]
  for (int p = threadIdx.x; p < ma; p += blockDim.x) {
    const int64_t c = cells[q * ma_row + p];
    int64_t b = 0, e = 0;
    if (c >= 0) {
      b = offsets[c];
      e = offsets[c + 1];
    }
    s_b[p] = b;
    s_len[p] = (int)min((int64_t)spl, e - b);
    s_pd[p] = (float)pdist[q * ma_row + p];
  }
  __syncthreads();
  unsigned int valid = 0, kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll 4
  for (int s2 = threadIdx.x; s2 < ns; s2 += blockDim.x) {
    const int p = s2 / spl, i = s2 - p * spl;
    unsigned int key = 0xFFFFFFFFu;
    {
      if (i < s_len[p]) {
        const int64_t pos = s_b[p] + i;
        float acc = s_pd[p] + V[pos];
        if (m == 8) {  // one 8-byte load per sampled code
          const uint2 cw = *reinterpret_cast<const uint2*>(codes + pos * 8);
#pragma unroll
          for (int j = 0; j < 4; ++j) acc += su[j * k + ((cw.x >> (8 * j)) & 255u)];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc += su[(4 + j) * k + ((cw.y >> (8 * j)) & 255u)];
        } else {
          for (int j = 0; j < m; ++j) acc += su[j * k + codes[pos * m + j]];
        }
        key = fkey(acc);
        ++valid;
        kmin = min(kmin, key);
        kmax = max(kmax, key);
      }
    }
    keys[s2] = key;
  }
  atomicAdd(&s_valid, valid);
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_kmin, kmin);
    atomicMax(&s_kmax, kmax);
  }
  __syncthreads();
  if (s_valid < (unsigned)r) {
    if (threadIdx.x == 0) theta[q] = __int_as_float(0x7f800000);
    return;
  }
  // digits from the highest bit where the keys differ (fkeys share their
  // sign/exponent bits: a fixed 24-bit first shift would pile them into a
  // few hot bins); the common high bits seed the prefix
  const unsigned kdiff = s_kmin ^ s_kmax;
  const int top0 = kdiff ? 32 - __clz((int)kdiff) : 0;
  const unsigned prefix0 = top0 >= 32 ? 0u : (s_kmin >> top0) << top0;
  // k-th smallest (0-based) of the valid keys arr[i * stride], i < n: MSD radix
  // select, 8-bit digits, shared histogram; result in s_prefix
  auto radix_kth = [&](const unsigned int* arr, int n, int stride, unsigned kth) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_prefix = prefix0;
      s_k = kth;
    }
    __syncthreads();
    for (int top = top0; top > 0;) {
      const int width = top < 8 ? top : 8, shift = top - width;
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const unsigned prefix = s_prefix;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned key = arr[i * stride];
        if (key == 0xFFFFFFFFu) continue;
        const bool match = top >= 32 ? true : ((key ^ prefix) >> top) == 0;
        if (match) atomicAdd(&hist[(key >> shift) & ((1u << width) - 1u)], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // lane-parallel digit search: each lane owns 8 bins
        const int lane = threadIdx.x;
        unsigned int s8 = 0;
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) s8 += hist[lane * 8 + bb];
        unsigned int incl = s8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const unsigned int kk = s_k, excl = incl - s8;
        if (kk >= excl && kk < incl) {
          unsigned int cc = excl;
          int d = lane * 8;
          for (int bb = 0; bb < 8; ++bb) {
            const unsigned int h = hist[lane * 8 + bb];
            if (kk < cc + h) {
              d = lane * 8 + bb;
              break;
            }
            cc += h;
          }
          s_k = kk - cc;
          s_prefix = prefix | ((unsigned)d << shift);
        }
      }
      __syncthreads();
      top = shift;
    }
  };
  // The r-th smallest of ~16k keys is a low quantile: take a pivot from a
  // strided subsample (rank ~3 r scaled to the subsample), compact the keys
  // below it (a few hundred) and select among those; the full-array select
  // runs only if the pivot missed (fewer than r keys below it, or too many).
  constexpr int SUB = 1024;
  const unsigned int SMALL = (unsigned)min(2048, m * k);  // the compacted keys reuse the table area
  bool done = false;
  if (ns >= 4 * SUB && (int)s_valid >= 8 * r) {
    const int stride = ns / SUB;
    // valid keys of the subsample (slots past a list's end hold 0xFFFFFFFF)
    if (threadIdx.x == 0) s_cnt2 = 0;
    __syncthreads();
    unsigned int sv = 0;
    for (int i = threadIdx.x; i < SUB; i += blockDim.x) sv += keys[i * stride] != 0xFFFFFFFFu;
    atomicAdd(&s_cnt2, sv);
    __syncthreads();
    const unsigned int subv = s_cnt2;
    const unsigned int want = (unsigned)((3ull * (unsigned)r * subv + s_valid - 1) / s_valid) + 8u;  // rank in the subsample
    if (want < subv) {
      radix_kth(keys, SUB, stride, want);
      const unsigned int pivot = s_prefix;
      __syncthreads();
      if (threadIdx.x == 0) s_cnt2 = 0;
      __syncthreads();
      unsigned int* small = reinterpret_cast<unsigned int*>(su);  // the tables are not needed any more
      for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        const unsigned key = keys[i];
        if (key <= pivot) {
          const unsigned int p = atomicAdd(&s_cnt2, 1u);
          if (p < SMALL) small[p] = key;
        }
      }
      __syncthreads();
      const unsigned int nsm = s_cnt2;
      if (nsm >= (unsigned)r && nsm <= SMALL) {
        radix_kth(small, (int)nsm, 1, (unsigned)(r - 1));
        done = true;
      }
    }
  }
  if (!done) radix_kth(keys, ns, 1, (unsigned)(r - 1));
  if (threadIdx.x == 0) {
    const double t = (double)fkey_inv(s_prefix) + 2.0 * (double)aerr[q];
    float f = (float)t;
    if ((double)f < t) f = nextafterf(f, __int_as_float(0x7f800000));
    theta[q] = nextafterf(f, __int_as_float(0x7f800000));
  }
}

// per query: codes in its probed lists (the r_eff of the overflow check and the
// evaluation count); per launch: slot evaluations of the list scan including
// the idle slots of partly filled 8-query passes
__global__ void ivf_probed_kernel(const int64_t* __restrict__ cells, const int64_t* __restrict__ offsets, int64_t nq,
                                  int ma, int64_t* __restrict__ tot) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int64_t t = 0;
  for (int p = 0; p < ma; ++p) {
    const int64_t c = cells[q * ma + p];
    if (c >= 0) t += offsets[c + 1] - offsets[c];
  }
  tot[q] = t;
}
__global__ void ivf_slot_evals_kernel(const int* __restrict__ lcnt, const int64_t* __restrict__ offsets, int64_t K,
                                      int lq, unsigned long long* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (c < K) v = (unsigned long long)(offsets[c + 1] - offsets[c]) * (unsigned long long)lq *
                 (unsigned long long)((lcnt[c] + lq - 1) / lq);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

__global__ void pair_count_kernel(const int64_t* __restrict__ cells, int64_t npairs, int* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < npairs && cells[i] >= 0) atomicAdd(cnt + cells[i], 1);
}

// exclusive scan of K ints (single CTA, K up to a few million)
__global__ void scan_kernel(const int* __restrict__ in, int64_t K, int64_t* __restrict__ out) {
  __shared__ int64_t part[1024];
  const int64_t per = cdiv(K, blockDim.x);
  const int64_t b = threadIdx.x * per, e = min(b + per, K);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int64_t t = part[i];
      part[i] = acc;
      acc += t;
    }
  }
  __syncthreads();
  int64_t acc = part[threadIdx.x];
  for (int64_t i = b; i < e; ++i) {
    out[i] = acc;
    acc += in[i];
  }
  if (threadIdx.x == blockDim.x - 1) out[K] = acc;
}

__global__ void pair_fill_kernel(const int64_t* __restrict__ cells, const double* __restrict__ pdist, int64_t nq, int ma,
                                 const int64_t* __restrict__ starts, int* __restrict__ fill, int* __restrict__ pq,
                                 float* __restrict__ pa, int* __restrict__ pcell, const float* __restrict__ sub8,
                                 const float* __restrict__ qscale, const uint32_t* __restrict__ qtint,
                                 float* __restrict__ ps, uint32_t* __restrict__ pt, float* __restrict__ pas) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nq * ma) return;
  const int64_t c = cells[i];
  if (c < 0) return;
  const int slot = atomicAdd(fill + c, 1);
  const int64_t o = starts[c] + slot;
  const int q = (int)(i / ma);
  pq[o] = q;
  pa[o] = (float)pdist[i];
  pcell[o] = (int)c;
  if (sub8) {  // packed list scan: the pair's scale, threshold and scaled sub-space terms a_qj * s_q
    const float sc = qscale[q];
    ps[o] = sc;
    pt[o] = qtint[q];
    const float4 a0 = *reinterpret_cast<const float4*>(sub8 + i * 8), a1 = *reinterpret_cast<const float4*>(sub8 + i * 8 + 4);
    *reinterpret_cast<float4*>(pas + o * 8) = make_float4(a0.x * sc, a0.y * sc, a0.z * sc, a0.w * sc);
    *reinterpret_cast<float4*>(pas + o * 8 + 4) = make_float4(a1.x * sc, a1.y * sc, a1.z * sc, a1.w * sc);
  }
}

// One CTA per inverted list (two resident per SM); the queries probing it are
// processed 8 at a time ("slots"): their U tables are staged in shared memory
// interleaved as [entry*m + j][slot] (row stride 8 words), a quarter-warp
// evaluates one code for all 8 slots (lane = slot, the code's bytes are a
// broadcast read), so the 8 lookups of one table row hit the 8 banks of
// window (row mod 4) = (j mod 4) when m % 4 == 0.  The four quarter-warps of
// a warp visit the components in rotated orders (quarter-warp w reads
// component (t + w) mod m at step t), so one warp-wide lookup touches four
// distinct windows: conflict-free for any codes.  Survivors are staged per
// slot in shared memory and appended to the query's candidate list with one
// global reservation per (list, slot).
constexpr int LQ = 8;
constexpr int LROW = LQ;           // row stride (words) of the slot-interleaved tables
constexpr int LIST_THREADS = 512;
constexpr int LCH = 1024;          // codes per chunk
constexpr int LSTAGE = 256;        // staged survivors per slot

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// streaming copy (codes / V are read once per list): L2 evict-first, so the
// query tables stay resident
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async4_stream(void* smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "l"(pol)
               : "memory");
}

__device__ __forceinline__ uint32_t prmt_b(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ float2 lds_f32x2(uint32_t addr) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

template <int MT, int KT>  // compile-time (m, k), or (0, 0) for runtime values
__global__ void __launch_bounds__(LIST_THREADS, 2) ivf_list_kernel(
    const float* __restrict__ U, const int64_t* __restrict__ starts, const int* __restrict__ pq,
    const float* __restrict__ pa, const int64_t* __restrict__ offsets, const uint8_t* __restrict__ codes,
    const float* __restrict__ V, int m_rt, int k_rt, const float* __restrict__ theta, uint64_t* __restrict__ cand,
    float* __restrict__ cand_apx, int* __restrict__ cand_cnt, int64_t cap, const int* __restrict__ order) {
  const int m = MT > 0 ? MT : m_rt;
  const int k = KT > 0 ? KT : k_rt;
  extern __shared__ __align__(16) unsigned char lsm[];
  float* su = (float*)lsm;                                         // [m*k][LROW]
  uint32_t* scode = (uint32_t*)(su + (size_t)m * k * LROW);        // [LCH][m/4] (m % 4 == 0) or bytes
  float* sv = (float*)(scode + (size_t)LCH * ((m + 3) / 4));       // [LCH]
  uint32_t* sst = (uint32_t*)(sv + LCH);                           // [LQ][LSTAGE] list offsets
  float* ssa = (float*)(sst + LQ * LSTAGE);                        // [LQ][LSTAGE] filter distances
  __shared__ int s_cnt[LQ], s_q[LQ];
  __shared__ float s_a[LQ], s_th[LQ];
  const int64_t c = order ? order[blockIdx.x] : blockIdx.x;  // spatially grouped list order (query-table reuse in L2)
  const int64_t p0 = starts[c], p1 = starts[c + 1];
  if (p0 == p1) return;
  const int64_t b = offsets[c], e = offsets[c + 1];
  if (b == e) return;
  const int mk = m * k;
  const int mw = (m + 3) / 4;   // code words per code
  const int slot = threadIdx.x & (LQ - 1);
  const int hw = threadIdx.x / LQ, nhw = blockDim.x / LQ;
  const float* su_s = su + slot;
  // rotated lookups (MT % 4 == 0): byte offset of component (t + qw) mod MT
  // within an entry's block of MT rows, and the entry stride as a shift
  const int qw = (threadIdx.x >> 3) & 3;
  constexpr int eshift = MT > 0 ? 31 - __builtin_clz(MT * LROW * 4) : 0;
  constexpr bool PAIR = MT == 8 && KT == 256;
  const int qw2 = (threadIdx.x >> 2) & 3;
  uint32_t jb2[8];
#pragma unroll
  for (int t = 0; t < 8; ++t)
    jb2[t] = (uint32_t)__cvta_generic_to_shared(su) + 8 * (threadIdx.x & 3) + ((t + qw2) & 7) * LROW * 4;
  uint32_t jb[MT > 0 ? MT : 1];  // shared-window byte addresses
#pragma unroll
  for (int t = 0; t < (MT > 0 ? MT : 1); ++t)
    jb[t] = (uint32_t)__cvta_generic_to_shared(su_s) + (MT > 0 ? ((t + qw) % (MT > 0 ? MT : 1)) * LROW * 4 : 0);
  for (int64_t g0 = p0; g0 < p1; g0 += LQ) {
    const int ns = (int)min((int64_t)LQ, p1 - g0);
    __syncthreads();
    if (threadIdx.x < LQ) {
      const bool ok = threadIdx.x < ns;
      s_q[threadIdx.x] = ok ? pq[g0 + threadIdx.x] : 0;
      s_a[threadIdx.x] = ok ? pa[g0 + threadIdx.x] : 0.f;
      s_th[threadIdx.x] = ok ? theta[pq[g0 + threadIdx.x]] : -__int_as_float(0x7f800000);
      s_cnt[threadIdx.x] = 0;
    }
    __syncthreads();
    // stage the tables (asynchronous, completed with the first code chunk):
    // a warp copies runs of 8 consecutive entries (one 32 B sector) of 4
    // slots' tables; shared writes are 2-way conflicted at most
    {
      static_assert(LQ == 8 && LIST_THREADS % 64 == 0, "staging map assumes 8 slots");
      const int u = threadIdx.x & 7, g8 = threadIdx.x >> 3, sl = g8 & 7;
      if (sl < ns) {
        const float* src = U + (int64_t)s_q[sl] * mk;
        // 64 threads per slot: 8 runs of 8 consecutive entries per step
        for (int i = (g8 >> 3) * 8 + u; i < mk; i += 64) cp_async4(su + i * LROW + sl, src + i);
      }
    }
    const int q = s_q[slot];
    const float A = s_a[slot], th = s_th[slot];
    // idle slots (ns < LQ) read unstaged table rows: whatever they sum to
    // (even -inf) must not emit
    const bool live = slot < ns;
    const int ps0 = 2 * (threadIdx.x & 3);  // PAIR: this lane's slots ps0, ps0 + 1
    const int q0 = s_q[ps0], q1 = s_q[ps0 + 1];
    const float A0 = s_a[ps0], A1 = s_a[ps0 + 1], th0 = s_th[ps0], th1 = s_th[ps0 + 1];
    const bool live0 = ps0 < ns, live1 = ps0 + 1 < ns;
    for (int64_t cb = b; cb < e; cb += LCH) {
      const int nc = (int)min((int64_t)LCH, e - cb);
      __syncthreads();
      // codes and V of the chunk: asynchronous copies, all in flight at once
      const uint64_t pol = evict_first_policy();
      if ((m & 3) == 0) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(codes + cb * m);
        for (int i = threadIdx.x; i < nc * mw; i += blockDim.x) cp_async4_stream(scode + i, src + i, pol);
      } else {
        uint8_t* sc8 = (uint8_t*)scode;
        for (int i = threadIdx.x; i < nc * m; i += blockDim.x) sc8[i] = codes[cb * m + i];
      }
      for (int i = threadIdx.x; i < nc; i += blockDim.x) cp_async4_stream(sv + i, V + cb + i, pol);
      cp_async_wait_all();
      __syncthreads();
      auto emit = [&](int sl, int qs, float acc, int i) {
        const int pos = atomicAdd(&s_cnt[sl], 1);
        const uint32_t off = (uint32_t)(cb - b + i);
        if (pos < LSTAGE) {
          sst[sl * LSTAGE + pos] = off;
          ssa[sl * LSTAGE + pos] = acc;
        } else {  // stage full: direct append
          const int gp = atomicAdd(cand_cnt + qs, 1);
          if (gp < cap) {
            cand[(int64_t)qs * cap + gp] = ((uint64_t)c << 32) | (uint64_t)(uint32_t)(b + off);
            cand_apx[(int64_t)qs * cap + gp] = acc;
          }
        }
      };
      if constexpr (PAIR) {
        // 4 lanes per code, two slots per lane (one 8-byte lookup = the
        // entries of slots 2l, 2l+1): 8 codes per warp, each half-warp's four
        // codes in distinct bank windows (rotation by code index mod 4)
        for (int i = threadIdx.x >> 2; i < nc; i += LIST_THREADS / 4) {
          const uint32_t c0 = scode[2 * i], c1 = scode[2 * i + 1];  // broadcast to the 4 lanes
          const uint32_t r0 = __funnelshift_r(c0, c1, 8 * qw2), r1 = __funnelshift_r(c1, c0, 8 * qw2);
          float2 t8[8];
#pragma unroll
          for (int t = 0; t < 4; ++t) t8[t] = lds_f32x2(jb2[t] + (__byte_perm(r0, 0u, 0x4440 + t) << eshift));
#pragma unroll
          for (int t = 0; t < 4; ++t) t8[4 + t] = lds_f32x2(jb2[4 + t] + (__byte_perm(r1, 0u, 0x4440 + t) << eshift));
          const float vv = sv[i];
          const float s0 = ((t8[0].x + t8[1].x) + (t8[2].x + t8[3].x)) + ((t8[4].x + t8[5].x) + (t8[6].x + t8[7].x));
          const float s1 = ((t8[0].y + t8[1].y) + (t8[2].y + t8[3].y)) + ((t8[4].y + t8[5].y) + (t8[6].y + t8[7].y));
          const float acc0 = (A0 + vv) + s0, acc1 = (A1 + vv) + s1;
          if (live0 && acc0 <= th0) emit(ps0, q0, acc0, i);
          if (live1 && acc1 <= th1) emit(ps0 + 1, q1, acc1, i);
        }
        continue;
      }
      for (int i = hw; i < nc; i += nhw) {
        float acc = A + sv[i];
        if (MT > 0 && (MT & 3) == 0) {
          // rotated component order (conflict-free windows); the sum is
          // pairwise -- the filter bound holds for any summation order
          constexpr int W = MT >= 4 ? MT / 4 : 1;
          uint32_t cw[W], rot[W];
#pragma unroll
          for (int w = 0; w < W; ++w) cw[w] = scode[i * W + w];  // broadcast
#pragma unroll
          for (int w = 0; w < W; ++w) rot[w] = __funnelshift_r(cw[w], cw[(w + 1) % W], 8 * qw);
          float part[W];
#pragma unroll
          for (int w = 0; w < W; ++w) {
            float t4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
              t4[t] = lds_f32(jb[4 * w + t] + (__byte_perm(rot[w], 0u, 0x4440 + t) << eshift));
            part[w] = (t4[0] + t4[1]) + (t4[2] + t4[3]);
          }
#pragma unroll
          for (int w = 1; w < W; ++w) part[0] += part[w];
          acc += part[0];
        } else if ((m & 3) == 0) {
          for (int w = 0; w < mw; ++w) {
            const uint32_t cw = scode[i * mw + w];  // broadcast
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int j = 4 * w + t;
              acc += su_s[((int)((cw >> (8 * t)) & 255u) * m + j) * LROW];
            }
          }
        } else {
          const uint8_t* cd = (const uint8_t*)scode + i * m;
          for (int j = 0; j < m; ++j) acc += su_s[(cd[j] * m + j) * LROW];
        }
        if (live && acc <= th) emit(slot, q, acc, i);
      }
    }
    __syncthreads();
    // flush the staged survivors: one reservation per slot (warp w handles slot w)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < ns) {
      const int n = min(s_cnt[w], LSTAGE);
      const int qq = s_q[w];
      int base = 0;
      if (lane == 0 && n) base = atomicAdd(cand_cnt + qq, n);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (int i = lane; i < n; i += 32)
        if (base + i < cap) {
          cand[(int64_t)qq * cap + base + i] = ((uint64_t)c << 32) | (uint64_t)(uint32_t)(b + sst[w * LSTAGE + i]);
          cand_apx[(int64_t)qq * cap + base + i] = ssa[w * LSTAGE + i];
        }
    }
  }
}



// ------------------------------------------------------------------ K8p
// Packed list scan (m = 8, k = 256): an integer version of the list-major
// scan with two queries per table word, as in scan8.cu (K3p).  Per (list c,
// pass of 8 probing queries) the CTA builds the residual tables of the pass
// in shared memory,
//   T[j][e] = U_q[j][e] + W_c[j][e] + a_qj        (a_qj = ||q_j - c_j||^2)
//           = ||(q - c)_j - C_j[e]||^2 >= 0       (W_c[j][e] = 2 <c_j, C_j[e]>)
// -- no cancellation is left for the scan (the entries are true sub-space
// distances), so they quantise to 12-bit integers t' = min(4095, floor(s_q T))
// at a per-query power-of-two scale s_q that puts the query's threshold near
// 4080.  Word (e, j, h) = t'(slot h) | t'(slot h + 4) << 16 sits at byte
// e * 256 + par * 128 + j * 16 + h * 4 (par = pass parity: the two halves of a
// 256-byte row hold alternate passes), so one PRMT builds the offset (code
// byte into byte 1).  An octet of lanes (4 lanes x 2 slots) evaluates one
// code; the eight octets of a warp walk the components in rotated order
// (component (t + o) mod 8 at step t): one warp-wide LDS.32 reads eight
// disjoint 4-bank windows -- conflict-free, 64 lookups per wavefront, and a
// pass of 8 slots wastes no lanes on lists probed by few queries.
// Every code with L <= Tint_q becomes a candidate with the filter distance
// L / s_q, certified within aerr2_q of the reference distance (see
// ivf_qparams_kernel): the scan reads no per-code V, no fp32 tables and
// needs no fp32 re-filter.
constexpr int L8_Q = 8;
constexpr int L8_CH = 3072;    // codes per staged chunk
constexpr uint32_t L8_CLIP = 4095u;
constexpr double L8_TARGET = 4080.0;

// W[c][e * m + j] = 2 <c_j, C_j[e]> (fp64 -> fp32) and max |W|
__global__ void ivf_w_kernel(const float* __restrict__ coarse, const float* __restrict__ books, int m, int k, int dsub,
                             float* __restrict__ W, float* __restrict__ wmax) {
  const int64_t c = blockIdx.x;
  const int d = m * dsub;
  float mx = 0.f;
  for (int i = threadIdx.x; i < m * k; i += blockDim.x) {
    const int e = i / m, j = i - e * m;
    const float* cb = books + ((int64_t)j * k + e) * dsub;
    const float* g = coarse + c * d + j * dsub;
    double s = 0.0;
    for (int t = 0; t < dsub; ++t) s += (double)g[t] * (double)cb[t];
    const float w = (float)(2.0 * s);
    W[c * (int64_t)m * k + i] = w;
    mx = fmaxf(mx, fabsf(w));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(wmax), __float_as_int(mx));
}

// Per query: scale s_q = 2^e, integer threshold Tint_q and the certified error
// aerr2_q of the packed scan's filter distance L / s_q.
//  * theta_q >= (r-th smallest reference distance d_ref over the probed lists)
//    + aerr_q (ivf_theta_kernel), so every code the search can return has
//    D <= theta' = (theta + aerr)(1 + 4u): D is the exact sum of the exact
//    sub-space distances, d_ref the sum of their float32 roundings.
//  * one table entry: T32 = fl(fl(U32 + W32) + a32) with |U32 - U| <= u |U|,
//    |W32 - W| <= u |W|, |a32 - a| <= u a, so |T32 - T| <= epsT = 1.5 x 3u
//    (usum + wmax + amax) (|U| <= usum = sum_j max_e |U|, a <= max probe
//    distance).  The builder stores t' with  s max(T32, 0) - 2 < t' <=
//    s max(T32, 0)  unless it clips at 4095 (floor, minus one more on a
//    round-to-even tie of the magic-number conversion).
//  * hence  L <= s (D + m epsT)  for every code, and  s D <= L + 2 m + s m
//    epsT  for every code without a clipped entry.  Tint = floor(s theta') +
//    m + 2 < 4095 keeps every returnable code and rejects every clipped one,
//    so all candidates obey |(L + m) / s - d_ref| <= aerr2 = m / s + m epsT +
//    4u theta' (the candidates carry the centred estimate (L + m) / s).
// theta = +inf (sample shorter than r): s = 0 -- every probed code is kept.
__global__ void ivf_qparams_kernel(const float* __restrict__ U, const double* __restrict__ pdist,
                                   const float* __restrict__ theta, const float* __restrict__ aerr,
                                   const float* __restrict__ wmax, int64_t nq, int ma, int m, int k,
                                   float* __restrict__ qscale, uint32_t* __restrict__ qtint,
                                   float* __restrict__ aerr2) {
  const int64_t q = blockIdx.x;
  __shared__ double part[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double s = 0.0;
  for (int j = warp; j < m; j += nw) {
    float mx = 0.f;
    for (int i = lane; i < k; i += 32) mx = fmaxf(mx, fabsf(U[(q * k + i) * (int64_t)m + j]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    s += (double)mx;
  }
  if (lane == 0) part[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double usum = 0.0;
    for (int i = 0; i < nw; ++i) usum += part[i];
    double amax = 0.0;
    for (int p = 0; p < ma; ++p) amax = fmax(amax, pdist[q * ma + p]);
    const double u = 5.9604644775390625e-08;
    const double epsT = 1.5 * u * 3.0 * (usum + (double)wmax[0] + amax);
    const float th = theta[q];
    if (!(th < __int_as_float(0x7f800000))) {
      qscale[q] = 0.f;
      qtint[q] = L8_CLIP - 1u;
      aerr2[q] = __int_as_float(0x7f800000);
    } else {
      const double tp = ((double)th + (double)aerr[q]) * (1.0 + 4.0 * u) + (double)m * epsT;
      int e = 0;
      if (tp > 0.0) e = (int)floor(log2(L8_TARGET / tp));
      e = max(-100, min(100, e));
      qscale[q] = (float)ldexp(1.0, e);
      const double t = (tp > 0.0 ? floor(ldexp(tp, e)) : 0.0) + (double)m + 2.0;
      qtint[q] = t >= (double)(L8_CLIP - 1u) ? L8_CLIP - 1u : (uint32_t)t;
      // the candidates carry (L + m) / s: |(L + m) / s - D| <= m / s + m epsT
      const double a2 = ldexp((double)m, -e) + (double)m * epsT + 4.0 * u * tp;
      float f = (float)a2;
      if ((double)f < a2) f = nextafterf(f, __int_as_float(0x7f800000));
      aerr2[q] = f;
    }
  }
}

// one descriptor per list in scan order: the producer warps prefetch it
struct ListDesc {
  int c;          // cell
  int np;         // probing pairs
  int64_t p0;     // first pair
  int64_t b;      // first code
  int64_t n;      // codes
};
__global__ void ivf_desc_kernel(const int* __restrict__ order, const int64_t* __restrict__ starts,
                                const int64_t* __restrict__ offsets, int64_t K, ListDesc* __restrict__ desc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int64_t c = order ? order[i] : i;
  ListDesc d;
  d.c = (int)c;
  d.p0 = starts[c];
  d.np = (int)(starts[c + 1] - starts[c]);
  d.b = offsets[c];
  d.n = offsets[c + 1] - offsets[c];
  desc[i] = d;
}

struct List8Args {
  const float* U;         // [nq][k * m] (entry-major, component fastest)
  const float* W;         // [K][k * m]
  const ListDesc* desc;   // (K,) lists in scan order
  int64_t K;
  const int* pq;          // pair -> query
  const float* ps;        // pair -> scale
  const uint32_t* pt;     // pair -> integer threshold
  const float* pas;       // pair -> a_qj * s_q (8 per pair)
  const uint8_t* codes;   // (n, 8) row-major, list order
  uint64_t* cand;         // per query: list << 32 | position
  float* cand_apx;        // per query: L / s_q
  int* cand_cnt;
  int64_t cap;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}

// Persistent, warp-specialised: L8_PW producer warps fetch the list
// descriptors (CTA i takes lists i, i + grid, ... of the scan order, the next
// descriptor / W table / pass parameters prefetched in registers), stage the
// code chunks (cp.async) and build the packed tables of pass p + 1 while
// L8_CW consumer warps scan pass p.  Stages (one code chunk each, two
// buffers) and the two table halves are handed over with full / empty
// mbarriers; the candidate path is per consumer warp (own stage, no block
// barrier anywhere in the steady state).
constexpr int L8_PW = 8, L8_CW = 16;
constexpr int L8_PT = L8_PW * 32;
constexpr int L8_THREADS = (L8_PW + L8_CW) * 32;
constexpr int L8_WST = 96;     // staged candidates per consumer warp

struct L8Stage {   // what the consumers need to scan one chunk
  int nc;          // codes in the chunk; < 0: no more work
  uint32_t loff0;  // list offset of its first code
  int par;         // table half
  int last;        // last chunk of the pass: flush, release the table half
  int ns;          // live slots
  int c;           // cell
  int64_t b;       // list base position
  int q[L8_Q];
  float inv[L8_Q];
  uint32_t t[L8_Q];
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(L8_THREADS, 1) ivf_list8_kernel(List8Args a) {
  constexpr int M = 8, KK = 256, MK = M * KK;
  extern __shared__ __align__(256) unsigned char l8[];
  // the 64 KB table slot sits at a 64 KB-aligned shared-window address, so a
  // lookup address is one PRMT of the code byte into byte 1 of the lane's
  // base (no add); the code chunks and candidate stages fill the region
  // below it, the list table the region above
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(l8);
  const uint32_t slot_w = (sb + 65535u) & ~65535u;  // window address of the slot
  unsigned char* slot = l8 + (slot_w - sb);                              // 64 KB: packed tables, two interleaved halves
  float* sW = reinterpret_cast<float*>(slot + 65536);                    // [MK] list table (producers only)
  float* raw = sW + MK;                                                  // [L8_Q][MK] the pass's U tables (producers only)
  uint2* scode = reinterpret_cast<uint2*>(l8);                           // [2][L8_CH] code rows
  uint64_t* wst = reinterpret_cast<uint64_t*>(scode + 2 * L8_CH);        // [L8_CW][L8_WST] candidate records
  if (2u * L8_CH * 8u + L8_CW * L8_WST * 8u > slot_w - sb) __trap();
  __shared__ L8Stage sinfo[2];
  __shared__ __align__(8) uint64_t st_full[2], st_empty[2], tab_empty[2], raw_full;
  __shared__ int pp_q[2][L8_Q], s_wcnt[L8_CW];
  __shared__ float pp_s[2][L8_Q], pp_as[2][L8_Q][M];
  __shared__ uint32_t pp_t[2][L8_Q];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&st_full[i], 1);
      tc::mbar_init(&st_empty[i], L8_CW);
      tc::mbar_init(&tab_empty[i], L8_CW);
    }
    tc::mbar_init(&raw_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp < L8_PW) {
    // =============================== producers ===============================
    // Everything a pass needs from global memory is requested one pass ahead:
    // the next list's descriptor and W slice and the next pass's parameters
    // travel in registers, the next pass's eight raw U tables (64 KB) in a
    // TMA bulk copies (one 8 KB copy per slot) that land during the current
    // build -- the build itself reads shared memory only.
    const int ptid = threadIdx.x;
    const int bj = lane & 7, be = lane >> 3;
    int sidx = 0, pc = 0;  // stage and pass counters (buffer = & 1)
    for (int i = ptid; i < L8_Q * MK / 4; i += L8_PT) reinterpret_cast<float4*>(raw)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the zero fill is ordered before the bulk copies
    // list cursor: `d` current, `nd` / wreg the prefetched next live list
    ListDesc nd;
    nd.np = 0;
    nd.n = 0;
    float wreg[MK / L8_PT];
    int64_t nli = (int64_t)blockIdx.x - gridDim.x;
    bool more = true;
    auto fetch_list = [&]() {  // advance to the next list with work (descriptor + W slice into registers)
      for (;;) {
        nli += gridDim.x;
        if (nli >= a.K) {
          more = false;
          return;
        }
        nd = a.desc[nli];
        if (nd.np > 0 && nd.n > 0) break;
      }
#pragma unroll
      for (int i = 0; i < MK / L8_PT; ++i) wreg[i] = __ldg(a.W + (int64_t)nd.c * MK + ptid + i * L8_PT);
    };
    // pass parameters in registers: thread t < 8 -> (q, s, tint) of slot t; threads 32..95 -> a_qj * s_q
    int rq = 0;
    float rs = 0.f, ras = 0.f;
    uint32_t rt = 0;
    auto fetch_pass = [&](const ListDesc& dd, int g0) {
      const int ns = min(L8_Q, dd.np - g0);
      if (ptid < L8_Q) {
        const bool ok = ptid < ns;
        rq = ok ? a.pq[dd.p0 + g0 + ptid] : 0;
        rs = ok ? a.ps[dd.p0 + g0 + ptid] : 0.f;
        rt = ok ? a.pt[dd.p0 + g0 + ptid] : 0u;
      } else if (ptid >= 32 && ptid < 32 + L8_Q * M) {
        const int t = ptid - 32;
        ras = (t >> 3) < ns ? a.pas[(dd.p0 + g0) * M + t] : 0.f;
      }
    };
    auto store_pass = [&](int pb) {
      if (ptid < L8_Q) {
        pp_q[pb][ptid] = rq;
        pp_s[pb][ptid] = rs;
        pp_t[pb][ptid] = rt;
      } else if (ptid >= 32 && ptid < 32 + L8_Q * M) {
        pp_as[pb][(ptid - 32) >> 3][(ptid - 32) & 7] = ras;
      }
    };
    auto issue_raw = [&](int pb, int ns) {  // one 8 KB bulk copy (TMA) per live slot, completing on raw_full
      if (ptid == 0) {
        tc::mbar_expect_tx(&raw_full, (uint32_t)ns * MK * 4u);
        for (int sl = 0; sl < ns; ++sl)
          tc::bulk_g2s(raw + sl * MK, a.U + (int64_t)pp_q[pb][sl] * MK, MK * 4u, &raw_full);
      }
    };
    fetch_list();
    if (more) {
      ListDesc d = nd;
      int g0 = 0;
      bool new_list = true;
      fetch_pass(d, 0);
      store_pass(0);
      named_bar_sync(1, L8_PT);
      issue_raw(0, min(L8_Q, d.np));
      for (;;) {  // one iteration per pass
        const int ns = min(L8_Q, d.np - g0);
        const int par = pc & 1, pb = pc & 1;
        if (new_list) {
          named_bar_sync(1, L8_PT);  // the previous list's builds are done with sW
#pragma unroll
          for (int i = 0; i < MK / L8_PT; ++i) sW[ptid + i * L8_PT] = wreg[i];
          fetch_list();  // the list after this one: in flight during this list
          new_list = false;
        }
        // the pass after this one
        const bool last_pass = g0 + L8_Q >= d.np;
        const bool have_next = !last_pass || more;
        const ListDesc dn = last_pass ? nd : d;
        const int gn = last_pass ? 0 : g0 + L8_Q;
        if (have_next) fetch_pass(dn, gn);
        bool built = false;
        for (int64_t cb = 0; cb < d.n; cb += L8_CH, ++sidx) {
          const int nc = (int)min((int64_t)L8_CH, d.n - cb);
          const int buf = sidx & 1;
          if (ptid == 0) tc::mbar_wait(&st_empty[buf], (uint32_t)(((sidx >> 1) & 1) ^ 1));
          named_bar_sync(1, L8_PT);  // one thread polls, the others park on the hardware barrier
          {
            const uint2* src = reinterpret_cast<const uint2*>(a.codes) + d.b + cb;
            uint2* dst = scode + buf * L8_CH;
            for (int i = ptid; i < nc; i += L8_PT) cp_async8(dst + i, src + i);
            asm volatile("cp.async.commit_group;" ::: "memory");
          }
          if (!built) {
            built = true;
            if (ptid == 0) {
              tc::mbar_wait(&tab_empty[par], (uint32_t)(((pc >> 1) & 1) ^ 1));
              tc::mbar_wait(&raw_full, (uint32_t)(pc & 1));  // this pass's raw tables landed
            }
            named_bar_sync(1, L8_PT);
            tc::mbar_wait(&raw_full, (uint32_t)(pc & 1));  // passes at once: every reader observes the phase itself
            // ---- table build from shared memory: 8 loads (one per slot), 4 packed words, one STS.128
            {
              float as[L8_Q], sc[L8_Q];
#pragma unroll
              for (int i = 0; i < L8_Q; ++i) {
                as[i] = pp_as[pb][i][bj];
                sc[i] = pp_s[pb][i];
              }
#pragma unroll 2
              for (int e0 = warp * 4 + be; e0 < KK; e0 += 4 * L8_PW) {
                const float wv = sW[e0 * M + bj];
                uint32_t tq[L8_Q];
#pragma unroll
                for (int i = 0; i < L8_Q; ++i) {
                  float x = fmaf(raw[i * MK + e0 * M + bj] + wv, sc[i], as[i]);
                  x = fminf(fmaxf(x, 0.5f), (float)L8_CLIP + 0.5f);
                  tq[i] = __float_as_uint(x + 8388607.5f);  // low 16 bits: floor(x), or floor(x) - 1 on a rounding tie
                }
                uint4 w4;  // one PRMT packs the low halves of two slots' words
                w4.x = __byte_perm(tq[0], tq[4], 0x5410);
                w4.y = __byte_perm(tq[1], tq[5], 0x5410);
                w4.z = __byte_perm(tq[2], tq[6], 0x5410);
                w4.w = __byte_perm(tq[3], tq[7], 0x5410);
                *reinterpret_cast<uint4*>(slot + e0 * 256 + par * 128 + bj * 16) = w4;
              }
            }
            named_bar_sync(1, L8_PT);  // every thread is done with raw and pp[pb ^ 1]'s previous user
            if (have_next) {
              store_pass(pb ^ 1);
              named_bar_sync(1, L8_PT);
              issue_raw(pb ^ 1, min(L8_Q, dn.np - gn));
            }
          }
          asm volatile("cp.async.wait_group 0;" ::: "memory");  // the code chunk
          if (ptid == 0) {
            L8Stage& si = sinfo[buf];
            si.nc = nc;
            si.loff0 = (uint32_t)cb;
            si.par = par;
            si.last = cb + L8_CH >= d.n ? 1 : 0;
            si.ns = ns;
            si.c = d.c;
            si.b = d.b;
          }
          if (ptid < L8_Q) {
            L8Stage& si = sinfo[buf];
            si.q[ptid] = pp_q[pb][ptid];
            si.inv[ptid] = pp_s[pb][ptid] > 0.f ? 1.0f / pp_s[pb][ptid] : 0.f;  // exact: a power of two
            si.t[ptid] = pp_t[pb][ptid];
          }
          named_bar_sync(1, L8_PT);  // tables, codes and the stage record are written
          if (ptid == 0) tc::mbar_arrive(&st_full[buf]);
        }
        ++pc;
        if (!have_next) break;
        if (last_pass) {
          d = dn;
          g0 = 0;
          new_list = true;
        } else {
          g0 += L8_Q;
        }
      }
    }
    // no more work
    {
      const int buf = sidx & 1;
      tc::mbar_wait(&st_empty[buf], (uint32_t)(((sidx >> 1) & 1) ^ 1));
      if (ptid == 0) {
        sinfo[buf].nc = -1;
        tc::mbar_arrive(&st_full[buf]);
      }
    }
  } else {
    // =============================== consumers ===============================
    // A duet of lanes evaluates one code: lane h2 of the duet reads the two
    // adjacent words (slots 2 h2 | 2 h2 + 4 and 2 h2 + 1 | 2 h2 + 5) of a
    // table row with one LDS.64 -- one address PRMT and two adds per four
    // lookups.  The 16 duets of a warp take 16 codes; duets d and d + 8 share
    // a component window (rotation (t + d) mod 8), which a 64-bit access
    // spends as its second wavefront anyway.
    const int cw = warp - L8_PW;
    const int o = lane >> 1, h2 = lane & 1;
    const int rsh = 8 * (o & 3);
    const bool rswap = (o & 4) != 0;
    uint64_t* mst = wst + cw * L8_WST;  // this warp's candidate stage
    int* mcnt = &s_wcnt[cw];            // its fill count (shared atomics of the hitting lanes)
    if (lane == 0) *mcnt = 0;
    __syncwarp();
    for (int sidx = 0;; ++sidx) {
      const int buf = sidx & 1;
      tc::mbar_wait(&st_full[buf], (uint32_t)((sidx >> 1) & 1));
      const L8Stage& si = sinfo[buf];
      const int nc = si.nc;
      if (nc < 0) break;
      const int ns = si.ns;
      const uint32_t par = (uint32_t)si.par * 128u;
      // accumulator A: slots 2 h2 (low half) and 2 h2 + 4 (high); B: 2 h2 + 1 and 2 h2 + 5
      const int sA = 2 * h2, sB = 2 * h2 + 1;
      const uint32_t thA = (sA < ns ? si.t[sA] : 0u) | ((sA + 4 < ns ? si.t[sA + 4] : 0u) << 16) | 0x80008000u;
      const uint32_t thB = (sB < ns ? si.t[sB] : 0u) | ((sB + 4 < ns ? si.t[sB + 4] : 0u) << 16) | 0x80008000u;
      const uint32_t vmA = (sA < ns ? 0x8000u : 0u) | (sA + 4 < ns ? 0x80000000u : 0u);
      const uint32_t vmB = (sB < ns ? 0x8000u : 0u) | (sB + 4 < ns ? 0x80000000u : 0u);
      const uint32_t loff0 = si.loff0;
      // candidate record (list offset | L << 32 | slot << 48) -> the query's list
      auto append = [&](uint64_t rcd) {
        const int sl = (int)(rcd >> 48);
        const int qs = si.q[sl];
        const int gp = atomicAdd(a.cand_cnt + qs, 1);
        if (gp < a.cap) {
          a.cand[(int64_t)qs * a.cap + gp] = ((uint64_t)(uint32_t)si.c << 32) | (uint64_t)(uint32_t)(si.b + (uint32_t)rcd);
          // centred estimate: s D lies in [L - s m epsT, L + 2 m + s m epsT]
          a.cand_apx[(int64_t)qs * a.cap + gp] = (float)(((uint32_t)(rcd >> 32) & 0x7FFFu) + 8u) * si.inv[sl];
        }
      };
      auto flush = [&]() {
        __syncwarp();
        const int n = min(*reinterpret_cast<volatile int*>(mcnt), L8_WST);
        for (int i = lane; i < n; i += 32) {
          const uint64_t rcd = mst[i];
          if (rcd != ~0ull) append(rcd);
        }
        __syncwarp();
        if (lane == 0) *mcnt = 0;
        __syncwarp();
      };
      // one packed sum -> its (at most two) candidates
      auto emit = [&](uint32_t hit, uint32_t acc, int slo, uint32_t loff) {
        const uint32_t two = hit & (hit << 16);
        const int sp = atomicAdd(mcnt, two ? 2 : 1);
        const uint32_t m0 = (acc & 0x7FFFu) | ((uint32_t)slo << 16);  // L | slot << 16
        const uint32_t m1 = ((acc >> 16) & 0x7FFFu) | ((uint32_t)(slo + 4) << 16);
        uint2* m2 = reinterpret_cast<uint2*>(mst);
        if (sp + 2 <= L8_WST) {
          m2[sp] = make_uint2(loff, (hit & 0x8000u) ? m0 : m1);
          if (two) m2[sp + 1] = make_uint2(loff, m1);
        } else {  // stage full: direct append (a skipped last slot is marked)
          if (sp == L8_WST - 1) mst[sp] = ~0ull;
          if (hit & 0x8000u) append((uint64_t)loff | ((uint64_t)m0 << 32));
          if (hit & 0x80000000u) append((uint64_t)loff | ((uint64_t)m1 << 32));
        }
      };
      uint32_t lbase[M];
#pragma unroll
      for (int t = 0; t < M; ++t) lbase[t] = slot_w + par + (uint32_t)(((t + o) & 7) * 16 + h2 * 8);
      const uint2* sc = scode + buf * L8_CH;
      constexpr int ILP = 2, STEP = 16 * L8_CW;
      for (int ib = cw * 16; ib < nc; ib += ILP * STEP) {  // warp-uniform trip count
        const int i0 = ib + o;
        if (*reinterpret_cast<volatile int*>(mcnt) > L8_WST / 2) flush();  // warp-uniform: only this warp changes it
        uint32_t accA[ILP], accB[ILP];
        uint2 cwd[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) cwd[u] = sc[min(i0 + u * STEP, nc - 1)];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
          const uint32_t x = rswap ? cwd[u].y : cwd[u].x, y = rswap ? cwd[u].x : cwd[u].y;
          const uint32_t r0 = __funnelshift_r(x, y, rsh), r1 = __funnelshift_r(y, x, rsh);
          uint32_t sa = 0u, sb2 = 0u;
#pragma unroll
          for (int t = 0; t < M; ++t) {
            uint32_t va, vb;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                         : "=r"(va), "=r"(vb)
                         : "r"(prmt_b(t < 4 ? r0 : r1, lbase[t], 0x7604u | ((uint32_t)(t & 3) << 4))));
            sa += va;
            sb2 += vb;
          }
          accA[u] = sa;
          accB[u] = sb2;
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
          const int i = i0 + u * STEP;
          const uint32_t hitA = i < nc ? (thA - accA[u]) & vmA : 0u;
          const uint32_t hitB = i < nc ? (thB - accB[u]) & vmB : 0u;
          if (hitA | hitB) {  // rare per lane; kept small
            const uint32_t loff = loff0 + (uint32_t)i;
            if (hitA) emit(hitA, accA[u], sA, loff);
            if (hitB) emit(hitB, accB[u], sB, loff);
          }
        }
      }
      if (si.last) {
        flush();  // reads the stage record: before the release below
        if (lane == 0) tc::mbar_arrive(&tab_empty[si.par]);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&st_empty[buf]);
    }
  }
}

// After the list scan: every probed code with filter distance <= theta is a
// candidate, and theta >= the r-th smallest filter distance, so the r-th
// smallest candidate filter distance is the r-th smallest overall; a code can
// only be in the exact top-r if its filter distance is within 2 * aerr of it
// (|filter - exact| <= aerr).  Those candidates are compacted into out (count
// cnt2) for the exact re-score; lists past cap are left whole (the caller's
// fallback re-runs those queries).
constexpr int CT_THREADS = 256;
constexpr int CT_SMEM = 4096;

__global__ void __launch_bounds__(CT_THREADS) ivf_cand_theta_kernel(const uint64_t* __restrict__ cand,
                                                                    const float* __restrict__ apx,
                                                                    const int* __restrict__ cand_cnt, int64_t cap,
                                                                    int r, const float* __restrict__ aerr,
                                                                    uint64_t* __restrict__ out, int* __restrict__ cnt2) {
  __shared__ unsigned int keys[CT_SMEM];
  __shared__ unsigned int hist[256];
  __shared__ unsigned int s_prefix, s_k;
  __shared__ int s_n;
  const int64_t q = blockIdx.x;
  const int64_t M = min((int64_t)cand_cnt[q], cap);
  const uint64_t* cq = cand + q * cap;
  const float* aq = apx + q * cap;
  uint64_t* oq = out + q * cap;
  float th2 = __int_as_float(0x7f800000);
  if (cand_cnt[q] <= cap && M > r && M <= CT_SMEM) {
    for (int i = threadIdx.x; i < M; i += blockDim.x) keys[i] = fkey(aq[i]);
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_k = (unsigned)(r - 1);
    }
    __syncthreads();
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const unsigned prefix = s_prefix;
      for (int i = threadIdx.x; i < M; i += blockDim.x) {
        const unsigned key = keys[i];
        const bool match = (shift == 24) ? true : ((key ^ prefix) >> (shift + 8)) == 0;
        if (match) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        unsigned int s8 = 0;
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) s8 += hist[lane * 8 + bb];
        unsigned int incl = s8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const unsigned int kk = s_k, excl = incl - s8;
        if (kk >= excl && kk < incl) {
          unsigned int cc = excl;
          int d = lane * 8;
          for (int bb = 0; bb < 8; ++bb) {
            const unsigned int h = hist[lane * 8 + bb];
            if (kk < cc + h) {
              d = lane * 8 + bb;
              break;
            }
            cc += h;
          }
          s_k = kk - cc;
          s_prefix = prefix | ((unsigned)d << shift);
        }
      }
      __syncthreads();
    }
    const double t = (double)fkey_inv(s_prefix) + 2.0 * (double)aerr[q];
    float f = (float)t;
    if ((double)f < t) f = nextafterf(f, __int_as_float(0x7f800000));
    th2 = nextafterf(f, __int_as_float(0x7f800000));
  }
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    if (aq[i] <= th2) {
      const int p = atomicAdd(&s_n, 1);
      oq[p] = cq[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cnt2[q] = s_n;
}

// K6 for IVF: exact fp64 re-score of every candidate (list << 32 | pos), in
// place: the slot gets dkey(distance), pids the stored id.  Reference
// arithmetic (query_ivf, ivf.py:179-183 -> compute_tables scan.py:45-56 ->
// scan_distances scan.py:77-81): r = fp64(q) - fp64(coarse[c]); table entry
// j = fp32(sum_t (r_t - C_j[code_j][t])^2) summed over t in order; distance =
// fp64 sum over j in order.  8 lanes per candidate (lane j0 builds entries
// j0, j0 + 8, ...), the ordered j-sum by shuffles; grid (query, slice).
constexpr int RERANK_THREADS = 256;

template <int DSUB>  // compile-time sub-space dimension (all loads of a sub-space in flight), 0: runtime
__global__ void __launch_bounds__(RERANK_THREADS, 4) ivf_rerank_kernel(
    uint64_t* __restrict__ cand, const int* __restrict__ cand_cnt, int64_t cap, const int64_t* __restrict__ ids,
    QVec queries, const float* __restrict__ coarse, const float* __restrict__ books,
    const uint8_t* __restrict__ codes, int m, int k, int d, int dsub_rt, int64_t* __restrict__ pids) {
  const int dsub = DSUB > 0 ? DSUB : dsub_rt;
  const int64_t q = blockIdx.x;
  const int64_t M = min((int64_t)cand_cnt[q], cap);
  uint64_t* cq = cand + q * cap;
  int64_t* iq = pids + q * cap;
  const QVec qv = queries.offset(q * (int64_t)d);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane >> 3, j0 = lane & 7;
  const int64_t step = (int64_t)gridDim.y * (RERANK_THREADS / 32) * 4;
  for (int64_t base = ((int64_t)blockIdx.y * (RERANK_THREADS / 32) + warp) * 4; base < M; base += step) {
    const int64_t i = base + sub;
    const bool valid = i < M;
    const uint64_t e = valid ? cq[i] : 0ull;
    const int64_t pos = (int64_t)(uint32_t)e;
    const int64_t c = (int64_t)(e >> 32);
    const float* g = coarse + c * (int64_t)d;
    const uint8_t* code = codes + pos * (int64_t)m;
    double acc = 0.0;
    for (int jb = 0; jb < m; jb += 8) {
      const int j = jb + j0;
      float tf = 0.f;
      if (valid && j < m) {
        const float* cb = books + ((int64_t)j * k + code[j]) * dsub;
        double t = 0.0;
        if constexpr (DSUB > 0 && DSUB % 4 == 0) {
          // the sub-space's coordinates of the centroid and the codeword as
          // 16-byte loads, all issued before the ordered fp64 sum
          float gv[DSUB], cv[DSUB];
          double qd[DSUB];
#pragma unroll
          for (int s4 = 0; s4 < DSUB / 4; ++s4) {
            const float4 a4 = __ldg(reinterpret_cast<const float4*>(g + j * DSUB) + s4);
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(cb) + s4);
            gv[4 * s4] = a4.x, gv[4 * s4 + 1] = a4.y, gv[4 * s4 + 2] = a4.z, gv[4 * s4 + 3] = a4.w;
            cv[4 * s4] = b4.x, cv[4 * s4 + 1] = b4.y, cv[4 * s4 + 2] = b4.z, cv[4 * s4 + 3] = b4.w;
          }
#pragma unroll
          for (int s2 = 0; s2 < DSUB; ++s2) qd[s2] = qv.at(j * DSUB + s2);
#pragma unroll
          for (int s2 = 0; s2 < DSUB; ++s2) {
            const double rr = __dsub_rn(qd[s2], (double)gv[s2]);
            const double df = __dsub_rn(rr, (double)cv[s2]);
            t = __dadd_rn(t, __dmul_rn(df, df));
          }
        } else {
          for (int s2 = 0; s2 < dsub; ++s2) {
            const int dd = j * dsub + s2;
            const double rr = __dsub_rn(qv.at(dd), (double)__ldg(g + dd));
            const double df = __dsub_rn(rr, (double)__ldg(cb + s2));
            t = __dadd_rn(t, __dmul_rn(df, df));
          }
        }
        tf = __double2float_rn(t);
      }
      const int nj = min(8, m - jb);
      for (int u = 0; u < nj; ++u) acc = __dadd_rn(acc, (double)__shfl_sync(0xffffffffu, tf, (sub << 3) + u));
    }
    if (valid && j0 == 0) {
      cq[i] = dkey(acc);
      iq[i] = ids[pos];
    }
  }
}

// fallback: every code of the query's probed lists becomes a candidate
__global__ void ivf_all_kernel(const int64_t* __restrict__ cells_row, int ma, const int64_t* __restrict__ offsets,
                               uint64_t* __restrict__ cand, int* __restrict__ cnt, int64_t cap) {
  for (int p = 0; p < ma; ++p) {
    const int64_t c = cells_row[p];
    if (c < 0) continue;
    const int64_t b = offsets[c], e = offsets[c + 1];
    for (int64_t pos = b + threadIdx.x; pos < e; pos += blockDim.x) {
      const int s = atomicAdd(cnt, 1);
      if (s < cap) cand[s] = ((uint64_t)c << 32) | (uint64_t)(uint32_t)pos;
    }
  }
}

}  // namespace

void ivf_destroy_impl(pqs_ivf* iv);
int probe_build_index(pqs_ctx* ctx, pqs_ivf* iv);

// ---------------------------------------------------------------------------
int device_max_u8(pqs_ctx* ctx, const uint8_t* d, int64_t count, int* out);

// coarse, codes and ids: host or device pointers (io); list_sizes: host
int ivf_create_impl(pqs_ctx* ctx, const pqs_pq* pq, const float* coarse, int64_t K, const int64_t* list_sizes,
                    const uint8_t* codes, const int64_t* ids, int io, pqs_ivf** out) {
  *out = nullptr;
  PQS_CHECK(ctx, K >= 1, "need at least one coarse centroid");
  PQS_CHECK(ctx, pq->k <= 256, "IVF lists need b <= 8");
  std::vector<int64_t> offs(K + 1, 0);
  int64_t mx = 0;
  for (int64_t c = 0; c < K; ++c) {
    PQS_CHECK(ctx, list_sizes[c] >= 0, "list sizes must be >= 0");
    offs[c + 1] = offs[c] + list_sizes[c];
    mx = std::max(mx, list_sizes[c]);
  }
  const int64_t n = offs[K];
  PQS_CHECK(ctx, n < (1ll << 32), "an IVF shard holds at most 2^32 - 1 codes");
  PQS_CHECK(ctx, K < (1ll << 31), "K must be < 2^31");
  (void)io;  // copies below use cudaMemcpyDefault (host or device sources)
  pqs_ivf* iv = new pqs_ivf();
  iv->K = K;
  iv->n = n;
  iv->m = pq->m;
  iv->k = pq->k;
  iv->d = pq->d;
  iv->dsub = pq->dsub;
  iv->h_offsets = offs;
  iv->max_list = mx;
  const int d = pq->d;
  auto al = [&](void** p, size_t bytes) { return cudaMalloc(p, std::max<size_t>(bytes, 16)) == cudaSuccess; };
  bool ok = al((void**)&iv->coarse, (size_t)K * d * 4) && al((void**)&iv->cnorm, (size_t)K * 8) && al((void**)&iv->cnormf, (size_t)K * 4) &&
            al((void**)&iv->books, (size_t)pq->m * pq->k * pq->dsub * 4) && al((void**)&iv->offsets, (size_t)(K + 1) * 8) &&
            al((void**)&iv->codes, (size_t)n * pq->m) && al((void**)&iv->ids, (size_t)n * 8) &&
            al((void**)&iv->gnorm, (size_t)K * 4 /* gnorm */ + 16) && al((void**)&iv->vtab, (size_t)n * 4) &&
            al((void**)&iv->vmax, 16);
  if (!ok) {
    cudaGetLastError();
    ivf_destroy_impl(iv);
    return set_err(ctx, PQS_ERR_NOMEM, "IVF allocation failed");
  }
  PQS_TRY(upload(ctx, iv->coarse, coarse, (size_t)K * d * 4));
  PQS_TRY(upload(ctx, iv->books, pq->books, (size_t)pq->m * pq->k * pq->dsub * 4));
  PQS_TRY(upload(ctx, iv->offsets, offs.data(), (size_t)(K + 1) * 8));
  if (n) {
    PQS_TRY(upload(ctx, iv->codes, codes, (size_t)n * pq->m));
    PQS_TRY(upload(ctx, iv->ids, ids, (size_t)n * 8));
    int maxc = 0;
    PQS_TRY(device_max_u8(ctx, iv->codes, n * pq->m, &maxc));
    if (maxc >= pq->k) {
      ivf_destroy_impl(iv);
      return set_err(ctx, PQS_ERR_INVALID, "code component out of range");
    }
  }
  PQS_CUDA(ctx, cudaMemsetAsync(iv->vmax, 0, 16, ctx->stream));
  cnorm_kernel<<<(unsigned)cdiv(K, 256), 256, 0, ctx->stream>>>(iv->coarse, K, d, iv->cnorm, iv->gnorm, iv->cnormf);
  PQS_LAUNCHED(ctx);
  {
    const int st = probe_build_index(ctx, iv);
    if (st != PQS_OK) {
      cudaGetLastError();
      ivf_destroy_impl(iv);
      return st;
    }
  }
  v_kernel<<<(unsigned)K, 256, 0, ctx->stream>>>(iv->coarse, iv->books, iv->offsets, iv->codes, iv->m, iv->k, iv->dsub,
                                                 d, iv->vtab, iv->vmax);
  PQS_LAUNCHED(ctx);
  // W tables of the packed list scan (m = 8, k = 256): K x 8 KB
  static const int use_w = getenv("PQS_IVF_W") ? atoi(getenv("PQS_IVF_W")) : 1;
  if (use_w && iv->m == 8 && iv->k == 256) {
    if (cudaMalloc(&iv->wtab, (size_t)K * iv->m * iv->k * 4) == cudaSuccess && cudaMalloc(&iv->wmax, 16) == cudaSuccess) {
      PQS_CUDA(ctx, cudaMemsetAsync(iv->wmax, 0, 16, ctx->stream));
      ivf_w_kernel<<<(unsigned)K, 256, 0, ctx->stream>>>(iv->coarse, iv->books, iv->m, iv->k, iv->dsub, iv->wtab,
                                                        iv->wmax);
      PQS_LAUNCHED(ctx);
    } else {  // no room: the float list scan needs no W
      cudaGetLastError();
      if (iv->wtab) cudaFree(iv->wtab);
      iv->wtab = nullptr;
    }
  }
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  // list scan order: cells grouped by their nearest of P = sqrt(K) pivot cells
  // (PQS_LIST_ORDER=0 keeps cell order)
  static const int use_order = getenv("PQS_LIST_ORDER") ? atoi(getenv("PQS_LIST_ORDER")) : 1;
  if (use_order && K >= 1024) {
    int P = 1;
    while ((int64_t)P * P < K) ++P;
    int* asg = nullptr;
    PQS_CUDA(ctx, cudaMalloc(&asg, sizeof(int) * K));
    pivot_assign_kernel<<<(unsigned)cdiv(K, 128), 128, 0, ctx->stream>>>(iv->coarse, K, d, P, asg);
    PQS_LAUNCHED(ctx);
    std::vector<int> ha((size_t)K), ord((size_t)K);
    const int dl = download(ctx, ha.data(), asg, sizeof(int) * K);
    cudaFree(asg);
    PQS_TRY(dl);
    for (int64_t c = 0; c < K; ++c) ord[c] = (int)c;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return ha[x] < ha[y]; });
    PQS_CUDA(ctx, cudaMalloc(&iv->list_order, sizeof(int) * K));
    PQS_TRY(upload(ctx, iv->list_order, ord.data(), sizeof(int) * K));
  }
  // gmax on host
  std::vector<float> gn(K);
  PQS_TRY(download(ctx, gn.data(), iv->gnorm, (size_t)K * 4));
  float gm = 0.f;
  for (float v : gn) gm = std::max(gm, v);
  iv->gmax = gm;
  *out = iv;
  return PQS_OK;
}

// Coarse-only handle (no lists, no residual quantizer): what the probe needs
// to answer nearest / nearest_k over a centroid set (_dist.py:24-67), used by
// pqs_nearest for the index build's assignment (ivf.py:122).
int coarse_index_create(pqs_ctx* ctx, const float* centroids, int64_t K, int d, pqs_ivf** out) {
  *out = nullptr;
  PQS_CHECK(ctx, K >= 1 && K < (1ll << 31), "need 1 <= K < 2^31 centroids");
  PQS_CHECK(ctx, d >= 1, "d must be >= 1");
  pqs_ivf* iv = new pqs_ivf();
  iv->K = K;
  iv->d = d;
  auto al = [&](void** p, size_t bytes) { return cudaMalloc(p, std::max<size_t>(bytes, 16)) == cudaSuccess; };
  if (!(al((void**)&iv->coarse, (size_t)K * d * 4) && al((void**)&iv->cnorm, (size_t)K * 8) &&
        al((void**)&iv->cnormf, (size_t)K * 4) && al((void**)&iv->gnorm, (size_t)K * 4 + 16))) {
    cudaGetLastError();
    ivf_destroy_impl(iv);
    return set_err(ctx, PQS_ERR_NOMEM, "centroid allocation failed");
  }
  int st = upload(ctx, iv->coarse, centroids, (size_t)K * d * 4);
  if (st == PQS_OK) {
    cnorm_kernel<<<(unsigned)cdiv(K, 256), 256, 0, ctx->stream>>>(iv->coarse, K, d, iv->cnorm, iv->gnorm, iv->cnormf);
    ctx->launches++;
    st = probe_build_index(ctx, iv);
  }
  std::vector<float> gn(K);
  if (st == PQS_OK) st = download(ctx, gn.data(), iv->gnorm, (size_t)K * 4);
  if (st != PQS_OK) {
    cudaGetLastError();
    ivf_destroy_impl(iv);
    return st;
  }
  float gm = 0.f;
  for (float v : gn) gm = std::max(gm, v);
  iv->gmax = gm;
  *out = iv;
  return PQS_OK;
}

void ivf_destroy_impl(pqs_ivf* iv) {
  if (!iv) return;
  cudaFree(iv->coarse);
  cudaFree(iv->gnorm);
  cudaFree(iv->cnorm);
  cudaFree(iv->cnormf);
  cudaFree(iv->books);
  cudaFree(iv->offsets);
  cudaFree(iv->codes);
  cudaFree(iv->ids);
  cudaFree(iv->vtab);
  cudaFree(iv->vmax);
  if (iv->list_order) cudaFree(iv->list_order);
  if (iv->wtab) cudaFree(iv->wtab);
  if (iv->wmax) cudaFree(iv->wmax);
  if (iv->probe_b) cudaFree(iv->probe_b);
  delete iv;
}

int run_ivf_search(pqs_ctx* ctx, const pqs_ivf* iv, QVec d_queries, int64_t nq, int ma, int r, double* d_dist,
                   int64_t* d_ids, int32_t* d_count) {
  const int64_t K = iv->K;
  const int m = iv->m, k = iv->k;
  // probes
  int64_t* cells = nullptr;
  double* pdist = nullptr;
  PQS_TRY(scratch(ctx, S_PROBE, (size_t)(nq * ma), &cells));
  PQS_TRY(scratch(ctx, S_PROBE_D, (size_t)(nq * ma), &pdist));
  // PQS_IVF_TIMING=1: device time of each phase of the search (CUDA events on
  // the context stream, printed to stderr after the search) -- the in-pipeline,
  // warm-cache counterpart of the serialised ncu launch list
  static const bool phase_timing = getenv("PQS_IVF_TIMING") != nullptr;
  struct Phase {
    const char* name;
    cudaEvent_t ev;
  };
  std::vector<Phase> phases;
  auto mark = [&](const char* name) {
    if (!phase_timing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, ctx->stream);
    phases.push_back({name, e});
  };
  mark("start");
  // packed list scan: the probe's exact re-score also emits the sub-space terms
  // a_qj = ||q_j - c_j||^2 of the selected cells (no separate pass over the pairs)
  if (ctx->ivf_engine == 2 && !iv->wtab)
    return set_err(ctx, PQS_ERR_UNSUPPORTED, "packed IVF list scan needs m = 8, k = 256 (W tables)");
  const bool packed = ctx->ivf_engine != 1 && iv->wtab != nullptr && nq < (1ll << 21);
  float* sub8 = nullptr;
  if (packed) PQS_TRY(scratch(ctx, S_TC_B, (size_t)(nq * ma) * 8, &sub8));
  PQS_TRY(run_ivf_probe(ctx, iv, d_queries, nq, ma, cells, pdist, sub8, packed ? m : 0));
  mark("probe");
  // per-query tables + bound
  float* U = nullptr;
  float* aerr = nullptr;
  PQS_TRY(scratch(ctx, S_TABLES, (size_t)(nq * m * k), &U));
  PQS_TRY(scratch(ctx, S_AERR, (size_t)nq, &aerr));
  {
    const size_t usz = ((size_t)UQ * m * k + 1) * 4 + (size_t)UQ * iv->d * 8;
    PQS_CHECK(ctx, usz <= 200 * 1024, "IVF query tables: m * k too large");
    PQS_CUDA(ctx, cudaFuncSetAttribute(utables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usz));
    utables_kernel<<<(unsigned)cdiv(nq, UQ), 256, usz, ctx->stream>>>(d_queries, iv->books, nq, m, k, iv->dsub, U);
  }
  PQS_LAUNCHED(ctx);
  ivf_bound_kernel<<<(unsigned)nq, 256, 0, ctx->stream>>>(U, pdist, nq, ma, m, k, iv->vmax, aerr);
  PQS_LAUNCHED(ctx);
  // threshold from the sample (the first spl codes of every probed list)
  static const int theta_cap = getenv("PQS_THETA_CAP") ? std::min(THETA_SAMPLE_CAP, atoi(getenv("PQS_THETA_CAP")))
                                                        : THETA_SAMPLE_CAP;  // tuning experiments
  // The sample: the first spl codes of the mas NEAREST probed lists.  Any >= r
  // probed codes give a valid threshold (an upper bound of the r-th smallest
  // distance); the nearest lists hold most of the true neighbours, so their
  // r-th smallest is tighter than that of a sample spread over all ma lists
  // (cfg3: 1742 -> fewer candidates per query) and the reads are longer runs.
  // mas: enough of them for ~32 r sampled codes at the average list length,
  // at least 8 (PQS_THETA_PROBES / PQS_THETA_SPL override, tuning experiments);
  // cfg3 sweep (probes x codes -> ms/step): 64x256 8.60, 32x512 8.38, 16x1024
  // 8.28, 8x2048 8.20, 8x1024 7.96.
  static const int theta_probes = getenv("PQS_THETA_PROBES") ? std::max(1, atoi(getenv("PQS_THETA_PROBES"))) : 0;
  static const int theta_spl = getenv("PQS_THETA_SPL") ? std::max(1, atoi(getenv("PQS_THETA_SPL"))) : 1024;
  const int64_t avg_list = std::max<int64_t>(1, iv->n / std::max<int64_t>(1, K));
  const int64_t per_list = std::min<int64_t>(theta_spl, avg_list);
  const int mas = std::min<int64_t>(ma, theta_probes > 0 ? theta_probes : std::max<int64_t>(8, cdiv(32 * (int64_t)r, per_list)));
  const int spl = std::min(theta_spl, std::max(1, theta_cap / std::max(mas, 1)));
  float* theta = nullptr;
  PQS_TRY(scratch(ctx, S_THETA, (size_t)nq * 4, (uint8_t**)&theta));
  const size_t usm = (size_t)m * k * 4;
  const size_t tsm = usm + (size_t)mas * spl * 4 + 8 + (size_t)mas * 16;
  PQS_CHECK(ctx, tsm <= 200 * 1024, "IVF threshold sample: m * k too large");
  PQS_CUDA(ctx, cudaFuncSetAttribute(ivf_theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
  mark("utables+bound");
  ivf_theta_kernel<<<(unsigned)nq, THETA_THREADS, tsm, ctx->stream>>>(U, cells, pdist, iv->offsets, iv->codes,
                                                                     iv->vtab, ma, mas, spl, m, k, r, aerr, theta);
  PQS_LAUNCHED(ctx);
  mark("theta sample");
  // packed list scan: per-query scale / integer threshold / error bound, then the
  // pair kernels below also lay out the per-pair parameters
  float* qscale = nullptr;
  uint32_t* qtint = nullptr;
  float *aerr2 = nullptr, *ps = nullptr, *pas = nullptr;
  uint32_t* pt = nullptr;
  if (packed) {
    PQS_TRY(scratch(ctx, S_QT_WORK, (size_t)nq * 3 + (size_t)(nq * ma) * 10 + 8, &qscale));
    qtint = reinterpret_cast<uint32_t*>(qscale + nq);
    aerr2 = qscale + 2 * nq;
    ps = qscale + 3 * nq + ((4 - (3 * nq) % 4) % 4);  // 16-byte aligned rows for the float4 stores of pas
    pt = reinterpret_cast<uint32_t*>(ps + nq * ma);
    pas = ps + 2 * nq * ma + ((4 - (2 * nq * ma) % 4) % 4);
    ivf_qparams_kernel<<<(unsigned)nq, 256, 0, ctx->stream>>>(U, pdist, theta, aerr, iv->wmax, nq, ma, m, k, qscale,
                                                             qtint, aerr2);
    PQS_LAUNCHED(ctx);
  }
  // bucket (query, probe) pairs by list
  int* lcnt = nullptr;
  int64_t* starts = nullptr;
  int* pq_ = nullptr;
  float* pa = nullptr;
  PQS_TRY(scratch(ctx, S_IVF_WORK2, (size_t)(K + 1), &lcnt));
  PQS_TRY(scratch(ctx, S_IVF_WORK3, (size_t)(K + 1), &starts));
  PQS_TRY(scratch(ctx, S_MISC, (size_t)(nq * ma) * 3, &pq_));
  pa = (float*)(pq_ + nq * ma);
  int* pcell = pq_ + 2 * nq * ma;
  PQS_CUDA(ctx, cudaMemsetAsync(lcnt, 0, sizeof(int) * (K + 1), ctx->stream));
  pair_count_kernel<<<(unsigned)cdiv(nq * ma, 256), 256, 0, ctx->stream>>>(cells, nq * ma, lcnt);
  PQS_LAUNCHED(ctx);
  scan_kernel<<<1, 1024, 0, ctx->stream>>>(lcnt, K, starts);
  PQS_LAUNCHED(ctx);
  PQS_CUDA(ctx, cudaMemsetAsync(lcnt, 0, sizeof(int) * (K + 1), ctx->stream));
  pair_fill_kernel<<<(unsigned)cdiv(nq * ma, 256), 256, 0, ctx->stream>>>(cells, pdist, nq, ma, starts, lcnt, pq_, pa, pcell,
                                                                          sub8, qscale, qtint, ps, pt, pas);
  PQS_LAUNCHED(ctx);
  // list-major filtered scan
  const int64_t cap = ctx->cand_cap;
  uint64_t* cand = nullptr;
  int* cnt = nullptr;
  PQS_TRY(scratch(ctx, S_CAND, (size_t)(nq * cap), &cand));
  PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)nq, &cnt));
  PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
  const size_t lsm = (size_t)m * k * LROW * 4 + (size_t)LCH * ((m + 3) / 4) * 4 + (size_t)LCH * 4 +
                     (size_t)LQ * LSTAGE * 8;
  float* capx = nullptr;
  PQS_TRY(scratch(ctx, S_IVF_APX, (size_t)(nq * cap), &capx));
  PQS_CHECK(ctx, lsm <= 220 * 1024, "IVF list scan: m * k too large for the shared-memory tables");
  auto list_kernel = (m == 8 && k == 256) ? ivf_list_kernel<8, 256> : ivf_list_kernel<0, 0>;
  PQS_CUDA(ctx, cudaFuncSetAttribute(list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
  const float* aerr_ct = aerr;  // error bound of the candidates' filter distances (ivf_cand_theta_kernel)
  if (packed) {
    // integer list scan (K8p): candidates carry L / s_q, certified within aerr2
    ListDesc* desc = nullptr;
    PQS_TRY(scratch(ctx, S_TC_REC, (size_t)K, &desc));
    ivf_desc_kernel<<<(unsigned)cdiv(K, 256), 256, 0, ctx->stream>>>(iv->list_order, starts, iv->offsets, K, desc);
    PQS_LAUNCHED(ctx);
    List8Args la{};
    la.U = U;
    la.W = iv->wtab;
    la.desc = desc;
    la.K = K;
    la.pq = pq_;
    la.ps = ps;
    la.pt = pt;
    la.pas = pas;
    la.codes = iv->codes;
    la.cand = cand;
    la.cand_apx = capx;
    la.cand_cnt = cnt;
    la.cap = cap;
    const size_t l8sm = 65536 /* below the aligned slot */ + 65536 + (size_t)m * k * 4 * (1 + L8_Q);
    PQS_CUDA(ctx, cudaFuncSetAttribute(ivf_list8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l8sm));
    PQS_TRY(scan_timer_begin(ctx));
    ivf_list8_kernel<<<(unsigned)std::min<int64_t>(K, ctx->sm_count), L8_THREADS, l8sm, ctx->stream>>>(la);
    PQS_LAUNCHED(ctx);
    PQS_TRY(scan_timer_end(ctx));
    ctx->last_scan_launches = 1;
    ctx->last_scan_engine = 6;
    aerr_ct = aerr2;
  }
  if (!packed) {
    PQS_TRY(scan_timer_begin(ctx));
    list_kernel<<<(unsigned)K, LIST_THREADS, lsm, ctx->stream>>>(U, starts, pq_, pa, iv->offsets, iv->codes, iv->vtab,
                                                                m, k, theta, cand, capx, cnt, cap, iv->list_order);
    PQS_LAUNCHED(ctx);
    PQS_TRY(scan_timer_end(ctx));
    ctx->last_scan_launches = 1;
    ctx->last_scan_engine = 4;
  }
  // tighten to the candidates within 2 aerr of the r-th filter distance,
  // exact rerank (keys in place in cand2, ids into cand) + select
  uint64_t* cand2 = nullptr;
  int* cnt2 = nullptr;
  PQS_TRY(scratch(ctx, S_PIDS, (size_t)(nq * cap), &cand2));
  PQS_TRY(scratch(ctx, S_IVF_CNT2, (size_t)nq, &cnt2));
  mark("pairs+params+list scan");
  ivf_cand_theta_kernel<<<(unsigned)nq, CT_THREADS, 0, ctx->stream>>>(cand, capx, cnt, cap, r, aerr_ct, cand2, cnt2);
  PQS_LAUNCHED(ctx);
  mark("cand tighten");
  int64_t* pids = reinterpret_cast<int64_t*>(cand);
  auto rerank = [&](uint64_t* cd, const int* cc, int64_t cp, QVec qs, int64_t nqr, int64_t* pi) -> int {
    dim3 rg((unsigned)nqr, 8);
    // float4 loads need 16-byte aligned sub-vectors: dsub % 4 == 0 (cudaMalloc'd bases)
    auto rk = iv->dsub == 16 ? ivf_rerank_kernel<16> : iv->dsub == 8 ? ivf_rerank_kernel<8>
              : iv->dsub == 4 ? ivf_rerank_kernel<4> : ivf_rerank_kernel<0>;
    rk<<<rg, RERANK_THREADS, 0, ctx->stream>>>(cd, cc, cp, iv->ids, qs, iv->coarse, iv->books, iv->codes, m, k, iv->d,
                                               iv->dsub, pi);
    PQS_LAUNCHED(ctx);
    return PQS_OK;
  };
  PQS_TRY(rerank(cand2, cnt2, cap, d_queries, nq, pids));
  mark("exact rerank");
  uint64_t* gk = nullptr;
  int64_t* gi = nullptr;
  PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * cap), &gk));
  PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * cap), &gi));
  SelArgs s{};
  s.src = SEL_KEYS;
  s.nq = nq;
  s.r = r;
  s.cand = cand2;
  s.cand_cnt = cnt2;
  s.cap = cap;
  s.pids = pids;
  s.out_d = d_dist;
  s.out_i = d_ids;
  s.out_c = d_count;
  s.gkeys = gk;
  s.gids = gi;
  s.gcap = cap;
  PQS_TRY(launch_select(ctx, s));
  mark("select");
  // overflow / sanity check against the exact probed totals; the totals and
  // the statistics are reduced on the device and land in one pinned buffer
  int64_t* d_tot = nullptr;
  PQS_TRY(scratch(ctx, S_IVF_WORK, (size_t)nq + 1, &d_tot));
  ivf_probed_kernel<<<(unsigned)cdiv(nq, 256), 256, 0, ctx->stream>>>(cells, iv->offsets, nq, ma, d_tot);
  PQS_LAUNCHED(ctx);
  PQS_CUDA(ctx, cudaMemsetAsync(d_tot + nq, 0, 8, ctx->stream));
  ivf_slot_evals_kernel<<<(unsigned)cdiv(K, 256), 256, 0, ctx->stream>>>(
      lcnt, iv->offsets, K, LQ, reinterpret_cast<unsigned long long*>(d_tot + nq));
  PQS_LAUNCHED(ctx);
  const int64_t need = 4 * nq + 2;
  if (ctx->h_cnt_cap < need) {
    if (ctx->h_cnt) {
      PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFreeHost(ctx->h_cnt);
      ctx->h_cnt = nullptr;
    }
    PQS_CUDA(ctx, cudaHostAlloc((void**)&ctx->h_cnt, sizeof(int) * (size_t)need, cudaHostAllocDefault));
    ctx->h_cnt_cap = need;
  }
  int* hcnt = ctx->h_cnt;
  int* hcnt2 = ctx->h_cnt + nq;
  int64_t* htot = reinterpret_cast<int64_t*>(ctx->h_cnt + 2 * nq);
  PQS_CUDA(ctx, cudaMemcpyAsync(hcnt2, cnt2, sizeof(int) * nq, cudaMemcpyDeviceToHost, ctx->stream));
  PQS_CUDA(ctx, cudaMemcpyAsync(hcnt, cnt, sizeof(int) * nq, cudaMemcpyDeviceToHost, ctx->stream));
  PQS_CUDA(ctx, cudaMemcpyAsync(htot, d_tot, sizeof(int64_t) * (nq + 1), cudaMemcpyDeviceToHost, ctx->stream));
  mark("stats");
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  PQS_TRY(scan_timer_collect(ctx));
  if (phase_timing) {
    for (size_t i = 1; i < phases.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, phases[i - 1].ev, phases[i].ev);
      fprintf(stderr, "pqs ivf phase %-24s %8.3f ms\n", phases[i].name, ms);
    }
    for (auto& ph : phases) cudaEventDestroy(ph.ev);
  }
  std::vector<int> over;
  int64_t mx = 0, ctot = 0, total_evals = 0, worst_total = 0;
  for (int64_t q = 0; q < nq; ++q) {
    const int64_t tot = htot[q];
    total_evals += tot;
    mx = std::max<int64_t>(mx, hcnt[q]);
    ctot += hcnt[q];
    const int64_t r_eff = std::min<int64_t>(r, tot);
    if (hcnt[q] > cap || hcnt[q] < r_eff || ctx->force_fallback) {
      static const bool dbg = getenv("PQS_DEBUG") != nullptr;
      if (dbg)
        fprintf(stderr, "pqs ivf: query %lld falls back: %d candidates (cap %lld, r_eff %lld, probed %lld)\n",
                (long long)q, hcnt[q], (long long)cap, (long long)r_eff, (long long)tot);
      over.push_back((int)q);
      worst_total = std::max(worst_total, tot);
    }
  }
  ctx->last_evals = total_evals;
  ctx->last_scan_work = (double)total_evals * (double)m;
  ctx->last_slot_evals = htot[nq];
  ctx->last_max_cand = mx;
  ctx->last_cand_total = ctot;
  {
    int64_t rt = 0;
    for (int64_t q = 0; q < nq; ++q) rt += hcnt2[q];
    ctx->last_rerank_total = rt;
  }
  ctx->last_overflow = (int64_t)over.size();
  if (!over.empty()) {
    const int64_t fcap = std::max<int64_t>(worst_total, 1);
    uint64_t* fc = nullptr;
    int* fcnt = nullptr;
    for (size_t i = 0; i < over.size(); ++i) {
      // one query at a time: its whole probed set is the candidate list
      PQS_TRY(scratch(ctx, S_DENSE, (size_t)fcap * (nq > 0 ? 1 : 1) * 2 + 2, &fc));
      fcnt = (int*)(fc + fcap);
      PQS_TRY(scratch(ctx, S_KEYS, (size_t)fcap, &gk));
      PQS_TRY(scratch(ctx, S_IDS, (size_t)fcap, &gi));
      PQS_CUDA(ctx, cudaMemsetAsync(fcnt, 0, sizeof(int) * 1, ctx->stream));
      // candidates are indexed by the global query id; use a 1-row view
      const int qg = over[i];
      ivf_all_kernel<<<1, 256, 0, ctx->stream>>>(cells + (int64_t)qg * ma, ma, iv->offsets, fc, fcnt, fcap);
      PQS_LAUNCHED(ctx);
      int64_t* fpi = nullptr;
      PQS_TRY(scratch(ctx, S_PIDS, (size_t)fcap, &fpi));
      PQS_TRY(rerank(fc, fcnt, fcap, d_queries.offset((int64_t)qg * iv->d), 1, fpi));
      SelArgs f = s;
      f.nq = 1;
      f.cand = fc;
      f.cand_cnt = fcnt;
      f.cap = fcap;
      f.pids = fpi;
      f.out_d = d_dist + (int64_t)qg * r;
      f.out_i = d_ids + (int64_t)qg * r;
      f.out_c = d_count + qg;
      f.gkeys = gk;
      f.gids = gi;
      f.gcap = fcap;
      PQS_TRY(launch_select(ctx, f));
    }
  }
  return PQS_OK;
}
