// select.cu -- K5/K6/K10: per-query top-r by (distance, id).
//
// Reference semantics: _select_best (scan.py:142-154) -- the r smallest
// (distance, id) pairs, ascending, r > n returns n; NeighborSet.push keeps the
// lower id on distance ties (scan.py:109-118).  One CTA per query:
//   1. materialise (key, id) for the query's elements (candidates from a
//      filtered scan, a dense row, or G shard lists);  for SEL_CAND_ADC the
//      key is the exact fp64 ADC distance recomputed in the reference's
//      summation order (scan.py:77-81) -- the "rerank" (K6);
//   2. MSD radix select (8-bit digits, smem histogram) of the r-th key;
//   3. if the cut key is tied beyond r, a second radix select on ids;
//   4. gather exactly r elements, bitonic sort by (key, id), write out.
#include <cuda_runtime.h>

#include <algorithm>

#include "pqs_common.cuh"
#include "select_dev.cuh"

namespace {

using namespace seldev;

constexpr int SEL_THREADS = 256;
constexpr int SMEM_CAP = 2048;  // materialised elements kept in shared memory (more: global scratch)

// Element access -----------------------------------------------------------
struct ElemSrc {
  const SelArgs* a;
  int64_t q;    // global query index (tables, candidates, outputs)
  int64_t ql;   // local (block) index (dense rows, global scratch)
  const uint64_t* K;  // materialised keys (smem or global) or nullptr
  const int64_t* I;
};

__device__ __forceinline__ int64_t map_id(const SelArgs& a, int64_t idx) {
  return a.ids ? a.ids[idx] : a.id_base + idx;
}

__device__ __forceinline__ void get_elem(const ElemSrc& e, int64_t i, uint64_t& key, int64_t& id) {
  if (e.K) {
    key = e.K[i];
    id = e.I[i];
    return;
  }
  const SelArgs& a = *e.a;
  if (a.src == SEL_DENSE_F64) {
    key = dkey(((const double*)a.dense)[e.ql * a.n + i]);
  } else {  // SEL_DENSE_U8
    key = ((const uint8_t*)a.dense)[e.ql * a.n + i];
  }
  id = map_id(a, i);
}

// exact fp64 ADC of one stored code, sub-space order (scan.py:77-81)
__device__ __forceinline__ double adc_exact(const float* __restrict__ T, const uint8_t* __restrict__ codes8,
                                            int m, int k, int64_t idx) {
  const int64_t tile = idx / TILE8;
  const int c = (int)(idx % TILE8);
  const uint8_t* base = codes8 + tile * (int64_t)m * TILE8 + c;
  double acc = 0.0;
  for (int j0 = 0; j0 < m; j0 += 8) {  // 8 components' codes and entries in flight, then the ordered sum
    int code[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) code[u] = j0 + u < m ? base[(int64_t)(j0 + u) * TILE8] : 0;
    float t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = j0 + u < m ? __ldg(T + (int64_t)(j0 + u) * k + code[u]) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u < m) acc = __dadd_rn(acc, (double)t[u]);
  }
  return acc;
}

// the same sum from a row-major code row: all m code bytes and table entries
// of a 16-component block are in flight before the ordered fp64 sum
__device__ __forceinline__ double adc_exact_rm(const float* __restrict__ T, const uint8_t* __restrict__ row, int m,
                                               int k) {
  double acc = 0.0;
  for (int j0 = 0; j0 < m; j0 += 16) {
    uint32_t w[4];
    if ((m & 15) == 0) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + j0));
      w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else if ((m & 7) == 0) {
      const uint2 v0 = __ldg(reinterpret_cast<const uint2*>(row + j0));
      const uint2 v1 = j0 + 8 < m ? __ldg(reinterpret_cast<const uint2*>(row + j0 + 8)) : make_uint2(0u, 0u);
      w[0] = v0.x, w[1] = v0.y, w[2] = v1.x, w[3] = v1.y;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t x = 0;
        for (int b = 0; b < 4; ++b)
          if (j0 + 4 * u + b < m) x |= (uint32_t)row[j0 + 4 * u + b] << (8 * b);
        w[u] = x;
      }
    }
    float t[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      t[u] = j0 + u < m ? __ldg(T + (int64_t)(j0 + u) * k + ((w[u >> 2] >> (8 * (u & 3))) & 255u)) : 0.f;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (j0 + u < m) acc = __dadd_rn(acc, (double)t[u]);
  }
  return acc;
}

__device__ void materialise(const SelArgs& a, int64_t q, int64_t M, uint64_t* K, int64_t* I,
                            SelShared& sh) {
  if (a.src == SEL_KEYS) {
    const uint64_t* ck = a.cand + q * a.cap;
    const int64_t* ci = a.pids + q * a.cap;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      K[i] = ck[i];
      I[i] = ci[i];
    }
  } else if (a.src == SEL_CAND_BIN || a.src == SEL_CAND_ADC) {
    const uint64_t* cand = a.cand + q * a.cap;
    const float* T = a.tables ? a.tables + q * (int64_t)a.m * a.k : nullptr;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      const uint64_t e = cand[i];
      const int64_t idx = (int64_t)(uint32_t)e;
      uint64_t key;
      if (a.src == SEL_CAND_BIN) key = min(e >> 32, (uint64_t)127);  // bin = min(sum, 127)
      else key = dkey(a.codes_rm ? adc_exact_rm(T, a.codes_rm + idx * a.m, a.m, a.k)
                                 : adc_exact(T, a.codes8, a.m, a.k, idx));
      K[i] = key;
      I[i] = map_id(a, idx);
    }
  } else {  // SEL_MERGE: G lists of r_in entries
    int64_t off = 0;
    for (int g = 0; g < a.G; ++g) {
      const int64_t row = ((int64_t)g * a.nq + q);
      const int cnt = a.mcnt[row];
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        K[off + i] = dkey(a.mdist[row * a.r_in + i]);
        I[off + i] = a.mids[row * a.r_in + i];
      }
      off += cnt;
    }
  }
}

// NT threads per query CTA: 128 for candidate lists (a 1000-query batch is
// one wave at 8 CTAs/SM), 256 for dense rows and merges
template <int NT>
__global__ void __launch_bounds__(NT, NT == 128 ? 8 : 1) select_kernel(SelArgs a, int sortP, int scap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelShared sh;
  uint64_t* s_keys = (uint64_t*)smem_raw;
  int64_t* s_ids = (int64_t*)(s_keys + scap);
  uint64_t* o_keys = (uint64_t*)(s_ids + scap);
  int64_t* o_ids = (int64_t*)(o_keys + sortP);

  const int64_t ql = blockIdx.x;
  const int64_t q = a.qmap ? a.qmap[ql] : ql;

  if (threadIdx.x == 0) {
    long long M = 0;
    if (a.src == SEL_CAND_BIN || a.src == SEL_CAND_ADC || a.src == SEL_KEYS) {
      long long c = a.cand_cnt[q];
      M = c < a.cap ? c : a.cap;
    } else if (a.src == SEL_MERGE) {
      for (int g = 0; g < a.G; ++g) M += a.mcnt[(int64_t)g * a.nq + q];
    } else {
      M = a.n;
    }
    sh.M = M;
    sh.r_eff = M < a.r ? M : a.r;
    sh.out_cnt = 0;
  }
  __syncthreads();
  const int64_t M = sh.M;
  const int64_t r_eff = sh.r_eff;

  ElemSrc es{&a, q, ql, nullptr, nullptr};
  if (a.src != SEL_DENSE_F64 && a.src != SEL_DENSE_U8) {
    uint64_t* K = M <= scap ? s_keys : a.gkeys + ql * a.gcap;
    int64_t* I = M <= scap ? s_ids : a.gids + ql * a.gcap;
    materialise(a, q, M, K, I, sh);
    es.K = K;
    es.I = I;
    __syncthreads();
  }

  unsigned long long kstar = ~0ull;
  long long istar = 0x7FFFFFFFFFFFFFFFll;
  bool take_all_ties = true;
  if (r_eff > 0 && r_eff < M) {
    auto getk = [&](int64_t i, uint64_t& v) {
      int64_t id;
      get_elem(es, i, v, id);
      return true;
    };
    if (a.src == SEL_CAND_BIN) {
      // bins < 128: one shared histogram pass finds the cut bin
      for (int i = threadIdx.x; i < 128; i += blockDim.x) sh.hist[i] = 0;
      __syncthreads();
      for (int64_t i = threadIdx.x; i < M; i += blockDim.x) atomicAdd(&sh.hist[es.K[i]], 1u);
      __syncthreads();
      if (threadIdx.x < 32) {
        // warp-parallel cut: lane l owns bins 4l..4l+3; the cut bin is the
        // first whose inclusive count reaches r_eff (every bin is < 128)
        const int lane = threadIdx.x;
        unsigned int h[4], s4 = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) s4 += (h[u] = sh.hist[4 * lane + u]);
        unsigned int incl = s4;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const unsigned long long re = (unsigned long long)r_eff;
        const unsigned int excl = incl - s4;
        if (excl < re && incl >= re) {
          unsigned int c = excl;
          int u = 0;
          while (c + h[u] < re) c += h[u++];
          sh.prefix = (unsigned long long)(4 * lane + u);
          sh.less = c;
          sh.eq = h[u];
        }
      }
      __syncthreads();
    } else {
      block_radix_select(M, getk, (unsigned long long)(r_eff - 1), sh);
    }
    kstar = sh.prefix;
    const unsigned long long less = sh.less, eq = sh.eq;
    const unsigned long long need = (unsigned long long)r_eff - less;
    __syncthreads();
    if (eq > need) {
      take_all_ties = false;
      auto geti = [&](int64_t i, uint64_t& v) {
        uint64_t key;
        int64_t id;
        get_elem(es, i, key, id);
        v = (uint64_t)id ^ 0x8000000000000000ull;
        return key == kstar;
      };
      block_radix_select(M, geti, need - 1, sh);
      istar = (long long)(sh.prefix ^ 0x8000000000000000ull);
      __syncthreads();
    }
  }
  // gather
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    uint64_t key;
    int64_t id;
    get_elem(es, i, key, id);
    const bool sel = key < kstar || (key == kstar && (take_all_ties || id <= istar));
    if (sel) {
      const int p = atomicAdd(&sh.out_cnt, 1);
      if (p < sortP) {
        o_keys[p] = key;
        o_ids[p] = id;
      }
    }
  }
  __syncthreads();
  const int cnt = min((int)r_eff, sortP);
  for (int p = cnt + threadIdx.x; p < sortP; p += blockDim.x) {
    o_keys[p] = ~0ull;
    o_ids[p] = 0x7FFFFFFFFFFFFFFFll;
  }
  __syncthreads();
  bitonic_sort(o_keys, o_ids, sortP);
  // write
  const bool is_float = (a.src != SEL_CAND_BIN && a.src != SEL_DENSE_U8);
  for (int p = threadIdx.x; p < a.r; p += blockDim.x) {
    const int64_t o = q * a.r + p;
    if (p < cnt) {
      if (a.out_d) a.out_d[o] = is_float ? dkey_inv(o_keys[p]) : (double)o_keys[p];
      if (a.out_b) a.out_b[o] = (uint8_t)o_keys[p];
      a.out_i[o] = o_ids[p];
    } else {
      if (a.out_d) a.out_d[o] = __longlong_as_double(0x7FF0000000000000ll);
      if (a.out_b) a.out_b[o] = 255;
      a.out_i[o] = -1;
    }
  }
  if (threadIdx.x == 0 && a.out_c) a.out_c[q] = cnt;
}

}  // namespace

int launch_select(pqs_ctx* ctx, const SelArgs& a) {
  if (a.r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  int nql = (int)a.nq;
  if (nql == 0) return PQS_OK;
  int P = 1;
  while (P < a.r) P <<= 1;
  if (P < 2) P = 2;
  const bool narrow = a.src == SEL_CAND_BIN || a.src == SEL_CAND_ADC || a.src == SEL_KEYS;
  const int scap = narrow ? SMEM_CAP / 2 : SMEM_CAP;  // narrow: 18 KB + P -> 8 CTAs/SM
  const size_t smem = (size_t)scap * 16 + (size_t)P * 16;
  auto kern = narrow ? select_kernel<128> : select_kernel<SEL_THREADS>;
  PQS_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((size_t)SMEM_CAP * 16 + (size_t)MAX_R * 16)));
  kern<<<nql, narrow ? 128 : SEL_THREADS, smem, ctx->stream>>>(a, P, scap);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}
