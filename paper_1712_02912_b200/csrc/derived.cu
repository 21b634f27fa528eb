// derived.cu -- derived-quantizer two-pass search (derived.py:143-409,
// SURVEY 8f row 4) and query_ivf kernel='derived' (ivf.py:191-195).
//
// Reference semantics of search_two_pass(dpq, db, query, r, r2):
//   compact = compute_compact_tables: fp32(||y_j - D_j[l]||^2) over the
//             2^bbar derived centroids (fp64, scipy order)      derived.py:129-140
//   qt      = quantize_compact_tables: qmin = min(compact); qmax = max fp64
//             ADC (low index bits) of the first min(r2, n) codes; 255-bin
//             quantization (255 at/above qmax)                   derived.py:143-198
//   cand    = scan_candidates: d = min(255, sum_j qt[j][c_j & (kbar-1)]);
//             if >= r2 codes have d <= 254: keep d <= the bucket where the
//             running count reaches r2; else keep every d <= 254 plus the
//             d = 255 codes admitted while fewer than r2 were held -- the
//             count before storage position p is exactly p, so those are
//             the d = 255 codes at positions < r2               derived.py:294-326
//   result  = rerank: exact fp64 distances (sum over j of the fp32 full-table
//             entries) of every kept code -- the bucket walk stops only after
//             the last kept bucket -- and the r best by (distance, id)
//                                                                derived.py:362-399
// B200 design, exhaustive list (batched queries): K1 builds the full and the
// compact tables; dv_params_kernel (per query) the 255-bin tables;
// dv_hist_kernel (grid tiles x queries) the 256-bin histogram of d;
// dv_bound_kernel the admission rule; dv_collect_kernel the kept indices;
// K5 (SEL_CAND_ADC) re-scores them exactly and selects.  IVF: one CTA per
// (query, probe) does all of it for its list on chip, emitting the list's r
// best (distance, id); K5 (SEL_KEYS) merges the probes.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "pqs_common.cuh"
#include "select_dev.cuh"

namespace {

using namespace seldev;

constexpr int DV_THREADS = 256;
constexpr int DV_TILE = 4096;  // codes per histogram / collect CTA

// quantize_255 (derived.py:143-154): 255 at or above qmax, else
// clip(floor((v - qmin) * (255 / span)), 0, 254); all 0 for an empty span
__device__ __forceinline__ uint8_t quantize255(double v, double qmin, double qmax, double span) {
  if (!(span > 0.0)) return 0;
  if (v >= qmax) return 255;
  double f = floor(__dmul_rn(__dsub_rn(v, qmin), __ddiv_rn(255.0, span)));
  f = f < 0.0 ? 0.0 : (f > 254.0 ? 254.0 : f);
  return (uint8_t)f;
}

__device__ __forceinline__ int code8_at(const uint8_t* __restrict__ codes8, int m, int64_t i, int j) {
  return codes8[(i / TILE8) * (int64_t)m * TILE8 + (int64_t)j * TILE8 + (i % TILE8)];
}

struct DvQuery {
  double qmin, qmax;
  int mode;      // 0: keep d <= bound; 1: keep d <= 254 or position < r2
  int bound;
  long long kept;
};

// per query: qmin, qmax, 255-bin compact tables
__global__ void __launch_bounds__(DV_THREADS) dv_params_kernel(const float* __restrict__ ctab, const uint8_t* __restrict__ codes8,
                                                               int64_t n, int m, int kbar, int64_t r2,
                                                               DvQuery* __restrict__ qs, uint8_t* __restrict__ qct) {
  __shared__ float fmn[DV_THREADS / 32];
  __shared__ double dmx[DV_THREADS / 32];
  __shared__ double s_q[2];
  const int64_t q = blockIdx.x;
  const float* T = ctab + q * (int64_t)m * kbar;
  const int mask = kbar - 1;
  float mn = __int_as_float(0x7f800000);
  for (int i = threadIdx.x; i < m * kbar; i += DV_THREADS) mn = fminf(mn, T[i]);
  double mx = -1.0;  // distances are >= 0
  const int64_t head = min(r2, n);
  for (int64_t i = threadIdx.x; i < head; i += DV_THREADS) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, (double)T[j * kbar + (code8_at(codes8, m, i, j) & mask)]);
    mx = fmax(mx, acc);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    fmn[threadIdx.x >> 5] = mn;
    dmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = fmn[0];
    double b = dmx[0];
    for (int w = 1; w < DV_THREADS / 32; ++w) {
      a = fminf(a, fmn[w]);
      b = fmax(b, dmx[w]);
    }
    const double qmin = (double)a;
    const double qmax = b > qmin ? b : qmin;
    s_q[0] = qmin;
    s_q[1] = qmax;
    qs[q].qmin = qmin;
    qs[q].qmax = qmax;
  }
  __syncthreads();
  const double qmin = s_q[0], qmax = s_q[1], span = __dsub_rn(qmax, qmin);
  for (int i = threadIdx.x; i < m * kbar; i += DV_THREADS)
    qct[q * (int64_t)m * kbar + i] = quantize255((double)T[i], qmin, qmax, span);
}

// adc_low_bits (derived.py:201-211): saturating sum of the 255-bin entries
__device__ __forceinline__ int low_adc(const uint8_t* __restrict__ sq, const uint8_t* __restrict__ codes8, int m,
                                       int kbar, int64_t i) {
  const uint8_t* cp = codes8 + (i / TILE8) * (int64_t)m * TILE8 + (i % TILE8);
  const int mask = kbar - 1;
  int acc = 0;
  for (int j = 0; j < m; ++j) acc += sq[j * kbar + (cp[(int64_t)j * TILE8] & mask)];
  return acc < 255 ? acc : 255;
}

__global__ void __launch_bounds__(DV_THREADS) dv_hist_kernel(const uint8_t* __restrict__ codes8, int64_t n, int m,
                                                             int kbar, const uint8_t* __restrict__ qct,
                                                             unsigned int* __restrict__ hist) {
  extern __shared__ uint8_t sq[];
  __shared__ unsigned int h[256];
  const int64_t q = blockIdx.y;
  for (int i = threadIdx.x; i < 256; i += DV_THREADS) h[i] = 0;
  for (int i = threadIdx.x; i < m * kbar; i += DV_THREADS) sq[i] = qct[q * (int64_t)m * kbar + i];
  __syncthreads();
  const int64_t b = (int64_t)blockIdx.x * DV_TILE, e = min(n, b + DV_TILE);
  for (int64_t i = b + threadIdx.x; i < e; i += DV_THREADS) atomicAdd(&h[low_adc(sq, codes8, m, kbar, i)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += DV_THREADS)
    if (h[i]) atomicAdd(hist + q * 256 + i, h[i]);
}

// one warp per query: the admission rule of scan_candidates
__global__ void dv_bound_kernel(const unsigned int* __restrict__ hist, int64_t nq, int64_t n, int64_t r2,
                                DvQuery* __restrict__ qs) {
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const int lane = threadIdx.x & 31;
  const unsigned int* hq = hist + q * 256;
  unsigned long long c[8], s8 = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s8 += (c[u] = hq[8 * lane + u]);
  unsigned long long incl = s8;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned long long excl = incl - s8;
  const unsigned long long small = __shfl_sync(0xffffffffu, incl - c[7], 31);  // bins 0..254
  if (small >= (unsigned long long)r2) {
    int bnd = 1 << 30;
    if (excl < (unsigned long long)r2 && incl >= (unsigned long long)r2) {
      unsigned long long a = excl;
      for (int u = 0; u < 8; ++u) {
        a += c[u];
        if (a >= (unsigned long long)r2) {
          bnd = 8 * lane + u;
          break;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) bnd = min(bnd, __shfl_xor_sync(0xffffffffu, bnd, o));
    // kept = codes with d <= bnd
    unsigned long long kk = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) kk += (8 * lane + u <= bnd) ? c[u] : 0ull;
    for (int o = 16; o > 0; o >>= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
    if (lane == 0) {
      qs[q].mode = 0;
      qs[q].bound = bnd;
      qs[q].kept = (long long)kk;
    }
  } else if (lane == 0) {
    qs[q].mode = 1;
    qs[q].bound = 254;
    qs[q].kept = (long long)small + min(r2, n);  // upper bound (exact count from the collect)
  }
}

__global__ void __launch_bounds__(DV_THREADS) dv_collect_kernel(const uint8_t* __restrict__ codes8, int64_t n, int m,
                                                                int kbar, int64_t r2, const uint8_t* __restrict__ qct,
                                                                const DvQuery* __restrict__ qs,
                                                                uint64_t* __restrict__ cand, int* __restrict__ cnt,
                                                                int64_t cap) {
  extern __shared__ uint8_t sq[];
  const int64_t q = blockIdx.y;
  for (int i = threadIdx.x; i < m * kbar; i += DV_THREADS) sq[i] = qct[q * (int64_t)m * kbar + i];
  __syncthreads();
  const DvQuery Q = qs[q];
  const int64_t b = (int64_t)blockIdx.x * DV_TILE, e = min(n, b + DV_TILE);
  for (int64_t i0 = b; i0 < e; i0 += DV_THREADS) {
    const int64_t i = i0 + threadIdx.x;
    bool keep = false;
    if (i < e) {
      const int d = low_adc(sq, codes8, m, kbar, i);
      keep = Q.mode == 0 ? d <= Q.bound : (d <= 254 || i < r2);
    }
    // warp-aggregated append
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    int base = 0;
    if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(cnt + q, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
      const int s = base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
      if (s < cap) cand[q * cap + s] = (uint64_t)(uint32_t)i;
    }
  }
}

// ------------------------------------------------------------------ IVF
// One CTA per (query, probe): residual full tables (m x k) and compact
// tables (m x kbar) in shared memory, then the whole search_two_pass of the
// list; the list's r best (exact distance, id) go to the query's candidate
// row (one reservation), merged by K5.
struct DvIvfArgs {
  QVec queries;
  const float* coarse;
  const float* books;     // (m, k, dsub)
  const float* dbooks;    // (m, kbar, dsub)
  const int64_t* offsets;
  const uint8_t* codes;   // (n, m) row-major
  const int64_t* ids;
  const int64_t* cells;
  int64_t q0;
  int ma, m, k, kbar, d, dsub, r;
  int64_t r2;
  uint64_t* cand;
  int64_t* pids;
  int* cnt;
  int64_t cap;
};

struct DvShared {
  SelShared sel;
  unsigned int hist[256];
  float fred[DV_THREADS / 32];
  double dred[DV_THREADS / 32];
  double qmin, qmax;
  int mode, bound, emitted, eqleft, tiebreak;
  long long base;
  unsigned long long kstar, istar;
};

__device__ __forceinline__ double table_entry(QVec qv, const float* g, const float* cb, int j, int dsub) {
  double t = 0.0;
  for (int s = 0; s < dsub; ++s) {
    const int dd = j * dsub + s;
    const double rr = __dsub_rn(qv.at(dd), (double)__ldg(g + dd));
    const double df = __dsub_rn(rr, (double)__ldg(cb + s));
    t = __dadd_rn(t, __dmul_rn(df, df));
  }
  return t;
}

__global__ void __launch_bounds__(DV_THREADS) dv_ivf_kernel(DvIvfArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ DvShared sh;
  const int m = a.m, k = a.k, kbar = a.kbar, mask = kbar - 1;
  float* T = (float*)dsm;                      // (m, k) full residual tables
  float* C = T + (size_t)m * k;                // (m, kbar) compact tables
  uint8_t* Q = (uint8_t*)(C + (size_t)m * kbar);  // (m, kbar) 255-bin tables
  const int64_t pair = blockIdx.x;
  const int64_t ql = pair / a.ma;
  const int64_t c = a.cells[(a.q0 + ql) * a.ma + pair % a.ma];
  if (c < 0) return;
  const int64_t lb = a.offsets[c], n = a.offsets[c + 1] - lb;
  if (n == 0) return;  // ivf.py:176-177
  const QVec qv = a.queries.offset((a.q0 + ql) * (int64_t)a.d);
  const float* g = a.coarse + c * (int64_t)a.d;
  const uint8_t* lc = a.codes + lb * (int64_t)m;
  const int64_t* li = a.ids + lb;
  for (int e = threadIdx.x; e < m * k; e += DV_THREADS)
    T[e] = __double2float_rn(table_entry(qv, g, a.books + (int64_t)e * a.dsub, e / k, a.dsub));
  float mn = __int_as_float(0x7f800000);
  for (int e = threadIdx.x; e < m * kbar; e += DV_THREADS) {
    const float v = __double2float_rn(table_entry(qv, g, a.dbooks + (int64_t)e * a.dsub, e / kbar, a.dsub));
    C[e] = v;
    mn = fminf(mn, v);
  }
  for (int i = threadIdx.x; i < 256; i += DV_THREADS) sh.hist[i] = 0;
  __syncthreads();
  // qmax: the largest compact ADC of the first min(r2, n) codes
  double mx = -1.0;
  for (int64_t i = threadIdx.x; i < min(a.r2, n); i += DV_THREADS) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, (double)C[j * kbar + (lc[i * m + j] & mask)]);
    mx = fmax(mx, acc);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    sh.fred[threadIdx.x >> 5] = mn;
    sh.dred[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a0 = sh.fred[0];
    double b0 = sh.dred[0];
    for (int w = 1; w < DV_THREADS / 32; ++w) {
      a0 = fminf(a0, sh.fred[w]);
      b0 = fmax(b0, sh.dred[w]);
    }
    sh.qmin = (double)a0;
    sh.qmax = b0 > sh.qmin ? b0 : sh.qmin;
  }
  __syncthreads();
  {
    const double qmin = sh.qmin, qmax = sh.qmax, span = __dsub_rn(qmax, qmin);
    for (int e = threadIdx.x; e < m * kbar; e += DV_THREADS) Q[e] = quantize255((double)C[e], qmin, qmax, span);
  }
  __syncthreads();
  auto dlow = [&](int64_t i) -> int {
    int acc = 0;
    for (int j = 0; j < m; ++j) acc += Q[j * kbar + (lc[i * m + j] & mask)];
    return acc < 255 ? acc : 255;
  };
  for (int64_t i = threadIdx.x; i < n; i += DV_THREADS) atomicAdd(&sh.hist[dlow(i)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    long long small = 0;
    for (int b = 0; b < 255; ++b) small += sh.hist[b];
    if (small >= a.r2) {
      long long cum = 0;
      int b = 0;
      for (; b < 255; ++b) {
        cum += sh.hist[b];
        if (cum >= a.r2) break;
      }
      sh.mode = 0;
      sh.bound = b;
    } else {
      sh.mode = 1;
      sh.bound = 254;
    }
  }
  __syncthreads();
  const int mode = sh.mode, bound = sh.bound;
  const int64_t r2 = a.r2;
  // exact distance of a kept code (rerank, derived.py:362-399), else no key
  auto kept = [&](int64_t i) -> bool {
    const int dl = dlow(i);
    return mode == 0 ? dl <= bound : (dl <= 254 || i < r2);
  };
  auto exact = [&](int64_t i) -> double {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, (double)T[j * k + lc[i * m + j]]);
    return acc;
  };
  // number kept
  if (threadIdx.x == 0) sh.emitted = 0;
  __syncthreads();
  {
    int local = 0;
    for (int64_t i = threadIdx.x; i < n; i += DV_THREADS) local += kept(i) ? 1 : 0;
    atomicAdd(&sh.emitted, local);
  }
  __syncthreads();
  const int64_t M = sh.emitted;
  const int64_t r_eff = min((int64_t)a.r, M);
  unsigned long long kstar = ~0ull, istar = ~0ull;
  bool tb = false;
  if (r_eff < M) {
    auto getk = [&](int64_t i, uint64_t& v) -> bool {
      if (!kept(i)) return false;
      v = dkey(exact(i));
      return true;
    };
    block_radix_select(n, getk, (unsigned long long)(r_eff - 1), sh.sel);
    kstar = sh.sel.prefix;
    const unsigned long long less = sh.sel.less, eq = sh.sel.eq, need = (unsigned long long)r_eff - less;
    __syncthreads();
    if (eq > need) {
      tb = true;
      auto geti = [&](int64_t i, uint64_t& v) -> bool {
        if (!kept(i) || dkey(exact(i)) != kstar) return false;
        v = (uint64_t)li[i] ^ 0x8000000000000000ull;
        return true;
      };
      block_radix_select(n, geti, need - 1, sh.sel);
      istar = sh.sel.prefix;
      if (threadIdx.x == 0) sh.eqleft = (int)(need - sh.sel.less);
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    sh.emitted = 0;
    sh.base = atomicAdd(a.cnt + ql, (int)r_eff);
  }
  __syncthreads();
  uint64_t* crow = a.cand + ql * a.cap + sh.base;
  int64_t* prow = a.pids + ql * a.cap + sh.base;
  for (int64_t i = threadIdx.x; i < n; i += DV_THREADS) {
    if (!kept(i)) continue;
    const double dist = exact(i);
    const uint64_t key = dkey(dist);
    bool take = key < kstar || (key == kstar && !tb);
    if (!take && key == kstar) {
      const uint64_t ik = (uint64_t)li[i] ^ 0x8000000000000000ull;
      take = ik < istar || (ik == istar && atomicSub(&sh.eqleft, 1) > 0);
    }
    if (take) {
      const int s = atomicAdd(&sh.emitted, 1);
      crow[s] = key;
      prow[s] = li[i];
    }
  }
}

}  // namespace

// Exhaustive search_two_pass for a batch: full tables (nq, m, k) and compact
// tables (nq, m, kbar), both exact fp32 (K1); db b = 8.
int run_derived_search(pqs_ctx* ctx, const pqs_db* db, const float* d_full, int k, const float* d_compact, int64_t nq,
                       int kbar, int r, int64_t r2, double* d_dist, int64_t* d_ids, int32_t* d_count) {
  const int64_t n = db->n;
  const int m = db->m;
  DvQuery* qs = nullptr;
  uint8_t* qct = nullptr;
  unsigned int* hist = nullptr;
  PQS_TRY(scratch(ctx, S_QMINMAX, (size_t)nq * sizeof(DvQuery) / 8 + 1, (double**)&qs));
  PQS_TRY(scratch(ctx, S_QT_WORK, (size_t)nq * m * kbar, &qct));
  PQS_TRY(scratch(ctx, S_SAMPLE, (size_t)nq * 256, &hist));
  PQS_CUDA(ctx, cudaMemsetAsync(hist, 0, sizeof(unsigned int) * nq * 256, ctx->stream));
  dv_params_kernel<<<(unsigned)nq, DV_THREADS, 0, ctx->stream>>>(d_compact, db->codes8, n, m, kbar, r2, qs, qct);
  PQS_LAUNCHED(ctx);
  const dim3 grid((unsigned)cdiv(n, DV_TILE), (unsigned)nq);
  const size_t qsm = (size_t)m * kbar;
  dv_hist_kernel<<<grid, DV_THREADS, qsm, ctx->stream>>>(db->codes8, n, m, kbar, qct, hist);
  PQS_LAUNCHED(ctx);
  dv_bound_kernel<<<(unsigned)cdiv(nq, 4), 128, 0, ctx->stream>>>(hist, nq, n, r2, qs);
  PQS_LAUNCHED(ctx);
  // candidate capacity: the largest kept count (one host sync)
  std::vector<DvQuery> hq((size_t)nq);
  PQS_CUDA(ctx, cudaMemcpyAsync(hq.data(), qs, sizeof(DvQuery) * nq, cudaMemcpyDeviceToHost, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int64_t cap = 1;
  for (const DvQuery& x : hq) cap = std::max<int64_t>(cap, std::min<int64_t>(x.kept, n));
  PQS_CHECK(ctx, cap < (1ll << 31), "derived search: too many kept candidates");
  uint64_t* cand = nullptr;
  int* cnt = nullptr;
  uint64_t* gk = nullptr;
  int64_t* gi = nullptr;
  PQS_TRY(scratch(ctx, S_CAND, (size_t)(nq * cap), &cand));
  PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)nq, &cnt));
  PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * cap), &gk));
  PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * cap), &gi));
  PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
  PQS_TRY(scan_timer_begin(ctx));
  dv_collect_kernel<<<grid, DV_THREADS, qsm, ctx->stream>>>(db->codes8, n, m, kbar, r2, qct, qs, cand, cnt, cap);
  PQS_LAUNCHED(ctx);
  SelArgs s{};
  s.src = SEL_CAND_ADC;
  s.nq = nq;
  s.r = r;
  s.cand = cand;
  s.cand_cnt = cnt;
  s.cap = cap;
  s.tables = d_full;
  s.codes8 = db->codes8;
  s.codes_rm = db->codes_rm;
  s.m = m;
  s.k = k;
  s.ids = db->ids;
  s.id_base = db->id_base;
  s.out_d = d_dist;
  s.out_i = d_ids;
  s.out_c = d_count;
  s.gkeys = gk;
  s.gids = gi;
  s.gcap = cap;
  PQS_TRY(launch_select(ctx, s));
  PQS_TRY(scan_timer_end(ctx));
  ctx->last_scan_launches = 1;
  ctx->last_scan_engine = 6;
  ctx->last_evals = n * nq;
  int64_t tot = 0;
  for (const DvQuery& x : hq) tot += std::min<int64_t>(x.kept, n);
  ctx->last_cand_total = tot;
  ctx->last_overflow = 0;
  return PQS_OK;
}

// query_ivf kernel='derived' for a batch of queries
int run_ivf_derived_search(pqs_ctx* ctx, const pqs_ivf* iv, const float* d_dbooks, int kbar, QVec d_queries,
                           int64_t nq, int ma, int r, int64_t r2, double* d_dist, int64_t* d_ids, int32_t* d_count) {
  const int m = iv->m, k = iv->k;
  const size_t smem = (size_t)m * k * 4 + (size_t)m * kbar * 4 + (size_t)m * kbar;
  PQS_CHECK(ctx, smem <= 200 * 1024, "derived IVF kernel: m * k too large for the shared-memory tables");
  int64_t* cells = nullptr;
  double* pdist = nullptr;
  PQS_TRY(scratch(ctx, S_PROBE, (size_t)(nq * ma), &cells));
  PQS_TRY(scratch(ctx, S_PROBE_D, (size_t)(nq * ma), &pdist));
  PQS_TRY(run_ivf_probe(ctx, iv, d_queries, nq, ma, cells, pdist));
  const int64_t cap = (int64_t)ma * r;
  const int64_t QB = std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t)(32ll << 20) / cap));
  uint64_t* cand = nullptr;
  int64_t* pids = nullptr;
  int* cnt = nullptr;
  uint64_t* gk = nullptr;
  int64_t* gi = nullptr;
  PQS_TRY(scratch(ctx, S_CAND, (size_t)(QB * cap), &cand));
  PQS_TRY(scratch(ctx, S_PIDS, (size_t)(QB * cap), &pids));
  PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)QB, &cnt));
  PQS_TRY(scratch(ctx, S_KEYS, (size_t)(QB * cap), &gk));
  PQS_TRY(scratch(ctx, S_IDS, (size_t)(QB * cap), &gi));
  PQS_CUDA(ctx, cudaFuncSetAttribute(dv_ivf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PQS_TRY(scan_timer_begin(ctx));
  for (int64_t q0 = 0; q0 < nq; q0 += QB) {
    const int64_t nb = std::min(QB, nq - q0);
    PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nb, ctx->stream));
    DvIvfArgs a{};
    a.queries = d_queries;
    a.coarse = iv->coarse;
    a.books = iv->books;
    a.dbooks = d_dbooks;
    a.offsets = iv->offsets;
    a.codes = iv->codes;
    a.ids = iv->ids;
    a.cells = cells;
    a.q0 = q0;
    a.ma = ma;
    a.m = m;
    a.k = k;
    a.kbar = kbar;
    a.d = iv->d;
    a.dsub = iv->dsub;
    a.r = r;
    a.r2 = r2;
    a.cand = cand;
    a.pids = pids;
    a.cnt = cnt;
    a.cap = cap;
    dv_ivf_kernel<<<(unsigned)(nb * ma), DV_THREADS, smem, ctx->stream>>>(a);
    PQS_LAUNCHED(ctx);
    SelArgs s{};
    s.src = SEL_KEYS;
    s.nq = nb;
    s.r = r;
    s.cand = cand;
    s.cand_cnt = cnt;
    s.cap = cap;
    s.pids = pids;
    s.out_d = d_dist + q0 * r;
    s.out_i = d_ids + q0 * r;
    s.out_c = d_count + q0;
    s.gkeys = gk;
    s.gids = gi;
    s.gcap = cap;
    PQS_TRY(launch_select(ctx, s));
  }
  PQS_TRY(scan_timer_end(ctx));
  ctx->last_scan_engine = 7;
  std::vector<int64_t> hcells((size_t)(nq * ma));
  PQS_CUDA(ctx, cudaMemcpyAsync(hcells.data(), cells, sizeof(int64_t) * nq * ma, cudaMemcpyDeviceToHost, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  PQS_TRY(scan_timer_collect(ctx));
  int64_t total = 0;
  for (int64_t c : hcells)
    if (c >= 0) total += iv->h_offsets[c + 1] - iv->h_offsets[c];
  ctx->last_evals = total;
  ctx->last_overflow = 0;
  return PQS_OK;
}
