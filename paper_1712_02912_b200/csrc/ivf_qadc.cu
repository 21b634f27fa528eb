// ivf_qadc.cu -- IVF probing with the Quick ADC list kernel
// (query_ivf kernel='quick-adc', ivf.py:185-190).
//
// Reference semantics, per (query, probed cell c) with a non-empty list:
//   residual  = fp64(q) - fp64(coarse[c])                       ivf.py:179
//   tables    = compute_tables(pq, residual)   (m, 16) fp32    scan.py:45-56
//   part, qt  = qadc_scan(list, tables, min(init_count, n), r)  quickadc.py:104-141
//               (qmax from the list's first n_init codes, 127-bin saturated
//                sums, the list's r best by (bin, id))
//   merged.push(qt.rescale(bin), id) for every kept (bin, id)  quickadc.py:50-54
// and the answer is the r smallest (rescaled distance, id) over all probes
// (NeighborSet, scan.py:84-139).
//
// B200 design: probes come from K7 (run_ivf_probe, exact probe sets and
// order).  One CTA per (query, probe) pair does the whole per-list Quick ADC
// on chip: exact residual tables in shared memory (fp64, scipy's sequential
// order), qmax by a radix select over the prefix's fp64 ADC (recomputed per
// pass, no buffer), the 127-bin tables, a shared-memory bin histogram of the
// list (the per-list cut bin), a radix select over ids only when the cut bin
// holds more codes than needed, and the emission of exactly min(r, n)
// (rescaled distance key, id) pairs into the query's candidate row with one
// reservation.  K5 (select_kernel, SEL_KEYS) then takes the r smallest
// (distance, id) of the <= ma * r candidates.  Per-list selection by bin and
// the rescale-then-merge order are kept exactly as the reference does them:
// the rescale is monotone but not strictly, so merging bins instead would
// change tie-breaks.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "pqs_common.cuh"
#include "select_dev.cuh"

namespace {

using namespace seldev;

constexpr int QI_THREADS = 256;
constexpr int QI_MAX_M = 64;  // m * 16 table entries in shared memory

struct QiShared {
  SelShared sel;
  float T[QI_MAX_M * 16];
  uint8_t qt[QI_MAX_M * 16];
  unsigned int hist[128];
  float fred[QI_THREADS / 32];
  double qmin, qmax, span;
  int cut, need, tiebreak, emitted, eqleft;
  long long base;
  unsigned long long idcut;
};

__device__ __forceinline__ uint64_t id_key(int64_t id) { return (uint64_t)id ^ 0x8000000000000000ull; }

__global__ void __launch_bounds__(QI_THREADS) ivf_qadc_kernel(
    QVec queries, const float* __restrict__ coarse, const float* __restrict__ books,
    const int64_t* __restrict__ offsets, const uint8_t* __restrict__ codes, const int64_t* __restrict__ ids,
    const int64_t* __restrict__ cells, int64_t q0, int ma, int m, int d, int dsub, int init_count, int r,
    uint64_t* __restrict__ cand, int64_t* __restrict__ pids, int* __restrict__ cnt, int64_t cap) {
  __shared__ QiShared sh;
  const int64_t pair = blockIdx.x;           // (local query, probe)
  const int64_t ql = pair / ma;
  const int64_t c = cells[(q0 + ql) * ma + pair % ma];
  if (c < 0) return;
  const int64_t lb = offsets[c];
  const int64_t n = offsets[c + 1] - lb;
  if (n == 0) return;  // ivf.py:176-177
  const QVec qv = queries.offset((q0 + ql) * (int64_t)d);
  const float* g = coarse + c * (int64_t)d;
  const uint8_t* lc = codes + lb * (int64_t)m;
  const int64_t* li = ids + lb;
  const int ne = m * 16;

  // exact residual tables (ivf.py:179 -> scan.py:45-56 -> _dist.py:13-21)
  float mn = __int_as_float(0x7f800000);
  for (int e = threadIdx.x; e < ne; e += QI_THREADS) {
    const int j = e >> 4;
    const float* cb = books + (int64_t)e * dsub;
    double t = 0.0;
    for (int s = 0; s < dsub; ++s) {
      const int dd = j * dsub + s;
      const double rr = __dsub_rn(qv.at(dd), (double)__ldg(g + dd));
      const double df = __dsub_rn(rr, (double)__ldg(cb + s));
      t = __dadd_rn(t, __dmul_rn(df, df));
    }
    const float tf = __double2float_rn(t);
    sh.T[e] = tf;
    mn = fminf(mn, tf);
  }
  for (int i = threadIdx.x; i < 128; i += QI_THREADS) sh.hist[i] = 0;
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) sh.fred[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = sh.fred[0];
    for (int i = 1; i < QI_THREADS / 32; ++i) a = fminf(a, sh.fred[i]);
    sh.qmin = (double)a;  // qmin = float(tables.min()), quickadc.py:133
  }

  // qmax: the r-th smallest fp64 ADC of the first n_init codes (quickadc.py:129-132)
  const int64_t n_init = min((int64_t)init_count, n);
  const unsigned long long kq = (unsigned long long)(n_init >= r ? r - 1 : n_init - 1);
  const float* T = sh.T;
  auto prefix_get = [&](int64_t i, uint64_t& v) -> bool {
    if (i >= n_init) return false;
    const uint8_t* cp = lc + i * m;
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, (double)T[j * 16 + cp[j]]);  // scan.py:77-81
    v = dkey(acc);
    return true;
  };
  block_radix_select(n_init, prefix_get, kq, sh.sel);
  if (threadIdx.x == 0) {
    const double qmin = sh.qmin;
    double qmax = dkey_inv(sh.sel.prefix);
    qmax = qmax > qmin ? qmax : qmin;  // QuantParams(qmin, max(qmax, qmin))
    sh.qmax = qmax;
    sh.span = __dsub_rn(qmax, qmin);
  }
  __syncthreads();
  {
    const double qmin = sh.qmin, qmax = sh.qmax, span = sh.span;
    const double scale = span > 0.0 ? __ddiv_rn(127.0, span) : 0.0;  // fastscan.py:43-46
    for (int e = threadIdx.x; e < ne; e += QI_THREADS) sh.qt[e] = quantize1((double)T[e], qmin, qmax, scale);
  }
  __syncthreads();

  // saturated sums (quickadc.py:87-101: entries >= 0, so clamping once at the end is exact)
  const uint8_t* qt = sh.qt;
  auto bin_of = [&](int64_t i) -> int {
    const uint8_t* cp = lc + i * m;
    int s = 0;
    if ((m & 15) == 0) {
      for (int j0 = 0; j0 < m; j0 += 16) {
        const uint4 w = *reinterpret_cast<const uint4*>(cp + j0);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 16; ++u) s += qt[(j0 + u) * 16 + ((ws[u >> 2] >> (8 * (u & 3))) & 15u)];
      }
    } else {
      for (int j = 0; j < m; ++j) s += qt[j * 16 + cp[j]];
    }
    return s < 127 ? s : 127;
  };
  for (int64_t i = threadIdx.x; i < n; i += QI_THREADS) atomicAdd(&sh.hist[bin_of(i)], 1u);
  __syncthreads();
  const int r_eff = (int)min((int64_t)r, n);
  if (threadIdx.x == 0) {
    int cum = 0, b = 0;
    for (; b < 128; ++b) {
      if (cum + (int)sh.hist[b] >= r_eff) break;
      cum += (int)sh.hist[b];
    }
    sh.cut = b;
    sh.need = r_eff - cum;
    sh.tiebreak = (int)sh.hist[b] > sh.need;
    sh.emitted = 0;
    sh.base = atomicAdd(cnt + ql, r_eff);
  }
  __syncthreads();
  const int cut = sh.cut;
  // ties at the cut bin: the `need` smallest ids (_select_best lexsort, scan.py:150-154)
  if (sh.tiebreak) {
    auto tie_get = [&](int64_t i, uint64_t& v) -> bool {
      if (bin_of(i) != cut) return false;
      v = id_key(li[i]);
      return true;
    };
    block_radix_select(n, tie_get, (unsigned long long)(sh.need - 1), sh.sel);
    if (threadIdx.x == 0) {
      sh.idcut = sh.sel.prefix;
      sh.eqleft = sh.need - (int)sh.sel.less;
    }
    __syncthreads();
  }
  const bool tb = sh.tiebreak;
  const unsigned long long idcut = sh.idcut;
  const double qmin = sh.qmin, span = sh.span;
  uint64_t* crow = cand + ql * cap + sh.base;
  int64_t* prow = pids + ql * cap + sh.base;
  for (int64_t i = threadIdx.x; i < n; i += QI_THREADS) {
    const int b = bin_of(i);
    if (b > cut) continue;
    bool take = b < cut || !tb;
    if (!take) {
      const uint64_t k = id_key(li[i]);
      take = k < idcut || (k == idcut && atomicSub(&sh.eqleft, 1) > 0);
    }
    if (take) {
      const int s = atomicAdd(&sh.emitted, 1);
      // QuantizedTables4.rescale: bins * (qmax - qmin) / 127 + qmin (quickadc.py:50-54)
      const double v = __dadd_rn(__ddiv_rn(__dmul_rn((double)b, span), 127.0), qmin);
      crow[s] = dkey(v);
      prow[s] = li[i];
    }
  }
}

}  // namespace

// Batched query_ivf(kernel='quick-adc'): probes, per-(query, probe) Quick ADC
// top-r, K5 merge.  Queries are processed in batches so the candidate rows
// (ma * r per query) stay within a bounded scratch.
int run_ivf_qadc_search(pqs_ctx* ctx, const pqs_ivf* iv, QVec d_queries, int64_t nq, int ma, int r,
                        int init_count, double* d_dist, int64_t* d_ids, int32_t* d_count) {
  const int m = iv->m;
  PQS_CHECK(ctx, iv->k == 16, "the quick-adc kernel requires b = 4 (16-entry tables)");
  PQS_CHECK(ctx, m % 2 == 0, "quick-adc kernel requires b=4 and even m");
  PQS_CHECK(ctx, m <= QI_MAX_M, "quick-adc IVF kernel: m <= 64");
  PQS_CHECK(ctx, init_count >= 1, "init_count must be >= 1");
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
  PQS_TRY(scan_timer_begin(ctx));
  int64_t launches = 0;
  for (int64_t q0 = 0; q0 < nq; q0 += QB) {
    const int64_t nb = std::min(QB, nq - q0);
    PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nb, ctx->stream));
    ivf_qadc_kernel<<<(unsigned)(nb * ma), QI_THREADS, 0, ctx->stream>>>(
        d_queries, iv->coarse, iv->books, iv->offsets, iv->codes, iv->ids, cells, q0, ma, m, iv->d, iv->dsub,
        init_count, r, cand, pids, cnt, cap);
    PQS_LAUNCHED(ctx);
    ++launches;
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
  ctx->last_scan_launches = launches;
  ctx->last_scan_engine = 5;
  // evaluated codes (the metric's unit): every code of every probed list
  std::vector<int64_t> hcells((size_t)(nq * ma));
  PQS_CUDA(ctx, cudaMemcpyAsync(hcells.data(), cells, sizeof(int64_t) * nq * ma, cudaMemcpyDeviceToHost, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  PQS_TRY(scan_timer_collect(ctx));
  int64_t total = 0;
  for (int64_t c : hcells)
    if (c >= 0) total += iv->h_offsets[c + 1] - iv->h_offsets[c];
  ctx->last_evals = total;
  ctx->last_scan_work = (double)total * (double)m;
  ctx->last_overflow = 0;
  ctx->last_cand_total = 0;
  return PQS_OK;
}
