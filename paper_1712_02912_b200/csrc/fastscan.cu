// fastscan.cu -- PQ Fast Scan (fastscan.py:328-386) on the device.
//
// The reference's fast_scan returns exactly scan()'s neighbour set (its
// pruning is certified) plus ScanStats counting the codes whose exact
// distance it evaluated.  That count follows from a sequential process: the
// first n_init = ceil(init * n) codes are scanned exactly; then, chunk by
// chunk of 1024 codes, a code is evaluated iff its 8-bit lower bound
// lb = min(127, sum_{j<4} qt[j][c_j] + sum_{j>=4} min16(qt[j])[c_j >> 4])
// is <= quantize(params, worst), worst = the current r-th best distance.
//
// Pruned codes can never enter the top-r (lb <= quantize(d) and quantize is
// monotone), so before chunk c the neighbour set holds exactly the r best of
// all codes in [0, start_c), and quantize(worst_c) = the smallest bin t such
// that at least r of those codes have quantize(d) <= t (127 -- or 0 when the
// scale is 0 -- while fewer than r are held).  The device therefore needs no
// sequential scan over codes:
//   fs_params_kernel  per query: qmin, qmax (r-th smallest exact distance of
//                     the prefix, quickadc-style), the 127-bin tables and the
//                     4 x 16 portion minima of tables 4-7;
//   fs_hist_kernel    per (chunk, query): histograms of quantize(d) and of lb
//                     over the chunk (the prefix is chunk "-1");
//   fs_count_kernel   per query, one warp: walks the chunk histograms in
//                     order, deriving each chunk's threshold from the running
//                     bin counts, and sums the evaluated codes.
// Exact distances come from the dense ADC kernel (scan8.cu).  The neighbour
// set itself is scan()'s, computed by the float ADC path.
#include <cuda_runtime.h>

#include <algorithm>

#include "pqs_common.cuh"
#include "select_dev.cuh"

namespace {

using namespace seldev;

constexpr int FS_CHUNK = 1024;   // fastscan.py:325 (_CHUNK)
constexpr int FS_THREADS = 256;

struct FsParams {
  double qmin, qmax, scale;
};

// one CTA per query: params, quantized tables (8 x 256) and minima (4 x 16)
__global__ void __launch_bounds__(FS_THREADS) fs_params_kernel(const float* __restrict__ tables,
                                                               const double* __restrict__ dist, int64_t n,
                                                               int64_t n_init, int r, FsParams* __restrict__ prm,
                                                               uint8_t* __restrict__ qt_out) {
  __shared__ SelShared sh;
  __shared__ float fred[FS_THREADS / 32];
  __shared__ uint8_t qt[8 * 256];
  __shared__ double s_q[2];
  const int64_t q = blockIdx.x;
  const float* T = tables + q * 2048;
  const double* dq = dist + q * n;
  float mn = __int_as_float(0x7f800000);
  for (int i = threadIdx.x; i < 2048; i += FS_THREADS) mn = fminf(mn, T[i]);
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) fred[threadIdx.x >> 5] = mn;
  // qmax: r-th smallest of the prefix distances, largest when n_init < r
  // (compute_quant_params / fast_scan, fastscan.py:355-358)
  auto get = [&](int64_t i, uint64_t& v) -> bool {
    v = dkey(dq[i]);
    return true;
  };
  block_radix_select(n_init, get, (unsigned long long)(n_init >= r ? r - 1 : n_init - 1), sh);
  if (threadIdx.x == 0) {
    float a = fred[0];
    for (int i = 1; i < FS_THREADS / 32; ++i) a = fminf(a, fred[i]);
    const double qmin = (double)a;
    double qmax = dkey_inv(sh.prefix);
    qmax = qmax > qmin ? qmax : qmin;  // QuantParams(qmin, max(qmax, qmin))
    const double span = __dsub_rn(qmax, qmin);
    const double scale = span > 0.0 ? __ddiv_rn(127.0, span) : 0.0;
    prm[q] = FsParams{qmin, qmax, scale};
    s_q[0] = qmin;
    s_q[1] = qmax;
  }
  __syncthreads();
  const double qmin = s_q[0], qmax = s_q[1];
  const double span = __dsub_rn(qmax, qmin);
  const double scale = span > 0.0 ? __ddiv_rn(127.0, span) : 0.0;
  for (int i = threadIdx.x; i < 2048; i += FS_THREADS) qt[i] = quantize1((double)T[i], qmin, qmax, scale);
  __syncthreads();
  uint8_t* o = qt_out + q * (2048 + 64);
  for (int i = threadIdx.x; i < 2048; i += FS_THREADS) o[i] = qt[i];
  // _min_tables (fastscan.py:258-260): minima of the 16 portions of tables 4-7
  if (threadIdx.x < 64) {
    const int j = 4 + (threadIdx.x >> 4), p = threadIdx.x & 15;
    int mv = 255;
    for (int u = 0; u < 16; ++u) mv = min(mv, (int)qt[j * 256 + p * 16 + u]);
    o[2048 + threadIdx.x] = (uint8_t)mv;
  }
}

// grid (n_chunks + 1, nq): histograms of quantize(d) (all chunks incl. the
// prefix = blockIdx.x 0) and of the lower bound (chunks only)
__global__ void __launch_bounds__(FS_THREADS) fs_hist_kernel(const uint8_t* __restrict__ codes8, int64_t n,
                                                             int64_t n_init, const double* __restrict__ dist,
                                                             const FsParams* __restrict__ prm,
                                                             const uint8_t* __restrict__ qt_all,
                                                             unsigned int* __restrict__ binh,
                                                             unsigned int* __restrict__ lbh, int64_t nch) {
  __shared__ unsigned int hb[128], hl[128];
  __shared__ uint8_t qt[2048 + 64];
  const int64_t q = blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x - 1;
  const int64_t b = c < 0 ? 0 : n_init + c * FS_CHUNK;
  const int64_t e = c < 0 ? n_init : min(n, b + FS_CHUNK);
  for (int i = threadIdx.x; i < 128; i += FS_THREADS) hb[i] = hl[i] = 0;
  const uint8_t* qg = qt_all + q * (2048 + 64);
  for (int i = threadIdx.x; i < 2048 + 64; i += FS_THREADS) qt[i] = qg[i];
  __syncthreads();
  const FsParams P = prm[q];
  const double* dq = dist + q * n;
  for (int64_t i = b + threadIdx.x; i < e; i += FS_THREADS) {
    atomicAdd(&hb[quantize1(dq[i], P.qmin, P.qmax, P.scale)], 1u);
    if (c >= 0) {
      // tile-transposed layout: byte (t, j, cc) at t*8*1024 + j*1024 + cc
      const uint8_t* cp = codes8 + (i / TILE8) * 8 * TILE8 + (i % TILE8);
      int acc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc += qt[j * 256 + cp[j * TILE8]];
#pragma unroll
      for (int j = 4; j < 8; ++j) acc += qt[2048 + (j - 4) * 16 + (cp[j * TILE8] >> 4)];
      atomicAdd(&hl[acc < 127 ? acc : 127], 1u);
    }
  }
  __syncthreads();
  unsigned int* ob = binh + (q * (nch + 1) + blockIdx.x) * 128;
  for (int i = threadIdx.x; i < 128; i += FS_THREADS) ob[i] = hb[i];
  if (c >= 0) {
    unsigned int* ol = lbh + (q * nch + c) * 128;
    for (int i = threadIdx.x; i < 128; i += FS_THREADS) ol[i] = hl[i];
  }
}

// one warp per query: the sequential threshold refresh of fast_scan
// (fastscan.py:364-383) from the per-chunk histograms; lane l owns bins 4l..4l+3
__global__ void fs_count_kernel(const unsigned int* __restrict__ binh, const unsigned int* __restrict__ lbh,
                                const FsParams* __restrict__ prm, int64_t nq, int64_t nch, int64_t n_init, int r,
                                int64_t* __restrict__ checked) {
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const uint8_t empty_thr = prm[q].scale == 0.0 ? 0 : 127;  // quantize(params, inf)
  const unsigned int* bh = binh + q * (nch + 1) * 128;
  const unsigned int* lh = lbh + q * nch * 128;
  unsigned long long cum[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) cum[u] = bh[4 * lane + u];
  unsigned long long tot = (unsigned long long)n_init;
  for (int64_t c = 0; c < nch; ++c) {
    // threshold = smallest bin t with >= r codes at bins <= t (else empty_thr)
    unsigned long long s4 = cum[0] + cum[1] + cum[2] + cum[3], incl = s4;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(full, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned long long excl = incl - s4;
    int cand = 128;
    if (excl < (unsigned long long)r && incl >= (unsigned long long)r) {
      unsigned long long a = excl;
      for (int u = 0; u < 4; ++u) {
        a += cum[u];
        if (a >= (unsigned long long)r) {
          cand = 4 * lane + u;
          break;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(full, cand, o));
    const int thr = cand < 128 ? cand : empty_thr;
    // evaluated codes of the chunk: lower bound <= threshold
    const unsigned int* l = lh + c * 128;
    unsigned long long k = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) k += (4 * lane + u <= thr) ? l[4 * lane + u] : 0u;
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(full, k, o);
    tot += k;
    const unsigned int* nb = bh + (c + 1) * 128;
#pragma unroll
    for (int u = 0; u < 4; ++u) cum[u] += nb[4 * lane + u];
  }
  if (lane == 0) checked[q] = (int64_t)tot;
}

}  // namespace

// ScanStats.checked of fast_scan for a batch of tables (nq, 8, 256); the
// code list is the grouped database's codes in storage order (b = 8, m = 8)
int run_fastscan_checked(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, int64_t n_init, int r,
                         int64_t* d_checked) {
  const int64_t n = db->n;
  const int64_t nch = cdiv(std::max<int64_t>(n - n_init, 0), FS_CHUNK);
  const int64_t QB = std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t)(512ll << 20) / (8 * std::max<int64_t>(n, 1))));
  double* dist = nullptr;
  FsParams* prm = nullptr;
  uint8_t* qt = nullptr;
  unsigned int* binh = nullptr;
  unsigned int* lbh = nullptr;
  PQS_TRY(scratch(ctx, S_DENSE, (size_t)(QB * n), &dist));
  PQS_TRY(scratch(ctx, S_QMINMAX, (size_t)QB * 3, (double**)&prm));
  PQS_TRY(scratch(ctx, S_QT_WORK, (size_t)QB * (2048 + 64), &qt));
  PQS_TRY(scratch(ctx, S_KEYS, (size_t)QB * (nch + 1) * 128, &binh));
  PQS_TRY(scratch(ctx, S_IDS, (size_t)QB * std::max<int64_t>(nch, 1) * 128, &lbh));
  pqs_db dbk = *db;
  dbk.k = 256;
  for (int64_t q0 = 0; q0 < nq; q0 += QB) {
    const int64_t nb = std::min(QB, nq - q0);
    const float* t = d_tables + q0 * 2048;
    PQS_TRY(launch_scan_distances(ctx, &dbk, t, nb, dist));
    fs_params_kernel<<<(unsigned)nb, FS_THREADS, 0, ctx->stream>>>(t, dist, n, n_init, r, prm, qt);
    PQS_LAUNCHED(ctx);
    fs_hist_kernel<<<dim3((unsigned)(nch + 1), (unsigned)nb), FS_THREADS, 0, ctx->stream>>>(
        db->codes8, n, n_init, dist, prm, qt, binh, lbh, nch);
    PQS_LAUNCHED(ctx);
    fs_count_kernel<<<(unsigned)cdiv(nb, 4), 128, 0, ctx->stream>>>(binh, lbh, prm, nb, nch, n_init, r,
                                                                    d_checked + q0);
    PQS_LAUNCHED(ctx);
  }
  return PQS_OK;
}
