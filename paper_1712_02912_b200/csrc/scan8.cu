// scan8.cu -- float ADC over 8-bit codes (K3 scan, K6 rerank via select.cu).
//
// Reference: scan_distances / scan (scan.py:68-81, 197-203).
//
// K3 design: lane = query.  A CTA owns a group of 32
// queries and W warps; all warps share the group's tables, staged in shared
// memory in [component][entry][lane] fp32 order so that 32 lanes reading the
// same entry of their own table hit 32 distinct banks (conflict-free for any
// code).  Codes are broadcast: the device layout is tile-transposed
// ([tile][component][1024 codes]) so a warp reads 16 codes' bytes of one
// component with one broadcast LDS.128.  Each warp owns 64 codes of the 1024
// code tile and keeps 64 fp32 partial sums per lane in registers while the
// tables stream through shared memory in component chunks.  Chunks (tables +
// the tile's matching code bytes) are double-buffered with TMA bulk copies
// (cp.async.bulk + mbarrier).  The fp32 sums are a filter only: every code
// whose fp32 distance is within the certified error bound of the threshold
// becomes a candidate, and candidates are re-scored exactly in fp64 in the
// reference's order before the (distance, id) selection.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "pqs_common.cuh"

namespace {

constexpr int W8 = 16;              // warps per CTA
constexpr int C8 = TILE8 / W8;     // codes per warp (64)
constexpr int SCAN8_THREADS = W8 * 32;
constexpr int CHUNK_BUDGET = 96 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------- table layout
// tables (nq, m, k) -> tt [qg][j][c][32]; aerr[q] = certified bound on
// |fp32 sum - fp64 sum| of any code's distance (recursive summation).
__global__ void tables_scan8_kernel(const float* __restrict__ tables, int64_t nq, int m, int k,
                                    float* __restrict__ tt) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nqg = cdiv(nq, 32);
  const int64_t total = nqg * m * (int64_t)k * 32;
  if (gid >= total) return;
  const int lane = (int)(gid & 31);
  int64_t t = gid >> 5;
  const int c = (int)(t % k);
  t /= k;
  const int j = (int)(t % m);
  const int64_t qg = t / m;
  const int64_t q = qg * 32 + lane;
  tt[gid] = q < nq ? tables[(q * m + j) * (int64_t)k + c] : 0.0f;
}

__global__ void aerr_kernel(const float* __restrict__ tables, int64_t nq, int m, int k, float* __restrict__ aerr) {
  const int64_t q = blockIdx.x;
  __shared__ double part[32];
  double s = 0.0;
  // one warp per component round-robin
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < m; j += nw) {
    float mx = 0.f;
    for (int c = lane; c < k; c += 32) mx = fmaxf(mx, fabsf(tables[(q * m + j) * (int64_t)k + c]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    s += (double)mx;
  }
  if (lane == 0) part[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int i = 0; i < nw; ++i) tot += part[i];
    // gamma_{m} for fp32 (u = 2^-24) plus fp64 (u = 2^-53), with slack
    const double u32 = 5.9604644775390625e-08, u64 = 1.1102230246251565e-16;
    const double g = (double)m * u32 / (1.0 - (double)m * u32) + (double)m * u64 * 2.0;
    aerr[q] = (float)(tot * g * 1.01 + 1e-30);
  }
}

// --------------------------------------------------------------- K3 kernel
enum { MODE8_DENSE = 0, MODE8_FILTER = 1 };

struct Scan8Args {
  const float* tt;         // [nqg][m][k][32]
  const uint8_t* codes;    // [ntiles][m][TILE8]
  int64_t n;
  int m, k, mc;
  int64_t nq;
  int64_t nvt, tile_off, tile_step, per_cta;
  float* out;              // dense [q][ld]
  int64_t ld;
  const float* theta;      // filter
  uint64_t* cand;
  int* cand_cnt;
  int64_t cap;
};

template <int MODE>
__global__ void __launch_bounds__(SCAN8_THREADS, 1) scan8_kernel(Scan8Args a) {
  extern __shared__ __align__(128) unsigned char sm8[];
  __shared__ __align__(8) uint64_t bars[2];
  const int m = a.m, k = a.k, mc = a.mc;
  const uint32_t tab_bytes = (uint32_t)mc * k * 32 * 4;
  const uint32_t code_bytes = (uint32_t)mc * TILE8;
  // buffer b: tables at sm8 + b*tab_bytes, codes at sm8 + 2*tab_bytes + b*code_bytes

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t qg = blockIdx.y;
  const int64_t q = qg * 32 + lane;
  const bool qvalid = q < a.nq;
  const float theta = (MODE == MODE8_FILTER && qvalid) ? a.theta[q] : 0.f;

  const int64_t i0 = blockIdx.x * a.per_cta;
  const int64_t i1 = min(i0 + a.per_cta, a.nvt);
  if (i0 >= i1) return;
  const int nch = (m + mc - 1) / mc;
  const int64_t S = (i1 - i0) * nch;  // stages

  const float* tt_q = a.tt + qg * (int64_t)m * k * 32;
  auto issue_at = [&](int b, int64_t vi, int ch) {
    const int j0 = ch * mc;
    const int mcur = min(mc, m - j0);
    const int64_t tile = a.tile_off + vi * a.tile_step;
    const uint32_t tb = (uint32_t)mcur * k * 32 * 4, cb = (uint32_t)mcur * TILE8;
    mbar_expect_tx(&bars[b], tb + cb);
    bulk_g2s(sm8 + b * tab_bytes, tt_q + (int64_t)j0 * k * 32, tb, &bars[b]);
    bulk_g2s(sm8 + 2 * tab_bytes + b * code_bytes, a.codes + (tile * m + j0) * (int64_t)TILE8, cb, &bars[b]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    issue_at(0, i0, 0);
    if (S > 1) {
      if (nch > 1) issue_at(1, i0, 1);
      else issue_at(1, i0 + 1, 0);
    }
  }

  float part[C8];
#pragma unroll
  for (int c = 0; c < C8; ++c) part[c] = 0.f;

  int64_t s = 0;
  for (int64_t vi = i0; vi < i1; ++vi) {
    const int64_t tile = a.tile_off + vi * a.tile_step;
    for (int ch = 0; ch < nch; ++ch, ++s) {
      const int b = (int)(s & 1);
      mbar_wait(&bars[b], (uint32_t)((s >> 1) & 1));
      const int mcur = min(mc, m - ch * mc);
      const float* T = reinterpret_cast<const float*>(sm8 + b * tab_bytes) + lane;
      const uint8_t* cb = sm8 + 2 * tab_bytes + b * code_bytes + warp * C8;
#pragma unroll
      for (int v = 0; v < C8 / 16; ++v) {
        const uint8_t* cv = cb + v * 16;
        for (int jj = 0; jj < mcur; ++jj) {
          const float* Tj = T + jj * k * 32;
          const uint4 w = *reinterpret_cast<const uint4*>(cv + jj * TILE8);
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t code = (ws[e >> 2] >> (8 * (e & 3))) & 0xFFu;
            part[v * 16 + e] += Tj[code * 32];
          }
        }
      }
      if (ch == nch - 1) {
        const int64_t c0 = tile * TILE8 + warp * C8;
        if (MODE == MODE8_FILTER) {
          if (qvalid) {
#pragma unroll
            for (int c = 0; c < C8; ++c) {
              if (part[c] <= theta && c0 + c < a.n) {
                const int pos = atomicAdd(a.cand_cnt + q, 1);
                if (pos < a.cap) a.cand[q * a.cap + pos] = (uint64_t)(uint32_t)(c0 + c);
              }
            }
          }
        } else {
          if (qvalid) {
            const int64_t col = vi * TILE8 + warp * C8;
            const float inf = __int_as_float(0x7f800000);
#pragma unroll
            for (int c = 0; c < C8; c += 4) {
              float4 o;
              o.x = (c0 + c + 0 < a.n) ? part[c + 0] : inf;
              o.y = (c0 + c + 1 < a.n) ? part[c + 1] : inf;
              o.z = (c0 + c + 2 < a.n) ? part[c + 2] : inf;
              o.w = (c0 + c + 3 < a.n) ? part[c + 3] : inf;
              if (col + c + 3 < a.ld) *reinterpret_cast<float4*>(a.out + q * a.ld + col + c) = o;
            }
          }
        }
#pragma unroll
        for (int c = 0; c < C8; ++c) part[c] = 0.f;
      }
      __syncthreads();
      if (threadIdx.x == 0 && s + 2 < S) {
        // stage s+2 lives in buffer b: its tile/chunk follow (vi, ch) by two steps
        int ch2 = ch + 2;
        int64_t vi2 = vi;
        while (ch2 >= nch) {
          ch2 -= nch;
          ++vi2;
        }
        issue_at(b, vi2, ch2);
      }
    }
  }
}

int pick_mc(int m, int k) {
  int mc = CHUNK_BUDGET / (k * 128 + TILE8);
  mc = std::max(1, std::min(mc, m));
  return mc;
}

template <int MODE>
int launch_scan8(pqs_ctx* ctx, Scan8Args a) {
  a.mc = pick_mc(a.m, a.k);
  const size_t smem = 2 * ((size_t)a.mc * a.k * 128 + (size_t)a.mc * TILE8);
  PQS_CUDA(ctx, cudaFuncSetAttribute(scan8_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t qgroups = cdiv(a.nq, 32);
  const int64_t target = (int64_t)ctx->sm_count * 4;
  int64_t splits = std::max<int64_t>(1, cdiv(target, qgroups));
  splits = std::min<int64_t>(splits, a.nvt);
  a.per_cta = cdiv(a.nvt, splits);
  splits = cdiv(a.nvt, a.per_cta);
  dim3 grid((unsigned)splits, (unsigned)qgroups);
  scan8_kernel<MODE><<<grid, SCAN8_THREADS, smem, ctx->stream>>>(a);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

// float threshold: theta = r-th smallest valid sample value + 2*aerr, rounded up
__global__ void theta8_kernel(const float* __restrict__ sample, int64_t ns, int r, const float* __restrict__ aerr,
                              float* __restrict__ theta) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned int s_prefix, s_k, s_valid;
  const int64_t q = blockIdx.x;
  const float* row = sample + q * ns;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_k = (unsigned)(r - 1);
    s_valid = 0;
  }
  __syncthreads();
  unsigned int valid = 0;
  for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) valid += isfinite(row[i]) ? 1u : 0u;
  atomicAdd(&s_valid, valid);
  __syncthreads();
  if (s_valid < (unsigned)r) {
    if (threadIdx.x == 0) theta[q] = __int_as_float(0x7f800000);
    return;
  }
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned prefix = s_prefix;
    for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
      const float v = row[i];
      if (!isfinite(v)) continue;
      const unsigned key = fkey(v);
      const bool match = (shift == 24) ? true : ((key ^ prefix) >> (shift + 8)) == 0;
      if (match) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned c = 0, kk = s_k;
      int d = 0;
      for (; d < 256; ++d) {
        if (kk < c + hist[d]) break;
        c += hist[d];
      }
      s_k = kk - c;
      s_prefix = prefix | ((unsigned)d << shift);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double t = (double)fkey_inv(s_prefix) + 2.0 * (double)aerr[q];
    float f = (float)t;
    if ((double)f < t) f = nextafterf(f, __int_as_float(0x7f800000));
    theta[q] = nextafterf(f, __int_as_float(0x7f800000));
  }
}

__global__ void fill_f32_kernel(float* p, int64_t n, float v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// dense exact fp64 ADC (scan_distances), optional query map
__global__ void dense_adc_kernel(const float* __restrict__ tables, const uint8_t* __restrict__ codes, int64_t n, int m,
                                 int k, int64_t nq, const int* __restrict__ qmap, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t ql = blockIdx.y;
  if (i >= n) return;
  const int64_t q = qmap ? qmap[ql] : ql;
  const float* T = tables + q * (int64_t)m * k;
  const uint8_t* base = codes + (i / TILE8) * (int64_t)m * TILE8 + (i % TILE8);
  double acc = 0.0;
  for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, (double)__ldg(T + (int64_t)j * k + base[(int64_t)j * TILE8]));
  out[ql * n + i] = acc;
}

}  // namespace

// ---------------------------------------------------------------------------
int build_db8(pqs_ctx* ctx, pqs_db* db, const uint8_t* h_codes) {
  // host-side tile transpose into pinned staging, then one copy
  const int64_t n = db->n, m = db->m;
  const size_t bytes = (size_t)db->ntiles * m * TILE8;
  std::vector<uint8_t> h(bytes, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t t = i / TILE8, c = i % TILE8;
    uint8_t* dst = h.data() + t * m * TILE8 + c;
    const uint8_t* src = h_codes + i * m;
    for (int64_t j = 0; j < m; ++j) dst[j * TILE8] = src[j];
  }
  PQS_CUDA(ctx, cudaMemcpyAsync(db->codes8, h.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PQS_OK;
}

int launch_scan_distances(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, double* d_out) {
  if (db->n == 0 || nq == 0) return PQS_OK;
  dim3 grid((unsigned)cdiv(db->n, 256), (unsigned)nq);
  dense_adc_kernel<<<grid, 256, 0, ctx->stream>>>(d_tables, db->codes8, db->n, db->m, db->k, nq, nullptr, d_out);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int launch_tables_scan8(pqs_ctx* ctx, const float* d_tables, int64_t nq, int m, int k, float* d_tt, float* d_aerr) {
  const int64_t total = cdiv(nq, 32) * m * (int64_t)k * 32;
  tables_scan8_kernel<<<(unsigned)cdiv(total, 256), 256, 0, ctx->stream>>>(d_tables, nq, m, k, d_tt);
  PQS_LAUNCHED(ctx);
  aerr_kernel<<<(unsigned)nq, 256, 0, ctx->stream>>>(d_tables, nq, m, k, d_aerr);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int run_adc_topr(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, int r, double* d_dist,
                 int64_t* d_ids, int32_t* d_count) {
  const int64_t n = db->n;
  const int m = db->m, k = db->k;
  if (n == 0) {
    // nothing to scan: every row is empty
    SelArgs s{};
    s.src = SEL_DENSE_F64;
    s.nq = nq;
    s.r = r;
    s.n = 0;
    s.dense = nullptr;
    s.out_d = d_dist;
    s.out_i = d_ids;
    s.out_c = d_count;
    return launch_select(ctx, s);
  }
  float* tt = nullptr;
  float* aerr = nullptr;
  PQS_TRY(scratch(ctx, S_TABLES_T, (size_t)(cdiv(nq, 32) * 32 * m * k), &tt));
  PQS_TRY(scratch(ctx, S_AERR, (size_t)nq, &aerr));
  PQS_TRY(launch_tables_scan8(ctx, d_tables, nq, m, k, tt, aerr));

  float* theta = nullptr;
  PQS_TRY(scratch(ctx, S_THETA, (size_t)nq * 4, (uint8_t**)&theta));
  const int64_t cap = std::min<int64_t>(ctx->cand_cap, n);
  const int64_t r_eff = std::min<int64_t>(r, n);
  if (n <= cap) {
    fill_f32_kernel<<<(unsigned)cdiv(nq, 256), 256, 0, ctx->stream>>>(theta, nq, __builtin_huge_valf());
    PQS_LAUNCHED(ctx);
  } else {
    int64_t st = std::max<int64_t>(cdiv(db->ntiles, ctx->sample_div), cdiv(16 * r_eff, TILE8));
    st = std::min<int64_t>(st, db->ntiles);
    const int64_t step = std::max<int64_t>(1, db->ntiles / st);
    const int64_t ns = st * TILE8;
    float* sample = nullptr;
    PQS_TRY(scratch(ctx, S_SAMPLE, (size_t)(nq * ns) * 4, (uint8_t**)&sample));
    Scan8Args a{};
    a.tt = tt;
    a.codes = db->codes8;
    a.n = n;
    a.m = m;
    a.k = k;
    a.nq = nq;
    a.nvt = st;
    a.tile_off = 0;
    a.tile_step = step;
    a.out = sample;
    a.ld = ns;
    PQS_TRY(launch_scan8<MODE8_DENSE>(ctx, a));
    theta8_kernel<<<(unsigned)nq, 256, 0, ctx->stream>>>(sample, ns, (int)r_eff, aerr, theta);
    PQS_LAUNCHED(ctx);
  }

  uint64_t* cand = nullptr;
  int* cnt = nullptr;
  PQS_TRY(scratch(ctx, S_CAND, (size_t)(nq * cap), &cand));
  PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)nq, &cnt));
  PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
  {
    Scan8Args a{};
    a.tt = tt;
    a.codes = db->codes8;
    a.n = n;
    a.m = m;
    a.k = k;
    a.nq = nq;
    a.nvt = db->ntiles;
    a.tile_off = 0;
    a.tile_step = 1;
    a.theta = theta;
    a.cand = cand;
    a.cand_cnt = cnt;
    a.cap = cap;
    PQS_TRY(scan_timer_begin(ctx));
    PQS_TRY(launch_scan8<MODE8_FILTER>(ctx, a));
    PQS_TRY(scan_timer_end(ctx));
    ctx->last_scan_launches = 1;
  }
  ctx->last_evals = nq * n;

  uint64_t* gk = nullptr;
  int64_t* gi = nullptr;
  PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * cap), &gk));
  PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * cap), &gi));
  SelArgs s{};
  s.src = SEL_CAND_ADC;
  s.nq = nq;
  s.r = r;
  s.cand = cand;
  s.cand_cnt = cnt;
  s.cap = cap;
  s.ids = db->ids;
  s.id_base = db->id_base;
  s.tables = d_tables;
  s.codes8 = db->codes8;
  s.m = m;
  s.k = k;
  s.out_d = d_dist;
  s.out_i = d_ids;
  s.out_c = d_count;
  s.gkeys = gk;
  s.gids = gi;
  s.gcap = cap;
  PQS_TRY(launch_select(ctx, s));

  std::vector<int> hcnt(nq);
  PQS_CUDA(ctx, cudaMemcpyAsync(hcnt.data(), cnt, sizeof(int) * nq, cudaMemcpyDeviceToHost, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  PQS_TRY(scan_timer_collect(ctx));
  std::vector<int> over;
  int64_t mx = 0;
  for (int64_t q = 0; q < nq; ++q) {
    mx = std::max<int64_t>(mx, hcnt[q]);
    if (hcnt[q] > cap || hcnt[q] < r_eff || ctx->force_fallback) over.push_back((int)q);
  }
  ctx->last_max_cand = mx;
  ctx->last_overflow = (int64_t)over.size();
  if (!over.empty()) {
    const int64_t B = std::max<int64_t>(1, std::min<int64_t>((int64_t)over.size(), (int64_t)(1ll << 27) / n));
    int* d_qmap = nullptr;
    double* dense = nullptr;
    PQS_TRY(scratch(ctx, S_MISC, (size_t)over.size(), &d_qmap));
    PQS_TRY(scratch(ctx, S_DENSE, (size_t)(B * n), &dense));
    PQS_CUDA(ctx, cudaMemcpyAsync(d_qmap, over.data(), sizeof(int) * over.size(), cudaMemcpyHostToDevice, ctx->stream));
    for (int64_t b0 = 0; b0 < (int64_t)over.size(); b0 += B) {
      const int64_t nb = std::min<int64_t>(B, (int64_t)over.size() - b0);
      dim3 grid((unsigned)cdiv(n, 256), (unsigned)nb);
      dense_adc_kernel<<<grid, 256, 0, ctx->stream>>>(d_tables, db->codes8, n, m, k, nb, d_qmap + b0, dense);
      PQS_LAUNCHED(ctx);
      SelArgs f{};
      f.src = SEL_DENSE_F64;
      f.nq = nb;
      f.r = r;
      f.dense = dense;
      f.n = n;
      f.ids = db->ids;
      f.id_base = db->id_base;
      f.qmap = d_qmap + b0;
      f.out_d = d_dist;
      f.out_i = d_ids;
      f.out_c = d_count;
      PQS_TRY(launch_select(ctx, f));
    }
  }
  return PQS_OK;
}
