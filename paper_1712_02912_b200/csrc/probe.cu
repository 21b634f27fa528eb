// probe.cu -- K7: IVF probe selection on the tensor cores (tcgen05 kind::tf32).
//
// Reference: query_ivf probes the ma nearest coarse cells of the fp64 query
// (ivf.py:170-173) with nearest_k (_dist.py:42-67): fp64 cdist to every
// centroid, the ma smallest by (distance, cell index).  Output here: the same
// cells in the same order with the same fp64 distances (scipy's sequential
// sum of (q_t - c_t)^2), for a whole batch of queries.
//
// B200 design.  The distance ranking only needs key(c) = ||c||^2 - 2 q.c
// (= ||q - c||^2 - ||q||^2), a GEMM: the probe runs it on tcgen05 in TF32 with
// the norm folded into K -- A[q] = (q, 1, 1), B[c] = (-2c, hi(||c||^2),
// lo(||c||^2)) -- so the accumulator IS the key and the epilogue is a compare.
// Every approximation is covered by a certified bound eps_q (probe_eps_kernel)
// and every survivor is re-scored exactly, so the probe sets are exact:
//   pass 1 (MIN)     GEMM over a strided subset of the cell tiles; per query
//                    and 128-cell group the minimum key (one float).  The ma
//                    smallest group minima come from ma distinct cells, so
//                    the ma-th smallest of them bounds the ma-th smallest key
//                    of all cells from above (certified, no sampling risk).
//   theta            theta_q = that bound + 2 eps_q.
//   pass 2 (FILTER)  GEMM over all cells; the epilogue appends (key, cell) of
//                    every key <= theta_q to the query's candidate row -- no
//                    (nq, K) product block ever reaches HBM.
//   final            per query: the ma-th smallest candidate key t (= the
//                    ma-th smallest overall: every key <= theta was kept);
//                    cells with key <= t + 2 eps_q re-scored in fp64 (scipy
//                    order), the ma best by (distance, cell) sorted out.  A
//                    query whose candidate row overflowed is solved exactly by
//                    streaming all K cells (recomputed per radix pass).
// GEMM kernel: persistent, one CTA per SM, warp-specialised: a TMA warp
// bulk-copies the query block (A, resident, <= 128 x 256 tf32) and the cell
// tiles (B, 256 cells, in K stages of 4 MMA steps), one thread issues
// tcgen05.mma.kind::tf32 M=128 N=256 K=8 into two TMEM accumulators (2 x 256
// columns), 8 epilogue warps drain them (lane = query, column = cell).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pqs_common.cuh"
#include "select_dev.cuh"
#include "tc_common.cuh"

namespace {

using namespace seldev;

constexpr int PM = 128;                    // queries per block (TMEM lanes)
constexpr int PN = 256;                    // cells per tile (accumulator columns)
constexpr int PKS = 8;                     // tf32 elements per MMA K step (32 bytes)
constexpr int PSTEPS_PER_STAGE = 4;        // K steps per B stage
constexpr int PB_STEP = PN * PKS * 4;      // 8 KB of a B tile per K step
constexpr int PLBO_A = (PM / 8) * 128;     // 2048: byte distance of 16-byte K chunks in A
constexpr int PLBO_B = (PN / 8) * 128;     // 4096: ... in B
constexpr int P_EPI_WARPS = 8;
constexpr int P_THREADS = (P_EPI_WARPS + 2) * 32;  // + MMA warp + TMA warp
constexpr int P_DPAD_MAX = 256;            // A resident in shared memory: d + 2 <= 256
constexpr uint32_t P_IDESC = tc::idesc(1u, 2u, 2u, PM, PN);  // f32 <- tf32 x tf32, K-major

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// element (row, k) of a canonical K-major no-swizzle operand block with
// `rows` rows: 16-byte K chunks of 4 tf32 at stride (rows / 8) * 128
__host__ __device__ __forceinline__ int64_t canon_off(int row, int k, int rows) {
  return (int64_t)(k >> 2) * ((rows / 8) * 128) + (row >> 3) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

// ---------------------------------------------------------------- layouts
// B tiles (index build): cell c of tile t, k < d: -2 c_k; k = d, d+1: the
// fp32 norm ||c||^2 split into tf32 hi + lo; k >= d+2: 0.  Padding cells
// (c >= K) carry 1e30 in the hi column (their key never passes a filter).
__global__ void probe_build_b_kernel(const float* __restrict__ coarse, const double* __restrict__ cnorm, int64_t K,
                                     int d, int dpad, int64_t ntiles, float* __restrict__ B) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one per (tile, cell, 4-element chunk)
  const int nch = dpad / 4;
  if (gid >= ntiles * PN * nch) return;
  const int ch = (int)(gid % nch);
  const int n = (int)((gid / nch) % PN);
  const int64_t t = gid / ((int64_t)nch * PN);
  const int64_t c = t * PN + n;
  float v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = ch * 4 + u;
    float x = 0.f;
    if (c < K) {
      if (k < d) {
        x = tf32_rna(-2.f * coarse[c * d + k]);
      } else if (k == d || k == d + 1) {
        const float cn = (float)cnorm[c];
        const float hi = tf32_rna(cn);
        x = k == d ? hi : tf32_rna(cn - hi);
      }
    } else if (k == d) {
      x = 1e30f;
    }
    v[u] = x;
  }
  float* tb = B + t * (int64_t)(dpad * PN);
  *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(tb) + canon_off(n, ch * 4, PN)) =
      make_float4(v[0], v[1], v[2], v[3]);
}

// A blocks (per search): query q of block b, k < d: tf32(fp32(q_k)); k = d,
// d+1: 1; else 0.  Rows beyond nq are zero.
__global__ void probe_build_a_kernel(QVec q, int64_t nq, int d, int dpad, int64_t nblocks, float* __restrict__ A) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one per (block, row, chunk)
  const int nch = dpad / 4;
  if (gid >= nblocks * PM * nch) return;
  const int ch = (int)(gid % nch);
  const int row = (int)((gid / nch) % PM);
  const int64_t b = gid / ((int64_t)nch * PM);
  const int64_t qi = b * PM + row;
  float v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = ch * 4 + u;
    float x = 0.f;
    if (qi < nq) {
      if (k < d) x = tf32_rna((float)q.at(qi * d + k));
      else if (k == d || k == d + 1) x = 1.f;
    }
    v[u] = x;
  }
  float* ab = A + b * (int64_t)(dpad * PM);
  *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(ab) + canon_off(row, ch * 4, PM)) =
      make_float4(v[0], v[1], v[2], v[3]);
}

// eps_q: certified bound of |accumulator - (||c||^2 - 2 q.c)| for every cell
// (Q = ||q||, G = max ||c||):
//   operands rounded to tf32 (q also fp64 -> fp32): each product within
//     (2^-9 + 2^-18) |2 q_t c_t|                     -> (2^-9 + 2^-18) 2 Q G
//   the norm as fp32 (u G^2) split hi + lo (lo in tf32: 2^-21 G^2)
//   fp32 accumulation, <= 2^-22 of the magnitude per add (d + 2 adds;
//     4x the fp32 unit roundoff, generous for the tensor-core adder tree)
//   + the rounding of the fp64 reference distances themselves (1e-9 scale)
__global__ void probe_eps_kernel(QVec q, int64_t nq, int d, float gmax, double* __restrict__ eps) {
  const int64_t qi = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (qi >= nq) return;
  double s = 0.0;
  for (int t = lane; t < d; t += 32) {
    const double x = q.at(qi * d + t);
    s += x * x;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const double Q = sqrt(s) * (1.0 + 1e-12), G = (double)gmax * 1.0001;
    const double e = (1.953125e-3 + 3.814697265625e-06) * 2.0 * Q * G +
                     (5.9604644775390625e-08 + 4.76837158203125e-07) * G * G +
                     (double)(d + 2) * 2.384185791015625e-07 * (2.0 * Q * G + G * G);
    eps[qi] = e * 1.01 + 1e-9 * (Q * Q + G * G) + 1e-30;
  }
}

// ---------------------------------------------------------------- GEMM
struct ProbeGemmArgs {
  const float* A;        // (nblocks, PM x dpad) canonical
  const float* B;        // (ntiles, PN x dpad) canonical
  int64_t nq, K;
  int dpad, nsteps;      // dpad / 8 MMA K steps
  int64_t nblocks;
  int64_t ntiles_pass;   // tiles visited by this pass: t = i * tstride
  int tstride;
  // MIN: per (query, 128-cell group of the visited tiles) minimum key
  float* gmin;           // (nq, 2 * ntiles_pass)
  // FILTER: per-CTA record lists (q_local << 32 | cell), bucketed afterwards
  const float* theta;    // (nq,)
  uint64_t* rec;         // (gridDim, rec_cap)
  int* rec_cnt;          // (gridDim,) records produced (may exceed rec_cap: overflow)
  int64_t rec_cap;
};

template <int MODE>  // 0 MIN, 1 FILTER
__global__ void __launch_bounds__(P_THREADS, 1) probe_gemm_kernel(ProbeGemmArgs a) {
  extern __shared__ __align__(1024) uint8_t psm[];
  __shared__ __align__(8) uint64_t bar_a, bar_adone, bar_full[3], bar_empty[3], bar_accfull[2], bar_accempty[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_rec;
  const int nstages = a.dpad <= 192 ? 3 : 2;
  uint8_t* sA = psm;                                     // PM x dpad fp32
  uint8_t* sB = psm + (size_t)a.dpad * PM * 4;           // nstages x (4 K steps of a B tile)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.nblocks * a.ntiles_pass;
  const int64_t w0 = (int64_t)blockIdx.x * total / gridDim.x;
  const int64_t w1 = (int64_t)(blockIdx.x + 1) * total / gridDim.x;
  const int nch = (a.nsteps + PSTEPS_PER_STAGE - 1) / PSTEPS_PER_STAGE;  // B stages per item

  if (threadIdx.x == 0) {
    tc::mbar_init(&bar_a, 1);
    tc::mbar_init(&bar_adone, 1);
    for (int i = 0; i < 3; ++i) {
      tc::mbar_init(&bar_full[i], 1);
      tc::mbar_init(&bar_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_accfull[i], 1);
      tc::mbar_init(&bar_accempty[i], P_EPI_WARPS);
    }
    s_rec = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = s_tmem;

  if (w0 < w1) {
    if (warp == P_EPI_WARPS + 1) {
      // ---------------- TMA producer: A per query block, B stages per item ----------------
      if (lane == 0) {
        int64_t cur_b = -1;
        int na = 0;
        int64_t gc = 0;  // global B stage counter
        for (int64_t w = w0; w < w1; ++w) {
          const int64_t b = w / a.ntiles_pass;
          const int64_t tile = (w % a.ntiles_pass) * a.tstride;
          if (b != cur_b) {
            // the MMAs of the previous block must be done with A
            if (na > 0) tc::mbar_wait(&bar_adone, (uint32_t)((na - 1) & 1));
            const uint32_t abytes = (uint32_t)a.dpad * PM * 4;
            tc::mbar_expect_tx(&bar_a, abytes);
            tc::bulk_g2s(sA, a.A + b * (int64_t)a.dpad * PM, abytes, &bar_a);
            ++na;
            cur_b = b;
          }
          const uint8_t* bt = reinterpret_cast<const uint8_t*>(a.B) + tile * (int64_t)a.dpad * PN * 4;
          for (int j = 0; j < nch; ++j, ++gc) {
            const int st = (int)(gc % nstages);
            tc::mbar_wait(&bar_empty[st], (uint32_t)(((gc / nstages) & 1) ^ 1));
            const int s0 = j * PSTEPS_PER_STAGE, s1 = min(a.nsteps, s0 + PSTEPS_PER_STAGE);
            const uint32_t bytes = (uint32_t)(s1 - s0) * PB_STEP;
            tc::mbar_expect_tx(&bar_full[st], bytes);
            tc::bulk_g2s(sB + (size_t)st * PSTEPS_PER_STAGE * PB_STEP, bt + (int64_t)s0 * PB_STEP, bytes,
                         &bar_full[st]);
          }
        }
      }
    } else if (warp == P_EPI_WARPS) {
      // ---------------- MMA issuer ----------------
      if (lane == 0) {
        int64_t cur_b = -1;
        int na = 0;
        int64_t gc = 0;
        for (int64_t w = w0; w < w1; ++w) {
          const int64_t it = w - w0;
          const int64_t b = w / a.ntiles_pass;
          if (b != cur_b) {
            if (na > 0) tc::mma_commit(&bar_adone);  // every MMA on the old A (issued before) retires first
            tc::mbar_wait(&bar_a, (uint32_t)(na & 1));
            ++na;
            cur_b = b;
          }
          const int ab = (int)(it & 1);
          tc::mbar_wait(&bar_accempty[ab], (uint32_t)(((it >> 1) & 1) ^ 1));
          tc::fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(ab * PN);
          const uint32_t a_base = tc::smem_u32(sA);
          for (int j = 0; j < nch; ++j, ++gc) {
            const int st = (int)(gc % nstages);
            tc::mbar_wait(&bar_full[st], (uint32_t)((gc / nstages) & 1));
            tc::fence_after();
            const uint32_t b_base = tc::smem_u32(sB + (size_t)st * PSTEPS_PER_STAGE * PB_STEP);
            const int s0 = j * PSTEPS_PER_STAGE, s1 = min(a.nsteps, s0 + PSTEPS_PER_STAGE);
            for (int s = s0; s < s1; ++s) {
              const uint64_t da = tc::make_desc(a_base + (uint32_t)s * (2 * PLBO_A), PLBO_A, 128);
              const uint64_t db = tc::make_desc(b_base + (uint32_t)(s - s0) * PB_STEP, PLBO_B, 128);
              const uint32_t acc = s > 0 ? 1u : 0u;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
                  "l"(da), "l"(db), "r"(P_IDESC), "r"(acc)
                  : "memory");
            }
            tc::mma_commit(&bar_empty[st]);
          }
          tc::mma_commit(&bar_accfull[ab]);
        }
      }
    } else {
      // ---------------- epilogue: lane = query, 128 cells per warp ----------------
      const int quad = warp & 3, half = warp >> 2;
      const int row = quad * 32 + lane;
      int64_t cur_b = -1;
      float th = -__int_as_float(0x7f800000);
      int64_t q = 0;
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        const int64_t b = w / a.ntiles_pass;
        const int64_t ti = w % a.ntiles_pass;
        if (b != cur_b) {
          cur_b = b;
          q = b * PM + row;
          if (MODE == 1) th = q < a.nq ? __ldg(a.theta + q) : -__int_as_float(0x7f800000);
        }
        const int ab = (int)(it & 1);
        tc::mbar_wait(&bar_accfull[ab], (uint32_t)((it >> 1) & 1));
        tc::fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * PN + half * 128);
        const int64_t cell0 = ti * a.tstride * PN + half * 128;
        float mn = __int_as_float(0x7f800000);
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 64) {
          uint32_t v[64];
          TC_TMEM_LD64(tbase + (uint32_t)c0, v);
          tc::tmem_wait_ld();
          float lm = __uint_as_float(v[0]);
#pragma unroll
          for (int i = 1; i < 64; ++i) lm = fminf(lm, __uint_as_float(v[i]));
          if (MODE == 0) {
            mn = fminf(mn, lm);
          } else if (__any_sync(0xffffffffu, lm <= th)) {
            // rare: this warp's hits -> the CTA's record list; one shared
            // atomic per warp reserves the slots (no global round trip on
            // the accumulator's critical path)
            const int64_t cb = cell0 + c0;
            uint64_t mask = 0;
#pragma unroll
            for (int i = 0; i < 64; ++i) mask |= (uint64_t)(__uint_as_float(v[i]) <= th) << i;
            if (cb + 64 > a.K) mask &= cb >= a.K ? 0ull : (~0ull >> (64 - (a.K - cb)));
            const int nh = __popcll(mask);
            int incl = nh;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += t;
            }
            int base = 0;
            if (lane == 31 && incl) base = atomicAdd(&s_rec, incl);
            base = __shfl_sync(0xffffffffu, base, 31) + incl - nh;
            const uint64_t qtag = (uint64_t)q << 32;
            while (mask) {
              const int i = __ffsll((long long)mask) - 1;
              mask &= mask - 1;
              if (base < a.rec_cap) a.rec[(int64_t)blockIdx.x * a.rec_cap + base] = qtag | (uint64_t)(uint32_t)(cb + i);
              ++base;
            }
          }
        }
        if (MODE == 0 && q < a.nq) a.gmin[q * (2 * a.ntiles_pass) + 2 * ti + half] = mn;
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bar_accempty[ab]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (MODE == 1 && threadIdx.x == 0) a.rec_cnt[blockIdx.x] = s_rec;
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// per-CTA records -> per-query candidate rows: shared histogram over the
// batch's queries, one global reservation per (region, query), scatter;
// *ovf set when a region overflowed its capacity (the host re-runs larger)
__global__ void __launch_bounds__(1024) probe_bucket_kernel(const uint64_t* __restrict__ rec,
                                                            const int* __restrict__ rec_cnt, int64_t rec_cap,
                                                            int64_t nq, uint64_t* __restrict__ cand,
                                                            int* __restrict__ cnt, int64_t cap,
                                                            int* __restrict__ ovf) {
  extern __shared__ int bsm[];
  int* hist = bsm;        // [nq]
  int* basev = bsm + nq;  // [nq]
  const int b = blockIdx.x;
  if (threadIdx.x == 0 && rec_cnt[b] > rec_cap) atomicOr(ovf, 1);
  const int n = (int)min((int64_t)rec_cnt[b], rec_cap);
  const uint64_t* r = rec + (int64_t)b * rec_cap;
  for (int64_t i = threadIdx.x; i < nq; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&hist[r[i] >> 32], 1);
  __syncthreads();
  for (int64_t i = threadIdx.x; i < nq; i += blockDim.x) {
    const int h = hist[i];
    basev[i] = h ? atomicAdd(cnt + i, h) : 0;
    hist[i] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t x = r[i];
    const int64_t q = (int64_t)(x >> 32);
    const int pos = basev[q] + atomicAdd(&hist[q], 1);
    if (pos < cap) cand[q * cap + pos] = x & 0xFFFFFFFFull;
  }
}

// theta_q = (ma-th smallest group minimum) + 2 eps_q, rounded up; +inf when
// there are fewer than ma groups
__global__ void __launch_bounds__(256) probe_theta_kernel(const float* __restrict__ gmin, int64_t G, int ma,
                                                          const double* __restrict__ eps, float* __restrict__ theta) {
  __shared__ SelShared sh;
  const int64_t q = blockIdx.x;
  if ((int64_t)ma > G) {
    if (threadIdx.x == 0) theta[q] = __int_as_float(0x7f800000);
    return;
  }
  const float* g = gmin + q * G;
  auto get = [&](int64_t i, uint64_t& v) {
    v = (uint64_t)fkey(g[i]);
    return true;
  };
  block_radix_select(G, get, (unsigned long long)(ma - 1), sh);
  if (threadIdx.x == 0) {
    const double t = (double)fkey_inv((uint32_t)sh.prefix) + 2.0 * eps[q];
    theta[q] = __double2float_ru(t);
  }
}

// ---------------------------------------------------------------- final
constexpr int PF_THREADS = 256;
constexpr int PF_SMEM_CAP = 1024;   // candidates staged in shared memory (more: in place in global scratch)

struct ProbeFinalArgs {
  QVec queries;          // batch-offset applied
  const float* coarse;   // (K, d)
  const uint64_t* cand;  // (nb, cap)
  const int* cnt;
  int64_t cap;
  int64_t K;
  int d, ma;
  int all_exact;         // 1: every query takes the exact streaming path
  int64_t q0;            // global index of batch row 0
  uint64_t* gkeys;       // (nb, cap) scratch for rows beyond PF_SMEM_CAP
  int64_t* gids;
  int64_t* out_cells;    // (nq, ma)
  double* out_dist;
  float* out_sub;        // optional (nq, ma, nsub): ||q_j - c_j||^2 per sub-space of the selected cells
  int nsub;
};

// exact fp64 squared distance, scipy cdist order (sequential over t).  The
// centroid row streams through registers 32 coordinates at a time with the
// next chunk's loads issued before the current chunk's (dependent) fp64 sum,
// so one L2 round trip is exposed per row instead of one per chunk.
__device__ __forceinline__ void load_chunk(const float* g, int t0, int d, float (&ga)[32]) {
  if ((d & 3) == 0 && t0 + 32 <= d) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(g + t0) + u);
      ga[4 * u] = v.x, ga[4 * u + 1] = v.y, ga[4 * u + 2] = v.z, ga[4 * u + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < 32; ++u) ga[u] = t0 + u < d ? __ldg(g + t0 + u) : 0.f;
  }
}
__device__ __forceinline__ double exact_dist(const double* qx, const float* g, int d) {
  double s = 0.0;
  float cur[32], nxt[32];
  load_chunk(g, 0, d, cur);
  for (int t0 = 0; t0 < d; t0 += 32) {
    if (t0 + 32 < d) load_chunk(g, t0 + 32, d, nxt);
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      if (t0 + u < d) {
        const double df = __dsub_rn(qx[t0 + u], (double)cur[u]);
        s = __dadd_rn(s, __dmul_rn(df, df));
      }
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) cur[u] = nxt[u];
  }
  return s;
}

// Per query: every candidate (all keys <= theta, a superset of the exact
// probe set) re-scored exactly, the ma smallest by (distance, cell) selected
// and sorted.  A row that overflowed its capacity (or all_exact) streams all
// K cells instead, recomputing the distance in every radix pass.
__global__ void __launch_bounds__(PF_THREADS) probe_final_kernel(ProbeFinalArgs a, int sortP) {
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ SelShared sh;
  __shared__ int s_cnt;
  uint64_t* ck = (uint64_t*)fsm;                 // PF_SMEM_CAP keys
  int64_t* ci = (int64_t*)(ck + PF_SMEM_CAP);    // PF_SMEM_CAP cells
  uint64_t* ok = (uint64_t*)(ci + PF_SMEM_CAP);  // sortP
  int64_t* oi = (int64_t*)(ok + sortP);
  double* qx = (double*)(oi + sortP);            // d (fp64 query)
  const int64_t ql = blockIdx.x, q = a.q0 + ql;
  const int ma = a.ma;
  for (int t = threadIdx.x; t < a.d; t += blockDim.x) qx[t] = a.queries.at(ql * a.d + t);
  const int64_t raw = a.all_exact ? a.cap + 1 : (int64_t)a.cnt[ql];
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const bool streaming = raw > a.cap;
  const int64_t M = streaming ? a.K : raw;
  uint64_t* KK = ck;
  int64_t* II = ci;
  if (!streaming) {
    if (M > PF_SMEM_CAP) {
      KK = a.gkeys + ql * a.cap;
      II = a.gids + ql * a.cap;
    }
    const uint64_t* cr = a.cand + ql * a.cap;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      const int64_t c = (int64_t)(uint32_t)cr[i];
      II[i] = c;
      KK[i] = dkey(exact_dist(qx, a.coarse + c * a.d, a.d));
    }
    __syncthreads();
  }
  auto key_of = [&](int64_t i, uint64_t& v) {
    v = streaming ? dkey(exact_dist(qx, a.coarse + i * a.d, a.d)) : KK[i];
    return true;
  };
  auto id_of = [&](int64_t i) -> int64_t { return streaming ? i : II[i]; };
  unsigned long long kstar = ~0ull;
  long long istar = 0x7FFFFFFFFFFFFFFFll;
  bool all_ties = true;
  const int64_t r_eff = ma < M ? ma : M;
  if (r_eff < M) {
    block_radix_select(M, key_of, (unsigned long long)(r_eff - 1), sh);
    kstar = sh.prefix;
    const unsigned long long less = sh.less, eq = sh.eq, need = r_eff - less;
    __syncthreads();
    if (eq > need) {
      all_ties = false;
      auto geti = [&](int64_t i, uint64_t& v) {
        uint64_t kv;
        key_of(i, kv);
        v = (uint64_t)id_of(i) ^ 0x8000000000000000ull;
        return kv == kstar;
      };
      block_radix_select(M, geti, need - 1, sh);
      istar = (long long)(sh.prefix ^ 0x8000000000000000ull);
      __syncthreads();
    }
  }
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    uint64_t key;
    key_of(i, key);
    const int64_t id = id_of(i);
    if (key < kstar || (key == kstar && (all_ties || id <= istar))) {
      const int p = atomicAdd(&s_cnt, 1);
      if (p < sortP) {
        ok[p] = key;
        oi[p] = id;
      }
    }
  }
  __syncthreads();
  for (int p = (int)r_eff + threadIdx.x; p < sortP; p += blockDim.x) {
    ok[p] = ~0ull;
    oi[p] = 0x7FFFFFFFFFFFFFFFll;
  }
  __syncthreads();
  bitonic_sort(ok, oi, sortP);
  for (int p = threadIdx.x; p < ma; p += blockDim.x) {
    a.out_cells[q * ma + p] = p < r_eff ? oi[p] : -1;
    if (a.out_dist) a.out_dist[q * ma + p] = p < r_eff ? dkey_inv(ok[p]) : __longlong_as_double(0x7FF0000000000000ll);
  }
  if (a.out_sub) {  // sub-space terms of the selected cells (the packed IVF scan's a_qj), fp64 -> fp32
    const int dsub = a.d / a.nsub;
    const int lps = dsub >> 2;  // lanes per sub-space when a lane takes 4 coordinates
    if ((dsub & 3) == 0 && lps <= 32 && (lps & (lps - 1)) == 0 && (a.d & 3) == 0) {
      // a warp per selected cell: coalesced 16-byte loads of the centroid row,
      // 4 coordinates per lane, the sub-space sums by a shuffle tree
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      constexpr int UN = 4;  // cells in flight per warp
      for (int base = 0; base < a.d; base += 128) {
        const int t = base + lane * 4;
        for (int p0 = warp * UN; p0 < ma; p0 += nw * UN) {
          float4 gv[UN];
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            const int p = p0 + u;
            gv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p < r_eff && t < a.d) gv[u] = __ldg(reinterpret_cast<const float4*>(a.coarse + oi[p] * a.d + t));
          }
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            const int p = p0 + u;
            double s = 0.0;
            if (p < r_eff && t < a.d) {
              const double d0 = qx[t] - (double)gv[u].x, d1 = qx[t + 1] - (double)gv[u].y,
                           d2 = qx[t + 2] - (double)gv[u].z, d3 = qx[t + 3] - (double)gv[u].w;
              s = (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
            }
            for (int o = lps >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (p < ma && (lane & (lps - 1)) == 0 && t < a.d) a.out_sub[(q * ma + p) * a.nsub + t / dsub] = (float)s;
          }
        }
      }
    } else
    for (int idx = threadIdx.x; idx < ma * a.nsub; idx += blockDim.x) {
      const int p = idx / a.nsub, j = idx - p * a.nsub;
      double s = 0.0;
      if (p < r_eff) {
        const float* g = a.coarse + oi[p] * a.d + j * dsub;
        for (int t = 0; t < dsub; ++t) {
          const double df = qx[j * dsub + t] - (double)__ldg(g + t);
          s += df * df;
        }
      }
      a.out_sub[(q * ma + p) * a.nsub + j] = (float)s;
    }
  }
}

}  // namespace

// index build: the canonical B tiles of the probe GEMM (pqs_ivf::probe_b)
int probe_build_index(pqs_ctx* ctx, pqs_ivf* iv) {
  iv->probe_dpad = 0;
  iv->probe_b = nullptr;
  if (iv->d + 2 > P_DPAD_MAX) return PQS_OK;  // exact streaming probes only
  const int dpad = (iv->d + 2 + PKS - 1) / PKS * PKS;
  const int64_t ntiles = cdiv(iv->K, PN);
  const size_t bytes = (size_t)ntiles * PN * dpad * 4;
  PQS_CUDA(ctx, cudaMalloc(&iv->probe_b, bytes));
  const int64_t total = ntiles * PN * (dpad / 4);
  probe_build_b_kernel<<<(unsigned)cdiv(total, 256), 256, 0, ctx->stream>>>(iv->coarse, iv->cnorm, iv->K, iv->d, dpad,
                                                                          ntiles, iv->probe_b);
  PQS_LAUNCHED(ctx);
  iv->probe_dpad = dpad;
  iv->probe_ntiles = ntiles;
  return PQS_OK;
}

int run_ivf_probe(pqs_ctx* ctx, const pqs_ivf* iv, QVec d_queries, int64_t nq, int ma, int64_t* d_cells,
                  double* d_dist, float* d_sub, int nsub) {
  const int64_t K = iv->K;
  const int d = iv->d;
  int P = 1;
  while (P < ma) P <<= 1;
  if (P < 2) P = 2;
  PQS_CHECK(ctx, P <= 4096, "ma too large for the device probe select (<= 4096)");
  static const int64_t cap_env = getenv("PQS_PROBE_CAP") ? atoll(getenv("PQS_PROBE_CAP")) : 0;  // testing
  const int64_t cap = cap_env > 0 ? std::min<int64_t>(cap_env, 4096) : 2048;
  const bool tc_path = iv->probe_b != nullptr && getenv("PQS_PROBE_EXACT") == nullptr;
  const size_t fsmem = (size_t)PF_SMEM_CAP * 16 + (size_t)P * 16 + (size_t)d * 8;
  PQS_CHECK(ctx, fsmem <= 200 * 1024, "probe: d too large for the shared-memory query stage");
  PQS_CUDA(ctx, cudaFuncSetAttribute(probe_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
  // query batches of QB (multiple of PM): candidate rows QB x cap
  // balanced batches of at most 12,288 queries (10,000 queries run as ONE batch: a short tail batch would run the
  // GEMM over all K cells with a few query blocks only)
  const int64_t nbatch = std::max<int64_t>(1, cdiv(nq, 12288));
  const int64_t QB = cdiv(cdiv(nq, nbatch), PM) * PM;
  double* eps = nullptr;
  PQS_TRY(scratch(ctx, S_AERR, (size_t)QB * 2, (float**)&eps));
  uint64_t* cand = nullptr;
  int* cnt = nullptr;
  float* A = nullptr;
  float* gmin = nullptr;
  float* theta = nullptr;
  const int dpad = iv->probe_dpad;
  const int64_t ntiles = iv->probe_ntiles;
  // pass 1 visits every tstride-th tile: >= 2 ma groups of 128 cells
  int tstride = 1;
  static const int ts_env = getenv("PQS_PROBE_TSTRIDE") ? atoi(getenv("PQS_PROBE_TSTRIDE")) : 2;  // tuning
  if (tc_path) {
    const int64_t groups = 2 * ntiles;
    tstride = (int)std::max<int64_t>(1, std::min<int64_t>(ts_env, groups / std::max<int64_t>(1, 2 * (int64_t)ma)));
  }
  const int64_t ntp1 = cdiv(ntiles, tstride);
  uint64_t* gk = nullptr;
  int64_t* gi = nullptr;
  if (tc_path) {
    PQS_TRY(scratch(ctx, S_KEYS, (size_t)(QB * cap), &gk));
    PQS_TRY(scratch(ctx, S_IDS, (size_t)(QB * cap), &gi));
    PQS_TRY(scratch(ctx, S_CAND, (size_t)(QB * cap), &cand));
    PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)QB, &cnt));
    PQS_TRY(scratch(ctx, S_IVF_WORK, (size_t)(QB * dpad), &A));
    PQS_TRY(scratch(ctx, S_IVF_WORK2, (size_t)(QB * 2 * ntp1), &gmin));
    PQS_TRY(scratch(ctx, S_THETA, (size_t)QB * 4, (uint8_t**)&theta));
  }
  const size_t gsmem = (size_t)dpad * PM * 4 + (size_t)(dpad <= 192 ? 3 : 2) * PSTEPS_PER_STAGE * PB_STEP;
  const size_t bsmem = (size_t)QB * 2 * sizeof(int);
  PQS_CUDA(ctx, cudaFuncSetAttribute(probe_bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
  for (int64_t q0 = 0; q0 < nq; q0 += QB) {
    const int64_t nb = std::min(QB, nq - q0);
    const QVec qb = d_queries.offset(q0 * d);
    ProbeFinalArgs f{};
    f.queries = qb;
    f.coarse = iv->coarse;
    f.cap = cap;
    f.K = K;
    f.d = d;
    f.ma = ma;
    f.q0 = q0;
    f.out_cells = d_cells;
    f.out_dist = d_dist;
    f.out_sub = (d_sub && nsub > 0 && d % nsub == 0) ? d_sub : nullptr;
    f.nsub = nsub;
    if (tc_path) {
      const int64_t nblocks = cdiv(nb, PM);
      probe_build_a_kernel<<<(unsigned)cdiv(nblocks * PM * (dpad / 4), 256), 256, 0, ctx->stream>>>(qb, nb, d, dpad,
                                                                                                    nblocks, A);
      PQS_LAUNCHED(ctx);
      probe_eps_kernel<<<(unsigned)cdiv(nb, 8), 256, 0, ctx->stream>>>(qb, nb, d, iv->gmax, eps);
      PQS_LAUNCHED(ctx);
      ProbeGemmArgs g{};
      g.A = A;
      g.B = iv->probe_b;
      g.nq = nb;
      g.K = K;
      g.dpad = dpad;
      g.nsteps = dpad / PKS;
      g.nblocks = nblocks;
      g.gmin = gmin;
      g.theta = theta;
      // pass 1: group minima over the strided tiles
      g.ntiles_pass = ntp1;
      g.tstride = tstride;
      PQS_CUDA(ctx, cudaFuncSetAttribute(probe_gemm_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
      PQS_CUDA(ctx, cudaFuncSetAttribute(probe_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
      probe_gemm_kernel<0><<<(unsigned)std::min<int64_t>(ctx->sm_count, nblocks * ntp1), P_THREADS, gsmem,
                             ctx->stream>>>(g);
      PQS_LAUNCHED(ctx);
      probe_theta_kernel<<<(unsigned)nb, 256, 0, ctx->stream>>>(gmin, 2 * ntp1, ma, eps, theta);
      PQS_LAUNCHED(ctx);
      // pass 2: every tile, keys <= theta -> per-CTA records -> candidate rows
      g.ntiles_pass = ntiles;
      g.tstride = 1;
      const int64_t nct = std::min<int64_t>(ctx->sm_count, nblocks * ntiles);
      int64_t rec_cap = std::max<int64_t>(16384, cdiv(nb * 1024, nct));
      for (int attempt = 0;; ++attempt) {
        uint64_t* rec = nullptr;
        int* rec_cnt = nullptr;
        PQS_TRY(scratch(ctx, S_TC_REC, (size_t)(nct * rec_cap), &rec));
        PQS_TRY(scratch(ctx, S_TC_RECCNT, (size_t)nct + 1, &rec_cnt));
        int* ovf = rec_cnt + nct;
        g.rec = rec;
        g.rec_cnt = rec_cnt;
        g.rec_cap = rec_cap;
        PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nb, ctx->stream));
        PQS_CUDA(ctx, cudaMemsetAsync(ovf, 0, sizeof(int), ctx->stream));
        probe_gemm_kernel<1><<<(unsigned)nct, P_THREADS, gsmem, ctx->stream>>>(g);
        PQS_LAUNCHED(ctx);
        probe_bucket_kernel<<<(unsigned)nct, 1024, bsmem, ctx->stream>>>(rec, rec_cnt, rec_cap, nb, cand, cnt, cap,
                                                                         ovf);
        PQS_LAUNCHED(ctx);
        int h_ovf = 0;
        PQS_TRY(download(ctx, &h_ovf, ovf, sizeof(int)));
        if (!h_ovf) break;
        PQS_CHECK(ctx, attempt < 6, "probe: candidate records overflow");
        rec_cap *= 4;
      }
      f.cand = cand;
      f.cnt = cnt;
      f.gkeys = gk;
      f.gids = gi;
      f.all_exact = 0;
    } else {
      f.all_exact = 1;
    }
    probe_final_kernel<<<(unsigned)nb, PF_THREADS, fsmem, ctx->stream>>>(f, P);
    PQS_LAUNCHED(ctx);
    static const bool dbg = getenv("PQS_PROBE_DEBUG") != nullptr;
    if (dbg && tc_path) {
      std::vector<int> hc((size_t)nb);
      std::vector<float> ht((size_t)nb), hg((size_t)(2 * ntp1) * 4);
      std::vector<double> he((size_t)nb);
      PQS_TRY(download(ctx, hc.data(), cnt, sizeof(int) * nb));
      PQS_TRY(download(ctx, ht.data(), theta, sizeof(float) * nb));
      PQS_TRY(download(ctx, he.data(), eps, sizeof(double) * nb));
      PQS_TRY(download(ctx, hg.data(), gmin, sizeof(float) * 2 * ntp1 * 4));
      int64_t tot = 0, mx = 0, over = 0;
      for (int64_t i = 0; i < nb; ++i) {
        tot += hc[i];
        mx = std::max<int64_t>(mx, hc[i]);
        over += hc[i] > cap;
      }
      fprintf(stderr, "probe batch q0=%lld nb=%lld tstride=%d groups=%lld: candidates mean %.1f max %lld overflow %lld\n",
              (long long)q0, (long long)nb, tstride, (long long)(2 * ntp1), (double)tot / nb, (long long)mx,
              (long long)over);
      for (int i = 0; i < 4 && i < nb; ++i) {
        float mn = 1e38f;
        for (int64_t g2 = 0; g2 < 2 * ntp1; ++g2) mn = std::min(mn, hg[(size_t)i * 2 * ntp1 + g2]);
        fprintf(stderr, "  q%d: cnt %d theta %.6g eps %.6g min group %.6g\n", i, hc[i], ht[i], he[i], mn);
      }
    }
  }
  return PQS_OK;
}
