// scan8.cu -- float ADC over 8-bit codes (K3 scan, K6 rerank via select.cu).
//
// Reference: scan_distances / scan (scan.py:68-81, 197-203).
//
// K3 design: lane = query.  A CTA owns a group of 32
// queries and W warps; all warps share the group's tables, staged in shared
// memory in [component][entry][lane] order so that 32 lanes reading the same
// entry of their own table hit distinct banks (conflict-free for any code).
// The scan tables are u16 fixed-point LOWER BOUNDS of the exact fp32 tables:
//   t'[j][c] = min(65535, floor((T[j][c] - o_j) * 2^e))   (o_j = min_c T[j][c])
// so every code's integer sum L satisfies  L <= 2^e (d - O) <= L + m  (d the
// exact distance, O = sum_j o_j) -- exact integer bounds, no fp error
// analysis.  Two u16 tables (32 queries x 8 x 256) fit in 128 KB, so for the
// cfg0 shape the tables stay resident; larger tables stream in component
// chunks (TMA bulk copies, cp.async.bulk + mbarrier, double-buffered) while
// each lane keeps 64 u32 partial sums in registers.  Codes are broadcast:
// the device layout is tile-transposed ([tile][component][1024 codes]), one
// LDS.128 returns 16 codes' bytes of a component.  A sample pass (scale e0,
// no saturation) gives an upper bound D' on the r-th smallest d - O; the
// filter pass (finer scale e1) keeps every code with L <= floor(2^e1 D'),
// which provably contains the reference's top-r; survivors are re-scored
// exactly in fp64 (reference order) and selected by (distance, id).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "pqs_common.cuh"
#include "select_dev.cuh"

namespace {

constexpr int W8 = 16;              // warps per CTA
constexpr int C8 = TILE8 / W8;     // codes per warp (64)
constexpr int SCAN8_THREADS = W8 * 32;
constexpr int CHUNK_BUDGET = 176 * 1024;

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// --------------------------------------------------------- u16 tables
// per query: o_j = min_c T[j][c] (fp32), e0 = floor(log2(65535 / max_j max_c (T - o_j)))
__global__ void tables_u16_stats_kernel(const float* __restrict__ tables, int64_t nq, int m, int k,
                                        float* __restrict__ off, int* __restrict__ e0, double* __restrict__ slack) {
  const int64_t q = blockIdx.x;
  __shared__ double s_max[32], s_abs[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double mx = 0.0, absum = 0.0;
  for (int j = warp; j < m; j += nw) {
    const float* row = tables + (q * m + j) * (int64_t)k;
    float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000), am = 0.f;
    for (int c = lane; c < k; c += 32) {
      const float v = row[c];
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
      am = fmaxf(am, fabsf(v));
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
    }
    if (lane == 0) off[q * m + j] = lo;
    mx = fmax(mx, (double)hi - (double)lo);
    absum += (double)am;
  }
  if (lane == 0) {
    s_max[warp] = mx;
    s_abs[warp] = absum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double M = 0.0, A = 0.0;
    for (int i = 0; i < nw; ++i) {
      M = fmax(M, s_max[i]);
      A += s_abs[i];
    }
    int e = 0;
    if (M > 0.0) e = (int)floor(log2(65535.0 / M));
    while (M > 0.0 && ldexp(M, e) > 65535.0) --e;
    e0[q] = e;
    // covers the reference's fp64 rounding of d and of the offset sum
    slack[q] = A * 4.0 * (double)(m + 2) * 1.1102230246251565e-16;
  }
}

// t'[qg][j][c][lane] = min(65535, floor((T - o_j) * 2^e_q)); exact in fp64.
// One CTA per (query group, component): the 32 queries' rows of k entries are
// read coalesced and transposed through shared memory, so the [c][lane]
// output is written coalesced too
constexpr int TU16_THREADS = 256;
__global__ void __launch_bounds__(TU16_THREADS) tables_u16_t_kernel(const float* __restrict__ tables,
                                                                   const float* __restrict__ off,
                                                                   const int* __restrict__ ex, int64_t nq, int m,
                                                                   int k, uint16_t* __restrict__ tt) {
  __shared__ float st[32][257];  // k <= 256
  __shared__ double so[32];
  __shared__ int se[32];
  const int64_t qg = blockIdx.x / m;
  const int j = (int)(blockIdx.x - qg * m);
  if (threadIdx.x < 32) {
    const int64_t q = qg * 32 + threadIdx.x;
    so[threadIdx.x] = q < nq ? (double)off[q * m + j] : 0.0;
    se[threadIdx.x] = q < nq ? ex[q] : 0;
  }
  for (int i = threadIdx.x; i < 32 * k; i += TU16_THREADS) {
    const int l = i / k, c = i - l * k;
    const int64_t q = qg * 32 + l;
    st[l][c] = q < nq ? tables[(q * m + j) * (int64_t)k + c] : 0.f;
  }
  __syncthreads();
  uint16_t* dst = tt + (qg * m + j) * (int64_t)k * 32;
  for (int i = threadIdx.x; i < 32 * k; i += TU16_THREADS) {
    const int l = i & 31, c = i >> 5;
    uint16_t v = 0;
    if (qg * 32 + l < nq) {
      const double d = (double)st[l][c] - so[l];
      const double f = floor(ldexp(d, se[l]));
      v = f >= 65535.0 ? (uint16_t)65535 : (uint16_t)f;
    }
    dst[i] = v;
  }
}

// --------------------------------------------------------------- K3 kernel
enum { MODE8_DENSE = 0, MODE8_FILTER = 1 };
constexpr int CSTAGE8 = 16;

struct Scan8Args {
  const uint16_t* tt;      // [nqg][m][k][32]
  const uint8_t* codes;    // [ntiles][m][TILE8]
  int64_t n;
  int m, k, mc, resident;
  int64_t nq;
  int64_t nvt, tile_off, tile_step, per_cta;
  int64_t nqg;             // query groups of 32
  uint32_t* out;           // dense [q][ld] u32 lower-bound sums (0xFFFFFFFF = no code)
  int64_t ld;
  const uint32_t* theta;   // filter: keep L <= theta[q]
  uint64_t* cand;
  int* cand_cnt;
  int64_t cap;
  uint32_t one;
  uint32_t c64;            // runtime 64 (entry row stride), keeps the IMAD on the FMA pipe
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

__device__ __forceinline__ uint32_t imad8(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int MODE, bool RES>
__global__ void __launch_bounds__(SCAN8_THREADS, 1) scan8_kernel(Scan8Args a) {
  extern __shared__ __align__(128) unsigned char sm8[];
  __shared__ __align__(8) uint64_t bars[3];  // 0/1: stage buffers, 2: resident tables
  const int m = a.m, k = a.k, mc = a.mc;
  const uint32_t row_bytes = (uint32_t)k * 32 * 2;  // one component of 32 queries' tables
  const uint32_t tab_bytes = RES ? (uint32_t)m * row_bytes : (uint32_t)mc * row_bytes;
  const uint32_t tab_region = RES ? tab_bytes : 2 * tab_bytes;
  const uint32_t code_bytes = (uint32_t)mc * TILE8;
  uint8_t* code_base = sm8 + tab_region;
  uint32_t* stage = reinterpret_cast<uint32_t*>(code_base + 2 * code_bytes) + threadIdx.x;
  int ncand = 0;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t one = a.one;
  const uint32_t c64 = a.c64;

  // persistent CTA over a balanced range of the linearised (query group, tile) list
  const int64_t total = a.nqg * a.nvt;
  const int64_t w0 = (int64_t)blockIdx.x * total / gridDim.x;
  const int64_t w1 = (int64_t)(blockIdx.x + 1) * total / gridDim.x;
  if (w0 >= w1) return;
  const int nch = RES ? 1 : (m + mc - 1) / mc;
  const int64_t S = (w1 - w0) * nch;  // stages

  auto issue_at = [&](int b, int64_t w, int ch) {
    const int64_t qg = w / a.nvt;
    const int64_t tile = a.tile_off + (w - qg * a.nvt) * a.tile_step;
    const int j0 = ch * mc;
    const int mcur = min(mc, m - j0);
    const uint32_t cb = (uint32_t)mcur * TILE8;
    const uint32_t tb = RES ? 0u : (uint32_t)mcur * row_bytes;
    mbar_expect_tx(&bars[b], tb + cb);
    if (!RES) bulk_g2s(sm8 + b * tab_bytes, a.tt + (qg * m + j0) * (int64_t)k * 32, tb, &bars[b]);
    bulk_g2s(code_base + b * code_bytes, a.codes + (tile * m + j0) * (int64_t)TILE8, cb, &bars[b]);
  };
  auto next_of = [&](int64_t w, int ch, int steps, int64_t& w2, int& ch2) {
    ch2 = ch + steps;
    w2 = w;
    while (ch2 >= nch) {
      ch2 -= nch;
      ++w2;
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    issue_at(0, w0, 0);
    if (S > 1) {
      int64_t w2;
      int ch2;
      next_of(w0, 0, 1, w2, ch2);
      issue_at(1, w2, ch2);
    }
  }

  int64_t q = -1, cur_qg = -1;
  bool qvalid = false;
  uint32_t theta = 0;
  uint32_t tphase = 0;

  auto flush = [&]() {
    if (MODE == MODE8_FILTER && ncand > 0) {
      const int pos = atomicAdd(a.cand_cnt + q, ncand);
      for (int i = 0; i < ncand; ++i)
        if (pos + i < a.cap) a.cand[q * a.cap + pos + i] = (uint64_t)stage[i * SCAN8_THREADS];
      ncand = 0;
    }
  };
  // epilogue for the NV consecutive codes of this warp starting at code c0 / column col
  auto emit = [&](const auto& vals, int64_t c0, int64_t col) {
    constexpr int nv = (int)(sizeof(vals) / sizeof(vals[0]));
    if (!qvalid) return;
    if (MODE == MODE8_FILTER) {
      unsigned long long hit = 0;
#pragma unroll
      for (int c = 0; c < nv; ++c) hit |= (unsigned long long)(vals[c] <= theta) << c;
      if (hit) {  // rare: one divergent branch per nv codes
        const int64_t valid = a.n - c0;
        if (valid < nv) hit &= valid <= 0 ? 0ull : ((1ull << valid) - 1ull);
        while (hit) {
          const int c = __ffsll((long long)hit) - 1;
          hit &= hit - 1;
          stage[ncand * SCAN8_THREADS] = (uint32_t)(c0 + c);
          if (++ncand == CSTAGE8) flush();
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < nv; c += 4) {
        uint4 o;
        o.x = (c0 + c + 0 < a.n) ? vals[c + 0] : 0xFFFFFFFFu;
        o.y = (c0 + c + 1 < a.n) ? vals[c + 1] : 0xFFFFFFFFu;
        o.z = (c0 + c + 2 < a.n) ? vals[c + 2] : 0xFFFFFFFFu;
        o.w = (c0 + c + 3 < a.n) ? vals[c + 3] : 0xFFFFFFFFu;
        *reinterpret_cast<uint4*>(a.out + q * a.ld + col + c) = o;
      }
    }
  };
  // 2 x 16 lookups (components jj, jj+1 of 16 codes), one IADD3 per code
  auto lookup16x2 = [&](uint32_t tj0, const uint4& w0v, uint32_t tj1, const uint4& w1v, uint32_t* acc) {
    const uint32_t a0[4] = {w0v.x, w0v.y, w0v.z, w0v.w};
    const uint32_t a1[4] = {w1v.x, w1v.y, w1v.z, w1v.w};
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const uint32_t c0 = prmt(a0[e >> 2], 0u, 0x4440u | (uint32_t)(e & 3));
      const uint32_t c1 = prmt(a1[e >> 2], 0u, 0x4440u | (uint32_t)(e & 3));
      uint32_t t0, t1;
      asm volatile("ld.shared.u16 %0, [%1];" : "=r"(t0) : "r"(imad8(c0, c64, tj0)));
      asm volatile("ld.shared.u16 %0, [%1];" : "=r"(t1) : "r"(imad8(c1, c64, tj1)));
      acc[e] = acc[e] + t0 + t1;
    }
  };
  auto lookup16 = [&](uint32_t tj, const uint4& w, uint32_t* acc) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const uint32_t code = prmt(ws[e >> 2], 0u, 0x4440u | (uint32_t)(e & 3));
      uint32_t t;
      asm volatile("ld.shared.u16 %0, [%1];" : "=r"(t) : "r"(imad8(code, c64, tj)));
      acc[e] = imad8(t, one, acc[e]);
    }
  };
  auto switch_group = [&](int64_t qg) {
    flush();
    q = qg * 32 + lane;
    qvalid = q < a.nq;
    theta = (MODE == MODE8_FILTER && qvalid) ? a.theta[q] : 0u;
    cur_qg = qg;
  };

  if constexpr (RES) {
    int64_t s = 0;
    for (int64_t w = w0; w < w1; ++w, ++s) {
      const int64_t qg = w / a.nvt;
      const int64_t vi = w - qg * a.nvt;
      const int64_t tile = a.tile_off + vi * a.tile_step;
      if (qg != cur_qg) {
        switch_group(qg);
        __syncthreads();  // every warp is done with the previous group's tables
        if (threadIdx.x == 0) {
          mbar_expect_tx(&bars[2], tab_bytes);
          bulk_g2s(sm8, a.tt + qg * (int64_t)m * k * 32, tab_bytes, &bars[2]);
        }
        mbar_wait(&bars[2], tphase);
        tphase ^= 1;
      }
      const int b = (int)(s & 1);
      mbar_wait(&bars[b], (uint32_t)((s >> 1) & 1));
      const uint32_t tbase = smem_u32(sm8) + 2u * lane;
      const uint8_t* cb = code_base + b * code_bytes + warp * C8;
      // component pairs outermost over all C8 codes of the warp (64 sums in
      // fixed registers); the epilogue runs once per tile after the barrier
      uint32_t acc[C8];
#pragma unroll
      for (int e = 0; e < C8; ++e) acc[e] = 0u;
      int jj = 0;
      for (; jj + 1 < m; jj += 2) {
#pragma unroll
        for (int v = 0; v < C8 / 16; ++v) {
          const uint8_t* cv = cb + v * 16;
          lookup16x2(tbase + (uint32_t)jj * row_bytes, *reinterpret_cast<const uint4*>(cv + jj * TILE8),
                     tbase + (uint32_t)(jj + 1) * row_bytes, *reinterpret_cast<const uint4*>(cv + (jj + 1) * TILE8),
                     acc + v * 16);
        }
      }
      if (jj < m) {
#pragma unroll
        for (int v = 0; v < C8 / 16; ++v)
          lookup16(tbase + (uint32_t)jj * row_bytes, *reinterpret_cast<const uint4*>(cb + v * 16 + jj * TILE8),
                   acc + v * 16);
      }
      __syncthreads();
      if (threadIdx.x == 0 && s + 2 < S) issue_at(b, w + 2, 0);
      emit(acc, tile * TILE8 + warp * C8, vi * TILE8 + warp * C8);
    }
  } else {
    uint32_t part[C8];
#pragma unroll
    for (int c = 0; c < C8; ++c) part[c] = 0u;
    int64_t s = 0;
    for (int64_t w = w0; w < w1; ++w) {
      const int64_t qg = w / a.nvt;
      const int64_t vi = w - qg * a.nvt;
      const int64_t tile = a.tile_off + vi * a.tile_step;
      if (qg != cur_qg) switch_group(qg);
      for (int ch = 0; ch < nch; ++ch, ++s) {
        const int b = (int)(s & 1);
        mbar_wait(&bars[b], (uint32_t)((s >> 1) & 1));
        const int mcur = min(mc, m - ch * mc);
        const uint32_t tbase = smem_u32(sm8 + b * tab_bytes) + 2u * lane;
        const uint8_t* cb = code_base + b * code_bytes + warp * C8;
        // component pairs outermost: all C8 partial sums stay in fixed registers
        int jj = 0;
        for (; jj + 1 < mcur; jj += 2) {
#pragma unroll
          for (int v = 0; v < C8 / 16; ++v) {
            const uint8_t* cv = cb + v * 16;
            lookup16x2(tbase + (uint32_t)jj * row_bytes, *reinterpret_cast<const uint4*>(cv + jj * TILE8),
                       tbase + (uint32_t)(jj + 1) * row_bytes,
                       *reinterpret_cast<const uint4*>(cv + (jj + 1) * TILE8), part + v * 16);
          }
        }
        if (jj < mcur) {
#pragma unroll
          for (int v = 0; v < C8 / 16; ++v)
            lookup16(tbase + (uint32_t)jj * row_bytes, *reinterpret_cast<const uint4*>(cb + v * 16 + jj * TILE8),
                     part + v * 16);
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < S) {
          int64_t w2;
          int ch2;
          next_of(w, ch, 2, w2, ch2);
          issue_at(b, w2, ch2);
        }
      }
      // the epilogue reads registers and the stage area only, so it runs after
      // the chunk loop: the lookup loop carries no epilogue register pressure
      emit(part, tile * TILE8 + warp * C8, vi * TILE8 + warp * C8);
#pragma unroll
      for (int c = 0; c < C8; ++c) part[c] = 0u;
    }
  }
  flush();
}


// ===================================================================== packed
// K3p -- the filter pass with two queries per table word.
//
// The u16 lane=query kernel above issues ~4.5 instructions per lookup and its
// LDS.U16 uses half of the 128-byte shared-memory wavefront.  Here one 32-bit
// word holds the (15-bit) lower-bound entries of two queries, so one LDS.32
// is 64 lookups and the partial sums of both queries advance with ONE integer
// add.  Layout of a 32-query group's tables, per component quad Q = j / 4:
//   word[(Q*k + c) * 64 + (j % 4) * 16 + h] = t'(query h)[j][c] | t'(query h+16)[j][c] << 16
// i.e. one 256-byte row per entry c.  A quad's 256 rows are exactly 64 KB and
// are staged at a 64 KB-aligned shared-memory window address, so the address
// of a lookup is  slot | code << 8 | (j%4)*64 + h*4  -- formed by ONE PRMT
// that drops the code byte into byte 1 of the lane's base register (no IMAD,
// no shift).  Half-warp P = lane / 16 takes component parity P: lanes 0-15
// read sub-slot 2i (banks 0-15 or 16-31 alternating with i), lanes 16-31
// sub-slot 2i+1 (the other 16 banks) -> every LDS.32 is one conflict-free
// 128-byte wavefront.  To let one SHFL finish two codes, the upper half-warp
// walks each code pair in swapped order (acc[e] <-> code e^1): after
//   tot = acc[e] + shfl_xor(acc[e+1], 16)
// lanes 0-15 hold the total of code e and lanes 16-31 that of code e+1.
// Entries are clipped to floor(32767 / m) (a clipped entry is still a lower
// bound) so a half never carries into its neighbour and bit 15 of each half
// stays free: (theta | 0x8000) - tot keeps bit 15 set iff tot <= theta, one
// subtraction tests both queries.  Per 2 lookups: PRMT + LDS.32 + IADD.
constexpr int CST8P = 8;          // staged candidates per thread and query half
constexpr int P16_MAX_M = 64;     // clip = floor(32767 / m) >= 511
constexpr uint32_t P16_TMAX = 32767u;
constexpr double P16_TARGET = 8191.0;
constexpr int P16_RUN = 4;        // streamed tables: tiles per run of one query group

// one CTA per (query group, padded component): rows read coalesced, transposed
// through shared memory, written as 64-byte runs of the packed layout
__global__ void __launch_bounds__(TU16_THREADS) tables_p16_kernel(const float* __restrict__ tables,
                                                                 const float* __restrict__ off,
                                                                 const int* __restrict__ ex, int64_t nq, int m, int k,
                                                                 uint32_t clip, uint32_t* __restrict__ tp) {
  __shared__ float st[32][257];
  __shared__ double so[32];
  __shared__ int se[32];
  const int mq = ((m + 3) >> 2) << 2;
  const int64_t qg = blockIdx.x / mq;
  const int j = (int)(blockIdx.x - qg * mq);
  uint32_t* dst = tp + ((qg * (mq >> 2) + (j >> 2)) * (int64_t)k) * 64 + (j & 3) * 16;
  if (j >= m) {  // padding component of the last quad: zero rows
    for (int i = threadIdx.x; i < 16 * k; i += TU16_THREADS) dst[(int64_t)(i >> 4) * 64 + (i & 15)] = 0u;
    return;
  }
  if (threadIdx.x < 32) {
    const int64_t q = qg * 32 + threadIdx.x;
    so[threadIdx.x] = q < nq ? (double)off[q * m + j] : 0.0;
    se[threadIdx.x] = q < nq ? ex[q] : 0;
  }
  for (int i = threadIdx.x; i < 32 * k; i += TU16_THREADS) {
    const int l = i / k, c = i - l * k;
    const int64_t q = qg * 32 + l;
    st[l][c] = q < nq ? tables[(q * m + j) * (int64_t)k + c] : 0.f;
  }
  __syncthreads();
  auto val = [&](int l, int c) -> uint32_t {
    if (qg * 32 + l >= nq) return 0u;
    const double f = floor(ldexp((double)st[l][c] - so[l], se[l]));
    return f >= (double)clip ? clip : (f <= 0.0 ? 0u : (uint32_t)f);
  };
  for (int i = threadIdx.x; i < 16 * k; i += TU16_THREADS) {
    const int h = i & 15, c = i >> 4;
    dst[(int64_t)c * 64 + h] = val(h, c) | (val(h + 16, c) << 16);
  }
}

struct Scan8PArgs {
  const uint32_t* tp;    // [nqg][nQ][k][64]
  const uint8_t* codes;  // [ntiles][m][TILE8]
  int64_t n;
  int m, k;
  int64_t nq, nvt, nqg;
  int64_t tile0;          // first tile of this launch (nvt tiles from there)
  const uint32_t* theta;  // keep L <= theta[q] (<= P16_TMAX)
  uint64_t* cand;
  int* cand_cnt;
  int64_t cap;
};

template <int OFF>
__device__ __forceinline__ uint32_t lds32_off(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
  return v;
}

template <bool RES>
__global__ void __launch_bounds__(SCAN8_THREADS, 1) scan8p_kernel(Scan8PArgs a) {
  extern __shared__ __align__(128) unsigned char smp[];
  const int m = a.m, k = a.k;
  const int nQ = (m + 3) >> 2;
  const uint32_t sb = smem_u32(smp);
  const uint32_t slot0 = (sb + 65535u) & ~65535u;  // two 64 KB table slots at slot0, slot0 + 64 KB
  unsigned char* slot_ptr = smp + (slot0 - sb);
  // low region [sb, slot0): barriers, code buffers, candidate stage
  // stage buffers: NB code buffers (+ the two table slots when the tables
  // stream).  full[b]: the bulk copies of a stage landed; empty[b]: all W8
  // warps are done with it (no block-wide barrier per stage: a warp delayed by
  // its candidate path does not hold the others back)
  constexpr int NB = RES ? 3 : 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smp);
  uint64_t* empty = full + NB;
  uint64_t* tabbar = empty + NB;  // resident tables
  const int crows = RES ? nQ * 4 : 4;
  const uint32_t code_bytes = (uint32_t)crows * TILE8;
  uint8_t* code_base = smp + 128;
  uint32_t* stage = reinterpret_cast<uint32_t*>(code_base + NB * code_bytes) + threadIdx.x;
  if (128u + NB * code_bytes + 2u * CST8P * SCAN8_THREADS * 4u > slot0 - sb) __trap();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane & 15, P = lane >> 4;
  const uint32_t lb = slot0 + (uint32_t)h * 4u + (uint32_t)P * 64u;
  uint32_t sel[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) sel[b] = 0x7604u | ((uint32_t)(b ^ P) << 4);

  // items = (query group, tile) pairs.  Resident tables: a balanced contiguous
  // range of the group-major list (tables reloaded at a group change only).
  // Streamed tables (every item streams its quads anyway): runs of P16_RUN
  // consecutive tiles of one group, runs in tile-major order, CTA i takes runs
  // i, i + grid, ... -- at any time the CTAs share a few tile blocks, so each
  // code tile comes from DRAM once and the (small) tables cycle through L2.
  // Runs of the last tile block are padded with empty items (tile >= nvt).
  const int64_t total = a.nqg * a.nvt;
  const int nch = RES ? 1 : nQ;
  const int nvt = (int)a.nvt, nqg = (int)a.nqg;
  int nw, g0 = 0, t0 = 0;
  if (RES) {
    const int64_t w0 = (int64_t)blockIdx.x * total / gridDim.x;
    const int64_t w1 = (int64_t)(blockIdx.x + 1) * total / gridDim.x;
    nw = (int)(w1 - w0);
    g0 = (int)(w0 / a.nvt);
    t0 = (int)(w0 - (int64_t)g0 * a.nvt);
  } else {
    const int64_t nruns = (int64_t)((nvt + P16_RUN - 1) / P16_RUN) * nqg;
    nw = (int)((nruns - blockIdx.x + gridDim.x - 1) / gridDim.x) * P16_RUN;
  }
  if (nw <= 0) return;
  const int S = nw * nch;
  auto item = [&](int wi, int& qg, int& tile) {  // wi: index into this CTA's items
    if (RES) {
      const int lin = t0 + wi;
      qg = g0 + lin / nvt;
      tile = lin % nvt;
    } else {
      const int64_t rw = (int64_t)blockIdx.x + (int64_t)(wi / P16_RUN) * gridDim.x;
      const int tb = (int)(rw / nqg);
      qg = (int)(rw - (int64_t)tb * nqg);
      tile = tb * P16_RUN + wi % P16_RUN;
    }
  };
  const uint32_t quad_bytes = (uint32_t)k * 256u;

  auto issue_at = [&](int b, int wi, int ch) {
    int qgi, tli;
    item(wi, qgi, tli);
    const int64_t qg = qgi, tile = tli + a.tile0;
    if (!RES && tli >= nvt) {  // padding item: complete the phase with no bytes
      mbar_expect_tx(&full[b], 0u);
      return;
    }
    if (RES) {
      mbar_expect_tx(&full[b], (uint32_t)m * TILE8);
      bulk_g2s(code_base + b * code_bytes, a.codes + tile * m * (int64_t)TILE8, (uint32_t)m * TILE8, &full[b]);
    } else {
      const int mcur = min(4, m - 4 * ch);
      mbar_expect_tx(&full[b], quad_bytes + (uint32_t)mcur * TILE8);
      bulk_g2s(slot_ptr + b * 65536, a.tp + (qg * nQ + ch) * (int64_t)k * 64, quad_bytes, &full[b]);
      bulk_g2s(code_base + b * code_bytes, a.codes + (tile * m + 4 * ch) * (int64_t)TILE8, (uint32_t)mcur * TILE8,
               &full[b]);
    }
  };
  auto issue_stage = [&](int st) { issue_at(st % NB, st / nch, st % nch); };
  // code rows of padding components must hold valid codes (their table rows
  // are zero): clear both buffers once, before any bulk copy lands in them
  for (uint32_t i = threadIdx.x; i < NB * code_bytes / 16; i += SCAN8_THREADS)
    reinterpret_cast<uint4*>(code_base)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], W8);
    }
    mbar_init(tabbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0)
    for (int st = 0; st < NB - 1 && st < S; ++st) issue_stage(st);

  int q0 = -1, cur_qg = -1;  // nq < 2^31
  uint32_t thg = 0, vmask = 0, tphase = 0;
  uint32_t ncp = 0;  // staged candidates: query half 0 in byte 0, half 1 in byte 1
  // append the staged candidates of query half hf to its global list
  auto flush = [&](int hf) {
    const int nc = (int)((ncp >> (8 * hf)) & 0xffu);
    if (nc > 0) {
      const int64_t q = q0 + 16 * hf;
      const int pos = atomicAdd(a.cand_cnt + q, nc);
      const uint32_t* st = stage + hf * CST8P * SCAN8_THREADS;
      for (int i = 0; i < nc; ++i)
        if (pos + i < a.cap) a.cand[q * a.cap + pos + i] = (uint64_t)st[i * SCAN8_THREADS];
      ncp &= ~(0xffu << (8 * hf));
    }
  };
  auto switch_group = [&](int qg) {
    flush(0);
    flush(1);
    q0 = qg * 32 + h;
    const bool v0 = q0 < a.nq, v1 = q0 + 16 < a.nq;
    const uint32_t t0 = v0 ? min(a.theta[q0], P16_TMAX) : 0u, t1 = v1 ? min(a.theta[q0 + 16], P16_TMAX) : 0u;
    thg = t0 | (t1 << 16) | 0x80008000u;
    vmask = (v0 ? 0x8000u : 0u) | (v1 ? 0x80000000u : 0u);
    cur_qg = qg;
  };
  // one component pair (sub-slots 2*IP and 2*IP+1 of the quad at B) of the warp's 64 codes
  auto pair_pass = [&](auto ip_tag, uint32_t B, const uint8_t* crow, uint32_t* acc) {
    constexpr int IP = decltype(ip_tag)::value;
#pragma unroll
    for (int v = 0; v < C8 / 16; ++v) {
      const uint4 cw = *reinterpret_cast<const uint4*>(crow + v * 16);
      const uint32_t ws[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[v * 16 + e] += lds32_off<IP * 128>(prmt(ws[e >> 2], B, sel[e & 3]));
    }
  };
  // totals of the warp's code pairs and the filter test: the hit bits of a
  // group of 8 totals shift into one mask word (half 0 in bits 8..15, half 1
  // in bits 24..31); the rare hits are walked in a compact loop (the kernel
  // must stay small: a fully unrolled slow path thrashes the instruction cache)
  auto emit = [&](uint32_t* acc, int64_t c0) {
    uint32_t M[C8 / 16];
#pragma unroll
    for (int g = 0; g < C8 / 16; ++g) M[g] = 0u;
#pragma unroll
    for (int e = 0; e < C8; e += 2) {
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e + 1], 16);
      M[e >> 4] = (M[e >> 4] >> 1) | ((thg - acc[e]) & vmask);
    }
#pragma unroll
    for (int g = 0; g < C8 / 16; ++g) {
      uint32_t mm = M[g];
      while (mm) {
        const int p = __ffs((int)mm) - 1;
        mm &= mm - 1;
        const int hf = p >> 4;
        const int64_t code = c0 + g * 16 + 2 * ((p & 15) - 8) + P;
        if (code < a.n) {
          const uint32_t nc = (ncp >> (8 * hf)) & 0xffu;
          stage[(hf * CST8P + nc) * SCAN8_THREADS] = (uint32_t)code;
          ncp += 1u << (8 * hf);
          if (nc + 1 == CST8P) flush(hf);
        }
      }
    }
  };

  uint32_t acc[C8];
#pragma unroll
  for (int e = 0; e < C8; ++e) acc[e] = 0u;
  int s = 0;
  for (int w = 0; w < nw; ++w) {
    int qg, tile;
    item(w, qg, tile);
    if (qg != cur_qg) {
      switch_group(qg);
      if (RES) {
        __syncthreads();  // every warp is done with the previous group's tables
        if (threadIdx.x == 0) {
          mbar_expect_tx(tabbar, (uint32_t)nQ * quad_bytes);
          for (int Q = 0; Q < nQ; ++Q)
            bulk_g2s(slot_ptr + Q * 65536, a.tp + ((int64_t)qg * nQ + Q) * (int64_t)k * 64, quad_bytes, tabbar);
        }
        mbar_wait(tabbar, tphase);
        tphase ^= 1;
      }
    }
    for (int ch = 0; ch < nch; ++ch, ++s) {
      const int b = s % NB;
      // warp 0 keeps NB - 1 stages in flight: stage s + NB - 1 reuses the
      // buffer of stage s - 1, once every warp has released it
      if (warp == 0 && s + NB - 1 < S) {
        if (lane == 0) {
          if (s >= 1) mbar_wait(&empty[(s - 1) % NB], (uint32_t)(((s - 1) / NB) & 1));
          issue_stage(s + NB - 1);
        }
        __syncwarp();
      }
      mbar_wait(&full[b], (uint32_t)((s / NB) & 1));
      const uint8_t* cb = code_base + b * code_bytes + warp * C8 + P * TILE8;
      if (!RES && tile >= nvt) {
        // padding item: nothing to scan
      } else if (RES) {
        for (int Q = 0; Q < nQ; ++Q) {
          const uint32_t B = lb + (uint32_t)Q * 65536u;
          pair_pass(std::integral_constant<int, 0>{}, B, cb + (4 * Q) * TILE8, acc);
          if (4 * Q + 2 < m) pair_pass(std::integral_constant<int, 1>{}, B, cb + (4 * Q + 2) * TILE8, acc);
        }
      } else {
        const uint32_t B = lb + (uint32_t)b * 65536u;
        pair_pass(std::integral_constant<int, 0>{}, B, cb, acc);
        if (4 * ch + 2 < m) pair_pass(std::integral_constant<int, 1>{}, B, cb + 2 * TILE8, acc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    if (RES || tile < nvt) {
      emit(acc, ((int64_t)tile + a.tile0) * TILE8 + warp * C8);
#pragma unroll
      for (int e = 0; e < C8; ++e) acc[e] = 0u;
    }
  }
  flush(0);
  flush(1);
}

int launch_scan8p(pqs_ctx* ctx, Scan8PArgs a) {
  const int nQ = (a.m + 3) / 4;
  const bool res = nQ <= 2;
  const int smem = 227 * 1024;
  auto kern = res ? scan8p_kernel<true> : scan8p_kernel<false>;
  static uint64_t attr_set[2] = {0, 0};  // per device
  if (!((attr_set[res] >> (ctx->device & 63)) & 1)) {
    PQS_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set[res] |= 1ull << (ctx->device & 63);
  }
  a.nqg = cdiv(a.nq, 32);
  const int64_t total = a.nqg * a.nvt;
  if (total <= 0) return PQS_OK;
  const int64_t nctas = std::min<int64_t>(total, (int64_t)ctx->sm_count);
  kern<<<(unsigned)nctas, SCAN8_THREADS, smem, ctx->stream>>>(a);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

constexpr int RESIDENT_BUDGET = 160 * 1024;

template <int MODE>
int launch_scan8(pqs_ctx* ctx, Scan8Args a) {
  const size_t row_bytes = (size_t)a.k * 64;
  a.resident = (size_t)a.m * row_bytes <= RESIDENT_BUDGET ? 1 : 0;
  if (a.resident) {
    a.mc = a.m;
  } else {
    int mc = (int)(CHUNK_BUDGET / (2 * row_bytes + 2 * TILE8));
    a.mc = std::max(1, std::min(mc, a.m));
  }
  const size_t tab = a.resident ? (size_t)a.m * row_bytes : 2 * (size_t)a.mc * row_bytes;
  size_t smem = tab + 2 * (size_t)a.mc * TILE8;
  if (MODE == MODE8_FILTER) smem += (size_t)CSTAGE8 * SCAN8_THREADS * 4;
  if (smem > 227 * 1024) return set_err(ctx, PQS_ERR_UNSUPPORTED, "scan8: table chunk does not fit shared memory");
  auto kern = a.resident ? scan8_kernel<MODE, true> : scan8_kernel<MODE, false>;
  PQS_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  a.nqg = cdiv(a.nq, 32);
  const int64_t total = a.nqg * a.nvt;
  if (total <= 0) return PQS_OK;
  const int64_t nctas = std::min<int64_t>(total, (int64_t)ctx->sm_count);  // 1 CTA / SM (smem)
  a.one = 1u;
  a.c64 = 64u;
  dim3 grid((unsigned)nctas);
  kern<<<grid, SCAN8_THREADS, smem, ctx->stream>>>(a);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

// threshold from the u32 lower-bound sample (scale e0): t = r-th smallest;
// D' = (t + m) * 2^-e0 + slack bounds the r-th smallest d - O; the filter
// scale e1 puts D' near 2^16 * max(1, m/8); theta = floor(D' * 2^e1).
__global__ void theta8_kernel(const uint32_t* __restrict__ sample, int64_t ns, int r, int m,
                              const int* __restrict__ e0, const double* __restrict__ slack, int* __restrict__ e1,
                              uint32_t* __restrict__ theta, double target, uint32_t tmax) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned int s_prefix, s_k, s_valid, s_vmax;
  const int64_t q = blockIdx.x;
  const uint32_t* row = sample + q * ns;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_k = (unsigned)(r - 1);
    s_valid = 0;
    s_vmax = 0;
  }
  __syncthreads();
  unsigned int valid = 0, vmax = 0;
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
    const uint32_t v = row[i];
    if (v != 0xFFFFFFFFu) {
      ++valid;
      vmax = max(vmax, v);
    }
  }
  atomicAdd(&s_valid, valid);
  for (int o = 16; o > 0; o >>= 1) vmax = max(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&s_vmax, vmax);
  __syncthreads();
  if (s_valid < (unsigned)r) {
    if (threadIdx.x == 0) {
      e1[q] = e0[q];
      theta[q] = tmax;
    }
    return;
  }
  // MSD radix select over the significant bits only: the first digit is the
  // top 8 bits below the largest value's leading one (all 256 bins in use,
  // no hot-bin atomics), then 8-bit digits down to bit 0.  k-th smallest
  // (0-based) of the valid values arr[i * stride], i < n; result in s_prefix
  const int top0 = 32 - __clz((int)s_vmax);
  auto radix_kth = [&](const uint32_t* arr, int64_t n, int64_t stride, unsigned kth) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_k = kth;
    }
    __syncthreads();
    for (int top = top0; top > 0;) {
      const int width = top < 8 ? top : 8, shift = top - width;
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const unsigned prefix = s_prefix;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t v = arr[i * stride];
        if (v == 0xFFFFFFFFu) continue;
        const bool match = top >= 32 ? true : ((v ^ prefix) >> top) == 0;
        if (match) atomicAdd(&hist[(v >> shift) & ((1u << width) - 1u)], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // warp-parallel digit search: lane l owns bins 8l..8l+7
        const int lane = threadIdx.x;
        unsigned h8[8], s8 = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) s8 += (h8[u] = hist[8 * lane + u]);
        unsigned incl = s8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const unsigned kk = s_k, excl = incl - s8;
        if (kk >= excl && kk < incl) {
          unsigned c = excl;
          int u = 0;
          while (kk >= c + h8[u]) c += h8[u++];
          s_k = kk - c;
          s_prefix = prefix | ((unsigned)(8 * lane + u) << shift);
        }
      }
      __syncthreads();
      top = shift;
    }
  };
  // The r-th smallest of a few 10^4 sums is a low quantile: a pivot from a
  // strided subsample (rank ~3 r scaled to it), the values below it compacted
  // into shared memory (a few hundred), the select among those -- two passes
  // over the sample instead of five.  The full-array select runs only when
  // the pivot missed.
  constexpr int SUB = 1024, SMALL = 2048;
  __shared__ uint32_t small[SMALL];
  __shared__ unsigned int s_cnt2;
  bool done = false;
  if (ns >= 8 * SUB && (int64_t)s_valid >= 8ll * r) {
    const int64_t stride = ns / SUB;
    if (threadIdx.x == 0) s_cnt2 = 0;
    __syncthreads();
    unsigned int sv = 0;
    for (int i = threadIdx.x; i < SUB; i += blockDim.x) sv += row[i * stride] != 0xFFFFFFFFu;
    atomicAdd(&s_cnt2, sv);
    __syncthreads();
    const unsigned int subv = s_cnt2;
    const unsigned int want = (unsigned)((3ull * (unsigned)r * subv + s_valid - 1) / s_valid) + 8u;
    if (want < subv) {
      radix_kth(row, SUB, stride, want);
      const uint32_t pivot = s_prefix;
      __syncthreads();
      if (threadIdx.x == 0) s_cnt2 = 0;
      __syncthreads();
      for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
        const uint32_t v = row[i];
        if (v <= pivot) {
          const unsigned int p = atomicAdd(&s_cnt2, 1u);
          if (p < SMALL) small[p] = v;
        }
      }
      __syncthreads();
      const unsigned int nsm = s_cnt2;
      if (nsm >= (unsigned)r && nsm <= SMALL) {
        radix_kth(small, nsm, 1, (unsigned)(r - 1));
        done = true;
      }
    }
  }
  if (!done) radix_kth(row, ns, 1, (unsigned)(r - 1));
  if (threadIdx.x == 0) {
    const double Dp = ldexp((double)s_prefix + (double)m, -e0[q]) + slack[q];
    int e = e0[q];
    if (Dp > 0.0) {
      e = (int)floor(log2(target / Dp));
      e = max(-1000, min(1000, e));
    }
    const double th = floor(ldexp(Dp, e) * (1.0 + 1e-12));
    e1[q] = e;
    theta[q] = th >= (double)tmax ? tmax : (uint32_t)th;
  }
}

// Second threshold of the packed filter: the exact r-th smallest distance D2
// among the candidates of the first tiles (select_kernel's output) bounds the
// r-th smallest overall, so the remaining tiles are filtered with
// floor(2^e1 (D2 - O + slack)) -- the same certified form as theta8_kernel's,
// from an exact distance instead of a sampled lower bound.
__global__ void theta8_refine_kernel(const double* __restrict__ topd, const int32_t* __restrict__ topc, int64_t nq,
                                     int r, int m, const float* __restrict__ off, const double* __restrict__ slack,
                                     const int* __restrict__ e1, uint32_t* __restrict__ theta) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq || topc[q] < r) return;
  double O = 0.0;
  for (int j = 0; j < m; ++j) O += (double)off[q * m + j];
  const double Dp = (topd[q * r + r - 1] - O) + slack[q];
  if (!(Dp >= 0.0)) return;
  const double th = floor(ldexp(Dp, e1[q]) * (1.0 + 1e-12)) + 1.0;
  if (th < (double)theta[q]) theta[q] = (uint32_t)th;
}

__global__ void fill_u32_kernel(uint32_t* p, int64_t n, uint32_t v) {
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
int launch_scan_distances(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, double* d_out) {
  if (db->n == 0 || nq == 0) return PQS_OK;
  dim3 grid((unsigned)cdiv(db->n, 256), (unsigned)nq);
  dense_adc_kernel<<<grid, 256, 0, ctx->stream>>>(d_tables, db->codes8, db->n, db->m, db->k, nq, nullptr, d_out);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int run_adc_topr(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, int r, double* d_dist,
                 int64_t* d_ids, int32_t* d_count) {
  const int64_t n = db->n;
  const int m = db->m, k = db->k;
  if (n == 0) {
    SelArgs s{};
    s.src = SEL_DENSE_F64;
    s.nq = nq;
    s.r = r;
    s.n = 0;
    s.out_d = d_dist;
    s.out_i = d_ids;
    s.out_c = d_count;
    return launch_select(ctx, s);
  }
  // ---- u16 lower-bound tables, scale e0 (no saturation)
  float* off = nullptr;
  int* e0 = nullptr;
  int* e1 = nullptr;
  double* slack = nullptr;
  uint16_t* tt = nullptr;
  uint32_t* theta = nullptr;
  PQS_TRY(scratch(ctx, S_AERR, (size_t)(nq * m), &off));
  PQS_TRY(scratch(ctx, S_QMINMAX, (size_t)nq * 2, &e0));
  e1 = e0 + nq;
  PQS_TRY(scratch(ctx, S_PREFIX, (size_t)nq, &slack));
  // the filter pass runs the packed two-queries-per-word kernel (K3p) when the
  // entries keep >= 9 bits (m <= 64); PQS_OPT_SCAN8_ENGINE = 1 keeps the u16 kernel
  if (ctx->scan8_engine == 2 && m > P16_MAX_M)
    return set_err(ctx, PQS_ERR_UNSUPPORTED, "packed scan8 engine takes m <= 64");
  const bool packed = ctx->scan8_engine != 1 && m <= P16_MAX_M;
  // threshold scale of the packed filter: entries clip at floor(32767 / m).  For
  // m <= 8 the threshold stays below the clip value, so a code with a clipped
  // entry can never pass (no false candidates from clipping; cfg0: 3836 ->
  // fewer candidates per query); for larger m that would leave too few bits
  // (m = 64: clip 511), so the threshold sits at 8191 = 16 clip / m x the
  // average entry of a threshold-distance code
  static const double tgt_env = getenv("PQS_P16_TARGET") ? atof(getenv("PQS_P16_TARGET")) : 0.0;  // tuning
  const double p16_target = tgt_env > 0.0 ? tgt_env : (m <= 8 ? std::min(P16_TARGET, (double)(P16_TMAX / (uint32_t)m) - 1.0) : P16_TARGET);
  const int mq = ((m + 3) / 4) * 4;
  PQS_TRY(scratch(ctx, S_TABLES_T, (size_t)(cdiv(nq, 32) * 32 * (packed ? mq : m) * k), &tt));
  PQS_TRY(scratch(ctx, S_THETA, (size_t)nq, &theta));
  tables_u16_stats_kernel<<<(unsigned)nq, 256, 0, ctx->stream>>>(d_tables, nq, m, k, off, e0, slack);
  PQS_LAUNCHED(ctx);
  const int64_t tt_total = cdiv(nq, 32) * m * (int64_t)k * 32;
  tables_u16_t_kernel<<<(unsigned)(cdiv(nq, 32) * m), TU16_THREADS, 0, ctx->stream>>>(d_tables, off, e0, nq, m, k, tt);
  PQS_LAUNCHED(ctx);

  const int64_t cap = std::min<int64_t>(ctx->cand_cap, n);
  const int64_t r_eff = std::min<int64_t>(r, n);
  if (n <= cap) {
    fill_u32_kernel<<<(unsigned)cdiv(nq, 256), 256, 0, ctx->stream>>>(theta, nq, packed ? P16_TMAX : 0xFFFFFFFEu);
    PQS_LAUNCHED(ctx);
    if (packed) {
      tables_p16_kernel<<<(unsigned)(cdiv(nq, 32) * mq), TU16_THREADS, 0, ctx->stream>>>(
          d_tables, off, e0, nq, m, k, P16_TMAX / (uint32_t)m, reinterpret_cast<uint32_t*>(tt));
      PQS_LAUNCHED(ctx);
    }
  } else {
    int64_t st = std::max<int64_t>(cdiv(db->ntiles, ctx->sample_div), cdiv(16 * r_eff, TILE8));
    st = std::min<int64_t>(st, db->ntiles);
    const int64_t step = std::max<int64_t>(1, db->ntiles / st);
    const int64_t ns = st * TILE8;
    uint32_t* sample = nullptr;
    PQS_TRY(scratch(ctx, S_SAMPLE, (size_t)(nq * ns), &sample));
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
    theta8_kernel<<<(unsigned)nq, 256, 0, ctx->stream>>>(
        sample, ns, (int)r_eff, m, e0, slack, e1, theta, packed ? p16_target : 65536.0 * (m > 8 ? m / 8.0 : 1.0),
        packed ? P16_TMAX : 0xFFFFFFFEu);
    PQS_LAUNCHED(ctx);
    // rebuild the tables at the filter scale e1
    if (packed)
      tables_p16_kernel<<<(unsigned)(cdiv(nq, 32) * mq), TU16_THREADS, 0, ctx->stream>>>(
          d_tables, off, e1, nq, m, k, P16_TMAX / (uint32_t)m, reinterpret_cast<uint32_t*>(tt));
    else
      tables_u16_t_kernel<<<(unsigned)(cdiv(nq, 32) * m), TU16_THREADS, 0, ctx->stream>>>(d_tables, off, e1, nq, m, k, tt);
    PQS_LAUNCHED(ctx);
  }

  uint64_t* cand = nullptr;
  int* cnt = nullptr;
  PQS_TRY(scratch(ctx, S_CAND, (size_t)(nq * cap), &cand));
  PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)nq, &cnt));
  PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
  if (packed) {
    Scan8PArgs a{};
    a.tp = reinterpret_cast<const uint32_t*>(tt);
    a.codes = db->codes8;
    a.n = n;
    a.m = m;
    a.k = k;
    a.nq = nq;
    a.nvt = db->ntiles;
    a.theta = theta;
    a.cand = cand;
    a.cand_cnt = cnt;
    a.cap = cap;
    // Two steps when the list is long: the first 1/8 of the tiles with the
    // sampled threshold, then the exact r-th distance among their candidates
    // (one small select) tightens the threshold for the other 7/8 -- about 3x
    // fewer candidates for the exact re-score and the final select.
    static const int t1div = getenv("PQS_ADC_T1_DIV") ? std::max(2, atoi(getenv("PQS_ADC_T1_DIV"))) : 8;  // tuning
    const int64_t t1 = (n > cap && db->ntiles >= 64 && r_eff == r) ? std::max<int64_t>(1, db->ntiles / t1div) : 0;
    PQS_TRY(scan_timer_begin(ctx));
    if (t1 > 0) {
      a.nvt = t1;
      a.tile0 = 0;
      PQS_TRY(launch_scan8p(ctx, a));
      uint64_t* gk1 = nullptr;
      int64_t* gi1 = nullptr;
      PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * cap), &gk1));
      PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * cap), &gi1));
      SelArgs s1{};
      s1.src = SEL_CAND_ADC;
      s1.nq = nq;
      s1.r = r;
      s1.cand = cand;
      s1.cand_cnt = cnt;
      s1.cap = cap;
      s1.ids = db->ids;
      s1.id_base = db->id_base;
      s1.tables = d_tables;
      s1.codes8 = db->codes8;
      s1.codes_rm = db->codes_rm;
      s1.m = m;
      s1.k = k;
      s1.out_d = d_dist;  // scratch here: the final select overwrites them
      s1.out_i = d_ids;
      s1.out_c = d_count;
      s1.gkeys = gk1;
      s1.gids = gi1;
      s1.gcap = cap;
      PQS_TRY(launch_select(ctx, s1));
      theta8_refine_kernel<<<(unsigned)cdiv(nq, 128), 128, 0, ctx->stream>>>(d_dist, d_count, nq, r, m, off, slack, e1,
                                                                            theta);
      PQS_LAUNCHED(ctx);
      a.nvt = db->ntiles - t1;
      a.tile0 = t1;
    }
    PQS_TRY(launch_scan8p(ctx, a));
    PQS_TRY(scan_timer_end(ctx));
    ctx->last_scan_launches = t1 > 0 ? 2 : 1;
    ctx->last_scan_engine = 5;
    ctx->last_scan_work = (double)nq * (double)n * (double)m;
  } else {
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
    ctx->last_scan_engine = 3;
    ctx->last_scan_work = (double)nq * (double)n * (double)m;
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
  s.codes_rm = db->codes_rm;
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
  int64_t mx = 0, ctot = 0;
  for (int64_t q = 0; q < nq; ++q) {
    mx = std::max<int64_t>(mx, hcnt[q]);
    ctot += hcnt[q];
    if (hcnt[q] > cap || hcnt[q] < r_eff || ctx->force_fallback) over.push_back((int)q);
  }
  ctx->last_max_cand = mx;
  ctx->last_cand_total = ctot;
  ctx->last_rerank_total = ctot;  // every candidate is re-scored exactly
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
