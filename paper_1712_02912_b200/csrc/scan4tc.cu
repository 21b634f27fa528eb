// scan4tc.cu -- Quick ADC scan on the 5th-gen tensor cores (tcgen05, kind::i8).
//
// Reference semantics: quantized_distances / qadc_scan (quickadc.py:87-141):
// bin(code) = min(sum_j qt[j][code_j], 127) with qt entries in [0, 127].
//
// The sum is an exact integer GEMM: with A[code][16j + i] = (code_j == i)
// (one-hot, K = 16 m = 256 for m = 16) and B[q][16j + i] = qt_q[j][i],
//   S[code][q] = sum_k A[code][k] * B[q][k]         (u8 x u8 -> s32, exact)
// and the filter keeps (code, q) with S <= theta_q (theta_q <= 127, so
// S = bin for every survivor).  Per CTA (persistent, one per SM):
//   * B for a group of 256 queries (64 KB, canonical K-major no-swizzle
//     layout) is TMA-bulk-copied once per group (double-buffered);
//   * warps 4-7 expand 128 codes per tile from the 4-bit quad layout into the
//     one-hot A tile (32 KB, double-buffered) with 16-byte shared stores;
//   * one elected thread of warp 8 issues 8 tcgen05.mma (M=128, N=256, K=32)
//     per tile into a TMEM accumulator (2 x 256 columns, double-buffered) and
//     commits to mbarriers;
//   * warps 0-3 tcgen05.ld the accumulator (lane = code, column = query),
//     compare against the per-query threshold with a sign-bit OR (1.5
//     instr/value) and append the rare survivors to a per-CTA record list.
// A small bucketing kernel turns the records into the per-query candidate
// lists consumed by select_kernel (SEL_CAND_BIN), exactly as the PRMT scan.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "pqs_common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int TC_M = 128;          // codes per tile (TMEM lanes)
constexpr int TC_N = 256;          // queries per group (TMEM columns per accumulator)
constexpr int TC_K = 256;          // one-hot width (16 components x 16 values)
constexpr int TC_KB = TC_K + 32;   // + one K step carrying the per-query threshold (A: ones, B: -(theta+1))
constexpr int A32_BYTES = TC_M * TC_K;   // 32 KB: one-hot tile with the threshold folded into B
constexpr int SS_NA = 3;                 // one-hot tile buffers of the SS filter
constexpr int B_BYTES = TC_N * TC_KB;    // 72 KB per 256-query group
constexpr int B_ONEHOT_BYTES = TC_N * TC_K;  // its first 64 KB: the quantized tables
constexpr int LBO_A = (TC_M / 8) * 128;  // byte distance between K-chunks of A (2048)
constexpr int LBO_B = (TC_N / 8) * 128;  // ... of B (4096)
constexpr int TC_THREADS = 13 * 32;      // 8 epilogue + 4 producer + 1 MMA warp
constexpr int EPI_WARPS = 8;
constexpr int ESTAGE = 48;  // per-thread survivor staging slots (u32)

using tc::bulk_g2s;
using tc::make_desc;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::mbar_wait_sleep;
using tc::mma_commit;
using tc::smem_u32;
__device__ __forceinline__ void tc_fence_before() { tc::fence_before(); }
__device__ __forceinline__ void tc_fence_after() { tc::fence_after(); }

// instruction descriptor: u8 x u8 -> s32, K-major A and B, M=128, N=256
// A unsigned (one-hot), B signed (tables <= 127 and the negative threshold column)
constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                           ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate)
      : "memory");
}
#define TMEM_LD32(taddr, v) TC_TMEM_LD32(taddr, v)
#define TMEM_LD64(taddr, v) TC_TMEM_LD64(taddr, v)

struct Scan4TcArgs {
  const uint32_t* words;   // 4-bit quad layout (mp = 16: 8 words per quad)
  int64_t n;
  const uint8_t* bglob;    // [nqg][B_BYTES] canonical B tiles
  const uint16_t* nadd;    // [nqg][256] per column: S = D + nadd (the threshold folded into B, build_bias_kernel)
  int64_t nq, nqg, ntiles; // ntiles of TC_M codes in this launch's range
  int64_t tile0;           // first tile of the range
  uint64_t* rec;           // [gridDim][rec_cap] (q << 40 | bin << 32 | idx)
  int* rec_cnt;            // [gridDim]
  int64_t rec_cap;
  unsigned long long* dbg;  // optional per-tile timestamps of CTA 0 (ns), 8 per tile
  int dbg_mode;             // timing experiments (PQS_TC_MODE): bit 0 skip the epilogue work, bit 1 skip the one-hot writes
};

using tc::gtime;

__global__ void __launch_bounds__(TC_THREADS, 1) scan4tc_kernel(Scan4TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smtc[];
  uint8_t* sB = smtc;                           // 64 KB (one query group)
  uint8_t* sA = smtc + B_ONEHOT_BYTES;          // SS_NA x 32 KB one-hot tiles
  uint16_t* sAdd = reinterpret_cast<uint16_t*>(smtc + B_ONEHOT_BYTES + SS_NA * A32_BYTES);  // [2 buffers][256]
  uint32_t* stage = reinterpret_cast<uint32_t*>(smtc + B_ONEHOT_BYTES + SS_NA * A32_BYTES + 2 * TC_N * 2);
  __shared__ __align__(8) uint64_t bar_b[2], bar_afull[SS_NA], bar_aempty[SS_NA], bar_accfull[2], bar_accempty[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_cnt;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.nqg * a.ntiles;
  // a CTA range spans <= 2 query groups: (group, tile) of item w without division
  const int64_t gfirst = ((int64_t)blockIdx.x * total / gridDim.x) / a.ntiles;
  const int64_t wsplit = (gfirst + 1) * a.ntiles;
  auto group_of = [&](int64_t w) { return w < wsplit ? gfirst : gfirst + 1; };
  auto tile_of = [&](int64_t w) { return w < wsplit ? w - gfirst * a.ntiles : w - wsplit; };
  const int64_t w0 = (int64_t)blockIdx.x * total / gridDim.x;
  const int64_t w1 = (int64_t)(blockIdx.x + 1) * total / gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_b[i], 1);
      mbar_init(&bar_accfull[i], 1);   // tcgen05.commit
      mbar_init(&bar_accempty[i], EPI_WARPS);  // one arrive per epilogue warp
    }
    for (int i = 0; i < SS_NA; ++i) {
      mbar_init(&bar_afull[i], 4);     // one arrive per producer warp
      mbar_init(&bar_aempty[i], 1);    // tcgen05.commit
    }
    s_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: 2 accumulators x 256 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (w0 < w1) {
    if (warp == EPI_WARPS + 4) {
      // ---------------- MMA issuer (+ B loader) ----------------
      if (lane == 0) {
        int64_t cur_g = -1;
        int gi = -1;
        for (int64_t w = w0; w < w1; ++w) {
          const int64_t it = w - w0;
          const int64_t g = group_of(w);
          if (g != cur_g) {
            ++gi;
            const int bb = gi & 1;
            if (it > 0) {
              // B is single-buffered: every MMA of the previous group must be done
              // (its last commit to bar_aempty) before the new B overwrites it
              mbar_wait(&bar_aempty[(it - 1) % SS_NA], (uint32_t)(((it - 1) / SS_NA) & 1));
            }
            mbar_expect_tx(&bar_b[bb], (uint32_t)(B_ONEHOT_BYTES + TC_N * 2));
            bulk_g2s(sB, a.bglob + g * (int64_t)B_BYTES, B_ONEHOT_BYTES, &bar_b[bb]);
            bulk_g2s(sAdd + bb * TC_N, a.nadd + g * TC_N, TC_N * 2, &bar_b[bb]);
            mbar_wait(&bar_b[bb], 0);
            cur_g = g;
          }
          const int ab = (int)(it & 1);
          const uint32_t ph = (uint32_t)((it >> 1) & 1);
          const int aq = (int)(it % SS_NA);
          const uint32_t aph = (uint32_t)((it / SS_NA) & 1);
          if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it * 8 + 0] = gtime();
          mbar_wait(&bar_afull[aq], aph);         // one-hot tile written (spin: critical path)
          if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it * 8 + 1] = gtime();
          mbar_wait(&bar_accempty[ab], ph ^ 1);   // accumulator drained (first use passes)
          if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it * 8 + 2] = gtime();
          tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(ab * TC_N);
          const uint32_t a_base = smem_u32(sA + aq * A32_BYTES);
          const uint32_t b_base = smem_u32(sB);
#pragma unroll
          for (int s = 0; s < TC_K / 32; ++s) {  // K = 256: the threshold is folded into component 0 of B
            const uint64_t da = make_desc(a_base + (uint32_t)(2 * s) * LBO_A, LBO_A, 128);
            const uint64_t db = make_desc(b_base + (uint32_t)(2 * s) * LBO_B, LBO_B, 128);
            mma_i8(d_tmem, da, db, s > 0 ? 1u : 0u);
          }
          mma_commit(&bar_aempty[aq]);
          mma_commit(&bar_accfull[ab]);
        }
      }
    } else if (warp >= EPI_WARPS) {
      // ---------------- one-hot producers: thread = code row ----------------
      const int row = (warp - EPI_WARPS) * 32 + lane;  // 0..127
      const uint32_t row_off = (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
      // the code words of the next two tiles are loaded ahead (registers), so
      // the L2/HBM latency of the 4-bit codes hides behind the MMAs
      auto load_words = [&](int64_t w, uint4& x0, uint4& x1) {
        x0 = make_uint4(0u, 0u, 0u, 0u);
        x1 = x0;
        if (w < w1) {
          const int64_t c = (a.tile0 + tile_of(w)) * TC_M + row;
          if (c < a.n) {
            const uint4* src = reinterpret_cast<const uint4*>(a.words + (c >> 2) * 8);
            x0 = __ldg(src);
            x1 = __ldg(src + 1);
          }
        }
      };
      uint4 n0a, n0b, n1a, n1b;
      load_words(w0, n0a, n0b);
      load_words(w0 + 1, n1a, n1b);
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        const int aq = (int)(it % SS_NA);
        const uint32_t aph = (uint32_t)((it / SS_NA) & 1);
        const uint4 x0 = n0a, x1 = n0b;
        n0a = n1a;
        n0b = n1b;
        load_words(w + 2, n1a, n1b);
        mbar_wait_sleep(&bar_aempty[aq], aph ^ 1);  // MMA finished reading this buffer
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == EPI_WARPS * 32) a.dbg[it * 8 + 3] = gtime();
        const int64_t tile = a.tile0 + tile_of(w);
        const int64_t code = tile * TC_M + row;
        const uint32_t wd[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const int sh = 4 * (int)(code & 3);
        uint8_t* dst = sA + aq * A32_BYTES + row_off;
        if (a.dbg_mode & 2) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_afull[aq]);
          continue;
        }
#pragma unroll
        for (int p = 0; p < 8; ++p) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t v = (wd[p] >> (16 * h + sh)) & 15u;  // component 2p+h
            const uint32_t one = 1u << (8 * (v & 3));
            uint4 o;
            o.x = (v >> 2) == 0 ? one : 0u;
            o.y = (v >> 2) == 1 ? one : 0u;
            o.z = (v >> 2) == 2 ? one : 0u;
            o.w = (v >> 2) == 3 ? one : 0u;
            *reinterpret_cast<uint4*>(dst + (2 * p + h) * LBO_A) = o;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == EPI_WARPS * 32) a.dbg[it * 8 + 4] = gtime();
        if (lane == 0) mbar_arrive(&bar_afull[aq]);
      }
    } else {
      // ---------------- epilogue: warp w reads TMEM lanes 32w..32w+31 (lane = code) ----------------
      // survivors are staged per thread as 32-bit records (tile-iteration << 15 |
      // column << 7 | bin) with predicated stores -- no divergent branches per value
      uint32_t* my_stage = stage + threadIdx.x;  // [slot][EPI thread]
      uint32_t* my_x = stage + ESTAGE * EPI_WARPS * 32 + threadIdx.x;  // [16][EPI thread] word stash
      const int quad = warp & 3, half = warp >> 2;  // TMEM lane quadrant, query-column half
      const int row = quad * 32 + lane;
      int ncand = 0;
      auto flush = [&]() {
        const int base = atomicAdd(&s_cnt, ncand);
        for (int i = 0; i < ncand; ++i) {
          const uint32_t r = my_stage[i * (EPI_WARPS * 32)];
          const int64_t wi = w0 + (int64_t)(r >> 15);
          const int64_t gg = group_of(wi);
          const int64_t code = (a.tile0 + tile_of(wi)) * TC_M + row;
          const int64_t q = gg * TC_N + ((r >> 7) & 255u);
          if (base + i < a.rec_cap)
            a.rec[(int64_t)blockIdx.x * a.rec_cap + base + i] =
                ((uint64_t)q << 40) | ((uint64_t)(r & 127u) << 32) | (uint64_t)(uint32_t)code;
        }
        ncand = 0;
      };
      int64_t cur_g = -1;
      int gi = -1;
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        const int64_t g = group_of(w);
        if (g != cur_g) {
          ++gi;
          mbar_wait(&bar_b[gi & 1], 0);  // biases of this group are in smem
          cur_g = g;
        }
        const int ab = (int)(it & 1);
        const uint32_t ph = (uint32_t)((it >> 1) & 1);
        mbar_wait(&bar_accfull[ab], ph);
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == 0) a.dbg[it * 8 + 5] = gtime();
        tc_fence_after();
        const int64_t tile = a.tile0 + tile_of(w);
        const bool cvalid = tile * TC_M + row < a.n;
        const uint16_t* nadd = sAdd + (gi & 1) * TC_N;
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * TC_N);
        const uint32_t itag = (uint32_t)it << 15;
        if (!(a.dbg_mode & 1)) {
          // the warp's 128 query columns in one load: .pack::16b keeps the low
          // 16 bits of every column (|D| < 2^15), two columns per register
          // (column 2i in the low half) -- half the TMEM read and OR work
          const int c0 = half * (TC_N / 2);
          uint32_t v[64];
          TC_TMEM_LD64_PACK16(tbase + (uint32_t)c0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (a.dbg && blockIdx.x == 0 && it < 64 && lane == 0) a.dbg[512 + it * 16 + warp] = gtime();
          // the accumulator is in registers: release it to the MMA now (the
          // hit test and the rare survivor path run off its critical path)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_accempty[ab]);
          // D = S - (theta + 1) per query column: a survivor is a negative D
          uint32_t orv = 0;
#pragma unroll
          for (int i = 0; i < 64; ++i) orv |= v[i];
          if ((orv & 0x80008000u) && cvalid) {  // lane-local, rare
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {  // four 32-column quarters
              const int cc = c0 + 32 * hh;
              // hit mask: bit i <- column cc+2i, bit 16+i <- column cc+2i+1 (sign of D);
              // the packed D pairs go to a per-thread stash for the dynamic reads below
              uint32_t mask = 0;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const uint32_t x = v[16 * hh + i];
                mask |= (x >> (15 - i)) & (0x00010001u << i);
                my_x[i * (EPI_WARPS * 32)] = x;
              }
              const uint32_t base = itag | ((uint32_t)cc << 7);
              while (mask) {
                const int bi = __ffs(mask) - 1;
                mask &= mask - 1;
                const int i = bi & 15, h = bi >> 4;
                const int col = cc + 2 * i + h;
                const int D = (int)(int16_t)(my_x[i * (EPI_WARPS * 32)] >> (16 * h));
                const uint32_t S = (uint32_t)(D + (int)nadd[col]);
                my_stage[ncand * (EPI_WARPS * 32)] = base + ((uint32_t)(2 * i + h) << 7) + min(S, 127u);
                ++ncand;
              }
              if (ncand > ESTAGE - 32) flush();  // rare
            }
          }
        }
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == 0) a.dbg[it * 8 + 6] = gtime();
        if (a.dbg && blockIdx.x == 0 && it < 64 && lane == 0) a.dbg[512 + it * 16 + 8 + warp] = gtime();
        if (a.dbg_mode & 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_accempty[ab]);
        }
      }
      if (ncand > 0) flush();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) a.rec_cnt[blockIdx.x] = s_cnt;
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}


// ---------------------------------------------------------------------------
// Threshold-sample histogram on tcgen05 (roles transposed w.r.t. the filter):
// A = the quantized tables of 128 queries (one half of a 256-query group's B
// tile, read in place: rows n in [128h, 128h+128) sit at byte offset 2048h
// of every 4096-byte K chunk), B = the one-hot of 256 codes (N = 256,
// K-major, K chunk stride 4096), D = 128 query lanes x 256 code columns in
// TMEM.  Each epilogue thread owns one query lane and adds its 256 sums'
// bins into shared u32 counters [pair of bins][query] (shared atomics,
// conflict-free: consecutive lanes are consecutive words), flushed to the
// global (nq, 128) histogram at each pair's upper bin.  Codes >= nh are
// zero rows (sum 0 -> pair 0); the caller subtracts them.
constexpr int HN = 256;                       // codes per tile (N)
constexpr int HO_BYTES = HN * TC_K;           // one-hot tile, 64 KB
constexpr int LBO_O = (HN / 8) * 128;         // 4096
constexpr int H_EPI_WARPS = 8;                // 2 per TMEM lane quadrant, 128 code columns each
constexpr int H_THREADS = (H_EPI_WARPS + 8 + 1) * 32;  // epilogue + 8 producer + 1 MMA warp
constexpr int H_PAIRS = 64;
constexpr uint32_t IDESC_H = (2u << 4) | ((uint32_t)(HN >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);

struct HistTcArgs {
  const uint32_t* words;
  int64_t nh;              // codes [0, nh) are counted
  const uint8_t* bglob;    // [nqg][B_BYTES]
  int64_t nq, nqg, ntiles; // ntiles of HN codes
  unsigned int* ghist;     // (nq, 128)
};

__device__ __forceinline__ void mma_i8_h(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC_H), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(H_THREADS, 1) scan4tc_hist_kernel(HistTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smh[];
  uint8_t* sG = smh;                                    // 64 KB: query tables of one group
  uint8_t* sO = smh + B_ONEHOT_BYTES;                   // 64 KB: one-hot of 256 codes
  unsigned int* hist = reinterpret_cast<unsigned int*>(smh + B_ONEHOT_BYTES + HO_BYTES);  // [64][256]
  __shared__ __align__(8) uint64_t bar_g, bar_ofull, bar_oempty, bar_accfull[2], bar_accempty[2];
  __shared__ uint32_t s_tmem;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.nqg * a.ntiles;
  const int64_t w0 = (int64_t)blockIdx.x * total / gridDim.x;
  const int64_t w1 = (int64_t)(blockIdx.x + 1) * total / gridDim.x;

  if (threadIdx.x == 0) {
    mbar_init(&bar_g, 1);
    mbar_init(&bar_ofull, 8);       // one arrive per producer warp
    mbar_init(&bar_oempty, 1);      // tcgen05.commit after both halves
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_accfull[i], 1);
      mbar_init(&bar_accempty[i], H_EPI_WARPS);  // every epilogue warp reads both query halves
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < H_PAIRS * TC_N; i += blockDim.x) hist[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (w0 < w1) {
    if (warp == H_EPI_WARPS + 8) {
      // ---------------- MMA issuer (+ group table loader) ----------------
      if (lane == 0) {
        int64_t cur_g = -1;
        int gi = -1;
        for (int64_t w = w0; w < w1; ++w) {
          const int64_t it = w - w0;
          const int64_t g = w / a.ntiles;
          if (g != cur_g) {
            ++gi;
            if (it > 0) mbar_wait(&bar_oempty, (uint32_t)((it - 1) & 1));  // all MMAs on the old tables done
            mbar_expect_tx(&bar_g, (uint32_t)B_ONEHOT_BYTES);
            bulk_g2s(sG, a.bglob + g * (int64_t)B_BYTES, B_ONEHOT_BYTES, &bar_g);
            mbar_wait(&bar_g, (uint32_t)(gi & 1));
            cur_g = g;
          }
          const uint32_t ph = (uint32_t)(it & 1);
          mbar_wait(&bar_ofull, ph);  // one-hot of this tile written
          const uint32_t o_base = smem_u32(sO);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait(&bar_accempty[h], ph ^ 1u);  // previous tile's half h drained
            tc_fence_after();
            const uint32_t g_base = smem_u32(sG) + (uint32_t)h * 2048u;
            const uint32_t d_tmem = tmem + (uint32_t)(h * HN);
#pragma unroll
            for (int s2 = 0; s2 < TC_K / 32; ++s2) {
              const uint64_t da = make_desc(g_base + (uint32_t)(2 * s2) * LBO_B, LBO_B, 128);
              const uint64_t db = make_desc(o_base + (uint32_t)(2 * s2) * LBO_O, LBO_O, 128);
              mma_i8_h(d_tmem, da, db, s2 > 0 ? 1u : 0u);
            }
            mma_commit(&bar_accfull[h]);
          }
          mma_commit(&bar_oempty);
        }
      }
    } else if (warp >= H_EPI_WARPS) {
      // ---------------- one-hot producers: thread = code row (256 rows) ----------------
      const int row = (warp - H_EPI_WARPS) * 32 + lane;  // 0..255
      const uint32_t row_off = (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u;
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        mbar_wait_sleep(&bar_oempty, (uint32_t)((it & 1) ^ 1));  // MMAs of the previous tile done
        const int64_t tile = w % a.ntiles;
        const int64_t code = tile * HN + row;
        uint8_t* dst = sO + row_off;
        if (code < a.nh) {
          const uint4* src = reinterpret_cast<const uint4*>(a.words + (code >> 2) * 8);
          const uint4 x0 = __ldg(src), x1 = __ldg(src + 1);
          const uint32_t wd[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
          const int sh = 4 * (int)(code & 3);
#pragma unroll
          for (int p = 0; p < 8; ++p) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t v = (wd[p] >> (16 * h + sh)) & 15u;  // component 2p+h
              const uint32_t one = 1u << (8 * (v & 3));
              uint4 o;
              o.x = (v >> 2) == 0 ? one : 0u;
              o.y = (v >> 2) == 1 ? one : 0u;
              o.z = (v >> 2) == 2 ? one : 0u;
              o.w = (v >> 2) == 3 ? one : 0u;
              *reinterpret_cast<uint4*>(dst + (2 * p + h) * LBO_O) = o;
            }
          }
        } else {  // beyond the counted range: an all-zero row (sum 0)
#pragma unroll
          for (int k = 0; k < 16; ++k) *reinterpret_cast<uint4*>(dst + k * LBO_O) = make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_ofull);
      }
    } else {
      // ---------------- epilogue: thread = query lane, 128 code columns per warp ----------------
      const int quad = warp & 3, half_c = warp >> 2;
      const int row = quad * 32 + lane;  // query lane within the 128-query half
      int64_t cur_g = -1;
      auto flush = [&](int64_t g) {
        // the 8 epilogue warps' 256 threads own the 256 queries of the group
        asm volatile("bar.sync 1, %0;" ::"r"(H_EPI_WARPS * 32));
        const int t = warp * 32 + lane;
        const int64_t q = g * TC_N + t;
        for (int b = 0; b < H_PAIRS; ++b) {
          const unsigned int v = hist[b * TC_N + t];
          if (v) {
            if (q < a.nq) atomicAdd(a.ghist + q * 128 + 2 * b + 1, v);
            hist[b * TC_N + t] = 0;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(H_EPI_WARPS * 32));
      };
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        const int64_t g = w / a.ntiles;
        if (g != cur_g) {
          if (cur_g >= 0) flush(cur_g);
          cur_g = g;
        }
        const uint32_t ph = (uint32_t)(it & 1);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&bar_accfull[h], ph);
          tc_fence_after();
          unsigned int* hq = hist + h * 128 + row;  // this lane's query column
          const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(h * HN + half_c * 128);
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 64) {
            uint32_t v[64];
            TMEM_LD64(tbase + (uint32_t)c0, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 64; ++i) atomicAdd(hq + (min(v[i], 127u) >> 1) * TC_N, 1u);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_accempty[h]);
        }
      }
      if (cur_g >= 0) flush(cur_g);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// B tiles in the canonical K-major no-swizzle layout + negated thresholds:
// B[n][k] at (k/16) * LBO_B + (n/8) * 128 + (n%8) * 16 + k%16, k = 16 j + i.
__global__ void build_b_kernel(const uint8_t* __restrict__ qt, int64_t nq, int m, int64_t nqg,
                               uint8_t* __restrict__ bglob) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one per (group, n, j)
  if (gid >= nqg * TC_N * 16) return;
  const int j = (int)(gid % 16);
  const int n = (int)((gid / 16) % TC_N);
  const int64_t g = gid / (16 * TC_N);
  const int64_t q = g * TC_N + n;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (q < nq && j < m) v = *reinterpret_cast<const uint4*>(qt + (q * m + j) * 16);
  *reinterpret_cast<uint4*>(bglob + g * (int64_t)B_BYTES + (int64_t)j * LBO_B + (n >> 3) * 128 + (n & 7) * 16) = v;
}


// ---------------------------------------------------------------------------
// The filter with the one-hot operand in TENSOR MEMORY (tcgen05.mma A from
// TMEM, "TS"): the producers tcgen05.st each code's one-hot row straight into
// TMEM, so shared memory only carries B (the query tables) to the tensor core
// -- the SS kernel above moves 3 bytes of shared memory per 2 it feeds to the
// MMA (A written + read, B read) and is co-limited by shared-memory bandwidth.
// The threshold is folded into component 0 of B instead of an extra K step:
// every code selects exactly one entry of each component, so B[q][i] =
// qt_q[0][i] - (theta_q + 1) (fits s8: qt <= 127, theta + 1 <= 128) gives
// D = S - (theta + 1); theta 127 (admit everything) adds -128 to every
// component (D = S - 2048 < 0); padding queries / THETA_NONE: no bias.
// K = 256 = 8 MMA K steps (the SS kernel issues 9).  TMEM: 2 accumulators of
// TS_N = 192 query columns + 2 one-hot buffers of 64 columns = 512.
constexpr int TS_N = 192;                 // queries per group
constexpr int TS_K = 256;                 // one-hot width (16 components x 16 values)
constexpr int TS_B_BYTES = TS_N * TS_K;   // 48 KB per group
constexpr int LBO_TS = (TS_N / 8) * 128;  // 3072: byte distance of 16-byte K chunks of B
constexpr int TS_ACOL = 2 * TS_N;         // first one-hot buffer column (384)
constexpr int TS_THREADS = 13 * 32;       // 8 epilogue + 4 producer + 1 MMA warp
constexpr uint32_t IDESC_TS = tc::idesc(2u, 0u, 1u, TC_M, TS_N);  // s32 <- u8 (A) x s8 (B)

__global__ void __launch_bounds__(TS_THREADS, 1) scan4ts_kernel(Scan4TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smts[];
  uint8_t* sB = smts;                                                        // 48 KB (one query group)
  uint16_t* sAdd = reinterpret_cast<uint16_t*>(smts + TS_B_BYTES);          // [2][TS_N]
  uint32_t* stage = reinterpret_cast<uint32_t*>(smts + TS_B_BYTES + 2 * TS_N * 2);
  __shared__ __align__(8) uint64_t bar_b[2], bar_afull[2], bar_aempty[2], bar_accfull[2], bar_accempty[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_cnt;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = a.nqg * a.ntiles;
  const int64_t gfirst = ((int64_t)blockIdx.x * total / gridDim.x) / a.ntiles;
  const int64_t wsplit = (gfirst + 1) * a.ntiles;
  auto group_of = [&](int64_t w) { return w < wsplit ? gfirst : gfirst + 1; };
  auto tile_of = [&](int64_t w) { return w < wsplit ? w - gfirst * a.ntiles : w - wsplit; };
  const int64_t w0 = (int64_t)blockIdx.x * total / gridDim.x;
  const int64_t w1 = (int64_t)(blockIdx.x + 1) * total / gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_b[i], 1);
      mbar_init(&bar_afull[i], 4);            // one arrive per producer warp
      mbar_init(&bar_aempty[i], 1);           // tcgen05.commit
      mbar_init(&bar_accfull[i], 1);          // tcgen05.commit
      mbar_init(&bar_accempty[i], EPI_WARPS); // one arrive per epilogue warp
    }
    s_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (w0 < w1) {
    if (warp == EPI_WARPS + 4) {
      // ---------------- MMA issuer (+ B loader) ----------------
      if (lane == 0) {
        int64_t cur_g = -1;
        int gi = -1;
        for (int64_t w = w0; w < w1; ++w) {
          const int64_t it = w - w0;
          const int64_t g = group_of(w);
          if (g != cur_g) {
            ++gi;
            const int bb = gi & 1;
            if (it > 0) mbar_wait(&bar_aempty[(it - 1) & 1], (uint32_t)(((it - 1) >> 1) & 1));
            mbar_expect_tx(&bar_b[bb], (uint32_t)(TS_B_BYTES + TS_N * 2));
            bulk_g2s(sB, a.bglob + g * (int64_t)TS_B_BYTES, TS_B_BYTES, &bar_b[bb]);
            bulk_g2s(sAdd + bb * TS_N, a.nadd + g * TS_N, TS_N * 2, &bar_b[bb]);
            mbar_wait(&bar_b[bb], 0);
            cur_g = g;
          }
          const int ab = (int)(it & 1);
          const uint32_t ph = (uint32_t)((it >> 1) & 1);
          if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it * 8 + 0] = gtime();
          mbar_wait(&bar_afull[ab], ph);         // one-hot rows stored to TMEM
          if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it * 8 + 1] = gtime();
          mbar_wait(&bar_accempty[ab], ph ^ 1);  // accumulator drained (first use passes)
          if (a.dbg && blockIdx.x == 0 && it < 64) a.dbg[it * 8 + 2] = gtime();
          tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(ab * TS_N);
          const uint32_t a_tmem = tmem + (uint32_t)(TS_ACOL + ab * (TS_K / 4));
          const uint32_t b_base = smem_u32(sB);
#pragma unroll
          for (int s = 0; s < TS_K / 32; ++s) {
            const uint64_t db = make_desc(b_base + (uint32_t)(2 * s) * LBO_TS, LBO_TS, 128);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
                "r"(a_tmem + (uint32_t)(8 * s)), "l"(db), "r"(IDESC_TS), "r"(s > 0 ? 1u : 0u)
                : "memory");
          }
          mma_commit(&bar_aempty[ab]);
          mma_commit(&bar_accfull[ab]);
        }
      }
    } else if (warp >= EPI_WARPS) {
      // ---------------- one-hot producers: thread = code row = TMEM lane ----------------
      const int quad = warp & 3;
      const int row = quad * 32 + lane;
      // the code words of the next two tiles are loaded ahead (registers), so
      // the HBM/L2 latency of the 4-bit codes hides behind the MMAs
      auto load_words = [&](int64_t w, uint4& x0, uint4& x1) {
        x0 = make_uint4(0u, 0u, 0u, 0u);
        x1 = x0;
        if (w < w1) {
          const int64_t code = (a.tile0 + tile_of(w)) * TC_M + row;
          if (code < a.n) {
            const uint4* src = reinterpret_cast<const uint4*>(a.words + (code >> 2) * 8);
            x0 = __ldg(src);
            x1 = __ldg(src + 1);
          }
        }
      };
      uint4 n0a, n0b, n1a, n1b;
      load_words(w0, n0a, n0b);
      load_words(w0 + 1, n1a, n1b);
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        const int ab = (int)(it & 1);
        const uint32_t ph = (uint32_t)((it >> 1) & 1);
        const uint4 x0 = n0a, x1 = n0b;
        n0a = n1a;
        n0b = n1b;
        load_words(w + 2, n1a, n1b);
        mbar_wait_sleep(&bar_aempty[ab], ph ^ 1);  // the MMAs reading this buffer are done
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == EPI_WARPS * 32) a.dbg[it * 8 + 3] = gtime();
        tc_fence_after();
        const int64_t tile = a.tile0 + tile_of(w);
        const int64_t code = tile * TC_M + row;
        uint32_t wd[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const int sh = 4 * (int)(code & 3);
        if (a.dbg_mode & 2) {  // timing experiment: no one-hot stores
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_afull[ab]);
          continue;
        }
        uint32_t o[64];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t v = (wd[p] >> (16 * h + sh)) & 15u;  // component 2p+h
            const uint32_t one = 1u << (8 * (v & 3));
            const int c = 2 * p + h;
            o[4 * c + 0] = (v >> 2) == 0 ? one : 0u;
            o[4 * c + 1] = (v >> 2) == 1 ? one : 0u;
            o[4 * c + 2] = (v >> 2) == 2 ? one : 0u;
            o[4 * c + 3] = (v >> 2) == 3 ? one : 0u;
          }
        }
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(TS_ACOL + ab * (TS_K / 4));
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,"
            "%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(
                taddr),
            "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]),
            "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]), "r"(o[16]),
            "r"(o[17]), "r"(o[18]), "r"(o[19]), "r"(o[20]), "r"(o[21]), "r"(o[22]), "r"(o[23]), "r"(o[24]),
            "r"(o[25]), "r"(o[26]), "r"(o[27]), "r"(o[28]), "r"(o[29]), "r"(o[30]), "r"(o[31]), "r"(o[32]),
            "r"(o[33]), "r"(o[34]), "r"(o[35]), "r"(o[36]), "r"(o[37]), "r"(o[38]), "r"(o[39]), "r"(o[40]),
            "r"(o[41]), "r"(o[42]), "r"(o[43]), "r"(o[44]), "r"(o[45]), "r"(o[46]), "r"(o[47]), "r"(o[48]),
            "r"(o[49]), "r"(o[50]), "r"(o[51]), "r"(o[52]), "r"(o[53]), "r"(o[54]), "r"(o[55]), "r"(o[56]),
            "r"(o[57]), "r"(o[58]), "r"(o[59]), "r"(o[60]), "r"(o[61]), "r"(o[62]), "r"(o[63])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == EPI_WARPS * 32) a.dbg[it * 8 + 4] = gtime();
        if (lane == 0) mbar_arrive(&bar_afull[ab]);
      }
    } else {
      // ---------------- epilogue: warp w reads TMEM lanes of quadrant w & 3, 96 query columns ----------------
      uint32_t* my_stage = stage + threadIdx.x;
      uint32_t* my_x = stage + ESTAGE * EPI_WARPS * 32 + threadIdx.x;
      const int quad = warp & 3, half = warp >> 2;
      const int row = quad * 32 + lane;
      int ncand = 0;
      auto flush = [&]() {
        const int base = atomicAdd(&s_cnt, ncand);
        for (int i = 0; i < ncand; ++i) {
          const uint32_t r = my_stage[i * (EPI_WARPS * 32)];
          const int64_t wi = w0 + (int64_t)(r >> 15);
          const int64_t gg = group_of(wi);
          const int64_t code = (a.tile0 + tile_of(wi)) * TC_M + row;
          const int64_t q = gg * TS_N + ((r >> 7) & 255u);
          if (base + i < a.rec_cap)
            a.rec[(int64_t)blockIdx.x * a.rec_cap + base + i] =
                ((uint64_t)q << 40) | ((uint64_t)(r & 127u) << 32) | (uint64_t)(uint32_t)code;
        }
        ncand = 0;
      };
      int64_t cur_g = -1;
      int gi = -1;
      for (int64_t w = w0; w < w1; ++w) {
        const int64_t it = w - w0;
        const int64_t g = group_of(w);
        if (g != cur_g) {
          ++gi;
          mbar_wait(&bar_b[gi & 1], 0);  // biases of this group are in smem
          cur_g = g;
        }
        const int ab = (int)(it & 1);
        const uint32_t ph = (uint32_t)((it >> 1) & 1);
        mbar_wait(&bar_accfull[ab], ph);
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == 0) a.dbg[it * 8 + 5] = gtime();
        tc_fence_after();
        const int64_t tile = a.tile0 + tile_of(w);
        const bool cvalid = tile * TC_M + row < a.n;
        const uint16_t* nadd = sAdd + (gi & 1) * TS_N;
        const int c0 = half * (TS_N / 2);
        const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * TS_N + c0);
        const uint32_t itag = (uint32_t)it << 15;
        if (a.dbg_mode & 1) {  // timing experiment: no epilogue work
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_accempty[ab]);
          continue;
        }
        // 96 columns as 48 registers of 16-bit pairs (.pack::16b: |D| < 2^15)
        uint32_t v[48];
        TC_TMEM_LD64_PACK16(tbase, v);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
            "%15}, [%16];"
            : "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]),
              "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]),
              "=r"(v[46]), "=r"(v[47])
            : "r"(tbase + 64u));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the accumulator is in registers: release it to the MMA now
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_accempty[ab]);
        uint32_t orv = 0;
#pragma unroll
        for (int i = 0; i < 48; ++i) orv |= v[i];
        if ((orv & 0x80008000u) && cvalid) {  // lane-local, rare
#pragma unroll
          for (int hh = 0; hh < 3; ++hh) {  // three 32-column groups
            const int cc = c0 + 32 * hh;
            uint32_t mask = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t x = v[16 * hh + i];
              mask |= (x >> (15 - i)) & (0x00010001u << i);
              my_x[i * (EPI_WARPS * 32)] = x;
            }
            const uint32_t base = itag | ((uint32_t)cc << 7);
            while (mask) {
              const int bi = __ffs(mask) - 1;
              mask &= mask - 1;
              const int i = bi & 15, h = bi >> 4;
              const int col = cc + 2 * i + h;
              const int D = (int)(int16_t)(my_x[i * (EPI_WARPS * 32)] >> (16 * h));
              const uint32_t S = (uint32_t)(D + (int)nadd[col]);
              my_stage[ncand * (EPI_WARPS * 32)] = base + ((uint32_t)(2 * i + h) << 7) + min(S, 127u);
              ++ncand;
            }
            if (ncand > ESTAGE - 32) flush();  // rare
          }
        }
        if (a.dbg && blockIdx.x == 0 && it < 64 && threadIdx.x == 0) a.dbg[it * 8 + 6] = gtime();
      }
      if (ncand > 0) flush();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) a.rec_cnt[blockIdx.x] = s_cnt;
  if (warp == 0) {
    tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// B tiles of the filter (canonical K-major, QN queries per group: 256 for
// SS, TS_N for TS) with the threshold folded into the tables: B[n][16 j + i] = qt[q][j][i], minus
// (theta + 1) on component 0 (theta <= 126) or minus 128 on every component
// (theta 127: admit every sum, D = S - 2048); THETA_NONE (255) and padding
// queries: plain tables (D = S >= 0, never a survivor).  nadd[n] = the bias.
template <int QN, int LBO, int GBYTES>
__global__ void build_b_fold_kernel(const uint8_t* __restrict__ qt, const uint8_t* __restrict__ theta, int64_t nq,
                                    int m, int64_t nqg, uint8_t* __restrict__ bglob, uint16_t* __restrict__ nadd) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one per (group, n, component j)
  if (gid >= nqg * QN * 16) return;
  const int j = (int)(gid % 16);
  const int n = (int)((gid / 16) % QN);
  const int64_t g = gid / (16 * QN);
  const int64_t q = g * QN + n;
  const uint32_t t = q < nq ? theta[q] : 255u;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (q < nq && j < m) v = *reinterpret_cast<const uint4*>(qt + (q * m + j) * 16);
  int bias = 0;
  if (t == 127u) bias = 128;
  else if (t != 255u && j == 0) bias = (int)t + 1;
  if (bias) {
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
    for (int k = 0; k < 4; ++k) {
      uint32_t x = 0;
      for (int b = 0; b < 4; ++b) x |= (uint32_t)(uint8_t)(int8_t)((int)((w[k] >> (8 * b)) & 255u) - bias) << (8 * b);
      w[k] = x;
    }
  }
  *reinterpret_cast<uint4*>(bglob + g * (int64_t)GBYTES + (int64_t)j * LBO + (n >> 3) * 128 + (n & 7) * 16) = v;
  if (j == 0) nadd[g * QN + n] = (uint16_t)(t == 127u ? 2048u : (t == 255u ? 0u : t + 1));
}

// per-CTA survivor records -> per-query candidate lists (bin << 32 | idx).
// One CTA per record region: shared histogram over queries, one global
// reservation per (region, query), then a scatter -- ~nq global atomics per
// region instead of one per record.
__global__ void bucket_kernel(const uint64_t* __restrict__ rec, const int* __restrict__ rec_cnt, int64_t rec_cap,
                              int64_t nq, uint64_t* __restrict__ cand, int* __restrict__ cand_cnt, int64_t cap,
                              int* __restrict__ ovf) {
  extern __shared__ int bsm[];
  int* hist = bsm;        // [nq]
  int* basev = bsm + nq;  // [nq]
  const int b = blockIdx.x;
  if (threadIdx.x == 0 && rec_cnt[b] > rec_cap) atomicOr(ovf, 1);
  const int cnt = (int)min((int64_t)rec_cnt[b], rec_cap);
  const uint64_t* r = rec + (int64_t)b * rec_cap;
  for (int64_t i = threadIdx.x; i < nq; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) atomicAdd(&hist[r[i] >> 40], 1);
  __syncthreads();
  for (int64_t i = threadIdx.x; i < nq; i += blockDim.x) {
    const int h = hist[i];
    basev[i] = h ? atomicAdd(cand_cnt + i, h) : 0;
    hist[i] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint64_t x = r[i];
    const int64_t q = (int64_t)(x >> 40);
    const int pos = basev[q] + atomicAdd(&hist[q], 1);
    if (pos < cap) cand[q * cap + pos] = x & 0xFFFFFFFFFFull;
  }
}

// fallback for very large query batches (histograms beyond shared memory)
__global__ void bucket_atomic_kernel(const uint64_t* __restrict__ rec, const int* __restrict__ rec_cnt,
                                     int64_t rec_cap, uint64_t* __restrict__ cand, int* __restrict__ cand_cnt,
                                     int64_t cap, int* __restrict__ ovf) {
  const int b = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0 && rec_cnt[b] > rec_cap) atomicOr(ovf, 1);
  const int cnt = (int)min((int64_t)rec_cnt[b], rec_cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const uint64_t r = rec[(int64_t)b * rec_cap + i];
    const int64_t q = (int64_t)(r >> 40);
    const int pos = atomicAdd(cand_cnt + q, 1);
    if (pos < cap) cand[q * cap + pos] = r & 0xFFFFFFFFFFull;
  }
}

}  // namespace

// PQS_TC_DEBUG: per-tile role timestamps of CTA 0 (ns since its first tile)
static int dump_debug(pqs_ctx* ctx, const unsigned long long* dbg) {
  std::vector<unsigned long long> d(64 * 8 + 64 * 16);
  PQS_CUDA(ctx, cudaMemcpy(d.data(), dbg, (64 * 8 + 64 * 16) * 8, cudaMemcpyDeviceToHost));
  const unsigned long long t0 = d[0];
  for (int it = 0; it < 24; ++it) {
    fprintf(stderr, "tile %2d:", it);
    for (int k = 0; k < 7; ++k) fprintf(stderr, " %8lld", d[it * 8 + k] ? (long long)(d[it * 8 + k] - t0) : -1ll);
    fprintf(stderr, " | ld");
    for (int k = 0; k < 8; ++k) {
      const unsigned long long x = d[512 + it * 16 + k];
      fprintf(stderr, " %6lld", x ? (long long)(x - t0) : -1ll);
    }
    fprintf(stderr, " | end");
    for (int k = 0; k < 8; ++k) {
      const unsigned long long x = d[512 + it * 16 + 8 + k];
      fprintf(stderr, " %6lld", x ? (long long)(x - t0) : -1ll);
    }
    fprintf(stderr, "\n");
  }
  return PQS_OK;
}

// Filtered Quick ADC scan on tcgen05 over the 128-code tiles [tile_begin,
// tile_end) with per-query thresholds theta (build_b: also (re)build the B
// tiles of the quantized tables).  Survivors are appended to the per-query
// candidate lists; a per-CTA record overflow sets *d_ovf (the caller re-runs
// the scan on the PRMT engine).  No host synchronisation.  Returns
// PQS_ERR_UNSUPPORTED when the shape is outside this kernel.
// queries per group of the filter kernel in use: SS (one-hot in shared
// memory, 3 one-hot buffers; default) or TS (PQS_TC_TS=1: one-hot in TMEM,
// 192-query groups -- measured slower on cfg4: 237 vs 195 ms per search)
static bool tc_use_ss() {
  static const bool ss = getenv("PQS_TC_TS") == nullptr;
  return ss;
}
int tc_query_group() { return tc_use_ss() ? TC_N : TS_N; }
int tc_k_per_eval() { return TC_K; }

int launch_scan4_tc(pqs_ctx* ctx, const pqs_db* db, const uint8_t* d_qt, const uint8_t* d_theta, int64_t nq,
                    int64_t tile_begin, int64_t tile_end, bool build_b, uint64_t* cand, int* cand_cnt, int64_t cap,
                    int* d_ovf) {
  if (db->mp != 16) return PQS_ERR_UNSUPPORTED;
  const bool ss = tc_use_ss();
  const int qn = ss ? TC_N : TS_N;
  const int64_t nqg = cdiv(nq, qn);
  const int64_t nctas_max = (int64_t)ctx->sm_count;
  if (tile_end <= tile_begin) return PQS_OK;
  // every CTA range must span <= 2 query groups (single-buffered B, decode of
  // the staged records) and fit the 17-bit tile-iteration field of a record:
  // long ranges are scanned in chunks of tiles, one launch each
  if (nqg >= nctas_max) return PQS_ERR_UNSUPPORTED;
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(tile_end - tile_begin, ((1 << 17) - 2) * nctas_max / nqg));
  // Every query group re-reads the launch's codes: keep them L2-resident.  16 MB
  // of codes per launch (16,384 tiles at m = 16) are read from DRAM once and
  // hit L2 for the other groups (cfg4: 11.2 GB -> 1.1 GB of DRAM reads per
  // search, 1.08x the code bytes, and ~3% less time; sweep 4k..64k tiles in
  // DESIGN.md); equal-sized chunks, so no launch is left with a sliver.
  if (nqg > 1) chunk = std::min<int64_t>(chunk, std::max<int64_t>(1, (16ll << 20) / ((int64_t)TC_M * db->mp / 2)));
  if (ctx->tc_chunk_tiles > 0) chunk = std::min<int64_t>(chunk, ctx->tc_chunk_tiles);
  chunk = cdiv(tile_end - tile_begin, cdiv(tile_end - tile_begin, chunk));
  for (int64_t c0 = tile_begin; c0 < tile_end; c0 += chunk) {
    const int64_t ntiles = std::min<int64_t>(chunk, tile_end - c0);
    const int64_t total = nqg * ntiles;
    // a CTA range no longer than a group's tile count spans <= 2 groups
    if (nqg > 1 && cdiv(total, std::min<int64_t>(nctas_max, total)) >= ntiles) return PQS_ERR_UNSUPPORTED;
  }
  uint8_t* bglob = nullptr;
  uint16_t* nadd = nullptr;
  uint64_t* rec = nullptr;
  int* rec_cnt = nullptr;
  PQS_TRY(scratch(ctx, S_TC_B, (size_t)(nqg * (ss ? B_BYTES : TS_B_BYTES)), &bglob));
  PQS_TRY(scratch(ctx, S_TC_TH, (size_t)(nqg * qn), &nadd));
  // survivors per CTA: expect ~nq*cap_used/nctas; size generously
  const int64_t rec_cap = std::max<int64_t>(1 << 16, cdiv(nq * std::min<int64_t>(cap, 8192), nctas_max) * 2);
  PQS_TRY(scratch(ctx, S_TC_REC, (size_t)(nctas_max * rec_cap), &rec));
  PQS_TRY(scratch(ctx, S_TC_RECCNT, (size_t)nctas_max, &rec_cnt));
  (void)build_b;  // the tables are rebuilt per launch with this launch's thresholds folded in
  if (ss) {
    build_b_fold_kernel<TC_N, LBO_B, B_BYTES><<<(unsigned)cdiv(nqg * TC_N * 16, 256), 256, 0, ctx->stream>>>(
        d_qt, d_theta, nq, db->m, nqg, bglob, nadd);
    PQS_LAUNCHED(ctx);
  } else {  // TS: the tables with this launch's thresholds folded in
    build_b_fold_kernel<TS_N, LBO_TS, TS_B_BYTES><<<(unsigned)cdiv(nqg * TS_N * 16, 256), 256, 0, ctx->stream>>>(
        d_qt, d_theta, nq, db->m, nqg, bglob, nadd);
    PQS_LAUNCHED(ctx);
  }
  const size_t smem = ss ? (size_t)B_ONEHOT_BYTES + SS_NA * (size_t)A32_BYTES + 2 * TC_N * 2 +
                               (size_t)(ESTAGE + 16) * EPI_WARPS * 32 * 4
                         : (size_t)TS_B_BYTES + 2 * TS_N * 2 + (size_t)(ESTAGE + 16) * EPI_WARPS * 32 * 4;
  if (ss)
    PQS_CUDA(ctx, cudaFuncSetAttribute(scan4tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  else
    PQS_CUDA(ctx, cudaFuncSetAttribute(scan4ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const size_t bsmem = (size_t)nq * 2 * sizeof(int);
  if (bsmem <= 200 * 1024)
    PQS_CUDA(ctx, cudaFuncSetAttribute(bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
  const int dbg_mode = getenv("PQS_TC_MODE") ? atoi(getenv("PQS_TC_MODE")) : 0;
  for (int64_t c0 = tile_begin; c0 < tile_end; c0 += chunk) {
    const int64_t ntiles = std::min<int64_t>(chunk, tile_end - c0);
    const int64_t total = nqg * ntiles;
    const int64_t nctas = std::min<int64_t>(nctas_max, total);
    Scan4TcArgs a{};
    a.words = db->words4;
    a.n = db->n;
    a.bglob = bglob;
    a.nadd = nadd;
    a.nq = nq;
    a.nqg = nqg;
    a.ntiles = ntiles;
    a.tile0 = c0;
    a.rec = rec;
    a.rec_cnt = rec_cnt;
    a.rec_cap = rec_cap;
    a.dbg = nullptr;
    a.dbg_mode = dbg_mode;
    if (getenv("PQS_TC_DEBUG")) {
      PQS_TRY(scratch(ctx, S_MISC, 64 * 8 + 64 * 16, &a.dbg));
      PQS_CUDA(ctx, cudaMemsetAsync(a.dbg, 0, (64 * 8 + 64 * 16) * 8, ctx->stream));
    }
    if (ss)
      scan4tc_kernel<<<(unsigned)nctas, TC_THREADS, smem, ctx->stream>>>(a);
    else
      scan4ts_kernel<<<(unsigned)nctas, TS_THREADS, smem, ctx->stream>>>(a);
    PQS_LAUNCHED(ctx);
    if (bsmem <= 200 * 1024) {
      bucket_kernel<<<(unsigned)nctas, 1024, bsmem, ctx->stream>>>(rec, rec_cnt, rec_cap, nq, cand, cand_cnt, cap,
                                                                    d_ovf);
    } else {
      dim3 bg(64, (unsigned)nctas);
      bucket_atomic_kernel<<<bg, 256, 0, ctx->stream>>>(rec, rec_cnt, rec_cap, cand, cand_cnt, cap, d_ovf);
    }
    PQS_LAUNCHED(ctx);
    if (a.dbg) PQS_TRY(dump_debug(ctx, a.dbg));
  }
  return PQS_OK;
}

// Bin histogram of the codes [0, nh) for every query on tcgen05 (see
// scan4tc_hist_kernel); adds into ghist (nq, 128) at each bin pair's upper
// bin; the zero rows padding the last 256-code tile land in bin 1 (the
// caller subtracts cdiv(nh, 256) * 256 - nh there).  Builds the B tiles
// (query tables) that launch_scan4_tc then reuses (build_b = false).
int launch_hist_tc(pqs_ctx* ctx, const pqs_db* db, const uint8_t* d_qt, int64_t nq, int64_t nh,
                   unsigned int* ghist) {
  if (db->mp != 16) return PQS_ERR_UNSUPPORTED;
  const int64_t nqg = cdiv(nq, TC_N);
  const int64_t ntiles = cdiv(nh, HN);
  const int64_t total = nqg * ntiles;
  if (total == 0) return PQS_OK;
  uint8_t* bglob = nullptr;
  PQS_TRY(scratch(ctx, S_TC_B, (size_t)(nqg * B_BYTES), &bglob));
  build_b_kernel<<<(unsigned)cdiv(nqg * TC_N * 16, 256), 256, 0, ctx->stream>>>(d_qt, nq, db->m, nqg, bglob);
  PQS_LAUNCHED(ctx);
  HistTcArgs a{};
  a.words = db->words4;
  a.nh = nh;
  a.bglob = bglob;
  a.nq = nq;
  a.nqg = nqg;
  a.ntiles = ntiles;
  a.ghist = ghist;
  const size_t smem = (size_t)B_ONEHOT_BYTES + HO_BYTES + (size_t)H_PAIRS * TC_N * 4;
  PQS_CUDA(ctx, cudaFuncSetAttribute(scan4tc_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t nctas = std::min<int64_t>((int64_t)ctx->sm_count, total);
  scan4tc_hist_kernel<<<(unsigned)nctas, H_THREADS, smem, ctx->stream>>>(a);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}
