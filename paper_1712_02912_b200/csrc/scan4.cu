// scan4.cu -- Quick ADC over 4-bit codes (K2 layout, K9 params, K4 scan).
//
// Reference: qadc_scan (quickadc.py:104-141), quantize (fastscan.py:42-57),
// quantized_distances / qadc_block (quickadc.py:66-101).
//
// K4 design: one thread per query holds that query's m
// quantized 16-entry tables in registers (4 x u32 per component).  Codes are
// stored as 4-code quads: one u32 per (quad, component pair) whose low/high
// 16 bits are PRMT selectors for components 2p / 2p+1.  Each tile of 1024
// codes is expanded once per CTA into shared memory as (s, s^0x8888, s>>16,
// (s^0x8888)>>16) and read by every thread with a broadcast LDS.128.  A
// 16-entry lookup of 4 codes is two PRMTs: entries 0-7 with the raw selector
// (a set nibble msb sign-replicates a byte <= 127 -> 0), entries 8-15 with
// the msb-flipped selector.  Two components are summed in byte lanes (<= 254)
// and widened into 16-bit lanes; min(sum,127) equals the reference's clamp
// after every add because entries are non-negative (quickadc.py:87-92).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "pqs_common.cuh"

namespace {

constexpr int SCAN4_THREADS = 256;
// K9: 128 threads per query CTA so a 1000-query batch is one wave (12 CTAs/SM)
constexpr int PARAMS_THREADS = 128;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

// FMA-pipe integer ops.  The multiplier comes from a kernel argument (runtime
// value 1 or 2^24) so ptxas cannot strength-reduce them into ALU-pipe
// IADD3/SHF: the PRMT lookups keep the ALU pipe busy, the byte-lane sums and
// the widening shift run on the otherwise idle FMA pipe (IMAD / IMAD.HI).
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t imulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// ---------------------------------------------------------------- K2 layout
// codes (n, m) row-major -> words[(tile*QUADS4 + g) * (mp/2) + p]
__global__ void build_words4_kernel(const uint8_t* __restrict__ codes, int64_t n, int m, int mp,
                                    int64_t nquads, uint32_t* __restrict__ words) {
  const int hp = mp / 2;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= nquads * hp) return;
  const int p = (int)(gid % hp);
  const int64_t g = gid / hp;
  uint32_t w = 0;
  for (int i = 0; i < 4; ++i) {
    const int64_t c = g * 4 + i;
    if (c >= n) continue;
    const int j0 = 2 * p, j1 = 2 * p + 1;
    const uint32_t v0 = j0 < m ? (codes[c * m + j0] & 15u) : 0u;
    const uint32_t v1 = j1 < m ? (codes[c * m + j1] & 15u) : 0u;
    w |= v0 << (4 * i);
    w |= v1 << (16 + 4 * i);
  }
  words[gid] = w;
}

__device__ __forceinline__ int code4_at(const pqs_db& db, const uint32_t* __restrict__ words, int64_t i,
                                        int j) {
  const int hp = db.mp / 2;
  const uint32_t w = words[(i >> 2) * hp + (j >> 1)];
  const uint32_t sel = (j & 1) ? (w >> 16) : (w & 0xFFFFu);
  return (int)((sel >> (4 * (i & 3))) & 15u);
}

__global__ void quantize_kernel(const double* __restrict__ v, int64_t n, double qmin, double qmax, double scale,
                                uint8_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = quantize1(v[i], qmin, qmax, scale);
}

// ---------------------------------------------------------------- K9 params
// One CTA per query.  qmin = global fp32 table min; qmax = r-th smallest fp64
// ADC over the first n_init codes in storage order (max if n_init < r);
// qmax = max(qmax, qmin); quantize with fp64 scale = 127/span (0 if span==0).
struct ParamShared {
  unsigned int hist[256];
  unsigned long long red[SCAN4_THREADS / 32];
  float fred[SCAN4_THREADS / 32];
  unsigned long long prefix, k, vmin, vmax;
  double qmin, qmax;
};

__device__ __forceinline__ bool match_above4(uint64_t v, uint64_t prefix, int s) {
  return s >= 64 ? true : ((v ^ prefix) >> s) == 0;
}

// k-th smallest (0-based) of M keys in keys[] (block-wide), small helper
__device__ unsigned long long kth_smallest(const unsigned long long* keys, int64_t M, unsigned long long k,
                                           ParamShared& sh) {
  // min / max
  unsigned long long lo = ~0ull, hi = 0;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    lo = min(lo, keys[i]);
    hi = max(hi, keys[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = lo;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = ~0ull;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a = min(a, sh.red[i]);
    sh.vmin = a;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b = max(b, sh.red[i]);
    sh.vmax = b;
  }
  __syncthreads();
  const unsigned long long vmin = sh.vmin, vmax = sh.vmax;
  if (vmin == vmax) return vmin;
  const int hib = 63 - __clzll((long long)(vmin ^ vmax));
  int shift = (hib / 8) * 8;
  if (threadIdx.x == 0) {
    const int s = shift + 8;
    sh.prefix = s >= 64 ? 0ull : (vmin >> s) << s;
    sh.k = k;
  }
  __syncthreads();
  for (; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sh.prefix;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
      const unsigned long long v = keys[i];
      if (match_above4(v, prefix, shift + 8)) atomicAdd(&sh.hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // lane-parallel digit search: each lane owns 8 bins
      const int lane = threadIdx.x;
      unsigned int s8 = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) s8 += sh.hist[lane * 8 + b];
      unsigned int incl = s8;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const unsigned long long kk = sh.k;
      const unsigned int excl = incl - s8;
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
        sh.k = kk - c;
        sh.prefix = prefix | ((unsigned long long)d << shift);
      }
    }
    __syncthreads();
  }
  return sh.prefix;
}

// k-th smallest of a few hundred keys by rank counting (broadcast reads):
// the key with #less <= k < #less + #equal.  Each thread ranks two keys in
// one unrolled pass (the shared loads stay in flight).
__device__ unsigned long long kth_smallest_small(const unsigned long long* keys, int M, int k, ParamShared& sh) {
  for (int t0 = threadIdx.x; t0 < M; t0 += 2 * blockDim.x) {
    const int t1 = t0 + blockDim.x;
    const unsigned long long v0 = keys[t0], v1 = t1 < M ? keys[t1] : ~0ull;
    int l0 = 0, e0 = 0, l1 = 0, e1 = 0;
#pragma unroll 8
    for (int i = 0; i < M; ++i) {
      const unsigned long long w = keys[i];
      l0 += w < v0 ? 1 : 0;
      e0 += w == v0 ? 1 : 0;
      l1 += w < v1 ? 1 : 0;
      e1 += w == v1 ? 1 : 0;
    }
    if (l0 <= k && k < l0 + e0) sh.prefix = v0;  // every writer holds the same value
    if (t1 < M && l1 <= k && k < l1 + e1) sh.prefix = v1;
  }
  __syncthreads();
  return sh.prefix;
}

__global__ void __launch_bounds__(PARAMS_THREADS) qadc_params_kernel(
    pqs_db db, const float* __restrict__ tables, int64_t nq, int init_count, int r,
    unsigned long long* __restrict__ gscratch, int64_t gscratch_ld, uint8_t* __restrict__ qt_out,
    double* __restrict__ qmm_out) {
  __shared__ ParamShared sh;
  __shared__ unsigned long long s_keys[2048];
  __shared__ float sT[32 * 16];
  __shared__ __align__(16) uint32_t s_src[2048];  // prefix codes (<= 256 codes: words or bytes)
  const int64_t q = blockIdx.x;
  const int m = db.m;
  const float* Tg = tables + q * (int64_t)m * 16;
  for (int i = threadIdx.x; i < m * 16; i += blockDim.x) sT[i] = Tg[i];
  const float* T = sT;
  // qmin
  float mn = __int_as_float(0x7f800000);
  for (int i = threadIdx.x; i < m * 16; i += blockDim.x) mn = fminf(mn, T[i]);
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) sh.fred[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = sh.fred[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) a = fminf(a, sh.fred[i]);
    sh.qmin = (double)a;
  }
  __syncthreads();
  // prefix distances
  const int64_t n_src = db.prefix ? db.n_prefix : db.n;
  const int64_t n_init = min((int64_t)init_count, n_src);
  unsigned long long* keys = n_init <= 2048 ? s_keys : gscratch + q * gscratch_ld;
  const int hp = db.mp / 2;
  if (n_init <= 256) {
    // stage the prefix codes with one coalesced pass (the per-code decode
    // below then reads shared memory instead of dependent global loads)
    if (db.prefix) {  // 16-byte loads (cudaMalloc'd, row-major prefix)
      const int nb = (int)n_init * m;
      for (int i = threadIdx.x; i < nb / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(s_src)[i] = reinterpret_cast<const uint4*>(db.prefix)[i];
      for (int i = (nb & ~15) + threadIdx.x; i < nb; i += blockDim.x) ((uint8_t*)s_src)[i] = db.prefix[i];
    } else {
      const int nw = (int)((n_init + 3) / 4) * hp;
      for (int i = threadIdx.x; i < nw; i += blockDim.x) s_src[i] = db.words4[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (int)n_init; i += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < m; ++j) {
        int c;
        if (db.prefix) {
          c = ((const uint8_t*)s_src)[i * m + j];
        } else {
          const uint32_t w = s_src[(i >> 2) * hp + (j >> 1)];
          c = (int)((((j & 1) ? (w >> 16) : w) >> (4 * (i & 3))) & 15u);
        }
        acc = __dadd_rn(acc, (double)T[j * 16 + c]);
      }
      keys[i] = dkey(acc);
    }
  } else {
    for (int64_t i = threadIdx.x; i < n_init; i += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < m; ++j) {
        const int c = db.prefix ? db.prefix[i * m + j] : code4_at(db, db.words4, i, j);
        acc = __dadd_rn(acc, (double)T[j * 16 + c]);
      }
      keys[i] = dkey(acc);
    }
  }
  __syncthreads();
  double qmax;
  const int64_t kq = n_init >= r ? r - 1 : n_init - 1;
  if (n_init <= 256) {
    qmax = dkey_inv(kth_smallest_small(keys, (int)n_init, (int)kq, sh));
  } else {
    qmax = dkey_inv(kth_smallest(keys, n_init, (unsigned long long)kq, sh));
  }
  const double qmin = sh.qmin;
  qmax = qmax > qmin ? qmax : qmin;
  const double span = __dsub_rn(qmax, qmin);
  const double scale = span > 0.0 ? __ddiv_rn(127.0, span) : 0.0;
  for (int i = threadIdx.x; i < m * 16; i += blockDim.x)
    qt_out[q * (int64_t)m * 16 + i] = quantize1((double)T[i], qmin, qmax, scale);
  if (threadIdx.x == 0) {
    qmm_out[2 * q] = qmin;
    qmm_out[2 * q + 1] = qmax;
  }
}

// ---------------------------------------------------------------- K4 scan
enum { MODE_DENSE = 0, MODE_FILTER = 1, MODE_HIST = 2 };

// theta value meaning "no survivors" (a strict threshold below bin 0)
constexpr uint8_t THETA_NONE = 255;

struct Scan4Args {
  const uint32_t* words;
  int64_t n;
  int m;
  const uint8_t* qt;       // (nq, m, 16)
  int64_t nq;
  // virtual tiles: tile(i) = tile_off + i * tile_step, i in [0, nvt)
  int64_t nvt, tile_off, tile_step, per_cta;
  int64_t nqg;             // query groups of SCAN4_THREADS
  int parts;               // work items per tile (quarter tiles give the small sample pass more CTAs)
  unsigned long long* work;  // dynamic tile counter (zeroed before launch)
  // dense
  uint8_t* out;
  int64_t ld;
  uint32_t one;            // runtime 1 (see imad)
  uint32_t k24;            // runtime 2^24 (v >> 8 as a high multiply)
  // filter
  const uint8_t* theta;
  uint64_t* cand;
  int* cand_cnt;
  int64_t cap;
  // hist
  unsigned int* ghist;     // (nq, 128) bin histograms of the scanned codes
};

template <int MP>
__device__ __forceinline__ void load_tile_raw(const uint32_t* __restrict__ words, int64_t tile, uint4* regs,
                                              int nthreads) {
  constexpr int HP = MP / 2;
  constexpr int WORDS = QUADS4 * HP;            // words per tile
  constexpr int V4 = WORDS / 4;                 // uint4 per tile
  const uint4* src = reinterpret_cast<const uint4*>(words + tile * (int64_t)WORDS);
  constexpr int PER = (V4 + SCAN4_THREADS - 1) / SCAN4_THREADS;
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    const int i = threadIdx.x + v * nthreads;
    if (i < V4) regs[v] = __ldg(src + i);
  }
}

template <int MP>
__device__ __forceinline__ void store_tile_pred(const uint4* regs, uint4* __restrict__ buf, int nthreads) {
  constexpr int HP = MP / 2;
  constexpr int WORDS = QUADS4 * HP;
  constexpr int V4 = WORDS / 4;
  constexpr int PER = (V4 + SCAN4_THREADS - 1) / SCAN4_THREADS;
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    const int i = threadIdx.x + v * nthreads;
    if (i < V4) {
      const uint32_t w4[4] = {regs[v].x, regs[v].y, regs[v].z, regs[v].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t w = w4[e];
        const uint32_t x = w ^ 0x88888888u;
        buf[i * 4 + e] = make_uint4(w, x, w >> 16, x >> 16);
      }
    }
  }
}

// Candidates are staged per thread in shared memory ([slot][thread], no
// atomics) and flushed to the query's global list CSTAGE at a time with one
// global atomicAdd, so the scan never waits on an atomic's return value.
constexpr int CSTAGE = 16;

__device__ __forceinline__ void flush_cands(const uint64_t* stage, int cnt, int64_t q, uint64_t* cand,
                                            int* cand_cnt, int64_t cap) {
  const int pos = atomicAdd(cand_cnt + q, cnt);
  for (int i = 0; i < cnt; ++i)
    if (pos + i < cap) cand[q * cap + pos + i] = stage[i * SCAN4_THREADS];
}

// MODE_HIST: per-thread (= per-query) u16 counters in shared memory, one per
// PAIR of bins (2k, 2k+1) -- 32 KB, two CTAs per SM -- laid out
// [pair][thread] so a warp's 32 increments touch 16 distinct words of 16
// banks whatever the bins (conflict-free).  Flushed to the global (nq, 128)
// histogram at the pair's upper bin 2k+1 (the threshold derived from it is
// then >= the exact one: certified) before a counter can wrap.
constexpr int HIST_PAIRS = 64;
constexpr int HIST_FLUSH_CODES = 60000;

__device__ __forceinline__ void flush_hist(uint16_t* h, int64_t q, bool valid, unsigned int* ghist) {
#pragma unroll 4
  for (int b = 0; b < HIST_PAIRS; ++b) {
    const unsigned int v = h[b * SCAN4_THREADS];
    if (v) {
      if (valid) atomicAdd(ghist + q * 128 + 2 * b + 1, v);
      h[b * SCAN4_THREADS] = 0;
    }
  }
}

template <int MP, int MODE>
__global__ void __launch_bounds__(SCAN4_THREADS, (MP <= 16 ? 2 : 1)) scan4_kernel(Scan4Args a) {
  constexpr int HP = MP / 2;
  constexpr int WORDS = QUADS4 * HP;
  constexpr int V4 = WORDS / 4;
  constexpr int PER = (V4 + SCAN4_THREADS - 1) / SCAN4_THREADS;
  extern __shared__ __align__(16) uint4 s_pred[];  // 2 buffers of WORDS uint4 (+ candidate stage)
  const int nthreads = blockDim.x;
  uint64_t* stage = reinterpret_cast<uint64_t*>(s_pred + 2 * WORDS) + threadIdx.x;
  uint16_t* hist = reinterpret_cast<uint16_t*>(s_pred + 2 * WORDS) + threadIdx.x;
  int ncand = 0;
  int hcodes = 0;  // codes counted since the last histogram flush
  if (MODE == MODE_HIST) {
    for (int b = 0; b < HIST_PAIRS; ++b) hist[b * SCAN4_THREADS] = 0;
  }

  // persistent CTAs grab tiles of the linearised (query group, tile) list from
  // a global counter (dynamic balance); tables are reloaded at group switches
  const long long per_group = a.nvt * a.parts;
  const long long total = a.nqg * per_group;
  const int gq = QUADS4 / a.parts;  // quads per work item
  __shared__ long long s_w[2];
  if (threadIdx.x == 0) {
    s_w[0] = atomicAdd(a.work, 1ull);
    s_w[1] = atomicAdd(a.work, 1ull);
  }
  __syncthreads();
  long long w = s_w[0], wn = s_w[1];
  if (w >= total) return;

  int64_t q = -1, cur_qg = -1;
  bool qvalid = false;
  uint32_t T[MP][4];
  uint32_t theta = 0, bias = 0;
  const uint32_t one = a.one, k24 = a.k24;
  auto load_group = [&](int64_t qg) {
    q = qg * SCAN4_THREADS + threadIdx.x;
    qvalid = q < a.nq;
#pragma unroll
    for (int j = 0; j < MP; ++j) {
      if (qvalid && j < a.m) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(a.qt + (q * a.m + j) * 16));
        T[j][0] = t.x;
        T[j][1] = t.y;
        T[j][2] = t.z;
        T[j][3] = t.w;
      } else {
        T[j][0] = T[j][1] = T[j][2] = T[j][3] = 0u;
      }
    }
    theta = (MODE == MODE_FILTER && qvalid) ? a.theta[q] : 0u;
    // theta 127 admits every code: bin = min(S, 127) <= 127 for any sum S
    if (theta == 127u) theta = 0x7FFFu;
    // THETA_NONE: bit 15 of every lane stays set -> no survivors
    bias = theta == THETA_NONE ? 0x80008000u : (0x7FFFu - theta) * 0x00010001u;
  };

  uint4 regs[PER];
  load_tile_raw<MP>(a.words, a.tile_off + ((w % per_group) / a.parts) * a.tile_step, regs, nthreads);
  store_tile_pred<MP>(regs, s_pred, nthreads);
  __syncthreads();

  int cur = 0;
  for (int it = 0;; ++it) {
    const int64_t qg = w / per_group;
    const int64_t rem = w - qg * per_group;
    const int64_t i = rem / a.parts;
    const int part = (int)(rem - i * a.parts);
    if (qg != cur_qg) {
      if (MODE == MODE_FILTER && ncand > 0) {
        flush_cands(stage, ncand, q, a.cand, a.cand_cnt, a.cap);
        ncand = 0;
      }
      if (MODE == MODE_HIST && hcodes > 0) {
        flush_hist(hist, q, qvalid, a.ghist);
        hcodes = 0;
      }
      load_group(qg);
      cur_qg = qg;
    }
    const bool has_next = (wn < total);
    if (has_next) load_tile_raw<MP>(a.words, a.tile_off + ((wn % per_group) / a.parts) * a.tile_step, regs, nthreads);
    const uint4* buf = s_pred + cur * WORDS;
    const int64_t tile = a.tile_off + i * a.tile_step;
    const int64_t code0 = tile * TILE4;
#pragma unroll 2
    for (int g = part * gq; g < (part + 1) * gq; ++g) {
      uint32_t ae = 0, ao = 0;
#pragma unroll
      for (int p = 0; p < HP; ++p) {
        const uint4 s = buf[g * HP + p];
        const uint32_t lo0 = prmt(T[2 * p][0], T[2 * p][1], s.x);
        const uint32_t hi0 = prmt(T[2 * p][2], T[2 * p][3], s.y);
        const uint32_t lo1 = prmt(T[2 * p + 1][0], T[2 * p + 1][1], s.z);
        const uint32_t hi1 = prmt(T[2 * p + 1][2], T[2 * p + 1][3], s.w);
        // two components per byte lane (each entry <= 127, sum <= 254)
        const uint32_t v = imad(imad(lo0, one, hi0), one, imad(lo1, one, hi1));
        ae = imad(v & 0x00FF00FFu, one, ae);
        ao = imad(imulhi(v, k24) & 0x00FF00FFu, one, ao);
      }
      const int64_t c = code0 + 4 * g;
      if (MODE == MODE_FILTER) {
        const uint32_t t = imad(ae, one, bias) & imad(ao, one, bias) & 0x80008000u;
        if (t != 0x80008000u && qvalid) {
          const uint32_t S[4] = {ae & 0xFFFFu, ao & 0xFFFFu, ae >> 16, ao >> 16};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (S[e] <= theta && c + e < a.n) {
              stage[ncand * SCAN4_THREADS] = ((uint64_t)S[e] << 32) | (uint64_t)(uint32_t)(c + e);
              if (++ncand == CSTAGE) {
                flush_cands(stage, ncand, q, a.cand, a.cand_cnt, a.cap);
                ncand = 0;
              }
            }
          }
        }
      } else if (MODE == MODE_HIST) {
        const uint32_t S[4] = {ae & 0xFFFFu, ao & 0xFFFFu, ae >> 16, ao >> 16};
        const int nv = (int)min((int64_t)4, a.n - c);  // valid codes of this quad
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t b = (S[e] < 127u ? S[e] : 127u) >> 1;
          if (e < nv) hist[b * SCAN4_THREADS] += 1;
        }
      } else {
        if (qvalid) {
          const uint32_t S[4] = {ae & 0xFFFFu, ao & 0xFFFFu, ae >> 16, ao >> 16};
          const int64_t col = i * TILE4 + 4 * g;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t b = S[e] < 127u ? S[e] : 127u;
            if (col + e < a.ld) a.out[q * a.ld + col + e] = (c + e < a.n) ? (uint8_t)b : (uint8_t)255;
          }
        }
      }
    }
    if (MODE == MODE_HIST) {
      hcodes += 4 * gq;
      if (hcodes > HIST_FLUSH_CODES - 4 * gq) {
        flush_hist(hist, q, qvalid, a.ghist);
        hcodes = 0;
      }
    }
    if (has_next) store_tile_pred<MP>(regs, s_pred + (cur ^ 1) * WORDS, nthreads);
    if (threadIdx.x == 0 && has_next) s_w[it & 1] = atomicAdd(a.work, 1ull);
    __syncthreads();
    if (!has_next) break;
    w = wn;
    wn = s_w[it & 1];
    cur ^= 1;
  }
  if (MODE == MODE_FILTER && ncand > 0 && q >= 0) flush_cands(stage, ncand, q, a.cand, a.cand_cnt, a.cap);
  if (MODE == MODE_HIST && hcodes > 0) flush_hist(hist, q, qvalid, a.ghist);
}

template <int MP, int MODE>
int launch_scan4_t(pqs_ctx* ctx, Scan4Args a, int64_t nq) {
  constexpr int HP = MP / 2;
  const size_t smem = 2 * (size_t)QUADS4 * HP * sizeof(uint4) +
                      (MODE == MODE_FILTER ? (size_t)CSTAGE * SCAN4_THREADS * sizeof(uint64_t) : 0) +
                      (MODE == MODE_HIST ? (size_t)HIST_PAIRS * SCAN4_THREADS * sizeof(uint16_t) : 0);
  PQS_CUDA(ctx, cudaFuncSetAttribute(scan4_kernel<MP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  const int threads = SCAN4_THREADS;  // the tile loader assumes a full CTA
  a.nqg = cdiv(nq, threads);
  if (a.parts <= 0) a.parts = 1;
  const int64_t total = a.nqg * a.nvt * a.parts;
  if (total <= 0) return PQS_OK;
  int per_sm = 0;
  PQS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan4_kernel<MP, MODE>, threads, smem));
  const int64_t nctas = std::min<int64_t>(total, (int64_t)ctx->sm_count * std::max(per_sm, 1));
  a.one = 1u;
  a.k24 = 1u << 24;
  PQS_TRY(scratch(ctx, S_WORK, 1, &a.work));
  PQS_CUDA(ctx, cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), ctx->stream));
  dim3 grid((unsigned)nctas);
  scan4_kernel<MP, MODE><<<grid, threads, smem, ctx->stream>>>(a);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

template <int MODE>
int launch_scan4(pqs_ctx* ctx, int mp, const Scan4Args& a, int64_t nq) {
  switch (mp) {
    case 2: return launch_scan4_t<2, MODE>(ctx, a, nq);
    case 4: return launch_scan4_t<4, MODE>(ctx, a, nq);
    case 8: return launch_scan4_t<8, MODE>(ctx, a, nq);
    case 16: return launch_scan4_t<16, MODE>(ctx, a, nq);
    case 32: return launch_scan4_t<32, MODE>(ctx, a, nq);
  }
  return set_err(ctx, PQS_ERR_UNSUPPORTED, "scan4: unsupported padded m");
}

// theta[q] = the r-th smallest bin of the histogram pass (127 if fewer than r);
// pad1 zero-sum padding codes counted in bin 1 are removed
__global__ void theta4_final_kernel(const unsigned int* __restrict__ ghist, int64_t nq, int r, unsigned int pad1,
                                    uint8_t* __restrict__ theta) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  unsigned long long c = 0;
  int t = 127;
  for (int b = 0; b < 128; ++b) {
    c += ghist[q * 128 + b] - (b == 1 ? pad1 : 0u);
    if (c >= (unsigned long long)r) {
      t = b;
      break;
    }
  }
  theta[q] = (uint8_t)t;
}

// after the prefix pass: theta_main from the prefix candidates (every prefix
// code with bin <= t0, and t0 >= the prefix's r-th smallest bin t): the r-th
// smallest candidate bin is t exactly.  An overflowed list (count > cap, the
// query takes the exact fallback) gets THETA_NONE.
__global__ void cand_theta_kernel(const uint64_t* __restrict__ cand, const int* __restrict__ cand_cnt, int64_t cap,
                                  int r, int strict, uint8_t* __restrict__ theta_main) {
  __shared__ unsigned int hist[128];
  const int64_t q = blockIdx.x;
  const int cnt = cand_cnt[q];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  if (cnt > cap) {
    if (threadIdx.x == 0) theta_main[q] = THETA_NONE;
    return;
  }
  const uint64_t* c = cand + q * cap;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint64_t b = c[i] >> 32;
    atomicAdd(&hist[b < 127 ? b : 127], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int acc = 0;
    int t = 127;
    for (int b = 0; b < 128; ++b) {
      acc += hist[b];
      if (acc >= (unsigned)r) {
        t = b;
        break;
      }
    }
    theta_main[q] = strict ? (t == 0 ? THETA_NONE : (uint8_t)(t - 1)) : (uint8_t)t;
  }
}

__global__ void fill_u8_kernel(uint8_t* p, int64_t n, uint8_t v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void gather_rows_u8_kernel(const uint8_t* __restrict__ src, const int* __restrict__ qmap, int64_t rows,
                                      int64_t width, uint8_t* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * width) return;
  const int64_t r = i / width, c = i % width;
  dst[i] = src[(int64_t)qmap[r] * width + c];
}

}  // namespace

int tc_query_group();
int tc_k_per_eval();
int launch_scan4_tc(pqs_ctx* ctx, const pqs_db* db, const uint8_t* d_qt, const uint8_t* d_theta, int64_t nq,
                    int64_t tile_begin, int64_t tile_end, bool build_b, uint64_t* cand, int* cand_cnt, int64_t cap,
                    int* d_ovf);
int launch_hist_tc(pqs_ctx* ctx, const pqs_db* db, const uint8_t* d_qt, int64_t nq, int64_t nh,
                   unsigned int* ghist);

// ---------------------------------------------------------------------------
int build_db4(pqs_ctx* ctx, pqs_db* db, const uint8_t* d_codes) {
  const int hp = db->mp / 2;
  const int64_t nquads = db->ntiles * QUADS4;
  const int64_t total = nquads * hp;
  build_words4_kernel<<<(unsigned)cdiv(total, 256), 256, 0, ctx->stream>>>(d_codes, db->n, db->m, db->mp,
                                                                           nquads, db->words4);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int launch_quantize(pqs_ctx* ctx, double qmin, double qmax, const double* d_v, int64_t n, uint8_t* d_out) {
  if (n == 0) return PQS_OK;
  const double span = qmax - qmin;
  const double scale = span > 0.0 ? 127.0 / span : 0.0;
  quantize_kernel<<<(unsigned)cdiv(n, 256), 256, 0, ctx->stream>>>(d_v, n, qmin, qmax, scale, d_out);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int launch_scan4_dense(pqs_ctx* ctx, const pqs_db* db, const uint8_t* d_qtables, int64_t nq, uint8_t* d_out,
                       int64_t ld_out) {
  Scan4Args a{};
  a.words = db->words4;
  a.n = db->n;
  a.m = db->m;
  a.qt = d_qtables;
  a.nq = nq;
  a.nvt = db->ntiles;
  a.tile_off = 0;
  a.tile_step = 1;
  a.out = d_out;
  a.ld = ld_out;
  return launch_scan4<MODE_DENSE>(ctx, db->mp, a, nq);
}

// ---------------------------------------------------------------------------
// Quick ADC top-r search.  The device phase (params -> threshold sample ->
// filtered scan -> select -> candidate counts into pinned host memory) makes
// no host decision that depends on device data, so it is captured once per
// (list, batch shape, options, scratch layout) as a CUDA graph and replayed;
// the host phase (record-overflow redo, exact dense fallback, statistics)
// runs after the single synchronisation.
namespace {

struct QadcRun {
  pqs_ctx* ctx;
  const pqs_db* db;
  const float* d_tables;
  int64_t nq;
  int init_count, r;
  uint8_t *d_bins, *d_qt;
  int64_t* d_ids;
  int32_t* d_count;
  double* d_qmm;
  // plan
  int64_t n = 0, cap = 0, r_eff = 0, st = 0, t1 = 0;
  int m = 0;
  bool second = false, used_tc = false;
  // buffers
  uint8_t *theta = nullptr, *theta_main = nullptr;
  uint64_t* cand = nullptr;
  int* cnt = nullptr;
  int* d_ovf = nullptr;
  SelArgs sel{};

  int main_theta() {
    cand_theta_kernel<<<(unsigned)nq, 128, 0, ctx->stream>>>(cand, cnt, cap, (int)r_eff, db->ids == nullptr ? 1 : 0,
                                                            theta_main);
    PQS_LAUNCHED(ctx);
    return PQS_OK;
  }

  // PRMT engine over the same two ranges
  int scan_prmt() {
    Scan4Args a{};
    a.words = db->words4;
    a.n = n;
    a.m = m;
    a.qt = d_qt;
    a.nq = nq;
    a.tile_step = 1;
    a.cand = cand;
    a.cand_cnt = cnt;
    a.cap = cap;
    a.nvt = t1;
    a.tile_off = 0;
    a.theta = theta;
    PQS_TRY(launch_scan4<MODE_FILTER>(ctx, db->mp, a, nq));
    if (second) {
      PQS_TRY(main_theta());
      a.nvt = db->ntiles - t1;
      a.tile_off = t1;
      a.theta = theta_main;
      PQS_TRY(launch_scan4<MODE_FILTER>(ctx, db->mp, a, nq));
    }
    ctx->last_scan_engine = 1;
    ctx->last_scan_work = (double)nq * (double)n * (double)m;
    return PQS_OK;
  }

  int device_phase() {
    n = db->n;
    m = db->m;
    // ---- K9: params + quantized tables
    const int64_t n_src = db->prefix ? db->n_prefix : n;
    const int64_t n_init = std::min<int64_t>(init_count, n_src);
    unsigned long long* pscratch = nullptr;
    if (n_init > 2048) PQS_TRY(scratch(ctx, S_PREFIX, (size_t)(nq * n_init), &pscratch));
    qadc_params_kernel<<<(unsigned)nq, PARAMS_THREADS, 0, ctx->stream>>>(*db, d_tables, nq, init_count, r, pscratch,
                                                                       n_init, d_qt, d_qmm);
    PQS_LAUNCHED(ctx);

    // ---- threshold: exact when every code fits the candidate buffer.
    // Otherwise certified thresholds from the first st tiles (the "prefix"):
    //   1. t0 = the r-th smallest bin of the first s0 tiles (histogram pass);
    //   2. the prefix is filtered with t0 (>= the prefix's r-th smallest bin t);
    //   3. t = the r-th smallest prefix candidate bin (cand_theta_kernel): every
    //      top-r code has bin <= t, and -- ids increasing in storage order -- a
    //      code after the prefix needs bin < t (the prefix holds r codes with
    //      bin <= t and smaller ids), so the rest is filtered with t - 1.
    PQS_TRY(scratch(ctx, S_THETA, (size_t)(2 * nq), &theta));
    theta_main = theta + nq;
    cap = std::min<int64_t>(ctx->cand_cap, std::max<int64_t>(n, 1));
    r_eff = std::min<int64_t>(r, n);
    st = 0;  // prefix tiles (TILE4 codes each); 0 = no sample
    bool b_built = false;  // tcgen05 B tiles (query tables) already built by the histogram pass
    if (n <= cap) {
      fill_u8_kernel<<<(unsigned)cdiv(nq, 256), 256, 0, ctx->stream>>>(theta, nq, 127);
      PQS_LAUNCHED(ctx);
    } else {
      const int64_t tmin = cdiv(16 * r_eff, TILE4);
      // prefix: 1/sample_div of the list, but at least min(1/4 of it, 256 tiles)
      // -- small lists get a larger prefix (fewer candidates after it)
      static const int pdiv = getenv("PQS_PREFIX_DIV") ? atoi(getenv("PQS_PREFIX_DIV")) : 4;  // tuning experiments
      static const int s0div = getenv("PQS_S0_DIV") ? atoi(getenv("PQS_S0_DIV")) : 2;
      st = std::max<int64_t>(cdiv(db->ntiles, ctx->sample_div), std::min<int64_t>(cdiv(db->ntiles, pdiv), 1024 / pdiv));
      st = std::min<int64_t>(std::max<int64_t>(st, tmin), db->ntiles);
      const int64_t s0 = std::min<int64_t>(std::max<int64_t>(cdiv(st, s0div), tmin), st);
      unsigned int* ghist = nullptr;
      PQS_TRY(scratch(ctx, S_IVF_WORK3, (size_t)(nq * 128), &ghist));
      PQS_CUDA(ctx, cudaMemsetAsync(ghist, 0, sizeof(unsigned int) * nq * 128, ctx->stream));
      // the histogram of the first s0 tiles: tcgen05 when the filter will run there
      const int64_t nh = std::min<int64_t>(s0 * TILE4, n);
      unsigned int pad1 = 0;
      int hrc = PQS_ERR_UNSUPPORTED;
      if (ctx->scan4_engine != 1 && cdiv(nq, 256) < ctx->sm_count) {
        hrc = launch_hist_tc(ctx, db, d_qt, nq, nh, ghist);
        if (hrc != PQS_OK && hrc != PQS_ERR_UNSUPPORTED) return hrc;
        if (hrc == PQS_OK) {
          pad1 = (unsigned int)(cdiv(nh, 256) * 256 - nh);
          b_built = true;
        }
      }
      if (hrc != PQS_OK) {
        Scan4Args a{};
        a.parts = 4;
        a.words = db->words4;
        a.n = n;
        a.m = m;
        a.qt = d_qt;
        a.nq = nq;
        a.nvt = s0;
        a.tile_off = 0;
        a.tile_step = 1;
        a.ghist = ghist;
        PQS_TRY(launch_scan4<MODE_HIST>(ctx, db->mp, a, nq));
      }
      theta4_final_kernel<<<(unsigned)cdiv(nq, 128), 128, 0, ctx->stream>>>(ghist, nq, (int)r_eff, pad1, theta);
      PQS_LAUNCHED(ctx);
    }

    // ---- K4 filtered scan
    PQS_TRY(scratch(ctx, S_CAND, (size_t)(nq * cap), &cand));
    PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)nq, &cnt));
    PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
    t1 = st > 0 ? st : db->ntiles;  // end of the first range
    second = st > 0 && st < db->ntiles;
    PQS_TRY(scratch(ctx, S_TC_OVF, 1, &d_ovf));
    PQS_CUDA(ctx, cudaMemsetAsync(d_ovf, 0, sizeof(int), ctx->stream));
    used_tc = false;
    PQS_TRY(scan_timer_begin(ctx));
    if (st > 0 && ctx->scan4_engine != 1) {
      // tcgen05 engine (128-code tiles); UNSUPPORTED for shapes outside it
      const int64_t nt128 = cdiv(n, 128);
      const int64_t p128 = std::min<int64_t>(t1 * (TILE4 / 128), nt128);
      int rc = launch_scan4_tc(ctx, db, d_qt, theta, nq, 0, p128, !b_built, cand, cnt, cap, d_ovf);
      if (rc == PQS_OK && second) {
        PQS_TRY(main_theta());
        rc = launch_scan4_tc(ctx, db, d_qt, theta_main, nq, p128, nt128, false, cand, cnt, cap, d_ovf);
      }
      if (rc == PQS_OK) {
        used_tc = true;
        ctx->last_scan_engine = 2;
        // int8 MMA ops issued: 2 x K per (query, code) over padded query groups and 128-code tiles
        const int qg = tc_query_group();
        ctx->last_scan_work = 2.0 * (double)cdiv(nq, qg) * qg * (double)nt128 * 128.0 * (double)tc_k_per_eval();
      } else if (rc == PQS_ERR_UNSUPPORTED) {
        if (ctx->scan4_engine == 2)
          return set_err(ctx, PQS_ERR_UNSUPPORTED, "tcgen05 Quick ADC scan: unsupported shape (needs m <= 16)");
        PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
      } else {
        return rc;
      }
    }
    if (!used_tc) PQS_TRY(scan_prmt());
    PQS_TRY(scan_timer_end(ctx));
    ctx->last_scan_launches = second ? 2 : 1;

    // ---- K5 select (bins, ties by id)
    uint64_t* gk = nullptr;
    int64_t* gi = nullptr;
    PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * cap), &gk));
    PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * cap), &gi));
    sel = SelArgs{};
    sel.src = SEL_CAND_BIN;
    sel.nq = nq;
    sel.r = r;
    sel.cand = cand;
    sel.cand_cnt = cnt;
    sel.cap = cap;
    sel.ids = db->ids;
    sel.id_base = db->id_base;
    sel.out_b = d_bins;
    sel.out_i = d_ids;
    sel.out_c = d_count;
    sel.gkeys = gk;
    sel.gids = gi;
    sel.gcap = cap;
    PQS_TRY(launch_select(ctx, sel));
    // candidate counts + the tcgen05 record-overflow flag into pinned host memory
    PQS_CUDA(ctx, cudaMemcpyAsync(ctx->h_cnt, cnt, sizeof(int) * nq, cudaMemcpyDeviceToHost, ctx->stream));
    PQS_CUDA(ctx, cudaMemcpyAsync(ctx->h_cnt + nq, d_ovf, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    return PQS_OK;
  }

  int host_phase() {
    const int* hcnt = ctx->h_cnt;
    if (used_tc && ctx->h_cnt[nq]) {  // a CTA record list overflowed: redo the scan on the PRMT engine
      PQS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int) * nq, ctx->stream));
      PQS_TRY(scan_timer_begin(ctx));
      PQS_TRY(scan_prmt());
      PQS_TRY(scan_timer_end(ctx));
      PQS_TRY(launch_select(ctx, sel));
      PQS_CUDA(ctx, cudaMemcpyAsync(ctx->h_cnt, cnt, sizeof(int) * nq, cudaMemcpyDeviceToHost, ctx->stream));
      PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    ctx->last_evals = nq * n;
    // ---- overflow check -> exact dense fallback for those queries
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
    ctx->last_overflow = (int64_t)over.size();
    if (!over.empty()) {
      const int64_t B =
          std::max<int64_t>(1, std::min<int64_t>((int64_t)over.size(), (int64_t)(1ll << 30) / std::max<int64_t>(n, 1)));
      int* d_qmap = nullptr;
      uint8_t* qt_sub = nullptr;
      uint8_t* dense = nullptr;
      PQS_TRY(scratch(ctx, S_MISC, (size_t)over.size(), &d_qmap));
      PQS_TRY(scratch(ctx, S_QTABLES, (size_t)(B * m * 16), &qt_sub));
      PQS_TRY(scratch(ctx, S_DENSE, (size_t)(B * n), &dense));
      PQS_CUDA(ctx, cudaMemcpyAsync(d_qmap, over.data(), sizeof(int) * over.size(), cudaMemcpyHostToDevice,
                                    ctx->stream));
      for (int64_t b0 = 0; b0 < (int64_t)over.size(); b0 += B) {
        const int64_t nb = std::min<int64_t>(B, (int64_t)over.size() - b0);
        gather_rows_u8_kernel<<<(unsigned)cdiv(nb * m * 16, 256), 256, 0, ctx->stream>>>(d_qt, d_qmap + b0, nb,
                                                                                       (int64_t)m * 16, qt_sub);
        PQS_LAUNCHED(ctx);
        PQS_TRY(launch_scan4_dense(ctx, db, qt_sub, nb, dense, n));
        SelArgs f{};
        f.src = SEL_DENSE_U8;
        f.nq = nb;
        f.r = r;
        f.dense = dense;
        f.n = n;
        f.ids = db->ids;
        f.id_base = db->id_base;
        f.qmap = d_qmap + b0;
        f.out_b = d_bins;
        f.out_i = d_ids;
        f.out_c = d_count;
        PQS_TRY(launch_select(ctx, f));
      }
    }
    return PQS_OK;
  }
};

}  // namespace

int run_qadc_topr(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, int init_count, int r,
                  uint8_t* d_bins, int64_t* d_ids, int32_t* d_count, uint8_t* d_qt, double* d_qmm) {
  // pinned landing buffer for the counts (+ overflow flag); growing it drops the graph
  if (ctx->h_cnt_cap < nq + 1) {
    if (ctx->h_cnt) {
      PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFreeHost(ctx->h_cnt);
      ctx->h_cnt = nullptr;
    }
    PQS_CUDA(ctx, cudaHostAlloc((void**)&ctx->h_cnt, sizeof(int) * (size_t)(nq + 1), cudaHostAllocDefault));
    ctx->h_cnt_cap = nq + 1;
    ctx->scratch_epoch++;
  }
  QadcRun run{ctx, db, d_tables, nq, init_count, r, d_bins, d_qt, d_ids, d_count, d_qmm};
  // db->gen is unique per handle and content version (never reused), so a graph
  // captured for a destroyed or re-prefixed list can never replay on another
  const std::vector<int64_t> key = {db->gen, db->n, (int64_t)(uintptr_t)db->prefix, db->n_prefix,
                                    (int64_t)(uintptr_t)d_tables, nq, init_count, r, ctx->cand_cap, ctx->sample_div,
                                    ctx->scan4_engine, ctx->tc_chunk_tiles, (int64_t)(uintptr_t)d_bins,
                                    (int64_t)(uintptr_t)d_ids, (int64_t)(uintptr_t)d_count, (int64_t)(uintptr_t)d_qt,
                                    (int64_t)(uintptr_t)d_qmm, (int64_t)(uintptr_t)ctx->h_cnt};
  static const bool no_graph = getenv("PQS_NO_GRAPH") != nullptr || getenv("PQS_TC_DEBUG") != nullptr;
  auto& g = ctx->qg;
  if (!no_graph && g.exec && g.key == key && g.epoch == ctx->scratch_epoch) {
    // replay: the plan is the captured one (it only depends on the key)
    PQS_CUDA(ctx, cudaGraphLaunch(g.exec, ctx->stream));
    ctx->launches += g.launches;
    run.n = db->n;
    run.m = db->m;
    run.cap = std::min<int64_t>(ctx->cand_cap, std::max<int64_t>(db->n, 1));
    run.r_eff = std::min<int64_t>(r, db->n);
    run.used_tc = g.used_tc != 0;
    run.second = g.second != 0;
    ctx->last_scan_engine = run.used_tc ? 2 : 1;
    ctx->last_scan_work = g.scan_work;
    ctx->last_scan_launches = run.second ? 2 : 1;
    // buffers for a possible host-phase redo (same scratch layout: the epoch matched)
    PQS_TRY(scratch(ctx, S_THETA, (size_t)(2 * nq), &run.theta));
    run.theta_main = run.theta + nq;
    PQS_TRY(scratch(ctx, S_CAND, (size_t)(nq * run.cap), &run.cand));
    PQS_TRY(scratch(ctx, S_CAND_CNT, (size_t)nq, &run.cnt));
    if (run.used_tc) {  // the PRMT redo needs the prefix split
      const int64_t tmin = cdiv(16 * run.r_eff, TILE4);
      static const int pdiv = getenv("PQS_PREFIX_DIV") ? atoi(getenv("PQS_PREFIX_DIV")) : 4;
      int64_t st = std::max<int64_t>(cdiv(db->ntiles, ctx->sample_div), std::min<int64_t>(cdiv(db->ntiles, pdiv), 1024 / pdiv));
      st = std::min<int64_t>(std::max<int64_t>(st, tmin), db->ntiles);
      run.st = run.n <= run.cap ? 0 : st;
      run.t1 = run.st > 0 ? run.st : db->ntiles;
      uint64_t* gk = nullptr;
      int64_t* gi = nullptr;
      PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * run.cap), &gk));
      PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * run.cap), &gi));
      run.sel.src = SEL_CAND_BIN;
      run.sel.nq = nq;
      run.sel.r = r;
      run.sel.cand = run.cand;
      run.sel.cand_cnt = run.cnt;
      run.sel.cap = run.cap;
      run.sel.ids = db->ids;
      run.sel.id_base = db->id_base;
      run.sel.out_b = d_bins;
      run.sel.out_i = d_ids;
      run.sel.out_c = d_count;
      run.sel.gkeys = gk;
      run.sel.gids = gi;
      run.sel.gcap = run.cap;
    }
  } else if (!no_graph && g.seen == key && g.epoch == ctx->scratch_epoch) {
    // second identical call (scratch already sized): capture the device phase on the
    // context's own stream and launch the graph on the caller's stream
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    cudaStream_t user = ctx->stream;
    PQS_CUDA(ctx, cudaStreamSynchronize(user));
    ctx->stream = ctx->own_stream;
    const int64_t l0 = ctx->launches, e0 = ctx->scratch_epoch;
    cudaGraph_t graph = nullptr;
    int rc = PQS_OK;
    if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      rc = PQS_ERR_CUDA;
    } else {
      rc = run.device_phase();
      const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
      if (rc == PQS_OK && ce != cudaSuccess) rc = PQS_ERR_CUDA;
    }
    ctx->stream = user;
    cudaGetLastError();
    if (rc == PQS_OK && graph && ctx->scratch_epoch == e0 &&
        cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess) {
      g.key = key;
      g.epoch = ctx->scratch_epoch;
      g.launches = ctx->launches - l0;
      g.used_tc = run.used_tc;
      g.second = run.second;
      g.scan_work = ctx->last_scan_work;
      if (graph) cudaGraphDestroy(graph);
      PQS_CUDA(ctx, cudaGraphLaunch(g.exec, ctx->stream));
    } else {  // not capturable here: run it directly (and do not try again for this key)
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      g.exec = nullptr;
      g.seen.clear();
      ctx->launches = l0;
      PQS_TRY(run.device_phase());
    }
  } else {
    PQS_TRY(run.device_phase());
    g.seen = key;
    g.epoch = ctx->scratch_epoch;
  }
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return run.host_phase();
}
