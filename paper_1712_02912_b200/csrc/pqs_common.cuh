// pqs_common.cuh -- shared types of libpqs.so (B200 / sm_100a ADC-scan engine).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/pqs.h"

// ---------------------------------------------------------------------------
// tile geometry (device layouts)
// ---------------------------------------------------------------------------
// scan8: codes are stored tile-transposed, TILE8 codes per tile, component
// major inside a tile: byte (t, j, c) at t*m*TILE8 + j*TILE8 + c.
constexpr int TILE8 = 1024;
// scan4: 4-code "quads"; one 32-bit word per (quad, component pair) holds the
// PRMT selectors of components 2p (low half) and 2p+1 (high half):
// selector nibble i = component value of code 4g+i.  TILE4 codes per tile.
constexpr int TILE4 = 1024;
constexpr int QUADS4 = TILE4 / 4;
constexpr int MAX_R = 4096;  // largest r the device select handles

// Query (or vector) rows as the caller passed them: float32 or float64.  The
// reference computes from float64(query) (ProductQuantizer.rotate,
// quantizer.py:85-89; query_ivf ivf.py:170), so every exact kernel reads
// the rows through at() in fp64; float32 input is widened exactly.
struct QVec {
  const void* p = nullptr;
  int f64 = 0;
  __host__ __device__ QVec offset(int64_t i) const {
    return QVec{f64 ? (const void*)((const double*)p + i) : (const void*)((const float*)p + i), f64};
  }
#ifdef __CUDACC__
  __device__ __forceinline__ double at(int64_t i) const {
    return f64 ? __ldg((const double*)p + i) : (double)__ldg((const float*)p + i);
  }
#endif
};

struct Scratch {
  void* p = nullptr;
  size_t cap = 0;
};

enum ScratchSlot {
  S_QUERIES = 0,
  S_TABLES,
  S_TABLES_T,   // scan8 table layout
  S_QTABLES,
  S_QMINMAX,
  S_THETA,
  S_AERR,
  S_CAND,
  S_CAND_CNT,
  S_SAMPLE,
  S_KEYS,
  S_IDS,
  S_OUT_D,
  S_OUT_I,
  S_OUT_C,
  S_OUT_B,
  S_PREFIX,
  S_FLAG,
  S_DENSE,
  S_PROBE,
  S_PROBE_D,
  S_IVF_WORK,
  S_IVF_WORK2,
  S_IVF_WORK3,
  S_MISC,
  S_WORK,     // dynamic work counters
  S_QT_WORK,  // quantized tables of a Quick ADC search
  S_TC_B, S_TC_TH, S_TC_REC, S_TC_RECCNT, S_TC_OVF,
  S_PIDS,     // compacted IVF candidates (then their exact keys)
  S_IVF_APX,  // IVF candidates' filter distances
  S_IVF_CNT2, // IVF compacted candidate counts
  S_QUERIES32,// float32 copy of float64 queries (probe GEMM operand)
  S_NSLOTS
};

struct pqs_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  std::string err;
  int64_t cand_cap = 32768;
  int sample_div = 32;
  int force_fallback = 0;
  int scan4_engine = 0;  // 0 auto (tcgen05 when possible), 1 PRMT, 2 tcgen05
  int scan8_engine = 0;  // 0 auto (packed when m <= 64), 1 u16 lane=query, 2 packed
  int ivf_engine = 0;    // 0 auto (packed list scan when the index has W tables), 1 float list scan, 2 packed
  int64_t tc_chunk_tiles = 0;  // tcgen05 scan: max 128-code tiles per launch (0 = auto)
  int64_t launches = 0;
  int64_t last_max_cand = 0;
  int64_t last_overflow = 0;
  int64_t last_evals = 0;
  int64_t last_scan_ns = 0;
  int64_t last_scan_launches = 0;
  int64_t last_cand_total = 0;
  int64_t last_rerank_total = 0;  // candidates left for the exact re-score after tightening
  int64_t last_scan_engine = 0;
  int64_t last_slot_evals = 0;    // IVF list scan: slot-evaluations incl. idle slots
  double last_scan_work = 0;
  cudaEvent_t scan_ev[2] = {nullptr, nullptr};
  Scratch scratch[S_NSLOTS];
  int64_t scratch_epoch = 0;  // bumped whenever a scratch slot is (re)allocated
  int* host_flag = nullptr;  // pinned
  // pinned host landing buffers of the per-query candidate counts (+ flags)
  int* h_cnt = nullptr;
  int64_t h_cnt_cap = 0;
  // captured Quick ADC search pipeline (CUDA graph), see run_qadc_topr
  struct QGraph {
    std::vector<int64_t> key, seen;
    cudaGraphExec_t exec = nullptr;
    int64_t epoch = -1;
    int64_t launches = 0;
    int used_tc = 0, second = 0;
    double scan_work = 0;
  } qg;
};

struct pqs_pq {
  int m = 0, b = 0, d = 0, k = 0, dsub = 0;
  float* books = nullptr;  // device (m, k, dsub)
};

// every pqs_db gets a process-unique generation number at creation and a new
// one whenever its device content changes (pqs_db_set_prefix): captured CUDA
// graphs are keyed on it, never on the (reusable) host address of the handle
inline int64_t next_db_generation() {
  static std::atomic<int64_t> g{0};
  return ++g;
}

struct pqs_db {
  int64_t gen = 0;        // next_db_generation() at create / prefix change
  int64_t n = 0;
  int m = 0, b = 0, k = 0;
  int mp = 0;             // b==4: padded component count (2,4,8,16,32)
  int max_code = 0;       // largest stored component value
  int64_t ntiles = 0;
  uint8_t* codes8 = nullptr;    // b==8 tile-transposed
  uint8_t* codes_rm = nullptr;  // b==8 row-major copy (n, m): exact re-score reads one row per candidate
  uint32_t* words4 = nullptr;   // b==4 quad words (ntiles*QUADS4, mp/2)
  int64_t* ids = nullptr;       // explicit ids or nullptr
  int64_t id_base = 0;
  uint8_t* prefix = nullptr;    // b==4: optional global prefix (n_prefix, m) row-major
  int64_t n_prefix = 0;
};

struct pqs_ivf {
  int64_t K = 0, n = 0;
  int m = 0, k = 0, d = 0, dsub = 0;
  float* coarse = nullptr;        // (K, d)
  float* gnorm = nullptr;         // (K,) ||c|| (fp32, for the probe error bound)
  float gmax = 0.f;               // max ||c||
  double* cnorm = nullptr;        // (K,) fp64 ||c||^2
  float* cnormf = nullptr;        // (K,) fp32 ||c||^2 (probe keys)
  float* vtab = nullptr;          // (n,) V = 2 sum_j <c_j, C_j[code_j]> per stored code
  float* vmax = nullptr;          // (1,) max |V|
  float* books = nullptr;         // (m, k, dsub)
  int64_t* offsets = nullptr;     // (K+1,) device
  std::vector<int64_t> h_offsets; // host copy
  uint8_t* codes = nullptr;       // (n, m) row-major, list order
  int64_t* ids = nullptr;         // (n,)
  int64_t max_list = 0;
  int* list_order = nullptr;      // (K,) list-scan order (cells grouped by nearest pivot) or null
  float* wtab = nullptr;          // (K, k*m) W_c[e*m + j] = 2 <c_j, C_j[e]> (packed list scan, m = 8, k = 256) or null
  float* wmax = nullptr;          // (1,) max |W|
  // probe GEMM (probe.cu): canonical tf32 B tiles of (-2c, ||c||^2 hi, lo),
  // 256 cells per tile, dpad = d + 2 rounded up to 8 (0: d + 2 > 256, exact probes)
  float* probe_b = nullptr;
  int probe_dpad = 0;
  int64_t probe_ntiles = 0;
};

// ---------------------------------------------------------------------------
// error helpers
// ---------------------------------------------------------------------------
int set_err(pqs_ctx* ctx, int code, const std::string& msg);

#define PQS_CUDA(ctx, call)                                                        \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_err((ctx), PQS_ERR_CUDA,                                          \
                     std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

#define PQS_LAUNCHED(ctx)                                                          \
  do {                                                                             \
    (ctx)->launches++;                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return set_err((ctx), PQS_ERR_CUDA,                                          \
                     std::string("kernel launch: ") + cudaGetErrorString(e_));     \
  } while (0)

#define PQS_CHECK(ctx, cond, msg)                                                  \
  do {                                                                             \
    if (!(cond)) return set_err((ctx), PQS_ERR_INVALID, (msg));                    \
  } while (0)

#define PQS_TRY(x)            \
  do {                        \
    int s_ = (x);             \
    if (s_ != PQS_OK) return s_; \
  } while (0)

int scratch_get(pqs_ctx* ctx, int slot, size_t bytes, void** out);
// CUDA events around the main scan kernel of a search (PQS_STAT_LAST_SCAN_NS)
int scan_timer_begin(pqs_ctx* ctx);
int scan_timer_end(pqs_ctx* ctx);
int scan_timer_collect(pqs_ctx* ctx);  // after a stream sync
// host <-> device copies ordered on the context stream and completed on return
int upload(pqs_ctx* ctx, void* dst, const void* src, size_t bytes);
int download(pqs_ctx* ctx, void* dst, const void* src, size_t bytes);
template <class T>
inline int scratch(pqs_ctx* ctx, int slot, size_t count, T** out) {
  void* p = nullptr;
  int s = scratch_get(ctx, slot, count * sizeof(T), &p);
  *out = (T*)p;
  return s;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
// Order-preserving map of a double to uint64 (total order of finite values,
// -0.0 and +0.0 kept distinct; ADC sums never produce -0.0).
__host__ __device__ inline uint64_t dkey(double d) {
  uint64_t b;
#ifdef __CUDA_ARCH__
  b = (uint64_t)__double_as_longlong(d);
#else
  memcpy(&b, &d, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double d;
#ifdef __CUDA_ARCH__
  d = __longlong_as_double((long long)b);
#else
  memcpy(&d, &b, 8);
#endif
  return d;
}
__host__ __device__ inline uint32_t fkey(float f) {
  uint32_t b;
#ifdef __CUDA_ARCH__
  b = __float_as_uint(f);
#else
  memcpy(&b, &f, 4);
#endif
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__host__ __device__ inline float fkey_inv(uint32_t k) {
  uint32_t b = (k >> 31) ? (k & 0x7FFFFFFFu) : ~k;
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(b);
#else
  memcpy(&f, &b, 4);
#endif
  return f;
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

#ifdef __CUDACC__
// fastscan.py:48-57 in fp64: 127 at or above qmax, else floor((v-qmin)*scale)
// clamped to [0, 126]; 0 everywhere when the span is empty.
__device__ __forceinline__ uint8_t quantize1(double v, double qmin, double qmax, double scale) {
  if (scale == 0.0) return 0;
  if (v >= qmax) return 127;
  double f = floor(__dmul_rn(__dsub_rn(v, qmin), scale));
  f = f < 0.0 ? 0.0 : (f > 126.0 ? 126.0 : f);
  return (uint8_t)f;
}
#endif

// ---------------------------------------------------------------------------
// launchers (defined in the .cu files)
// ---------------------------------------------------------------------------
// tables.cu
int launch_tables_exact(pqs_ctx* ctx, const pqs_pq* pq, QVec d_queries, int64_t nq, float* d_tables);
// scan8.cu
int launch_scan_distances(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq,
                          double* d_out);
int run_adc_topr(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, int r,
                 double* d_dist, int64_t* d_ids, int32_t* d_count);
// scan4.cu
int run_qadc_topr(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq,
                  int init_count, int r, uint8_t* d_bins, int64_t* d_ids, int32_t* d_count,
                  uint8_t* d_qtables_out, double* d_qminmax_out);
int launch_scan4_dense(pqs_ctx* ctx, const pqs_db* db, const uint8_t* d_qtables, int64_t nq,
                       uint8_t* d_out, int64_t ld_out);
// select.cu
enum SelSource {
  SEL_CAND_BIN = 0,   // candidates (bin<<32 | idx), key = bin
  SEL_CAND_ADC = 1,   // candidates idx, key = exact fp64 ADC (rerank)
  SEL_DENSE_F64 = 2,  // dense fp64 [q][n], key = value
  SEL_DENSE_U8 = 3,   // dense u8 [q][n], key = value
  SEL_MERGE = 4,      // G lists of (double, id)
  SEL_KEYS = 6        // precomputed keys (cand) and ids (pids) per candidate slot (IVF: ivf_rerank_kernel)
};
struct SelArgs {
  int src = 0;
  int64_t nq = 0;
  int r = 0;
  // candidates
  const uint64_t* cand = nullptr;
  const int* cand_cnt = nullptr;
  int64_t cap = 0;
  // dense
  const void* dense = nullptr;
  int64_t n = 0;
  // id mapping
  const int64_t* ids = nullptr;
  int64_t id_base = 0;
  // rerank (SEL_CAND_ADC)
  const float* tables = nullptr;  // (nq, m, k)
  const uint8_t* codes8 = nullptr;
  const uint8_t* codes_rm = nullptr;  // optional row-major codes (faster exact re-score)
  int m = 0, k = 0;
  // precomputed ids (SEL_KEYS; keys in cand)
  const int64_t* pids = nullptr;
  // merge
  int G = 0;
  int r_in = 0;
  const double* mdist = nullptr;
  const int64_t* mids = nullptr;
  const int32_t* mcnt = nullptr;
  // query subset: q_local -> q_global (nullptr = identity)
  const int* qmap = nullptr;
  // outputs
  double* out_d = nullptr;
  uint8_t* out_b = nullptr;
  int64_t* out_i = nullptr;
  int32_t* out_c = nullptr;
  // scratch for large selections (nq_blocks * cap)
  uint64_t* gkeys = nullptr;
  int64_t* gids = nullptr;
  int64_t gcap = 0;
};
int launch_select(pqs_ctx* ctx, const SelArgs& a);
// ivf.cu
// d_sub (optional): (nq, ma, nsub) float32 ||q_j - c_j||^2 per sub-space of the selected cells
int run_ivf_probe(pqs_ctx* ctx, const pqs_ivf* ivf, QVec d_queries, int64_t nq, int ma,
                  int64_t* d_cells, double* d_dist, float* d_sub = nullptr, int nsub = 0);
int run_ivf_search(pqs_ctx* ctx, const pqs_ivf* ivf, QVec d_queries, int64_t nq, int ma,
                   int r, double* d_dist, int64_t* d_ids, int32_t* d_count);
// fastscan.cu
int run_fastscan_checked(pqs_ctx* ctx, const pqs_db* db, const float* d_tables, int64_t nq, int64_t n_init,
                         int r, int64_t* d_checked);
// derived.cu
int run_derived_search(pqs_ctx* ctx, const pqs_db* db, const float* d_full, int k, const float* d_compact,
                       int64_t nq, int kbar, int r, int64_t r2, double* d_dist, int64_t* d_ids, int32_t* d_count);
int run_ivf_derived_search(pqs_ctx* ctx, const pqs_ivf* iv, const float* d_dbooks, int kbar, QVec d_queries,
                           int64_t nq, int ma, int r, int64_t r2, double* d_dist, int64_t* d_ids, int32_t* d_count);
// ivf_qadc.cu
int run_ivf_qadc_search(pqs_ctx* ctx, const pqs_ivf* ivf, QVec d_queries, int64_t nq, int ma,
                        int r, int init_count, double* d_dist, int64_t* d_ids, int32_t* d_count);
