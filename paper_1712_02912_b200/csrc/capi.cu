// capi.cu -- extern "C" entry points of libpqs.so (include/pqs.h).
//
// Host orchestration only: argument validation mirroring the reference's
// ValueError conditions, host<->device staging for PQS_IO_HOST calls, and the
// kernel pipelines in tables.cu / scan4.cu / scan8.cu / select.cu / ivf.cu.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "pqs_common.cuh"

int build_db4(pqs_ctx* ctx, pqs_db* db, const uint8_t* d_codes);
int build_db8(pqs_ctx* ctx, pqs_db* db, const uint8_t* d_codes);
int device_max_u8(pqs_ctx* ctx, const uint8_t* d, int64_t count, int* out);
int launch_unpack_nibbles(pqs_ctx* ctx, const uint8_t* d_packed, int64_t n, int m, uint8_t* d_out);
int launch_encode(pqs_ctx* ctx, const pqs_pq* pq, QVec d_x, int64_t n, const float* d_coarse,
                  const int64_t* d_cells, uint8_t* d_out);
int launch_quantize(pqs_ctx* ctx, double qmin, double qmax, const double* d_v, int64_t n, uint8_t* d_out);
int ivf_create_impl(pqs_ctx* ctx, const pqs_pq* pq, const float* coarse, int64_t K, const int64_t* list_sizes,
                    const uint8_t* codes, const int64_t* ids, int io, pqs_ivf** out);
void ivf_destroy_impl(pqs_ivf* ivf);
int coarse_index_create(pqs_ctx* ctx, const float* centroids, int64_t K, int d, pqs_ivf** out);

int set_err(pqs_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int scratch_get(pqs_ctx* ctx, int slot, size_t bytes, void** out) {
  Scratch& s = ctx->scratch[slot];
  if (bytes == 0) bytes = 16;
  if (s.cap < bytes) {
    if (s.p) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(s.p);
      s.p = nullptr;
      s.cap = 0;
    }
    size_t want = std::max(bytes, (size_t)(s.cap * 5 / 4));
    want = (want + 255) & ~(size_t)255;
    ctx->scratch_epoch++;
    cudaError_t e = cudaMalloc(&s.p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      s.p = nullptr;
      return set_err(ctx, PQS_ERR_NOMEM, std::string("scratch allocation failed: ") + cudaGetErrorString(e));
    }
    s.cap = want;
  }
  *out = s.p;
  return PQS_OK;
}

// inside a stream capture the record must be "external" to become an
// event-record node of the graph (a plain record only orders the capture)
static int record_timer(pqs_ctx* ctx, cudaEvent_t ev) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PQS_CUDA(ctx, cudaStreamIsCapturing(ctx->stream, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    PQS_CUDA(ctx, cudaEventRecordWithFlags(ev, ctx->stream, cudaEventRecordExternal));
  else
    PQS_CUDA(ctx, cudaEventRecord(ev, ctx->stream));
  return PQS_OK;
}

int scan_timer_begin(pqs_ctx* ctx) {
  if (!ctx->scan_ev[0]) {
    PQS_CUDA(ctx, cudaEventCreate(&ctx->scan_ev[0]));
    PQS_CUDA(ctx, cudaEventCreate(&ctx->scan_ev[1]));
  }
  return record_timer(ctx, ctx->scan_ev[0]);
}

int scan_timer_end(pqs_ctx* ctx) {
  return record_timer(ctx, ctx->scan_ev[1]);
}

int scan_timer_collect(pqs_ctx* ctx) {
  float ms = 0.f;
  PQS_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->scan_ev[0], ctx->scan_ev[1]));
  ctx->last_scan_ns = (int64_t)((double)ms * 1e6);
  return PQS_OK;
}

int upload(pqs_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PQS_OK;
}

int download(pqs_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PQS_OK;
}

namespace {

// input staging: device pointer as-is, host pointer copied into a scratch slot
template <class T>
int stage_in(pqs_ctx* ctx, int slot, const T* p, size_t count, int io, const T** out);

// query rows (float32 or float64, as the caller passed them) -> device QVec
int stage_q(pqs_ctx* ctx, const void* p, size_t count, int io, int f64, QVec* out) {
  out->f64 = f64;
  if (f64) {
    const double* d = nullptr;
    PQS_TRY(stage_in(ctx, S_QUERIES, (const double*)p, count, io, &d));
    out->p = d;
  } else {
    const float* d = nullptr;
    PQS_TRY(stage_in(ctx, S_QUERIES, (const float*)p, count, io, &d));
    out->p = d;
  }
  return PQS_OK;
}

template <class T>
int stage_in(pqs_ctx* ctx, int slot, const T* p, size_t count, int io, const T** out) {
  if (io == PQS_IO_DEVICE) {
    *out = p;
    return PQS_OK;
  }
  T* d = nullptr;
  PQS_TRY(scratch(ctx, slot, count, &d));
  if (count) PQS_CUDA(ctx, cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  *out = d;
  return PQS_OK;
}

template <class T>
int stage_out(pqs_ctx* ctx, int slot, T* p, size_t count, int io, T** out) {
  if (io == PQS_IO_DEVICE || p == nullptr) {
    *out = p;
    if (p == nullptr && count) {
      T* d = nullptr;
      PQS_TRY(scratch(ctx, slot, count, &d));
      *out = d;
    }
    return PQS_OK;
  }
  T* d = nullptr;
  PQS_TRY(scratch(ctx, slot, count, &d));
  *out = d;
  return PQS_OK;
}

template <class T>
int copy_out(pqs_ctx* ctx, T* host, const T* dev, size_t count, int io) {
  if (io == PQS_IO_DEVICE || host == nullptr || count == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  return PQS_OK;
}

// copy a scratch result to the caller's buffer (host or device)
template <class T>
int copy_any(pqs_ctx* ctx, T* dst, const T* dev, size_t count, int io) {
  if (dst == nullptr || count == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaMemcpyAsync(dst, dev, count * sizeof(T),
                                io == PQS_IO_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
  return PQS_OK;
}

int finish(pqs_ctx* ctx, int io) {
  if (io == PQS_IO_HOST) PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PQS_OK;
}

int check_io(pqs_ctx* ctx, int io) {
  PQS_CHECK(ctx, io == PQS_IO_HOST || io == PQS_IO_DEVICE, "io must be PQS_IO_HOST or PQS_IO_DEVICE");
  return PQS_OK;
}

}  // namespace

extern "C" {

int pqs_api_version(void) { return PQS_API_VERSION; }

int pqs_ctx_create(int device, pqs_ctx** out) {
  if (!out) return PQS_ERR_INVALID;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return PQS_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) return PQS_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return PQS_ERR_CUDA;
  pqs_ctx* ctx = new pqs_ctx();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return PQS_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  *out = ctx;
  return PQS_OK;
}

void pqs_ctx_destroy(pqs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& s : ctx->scratch)
    if (s.p) cudaFree(s.p);
  if (ctx->qg.exec) cudaGraphExecDestroy(ctx->qg.exec);
  if (ctx->h_cnt) cudaFreeHost(ctx->h_cnt);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  for (auto& e : ctx->scan_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
}

int pqs_ctx_set_stream(pqs_ctx* ctx, void* stream) {
  if (!ctx) return PQS_ERR_INVALID;
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return PQS_OK;
}

int pqs_ctx_synchronize(pqs_ctx* ctx) {
  if (!ctx) return PQS_ERR_INVALID;
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return PQS_OK;
}

int pqs_ctx_set_option(pqs_ctx* ctx, int option, int64_t value) {
  if (!ctx) return PQS_ERR_INVALID;
  switch (option) {
    case PQS_OPT_CAND_CAP:
      PQS_CHECK(ctx, value >= 1 && value <= (1ll << 30), "candidate capacity out of range");
      ctx->cand_cap = value;
      return PQS_OK;
    case PQS_OPT_SAMPLE_DIV:
      PQS_CHECK(ctx, value >= 1, "sample divisor must be >= 1");
      ctx->sample_div = (int)value;
      return PQS_OK;
    case PQS_OPT_FORCE_FALLBACK:
      ctx->force_fallback = value ? 1 : 0;
      return PQS_OK;
    case PQS_OPT_SCAN4_ENGINE:
      PQS_CHECK(ctx, value >= 0 && value <= 2, "scan4 engine must be 0, 1 or 2");
      ctx->scan4_engine = (int)value;
      return PQS_OK;
    case PQS_OPT_SCAN8_ENGINE:
      PQS_CHECK(ctx, value >= 0 && value <= 2, "scan8 engine must be 0, 1 or 2");
      ctx->scan8_engine = (int)value;
      return PQS_OK;
    case PQS_OPT_IVF_ENGINE:
      PQS_CHECK(ctx, value >= 0 && value <= 2, "ivf engine must be 0, 1 or 2");
      ctx->ivf_engine = (int)value;
      return PQS_OK;
    case PQS_OPT_TC_CHUNK_TILES:
      PQS_CHECK(ctx, value >= 0, "chunk must be >= 0");
      ctx->tc_chunk_tiles = value;
      return PQS_OK;
  }
  return set_err(ctx, PQS_ERR_INVALID, "unknown option");
}

int pqs_ctx_get_stat(pqs_ctx* ctx, int stat, int64_t* out) {
  if (!ctx || !out) return PQS_ERR_INVALID;
  switch (stat) {
    case PQS_STAT_LAUNCHES: *out = ctx->launches; return PQS_OK;
    case PQS_STAT_LAST_MAX_CAND: *out = ctx->last_max_cand; return PQS_OK;
    case PQS_STAT_LAST_OVERFLOW: *out = ctx->last_overflow; return PQS_OK;
    case PQS_STAT_LAST_EVALS: *out = ctx->last_evals; return PQS_OK;
    case PQS_STAT_LAST_SCAN_NS: *out = ctx->last_scan_ns; return PQS_OK;
    case PQS_STAT_LAST_SCAN_LAUNCHES: *out = ctx->last_scan_launches; return PQS_OK;
    case PQS_STAT_LAST_CAND_TOTAL: *out = ctx->last_cand_total; return PQS_OK;
    case PQS_STAT_LAST_SCAN_ENGINE: *out = ctx->last_scan_engine; return PQS_OK;
    case PQS_STAT_LAST_SCAN_WORK: *out = (int64_t)ctx->last_scan_work; return PQS_OK;
    case PQS_STAT_LAST_RERANK_TOTAL: *out = ctx->last_rerank_total; return PQS_OK;
    case PQS_STAT_LAST_SLOT_EVALS: *out = ctx->last_slot_evals; return PQS_OK;
  }
  return set_err(ctx, PQS_ERR_INVALID, "unknown stat");
}

const char* pqs_last_error(const pqs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// ---------------------------------------------------------------- quantizer
int pqs_pq_create(pqs_ctx* ctx, int m, int b, int d, const float* codebooks, pqs_pq** out) {
  if (!ctx || !out) return PQS_ERR_INVALID;
  *out = nullptr;
  PQS_CHECK(ctx, m >= 1 && d >= 1 && d % m == 0, "d not divisible by m");
  PQS_CHECK(ctx, b >= 1 && b <= 8, "b must be in [1, 8] for the device quantizer");
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  pqs_pq* pq = new pqs_pq();
  pq->m = m;
  pq->b = b;
  pq->d = d;
  pq->k = 1 << b;
  pq->dsub = d / m;
  const size_t bytes = (size_t)m * pq->k * pq->dsub * sizeof(float);
  if (cudaMalloc(&pq->books, bytes) != cudaSuccess) {
    cudaGetLastError();
    delete pq;
    return set_err(ctx, PQS_ERR_NOMEM, "codebook allocation failed");
  }
  PQS_TRY(upload(ctx, pq->books, codebooks, bytes));
  *out = pq;
  return PQS_OK;
}

void pqs_pq_destroy(pqs_pq* pq) {
  if (!pq) return;
  cudaFree(pq->books);
  delete pq;
}

// ---------------------------------------------------------------- code lists
int pqs_db_create(pqs_ctx* ctx, const uint8_t* codes, int64_t n, int m, int b, const int64_t* ids, int64_t id_base,
                  int io, pqs_db** out) {
  if (!ctx || !out) return PQS_ERR_INVALID;
  *out = nullptr;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, n >= 0, "n must be >= 0");
  PQS_CHECK(ctx, m >= 1, "m must be >= 1");
  PQS_CHECK(ctx, n < (1ll << 32), "a device code list holds at most 2^32 - 1 codes (shard larger lists)");
  PQS_CHECK(ctx, b == 4 || b == 8, "device code lists support b = 4 (Quick ADC) or b = 8 (float ADC)");
  if (b == 4) {
    PQS_CHECK(ctx, m % 2 == 0, "b=4 transposition needs even m");
    PQS_CHECK(ctx, m <= 32, "Quick ADC device layout supports m <= 32");
  }
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  // codes on the device (caller's pointer or a temporary copy)
  uint8_t* tmp = nullptr;
  const uint8_t* d_codes = codes;
  if (io == PQS_IO_HOST && n) {
    if (cudaMalloc(&tmp, (size_t)n * m) != cudaSuccess) {
      cudaGetLastError();
      return set_err(ctx, PQS_ERR_NOMEM, "staging allocation failed");
    }
    d_codes = tmp;
    const int s = upload(ctx, tmp, codes, (size_t)n * m);
    if (s != PQS_OK) {
      cudaFree(tmp);
      return s;
    }
  }
  pqs_db* db = new pqs_db();
  db->gen = next_db_generation();
  auto fail = [&](int code, const std::string& msg) {
    cudaStreamSynchronize(ctx->stream);
    if (tmp) cudaFree(tmp);
    if (db->codes8) cudaFree(db->codes8);
    if (db->codes_rm) cudaFree(db->codes_rm);
    if (db->words4) cudaFree(db->words4);
    if (db->ids) cudaFree(db->ids);
    delete db;
    cudaGetLastError();
    return set_err(ctx, code, msg);
  };
  int maxc = 0;
  if (n && device_max_u8(ctx, d_codes, n * m, &maxc) != PQS_OK) return fail(PQS_ERR_CUDA, ctx->err);
  if (b == 4 && maxc >= 16) return fail(PQS_ERR_INVALID, "component out of range for b=4");
  db->n = n;
  db->m = m;
  db->b = b;
  db->k = b == 4 ? 16 : 256;
  db->max_code = maxc;
  db->id_base = id_base;
  if (b == 8) {
    db->ntiles = cdiv(n, TILE8);
    if (db->ntiles) {
      if (cudaMalloc(&db->codes8, (size_t)db->ntiles * m * TILE8) != cudaSuccess)
        return fail(PQS_ERR_NOMEM, "code allocation failed");
      const int s = build_db8(ctx, db, d_codes);
      if (s != PQS_OK) return fail(s, ctx->err);
      if (cudaMalloc(&db->codes_rm, (size_t)n * m) != cudaSuccess) return fail(PQS_ERR_NOMEM, "code allocation failed");
      if (cudaMemcpyAsync(db->codes_rm, d_codes, (size_t)n * m, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
        return fail(PQS_ERR_CUDA, "code copy failed");
    }
  } else {
    int mp = 2;
    while (mp < m) mp <<= 1;
    db->mp = mp;
    db->ntiles = cdiv(n, TILE4);
    if (db->ntiles) {
      const size_t words = (size_t)db->ntiles * QUADS4 * (mp / 2);
      if (cudaMalloc(&db->words4, words * 4) != cudaSuccess) return fail(PQS_ERR_NOMEM, "code allocation failed");
      const int s = build_db4(ctx, db, d_codes);
      if (s != PQS_OK) return fail(s, ctx->err);
    }
  }
  if (ids && n) {
    if (cudaMalloc(&db->ids, (size_t)n * 8) != cudaSuccess) return fail(PQS_ERR_NOMEM, "id allocation failed");
    if (upload(ctx, db->ids, ids, (size_t)n * 8) != PQS_OK) return fail(PQS_ERR_CUDA, "id upload failed");
  }
  PQS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (tmp) cudaFree(tmp);
  *out = db;
  return PQS_OK;
}

// code list straight from a PQL1 payload (scan.py:290-359): b_file <= 4 ->
// nibble-packed (m+1)/2 bytes per code, unpacked on the device; 4 < b_file <= 8
// -> one byte per component.  layout_b selects the device layout (4 or 8).
int pqs_db_create_packed(pqs_ctx* ctx, const uint8_t* payload, int64_t n, int m, int b_file, int layout_b,
                         const int64_t* ids, int64_t id_base, int io, pqs_db** out) {
  if (!ctx || !out) return PQS_ERR_INVALID;
  *out = nullptr;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, n >= 0 && m >= 1, "bad code list shape");
  PQS_CHECK(ctx, b_file >= 1 && b_file <= 8, "device code lists hold b <= 8 components");
  if (b_file > 4) return pqs_db_create(ctx, payload, n, m, layout_b, ids, id_base, io, out);
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t pbytes = (size_t)n * ((m + 1) / 2);
  uint8_t* dp = nullptr;
  uint8_t* dc = nullptr;
  if (cudaMalloc(&dc, std::max<size_t>((size_t)n * m, 16)) != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, PQS_ERR_NOMEM, "unpack allocation failed");
  }
  const uint8_t* src = payload;
  if (io == PQS_IO_HOST && pbytes) {
    if (cudaMalloc(&dp, pbytes) != cudaSuccess) {
      cudaFree(dc);
      cudaGetLastError();
      return set_err(ctx, PQS_ERR_NOMEM, "staging allocation failed");
    }
    int st = upload(ctx, dp, payload, pbytes);
    if (st != PQS_OK) {
      cudaFree(dp);
      cudaFree(dc);
      return st;
    }
    src = dp;
  }
  int st = launch_unpack_nibbles(ctx, src, n, m, dc);
  // ids follow the caller's io; codes are now on the device
  if (st == PQS_OK && io == PQS_IO_HOST && ids && n) {
    // pqs_db_create takes one io for codes and ids: stage the ids too
    int64_t* di = nullptr;
    if (cudaMalloc(&di, (size_t)n * 8) != cudaSuccess) {
      st = set_err(ctx, PQS_ERR_NOMEM, "id staging failed");
    } else {
      st = upload(ctx, di, ids, (size_t)n * 8);
      if (st == PQS_OK) st = pqs_db_create(ctx, dc, n, m, layout_b, di, id_base, PQS_IO_DEVICE, out);
      cudaStreamSynchronize(ctx->stream);
      cudaFree(di);
    }
  } else if (st == PQS_OK) {
    st = pqs_db_create(ctx, dc, n, m, layout_b, ids, id_base, PQS_IO_DEVICE, out);
  }
  cudaStreamSynchronize(ctx->stream);
  if (dp) cudaFree(dp);
  cudaFree(dc);
  return st;
}

int pqs_db_set_prefix(pqs_ctx* ctx, pqs_db* db, const uint8_t* prefix, int64_t n_prefix, int io) {
  if (!ctx || !db) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, db->b == 4, "a global prefix applies to Quick ADC (b=4) lists");
  PQS_CHECK(ctx, n_prefix >= 1, "prefix must hold at least one code");
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  if (db->prefix) cudaFree(db->prefix);
  db->prefix = nullptr;
  db->n_prefix = 0;
  db->gen = next_db_generation();
  PQS_CUDA(ctx, cudaMalloc(&db->prefix, (size_t)n_prefix * db->m));
  PQS_TRY(upload(ctx, db->prefix, prefix, (size_t)n_prefix * db->m));
  int maxc = 0;
  PQS_TRY(device_max_u8(ctx, db->prefix, n_prefix * db->m, &maxc));
  if (maxc >= 16) {
    cudaFree(db->prefix);
    db->prefix = nullptr;
    return set_err(ctx, PQS_ERR_INVALID, "component out of range for b=4");
  }
  db->n_prefix = n_prefix;
  db->gen = next_db_generation();
  return PQS_OK;
}

void pqs_db_destroy(pqs_db* db) {
  if (!db) return;
  db->gen = -1;
  if (db->codes8) cudaFree(db->codes8);
  if (db->codes_rm) cudaFree(db->codes_rm);
  if (db->words4) cudaFree(db->words4);
  if (db->ids) cudaFree(db->ids);
  if (db->prefix) cudaFree(db->prefix);
  delete db;
}

// ---------------------------------------------------------------- tables
static int compute_tables_impl(pqs_ctx* ctx, const pqs_pq* pq, const void* queries, int f64, int64_t nq,
                               float* out_tables, int io) {
  if (!ctx || !pq) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, nq >= 0, "nq must be >= 0");
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  float* dt = nullptr;
  const size_t tcount = (size_t)nq * pq->m * pq->k;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * pq->d, io, f64, &dq));
  PQS_TRY(stage_out(ctx, S_TABLES, out_tables, tcount, io, &dt));
  PQS_TRY(launch_tables_exact(ctx, pq, dq, nq, dt));
  PQS_TRY(copy_out(ctx, out_tables, dt, tcount, io));
  return finish(ctx, io);
}
int pqs_compute_tables(pqs_ctx* ctx, const pqs_pq* pq, const float* queries, int64_t nq, float* out_tables, int io) {
  return compute_tables_impl(ctx, pq, queries, 0, nq, out_tables, io);
}
int pqs_compute_tables_f64(pqs_ctx* ctx, const pqs_pq* pq, const double* queries, int64_t nq, float* out_tables,
                           int io) {
  return compute_tables_impl(ctx, pq, queries, 1, nq, out_tables, io);
}

// ---------------------------------------------------------------- float ADC
int pqs_scan_distances(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq, int k, double* out, int io) {
  if (!ctx || !db) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, db->b == 8, "scan_distances needs a b=8 code list");
  PQS_CHECK(ctx, k >= 1 && k <= 256, "device tables support k <= 256");
  PQS_CHECK(ctx, db->n == 0 || db->max_code < k, "code component out of range for the tables");
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  pqs_db dbk = *db;
  dbk.k = k;
  const float* dt = nullptr;
  double* dout = nullptr;
  PQS_TRY(stage_in(ctx, S_TABLES, tables, (size_t)nq * db->m * k, io, &dt));
  PQS_TRY(stage_out(ctx, S_DENSE, out, (size_t)nq * db->n, io, &dout));
  PQS_TRY(launch_scan_distances(ctx, &dbk, dt, nq, dout));
  PQS_TRY(copy_out(ctx, out, dout, (size_t)nq * db->n, io));
  return finish(ctx, io);
}

static int adc_common(pqs_ctx* ctx, const pqs_db* db, const float* dt, int64_t nq, int k, int r, double* out_dist,
                      int64_t* out_ids, int32_t* out_count, int io) {
  pqs_db dbk = *db;
  dbk.k = k;
  double* dd = nullptr;
  int64_t* di = nullptr;
  int32_t* dc = nullptr;
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * r, io, &dd));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_ids, (size_t)nq * r, io, &di));
  PQS_TRY(stage_out(ctx, S_OUT_C, out_count, (size_t)nq, io, &dc));
  PQS_TRY(run_adc_topr(ctx, &dbk, dt, nq, r, dd, di, dc));
  PQS_TRY(copy_out(ctx, out_dist, dd, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_ids, di, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_count, dc, (size_t)nq, io));
  return finish(ctx, io);
}

int pqs_adc_scan(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq, int k, int r, double* out_dist,
                 int64_t* out_ids, int32_t* out_count, int io) {
  if (!ctx || !db) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, db->b == 8, "scan needs a b=8 code list");
  PQS_CHECK(ctx, k >= 1 && k <= 256, "device tables support k <= 256");
  PQS_CHECK(ctx, db->n == 0 || db->max_code < k, "code component out of range for the tables");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const float* dt = nullptr;
  PQS_TRY(stage_in(ctx, S_TABLES, tables, (size_t)nq * db->m * k, io, &dt));
  return adc_common(ctx, db, dt, nq, k, r, out_dist, out_ids, out_count, io);
}

static int adc_search_impl(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const void* queries, int f64, int64_t nq,
                           int r, double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  if (!ctx || !db || !pq) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, db->b == 8, "scan needs a b=8 code list");
  PQS_CHECK(ctx, pq->m == db->m, "quantizer m does not match the code list");
  PQS_CHECK(ctx, db->n == 0 || db->max_code < pq->k, "code component out of range for the quantizer");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  float* dt = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * pq->d, io, f64, &dq));
  PQS_TRY(scratch(ctx, S_TABLES, (size_t)nq * pq->m * pq->k, &dt));
  PQS_TRY(launch_tables_exact(ctx, pq, dq, nq, dt));
  return adc_common(ctx, db, dt, nq, pq->k, r, out_dist, out_ids, out_count, io);
}
int pqs_adc_search(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const float* queries, int64_t nq, int r,
                   double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  return adc_search_impl(ctx, db, pq, queries, 0, nq, r, out_dist, out_ids, out_count, io);
}
int pqs_adc_search_f64(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const double* queries, int64_t nq, int r,
                       double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  return adc_search_impl(ctx, db, pq, queries, 1, nq, r, out_dist, out_ids, out_count, io);
}

// ---------------------------------------------------------------- Quick ADC
static int qadc_common(pqs_ctx* ctx, const pqs_db* db, const float* dt, int64_t nq, int init_count, int r,
                       uint8_t* out_bins, int64_t* out_ids, int32_t* out_count, uint8_t* out_qt, double* out_qmm,
                       int io) {
  // results land in the context's scratch (stable addresses: the device phase
  // is replayed as a CUDA graph, see run_qadc_topr) and are copied out
  uint8_t* db_ = nullptr;
  int64_t* di = nullptr;
  int32_t* dc = nullptr;
  uint8_t* qt_work = nullptr;
  double* dqmm = nullptr;
  PQS_TRY(scratch(ctx, S_OUT_B, (size_t)nq * r, &db_));
  PQS_TRY(scratch(ctx, S_OUT_I, (size_t)nq * r, &di));
  PQS_TRY(scratch(ctx, S_OUT_C, (size_t)nq, &dc));
  PQS_TRY(scratch(ctx, S_QT_WORK, (size_t)nq * db->m * 16, &qt_work));
  PQS_TRY(scratch(ctx, S_QMINMAX, (size_t)nq * 2, &dqmm));
  PQS_TRY(run_qadc_topr(ctx, db, dt, nq, init_count, r, db_, di, dc, qt_work, dqmm));
  PQS_TRY(copy_any(ctx, out_bins, db_, (size_t)nq * r, io));
  PQS_TRY(copy_any(ctx, out_ids, di, (size_t)nq * r, io));
  PQS_TRY(copy_any(ctx, out_count, dc, (size_t)nq, io));
  PQS_TRY(copy_any(ctx, out_qt, (const uint8_t*)qt_work, (size_t)nq * db->m * 16, io));
  PQS_TRY(copy_any(ctx, out_qmm, dqmm, (size_t)nq * 2, io));
  return finish(ctx, io);
}

static int qadc_validate(pqs_ctx* ctx, const pqs_db* db, int init_count, int r) {
  PQS_CHECK(ctx, db->b == 4, "quick scan requires 4-bit codes");
  PQS_CHECK(ctx, db->m % 2 == 0, "quick scan needs even m");
  PQS_CHECK(ctx, init_count >= 1, "init_count must be >= 1");
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, db->n > 0, "empty code list");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  return PQS_OK;
}

int pqs_qadc_scan(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq, int init_count, int r,
                  uint8_t* out_bins, int64_t* out_ids, int32_t* out_count, uint8_t* out_qt, double* out_qmm, int io) {
  if (!ctx || !db) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_TRY(qadc_validate(ctx, db, init_count, r));
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const float* dt = nullptr;
  PQS_TRY(stage_in(ctx, S_TABLES, tables, (size_t)nq * db->m * 16, io, &dt));
  return qadc_common(ctx, db, dt, nq, init_count, r, out_bins, out_ids, out_count, out_qt, out_qmm, io);
}

static int qadc_search_impl(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const void* queries, int f64,
                            int64_t nq, int init_count, int r, uint8_t* out_bins, int64_t* out_ids,
                            int32_t* out_count, uint8_t* out_qt, double* out_qmm, int io) {
  if (!ctx || !db || !pq) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_TRY(qadc_validate(ctx, db, init_count, r));
  PQS_CHECK(ctx, pq->k == 16 && pq->m == db->m, "tables do not match the code list shape");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  float* dt = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * pq->d, io, f64, &dq));
  PQS_TRY(scratch(ctx, S_TABLES, (size_t)nq * pq->m * 16, &dt));
  PQS_TRY(launch_tables_exact(ctx, pq, dq, nq, dt));
  return qadc_common(ctx, db, dt, nq, init_count, r, out_bins, out_ids, out_count, out_qt, out_qmm, io);
}
int pqs_qadc_search(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const float* queries, int64_t nq,
                    int init_count, int r, uint8_t* out_bins, int64_t* out_ids, int32_t* out_count, uint8_t* out_qt,
                    double* out_qmm, int io) {
  return qadc_search_impl(ctx, db, pq, queries, 0, nq, init_count, r, out_bins, out_ids, out_count, out_qt, out_qmm,
                          io);
}
int pqs_qadc_search_f64(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const double* queries, int64_t nq,
                        int init_count, int r, uint8_t* out_bins, int64_t* out_ids, int32_t* out_count,
                        uint8_t* out_qt, double* out_qmm, int io) {
  return qadc_search_impl(ctx, db, pq, queries, 1, nq, init_count, r, out_bins, out_ids, out_count, out_qt, out_qmm,
                          io);
}

int pqs_quantize(pqs_ctx* ctx, double qmin, double qmax, const double* values, int64_t n, uint8_t* out, int io) {
  if (!ctx) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, std::isfinite(qmin) && std::isfinite(qmax), "quantization bounds must be finite");
  PQS_CHECK(ctx, qmax >= qmin, "qmax must be >= qmin");
  if (n == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const double* dv = nullptr;
  uint8_t* dout = nullptr;
  PQS_TRY(stage_in(ctx, S_MISC, values, (size_t)n, io, &dv));
  PQS_TRY(stage_out(ctx, S_DENSE, out, (size_t)n, io, &dout));
  PQS_TRY(launch_quantize(ctx, qmin, qmax, dv, n, dout));
  PQS_TRY(copy_out(ctx, out, dout, (size_t)n, io));
  return finish(ctx, io);
}

int pqs_quantized_distances(pqs_ctx* ctx, const pqs_db* db, const uint8_t* qtables, int64_t nq, uint8_t* out, int io) {
  if (!ctx || !db) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, db->b == 4, "quantized distances need a b=4 code list");
  if (nq == 0 || db->n == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const uint8_t* dqt = nullptr;
  uint8_t* dout = nullptr;
  PQS_TRY(stage_in(ctx, S_QTABLES, qtables, (size_t)nq * db->m * 16, io, &dqt));
  PQS_TRY(stage_out(ctx, S_DENSE, out, (size_t)nq * db->n, io, &dout));
  PQS_TRY(launch_scan4_dense(ctx, db, dqt, nq, dout, db->n));
  PQS_TRY(copy_out(ctx, out, dout, (size_t)nq * db->n, io));
  return finish(ctx, io);
}

// ---------------------------------------------------------------- IVF
int pqs_ivf_create(pqs_ctx* ctx, const pqs_pq* pq, const float* coarse, int64_t K, const int64_t* list_sizes,
                   const uint8_t* codes, const int64_t* ids, int io, pqs_ivf** out) {
  if (!ctx || !pq || !out) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  return ivf_create_impl(ctx, pq, coarse, K, list_sizes, codes, ids, io, out);
}

// ---------------------------------------------------------------- encode
static int encode_impl(pqs_ctx* ctx, const pqs_pq* pq, const void* x, int f64, int64_t n, const float* coarse,
                       int64_t K, const int64_t* cells, uint8_t* out_codes, int io) {
  if (!ctx || !pq) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, n >= 0, "n must be >= 0");
  PQS_CHECK(ctx, pq->k <= 256, "device encode supports b <= 8 (uint8 codes)");
  PQS_CHECK(ctx, (coarse == nullptr) == (cells == nullptr), "coarse and cells go together");
  PQS_CHECK(ctx, coarse == nullptr || K >= 1, "K must be >= 1");
  if (n == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dx;
  const float* dg = nullptr;
  const int64_t* dc = nullptr;
  uint8_t* dout = nullptr;
  PQS_TRY(stage_q(ctx, x, (size_t)n * pq->d, io, f64, &dx));
  if (coarse) {
    PQS_TRY(stage_in(ctx, S_IVF_WORK, coarse, (size_t)K * pq->d, io, &dg));
    PQS_TRY(stage_in(ctx, S_PROBE, cells, (size_t)n, io, &dc));
  }
  PQS_TRY(stage_out(ctx, S_OUT_B, out_codes, (size_t)n * pq->m, io, &dout));
  PQS_TRY(launch_encode(ctx, pq, dx, n, dg, dc, dout));
  PQS_TRY(copy_out(ctx, out_codes, dout, (size_t)n * pq->m, io));
  return finish(ctx, io);
}
int pqs_encode(pqs_ctx* ctx, const pqs_pq* pq, const float* x, int64_t n, const float* coarse, int64_t K,
               const int64_t* cells, uint8_t* out_codes, int io) {
  return encode_impl(ctx, pq, x, 0, n, coarse, K, cells, out_codes, io);
}
int pqs_encode_f64(pqs_ctx* ctx, const pqs_pq* pq, const double* x, int64_t n, const float* coarse, int64_t K,
                   const int64_t* cells, uint8_t* out_codes, int io) {
  return encode_impl(ctx, pq, x, 1, n, coarse, K, cells, out_codes, io);
}

void pqs_ivf_destroy(pqs_ivf* ivf) { ivf_destroy_impl(ivf); }

static int ivf_probe_impl(pqs_ctx* ctx, const pqs_ivf* ivf, const void* queries, int f64, int64_t nq, int ma,
                          int64_t* out_cells, double* out_dist, int io) {
  if (!ctx || !ivf) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, ma >= 1 && ma <= ivf->K, "ma must be in [1, K]");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  int64_t* dc = nullptr;
  double* dd = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * ivf->d, io, f64, &dq));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_cells, (size_t)nq * ma, io, &dc));
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * ma, io, &dd));
  PQS_TRY(run_ivf_probe(ctx, ivf, dq, nq, ma, dc, dd));
  PQS_TRY(copy_out(ctx, out_cells, dc, (size_t)nq * ma, io));
  PQS_TRY(copy_out(ctx, out_dist, dd, (size_t)nq * ma, io));
  return finish(ctx, io);
}
int pqs_ivf_probe(pqs_ctx* ctx, const pqs_ivf* ivf, const float* queries, int64_t nq, int ma, int64_t* out_cells,
                  double* out_dist, int io) {
  return ivf_probe_impl(ctx, ivf, queries, 0, nq, ma, out_cells, out_dist, io);
}
int pqs_ivf_probe_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const double* queries, int64_t nq, int ma,
                      int64_t* out_cells, double* out_dist, int io) {
  return ivf_probe_impl(ctx, ivf, queries, 1, nq, ma, out_cells, out_dist, io);
}

// nearest (_dist.py:24-39): the probe with ma = 1 over a coarse-only handle
static int nearest_impl(pqs_ctx* ctx, const float* centroids, int64_t K, int d, const void* points, int f64,
                        int64_t n, int64_t* out_idx, double* out_dist, int io) {
  if (!ctx || !centroids || !out_idx) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, n >= 0, "n must be >= 0");
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  pqs_ivf* iv = nullptr;
  PQS_TRY(coarse_index_create(ctx, centroids, K, d, &iv));
  int st = PQS_OK;
  if (n > 0) {
    QVec dq;
    int64_t* dc = nullptr;
    double* dd = nullptr;
    st = stage_q(ctx, points, (size_t)n * d, io, f64, &dq);
    if (st == PQS_OK) st = stage_out(ctx, S_OUT_I, out_idx, (size_t)n, io, &dc);
    if (st == PQS_OK) st = stage_out(ctx, S_OUT_D, out_dist, (size_t)n, io, &dd);
    if (st == PQS_OK) st = run_ivf_probe(ctx, iv, dq, n, 1, dc, dd);
    if (st == PQS_OK) st = copy_out(ctx, out_idx, dc, (size_t)n, io);
    if (st == PQS_OK) st = copy_out(ctx, out_dist, dd, (size_t)n, io);
  }
  // the handle's buffers are read by work queued on the stream: drain it first
  cudaStreamSynchronize(ctx->stream);
  ivf_destroy_impl(iv);
  if (st != PQS_OK) return st;
  return finish(ctx, io);
}
int pqs_nearest(pqs_ctx* ctx, const float* centroids, int64_t K, int d, const float* points, int64_t n,
                int64_t* out_idx, double* out_dist, int io) {
  return nearest_impl(ctx, centroids, K, d, points, 0, n, out_idx, out_dist, io);
}
int pqs_nearest_f64(pqs_ctx* ctx, const float* centroids, int64_t K, int d, const double* points, int64_t n,
                    int64_t* out_idx, double* out_dist, int io) {
  return nearest_impl(ctx, centroids, K, d, points, 1, n, out_idx, out_dist, io);
}

static int ivf_search_impl(pqs_ctx* ctx, const pqs_ivf* ivf, const void* queries, int f64, int64_t nq, int ma, int r,
                           double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  if (!ctx || !ivf) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, ma >= 1 && ma <= ivf->K, "ma must be in [1, K]");
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  double* dd = nullptr;
  int64_t* di = nullptr;
  int32_t* dc = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * ivf->d, io, f64, &dq));
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * r, io, &dd));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_ids, (size_t)nq * r, io, &di));
  PQS_TRY(stage_out(ctx, S_OUT_C, out_count, (size_t)nq, io, &dc));
  PQS_TRY(run_ivf_search(ctx, ivf, dq, nq, ma, r, dd, di, dc));
  PQS_TRY(copy_out(ctx, out_dist, dd, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_ids, di, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_count, dc, (size_t)nq, io));
  return finish(ctx, io);
}
int pqs_ivf_search(pqs_ctx* ctx, const pqs_ivf* ivf, const float* queries, int64_t nq, int ma, int r,
                   double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  return ivf_search_impl(ctx, ivf, queries, 0, nq, ma, r, out_dist, out_ids, out_count, io);
}
int pqs_ivf_search_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const double* queries, int64_t nq, int ma, int r,
                       double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  return ivf_search_impl(ctx, ivf, queries, 1, nq, ma, r, out_dist, out_ids, out_count, io);
}

static int ivf_qadc_search_impl(pqs_ctx* ctx, const pqs_ivf* ivf, const void* queries, int f64, int64_t nq, int ma,
                                int r, int init_count, double* out_dist, int64_t* out_ids, int32_t* out_count,
                                int io) {
  if (!ctx || !ivf) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, ma >= 1 && ma <= ivf->K, "ma must be in [1, K]");
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, ivf->k == 16 && ivf->m % 2 == 0, "quick-adc kernel requires b=4 and even m");
  PQS_CHECK(ctx, init_count >= 1, "init_count must be >= 1");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (ivf->m > 64) return set_err(ctx, PQS_ERR_UNSUPPORTED, "quick-adc IVF kernel supports m <= 64");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  double* dd = nullptr;
  int64_t* di = nullptr;
  int32_t* dc = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * ivf->d, io, f64, &dq));
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * r, io, &dd));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_ids, (size_t)nq * r, io, &di));
  PQS_TRY(stage_out(ctx, S_OUT_C, out_count, (size_t)nq, io, &dc));
  PQS_TRY(run_ivf_qadc_search(ctx, ivf, dq, nq, ma, r, init_count, dd, di, dc));
  PQS_TRY(copy_out(ctx, out_dist, dd, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_ids, di, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_count, dc, (size_t)nq, io));
  return finish(ctx, io);
}
int pqs_ivf_qadc_search(pqs_ctx* ctx, const pqs_ivf* ivf, const float* queries, int64_t nq, int ma, int r,
                        int init_count, double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  return ivf_qadc_search_impl(ctx, ivf, queries, 0, nq, ma, r, init_count, out_dist, out_ids, out_count, io);
}
int pqs_ivf_qadc_search_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const double* queries, int64_t nq, int ma, int r,
                            int init_count, double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  return ivf_qadc_search_impl(ctx, ivf, queries, 1, nq, ma, r, init_count, out_dist, out_ids, out_count, io);
}

int pqs_fastscan_checked(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq, int64_t n_init, int r,
                         int64_t* out_checked, int io) {
  if (!ctx || !db) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, db->b == 8 && db->m == 8, "fast scan requires m=8, b=8 lookup tables");
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, db->n >= 1, "empty code list");
  PQS_CHECK(ctx, n_init >= 1 && n_init <= db->n, "n_init must be in [1, n]");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const float* dt = nullptr;
  int64_t* dc = nullptr;
  PQS_TRY(stage_in(ctx, S_TABLES, tables, (size_t)nq * 8 * 256, io, &dt));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_checked, (size_t)nq, io, &dc));
  PQS_TRY(run_fastscan_checked(ctx, db, dt, nq, n_init, r, dc));
  PQS_TRY(copy_out(ctx, out_checked, dc, (size_t)nq, io));
  return finish(ctx, io);
}

static int derived_search_impl(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* full, const pqs_pq* derived,
                               const void* queries, int f64, int64_t nq, int r, int64_t r2, double* out_dist,
                               int64_t* out_ids, int32_t* out_count, int io) {
  if (!ctx || !db || !full || !derived) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, db->n >= 1, "empty code list");
  PQS_CHECK(ctx, r2 >= 1, "r2 must be >= 1");
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, db->b == 8 && db->m == full->m, "derived search needs a b=8 code list matching the quantizer");
  PQS_CHECK(ctx, derived->m == full->m && derived->d == full->d && derived->k <= full->k,
            "derived codebooks do not match the full quantizer");
  PQS_CHECK(ctx, db->max_code < full->k, "code component out of range for the quantizer");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  float* tf = nullptr;
  float* tc = nullptr;
  double* dd = nullptr;
  int64_t* di = nullptr;
  int32_t* dc = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * full->d, io, f64, &dq));
  PQS_TRY(scratch(ctx, S_TABLES, (size_t)nq * full->m * full->k, &tf));
  PQS_TRY(scratch(ctx, S_TABLES_T, (size_t)nq * derived->m * derived->k, &tc));
  PQS_TRY(launch_tables_exact(ctx, full, dq, nq, tf));
  PQS_TRY(launch_tables_exact(ctx, derived, dq, nq, tc));
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * r, io, &dd));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_ids, (size_t)nq * r, io, &di));
  PQS_TRY(stage_out(ctx, S_OUT_C, out_count, (size_t)nq, io, &dc));
  PQS_TRY(run_derived_search(ctx, db, tf, full->k, tc, nq, derived->k, r, r2, dd, di, dc));
  PQS_TRY(copy_out(ctx, out_dist, dd, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_ids, di, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_count, dc, (size_t)nq, io));
  return finish(ctx, io);
}
int pqs_derived_search(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* full, const pqs_pq* derived,
                       const float* queries, int64_t nq, int r, int64_t r2, double* out_dist, int64_t* out_ids,
                       int32_t* out_count, int io) {
  return derived_search_impl(ctx, db, full, derived, queries, 0, nq, r, r2, out_dist, out_ids, out_count, io);
}
int pqs_derived_search_f64(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* full, const pqs_pq* derived,
                           const double* queries, int64_t nq, int r, int64_t r2, double* out_dist, int64_t* out_ids,
                           int32_t* out_count, int io) {
  return derived_search_impl(ctx, db, full, derived, queries, 1, nq, r, r2, out_dist, out_ids, out_count, io);
}

static int ivf_derived_search_impl(pqs_ctx* ctx, const pqs_ivf* ivf, const pqs_pq* derived, const void* queries,
                                   int f64, int64_t nq, int ma, int r, int64_t r2, double* out_dist,
                                   int64_t* out_ids, int32_t* out_count, int io) {
  if (!ctx || !ivf || !derived) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, ma >= 1 && ma <= ivf->K, "ma must be in [1, K]");
  PQS_CHECK(ctx, r >= 1, "r must be >= 1");
  PQS_CHECK(ctx, r2 >= 1, "r2 must be >= 1");
  PQS_CHECK(ctx, derived->m == ivf->m && derived->d == ivf->d && derived->k <= ivf->k,
            "derived codebooks do not match the index quantizer");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  QVec dq;
  double* dd = nullptr;
  int64_t* di = nullptr;
  int32_t* dc = nullptr;
  PQS_TRY(stage_q(ctx, queries, (size_t)nq * ivf->d, io, f64, &dq));
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * r, io, &dd));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_ids, (size_t)nq * r, io, &di));
  PQS_TRY(stage_out(ctx, S_OUT_C, out_count, (size_t)nq, io, &dc));
  PQS_TRY(run_ivf_derived_search(ctx, ivf, derived->books, derived->k, dq, nq, ma, r, r2, dd, di, dc));
  PQS_TRY(copy_out(ctx, out_dist, dd, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_ids, di, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_count, dc, (size_t)nq, io));
  return finish(ctx, io);
}
int pqs_ivf_derived_search(pqs_ctx* ctx, const pqs_ivf* ivf, const pqs_pq* derived, const float* queries, int64_t nq,
                           int ma, int r, int64_t r2, double* out_dist, int64_t* out_ids, int32_t* out_count,
                           int io) {
  return ivf_derived_search_impl(ctx, ivf, derived, queries, 0, nq, ma, r, r2, out_dist, out_ids, out_count, io);
}
int pqs_ivf_derived_search_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const pqs_pq* derived, const double* queries,
                               int64_t nq, int ma, int r, int64_t r2, double* out_dist, int64_t* out_ids,
                               int32_t* out_count, int io) {
  return ivf_derived_search_impl(ctx, ivf, derived, queries, 1, nq, ma, r, r2, out_dist, out_ids, out_count, io);
}

// ---------------------------------------------------------------- merge
int pqs_merge_topr(pqs_ctx* ctx, int G, const double* dists, const int64_t* ids, const int32_t* counts, int64_t nq,
                   int r_in, int r, double* out_dist, int64_t* out_ids, int32_t* out_count, int io) {
  if (!ctx) return PQS_ERR_INVALID;
  PQS_TRY(check_io(ctx, io));
  PQS_CHECK(ctx, G >= 1 && r_in >= 1 && r >= 1, "G, r_in and r must be >= 1");
  if (r > MAX_R) return set_err(ctx, PQS_ERR_UNSUPPORTED, "r > 4096 is not supported by the device select");
  if (nq == 0) return PQS_OK;
  PQS_CUDA(ctx, cudaSetDevice(ctx->device));
  const double* dd = nullptr;
  const int64_t* di = nullptr;
  const int32_t* dc = nullptr;
  PQS_TRY(stage_in(ctx, S_PROBE_D, dists, (size_t)G * nq * r_in, io, &dd));
  PQS_TRY(stage_in(ctx, S_PROBE, ids, (size_t)G * nq * r_in, io, &di));
  PQS_TRY(stage_in(ctx, S_IVF_WORK, counts, (size_t)G * nq, io, &dc));
  double* od = nullptr;
  int64_t* oi = nullptr;
  int32_t* oc = nullptr;
  PQS_TRY(stage_out(ctx, S_OUT_D, out_dist, (size_t)nq * r, io, &od));
  PQS_TRY(stage_out(ctx, S_OUT_I, out_ids, (size_t)nq * r, io, &oi));
  PQS_TRY(stage_out(ctx, S_OUT_C, out_count, (size_t)nq, io, &oc));
  const int64_t gcap = (int64_t)G * r_in;
  uint64_t* gk = nullptr;
  int64_t* gi = nullptr;
  if (gcap > 2048) {
    PQS_TRY(scratch(ctx, S_KEYS, (size_t)(nq * gcap), &gk));
    PQS_TRY(scratch(ctx, S_IDS, (size_t)(nq * gcap), &gi));
  }
  SelArgs s{};
  s.src = SEL_MERGE;
  s.nq = nq;
  s.r = r;
  s.G = G;
  s.r_in = r_in;
  s.mdist = dd;
  s.mids = di;
  s.mcnt = dc;
  s.out_d = od;
  s.out_i = oi;
  s.out_c = oc;
  s.gkeys = gk;
  s.gids = gi;
  s.gcap = gcap;
  PQS_TRY(launch_select(ctx, s));
  PQS_TRY(copy_out(ctx, out_dist, od, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_ids, oi, (size_t)nq * r, io));
  PQS_TRY(copy_out(ctx, out_count, oc, (size_t)nq, io));
  return finish(ctx, io);
}

}  // extern "C"
