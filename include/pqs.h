/*
 * pqs.h -- C ABI of libpqs.so, the B200 (sm_100a) ADC-scan engine.
 *
 * This is the drop-in boundary for the PQ ADC scan path of the reference
 * package `pqscan` (arxiv/paper_1712_02912, /root/reference/pkg/src/pqscan).
 * The reference has no FFI of its own (it is pure NumPy/SciPy); its
 * "operator API" is the Python function surface listed in SURVEY.md 8(b).
 * Each entry point below names the reference function it replaces; the
 * Python package `paper_1712_02912_b200` binds these through ctypes and
 * re-exports the reference names (see INTEGRATION.md for the binding a
 * reference maintainer would add).
 *
 * Conventions
 *   - Plain pointers and sizes, no framework types.  Every call returns an
 *     int status (PQS_OK == 0); on failure pqs_last_error(ctx) holds a
 *     message.  Argument errors the reference raises as ValueError map to
 *     PQS_ERR_INVALID.
 *   - `io` says where the per-call arrays (queries/tables in, results out)
 *     live: PQS_IO_HOST (host memory; copies happen inside the call) or
 *     PQS_IO_DEVICE (device pointers, e.g. torch.Tensor.data_ptr()).
 *     Quantizer / code-list / index handles always own device copies; their
 *     create calls take host or device source arrays by the same flag.
 *   - All work of a context is issued on one CUDA stream (its own, or the
 *     one set with pqs_ctx_set_stream).  A context is single-writer, like
 *     the reference NeighborSet; separate contexts may run
 *     concurrently.
 *   - Query (and vector) rows: every entry point that takes them as
 *     `const float*` has a `_f64` twin taking `const double*`.  The reference
 *     computes from float64(query) (ProductQuantizer.rotate,
 *     quantizer.py:85-89; query_ivf ivf.py:170; encode quantizer.py:319-323),
 *     so the exact kernels read the rows in fp64 either way; float32 rows are
 *     widened exactly, float64 rows are used as given.
 *   - Results are (nq, r) row-major arrays ascending by (distance, id);
 *     out_count[q] = number of valid entries (min(r, candidates)); unused
 *     slots hold distance +inf (bins 255) and id -1.
 */
#ifndef PQS_H
#define PQS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQS_API_VERSION 3

typedef struct pqs_ctx pqs_ctx;
typedef struct pqs_pq pqs_pq;
typedef struct pqs_db pqs_db;
typedef struct pqs_ivf pqs_ivf;

enum pqs_status {
  PQS_OK = 0,
  PQS_ERR_INVALID = 1,     /* the reference raises ValueError here */
  PQS_ERR_CUDA = 2,
  PQS_ERR_NOMEM = 3,
  PQS_ERR_UNSUPPORTED = 4  /* valid for the reference, outside this engine's limits */
};

enum pqs_io { PQS_IO_HOST = 0, PQS_IO_DEVICE = 1 };

enum pqs_option {
  PQS_OPT_CAND_CAP = 1,     /* candidate slots per query in a filtered scan (default 32768) */
  PQS_OPT_SAMPLE_DIV = 2,   /* threshold sample = 1/SAMPLE_DIV of the code tiles (default 32) */
  PQS_OPT_FORCE_FALLBACK = 3,/* 1: run the exact dense fallback for every query (testing) */
  PQS_OPT_SCAN4_ENGINE = 4, /* Quick ADC scan: 0 auto (tcgen05 int8 when possible), 1 PRMT, 2 tcgen05 */
  PQS_OPT_TC_CHUNK_TILES = 5,/* tcgen05 scan: cap on 128-code tiles per launch (0 = automatic; testing) */
  PQS_OPT_SCAN8_ENGINE = 6, /* float ADC filter: 0 auto (packed two-query words when m <= 64), 1 u16 lane=query, 2 packed */
  PQS_OPT_IVF_ENGINE = 7    /* IVF 'adc' list scan: 0 auto (packed integer pre-filter when m = 8, k = 256), 1 float, 2 packed */
};

enum pqs_stat {
  PQS_STAT_LAUNCHES = 1,       /* kernels launched by this context since creation */
  PQS_STAT_LAST_MAX_CAND = 2,  /* largest per-query candidate count of the last search */
  PQS_STAT_LAST_OVERFLOW = 3,  /* queries that took the dense fallback in the last search */
  PQS_STAT_LAST_EVALS = 4,     /* (query, code) evaluations of the last search (IVF: exact count) */
  PQS_STAT_LAST_SCAN_NS = 5,   /* device time of the last search's main scan kernel (CUDA events) */
  PQS_STAT_LAST_SCAN_LAUNCHES = 6, /* launches of that kernel in the last search */
  PQS_STAT_LAST_CAND_TOTAL = 7,    /* sum over queries of the candidates of the last search */
  PQS_STAT_LAST_SCAN_ENGINE = 8,   /* 1 PRMT scan4, 2 tcgen05 scan4, 3 scan8 (u16), 4 IVF list scan (float), 5 scan8 packed, 6 IVF list scan (packed) */
  PQS_STAT_LAST_SCAN_WORK = 9,     /* work units of that kernel: tcgen05 -> int8 MMA ops; others -> table lookups */
  PQS_STAT_LAST_RERANK_TOTAL = 10, /* float / IVF: candidates re-scored exactly after the bound tightening (sum over queries) */
  PQS_STAT_LAST_SLOT_EVALS = 11    /* IVF list scan: (slot, code) evaluations incl. idle slots of partly filled 8-query groups */
};

int pqs_api_version(void);

/* ---- context --------------------------------------------------------- */
int pqs_ctx_create(int device, pqs_ctx** out);
void pqs_ctx_destroy(pqs_ctx* ctx);
int pqs_ctx_set_stream(pqs_ctx* ctx, void* cuda_stream); /* NULL -> context's own stream */
int pqs_ctx_synchronize(pqs_ctx* ctx);
int pqs_ctx_set_option(pqs_ctx* ctx, int option, int64_t value);
int pqs_ctx_get_stat(pqs_ctx* ctx, int stat, int64_t* out);
const char* pqs_last_error(const pqs_ctx* ctx);

/* ---- quantizer: ProductQuantizer (quantizer.py:38-89, identity rotation) */
/* codebooks: host float32 (m, 2^b, d/m) C-contiguous. */
int pqs_pq_create(pqs_ctx* ctx, int m, int b, int d, const float* codebooks, pqs_pq** out);
void pqs_pq_destroy(pqs_pq* pq);

/* ---- code lists: CodeList (scan.py:157-194) / TransposedCodeList (scan.py:209-245)
 * codes: uint8 (n, m) row-major component values (< 2^b), host or device (io).
 * b == 8: float-ADC layout (scan8), any m >= 1, 2 <= k <= 256.
 * b == 4: Quick ADC layout (scan4, 4-code PRMT-selector quads), even m <= 32.
 * ids:  int64 (n,) (same io) or NULL for implicit ids id_base + i (CodeList
 *       default ids = arange(n), scan.py:170-171).                         */
int pqs_db_create(pqs_ctx* ctx, const uint8_t* codes, int64_t n, int m, int b,
                  const int64_t* ids, int64_t id_base, int io, pqs_db** out);
/* code list straight from a PQL1 file payload (scan.py:290-359, save_codes):
 * b_file <= 4 -> (m+1)/2 nibble-packed bytes per code (even component low),
 * unpacked on the device; 4 < b_file <= 8 -> one byte per component.
 * layout_b = 4 (Quick ADC, even m, components < 16) or 8 (float ADC).    */
int pqs_db_create_packed(pqs_ctx* ctx, const uint8_t* payload, int64_t n, int m, int b_file,
                         int layout_b, const int64_t* ids, int64_t id_base, int io, pqs_db** out);
/* Quick ADC under sharding: qmax must come from the first init_count codes of
 * the GLOBAL list (quickadc.py:130-137).  Supplies them (uint8 (n_prefix, m)). */
int pqs_db_set_prefix(pqs_ctx* ctx, pqs_db* db, const uint8_t* prefix_codes, int64_t n_prefix,
                      int io);
void pqs_db_destroy(pqs_db* db);

/* ---- tables: compute_tables (scan.py:45-56; sqdist_matrix _dist.py:13-21)
 * queries (nq, d) float32 -> out_tables (nq, m, k) float32, bit-identical. */
int pqs_compute_tables(pqs_ctx* ctx, const pqs_pq* pq, const float* queries, int64_t nq,
                       float* out_tables, int io);
int pqs_compute_tables_f64(pqs_ctx* ctx, const pqs_pq* pq, const double* queries, int64_t nq,
                           float* out_tables, int io);

/* ---- dense fp64 ADC: scan_distances (scan.py:68-81), b == 8 list
 * tables (nq, m, k) float32 (k <= 256, every code < k) -> out (nq, n)
 * float64, bit-identical.                                                 */
int pqs_scan_distances(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq,
                       int k, double* out, int io);

/* ---- float ADC top-r: scan (scan.py:197-203), b == 8 list, given tables. */
int pqs_adc_scan(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq, int k,
                 int r, double* out_dist, int64_t* out_ids, int32_t* out_count, int io);
/* batched search from queries: compute_tables + scan for every query.     */
int pqs_adc_search(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const float* queries,
                   int64_t nq, int r, double* out_dist, int64_t* out_ids, int32_t* out_count,
                   int io);
int pqs_adc_search_f64(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const double* queries,
                       int64_t nq, int r, double* out_dist, int64_t* out_ids, int32_t* out_count,
                       int io);

/* ---- Quick ADC: qadc_scan (quickadc.py:104-141), b == 4 list, given tables
 * (nq, m, 16) float32.  Outputs bins (nq, r) uint8 ascending by (bin, id),
 * ids, counts, the quantized tables (nq, m, 16) uint8 and (qmin, qmax)
 * (nq, 2) float64 -- QuantizedTables4 (quickadc.py:32-54).  Output pointers
 * out_qtables / out_qminmax may be NULL.                                   */
int pqs_qadc_scan(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq,
                  int init_count, int r, uint8_t* out_bins, int64_t* out_ids,
                  int32_t* out_count, uint8_t* out_qtables, double* out_qminmax, int io);
int pqs_qadc_search(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const float* queries,
                    int64_t nq, int init_count, int r, uint8_t* out_bins, int64_t* out_ids,
                    int32_t* out_count, uint8_t* out_qtables, double* out_qminmax, int io);
int pqs_qadc_search_f64(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* pq, const double* queries,
                        int64_t nq, int init_count, int r, uint8_t* out_bins, int64_t* out_ids,
                        int32_t* out_count, uint8_t* out_qtables, double* out_qminmax, int io);

/* ---- quantize (fastscan.py:48-57): 127-bin fp64 quantization of values
 * (n,) float64 with QuantParams(qmin, qmax) -> out (n,) uint8.            */
int pqs_quantize(pqs_ctx* ctx, double qmin, double qmax, const double* values, int64_t n,
                 uint8_t* out, int io);

/* ---- quantized_distances (quickadc.py:87-101), b == 4 list:
 * qtables (nq, m, 16) uint8 (entries <= 127) -> out (nq, n) uint8.          */
int pqs_quantized_distances(pqs_ctx* ctx, const pqs_db* db, const uint8_t* qtables,
                            int64_t nq, uint8_t* out, int io);

/* ---- IVFADC: IvfIndex (ivf.py:58-86) + query_ivf kernel='adc' (ivf.py:148-196)
 * coarse (K, d) float32; lists concatenated in cell order: list_sizes (K,),
 * codes (sum, m) uint8 (b == 8), ids (sum,) int64.  coarse/codes/ids host
 * or device (io); list_sizes always host.                                  */
int pqs_ivf_create(pqs_ctx* ctx, const pqs_pq* pq, const float* coarse, int64_t K,
                   const int64_t* list_sizes, const uint8_t* codes, const int64_t* ids,
                   int io, pqs_ivf** out);
void pqs_ivf_destroy(pqs_ivf* ivf);
/* probes only: nearest_k (_dist.py:42-67) -> out_cells (nq, ma) int64,
 * out_dist (nq, ma) float64 (may be NULL), ascending by (distance, cell).  */
int pqs_ivf_probe(pqs_ctx* ctx, const pqs_ivf* ivf, const float* queries, int64_t nq, int ma,
                  int64_t* out_cells, double* out_dist, int io);
int pqs_ivf_probe_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const double* queries, int64_t nq, int ma,
                      int64_t* out_cells, double* out_dist, int io);
int pqs_ivf_search(pqs_ctx* ctx, const pqs_ivf* ivf, const float* queries, int64_t nq, int ma,
                   int r, double* out_dist, int64_t* out_ids, int32_t* out_count, int io);
int pqs_ivf_search_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const double* queries, int64_t nq, int ma,
                       int r, double* out_dist, int64_t* out_ids, int32_t* out_count, int io);
/* ---- PQ Fast Scan statistics (fast_scan, fastscan.py:328-386): the number
 * of codes whose exact distance the reference's pruned scan evaluates
 * (ScanStats.checked; pruned = n - checked).  db: the grouped database's
 * codes in storage order (GroupedDatabase.reconstruct_codes, b == 8, m ==
 * 8); tables (nq, 8, 256) float32; n_init = ceil(init * n) in [1, n].  The
 * neighbour set equals pqs_adc_scan's (fast_scan is exact).              */
int pqs_fastscan_checked(pqs_ctx* ctx, const pqs_db* db, const float* tables, int64_t nq,
                         int64_t n_init, int r, int64_t* out_checked, int io);

/* ---- derived-quantizer two-pass search: search_two_pass (derived.py:402-409)
 * over a b == 8 list; full: the DerivedPQ's quantizer (m, 2^b), derived: its
 * 2^bbar codebooks as a quantizer handle (same m, d).  r2 >= 1 candidates
 * for the exact rerank (default_r2, ivf.py:51-53).  Outputs as
 * pqs_adc_search (exact fp64 distances of the reranked codes).           */
int pqs_derived_search(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* full, const pqs_pq* derived,
                       const float* queries, int64_t nq, int r, int64_t r2, double* out_dist,
                       int64_t* out_ids, int32_t* out_count, int io);
int pqs_derived_search_f64(pqs_ctx* ctx, const pqs_db* db, const pqs_pq* full, const pqs_pq* derived,
                           const double* queries, int64_t nq, int r, int64_t r2, double* out_dist,
                           int64_t* out_ids, int32_t* out_count, int io);
/* ---- query_ivf kernel='derived' (ivf.py:191-195): search_two_pass per
 * probed list on the residual, merged by (distance, id).                 */
int pqs_ivf_derived_search(pqs_ctx* ctx, const pqs_ivf* ivf, const pqs_pq* derived,
                           const float* queries, int64_t nq, int ma, int r, int64_t r2,
                           double* out_dist, int64_t* out_ids, int32_t* out_count, int io);
int pqs_ivf_derived_search_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const pqs_pq* derived,
                               const double* queries, int64_t nq, int ma, int r, int64_t r2,
                               double* out_dist, int64_t* out_ids, int32_t* out_count, int io);

/* ---- query_ivf kernel='quick-adc' (ivf.py:185-190): per probed list the
 * Quick ADC scan (quickadc.py:104-141, init_count = min(init_count, list
 * size)), its r best by (bin, id) rescaled (quickadc.py:50-54) and merged by
 * (distance, id).  b == 4, even m <= 64; init_count >= 1.  Outputs as
 * pqs_ivf_search (out_dist = rescaled fp64 distances).                    */
int pqs_ivf_qadc_search(pqs_ctx* ctx, const pqs_ivf* ivf, const float* queries, int64_t nq,
                        int ma, int r, int init_count, double* out_dist, int64_t* out_ids,
                        int32_t* out_count, int io);
int pqs_ivf_qadc_search_f64(pqs_ctx* ctx, const pqs_ivf* ivf, const double* queries, int64_t nq,
                            int ma, int r, int init_count, double* out_dist, int64_t* out_ids,
                            int32_t* out_count, int io);

/* ---- encode (quantizer.py:308-325, nearest _dist.py:24-39): per sub-space
 * the nearest centroid by the fp64 cdist sum, ties to the lowest index.
 * x (n, d) float32 -> out_codes (n, m) uint8 (b <= 8), bit-identical.  With
 * coarse (K, d) float32 and cells (n,) int64 the residual
 * fp64(x) - fp64(coarse[cell]) is encoded (build_ivf, ivf.py:137-140);
 * both NULL for plain PQ.                                                  */
int pqs_encode(pqs_ctx* ctx, const pqs_pq* pq, const float* x, int64_t n, const float* coarse,
               int64_t K, const int64_t* cells, uint8_t* out_codes, int io);
int pqs_encode_f64(pqs_ctx* ctx, const pqs_pq* pq, const double* x, int64_t n, const float* coarse,
                   int64_t K, const int64_t* cells, uint8_t* out_codes, int io);

/* ---- nearest (_dist.py:24-39), the assignment step of build_ivf (ivf.py:122):
 * per point the index of its nearest centroid by the fp64 cdist sum, ties to
 * the lowest index, and that squared distance.  centroids (K, d) float32
 * (the reference widens them with astype(float64)), points (n, d); out_idx
 * (n,) int64, out_dist (n,) float64 or NULL.  Runs the probe GEMM (tcgen05
 * kind::tf32 shortlist with a certified bound) and its exact fp64 re-score,
 * i.e. nearest_k with k = 1; centroids/points host or device by io.        */
int pqs_nearest(pqs_ctx* ctx, const float* centroids, int64_t K, int d, const float* points,
                int64_t n, int64_t* out_idx, double* out_dist, int io);
int pqs_nearest_f64(pqs_ctx* ctx, const float* centroids, int64_t K, int d, const double* points,
                    int64_t n, int64_t* out_idx, double* out_dist, int io);

/* ---- sharded merge: top-r of the union of G per-shard top-r lists by
 * (distance, id) -- NeighborSet.push semantics (scan.py:109-118).
 * dists (G, nq, r_in) float64, ids (G, nq, r_in), counts (G, nq).          */
int pqs_merge_topr(pqs_ctx* ctx, int G, const double* dists, const int64_t* ids,
                   const int32_t* counts, int64_t nq, int r_in, int r, double* out_dist,
                   int64_t* out_ids, int32_t* out_count, int io);

#ifdef __cplusplus
}
#endif
#endif /* PQS_H */
