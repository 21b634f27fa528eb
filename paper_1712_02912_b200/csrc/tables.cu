// tables.cu -- K1: exact per-query lookup tables.
//
// Reference: compute_tables (scan.py:45-56) calls sqdist_matrix
// (_dist.py:13-21 = scipy cdist 'sqeuclidean' in fp64) per sub-space on the
// fp64-cast query (quantizer.py:85-89; float32 or float64 rows, QVec) and rounds each row to fp32.  scipy
// sums (u_t - v_t)^2 sequentially over t; this kernel does the same with
// explicit round-to-nearest fp64 ops (no FMA contraction), so every entry is
// bit-identical (tests/test_gpu_parity.py::test_tables_bitwise).
//
// One thread per (query, sub-space, centroid).  The codebook of a CTA's
// sub-space and the query sub-vector are read through L1; the work is tiny
// next to the scan (cfg0: 2M entries x 16 dims per 1000 queries).
#include <cuda_runtime.h>

#include "pqs_common.cuh"

namespace {

__global__ void tables_exact_kernel(const float* __restrict__ books, QVec queries, int64_t nq,
                                    int m, int k, int dsub, float* __restrict__ out) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = nq * m * (int64_t)k;
  if (gid >= total) return;
  const int i = (int)(gid % k);
  const int64_t t = gid / k;
  const int j = (int)(t % m);
  const int64_t q = t / m;
  const int64_t y = q * (int64_t)m * dsub + (int64_t)j * dsub;
  const float* c = books + ((int64_t)j * k + i) * dsub;
  double acc = 0.0;
  for (int s = 0; s < dsub; ++s) {
    const double d = __dsub_rn(queries.at(y + s), (double)__ldg(c + s));
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  out[gid] = __double2float_rn(acc);
}

}  // namespace

int launch_tables_exact(pqs_ctx* ctx, const pqs_pq* pq, QVec d_queries, int64_t nq, float* d_tables) {
  const int64_t total = nq * pq->m * (int64_t)pq->k;
  if (total == 0) return PQS_OK;
  tables_exact_kernel<<<(unsigned)cdiv(total, 256), 256, 0, ctx->stream>>>(pq->books, d_queries, nq, pq->m, pq->k,
                                                                         pq->dsub, d_tables);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}
