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

// DSUB > 0: compile-time sub-space dimension -- the centroid's and the query's
// coordinates are all loaded (16-byte loads when DSUB % 4 == 0) before the
// sequential fp64 chain, whose order is unchanged; DSUB == 0: runtime dsub
template <int DSUB>
__global__ void tables_exact_kernel(const float* __restrict__ books, QVec queries, int64_t nq,
                                    int m, int k, int dsub_rt, float* __restrict__ out) {
  const int dsub = DSUB > 0 ? DSUB : dsub_rt;
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
  if constexpr (DSUB > 0) {
    float cv[DSUB];
    double qv[DSUB];
    if constexpr (DSUB % 4 == 0) {
#pragma unroll
      for (int s4 = 0; s4 < DSUB / 4; ++s4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(c) + s4);
        cv[4 * s4] = v.x, cv[4 * s4 + 1] = v.y, cv[4 * s4 + 2] = v.z, cv[4 * s4 + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int s = 0; s < DSUB; ++s) cv[s] = __ldg(c + s);
    }
#pragma unroll
    for (int s = 0; s < DSUB; ++s) qv[s] = queries.at(y + s);
#pragma unroll
    for (int s = 0; s < DSUB; ++s) {
      const double d = __dsub_rn(qv[s], (double)cv[s]);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  } else {
    for (int s = 0; s < dsub; ++s) {
      const double d = __dsub_rn(queries.at(y + s), (double)__ldg(c + s));
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  }
  out[gid] = __double2float_rn(acc);
}

}  // namespace

int launch_tables_exact(pqs_ctx* ctx, const pqs_pq* pq, QVec d_queries, int64_t nq, float* d_tables) {
  const int64_t total = nq * pq->m * (int64_t)pq->k;
  if (total == 0) return PQS_OK;
  auto kern = tables_exact_kernel<0>;
  // the BASELINE shapes with an even sub-space dimension (cfg0/3: 16, cfg1: 8, cfg4: 6) and small sub-spaces;
  // odd dimensions (cfg2: 15) keep the runtime loop -- unrolled scalar loads measured slower there (224 vs 187 us)
  switch (pq->dsub) {
    case 16: kern = tables_exact_kernel<16>; break;
    case 8: kern = tables_exact_kernel<8>; break;
    case 6: kern = tables_exact_kernel<6>; break;
    case 4: kern = tables_exact_kernel<4>; break;
    case 2: kern = tables_exact_kernel<2>; break;
    default: break;
  }
  kern<<<(unsigned)cdiv(total, 256), 256, 0, ctx->stream>>>(pq->books, d_queries, nq, pq->m, pq->k, pq->dsub, d_tables);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}
