// encode.cu -- PQ encoding and device-side code-list builders.
//
// Reference: encode (quantizer.py:308-325) -> nearest (_dist.py:24-39) ->
// sqdist_matrix (_dist.py:13-21, scipy cdist 'sqeuclidean'): per sub-space j
// the index of the nearest centroid by the fp64 sum over t of
// (fp64 z_t - fp64 C_j[i][t])^2 accumulated in t order, ties to the lowest
// index (np.argmin).  With an IVF coarse quantizer the encoded vector is the
// residual z = fp64(x) - fp64(coarse[cell]) (build_ivf, ivf.py:137-140).
//
// One thread per (vector, sub-space): the sub-space's centroids are staged in
// shared memory as fp64 (broadcast reads, no per-use conversion), the
// thread's sub-vector lives in registers (DSUB template) and the distance is
// accumulated with explicit __dsub_rn/__dmul_rn/__dadd_rn (no FMA
// contraction), exactly as the reference's scipy loop.
#include <cuda_runtime.h>

#include <algorithm>

#include "pqs_common.cuh"

namespace {

constexpr int ENC_THREADS = 128;

template <int DSUB>
__global__ void __launch_bounds__(ENC_THREADS) encode_kernel(QVec x, int64_t n, int d,
                                                             const float* __restrict__ books, int k, int dsub_rt,
                                                             const float* __restrict__ coarse,
                                                             const int64_t* __restrict__ cells, int m,
                                                             uint8_t* __restrict__ out) {
  extern __shared__ double cs[];  // (k, dsub) fp64
  const int dsub = DSUB > 0 ? DSUB : dsub_rt;
  const int j = blockIdx.y;
  const float* bj = books + (int64_t)j * k * dsub;
  for (int i = threadIdx.x; i < k * dsub; i += blockDim.x) cs[i] = (double)bj[i];
  __syncthreads();
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const QVec xv = x.offset(v * d + (int64_t)j * dsub);
  const float* gv = coarse ? coarse + cells[v] * d + (int64_t)j * dsub : nullptr;
  if (DSUB > 0) {
    double z[DSUB > 0 ? DSUB : 1];
#pragma unroll
    for (int t = 0; t < DSUB; ++t) z[t] = gv ? __dsub_rn(xv.at(t), (double)gv[t]) : xv.at(t);
    double best = 0.0;
    int bi = 0;
    for (int i = 0; i < k; ++i) {
      const double* c = cs + i * DSUB;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < DSUB; ++t) {
        const double df = __dsub_rn(z[t], c[t]);
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
      if (i == 0 || acc < best) {
        best = acc;
        bi = i;
      }
    }
    out[v * m + j] = (uint8_t)bi;
  } else {
    double best = 0.0;
    int bi = 0;
    for (int i = 0; i < k; ++i) {
      const double* c = cs + i * dsub;
      double acc = 0.0;
      for (int t = 0; t < dsub; ++t) {
        const double zt = gv ? __dsub_rn(xv.at(t), (double)gv[t]) : xv.at(t);
        const double df = __dsub_rn(zt, c[t]);
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
      if (i == 0 || acc < best) {
        best = acc;
        bi = i;
      }
    }
    out[v * m + j] = (uint8_t)bi;
  }
}

__global__ void max_u8_kernel(const uint8_t* __restrict__ p, int64_t count, unsigned int* __restrict__ out) {
  unsigned int mx = 0;
  const int64_t n16 = count / 16;
  const uint4* p16 = reinterpret_cast<const uint4*>(p);
  const bool aligned = (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail0 = 0;
  if (aligned) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
      const uint4 w = p16[i];
      const uint32_t t = __vmaxu4(__vmaxu4(w.x, w.y), __vmaxu4(w.z, w.w));  // per-byte max
      mx = max(mx, max(max(t & 255u, (t >> 8) & 255u), max((t >> 16) & 255u, t >> 24)));
    }
    tail0 = n16 * 16;
  }
  for (int64_t i = tail0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += stride) mx = max(mx, (unsigned int)p[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// (n, m) row-major codes -> the scan8 tile layout: byte (t, j, c) at
// t*m*TILE8 + j*TILE8 + c, zero padding in the last tile
__global__ void build_db8_kernel(const uint8_t* __restrict__ codes, int64_t n, int m, int64_t total,
                                 uint8_t* __restrict__ out) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= total) return;
  const int64_t c = o % TILE8;
  const int64_t tj = o / TILE8;
  const int64_t j = tj % m, t = tj / m;
  const int64_t i = t * TILE8 + c;
  out[o] = i < n ? codes[i * m + j] : (uint8_t)0;
}

// PQL1 payload with b <= 4 (scan.py:293-316): (m+1)/2 bytes per code, even
// component in the low nibble, odd component in the high nibble
__global__ void unpack_nibbles_kernel(const uint8_t* __restrict__ packed, int64_t n, int m,
                                      uint8_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * m) return;
  const int64_t c = i / m;
  const int j = (int)(i - c * m);
  const uint8_t v = packed[c * ((m + 1) / 2) + (j >> 1)];
  out[i] = (j & 1) ? (uint8_t)(v >> 4) : (uint8_t)(v & 15);
}

}  // namespace

int launch_unpack_nibbles(pqs_ctx* ctx, const uint8_t* d_packed, int64_t n, int m, uint8_t* d_out) {
  if (n == 0) return PQS_OK;
  unpack_nibbles_kernel<<<(unsigned)cdiv(n * m, 256), 256, 0, ctx->stream>>>(d_packed, n, m, d_out);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int device_max_u8(pqs_ctx* ctx, const uint8_t* d, int64_t count, int* out) {
  *out = 0;
  if (count <= 0) return PQS_OK;
  unsigned int* dm = nullptr;
  PQS_TRY(scratch(ctx, S_FLAG, 1, &dm));
  PQS_CUDA(ctx, cudaMemsetAsync(dm, 0, sizeof(unsigned int), ctx->stream));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(count, 256 * 16), 4 * (int64_t)ctx->sm_count));
  max_u8_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(d, count, dm);
  PQS_LAUNCHED(ctx);
  unsigned int h = 0;
  PQS_TRY(download(ctx, &h, dm, sizeof(h)));
  *out = (int)h;
  return PQS_OK;
}

int build_db8(pqs_ctx* ctx, pqs_db* db, const uint8_t* d_codes) {
  const int64_t total = db->ntiles * db->m * TILE8;
  build_db8_kernel<<<(unsigned)cdiv(total, 256), 256, 0, ctx->stream>>>(d_codes, db->n, db->m, total, db->codes8);
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}

int launch_encode(pqs_ctx* ctx, const pqs_pq* pq, QVec d_x, int64_t n, const float* d_coarse,
                  const int64_t* d_cells, uint8_t* d_out) {
  if (n == 0) return PQS_OK;
  const int k = pq->k, dsub = pq->dsub;
  const size_t smem = (size_t)k * dsub * sizeof(double);
  PQS_CHECK(ctx, smem <= 200 * 1024, "encode: k * dsub too large for the shared-memory codebook stage");
  dim3 grid((unsigned)cdiv(n, ENC_THREADS), (unsigned)pq->m);
  PQS_CHECK(ctx, cdiv(n, ENC_THREADS) < (1ll << 31), "encode: too many vectors for one call");
#define PQS_ENC(DS)                                                                                              \
  do {                                                                                                          \
    PQS_CUDA(ctx, cudaFuncSetAttribute(encode_kernel<DS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    encode_kernel<DS><<<grid, ENC_THREADS, smem, ctx->stream>>>(d_x, n, pq->d, pq->books, k, dsub, d_coarse,    \
                                                              d_cells, pq->m, d_out);                           \
  } while (0)
  switch (dsub) {
    case 2: PQS_ENC(2); break;
    case 4: PQS_ENC(4); break;
    case 6: PQS_ENC(6); break;
    case 8: PQS_ENC(8); break;
    case 12: PQS_ENC(12); break;
    case 15: PQS_ENC(15); break;
    case 16: PQS_ENC(16); break;
    case 32: PQS_ENC(32); break;
    default: PQS_ENC(0); break;
  }
#undef PQS_ENC
  PQS_LAUNCHED(ctx);
  return PQS_OK;
}
