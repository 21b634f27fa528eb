// peaks.cu -- microbenchmarked peaks for the roofline denominators of the
// ADC-scan kernels.  Standalone binary:
//   make peaks && tools/bin/pqs_peaks > profiles/peaks_rNN.json
//
// Measured, one CTA per SM over all SMs, CUDA-event timed, with the effective
// SM clock of each run read from clock64 / %globaltimer inside the kernel:
//   i8_mma      tcgen05.mma.cta_group::1.kind::i8, M=128 N=256 K=32, back to
//               back into two TMEM accumulators (operands resident in shared
//               memory, no epilogue) -- the int8 tensor peak of scan4tc.
//   f16_mma     the same for kind::f16 (bf16 inputs, f32 accumulate, K=16) --
//               cross-check against MEASURED_PEAKS.json's cuBLAS bf16 figure.
//   tf32_mma    kind::tf32 (K=8) -- the peak of the IVF probe GEMM.
//   tmem_ld     tcgen05.ld 32x32b.x64 (64 columns -> 64 registers) and
//               32x32b.x64.pack::16b (128 columns -> 64 registers, low 16 bits
//               of each column) throughput, 8 warps (2 per lane quadrant) --
//               the bound of the scan4tc filter epilogue.
//   prmt        PRMT issue rate (byte-permute): a 16-entry register LUT
//               resolves 4 lookups with 2 PRMT (scan4 engine).
//   smem_lut    conflict-free shared-memory lookups (lane = query, one 32-bit
//               word per lane per lookup, distinct banks) -- the LUT rate of
//               the float scans.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));   \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

struct Clk {
  unsigned long long c0, c1, t0, t1;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// ------------------------------------------------------------------ MMA peaks
// kind: 0 i8 (u8 x s8 -> s32), 1 f16 (bf16 x bf16 -> f32), 2 tf32 (-> f32)
constexpr int MM = 128, MN = 256;
template <int KIND>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters, Clk* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  constexpr int KB = 64;                  // bytes of K per row per tile (two 32-byte MMA K steps)
  uint8_t* sA = sm;                       // MM x KB
  uint8_t* sB = sm + MM * KB;             // MN x KB
  for (int i = threadIdx.x; i < (MM + MN) * KB / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = KIND == 0 ? (i * 2654435761u) & 0x3F3F3F3Fu : 0x3F803F80u ^ (i & 0x00070007u);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    unsigned long long c0 = clock64(), t0 = gtime();
    // idesc: D type (bits 4-5: 1 f32, 2 s32), A/B type (7-9, 10-12), N>>3 (17-22), M>>4 (24-28)
    constexpr uint32_t idesc = KIND == 0   ? ((2u << 4) | (0u << 7) | (1u << 10))
                               : KIND == 1 ? ((1u << 4) | (1u << 7) | (1u << 10))
                                           : ((1u << 4) | (2u << 7) | (2u << 10));
    constexpr uint32_t IDESC = idesc | ((uint32_t)(MN >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((it & 1) * MN);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        // K-major no-swizzle: 16-byte core rows; two 16-byte K chunks per 32-byte MMA step
        const uint32_t ks = (uint32_t)(s & 1) * 2;
        const uint64_t da = make_desc(a0 + ks * (MM / 8) * 128, (MM / 8) * 128, 128);
        const uint64_t db = make_desc(b0 + ks * (MN / 8) * 128, (MN / 8) * 128, 128);
        const uint32_t acc = s > 0 ? 1u : 0u;
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(da), "l"(db), "r"(IDESC), "r"(acc) : "memory");
        else if (KIND == 1)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(da), "l"(db), "r"(IDESC), "r"(acc) : "memory");
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(da), "l"(db), "r"(IDESC), "r"(acc) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    mbar_wait(&bar, 0);
    unsigned long long c1 = clock64(), t1 = gtime();
    if (blockIdx.x == 0) *clk = Clk{c0, c1, t0, t1};
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ TMEM load
#define LD64(taddr, v, OP)                                                                                          \
  asm volatile(OP                                                                                                   \
               " {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26," \
               "%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51," \
               "%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"                                             \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),          \
                 "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),        \
                 "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),        \
                 "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]),        \
                 "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]),        \
                 "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),        \
                 "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),        \
                 "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])         \
               : "r"(taddr))

template <int PACK>
__global__ void __launch_bounds__(256, 1) tmem_ld_kernel(int iters, Clk* clk, uint32_t* sink) {
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int quad = warp & 3, half = warp >> 2;
  const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * 256);
  unsigned long long c0 = clock64(), t0 = gtime();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    // 256 columns per warp per iteration
#pragma unroll 1
    for (int c = 0; c < 256; c += (PACK ? 128 : 64)) {
      uint32_t v[64];
      if (PACK)
        LD64(base + (uint32_t)c, v, "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32");
      else
        LD64(base + (uint32_t)c, v, "tcgen05.ld.sync.aligned.32x32b.x64.b32");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 64; ++i) acc |= v[i];
    }
  }
  unsigned long long c1 = clock64(), t1 = gtime();
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1, t0, t1};
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ PRMT
__global__ void __launch_bounds__(1024, 1) prmt_kernel(int iters, Clk* clk, uint32_t* sink, uint32_t seed) {
  uint32_t t0 = seed * 0x9E3779B9u, t1 = t0 ^ 0x5bd1e995u;
  uint32_t x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = (threadIdx.x * 8 + u) * 0x01234567u;
  unsigned long long c0 = clock64(), g0 = gtime();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __byte_perm(t0, t1, x[u]) ^ t0;  // PRMT (+ LOP3 folded by ptxas? see SASS)
  }
  unsigned long long c1 = clock64(), g1 = gtime();
  uint32_t acc = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) acc ^= x[u];
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1, g0, g1};
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

// pure PRMT chains (no other ALU op): x = prmt(t0, x, s) with the selector
// in a separate register -> 32 PRMT per iteration per thread
__global__ void __launch_bounds__(1024, 1) prmt_only_kernel(int iters, Clk* clk, uint32_t* sink, uint32_t seed) {
  const uint32_t t0 = seed * 0x9E3779B9u;
  uint32_t x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = (threadIdx.x * 8 + u) * 0x01234567u;
  const uint32_t s = 0x3210u + (seed & 1);
  unsigned long long c0 = clock64(), g0 = gtime();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __byte_perm(x[u], t0, s ^ (uint32_t)r);
  }
  unsigned long long c1 = clock64(), g1 = gtime();
  uint32_t acc = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) acc ^= x[u];
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1, g0, g1};
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

// ------------------------------------------------------------------ smem LUT
// lane = query: table word (entry e, lane l) at e * 32 + l -> 32 distinct banks
// for any warp-uniform entry; 8 independent lookups in flight per thread.
__global__ void __launch_bounds__(1024, 1) smem_lut_kernel(int iters, Clk* clk, uint32_t* sink, uint32_t seed) {
  __shared__ uint32_t tab[256 * 32];  // 32 KB: 256 entries x 32 lanes
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t e[8], acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    e[u] = (seed + u * 77 + (threadIdx.x >> 5)) & 255;
    acc[u] = 0;
  }
  unsigned long long c0 = clock64(), g0 = gtime();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t v = tab[e[u] * 32 + lane];
      acc[u] += v;
      e[u] = (e[u] + 97 + u) & 255;  // warp-uniform next entry
    }
  }
  unsigned long long c1 = clock64(), g1 = gtime();
  uint32_t a = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) a ^= acc[u];
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1, g0, g1};
  if (a == 0x12345678u) sink[threadIdx.x] = a;
}

// ------------------------------------------------------------------ host
static int g_sms = 148;

template <class F>
static double timed(F launch, Clk* d_clk, double* mhz) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  Clk c{};
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) {
      best = ms;
      CK(cudaMemcpy(&c, d_clk, sizeof(Clk), cudaMemcpyDeviceToHost));
    }
  }
  CK(cudaGetLastError());
  *mhz = (double)(c.c1 - c.c0) / (double)(c.t1 - c.t0) * 1e3;
  return best * 1e-3;
}

// `pqs_peaks i8 [seconds]`: the int8 MMA peak only -- a burst (best of 5
// launches of ~20 ms) and a sustained figure (back-to-back launches for the
// given seconds, default 3, the regime of a kernel timed inside a long step)
static int i8_only(double seconds) {
  Clk* d_clk;
  CK(cudaMalloc(&d_clk, sizeof(Clk)));
  const int smem = (MM + MN) * 64;
  const int iters = 40000;
  double mhz = 0;
  auto launch = [&]() { mma_peak_kernel<0><<<g_sms, 128, smem>>>(iters, d_clk); };
  const double s = timed(launch, d_clk, &mhz);
  const double macs = (double)g_sms * iters * 8 * MM * MN * 32;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int nl = (int)(seconds / s) + 1;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < nl; ++i) launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  Clk c{};
  CK(cudaMemcpy(&c, d_clk, sizeof(Clk), cudaMemcpyDeviceToHost));
  const double mhz_last = (double)(c.c1 - c.c0) / (double)(c.t1 - c.t0) * 1e3;
  printf("{\"i8_mma\": {\"tops\": %.1f, \"sm_mhz\": %.0f, \"ms\": %.3f, \"shape\": \"M128 N256 K32 cta_group::1\"}, "
         "\"i8_mma_sustained\": {\"tops\": %.1f, \"seconds\": %.2f, \"launches\": %d, \"sm_mhz_last\": %.0f}}\n",
         2 * macs / s / 1e12, mhz, s * 1e3, 2 * macs * nl / (ms * 1e-3) / 1e12, ms * 1e-3, nl, mhz_last);
  return 0;
}

int main(int argc, char** argv) {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  g_sms = p.multiProcessorCount;
  if (argc > 1 && std::string(argv[1]) == "i8") return i8_only(argc > 2 ? atof(argv[2]) : 3.0);
  Clk* d_clk;
  uint32_t* sink;
  CK(cudaMalloc(&d_clk, sizeof(Clk)));
  CK(cudaMalloc(&sink, 1 << 16));
  printf("{\"device\": \"%s\", \"sm_count\": %d", p.name, g_sms);

  // ---- MMA peaks
  const int smem = (MM + MN) * 64;
  const char* names[3] = {"i8_mma", "f16_mma", "tf32_mma"};
  const double kper[3] = {32, 16, 8};
  for (int kind = 0; kind < 3; ++kind) {
    const int iters = kind == 0 ? 40000 : 20000;
    double mhz = 0;
    auto launch = [&]() {
      if (kind == 0) mma_peak_kernel<0><<<g_sms, 128, smem>>>(iters, d_clk);
      else if (kind == 1) mma_peak_kernel<1><<<g_sms, 128, smem>>>(iters, d_clk);
      else mma_peak_kernel<2><<<g_sms, 128, smem>>>(iters, d_clk);
    };
    const double s = timed(launch, d_clk, &mhz);
    const double macs = (double)g_sms * iters * 8 * MM * MN * kper[kind];
    const double per_clk_sm = macs / g_sms / (s * mhz * 1e6);
    printf(", \"%s\": {\"tops\": %.1f, \"macs_per_clk_sm\": %.1f, \"sm_mhz\": %.0f, \"shape\": \"M128 N256 K%d cta_group::1\", \"ms\": %.3f}",
           names[kind], 2 * macs / s / 1e12, per_clk_sm, mhz, (int)kper[kind], s * 1e3);
  }
  // ---- TMEM load
  for (int pack = 0; pack < 2; ++pack) {
    const int iters = 20000;
    double mhz = 0;
    auto launch = [&]() {
      if (pack) tmem_ld_kernel<1><<<g_sms, 256>>>(iters, d_clk, sink);
      else tmem_ld_kernel<0><<<g_sms, 256>>>(iters, d_clk, sink);
    };
    const double s = timed(launch, d_clk, &mhz);
    // per CTA per iteration: 8 warps x 256 columns x 32 lanes x 4 bytes of TMEM
    const double bytes = (double)g_sms * iters * 8 * 256 * 32 * 4;
    printf(", \"tmem_ld%s\": {\"tmem_bytes_per_clk_sm\": %.1f, \"reg_bytes_per_clk_sm\": %.1f, \"sm_mhz\": %.0f, \"op\": \"%s\"}",
           pack ? "_pack16" : "", bytes / g_sms / (s * mhz * 1e6), bytes / (pack ? 2 : 1) / g_sms / (s * mhz * 1e6), mhz,
           pack ? "tcgen05.ld.32x32b.x64.pack::16b (128 columns)" : "tcgen05.ld.32x32b.x64 (64 columns)");
  }
  // ---- PRMT
  for (int only = 0; only < 2; ++only) {
    const int iters = 20000;
    double mhz = 0;
    auto launch = [&]() {
      if (only) prmt_only_kernel<<<g_sms, 1024>>>(iters, d_clk, sink, 7);
      else prmt_kernel<<<g_sms, 1024>>>(iters, d_clk, sink, 7);
    };
    const double s = timed(launch, d_clk, &mhz);
    const double prmts = (double)g_sms * 1024 * iters * 32;
    const double per_clk = prmts / g_sms / (s * mhz * 1e6);
    printf(", \"%s\": {\"prmt_per_clk_sm\": %.1f, \"lut16_lookups_per_s\": %.4e, \"lut16_lookups_per_clk_sm\": %.1f, \"sm_mhz\": %.0f, \"note\": \"%s\"}",
           only ? "prmt" : "prmt_xor", per_clk, prmts * 2 / s, per_clk * 2, mhz,
           only ? "PRMT chains only; a 16-entry u8 LUT resolves 4 lookups with 2 PRMT"
                : "PRMT + LOP3 per step (ALU pipe shared)");
  }
  // ---- smem LUT
  {
    const int iters = 20000;
    double mhz = 0;
    auto launch = [&]() { smem_lut_kernel<<<g_sms, 1024>>>(iters, d_clk, sink, 3); };
    const double s = timed(launch, d_clk, &mhz);
    const double lookups = (double)g_sms * 1024 * iters * 8;
    printf(", \"smem_lut\": {\"lookups_per_s\": %.4e, \"lookups_per_clk_sm\": %.2f, \"sm_mhz\": %.0f, \"layout\": \"lane = query, 32 distinct banks, warp-uniform entry\"}",
           lookups / s, lookups / g_sms / (s * mhz * 1e6), mhz);
  }
  printf("}\n");
  return 0;
}
