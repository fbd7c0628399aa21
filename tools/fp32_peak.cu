// fp32_peak.cu -- measure the B200 FP32 / ALU / MUFU issue ceilings that bound
// the filter kernels.  Every op is an asm volatile PTX
// instruction so that nvcc cannot contract or fold the chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048
#define ACC 8

#define KERNEL(NAME, BODY)                                                   \
  __global__ void NAME(float* out, float b, float c) {                      \
    float a[ACC], bb[ACC], cc[ACC];                                          \
    _Pragma("unroll") for (int k = 0; k < ACC; ++k) {                        \
      a[k] = threadIdx.x * 1e-3f + k; bb[k] = b + k * 1e-3f; cc[k] = c + k;  \
    }                                                                        \
    for (int i = 0; i < ITERS; ++i) {                                        \
      _Pragma("unroll") for (int k = 0; k < ACC; ++k) { BODY; }              \
    }                                                                        \
    float s = 0;                                                             \
    _Pragma("unroll") for (int k = 0; k < ACC; ++k) s += a[k] + bb[k] + cc[k]; \
    if (s == 12345.f) out[threadIdx.x] = s;                                  \
  }

// FFMA, register a, b and immediate c
KERNEL(k_ffma_imm, asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k])))
// FFMA, three registers, b shared (reuse cache can help)
KERNEL(k_ffma_reg, asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(bb[0]), "f"(cc[k])))
// FFMA, three distinct registers per instruction
KERNEL(k_ffma_reg3, asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(bb[k]), "f"(cc[k])))
// FADD register + register
KERNEL(k_fadd, asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[k]) : "f"(bb[k])))
// FMUL register * register
KERNEL(k_fmul, asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[k]) : "f"(bb[k])))
// FMNMX (ALU pipe)
KERNEL(k_fmax, asm volatile("max.f32 %0, %0, %1;" : "+f"(a[k]) : "f"(bb[k])))
// FSEL-like select on predicate (ALU pipe)
KERNEL(k_fsetp_sel, asm volatile("{.reg .pred p; setp.lt.f32 p, %0, %1; selp.f32 %0, %0, %2, p;}" : "+f"(a[k]) : "f"(bb[k]), "f"(cc[k])))
// MUFU.RSQ
KERNEL(k_rsq, asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a[k])))
// MUFU.RCP
KERNEL(k_rcp, asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[k])); asm volatile("add.f32 %0, %0, 0f3F000000;" : "+f"(a[k])))
// 1 FFMA (imm) + 1 FADD interleaved on independent chains
KERNEL(k_ffma_fadd, asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k]));
       asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(cc[k]) : "f"(bb[k])))
// 1 FFMA (imm) + 1 FMNMX interleaved
KERNEL(k_ffma_fmax, asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k]));
       asm volatile("max.f32 %0, %0, %1;" : "+f"(cc[k]) : "f"(bb[k])))
// 4 FFMA (imm) + 1 MUFU.RSQ
KERNEL(k_ffma4_rsq, asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k]));
       asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k]));
       asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k]));
       asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(a[k]) : "f"(bb[k]));
       asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(cc[k])))

// packed FP32 pairs (sm_100: fma/add/mul.rn.f32x2 -> FFMA2 / FADD2 / FMUL2)
#define K2KERNEL(NAME, BODY)                                                 \
  __global__ void NAME(float* out, float b, float c) {                      \
    unsigned long long a[ACC], bb[ACC], cc[ACC];                             \
    _Pragma("unroll") for (int k = 0; k < ACC; ++k) {                        \
      float2 x = make_float2(threadIdx.x * 1e-3f + k, k);                    \
      float2 y = make_float2(b + k * 1e-3f, b);                              \
      float2 z = make_float2(c + k, c);                                      \
      a[k] = *(unsigned long long*)&x; bb[k] = *(unsigned long long*)&y;     \
      cc[k] = *(unsigned long long*)&z;                                      \
    }                                                                        \
    for (int i = 0; i < ITERS; ++i) {                                        \
      _Pragma("unroll") for (int k = 0; k < ACC; ++k) { BODY; }              \
    }                                                                        \
    float s = 0;                                                             \
    _Pragma("unroll") for (int k = 0; k < ACC; ++k) {                        \
      float2 x = *(float2*)&a[k]; s += x.x + x.y; }                          \
    if (s == 12345.f) out[threadIdx.x] = s;                                  \
  }
K2KERNEL(k_ffma2, asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(bb[k]), "l"(cc[k])))
// Horner-like: a = a * x + c with x, c shared by all chains (register reuse)
K2KERNEL(k_ffma2_shared, asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(bb[0]), "l"(cc[0])))
// a = a * a + c_shared
K2KERNEL(k_ffma2_sq, asm volatile("fma.rn.f32x2 %0, %0, %0, %1;" : "+l"(a[k]) : "l"(cc[0])))
K2KERNEL(k_fadd2, asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[k]) : "l"(bb[k])))
K2KERNEL(k_fmul2, asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[k]) : "l"(bb[k])))
// 1 FFMA2 + 1 FFMA interleaved
K2KERNEL(k_ffma2_ffma, asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(bb[k]), "l"(cc[k]));
         asm volatile("{.reg .f32 lo, hi; mov.b64 {lo, hi}, %0; fma.rn.f32 lo, lo, lo, 0f3F000000; mov.b64 %0, {lo, hi};}" : "+l"(cc[k])))

// integer kernels on packed bytes
#define IKERNEL(NAME, BODY)                                                  \
  __global__ void NAME(float* out, float b, float c) {                      \
    unsigned a[ACC], bb[ACC];                                                \
    _Pragma("unroll") for (int k = 0; k < ACC; ++k) {                        \
      a[k] = threadIdx.x * 7919u + k; bb[k] = 0x01020304u * (k + 1);         \
    }                                                                        \
    for (int i = 0; i < ITERS; ++i) {                                        \
      _Pragma("unroll") for (int k = 0; k < ACC; ++k) { BODY; }              \
    }                                                                        \
    unsigned s = 0;                                                          \
    _Pragma("unroll") for (int k = 0; k < ACC; ++k) s += a[k];               \
    if (s == 12345u) out[threadIdx.x] = s;                                   \
  }
IKERNEL(k_vabsdiff4, asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %0, %0;" : "+r"(a[k]) : "r"(bb[k])))
IKERNEL(k_dp4a, asm volatile("dp4a.u32.u32 %0, %1, %0, %0;" : "+r"(a[k]) : "r"(bb[k])))
IKERNEL(k_iadd, asm volatile("add.u32 %0, %1, %0;" : "+r"(a[k]) : "r"(bb[k])))

template <typename F>
float timeit(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 10;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  float* out;
  cudaMalloc(&out, 4096);
  const int blocks = sms * 8, threads = 256;
  const double n = (double)blocks * threads * ITERS * ACC;   // instructions (thread level) per "op slot"
  printf("{\"sms\": %d", sms);
#define RUN(K, LABEL, PER) { float ms = timeit([&] { K<<<blocks, threads>>>(out, 0.999f, 0.5f); }); \
    printf(", \"%s\": %.3f", LABEL, (PER) * n / ms / 1e9); }
  RUN(k_ffma_imm, "ffma_imm_Tinst_per_s", 1)
  RUN(k_ffma_reg, "ffma_reg_Tinst_per_s", 1)
  RUN(k_ffma_reg3, "ffma_reg3_Tinst_per_s", 1)
  RUN(k_fadd, "fadd_Tinst_per_s", 1)
  RUN(k_fmul, "fmul_Tinst_per_s", 1)
  RUN(k_fmax, "fmnmx_Tinst_per_s", 1)
  RUN(k_fsetp_sel, "fsetp_fsel_Tinst_per_s", 2)
  RUN(k_rsq, "mufu_rsq_Tinst_per_s", 1)
  RUN(k_rcp, "mufu_rcp_plus_fadd_Tinst_per_s", 2)
  RUN(k_ffma_fadd, "ffma_plus_fadd_Tinst_per_s", 2)
  RUN(k_ffma_fmax, "ffma_plus_fmnmx_Tinst_per_s", 2)
  RUN(k_ffma4_rsq, "4ffma_plus_rsq_Tinst_per_s", 5)
  RUN(k_ffma2, "ffma2_Tinst_per_s", 1)
  RUN(k_ffma2_shared, "ffma2_shared_xc_Tinst_per_s", 1)
  RUN(k_ffma2_sq, "ffma2_sq_Tinst_per_s", 1)
  RUN(k_fadd2, "fadd2_Tinst_per_s", 1)
  RUN(k_fmul2, "fmul2_Tinst_per_s", 1)
  RUN(k_ffma2_ffma, "ffma2_plus_ffma_Tinst_per_s", 2)
  RUN(k_vabsdiff4, "vabsdiff4_Tinst_per_s", 1)
  RUN(k_dp4a, "idp4a_Tinst_per_s", 1)
  RUN(k_iadd, "iadd_Tinst_per_s", 1)
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf(", \"clock_khz_attr\": %d, \"note\": \"thread-instructions per second; FFMA flops = 2x, FFMA2 flops = 4x\"}\n", clk);
  return 0;
}
