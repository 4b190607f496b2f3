// Throughput microbenchmarks for the B200 design decision:
// FP32 FFMA, packed FFMA2 (fma.rn.f32x2), MUFU ex2, and legacy mma.sync
// (tf32 m16n8k8, f16/bf16 m16n8k16) on sm_100a.  Dev tooling, not product.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

#define ITERS 4096

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&bv);
  for (int i = 0; i < 8; i++) { float2 t = make_float2(threadIdx.x*0.001f+i, i); x[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  }
  float s = 0; for (int i = 0; i < 8; i++) { float2 t = *reinterpret_cast<float2*>(&x[i]); s += t.x + t.y; }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ex2(float* out, float a) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-6f + i * 1e-3f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i])); x[i] = y * a; }
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_mma_tf32(float* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; i++) a[i] = __float_as_uint(1.0f + threadIdx.x);
  for (int i = 0; i < 2; i++) b[i] = __float_as_uint(0.5f);
  float c[8][4] = {};
  for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0; for (int j = 0; j < 8; j++) for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 12345.f) out[0] = s;
}

template <bool BF>
__global__ void k_mma_16(float* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; i++) a[i] = 0x3c003c00u + threadIdx.x;
  for (int i = 0; i < 2; i++) b[i] = 0x3c003c00u;
  float c[8][4] = {};
  for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (BF)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  float s = 0; for (int j = 0; j < 8; j++) for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 12345.f) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4);
  printf("SMs=%d clock_khz=%d\n", sms, clk);
  for (int tpb : {256, 512, 1024}) {
    dim3 g(sms * 4), blk(tpb);
    double thr = (double)g.x * tpb;
    float ms = timeit([&] { k_ffma<<<g, blk>>>(out, 0.999f, 0.001f); });
    printf("tpb=%d FFMA   : %.1f TFLOP/s\n", tpb, thr * ITERS * 8 * 2 / ms / 1e9);
    ms = timeit([&] { k_ffma2<<<g, blk>>>(out, 0.999f, 0.001f); });
    printf("tpb=%d FFMA2  : %.1f TFLOP/s (fp32 flops)\n", tpb, thr * ITERS * 8 * 4 / ms / 1e9);
    ms = timeit([&] { k_ex2<<<g, blk>>>(out, 0.999f); });
    printf("tpb=%d EX2    : %.2f Tex2/s\n", tpb, thr * ITERS * 8 / ms / 1e9);
    double warps = thr / 32;
    ms = timeit([&] { k_mma_tf32<<<g, blk>>>(out); });
    printf("tpb=%d mma tf32 m16n8k8 : %.1f TFLOP/s\n", tpb, warps * (ITERS / 4) * 8 * 16 * 8 * 8 * 2 / ms / 1e9);
    ms = timeit([&] { k_mma_16<false><<<g, blk>>>(out); });
    printf("tpb=%d mma f16 m16n8k16 : %.1f TFLOP/s\n", tpb, warps * (ITERS / 4) * 8 * 16 * 8 * 16 * 2 / ms / 1e9);
    ms = timeit([&] { k_mma_16<true><<<g, blk>>>(out); });
    printf("tpb=%d mma bf16 m16n8k16: %.1f TFLOP/s\n", tpb, warps * (ITERS / 4) * 8 * 16 * 8 * 16 * 2 / ms / 1e9);
  }
  cudaError_t e = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
