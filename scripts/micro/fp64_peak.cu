// FP64 peak probes on B200: DMMA (mma.sync m16n8k4 / m16n8k8 / m16n8k16 f64) vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_k4(double* out, int iters) {
  double c[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = 1.0 + a0, b0 = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_k16(double* out, int iters) {
  double c[8][4] = {};
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma(double* out, int iters) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  double s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    dim3 g(sms * 2), b(32 * warps);
    dmma_k4<<<g, b>>>(out, 16); cudaEventRecord(e0); dmma_k4<<<g, b>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 4 * 8 * (double)iters * g.x * (b.x / 32);
    printf("DMMA m16n8k4  warps/CTA=%2d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    dmma_k16<<<g, b>>>(out, 16); cudaEventRecord(e0); dmma_k16<<<g, b>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 8 * (double)iters * g.x * (b.x / 32);
    printf("DMMA m16n8k16 warps/CTA=%2d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    dfma<<<g, b>>>(out, 16); cudaEventRecord(e0); dfma<<<g, b>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * (double)iters * g.x * b.x;
    printf("DFMA          warps/CTA=%2d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
