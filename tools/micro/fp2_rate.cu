// Issue-rate microbenchmark of the packed-FP32 forms the interior kernel uses (sm_100a):
// cycles per warp instruction per SMSP for FADD2 / FFMA2 / FMUL2 in register and immediate
// forms, 8 independent chains per thread, 16 warps per SM.   nvcc -arch=sm_100a -O3 fp2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N_ITER 4096
typedef float2 V;

template <int OP>
__global__ void k(float* out, float a0, float b0, long long* cyc) {
  V x[8], y = make_float2(a0, b0), z = make_float2(b0, a0);
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(a0 + i, b0 - i);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __fadd2_rn(x[i], y);                          // FADD2 R, R
      if (OP == 1) x[i] = __ffma2_rn(x[i], make_float2(1.0001f, 1.0001f), y);   // FFMA2 R, imm, R
      if (OP == 2) x[i] = __ffma2_rn(x[i], z, y);                       // FFMA2 R, R, R
      if (OP == 3) x[i] = __fmul2_rn(x[i], make_float2(0.9999f, 0.9999f));       // FMUL2 R, imm
      if (OP == 4) x[i].x = __fadd_rn(x[i].x, y.x);                     // FADD scalar R, R
      if (OP == 5) x[i].x = __fmaf_rn(x[i].x, 1.0001f, y.x);            // FFMA scalar R, imm, R
      if (OP == 6) x[i] = __fadd2_rn(x[i], make_float2(0.5f, 0.5f));    // FADD2 R, imm
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 512 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const char* names[] = {"FADD2 r,r", "FFMA2 r,imm,r", "FFMA2 r,r,r", "FMUL2 r,imm", "FADD r,r", "FFMA r,imm,r", "FADD2 r,imm"};
  void (*ks[])(float*, float, float, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  for (int o = 0; o < 7; ++o) {
    ks[o]<<<148, 512>>>(out, 1.f, 2.f, cyc);
    ks[o]<<<148, 512>>>(out, 1.f, 2.f, cyc);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += c[i];
    avg /= 148;
    // 16 warps/SM = 4 warps per SMSP, each issuing 8*N_ITER instructions
    printf("%-16s %.3f cycles per warp instruction per SMSP\n", names[o], avg / (4.0 * 8 * N_ITER));
  }
  return 0;
}
