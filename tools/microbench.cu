// Microbenchmarks for the deposit design on sm_100a: DP/FP32 issue rate,
// correctly-rounded DP divide, global RED.F32, shared CAS-float and int atomics.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dp_mul_add(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(__dmul_rn(x0, a), 1e-9); x1 = __dadd_rn(__dmul_rn(x1, a), 1e-9);
    x2 = __dadd_rn(__dmul_rn(x2, a), 1e-9); x3 = __dadd_rn(__dmul_rn(x3, a), 1e-9);
    x4 = __dadd_rn(__dmul_rn(x4, a), 1e-9); x5 = __dadd_rn(__dmul_rn(x5, a), 1e-9);
    x6 = __dadd_rn(__dmul_rn(x6, a), 1e-9); x7 = __dadd_rn(__dmul_rn(x7, a), 1e-9);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void dp_div(double* out, int iters, double a) {
  double x0 = threadIdx.x + 1.0, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) { x0 = a / x0 + 1.0; x1 = a / x1 + 1.0; x2 = a / x2 + 1.0; x3 = a / x3 + 1.0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3;
}
__global__ void fp32_fma(float* out, int iters, float a) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    x0 = __fmaf_rn(x0, a, 1e-9f); x1 = __fmaf_rn(x1, a, 1e-9f); x2 = __fmaf_rn(x2, a, 1e-9f); x3 = __fmaf_rn(x3, a, 1e-9f);
    x4 = __fmaf_rn(x4, a, 1e-9f); x5 = __fmaf_rn(x5, a, 1e-9f); x6 = __fmaf_rn(x6, a, 1e-9f); x7 = __fmaf_rn(x7, a, 1e-9f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void red_spread(float* buf, unsigned mask, int iters) {
  unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) atomicAdd(buf + (hash(t * 7919u + i) & mask), 1.0f);
}
__global__ void red_tile(float* buf, unsigned mask, int iters) {
  // warp lanes hit 32 consecutive floats of a per-block window (deposit-flush-like)
  unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) atomicAdd(buf + ((blockIdx.x * 4096u + (i * 256u + threadIdx.x)) & mask), 1.0f);
}
__global__ void smem_cas_float(float* out, int iters) {
  __shared__ float tile[3456];
  for (int i = threadIdx.x; i < 3456; i += blockDim.x) tile[i] = 0;
  __syncthreads();
  unsigned t = threadIdx.x;
  for (int i = 0; i < iters; ++i) atomicAdd(&tile[hash(t * 31u + i) % 3456u], 1.0f);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = tile[5];
}
__global__ void smem_int_atom(int* out, int iters) {
  __shared__ int tile[3456];
  for (int i = threadIdx.x; i < 3456; i += blockDim.x) tile[i] = 0;
  __syncthreads();
  unsigned t = threadIdx.x;
  for (int i = 0; i < iters; ++i) atomicAdd(&tile[hash(t * 31u + i) % 3456u], 1);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = tile[5];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; float* f; int* ii; float* big;
  CK(cudaMalloc(&d, 1 << 26)); CK(cudaMalloc(&f, 1 << 26)); CK(cudaMalloc(&ii, 1 << 26));
  CK(cudaMalloc(&big, 64u << 20)); cudaMemset(big, 0, 64u << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  int blocks = sms * 8, th = 256, it = 4096;
  auto T = [&](const char* name, double ops, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %10.3f ms  %10.3e ops/s  %8.2f ops/clk/SM (@1.965GHz)\n", name, ms, ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / 1.965e9);
  };
  double n = (double)blocks * th;
  T("dp mul+add (ops)", n * it * 16, [&] { dp_mul_add<<<blocks, th>>>(d, it, 0.999999); });
  T("dp divide", n * (it / 4) * 4, [&] { dp_div<<<blocks, th>>>(d, it / 4, 3.0); });
  T("fp32 fma", n * it * 8, [&] { fp32_fma<<<blocks, th>>>(f, it, 0.9999f); });
  T("red.f32 spread 16MB", n * 256, [&] { red_spread<<<blocks, th>>>(big, (4u << 20) - 1, 256); });
  T("red.f32 spread 256KB", n * 256, [&] { red_spread<<<blocks, th>>>(big, (64u << 10) - 1, 256); });
  T("red.f32 tile", n * 256, [&] { red_tile<<<blocks, th>>>(big, (16u << 20) - 1, 256); });
  T("smem cas-float atomicAdd", n * 1024, [&] { smem_cas_float<<<blocks, th>>>(f, 1024); });
  T("smem int atomicAdd", n * 1024, [&] { smem_int_atom<<<blocks, th>>>(ii, 1024); });
  return 0;
}
