// Shared-memory float add on sm_100a: which SASS does each spelling compile
// to, and what does it cost?  (atomicAdd on a shared pointer compiles to an
// ATOMS.CAST.SPIN loop; does red/atom through a generic address do better?)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_fadd_probe smem_fadd_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters) {
    __shared__ float s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 0.f;
    __syncthreads();
    const int t = threadIdx.x;
    float v = 1.0f + t * 1e-3f;
    for (int i = 0; i < iters; ++i) {
        const int idx = (t * 7 + i * 13) & 1023;
        float *p = &s[idx];
        if (MODE == 0) {
            atomicAdd(p, v);                                  // shared CAS loop
        } else if (MODE == 1) {
            unsigned a = (unsigned)__cvta_generic_to_shared(p);
            asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
        } else if (MODE == 2) {
            float *g = p;
            asm volatile("" : "+l"(g));                       // hide the state space
            asm volatile("red.add.f32 [%0], %1;" ::"l"(g), "f"(v) : "memory");
        } else if (MODE == 3) {
            // plain read-add-write (no atomicity; lower bound)
            s[idx] = s[idx] + v;
        }
    }
    __syncthreads();
    float acc = 0.f;
    for (int i = t; i < 1024; i += blockDim.x) acc += s[i];
    atomicAdd(out, acc);
}

template <int MODE>
float run(const char *name, int blocks, int iters, float *d) {
    cudaMemset(d, 0, sizeof(float));
    k<MODE><<<blocks, 256>>>(d, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<blocks, 256>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    float h; cudaMemcpy(&h, d, sizeof(float), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    double ops = (double)blocks * 256 * iters;
    printf("%-34s %8.3f ms  %9.3e adds/s  sum %.6e  %s\n", name, ms, ops / ms * 1e3, h,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    return ms;
}

int main() {
    float *d;
    cudaMalloc(&d, sizeof(float));
    const int blocks = 148 * 8, iters = 4096;
    run<0>("atomicAdd(shared float*)", blocks, iters, d);
    run<1>("red.shared.add.f32", blocks, iters, d);
    run<2>("red.add.f32 (generic address)", blocks, iters, d);
    run<3>("plain read-add-write (racy)", blocks, iters, d);
    return 0;
}
