// TMA probe, one mode per process (argv[1]): 0 = 1-D cp.async.bulk (no tensor
// map), 1 = 2-D tensor map in param space, 2 = 2-D tensor map in global
// memory, 3 = 4-D param (the advance kernel's shape).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
__constant__ unsigned c_box_bytes;
__constant__ int c_coord[3];
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait0(uint64_t *m) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(su32(m)) : "memory");
}
__global__ void k(int mode, const __grid_constant__ CUtensorMap tm, const CUtensorMap *gtm, const float *src, float *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t mbar;
    float *buf = reinterpret_cast<float *>(sm);
    const unsigned bytes = mode == 0 ? 4096 : (mode == 3 ? c_box_bytes : 16 * 8 * 4);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)), "r"(bytes) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(buf)), "l"(src), "r"(bytes), "r"(su32(&mbar)) : "memory");
        else if (mode == 1)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(su32(&mbar)) : "memory");
        else if (mode == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(gtm)), "r"(0), "r"(0), "r"(su32(&mbar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c_coord[0]), "r"(c_coord[1]), "r"(c_coord[2]), "r"(0), "r"(su32(&mbar)) : "memory");
    }
    wait0(&mbar);
    for (unsigned i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char **argv) {
    const int mode = atoi(argv[1]);
    const int nx = 32, ny = 32, nz = 16, nl = 6;
    std::vector<float> h((size_t)nx * ny * nz * nl);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 1 << 16);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    CUresult r;
    if (mode == 3) {
        cuuint64_t dims[4] = {nx, ny, nz, nl}, str[3] = {nx * 4ull, nx * ny * 4ull, nx * ny * nz * 4ull};
        cuuint32_t box[4] = {(cuuint32_t)atoi(argv[2]), (cuuint32_t)atoi(argv[3]), (cuuint32_t)atoi(argv[4]), (cuuint32_t)atoi(argv[5])}, es[4] = {1, 1, 1, 1};
        unsigned bb = box[0] * box[1] * box[2] * box[3] * 4;
        int cc[3] = {atoi(argv[6]), atoi(argv[7]), atoi(argv[8])};
        cudaMemcpyToSymbol(c_coord, cc, 12);
        cudaMemcpyToSymbol(c_box_bytes, &bb, 4);
        r = ((EncodeFn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, atoi(argv[9]) ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[2] = {nx, ny * nz * nl}, str[1] = {nx * 4ull};
        cuuint32_t box[2] = {16, 8}, es[2] = {1, 1};
        r = ((EncodeFn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    CUtensorMap *g;
    cudaMalloc(&g, sizeof(tm));
    cudaMemcpy(g, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    k<<<1, 128, 32768>>>(mode, tm, g, d, o);
    cudaError_t e = cudaDeviceSynchronize();
    float v[4];
    cudaMemcpy(v, o, 16, cudaMemcpyDeviceToHost);
    printf("mode %d encode %d: %s  out[0..3] = %g %g %g %g\n", mode, (int)r, cudaGetErrorString(e), v[0], v[1], v[2], v[3]);
    return 0;
}
