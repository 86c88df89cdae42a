// Minimal TMA probe: 4-D tiled load and reduce-add through a __grid_constant__
// tensor map, encoder from cudaGetDriverEntryPoint.  nvcc -arch=sm_100a.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tm_param, float *out, const CUtensorMap *tm_glob) {
    const CUtensorMap &tm = tm_glob ? *tm_glob : tm_param;
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t mbar;
    float *buf = reinterpret_cast<float *>(sm);
    if (MODE == 0) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)), "r"(12 * 10 * 6 * 6 * 4) : "memory");
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(7), "r"(7), "r"(3), "r"(0), "r"(su32(&mbar)) : "memory");
        }
        __syncthreads();
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(su32(&mbar)) : "memory");
        for (int i = threadIdx.x; i < 12 * 10 * 6 * 6; i += blockDim.x) out[i] = buf[i];
    } else {
        for (int i = threadIdx.x; i < 12 * 10 * 6 * 6; i += blockDim.x) buf[i] = 1.0f;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                         ::"l"(reinterpret_cast<uint64_t>(&tm)), "r"(7), "r"(7), "r"(3), "r"(0), "r"(su32(buf)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
}

int main() {
    const int nx = 32, ny = 32, nz = 16, nl = 6;
    std::vector<float> h((size_t)nx * ny * nz * nl);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 12 * 10 * 6 * 6 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    printf("entry point: %s q=%d p=%p\n", cudaGetErrorString(e), (int)q, p);
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    cuuint64_t dims[4] = {nx, ny, nz, nl};
    cuuint64_t str[3] = {nx * 4ull, nx * ny * 4ull, nx * ny * nz * 4ull};
    cuuint32_t box[4] = {12, 10, 6, 6}, es[4] = {1, 1, 1, 1};
    CUresult r = ((EncodeFn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    CUtensorMap *dtm;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    for (int v = 0; v < 2; ++v) {
    probe<0><<<1, 128, 20000>>>(tm, o, v ? dtm : nullptr);
    e = cudaDeviceSynchronize();
    printf("variant %s load: %s\n", v ? "global" : "param", cudaGetErrorString(e));
    if (e != cudaSuccess) break;
    }
    std::vector<float> ho(12 * 10 * 6 * 6);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    // expected element (x=7+a, y=7+b, z=3+c, l)
    int bad = 0;
    for (int l = 0; l < 6; ++l) for (int c = 0; c < 6; ++c) for (int b = 0; b < 10; ++b) for (int a = 0; a < 12; ++a) {
        float want = h[(((size_t)l * nz + 3 + c) * ny + 7 + b) * nx + 7 + a];
        if (ho[((l * 6 + c) * 10 + b) * 12 + a] != want) ++bad;
    }
    printf("load mismatches: %d\n", bad);
    probe<1><<<1, 128, 20000>>>(tm, o, nullptr);
    e = cudaDeviceSynchronize();
    printf("reduce: %s\n", cudaGetErrorString(e));
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("after reduce: %f (expect %f)\n", h[(((size_t)0 * nz + 3) * ny + 7) * nx + 7], (float)((3 * ny + 7) * nx + 7) + 1.0f);
    return 0;
}
