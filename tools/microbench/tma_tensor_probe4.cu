// Probe: the K1b sequence (two boxes on one barrier, the mirror box partially out of range)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int x0, int x1, int boff_f2) {
#ifdef GDC
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    extern __shared__ __align__(128) float sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(2 * 16 * 4 * 256) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(sm)), "l"(&tm), "r"(x0), "r"(0), "r"(smem_u32(&bar)) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(sm + 2 * boff_f2)), "l"(&tm), "r"(x1), "r"(0), "r"(smem_u32(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) { out[i] = sm[i]; out[4096 + i] = sm[2 * boff_f2 + i]; }
}
int main(int argc, char** argv) {
    const int N = 256, rows = 1024;
    const int boff = argc > 1 ? atoi(argv[1]) : 2064;
    std::vector<float> h((size_t)rows * 2 * N);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 2 * 4096 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap tm;
    cuuint64_t dims[2] = {2 * (cuuint64_t)N, (cuuint64_t)rows}; cuuint64_t strides[1] = {2 * (cuuint64_t)N * 4};
    cuuint32_t box[2] = {16, 256}, es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = (2 * boff + 2 * 2048) * 4 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int x0 = 0, x1 = argc > 2 ? atoi(argv[2]) : 498;
    k<<<1, 256, smem>>>(tm, o, x0, x1, boff);
    cudaError_t e = cudaDeviceSynchronize();
    printf("encode %d boff %d x1 %d kernel %s\n", (int)r, boff, x1, cudaGetErrorString(e));
    return 0;
}
