// Issue rate of the packed fp32 instructions (FADD2 / FFMA2, sm_100a) against
// their scalar forms: the same number of fp32 operations per thread either as
// 2n scalar or n packed instructions, 8 independent chains per thread.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f32x2_probe f32x2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 r;
    asm volatile("{ .reg .b64 ra, rb, rr;\n\t mov.b64 ra, {%2,%3};\n\t mov.b64 rb, {%4,%5};\n\t add.rn.f32x2 rr, ra, rb;\n\t"
                 " mov.b64 {%0,%1}, rr; }"
                 : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm volatile("{ .reg .b64 ra, rb, rc, rr;\n\t mov.b64 ra, {%2,%3};\n\t mov.b64 rb, {%4,%5};\n\t mov.b64 rc, {%6,%7};\n\t"
                 " fma.rn.f32x2 rr, ra, rb, rc;\n\t mov.b64 {%0,%1}, rr; }"
                 : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

template <int MODE>
__global__ void k(float2* out, float2 seed, int iters) {
    float2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = make_float2(seed.x + j + threadIdx.x, seed.y - j);
    const float2 w = make_float2(seed.y, seed.x);
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (MODE == 0) {  // scalar adds
                    asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(v[j].x) : "f"(w.x));
                    asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(v[j].y) : "f"(w.y));
                } else if (MODE == 1) {
                    v[j] = add2(v[j], w);
                } else if (MODE == 2) {  // scalar fmas
                    asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[j].x) : "f"(w.x), "f"(w.y));
                    asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[j].y) : "f"(w.y), "f"(w.x));
                } else {
                    v[j] = fma2(v[j], w, w);
                }
            }
        }
    }
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 8; ++j) { s.x += v[j].x; s.y += v[j].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, float2* d) {
    const int blocks = 148 * 8, threads = 256, iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<blocks, threads>>>(d, make_float2(1e-3f, 2e-3f), 10);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(d, make_float2(1e-3f, 2e-3f), iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 64 * 2;  // fp32 operations (an fma counts once)
    printf("%-12s %8.3f ms  %7.2f T fp32-op/s\n", name, ms, ops / ms / 1e9);
}

int main() {
    float2* d; cudaMalloc(&d, 148 * 8 * 256 * sizeof(float2));
    run<0>("FADD", d); run<1>("FADD2", d); run<2>("FFMA", d); run<3>("FFMA2", d);
    run<0>("FADD", d); run<1>("FADD2", d); run<2>("FFMA", d); run<3>("FFMA2", d);
    return 0;
}
