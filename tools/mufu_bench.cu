// Microbenchmark: sustained throughput of each MUFU op (and FFMA) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bench mufu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define OP_KERNEL(NAME, ASM)                                                    \
__global__ void NAME(float* out, int iters) {                                   \
    float x[8];                                                                 \
    for (int i = 0; i < 8; ++i) x[i] = 0.5f + 0.001f * (threadIdx.x + i);       \
    for (int it = 0; it < iters; ++it) {                                        \
        _Pragma("unroll") for (int i = 0; i < 8; ++i) {                         \
            float y; asm volatile(ASM : "=f"(y) : "f"(x[i])); x[i] = y;         \
        }                                                                       \
    }                                                                           \
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];                         \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                             \
}
OP_KERNEL(k_ex2, "ex2.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_lg2, "lg2.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_sqrt, "sqrt.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_rsqrt, "rsqrt.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_sin, "sin.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_cos, "cos.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_rcp, "rcp.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_tanh, "tanh.approx.f32 %0, %1;")
OP_KERNEL(k_ffma, "fma.rn.f32 %0, %1, 0f3F800001, 0f3A800000;")

typedef void (*kfn)(float*, int);
int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float* out;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    struct { const char* name; kfn f; } ks[] = {{"ex2", k_ex2}, {"lg2", k_lg2}, {"sqrt", k_sqrt},
        {"rsqrt", k_rsqrt}, {"sin", k_sin}, {"cos", k_cos}, {"rcp", k_rcp}, {"tanh", k_tanh},
        {"ffma", k_ffma}};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (auto& k : ks) {
        k.f<<<blocks, threads>>>(out, 64);
        cudaEventRecord(a);
        k.f<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters * 8;
        double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("%-6s %8.3f ms  %7.2f ops/clk/SM (at %d MHz nominal)\n", k.name, ms, per_clk_sm, clk / 1000);
    }
    return 0;
}
