// Microbenchmark: sustained issue throughput of each MUFU op (and FFMA) on
// sm_100a, in ops per SM clock -- the denominator of bench.py's roofline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bench tools/mufu_bench.cu
//   tools/mufu_bench > profiles/r02_mufu_peak.json
// Cycles are measured in the kernel (clock64 per block, one resident wave:
// 8 blocks x 256 threads per SM), so the figure does not depend on which SM
// clock the driver picked; the CUDA-event time is reported beside it.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define OP_KERNEL(NAME, ASM)                                                    \
__global__ void NAME(float* out, long long* cyc, int iters) {                   \
    float x[8];                                                                 \
    for (int i = 0; i < 8; ++i) x[i] = 0.5f + 0.001f * (threadIdx.x + i);       \
    __syncthreads();                                                            \
    const long long t0 = clock64();                                             \
    for (int it = 0; it < iters; ++it) {                                        \
        _Pragma("unroll") for (int i = 0; i < 8; ++i) {                         \
            float y; asm volatile(ASM : "=f"(y) : "f"(x[i])); x[i] = y;         \
        }                                                                       \
    }                                                                           \
    __syncthreads();                                                            \
    const long long t1 = clock64();                                             \
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];                         \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                             \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                            \
}
OP_KERNEL(k_ex2, "ex2.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_lg2, "lg2.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_sqrt, "sqrt.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_rsqrt, "rsqrt.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_sin, "sin.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_cos, "cos.approx.ftz.f32 %0, %1;")
OP_KERNEL(k_tanh, "tanh.approx.f32 %0, %1;")
OP_KERNEL(k_ffma, "fma.rn.f32 %0, %1, 0f3F800001, 0f3A800000;")

typedef void (*kfn)(float*, long long*, int);
int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, dev);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float* out;
    long long* cyc;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    std::vector<long long> h(blocks);
    struct { const char* name; kfn f; } ks[] = {{"ex2", k_ex2}, {"lg2", k_lg2}, {"sqrt", k_sqrt},
        {"rsqrt", k_rsqrt}, {"sin", k_sin}, {"cos", k_cos}, {"tanh", k_tanh},
        {"ffma", k_ffma}};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"nominal_mhz\": %d, \"blocks_per_sm\": 8, \"threads\": %d, "
           "\"what\": \"ops per SM clock (clock64 in-kernel, max block cycles) and at the event time\", "
           "\"ops\": {", prop.name, sms, clk / 1000, threads);
    bool first = true;
    for (auto& k : ks) {
        k.f<<<blocks, threads>>>(out, cyc, 64);
        cudaEventRecord(a);
        k.f<<<blocks, threads>>>(out, cyc, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaMemcpy(h.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
        const long long cmax = *std::max_element(h.begin(), h.end());
        const double per_sm = (double)threads * 8 * iters * 8;  // one wave: 8 blocks per SM
        const double per_clk = per_sm / (double)cmax;
        const double eff_mhz = (double)cmax / (ms * 1e-3) / 1e6;
        printf("%s\"%s\": {\"ops_per_clk_per_sm\": %.3f, \"ms\": %.4f, \"cycles\": %lld, \"implied_sm_mhz\": %.0f}",
               first ? "" : ", ", k.name, per_clk, ms, cmax, eff_mhz);
        first = false;
    }
    printf("}}\n");
    return 0;
}
