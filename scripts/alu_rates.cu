// alu_rates.cu — per-op issue throughput on this GPU (measurement aid for the k-NN
// kernel's ALU roofline; "measure the sm_100 rate of IMAD.WIDE, IADD3
// and 64-bit compare ... and scale the floor if any of them is half-rate").
//
// Each kernel runs 8 independent dependency chains of one operation per thread
// (enough to cover the 4-cycle pipe latency), over a grid of 8 resident blocks of 256
// threads per SM.  Reports lane-ops/s and lane-ops per clock per SM (the nominal full
// rate is 128 = 4 SMSPs x 32 lanes).  Not part of the product; built by
// scripts/alu_rates.py with nvcc -arch sm_100a.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;        // independent chains per thread
constexpr int ITERS = 4096;  // iterations per chain

__global__ void k_ffma(float* out, float b, float c) {
    float a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fmnmx(float* out, float b, float c) {
    float a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
            asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c));
        }
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3-input fp32 max (FMNMX3 on sm_100a: the k-NN box test's per-axis gap)
__global__ void k_fmnmx3(float* out, float b, float c) {
    float a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
    float s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_iadd3(int* out, int b, int c) {
    int a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
        }
    int s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_wide(long long* out, int b, int c) {
    long long a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    const int x = b ^ (int)threadIdx.x;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(a[i]) : "r"(x), "r"(c));
    long long s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imnmx(int* out, int b, int c) {
    int a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("max.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            asm volatile("min.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
        }
    int s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 64-bit compare + select (setp.lt.s64 + selp.b64): the candidate test of the 2D path
__global__ void k_cmp64(long long* out, long long b, long long c) {
    long long a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i)
            asm volatile("{ .reg .pred p; setp.lt.s64 p, %0, %1; selp.b64 %0, %2, %0, p; }" : "+l"(a[i]) : "l"(b), "l"(c));
    long long s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// packed bf16x2 / f16x2 min + max (HMNMX2): candidate k-best list in packed halves
__global__ void k_hmnmx2_bf16(unsigned* out, unsigned b, unsigned c) {
    unsigned a[CH];
    for (int i = 0; i < CH; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("max.bf16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            asm volatile("min.bf16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
        }
    unsigned s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_hmnmx2_f16(unsigned* out, unsigned b, unsigned c) {
    unsigned a[CH];
    for (int i = 0; i < CH; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("max.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            asm volatile("min.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
        }
    unsigned s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// byte permute (PRMT): pairs the halves of two packed registers
__global__ void k_prmt(unsigned* out, unsigned b, unsigned c) {
    unsigned a[CH];
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("prmt.b32 %0, %0, %1, 0x5432;" : "+r"(a[i]) : "r"(b));
    unsigned s = 0;
    for (int i = 0; i < CH; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static double run(F launch, int blocks, int threads, double ops_per_thread) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();   // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return (double)blocks * threads * ops_per_thread / (best * 1e-3);
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int threads = 256, blocks = sms * 8;
    void* buf = nullptr;
    cudaMalloc(&buf, (size_t)blocks * threads * 8);
    const double per = (double)ITERS * CH;
    struct R { const char* name; double ops; } res[12];
    int nr = 0;
    res[nr++] = {"FFMA", run([&] { k_ffma<<<blocks, threads>>>((float*)buf, 1.0001f, 0.5f); }, blocks, threads, per)};
    res[nr++] = {"FMNMX", run([&] { k_fmnmx<<<blocks, threads>>>((float*)buf, 1.0f, 2.0f); }, blocks, threads, 2 * per)};
    res[nr++] = {"FMNMX3", run([&] { k_fmnmx3<<<blocks, threads>>>((float*)buf, 1.0f, 2.0f); }, blocks, threads, per)};
    res[nr++] = {"IMNMX", run([&] { k_imnmx<<<blocks, threads>>>((int*)buf, 3, 1 << 20); }, blocks, threads, 2 * per)};
    res[nr++] = {"IADD", run([&] { k_iadd3<<<blocks, threads>>>((int*)buf, 3, 5); }, blocks, threads, 2 * per)};
    res[nr++] = {"IMAD.WIDE", run([&] { k_imad_wide<<<blocks, threads>>>((long long*)buf, 3, 5); }, blocks, threads, per)};
    res[nr++] = {"ISETP64+SEL", run([&] { k_cmp64<<<blocks, threads>>>((long long*)buf, 1000, 7); }, blocks, threads, per)};
    res[nr++] = {"HMNMX2.BF16 (pairs)", run([&] { k_hmnmx2_bf16<<<blocks, threads>>>((unsigned*)buf, 0x3f003f00u, 0x40004000u); }, blocks, threads, 2 * per)};
    res[nr++] = {"HMNMX2.F16 (pairs)", run([&] { k_hmnmx2_f16<<<blocks, threads>>>((unsigned*)buf, 0x38003800u, 0x40004000u); }, blocks, threads, 2 * per)};
    res[nr++] = {"PRMT", run([&] { k_prmt<<<blocks, threads>>>((unsigned*)buf, 7u, 0u); }, blocks, threads, per)};
    printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"ops\": {", sms, clk_khz / 1e3);
    for (int i = 0; i < nr; ++i)
        printf("%s\"%s\": {\"lane_ops_per_s\": %.4g}", i ? ", " : "", res[i].name, res[i].ops);
    printf("}}\n");
    cudaFree(buf);
    return 0;
}
