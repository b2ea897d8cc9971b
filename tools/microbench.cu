// microbench.cu -- B200 pipe-throughput probes used to set the rooflines in DESIGN.md.
//   FFMA  (3-register form, independent chains)  -> CUDA-core FP32 peak
//   FFMA2 (fma.rn.f32x2)                           -> packed FP32 peak
//   HMMA  (mma.sync m16n8k16 bf16 -> fp32)         -> legacy warp-level tensor path
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 0.001f + i;
    float x = a + threadIdx.x, y = b;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], x, y);
        x += 1e-7f;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// broadcast-operand form used by the SpMM inner loop: acc[r][c] += v[r] * b[c]
__global__ void ffma_outer_kernel(float* out, const float* src) {
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
    float v[4], b[8];
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = src[r] + threadIdx.x;
#pragma unroll
    for (int c = 0; c < 8; ++c) b[c] = src[4 + c] - threadIdx.x;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(v[r], b[c], acc[r][c]);
#pragma unroll
        for (int c = 0; c < 8; ++c) b[c] = __int_as_float(__float_as_int(b[c]) ^ 1);
    }
    float s = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) s += acc[r][c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

__global__ void ffma2_kernel(float* out, float a, float b) {
    unsigned long long acc[8];
    for (int i = 0; i < 8; ++i) {
        float2 t = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
        acc[i] = *reinterpret_cast<unsigned long long*>(&t);
    }
    float2 xx = make_float2(a, a + 1), yy = make_float2(b, b);
    unsigned long long x = *reinterpret_cast<unsigned long long*>(&xx);
    unsigned long long y = *reinterpret_cast<unsigned long long*>(&yy);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) ffma2(acc[i], x, y);
        x ^= 1ull;
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) {
        float2 t = *reinterpret_cast<float2*>(&acc[i]);
        s += t.x + t.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void hmma_kernel(float* out, uint32_t seed) {
    float d[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) d[j][e] = 0.f;
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = seed * 11, b1 = seed * 13;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) s += d[j][e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_kernel(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    float* out;
    CHK(cudaMalloc(&out, size_t(sms) * 8 * 1024 * sizeof(float)));
    float* src;
    CHK(cudaMalloc(&src, 64 * sizeof(float)));
    CHK(cudaMemset(src, 0, 64 * sizeof(float)));
    const int blocks = sms * 8, threads = 256;   // 64 warps / SM
    double n_thr = double(blocks) * threads;

    float ms = time_kernel([&] { ffma_kernel<<<blocks, threads>>>(out, 1.0001f, 0.5f); });
    double tf = n_thr * ITERS * 16 * 2 / (ms * 1e-3) / 1e12;
    printf("{\"probe\": \"ffma\", \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d, \"attr_clock_mhz\": %d}\n", tf, ms, sms,
           clk_khz / 1000);
    ms = time_kernel([&] { ffma_outer_kernel<<<blocks, threads>>>(out, src); });
    tf = n_thr * ITERS * 32 * 2 / (ms * 1e-3) / 1e12;
    printf("{\"probe\": \"ffma_outer_4x8\", \"tflops\": %.2f, \"ms\": %.3f}\n", tf, ms);
    ms = time_kernel([&] { ffma2_kernel<<<blocks, threads>>>(out, 1.0001f, 0.5f); });
    tf = n_thr * ITERS * 8 * 4 / (ms * 1e-3) / 1e12;
    printf("{\"probe\": \"ffma2\", \"tflops\": %.2f, \"ms\": %.3f}\n", tf, ms);
    ms = time_kernel([&] { hmma_kernel<<<blocks, threads>>>(out, 12345u); });
    tf = n_thr / 32 * (ITERS / 4) * 4 * (16.0 * 8 * 16 * 2) / (ms * 1e-3) / 1e12;
    printf("{\"probe\": \"hmma_m16n8k16_bf16\", \"tflops\": %.2f, \"ms\": %.3f}\n", tf, ms);
    return 0;
}
