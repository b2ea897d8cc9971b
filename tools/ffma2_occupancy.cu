// FFMA2 outer-product throughput vs resident warps (tools only): acc[SUB][4][8] += v[4] (broadcast) x
// b[8] (pairs), the K3 inner-loop pattern with registers only, at 4 / 8 / 16 warps per scheduler.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int SUB>
__global__ void outer2(float* out, const float* src) {
    float2 acc[SUB][4][4];
#pragma unroll
    for (int q = 0; q < SUB; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[q][r][c] = make_float2(0.f, 0.f);
    float v[4];
    float2 b[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = src[r] + threadIdx.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) b[c] = make_float2(src[4 + c] - threadIdx.x, src[8 + c]);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int q = 0; q < SUB; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[q][r][c] = __ffma2_rn(make_float2(v[r], v[r]), b[c], acc[q][r][c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) b[c].x = __int_as_float(__float_as_int(b[c].x) ^ 1);
    }
    float s = 0;
#pragma unroll
    for (int q = 0; q < SUB; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) s += acc[q][r][c].x + acc[q][r][c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int SUB>
void run(int sms, int threads, int blocks_per_sm, float* out, const float* src) {
    const int blocks = sms * blocks_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    outer2<SUB><<<blocks, threads>>>(out, src);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) outer2<SUB><<<blocks, threads>>>(out, src);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    const double flops = 2.0 * 2 * 16 * SUB * double(ITERS) * blocks * threads;
    printf("{\"sub\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", SUB, threads / 32 * blocks_per_sm, flops / ms / 1e9);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out, *src;
    cudaMalloc(&out, size_t(sms) * 8 * 1024 * 4); cudaMalloc(&src, 64 * 4); cudaMemset(src, 0, 256);
    run<1>(sms, 512, 1, out, src); run<1>(sms, 512, 2, out, src); run<1>(sms, 512, 4, out, src);
    run<2>(sms, 512, 1, out, src); run<2>(sms, 512, 2, out, src); run<2>(sms, 256, 1, out, src);
    return 0;
}
