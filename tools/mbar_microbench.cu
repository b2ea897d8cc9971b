// mbar_microbench.cu -- latency of mbarrier operations on this B200 (tools only).
#include <cstdio>
#include "common.cuh"
using namespace sten;

STEN_DEVICE_INLINE bool try_once(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    return ok;
}
STEN_DEVICE_INLINE bool test_once(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    return ok;
}

__global__ void probe(unsigned long long* out) {
    __shared__ __align__(8) uint64_t bar[4];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        mbar_arrive(&bar[0]);           // phase 0 of bar 0 complete
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int R = 64;
        unsigned acc = 0;
        long long t0 = clock64();
        for (int i = 0; i < R; ++i) acc += try_once(&bar[0], 0);
        long long t1 = clock64();
        for (int i = 0; i < R; ++i) acc += test_once(&bar[0], 0);
        long long t2 = clock64();
        for (int i = 0; i < R; ++i) mbar_wait(&bar[0], 0);
        long long t3 = clock64();
        for (int i = 0; i < R; ++i) acc += try_once(&bar[1], 0);    // not complete: try_wait times out
        long long t4 = clock64();
        for (int i = 0; i < R; ++i) acc += test_once(&bar[1], 0);
        long long t5 = clock64();
        out[0] = (t1 - t0) / R; out[1] = (t2 - t1) / R; out[2] = (t3 - t2) / R; out[3] = (t4 - t3) / R;
        out[4] = (t5 - t4) / R; out[5] = acc;
    }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    probe<<<1, 32>>>(d);
    probe<<<1, 32>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[6];
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("{\"err\": \"%s\", \"try_wait_done\": %llu, \"test_wait_done\": %llu, \"mbar_wait_done\": %llu, "
           "\"try_wait_pending\": %llu, \"test_wait_pending\": %llu, \"acc\": %llu}\n",
           cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5]);
    return 0;
}
