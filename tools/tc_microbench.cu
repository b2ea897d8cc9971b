// tc_microbench.cu -- issue-rate probes for tcgen05.mma on this B200 (tools only, not the product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2304_07613_b200/csrc \
//        tools/tc_microbench.cu -o gpurun_out/tc_microbench && gpurun_out/tc_microbench
// One CTA per SM; thread 0 issues `iters` back-to-back MMAs (M = 128, N, K = 16, bf16 -> fp32)
// into one accumulator, A from TMEM (.ts) or from shared memory (.ss); optional "noise" warps
// write TMEM with tcgen05.st or read shared memory with ldmatrix concurrently.
#include <cstdio>
#include <vector>
#include "sten.h"
#include "spmm_tc.cuh"

using namespace sten;

STEN_DEVICE_INLINE void tc_mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

STEN_DEVICE_INLINE bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(pred));
    return pred != 0;
}

// MODE 0: A in TMEM; 1: A in smem; +2: tcgen05.st noise; +4: ldmatrix noise; +8: converged warp + elect.sync;
// +16: no "memory" clobber
template <int N, int MODE>
__global__ void __launch_bounds__(256, 1) tc_rate(unsigned long long* out, int iters, int dsets) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 64);
    volatile int* stop = reinterpret_cast<volatile int*>(smem + 128);
    unsigned char* sA = smem + 1024;             // 128 rows x 128 B, SW128
    unsigned char* sB = smem + 1024 + 16384;     // N rows x 128 B, SW128
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) { mbar_init(bar, 1); *stop = 0; fence_mbar_init(); }
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sA)[i] = 0x3c003c00u;
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (warp == 0 && (MODE & 8)) {
        const uint32_t idesc = tc_idesc(N);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tb + uint32_t((i & (dsets - 1)) * N);
            const int kt = i & 3;
            const uint64_t bd = tc_sdesc_sw128(smem_u32(sB) + kt * 32);
            if (elect_one()) {
                if ((MODE & 1) == 0) tc_mma_ts(d, tb + 256 + uint32_t(kt * 8), bd, idesc, 1u);
                else tc_mma_ss(d, tc_sdesc_sw128(smem_u32(sA) + kt * 32), bd, idesc, 1u);
            }
            __syncwarp();
        }
        const long long t1 = clock64();
        if (elect_one()) tc_commit(bar);
        __syncwarp();
        mbar_wait(bar, 0);
        const long long t2 = clock64();
        if (lane == 0) {
            *stop = 1;
            if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            const uint32_t idesc = tc_idesc(N);
            const long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t d = tb + uint32_t((i & (dsets - 1)) * N);
                const int kt = i & 3;
                const uint64_t bd = tc_sdesc_sw128(smem_u32(sB) + kt * 32);
                if ((MODE & 1) == 0)
                    tc_mma_ts(d, tb + 256 + uint32_t(kt * 8), bd, idesc, 1u);
                else
                    tc_mma_ss(d, tc_sdesc_sw128(smem_u32(sA) + kt * 32), bd, idesc, 1u);
            }
            const long long t1 = clock64();
            tc_commit(bar);
            mbar_wait(bar, 0);
            const long long t2 = clock64();
            *stop = 1;
            if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
        }
        __syncwarp();
    } else if (warp >= 4) {
        const int q = warp % 4;
        long long cnt = 0;
        while (!*stop) {
            if (MODE & 2) {
                for (int j = 0; j < 8; ++j)
                    tmem_st_16x256b(tb + 288 + uint32_t(j * 8) + (uint32_t(32 * q) << 16), 1u, 2u, 3u, 4u);
                tmem_wait_st();
            }
            if (MODE & 4) {
                uint32_t r0, r1, r2, r3;
                for (int j = 0; j < 8; ++j) {
                    ldsm_x4_trans(smem_u32(sA) + uint32_t(((lane + j) & 127) * 128 + ((lane & 7) * 16)), r0, r1, r2, r3);
                    cnt += r0 ^ r3;
                }
            }
            ++cnt;
        }
        if (cnt == 12345678) out[2] = cnt;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int N, int MODE>
void run(const char* name, int dsets) {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    const int iters = 4096;
    const size_t sm = 1024 + 16384 + N * 128;
    cudaFuncSetAttribute(tc_rate<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    tc_rate<N, MODE><<<148, 256, sm>>>(d, iters, dsets);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * 16;
    printf("{\"probe\": \"%s\", \"N\": %d, \"dsets\": %d, \"err\": \"%s\", \"issue_cyc_per_mma\": %.1f, "
           "\"done_cyc_per_mma\": %.1f, \"flop_per_clk\": %.0f}\n",
           name, N, dsets, cudaGetErrorString(e), double(h[0]) / iters, double(h[1]) / iters,
           flops * iters / double(h[1]));
    cudaFree(d);
}

int main() {
    run<16, 8>("ts_elect", 1);
    run<32, 8>("ts_elect", 1);
    run<16, 8>("ts_elect", 16);
    run<64, 8>("ts_elect", 1);
    run<256, 8>("ts_elect", 1);
    run<64, 9>("ss_elect", 1);
    run<64, 0>("ts", 1);
    run<64, 0>("ts", 4);
    run<64, 1>("ss", 1);
    run<64, 1>("ss", 4);
    run<16, 0>("ts", 1);
    run<16, 0>("ts", 16);
    run<16, 1>("ss", 1);
    run<128, 0>("ts", 1);
    run<128, 1>("ss", 1);
    run<256, 0>("ts", 1);
    run<256, 1>("ss", 1);
    run<64, 2>("ts+st_noise", 1);
    run<64, 4>("ts+ldsm_noise", 1);
    run<64, 6>("ts+st+ldsm_noise", 1);
    run<64, 3>("ss+st_noise", 1);
    run<16, 14>("ts_elect+st+ldsm_noise", 1);
    run<64, 14>("ts_elect+st+ldsm_noise", 1);
    return 0;
}
