// sp_rate.cu -- issue/complete rate of tcgen05.mma variants relevant to K6 (tools only):
// dense vs 2:4-sparse kind::f16, B K-major vs MN-major (SWIZZLE_128B), with / without a
// tcgen05.cp of metadata every 4 MMAs.  One CTA per SM, one elected lane issues `iters` MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2304_07613_b200/csrc -I include \
//        tools/sp_rate.cu -o tools/_bin/sp_rate && tools/_bin/sp_rate
#include <cstdio>
#include <cstdlib>
#include "sten.h"
#include "spmm_sp24.cuh"

using namespace sten;

STEN_DEVICE_INLINE void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                 : "memory");
}

// MODE bits: 1 sparse, 2 B MN-major, 4 tcgen05.cp every 4 MMAs, 8 A SWIZZLE_64B, 16 two accumulators
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) rate(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 64);
    unsigned char* sA = smem + 1024;              // 128 rows x 128 B
    unsigned char* sB = smem + 1024 + 16384;      // up to 256 x 128 B
    unsigned char* sE = smem + 1024 + 16384 + 32768;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < (16384 + 32768 + 2048) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sA)[i] = (MODE & 1) && i >= (16384 + 32768) / 4 ? 0x44444444u : 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(slot, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (warp == 0) {
        uint32_t idesc = tc_idesc(N);
        if (MODE & 1) idesc |= 1u << 2;
        if (MODE & 2) idesc |= 1u << 16;
        const uint32_t te = tb + 256;
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int kt = i & 3;
            const uint64_t ad = (MODE & 8) ? tc_sdesc_sw(smem_u32(sA) + (kt & 1) * 32 + (kt >> 1) * 8192, 64)
                                            : tc_sdesc_sw128(smem_u32(sA) + kt * 32);
            const uint64_t bd = (MODE & 2) ? tc_sdesc_mn_sw128(smem_u32(sB) + kt * ((MODE & 1) ? 4096 : 2048) / 4, 4096)
                                           : tc_sdesc_sw128(smem_u32(sB) + kt * 32);
            if (elect_one()) {
                if ((MODE & 4) && kt == 0) tc_cp_128x128b(te + 4 * ((i >> 2) & 3), tc_sdesc(smem_u32(sE), 16, 128));
                if (MODE & 1) tc_mma_sp_ss(tb + ((MODE & 16) ? uint32_t((i >> 1) & 1) * N : 0u), ad, bd, te + 4 * ((i >> 2) & 3) + (kt & 2), idesc | uint32_t(kt & 1), 1u);
                else mma_ss(tb, ad, bd, idesc);
            }
            __syncwarp();
        }
        const long long t1 = clock64();
        if (elect_one()) tc_commit(bar);
        __syncwarp();
        mbar_wait(bar, 0);
        const long long t2 = clock64();
        if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int N, int MODE>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    const int iters = 4096;
    const size_t sm = 1024 + 16384 + 32768 + 2048 + 1024;
    cudaFuncSetAttribute(rate<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    rate<N, MODE><<<148, 128, sm>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double kl = (MODE & 1) ? 32 : 16;      // logical k per MMA
    printf("{\"probe\": \"%s\", \"N\": %d, \"err\": \"%s\", \"issue_cyc_per_mma\": %.1f, \"done_cyc_per_mma\": %.1f, "
           "\"logical_flop_per_clk\": %.0f}\n",
           name, N, cudaGetErrorString(e), double(h[0]) / iters, double(h[1]) / iters,
           2.0 * 128 * N * kl * iters / double(h[1]));
    cudaFree(d);
}

int main(int argc, char** argv) {
    const int sel = argc > 1 ? atoi(argv[1]) : -1;
    int k = 0;
#define RUN(N, M, name) if (sel < 0 || sel == k++) run<N, M>(name);
    RUN(128, 0, "dense_Bk") RUN(256, 0, "dense_Bk") RUN(128, 2, "dense_Bmn") RUN(256, 2, "dense_Bmn")
    RUN(128, 1, "sparse_Bk") RUN(256, 1, "sparse_Bk") RUN(128, 3, "sparse_Bmn") RUN(256, 3, "sparse_Bmn")
    RUN(128, 7, "sparse_Bmn_cp") RUN(256, 7, "sparse_Bmn_cp") RUN(64, 3, "sparse_Bmn") RUN(192, 3, "sparse_Bmn")
    RUN(192, 11, "sparse_Bmn_A64") RUN(192, 27, "sparse_Bmn_A64_2acc") RUN(128, 11, "sparse_Bmn_A64") RUN(256, 11, "sparse_Bmn_A64")
    return 0;
}
