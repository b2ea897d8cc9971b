// tma_microbench.cu -- per-SM L2 -> shared memory ingest rate of TMA tile loads (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2304_07613_b200/csrc \
//        tools/tma_microbench.cu -o tools/_bin/tma_microbench -lcuda
// One CTA per SM streams `iters` boxes of [rows][inner bytes] through a ring of `stages` buffers
// (one producer thread, mbarrier completion, no consumer work), from a source of `src_mb` MB that
// each CTA walks at its own offset.  Reports bytes per SM clock per SM and aggregate GB/s.
#include <cstdio>
#include <cstring>
#include <vector>
#include "common.cuh"
#include "tma_host.h"

using namespace sten;

STEN_DEVICE_INLINE void wait_plain(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
STEN_DEVICE_INLINE void wait_test(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ int g_wait_mode;

__global__ void __launch_bounds__(128, 1)
tma_stream(const __grid_constant__ CUtensorMap tm, int iters, int stages, int box_rows, int rows_total, uint32_t box_bytes,
           unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    unsigned char* buf = smem + 1024;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        int row = (blockIdx.x * 7919 * box_rows) % rows_total;
        for (int i = 0; i < iters + stages; ++i) {
            const int s = i % stages;
            const long long tw = clock64();
            if (i >= stages) {
                const uint32_t ph = uint32_t(((i / stages) - 1) & 1);
                if (g_wait_mode == 0) mbar_wait(&full[s], ph);
                else if (g_wait_mode == 1) wait_plain(&full[s], ph);
                else wait_test(&full[s], ph);
            }
            const long long tw2 = clock64();
            if (i < iters) {
                mbar_arrive_expect_tx(&full[s], box_bytes);
                tma_load_2d(buf + size_t(s) * box_bytes, &tm, &full[s], 0, row);
                row += box_rows;
                if (row + box_rows > rows_total) row = 0;
            }
            if (blockIdx.x == 0 && i >= 64 && i < 96) {
                const long long te = clock64();
                out[1024 + 2 * (i - 64)] = (unsigned long long)(te - tw);
                out[1025 + 2 * (i - 64)] = (unsigned long long)(tw2 - tw);
            }
        }
        const long long t1 = clock64();
        out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
}

// burst: thread 0 issues `nbox` boxes back to back onto distinct barriers, then waits for all;
// out = {issue cycles, completion cycles} of CTA 0
__global__ void __launch_bounds__(128, 1)
tma_burst(const __grid_constant__ CUtensorMap tm, int nbox, int box_rows, uint32_t box_bytes, int prefetch,
          unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    unsigned char* buf = smem + 1024;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nbox; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        if (prefetch) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int rep = 0; rep < 2; ++rep) {
            const long long t0 = clock64();
            for (int i = 0; i < nbox; ++i) {
                mbar_arrive_expect_tx(&full[i], box_bytes);
                tma_load_2d(buf + size_t(i) * box_bytes, &tm, &full[i], 0, (blockIdx.x * 64 + i) * box_rows);
            }
            const long long t1 = clock64();
            for (int i = 0; i < nbox; ++i) mbar_wait(&full[i], uint32_t(rep));
            const long long t2 = clock64();
            if (blockIdx.x == 0 && rep == 1) { out[0] = t1 - t0; out[1] = t2 - t0; }
        }
    }
}

static void burst(void* src, int box_rows, int nbox, int ctas, int prefetch) {
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    const int rows_total = int((size_t(48) << 20) / 128);
    const uint64_t dims[2] = {64, uint64_t(rows_total)};
    const uint64_t strides[1] = {128};
    const uint32_t box[2] = {64, uint32_t(box_rows)};
    make_tmap_nd(&tm, src, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    const uint32_t box_bytes = 128u * box_rows;
    const size_t smem = 1024 + size_t(nbox) * box_bytes;
    cudaFuncSetAttribute(tma_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    unsigned long long* d;
    cudaMalloc(&d, 16);
    tma_burst<<<ctas, 128, smem>>>(tm, nbox, box_rows, box_bytes, prefetch, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"burst\": 1, \"box_rows\": %d, \"nbox\": %d, \"ctas\": %d, \"prefetch\": %d, \"err\": \"%s\", "
           "\"issue_cyc_per_box\": %.1f, \"done_cyc\": %llu, \"B_per_clk\": %.1f}\n",
           box_rows, nbox, ctas, prefetch, cudaGetErrorString(err), double(h[0]) / nbox, h[1],
           double(nbox) * box_bytes / double(h[1]));
    cudaFree(d);
}

static int g_mode = 0;
static void run(void* src, int inner_bytes, int box_rows, int stages, int ctas, size_t src_bytes, int swz) {
    cudaMemcpyToSymbol(g_wait_mode, &g_mode, sizeof(int));
    const int rows_total = int(src_bytes / inner_bytes);
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    const uint64_t dims[2] = {uint64_t(inner_bytes / 2), uint64_t(rows_total)};
    const uint64_t strides[1] = {uint64_t(inner_bytes)};
    const uint32_t box[2] = {uint32_t(inner_bytes / 2), uint32_t(box_rows)};
    const CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (!make_tmap_nd(&tm, src, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims, strides, box, sw)) {
        printf("{\"err\": \"tmap\", \"inner\": %d, \"rows\": %d}\n", inner_bytes, box_rows);
        return;
    }
    const uint32_t box_bytes = uint32_t(inner_bytes * box_rows);
    const size_t smem = 1024 + size_t(stages) * box_bytes;
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    unsigned long long* d;
    cudaMalloc(&d, 16384);
    const int iters = int((64ull << 20) / box_bytes);     // 64 MB per CTA
    tma_stream<<<ctas, 128, smem>>>(tm, 4, stages, box_rows, rows_total, box_bytes, d);   // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_stream<<<ctas, 128, smem>>>(tm, iters, stages, box_rows, rows_total, box_bytes, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(ctas);
    cudaMemcpy(h.data(), d, ctas * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += double(v) / ctas;
    unsigned long long it[64];
    cudaMemcpy(it, d + 1024, sizeof(it), cudaMemcpyDeviceToHost);
    printf("iter cycles:");
    for (int k = 0; k < 32; ++k) printf(" %llu/%llu", it[2 * k], it[2 * k + 1]);
    printf("\n");
    const double bytes = double(iters) * box_bytes;
    printf("{\"wait\": %d, \"inner_B\": %d, \"box_rows\": %d, \"box_KB\": %.0f, \"stages\": %d, \"ctas\": %d, \"src_MB\": %zu, "
           "\"swz\": %d, \"err\": \"%s\", \"B_per_clk_per_sm\": %.1f, \"aggregate_GBps\": %.0f}\n",
           g_mode, inner_bytes, box_rows, box_bytes / 1024.0, stages, ctas, src_bytes >> 20, swz, cudaGetErrorString(err),
           bytes / mean, bytes * ctas / (ms * 1e-3) / 1e9);
    cudaFree(d);
}

int main() {
    void* src;
    const size_t big = size_t(1) << 30;
    cudaMalloc(&src, big);
    cudaMemset(src, 0, big);
    const size_t l2 = size_t(48) << 20;    // L2-resident source
    for (int pf = 0; pf < 0; ++pf) {
        burst(src, 32, 16, 1, pf);
        burst(src, 32, 16, 148, pf);
        burst(src, 8, 32, 1, pf);
        burst(src, 256, 4, 1, pf);
        burst(src, 256, 4, 148, pf);
    }
    for (g_mode = 0; g_mode < 1; ++g_mode) {
        run(src, 128, 256, 3, 148, l2, 128);
        run(src, 128, 64, 8, 148, l2, 128);
        run(src, 128, 32, 16, 148, l2, 128);
        run(src, 128, 32, 16, 16, l2, 128);
    }
    g_mode = 1;
    run(src, 128, 128, 3, 148, l2, 128);
    run(src, 64, 256, 3, 148, l2, 64);
    run(src, 128, 256, 3, 148, big, 128);
    return 0;
}
