// tcgen05 kind::tf32 issue rate on B200: one CTA per SM, lane 0 of warp 0 issues
// `iters` MMAs (M = 128, K = 8, A from TMEM, B from smem) into one accumulator,
// then commits and waits; cycles per MMA from clock64.  Prints one JSON line per N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_rate tools/tc_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void rate(int N, int iters, int chain, int ss, unsigned long long *cyc) {
    __shared__ __align__(1024) float sB[128 * 64];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int j = tid; j < 128 * 64; j += blockDim.x) sB[j] = 0.001f * (j % 7);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tbase;
    if (ss == 2) {
        if (tid < 32) {
            const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
            const uint64_t desc = (uint64_t)((smem_u32(sB) >> 4) & 0x3FFF) | (8ull << 16) |
                                  ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
            const unsigned long long t0 = clock64();
#pragma unroll 8
            for (int i = 0; i < iters; ++i) {
                const uint32_t d = tb + 128 + ((chain || 2 * N > 384) ? 0 : (i & 1) * N);
                asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tb + (i & 7) * 16), "l"(desc), "r"(id), "r"(i > 3 ? 1 : 0));
            }
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                smem_u32(&mbar)));
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&mbar)));
            const unsigned long long t1 = clock64();
            if (tid == 0) cyc[blockIdx.x] = t1 - t0;
        }
    } else if (tid == 0) {
        const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const uint64_t desc = (uint64_t)((smem_u32(sB) >> 4) & 0x3FFF) | (8ull << 16) | ((uint64_t)(256 >> 4) << 32) |
                              (1ull << 46);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            // chain = 1: every MMA accumulates into one D; chain = 0: two independent D tiles
            const uint32_t d = tb + 128 + ((chain || 2 * N > 384) ? 0 : (i & 1) * N);
            if (ss)  // A from shared memory too (128 x 8 K-major, same descriptor form)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(desc), "l"(desc), "r"(id), "r"(i > 3 ? 1 : 0));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tb + (i & 7) * 16), "l"(desc), "r"(id), "r"(i > 3 ? 1 : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&mbar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&mbar)));
        const unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
    unsigned long long *d, h[148];
    cudaMalloc(&d, sizeof h);
    const int iters = 4096;
    printf("[");
    bool first = true;
    for (int ss = 0; ss < 3; ++ss)
    for (int chain = 0; chain < 2; ++chain)
        for (int N : {16, 48, 64, 96, 112, 128, 256}) {
            rate<<<148, 128>>>(N, iters, chain, ss, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("{\"error\": \"%s\"}]\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            double mean = 0;
            for (int i = 0; i < 148; ++i) mean += h[i];
            mean /= 148;
            printf("%s{\"A\": \"%s\", \"N\": %d, \"chained\": %d, \"cycles_per_mma\": %.1f, \"model_128N_over_256\": %.1f}",
                   first ? "" : ",\n ", ss == 2 ? "tmem, warp-elected" : ss ? "smem" : "tmem", N, chain, mean / iters, 128.0 * N / 256);
            first = false;
        }
    printf("]\n");
    return 0;
}
