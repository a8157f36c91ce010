// tcgen05 kind::tf32 probe (sm_100a): A in TMEM (written by tcgen05.st, lane = row),
// B in shared memory (K-major, no swizzle), D in TMEM, read back by tcgen05.ld.
// Checks the operand layouts and the 3xTF32 split (A_hi B_hi + A_hi B_lo + A_lo B_hi)
// against a double-precision host product.  Usage: tc_probe  (prints one JSON line)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int M = 128, KMAX = 64;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t b = __float_as_uint(x);
    return __uint_as_float((b + 0x1000u) & 0xFFFFE000u);
}

// B element (n, k) of an N x K K-major no-swizzle operand: 8-row x 16-byte core
// matrices, K chunks LBO = 128 B apart, 8-row groups SBO = (K/4)*128 B apart.
__device__ __forceinline__ int b_off(int n, int k, int K) {
    return ((n >> 3) * (K >> 2) + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3);
}

__device__ __forceinline__ uint64_t desc_b(uint32_t addr, int K) {
    const uint64_t lbo = 128 >> 4, sbo = (uint64_t)((K / 4) * 128) >> 4;
    return (uint64_t)((addr >> 4) & 0x3FFF) | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

__device__ __forceinline__ uint32_t idesc_tf32(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, int acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void probe(const float *A, const float *B, float *D, int N, int K, int split) {
    __shared__ __align__(1024) float sB[2][64 * KMAX];  // hi, lo
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int j = tid; j < N * K; j += blockDim.x) {
        const int n = j / K, k = j % K;
        const float x = B[j], h = tf32_hi(x);
        sB[0][b_off(n, k, K)] = h;
        sB[1][b_off(n, k, K)] = x - h;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy (MMA)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    // A row m = tid: hi at columns [0, K), lo at [K, 2K)
    for (int k0 = 0; k0 < K; k0 += 8) {
        uint32_t h[8], l[8];
        for (int j = 0; j < 8; ++j) {
            const float x = A[tid * K + k0 + j], hh = tf32_hi(x);
            h[j] = __float_as_uint(hh);
            l[j] = __float_as_uint(x - hh);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     ::"r"(tb + lane_base + k0), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]),
                     "r"(h[6]), "r"(h[7]));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     ::"r"(tb + lane_base + K + k0), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]),
                     "r"(l[5]), "r"(l[6]), "r"(l[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    const uint32_t dcol = 128;
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t id = idesc_tf32(N);
        int acc = 0;
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t bh = desc_b(smem_u32(&sB[0][0]) + s * 256, K);
            const uint64_t bl = desc_b(smem_u32(&sB[1][0]) + s * 256, K);
            if (split) {
                mma_tf32(tb + dcol, tb + K + 8 * s, bh, id, acc); acc = 1;   // A_lo B_hi
                mma_tf32(tb + dcol, tb + 8 * s, bl, id, 1);                 // A_hi B_lo
            }
            mma_tf32(tb + dcol, tb + 8 * s, bh, id, acc); acc = 1;          // A_hi B_hi
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&mbar)));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int n0 = 0; n0 < N; n0 += 16) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tb + lane_base + dcol + n0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16 && n0 + j < N; ++j) D[tid * N + n0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}

int main() {
    srand(12345);
    printf("[");
    bool first = true;
    const int Ns[] = {48, 64, 56, 16};
    const int Ks[] = {8, 56, 48};
    for (int split = 0; split < 2; ++split)
        for (int K : Ks)
            for (int N : Ns) {
                std::vector<float> A(M * K), B(N * K), D(M * N);
                for (auto &x : A) x = (float)((rand() / (double)RAND_MAX) * 2 - 1);
                for (auto &x : B) x = (float)((rand() / (double)RAND_MAX) * 2 - 1);
                float *dA, *dB, *dD;
                CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
                CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
                CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
                CK(cudaMemset(dD, 0xff, D.size() * 4));
                probe<<<1, 128>>>(dA, dB, dD, N, K, split);
                CK(cudaGetLastError());
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
                double maxrel = 0, maxabs = 0, scale = 0;
                int bad = 0;
                for (int m = 0; m < M; ++m)
                    for (int n = 0; n < N; ++n) {
                        double ref = 0, mag = 0;
                        for (int k = 0; k < K; ++k) {
                            ref += (double)A[m * K + k] * B[n * K + k];
                            mag += fabs((double)A[m * K + k] * B[n * K + k]);
                        }
                        const double e = fabs(D[m * N + n] - ref);
                        if (!(e == e) || e > 1e-2 * mag + 1e-6) ++bad;
                        maxabs = fmax(maxabs, e);
                        maxrel = fmax(maxrel, e / mag);
                        scale = fmax(scale, mag);
                    }
                printf("%s{\"split\": %d, \"K\": %d, \"N\": %d, \"max_err_over_sum_abs\": %.3e, \"bad\": %d}",
                       first ? "" : ",\n ", split, K, N, maxrel, bad);
                first = false;
                cudaFree(dA); cudaFree(dB); cudaFree(dD);
            }
    printf("]\n");
    return 0;
}
