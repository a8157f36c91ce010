// Probe (sm_100a) for the persistent stage kernel's two new data paths:
//  (1) tcgen05.cp.cta_group::1.128x256b: a 128-row x 8-word block of a K-major,
//      no-swizzle shared-memory operand (8-row x 16-byte core matrices, LBO = 128 B
//      between the two 16-byte column halves, SBO = 256 B between 8-row groups) into
//      TMEM lanes 0..127, columns c..c+7; read back with tcgen05.ld;
//  (2) the same copy followed in the tensor pipe by a kind::tf32 MMA reading that TMEM
//      block as A (issue order, no wait in between): D = A B against a host product;
//  (3) cp.async.bulk.tensor.3d (TMA) of one 72-float row box from a [B][H][ld] fp32
//      tensor into shared memory, at in-range and negative / past-the-end x coordinates
//      (out-of-bounds elements are zero-filled).  Measured on the B200: the innermost
//      box start must be a multiple of 16 bytes (x % 4 == 0 for fp32) -- x = 5 or -7
//      raises cudaErrorIllegalInstruction, x = 0, 4, 8, -4 work.
// Prints one JSON line.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/cp_probe tools/cp_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc_tf32(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}

// E-ring element (pixel px of a 128-pixel block, word j of 8): K-major core matrices
__device__ __forceinline__ int e_off(int px, int j) { return ((px >> 3) * 2 + (j >> 2)) * 32 + (px & 7) * 4 + (j & 3); }

__global__ void cp_probe(const float *B8x16, float *out_cp, float *out_d, const __grid_constant__ CUtensorMap tm,
                         float *out_tma, const CUtensorMap *gtm, const float *img) {
    __shared__ __align__(1024) float sE[128 * 8];
    __shared__ __align__(1024) float sB[16 * 8];     // B: N = 16 rows x K = 8, K-major
    __shared__ __align__(128) float sT[3][96];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int px = i / 8, j = i % 8;
        sE[e_off(px, j)] = (float)(px * 8 + j) * 0.25f;   // exact in TF32
    }
    for (int i = tid; i < 16 * 8; i += blockDim.x) {
        const int n = i / 8, k = i % 8;
        sB[((n >> 3) * 2 + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3)] = B8x16[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm0 = tbase;
    if (tid == 0) {
        // (1) + (2): copy A into columns 0..7, then D (cols 16..31) = A (128x8) * B^T (8x16)
#ifndef NO_CP
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm0), "l"(desc(smem_u32(sE), 128, 256)));
#endif
#ifndef NO_MMA
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tm0 + 16), "r"(tm0), "l"(desc(smem_u32(sB), 128, 256)), "r"(idesc_tf32(16)), "r"(0));
#endif
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
        // (3) TMA: three row boxes at x = 5, x = -7 and x = W - 40 of row 3 of image 1
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[1])), "r"(3 * 72 * 4) : "memory");
        const int xs[3] = {4, -8, 100 - 40};
#ifdef BULK1D
        for (int q = 0; q < 3; ++q)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sT[q])), "l"(img + 2 * 8 * 104 / 2 + 3 * 104 + 4 * q), "r"(288), "r"(smem_u32(&bar[1])) : "memory");
        if (0)
#endif
        for (int q = 0; q < 3; ++q)
#ifdef NO_TMA
            if (q < 0)
#endif
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(sT[q])), 
#ifdef GMAP
                         "l"(reinterpret_cast<uint64_t>(gtm))
#else
                         "l"(reinterpret_cast<uint64_t>(&tm))
#endif
                         , "r"(xs[q]), "r"(3), "r"(1),
                         "r"(smem_u32(&bar[1])) : "memory");
    }
    __syncwarp();
    mbar_wait(&bar[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        uint32_t r[8], d[16];
        const uint32_t ta = tm0 + ((uint32_t)(warp * 32) << 16);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]) : "r"(ta + 16));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]) : "r"(ta + 24));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int m = warp * 32 + lane;
        for (int j = 0; j < 8; ++j) out_cp[m * 8 + j] = __uint_as_float(r[j]);
        for (int n = 0; n < 16; ++n) out_d[m * 16 + n] = __uint_as_float(d[n]);
    }
#ifndef NO_TMA
    mbar_wait(&bar[1], 0);
#endif
    for (int i = tid; i < 3 * 72; i += blockDim.x) out_tma[i] = sT[i / 72][i % 72];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm0));
}

int main() {
    const int Bn = 2, H = 8, W = 100, ld = 104;
    std::vector<float> img((size_t)Bn * H * ld);
    for (size_t i = 0; i < img.size(); ++i) img[i] = (float)i;
    float *d_img, *d_B, *d_cp, *d_d, *d_t;
    CK(cudaMalloc(&d_img, img.size() * 4));
    CK(cudaMemcpy(d_img, img.data(), img.size() * 4, cudaMemcpyHostToDevice));
    std::vector<float> Bh(16 * 8);
    for (int i = 0; i < 16 * 8; ++i) Bh[i] = (float)((i * 7) % 11 - 5) * 0.5f;
    CK(cudaMalloc(&d_B, 16 * 8 * 4));
    CK(cudaMemcpy(d_B, Bh.data(), 16 * 8 * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&d_cp, 128 * 8 * 4));
    CK(cudaMalloc(&d_d, 128 * 16 * 4));
    CK(cudaMalloc(&d_t, 3 * 72 * 4));
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                            const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)Bn};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)H * ld * 4};
#ifdef BOX64
    cuuint32_t box[3] = {64, 1, 1}, es[3] = {1, 1, 1};
#else
    cuuint32_t box[3] = {72, 1, 1}, es[3] = {1, 1, 1};
#endif
    printf("{\"encode_fn\": \"%p\", \"query\": %d}\n", fn, (int)q);
#ifdef DIRECT
    CUresult cr = cuTensorMapEncodeTiled(&tm,
#else
    CUresult cr = ((Enc)fn)(&tm,
#endif
                            CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_img, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("{\"error\": \"encode %d\"}\n", (int)cr); return 1; }
    CUtensorMap *gtm;
    CK(cudaMalloc(&gtm, sizeof(CUtensorMap)));
    CK(cudaMemcpy(gtm, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    printf("{\"host_tm_mod64\": %d, \"sizeof\": %d}\n", (int)(((uintptr_t)&tm) % 64), (int)sizeof(CUtensorMap));
    cp_probe<<<1, 256>>>(d_B, d_cp, d_d, tm, d_t, gtm, d_img);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> cp(128 * 8), dd(128 * 16), tt(3 * 72);
    CK(cudaMemcpy(cp.data(), d_cp, cp.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(dd.data(), d_d, dd.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tt.data(), d_t, tt.size() * 4, cudaMemcpyDeviceToHost));
    int bad_cp = 0, bad_d = 0, bad_t = 0;
    for (int m = 0; m < 128; ++m)
        for (int j = 0; j < 8; ++j) bad_cp += cp[m * 8 + j] != (float)(m * 8 + j) * 0.25f;
    double maxd = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            double s = 0;
            for (int k = 0; k < 8; ++k) s += (double)((m * 8 + k) * 0.25f) * Bh[n * 8 + k];
            maxd = fmax(maxd, fabs(s - dd[m * 16 + n]));
            bad_d += fabs(s - dd[m * 16 + n]) > 1e-3 * (1 + fabs(s));
        }
    const int xs[3] = {4, -8, 60};
    for (int q2 = 0; q2 < 3; ++q2)
        for (int c = 0; c < 72; ++c) {
            const int x = xs[q2] + c;
            const float want = (x >= 0 && x < W) ? img[(size_t)1 * H * ld + 3 * ld + x] : 0.0f;
            bad_t += tt[q2 * 72 + c] != want;
        }
    printf("{\"cp_128x256b_bad\": %d, \"cp_then_mma_bad\": %d, \"mma_max_abs_err\": %.3g, \"tma_row_bad\": %d, "
           "\"cp0\": [%g, %g, %g], \"cp_lane127\": [%g, %g]}\n",
           bad_cp, bad_d, maxd, bad_t, cp[0], cp[1], cp[8], cp[127 * 8], cp[127 * 8 + 7]);
    return 0;
}
