// Unit probe of tnrd::launch_tc_kgrad against a CPU loop (R1 and R2):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -Ipaper_1510_02930_b200/csrc \
//        -o tools/kg_probe tools/kg_probe.cu paper_1510_02930_b200/csrc/tnrd_tc.cu
// prints the max error per (inner|outer) and the worst (f, t).
#include "tnrd_internal.h"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

static int mir(int x, int n) { x = x < 0 ? -1 - x : x; x = x >= n ? 2 * n - 1 - x : x; return x; }

int main(int argc, char **argv) {
    const int K = 7, NK = 48, R = 3, KT = 49;
    const int B = argc > 1 ? atoi(argv[1]) : 1, H = argc > 2 ? atoi(argv[2]) : 8, W = argc > 3 ? atoi(argv[3]) : 64;
    const int bnd = argc > 4 ? atoi(argv[4]) : 0, mode = argc > 5 ? atoi(argv[5]) : 0;
    const long long n = (long long)B * H * W;
    std::vector<float> u(n), e(n), b(NK * n), w(NK * n);
    srand(1);
    auto rnd = [] { return (float)rand() / RAND_MAX - 0.5f; };
    for (auto &x : u) x = mode == 1 ? 1.0f : rnd();
    for (auto &x : e) x = mode == 1 ? 1.0f : rnd();
    for (long long i = 0; i < NK * n; ++i) { b[i] = mode == 1 ? (float)(i / n + 1) : rnd(); w[i] = mode == 1 ? 1.0f : rnd(); }
    if (getenv("KG_IN")) {   // real inputs dumped by the debug hook
        FILE *fp = fopen(getenv("KG_IN"), "rb");
        int hdr[4];
        if (fread(hdr, 4, 4, fp) != 4 || hdr[0] != B || hdr[1] != H || hdr[2] != W || hdr[3] != NK) { printf("hdr mismatch\n"); return 1; }
        size_t ok = fread(u.data(), 4, n, fp) + fread(e.data(), 4, n, fp) + fread(b.data(), 4, NK * n, fp) + fread(w.data(), 4, NK * n, fp);
        fclose(fp);
        printf("loaded %zu floats\n", ok);
        double mx[4] = {0, 0, 0, 0};
        for (long long i = 0; i < n; ++i) { mx[0] = fmax(mx[0], fabs(u[i])); mx[1] = fmax(mx[1], fabs(e[i])); }
        for (long long i = 0; i < NK * n; ++i) { mx[2] = fmax(mx[2], fabs(b[i])); mx[3] = fmax(mx[3], fabs(w[i])); }
        printf("max |u| %g |e| %g |b| %g |w| %g\n", mx[0], mx[1], mx[2], mx[3]);
    }
    std::vector<double> ref(NK * 2 * KT, 0.0);
    for (int f = 0; f < NK; ++f)
        for (int bi = 0; bi < B; ++bi)
            for (int y = 0; y < H; ++y)
                for (int x = 0; x < W; ++x) {
                    const long long p = (long long)bi * H * W + y * W + x;
                    const double bp = b[f * n + p];
                    const double op = bnd == 1 ? w[f * n + p] : e[p];
                    for (int a = 0; a < K; ++a)
                        for (int c = 0; c < K; ++c) {
                            const long long o = (long long)bi * H * W + mir(y - (a - R), H) * W + mir(x - (c - R), W);
                            ref[f * 2 * KT + a * K + c] += bp * u[o];
                            ref[f * 2 * KT + KT + a * K + c] += op * (bnd == 1 ? e[o] : w[f * n + o]);
                        }
                }
    float *du, *de, *db, *dw, *dp;
    const int nblk = tnrd::tc_kgrad_blocks(B, H, W, 148);
    cudaMalloc(&du, 4 * n); cudaMalloc(&de, 4 * n); cudaMalloc(&db, 4 * NK * n); cudaMalloc(&dw, 4 * NK * n);
    cudaMalloc(&dp, 4 * NK * nblk * 2 * KT);
    cudaMemcpy(du, u.data(), 4 * n, cudaMemcpyHostToDevice); cudaMemcpy(de, e.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), 4 * NK * n, cudaMemcpyHostToDevice); cudaMemcpy(dw, w.data(), 4 * NK * n, cudaMemcpyHostToDevice);
    cudaError_t er = tnrd::launch_tc_kgrad(K, NK, du, de, db, dw, bnd, B, H, W, dp, nblk, 0);
    if (er == cudaSuccess) er = cudaDeviceSynchronize();
    if (er != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(er)); return 1; }
    std::vector<float> part(NK * nblk * 2 * KT);
    cudaMemcpy(part.data(), dp, 4 * part.size(), cudaMemcpyDeviceToHost);
    double emax[2] = {0, 0}, smax[2] = {0, 0};
    int wf[2] = {0, 0}, wt[2] = {0, 0};
    for (int f = 0; f < NK; ++f)
        for (int j = 0; j < 2 * KT; ++j) {
            double s = 0;
            for (int k = 0; k < nblk; ++k) s += part[((long long)f * nblk + k) * 2 * KT + j];
            const double r = ref[f * 2 * KT + j], d = fabs(s - r);
            const int h = j >= KT;
            smax[h] = fmax(smax[h], fabs(r));
            if (d > emax[h]) { emax[h] = d; wf[h] = f; wt[h] = j % KT; }
            if (f == 0 && j < KT && argc > 6) printf("t=%d ref %.4f got %.4f\n", j, r, s);
        }
    if (getenv("KG_PART")) {
        FILE *fp = fopen(getenv("KG_PART"), "rb");
        std::vector<float> lp(part.size());
        size_t got = fread(lp.data(), 4, lp.size(), fp); fclose(fp);
        double dm = 0; long long at = -1;
        for (size_t i = 0; i < got; ++i) if (fabs(lp[i] - part[i]) > dm) { dm = fabs(lp[i] - part[i]); at = (long long)i; }
        printf("lib partial vs probe partial: %zu floats, max diff %g at %lld\n", got, dm, at);
        if (at >= 0) for (int i = 0; i < 8; ++i) printf("  [%d] lib %g probe %g\n", i, lp[i], part[i]);
    }
    printf("B=%d H=%d W=%d bnd=%d nblk=%d inner: err %.3e of %.3e (f %d t %d)  outer: err %.3e of %.3e (f %d t %d)\n", B, H,
           W, bnd, nblk, emax[0], smax[0], wf[0], wt[0], emax[1], smax[1], wf[1], wt[1]);
    return 0;
}
