// Dev microbenchmark of tc_gemm_kernel shapes (not part of the product).
#include <cstdio>
#include <vector>
#include "../paper_2605_08975_b200/csrc/ctx.h"
#include "../paper_2605_08975_b200/csrc/tc_gemm.cuh"
using namespace alpa;

template <int TN, int EPI>
float run(int nf, int T, int K, int splits, const void* W, const void* X, float* bias, void* out,
          float* ws, int* cnt) {
    using Cf = GemmCfg<TN>;
    cudaFuncSetAttribute(tc_gemm_kernel<TN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    CUtensorMap tw, tx;
    make_tmap_bf16_2d(&tw, W, K, nf, K * 2, 64, 128);
    make_tmap_bf16_2d(&tx, X, K, T, K * 2, 64, TN);
    GemmArgs a{};
    a.nf = nf; a.t = T; a.k = K; a.bias = bias; a.out = out; a.ldo = nf;
    int KB = K / 64; a.splits = splits; a.kbs = KB / splits;
    if (TN % splits) return -1.f;
    dim3 grid(nf / 128, (T + TN - 1) / TN, a.splits);
    cudaLaunchConfig_t cfg{}; cfg.gridDim = grid; cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = Cf::SMEM;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = splits;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, tc_gemm_kernel<TN, EPI>, tw, tx, a);
    cudaEventRecord(e0);
    const int R = 20;
    for (int i = 0; i < R; ++i) cudaLaunchKernelEx(&cfg, tc_gemm_kernel<TN, EPI>, tw, tx, a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    return ms / R * 1000.f;
}

int main() {
    size_t big = (size_t)8192 * 8192;
    void *W, *X, *out; float *bias, *ws; int* cnt;
    cudaMalloc(&W, big * 2); cudaMalloc(&X, (size_t)4096 * 8192 * 2); cudaMalloc(&out, (size_t)4096 * 8192 * 4);
    cudaMalloc(&bias, 8192 * 4); cudaMalloc(&ws, (size_t)64 << 20); cudaMalloc(&cnt, 1 << 16);
    cudaMemset(W, 0, big * 2); cudaMemset(X, 0, (size_t)4096 * 8192 * 2); cudaMemset(bias, 0, 8192 * 4);
    cudaMemset(cnt, 0, 1 << 16);
    struct S { int nf, T, K; const char* name; };
    S shapes[] = {{8192, 384, 2048, "mlp1"}, {2048, 384, 8192, "mlp2"}, {3072, 384, 2048, "qkv"}, {2048, 384, 1024, "o"}, {8192, 4096, 8192, "big"}};
    for (auto s : shapes) {
        double fl = 2.0 * s.nf * s.T * s.K;
        for (int sp : {1, 2, 4}) {
            float t64n = run<64, EPI_NONE>(s.nf, s.T, s.K, sp, W, X, bias, out, ws, cnt);
            float t128n = run<128, EPI_NONE>(s.nf, s.T, s.K, sp, W, X, bias, out, ws, cnt);
            float t192n = run<192, EPI_NONE>(s.nf, s.T, s.K, sp, W, X, bias, out, ws, cnt);
            float t256n = run<256, EPI_NONE>(s.nf, s.T, s.K, sp, W, X, bias, out, ws, cnt);
            float t192g = run<192, EPI_GELU_BF16>(s.nf, s.T, s.K, sp, W, X, bias, out, ws, cnt);
            float t192r = run<192, EPI_RESID_F32>(s.nf, s.T, s.K, sp, W, X, bias, out, ws, cnt);
            printf("%-5s split%d  none: tn64 %7.1fus tn128 %7.1f tn192 %7.1f (%5.0f TF) tn256 %7.1f | tn192 gelu %7.1f resid %7.1f\n",
                   s.name, sp, t64n, t128n, t192n, fl / t192n / 1e6, t256n, t192g, t192r);
        }
    }
    return 0;
}
