// Dev microbenchmark of tc_gemm_kernel epilogue variants (not part of the product).
#include <cstdio>
#include <vector>
#include "../paper_2605_08975_b200/csrc/ctx.h"
#include "../paper_2605_08975_b200/csrc/tc_gemm.cuh"
using namespace alpa;

struct Bufs { void *W, *X, *out, *xb; float *bias, *colsum; float2* stats; };

static int g_copies = 1;  // >1: rotate through weight copies (larger than L2 -> cold weights)
template <int TN, int EPI>
float run(int nf, int T, int K, int splits, const Bufs& b) {
    using Cf = GemmCfg<TN>;
    cudaFuncSetAttribute(tc_gemm_kernel<TN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    CUtensorMap tw, tx;
    CUtensorMap twc[8];
    for (int c = 0; c < g_copies; ++c)
        make_tmap_bf16_2d(&twc[c], (uint8_t*)b.W + (size_t)c * 8192 * 8192 * 2, K, nf, K * 2, 64, 128);
    make_tmap_bf16_2d(&tw, b.W, K, nf, K * 2, 64, 128);
    make_tmap_bf16_2d(&tx, b.X, K, T, K * 2, 64, TN);
    GemmArgs a{};
    a.nf = nf; a.t = T; a.k = K; a.bias = b.bias; a.out = b.out; a.ldo = nf;
    a.splits = splits; a.kbs = K / 64 / splits;
    a.stats_in = b.stats; a.colsum = b.colsum; a.nft = 16; a.ln_n = 2048;
    if (EPI == EPI_RESID_F32) { a.stats_out = b.stats; a.xb_out = (__nv_bfloat16*)b.xb; }
    dim3 grid(nf / 128, (T + TN - 1) / TN, splits);
    cudaLaunchConfig_t cfg{}; cfg.gridDim = grid; cfg.blockDim = dim3(Cf::THREADS); cfg.dynamicSmemBytes = Cf::SMEM;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = splits;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, tc_gemm_kernel<TN, EPI>, tw, tx, a);
    cudaEventRecord(e0);
    const int R = 50;
    for (int i = 0; i < R; ++i) cudaLaunchKernelEx(&cfg, tc_gemm_kernel<TN, EPI>, g_copies > 1 ? twc[i % g_copies] : tw, tx, a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    return ms / R * 1000.f;
}

int main(int argc, char** argv) {
    Bufs b;
    if (argc > 1) g_copies = atoi(argv[1]);
    cudaMalloc(&b.W, (size_t)8192 * 8192 * 2 * (g_copies > 1 ? 8 : 1)); cudaMalloc(&b.X, (size_t)4096 * 8192 * 2);
    cudaMalloc(&b.out, (size_t)4096 * 8192 * 4); cudaMalloc(&b.xb, (size_t)4096 * 8192 * 2);
    cudaMalloc(&b.bias, 8192 * 4); cudaMalloc(&b.colsum, 8192 * 4); cudaMalloc(&b.stats, 4096 * 16 * 8);
    cudaMemset(b.W, 0, (size_t)8192 * 8192 * 2 * (g_copies > 1 ? 8 : 1)); cudaMemset(b.X, 0, (size_t)4096 * 8192 * 2);
    cudaMemset(b.bias, 0, 8192 * 4); cudaMemset(b.colsum, 0, 8192 * 4); cudaMemset(b.stats, 0, 4096 * 16 * 8);
    cudaMemset(b.out, 0, (size_t)4096 * 8192 * 4);
    printf("mlp1 (8192x384x2048, S=1): none %6.1f  bf16 %6.1f  gelu %6.1f  ln_gelu %6.1f  f32 %6.1f resid %6.1f us\n",
           run<192, EPI_NONE>(8192, 384, 2048, 1, b), run<192, EPI_BF16>(8192, 384, 2048, 1, b),
           run<192, EPI_GELU_BF16>(8192, 384, 2048, 1, b), run<192, EPI_LN_GELU_BF16>(8192, 384, 2048, 1, b),
           run<192, EPI_F32>(8192, 384, 2048, 1, b), run<192, EPI_RESID_F32>(8192, 384, 2048, 1, b));
    for (int s : {1, 2, 4})
        printf("mlp2 (2048x384x8192, S=%d): none %6.1f  resid %6.1f us\n", s,
               run<192, EPI_NONE>(2048, 384, 8192, s, b), run<192, EPI_RESID_F32>(2048, 384, 8192, s, b));
    for (int s : {1, 2, 4})
        printf("o    (2048x384x1024, S=%d): none %6.1f  resid %6.1f us\n", s,
               run<192, EPI_NONE>(2048, 384, 1024, s, b), run<192, EPI_RESID_F32>(2048, 384, 1024, s, b));
    for (int s : {1, 2})
        printf("qkv  (3072x384x2048, S=%d): none %6.1f  ln %6.1f us\n", s,
               run<192, EPI_NONE>(3072, 384, 2048, s, b), run<192, EPI_LN_BF16>(3072, 384, 2048, s, b));
    return 0;
}
