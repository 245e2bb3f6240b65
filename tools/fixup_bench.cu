// Dev microbenchmark: the persistent kernel's split-K fixup (mk::gemm_fixup)
// in isolation, O / MLP2 shape (nf 2048, M 384, TN 192, S 4, 128 CTAs).
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/mk.cuh"
using namespace alpa;
using namespace alpa::mk;

__global__ void __launch_bounds__(320, 1) fixup_kernel(Params p, const Op* ops, int reps) {
    __shared__ float mu_s[256], rs_s[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < 2) return;
    const int ew = warp - 2;
    const Op op = ops[0];
    const int it = blockIdx.x;
    GemmItem g = gemm_item(op, it, 192);
    const int rows = 192 / op.splits;
    const int rb = g.t0 + g.s * rows, re = min(p.M, rb + rows);
    for (int r = 0; r < reps; ++r) gemm_fixup(p, op, g, rb, re, ew, lane, mu_s, rs_s);
}

int main() {
    const int M = 384, nf = 2048, S = 4;
    Params p{};
    float *ws, *e, *bias;
    float2* stats;
    __nv_bfloat16* xb;
    cudaMalloc(&ws, (size_t)S * M * nf * 4);
    cudaMalloc(&e, (size_t)M * nf * 4);
    cudaMalloc(&bias, nf * 4);
    cudaMalloc(&stats, (size_t)M * 16 * 8);
    cudaMalloc(&xb, (size_t)M * nf * 2);
    cudaMemset(ws, 0, (size_t)S * M * nf * 4);
    cudaMemset(e, 0, (size_t)M * nf * 4);
    cudaMemset(bias, 0, nf * 4);
    p.ws = ws; p.M = M; p.ah = nf; p.nft = 16;
    Op op{};
    op.kind = OP_GEMM; op.epi = EPI_RESID_F32; op.nf = nf; op.k = 8192; op.splits = S; op.kbs = 32;
    op.tiles_f = 16; op.tiles_t = 2; op.n_items = 128; op.bias = bias; op.out = e; op.ldo = nf;
    op.stats_out = stats; op.xb_out = xb;
    Op* d_op;
    cudaMalloc(&d_op, sizeof(Op));
    cudaMemcpy(d_op, &op, sizeof(Op), cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int reps : {1, 2, 5}) {
        fixup_kernel<<<128, 320>>>(p, d_op, reps);
        cudaEventRecord(a);
        for (int i = 0; i < 20; ++i) fixup_kernel<<<128, 320>>>(p, d_op, reps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("fixup reps=%d: %.2f us per launch (%.2f us per fixup incl. launch)\n", reps, ms / 20 * 1000, ms / 20 * 1000 / reps);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
