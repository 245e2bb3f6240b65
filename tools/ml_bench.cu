// Dev microbenchmark (not part of the product): GEMM mainloop throughput of the
// persistent kernel's item shape with every SM busy, to decide the tiling of the
// decoder-block GEMMs (N = 6: 384 tokens).
//   mode 0  1-CTA items: W tile 128 x K (HBM stream) + X tile TN x K (L2), MMA 128 x TN
//   mode 1  cluster of 2, same items, X tile multicast (each CTA loads TN/2 rows for both)
//   mode 2  cta_group::2 pair: MMA 256 x TN, each CTA loads its 128 W rows + TN/2 X rows
//   +8      no MMA (the consumer releases every stage as it lands): pure TMA ingress
// Prints us per launch, aggregate smem ingress (TB/s) and TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ml_bench tools/ml_bench.cu \
//        paper_2605_08975_b200/csrc/tma.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_08975_b200/csrc/common.cuh"
#include "../paper_2605_08975_b200/csrc/ctx.h"

using namespace alpa;

namespace {

__device__ inline void mma_cg2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ inline void commit_cg2_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ inline void commit_cg1_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// TMA load whose completion is signalled on an mbarrier of either CTA of the pair
__device__ inline void tma_load_2d_cg2(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1,
                                       uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(pol)
        : "memory");
}
__device__ inline void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                      uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ inline void mbar_arrive_cluster(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ inline void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}

struct P {
    const CUtensorMap* tw;  // W [rows][K], box {64, 128}
    const CUtensorMap* tx;  // X [384][K], box {64, TN} (mode 0) / {64, TN/2}
    int K, tiles_f, tiles_t, TN, wrow0, reps, wl2, tiled, pfd, nox;
    const uint8_t* wbase;
};

template <int MODE, int STAGES, int TNMAX>
__global__ void __launch_bounds__(192, 1) kern(const __grid_constant__ P p) {
    constexpr bool NOMMA = MODE & 8;
    constexpr int M = MODE & 7;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int WB = 128 * 64 * 2;
    constexpr int SLOT = WB + TNMAX * 128;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SLOT);
    uint64_t* full = bars;
    uint64_t* empty = bars + 8;
    uint64_t* accf = bars + 16;  // [2]
    uint64_t* acce = bars + 18;  // [2]
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 24);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = M ? cluster_ctarank() : 0;
    const int units = M ? gridDim.x / 2 : gridDim.x;
    const int unit = M ? blockIdx.x / 2 : blockIdx.x;
    const int TN = p.TN;
    const int nitems = p.tiles_f * p.tiles_t * p.reps;
    const int KB = p.K / 64;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], M == 1 ? 2 : 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&accf[i], 1);
            mbar_init(&acce[i], M == 2 ? 2 : 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(slot, 512);
    tc_fence_before();
    if (M) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    const uint64_t pol = p.wl2 ? policy_evict_last() : policy_evict_first();
    if (warp == 0 && lane == 0) {
        uint32_t ks = 0;
        for (int it = unit; it < nitems; it += units) {
            const int rep = it / (p.tiles_f * p.tiles_t), ii = it % (p.tiles_f * p.tiles_t);
            const int f = ii % p.tiles_f, t = ii / p.tiles_f;
            // W rows: a pair (modes 1, 2) covers 256 rows, rank r its half
            const int wrow = p.wrow0 + rep * p.tiles_f * (M ? 256 : 128) + (M ? f * 256 + rank * 128 : f * 128);
            // tiled layout: every (128-row tile, k-block) box is one contiguous 16 KB chunk
            auto wc0 = [&](int i) { return p.tiled ? 0 : i * 64; };
            auto wc1 = [&](int i) { return p.tiled ? ((wrow / 128) * KB + i) * 128 : wrow; };
            // pfd > 0: tensor-box L2 prefetch; pfd < 0: 1-D bulk prefetch of the contiguous
            // 16 KB box (tiled layout only), -pfd k-blocks ahead
            auto pf = [&](int i) {
                if (p.pfd > 0) tma_prefetch_box_2d(p.tw, wc0(i), wc1(i));
                else l2_prefetch_hint(p.wbase + (size_t)wc1(i) * 128, 16384, pol);
            };
            const int pd = p.pfd > 0 ? p.pfd : -p.pfd;
            for (int i = 0; i < pd && i < KB; ++i) pf(i);
            for (int i = 0; i < KB; ++i, ++ks) {
                const uint32_t st = ks % STAGES, ph = (ks / STAGES) & 1;
                if (pd && i + pd < KB) pf(i + pd);
                mbar_wait_cluster(&empty[st], ph ^ 1);
                uint8_t* sb = smem + st * SLOT;
                if (M == 0) {
                    mbar_expect_tx(&full[st], WB + (p.nox ? 0 : TN * 128));
                    tma_load_2d_hint(sb, p.tw, &full[st], wc0(i), wc1(i), pol);
                    if (!p.nox) tma_load_2d(sb + WB, p.tx, &full[st], i * 64, t * TN);
                } else if (M == 1) {
                    // own W + the full X tile (half from each CTA's multicast)
                    mbar_expect_tx(&full[st], WB + TN * 128);
                    tma_load_2d_hint(sb, p.tw, &full[st], i * 64, wrow, pol);
                    tma_load_2d_mc(sb + WB + rank * (TN / 2) * 128, p.tx, &full[st], i * 64, t * TN + rank * (TN / 2),
                                   3);
                } else {
                    // pair: both CTAs' bytes complete on the leader's barrier
                    const uint32_t fb = dsmem_addr(smem_u32(&full[st]), 0);
                    if (rank == 0) mbar_expect_tx(&full[st], 2 * (WB + (TN / 2) * 128));
                    tma_load_2d_cg2(sb, p.tw, fb, wc0(i), wc1(i), pol);
                    tma_load_2d_cg2(sb + WB, p.tx, fb, i * 64, t * TN + rank * (TN / 2), pol);
                }
            }
        }
    } else if (warp == 1 && lane == 0 && (M != 2 || rank == 0)) {
        uint32_t ks = 0, n = 0;
        const uint32_t idesc = idesc_bf16(M == 2 ? 256 : 128, TN);
        for (int it = unit; it < nitems; it += units, ++n) {
            const uint32_t ab = n & 1;
            if (n >= 2) mbar_wait_cluster(&acce[ab], ((n - 2) >> 1) & 1);
            tc_fence_after();
            for (int i = 0; i < KB; ++i, ++ks) {
                const uint32_t st = ks % STAGES, ph = (ks / STAGES) & 1;
                mbar_wait(&full[st], ph);
                tc_fence_after();
                uint8_t* sb = smem + st * SLOT;
                if (!NOMMA) {
                    const uint64_t da = sdesc_k_sw128(sb), db = sdesc_k_sw128(sb + WB);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (M == 2) mma_cg2(tb + ab * 256, da + 2 * k, db + 2 * k, idesc, (i | k) ? 1u : 0u);
                        else tc_mma_bf16(tb + ab * 256, da + 2 * k, db + 2 * k, idesc, (i | k) ? 1u : 0u);
                    }
                }
                if (M == 2) commit_cg2_mc(&empty[st], 3);
                else if (M == 1) commit_cg1_mc(&empty[st], 3);
                else tc_commit(&empty[st]);
            }
            if (M == 2) commit_cg2_mc(&accf[ab], 3);
            else tc_commit(&accf[ab]);
        }
    } else if (warp >= 2 && threadIdx.x == 64) {
        uint32_t n = 0;
        for (int it = unit; it < nitems; it += units, ++n) {
            const uint32_t ab = n & 1;
            mbar_wait(&accf[ab], (n >> 1) & 1);
            tc_fence_after();
            if (M == 2) mbar_arrive_cluster(dsmem_addr(smem_u32(&acce[ab]), 0));
            else mbar_arrive(&acce[ab]);
        }
    }
    tc_fence_before();
    if (M) cluster_sync_all(); else __syncthreads();
    if (warp == 1) tmem_dealloc(tb, 512);
}

template <int MODE, int STAGES, int TNMAX>
void run(const char* name, void* W, size_t wrows_total, void* X, int K, int nf, int TN, int G, int reps = 8, int wl2 = 0,
         int tiled = 0, int pfd = 0, int nox = 0) {
    constexpr int M = MODE & 7;
    constexpr int SLOT = 128 * 64 * 2 + TNMAX * 128;
    const int smem = STAGES * SLOT + 1024 + 256;
    auto fn = kern<MODE, STAGES, TNMAX>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    CUtensorMap tw, tx;
    if (wl2) wrows_total = (size_t)nf * reps;
    if (tiled) make_tmap_bf16_2d(&tw, W, 64, wrows_total * (K / 64), 128, 64, 128);
    else make_tmap_bf16_2d(&tw, W, K, wrows_total, K * 2, 64, 128);
    make_tmap_bf16_2d(&tx, X, K, 384, K * 2, 64, M ? TN / 2 : TN);
    CUtensorMap* d;
    cudaMalloc(&d, 2 * sizeof(CUtensorMap));
    cudaMemcpy(d, &tw, sizeof(tw), cudaMemcpyHostToDevice);
    cudaMemcpy(d + 1, &tx, sizeof(tx), cudaMemcpyHostToDevice);
    P p{};
    p.tw = d;
    p.tx = d + 1;
    p.K = K;
    p.TN = TN;
    p.tiles_f = M ? nf / 256 : nf / 128;
    p.tiles_t = 384 / TN;
    p.reps = reps;
    p.wl2 = wl2;
    p.tiled = tiled;
    p.pfd = pfd;
    p.nox = nox;
    p.wbase = (const uint8_t*)W;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = M ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int rows_per_launch = nf * reps;
    const int nrot = (int)(wrows_total / rows_per_launch);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) {
        p.wrow0 = (i % nrot) * rows_per_launch;
        cudaLaunchKernelEx(&cfg, fn, p);
    }
    const int R = 40;
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) {
        p.wrow0 = ((i + 3) % nrot) * rows_per_launch;
        cudaLaunchKernelEx(&cfg, fn, p);
    }
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1000.0 / R;
    const int items = p.tiles_f * p.tiles_t;
    // bytes landed in smem (all CTAs): W once per (item), X once per CTA per item
    const double wbytes = (double)nf * K * 2 * p.tiles_t * reps;
    const double xbytes = nox ? 0.0 : (double)384 * K * 2 * (M == 1 ? p.tiles_f * 2 : p.tiles_f) * reps;
    const double flops = 2.0 * nf * 384 * K * reps;
    printf("%-34s G=%3d items=%4d  %7.2f us/rep  ingress %5.2f TB/s (W %5.1f MB X %5.1f MB)  %6.1f TFLOP/s  %s\n", name, G,
           items, us / reps, (wbytes + xbytes) / us * 1e-6, wbytes * 1e-6, xbytes * 1e-6, flops / us * 1e-6,
           e ? cudaGetErrorString(e) : "");
    cudaFree(d);
}

}  // namespace

int main(int argc, char** argv) {
    const int which = argc > 1 ? atoi(argv[1]) : 0;
    const size_t wrows = 8192 * 16;  // 16 x [8192][2048] bf16 = 512 MB weight rotation (> L2)
    void *W, *X;
    cudaMalloc(&W, wrows * 2048 * 2 * 2);  // K up to 4096
    cudaMalloc(&X, (size_t)384 * 8192 * 2);
    cudaMemset(W, 0, wrows * 2048 * 2 * 2);
    cudaMemset(X, 0, (size_t)384 * 8192 * 2);
    if (which == 0) {
    // MLP1: nf 8192, K 2048
    run<0, 4, 192>("mlp1 1cta TN192 S4", W, wrows, X, 2048, 8192, 192, 128);
    run<8, 4, 192>("mlp1 1cta TN192 S4 nomma", W, wrows, X, 2048, 8192, 192, 128);
    run<0, 4, 256>("mlp1 1cta TN128 S4", W, wrows, X, 2048, 8192, 128, 148);
    run<0, 3, 256>("mlp1 1cta TN256 S3", W, wrows, X, 2048, 8192, 256, 148);
    run<8, 3, 256>("mlp1 1cta TN256 S3 nomma", W, wrows, X, 2048, 8192, 256, 148);
    run<1, 4, 192>("mlp1 mc2 TN192 S4", W, wrows, X, 2048, 8192, 192, 128);
    run<9, 4, 192>("mlp1 mc2 TN192 S4 nomma", W, wrows, X, 2048, 8192, 192, 128);
    run<2, 4, 192>("mlp1 cg2 TN192 S4", W, wrows, X, 2048, 8192, 192, 128);
    run<2, 5, 192>("mlp1 cg2 TN192 S5", W, wrows, X, 2048, 8192, 192, 128);
    run<10, 5, 192>("mlp1 cg2 TN192 S5 nomma", W, wrows, X, 2048, 8192, 192, 128);
    run<2, 4, 256>("mlp1 cg2 TN256 S4", W, wrows, X, 2048, 8192, 256, 148);
    run<2, 6, 128>("mlp1 cg2 TN128 S6", W, wrows, X, 2048, 8192, 128, 148);
    // QKV: nf 3072, K 2048
    run<0, 8, 64>("qkv 1cta TN64 S8", W, wrows, X, 2048, 3072, 64, 144);
    run<8, 8, 64>("qkv 1cta TN64 S8 nomma", W, wrows, X, 2048, 3072, 64, 144);
    run<0, 5, 128>("qkv 1cta TN128 S5", W, wrows, X, 2048, 3072, 128, 144);
    run<2, 8, 64>("qkv cg2 TN64 S8", W, wrows, X, 2048, 3072, 64, 144);
    run<2, 6, 128>("qkv cg2 TN128 S6", W, wrows, X, 2048, 3072, 128, 144);
    run<10, 8, 64>("qkv cg2 TN64 S8 nomma", W, wrows, X, 2048, 3072, 64, 144);
    // O: nf 2048, K 1024
    run<0, 8, 64>("o 1cta TN64 S8", W, wrows, X, 1024, 2048, 64, 96);
    run<2, 8, 64>("o cg2 TN64 S8", W, wrows, X, 1024, 2048, 64, 96);
    } else if (which == 2) {
    // weights L2-resident (evict_last, re-read) vs streamed from HBM (evict_first)
    for (int wl2 : {0, 1}) {
        const char* sfx = wl2 ? " W-in-L2" : " W-HBM";
        char nm[64];
        snprintf(nm, sizeof nm, "qkv 1cta TN64 S8%s", sfx); run<0, 8, 64>(nm, W, wrows, X, 2048, 3072, 64, 144, 2, wl2);
        snprintf(nm, sizeof nm, "qkv 1cta TN64 S8 nomma%s", sfx); run<8, 8, 64>(nm, W, wrows, X, 2048, 3072, 64, 144, 2, wl2);
        snprintf(nm, sizeof nm, "mlp1 1cta TN192 S4%s", sfx); run<0, 4, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, wl2);
        snprintf(nm, sizeof nm, "mlp1 cg2 TN192 S5%s", sfx); run<2, 5, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, wl2);
        snprintf(nm, sizeof nm, "mlp1 cg2 TN192 S6%s", sfx); run<2, 6, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, wl2);
        snprintf(nm, sizeof nm, "o 1cta TN64 S8%s", sfx); run<0, 8, 64>(nm, W, wrows, X, 1024, 2048, 64, 96, 2, wl2);
        snprintf(nm, sizeof nm, "mlp1 cg2 TN96 S8%s", sfx); run<2, 8, 96>(nm, W, wrows, X, 2048, 8192, 96, 148, 2, wl2);
        snprintf(nm, sizeof nm, "mlp1 1cta TN96 S8%s", sfx); run<0, 8, 96>(nm, W, wrows, X, 2048, 8192, 96, 148, 2, wl2);
    }
    } else if (which == 3) {
    // weights from HBM: row-major vs tiled (contiguous 16 KB boxes), L2 lookahead prefetch distance
    for (int tiled : {0, 1})
        for (int pfd : {0, 4, 8, 16}) {
            char nm[64];
            snprintf(nm, sizeof nm, "mlp1 1cta TN192 S4 t%d pf%d", tiled, pfd); run<0, 4, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, 0, tiled, pfd);
            snprintf(nm, sizeof nm, "mlp1 cg2 TN192 S5 t%d pf%d", tiled, pfd); run<2, 5, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, 0, tiled, pfd);
            snprintf(nm, sizeof nm, "qkv 1cta TN128 S5 t%d pf%d", tiled, pfd); run<0, 5, 128>(nm, W, wrows, X, 2048, 3072, 128, 144, 2, 0, tiled, pfd);
            snprintf(nm, sizeof nm, "qkv 1cta TN64 S8 t%d pf%d", tiled, pfd); run<0, 8, 64>(nm, W, wrows, X, 2048, 3072, 64, 144, 2, 0, tiled, pfd);
            snprintf(nm, sizeof nm, "o 1cta TN128 S5 t%d pf%d", tiled, pfd); run<0, 5, 128>(nm, W, wrows, X, 1024, 2048, 128, 148, 2, 0, tiled, pfd);
            snprintf(nm, sizeof nm, "o 1cta TN64 S8 t%d pf%d", tiled, pfd); run<0, 8, 64>(nm, W, wrows, X, 1024, 2048, 64, 148, 2, 0, tiled, pfd);
        }
    } else if (which == 4) {
    // pure HBM weight streaming (no X, no MMA): unique rows per CTA (tiles_t = 1 via TN = 384 is not
    // supported, so TN = 192 with 2 token tiles re-reads each W tile twice -> report both)
    for (int G : {64, 128, 148}) {
        char nm[64];
        snprintf(nm, sizeof nm, "W only S4 G%d", G); run<8, 4, 192>(nm, W, wrows, X, 2048, 8192, 192, G, 2, 0, 0, 0, 1);
        snprintf(nm, sizeof nm, "W only S8 G%d", G); run<8, 8, 64>(nm, W, wrows, X, 2048, 8192, 192, G, 2, 0, 0, 0, 1);
        snprintf(nm, sizeof nm, "W only tiled S8 G%d", G); run<8, 8, 64>(nm, W, wrows, X, 2048, 8192, 192, G, 2, 0, 1, 0, 1);
    }
    } else if (which == 5) {
    // pure HBM streaming (W only, tiled) with L2 lookahead prefetch; then the MLP1 mainloop with it
    for (int pfd : {0, -4, -8, -16, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "W only tiled S4 G128 pf%d", pfd); run<8, 4, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, 0, 1, pfd, 1);
        snprintf(nm, sizeof nm, "W only tiled S8 G128 pf%d", pfd); run<8, 8, 64>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, 0, 1, pfd, 1);
        snprintf(nm, sizeof nm, "mlp1 1cta TN192 S4 tiled pf%d", pfd); run<0, 4, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, 0, 1, pfd);
        snprintf(nm, sizeof nm, "mlp1 cg2 TN192 S5 tiled pf%d", pfd); run<2, 5, 192>(nm, W, wrows, X, 2048, 8192, 192, 128, 2, 0, 1, pfd);
        snprintf(nm, sizeof nm, "qkv 1cta TN128 S5 tiled pf%d", pfd); run<0, 5, 128>(nm, W, wrows, X, 2048, 3072, 128, 144, 2, 0, 1, pfd);
    }
    } else {
    // per-SM ingress vs grid size and stages (no MMA): is the limit per SM or per chip?
    for (int G : {16, 32, 64, 96, 128, 148}) {
        char nm[64];
        snprintf(nm, sizeof nm, "stream TN192 S4 nomma G%d", G);
        run<8, 4, 192>(nm, W, wrows, X, 2048, 8192, 192, G);
    }
    for (int G : {16, 64, 148}) {
        char nm[64];
        snprintf(nm, sizeof nm, "stream TN64 S8 nomma G%d", G);
        run<8, 8, 64>(nm, W, wrows, X, 2048, 3072, 64, G);
        snprintf(nm, sizeof nm, "stream TN64 S4 nomma G%d", G);
        run<8, 4, 64>(nm, W, wrows, X, 2048, 3072, 64, G);
        snprintf(nm, sizeof nm, "stream TN64 S2 nomma G%d", G);
        run<8, 2, 64>(nm, W, wrows, X, 2048, 3072, 64, G);
    }
    }
    return 0;
}
