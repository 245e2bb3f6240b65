// Dev microbenchmark: epilogue store patterns of the persistent kernel.
// 128 CTAs x 256 threads write a 384 x 8192 bf16 matrix in 128-feature x
// 192-token tiles (the MLP1 output).
#include <cstdio>
#include <cuda_bf16.h>
#include "../paper_2605_08975_b200/csrc/common.cuh"
using namespace alpa;

// (a) thread = feature, 96 tokens per thread (what the TMEM 32x32b layout gives)
__global__ void st_feature_major(__nv_bfloat16* out, int ldo, int gelu) {
  for (int rep = 0; rep < 10; ++rep) {
    const int tf = blockIdx.x % 64, tt = blockIdx.x / 64;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = tf * 128 + (w & 3) * 32 + lane;
    const int t0 = tt * 192 + (w >> 2) * 96;
    for (int c = 0; c < 96; c += 16) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            v[j] = (float)(f + j + c) * 1e-3f;
            if (gelu) v[j] = gelu_fast(v[j]);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[(int64_t)(t0 + c + j) * ldo + f] = __float2bfloat16_rn(v[j] + rep);
    }
  }
}
// (b) thread = 8 consecutive features of one token row (16-B stores, 256 B per row-warp)
__global__ void st_row_major(__nv_bfloat16* out, int ldo, int gelu) {
  for (int rep = 0; rep < 10; ++rep) {
    const int tf = blockIdx.x % 64, tt = blockIdx.x / 64;
    const int tid = threadIdx.x;
    // 192 rows x 16 chunks of 8 features = 3072 items / 256 threads = 12 each
    for (int it = tid; it < 192 * 16; it += 256) {
        const int r = it / 16, ch = it % 16;
        const int f = tf * 128 + ch * 8;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[j] = (float)(f + j + r) * 1e-3f;
            if (gelu) v[j] = gelu_fast(v[j]);
        }
        uint4 pk;
        __nv_bfloat162 b0 = __floats2bfloat162_rn(v[0], v[1]), b1 = __floats2bfloat162_rn(v[2], v[3]);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[4], v[5]), b3 = __floats2bfloat162_rn(v[6], v[7]);
        pk.x = *reinterpret_cast<uint32_t*>(&b0); pk.y = *reinterpret_cast<uint32_t*>(&b1);
        pk.z = *reinterpret_cast<uint32_t*>(&b2); pk.w = *reinterpret_cast<uint32_t*>(&b3);
        pk.x += rep;
        *reinterpret_cast<uint4*>(out + (int64_t)(tt * 192 + r) * ldo + f) = pk;
    }
  }
}

int main() {
    __nv_bfloat16* out;
    cudaMalloc(&out, (size_t)384 * 8192 * 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int gelu = 0; gelu < 2; ++gelu) {
        for (int k = 0; k < 2; ++k) {
            for (int i = 0; i < 3; ++i) k ? st_row_major<<<128, 256>>>(out, 8192, gelu) : st_feature_major<<<128, 256>>>(out, 8192, gelu);
            cudaEventRecord(a);
            for (int i = 0; i < 50; ++i) k ? st_row_major<<<128, 256>>>(out, 8192, gelu) : st_feature_major<<<128, 256>>>(out, 8192, gelu);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s gelu=%d: %.2f us per launch of 10 tile writes\n", k ? "row-major    " : "feature-major", gelu, ms / 50 * 1000);
        }
    }
    return 0;
}
