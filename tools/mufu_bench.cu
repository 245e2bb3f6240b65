// Dev microbenchmark: SFU (MUFU) throughput per SM on this part: ex2 / tanh /
// rcp with W warps per SM, 16 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bench tools/mufu_bench.cu
#include <cstdio>
template <int OP>
__global__ void k(float* out, int iters) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.001f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float y;
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
            else if (OP == 1) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
            else if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
            else asm volatile("fma.rn.f32 %0, %1, %1, %1;" : "=f"(y) : "f"(v[i]));
            v[i] = y;
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double per = (double)(t1 - t0) / (iters * 16.0);
        printf("op %d warps/SM %d: %.2f cycles per warp-instr per warp -> %.2f lanes/clk/SM\n", OP, blockDim.x / 32, per,
               32.0 * (blockDim.x / 32) / per);
    }
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 1024 * 4);
    for (int op = 0; op < 4; ++op)
        for (int w : {4, 8, 16}) {
            void (*f)(float*, int) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
            f<<<148, w * 32>>>(o, 2000);
            cudaDeviceSynchronize();
        }
    return 0;
}
