// Dev probe: register layout of tcgen05.ld.16x256b (which (lane, column) each
// thread receives), written via 32x32b stores of lane*1000 + column.
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/common.cuh"
using namespace alpa;

__global__ void probe(int* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = slot;
    if (warp == 0) {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = lane * 1000 + j;
        tmem_st8(tb, v);
        for (int j = 0; j < 8; ++j) v[j] = lane * 1000 + 8 + j;
        tmem_st8(tb + 8, v);
        tmem_st_wait();
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tb));
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tb + (16u << 16)));
        tmem_ld_wait();
        uint32_t q[4];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]) : "r"(tb));
        tmem_ld_wait();
        for (int j = 0; j < 4; ++j) out[lane * 12 + j] = q[j];
        for (int j = 0; j < 8; ++j) out[lane * 12 + 4 + j] = r[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 32);
}

int main() {
    int* d;
    cudaMalloc(&d, 32 * 12 * 4);
    probe<<<1, 128>>>(d);
    int h[32 * 12];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    for (int t = 0; t < 32; ++t) {
        printf("t%2d x1@lane0:", t);
        for (int j = 0; j < 4; ++j) printf(" %5d", h[t * 12 + j]);
        printf("   x2@lane16:");
        for (int j = 0; j < 8; ++j) printf(" %5d", h[t * 12 + 4 + j]);
        printf("\n");
    }
    return 0;
}
