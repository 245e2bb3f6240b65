// Open-loop evaluation metrics on the device for a batch of scenes
// (minivla eval.cpp:14-59): min_ade and diversity of the N generated
// trajectories of each scene.  fp64 with the reference's exact operation
// order (explicit round-to-nearest intrinsics, no FMA contraction), so the
// results are bit-identical to the reference's.
#include <cmath>
#include <vector>

#include "ctx.h"

namespace alpa {
namespace {

// mean_displacement (eval.cpp:14-25): mean over poses of sqrt(dx^2 + dy^2),
// double, summed in pose order.
__device__ double mean_disp(const float* a, const float* b, int steps) {
    double sum = 0.0;
    for (int i = 0; i < steps; ++i) {
        const double dx = __dsub_rn((double)a[i * 3], (double)b[i * 3]);
        const double dy = __dsub_rn((double)a[i * 3 + 1], (double)b[i * 3 + 1]);
        sum = __dadd_rn(sum, __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))));
    }
    return __ddiv_rn(sum, (double)steps);
}

// One thread per (scene, term): terms [0, n) = sample k vs the ground truth,
// terms [n, n + n(n-1)/2) = sample pairs (i < j) in row-major order.
__global__ void md_kernel(const float* __restrict__ traj, const float* __restrict__ gt, int scenes, int n,
                          int steps, double* __restrict__ md) {
    const int terms = n + n * (n - 1) / 2;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (tid >= (long long)scenes * terms) return;
    const int s = (int)(tid / terms), k = (int)(tid % terms);
    const float* ts = traj + (size_t)s * n * steps * 3;
    if (k < n) {
        md[tid] = gt ? mean_disp(ts + (size_t)k * steps * 3, gt + (size_t)s * steps * 3, steps) : 0.0;
        return;
    }
    int p = k - n, i = 0;
    while (p >= n - 1 - i) {
        p -= n - 1 - i;
        ++i;
    }
    const int j = i + 1 + p;
    md[tid] = mean_disp(ts + (size_t)i * steps * 3, ts + (size_t)j * steps * 3, steps);
}

// One thread per scene: min over samples in order (std::min keeps the first
// of equals, eval.cpp:39-46), pair sum in order / pair count (eval.cpp:48-59).
__global__ void reduce_kernel(const double* __restrict__ md, int scenes, int n, double* __restrict__ min_ade,
                              double* __restrict__ div) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= scenes) return;
    const int terms = n + n * (n - 1) / 2;
    const double* m = md + (size_t)s * terms;
    if (min_ade) {
        double best = m[0];
        for (int k = 1; k < n; ++k) best = m[k] < best ? m[k] : best;
        min_ade[s] = best;
    }
    if (div) {
        double sum = 0.0;
        long long pairs = 0;
        for (int k = n; k < terms; ++k) {
            sum = __dadd_rn(sum, m[k]);
            ++pairs;
        }
        div[s] = __ddiv_rn(sum, (double)pairs);
    }
}

}  // namespace

void eval_open_loop_device(Ctx& c, const float* d_traj, const float* d_gt, int64_t scenes, int64_t n,
                           int64_t steps, double* d_min_ade, double* d_div, cudaStream_t s) {
    if (n < 1) fail(ALPA_ERR_INTERNAL, "min_ade: no samples");
    if (d_div && n < 2) fail(ALPA_ERR_INTERNAL, "diversity: need at least 2 samples");
    if (d_min_ade && !d_gt) fail(ALPA_ERR_CONFIG, "min_ade needs the ground-truth trajectories");
    if (scenes < 1) return;
    const int64_t terms = n + n * (n - 1) / 2;
    const size_t need = (size_t)(scenes * terms) * sizeof(double);
    if (c.eval_scratch_bytes < need) {
        if (c.eval_scratch) c.dfree(c.eval_scratch);
        c.eval_scratch = c.dalloc(need);
        c.eval_scratch_bytes = need;
    }
    double* md = static_cast<double*>(c.eval_scratch);
    const long long total = scenes * terms;
    md_kernel<<<(unsigned)((total + 127) / 128), 128, 0, s>>>(d_traj, d_gt, (int)scenes, (int)n, (int)steps, md);
    ALPA_CUDA(cudaGetLastError());
    reduce_kernel<<<(unsigned)((scenes + 127) / 128), 128, 0, s>>>(md, (int)scenes, (int)n, d_min_ade, d_div);
    ALPA_CUDA(cudaGetLastError());
}

}  // namespace alpa
