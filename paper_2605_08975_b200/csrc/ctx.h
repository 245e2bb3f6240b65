// Internal context of the action-generation library (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/alpa_action.h"

namespace alpa {

// Error carrying one of the ALPA_ERR_* codes (reference taxonomy,
// common.hpp:10-23).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

#define ALPA_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            ::alpa::fail(ALPA_ERR_INTERNAL, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// One linear layer on device.  f32 path: w [in][out] (reference layout,
// model.hpp:57).  bf16 path: w = W^T [out][in] bf16 (K-major tcgen05 operand).
struct Linear {
    void* w = nullptr;
    float* b = nullptr;
    int64_t in = 0, out = 0;
    CUtensorMap tmap{};  // bf16: TMA map of W^T, box {64, 128}
    float* colsum = nullptr;  // bf16: sum_k W^T[f][k] (LayerNorm fold), LN consumers only
};

struct Block {
    Linear qkv;  // fused [ah -> 3kv]: q | k | v columns (model.cpp:574-576)
    Linear o, mlp1, mlp2;
};

struct Workspace {
    int64_t n = 0;  // lanes the buffers are sized for
    float* actions = nullptr;  // [N][64][2]
    float* traj = nullptr;     // [N][64][3]
    float* e = nullptr;        // residual stream f32 [M][ah]
    void* x = nullptr;         // LN output / encoder input: f32 or bf16 [M][ah]
    void* qkv = nullptr;       // [M][3kv]: q | action K | action V (in place, no copy)
    void* ctxb = nullptr;      // attention output [M][kv]
    void* h1 = nullptr;        // MLP hidden [M][4ah]
    int* counters = nullptr;   // scratch arrival counters
    float2* stats = nullptr;   // bf16 path: [M][ah/128] (sum, sumsq) of e rows per feature tile
    int32_t* lane_map = nullptr;  // [N] prefix index per lane
    CUtensorMap tm_x{}, tm_ctx{}, tm_h1{};  // bf16 activation maps (B operand)
    CUtensorMap tm_qkv{};                   // q | k | v rows, box {64, 128} (attention)
    int tn = 64;                            // token tile
};

// Per-kernel timing records (alpa_profile): an event pair around each launch.
struct ProfRec {
    const char* tag;
    cudaEvent_t a, b;
    double flops, bytes;
};
// Algorithmic work of one launch (SURVEY.md §8d accounting).
struct KInfo {
    const char* tag;
    double flops, bytes;
};

// Persistent iteration kernel plan (mk.cu): device op list, tensor maps,
// completion / split counters and the split-partial workspace.
struct MkState {
    bool valid = false;
    int64_t n = -1, uniform = -2, r = -1, cap = -1, prefix_n = -1;
    const void* prefix = nullptr;
    void* d_ops = nullptr;
    int n_ops = 0;
    CUtensorMap* d_maps = nullptr;
    int* d_counters = nullptr;
    size_t counter_ints = 0;
    float* ws = nullptr;
    float2* wsml = nullptr;
    unsigned long long* d_tstamp = nullptr;
    unsigned long long* d_trace = nullptr;  // ALPA_MK_TRACE=1: [n_ops][G][8] event times
    size_t trace_elems = 0;
    std::vector<const char*> tags;
    std::vector<double> flops;
    void* fn = nullptr;     // production kernel
    void* fn_tr = nullptr;  // instrumented twin (trace / per-op spans)
    int smem = 0, grid = 0;
};

// Per-op span inside a persistent launch (alpa_profile).
struct ProfSpan {
    const char* tag;
    double ms, flops;
};

struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    int64_t n = -1, k = -1, prefix_id = -2;
    int64_t nodes = 0;
};

// Reasoning-stage language model: reference-layout f32 weights
// ([in][out] + bias, model.cpp:72-101) and the static in-place KV it produces.
struct LangBlock {
    float *wq, *bq, *wk, *bk, *wv, *bv, *wo, *bo, *w1, *b1, *w2, *b2;
};
struct Reasoner {
    bool weights = false;
    std::vector<LangBlock> blocks;
    float *embed = nullptr, *lm_w = nullptr, *lm_b = nullptr;  // token_embed [V][h], lm_head
    int64_t lanes = 0, cap = 0, T = 0, len = 0;  // len: tokens appended per lane
    bool open = false;                 // begun, not sealed
    void* kv = nullptr;                // [lanes][B][2][cap][kv] in the context dtype (the action prefix)
    float* kv32 = nullptr;             // f32 working copy for the LM's own attention (bf16 contexts)
    float* pos = nullptr;              // [cap + 1][h] sinusoid (pipeline.cpp:291-295)
    float *x = nullptr, *xn = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *att = nullptr,
          *h1 = nullptr, *last = nullptr, *logits = nullptr;
    int32_t* ids = nullptr;            // [lanes] decode tokens / [n_prompt] prompt ids
    int64_t rows_cap = 0, ids_cap = 0;
    int64_t* dlen = nullptr;           // device cache length (position of the next token)
    int32_t* h_ids = nullptr;          // pinned [lanes]: the step graph's input ids
    float* h_logits = nullptr;         // pinned [lanes][vocab]: the step graph's output
    cudaGraphExec_t step = nullptr;    // one captured decode step, replayed per token
    std::vector<void*> bufs;           // per-begin allocations
};

struct Ctx {
    alpa_model_cfg cfg{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;

    bool weights_ready = false;
    Linear act_in, mlp1, mlp2, head;  // act_in/head always f32 [in][out]
    std::vector<Block> blocks;
    float* pos = nullptr;  // [64][ah] sinusoid (model.cpp:56-68)
    std::vector<void*> allocations;

    void* prefix = nullptr;  // [n_prefix][B][2][cap][kv] f32 or bf16, tokens [0, r) valid
    bool own_prefix = false;
    int64_t prefix_n = 0, prefix_r = 0;
    // rows per K / V section: the static reasoning capacity when the prefix
    // was produced in place on the device (KvLayout::reasoning_capacity,
    // pipeline.cpp:281-286), else r
    int64_t prefix_cap = 0;
    int64_t pcap() const { return prefix_cap > 0 ? prefix_cap : prefix_r; }
    std::vector<int32_t> lane_map_host;  // multi topology
    int64_t uniform_prefix = 0;          // prefix index shared by every lane, -1 if mixed
    CUtensorMap tm_pre{};                // 2-D view [n_prefix*B*2*cap][kv], box {64, 128}
    bool tm_pre_valid = false;

    Workspace ws;
    MkState mk;
    Reasoner rs;
    std::vector<ProfSpan> prof_spans;
    GraphCache graph;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float* d_scalars = nullptr;  // [0] = v0 (rollout), [1] = non-finite flag (int)
    float* pinned = nullptr;  // host staging
    size_t pinned_elems = 0;
    int64_t last_launches = 0;  // kernels enqueued by the last iteration body
    bool prof_on = false;
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_next = 0;
    std::vector<cudaEvent_t> iter_ev;  // K+1 timing events around the iterations
    int64_t iter_ev_used = 0;
    size_t dev_bytes = 0;              // device bytes allocated by the context
    void* eval_scratch = nullptr;  // eval.cu: per-(scene, term) mean displacements
    size_t eval_scratch_bytes = 0;
    void* io_scratch = nullptr;    // host-buffer entry points (rollout, eval): grown, never per call
    size_t io_scratch_bytes = 0;
    void* io(size_t bytes) {
        if (io_scratch_bytes < bytes) {
            if (io_scratch) dfree(io_scratch);
            io_scratch = dalloc(bytes);
            io_scratch_bytes = bytes;
        }
        return io_scratch;
    }

    bool bf16() const { return cfg.dtype == ALPA_DTYPE_BF16; }
    int64_t ah() const { return cfg.action_hidden_dim; }
    int64_t kv() const { return cfg.kv_dim; }
    int64_t steps() const { return cfg.action_steps; }
    size_t esz() const { return bf16() ? 2 : 4; }

    void* dalloc(size_t bytes) {
        void* p = nullptr;
        ALPA_CUDA(cudaMalloc(&p, bytes < 16 ? 16 : bytes));
        allocations.push_back(p);
        dev_bytes += bytes < 16 ? 16 : bytes;
        return p;
    }
    void dfree(void* p);
};

// weights.cu
void load_weights(Ctx& c, const float* host_arena, int64_t count, uint64_t seed, int64_t offset);
void make_prefix_synthetic(Ctx& c, uint64_t seed, int64_t r);
void synthesize_prefix_into(Ctx& c, void* dst, uint64_t seed, int64_t r);
void make_prefix_from_host(Ctx& c, const float* host, int64_t n_prefix, int64_t r);
int64_t stream_offset(const alpa_model_cfg& c);
// one f32 [in][out] linear (w then b) / a flat array drawn from the weight stream at `base`
void draw_linear_f32(Ctx& c, int64_t base, int64_t in, int64_t out, float* w, float* b);
void draw_array_f32(Ctx& c, int64_t base, int64_t n, float* dst);
// reasoning-stage KV producer (reason.cu)
void reasoning_begin(Ctx& c, int64_t lanes, int64_t capacity);
void reasoning_prefill(Ctx& c, const float* vision_rows, int64_t P, const int64_t* prompt_ids,
                       int64_t n_prompt, float* logits_out);
void reasoning_decode(Ctx& c, const int64_t* ids, float* logits_out);
int64_t reasoning_seal(Ctx& c);
void reasoning_release(Ctx& c);
int64_t param_count(const alpa_model_cfg& c);

// path.cu
void ensure_workspace(Ctx& c, int64_t n);
void enqueue_iteration(Ctx& c, int64_t n, cudaStream_t s);  // one diffusion iteration
void enqueue_rollout(Ctx& c, int64_t n, const float* d_actions, float* d_traj, cudaStream_t s);
void invalidate_graph(Ctx& c);
void refresh_prefix_map(Ctx& c);  // TMA map of the bound prefix (bf16)

// eval.cu: open-loop metrics (eval.cpp:14-59) of [scenes][n][steps][3] trajectories
void eval_open_loop_device(Ctx& c, const float* d_traj, const float* d_gt, int64_t scenes, int64_t n,
                           int64_t steps, double* d_min_ade, double* d_div, cudaStream_t s);

// mk.cu: persistent iteration kernel (bf16 path, uniform prefix)
double gemm_op_cost(int64_t M, int64_t nf, int64_t K, int tn_op, int tn_k, bool split_ok, int G);
bool mk_usable(const Ctx& c);
void mk_prepare(Ctx& c, int64_t n);
void mk_release(Ctx& c);
void mk_enqueue(Ctx& c, int64_t n, cudaStream_t s, unsigned long long* tstamp,
                unsigned long long* trace = nullptr);
// Host-side preparation that must happen outside stream capture.
void prepare_iteration(Ctx& c, int64_t n);

// tma.cu
void make_tmap_bf16_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
void make_tmap_f32_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
void make_tmap_panels(CUtensorMap* m, const void* base, bool f32, uint64_t cols, uint64_t rows,
                      uint64_t row_stride_bytes, uint32_t box_rows, uint32_t panels);
void make_tmap_f32_3d_sw128(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                            uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box1);

}  // namespace alpa
