// extern "C" boundary (include/alpa_action.h).  Maps the reference's
// exception taxonomy onto return codes and owns the K-loop CUDA graph.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "ctx.h"

using alpa::Ctx;
using alpa::Error;
using alpa::fail;

namespace {

thread_local std::string g_last_error;

template <typename Fn>
int guarded(Ctx* c, Fn&& fn) {
    try {
        fn();
        return ALPA_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        if (c) c->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        if (c) c->err = e.what();
        return ALPA_ERR_INTERNAL;
    }
}

// ModelConfig::validate (model.cpp:9-24) plus this build's kernel limits.
void validate(const alpa_model_cfg& c) {
    if (c.decoder_blocks < 1) fail(ALPA_ERR_CONFIG, "decoder_blocks must be >= 1");
    if (c.vision_blocks < 0) fail(ALPA_ERR_CONFIG, "vision_blocks must be >= 0");
    if (c.hidden_dim < 1 || c.action_hidden_dim < 1)
        fail(ALPA_ERR_CONFIG, "hidden dimensions must be positive");
    if (c.heads < 1 || c.kv_dim < 1 || c.kv_dim % c.heads != 0)
        fail(ALPA_ERR_CONFIG, "kv_dim must be a positive multiple of heads");
    if (c.vocab_size < 128) fail(ALPA_ERR_CONFIG, "vocab_size must be >= 128");
    if (c.patch_size < 1) fail(ALPA_ERR_CONFIG, "patch_size must be >= 1");
    if (c.action_steps != 64) fail(ALPA_ERR_CONFIG, "action_steps must be 64");
    if (c.diffusion_iters < 1) fail(ALPA_ERR_CONFIG, "diffusion_iters must be >= 1");
    if (!(c.update_scale > 0.0f)) fail(ALPA_ERR_CONFIG, "update_scale must be > 0");
    if (c.kv_dim / c.heads > 128) fail(ALPA_ERR_CONFIG, "head_dim must be <= 128 in this build");
    if (c.dtype != ALPA_DTYPE_F32 && c.dtype != ALPA_DTYPE_BF16)
        fail(ALPA_ERR_CONFIG, "dtype must be ALPA_DTYPE_F32 or ALPA_DTYPE_BF16");
    if (c.dtype == ALPA_DTYPE_BF16 && (c.action_hidden_dim % 128 != 0 || c.kv_dim % 128 != 0))
        fail(ALPA_ERR_CONFIG,
             "bf16 tensor-core path needs action_hidden_dim and kv_dim multiples of 128");
}

// Rng::normal (common.cpp:48-55) over splitmix64 (common.hpp:36-59): host
// side so the noise is bit-identical to the reference's (glibc logf/sqrtf/cosf).
struct HostRng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    float next_float() { return static_cast<float>(next() >> 40) * (1.0f / 16777216.0f); }
    float normal() {
        float u1 = next_float();
        float u2 = next_float();
        if (u1 < 1e-12f) u1 = 1e-12f;
        const float r = std::sqrt(-2.0f * std::log(u1));
        return r * std::cos(6.28318530717958647692f * u2);
    }
};

void* pinned(Ctx& c, size_t elems) {
    if (c.pinned_elems < elems) {
        if (c.pinned) cudaFreeHost(c.pinned);
        c.pinned = nullptr;
        ALPA_CUDA(cudaMallocHost(&c.pinned, elems * sizeof(float)));
        c.pinned_elems = elems;
    }
    return c.pinned;
}

void check_request(Ctx& c, const alpa_request& r) {
    if (!c.weights_ready) fail(ALPA_ERR_INTERNAL, "weights not loaded");
    if (r.num_trajectories < 1) fail(ALPA_ERR_CONFIG, "num_trajectories must be >= 1");
    if (r.executor == ALPA_EXEC_GRAPH && r.kv_strategy == ALPA_KV_DYNAMIC)
        fail(ALPA_ERR_CONFIG,
             "graph executor requires the static kv strategy (fixed buffer addresses)");
    if (!c.prefix) fail(ALPA_ERR_INTERNAL, "kv cache: action KV write before reasoning sealed");
    if (r.topology == ALPA_TOPOLOGY_SINGLE) {
        if (c.prefix_n != 1)
            fail(ALPA_ERR_INTERNAL, "replicate_for_batch: source cache must have batch 1");
    } else {
        // Multi topology: the cache batch must equal N (pipeline.cpp:411-413)
        // unless an explicit lane map was bound (alpa_set_lane_prefix).
        if (c.lane_map_host.empty() && c.prefix_n != r.num_trajectories)
            fail(ALPA_ERR_INTERNAL, "kv batch does not match the requested trajectory count");
    }
}

// actions_to_trajectory's speed check (pipeline.cpp:125-127): only when a
// trajectory is actually produced (the reference throws it in postprocessing).
void check_v0(const alpa_request& r) {
    if (!(r.v0 >= 0.0f) || !std::isfinite(r.v0))
        fail(ALPA_ERR_INTERNAL, "actions_to_trajectory: invalid initial speed");
}

void upload_lane_map(Ctx& c, const alpa_request& r) {
    const int64_t n = r.num_trajectories;
    std::vector<int32_t> map(n, 0);
    if (r.topology != ALPA_TOPOLOGY_SINGLE) {
        if (!c.lane_map_host.empty()) {
            for (int64_t l = 0; l < n; ++l)
                map[l] = c.lane_map_host[(size_t)std::min<int64_t>(l, (int64_t)c.lane_map_host.size() - 1)];
        } else if (c.prefix_n == n) {
            for (int64_t l = 0; l < n; ++l) map[l] = (int32_t)l;
        }
    }
    for (int32_t v : map)
        if (v < 0 || v >= c.prefix_n) fail(ALPA_ERR_CONFIG, "lane prefix index out of range");
    int64_t uni = map.empty() ? 0 : map[0];
    for (int32_t v : map)
        if (v != uni) uni = -1;
    if (uni != c.uniform_prefix) {
        c.uniform_prefix = uni;  // selects the attention kernel captured in the graph
        alpa::invalidate_graph(c);
    }
    ALPA_CUDA(cudaMemcpyAsync(c.ws.lane_map, map.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice,
                              c.stream));
}

// Timing events between the iterations (recorded as external event nodes
// when the loop is captured, so they time the graph replay too).
void iter_events(Ctx& c, int64_t K) {
    const int64_t need = std::min<int64_t>(K, ALPA_MAX_ITER_MS) + 1;
    while ((int64_t)c.iter_ev.size() < need) {
        cudaEvent_t e;
        ALPA_CUDA(cudaEventCreate(&e));
        c.iter_ev.push_back(e);
    }
}
void record_iter(Ctx& c, int64_t k, cudaStream_t s, bool capturing) {
    if (k >= (int64_t)c.iter_ev.size()) return;
    if (capturing)  // an event-record node of the graph, usable for timing
        ALPA_CUDA(cudaEventRecordWithFlags(c.iter_ev[k], s, cudaEventRecordExternal));
    else
        ALPA_CUDA(cudaEventRecord(c.iter_ev[k], s));
}

// Runs the whole K loop + rollout on c.ws buffers (actions already there).
// Graph executor: the K iterations and the rollout are ONE captured CUDA
// graph (model.cpp:607-636 captures one iteration and replays it K-2 times;
// here the whole loop replays with no host round-trip).  v0 and the
// non-finite flag live in device scalars so the graph is reusable.
void run_loop(Ctx& c, const alpa_request& r, int64_t K, alpa_stats* st) {
    const int64_t n = r.num_trajectories;
    cudaStream_t s = c.stream;
    const float v0 = r.v0;
    ALPA_CUDA(cudaMemcpyAsync(c.d_scalars, &v0, sizeof(float), cudaMemcpyHostToDevice, s));
    alpa::prepare_iteration(c, n);
    if (r.executor == ALPA_EXEC_GRAPH) {
        if (!c.graph.exec || c.graph.n != n || c.graph.k != K) {
            alpa::invalidate_graph(c);
            cudaGraph_t g = nullptr;
            ALPA_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            c.last_launches = 0;
            iter_events(c, K);
            try {
                record_iter(c, 0, s, true);
                for (int64_t it = 0; it < K; ++it) {
                    alpa::enqueue_iteration(c, n, s);
                    record_iter(c, it + 1, s, true);
                }
                alpa::enqueue_rollout(c, n, c.ws.actions, c.ws.traj, s);
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            ALPA_CUDA(cudaStreamEndCapture(s, &g));
            ALPA_CUDA(cudaGraphInstantiate(&c.graph.exec, g, 0));
            cudaGraphDestroy(g);
            c.graph.n = n;
            c.graph.k = K;
            c.graph.nodes = c.last_launches;
        }
        ALPA_CUDA(cudaGraphLaunch(c.graph.exec, s));
        if (st) {
            st->graph_launches = 1;
            st->graph_nodes = c.graph.nodes;
            st->kernel_launches = c.graph.nodes;
        }
    } else {
        c.last_launches = 0;
        iter_events(c, K);
        record_iter(c, 0, s, false);
        for (int64_t it = 0; it < K; ++it) {
            alpa::enqueue_iteration(c, n, s);
            record_iter(c, it + 1, s, false);
        }
        alpa::enqueue_rollout(c, n, c.ws.actions, c.ws.traj, s);
        if (st) {
            st->graph_launches = 0;
            st->graph_nodes = 0;
            st->kernel_launches = c.last_launches;
        }
    }
    c.iter_ev_used = std::min<int64_t>(K, ALPA_MAX_ITER_MS);
}

// After the stream synchronised: per-iteration times into the stats.
void fill_iter_ms(Ctx& c, alpa_stats* st) {
    if (!st) return;
    st->n_iter = c.iter_ev_used;
    for (int64_t k = 0; k < c.iter_ev_used; ++k) {
        float ms = 0.f;
        ALPA_CUDA(cudaEventElapsedTime(&ms, c.iter_ev[k], c.iter_ev[k + 1]));
        st->iter_ms[k] = ms;
    }
    st->bytes_allocated = (int64_t)c.dev_bytes;
}

int64_t kv_bytes(const Ctx& c, const alpa_request& r) {
    // footprint_bytes (kv_cache.cpp:365-372): live tokens r + 64 per lane of
    // the (replicated) cache, f32 elements, every block.
    return c.cfg.decoder_blocks * r.num_trajectories * (c.prefix_r + c.steps()) * c.kv() * 2 * 4;
}

}  // namespace

void alpa::Ctx::dfree(void* p) {
    for (size_t i = 0; i < allocations.size(); ++i)
        if (allocations[i] == p) {
            cudaFree(p);
            allocations.erase(allocations.begin() + i);
            return;
        }
}

extern "C" {

const char* alpa_version(void) { return "alpa_action 0.1 sm_100a"; }

void alpa_default_cfg(alpa_model_cfg* c) {
    // fixtures/default_config.json model block
    std::memset(c, 0, sizeof(*c));
    c->vision_blocks = 4;
    c->decoder_blocks = 6;
    c->hidden_dim = 64;
    c->action_hidden_dim = 32;
    c->kv_dim = 32;
    c->heads = 4;
    c->vocab_size = 512;
    c->patch_size = 14;
    c->action_steps = 64;
    c->diffusion_iters = 10;
    c->update_scale = 0.1f;
    c->dtype = ALPA_DTYPE_F32;
    c->weight_seed = 1234;
}

int alpa_validate_cfg(const alpa_model_cfg* cfg) {
    return guarded(nullptr, [&] {
        if (!cfg) fail(ALPA_ERR_CONFIG, "null config");
        validate(*cfg);
    });
}

int alpa_ctx_create(const alpa_model_cfg* cfg, int device, alpa_ctx** out) {
    Ctx* c = nullptr;
    int rc = guarded(nullptr, [&] {
        if (!cfg || !out) fail(ALPA_ERR_CONFIG, "null argument");
        validate(*cfg);
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
            fail(ALPA_ERR_INTERNAL, "no CUDA device available (this library has no CPU fallback)");
        if (device < 0 || device >= ndev) fail(ALPA_ERR_CONFIG, "device index out of range");
        ALPA_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        ALPA_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            fail(ALPA_ERR_INTERNAL, std::string("sm_100a build needs a Blackwell B200, got ") + prop.name);
        c = new Ctx();
        c->cfg = *cfg;
        c->device = device;
        ALPA_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        ALPA_CUDA(cudaEventCreate(&c->ev0));
        ALPA_CUDA(cudaEventCreate(&c->ev1));
        c->d_scalars = (float*)c->dalloc(16 * sizeof(float));
        ALPA_CUDA(cudaMemset(c->d_scalars, 0, 16 * sizeof(float)));
    });
    if (rc != ALPA_OK) {
        delete c;
        return rc;
    }
    *out = reinterpret_cast<alpa_ctx*>(c);
    return ALPA_OK;
}

void alpa_ctx_destroy(alpa_ctx* h) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->graph.exec) cudaGraphExecDestroy(c->graph.exec);
    try {
        alpa::reasoning_release(*c);  // decode-step graph, pinned slots
    } catch (...) {
    }
    for (void* p : c->allocations) cudaFree(p);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (cudaEvent_t e : c->iter_ev) cudaEventDestroy(e);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* alpa_last_error(const alpa_ctx* h) {
    const Ctx* c = reinterpret_cast<const Ctx*>(h);
    return c ? c->err.c_str() : g_last_error.c_str();
}

int alpa_set_stream(alpa_ctx* h, void* stream) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        cudaSetDevice(c->device);
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        if (!s) {
            if (!c->own_stream) {
                ALPA_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
                c->own_stream = true;
            }
            return;
        }
        if (c->own_stream && c->stream) {
            cudaStreamSynchronize(c->stream);
            cudaStreamDestroy(c->stream);
        }
        c->stream = s;
        c->own_stream = false;
    });
}

int64_t alpa_weight_stream_offset(const alpa_model_cfg* cfg) { return alpa::stream_offset(*cfg); }
int64_t alpa_action_param_count(const alpa_model_cfg* cfg) { return alpa::param_count(*cfg); }

int alpa_load_weights_seeded(alpa_ctx* h, uint64_t seed, int64_t offset) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        cudaSetDevice(c->device);
        if (c->weights_ready) fail(ALPA_ERR_INTERNAL, "weights already loaded on this context");
        alpa::load_weights(*c, nullptr, 0, seed, offset < 0 ? alpa::stream_offset(c->cfg) : offset);
    });
}

int alpa_load_weights_host(alpa_ctx* h, const float* arena, int64_t count) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !arena) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        if (c->weights_ready) fail(ALPA_ERR_INTERNAL, "weights already loaded on this context");
        alpa::load_weights(*c, arena, count, 0, 0);
    });
}

int alpa_bind_prefix(alpa_ctx* h, const float* kv, int64_t n_prefix, int64_t r) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !kv) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        alpa::make_prefix_from_host(*c, kv, n_prefix, r);
        alpa::invalidate_graph(*c);
    });
}

int alpa_bind_prefix_device(alpa_ctx* h, const void* kv, int64_t n_prefix, int64_t r) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !kv) fail(ALPA_ERR_CONFIG, "null argument");
        if (r < 1) fail(ALPA_ERR_INTERNAL, "kv cache: sealing an empty reasoning region");
        if (n_prefix < 1) fail(ALPA_ERR_CONFIG, "prefix count must be >= 1");
        if (c->prefix && c->own_prefix) c->dfree(c->prefix);
        c->prefix = const_cast<void*>(kv);
        c->own_prefix = false;
        c->prefix_n = n_prefix;
        c->prefix_r = r;
        c->prefix_cap = r;
        alpa::refresh_prefix_map(*c);
        alpa::invalidate_graph(*c);
    });
}

int alpa_bind_prefix_synthetic(alpa_ctx* h, uint64_t seed, int64_t r) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        cudaSetDevice(c->device);
        alpa::make_prefix_synthetic(*c, seed, r);
        alpa::invalidate_graph(*c);
    });
}

int alpa_synthesize_prefix(alpa_ctx* h, void* dst, uint64_t seed, int64_t r) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !dst) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        alpa::synthesize_prefix_into(*c, dst, seed, r);
    });
}

int alpa_prefix_device(alpa_ctx* h, void** ptr, int64_t* bytes) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !ptr || !bytes) fail(ALPA_ERR_CONFIG, "null argument");
        if (!c->prefix) fail(ALPA_ERR_INTERNAL, "no prefix bound");
        *ptr = c->prefix;
        *bytes = c->prefix_n * c->cfg.decoder_blocks * 2 * c->pcap() * c->kv() * (int64_t)c->esz();
    });
}

// ---------------------------------------------------------------- reasoning producer
int alpa_reasoning_begin(alpa_ctx* h, int64_t lanes, int64_t capacity) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        cudaSetDevice(c->device);
        alpa::reasoning_begin(*c, lanes, capacity);
    });
}

int alpa_reasoning_prefill(alpa_ctx* h, const float* vision_rows, int64_t P, const int64_t* prompt_ids,
                           int64_t n_prompt, float* logits_out) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        if (P < 0 || n_prompt < 0) fail(ALPA_ERR_CONFIG, "negative token count");
        cudaSetDevice(c->device);
        alpa::reasoning_prefill(*c, vision_rows, P, prompt_ids, n_prompt, logits_out);
    });
}

int alpa_reasoning_decode(alpa_ctx* h, const int64_t* token_ids, float* logits_out) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        cudaSetDevice(c->device);
        alpa::reasoning_decode(*c, token_ids, logits_out);
    });
}

int alpa_reasoning_seal(alpa_ctx* h, int64_t* r_out) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        cudaSetDevice(c->device);
        const int64_t r = alpa::reasoning_seal(*c);
        if (r_out) *r_out = r;
    });
}

int alpa_sample_token(const float* logits, int64_t vocab, int stochastic, uint64_t* rng_state,
                      int64_t* token_out) {
    // host logic only (no context): error text via alpa_last_error(NULL)
    return guarded(nullptr, [&] {
        if (!logits || !token_out || (stochastic && !rng_state)) fail(ALPA_ERR_CONFIG, "null argument");
        if (vocab < 1) fail(ALPA_ERR_INTERNAL, "sample_token: empty logits");
        for (int64_t i = 0; i < vocab; ++i)
            if (std::isnan(logits[i])) fail(ALPA_ERR_INTERNAL, "sample_token: NaN logits");
        if (!stochastic) {
            int64_t best = 0;
            for (int64_t i = 1; i < vocab; ++i)
                if (logits[i] > logits[best]) best = i;
            *token_out = best;
            return;
        }
        double mx = logits[0];
        for (int64_t i = 0; i < vocab; ++i) mx = std::max(mx, static_cast<double>(logits[i]));
        double sum = 0.0;
        for (int64_t i = 0; i < vocab; ++i) sum += std::exp(static_cast<double>(logits[i]) - mx);
        HostRng rng{*rng_state};
        const double u = static_cast<double>(rng.next_float()) * sum;
        *rng_state = rng.s;
        double acc = 0.0;
        for (int64_t i = 0; i < vocab; ++i) {
            acc += std::exp(static_cast<double>(logits[i]) - mx);
            if (u < acc) {
                *token_out = i;
                return;
            }
        }
        *token_out = vocab - 1;
    });
}

int alpa_set_lane_prefix(alpa_ctx* h, const int32_t* map, int64_t n) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c) fail(ALPA_ERR_CONFIG, "null context");
        c->lane_map_host.assign(map, map + (map ? n : 0));
    });
}

int alpa_generate(alpa_ctx* h, const alpa_request* req, float* actions_out, float* traj_out,
                  alpa_stats* st) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !req) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        const alpa_request& r = *req;
        check_request(*c, r);
        if (traj_out) check_v0(r);
        const int64_t n = r.num_trajectories, A = c->steps();
        const int64_t K = r.diffusion_iters > 0 ? r.diffusion_iters : c->cfg.diffusion_iters;
        alpa::ensure_workspace(*c, n);
        upload_lane_map(*c, r);
        const size_t na = n * A * 2, nt = n * A * 3;
        float* host = static_cast<float*>(pinned(*c, na + nt + 1));
        // host noise (pipeline.cpp:415-424), lane seeds keep the global index
        for (int64_t l = 0; l < n; ++l) {
            HostRng rng{r.action_init_seed + static_cast<uint64_t>(r.lane0 + l) * r.action_seed_stride};
            for (int64_t i = 0; i < A * 2; ++i) host[l * A * 2 + i] = rng.normal();
        }
        ALPA_CUDA(cudaEventRecord(c->ev0, c->stream));
        ALPA_CUDA(cudaMemcpyAsync(c->ws.actions, host, na * sizeof(float), cudaMemcpyHostToDevice,
                                  c->stream));
        if (st) std::memset(st, 0, sizeof(*st));
        run_loop(*c, r, K, st);
        float* hact = host;
        float* htraj = host + na;
        ALPA_CUDA(cudaMemcpyAsync(hact, c->ws.actions, na * sizeof(float), cudaMemcpyDeviceToHost,
                                  c->stream));
        ALPA_CUDA(cudaMemcpyAsync(htraj, c->ws.traj, nt * sizeof(float), cudaMemcpyDeviceToHost,
                                  c->stream));
        ALPA_CUDA(cudaMemcpyAsync(htraj + nt, c->d_scalars + 1, sizeof(int),
                                  cudaMemcpyDeviceToHost, c->stream));
        ALPA_CUDA(cudaEventRecord(c->ev1, c->stream));
        ALPA_CUDA(cudaStreamSynchronize(c->stream));
        ALPA_CUDA(cudaGetLastError());
        int bad = 0;
        std::memcpy(&bad, htraj + nt, sizeof(int));
        if (actions_out) std::memcpy(actions_out, hact, na * sizeof(float));
        // non-finite actions fail the rollout (pipeline.cpp:133-135): only an error
        // when trajectories were requested, like the reference's postprocessing
        if (bad && traj_out) fail(ALPA_ERR_INTERNAL, "actions_to_trajectory: non-finite action");
        if (traj_out) std::memcpy(traj_out, htraj, nt * sizeof(float));
        if (st) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, c->ev0, c->ev1);
            st->device_ms = ms;
            fill_iter_ms(*c, st);
            st->kv_bytes = kv_bytes(*c, r);
            st->h2d_bytes = (int64_t)(na * sizeof(float));
            st->d2h_bytes = (int64_t)((na + nt) * sizeof(float));
        }
    });
}

int alpa_generate_device(alpa_ctx* h, const alpa_request* req, const float* d_noise,
                         float* d_actions, float* d_traj, alpa_stats* st) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !req || !d_noise) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        const alpa_request& r = *req;
        check_request(*c, r);
        if (d_traj) check_v0(r);
        const int64_t n = r.num_trajectories, A = c->steps();
        const int64_t K = r.diffusion_iters > 0 ? r.diffusion_iters : c->cfg.diffusion_iters;
        alpa::ensure_workspace(*c, n);
        upload_lane_map(*c, r);
        const size_t na = n * A * 2, nt = n * A * 3;
        if (st) std::memset(st, 0, sizeof(*st));
        if (st) ALPA_CUDA(cudaEventRecord(c->ev0, c->stream));
        ALPA_CUDA(cudaMemcpyAsync(c->ws.actions, d_noise, na * sizeof(float),
                                  cudaMemcpyDeviceToDevice, c->stream));
        run_loop(*c, r, K, st);
        if (d_actions)
            ALPA_CUDA(cudaMemcpyAsync(d_actions, c->ws.actions, na * sizeof(float),
                                      cudaMemcpyDeviceToDevice, c->stream));
        if (d_traj)
            ALPA_CUDA(cudaMemcpyAsync(d_traj, c->ws.traj, nt * sizeof(float),
                                      cudaMemcpyDeviceToDevice, c->stream));
        if (st) {
            ALPA_CUDA(cudaEventRecord(c->ev1, c->stream));
            // the rollout's non-finite flag (pipeline.cpp:133-135) comes back with the
            // stats (the call synchronises anyway); without stats the device flag is
            // readable through alpa_last_rollout_flag_device
            int bad = 0;
            ALPA_CUDA(cudaMemcpyAsync(&bad, c->d_scalars + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            ALPA_CUDA(cudaStreamSynchronize(c->stream));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, c->ev0, c->ev1);
            st->device_ms = ms;
            fill_iter_ms(*c, st);
            st->kv_bytes = kv_bytes(*c, r);
            if (bad && d_traj) fail(ALPA_ERR_INTERNAL, "actions_to_trajectory: non-finite action");
        }
    });
}

int alpa_last_rollout_flag_device(alpa_ctx* h, const int** flag) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !flag) fail(ALPA_ERR_CONFIG, "null argument");
        *flag = reinterpret_cast<const int*>(c->d_scalars + 1);
    });
}

int alpa_profile(alpa_ctx* h, const alpa_request* req, int64_t iters, alpa_kernel_prof* out,
                 int32_t max_out, int32_t* n_out) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !req || !out || !n_out) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        const alpa_request& r = *req;
        check_request(*c, r);
        const int64_t n = r.num_trajectories, A = c->steps();
        alpa::ensure_workspace(*c, n);
        upload_lane_map(*c, r);
        std::vector<float> noise(n * A * 2);
        alpa_host_noise(r.action_init_seed, r.action_seed_stride, r.lane0, n, A, noise.data());
        ALPA_CUDA(cudaMemcpyAsync(c->ws.actions, noise.data(), noise.size() * sizeof(float),
                                  cudaMemcpyHostToDevice, c->stream));
        const float v0 = r.v0;
        ALPA_CUDA(cudaMemcpyAsync(c->d_scalars, &v0, sizeof(float), cudaMemcpyHostToDevice,
                                  c->stream));
        alpa::prepare_iteration(*c, n);
        c->prof.clear();
        c->prof_spans.clear();
        c->ev_next = 0;
        c->prof_on = true;
        try {
            for (int64_t it = 0; it < iters; ++it) alpa::enqueue_iteration(*c, n, c->stream);
            alpa::enqueue_rollout(*c, n, c->ws.actions, c->ws.traj, c->stream);
        } catch (...) {
            c->prof_on = false;
            throw;
        }
        c->prof_on = false;
        ALPA_CUDA(cudaStreamSynchronize(c->stream));
        std::vector<alpa_kernel_prof> agg;
        for (const auto& rec : c->prof) {
            float ms = 0.f;
            ALPA_CUDA(cudaEventElapsedTime(&ms, rec.a, rec.b));
            alpa_kernel_prof* slot = nullptr;
            for (auto& a : agg)
                if (std::strncmp(a.name, rec.tag, sizeof(a.name)) == 0) slot = &a;
            if (!slot) {
                agg.push_back(alpa_kernel_prof{});
                slot = &agg.back();
                std::strncpy(slot->name, rec.tag, sizeof(slot->name) - 1);
            }
            slot->launches += 1;
            slot->total_ms += ms;
            slot->flops += rec.flops;
            slot->bytes += rec.bytes;
        }
        for (const auto& sp : c->prof_spans) {
            // per-op spans inside the persistent launch, reported as "span:<op>"
            char name[sizeof(agg[0].name)] = {0};
            std::snprintf(name, sizeof(name), "span:%s", sp.tag);
            alpa_kernel_prof* slot = nullptr;
            for (auto& a : agg)
                if (std::strncmp(a.name, name, sizeof(a.name)) == 0) slot = &a;
            if (!slot) {
                agg.push_back(alpa_kernel_prof{});
                slot = &agg.back();
                std::strncpy(slot->name, name, sizeof(slot->name) - 1);
            }
            slot->launches += 1;
            slot->total_ms += sp.ms;
            slot->flops += sp.flops;
        }
        c->prof.clear();
        c->prof_spans.clear();
        const int32_t k = (int32_t)std::min<size_t>(agg.size(), (size_t)max_out);
        for (int32_t i = 0; i < k; ++i) out[i] = agg[i];
        *n_out = k;
    });
}


int alpa_debug_mk_trace(alpa_ctx* h, unsigned long long* out, int64_t max_elems, int64_t* n_ops,
                        int64_t* grid) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !out || !n_ops || !grid) fail(ALPA_ERR_CONFIG, "null argument");
        if (!c->mk.d_trace) fail(ALPA_ERR_INTERNAL, "no persistent-kernel trace (ALPA_MK_TRACE=1 + alpa_profile)");
        const size_t n = std::min<size_t>(c->mk.trace_elems, (size_t)max_elems);
        ALPA_CUDA(cudaMemcpy(out, c->mk.d_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        *n_ops = c->mk.n_ops;
        *grid = c->mk.grid;
    });
}

int alpa_eval_open_loop_device(alpa_ctx* h, const float* d_traj, const float* d_gt, int64_t scenes,
                               int64_t n, int64_t steps, double* d_min_ade, double* d_diversity) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !d_traj) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        alpa::eval_open_loop_device(*c, d_traj, d_gt, scenes, n, steps, d_min_ade, d_diversity, c->stream);
    });
}

int alpa_eval_open_loop(alpa_ctx* h, const float* traj, const float* gt, int64_t scenes, int64_t n,
                        int64_t steps, double* min_ade, double* diversity) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !traj) fail(ALPA_ERR_CONFIG, "null argument");
        cudaSetDevice(c->device);
        if (n < 1) fail(ALPA_ERR_INTERNAL, "min_ade: no samples");
        if (diversity && n < 2) fail(ALPA_ERR_INTERNAL, "diversity: need at least 2 samples");
        if (scenes < 1) return;
        const size_t tb = (size_t)(scenes * n * steps * 3) * sizeof(float);
        const size_t gb = gt ? (size_t)(scenes * steps * 3) * sizeof(float) : 0;
        const size_t ob = (size_t)scenes * sizeof(double);
        uint8_t* d = static_cast<uint8_t*>(c->io(tb + gb + 2 * ob + 64));
        float* dt = reinterpret_cast<float*>(d);
        float* dg = gt ? reinterpret_cast<float*>(d + tb) : nullptr;
        double* dm = reinterpret_cast<double*>(d + ((tb + gb + 15) & ~(size_t)15));
        double* dv = dm + scenes;
        ALPA_CUDA(cudaMemcpyAsync(dt, traj, tb, cudaMemcpyHostToDevice, c->stream));
        if (gt) ALPA_CUDA(cudaMemcpyAsync(dg, gt, gb, cudaMemcpyHostToDevice, c->stream));
        alpa::eval_open_loop_device(*c, dt, dg, scenes, n, steps, min_ade ? dm : nullptr,
                                    diversity ? dv : nullptr, c->stream);
        if (min_ade) ALPA_CUDA(cudaMemcpyAsync(min_ade, dm, ob, cudaMemcpyDeviceToHost, c->stream));
        if (diversity) ALPA_CUDA(cudaMemcpyAsync(diversity, dv, ob, cudaMemcpyDeviceToHost, c->stream));
        ALPA_CUDA(cudaStreamSynchronize(c->stream));
    });
}

void alpa_host_noise(uint64_t seed, uint64_t stride, int64_t lane0, int64_t n, int64_t steps,
                     float* out) {
    for (int64_t l = 0; l < n; ++l) {
        HostRng rng{seed + static_cast<uint64_t>(lane0 + l) * stride};
        for (int64_t i = 0; i < steps * 2; ++i) out[l * steps * 2 + i] = rng.normal();
    }
}

float alpa_initial_speed(const float* h) {
    // initial_speed_from_history (pipeline.cpp:150-156)
    const double dx = static_cast<double>(h[15 * 3]) - h[14 * 3];
    const double dy = static_cast<double>(h[15 * 3 + 1]) - h[14 * 3 + 1];
    return static_cast<float>(std::sqrt(dx * dx + dy * dy) / 0.1);
}

int alpa_rollout(alpa_ctx* h, const float* actions, int64_t n, float v0, float* traj) {
    Ctx* c = reinterpret_cast<Ctx*>(h);
    return guarded(c, [&] {
        if (!c || !actions || !traj) fail(ALPA_ERR_CONFIG, "null argument");
        if (!(v0 >= 0.0f) || !std::isfinite(v0))
            fail(ALPA_ERR_INTERNAL, "actions_to_trajectory: invalid initial speed");
        if (n < 1) return;
        cudaSetDevice(c->device);
        const int64_t A = c->steps();
        float* da = static_cast<float*>(c->io((size_t)n * A * 5 * sizeof(float)));
        float* dt = da + n * A * 2;
        ALPA_CUDA(cudaMemcpyAsync(da, actions, n * A * 2 * sizeof(float), cudaMemcpyHostToDevice,
                                  c->stream));
        ALPA_CUDA(cudaMemcpyAsync(c->d_scalars, &v0, sizeof(float), cudaMemcpyHostToDevice,
                                  c->stream));
        alpa::enqueue_rollout(*c, n, da, dt, c->stream);
        int hbad = 0;
        ALPA_CUDA(cudaMemcpyAsync(traj, dt, n * A * 3 * sizeof(float), cudaMemcpyDeviceToHost,
                                  c->stream));
        ALPA_CUDA(cudaMemcpyAsync(&hbad, c->d_scalars + 1, sizeof(int), cudaMemcpyDeviceToHost,
                                  c->stream));
        ALPA_CUDA(cudaStreamSynchronize(c->stream));
        if (hbad) fail(ALPA_ERR_INTERNAL, "actions_to_trajectory: non-finite action");
    });
}

int64_t alpa_kv_footprint_bytes(int64_t blocks, int64_t batch, int64_t tokens, int64_t kv_dim,
                                int64_t elem_bytes) {
    // kv_cache.cpp:22-26
    return blocks * batch * tokens * kv_dim * 2 * elem_bytes;
}

}  // extern "C"
