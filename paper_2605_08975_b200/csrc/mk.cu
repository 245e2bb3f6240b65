// Host side of the persistent iteration kernel (mk.cuh): builds the per-scene
// op plan (device Op[] + tensor maps + counters + split workspace) and
// launches one cooperative kernel per diffusion iteration.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctx.h"
#include "mk.cuh"

namespace alpa {

namespace {

using mk::Op;

int g_num_sms = 0;
int num_sms(Ctx& c) {
    if (!g_num_sms) {
        cudaDeviceProp prop{};
        ALPA_CUDA(cudaGetDeviceProperties(&prop, c.device));
        g_num_sms = prop.multiProcessorCount;
    }
    return g_num_sms;
}

template <int TN, int HD>
void* kernel_ptr(bool tr) {
    return tr ? reinterpret_cast<void*>(mk::iter_kernel<TN, HD, true>)
              : reinterpret_cast<void*>(mk::iter_kernel<TN, HD, false>);
}
template <int TN, int HD>
int kernel_smem() {
    return mk::Cfg<TN, HD>::SMEM;
}

struct KSel {
    void* fn;     // production kernel
    void* fn_tr;  // instrumented twin (ALPA_MK_TRACE / alpa_profile spans)
    int smem;
};
KSel select_kernel(int tn, int hd) {
#define ALPA_MK_CASE(T, D) \
    if (tn == T && hd == D) return {kernel_ptr<T, D>(false), kernel_ptr<T, D>(true), kernel_smem<T, D>()};
    ALPA_MK_CASE(64, 64) ALPA_MK_CASE(64, 128) ALPA_MK_CASE(128, 64) ALPA_MK_CASE(128, 128)
    ALPA_MK_CASE(192, 64) ALPA_MK_CASE(192, 128) ALPA_MK_CASE(256, 64) ALPA_MK_CASE(256, 128)
#undef ALPA_MK_CASE
    fail(ALPA_ERR_INTERNAL, "persistent kernel: unsupported token tile / head dim");
}

// Split-K count: one wave (tiles*S <= G, so the splits of a tile are
// co-resident), TN divisible by S (each split reduces TN/S rows), >= 2 k-blocks
// per split; maximise the CTAs used, prefer the smaller S on ties.
int pick_splits(int tiles, int KB, int tn, int G) {
    if (tiles >= G) return 1;
    int best = 1, used = tiles;
    for (int s = 2; s <= 4; ++s) {  // fix_t sums at most 4 split partials
        if (tn % s || (tn / s) % 16 || tiles * s > G || KB / s < 2) continue;
        const int kbs = (KB + s - 1) / s;
        if ((s - 1) * kbs >= KB) continue;  // every split must own >= 1 k-block
        if (tiles * s > used) {
            best = s;
            used = tiles * s;
        }
    }
    return best;
}

}  // namespace

bool mk_usable(const Ctx& c) {
    // default: the persistent kernel; ALPA_MK=0 selects the per-op kernel
    // sequence (A/B measurements and cross-checks)
    const char* e = getenv("ALPA_MK");
    if ((e && e[0] == '0') || !c.bf16() || !c.tm_pre_valid) return false;
    const int64_t hd = c.kv() / c.cfg.heads;
    return hd == 64 || hd == 128;
}

void mk_release(Ctx& c) {
    MkState& m = c.mk;
    for (void* p : {(void*)m.d_ops, (void*)m.d_maps, (void*)m.d_counters, (void*)m.ws, (void*)m.wsml,
                    (void*)m.d_tstamp, (void*)m.d_trace})
        if (p) c.dfree(p);
    m = MkState{};
}

void mk_prepare(Ctx& c, int64_t n) {
    MkState& m = c.mk;
    if (m.valid && m.n == n && m.prefix == c.prefix && m.uniform == c.uniform_prefix &&
        m.r == c.prefix_r && m.cap == c.pcap() && m.prefix_n == c.prefix_n)
        return;
    mk_release(c);
    const int G = num_sms(c);
    const int64_t A = c.steps(), M = n * A, ah = c.ah(), kv = c.kv(), H = c.cfg.heads, r = c.prefix_r;
    const int hd = (int)(kv / H);
    const int tn = c.ws.tn;
    const int64_t B = c.cfg.decoder_blocks;
    KSel ks = select_kernel(tn, hd);

    // ---- tensor maps (device copies; TMA reads them from global memory)
    std::vector<CUtensorMap> maps;
    auto add_map = [&](const CUtensorMap& t) {
        maps.push_back(t);
        return (int)maps.size() - 1;
    };
    const int mq128 = add_map(c.ws.tm_qkv);
    // activation maps (TMA load operand / TMA store target) per token tile
    std::vector<std::pair<std::pair<const void*, int64_t>, std::pair<int, int>>> act_cache;
    auto act_map = [&](void* base, int64_t inner, int rows) {
        for (auto& e : act_cache)
            if (e.first.first == base && e.first.second == inner && e.second.first == rows) return e.second.second;
        CUtensorMap t{};
        make_tmap_bf16_2d(&t, base, inner, M, inner * 2, 64, rows);
        const int id = add_map(t);
        act_cache.push_back({{base, inner}, {rows, id}});
        return id;
    };
    // token tile per op kind (qkv, o, mlp1, mlp2, enc1, enc2).  The few-feature-tile
    // ops (QKV: 3kv/128 tiles, O: ah/128) take the smallest tile (multiple of 32,
    // >= 64) that still fits one wave -- at N = 6 QKV 24 x 6 = 144 items, O 16 x 6 =
    // 96: their mainloops are bound by the bytes each SM streams, so spreading
    // wins (measured: 64/64 -0.5 ms/scene vs 96/96); the MLPs keep the full tile.
    // At N = 1 (M = 64) the ops are latency-bound with few items: 32-token tiles
    // double the SMs streaming QKV / O weights (measured -0.6 ms/scene at N = 1).
    const int min_tile = M <= 64 ? 32 : 64;
    auto few_tile = [&](int64_t nf) {
        const int64_t tf = nf / 128;
        int best = tn;
        for (int v = tn; v >= min_tile; v -= 32)
            if (tf * ((M + v - 1) / v) <= G) best = v;
        return best;
    };
    // the deep-K split-K ops (MLP2, encoder MLP2) may take a smaller token tile than
    // the kernel's when that packs more tiles x splits onto the SMs (cost model)
    auto split_tile = [&](int64_t nf, int64_t K) {
        int best = tn;
        double bt = gemm_op_cost(M, nf, K, tn, tn, true, G);
        for (int v = tn - 32; v >= 64; v -= 32) {
            const double t = gemm_op_cost(M, nf, K, v, tn, true, G);
            if (t < bt * 0.95) {
                bt = t;
                best = v;
            }
        }
        return best;
    };
    int tno[6] = {few_tile(3 * kv), few_tile(ah), tn, split_tile(ah, 4 * ah), tn, split_tile(ah, 4 * ah)};
    if (const char* e = getenv("ALPA_MK_TN"))
        std::sscanf(e, "%d,%d,%d,%d,%d,%d", &tno[0], &tno[1], &tno[2], &tno[3], &tno[4], &tno[5]);
    for (int& v : tno)
        if (v <= 0 || v > tn || v % 32) v = tn;  // drain: 16-token chunks per warp half
    CUtensorMap t64{};
    make_tmap_bf16_2d(&t64, c.ws.qkv, 3 * kv, M, 3 * kv * 2, 64, 64);
    const int mq64 = add_map(t64);
    const uint64_t pre_rows = (uint64_t)c.prefix_n * B * 2 * c.pcap();
    make_tmap_bf16_2d(&t64, c.prefix, (uint64_t)kv, pre_rows, (uint64_t)kv * 2, 64, 64);
    const int mpre = add_map(t64);
    const int menc1 = add_map(c.mlp1.tmap), menc2 = add_map(c.mlp2.tmap);
    std::vector<int> mblk(B * 4);
    for (int64_t b = 0; b < B; ++b) {
        mblk[b * 4 + 0] = add_map(c.blocks[b].qkv.tmap);
        mblk[b * 4 + 1] = add_map(c.blocks[b].o.tmap);
        mblk[b * 4 + 2] = add_map(c.blocks[b].mlp1.tmap);
        mblk[b * 4 + 3] = add_map(c.blocks[b].mlp2.tmap);
    }
    // ops reference maps by index until the device copy exists (fixed up below)
    auto dm = [&](int i) { return reinterpret_cast<const CUtensorMap*>((uintptr_t)(i + 1)); };

    // ---- ops
    std::vector<Op> ops;
    std::vector<const char*> tags;
    std::vector<double> flops;
    int split_ctr = 0;
    size_t ws_floats = 16, wsml_elems = 16;
    const float2* stats = c.ws.stats;
    auto wb = [](const Linear& L) { return (long long)(L.in * L.out * 2); };
    auto push = [&](Op op, const char* tag, double f) {
        op.dep = ops.empty() ? -1 : (int)ops.size() - 1;
        op.dep_count = ops.empty() ? 0 : ops.back().n_items;
        ops.push_back(op);
        tags.push_back(tag);
        flops.push_back(f);
    };
    // split-K caps per op kind (ALPA_MK_SPLITS="qkv,o,mlp1,mlp2,enc1,enc2"); a
    // split op pays an fp32 partial round trip through L2, so only the deep-K
    // MLP2 (K = 4 ah) splits by default
    int cap[6] = {1, 1, 1, 4, 1, 4};
    // L2 prefetch (cp.async.bulk.prefetch.L2, 1/G per CTA) of the next op's bytes,
    // per issuing op kind: bit 0 QKV -> its block's prefix K/V, 1 O -> MLP1 weights,
    // 2 MLP1 -> MLP2, 3 MLP2 -> next QKV, 4/5 encoder MLPs, 6 attention -> O weights.
    // The GEMM mainloops are bound by L2 -> SM throughput, not HBM: a prefetch issued
    // during a GEMM competes with it and slows the epilogues' L2 traffic (measured,
    // all on: +0.9 ms/scene).  Only attention (not L2-bound) pulls the O weights ahead.
    int pf_mask = 0x40;
    if (const char* e = getenv("ALPA_MK_PF")) pf_mask = (int)strtol(e, nullptr, 0);
    if (const char* e = getenv("ALPA_MK_SPLITS"))
        std::sscanf(e, "%d,%d,%d,%d,%d,%d", &cap[0], &cap[1], &cap[2], &cap[3], &cap[4], &cap[5]);
    auto gemm = [&](const Linear& L, int mw, void* xin, int epi, void* out, int64_t ldo, bool produce,
                    bool consume, const void* pf, long long pfb, const char* tag, int kind) {
        Op op{};
        const int pf_kind = kind;
        if (kind > 5) kind = 3;  // kind 7: MLP2 with the prefix prefetch (pf_mask bit 7)
        const int ttn = tno[kind];
        op.tn = ttn;
        op.kind = mk::OP_GEMM;
        op.epi = epi;
        op.nf = (int)L.out;
        op.k = (int)L.in;
        op.tiles_f = op.nf / 128;
        op.tiles_t = (int)((M + ttn - 1) / ttn);
        const int tiles = op.tiles_f * op.tiles_t, KB = op.k / 64;
        // split-K only for the fp32 residual producers (their finalisation runs in
        // the TMEM layout, tokens split evenly in 16-token halves per warp half)
        const bool splittable = epi == EPI_RESID_F32 || epi == EPI_F32;
        op.splits = splittable ? std::min(cap[kind], pick_splits(tiles, KB, ttn, G)) : 1;
        // the split finalisation stages its TN/S owned rows (fp32 + bf16 copy) in the
        // epilogue staging region and runs 4 threads per row: no split where that does not fit
        while (op.splits > 1) {
            const int orows = ttn / op.splits;
            if ((size_t)orows * (512 + 256) <= (size_t)tn * 256 && orows % 16 == 0 && orows <= 64) break;
            --op.splits;
            while (op.splits > 1 && ttn % op.splits) --op.splits;
        }
        op.kbs = (KB + op.splits - 1) / op.splits;
        op.n_items = tiles * op.splits;
        op.split_base = split_ctr;
        split_ctr += tiles;
        op.tmW = dm(mw);
        op.tmX = dm(act_map(xin, L.in, ttn));
        op.tmO = (out == c.ws.h1 || out == c.ws.qkv) ? dm(act_map(out, L.out, ttn)) : nullptr;
        op.tmXB = produce ? dm(act_map(c.ws.x, ah, ttn)) : nullptr;
        // progressive 16-row stores of the unsplit drain (ALPA_MK_PROG=0: one store per tile)
        const bool prog = !getenv("ALPA_MK_PROG") || getenv("ALPA_MK_PROG")[0] != '0';
        if (prog && (op.tmO || op.tmXB)) {
            // one store per 16-row chunk across both 64-feature panels (chunk-major staging)
            CUtensorMap tp{};
            if (op.tmO)
                make_tmap_panels(&tp, out, false, (uint64_t)L.out, (uint64_t)M, (uint64_t)L.out * 2, 16, 2);
            else
                make_tmap_panels(&tp, c.ws.x, false, (uint64_t)ah, (uint64_t)M, (uint64_t)ah * 2, 16, 2);
            op.tmO16 = dm(add_map(tp));
        }
        if (op.splits == 1 && (epi == EPI_RESID_F32 || epi == EPI_F32) && (size_t)ttn * (256 + 512) <= (size_t)tn * 256) {
            // unsplit fp32 producer whose fp32 tile fits the staging next to the bf16 tile:
            // TMA-stored through four SW128 panels of 32 fp32 (box {32, TN, 1})
            CUtensorMap te{};
            make_tmap_f32_3d_sw128(&te, out, (uint64_t)L.out, (uint64_t)M, 1, (uint64_t)ldo * 4,
                                   (uint64_t)ldo * 4 * M, (uint32_t)ttn);
            op.tmEs = dm(add_map(te));
            // progressive: one store per 16-row chunk across the four 32-fp32 panels
            make_tmap_panels(&te, out, true, (uint64_t)L.out, (uint64_t)M, (uint64_t)ldo * 4, 16, 4);
            op.tmE16 = dm(add_map(te));
        }
        if (op.splits > 1) {
            // split finalisation: TN/S owned rows, fp32 e + bf16 copy via TMA stores
            const int orows = ttn / op.splits;
            CUtensorMap te{};
            make_tmap_f32_2d(&te, out, (uint64_t)L.out, (uint64_t)M, (uint64_t)ldo * 4, 128, (uint32_t)orows);
            op.tmEs = dm(add_map(te));
            if (produce) op.tmXs = dm(act_map(c.ws.x, ah, orows));
        }
        op.bias = L.b;
        op.colsum = consume ? L.colsum : nullptr;
        op.out = out;
        op.ldo = ldo;
        if (produce) {
            op.stats_out = c.ws.stats;
            op.xb_out = (__nv_bfloat16*)c.ws.x;
        }
        if (consume) op.stats_in = stats;
        // L2 prefetch of a later op's bytes, per op kind (bit = kind, ALPA_MK_PF)
        op.pf_ptr = pf;
        op.pf_bytes = (pf_mask >> pf_kind) & 1 ? pfb : 0;
        // split partials: [tile][split][TN rows][128 features] fp32 blocks
        if (op.splits > 1) ws_floats = std::max(ws_floats, (size_t)tiles * op.splits * ttn * 128);
        push(op, tag, 2.0 * M * L.in * L.out);
    };
    const int64_t pcap = c.pcap();  // rows per K / V section of the prefix
    const int64_t pre_block = 2 * pcap * kv * 2;
    // mixed per-lane prefixes (multi topology): one query tile per lane, prefix
    // rows from the device lane map at run time
    const bool multi = c.uniform_prefix < 0;
    const int64_t upre = multi ? 0 : c.uniform_prefix;
    auto prefix_of = [&](int64_t b) {
        return (const void*)((const uint8_t*)c.prefix + (upre * B + b) * pre_block);
    };

    {
        Op op{};
        op.kind = mk::OP_ENCODE;
        op.tn = (int)std::max<int64_t>(1, (M + G - 1) / G);  // rows per item: spread over every SM
        op.n_items = (int)((M + op.tn - 1) / op.tn);
        push(op, "encode", 4.0 * M * ah);
    }
    gemm(c.mlp1, menc1, c.ws.x, EPI_GELU_BF16, c.ws.h1, 4 * ah, false, false, c.mlp2.w, wb(c.mlp2),
         "gemm_enc_mlp1", 4);
    gemm(c.mlp2, menc2, c.ws.h1, EPI_F32, c.ws.e, ah, true, false, c.blocks[0].qkv.w, wb(c.blocks[0].qkv),
         "gemm_enc_mlp2", 5);
    std::vector<std::pair<int, int>> attn_part_maps;  // (map index, splits)
    const int qtiles = multi ? (int)n : (int)((M + 127) / 128);
    const int prows = multi ? (int)n * 128 : (int)M;  // KV-split partial rows per split
    const int nbp = (int)((r + 63) / 64);
    for (int64_t b = 0; b < B; ++b) {
        const Block& blk = c.blocks[b];
        gemm(blk.qkv, mblk[b * 4 + 0], c.ws.x, EPI_LN_BF16, c.ws.qkv, 3 * kv, false, true, prefix_of(b),
             pre_block, "gemm_qkv", 0);
        {
            Op op{};
            op.kind = mk::OP_ATTN;
            op.tiles_f = (int)H;
            op.tiles_t = qtiles;
            const int tiles = (int)H * qtiles;
            const int nbt_min = nbp + 1;
            op.multi = multi ? 1 : 0;
            op.blk = (int)b;
            op.prows = prows;
            int smax = 6;  // attn_fixup merges at most 6 partials
            if (const char* e = getenv("ALPA_MK_ATTN_S")) smax = std::max(1, std::min(6, atoi(e)));
            op.splits = tiles >= G ? 1 : std::max(1, std::min({G / tiles, nbt_min, smax}));
            op.n_items = tiles * op.splits;
            op.split_base = split_ctr;
            split_ctr += tiles;
            op.nbp = nbp;
            op.tmW = dm(mpre);
            op.tmX = dm(mq64);
            op.tmQ = dm(mq128);
            op.out = c.ws.ctxb;
            const int64_t blkrow = (upre * B + b) * 2;
            op.pre_k_row = blkrow * pcap;
            op.pre_v_row = (blkrow + 1) * pcap;
            op.pf_ptr = blk.o.w;
            op.pf_bytes = (pf_mask >> 6) & 1 ? wb(blk.o) : 0;
            if (op.splits > 1) {
                // partial staging reuses the Q/P smem: one item per CTA (a next item's Q
                // load could otherwise land on it)
                if (op.n_items > G) fail(ALPA_ERR_INTERNAL, "persistent kernel: attention split plan exceeds one wave");
                const int mp = add_map(CUtensorMap{});  // encoded once the workspace exists
                attn_part_maps.push_back({mp, op.splits});
                op.tmXs = dm(mp);
            }
            ws_floats = std::max(ws_floats, (size_t)op.splits * prows * kv);
            wsml_elems = std::max(wsml_elems, (size_t)op.splits * prows * H);
            push(op, "attention", 4.0 * n * A * (r + A) * kv);
        }
        gemm(blk.o, mblk[b * 4 + 1], c.ws.ctxb, EPI_RESID_F32, c.ws.e, ah, true, false, blk.mlp1.w,
             wb(blk.mlp1), "gemm_o", 1);
        gemm(blk.mlp1, mblk[b * 4 + 2], c.ws.x, EPI_LN_GELU_BF16, c.ws.h1, 4 * ah, false, true, blk.mlp2.w,
             wb(blk.mlp2), "gemm_mlp1", 2);
        const bool last = b + 1 == B;
        // bit 7: MLP2 pulls the NEXT block's prefix K/V instead of its QKV weights
        const bool pf_pre = (pf_mask >> 7) & 1;
        gemm(blk.mlp2, mblk[b * 4 + 3], c.ws.h1, EPI_RESID_F32, c.ws.e, ah, true, false,
             last ? nullptr : (pf_pre ? prefix_of(b + 1) : c.blocks[b + 1].qkv.w),
             last ? 0 : (pf_pre ? pre_block : wb(c.blocks[b + 1].qkv)), "gemm_mlp2", pf_pre ? 7 : 3);
    }
    {
        Op op{};
        op.kind = mk::OP_HEAD;
        op.n_items = (int)((M + 7) / 8);
        push(op, "head_update", 4.0 * M * ah + 8.0 * M);
    }

    m.ws = (float*)c.dalloc(ws_floats * sizeof(float));
    m.wsml = (float2*)c.dalloc(wsml_elems * sizeof(float2));
    for (auto& pm : attn_part_maps)
        make_tmap_f32_3d_sw128(&maps[pm.first], m.ws, (uint64_t)kv, (uint64_t)prows, (uint64_t)pm.second,
                               (uint64_t)kv * 4, (uint64_t)prows * kv * 4, 128);
    m.d_maps = (CUtensorMap*)c.dalloc(maps.size() * sizeof(CUtensorMap));
    ALPA_CUDA(cudaMemcpy(m.d_maps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    auto fix = [&](const CUtensorMap*& t) {
        if (t) t = m.d_maps + ((uintptr_t)t - 1);
    };
    for (Op& op : ops) {
        fix(op.tmW);
        fix(op.tmX);
        fix(op.tmQ);
        fix(op.tmO);
        fix(op.tmXB);
        fix(op.tmEs);
        fix(op.tmXs);
        fix(op.tmO16);
        fix(op.tmE16);
    }
    m.n_ops = (int)ops.size();
    m.d_ops = (Op*)c.dalloc(ops.size() * sizeof(Op));
    ALPA_CUDA(cudaMemcpy(m.d_ops, ops.data(), ops.size() * sizeof(Op), cudaMemcpyHostToDevice));
    m.counter_ints = (size_t)m.n_ops + split_ctr;
    m.d_counters = (int*)c.dalloc(m.counter_ints * sizeof(int));
    if (getenv("ALPA_MK_DEBUG")) {  // plan dump (watchdog messages name counter addresses)
        std::printf("mk plan: counters at %p (done[0..%d], split counters after)\n", (void*)m.d_counters,
                    (int)ops.size());
        for (size_t o = 0; o < ops.size(); ++o)
            std::printf("  op %zu %s kind %d items %d splits %d tn %d dep %d/%d\n", o, tags[o], ops[o].kind,
                        ops[o].n_items, ops[o].splits, ops[o].tn, ops[o].dep, ops[o].dep_count);
    }
    ALPA_CUDA(cudaMemset(m.d_counters, 0, m.counter_ints * sizeof(int)));
    m.d_tstamp = (unsigned long long*)c.dalloc((m.n_ops + 1) * sizeof(unsigned long long));
    if (const char* e = getenv("ALPA_MK_TRACE"); e && e[0] == '1') {
        m.trace_elems = (size_t)m.n_ops * G * mk::TR_NSLOT;
        m.d_trace = (unsigned long long*)c.dalloc(m.trace_elems * sizeof(unsigned long long));
    }
    m.tags = tags;
    m.flops = flops;
    m.fn = ks.fn;
    m.fn_tr = ks.fn_tr;
    m.smem = ks.smem;
    m.grid = G;
    ALPA_CUDA(cudaFuncSetAttribute(ks.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ks.smem));
    ALPA_CUDA(cudaFuncSetAttribute(ks.fn_tr, cudaFuncAttributeMaxDynamicSharedMemorySize, ks.smem));
    int occ = 0;
    ALPA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.fn, mk::Cfg<64, 64>::THREADS, ks.smem));
    if (occ < 1) fail(ALPA_ERR_INTERNAL, "persistent kernel does not fit on an SM");
    m.n = n;
    m.prefix = c.prefix;
    m.uniform = c.uniform_prefix;
    m.r = r;
    m.cap = c.pcap();
    m.prefix_n = c.prefix_n;
    m.valid = true;
}

void mk_enqueue(Ctx& c, int64_t n, cudaStream_t s, unsigned long long* tstamp,
                unsigned long long* trace) {
    MkState& m = c.mk;
    if (!m.valid || m.n != n) fail(ALPA_ERR_INTERNAL, "persistent kernel plan not prepared");
    mk::Params p{};
    p.ops = (const Op*)m.d_ops;
    p.n_ops = m.n_ops;
    p.done = m.d_counters;
    p.splitc = m.d_counters + m.n_ops;
    p.ws = m.ws;
    p.wsml = m.wsml;
    p.M = (int)(n * c.steps());
    p.ah = (int)c.ah();
    p.kv = (int)c.kv();
    p.H = (int)c.cfg.heads;
    p.r = (int)c.prefix_r;
    p.rcap = (int)c.pcap();
    p.nft = (int)(c.ah() / 128);
    p.B = (int)c.cfg.decoder_blocks;
    p.lane_map = c.ws.lane_map;
    p.alpha = 1.0f / sqrtf((float)(c.kv() / c.cfg.heads));
    p.update_scale = c.cfg.update_scale;
    p.actions = c.ws.actions;
    p.w_in = (const float*)c.act_in.w;
    p.b_in = c.act_in.b;
    p.pos = c.pos;
    p.w_head = (const float*)c.head.w;
    p.b_head = c.head.b;
    p.e = c.ws.e;
    p.x = (__nv_bfloat16*)c.ws.x;
    p.tstamp = tstamp;
    p.trace = trace;
    if (const char* e = getenv("ALPA_MK_FLAGS")) p.flags = atoi(e);
    ALPA_CUDA(cudaMemsetAsync(m.d_counters, 0, m.counter_ints * sizeof(int), s));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)m.grid);
    cfg.blockDim = dim3(mk::Cfg<64, 64>::THREADS);
    cfg.dynamicSmemBytes = (size_t)m.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&p};
    ALPA_CUDA(cudaLaunchKernelExC(&cfg, (tstamp || trace) ? m.fn_tr : m.fn, args));
    c.last_launches++;
}

}  // namespace alpa
