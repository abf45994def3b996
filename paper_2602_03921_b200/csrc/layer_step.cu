// layer_step.cu -- the physical expert-cached MoE layer step (configs[1]).
//
// Decision and execution are split exactly as SURVEY.md section 7.1 asks:
//  * decisions: the replay kernel (replay.cu) runs the reference's logical
//    timeline for the request and streams its event records into mapped
//    host memory, publishing a per-layer progress counter;
//  * execution: this native runtime consumes each layer's records as soon
//    as they are published and drives the hardware:
//      EvictRec              -> the victim's HBM slot returns to the free list
//      PrefetchRec started   -> H2D copy pinned store -> a free slot, on the
//      AccessRec fetch          copy-engine stream, in decision order
//      PrefetchRec dropped   -> (cancelled in flight) slot returns; the DMA
//        superseded             already issued still completes (FIFO-safe)
//      AccessRec hit/wait    -> the expert executes from its slot
//      AccessRec subst       -> the substitute's slot runs the dropped
//                               expert's tokens
//      RouteRec              -> the layer's grouped FFN (ffn_gemm.cu) on
//                               the compute stream, then x += y
//    Hazards: landed[slot] (copy -> FFN, RAW) and freed[slot] (last FFN
//    reading the slot -> next copy into it, WAR) CUDA events. If a decision
//    evicts an expert the current layer has not executed yet (tiny caches),
//    the pending experts are flushed as a partial FFN first.
// The host never blocks on the GPU except to wait for decisions; copies
// stay back-to-back on the link, overlapped with compute.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/specmd_b200.h"

extern "C" int esim_tmap_bf16(void* out_map, const void* base, int64_t rows, int64_t cols, int32_t box_rows);
extern "C" int esim_ffn_gather(const void* d_x, const int32_t* d_tok_index, void* d_xg, int32_t n_exec, int32_t npad,
                               int32_t H, void* stream);
extern "C" int esim_ffn_residual(void* d_x, float* d_y, int64_t n, void* stream);
extern "C" int esim_ffn_experts_ex(const void* d_w1_maps, const void* d_w2_maps, const void* d_x_map,
                                   const void* d_act_map, const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                   const float* d_tok_weight, void* d_act, float* d_y, int32_t n_exec, int32_t npad,
                                   int32_t I, int32_t H, int32_t max_tok, void* stream);
extern "C" int esim_ffn_experts_gemv(const void* d_slots, int64_t slot_bytes, int32_t bits, const void* d_x,
                                     const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                     const float* d_tok_weight, float* d_y, int32_t n_exec, int32_t npad,
                                     int32_t max_tok, int32_t I, int32_t H, void* stream);
extern "C" int esim_ffn_experts_q(const void* d_slots, int64_t slot_bytes, int32_t bits, const void* d_x_map,
                                  const int32_t* d_exec_slot, const int32_t* d_tok_index, const float* d_tok_weight,
                                  float* d_y, int32_t n_exec, int32_t I, int32_t H, void* stream);
extern "C" int esim_ffn_experts(const void* d_w1_maps, const void* d_w2_maps, const void* d_x_map,
                                const void* d_act_map, const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                const float* d_tok_weight, void* d_act, float* d_y, int32_t n_exec, int32_t npad,
                                int32_t I, int32_t H, void* stream);
extern "C" int esim_router_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode,
                                  double overfetch, double percentile, void* stream);
extern "C" int esim_noise_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode, double noise,
                                 uint64_t seed, void* stream);
int esim_replay_launch_streamed(const EsimConfig* h_cfg, const EsimConfig* d_cfg, const EsimTraceDesc* d_traces,
                                const EsimRouterOut* d_routers, int32_t max_tokens, EsimCounters* d_counters,
                                int64_t* d_per_layer, int32_t pl_stride, EsimRec* d_recs, int64_t rec_cap,
                                int32_t* d_pexp, int64_t pe_cap, int64_t* progress, void* stream);

namespace {

constexpr int NPADS[4] = {16, 32, 64, 128};

__global__ void build_tables_kernel(const int16_t* __restrict__ row_sel, const float* __restrict__ row_w, int T,
                                    int K, const int32_t* __restrict__ pos_of_expert, int n_exec, int npad,
                                    int32_t* __restrict__ tok_index, float* __restrict__ tok_weight) {
    extern __shared__ int fill[];
    for (int i = threadIdx.x; i < n_exec * npad; i += blockDim.x) { tok_index[i] = -1; tok_weight[i] = 0.0f; }
    for (int i = threadIdx.x; i < n_exec; i += blockDim.x) fill[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < T * K; i += blockDim.x) {
        const int pos = pos_of_expert[row_sel[i]];
        if (pos < 0) continue;
        const int f = atomicAdd(&fill[pos], 1);        // the expert's f-th token -> entry pos + f / npad
        const int e = pos + f / npad, c = f % npad;     // (npad == 128 whenever an expert is split)
        if (e < n_exec) {
            tok_index[e * npad + c] = i / K;
            tok_weight[e * npad + c] = row_w[i];
        }
    }
}

// quantised expert (tile-major like the bf16 one, ffn.py; int8 codes, or
// int4 / int2 codes word-interleaved in 32-bit words (layer_step.py
// code_positions), two's complement; then fp32 scales: 2I gate/up rows, H down rows) -> bf16
// tile-major scratch entry: w = bf16(q * s_row). A thread converts 16
// consecutive codes of one row. pairs[2e] = source slot, pairs[2e+1] =
// scratch entry. grid: (chunks, n_entries of this precision)
template <int BITS>
__global__ void dequant_kernel(const uint8_t* __restrict__ slots, int64_t slot_bytes,
                               const int32_t* __restrict__ pairs, __nv_bfloat16* __restrict__ scratch, int I,
                               int H) {
    const uint8_t* src = slots + (int64_t)pairs[2 * blockIdx.y] * slot_bytes;
    const int64_t n1 = 2LL * I * H, n = 3LL * I * H;
    const float* s1 = reinterpret_cast<const float*>(src + n * BITS / 8);   // [2I]
    const float* s2 = s1 + 2 * I;                                          // [H]
    __nv_bfloat16* dst = scratch + (int64_t)pairs[2 * blockIdx.y + 1] * n;
    const int HT = H / 128;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n / 16; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = v * 16;
        float sc;
        if (j < n1) {                                   // w1 tile (m, k): [64 gate; 64 up] rows x 64
            const int64_t t = j / 8192;
            const int r = (int)((j % 8192) / 64);
            const int m = (int)(t / (H / 64));
            sc = r < 64 ? s1[m * 64 + r] : s1[I + m * 64 + (r - 64)];
        } else {                                        // w2 tile (m, ht): 128 down rows x 64
            const int64_t jj = j - n1;
            const int64_t t = jj / 8192;
            const int r = (int)((jj % 8192) / 64);
            sc = s2[(int)(t % HT) * 128 + r];
        }
        int8_t qb[16];
        if (BITS == 8) {
            const int4 q = reinterpret_cast<const int4*>(src)[v];
            const int8_t* b = reinterpret_cast<const int8_t*>(&q);
#pragma unroll
            for (int i = 0; i < 16; i++) qb[i] = b[i];
        } else {
            // word-interleaved codes (layer_step.py code_positions): element 2j at
            // position j, element 2j+1 at position PER/2 + j of its 32-bit word
            constexpr int PER = 32 / BITS;
            uint32_t w[2];
            if (BITS == 2) {
                w[0] = reinterpret_cast<const uint32_t*>(src)[v];
            } else {
                const uint2 q = reinterpret_cast<const uint2*>(src)[v];
                w[0] = q.x; w[1] = q.y;
            }
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const int wi = i / PER, k = i % PER, pos = (k & 1) ? PER / 2 + k / 2 : k / 2;
                qb[i] = (int8_t)((int)(w[wi] << (32 - BITS * (pos + 1))) >> (32 - BITS));   // sign-extended
            }
        }
        __align__(16) __nv_bfloat16 out[16];
#pragma unroll
        for (int i = 0; i < 16; i++) out[i] = __float2bfloat16((float)qb[i] * sc);
        reinterpret_cast<uint4*>(dst + j)[0] = reinterpret_cast<const uint4*>(out)[0];
        reinterpret_cast<uint4*>(dst + j)[1] = reinterpret_cast<const uint4*>(out)[1];
    }
}

// rows of bf16 between device and mapped host memory (zero-copy over the link)
__global__ void copy_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// shared expert of one layer (HF Qwen2MoeSparseMoeBlock): every token, weight
// sigmoid(x . gate). One warp per table row: entry j = row / npad, column
// c = row % npad, token t = j * npad + c (npad == 128 whenever T > 128).
__global__ void shared_tables_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ gate,
                                     int T, int H, int npad, int n_ent, int layer, int32_t* __restrict__ tok_index,
                                     float* __restrict__ tok_weight, int32_t* __restrict__ exec) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (r >= n_ent * npad) return;
    const int t = r;                                  // entries are consecutive npad-token chunks
    if (r % npad == 0 && lane == 0) exec[r / npad] = layer;
    if (t >= T) {
        if (lane == 0) { tok_index[r] = -1; tok_weight[r] = 0.0f; }
        return;
    }
    float acc = 0.0f;
    const __nv_bfloat162* xr = reinterpret_cast<const __nv_bfloat162*>(x + (size_t)t * H);
    const __nv_bfloat162* gr = reinterpret_cast<const __nv_bfloat162*>(gate);
    for (int i = lane; i < H / 2; i += 32) {
        const float2 a = __bfloat1622float2(xr[i]), b = __bfloat1622float2(gr[i]);
        acc = fmaf(a.x, b.x, fmaf(a.y, b.y, acc));
    }
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        tok_index[r] = t;
        tok_weight[r] = 1.0f / (1.0f + expf(-acc));
    }
}

struct Engine {
    EsimLSParams P;
    size_t expert_bytes = 0;             // working precision
    int mask = 0;                        // precisions in the store
    size_t fmt_bytes[4] = {};            // per expert, by precision code (0: absent)
    size_t store_off[4] = {};            // region offsets in the store
    size_t store_bytes = 0, slot_bytes = 0;
    int n_slot_maps = 0;                 // FFN maps over the slots (bf16 present), then scratch maps
    void* store = nullptr;               // pinned host: per precision [L][E][expert]
    char* slots = nullptr;               // device: [n_slots][slot_bytes]
    void *w1_maps = nullptr, *w2_maps = nullptr;
    void *xg = nullptr, *act = nullptr;
    void *x_maps[4] = {}, *act_maps[4] = {};
    float* y = nullptr;
    void* x = nullptr;
    int32_t* tok_index = nullptr;
    float* tok_weight = nullptr;
    cudaStream_t copy_st = nullptr, comp_st = nullptr, ctl_st = nullptr;
    std::vector<cudaEvent_t> landed, freed;
    cudaEvent_t ev_start = nullptr, ev_ttft = nullptr, ev_end = nullptr, ev_copy_end = nullptr;
    // mapped host (zero-copy) buffers
    EsimRec* recs = nullptr;
    int64_t rec_cap = 0;
    int32_t* pexp = nullptr;
    int64_t pe_cap = 0;
    int64_t* progress = nullptr;
    int32_t* tables = nullptr;           // pool of [2][E] int32 (pos_of_expert, exec_slot) per flush
    int64_t table_cap = 0;
    int max_entries = 0;                 // FFN entries per flush: experts + token-count splits at 128
    char* scratch = nullptr;             // quantised: [max_entries][3*H*I] bf16 tile-major
    bool fused_dequant = true;           // decode flushes over one quantised precision: ffn_decode_q_kernel
    bool decode_gemv = true;             // decode flushes over one precision: ffn_gemv_kernel (ESIM_FFN_DECODE=tc: off)
    // per-run device scratch
    void* dev_scratch = nullptr;
    size_t dev_scratch_bytes = 0;
    // always-resident shared expert (Qwen1.5-MoE: 2048 x 5632 per layer), attached by the caller
    int Is = 0;                          // its intermediate width (0: none)
    const void* shared_w = nullptr;      // device [L][3*H*Is] bf16 tile-major (caller-owned)
    const __nv_bfloat16* shared_gate = nullptr;   // device [L][H] bf16
    void *sw1_maps = nullptr, *sw2_maps = nullptr, *sact = nullptr;
    void* sact_maps[4] = {};
    int32_t* s_tok_index = nullptr;      // device tables of the shared entries
    float* s_tok_weight = nullptr;
    int32_t* s_exec = nullptr;
    int s_entries = 0;                   // ceil(max_tokens / 128)
    void* capture = nullptr;             // optional mapped host [sum over events of T][H] bf16: every layer's output
    int64_t capture_rows = 0;
    const int16_t* last_sel = nullptr;   // the last request's executed routing (in dev_scratch)
    const float* last_w = nullptr;
    int64_t last_rows = 0;
};

std::string g_ls_err;
int ls_fail(int code, const std::string& m) { g_ls_err = m; return code; }
int ls_cuda(cudaError_t e, const char* where) { return ls_fail(-3, std::string(where) + ": " + cudaGetErrorString(e)); }

#define CK(x)                                              \
    do {                                                   \
        cudaError_t _e = (x);                              \
        if (_e != cudaSuccess) return ls_cuda(_e, #x);     \
    } while (0)

int npad_for(int t) {
    for (int n : NPADS) if (t <= n) return n;
    return -1;
}
int npad_index(int n) {
    for (int i = 0; i < 4; i++) if (NPADS[i] == n) return i;
    return -1;
}

}  // namespace

extern "C" const char* esim_ls_last_error(void) { return g_ls_err.c_str(); }

extern "C" int esim_ls_create(const EsimLSParams* p, void** handle) {
    Engine* g = new Engine();
    g->P = *p;
    const int L = p->num_layers, E = p->experts, H = p->hidden, I = p->inter;
    if (H % 128 || I % 128 || p->max_tokens < 1 || p->max_tokens > 16384 || p->n_slots < 1) {
        delete g;
        return ls_fail(-1, "bad layer-step geometry");
    }
    // an expert with more than 128 tokens in a pass runs as several FFN entries of <= 128
    g->max_entries = E + (int)(((int64_t)p->max_tokens * p->top_k + 127) / 128);
    if (p->weight_format < 0 || p->weight_format > 3 || (p->prec_mask & ~0xF) ||
        (p->prec_mask && !(p->prec_mask >> p->weight_format & 1))) {
        delete g;
        return ls_fail(-1, "unknown weight format / precision mask");
    }
    g->mask = p->prec_mask ? p->prec_mask : 1 << p->weight_format;
    if (const char* v = getenv("ESIM_LS_SCRATCH_DEQUANT")) g->fused_dequant = v[0] != '1';   // A/B switch
    if (const char* v = getenv("ESIM_FFN_DECODE")) g->decode_gemv = !(v[0] == 't' && v[1] == 'c');
    const size_t bf16_bytes = (size_t)3 * H * I * 2;
    for (int pc = 0; pc < 4; pc++) {
        if (!(g->mask >> pc & 1)) continue;
        const int bits = 16 >> pc;                                    // 16, 8, 4, 2
        g->fmt_bytes[pc] = pc == 0 ? bf16_bytes : (size_t)3 * H * I * bits / 8 + (size_t)4 * (2 * I + H);
        g->store_off[pc] = g->store_bytes;
        g->store_bytes += g->fmt_bytes[pc] * L * E;
        g->slot_bytes = std::max(g->slot_bytes, (g->fmt_bytes[pc] + 255) & ~size_t(255));
    }
    g->expert_bytes = g->fmt_bytes[p->weight_format];
    CK(cudaHostAlloc(&g->store, g->store_bytes, cudaHostAllocDefault));
    CK(cudaMalloc((void**)&g->slots, g->slot_bytes * p->n_slots));
    // the FFN reads bf16 tile-major experts: the slots themselves (bf16) and/or
    // the per-entry scratch pool quantised slots are dequantised into
    g->n_slot_maps = (g->mask & 1) ? p->n_slots : 0;
    const int n_maps = g->n_slot_maps + ((g->mask & 0xE) ? g->max_entries : 0);
    if (g->mask & 0xE) {
        CK(cudaMalloc((void**)&g->scratch, bf16_bytes * g->max_entries));
    }
    std::vector<unsigned char> m1(128 * (size_t)n_maps), m2(128 * (size_t)n_maps);
    for (int s = 0; s < n_maps; s++) {
        const char* base = s < g->n_slot_maps ? g->slots + g->slot_bytes * s
                                               : g->scratch + bf16_bytes * (s - g->n_slot_maps);
        // tile-major expert layout (ffn.py): every TMA box is one contiguous run
        if (esim_tmap_bf16(&m1[128 * s], base, (int64_t)2 * I * H / 64, 64, 128) ||
            esim_tmap_bf16(&m2[128 * s], base + (size_t)2 * I * H * 2, (int64_t)I * H / 64, 64, 128))
            return ls_fail(-3, "tensor map encode failed");
    }
    CK(cudaMalloc(&g->w1_maps, m1.size()));
    CK(cudaMalloc(&g->w2_maps, m2.size()));
    CK(cudaMemcpy(g->w1_maps, m1.data(), m1.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(g->w2_maps, m2.data(), m2.size(), cudaMemcpyHostToDevice));
    const size_t maxrows = (size_t)g->max_entries * 128;
    CK(cudaMalloc(&g->xg, maxrows * H * 2));
    CK(cudaMalloc(&g->act, maxrows * I * 2));
    for (int i = 0; i < 4; i++) {
        unsigned char mx[128], ma[128];
        if (esim_tmap_bf16(mx, g->xg, (int64_t)g->max_entries * NPADS[i], H, NPADS[i]) ||
            esim_tmap_bf16(ma, g->act, (int64_t)g->max_entries * NPADS[i], I, NPADS[i]))
            return ls_fail(-3, "tensor map encode failed");
        CK(cudaMalloc(&g->x_maps[i], 128));
        CK(cudaMalloc(&g->act_maps[i], 128));
        CK(cudaMemcpy(g->x_maps[i], mx, 128, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(g->act_maps[i], ma, 128, cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc((void**)&g->y, (size_t)p->max_tokens * H * 4));
    CK(cudaMemset(g->y, 0, (size_t)p->max_tokens * H * 4));
    CK(cudaMalloc(&g->x, (size_t)p->max_tokens * H * 2));
    CK(cudaMalloc((void**)&g->tok_index, maxrows * 4));
    CK(cudaMalloc((void**)&g->tok_weight, maxrows * 4));
    CK(cudaStreamCreateWithFlags(&g->copy_st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g->comp_st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g->ctl_st, cudaStreamNonBlocking));
    g->landed.resize(p->n_slots);
    g->freed.resize(p->n_slots);
    for (int s = 0; s < p->n_slots; s++) {
        CK(cudaEventCreateWithFlags(&g->landed[s], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g->freed[s], cudaEventDisableTiming));
    }
    CK(cudaEventCreate(&g->ev_start));
    CK(cudaEventCreate(&g->ev_ttft));
    CK(cudaEventCreate(&g->ev_end));
    CK(cudaEventCreate(&g->ev_copy_end));
    *handle = g;
    return 0;
}

extern "C" void* esim_ls_store(void* handle) { return static_cast<Engine*>(handle)->store; }
extern "C" int64_t esim_ls_expert_bytes(void* handle) { return (int64_t) static_cast<Engine*>(handle)->expert_bytes; }
extern "C" int64_t esim_ls_format(void* handle, int32_t prec, int64_t* store_offset) {
    const Engine* g = static_cast<Engine*>(handle);
    if (prec < 0 || prec > 3 || !g->fmt_bytes[prec]) return 0;
    if (store_offset) *store_offset = (int64_t)g->store_off[prec];
    return (int64_t)g->fmt_bytes[prec];
}
// the last request's executed routing, [rows][K] (the router's top-k, or the
// cache-aware selection and its original-softmax weights for routing=cache_aware)
extern "C" int esim_ls_route_rows(void* handle, int16_t* sel_out, float* w_out, int64_t rows) {
    const Engine* g = static_cast<Engine*>(handle);
    if (!g->last_sel || rows > g->last_rows) return ls_fail(-1, "no such rows in the last request");
    const size_t n = (size_t)rows * g->P.top_k;
    if (cudaMemcpy(sel_out, g->last_sel, n * 2, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(w_out, g->last_w, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return ls_fail(-3, "route rows copy failed");
    return 0;
}
extern "C" int64_t esim_ls_store_bytes(void* handle) { return (int64_t) static_cast<Engine*>(handle)->store_bytes; }
extern "C" void* esim_ls_slots(void* handle) { return static_cast<Engine*>(handle)->slots; }

// Attach the always-resident shared expert (d_w: [L][3*H*inter] bf16 tile-major
// like a routed expert, d_gate: [L][H] bf16; both caller-owned device memory):
// every layer then adds sigmoid(x . gate_l) * shared_l(x) to the routed experts'
// output before the residual. inter = 0 detaches.
extern "C" int esim_ls_shared_expert(void* handle, const void* d_w, const void* d_gate, int32_t inter) {
    Engine* g = static_cast<Engine*>(handle);
    const int L = g->P.num_layers, H = g->P.hidden;
    cudaDeviceSynchronize();
    cudaFree(g->sw1_maps); cudaFree(g->sw2_maps); cudaFree(g->sact);
    for (int i = 0; i < 4; i++) { cudaFree(g->sact_maps[i]); g->sact_maps[i] = nullptr; }
    cudaFree(g->s_tok_index); cudaFree(g->s_tok_weight); cudaFree(g->s_exec);
    g->sw1_maps = g->sw2_maps = g->sact = nullptr;
    g->s_tok_index = nullptr; g->s_tok_weight = nullptr; g->s_exec = nullptr;
    g->Is = 0;
    if (inter == 0) return 0;
    if (inter < 0 || inter % 128 || !d_w || !d_gate) return ls_fail(-1, "bad shared expert");
    const int Is = inter;
    g->s_entries = (g->P.max_tokens + 127) / 128;
    if (g->s_entries > g->max_entries) return ls_fail(-1, "shared expert entries exceed the staging buffers");
    std::vector<unsigned char> m1(128 * (size_t)L), m2(128 * (size_t)L);
    for (int l = 0; l < L; l++) {
        const char* base = (const char*)d_w + (size_t)l * 3 * H * Is * 2;
        if (esim_tmap_bf16(&m1[128 * l], base, (int64_t)2 * Is * H / 64, 64, 128) ||
            esim_tmap_bf16(&m2[128 * l], base + (size_t)2 * Is * H * 2, (int64_t)Is * H / 64, 64, 128))
            return ls_fail(-3, "tensor map encode failed");
    }
    CK(cudaMalloc(&g->sw1_maps, m1.size()));
    CK(cudaMalloc(&g->sw2_maps, m2.size()));
    CK(cudaMemcpy(g->sw1_maps, m1.data(), m1.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(g->sw2_maps, m2.data(), m2.size(), cudaMemcpyHostToDevice));
    const size_t rows = (size_t)g->s_entries * 128;
    CK(cudaMalloc(&g->sact, rows * Is * 2));
    for (int i = 0; i < 4; i++) {
        unsigned char ma[128];
        if (esim_tmap_bf16(ma, g->sact, (int64_t)g->s_entries * NPADS[i], Is, NPADS[i]))
            return ls_fail(-3, "tensor map encode failed");
        CK(cudaMalloc(&g->sact_maps[i], 128));
        CK(cudaMemcpy(g->sact_maps[i], ma, 128, cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc((void**)&g->s_tok_index, rows * 4));
    CK(cudaMalloc((void**)&g->s_tok_weight, rows * 4));
    CK(cudaMalloc((void**)&g->s_exec, g->s_entries * 4));
    g->shared_w = d_w;
    g->shared_gate = (const __nv_bfloat16*)d_gate;
    g->Is = Is;
    return 0;
}

// Debug / parity hook: every layer's output hidden states (after the residual)
// of the following requests go to `host_buf` (page-locked or mapped host
// memory, [rows][H] bf16, events in order, T rows per event); NULL turns it off.
extern "C" int esim_ls_capture_layers(void* handle, void* host_buf, int64_t rows) {
    Engine* g = static_cast<Engine*>(handle);
    g->capture = host_buf;
    g->capture_rows = host_buf ? rows : 0;
    return 0;
}

extern "C" int esim_ls_destroy(void* handle) {
    Engine* g = static_cast<Engine*>(handle);
    if (!g) return 0;
    cudaDeviceSynchronize();
    cudaFreeHost(g->store);
    cudaFree(g->slots);
    if (g->scratch) cudaFree(g->scratch);
    cudaFree(g->w1_maps);
    cudaFree(g->w2_maps);
    cudaFree(g->xg);
    cudaFree(g->act);
    for (int i = 0; i < 4; i++) { cudaFree(g->x_maps[i]); cudaFree(g->act_maps[i]); }
    cudaFree(g->y);
    cudaFree(g->x);
    cudaFree(g->tok_index);
    cudaFree(g->tok_weight);
    if (g->recs) cudaFreeHost(g->recs);
    if (g->pexp) cudaFreeHost(g->pexp);
    if (g->progress) cudaFreeHost(g->progress);
    if (g->tables) cudaFreeHost(g->tables);
    if (g->dev_scratch) cudaFree(g->dev_scratch);
    esim_ls_shared_expert(g, nullptr, nullptr, 0);
    for (auto e : g->landed) cudaEventDestroy(e);
    for (auto e : g->freed) cudaEventDestroy(e);
    cudaEventDestroy(g->ev_start);
    cudaEventDestroy(g->ev_ttft);
    cudaEventDestroy(g->ev_end);
    cudaEventDestroy(g->ev_copy_end);
    cudaStreamDestroy(g->copy_st);
    cudaStreamDestroy(g->comp_st);
    cudaStreamDestroy(g->ctl_st);
    delete g;
    return 0;
}

// One request: the trace (device pointers in `trace`), the logical config
// (`cfg`, host), hidden-state inputs in pinned/mapped host memory:
// x_prefill [T0][H] bf16, x_decode [n_passes-1][H] bf16; outputs the last
// layer's hidden states of every pass to out (mapped host, [rows][H] bf16).
extern "C" int esim_ls_run(void* handle, const EsimTraceDesc* trace_dev, const int32_t* h_pass_tokens,
                           const EsimConfig* cfg, const void* x_prefill, const void* x_decode, void* out,
                           EsimCounters* counters_out, int64_t* per_layer_out, EsimLSResult* res) {
    Engine* g = static_cast<Engine*>(handle);
    const EsimLSParams& P = g->P;
    const int L = P.num_layers, E = P.experts, K = P.top_k, H = P.hidden, I = P.inter;
    const EsimTraceDesc& tr = *trace_dev;
    if (tr.num_layers != L || tr.experts != E || tr.top_k != K) return ls_fail(-1, "trace geometry mismatch");
    const int64_t n_events = tr.n_events;
    const int64_t wbytes = cfg->expert_bytes[cfg->working_prec];
    // every precision the decisions can fetch must be in the store; the slot
    // pool must hold the most residents the logical capacity allows
    int64_t min_bytes = wbytes;
    if (cfg->working_prec != P.weight_format || !g->fmt_bytes[cfg->working_prec])
        return ls_fail(-1, "working precision differs from the engine's weight format");
    if (cfg->miss == ESIM_MISS_FETCH_LOW || cfg->miss == ESIM_MISS_FETCH_PRIORITY) {
        for (int i = 0; i < cfg->n_precisions; i++) {
            const int pc = cfg->precisions[i];
            if (pc < 0 || pc > 3 || !g->fmt_bytes[pc])
                return ls_fail(-1, "mixed-precision miss policy: a ladder precision is missing from the store");
            min_bytes = std::min(min_bytes, cfg->expert_bytes[pc]);
        }
    }
    if (std::min<int64_t>(cfg->capacity_bytes / min_bytes, (int64_t)L * E) > P.n_slots)
        return ls_fail(-1, "more logical slots than physical slots");
    int max_t = 0;
    for (int p = 0; p < tr.n_passes; p++) max_t = std::max(max_t, h_pass_tokens[p]);
    if (max_t > P.max_tokens) return ls_fail(-1, "pass has more tokens than the engine was sized for");
    // ---- buffers: mapped record stream, progress, flush tables; device router/replay scratch
    const int64_t rec_cap = 64 + n_events * (6 + 12 * (int64_t)E) + tr.n_rows_total * K * 2;
    if (rec_cap > g->rec_cap) {
        if (g->recs) cudaFreeHost(g->recs);
        CK(cudaHostAlloc((void**)&g->recs, rec_cap * sizeof(EsimRec), cudaHostAllocMapped));
        g->rec_cap = rec_cap;
    }
    const int64_t pe_cap = n_events * E;
    if (pe_cap > g->pe_cap) {
        if (g->pexp) cudaFreeHost(g->pexp);
        CK(cudaHostAlloc((void**)&g->pexp, pe_cap * 4, cudaHostAllocMapped));
        g->pe_cap = pe_cap;
    }
    if (g->progress) cudaFreeHost(g->progress);
    CK(cudaHostAlloc((void**)&g->progress, (n_events + 2) * 8, cudaHostAllocMapped));
    volatile int64_t* prog = g->progress;
    for (int64_t i = 0; i < n_events + 2; i++) prog[i] = 0;
    const int64_t table_need = (n_events * 2 + 64) * (E + 3 * g->max_entries);
    if (table_need > g->table_cap) {
        if (g->tables) cudaFreeHost(g->tables);
        CK(cudaHostAlloc((void**)&g->tables, table_need * 4, cudaHostAllocMapped));
        g->table_cap = table_need;
    }
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const int64_t ne = n_events, nr = tr.n_rows_total;
    size_t need = al(ne * 4) * 3 + al(ne * E * 4) * 6 + al(ne * E * 8) + al(ne * 8) + al(nr * K * 2) + al(nr * K * 4) +
                  al(sizeof(EsimConfig)) + al(sizeof(EsimTraceDesc)) + al(sizeof(EsimRouterOut)) +
                  al(sizeof(EsimCounters)) + al(L * ESIM_PL_FIELDS * 8) + al(ne * 4) * 2 + al(L * 16) +
                  al(sizeof(EsimRouteSummary));
    if (need > g->dev_scratch_bytes) {
        if (g->dev_scratch) cudaFree(g->dev_scratch);
        CK(cudaMalloc(&g->dev_scratch, need));
        g->dev_scratch_bytes = need;
    }
    char* q = (char*)g->dev_scratch;
    auto take = [&](size_t b) { void* r = q; q += al(b); return r; };
    EsimRouterOut ro;
    ro.n_dem = (int32_t*)take(ne * 4); ro.n_pred = (int32_t*)take(ne * 4); ro.pred_clamped = (int32_t*)take(ne * 4);
    ro.dem_expert = (int32_t*)take(ne * E * 4); ro.dem_rank = (int32_t*)take(ne * E * 4);
    ro.dem_gate = (float*)take(ne * E * 4); ro.dem_tokens = (int32_t*)take(ne * E * 4);
    ro.pred_expert = (int32_t*)take(ne * E * 4); ro.pred_score = (float*)take(ne * E * 4);
    ro.dem_summed = (double*)take(ne * E * 8); ro.sel_mass = (double*)take(ne * 8);
    ro.row_sel = (int16_t*)take(nr * K * 2); ro.row_w = (float*)take(nr * K * 4);
    ro.route_mix = (uint32_t*)take(ne * 4); ro.pred_mix = (uint32_t*)take(ne * 4);
    ro.layer_pred = (int64_t*)take(L * 16); ro.summary = (EsimRouteSummary*)take(sizeof(EsimRouteSummary));
    g->last_sel = ro.row_sel;
    g->last_w = ro.row_w;
    g->last_rows = nr;
    EsimConfig* d_cfg = (EsimConfig*)take(sizeof(EsimConfig));
    EsimTraceDesc* d_tr = (EsimTraceDesc*)take(sizeof(EsimTraceDesc));
    EsimRouterOut* d_ro = (EsimRouterOut*)take(sizeof(EsimRouterOut));
    EsimCounters* d_cnt = (EsimCounters*)take(sizeof(EsimCounters));
    int64_t* d_pl = (int64_t*)take(L * ESIM_PL_FIELDS * 8);
    EsimConfig hc = *cfg;
    hc.flags |= ESIM_FLAG_FULL_LOG;
    hc.trace_id = 0;
    CK(cudaMemcpy(d_cfg, &hc, sizeof hc, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_tr, &tr, sizeof tr, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ro, &ro, sizeof ro, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());

    // ---- timed request --------------------------------------------------
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaEventRecord(g->ev_start, g->comp_st));
    CK(cudaStreamWaitEvent(g->copy_st, g->ev_start, 0));
    CK(cudaStreamWaitEvent(g->ctl_st, g->ev_start, 0));
    int rc = esim_router_launch(&tr, &ro, hc.prefetch, hc.overfetch, hc.percentile, g->ctl_st);
    if (rc) return ls_fail(rc, "router launch");
    if (hc.prefetch != ESIM_PF_NONE && hc.prefetch_noise > 0.0 &&      // prefetch.py:110-136 on the device
        (rc = esim_noise_launch(&tr, &ro, hc.prefetch, hc.prefetch_noise, hc.seed, g->ctl_st)))
        return ls_fail(rc, "prediction noise");
    rc = esim_replay_launch_streamed(&hc, d_cfg, d_tr, d_ro, max_t, d_cnt, d_pl, L, g->recs, rec_cap, g->pexp, pe_cap,
                                     g->progress, g->ctl_st);
    if (rc) return ls_fail(rc, "replay launch");

    std::vector<int> phys(L * E, -1);                // ident -> physical slot
    std::vector<int8_t> slot_prec(P.n_slots, -1);    // precision each slot holds
    std::vector<int> scratch_of(P.n_slots, -1);      // per flush: slot -> its dequantised scratch entry
    std::vector<int> free_slots;
    for (int s = P.n_slots - 1; s >= 0; s--) free_slots.push_back(s);
    std::vector<int> pend_slot;                      // pending executed slots of the current layer (positions)
    std::vector<int> pos_of_expert(E, -1);
    std::vector<char> slot_pending(P.n_slots, 0);
    std::vector<int> tok_of_pos;
    int64_t table_next = 0;
    int64_t n_copies = 0, n_demand = 0, n_prefetch = 0, n_cancel = 0, n_flush = 0, n_exec_total = 0, h2d = 0;
    int64_t row = 0;                                 // first token row of the current event
    int64_t rec_pos = 0;
    int64_t out_row = 0;
    int64_t cap_row = 0;
    auto issue_copy = [&](int ident, int prec) -> int {
        if (free_slots.empty()) return ls_fail(-2, "no free physical slot (decision stream inconsistent)");
        if (phys[ident] >= 0) return ls_fail(-2, "fetch of a resident expert (decision stream inconsistent)");
        if (prec < 0 || prec > 3 || !g->fmt_bytes[prec]) return ls_fail(-2, "fetch precision not in the store");
        const int s = free_slots.back();
        free_slots.pop_back();
        phys[ident] = s;
        slot_prec[s] = (int8_t)prec;
        const size_t nb = g->fmt_bytes[prec];
        CK(cudaStreamWaitEvent(g->copy_st, g->freed[s], 0));                       // WAR
        CK(cudaMemcpyAsync(g->slots + (size_t)s * g->slot_bytes, (char*)g->store + g->store_off[prec] + ident * nb,
                           nb, cudaMemcpyHostToDevice, g->copy_st));
        CK(cudaEventRecord(g->landed[s], g->copy_st));                              // RAW guard
        n_copies++;
        h2d += (int64_t)nb;
        return 0;
    };
    // the layer's shared expert (always resident): every token, weight sigmoid(x . gate)
    auto run_shared = [&](int layer, int T) -> int {
        const int npad = T > 128 ? 128 : npad_for(T);
        const int n_ent = (T + npad - 1) / npad;
        shared_tables_kernel<<<(n_ent * npad + 7) / 8, 256, 0, g->comp_st>>>(
            (const __nv_bfloat16*)g->x, g->shared_gate + (size_t)layer * H, T, H, npad, n_ent, layer, g->s_tok_index,
            g->s_tok_weight, g->s_exec);
        if (T <= 4 && g->decode_gemv) {              // decode: the GEMV straight from the layer's weights
            if (esim_ffn_experts_gemv(g->shared_w, (int64_t)3 * H * g->Is * 2, 16, g->x, g->s_exec, g->s_tok_index,
                                      g->s_tok_weight, g->y, n_ent, npad, T, g->Is, H, g->comp_st))
                return ls_fail(-3, "shared expert gemv launch failed");
            return 0;
        }
        if (esim_ffn_gather(g->x, g->s_tok_index, g->xg, n_ent, npad, H, g->comp_st) ||
            esim_ffn_experts_ex(g->sw1_maps, g->sw2_maps, g->x_maps[npad_index(npad)], g->sact_maps[npad_index(npad)],
                                g->s_exec, g->s_tok_index, g->s_tok_weight, g->sact, g->y, n_ent, npad, g->Is, H,
                                std::min(T, 128), g->comp_st))
            return ls_fail(-3, "shared expert ffn launch failed");
        return 0;
    };
    auto flush = [&](int layer_rows, const int16_t* rs, const float* rw, bool residual, int layer) -> int {
        const int n_exec = (int)pend_slot.size();
        if (n_exec > 0) {
            int maxtok = 0;
            for (int t : tok_of_pos) maxtok = std::max(maxtok, t);
            const int npad = npad_for(std::max(1, maxtok));
            if (npad < 0) return ls_fail(-1, "too many tokens per expert");
            if (table_next + E + 3 * g->max_entries > g->table_cap) {             // recycle the pool
                CK(cudaStreamSynchronize(g->comp_st));
                table_next = 0;
            }
            int32_t* tpos = g->tables + table_next;
            int32_t* tslot = tpos + E;                  // FFN map per position: slot (bf16) or scratch entry
            int32_t* tpair = tslot + g->max_entries;    // quantised: (slot, scratch entry) grouped by precision
            table_next += E + 3 * g->max_entries;
            for (int e = 0; e < E; e++) tpos[e] = pos_of_expert[e];
            for (int i = 0; i < n_exec; i++) CK(cudaStreamWaitEvent(g->comp_st, g->landed[pend_slot[i]], 0));
            // decode flush (<= 4 tokens per expert) whose slots all hold one
            // precision: the streaming GEMV reads the slots directly (bf16 or
            // quantised codes, no gather, no scratch); ESIM_FFN_DECODE=tc selects
            // the tcgen05 decode kernels instead (quantised: dequant fused into
            // the A operand; bf16: the per-slice kernel below)
            int fused_bits = 0, gemv_bits = 0;
            if (npad == 16 && maxtok <= 4) {
                const int pc = slot_prec[pend_slot[0]];
                bool uniform = true;
                for (int i = 1; i < n_exec && uniform; i++) uniform = slot_prec[pend_slot[i]] == pc;
                if (uniform && g->decode_gemv) gemv_bits = 16 >> pc;
                else if (uniform && pc > 0 && g->fused_dequant && H / 128 <= 16) fused_bits = 16 >> pc;
            }
            if (gemv_bits) {
                for (int i = 0; i < n_exec; i++) tslot[i] = pend_slot[i];
                build_tables_kernel<<<1, 256, n_exec * 4, g->comp_st>>>(rs, rw, layer_rows, K, tpos, n_exec, npad,
                                                                       g->tok_index, g->tok_weight);
                if (esim_ffn_experts_gemv(g->slots, (int64_t)g->slot_bytes, gemv_bits, g->x, tslot, g->tok_index,
                                          g->tok_weight, g->y, n_exec, npad, std::max(1, maxtok), I, H, g->comp_st))
                    return ls_fail(-3, "gemv ffn launch failed");
                fused_bits = -1;                        // done: skip the tcgen05 paths below
            } else if (fused_bits) {
                for (int i = 0; i < n_exec; i++) tslot[i] = pend_slot[i];
                build_tables_kernel<<<1, 256, n_exec * 4, g->comp_st>>>(rs, rw, layer_rows, K, tpos, n_exec, npad,
                                                                       g->tok_index, g->tok_weight);
                if (esim_ffn_gather(g->x, g->tok_index, g->xg, n_exec, npad, H, g->comp_st) ||
                    esim_ffn_experts_q(g->slots, (int64_t)g->slot_bytes, fused_bits, g->x_maps[npad_index(npad)],
                                       tslot, g->tok_index, g->tok_weight, g->y, n_exec, I, H, g->comp_st))
                    return ls_fail(-3, "quantised ffn launch failed");
            }
            int n_pair = 0;
            for (int pc = 0; pc < 4 && !fused_bits; pc++) {   // slots holding precision pc
                if (!(g->mask >> pc & 1)) continue;
                const int first = n_pair;
                for (int i = 0; i < n_exec; i++) {
                    const int sl = pend_slot[i];
                    if (slot_prec[sl] != pc) continue;
                    if (pc == 0) { tslot[i] = sl; continue; }
                    if (scratch_of[sl] < 0) {           // one dequant per slot (splits / substitutes share it)
                        scratch_of[sl] = n_pair;
                        tpair[2 * n_pair] = sl;
                        tpair[2 * n_pair + 1] = n_pair;
                        n_pair++;
                    }
                    tslot[i] = g->n_slot_maps + scratch_of[sl];
                }
                if (n_pair == first) continue;
                const dim3 grid(96, n_pair - first);
                const int32_t* pr = tpair + 2 * first;
                const uint8_t* sl = (const uint8_t*)g->slots;
                __nv_bfloat16* sc = (__nv_bfloat16*)g->scratch;
                if (pc == 1) dequant_kernel<8><<<grid, 256, 0, g->comp_st>>>(sl, g->slot_bytes, pr, sc, I, H);
                if (pc == 2) dequant_kernel<4><<<grid, 256, 0, g->comp_st>>>(sl, g->slot_bytes, pr, sc, I, H);
                if (pc == 3) dequant_kernel<2><<<grid, 256, 0, g->comp_st>>>(sl, g->slot_bytes, pr, sc, I, H);
            }
            if (!fused_bits) build_tables_kernel<<<1, 256, n_exec * 4, g->comp_st>>>(rs, rw, layer_rows, K, tpos,
                                                                                    n_exec, npad, g->tok_index,
                                                                                    g->tok_weight);
            if (!fused_bits && (esim_ffn_gather(g->x, g->tok_index, g->xg, n_exec, npad, H, g->comp_st) ||
                esim_ffn_experts_ex(g->w1_maps, g->w2_maps, g->x_maps[npad_index(npad)],
                                    g->act_maps[npad_index(npad)], tslot, g->tok_index, g->tok_weight, g->act, g->y,
                                    n_exec, npad, I, H, std::max(1, maxtok), g->comp_st)))
                return ls_fail(-3, "ffn launch failed");
            for (int i = 0; i < n_exec; i++) {
                CK(cudaEventRecord(g->freed[pend_slot[i]], g->comp_st));
                scratch_of[pend_slot[i]] = -1;
            }
            n_exec_total += n_exec;
            n_flush++;
        }
        for (int s : pend_slot) slot_pending[s] = 0;
        pend_slot.clear();
        tok_of_pos.clear();
        std::fill(pos_of_expert.begin(), pos_of_expert.end(), -1);
        if (residual && g->Is) {
            const int rc2 = run_shared(layer, layer_rows);
            if (rc2) return rc2;
        }
        if (residual && esim_ffn_residual(g->x, g->y, (int64_t)layer_rows * H, g->comp_st))
            return ls_fail(-3, "residual launch failed");
        return 0;
    };
    // one FFN entry per executed expert; a substitute serving several missing
    // experts appears once per expert (same slot, separate token lists), so
    // no entry ever holds more than one expert's tokens
    // (more than 128 tokens: consecutive entries of 128 on the same slot)
    auto execute = [&](int expert, int slot, int tokens, int prec) -> int {
        if (slot < 0 || slot_prec[slot] != prec)
            return ls_fail(-2, "executed expert not resident at its recorded precision (decision stream inconsistent)");
        slot_pending[slot] = 1;
        pos_of_expert[expert] = (int)pend_slot.size();
        do {
            pend_slot.push_back(slot);
            tok_of_pos.push_back(std::min(tokens, 128));
            tokens -= 128;
        } while (tokens > 0);
        return 0;
    };

    for (int64_t ev = 0; ev < n_events; ev++) {
        const int pass = (int)(ev / L), layer = (int)(ev % L);
        const int T = h_pass_tokens[pass];
        int64_t done;
        while ((done = prog[0]) <= ev) {
            if (done < 0) return ls_fail(-2, "replay kernel reported an error");
            std::this_thread::yield();
        }
        const int64_t end = prog[1 + ev];
        if (layer == 0) {                                // this pass's input rows -> x (zero-copy)
            const void* src = pass == 0 ? x_prefill : (const char*)x_decode + (size_t)(pass - 1) * H * 2;
            copy_rows_kernel<<<64, 256, 0, g->comp_st>>>((const uint4*)src, (uint4*)g->x, (int64_t)T * H / 8);
        }
        const int16_t* rs = ro.row_sel + row * K;
        const float* rw = ro.row_w + row * K;
        for (; rec_pos < end; rec_pos++) {
            const EsimRec& r = g->recs[rec_pos];
            if (r.kind == ESIM_REC_EVICT) {
                const int v = r.i0 * E + r.i1;
                const int s = phys[v];
                if (s >= 0) {
                    if (slot_pending[s] && (rc = flush(T, rs, rw, false, layer))) return rc;   // self-eviction
                    free_slots.push_back(s);
                    phys[v] = -1;
                }
            } else if (r.kind == ESIM_REC_PREFETCH) {
                if (r.i0 == 1) {                         // started (working precision, engine.py:684)
                    if ((rc = issue_copy(r.i1 * E + r.i2, cfg->working_prec))) return rc;
                    n_prefetch++;
                } else if (r.i0 == 4 && r.i3 == 4) {     // dropped superseded: cancelled in flight
                    const int id = r.i1 * E + r.i2;
                    if (phys[id] >= 0) { free_slots.push_back(phys[id]); phys[id] = -1; }
                    n_cancel++;
                }
            } else if (r.kind == ESIM_REC_ACCESS) {
                const int outcome = r.i3 & 0xFF;
                const int prec = ((r.i3 >> 16) & 0xFF) - 1;  // the precision it executes at
                const int id = r.layer * E + r.i0;
                if (outcome == 1) {                      // demand fetch (fetch_low / priority: below working)
                    if ((rc = issue_copy(id, prec))) return rc;
                    n_demand++;
                }
                if (outcome <= 2) {
                    if ((rc = execute(r.i0, phys[id], r.i1, prec))) return rc;
                } else if (outcome == 4) {               // substitute runs the missing expert's tokens
                    if ((rc = execute(r.i0, phys[r.layer * E + r.i4], r.i1, prec))) return rc;
                }
            } else if (r.kind == ESIM_REC_ROUTE) {
                if ((rc = flush(T, rs, rw, true, layer))) return rc;
                if (g->capture) {                        // this layer's output -> host (zero-copy)
                    if (cap_row + T > g->capture_rows) return ls_fail(-4, "layer capture buffer too small");
                    copy_rows_kernel<<<64, 256, 0, g->comp_st>>>((const uint4*)g->x,
                                                                 (uint4*)((char*)g->capture + (size_t)cap_row * H * 2),
                                                                 (int64_t)T * H / 8);
                    cap_row += T;
                }
                if (layer == L - 1) {                    // pass output -> host (zero-copy)
                    copy_rows_kernel<<<64, 256, 0, g->comp_st>>>((const uint4*)g->x,
                                                                 (uint4*)((char*)out + (size_t)out_row * H * 2),
                                                                 (int64_t)T * H / 8);
                    out_row += T;
                    if (pass == 0) CK(cudaEventRecord(g->ev_ttft, g->comp_st));
                }
            }
        }
        row += T;
    }
    CK(cudaEventRecord(g->ev_copy_end, g->copy_st));
    CK(cudaStreamWaitEvent(g->comp_st, g->ev_copy_end, 0));
    CK(cudaEventRecord(g->ev_end, g->comp_st));
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    CK(cudaEventSynchronize(g->ev_end));
    CK(cudaStreamSynchronize(g->ctl_st));
    float ttft = 0, total = 0;
    CK(cudaEventElapsedTime(&ttft, g->ev_start, g->ev_ttft));
    CK(cudaEventElapsedTime(&total, g->ev_start, g->ev_end));
    CK(cudaMemcpy(counters_out, d_cnt, sizeof(EsimCounters), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(per_layer_out, d_pl, (size_t)L * ESIM_PL_FIELDS * 8, cudaMemcpyDeviceToHost));
    res->ttft_ms = ttft;
    res->total_ms = total;
    res->decode_ms = total - ttft;
    res->host_enqueue_ms = host_ms;
    res->h2d_bytes = h2d;
    res->n_copies = n_copies;
    res->n_demand_copies = n_demand;
    res->n_prefetch_copies = n_prefetch;
    res->n_cancelled = n_cancel;
    res->n_ffn_batches = n_flush;
    res->n_exec_experts = n_exec_total;
    res->n_records = rec_pos;
    res->status = 0;
    return 0;
}
