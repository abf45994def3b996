// router.cu -- fused router kernel: softmax + stable top-k routing, demand
// aggregation and the next-layer prefetch predictor, one CTA per trace
// event, one warp per token row.
//
// Reference computation (all bit-exact):
//   routing.softmax_rows / topk_indices / route_event   routing.py:22-35, 109-142
//   engine.Simulation._aggregate_demand                 engine.py:578-594
//   RouteRec selected/original mass (builtin sum)       engine.py:630-631
//   prefetch.predict_event (topk / score / oracle)      prefetch.py:39-107
// The output is policy independent under standard routing, so one launch
// serves every replayed grid point of the trace.
//
// HBM roofline: each event reads T*E*4 B of logits once and writes
// T*k*6 B of selections plus <= E demand / prediction records.
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/specmd_b200.h"
#include "numpy_f32.cuh"
#include "digest.cuh"

namespace esim {

struct RouterArgs {
    EsimTraceDesc tr;
    EsimRouterOut out;
    int pred_mode;      // ESIM_PF_*
    int pred_count;     // topk predictor: min(ceil(k*overfetch), E)
    int pred_clamped;   // topk predictor: ceil(k*overfetch) > E
    int pct_rank;       // score predictor: nearest rank (1-based), host-computed in double
};

constexpr int kRouterWarps = 8;

// warp argmax over the row in smem, ties to the lower index; `taken` is the
// per-lane bitmask of already-chosen elements (element i owned by lane i%32,
// bit i/32). Returns the winning index (uniform across the warp).
__device__ __forceinline__ int warp_argmax(const float* s, int E, int lane, uint32_t taken) {
    float bv = -1.0f;
    int bi = 0x7fffffff;
    for (int i = lane, j = 0; i < E; i += 32, j++) {
        if (taken & (1u << j)) continue;
        float v = s[i];
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    return bi;
}

__device__ __forceinline__ void route_event_cta(const RouterArgs& a, int64_t ev, unsigned char* smem);

__global__ void __launch_bounds__(kRouterWarps * 32)
router_kernel(RouterArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    route_event_cta(a, blockIdx.x, smem);
}

// one launch over many traces: block b -> (trace t, event b - prefix[t])
struct RouterBatchArgs {
    const EsimTraceDesc* traces;
    const EsimRouterOut* outs;
    const int32_t* params;        // [n][4]: pred_mode, pred_count, pred_clamped, pct_rank
    const int64_t* prefix;        // [n+1] event prefix sums
    int n;
};

__global__ void __launch_bounds__(kRouterWarps * 32)
router_batch_kernel(RouterBatchArgs b) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t g = blockIdx.x;
    int lo = 0, hi = b.n - 1;
    while (lo < hi) {                       // last t with prefix[t] <= g
        const int mid = (lo + hi + 1) >> 1;
        if (b.prefix[mid] <= g) lo = mid; else hi = mid - 1;
    }
    RouterArgs a;
    a.tr = b.traces[lo];
    a.out = b.outs[lo];
    a.pred_mode = b.params[lo * 4 + 0];
    a.pred_count = b.params[lo * 4 + 1];
    a.pred_clamped = b.params[lo * 4 + 2];
    a.pct_rank = b.params[lo * 4 + 3];
    route_event_cta(a, g - b.prefix[lo], smem);
}

__device__ __forceinline__ void route_event_cta(const RouterArgs& a, int64_t ev, unsigned char* smem) {
    const int E = a.tr.experts, K = a.tr.top_k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* rowbuf = reinterpret_cast<float*>(smem) + warp * E;             // [warps][E]
    unsigned* best = reinterpret_cast<unsigned*>(smem) + kRouterWarps * E;  // [E] prediction union
    int* cnt = reinterpret_cast<int*>(best + E);                            // [2]

    const int64_t r0 = a.tr.row_offset[ev], r1 = a.tr.row_offset[ev + 1];
    const int T = (int)(r1 - r0);
    for (int i = threadIdx.x; i < E; i += blockDim.x) best[i] = 0u;
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    __syncthreads();

    const int nsel = a.pred_mode == ESIM_PF_TOPK ? max(K, a.pred_count) : K;
    for (int r = warp; r < T; r += kRouterWarps) {
        const float* x = a.tr.logits + (r0 + r) * (int64_t)E;
        float m = -__int_as_float(0x7f800000);
        for (int i = lane; i < E; i += 32) { float v = x[i]; rowbuf[i] = v; m = fmaxf(m, v); }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        for (int i = lane; i < E; i += 32) rowbuf[i] = np_expf(__fsub_rn(rowbuf[i], m));
        __syncwarp();
        float S = __fadd_rn(0.0f, warp_pw_sum(rowbuf, E, lane));
        __syncwarp();
        for (int i = lane; i < E; i += 32) rowbuf[i] = __fdiv_rn(rowbuf[i], S);
        __syncwarp();

        // stable top-nsel: repeated warp argmax (score desc, index asc)
        uint32_t taken = 0;
        int16_t* sel = a.out.row_sel + (r0 + r) * K;
        float* w = a.out.row_w + (r0 + r) * K;
        for (int j = 0; j < nsel; j++) {
            int b = warp_argmax(rowbuf, E, lane, taken);
            if ((b & 31) == lane) taken |= 1u << (b >> 5);
            if (lane == 0) {
                if (j < K) { sel[j] = (int16_t)b; w[j] = rowbuf[b]; }
                bool pred = (a.pred_mode == ESIM_PF_TOPK && j < a.pred_count) ||
                            (a.pred_mode == ESIM_PF_ORACLE && j < K);
                if (pred) atomicMax(&best[b], __float_as_uint(rowbuf[b]) + 1u);
            }
        }
        if (a.pred_mode == ESIM_PF_SCORE) {
            // nearest-rank percentile: the value at sorted position pct_rank-1
            float thr = 0.0f;
            bool found = false;
            for (int i = lane; i < E; i += 32) {
                float v = rowbuf[i];
                int less = 0, le = 0;
                for (int j = 0; j < E; j++) { float u = rowbuf[j]; less += (u < v); le += (u <= v); }
                if (less <= a.pct_rank - 1 && a.pct_rank - 1 < le) { thr = v; found = true; }
            }
            unsigned who = __ballot_sync(0xffffffffu, found);
            thr = __shfl_sync(0xffffffffu, thr, __ffs(who) - 1);
            for (int i = lane; i < E; i += 32)
                if (rowbuf[i] > thr) atomicMax(&best[i], __float_as_uint(rowbuf[i]) + 1u);
        }
        __syncwarp();
    }
    __syncthreads();

    // ---- predictions for this event as a target: sort (-score, expert) ----
    const int64_t eb = ev * E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        unsigned ke = best[e];
        if (!ke) continue;
        int pos = 0;
        for (int j = 0; j < E; j++) {
            unsigned kj = best[j];
            pos += (kj > ke) || (kj == ke && kj && j < e);
        }
        a.out.pred_expert[eb + pos] = e;
        a.out.pred_score[eb + pos] = __uint_as_float(ke - 1u);
        atomicAdd(&cnt[0], 1);
    }

    // ---- demand aggregation (engine.py:578-594) -------------------------
    // pass 1: per expert best (lowest) rank and max gate -> smem (reuses the
    // row buffers); pass 2: sort key (rank, -gate, expert) -> position, and
    // the row-ordered fp64 sum (plain +=, engine.py:592) + token count.
    __syncthreads();
    float* gate_s = reinterpret_cast<float*>(smem);
    int* rank_s = reinterpret_cast<int*>(smem) + E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int rank = 0x7fffffff;
        float gate = -1.0f;
        for (int r = 0; r < T; r++) {
            const int16_t* sel = a.out.row_sel + (r0 + r) * K;
            for (int j = 0; j < K; j++)
                if (sel[j] == e) {
                    rank = min(rank, j + 1);
                    gate = fmaxf(gate, a.out.row_w[(r0 + r) * K + j]);
                }
        }
        gate_s[e] = gate;
        rank_s[e] = rank;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int rk = rank_s[e];
        if (rk == 0x7fffffff) continue;
        const float g = gate_s[e];
        int pos = 0;
        for (int j = 0; j < E; j++) {
            int rj = rank_s[j];
            if (rj == 0x7fffffff || j == e) continue;
            float gj = gate_s[j];
            pos += (rj < rk) || (rj == rk && (gj > g || (gj == g && j < e)));
        }
        int tok = 0;
        double summed = 0.0;
        for (int r = 0; r < T; r++) {
            const int16_t* sel = a.out.row_sel + (r0 + r) * K;
            for (int j = 0; j < K; j++)
                if (sel[j] == e) {
                    double wv = (double)a.out.row_w[(r0 + r) * K + j];
                    summed = tok ? __dadd_rn(summed, wv) : wv;
                    tok++;
                }
        }
        a.out.dem_expert[eb + pos] = e;
        a.out.dem_rank[eb + pos] = rk;
        a.out.dem_gate[eb + pos] = g;
        a.out.dem_summed[eb + pos] = summed;
        a.out.dem_tokens[eb + pos] = tok;
        atomicAdd(&cnt[1], 1);
    }
    __syncthreads();

    // ---- RouteRec mass: sum(sum(dec.weights) for dec) with builtin sum ---
    if (threadIdx.x == 0) {
        PySum outer;
        outer.init();
        for (int r = 0; r < T; r++) {
            PySum in;
            in.init();
            for (int j = 0; j < K; j++) in.add((double)a.out.row_w[(r0 + r) * K + j]);
            outer.add(in.value());
        }
        a.out.sel_mass[ev] = outer.value();
        a.out.n_pred[ev] = cnt[0];
        a.out.n_dem[ev] = cnt[1];
        a.out.pred_clamped[ev] = (a.pred_mode == ESIM_PF_TOPK) ? a.pred_clamped : 0;
    }
}

// ---------------------------------------------------------------------------
// Router summary: the part of every replay that depends on the router output
// alone, computed once per trace instead of once per grid point.
//   * per event: the RouteRec digest word under standard routing with no
//     drop/substitution (faithful = T, modified = 0, executed = original
//     mass), the PredictionRec digest word of the predictions targeting the
//     event (emitted at layer l-1, engine.py:651-660);
//   * per trace: the prefetch precision/recall accounting
//     (metrics.py:150-187: |pred & dem| / |pred|, / |dem| for every event
//     with layer >= 1, Neumaier-summed in event order), the RouteRec
//     original-mass sum, rows, and per target layer the predicted-set sizes.
// ---------------------------------------------------------------------------
struct SumArgs {
    const EsimTraceDesc* traces;   // batch: device arrays; nullptr: the single trace below
    const EsimRouterOut* outs;
    const int32_t* params;         // [n][4], params[4t] = pred_mode
    const int64_t* prefix;         // [n+1]
    int n;
    EsimTraceDesc tr1;
    EsimRouterOut out1;
    int mode1;
};

__device__ __forceinline__ int sum_trace_of(const SumArgs& a, int64_t g) {
    int lo = 0, hi = a.n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.prefix[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// one warp per event
__global__ void __launch_bounds__(256) route_events_kernel(SumArgs a, int64_t total) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= total) return;
    int t = 0;
    int64_t ev = g;
    if (a.traces) { t = sum_trace_of(a, g); ev = g - a.prefix[t]; }
    const EsimTraceDesc& tr = a.traces ? a.traces[t] : a.tr1;
    const EsimRouterOut& o = a.traces ? a.outs[t] : a.out1;
    const int E = tr.experts, L = tr.num_layers;
    const int pass = (int)(ev / L), l = (int)(ev % L);
    const int np = o.n_pred[ev];
    uint32_t pm = 0;
    for (int j = lane; j < np; j += 32) pm += pe_mix_term(j, o.pred_expert[ev * E + j]);
    #pragma unroll
    for (int s = 16; s > 0; s >>= 1) pm += __shfl_xor_sync(0xffffffffu, pm, s);
    if (lane == 0) {
        const int T = (int)(tr.row_offset[ev + 1] - tr.row_offset[ev]);
        const double origm = o.sel_mass[ev];
        const double exm = __dadd_rn(origm, 0.0);
        o.route_mix[ev] = rec_mix(ESIM_REC_ROUTE, pass, l, T, T, 0, 0, 0, 0, __double_as_longlong(origm),
                                  __double_as_longlong(exm), origm);
        o.pred_mix[ev] = l >= 1 ? rec_mix(ESIM_REC_PREDICTION, pass, l - 1, l, np, o.pred_clamped[ev], 0, 0, 0, 0, 0,
                                          0.0) + pm
                                : 0u;
    }
}

__device__ __forceinline__ void nsum_add(double& f, double& c, double x) {   // PySum step (ps_add)
    const double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
    f = t;
}

// one warp per trace: events in chunks of 32 (lane i evaluates event base+i),
// folded in event order with warp-uniform Neumaier sums
__global__ void __launch_bounds__(32) route_totals_kernel(SumArgs a) {
    const int t = blockIdx.x, lane = threadIdx.x;
    const EsimTraceDesc& tr = a.traces ? a.traces[t] : a.tr1;
    const EsimRouterOut& o = a.traces ? a.outs[t] : a.out1;
    const int mode = a.traces ? a.params[4 * t] : a.mode1;
    const int E = tr.experts, L = tr.num_layers;
    const int64_t ne = tr.n_events;
    const bool pf = mode != ESIM_PF_NONE;
    EsimRouteSummary s;
    s.pf_tp = s.pf_pred = s.pf_dem = s.pf_records = s.pf_prec_parts = s.pf_empty = s.pf_rec_parts = 0;
    s.rows_total = 0;
    s.orig_f = s.orig_c = s.prec_f = s.prec_c = s.rec_f = s.rec_c = 0.0;
    for (int64_t base = 0; base < ne; base += 32) {
        const int64_t ev = base + lane;
        int T = 0, inter = 0, np = 0, nd = 0, has = 0;
        double origm = 0.0, pr = 0.0, rc = 0.0;
        if (ev < ne) {
            T = (int)(tr.row_offset[ev + 1] - tr.row_offset[ev]);
            origm = o.sel_mass[ev];
            if (pf && ev % L >= 1) {
                has = 1;
                np = o.n_pred[ev];
                nd = o.n_dem[ev];
                const int32_t* de = o.dem_expert + ev * E;
                const int32_t* pe = o.pred_expert + ev * E;
                for (int j = 0; j < np; j++) {
                    const int e = pe[j];
                    for (int i = 0; i < nd; i++) inter += de[i] == e;
                }
                if (np) pr = __ddiv_rn((double)inter, (double)np);
                rc = __ddiv_rn((double)inter, (double)nd);
            }
        }
        const int cnt = ne - base < 32 ? (int)(ne - base) : 32;
        for (int k = 0; k < cnt; k++) {
            const int Tk = __shfl_sync(0xffffffffu, T, k);
            const double ok = __shfl_sync(0xffffffffu, origm, k);
            const int hk = __shfl_sync(0xffffffffu, has, k);
            s.rows_total += Tk;
            nsum_add(s.orig_f, s.orig_c, ok);
            if (hk) {
                const int ik = __shfl_sync(0xffffffffu, inter, k);
                const int npk = __shfl_sync(0xffffffffu, np, k);
                const int ndk = __shfl_sync(0xffffffffu, nd, k);
                const double prk = __shfl_sync(0xffffffffu, pr, k);
                const double rck = __shfl_sync(0xffffffffu, rc, k);
                s.pf_tp += ik; s.pf_pred += npk; s.pf_dem += ndk; s.pf_records++;
                if (npk) { s.pf_prec_parts++; nsum_add(s.prec_f, s.prec_c, prk); }
                else s.pf_empty++;
                s.pf_rec_parts++;
                nsum_add(s.rec_f, s.rec_c, rck);
            }
        }
    }
    if (lane == 0) *o.summary = s;
    // per target layer (>= 1): predicted-set sizes and prediction events
    const int passes = tr.n_passes;
    for (int l = lane; l < L; l += 32) {
        int64_t n = 0, c = 0;
        if (pf && l >= 1)
            for (int p = 0; p < passes; p++) { n += o.n_pred[(int64_t)p * L + l]; c++; }
        o.layer_pred[2 * l] = n;
        o.layer_pred[2 * l + 1] = c;
    }
}

cudaError_t route_summary(const SumArgs& a, int n_traces, int64_t total_events, cudaStream_t st) {
    if (total_events <= 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((total_events * 32 + 255) / 256);
    route_events_kernel<<<blocks, 256, 0, st>>>(a, total_events);
    route_totals_kernel<<<n_traces, 32, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace esim

extern "C" int esim_router_launch_batch(const EsimTraceDesc* d_traces, const EsimRouterOut* d_outs,
                                        const int32_t* d_params, const int64_t* d_prefix, int32_t n_traces,
                                        int64_t total_events, int32_t max_experts, void* stream) {
    if (total_events <= 0) return 0;
    esim::RouterBatchArgs b{d_traces, d_outs, d_params, d_prefix, n_traces};
    const size_t smem = (size_t)(esim::kRouterWarps * max_experts + max_experts) * 4 + 16;
    esim::router_batch_kernel<<<(unsigned)total_events, esim::kRouterWarps * 32, smem, (cudaStream_t)stream>>>(b);
    esim::SumArgs s{};
    s.traces = d_traces; s.outs = d_outs; s.params = d_params; s.prefix = d_prefix; s.n = n_traces;
    if (esim::route_summary(s, n_traces, total_events, (cudaStream_t)stream) != cudaSuccess) return -3;
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

extern "C" int esim_route_summary_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode,
                                         void* stream) {
    esim::SumArgs s{};
    s.n = 1; s.tr1 = *tr; s.out1 = *out; s.mode1 = pred_mode;
    return esim::route_summary(s, 1, tr->n_events, (cudaStream_t)stream) == cudaSuccess ? 0 : -3;
}

// host launcher (declared in capi.cu)
cudaError_t esim_router_launch_impl(const EsimTraceDesc& tr, const EsimRouterOut& out, int pred_mode,
                                    int pred_count, int pred_clamped, int pct_rank, cudaStream_t st) {
    esim::RouterArgs a{tr, out, pred_mode, pred_count, pred_clamped, pct_rank};
    size_t smem = (size_t)(esim::kRouterWarps * tr.experts + tr.experts) * 4 + 16;
    if (tr.n_events == 0) return cudaSuccess;
    esim::router_kernel<<<(unsigned)tr.n_events, esim::kRouterWarps * 32, smem, st>>>(a);
    esim::SumArgs s{};
    s.n = 1; s.tr1 = tr; s.out1 = out; s.mode1 = pred_mode;
    return esim::route_summary(s, 1, tr.n_events, st);
}

// ---------------------------------------------------------------------------
// standalone plug-in kernels: routing.softmax_rows and routing.topk_indices
// (routing.py:22-35) over a (rows, E) matrix, one warp per row
// ---------------------------------------------------------------------------
namespace esim {
__global__ void softmax_rows_kernel(const float* __restrict__ x, int rows, int E, float* __restrict__ out) {
    extern __shared__ float sbuf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x >> 5) + warp;
    if (r >= rows) return;
    float* buf = sbuf + warp * E;
    float m = -__int_as_float(0x7f800000);
    for (int i = lane; i < E; i += 32) { float v = x[(int64_t)r * E + i]; buf[i] = v; m = fmaxf(m, v); }
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int i = lane; i < E; i += 32) buf[i] = np_expf(__fsub_rn(buf[i], m));
    __syncwarp();
    float S = __fadd_rn(0.0f, warp_pw_sum(buf, E, lane));
    for (int i = lane; i < E; i += 32) out[(int64_t)r * E + i] = __fdiv_rn(buf[i], S);
}

__global__ void topk_rows_kernel(const float* __restrict__ s, int rows, int E, int k, int32_t* __restrict__ idx) {
    extern __shared__ float sbuf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x >> 5) + warp;
    if (r >= rows) return;
    float* buf = sbuf + warp * E;
    for (int i = lane; i < E; i += 32) buf[i] = s[(int64_t)r * E + i];
    __syncwarp();
    uint32_t taken = 0;
    for (int j = 0; j < k; j++) {
        // stable argsort of -scores: larger first, ties to the lower index;
        // NaN-free inputs assumed (router scores)
        float bv = -__int_as_float(0x7f800000);
        int bi = 0x7fffffff;
        for (int i = lane, t = 0; i < E; i += 32, t++) {
            if (taken & (1u << t)) continue;
            float v = buf[i];
            if (bi == 0x7fffffff || v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi != 0x7fffffff && (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
        }
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == 0) idx[(int64_t)r * k + j] = bi;
    }
}
}  // namespace esim

extern "C" int esim_softmax_launch(const float* d_x, int32_t rows, int32_t E, float* d_out, void* stream) {
    if (E < 1 || E > ESIM_MAX_E) return -1;
    int wpb = 4;
    int blocks = (rows + wpb - 1) / wpb;
    if (blocks == 0) return 0;
    esim::softmax_rows_kernel<<<blocks, wpb * 32, wpb * E * 4, (cudaStream_t)stream>>>(d_x, rows, E, d_out);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

extern "C" int esim_topk_launch(const float* d_s, int32_t rows, int32_t E, int32_t k, int32_t* d_idx, void* stream) {
    if (E < 1 || E > ESIM_MAX_E || k < 1 || k > E) return -1;
    int wpb = 4;
    int blocks = (rows + wpb - 1) / wpb;
    if (blocks == 0) return 0;
    esim::topk_rows_kernel<<<blocks, wpb * 32, wpb * E * 4, (cudaStream_t)stream>>>(d_s, rows, E, k, d_idx);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---------------------------------------------------------------------------
// routing.route_event(policy=CACHE_AWARE) for one event (routing.py:143-161):
// rows in order (the running mean a row's bias uses includes every earlier
// row), one warp. cached: bit e of cached_mask set when expert e is resident
// at this layer. delta[0] = sums[layer], delta[1] = counts[layer] (in/out).
// ---------------------------------------------------------------------------
#include "warp_route.cuh"
namespace esim {
__global__ void route_cache_aware_kernel(const float* __restrict__ x, int T, int E, int K,
                                         const uint32_t* __restrict__ cached_mask, double lam, double* delta,
                                         int16_t* sel, float* w, int16_t* orig, float* ow, int32_t* modified) {
    extern __shared__ float rbuf[];
    float* buf = rbuf;          // [E]
    float* sc = rbuf + E;       // [E] original scores
    const int lane = threadIdx.x & 31;
    bool any_cached = false;
    for (int e = lane; e < E; e += 32) any_cached |= (cached_mask[e >> 5] >> (e & 31)) & 1;
    any_cached = __any_sync(0xffffffffu, any_cached);
    double sum = delta[0];
    double cnt = delta[1];
    for (int r = 0; r < T; r++) {
        const float* xr = x + (int64_t)r * E;
        for (int i = lane; i < E; i += 32) buf[i] = xr[i];
        __syncwarp();
        warp_softmax(buf, E, lane);
        for (int i = lane; i < E; i += 32) sc[i] = buf[i];
        __syncwarp();
        warp_topk(sc, E, K, lane, orig + r * K);
        const double mean = cnt != 0.0 ? __ddiv_rn(sum, cnt) : 0.0;
        const bool on = lam != 0.0 && mean != 0.0 && any_cached;
        const float bias = __double2float_rn(__dmul_rn(lam, mean));
        for (int i = lane; i < E; i += 32) {
            float v = xr[i];
            if (on && ((cached_mask[i >> 5] >> (i & 31)) & 1)) v = __fadd_rn(v, bias);
            buf[i] = v;
        }
        __syncwarp();
        warp_softmax(buf, E, lane);
        warp_topk(buf, E, K, lane, sel + r * K);
        for (int i = lane; i < E; i += 32) buf[i] = xr[i];
        __syncwarp();
        sum = __dadd_rn(sum, __dadd_rn(0.0, warp_pw_sum_f64(buf, E, lane)));
        cnt = __dadd_rn(cnt, (double)E);
        if (lane == 0) {
            bool same = true;
            for (int a = 0; a < K; a++) {
                bool f = false;
                for (int b = 0; b < K; b++) f |= sel[r * K + a] == orig[r * K + b];
                same &= f;
            }
            modified[r] = same ? 0 : 1;
            for (int a = 0; a < K; a++) { w[r * K + a] = sc[sel[r * K + a]]; ow[r * K + a] = sc[orig[r * K + a]]; }
        }
        __syncwarp();
    }
    if (lane == 0) { delta[0] = sum; delta[1] = cnt; }
}
}  // namespace esim

extern "C" int esim_route_cache_aware_launch(const float* d_x, int32_t rows, int32_t experts, int32_t top_k,
                                             const uint32_t* d_cached_mask, double lam, double* d_delta,
                                             int16_t* d_sel, float* d_w, int16_t* d_orig, float* d_ow,
                                             int32_t* d_modified, void* stream) {
    if (experts < 1 || experts > ESIM_MAX_E || top_k < 1 || top_k > ESIM_MAX_K || top_k > experts) return -1;
    esim::route_cache_aware_kernel<<<1, 32, 2 * experts * 4, (cudaStream_t)stream>>>(
        d_x, rows, experts, top_k, d_cached_mask, lam, d_delta, d_sel, d_w, d_orig, d_ow, d_modified);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
