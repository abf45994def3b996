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
#include <mutex>
#include <unordered_map>
#include <utility>

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

// per-event digest words of the router-fixed records (see the router
// summary below): RouteRec under standard routing, PredictionRec targeting ev
__device__ __forceinline__ void write_event_mixes(const EsimRouterOut& o, int64_t ev, int L, int T, int np,
                                                  uint32_t pm, double origm, int clamped) {
    const int pass = (int)(ev / L), l = (int)(ev % L);
    const double exm = __dadd_rn(origm, 0.0);
    o.route_mix[ev] = rec_mix(ESIM_REC_ROUTE, pass, l, T, T, 0, 0, 0, 0, __double_as_longlong(origm),
                              __double_as_longlong(exm), origm);
    o.pred_mix[ev] = l >= 1 ? rec_mix(ESIM_REC_PREDICTION, pass, l - 1, l, np, clamped, 0, 0, 0, 0, 0, 0.0) + pm : 0u;
}

// generic path (any E <= ESIM_MAX_E, any T): one CTA per event, one warp per row
__device__ __forceinline__ void route_event_cta_generic(const RouterArgs& a, int64_t ev, unsigned char* smem) {
    const int E = a.tr.experts, K = a.tr.top_k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* rowbuf = reinterpret_cast<float*>(smem) + warp * E;             // [warps][E]
    unsigned* best = reinterpret_cast<unsigned*>(smem) + kRouterWarps * E;  // [E] prediction union
    int* cnt = reinterpret_cast<int*>(best + E);                            // [2]

    const int64_t r0 = a.tr.row_offset[ev], r1 = a.tr.row_offset[ev + 1];
    const int T = (int)(r1 - r0);
    for (int i = threadIdx.x; i < E; i += blockDim.x) best[i] = 0u;
    if (threadIdx.x < 3) cnt[threadIdx.x] = 0;       // n_pred, n_dem, PredictionRec digest term
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
        atomicAdd(reinterpret_cast<unsigned*>(&cnt[2]), pe_mix_term(pos, e));
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
        const double origm = outer.value();
        const int clamped = (a.pred_mode == ESIM_PF_TOPK) ? a.pred_clamped : 0;
        a.out.sel_mass[ev] = origm;
        a.out.n_pred[ev] = cnt[0];
        a.out.n_dem[ev] = cnt[1];
        a.out.pred_clamped[ev] = clamped;
        write_event_mixes(a.out, ev, a.tr.num_layers, T, cnt[0], (uint32_t)cnt[2], origm, clamped);
    }
}

// ---------------------------------------------------------------------------
// E <= 64 fast path. A row's scores live in registers (element i of the row
// in lane i % 32, register i / 32) and are ordered once by a warp bitonic
// sort of the unique 64-bit keys (~score_bits << 32 | expert): position p of
// the sorted row is the p-th routed expert (stable top-k: score desc, index
// asc, routing.py:32-35), the top-count predictor's p-th pick, and the
// nearest-rank percentile (prefetch.py:30-36) is the key at descending
// position E - rank, so the score predictor's set (scores strictly above it,
// prefetch.py:57-64) is a prefix of the same order. Scores are softmax
// outputs (>= 0), so ~bits orders them exactly.
// ---------------------------------------------------------------------------
constexpr uint64_t kNoKey = ~0ull;

__device__ __forceinline__ uint64_t u64min(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t u64max(uint64_t a, uint64_t b) { return a < b ? b : a; }
__device__ __forceinline__ int key_expert(uint64_t k) { return (int)(uint32_t)k; }
__device__ __forceinline__ float key_score(uint64_t k) { return __uint_as_float(~(uint32_t)(k >> 32)); }

// ascending bitonic sort of N = 8, 16, 32 or 64 keys, element i = lane + 32 * reg
// (N < 32: lanes >= N sort their own padding, never mixed in)
template <int N>
__device__ __forceinline__ void bitonic_sort(uint64_t& a0, uint64_t& a1, int lane) {
    constexpr bool TWO = N == 64;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {                                  // k == 64: partner is the other register
                const uint64_t lo = u64min(a0, a1);
                a1 = u64max(a0, a1);
                a0 = lo;
                continue;
            }
            const bool lower = (lane & j) == 0;
            {
                const uint64_t p = __shfl_xor_sync(0xffffffffu, (unsigned long long)a0, j);
                const bool up = (lane & k) == 0;
                a0 = (lower == up) ? u64min(a0, p) : u64max(a0, p);
            }
            if (TWO) {
                const uint64_t p = __shfl_xor_sync(0xffffffffu, (unsigned long long)a1, j);
                const bool up = ((lane + 32) & k) == 0;
                a1 = (lower == up) ? u64min(a1, p) : u64max(a1, p);
            }
        }
    }
}

// softmax_rows of one row (bit-exact, routing.py:22-29) -> sorted keys.
// buf: this warp's E floats of shared memory (numpy's pairwise sum order).
template <int N>
__device__ __forceinline__ void row_keys64(const float* __restrict__ x, int E, int lane, float* buf, uint64_t& k0,
                                           uint64_t& k1) {
    constexpr bool TWO = N == 64;
    const float ninf = -__int_as_float(0x7f800000);
    const bool h0 = lane < E, h1 = TWO && lane + 32 < E;
    const float v0 = h0 ? x[lane] : ninf;
    const float v1 = h1 ? x[lane + 32] : ninf;
    float m = fmaxf(v0, v1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float e0 = h0 ? np_expf(__fsub_rn(v0, m)) : 0.0f;
    const float e1 = h1 ? np_expf(__fsub_rn(v1, m)) : 0.0f;
    if (h0) buf[lane] = e0;
    if (h1) buf[lane + 32] = e1;
    __syncwarp();
    const float S = __fadd_rn(0.0f, warp_pw_sum(buf, E, lane));
    __syncwarp();
    k0 = h0 ? ((uint64_t)(~__float_as_uint(__fdiv_rn(e0, S))) << 32) | (uint32_t)lane : kNoKey;
    k1 = h1 ? ((uint64_t)(~__float_as_uint(__fdiv_rn(e1, S))) << 32) | (uint32_t)(lane + 32) : kNoKey;
    bitonic_sort<N>(k0, k1, lane);
}

// number of predicted experts of one row in sorted order (prefix length)
template <int N>
__device__ __forceinline__ int row_pred_count(const RouterArgs& a, int E, int K, uint64_t k0, uint64_t k1) {
    constexpr bool TWO = N == 64;
    switch (a.pred_mode) {
    case ESIM_PF_TOPK: return a.pred_count;
    case ESIM_PF_ORACLE: return K;
    case ESIM_PF_SCORE: {
        int q = E - a.pct_rank;                               // descending position of the percentile
        q = q < 0 ? 0 : (q > E - 1 ? E - 1 : q);
        const uint64_t kq0 = __shfl_sync(0xffffffffu, (unsigned long long)k0, q & 31);
        const uint64_t kq1 = TWO ? __shfl_sync(0xffffffffu, (unsigned long long)k1, q & 31) : kNoKey;
        const float thr = key_score(q < 32 ? kq0 : kq1);
        const unsigned b0 = __ballot_sync(0xffffffffu, k0 != kNoKey && key_score(k0) > thr);
        const unsigned b1 = TWO ? __ballot_sync(0xffffffffu, k1 != kNoKey && key_score(k1) > thr) : 0u;
        return __popc(b0) + __popc(b1);
    }
    default: return 0;
    }
}

// inner RouteRec mass of one row: builtin sum over the K weights (lane 0's value)
__device__ __forceinline__ double row_mass(float w, int K, int lane) {
    PySum in;
    in.init();
    for (int j = 0; j < K; j++) {
        const float wj = __shfl_sync(0xffffffffu, w, j);
        in.add((double)wj);
    }
    return in.value();
}

// a single-row event (decode passes): one warp does everything
template <int N>
__device__ __forceinline__ void route_single_warp(const RouterArgs& a, int64_t ev, float* buf, int lane) {
    constexpr bool TWO = N == 64;
    const int E = a.tr.experts, K = a.tr.top_k;
    const int64_t r0 = a.tr.row_offset[ev];
    uint64_t k0, k1;
    row_keys64<N>(a.tr.logits + r0 * E, E, lane, buf, k0, k1);
    const int x0 = key_expert(k0), x1 = key_expert(k1);
    const float s0 = key_score(k0), s1 = key_score(k1);
    const int64_t eb = ev * E;
    if (lane < K) {                    // one row: demand rank j+1 = routing position j (engine.py:578-594)
        a.out.row_sel[r0 * K + lane] = (int16_t)x0;
        a.out.row_w[r0 * K + lane] = s0;
        a.out.dem_expert[eb + lane] = x0;
        a.out.dem_rank[eb + lane] = lane + 1;
        a.out.dem_gate[eb + lane] = s0;
        a.out.dem_summed[eb + lane] = (double)s0;
        a.out.dem_tokens[eb + lane] = 1;
    }
    const int c = row_pred_count<N>(a, E, K, k0, k1);
    if (lane < c) { a.out.pred_expert[eb + lane] = x0; a.out.pred_score[eb + lane] = s0; }
    if (TWO && lane + 32 < c) { a.out.pred_expert[eb + lane + 32] = x1; a.out.pred_score[eb + lane + 32] = s1; }
    const double inner = row_mass(s0, K, lane);
    uint32_t pm = (lane < c ? pe_mix_term(lane, x0) : 0u) + (TWO && lane + 32 < c ? pe_mix_term(lane + 32, x1) : 0u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pm += __shfl_xor_sync(0xffffffffu, pm, o);
    if (lane == 0) {
        PySum outer;
        outer.init();
        outer.add(inner);
        const double origm = outer.value();
        const int clamped = (a.pred_mode == ESIM_PF_TOPK) ? a.pred_clamped : 0;
        a.out.sel_mass[ev] = origm;
        a.out.n_pred[ev] = c;
        a.out.n_dem[ev] = K;
        a.out.pred_clamped[ev] = clamped;
        write_event_mixes(a.out, ev, a.tr.num_layers, 1, c, pm, origm, clamped);
    }
}

// shared memory of the multi-row E <= 64 CTA path
struct Multi64Smem {
    float rowbuf[kRouterWarps][64];
    float wgt[64][64];                // [expert][row within the 64-row chunk]
    unsigned long long mask[64];      // rows (within the chunk) that selected the expert
    double rmass[64];                 // inner RouteRec mass per row of the chunk
    unsigned best[64];                // prediction union: max score bits + 1
    unsigned gate[64];                // max gate bits (scores >= 0)
    int rank[64];                     // best (lowest) rank
    int cnt[2];
    unsigned pm;                      // PredictionRec expert-list digest term
};

// a multi-row event (prefill passes): rows spread over the warps in chunks
// of 64; per expert the row-ordered fp64 sum of weights (engine.py:592) is
// folded after each chunk from the row bitmask, so no O(E*T*K) rescans.
template <int N>
__device__ __forceinline__ void route_multi64_cta(const RouterArgs& a, int64_t ev, unsigned char* smem_raw) {
    constexpr bool TWO = N == 64;
    Multi64Smem& s = *reinterpret_cast<Multi64Smem*>(smem_raw);
    const int E = a.tr.experts, K = a.tr.top_k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int64_t r0 = a.tr.row_offset[ev], r1 = a.tr.row_offset[ev + 1];
    const int T = (int)(r1 - r0);
    const int64_t eb = ev * E;
    if (tid < 64) { s.best[tid] = 0u; s.gate[tid] = 0u; s.rank[tid] = 0x7fffffff; s.mask[tid] = 0ull; }
    if (tid < 2) s.cnt[tid] = 0;
    if (tid == 0) s.pm = 0u;
    double summed = 0.0;               // thread e < E: running row-ordered sum of expert e
    int tok = 0;
    PySum outer;
    outer.init();
    __syncthreads();
    for (int c0 = 0; c0 < T; c0 += 64) {
        const int cn = min(64, T - c0);
        for (int rr = warp; rr < cn; rr += kRouterWarps) {
            const int64_t row = r0 + c0 + rr;
            uint64_t k0, k1;
            row_keys64<N>(a.tr.logits + row * E, E, lane, s.rowbuf[warp], k0, k1);
            const int x0 = key_expert(k0), x1 = key_expert(k1);
            const float s0 = key_score(k0), s1 = key_score(k1);
            if (lane < K) {
                a.out.row_sel[row * K + lane] = (int16_t)x0;
                a.out.row_w[row * K + lane] = s0;
                atomicOr(&s.mask[x0], 1ull << rr);
                s.wgt[x0][rr] = s0;
                atomicMin(&s.rank[x0], lane + 1);
                atomicMax(&s.gate[x0], __float_as_uint(s0));
            }
            const int c = row_pred_count<N>(a, E, K, k0, k1);
            if (lane < c) atomicMax(&s.best[x0], __float_as_uint(s0) + 1u);
            if (TWO && lane + 32 < c) atomicMax(&s.best[x1], __float_as_uint(s1) + 1u);
            const double inner = row_mass(s0, K, lane);
            if (lane == 0) s.rmass[rr] = inner;
        }
        __syncthreads();
        if (tid < E) {
            unsigned long long m = s.mask[tid];
            while (m) {
                const int rr = __ffsll((long long)m) - 1;
                const double wv = (double)s.wgt[tid][rr];
                summed = tok ? __dadd_rn(summed, wv) : wv;
                tok++;
                m &= m - 1;
            }
            s.mask[tid] = 0ull;
        }
        if (tid == 0)
            for (int rr = 0; rr < cn; rr++) outer.add(s.rmass[rr]);
        __syncthreads();
    }
    // predictions for this event as a target: sort (-score, expert)
    if (tid < E) {
        const unsigned ke = s.best[tid];
        if (ke) {
            int pos = 0;
            for (int j = 0; j < E; j++) {
                const unsigned kj = s.best[j];
                pos += (kj > ke) || (kj == ke && j < tid);
            }
            a.out.pred_expert[eb + pos] = tid;
            a.out.pred_score[eb + pos] = __uint_as_float(ke - 1u);
            atomicAdd(&s.cnt[0], 1);
            atomicAdd(&s.pm, pe_mix_term(pos, tid));
        }
        // demand list sorted (rank, -gate, expert)  engine.py:578-594
        const int rk = s.rank[tid];
        if (rk != 0x7fffffff) {
            const unsigned g = s.gate[tid];
            int pos = 0;
            for (int j = 0; j < E; j++) {
                const int rj = s.rank[j];
                if (rj == 0x7fffffff || j == tid) continue;
                const unsigned gj = s.gate[j];
                pos += (rj < rk) || (rj == rk && (gj > g || (gj == g && j < tid)));
            }
            a.out.dem_expert[eb + pos] = tid;
            a.out.dem_rank[eb + pos] = rk;
            a.out.dem_gate[eb + pos] = __uint_as_float(g);
            a.out.dem_summed[eb + pos] = summed;
            a.out.dem_tokens[eb + pos] = tok;
            atomicAdd(&s.cnt[1], 1);
        }
    }
    __syncthreads();
    if (tid == 0) {
        const double origm = outer.value();
        const int clamped = (a.pred_mode == ESIM_PF_TOPK) ? a.pred_clamped : 0;
        a.out.sel_mass[ev] = origm;
        a.out.n_pred[ev] = s.cnt[0];
        a.out.n_dem[ev] = s.cnt[1];
        a.out.pred_clamped[ev] = clamped;
        write_event_mixes(a.out, ev, a.tr.num_layers, T, s.cnt[0], s.pm, origm, clamped);
    }
}

// ---------------------------------------------------------------------------
// One router launch over many traces (also the single-trace path):
//   classify_kernel: events that are not (one row, E <= 64) -> a work list;
//   router_persistent_kernel: one CTA per SM slot pulls multi-row events from
//   the list first (the long ones), then chunks of 64 single-row events (one
//   warp each), both through global work counters.
// ---------------------------------------------------------------------------
struct RouterBatchArgs {
    const EsimTraceDesc* traces;
    const EsimRouterOut* outs;
    const int32_t* params;        // [n][4]: pred_mode, pred_count, pred_clamped, pct_rank
    const int64_t* prefix;        // [n+1] event prefix sums
    int n;
    int64_t total;
    int64_t* multi;               // [total] work list
    int* ctl;                     // [0] n_multi, [1] next multi, [2] next single chunk
};

__device__ __forceinline__ int trace_of(const int64_t* prefix, int n, int64_t g) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {                       // last t with prefix[t] <= g
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ RouterArgs router_args(const RouterBatchArgs& b, int t) {
    RouterArgs a;
    a.tr = b.traces[t];
    a.out = b.outs[t];
    a.pred_mode = b.params[t * 4 + 0];
    a.pred_count = b.params[t * 4 + 1];
    a.pred_clamped = b.params[t * 4 + 2];
    a.pct_rank = b.params[t * 4 + 3];
    return a;
}

__global__ void __launch_bounds__(256) classify_kernel(RouterBatchArgs b) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= b.total) return;
    const int t = trace_of(b.prefix, b.n, g);
    const EsimTraceDesc& tr = b.traces[t];
    const int64_t ev = g - b.prefix[t];
    const int64_t T = tr.row_offset[ev + 1] - tr.row_offset[ev];
    if (!(T == 1 && tr.experts <= 64)) b.multi[atomicAdd(&b.ctl[0], 1)] = g;
}

__global__ void __launch_bounds__(kRouterWarps * 32, 3) router_persistent_kernel(RouterBatchArgs b) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int64_t s_item;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_multi = *(volatile int*)&b.ctl[0];
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(&b.ctl[1], 1);
        __syncthreads();
        const int64_t m = s_item;
        __syncthreads();
        if (m >= n_multi) break;
        const int64_t g = b.multi[m];
        const int t = trace_of(b.prefix, b.n, g);
        const RouterArgs a = router_args(b, t);
        const int64_t ev = g - b.prefix[t];
        const int E = a.tr.experts;
        if (E <= 8) route_multi64_cta<8>(a, ev, smem);
        else if (E <= 16) route_multi64_cta<16>(a, ev, smem);
        else if (E <= 32) route_multi64_cta<32>(a, ev, smem);
        else if (E <= 64) route_multi64_cta<64>(a, ev, smem);
        else route_event_cta_generic(a, ev, smem);
        __syncthreads();
    }
    float* buf = reinterpret_cast<float*>(smem) + warp * 64;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd((unsigned long long*)&b.ctl[4], 64ull);
        __syncthreads();
        const int64_t base = s_item;
        __syncthreads();
        if (base >= b.total) break;
        const int64_t end = base + 64 < b.total ? base + 64 : b.total;
        int t = trace_of(b.prefix, b.n, base + warp);    // a chunk rarely straddles traces
        int64_t t_lo = b.prefix[t], t_hi = b.prefix[t + 1];
        RouterArgs a = router_args(b, t);
        for (int64_t g = base + warp; g < end; g += kRouterWarps) {
            if (g >= t_hi) {
                t = trace_of(b.prefix, b.n, g);
                t_lo = b.prefix[t];
                t_hi = b.prefix[t + 1];
                a = router_args(b, t);
            }
            const int64_t ev = g - t_lo;
            if (a.tr.experts > 64 || a.tr.row_offset[ev + 1] - a.tr.row_offset[ev] != 1) continue;
            const int E = a.tr.experts;
            if (E <= 8) route_single_warp<8>(a, ev, buf, lane);
            else if (E <= 16) route_single_warp<16>(a, ev, buf, lane);
            else if (E <= 32) route_single_warp<32>(a, ev, buf, lane);
            else route_single_warp<64>(a, ev, buf, lane);
        }
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
    if (g_pysum_plain) {}                                        // CPython < 3.12: no compensation
    else if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
    f = t;
}

// one CTA per trace: per-event terms in parallel (chunks of 256 events),
// integer totals by shared atomics, the Neumaier sums (not associative)
// folded in event order by one thread with the three chains interleaved
__global__ void __launch_bounds__(256) route_totals_kernel(SumArgs a) {
    __shared__ double s_orig[256], s_pr[256], s_rc[256];
    __shared__ int s_flags[256];
    __shared__ unsigned long long s_int[8];
    const int t = blockIdx.x, tid = threadIdx.x;
    const EsimTraceDesc& tr = a.traces ? a.traces[t] : a.tr1;
    const EsimRouterOut& o = a.traces ? a.outs[t] : a.out1;
    const int mode = a.traces ? a.params[4 * t] : a.mode1;
    const int E = tr.experts, L = tr.num_layers;
    const int64_t ne = tr.n_events;
    const bool pf = mode != ESIM_PF_NONE;
    if (tid < 8) s_int[tid] = 0ull;
    long long acc[8] = {};             // integer totals of this thread's events (reduced at the end)
    double orig_f = 0.0, orig_c = 0.0, prec_f = 0.0, prec_c = 0.0, rec_f = 0.0, rec_c = 0.0;
    __syncthreads();
    for (int64_t base = 0; base < ne; base += 256) {
        const int64_t ev = base + tid;
        if (ev < ne) {
            const int T = (int)(tr.row_offset[ev + 1] - tr.row_offset[ev]);
            acc[7] += T;
            s_orig[tid] = o.sel_mass[ev];
            int flags = 0;
            if (pf && ev % L >= 1) {
                const int np = o.n_pred[ev], nd = o.n_dem[ev];
                const int32_t* de = o.dem_expert + ev * E;
                const int32_t* pe = o.pred_expert + ev * E;
                int inter = 0;
                if (E <= 64) {
                    unsigned long long dm = 0ull;
                    for (int i = 0; i < nd; i++) dm |= 1ull << de[i];
                    for (int j = 0; j < np; j++) inter += (int)((dm >> pe[j]) & 1ull);
                } else {
                    unsigned long long dm[ESIM_MAX_E / 64] = {};
                    for (int i = 0; i < nd; i++) { const int e = de[i]; dm[e >> 6] |= 1ull << (e & 63); }
                    for (int j = 0; j < np; j++) { const int e = pe[j]; inter += (int)((dm[e >> 6] >> (e & 63)) & 1ull); }
                }
                flags = 1 | (np ? 2 : 0);
                if (np) s_pr[tid] = __ddiv_rn((double)inter, (double)np);
                s_rc[tid] = __ddiv_rn((double)inter, (double)nd);
                acc[0] += inter;
                acc[1] += np;
                acc[2] += nd;
                acc[3] += 1;
                acc[4] += np ? 1 : 0;
                acc[5] += np ? 0 : 1;
            }
            s_flags[tid] = flags;
        }
        __syncthreads();
        // warp w < 3 folds chain w; a skipped term adds +0.0, an exact no-op
        // on these non-negative sums (f + 0 = f, compensation term 0)
        if ((tid & 31) == 0 && tid < 96) {
            const int w = tid >> 5;
            const int cnt = ne - base < 256 ? (int)(ne - base) : 256;
            const double* src = w == 0 ? s_orig : (w == 1 ? s_pr : s_rc);
            const int need = w == 0 ? 0 : (w == 1 ? 2 : 1);
            double f = w == 0 ? orig_f : (w == 1 ? prec_f : rec_f);
            double c = w == 0 ? orig_c : (w == 1 ? prec_c : rec_c);
#pragma unroll 8
            for (int k = 0; k < cnt; k++) {
                const double x = (need == 0 || (s_flags[k] & need)) ? src[k] : 0.0;
                const double t = __dadd_rn(f, x);
                const double e = g_pysum_plain ? 0.0
                                 : fabs(f) >= fabs(x) ? __dadd_rn(__dsub_rn(f, t), x) : __dadd_rn(__dsub_rn(x, t), f);
                c = __dadd_rn(c, e);
                f = t;
            }
            if (w == 0) { orig_f = f; orig_c = c; }
            else if (w == 1) { prec_f = f; prec_c = c; }
            else { rec_f = f; rec_c = c; }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        long long v = acc[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((tid & 31) == 0) atomicAdd(&s_int[i], (unsigned long long)v);
    }
    __shared__ double s_fc[6];
    if (tid == 32) { s_fc[2] = prec_f; s_fc[3] = prec_c; }
    if (tid == 64) { s_fc[4] = rec_f; s_fc[5] = rec_c; }
    __syncthreads();
    if (tid == 0) {
        prec_f = s_fc[2]; prec_c = s_fc[3]; rec_f = s_fc[4]; rec_c = s_fc[5];
        EsimRouteSummary s;
        s.pf_tp = (int64_t)s_int[0]; s.pf_pred = (int64_t)s_int[1]; s.pf_dem = (int64_t)s_int[2];
        s.pf_records = (int64_t)s_int[3]; s.pf_prec_parts = (int64_t)s_int[4]; s.pf_empty = (int64_t)s_int[5];
        s.pf_rec_parts = (int64_t)s_int[3];
        s.rows_total = (int64_t)s_int[7];
        s.orig_f = orig_f; s.orig_c = orig_c; s.prec_f = prec_f; s.prec_c = prec_c; s.rec_f = rec_f; s.rec_c = rec_c;
        *o.summary = s;
    }
    // per target layer (>= 1): predicted-set sizes and prediction events
    const int passes = tr.n_passes;
    for (int l = tid; l < L; l += blockDim.x) {
        int64_t n = 0, c = 0;
        if (pf && l >= 1)
            for (int p = 0; p < passes; p++) { n += o.n_pred[(int64_t)p * L + l]; c++; }
        o.layer_pred[2 * l] = n;
        o.layer_pred[2 * l + 1] = c;
    }
}

// with_events: recompute the per-event digest words (the router kernels
// write them themselves; esim_route_summary_launch needs them after the
// predictions were replaced)
cudaError_t route_summary(const SumArgs& a, int n_traces, int64_t total_events, cudaStream_t st, bool with_events) {
    if (total_events <= 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((total_events * 32 + 255) / 256);
    if (with_events) route_events_kernel<<<blocks, 256, 0, st>>>(a, total_events);
    route_totals_kernel<<<n_traces, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace esim

static size_t router_smem(int max_e) {
    const size_t generic = (size_t)(esim::kRouterWarps * max_e + max_e) * 4 + 16;
    return generic > sizeof(esim::Multi64Smem) ? generic : sizeof(esim::Multi64Smem);
}

// Router work-list scratch: one grow-only device buffer per stream (launches
// on one stream are ordered, so they can share it; other streams get their own)
static cudaError_t stream_scratch(cudaStream_t st, size_t bytes, void** out) {
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, std::pair<void*, size_t>> bufs;
    std::lock_guard<std::mutex> lock(mu);
    auto& b = bufs[st];
    if (b.second < bytes) {
        if (b.first) {
            cudaStreamSynchronize(st);
            cudaFree(b.first);
            b = {nullptr, 0};
        }
        const size_t cap = bytes + bytes / 4;
        cudaError_t e = cudaMalloc(&b.first, cap);
        if (e != cudaSuccess) return e;
        b.second = cap;
    }
    *out = b.first;
    return cudaSuccess;
}

// classify + persistent router + summary over device arrays of traces/outputs
static cudaError_t router_batch(const EsimTraceDesc* d_traces, const EsimRouterOut* d_outs, const int32_t* d_params,
                                const int64_t* d_prefix, int n_traces, int64_t total_events, int max_e,
                                cudaStream_t st) {
    if (total_events <= 0) return cudaSuccess;
    static int grid = 0;
    const size_t smem = router_smem(max_e > 64 ? max_e : 64);
    cudaError_t e = cudaFuncSetAttribute(esim::router_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (!grid) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, esim::router_persistent_kernel, esim::kRouterWarps * 32,
                                                      router_smem(ESIM_MAX_E));
        grid = sms * (per > 0 ? per : 1);
    }
    int64_t* scratch = nullptr;                 // ctl[8] (32 B) + work list
    if ((e = stream_scratch(st, 32 + (size_t)total_events * 8, (void**)&scratch)) != cudaSuccess) return e;
    int* ctl = reinterpret_cast<int*>(scratch);
    cudaMemsetAsync(ctl, 0, 32, st);
    esim::RouterBatchArgs b{d_traces, d_outs, d_params, d_prefix, n_traces, total_events, scratch + 4, ctl};
    esim::classify_kernel<<<(unsigned)((total_events + 255) / 256), 256, 0, st>>>(b);
    const int64_t want = (total_events + 63) / 64;
    esim::router_persistent_kernel<<<(unsigned)(want < grid ? want : grid), esim::kRouterWarps * 32, smem, st>>>(b);
    esim::SumArgs s{};
    s.traces = d_traces; s.outs = d_outs; s.params = d_params; s.prefix = d_prefix; s.n = n_traces;
    return esim::route_summary(s, n_traces, total_events, st, false);
}

extern "C" int esim_router_launch_batch(const EsimTraceDesc* d_traces, const EsimRouterOut* d_outs,
                                        const int32_t* d_params, const int64_t* d_prefix, int32_t n_traces,
                                        int64_t total_events, int32_t max_experts, void* stream) {
    if (total_events <= 0) return 0;
    return router_batch(d_traces, d_outs, d_params, d_prefix, n_traces, total_events, max_experts,
                        (cudaStream_t)stream) == cudaSuccess ? 0 : -3;
}

extern "C" int esim_route_summary_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode,
                                         void* stream) {
    esim::SumArgs s{};
    s.n = 1; s.tr1 = *tr; s.out1 = *out; s.mode1 = pred_mode;
    return esim::route_summary(s, 1, tr->n_events, (cudaStream_t)stream, true) == cudaSuccess ? 0 : -3;
}

// host launcher (declared in capi.cu): one trace through the batch path
cudaError_t esim_router_launch_impl(const EsimTraceDesc& tr, const EsimRouterOut& out, int pred_mode,
                                    int pred_count, int pred_clamped, int pct_rank, cudaStream_t st) {
    if (tr.n_events == 0) return cudaSuccess;
    struct Pack {
        EsimTraceDesc tr;
        EsimRouterOut out;
        int32_t params[4];
        int64_t prefix[2];
    } h{tr, out, {pred_mode, pred_count, pred_clamped, pct_rank}, {0, tr.n_events}};
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, Pack*> packs;   // one per stream, ordered like the launches
    Pack* d = nullptr;
    {
        std::lock_guard<std::mutex> lock(mu);
        Pack*& slot = packs[st];
        if (!slot) {
            cudaError_t e = cudaMalloc((void**)&slot, sizeof(Pack));
            if (e != cudaSuccess) { slot = nullptr; return e; }
        }
        d = slot;
    }
    cudaError_t e = cudaMemcpyAsync(d, &h, sizeof(Pack), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    return router_batch(&d->tr, &d->out, d->params, d->prefix, 1, tr.n_events, tr.experts, st);
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

// the host interpreter's sum() semantics for this translation unit's PySum
// chains (numpy_f32.cuh g_pysum_plain); called by esim_set_host_sum
int esim_router_set_sum_plain(int plain) {
    return cudaMemcpyToSymbol(esim::g_pysum_plain, &plain, sizeof(int)) == cudaSuccess ? 0 : -2;
}
