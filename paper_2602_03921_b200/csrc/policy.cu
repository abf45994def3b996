// policy.cu -- the eviction-policy plug-in objects (eviction.py:29-294) as
// device state + a one-warp op interpreter.
//
// `make_eviction_policy(name, ...)` objects on the host queue their
// begin_pass / note_access / note_admit / note_prefetch_hit calls and flush
// them with each select_victim, which needs an answer. Keys (layer, expert)
// are registered densely by the host; per key the device keeps the same
// flat state the replay kernel uses (stamp / generation+class / count+touch
// / fp64 signal), and every victim choice is a warp argmin with the
// reference's total order and tie-breaks.
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/specmd_b200.h"

namespace esim {
namespace pol {

enum Op : int32_t { OP_BEGIN = 0, OP_ACCESS = 1, OP_ADMIT = 2, OP_PREFETCH_HIT = 3, OP_SELECT = 4 };
constexpr uint8_t F_TRACKED = 1, F_HAS_COUNT = 2, F_HAS_SIGNAL = 4, F_CURRENT = 8;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t min64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(FULL, v, o);
        v = w < v ? w : v;
    }
    return v;
}

__device__ __forceinline__ uint64_t order_double(double d) {
    const uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}

// argmin over tracked keys of (primary, layer, expert) -> key index or -1
template <class F>
__device__ int argmin_keys(const EsimPolicyState& s, int lane, F primary, bool need_current, bool current) {
    uint64_t best_p = ~0ull;
    for (int i = lane; i < s.n_keys; i += 32) {
        const uint8_t f = s.flags[i];
        if (!(f & F_TRACKED)) continue;
        if (need_current && (((f & F_CURRENT) != 0) != current)) continue;
        const uint64_t p = primary(i);
        best_p = p < best_p ? p : best_p;
    }
    best_p = min64(best_p);
    if (best_p == ~0ull) return -1;
    uint64_t best_t = ~0ull;   // tie-break among equal primaries: (layer, expert) then index
    for (int i = lane; i < s.n_keys; i += 32) {
        const uint8_t f = s.flags[i];
        if (!(f & F_TRACKED)) continue;
        if (need_current && (((f & F_CURRENT) != 0) != current)) continue;
        if (primary(i) != best_p) continue;
        const uint64_t t = ((uint64_t)(uint32_t)s.layer[i] << 40) | ((uint64_t)(uint32_t)s.expert[i] << 20) | (uint64_t)i;
        best_t = t < best_t ? t : best_t;
    }
    best_t = min64(best_t);
    return (int)(best_t & 0xFFFFF);
}

__global__ void policy_kernel(EsimPolicyState s, const EsimPolicyOp* __restrict__ ops, int n_ops,
                              int32_t* __restrict__ results) {
    const int lane = threadIdx.x & 31;
    int64_t seq = s.seq[0];
    int nres = 0;
    for (int k = 0; k < n_ops; k++) {
        const EsimPolicyOp op = ops[k];
        const int i = op.key;
        if (op.op == OP_BEGIN) {
            if (s.policy == ESIM_EV_SB) {
                for (int j = lane; j < s.n_keys; j += 32)
                    if (s.flags[j] & F_HAS_SIGNAL) s.signal[j] = __dmul_rn(s.signal[j], s.decay);
            } else if (s.policy == ESIM_EV_LS) {
                for (int j = lane; j < s.n_keys; j += 32) s.flags[j] &= (uint8_t)~F_CURRENT;
            }
        } else if (op.op == OP_SELECT) {
            int v = -1;
            switch (s.policy) {
            case ESIM_EV_LRU:
                v = argmin_keys(s, lane, [&](int j) { return (uint64_t)s.key[j]; }, false, false);
                break;
            case ESIM_EV_LFU: case ESIM_EV_LHU:
                v = argmin_keys(s, lane, [&](int j) {
                    const uint64_t c = (s.flags[j] & F_HAS_COUNT) ? (uint64_t)(uint32_t)s.count[j] : 0;
                    return (c << 40) | (uint64_t)s.key[j];
                }, false, false);
                break;
            case ESIM_EV_FLD: {
                const int c = op.layer, L = s.num_layers;
                v = argmin_keys(s, lane, [&](int j) {
                    int d = (s.layer[j] - c) % L;
                    d = d < 0 ? d + L : d;
                    return ((uint64_t)(L - 1 - d) << 32) | (uint64_t)(uint32_t)s.expert[j];
                }, false, false);
                break;
            }
            case ESIM_EV_SB:
                v = argmin_keys(s, lane, [&](int j) {
                    return order_double((s.flags[j] & F_HAS_SIGNAL) ? s.signal[j] : 0.0);
                }, false, false);
                if (v >= 0 && lane == 0) { s.flags[v] &= (uint8_t)~F_HAS_SIGNAL; s.signal[v] = 0.0; }
                break;
            case ESIM_EV_LS:
                v = argmin_keys(s, lane, [&](int j) { return (uint64_t)s.key[j]; }, true, false);     // stale
                if (v < 0) {
                    if (!op.forced) {
                        if (lane == 0) s.counters[1]++;                                          // refusals
                    } else {
                        v = argmin_keys(s, lane, [&](int j) { return (uint64_t)s.key[j]; }, true, true);
                        if (v >= 0 && lane == 0) s.counters[0]++;                                // forced current
                    }
                }
                break;
            }
            if (v >= 0 && lane == 0) s.flags[v] &= (uint8_t)~(F_TRACKED | F_CURRENT);
            if (lane == 0) results[nres] = v;
            nres++;
        } else {
            // note_access / note_admit / note_prefetch_hit on key i
            if (lane == 0) {
                uint8_t f = s.flags[i];
                switch (s.policy) {
                case ESIM_EV_LRU:
                    if (op.op != OP_PREFETCH_HIT) { f |= F_TRACKED; s.key[i] = seq++; }
                    break;
                case ESIM_EV_LFU: case ESIM_EV_LHU:
                    if (op.op == OP_ACCESS) {
                        const int step = (s.policy == ESIM_EV_LFU || op.prec == s.highest_prec) ? 1 : 0;
                        s.count[i] = ((f & F_HAS_COUNT) ? s.count[i] : 0) + step;
                        f |= F_HAS_COUNT;
                        s.key[i] = seq++;
                    } else if (op.op == OP_ADMIT) {
                        f |= F_TRACKED;
                        if (!(f & F_HAS_COUNT)) { f |= F_HAS_COUNT; s.count[i] = 0; }
                        s.key[i] = seq++;
                    }
                    break;
                case ESIM_EV_FLD:
                    if (op.op != OP_PREFETCH_HIT) f |= F_TRACKED;
                    break;
                case ESIM_EV_SB:
                    if (op.op == OP_ACCESS) {
                        if (!isnan(op.gate)) s.signal[i] = __dadd_rn((f & F_HAS_SIGNAL) ? s.signal[i] : 0.0, op.gate);
                        else if (!(f & F_HAS_SIGNAL)) s.signal[i] = 0.0;
                        f |= F_HAS_SIGNAL;
                    } else if (op.op == OP_ADMIT) {
                        f |= F_TRACKED;
                        if (!(f & F_HAS_SIGNAL)) { f |= F_HAS_SIGNAL; s.signal[i] = 0.0; }
                    }
                    break;
                case ESIM_EV_LS:                                   // _touch: first touch of the pass fixes it
                    if (!((f & F_TRACKED) && (f & F_CURRENT))) {
                        f |= F_TRACKED | F_CURRENT;
                        s.key[i] = seq++;
                    }
                    break;
                }
                s.flags[i] = f;
            }
            seq = __shfl_sync(FULL, seq, 0);
        }
        __syncwarp();
    }
    if (lane == 0) s.seq[0] = seq;
}

}  // namespace pol
}  // namespace esim

extern "C" int esim_policy_apply(const EsimPolicyState* state, const EsimPolicyOp* d_ops, int32_t n_ops,
                                 int32_t* d_results, void* stream) {
    if (n_ops <= 0) return 0;
    esim::pol::policy_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*state, d_ops, n_ops, d_results);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---------------------------------------------------------------------------
// miss-handler plug-in decision (miss.py:66-140): one warp over the layer's
// demanded gate scores and the layer's residents. The fetch itself (making
// space, the transfer, blocking) belongs to the caller's fetch_fn.
// ---------------------------------------------------------------------------
namespace esim {
namespace pol {

__global__ void miss_decide_kernel(EsimMissQuery q, const double* __restrict__ scores,
                                   const int32_t* __restrict__ res_expert, const double* __restrict__ res_rec,
                                   EsimMissDecision* out) {
    const int lane = threadIdx.x;
    EsimMissDecision d{ESIM_MISS_OUT_FETCH, -1, ESIM_MISS_FETCH_WORKING, 0};
    if (q.policy == ESIM_MISS_DROP && q.rank > q.drop_rank_threshold) {
        d.kind = ESIM_MISS_OUT_DROP;                                   // miss.py:109-110
    } else {
        bool decided = false;
        if (q.policy == ESIM_MISS_SUBST) {
            // find_substitute (miss.py:66-79): min (|rec - gate|, expert) within tolerance
            // two passes: min diff, then min expert among equal diffs
            double bd = INFINITY;
            for (int i = lane; i < q.n_residents; i += 32) {
                const double diff = fabs(__dsub_rn(res_rec[i], q.gate_score));
                if (diff <= q.subst_tolerance && diff < bd) bd = diff;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bd = fmin(bd, __shfl_xor_sync(FULL, bd, o));
            int be = INT32_MAX;
            if (bd != INFINITY)
                for (int i = lane; i < q.n_residents; i += 32)
                    if (fabs(__dsub_rn(res_rec[i], q.gate_score)) == bd && res_expert[i] < be) be = res_expert[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) be = min(be, __shfl_xor_sync(FULL, be, o));
            if (bd != INFINITY) { d.kind = ESIM_MISS_OUT_SUBST; d.substitute = be; decided = true; }
        }
        if (!decided) {
            if (q.policy == ESIM_MISS_FETCH_LOW) {
                d.fetch = ESIM_MISS_FETCH_LOWEST;                       // miss.py:116-118
            } else if (q.policy == ESIM_MISS_FETCH_PRIORITY) {
                d.fetch = ESIM_MISS_FETCH_CASCADE;                      // miss.py:120-136
                if (q.ladder_len > 1 && q.n_scores > 0) {
                    // nearest-rank percentile (prefetch.py:30-36): the value whose
                    // ascending position holds rank - 1
                    double thr = 0.0;
                    bool found = false;
                    for (int i = lane; i < q.n_scores; i += 32) {
                        int lt = 0, le = 0;
                        for (int j = 0; j < q.n_scores; j++) {
                            lt += scores[j] < scores[i];
                            le += scores[j] <= scores[i];
                        }
                        if (lt <= q.pct_rank - 1 && q.pct_rank - 1 < le) { thr = scores[i]; found = true; }
                    }
                    const unsigned m = __ballot_sync(FULL, found);
                    thr = __shfl_sync(FULL, thr, __ffs(m) - 1);
                    if (q.gate_score < thr) d.start = 1;                // low-importance: one level lower
                }
            }
        }
    }
    if (lane == 0) *out = d;
}

}  // namespace pol
}  // namespace esim

extern "C" int esim_miss_decide(const EsimMissQuery* q, const double* h_scores, const int32_t* h_res_expert,
                                const double* h_res_rec, EsimMissDecision* decision) {
    if (!q || !decision || q->n_scores < 0 || q->n_residents < 0) return -1;
    const size_t ns = (size_t)q->n_scores, nr = (size_t)q->n_residents;
    char* d = nullptr;
    const size_t bytes = 8 * ns + 4 * nr + 8 * nr + sizeof(EsimMissDecision) + 64;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return -2;
    double* ds = (double*)d;
    double* dr = ds + ns;
    int32_t* de = (int32_t*)(dr + nr);
    EsimMissDecision* dd = (EsimMissDecision*)(((uintptr_t)(de + nr) + 15) & ~(uintptr_t)15);
    cudaError_t e = cudaSuccess;
    if (ns) e = cudaMemcpy(ds, h_scores, 8 * ns, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nr) e = cudaMemcpy(dr, h_res_rec, 8 * nr, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nr) e = cudaMemcpy(de, h_res_expert, 4 * nr, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        esim::pol::miss_decide_kernel<<<1, 32>>>(*q, ds, de, dr, dd);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(decision, dd, sizeof(EsimMissDecision), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : -2;
}
