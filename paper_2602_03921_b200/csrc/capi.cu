// capi.cu -- extern "C" entry points of libspecmd_b200.so (include/specmd_b200.h).
//
// Thin: argument checks, launch geometry, error translation. Errors are
// reported as negative return codes plus a thread-local message
// (esim_last_error), which the Python host re-raises as the reference's
// ConfigError / RuntimeError (models.py:31, engine.py:216-236).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/specmd_b200.h"

cudaError_t esim_router_launch_impl(const EsimTraceDesc& tr, const EsimRouterOut& out, int pred_mode,
                                    int pred_count, int pred_clamped, int pct_rank, cudaStream_t st);
cudaError_t esim_replay_launch_impl(const EsimConfig* d_cfg, int n, const EsimTraceDesc* d_traces,
                                    const EsimRouterOut* d_routers, EsimCounters* d_counters,
                                    int64_t* d_per_layer, EsimRec* d_recs, int64_t rec_cap, int32_t* d_pexp,
                                    int64_t pe_cap, int N, int S, int Q, int Lmax, int Emax, int Tmax, int Kmax,
                                    bool has_cnt, int warps_per_cta, cudaStream_t st);
int esim_replay_smem_bytes(int N, int S, int Q, int L, int E, int T, int K, bool ca, bool has_cnt);

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
    return fail(-3, std::string(where) + ": " + cudaGetErrorString(e));
}

extern "C" const char* esim_last_error(void) { return g_err.c_str(); }
extern "C" int esim_version(void) { return 1; }

// predictor constants resolved on the host exactly as the reference does in
// Python floats: count = ceil(k * overfetch) (prefetch.py:48), rank =
// max(1, ceil(p / 100 * E)) (prefetch.py:35)
static void predictor_consts(int k, int E, double overfetch, double percentile, int* count, int* clamped,
                             int* rank) {
    double c = std::ceil((double)k * overfetch);
    *clamped = c > (double)E;
    *count = (int)std::min<double>(c, (double)E);
    long r = (long)std::ceil(percentile / 100.0 * (double)E);
    *rank = (int)std::max<long>(1, r);
}

extern "C" int esim_router_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode,
                                  double overfetch, double percentile, void* stream) {
    if (!tr || !out) return fail(-1, "null argument");
    if (tr->experts < 1 || tr->experts > ESIM_MAX_E) return fail(-1, "experts out of range for the device router");
    if (tr->top_k < 1 || tr->top_k > ESIM_MAX_K || tr->top_k > tr->experts) return fail(-1, "top_k out of range");
    int count, clamped, rank;
    predictor_consts(tr->top_k, tr->experts, overfetch, percentile, &count, &clamped, &rank);
    cudaError_t e = esim_router_launch_impl(*tr, *out, pred_mode, count, clamped, rank, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "router launch");
    return 0;
}

struct Sizing { int N, S, Q, Lmax, Emax, Tmax, Kmax; bool ca, has_cnt; };

// queue_cap 0 = default ring size (64 entries, overflow -> status -5 and the
// caller re-launches with the exact bound queue_cap = -1: slots + 1)
static int replay_sizing(const EsimConfig* h, int n, int max_tokens, int pl_stride, int queue_cap, Sizing* z) {
    Sizing s{0, 1, 2, 0, 0, 0, 0, false, false};
    for (int i = 0; i < n; i++) {
        const EsimConfig& c = h[i];
        if (c.experts > ESIM_MAX_E || c.top_k > ESIM_MAX_K) return fail(-1, "geometry exceeds device limits");
        int N = c.num_layers * c.experts;
        if (N > 32767) return fail(-1, "num_layers * experts must be < 32768 on the device directory");
        int64_t minb = INT64_MAX;
        for (int p = 0; p < 4; p++)
            if (c.expert_bytes[p] > 0) minb = std::min(minb, c.expert_bytes[p]);
        if (minb == INT64_MAX) return fail(-1, "no precision available");
        int64_t slots = std::min<int64_t>(c.capacity_bytes / minb, N);
        s.N = std::max(s.N, N);
        s.S = std::max<int>(s.S, (int)std::max<int64_t>(slots, 1));
        s.Lmax = std::max(s.Lmax, c.num_layers);
        s.Emax = std::max(s.Emax, c.experts);
        s.Kmax = std::max(s.Kmax, c.top_k);
        if (c.routing == ESIM_ROUTE_CACHE_AWARE) s.ca = true;
        if (c.eviction == ESIM_EV_LFU || c.eviction == ESIM_EV_LHU) s.has_cnt = true;
    }
    if (s.S > 4095) return fail(-1, "more than 4095 resident experts per cache is not supported by the device directory");
    s.Q = queue_cap > 0 ? std::min(queue_cap, s.S + 1) : queue_cap < 0 ? s.S + 1 : std::min(64, s.S + 1);
    s.Tmax = s.ca ? std::max(1, max_tokens) : 0;
    if (pl_stride < s.Lmax) return fail(-1, "per-layer stride smaller than num_layers");
    s.Lmax = pl_stride;
    *z = s;
    return 0;
}

extern "C" int esim_replay_smem_per_point(const EsimConfig* h_cfg, int32_t n, int32_t max_tokens,
                                          int32_t pl_stride, int32_t queue_cap) {
    Sizing z;
    int rc = replay_sizing(h_cfg, n, max_tokens, pl_stride, queue_cap, &z);
    if (rc) return rc;
    return esim_replay_smem_bytes(z.N, z.S, z.Q, z.Lmax, z.Emax, z.Tmax, z.Kmax, z.ca, z.has_cnt);
}

extern "C" int esim_replay_launch(const EsimConfig* h_cfg, const EsimConfig* d_cfg, int32_t n,
                                  const EsimTraceDesc* d_traces, const EsimRouterOut* d_routers, int32_t max_tokens,
                                  EsimCounters* d_counters, int64_t* d_per_layer, int32_t pl_stride,
                                  EsimRec* d_recs, int64_t rec_cap, int32_t* d_pexp, int64_t pe_cap,
                                  int32_t warps_per_cta, int32_t queue_cap, void* stream) {
    if (n <= 0) return 0;
    Sizing z;
    int rc = replay_sizing(h_cfg, n, max_tokens, pl_stride, queue_cap, &z);
    if (rc) return rc;
    int per = esim_replay_smem_bytes(z.N, z.S, z.Q, z.Lmax, z.Emax, z.Tmax, z.Kmax, z.ca, z.has_cnt);
    const int budget = 227 * 1024;
    int w = warps_per_cta > 0 ? warps_per_cta : 4;
    while (w > 1 && per * w > budget) w--;
    if (per * w > budget) return fail(-1, "replay state of one grid point exceeds shared memory (" +
                                              std::to_string(per) + " B)");
    cudaError_t e = esim_replay_launch_impl(d_cfg, n, d_traces, d_routers, d_counters, d_per_layer, d_recs, rec_cap,
                                            d_pexp, pe_cap, z.N, z.S, z.Q, z.Lmax, z.Emax, z.Tmax, z.Kmax, z.has_cnt,
                                            w, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "replay launch");
    return 0;
}

// ---------------------------------------------------------------------------
// end-to-end host API: host buffers in, host results out
// ---------------------------------------------------------------------------
namespace {
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) cap = n;
        return e;
    }
};

struct HostCtx {
    cudaStream_t st = nullptr;
    std::vector<DevBuf> bufs;
};

HostCtx& ctx() {
    static HostCtx c;
    return c;
}
}  // namespace

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

extern "C" int esim_run_host(const EsimConfig* cfg, int32_t n, const EsimTraceDesc* traces, int32_t n_traces,
                             EsimCounters* counters, int64_t* per_layer, int32_t pl_stride, EsimRec* recs,
                             int64_t rec_cap, int32_t* pred_experts, int64_t pe_cap) {
    HostCtx& C = ctx();
    cudaError_t e;
    if (!C.st) {
        e = cudaStreamCreateWithFlags(&C.st, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e, "stream");
    }
    // predictor params per trace: taken from the first config that uses it
    std::vector<int> pmode(n_traces, 0);
    std::vector<double> pover(n_traces, 1.0), ppct(n_traces, 80.0);
    std::vector<char> seen(n_traces, 0);
    for (int i = 0; i < n; i++) {
        int t = cfg[i].trace_id;
        if (t < 0 || t >= n_traces) return fail(-1, "trace_id out of range");
        if (!seen[t]) { seen[t] = 1; pmode[t] = cfg[i].prefetch; pover[t] = cfg[i].overfetch; ppct[t] = cfg[i].percentile; }
        else if (pmode[t] != cfg[i].prefetch || pover[t] != cfg[i].overfetch || ppct[t] != cfg[i].percentile)
            return fail(-1, "configs sharing a trace_id must share the predictor");
    }
    // one device slab: traces, router outputs, configs, outputs
    size_t total = 0;
    std::vector<size_t> toff(n_traces), roff(n_traces);
    int max_tokens = 0;
    for (int t = 0; t < n_traces; t++) {
        const EsimTraceDesc& d = traces[t];
        int64_t ne = d.n_events, nr = d.n_rows_total, E = d.experts, K = d.top_k;
        toff[t] = total;
        total += al256(d.n_passes * 4) * 2 + al256((ne + 1) * 8) + al256(nr * E * 4);
        roff[t] = total;
        total += al256(ne * 4) * 3 + al256(ne * E * 4) * 6 + al256(ne * E * 8) + al256(ne * 8) +
                 al256(nr * K * 2) + al256(nr * K * 4) + al256(ne * 4);
        for (int p = 0; p < d.n_passes; p++) max_tokens = std::max(max_tokens, d.pass_tokens[p]);
    }
    size_t cfg_off = total; total += al256(sizeof(EsimConfig) * n);
    size_t td_off = total; total += al256(sizeof(EsimTraceDesc) * n_traces);
    size_t rd_off = total; total += al256(sizeof(EsimRouterOut) * n_traces);
    size_t cnt_off = total; total += al256(sizeof(EsimCounters) * n);
    size_t pl_off = total; total += al256(sizeof(int64_t) * n * pl_stride * ESIM_PL_FIELDS);
    size_t rec_off = total; total += recs ? al256(sizeof(EsimRec) * n * rec_cap) : 0;
    size_t pe_off = total; total += recs ? al256(sizeof(int32_t) * n * pe_cap) : 0;
    if (C.bufs.empty()) C.bufs.resize(1);
    e = C.bufs[0].ensure(total);
    if (e != cudaSuccess) return cuda_fail(e, "device alloc");
    char* base = (char*)C.bufs[0].p;
    std::vector<EsimTraceDesc> dtr(n_traces);
    std::vector<EsimRouterOut> dro(n_traces);
    for (int t = 0; t < n_traces; t++) {
        const EsimTraceDesc& h = traces[t];
        int64_t ne = h.n_events, nr = h.n_rows_total, E = h.experts, K = h.top_k;
        char* q = base + toff[t];
        EsimTraceDesc d = h;
        auto put = [&](const void* src, size_t bytes) -> void* {
            void* dst = q;
            if (bytes) cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, C.st);
            q += al256(bytes);
            return dst;
        };
        d.pass_tokens = (const int32_t*)put(h.pass_tokens, h.n_passes * 4);
        d.pass_kind = (const int32_t*)put(h.pass_kind, h.n_passes * 4);
        d.row_offset = (const int64_t*)put(h.row_offset, (ne + 1) * 8);
        d.logits = (const float*)put(h.logits, nr * E * 4);
        dtr[t] = d;
        char* r = base + roff[t];
        EsimRouterOut o;
        auto take = [&](size_t bytes) -> void* { void* x = r; r += al256(bytes); return x; };
        o.n_dem = (int32_t*)take(ne * 4);
        o.n_pred = (int32_t*)take(ne * 4);
        o.pred_clamped = (int32_t*)take(ne * 4);
        o.dem_expert = (int32_t*)take(ne * E * 4);
        o.dem_rank = (int32_t*)take(ne * E * 4);
        o.dem_gate = (float*)take(ne * E * 4);
        o.dem_tokens = (int32_t*)take(ne * E * 4);
        o.pred_expert = (int32_t*)take(ne * E * 4);
        o.pred_score = (float*)take(ne * E * 4);
        o.dem_summed = (double*)take(ne * E * 8);
        o.sel_mass = (double*)take(ne * 8);
        o.row_sel = (int16_t*)take(nr * K * 2);
        o.row_w = (float*)take(nr * K * 4);
        dro[t] = o;
        int rc = esim_router_launch(&d, &o, pmode[t], pover[t], ppct[t], C.st);
        if (rc) return rc;
    }
    cudaMemcpyAsync(base + cfg_off, cfg, sizeof(EsimConfig) * n, cudaMemcpyHostToDevice, C.st);
    cudaMemcpyAsync(base + td_off, dtr.data(), sizeof(EsimTraceDesc) * n_traces, cudaMemcpyHostToDevice, C.st);
    cudaMemcpyAsync(base + rd_off, dro.data(), sizeof(EsimRouterOut) * n_traces, cudaMemcpyHostToDevice, C.st);
    int rc = esim_replay_launch(cfg, (EsimConfig*)(base + cfg_off), n, (EsimTraceDesc*)(base + td_off),
                                (EsimRouterOut*)(base + rd_off), max_tokens, (EsimCounters*)(base + cnt_off),
                                (int64_t*)(base + pl_off), pl_stride, recs ? (EsimRec*)(base + rec_off) : nullptr,
                                rec_cap, recs ? (int32_t*)(base + pe_off) : nullptr, pe_cap, 0, 0, C.st);
    if (rc) return rc;
    cudaMemcpyAsync(counters, base + cnt_off, sizeof(EsimCounters) * n, cudaMemcpyDeviceToHost, C.st);
    cudaMemcpyAsync(per_layer, base + pl_off, sizeof(int64_t) * n * pl_stride * ESIM_PL_FIELDS,
                    cudaMemcpyDeviceToHost, C.st);
    if (recs) {
        cudaMemcpyAsync(recs, base + rec_off, sizeof(EsimRec) * n * rec_cap, cudaMemcpyDeviceToHost, C.st);
        cudaMemcpyAsync(pred_experts, base + pe_off, sizeof(int32_t) * n * pe_cap, cudaMemcpyDeviceToHost, C.st);
    }
    e = cudaStreamSynchronize(C.st);
    if (e != cudaSuccess) return cuda_fail(e, "esim_run_host");
    bool overflow = false;
    for (int i = 0; i < n; i++) overflow |= counters[i].status == -5;
    if (overflow) {   // channel deeper than the default ring: replay again with the exact bound
        rc = esim_replay_launch(cfg, (EsimConfig*)(base + cfg_off), n, (EsimTraceDesc*)(base + td_off),
                                (EsimRouterOut*)(base + rd_off), max_tokens, (EsimCounters*)(base + cnt_off),
                                (int64_t*)(base + pl_off), pl_stride, recs ? (EsimRec*)(base + rec_off) : nullptr,
                                rec_cap, recs ? (int32_t*)(base + pe_off) : nullptr, pe_cap, 0, -1, C.st);
        if (rc) return rc;
        cudaMemcpyAsync(counters, base + cnt_off, sizeof(EsimCounters) * n, cudaMemcpyDeviceToHost, C.st);
        cudaMemcpyAsync(per_layer, base + pl_off, sizeof(int64_t) * n * pl_stride * ESIM_PL_FIELDS,
                        cudaMemcpyDeviceToHost, C.st);
        if (recs) {
            cudaMemcpyAsync(recs, base + rec_off, sizeof(EsimRec) * n * rec_cap, cudaMemcpyDeviceToHost, C.st);
            cudaMemcpyAsync(pred_experts, base + pe_off, sizeof(int32_t) * n * pe_cap, cudaMemcpyDeviceToHost, C.st);
        }
        e = cudaStreamSynchronize(C.st);
        if (e != cudaSuccess) return cuda_fail(e, "esim_run_host");
    }
    for (int i = 0; i < n; i++)
        if (counters[i].status) {
            int s = (int)counters[i].status;
            return fail(s, s == -4 ? "record buffer too small" : s == -1 ? "config error during replay"
                                                                          : "runtime invariant broken during replay");
        }
    return 0;
}
