/*
 * specmd_b200.h -- C ABI of the B200-native expert-cached MoE layer step.
 *
 * This is the drop-in boundary for the path the reference implements in
 * pure Python (expertsim, /root/reference/pkg/src/expertsim):
 *
 *   reference symbol (file:line)                         replaced by
 *   -----------------------------------------------------------------------
 *   routing.softmax_rows / topk_indices / route_event     esim_router_launch
 *     (routing.py:22-35, 109-161)
 *   engine.Simulation._aggregate_demand (engine.py:578)   esim_router_launch
 *   prefetch.predict_event (prefetch.py:67-107)           esim_router_launch
 *   engine.Simulation.run / _run_layer / _handle_demand   esim_replay_launch
 *     / _fetch / _submit_prefetches / _settle
 *     (engine.py:422-748), eviction.* (eviction.py:29-294),
 *     miss.resolve_miss (miss.py:82-140),
 *     prefetch.watchdog_step (prefetch.py:163-221),
 *     engine.CacheState / Channel (engine.py:188-370),
 *     metrics.classify_miss (metrics.py:46-57)
 *   engine.run_simulation (engine.py:751)                 esim_run_host
 *   (no reference equivalent: the paper's real system)    esim_ffn_* /
 *                                                         esim_layer_step_*
 *
 * Conventions: plain pointers and sizes, no torch types. Functions return
 * 0 on success and a negative code on failure; esim_last_error() returns
 * the thread-local message. Codes: -1 config (ConfigError), -2 runtime
 * invariant (RuntimeError), -3 CUDA error, -4 capacity of an output buffer.
 * Device pointers are marked d_; streams are cudaStream_t passed as void*.
 */
#ifndef SPECMD_B200_H
#define SPECMD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- enums (strings in the reference) -------------------------------- */
enum { ESIM_FP16 = 0, ESIM_INT8 = 1, ESIM_INT4 = 2, ESIM_INT2 = 3 };          /* models.py:21-26 */
enum { ESIM_ROUTE_STANDARD = 0, ESIM_ROUTE_CACHE_AWARE = 1 };                  /* routing.py:16-17 */
enum { ESIM_EV_LRU = 0, ESIM_EV_LFU, ESIM_EV_LHU, ESIM_EV_FLD, ESIM_EV_SB, ESIM_EV_LS }; /* eviction.py:297 */
enum { ESIM_PF_NONE = 0, ESIM_PF_TOPK, ESIM_PF_SCORE, ESIM_PF_ORACLE };        /* prefetch.py:22-27 */
enum { ESIM_MISS_FETCH = 0, ESIM_MISS_FETCH_LOW, ESIM_MISS_FETCH_PRIORITY,
       ESIM_MISS_DROP, ESIM_MISS_SUBST };                                      /* miss.py:18-24 */
enum { ESIM_REC_ACCESS = 1, ESIM_REC_EVICT, ESIM_REC_PREFETCH, ESIM_REC_PREDICTION,
       ESIM_REC_ROUTE, ESIM_REC_PASS };                                        /* metrics.py:62-128 */

#define ESIM_FLAG_FULL_LOG 1   /* emit every EsimRec (else counters + digest only) */
#define ESIM_FLAG_NO_DIGEST 2  /* skip the record-stream digest (counters only) */
#define ESIM_FLAG_TIME32 4     /* caller-proven: the run's simulated clock stays below 2^31 us
                                  (esim_time32_ok); launches whose points all carry it run
                                  the 32-bit-clock replay kernels */
#define ESIM_MAX_E 256         /* experts per layer supported by the device path */
#define ESIM_MAX_K 16

/* One simulation config, resolved to integers/doubles on the host
 * (SimConfig engine.py:82-97 + HardwareSpec models.py:126-145 after
 * resolve_capacity models.py:148-165). */
typedef struct {
    int32_t num_layers, experts, top_k, n_precisions;
    int32_t precisions[4];        /* ladder, largest first (ModelSpec.precisions) */
    int64_t expert_bytes[4];      /* by precision code; 0 = not available */
    int64_t capacity_bytes;       /* resolved capacity */
    int64_t bandwidth;            /* bytes/s; 0 = infinitely fast link */
    int64_t compute_us;           /* per_layer_compute_us */
    int32_t working_prec;
    int32_t routing;
    double  lam;
    int32_t eviction;
    int32_t prefetch;
    double  sb_decay, overfetch, percentile;
    int32_t miss;
    int32_t drop_rank_threshold;
    double  subst_tolerance, degrade_percentile;
    int32_t flags;
    int32_t trace_id;             /* which router/trace buffer set this point replays */
    double  prefetch_noise;       /* SimConfig.prefetch_noise (engine.py:92): prefetch.py:110-136 */
    uint64_t seed;                /* SimConfig.seed (engine.py:97): np.random.default_rng(seed) */
} EsimConfig;                     /* 184 bytes */

/* One event-log record, 64 bytes; field mapping per kind is documented in
 * paper_2602_03921_b200/records.py:decode_records. */
typedef struct {
    int32_t kind, pass_id, layer, i0, i1, i2, i3, i4;
    int64_t t0, t1, t2;
    double  x0;
} EsimRec;

/* Report vector: everything metrics.build_report (metrics.py:190-316)
 * needs, accumulated in log order. Per-layer counters live in a separate
 * [L][ESIM_PL_FIELDS] int64 array. */
typedef struct {
    int64_t totals[15];           /* metrics.TOTAL_FIELDS order */
    int64_t ttft_us, total_us, decode_us, sync_overhead_us, passes, decode_passes;
    int64_t rows_total, faithful_rows, modified_rows;
    int64_t pf_tp, pf_pred_total, pf_dem_total, pf_records, pf_empty, pf_prec_parts, pf_rec_parts;
    int64_t ls_forced, ls_unforced, ls_refusals;
    int64_t n_recs, n_pred_experts;
    uint64_t digest;              /* FNV-1a over the canonical record stream */
    double  original_mass, executed_mass, pf_prec_sum, pf_rec_sum;
    int64_t status;               /* 0 ok, else negative error code */
    int64_t pad[3];
} EsimCounters;                   /* 360 bytes */

#define ESIM_PL_FIELDS 10         /* demanded hits misses compulsory collision capacity dropped substituted pred_size_sum pred_count */

/* Router output for one trace, policy independent under standard routing
 * (SURVEY.md section 7 decision 2). Event ev = pass*L + layer. Buffers are
 * sized by the caller: demands [n_events][E], rows [n_rows_total][K]. */
typedef struct {
    int32_t n_passes, num_layers, experts, top_k;
    int64_t n_events, n_rows_total;
    const int32_t *pass_tokens;   /* [n_passes] */
    const int32_t *pass_kind;     /* [n_passes] 0 prefill 1 decode */
    const int64_t *row_offset;    /* [n_events+1] first token row of each event */
    const float   *logits;        /* [n_rows_total][E] */
} EsimTraceDesc;

typedef struct {
    /* per event demand list, sorted (rank, -gate, expert)  engine.py:578-594 */
    int32_t *n_dem;               /* [n_events] */
    int32_t *dem_expert;          /* [n_events][E] */
    int32_t *dem_rank;            /* [n_events][E] */
    float   *dem_gate;            /* [n_events][E] */
    double  *dem_summed;          /* [n_events][E] */
    int32_t *dem_tokens;          /* [n_events][E] */
    double  *sel_mass;            /* [n_events] sum of sum(weights) in row order */
    /* per row top-k (selected == original under standard routing) */
    int16_t *row_sel;             /* [n_rows_total][K] */
    float   *row_w;               /* [n_rows_total][K] */
    /* per event next-layer prediction when this event is the target (prefetch.py:67-107) */
    int32_t *n_pred;              /* [n_events] */
    int32_t *pred_expert;         /* [n_events][E] */
    float   *pred_score;          /* [n_events][E] */
    int32_t *pred_clamped;        /* [n_events] */
    /* Policy-independent summary (filled by the router launchers, or by
     * esim_route_summary_launch after predictions are replaced): work every
     * grid point sharing this router output would otherwise repeat. */
    uint32_t *route_mix;          /* [n_events] RouteRec digest word (standard routing, no drop/subst) */
    uint32_t *pred_mix;           /* [n_events] digest word of the PredictionRec targeting the event */
    int64_t  *layer_pred;         /* [2*num_layers] per target layer: sum n_pred, prediction events */
    struct EsimRouteSummary *summary;  /* [1] */
} EsimRouterOut;

/* Router-only totals of a trace (metrics.py:150-187 P/R accounting under
 * standard routing; engine.py:625-643 RouteRec masses). Neumaier (f, c)
 * pairs in event order, exactly as the replay accumulates them. */
typedef struct EsimRouteSummary {
    int64_t pf_tp, pf_pred, pf_dem, pf_records, pf_prec_parts, pf_empty, pf_rec_parts;
    int64_t rows_total;
    double  orig_f, orig_c, prec_f, prec_c, rec_f, rec_c;
} EsimRouteSummary;                /* 112 bytes */

const char *esim_last_error(void);
/* Page-lock / release a caller-owned host buffer (trace arrays) so that
 * esim_run_host's host->device copies run as asynchronous DMA. */
int esim_host_register(void *ptr, size_t bytes);
int esim_host_unregister(void *ptr);
int esim_version(void);
/* 1 if a replay of `cfg` over `trace` provably keeps its simulated clock below
 * 2^31 us: trace events x compute_us + (demands + predictions) x the
 * working-precision transfer time, with demands <= min(rows x top_k,
 * events x experts) and predictions <= events x experts. The sweep plan sets
 * ESIM_FLAG_TIME32 itself; a direct esim_replay_launch caller may set it. */
int esim_time32_ok(const EsimConfig *cfg, const EsimTraceDesc *trace);
/* Host-semantics switch: the builtin sum() of the interpreter the device
 * must match (RouteRec masses engine.py:630-631, report sums
 * metrics.py:168-180, 267-270): neumaier = 1 for CPython >= 3.12 (the
 * compensated float path; the default), 0 for CPython <= 3.11 (plain left
 * fold). Process-wide; needs a device context. esim_get_host_sum reads it. */
int esim_set_host_sum(int neumaier);
int esim_get_host_sum(void);

/* Fused router over a whole trace: one CTA per event. `trace` and `out`
 * are host structs holding DEVICE pointers. pred_mode/overfetch/percentile
 * select the next-layer predictor (prefetch.py:67-107). */
int esim_router_launch(const EsimTraceDesc *trace, const EsimRouterOut *out,
                       int32_t pred_mode, double overfetch, double percentile, void *stream);

/* The same over many traces in ONE launch (one CTA per event of every
 * trace). Device arrays: traces[n], outs[n], params[n][4] = {pred_mode,
 * pred_count, pred_clamped, pct_rank} (see esim_predictor_params), prefix[n+1]
 * event prefix sums. */
int esim_router_launch_batch(const EsimTraceDesc *d_traces, const EsimRouterOut *d_outs,
                             const int32_t *d_params, const int64_t *d_prefix, int32_t n_traces,
                             int64_t total_events, int32_t max_experts, void *stream);
/* Host helper: the predictor constants the router uses, computed in double
 * exactly as the reference does (prefetch.py:35, 48). out[4] as above. */
/* Recompute the router summary (route_mix, pred_mix, layer_pred, summary)
 * of one router output after its predictions were replaced (noised
 * prediction streams, prefetch.py:110-160). `trace` / `out` are host structs
 * holding device pointers; pred_mode as for esim_router_launch. */
int esim_route_summary_launch(const EsimTraceDesc *trace, const EsimRouterOut *out, int32_t pred_mode,
                              void *stream);
/* prefetch.apply_prediction_noise (prefetch.py:110-136) over a routed
 * trace's whole prediction stream, in place, drawing from numpy's
 * default_rng(seed) (SeedSequence -> PCG64, restated on the device) in the
 * reference's submission order (engine.py:413, 653-666); then the router
 * summary is recomputed (as esim_route_summary_launch). noise 0 or pred_mode
 * NONE consumes nothing. Host structs holding device pointers. */
int esim_noise_launch(const EsimTraceDesc *trace, const EsimRouterOut *out, int32_t pred_mode, double noise,
                      uint64_t seed, void *stream);
int esim_predictor_params(int32_t top_k, int32_t experts, int32_t pred_mode, double overfetch,
                          double percentile, int32_t *out4);

/* Plug-in kernels behind routing.softmax_rows / topk_indices (routing.py:22-35):
 * one warp per row, numpy-exact. Device pointers. */
int esim_softmax_launch(const float *d_x, int32_t rows, int32_t experts, float *d_out, void *stream);
int esim_topk_launch(const float *d_scores, int32_t rows, int32_t experts, int32_t k, int32_t *d_idx, void *stream);

/* routing.route_event(policy=CACHE_AWARE) for one event (routing.py:143-161):
 * cached_mask bit e = expert e resident at the layer; delta[2] = (sum, count)
 * of the layer's DeltaAvgState, updated in place. Outputs per row: selected
 * and original top-k (int16 [rows][k]) with their original-softmax weights,
 * and the modified flag. Device pointers, one warp. */
int esim_route_cache_aware_launch(const float *d_x, int32_t rows, int32_t experts, int32_t top_k,
                                  const uint32_t *d_cached_mask, double lam, double *d_delta, int16_t *d_sel,
                                  float *d_w, int16_t *d_orig, float *d_ow, int32_t *d_modified, void *stream);

/* Eviction-policy plug-in objects (eviction.py:29-294) on the device.
 * op: 0 begin_pass, 1 note_access, 2 note_admit, 3 note_prefetch_hit,
 * 4 select_victim (result appended to d_results: key index or -1).
 * gate NaN = None; prec = precision code or -1. */
typedef struct {
    int32_t op, key, layer, prec;
    int32_t forced, pad;
    double gate;
} EsimPolicyOp;                    /* 32 bytes */

typedef struct {
    int32_t policy, num_layers, highest_prec, n_keys;
    double decay;
    int64_t *seq;                  /* device [1] */
    int64_t *counters;             /* device [2]: forced_current_evictions, refusals (LS) */
    uint8_t *flags;                /* device [n_keys] */
    int64_t *key;                  /* stamp / generation / touch */
    int32_t *count;                /* LFU / LHU */
    double *signal;                /* SB */
    int32_t *layer, *expert;
} EsimPolicyState;

/* Miss-handler plug-in decision (miss.py:66-140 resolve_miss/find_substitute):
 * policy = ESIM_MISS_* (models MISS_CODE order), rank = the missing expert's
 * 1-based rank by routing weight, scores = the gate scores demanded at this
 * layer event (degrade percentile, fetch_priority), residents = (expert,
 * recorded score) of the layer, pct_rank = max(1, ceil(p/100 * n_scores)).
 * Decision: kind DROP / SUBST (substitute = expert: min (|rec - gate|,
 * expert) within tolerance) / FETCH with fetch = WORKING, LOWEST, or CASCADE
 * down the ladder from `start` (1 when gate < the percentile). The caller
 * runs the fetch. Synchronous; host buffers in and out. */
enum { ESIM_MISS_OUT_FETCH = 0, ESIM_MISS_OUT_DROP = 1, ESIM_MISS_OUT_SUBST = 2 };
enum { ESIM_MISS_FETCH_WORKING = 0, ESIM_MISS_FETCH_LOWEST = 1, ESIM_MISS_FETCH_CASCADE = 2 };
typedef struct {
    int32_t policy, rank, drop_rank_threshold, n_scores;
    int32_t n_residents, ladder_len, pct_rank, pad;
    double gate_score, subst_tolerance;
} EsimMissQuery;
typedef struct { int32_t kind, substitute, fetch, start; } EsimMissDecision;
int esim_miss_decide(const EsimMissQuery *q, const double *scores, const int32_t *res_expert, const double *res_rec,
                     EsimMissDecision *decision);

int esim_policy_apply(const EsimPolicyState *state, const EsimPolicyOp *d_ops, int32_t n_ops, int32_t *d_results,
                      void *stream);

/* Shared memory one replayed grid point needs (for the host's grouping). */
int esim_replay_smem_per_point(const EsimConfig *h_cfg, int32_t n, int32_t max_tokens, int32_t pl_stride,
                               int32_t queue_cap);

/* Replay n grid points, one warp each. h_cfg/d_cfg: the same configs on
 * host (launch sizing) and device; cfg.trace_id indexes d_traces/d_routers
 * (device arrays of descriptors). Outputs (device): counters[n],
 * per_layer[n][pl_stride][ESIM_PL_FIELDS], and with ESIM_FLAG_FULL_LOG,
 * recs[n][rec_cap] + pred_experts[n][pe_cap]. max_tokens = largest token
 * count of any event (cache-aware scratch). warps_per_cta 0 = auto.
 * queue_cap: channel ring entries; <= 0 = the exact bound (resident slots
 * + 1, cannot overflow). A smaller positive cap saves shared memory; a point
 * whose channel outgrows it stops with counters.status = -5 and must be
 * re-launched with queue_cap = 0. */
int esim_replay_launch(const EsimConfig *h_cfg, const EsimConfig *d_cfg, int32_t n,
                       const EsimTraceDesc *d_traces, const EsimRouterOut *d_routers, int32_t max_tokens,
                       EsimCounters *d_counters, int64_t *d_per_layer, int32_t pl_stride,
                       EsimRec *d_recs, int64_t rec_cap, int32_t *d_pred_experts, int64_t pe_cap,
                       int32_t warps_per_cta, int32_t queue_cap, void *stream);
/* The same with a cap on the launch's CTAs. Common-path points (miss=fetch,
 * standard routing) replay in a persistent launch: one CTA of up to 12 warps
 * per SM, every warp pulling the next point of the launch order (put the
 * longest first). max_ctas > 0 limits the launch to that many CTAs (SMs), so
 * concurrent launches of different policies on different streams split the
 * GPU instead of interleaving; 0 = as many as fit. */
int esim_replay_launch_ex(const EsimConfig *h_cfg, const EsimConfig *d_cfg, int32_t n,
                          const EsimTraceDesc *d_traces, const EsimRouterOut *d_routers, int32_t max_tokens,
                          EsimCounters *d_counters, int64_t *d_per_layer, int32_t pl_stride,
                          EsimRec *d_recs, int64_t rec_cap, int32_t *d_pexp, int64_t pe_cap,
                          int32_t warps_per_cta, int32_t queue_cap, int32_t max_ctas, void *stream);

/* End-to-end host API (engine.run_simulation over many configs): host
 * traces (host pointers) and configs in; router + replay on the device;
 * host counters/per-layer/records out. Synchronous. Configs sharing a
 * trace_id must share the predictor (prefetch mode/overfetch/percentile)
 * and the prediction noise stream (prefetch_noise, seed): the noise is
 * applied on the device once per trace_id (esim_noise_launch). */
int esim_run_host(const EsimConfig *cfg, int32_t n, const EsimTraceDesc *traces, int32_t n_traces,
                  EsimCounters *counters, int64_t *per_layer, int32_t pl_stride,
                  EsimRec *recs, int64_t rec_cap, int32_t *pred_experts, int64_t pe_cap);

/* The same split into a reusable plan: create resolves everything that does
 * not change between runs (predictors, geometry groups and their order, the
 * device slab, descriptors); each run copies the step's inputs from the
 * caller's trace arrays (host pointers captured at create; page-lock them with
 * esim_host_register for DMA), routes, replays and writes counters[n] /
 * per_layer[n][pl_stride][ESIM_PL_FIELDS] (/ recs, pred_experts when rec_cap
 * > 0) straight into the caller's buffers, in the caller's config order.
 * Synchronous. esim_run_host = create + run + destroy. */
int esim_sweep_plan_create(const EsimConfig *cfg, int32_t n, const EsimTraceDesc *traces, int32_t n_traces,
                           int32_t pl_stride, int64_t rec_cap, int64_t pe_cap, void **plan);
int esim_sweep_plan_run(void *plan, EsimCounters *counters, int64_t *per_layer, EsimRec *recs,
                        int32_t *pred_experts);
int esim_sweep_plan_destroy(void *plan);
/* Pipelined steps over two device slabs (double buffering): submit enqueues one
 * step (H2D, router, replays, D2H into the given buffers, which must stay
 * untouched until its wait) and returns; wait blocks for the oldest submitted
 * step and checks its statuses. At most two steps in flight. Step k+1's copies
 * and router overlap step k's replays. esim_sweep_plan_run drains first. */
int esim_sweep_plan_submit(void *plan, EsimCounters *counters, int64_t *per_layer);
/* Opt-in profile-guided schedule: re-order every launch group longest-measured
 * first using the per-point replay times in `counters` (the output of one of
 * this plan's previous runs). Plans are created with a static order (the
 * traces' token-expert selections, longest first). */
int esim_sweep_plan_tune(void *plan, const EsimCounters *counters);
int esim_sweep_plan_wait(void *plan);

/* Report assembly for sweeps (metrics.flatten_report + emit csv,
 * metrics.py:190-316, 348-395): the result-dependent CSV columns (totals,
 * rates, timing, fidelity, prefetch) of n points, formatted exactly as the
 * reference's csv emission writes them (Python str(): shortest round-trip
 * floats, True/False). With prefixes (point i's fixed config columns =
 * prefixes[prefix_offsets[i] .. prefix_offsets[i+1]), ending in ","), each
 * point is one complete CSV line ending "\r\n"; without, only the result
 * columns. Point i's text is out[offsets[i] .. offsets[i+1]).
 * per_layer: [n][pl_stride][ESIM_PL_FIELDS] (identity checks). Host code, no
 * GPU needed. Returns 0, -1 (accounting identity broken), -4 (cap too small). */
int esim_report_csv(const EsimCounters *counters, const int64_t *per_layer, int32_t pl_stride,
                    const int32_t *num_layers, const int64_t *per_layer_compute_us, int32_t n,
                    const char *prefixes, const int64_t *prefix_offsets, char *out, int64_t cap,
                    int64_t *offsets);

/* ---- trace ingestion (trace.py:219-279 read_trace) --
 * esim_trace_jsonl_parse: the event lines of a reference JSON-lines trace
 * (text = the whole file, line 1 = the spec record, parsed by the host),
 * parsed natively in parallel line blocks (n_threads <= 0: all cores) into
 * float32 rows bit-identical to json.loads + np.asarray(float32). Returns 0
 * with *handle, *n_rows and *n_passes set; ESIM_TRACE_SLOW when the file
 * needs the reference-exact reader (malformed line, unexpected record or
 * key, out-of-order pass/layer, mixed kinds or row counts within a pass,
 * NaN/Infinity, truncated last pass): *bad_line = first such line (-1: end of
 * file), and the host re-parses to raise the reference's TraceFormatError.
 * esim_trace_jsonl_take copies rows (row-major [n_rows][experts]) and the
 * per-pass token counts / kinds (0 prefill, 1 decode) out and frees the
 * handle; esim_trace_jsonl_free drops it. Host code, no GPU needed.
 * Replaces: read_trace (trace.py:219-279) -- json.loads + np.asarray per line. */
#define ESIM_TRACE_SLOW 1
int esim_trace_jsonl_parse(const char *text, int64_t len, int32_t num_layers, int32_t experts, int32_t n_threads,
                           void **handle, int64_t *n_rows, int32_t *n_passes, int64_t *bad_line);
int esim_trace_jsonl_take(void *handle, float *logits, int32_t *pass_tokens, int32_t *pass_kind);
int esim_trace_jsonl_free(void *handle);
/* Device-side validation of uploaded logits (trace.py:94-95 "non-finite
 * logit value"): *d_first_bad (device int64) = index of the first
 * non-finite element, or -1. d_logits 16-byte aligned. Async on `stream`. */
int esim_trace_check_finite(const float *d_logits, int64_t n, int64_t *d_first_bad, void *stream);

/* ---- physical layer step (no reference equivalent; configs[1]) -------- */
typedef struct {
    int32_t num_layers, experts, top_k;
    int32_t hidden, inter;        /* OLMoE-1B-7B: 2048, 1024 (SwiGLU expert 3*H*I bf16) */
    int32_t n_slots;              /* HBM cache slots = capacity / working-precision expert bytes */
    int32_t max_tokens;           /* largest pass (<= 16384) */
    int32_t weight_format;        /* precision code of the working precision (models.PRECISION_ORDER):
                                     0: bf16 tile-major (3*H*I*2 B); 1: int8 / 2: int4 / 3: int2 tile-major
                                     codes (several per byte, lowest bits first, two's complement) +
                                     fp32 per-row scales (3*H*I*bits/8 + 4*(2*I+H) B), copied quantised
                                     and dequantised per layer into a bf16 scratch pool for the FFN */
    int32_t prec_mask;            /* precisions held in the store (bit = code); 0 = just weight_format.
                                     Mixed-precision miss policies (fetch_low / fetch_priority) need
                                     every rung of the ladder: each slot then holds whichever
                                     precision the decision stream fetched into it */
} EsimLSParams;

typedef struct {
    double ttft_ms, total_ms, decode_ms, host_enqueue_ms;
    int64_t h2d_bytes, n_copies, n_demand_copies, n_prefetch_copies, n_cancelled;
    int64_t n_ffn_batches, n_exec_experts, n_records;
    int64_t status;
} EsimLSResult;

/* Engine: pinned host expert store, one region [L][E][bytes(prec)] per
 * precision in prec_mask, ascending code (esim_ls_store returns it for
 * initialisation, esim_ls_format the per-expert bytes and region offset of
 * one precision, 0 if absent), n_slots HBM slots sized for the largest
 * precision with TMA descriptors, copy and compute streams, per-slot
 * RAW/WAR events. esim_ls_expert_bytes: the working precision's bytes. */
int esim_ls_create(const EsimLSParams *p, void **handle);
void *esim_ls_store(void *handle);
int64_t esim_ls_expert_bytes(void *handle);
int64_t esim_ls_format(void *handle, int32_t prec, int64_t *store_offset);
int64_t esim_ls_store_bytes(void *handle);
/* The last request's executed routing [rows][K] (expert, weight): the
 * router's top-k, or with routing=cache_aware the replay's re-routed
 * selection and its original-softmax weights (routing.py:147-160). */
int esim_ls_route_rows(void *handle, int16_t *sel_out, float *w_out, int64_t rows);
void *esim_ls_slots(void *handle);
/* Attach an always-resident shared expert (Qwen1.5-MoE-A2.7B, BASELINE.json
 * configs[3]: 2048 x 5632 per layer; not cache-managed -- the reference
 * models only routed experts): d_w [L][3*H*inter] bf16 in the
 * routed experts' tile-major layout, d_gate [L][H] bf16, caller-owned device
 * memory. Each layer then adds sigmoid(x . gate_l) * SwiGLU_l(x) for every
 * token to the routed output before the residual (HF Qwen2MoeSparseMoeBlock).
 * inter = 0 detaches. */
int esim_ls_shared_expert(void *handle, const void *d_w, const void *d_gate, int32_t inter);
/* Parity hook: every layer's output hidden states (after the residual) of
 * the following esim_ls_run calls are written to host_buf (page-locked /
 * mapped host memory, [rows][H] bf16, events in (pass, layer) order, the
 * pass's token count of rows per event); NULL turns it off. */
int esim_ls_capture_layers(void *handle, void *host_buf, int64_t rows);
int esim_ls_destroy(void *handle);
const char *esim_ls_last_error(void);
/* One request. trace: host struct with device pointers; h_pass_tokens: host
 * copy of its pass token counts; cfg: the logical config (decisions);
 * x_prefill [T0][H], x_decode [passes-1][H], out [rows][H]: pinned host bf16.
 * Timing: TTFT = start -> last prefill layer done; total = all passes and
 * copies done (CUDA events). counters_out / per_layer_out: the decision
 * stream's report vector (bit-exact with the reference for cfg). */
int esim_ls_run(void *handle, const EsimTraceDesc *trace, const int32_t *h_pass_tokens, const EsimConfig *cfg,
                const void *x_prefill, const void *x_decode, void *out, EsimCounters *counters_out,
                int64_t *per_layer_out, EsimLSResult *res);

/* FFN building blocks (ffn_gemm.cu): 2-D bf16 TMA descriptor (128B swizzle,
 * box [box_rows][64]); token gather; the grouped tcgen05 SwiGLU experts
 * (one persistent launch: w1 maps with 64-row boxes, w2 maps with 128-row
 * boxes); residual x += y. esim_ffn_set_trace: optional device buffer of
 * per-unit globaltimer stamps [units][4] for the following launches (NULL off). */
int esim_tmap_bf16(void *out_map, const void *base, int64_t rows, int64_t cols, int32_t box_rows);
int esim_ffn_gather(const void *d_x, const int32_t *d_tok_index, void *d_xg, int32_t n_exec, int32_t npad,
                    int32_t hidden, void *stream);
int esim_ffn_experts(const void *d_w1_maps, const void *d_w2_maps, const void *d_x_map, const void *d_act_map,
                     const int32_t *d_exec_slot, const int32_t *d_tok_index, const float *d_tok_weight,
                     void *d_act, float *d_y, int32_t n_exec, int32_t npad, int32_t inter, int32_t hidden,
                     void *stream);
/* The same with the largest token count of any executed expert: <= 4 (decode)
 * selects the fused per-slice kernel (no gemm1 -> gemm2 handoff across CTAs). */
int esim_ffn_experts_ex(const void *d_w1_maps, const void *d_w2_maps, const void *d_x_map, const void *d_act_map,
                        const int32_t *d_exec_slot, const int32_t *d_tok_index, const float *d_tok_weight,
                        void *d_act, float *d_y, int32_t n_exec, int32_t npad, int32_t inter, int32_t hidden,
                        int32_t max_tok, void *stream);
int esim_ffn_residual(void *d_x, float *d_y, int64_t n, void *stream);
int esim_ffn_set_trace(void *d_trace);
/* Decode-like layers (<= 4 tokens per expert) over quantised slots: slot
 * pool d_slots (slot_bytes apart, tile-major codes of `bits` 8 / 4 / 2 then
 * fp32 row scales, as the layer step stores them), d_exec_slot = slot per
 * executed expert; dequantisation is fused into the FFN's A operand
 * (ffn_decode_q_kernel). x map: the gathered tokens, box 16 rows. */
int esim_ffn_experts_q(const void *d_slots, int64_t slot_bytes, int32_t bits, const void *d_x_map,
                       const int32_t *d_exec_slot, const int32_t *d_tok_index, const float *d_tok_weight,
                       float *d_y, int32_t n_exec, int32_t inter, int32_t hidden, void *stream);

/* Decode layers (<= 4 tokens per expert) as a streaming GEMV straight from
 * the slots (ffn_gemv.cu): bits 16 = bf16 slots, 8 / 4 / 2 = quantised codes
 * + fp32 row scales (the layout above); x = the layer input [T][hidden]
 * (no gather), d_tok_index / d_tok_weight [n_exec][npad] (-1 = no token),
 * max_tok = the largest token count of any executed expert (1..4). */
int esim_ffn_experts_gemv(const void *d_slots, int64_t slot_bytes, int32_t bits, const void *d_x,
                          const int32_t *d_exec_slot, const int32_t *d_tok_index, const float *d_tok_weight,
                          float *d_y, int32_t n_exec, int32_t npad, int32_t max_tok, int32_t inter, int32_t hidden,
                          void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECMD_B200_H */
