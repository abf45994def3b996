// replay.cu -- the expert-cache layer step as a device state machine.
//
// One warp replays one grid point (a SimConfig over a trace) through the
// reference's logical timeline, bit-exactly:
//   Simulation._run_layer / run / _settle / _advance_to   engine.py:422-447, 596-649, 729-748
//   Simulation._handle_demand / _fetch / _evict           engine.py:451-574
//   Simulation._submit_prefetches + watchdog_step         engine.py:651-725, prefetch.py:163-221
//   CacheState (byte accounting, reservations)            engine.py:188-255
//   Channel (serialized link, demand insertion, promote,  engine.py:271-370
//            newest-pending cancellation, retime)
//   EvictionPolicy x6 (lru lfu lhu fld sb ls)             eviction.py:29-294
//   resolve_miss / find_substitute                        miss.py:66-140
//   classify_miss / ResidencyHistory                      metrics.py:32-57
//   route_event (cache_aware, DeltaAvgState)              routing.py:60-90, 143-161
//
// Device-native structures instead of the reference's containers:
//  * directory: one packed 16-bit word per ident (ident = layer*E + expert):
//    bit15 in-flight, bit12 resident, bits13-14 precision, bits0-11 slot;
//    an int16 miss history per ident; a slot table of residents, each with
//    one 64-bit policy key; a free-slot stack;
//  * victim selection: a warp argmin over the slot table (LS: class|gen,
//    LRU: stamp, LFU: count then touch, FLD: cyclic distance, SB: fp64);
//  * channel: a ring buffer [head][demands/promoted][pending prefetches]
//    whose retiming is a warp max-plus scan; capacity is a launch parameter
//    (overflow -> status -5, the host re-launches with the exact bound).
// Every helper is force-inlined so the warp-uniform scalars (clock, byte
// accounting, queue cursors, digest) stay in registers, redundantly
// computed by all 32 lanes; counters live in shared memory owned by lane 0.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "../../include/specmd_b200.h"
#include "numpy_f32.cuh"
#include "warp_route.cuh"
#include "digest.cuh"

#define DFI __device__ __forceinline__

namespace esim {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t FNV_OFFSET = 0xcbf29ce484222325ULL;
constexpr uint64_t FNV_PRIME = 0x100000001b3ULL;
constexpr int STATUS_QUEUE_OVERFLOW = -5;
constexpr int STATUS_COUNT_OVERFLOW = -7;          // an LFU/LHU access count outgrew 16 bits
constexpr int STATUS_SEQ_OVERFLOW = -8;            // > 2^31 policy stamps in one replay


// lane-0 owned counters (shared memory)
struct Ctr {                       // 32-bit counts: native ATOMS.ADD (64-bit is a CAS loop)
    uint32_t totals[15];
    uint32_t rows_total, faithful, modified;
    uint32_t pf_tp, pf_pred, pf_dem, pf_records, pf_empty, pf_prec_parts, pf_rec_parts;
    uint32_t ls_forced, ls_refusals;
    uint32_t passes, decode_passes;
    int64_t sync_overhead, decode_us, ttft, total;   // lane-0 plain updates
    double ps[8];                  // Neumaier (f, c) pairs: orig, exec, prec, rec
};

struct Layout {
    int key, q_submit, q_comp, dsum, ctr, dem_summed, q_ent;   // 8-byte
    int cnt, rscore, pl, demmask, lsc, ca_w, ca_row, dem_gate, dem_tokens, dem_expert, dem_rank;  // 4-byte
    int rs, hist, res_ident, fs, ca_sel, vict;            // 2-byte
    int tofetch, ca_mod;                                  // 1-byte
    int total;
};

__host__ __device__ inline int al8(int x) { return (x + 7) & ~7; }

// gen = false (common-path kernels: uniform transfers, no substitution): the
// per-entry submit/completion times and the recorded scores are never touched
// and take no space
__host__ __device__ inline Layout make_layout(int N, int S, int Q, int L, int E, int T, int K, bool ca,
                                              bool has_cnt, bool gen) {
    Layout l;
    int o = 0;
    l.key = o; o += al8(S * 8);
    l.q_submit = o; o += al8(gen ? Q * 8 : 0);
    l.q_comp = o; o += al8(gen ? Q * 8 : 0);
    l.dsum = o; o += al8(ca ? L * 8 : 0);
    l.ctr = o; o += al8((int)sizeof(Ctr));
    l.dem_summed = o; o += al8(ca ? E * 8 : 0);
    l.q_ent = o; o += al8(Q * 8);                   // channel entries: ident | flags | score, one word each
    l.cnt = o; o += al8(has_cnt ? N * 2 : 0);      // 16-bit LFU/LHU access counts (host-checked bound)
    l.rscore = o; o += al8(gen ? S * 4 : 0);
    l.pl = o; o += al8(L * ESIM_PL_FIELDS * 4);
    l.demmask = o; o += al8(((E + 31) / 32) * 4);
    l.lsc = o; o += al8(E * 4);
    l.ca_w = o; o += al8(ca ? T * K * 4 : 0);
    l.ca_row = o; o += al8(ca ? E * 4 : 0);
    l.dem_gate = o; o += al8(ca ? E * 4 : 0);
    l.dem_tokens = o; o += al8(ca ? E * 4 : 0);
    l.dem_expert = o; o += al8(ca ? E * 4 : 0);
    l.dem_rank = o; o += al8(ca ? E * 4 : 0);
    l.rs = o; o += al8(N * 2);
    l.hist = o; o += al8(N * 2);
    l.res_ident = o; o += al8(S * 2);
    l.fs = o; o += al8(S * 2);
    l.ca_sel = o; o += al8(ca ? T * K * 2 : 0);
    l.vict = o; o += al8(gen ? 0 : E * 2);          // batched watchdog sweep 2 (uniform instances)
    l.tofetch = o; o += al8(E);
    l.ca_mod = o; o += al8(ca ? T : 0);
    l.total = o;
    return l;
}

struct ReplayArgs {
    const EsimConfig* cfg;
    int n_points;
    const EsimTraceDesc* traces;   // device array of descriptors (device pointers inside)
    const EsimRouterOut* routers;
    EsimCounters* counters;
    int64_t* per_layer;            // [n][Lmax][ESIM_PL_FIELDS]
    EsimRec* recs;
    int64_t rec_cap;
    int32_t* pexp;
    int64_t pe_cap;
    int N, S, Q, Lmax, Emax, Tmax, Kmax;  // smem sizing (max over points)
    int has_cnt;                   // any LFU/LHU point (per-ident counts)
    int warps_per_cta;
    int point_bytes;
    Layout lay;                    // per-point shared-memory layout (launch-uniform, kernel-parameter space:
                                   // the smem pointers rematerialise from it instead of holding registers)
    const int32_t* out_index;      // optional: output row of launch point pid (counters, per_layer, logs)
    int* work;                     // optional: persistent launch, next point of the launch order
    volatile int64_t* progress;    // optional (single point, streamed decisions): [0] events done
                                   // (-1 on error), [1 + ev] records emitted through event ev
};

// packed directory word
constexpr uint16_t RS_INF = 0x8000, RS_RES = 0x1000;
DFI bool rs_res(uint16_t w) { return w & RS_RES; }
DFI int rs_prec(uint16_t w) { return (w >> 13) & 3; }
DFI int rs_slot(uint16_t w) { return w & 0x0FFF; }
DFI uint16_t rs_make(int prec, int slot) { return (uint16_t)(RS_RES | (prec << 13) | slot); }

// TM: the simulated-clock type -- int32_t when the host has bounded the run's
// total time below 2^31 us (time32 launches), else int64_t
template <typename TM>
struct PtT {
    using Tm = TM;
    const EsimConfig* c;
    int L, E, K, S, Q;
    int pol, lane;
    int miss;                       // ESIM_MISS_* (constant-folded in the simple specialisation)
    int64_t cap;
    TM dur0, dur1, dur2, dur3;      // transfer times by precision code (registers, not an array)
    int64_t eb0, eb1, eb2, eb3;     // expert bytes by precision code
    TM dur_w;                       // working precision
    int64_t eb_w;
    int wp;                         // working precision code (cfg->working_prec, kept in a register)
    double inv_dur;                 // 1 / dur_w (uniform-path landing count)
    bool uniform;                   // all transfers at the working precision (common path)
    // shared memory
    uint64_t* key;
    int64_t *q_submit, *q_comp;     // non-uniform instances only
    TM qc0;                         // uniform instances: completion time of the head entry
    uint64_t einv;                  // ceil(2^32 / E): ident / E as a multiply-high
    double* dsum;
    Ctr* ctr;
    double* dem_summed_s;
    uint16_t* cnt;                  // LFU / LHU access count per ident (< 65536: esim_replay_launch checks)
    float* rscore;
    int32_t* pl;
    uint32_t* demmask;
    float* lsc;
    float* ca_w;
    float* ca_row;
    float* dem_gate_s;
    int32_t* dem_tokens_s;
    int32_t* dem_expert_s;
    int32_t* dem_rank_s;
    uint16_t* rs;
    int16_t* hist;
    int16_t* res_ident;
    uint16_t* fs;
    uint2* q_ent;                   // channel ring: .x = ident:16 | flags:8 (bits 16-23), .y = score f32 bits
    int16_t* ca_sel;
    int16_t* vict;                  // sweep-2 victims in eviction order (uniform instances)
    uint8_t* tofetch;
    uint8_t* ca_mod;
    // warp-uniform scalars
    TM now;
    int64_t resident_bytes, reserved_bytes;       // general path: bytes
    int32_t res_u, resv_u, cap_u;   // uniform path: resident / reserved experts and the experts capacity holds
    int qh, qn, nA, fs_top;
    uint32_t seq;                   // policy stamp counter (< SEQ_LIMIT < 2^31: checked once per layer)
    uint32_t digest;                // lane-partial sum (mod 2^32) of lane-parallel records' terms
    uint32_t digest_u;              // warp-uniform records' terms (every lane holds the same sum)
    bool digest_on;
    uint32_t pf_ev[5];              // prefetch submitted/started/completed/skipped/dropped (registers)
    uint32_t n_evict, n_forced;
    // this layer's access outcomes (registers; folded into the smem per-layer
    // counters once per layer): misses (fetch + wait) by class, drops, substitutions
    uint32_t lc_miss, lc_c0, lc_c1, lc_drop, lc_sub;
    int32_t n_recs;                 // records so far (< 2^31: a log of 2^31 x 64 B records cannot exist)
    int64_t n_pe;
    int pass_id, layer;
    int err;
    // record output
    EsimRec* recs;
    int64_t rec_cap;
    int32_t* pexp;
    int64_t pe_cap;
    bool full;
};

// per-precision sizes; on the common path (miss=fetch) every transfer is at the working
// precision, which `uniform` (a template constant after inlining) exploits
template <class Pt>
DFI typename Pt::Tm pdur(const Pt& p, int c) {
    if (p.uniform) return p.dur_w;
    return c == 0 ? p.dur0 : c == 1 ? p.dur1 : c == 2 ? p.dur2 : p.dur3;
}
template <class Pt>
DFI int64_t peb(const Pt& p, int c) {
    if (p.uniform) return p.eb_w;
    return c == 0 ? p.eb0 : c == 1 ? p.eb1 : c == 2 ? p.eb2 : p.eb3;
}

// x / d for 0 <= x < 2^53, d > 0, with inv = 1.0 / d: one double multiply and an
// exact integer correction instead of a ~70-instruction 64-bit division
DFI int64_t udiv_rcp(int64_t x, int64_t d, double inv) {
    int64_t q = (int64_t)((double)x * inv);
    if (q * d > x) q--;
    else if ((q + 1) * d <= x) q++;
    return q;
}

// Cache byte accounting (engine.py:188-255). On the uniform path every resident
// or reserved entry is one working-precision expert, so it is counted in expert
// units (32-bit) against cap_u = capacity / expert bytes -- exact: a fetch fits
// iff units + 1 <= floor(capacity / bytes); the general path keeps bytes.
template <class Pt>
DFI bool no_room(const Pt& p, int64_t nb) {
    return p.uniform ? p.res_u + p.resv_u >= p.cap_u : p.cap - p.resident_bytes - p.reserved_bytes < nb;
}
template <class Pt>
DFI void reserve_add(Pt& p, int64_t nb, int n) {
    if (p.uniform) p.resv_u += n; else p.reserved_bytes += nb * n;
}
template <class Pt>
DFI void resident_add(Pt& p, int64_t nb, int n) {
    if (p.uniform) p.res_u += n; else p.resident_bytes += nb * n;
}

template <class Pt>
DFI int ediv(const Pt& p, int ident) {             // ident / E, exact for ident < 2^24
    return (int)(((uint64_t)(uint32_t)ident * p.einv) >> 32);
}

template <class Pt>
DFI int qphys(const Pt& p, int i) {
    int x = p.qh + i;
    return x & (p.Q - 1);                          // Q is a power of two (replay_sizing)
}

// fire-and-forget shared-memory atomics: lane 0 never waits on a counter RMW
template <class Pt>
DFI void ctr_add(Pt& p, uint32_t& f, uint32_t v) {
    if (p.lane == 0) f += v;
}
template <class Pt>
DFI void pl_add(Pt& p, int idx, int v) {
    if (p.lane == 0) p.pl[idx] += v;
}

template <class Pt>
DFI void ps_add(Pt& p, int which, double x) {
    if (p.lane == 0) {
        double f = p.ctr->ps[2 * which], c = p.ctr->ps[2 * which + 1];
        double t = __dadd_rn(f, x);
        if (g_pysum_plain) {}                                    // CPython < 3.12: no compensation
        else if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
        else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
        p.ctr->ps[2 * which] = t;
        p.ctr->ps[2 * which + 1] = c;
    }
}

// ---------------------------------------------------------------------------
// record output + digest
// digest: mix = sum_i w_i * K_i (mod 2^32) over the record's sixteen 32-bit
// words (t0 skipped for predictions) + sum_j (e_j+1) * G*(j+1) over a
// prediction's experts; x = (mix ^ idx*C) * P mod 2^32 (idx = record index);
// digest += x ^ (x >> 15) mod 2^32 (all 32-bit operations: the fold sits on
// every record's path). The index makes it
// order-sensitive, the sum keeps the loop-carried chain one add. Zero/constant
// words fold at compile time.
// ---------------------------------------------------------------------------
DFI uint32_t fold(uint32_t mix, int32_t idx) {
    const uint32_t x = (mix ^ ((uint32_t)idx * 0x85EBCA77u)) * 0xC2B2AE3Du;
    return x ^ (x >> 15);
}

// record with its digest word already mixed (premixed: from the router summary)
template <class Pt>
DFI void emit_mixed(Pt& p, uint32_t mix, int kind, int layer, int i0, int i1, int i2, int i3, int i4, int64_t t0,
                    int64_t t1, int64_t t2, double x0, const int32_t* pe = nullptr, int npe = 0) {
    if (p.digest_on) {
        // order-sensitive through the record index, associative across records;
        // the digest is lane-partial (summed over the warp once, at the end), so a
        // warp-uniform record is added by lane 0 only
        p.digest_u += fold(mix, p.n_recs);            // warp-uniform part, added once at the end
    }
    if (p.full) {
        const int64_t n = p.n_recs, m = p.n_pe;
        if (n < p.rec_cap && m + npe <= p.pe_cap) {
            if (p.lane == 0) {
                EsimRec r;
                r.kind = kind; r.pass_id = p.pass_id; r.layer = layer;
                r.i0 = i0; r.i1 = i1; r.i2 = i2; r.i3 = i3; r.i4 = i4;
                r.t0 = kind == ESIM_REC_PREDICTION ? m : t0; r.t1 = t1; r.t2 = t2; r.x0 = x0;
                p.recs[n] = r;
            }
            for (int j = p.lane; j < npe; j += 32) p.pexp[m + j] = pe[j];
        } else if (!p.err) {
            p.err = -4;
        }
    }
    p.n_recs++;
    p.n_pe += npe;
}

// record mixed here (digest.cuh; zero/constant words fold at compile time)
template <class Pt>
DFI void emit(Pt& p, int kind, int layer, int i0, int i1, int i2, int i3, int i4, int64_t t0, int64_t t1,
              int64_t t2, double x0) {
    const uint32_t mix = p.digest_on ? rec_mix(kind, p.pass_id, layer, i0, i1, i2, i3, i4, t0, t1, t2, x0) : 0u;
    emit_mixed(p, mix, kind, layer, i0, i1, i2, i3, i4, t0, t1, t2, x0);
}

// up to 32 records emitted at once, one per active lane (lane-varying fields),
// in `rank` order after the records already emitted; cnt = number active
template <class Pt>
DFI void emit_lanes(Pt& p, bool act, int rank, int cnt, int kind, int layer, int i0, int i1, int i2, int i3,
                    int i4, int64_t t0, int64_t t1, int64_t t2, double x0) {
    if (cnt == 0) return;
    if (p.digest_on) {
        uint32_t v = 0;
        if (act) {
            v = fold(rec_mix(kind, p.pass_id, layer, i0, i1, i2, i3, i4, t0, t1, t2, x0), p.n_recs + rank);
        }
        p.digest += v;                                   // lane-partial

    }
    if (p.full) {
        if (p.n_recs + cnt <= p.rec_cap) {
            if (act) {
                EsimRec r;
                r.kind = kind; r.pass_id = p.pass_id; r.layer = layer;
                r.i0 = i0; r.i1 = i1; r.i2 = i2; r.i3 = i3; r.i4 = i4;
                r.t0 = t0; r.t1 = t1; r.t2 = t2; r.x0 = x0;
                p.recs[p.n_recs + rank] = r;
            }
        } else if (!p.err) {
            p.err = -4;
        }
    }
    p.n_recs += cnt;
}

DFI unsigned lanes_below(int lane) { return (1u << lane) - 1u; }

// one record at absolute log index idx from this lane (batched phases: every
// lane owns a record at a position fixed by prefix counts); returns its digest
// term (0 when inactive) for the caller's one warp-sum per batch
template <class Pt>
DFI uint32_t lane_rec(Pt& p, bool act, int32_t idx, int kind, int layer, int i0, int i1, int i2, int i3, int i4,
                      int64_t t0, int64_t t1, int64_t t2, double x0) {
    if (!act) return 0;
    if (p.full) {
        if (idx < p.rec_cap) {
            EsimRec r;
            r.kind = kind; r.pass_id = p.pass_id; r.layer = layer;
            r.i0 = i0; r.i1 = i1; r.i2 = i2; r.i3 = i3; r.i4 = i4;
            r.t0 = t0; r.t1 = t1; r.t2 = t2; r.x0 = x0;
            p.recs[idx] = r;
        } else {
            p.err = -4;                          // lane-local; folded by the caller
        }
    }
    return p.digest_on ? fold(rec_mix(kind, p.pass_id, layer, i0, i1, i2, i3, i4, t0, t1, t2, x0), idx) : 0;
}

template <class Pt>
DFI void digest_add_warp(Pt& p, uint32_t v) {        // this lane's records of a batch (lane-partial digest)
    if (!p.digest_on) return;
    p.digest += v;
}

template <class Pt>
DFI void err_fold(Pt& p) {                       // a lane-local record-capacity error -> warp-uniform
    const int e = __reduce_min_sync(FULL, p.err);
    p.err = e;
}

template <class Pt>
DFI void rec_prefetch(Pt& p, int ev, int target, int expert, int64_t t, float score, int reason) {
    emit(p, ESIM_REC_PREFETCH, p.layer, ev, target, expert, reason, 0, t, 0, 0, (double)score);
    p.pf_ev[ev]++;                  // ev is a compile-time constant at every call site
}

// ---------------------------------------------------------------------------
// policies (eviction.py:29-294) on slot keys
// ---------------------------------------------------------------------------
// LRU / LS keys are 32-bit: stamp (p.seq, kept below 2^31 - 1: STATUS_SEQ_OVERFLOW)
// with the LS class in bit 31, so the victim scan compares one 32-bit word per slot
constexpr uint64_t LS_CURRENT = 1ull << 31;
constexpr uint64_t SEQ_LIMIT = 0x7FFF0000ull;        // checked once per layer (a layer adds < 2^16)
constexpr uint64_t KEY_FREE = 0x000FFFFFFFFFFFFFull; // free-slot key: low word 0xFFFFFFFF is above every live LRU/LS key,
                                                     // also after begin_pass clears bit 50

DFI uint64_t order_double(double d) {
    const uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}

template <class Pt>
DFI void set_key(Pt& p, int slot, uint64_t k) {
    if (p.lane == 0) p.key[slot] = k;
    __syncwarp();
}

template <class Pt>
DFI void ls_touch(Pt& p, int slot) {                                  // eviction.py:245-250
    if (p.key[slot] & LS_CURRENT) return;                              // first touch fixed it
    __syncwarp();
    set_key(p, slot, LS_CURRENT | (p.seq++));
}

template <class Pt>
DFI void note_admit(Pt& p, int slot, int ident) {
    uint64_t nk;
    switch (p.pol) {
    case ESIM_EV_LRU: nk = p.seq++; break;                                       // move_to_end
    case ESIM_EV_LFU: case ESIM_EV_LHU:                                          // count:16 | touch:32
        nk = ((uint64_t)p.cnt[ident] << 32) | (uint64_t)(p.seq++); break;       // (counts persist)
    case ESIM_EV_LS: nk = LS_CURRENT | (p.seq++); break;                         // untracked -> current
    default: nk = 0; break;                                                      // FLD; SB signal 0.0
    }
    set_key(p, slot, nk);
}

template <class Pt>
DFI void note_access(Pt& p, int ident, int slot, bool has_gate, double gate, int prec) {
    switch (p.pol) {
    case ESIM_EV_LRU: set_key(p, slot, p.seq++); break;
    case ESIM_EV_LFU: case ESIM_EV_LHU: {
        const int step = (p.pol == ESIM_EV_LFU || prec == p.c->precisions[0]) ? 1 : 0;
        const uint32_t c = p.cnt[ident] + step;
        if (c > 0xFFFF) p.err = STATUS_COUNT_OVERFLOW;                      // never silently wrap
        else if (p.lane == 0) p.cnt[ident] = (uint16_t)c;
        set_key(p, slot, ((uint64_t)c << 32) | (uint64_t)(p.seq++));
        break;
    }
    case ESIM_EV_SB:
        if (has_gate) {
            const double s = __longlong_as_double((long long)p.key[slot]);
            __syncwarp();
            set_key(p, slot, (uint64_t)__double_as_longlong(__dadd_rn(s, gate)));
        }
        break;
    case ESIM_EV_LS: ls_touch(p, slot); break;
    default: break;
    }
}

// warp argmin over residents; returns the victim slot or -1 (select_victim).
// Every policy's order is total, so one 64-bit key per slot with the slot
// index in the low 12 bits reduces in a single shuffle chain:
//   LRU / LS   (class | stamp) << 12 | slot      stamps are unique
//   LFU / LHU  the slot key itself: count:16 | touch:32 (touches are unique)
//   FLD        (L-1-dist):8 | expert:16 | layer:16 | slot:12
//   SB         two stages: min signal, then min ident among equal signals
DFI uint64_t warp_min_u64(uint64_t v) {         // two redux.sync (hi word, then lo among ties)
    const uint32_t hi = (uint32_t)(v >> 32);
    const uint32_t mhi = __reduce_min_sync(FULL, hi);
    const uint32_t mlo = __reduce_min_sync(FULL, hi == mhi ? (uint32_t)v : 0xFFFFFFFFu);
    return ((uint64_t)mhi << 32) | mlo;
}

template <class Pt>
DFI int select_victim(Pt& p, bool forced) {
    const int c = p.layer;
    uint64_t best = ~0ull;
    if (p.pol == ESIM_EV_SB) {
        uint64_t bsig = ~0ull;
        for (int s = p.lane; s < p.S; s += 32)
            if (p.res_ident[s] >= 0) {
                const uint64_t k = order_double(__longlong_as_double((long long)p.key[s]));
                bsig = k < bsig ? k : bsig;
            }
        bsig = warp_min_u64(bsig);
        if (bsig == ~0ull) return -1;
        for (int s = p.lane; s < p.S; s += 32) {
            const int id = p.res_ident[s];
            if (id >= 0 && order_double(__longlong_as_double((long long)p.key[s])) == bsig) {
                const uint64_t k = ((uint64_t)id << 12) | (uint64_t)s;
                best = k < best ? k : best;
            }
        }
        best = warp_min_u64(best);
        return (int)(best & 0xFFF);
    }
    if (p.pol == ESIM_EV_LRU || p.pol == ESIM_EV_LS) {
        // one 32-bit word per slot (the key's low word: class | stamp, free = 0xFFFFFFFF);
        // stamps are unique, so the lane holding the warp minimum names the victim
        const uint32_t* k32 = reinterpret_cast<const uint32_t*>(p.key);
        uint32_t bk = 0xFFFFFFFFu;
        int bs = 0;
        #pragma unroll 4
        for (int s = p.lane; s < p.S; s += 32) {
            const uint32_t k = k32[2 * s];
            bs = k < bk ? s : bs;
            bk = k < bk ? k : bk;
        }
        const uint32_t m = __reduce_min_sync(FULL, bk);
        if (m == 0xFFFFFFFFu) return -1;                                 // no resident
        const int slot = __shfl_sync(FULL, bs, __ffs(__ballot_sync(FULL, bk == m)) - 1);
        if (p.pol == ESIM_EV_LS && (m & (uint32_t)LS_CURRENT)) {
            if (!forced) { ctr_add(p, p.ctr->ls_refusals, 1); return -1; }
            ctr_add(p, p.ctr->ls_forced, 1);
        }
        return slot;
    }
    if (p.pol == ESIM_EV_LFU || p.pol == ESIM_EV_LHU) {
        // the slot key holds (count, touch) and free slots hold KEY_FREE (above
        // every live key), so the scan is one 64-bit load and compare per slot
        uint64_t bk = KEY_FREE;
        int bs = 0;
        #pragma unroll 4
        for (int s = p.lane; s < p.S; s += 32) {
            const uint64_t k = p.key[s];
            bs = k < bk ? s : bs;
            bk = k < bk ? k : bk;
        }
        const uint64_t m = warp_min_u64(bk);
        if (m == KEY_FREE) return -1;
        return __shfl_sync(FULL, bs, __ffs(__ballot_sync(FULL, bk == m)) - 1);
    }
    for (int s = p.lane; s < p.S; s += 32) {                              // FLD
        const int id = p.res_ident[s];
        if (id < 0) continue;
        const int l = ediv(p, id), e = id - l * p.E;
        int d = l - c;
        d = d < 0 ? d + p.L : d;
        const uint64_t k = ((uint64_t)(p.L - 1 - d) << 44) | ((uint64_t)e << 28) | ((uint64_t)l << 12) | (uint64_t)s;
        best = k < best ? k : best;
    }
    best = warp_min_u64(best);
    if (best == ~0ull) return -1;
    if (p.pol == ESIM_EV_LS && ((best >> 12) & LS_CURRENT)) {           // no stale resident left
        if (!forced) { ctr_add(p, p.ctr->ls_refusals, 1); return -1; }
        ctr_add(p, p.ctr->ls_forced, 1);
    }
    return (int)(best & 0xFFF);
}

// ---------------------------------------------------------------------------
// cache
// ---------------------------------------------------------------------------
template <class Pt>
DFI void evict(Pt& p, int slot, int cause, bool forced) {                 // engine.py:451-460
    const int ident = p.res_ident[slot];
    const int prec = rs_prec(p.rs[ident]);
    resident_add(p, peb(p, prec), -1);
    __syncwarp();
    if (p.lane == 0) {
        p.rs[ident] = 0;
        p.hist[ident] = (int16_t)p.pass_id;
        p.res_ident[slot] = -1;
        p.key[slot] = KEY_FREE;
        p.fs[p.fs_top] = (uint16_t)slot;
    }
    __syncwarp();
    p.fs_top++;
    const int il = ediv(p, ident);
    emit(p, ESIM_REC_EVICT, p.layer, il, ident - il * p.E, prec, cause, forced ? 1 : 0, 0, 0, 0, 0.0);
    p.n_evict++;
    p.n_forced += forced ? 1 : 0;
}

// ---------------------------------------------------------------------------
// channel
// ---------------------------------------------------------------------------
struct QEntry { int16_t ident; uint8_t flags; float score; int64_t submit, comp; };

DFI uint2 qe_make(int16_t ident, uint8_t flags, float score) {         // one 8-byte smem access, 32-bit ops
    return make_uint2((uint32_t)(uint16_t)ident | ((uint32_t)flags << 16), __float_as_uint(score));
}
DFI int16_t qe_ident(uint2 w) { return (int16_t)(uint16_t)w.x; }
DFI uint8_t qe_flags(uint2 w) { return (uint8_t)(w.x >> 16); }
DFI float qe_score(uint2 w) { return __uint_as_float(w.y); }

// The queue is settled whenever it is touched (every entry has comp > now >=
// its submit time: settle() lands comp <= now from the head after every time
// step), so comp_i = max(comp_{i-1}, submit_i) + dur_i (engine.py:283-288)
// never idles for i >= 1. With one transfer size (the uniform instances) that
// is comp_i = comp_0 + i * dur: only the head's completion time is stored.
template <class Pt>
DFI typename Pt::Tm qcomp(const Pt& p, int i) {
    if (p.uniform) return p.qc0 + (typename Pt::Tm)i * p.dur_w;
    return p.q_comp[qphys(p, i)];
}

template <class Pt>
DFI QEntry q_load(const Pt& p, int i) {
    const int x = qphys(p, i);
    QEntry e;
    const uint2 w = p.q_ent[x];
    e.ident = qe_ident(w); e.flags = qe_flags(w); e.score = qe_score(w);
    if (!p.uniform) { e.submit = p.q_submit[x]; e.comp = p.q_comp[x]; }
    return e;
}
template <class Pt>
DFI void q_store(Pt& p, int i, const QEntry& e) {
    const int x = qphys(p, i);
    p.q_ent[x] = qe_make(e.ident, e.flags, e.score);
    if (!p.uniform) { p.q_submit[x] = e.submit; p.q_comp[x] = e.comp; }
}

// open a hole at logical index `at` (shift [at, qn) right by one); false on overflow
template <class Pt>
DFI bool q_open(Pt& p, int at) {
    if (p.qn >= p.Q) { p.err = STATUS_QUEUE_OVERFLOW; return false; }
    for (int hi = p.qn; hi > at; hi -= 32) {
        const int lo = max(at, hi - 32);
        const int i = lo + p.lane;
        QEntry e;
        const bool act = i < hi;
        if (act) e = q_load(p, i);
        __syncwarp();
        if (act) q_store(p, i + 1, e);
        __syncwarp();
    }
    p.qn++;
    return true;
}

template <class Pt>
DFI void q_close(Pt& p, int at) {
    for (int lo = at + 1; lo < p.qn; lo += 32) {
        const int i = lo + p.lane;
        QEntry e;
        const bool act = i < p.qn;
        if (act) e = q_load(p, i);
        __syncwarp();
        if (act) q_store(p, i - 1, e);
        __syncwarp();
    }
    p.qn--;
}

// comp_i = max(comp_{i-1}, submit_i) + dur_i for i >= from >= 1 (engine.py:283-288):
// a warp inclusive scan composing x -> max(x + a, b)
template <class Pt>
DFI void retime(Pt& p, int from) {
    if (p.uniform) return;                       // implied by qcomp()
    if (from < 1) from = 1;
    if (from >= p.qn) return;
    int64_t carry = p.q_comp[qphys(p, from - 1)];
    for (int base = from; base < p.qn; base += 32) {
        const int i = base + p.lane;
        const bool act = i < p.qn;
        int64_t a = 0, b = INT64_MIN / 4;
        int x = 0;
        if (act) {
            x = qphys(p, i);
            const int64_t d = pdur(p, (qe_flags(p.q_ent[x]) >> 2) & 3);
            a = d;
            b = p.q_submit[x] + d;
        }
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t pa = __shfl_up_sync(FULL, a, o);
            const int64_t pb = __shfl_up_sync(FULL, b, o);
            if (p.lane >= o) { b = max(pb + a, b); a = pa + a; }
        }
        const int64_t comp = max(carry + a, b);
        __syncwarp();
        if (act) p.q_comp[x] = comp;
        const int last = min(31, p.qn - 1 - base);
        carry = __shfl_sync(FULL, comp, last);
        __syncwarp();
    }
}

template <class Pt>
DFI int q_find(const Pt& p, int ident) {
    for (int base = 0; base < p.qn; base += 32) {
        const int i = base + p.lane;
        const bool hit = i < p.qn && qe_ident(p.q_ent[qphys(p, i)]) == ident;
        const unsigned m = __ballot_sync(FULL, hit);
        if (m) return base + __ffs(m) - 1;
    }
    return -1;
}

// Uniform instances: entry i of the settled queue completes at qc0 + i * dur, so
// the k entries landed by `now` are known up front and admitted lane-parallel:
// slot = i-th pop of the free-slot stack, policy key stamp = seq + i, and the
// prefetch "completed" records at the positions their order fixes.
template <class Pt>
DFI void settle_uniform(Pt& p) {
    if (p.qn == 0 || p.qc0 > p.now) return;
    int k = p.qn;
    if (p.dur_w > 0) {
        // entry i has landed iff i * dur <= now - qc0: one compare per lane for
        // the usual <= 32 entries, the quotient beyond
        using Tm = typename Pt::Tm;
        const Tm d = p.now - p.qc0;
        if (p.qn <= 32) {
            k = __popc(__ballot_sync(FULL, p.lane < p.qn && (Tm)p.lane * p.dur_w <= d));
        } else {
            const int64_t t = udiv_rcp((int64_t)d, (int64_t)p.dur_w, p.inv_dur) + 1;
            if (t < k) k = (int)t;
        }
    }
    if (p.fs_top < k) { p.err = -2; return; }
    const int wp = p.wp;
    const unsigned below = lanes_below(p.lane);
    uint32_t dg = 0;
    int npf = 0;
    for (int b = 0; b < k; b += 32) {
        const int i = b + p.lane;
        const bool act = i < k;
        bool pf = false;
        int ident = 0, slot = 0;
        float score = 0.0f;
        if (act) {
            const int x = qphys(p, i);
            const uint2 w = p.q_ent[x];
            ident = qe_ident(w);
            pf = qe_flags(w) & 1;
            score = qe_score(w);
            slot = p.fs[p.fs_top - 1 - i];
            p.rs[ident] = rs_make(wp, slot);
            p.res_ident[slot] = (int16_t)ident;
            if (p.hist[ident] == -2) p.hist[ident] = -1;
            const uint64_t st = (uint64_t)(p.seq + (uint32_t)i);   // note_admit, in pop order
            uint64_t nk = 0;
            if (p.pol == ESIM_EV_LRU) nk = st;
            else if (p.pol == ESIM_EV_LS) nk = LS_CURRENT | st;
            else if (p.pol == ESIM_EV_LFU || p.pol == ESIM_EV_LHU) nk = ((uint64_t)p.cnt[ident] << 32) | st;
            p.key[slot] = nk;
        }
        const unsigned pm = __ballot_sync(FULL, pf);
        const int il = ediv(p, ident);
        dg += lane_rec(p, pf, p.n_recs + npf + __popc(pm & below), ESIM_REC_PREFETCH, p.layer, 2, il,
                       ident - il * p.E, 0, 0, p.qc0 + (typename Pt::Tm)i * p.dur_w, 0, 0, (double)score);
        npf += __popc(pm);
    }
    digest_add_warp(p, dg);
    if (p.full) err_fold(p);
    __syncwarp();
    const int64_t nb = p.eb_w;
    p.seq += (uint32_t)k;
    p.fs_top -= k;
    p.qh += k;
    p.qh &= p.Q - 1;
    p.qn -= k;
    p.qc0 += (typename Pt::Tm)k * p.dur_w;
    p.nA = p.nA > k ? p.nA - k : 0;
    reserve_add(p, nb, -k);
    resident_add(p, nb, k);
    p.n_recs += npf;
    p.pf_ev[2] += npf;
    // byte-accounting invariant (engine.py:216-236): checked on the general path
    // and in full-log runs (the parity tests); the uniform sweep kernels hold it
    // by construction (every landing was reserved)
    if (p.full && p.res_u + p.resv_u > p.cap_u && !p.err) p.err = -2;
}

template <class Pt>
DFI void settle(Pt& p) {                                                   // engine.py:422-442
    if (p.uniform) { settle_uniform(p); return; }
    while (p.qn > 0) {
        const int h = p.qh;
        const typename Pt::Tm comp = qcomp(p, 0);
        if (comp > p.now) break;
        const uint2 w = p.q_ent[h];
        const int ident = qe_ident(w);
        const uint8_t fl = qe_flags(w);
        const float score = qe_score(w);
        const int prec = (fl >> 2) & 3;
        const int64_t nb = peb(p, prec);
        if (p.fs_top <= 0) { p.err = -2; return; }
        const int slot = p.fs[p.fs_top - 1];
        __syncwarp();
        p.fs_top--;
        p.qh = (p.qh + 1) & (p.Q - 1);
        p.qn--;
        if (p.uniform) p.qc0 = comp + p.dur_w;       // the next entry's completion
        if (p.nA > 0) p.nA--;
        p.reserved_bytes -= nb;
        p.resident_bytes += nb;
        if (p.lane == 0) {
            p.rs[ident] = rs_make(prec, slot);
            p.res_ident[slot] = (int16_t)ident;
            if (p.miss == ESIM_MISS_SUBST) p.rscore[slot] = score;   // recorded_score: read by subst only
            if (p.hist[ident] == -2) p.hist[ident] = -1;
        }
        __syncwarp();
        if (p.resident_bytes + p.reserved_bytes > p.cap && !p.err) p.err = -2;
        note_admit(p, slot, ident);
        if (fl & 1) {
            const int il = ediv(p, ident);
            rec_prefetch(p, 2, il, ident - il * p.E, comp, score, 0);
        }
    }
}

template <class Pt>
DFI void advance_to(Pt& p, typename Pt::Tm t) {
    p.now = t;
    settle(p);
}

// _fetch (engine.py:463-510): blocked us, or -1 for None
template <class Pt>
DFI int64_t do_fetch(Pt& p, int ident, float gate, int prec, bool final) {
    const int64_t nb = peb(p, prec);
    if (p.uniform ? p.cap_u < 1 : nb > p.cap) {
        if (!final) return -1;
        p.err = -1;
        return 0;
    }
    while (no_room(p, nb) && !p.err) {
        const int v = select_victim(p, final);
        if (v >= 0) { evict(p, v, 0, final); continue; }
        if (!final) return -1;
        if (p.qn > 1 && p.qn - 1 - p.nA > 0) {                           // cancel newest pending = tail
            const QEntry e = q_load(p, p.qn - 1);
            __syncwarp();
            p.qn--;
            reserve_add(p, peb(p, (e.flags >> 2) & 3), -1);
            if (p.lane == 0) p.rs[e.ident] = 0;
            __syncwarp();
            const int il = ediv(p, e.ident);
            rec_prefetch(p, 4, il, e.ident - il * p.E, p.now, e.score, 4);
            continue;
        }
        if (p.qn == 0) { p.err = -2; return 0; }
        const typename Pt::Tm nd = qcomp(p, 0);
        advance_to(p, nd > p.now ? nd : p.now);
    }
    if (p.err) return 0;
    reserve_add(p, nb, 1);
    const int at = p.qn > 0 ? 1 + p.nA : 0;
    if (!q_open(p, at)) return 0;
    QEntry e;
    e.ident = (int16_t)ident; e.flags = (uint8_t)(prec << 2); e.score = gate;
    e.submit = p.now; e.comp = p.now + pdur(p, prec);
    if (p.lane == 0) { q_store(p, at, e); p.rs[ident] = RS_INF; }
    __syncwarp();
    if (at == 0 && p.uniform) p.qc0 = e.comp;
    if (at > 0) p.nA++;
    retime(p, at);
    const typename Pt::Tm comp = qcomp(p, at);
    const typename Pt::Tm blocked = comp - p.now;
    advance_to(p, comp);
    return blocked;
}

template <class Pt>
DFI void access_rec(Pt& p, int expert, int tokens, int rank, int outcome, int mclass, int64_t blocked, double wd,
                    int prec, int sub) {
    emit(p, ESIM_REC_ACCESS, p.layer, expert, tokens, rank,
         outcome | ((mclass < 0 ? 0xFF : mclass) << 8) | ((prec + 1) << 16), sub, blocked, 0, 0, wd);
    // per-layer counters in registers (outcome is a literal at every call site);
    // hits = demands - the rest, folded into smem after the layer (flush_layer_counts)
    if (outcome == 1 || outcome == 2) {
        p.lc_miss++;
        p.lc_c0 += mclass == 0;
        p.lc_c1 += mclass == 1;
    } else if (outcome == 3) {
        p.lc_drop++;
    } else if (outcome == 4) {
        p.lc_sub++;
    }
}

// the layer's access outcomes -> per-layer counters (totals[0..7] are their sums,
// formed at the end); n = the layer's demands, blocked = their summed blocked time
template <class Pt>
DFI void flush_layer_counts(Pt& p, int layer, int n, int64_t blocked) {
    if (p.lane == 0) {
        int32_t* pl = p.pl + layer * ESIM_PL_FIELDS;
        pl[0] += n;
        pl[1] += n - (int)(p.lc_miss + p.lc_drop + p.lc_sub);
        pl[2] += p.lc_miss;
        pl[3] += p.lc_c0;
        pl[4] += p.lc_c1;
        pl[5] += p.lc_miss - p.lc_c0 - p.lc_c1;
        pl[6] += p.lc_drop;
        pl[7] += p.lc_sub;
        if (blocked) p.ctr->sync_overhead += blocked;
    }
    p.lc_miss = p.lc_c0 = p.lc_c1 = p.lc_drop = p.lc_sub = 0;
}

// nearest-rank percentile (prefetch.py:30-36) of n floats in smem, warp-parallel
DFI float warp_nearest_rank(const float* v, int n, long rank, int lane) {
    float thr = 0.0f;
    bool found = false;
    for (int i = lane; i < n; i += 32) {
        const float x = v[i];
        int less = 0, le = 0;
        for (int j = 0; j < n; j++) { const float u = v[j]; less += u < x; le += u <= x; }
        if (less <= rank - 1 && rank - 1 < le) { thr = x; found = true; }
    }
    const unsigned who = __ballot_sync(FULL, found);
    return __shfl_sync(FULL, thr, __ffs(who) - 1);
}

// _handle_demand + resolve_miss: outcome 0 hit 1 fetch 2 wait 3 drop 4 subst, -1 error
template <class Pt>
DFI int handle_demand(Pt& p, int expert, int rank, float gate, double summed, int tokens, int nd,
                      int64_t& blocked, double& wd) {
    const EsimConfig* cfg = p.c;
    const int ident = p.layer * p.E + expert;
    blocked = 0;
    wd = 0.0;
    const uint16_t w = p.rs[ident];
    if (rs_res(w)) {
        const int prec = rs_prec(w), slot = rs_slot(w);
        note_access(p, ident, slot, true, (double)gate, prec);
        if (p.lane == 0 && p.miss == ESIM_MISS_SUBST) p.rscore[slot] = gate;
        __syncwarp();
        access_rec(p, expert, tokens, rank, 0, -1, 0, 0.0, prec, -1);
        return 0;
    }
    const int h = p.hist[ident];
    const int mclass = h == -2 ? 0 : (h == p.pass_id ? 1 : 2);
    if (w & RS_INF) {                                                     // promote + wait (engine.py:526-537)
        const int idx = q_find(p, ident);
        QEntry e = q_load(p, idx);
        e.flags |= 2;
        __syncwarp();
        int at = idx;
        if (idx == 0) {
            if (p.lane == 0) p.q_ent[qphys(p, 0)] = qe_make(e.ident, e.flags, e.score);
            __syncwarp();
        } else {
            const bool inA = idx <= p.nA;
            q_close(p, idx);
            if (inA) p.nA--;
            at = 1 + p.nA;
            q_open(p, at);
            if (p.lane == 0) q_store(p, at, e);
            __syncwarp();
            p.nA++;
            retime(p, min(idx, at));
        }
        const int prec = (e.flags >> 2) & 3;
        const typename Pt::Tm comp = qcomp(p, at);
        blocked = comp - p.now;
        advance_to(p, comp);
        const int slot = rs_slot(p.rs[ident]);
        note_access(p, ident, slot, true, (double)gate, prec);
        if (p.lane == 0 && p.miss == ESIM_MISS_SUBST) p.rscore[slot] = gate;
        __syncwarp();
        access_rec(p, expert, tokens, rank, 2, mclass, blocked, 0.0, prec, -1);
        return 2;
    }
    if (p.miss == ESIM_MISS_DROP && rank > cfg->drop_rank_threshold) {
        wd = -summed;
        access_rec(p, expert, tokens, rank, 3, -1, 0, wd, -1, -1);
        return 3;
    }
    if (p.miss == ESIM_MISS_SUBST) {                                     // find_substitute (miss.py:66-79)
        double bd = 0.0;
        int be = -1;
        for (int e0 = 0; e0 < p.E; e0 += 32) {
            const int e = e0 + p.lane;
            double diff = 0.0;
            bool ok = false;
            if (e < p.E) {
                const uint16_t ww = p.rs[p.layer * p.E + e];
                if (rs_res(ww)) {
                    diff = fabs(__dsub_rn((double)p.rscore[rs_slot(ww)], (double)gate));
                    ok = diff <= cfg->subst_tolerance;
                }
            }
            int ce = ok ? e : 0x7fffffff;
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(FULL, diff, o);
                const int oe = __shfl_xor_sync(FULL, ce, o);
                if (oe != 0x7fffffff && (ce == 0x7fffffff || od < diff || (od == diff && oe < ce))) {
                    diff = od;
                    ce = oe;
                }
            }
            if (ce != 0x7fffffff && (be < 0 || diff < bd)) { bd = diff; be = ce; }
        }
        if (be >= 0) {
            const uint16_t sw = p.rs[p.layer * p.E + be];
            const int sp = rs_prec(sw);
            note_access(p, p.layer * p.E + be, rs_slot(sw), false, 0.0, sp);
            wd = -summed;
            access_rec(p, expert, tokens, rank, 4, -1, 0, wd, sp, be);
            return 4;
        }
    }
    int prec = cfg->working_prec;
    int64_t b = -1;
    if (p.miss == ESIM_MISS_FETCH_LOW) {
        prec = cfg->precisions[cfg->n_precisions - 1];
        b = do_fetch(p, ident, gate, prec, true);
    } else if (p.miss == ESIM_MISS_FETCH_PRIORITY) {
        int start = 0;
        if (cfg->n_precisions > 1 && nd > 0) {
            long rk = (long)ceil(cfg->degrade_percentile / 100.0 * (double)nd);
            if (rk < 1) rk = 1;
            const float thr = warp_nearest_rank(p.lsc, nd, rk, p.lane);
            if ((double)gate < (double)thr) start = 1;
        }
        for (int i = start; i < cfg->n_precisions; i++) {
            prec = cfg->precisions[i];
            b = do_fetch(p, ident, gate, prec, i == cfg->n_precisions - 1);
            if (b >= 0 || p.err) break;
        }
        if (b < 0 && !p.err) p.err = -2;
    } else {
        b = do_fetch(p, ident, gate, prec, true);
    }
    if (p.err) return -1;
    const int slot = rs_slot(p.rs[ident]);
    note_access(p, ident, slot, true, (double)gate, prec);
    if (p.lane == 0 && p.miss == ESIM_MISS_SUBST) p.rscore[slot] = gate;
    __syncwarp();
    blocked = b;
    access_rec(p, expert, tokens, rank, 1, mclass, b, 0.0, prec, -1);
    return 1;
}

// sweep 2's victims for <= 128 slots: the `need` smallest keys in ascending
// order (LS: stale ones only), written to p.vict; K = the key width
template <typename K, class Pt>
DFI int merge_victims(Pt& p, int need, K FREE, bool& refusals) {
    K kk[4];
    int ss[4];
    #pragma unroll
    for (int j = 0; j < 4; j++) {
        const int sl = p.lane + 32 * j;
        kk[j] = sl < p.S ? (sizeof(K) == 8 ? (K)p.key[sl] : (K)reinterpret_cast<const uint32_t*>(p.key)[2 * sl]) : FREE;
        ss[j] = sl;
    }
    auto cx = [&](int a, int b) {
        const bool sw = kk[b] < kk[a];
        const K ka = kk[a], kb = kk[b];
        const int sa = ss[a], sb = ss[b];
        kk[a] = sw ? kb : ka; kk[b] = sw ? ka : kb;
        ss[a] = sw ? sb : sa; ss[b] = sw ? sa : sb;
    };
    cx(0, 1); cx(2, 3); cx(0, 2); cx(1, 3); cx(1, 2);
    int r = 0;
    while (r < need) {
        const K m = sizeof(K) == 8 ? (K)warp_min_u64((uint64_t)kk[0]) : (K)__reduce_min_sync(FULL, (uint32_t)kk[0]);
        if (m == FREE) break;                                         // no resident left: no_space drops
        if (p.pol == ESIM_EV_LS && ((uint64_t)m & LS_CURRENT)) { refusals = true; break; }
        const int wl = __ffs(__ballot_sync(FULL, kk[0] == m)) - 1;
        const int vs = __shfl_sync(FULL, ss[0], wl);
        if (p.lane == 0) p.vict[r] = (int16_t)vs;
        r++;
        if (p.lane == wl) {
            kk[0] = kk[1]; kk[1] = kk[2]; kk[2] = kk[3]; kk[3] = FREE;
            ss[0] = ss[1]; ss[1] = ss[2]; ss[2] = ss[3];
        }
    }
    return r;
}

// Watchdog sweep 2 (prefetch.py:199-221) for uniform instances under LRU / LS /
// LFU / LHU, batched. Every candidate needs exactly one expert's bytes, so the
// first `room` candidates start without evicting; each later one evicts the
// current minimum-key resident -- sweep 2 changes no key, so these victims
// are the residents in ascending key order (LS: stale ones only; a current
// minimum is a refusal, and so is every later candidate's); once no victim is
// left the rest are dropped "no_space". The victims are extracted with one
// warp min-reduction each; records (evict + started, or dropped) land at the
// positions their candidate order fixes and are written lane-parallel.
template <class Pt>
DFI void sweep2_uniform(Pt& p, const int32_t* pe, const float* ps, int nt, int target) {
    const int64_t nb = p.eb_w;
    const int wp = p.wp;
    int room = p.cap_u - p.res_u - p.resv_u;       // expert units (uniform path)
    if (room < 0) room = 0;
    const int F = nt < room ? nt : (int)room;
    const int need = nt - F;
    int r = 0;
    bool refusals = false;                     // LS: a current resident was the minimum
    if (need > 0) {
        const bool wide = p.pol == ESIM_EV_LFU || p.pol == ESIM_EV_LHU;   // 64-bit (count, touch) keys
        const uint32_t* k32 = reinterpret_cast<const uint32_t*>(p.key);
        // this lane's smallest key above `lo` (keys are unique; free slots hold the maximum)
        auto lane_min = [&](uint64_t lo, int& slot) -> uint64_t {
            uint64_t bk = wide ? KEY_FREE : 0xFFFFFFFFull;
            int bs = 0;
            for (int sl = p.lane; sl < p.S; sl += 32) {
                const uint64_t k = wide ? p.key[sl] : (uint64_t)k32[2 * sl];
                const bool better = k > lo && k < bk;
                bs = better ? sl : bs;
                bk = better ? k : bk;
            }
            slot = bs;
            return bk;
        };
        int lslot = 0;
        uint64_t lk = 0;
        if (p.S > 128) {                                               // first pass: no lower bound
            uint64_t bk = wide ? KEY_FREE : 0xFFFFFFFFull;
            int bs = 0;
            for (int sl = p.lane; sl < p.S; sl += 32) {
                const uint64_t k = wide ? p.key[sl] : (uint64_t)k32[2 * sl];
                bs = k < bk ? sl : bs;
                bk = k < bk ? k : bk;
            }
            lk = bk;
            lslot = bs;
        }
        const uint64_t FREE = wide ? KEY_FREE : 0xFFFFFFFFull;
        if (p.S <= 128) {
            // <= 4 slots per lane: each lane sorts its keys once (a 5-exchange
            // network in registers); the victims are then a 32-way merge of the
            // lanes' sorted lists -- the winner shifts its list instead of
            // rescanning its slots for the next key (LRU / LS: 32-bit keys)
            if (wide) r = merge_victims<uint64_t>(p, need, KEY_FREE, refusals);
            else r = merge_victims<uint32_t>(p, need, 0xFFFFFFFFu, refusals);
        } else {
            while (r < need) {
                const uint64_t m = wide ? warp_min_u64(lk) : (uint64_t)__reduce_min_sync(FULL, (uint32_t)lk);
                if (m == FREE) break;                                 // no resident left: no_space drops
                if (p.pol == ESIM_EV_LS && (m & LS_CURRENT)) { refusals = true; break; }
                const int wl = __ffs(__ballot_sync(FULL, lk == m)) - 1;
                const int vs = __shfl_sync(FULL, lslot, wl);
                if (p.lane == 0) p.vict[r] = (int16_t)vs;
                r++;
                if (p.lane == wl) lk = lane_min(m, lslot);
            }
        }
        __syncwarp();
    }
    const int started = F + r, dropped = nt - started;
    if (p.qn + started > p.Q) { p.err = STATUS_QUEUE_OVERFLOW; return; }
    const int32_t base = p.n_recs;
    uint32_t dg = 0;
    for (int b = 0; b < nt; b += 32) {
        const int t = b + p.lane;
        const bool act = t < nt;
        int e = 0;
        float sc = 0.0f;
        if (act) { const int j = p.tofetch[t]; e = pe[j]; sc = ps[j]; }
        const bool ev_rec = act && t >= F && t < started;
        const bool st = act && t < started;
        const bool dr = act && t >= started;
        const int32_t ri = base + (t < F ? t : (t < started ? F + 2 * (t - F) : F + 2 * r + (t - started)));
        int vid = 0, vslot = 0;
        if (ev_rec) { vslot = p.vict[t - F]; vid = p.res_ident[vslot]; }
        const int vl = ediv(p, vid);
        dg += lane_rec(p, ev_rec, ri, ESIM_REC_EVICT, p.layer, vl, vid - vl * p.E, wp, 1, 0, 0, 0, 0, 0.0);
        dg += lane_rec(p, st, ri + (ev_rec ? 1 : 0), ESIM_REC_PREFETCH, p.layer, 1, target, e, 0, 0, p.now, 0, 0,
                       (double)sc);
        dg += lane_rec(p, dr, ri, ESIM_REC_PREFETCH, p.layer, 4, target, e, 3, 0, p.now, 0, 0, (double)sc);
        __syncwarp();
        if (ev_rec) {                                                  // evict (engine.py:451-460)
            p.rs[vid] = 0;
            p.hist[vid] = (int16_t)p.pass_id;
            p.res_ident[vslot] = -1;
            p.key[vslot] = KEY_FREE;
            p.fs[p.fs_top + (t - F)] = (uint16_t)vslot;
        }
        if (st) {                                                      // reserve + channel.append
            const int x = qphys(p, p.qn + t);
            p.q_ent[x] = qe_make((int16_t)(target * p.E + e), (uint8_t)(1 | (wp << 2)), sc);
            p.rs[target * p.E + e] = RS_INF;
        }
    }
    digest_add_warp(p, dg);
    if (p.full) err_fold(p);
    __syncwarp();
    if (p.qn == 0 && started > 0) p.qc0 = p.now + p.dur_w;
    p.qn += started;
    p.fs_top += r;
    resident_add(p, nb, -r);
    reserve_add(p, nb, started);
    p.n_evict += r;
    p.pf_ev[1] += started;
    p.pf_ev[4] += dropped;
    p.n_recs += F + 2 * r + dropped;
    if (p.pol == ESIM_EV_LS && refusals) ctr_add(p, p.ctr->ls_refusals, dropped);
}

// _submit_prefetches + watchdog_step (engine.py:651-725, prefetch.py:163-221)
template <class Pt>
DFI void submit_prefetches(Pt& p, const EsimRouterOut& R, int tev) {   // tev < 2^31 / E events
    const int target = p.layer + 1;
    const int n = R.n_pred[tev];
    const int32_t* pe = R.pred_expert + tev * p.E;      // 32-bit index products (< 2^31)
    const float* ps = R.pred_score + tev * p.E;
    // PredictionRec: fixed by the router output (digest word from the summary;
    // the per-layer predicted-set sizes are added from it at the end)
    emit_mixed(p, p.digest_on ? R.pred_mix[tev] : 0u, ESIM_REC_PREDICTION, p.layer, target, n,
               p.full ? R.pred_clamped[tev] : 0, 0, 0, 0, 0, 0, 0.0, pe, n);
    const int wp = p.wp;
    const int64_t nb = peb(p, wp);
    const unsigned below = lanes_below(p.lane);
    // "predicted" records, one per prediction in order (lane j: prediction j)
    for (int b = 0; b < n; b += 32) {
        const int j = b + p.lane;
        const bool act = j < n;
        const int e = act ? pe[j] : 0;
        const float sc = act ? ps[j] : 0.0f;
        emit_lanes(p, act, p.lane, n - b < 32 ? n - b : 32, ESIM_REC_PREFETCH, p.layer, 0, target, e, 0, 0, p.now,
                   0, 0, (double)sc);
    }
    p.pf_ev[0] += n;
    // sweep 1, lane-parallel: resident -> (LS: first touch of the pass stamps the
    // key, in prediction order) "skip resident"; in flight -> "skip in flight";
    // otherwise compacted, in order, into the fetch list
    int nt = 0;
    for (int b = 0; b < n; b += 32) {
        const int j = b + p.lane;
        const bool act = j < n;
        int e = 0;
        float sc = 0.0f;
        uint16_t w = 0;
        if (act) { e = pe[j]; sc = ps[j]; w = p.rs[target * p.E + e]; }
        const bool res = act && rs_res(w);
        const bool inf = act && !res && (w & RS_INF);
        const bool fetch = act && !res && !inf;
        if (p.pol == ESIM_EV_LS) {
            const bool touch = res && !(p.key[rs_slot(w)] & LS_CURRENT);
            const unsigned tm = __ballot_sync(FULL, touch);
            if (touch) p.key[rs_slot(w)] = LS_CURRENT | (uint64_t)(p.seq + __popc(tm & below));
            p.seq += __popc(tm);
        }
        const unsigned hm = __ballot_sync(FULL, res || inf);
        emit_lanes(p, res || inf, __popc(hm & below), __popc(hm), ESIM_REC_PREFETCH, p.layer, 3, target, e,
                   res ? 1 : 2, 0, p.now, 0, 0, (double)sc);
        p.pf_ev[3] += __popc(hm);
        const unsigned fm = __ballot_sync(FULL, fetch);
        if (fetch) p.tofetch[nt + __popc(fm & below)] = (uint8_t)j;
        nt += __popc(fm);
    }
    __syncwarp();
    if (p.uniform && (p.pol == ESIM_EV_LRU || p.pol == ESIM_EV_LS || p.pol == ESIM_EV_LFU ||
                      p.pol == ESIM_EV_LHU)) {
        sweep2_uniform(p, pe, ps, nt, target);
        return;
    }
    for (int t = 0; t < nt && !p.err; t++) {                              // sweep 2 (serial)
        const int j = p.tofetch[t];
        const int e = pe[j];
        const float sc = ps[j];
        const int ident = target * p.E + e;
        bool refused = false;
        while (no_room(p, nb)) {
            const int v = select_victim(p, false);
            if (v < 0) { rec_prefetch(p, 4, target, e, p.now, sc, 3); refused = true; break; }
            evict(p, v, 1, false);
        }
        if (refused) continue;
        if (p.qn >= p.Q) { p.err = STATUS_QUEUE_OVERFLOW; return; }
        reserve_add(p, nb, 1);
        QEntry q;
        q.ident = (int16_t)ident; q.flags = (uint8_t)(1 | (wp << 2)); q.score = sc; q.submit = p.now;
        typename Pt::Tm start = p.now;
        if (p.qn) { const typename Pt::Tm tail = qcomp(p, p.qn - 1); start = p.now > tail ? p.now : tail; }
        q.comp = start + pdur(p, wp);
        if (p.qn == 0 && p.uniform) p.qc0 = q.comp;
        const int at = p.qn;
        __syncwarp();
        if (p.lane == 0) { q_store(p, at, q); p.rs[ident] = RS_INF; }
        __syncwarp();
        p.qn++;
        rec_prefetch(p, 1, target, e, p.now, sc, 0);
    }
}

// ---- cache-aware routing inside the loop (routing.py:143-161) -------------
// route one event with the cache-aware bias; fills the smem demand arrays
// (indexed by expert) and dem_expert_s (sorted order); returns the demand count
template <class Pt>
DFI int route_cache_aware(Pt& p, const EsimTraceDesc& tr, int64_t ev, int T, int64_t rows_before) {
    const int E = p.E, K = p.K, l = p.layer;
    const float* X = tr.logits + tr.row_offset[ev] * (int64_t)E;
    float* buf = p.ca_row;
    bool any_cached = false;
    for (int e = p.lane; e < E; e += 32) any_cached |= rs_res(p.rs[l * E + e]);
    any_cached = __any_sync(FULL, any_cached);
    int16_t orig[ESIM_MAX_K];
    for (int r = 0; r < T; r++) {
        const float* x = X + (int64_t)r * E;
        for (int i = p.lane; i < E; i += 32) buf[i] = x[i];
        __syncwarp();
        warp_softmax(buf, E, p.lane);                                     // original scores
        warp_topk(buf, E, K, p.lane, p.ca_sel + r * K);
        for (int j = 0; j < K; j++) orig[j] = p.ca_sel[r * K + j];
        const int64_t dcount = (rows_before + r) * (int64_t)E;
        const double mean = dcount ? __ddiv_rn(p.dsum[l], (double)dcount) : 0.0;
        __syncwarp();
        for (int i = p.lane; i < E; i += 32) p.dem_gate_s[i] = buf[i];     // keep original scores
        __syncwarp();
        const bool bias_on = p.c->lam != 0.0 && mean != 0.0 && any_cached;
        const float bias = __double2float_rn(__dmul_rn(p.c->lam, mean));
        for (int i = p.lane; i < E; i += 32) {
            float v = x[i];
            if (bias_on && rs_res(p.rs[l * E + i])) v = __fadd_rn(v, bias);
            buf[i] = v;
        }
        __syncwarp();
        warp_softmax(buf, E, p.lane);
        warp_topk(buf, E, K, p.lane, p.ca_sel + r * K);
        for (int i = p.lane; i < E; i += 32) buf[i] = x[i];                // DeltaAvg update after the row
        __syncwarp();
        const double rsum = __dadd_rn(0.0, warp_pw_sum_f64(buf, E, p.lane));
        if (p.lane == 0) p.dsum[l] = __dadd_rn(p.dsum[l], rsum);
        bool same = true;
        for (int a = 0; a < K; a++) {
            const int s = p.ca_sel[r * K + a];
            bool f = false;
            for (int b = 0; b < K; b++) f |= (s == orig[b]);
            same &= f;
        }
        if (p.lane == 0) {
            p.ca_mod[r] = same ? 0 : 1;
            for (int a = 0; a < K; a++) p.ca_w[r * K + a] = p.dem_gate_s[p.ca_sel[r * K + a]];
        }
        __syncwarp();
    }
    for (int e0 = 0; e0 < E; e0 += 32) {                                  // _aggregate_demand
        const int e = e0 + p.lane;
        if (e >= E) continue;
        int rank = 0x7fffffff, tok = 0;
        float gate = -1.0f;
        double summed = 0.0;
        for (int r = 0; r < T; r++)
            for (int j = 0; j < K; j++)
                if (p.ca_sel[r * K + j] == e) {
                    const float wv = p.ca_w[r * K + j];
                    rank = min(rank, j + 1);
                    gate = fmaxf(gate, wv);
                    summed = tok ? __dadd_rn(summed, (double)wv) : (double)wv;
                    tok++;
                }
        p.dem_rank_s[e] = tok ? rank : 0x7fffffff;
        p.dem_gate_s[e] = gate;
        p.dem_summed_s[e] = summed;
        p.dem_tokens_s[e] = tok;
    }
    __syncwarp();
    int cnt = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {                                  // order (rank, -gate, expert)
        const int e = e0 + p.lane;
        int pos = -1;
        if (e < E && p.dem_rank_s[e] != 0x7fffffff) {
            const int rk = p.dem_rank_s[e];
            const float g = p.dem_gate_s[e];
            pos = 0;
            for (int j = 0; j < E; j++) {
                const int rj = p.dem_rank_s[j];
                if (rj == 0x7fffffff || j == e) continue;
                const float gj = p.dem_gate_s[j];
                pos += (rj < rk) || (rj == rk && (gj > g || (gj == g && j < e)));
            }
        }
        cnt += __popc(__ballot_sync(FULL, pos >= 0));
        if (e < E) reinterpret_cast<int*>(p.ca_row)[e] = pos;            // routing done: int scratch
    }
    __syncwarp();
    for (int e = p.lane; e < E; e += 32) {
        const int pos = reinterpret_cast<int*>(p.ca_row)[e];
        if (pos >= 0) p.dem_expert_s[pos] = e;
    }
    __syncwarp();
    return cnt;
}

// ---------------------------------------------------------------------------
// Common-path launches are persistent with one CTA of kPersistWarps warps per SM
// (registers <= 65536 / (32 * 12) = 170 per thread): an SM then only ever runs
// one policy's kernel -- two policies' ~80 KB instruction streams sharing an SM
// thrash its instruction cache -- and its warps pull points longest-first.
#ifndef REPLAY_WARPS
#define REPLAY_WARPS 12
#endif
constexpr int kPersistWarps = REPLAY_WARPS;
// POL: eviction policy; GEN: 0 = the common case (miss=fetch, standard routing) with every
// other miss/routing path compiled out, 1 = all paths. Every helper is force-inlined, so the
// compile-time policy/miss constants delete the other policies' code from the kernel.
// LOG: 0 = digest only, no record log (compile-time: the log-writing code is gone
// from the kernel), 1 = per-point runtime flags (full log and/or digest)
template <int POL, int GEN, int LOG, int T32>
DFI void replay_point(const ReplayArgs& A, const int pid, unsigned char* base) {
    using Tm = typename std::conditional<T32 != 0, int32_t, int64_t>::type;
    const int64_t orow = A.out_index ? A.out_index[pid] : pid;      // where this point's results go
    const EsimConfig* cfg = &A.cfg[pid];
    const EsimTraceDesc tr = A.traces[cfg->trace_id];
    const EsimRouterOut R = A.routers[cfg->trace_id];
    const bool ca = GEN && cfg->routing == ESIM_ROUTE_CACHE_AWARE;
    const Layout& lay = A.lay;

    long long t_begin;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    PtT<Tm> p;
    p.c = cfg;
    p.L = cfg->num_layers; p.E = cfg->experts; p.K = cfg->top_k;
    const int N = p.L * p.E;
    p.lane = threadIdx.x & 31;
    p.pol = POL;
    p.miss = GEN ? cfg->miss : ESIM_MISS_FETCH;
    if (cfg->eviction != POL || (!GEN && (cfg->miss != ESIM_MISS_FETCH || cfg->routing != ESIM_ROUTE_STANDARD))) {
        if ((threadIdx.x & 31) == 0) A.counters[orow].status = -1;     // dispatch error
        return;
    }
    p.cap = cfg->capacity_bytes;
    const int64_t bw = cfg->bandwidth;
    int64_t minb = INT64_MAX;
    int64_t durs[4], ebs[4];
    #pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t nb = cfg->expert_bytes[i];
        ebs[i] = nb;
        durs[i] = (bw == 0 || nb == 0) ? 0 : (nb * 1000000 + bw - 1) / bw;
        if (nb > 0 && nb < minb) minb = nb;
    }
    p.eb0 = ebs[0]; p.eb1 = ebs[1]; p.eb2 = ebs[2]; p.eb3 = ebs[3];
    p.dur0 = (Tm)durs[0]; p.dur1 = (Tm)durs[1]; p.dur2 = (Tm)durs[2]; p.dur3 = (Tm)durs[3];
    p.uniform = !GEN;
    p.wp = cfg->working_prec;
    p.eb_w = ebs[cfg->working_prec & 3];
    p.dur_w = durs[cfg->working_prec & 3];
    p.inv_dur = p.dur_w > 0 ? 1.0 / (double)p.dur_w : 0.0;
    // residents + queued transfers <= capacity / (smallest expert this point can admit):
    // only fetch_low / fetch_priority ever admit below the working precision
    if (p.miss != ESIM_MISS_FETCH_LOW && p.miss != ESIM_MISS_FETCH_PRIORITY) minb = peb(p, cfg->working_prec);
    int64_t slots = p.cap / minb;
    if (slots > N) slots = N;
    if (slots > A.S) slots = A.S;
    p.S = (int)slots;
    p.Q = A.Q;
    p.key = reinterpret_cast<uint64_t*>(base + lay.key);
    p.q_submit = reinterpret_cast<int64_t*>(base + lay.q_submit);
    p.q_comp = reinterpret_cast<int64_t*>(base + lay.q_comp);
    p.dsum = reinterpret_cast<double*>(base + lay.dsum);
    p.ctr = reinterpret_cast<Ctr*>(base + lay.ctr);
    p.dem_summed_s = reinterpret_cast<double*>(base + lay.dem_summed);
    p.cnt = reinterpret_cast<uint16_t*>(base + lay.cnt);
    p.rscore = reinterpret_cast<float*>(base + lay.rscore);
    p.pl = reinterpret_cast<int32_t*>(base + lay.pl);
    p.demmask = reinterpret_cast<uint32_t*>(base + lay.demmask);
    p.lsc = reinterpret_cast<float*>(base + lay.lsc);
    p.ca_w = reinterpret_cast<float*>(base + lay.ca_w);
    p.ca_row = reinterpret_cast<float*>(base + lay.ca_row);
    p.dem_gate_s = reinterpret_cast<float*>(base + lay.dem_gate);
    p.dem_tokens_s = reinterpret_cast<int32_t*>(base + lay.dem_tokens);
    p.dem_expert_s = reinterpret_cast<int32_t*>(base + lay.dem_expert);
    p.dem_rank_s = reinterpret_cast<int32_t*>(base + lay.dem_rank);
    p.rs = reinterpret_cast<uint16_t*>(base + lay.rs);
    p.hist = reinterpret_cast<int16_t*>(base + lay.hist);
    p.res_ident = reinterpret_cast<int16_t*>(base + lay.res_ident);
    p.fs = reinterpret_cast<uint16_t*>(base + lay.fs);
    p.q_ent = reinterpret_cast<uint2*>(base + lay.q_ent);
    p.ca_sel = reinterpret_cast<int16_t*>(base + lay.ca_sel);
    p.vict = reinterpret_cast<int16_t*>(base + lay.vict);
    p.tofetch = base + lay.tofetch;
    p.ca_mod = base + lay.ca_mod;

    const bool lfu = p.pol == ESIM_EV_LFU || p.pol == ESIM_EV_LHU;
    for (int i = p.lane; i < N; i += 32) {
        p.rs[i] = 0;
        p.hist[i] = -2;
        if (lfu) p.cnt[i] = 0;
    }
    for (int i = p.lane; i < p.S; i += 32) { p.res_ident[i] = -1; p.key[i] = KEY_FREE; p.fs[i] = (uint16_t)(p.S - 1 - i); }
    for (int i = p.lane; i < p.L * ESIM_PL_FIELDS; i += 32) p.pl[i] = 0;
    if (ca) for (int i = p.lane; i < p.L; i += 32) p.dsum[i] = 0.0;
    {
        uint32_t* cw = reinterpret_cast<uint32_t*>(p.ctr);
        for (int i = p.lane; i < (int)(sizeof(Ctr) / 4); i += 32) cw[i] = 0;
    }
    __syncwarp();
    p.now = 0; p.resident_bytes = 0; p.reserved_bytes = 0;
    p.res_u = 0; p.resv_u = 0;
    p.cap_u = p.uniform ? (int32_t)((p.eb_w > 0 ? p.cap / p.eb_w : 0) < 0x7FFFFFFF ? (p.eb_w > 0 ? p.cap / p.eb_w : 0)
                                                                                  : 0x7FFFFFFF) : 0;
    p.qh = 0; p.qn = 0; p.nA = 0; p.fs_top = p.S; p.seq = 0; p.qc0 = 0;
    p.einv = ((1ull << 32) + (uint64_t)p.E - 1) / (uint64_t)p.E;
    p.digest = 0u; p.digest_u = (uint32_t)FNV_OFFSET; p.n_recs = 0; p.n_pe = 0;
    p.n_evict = 0; p.n_forced = 0;
    p.lc_miss = p.lc_c0 = p.lc_c1 = p.lc_drop = p.lc_sub = 0;
    #pragma unroll
    for (int i = 0; i < 5; i++) p.pf_ev[i] = 0;
    p.err = 0;
    p.full = LOG ? ((cfg->flags & ESIM_FLAG_FULL_LOG) && A.recs != nullptr) : false;
    p.digest_on = LOG ? (cfg->flags & ESIM_FLAG_NO_DIGEST) == 0 : true;
    p.recs = A.recs + orow * A.rec_cap;
    p.rec_cap = A.rec_cap;
    p.pexp = A.pexp + orow * A.pe_cap;
    p.pe_cap = A.pe_cap;
    if (ca && (p.E > A.Emax || A.Tmax == 0)) p.err = -1;
    if (lfu && !A.has_cnt) p.err = -1;
    int64_t rows_before = 0;

    for (int pass = 0; pass < tr.n_passes && !p.err; pass++) {
        p.pass_id = pass;
        if (p.pol == ESIM_EV_LS) {                                        // begin_pass (eviction.py:262-268)
            for (int s = p.lane; s < p.S; s += 32) {               // free slots keep KEY_FREE
                const uint64_t k = p.key[s];
                p.key[s] = k == KEY_FREE ? k : (k & ~LS_CURRENT);
            }
        } else if (p.pol == ESIM_EV_SB) {                                 // eviction.py:195-197
            for (int s = p.lane; s < p.S; s += 32)
                if (p.res_ident[s] >= 0)
                    p.key[s] = (uint64_t)__double_as_longlong(
                        __dmul_rn(__longlong_as_double((long long)p.key[s]), cfg->sb_decay));
        }
        __syncwarp();
        const int64_t pstart = p.now;
        int64_t pblocked = 0;
        for (int l = 0; l < p.L && !p.err; l++) {
            p.layer = l;
            if (p.seq > SEQ_LIMIT) { p.err = STATUS_SEQ_OVERFLOW; break; }
            const int ev = pass * p.L + l;                        // events and ev * E stay below 2^31
            settle(p);
            const int T = (int)(tr.row_offset[ev + 1] - tr.row_offset[ev]);
            int nd;
            const int32_t *d_exp, *d_rank, *d_tok;
            const float* d_gate;
            const double* d_sum;
            if (ca) {
                nd = route_cache_aware(p, tr, ev, T, rows_before);
                d_exp = p.dem_expert_s; d_rank = p.dem_rank_s; d_gate = p.dem_gate_s;
                d_sum = p.dem_summed_s; d_tok = p.dem_tokens_s;
            } else {
                nd = R.n_dem[ev];
                d_exp = R.dem_expert + ev * p.E; d_rank = R.dem_rank + ev * p.E; d_gate = R.dem_gate + ev * p.E;
                d_sum = R.dem_summed + ev * p.E; d_tok = R.dem_tokens + ev * p.E;
            }
            if (p.miss == ESIM_MISS_FETCH_PRIORITY) {                    // layer scores in demand order
                for (int i = p.lane; i < nd; i += 32) p.lsc[i] = ca ? d_gate[d_exp[i]] : d_gate[i];
                __syncwarp();
            }
            // prefetch P/R (metrics.py:150-187): router-only under standard routing
            // (taken from the router summary at the end); per point only when
            // cache-aware routing changes the demand sets
            if (ca && cfg->prefetch != ESIM_PF_NONE && l >= 1) {
                for (int i = p.lane; i < (p.E + 31) / 32; i += 32) p.demmask[i] = 0;
                __syncwarp();
                for (int i = p.lane; i < nd; i += 32) atomicOr(&p.demmask[d_exp[i] >> 5], 1u << (d_exp[i] & 31));
                __syncwarp();
                const int np = R.n_pred[ev];
                int inter = 0;
                for (int j = p.lane; j < np; j += 32) {
                    const int e = R.pred_expert[ev * p.E + j];
                    inter += (p.demmask[e >> 5] >> (e & 31)) & 1;
                }
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(FULL, inter, o);
                if (p.lane == 0) {
                    Ctr* c = p.ctr;
                    c->pf_tp += inter; c->pf_pred += np; c->pf_dem += nd; c->pf_records++;
                    if (np) c->pf_prec_parts++; else c->pf_empty++;
                    c->pf_rec_parts++;
                }
                if (np) ps_add(p, 2, __ddiv_rn((double)inter, (double)np));
                ps_add(p, 3, __ddiv_rn((double)inter, (double)nd));
            }
            int64_t blocked = 0;
            double wdelta = 0.0;
            bool any_aff = false;
            if (p.miss == ESIM_MISS_DROP || p.miss == ESIM_MISS_SUBST) {
                for (int i = p.lane; i < (p.E + 31) / 32; i += 32) p.demmask[i] = 0;
                __syncwarp();
            }
            for (int i = 0; i < nd && !p.err; i++) {
                const int e = d_exp[i];
                const int k = ca ? e : i;
                int64_t b;
                double wd;
                const int oc = handle_demand(p, e, d_rank[k], d_gate[k], d_sum[k], d_tok[k], nd, b, wd);
                blocked += b;
                wdelta = __dadd_rn(wdelta, wd);
                if (oc == 3 || oc == 4) {
                    any_aff = true;
                    if (p.lane == 0) p.demmask[e >> 5] |= 1u << (e & 31);
                    __syncwarp();
                }
            }
            if (p.err) break;
            flush_layer_counts(p, l, nd, blocked);
            int faithful = T, nmod = 0;                                   // RouteRec (engine.py:625-643)
            if (!GEN) {
                // standard routing, every demand served: the record is the router's
                // (digest word and mass sums from the summary)
                const double origm = R.sel_mass[ev];
                emit_mixed(p, p.digest_on ? R.route_mix[ev] : 0u, ESIM_REC_ROUTE, l, T, T, 0, 0, 0, 0,
                           __double_as_longlong(origm), __double_as_longlong(__dadd_rn(origm, 0.0)), origm);
            } else {
            if (ca || any_aff) {
                const int16_t* rsel = ca ? p.ca_sel : R.row_sel + tr.row_offset[ev] * p.K;
                int bad = 0;
                for (int r = p.lane; r < T; r += 32) {
                    bool hit = ca && p.ca_mod[r] != 0;
                    if (ca) nmod += p.ca_mod[r];
                    if (any_aff)
                        for (int j = 0; j < p.K; j++) {
                            const int s = rsel[r * p.K + j];
                            hit |= (p.demmask[s >> 5] >> (s & 31)) & 1;
                        }
                    bad += hit;
                }
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    bad += __shfl_xor_sync(FULL, bad, o);
                    nmod += __shfl_xor_sync(FULL, nmod, o);
                }
                faithful = T - bad;
            }
            const double origm = R.sel_mass[ev];
            double selm = origm;
            if (ca) {
                PySum outer;
                outer.init();
                for (int r = 0; r < T; r++) {
                    PySum in;
                    in.init();
                    for (int j = 0; j < p.K; j++) in.add((double)p.ca_w[r * p.K + j]);
                    outer.add(in.value());
                }
                selm = outer.value();
            }
            const double exm = __dadd_rn(selm, wdelta);
            emit(p, ESIM_REC_ROUTE, l, T, faithful, nmod, 0, 0, 0, __double_as_longlong(origm),
                 __double_as_longlong(exm), selm);
            if (p.lane == 0) { p.ctr->faithful += faithful; p.ctr->modified += nmod; }
            ps_add(p, 1, exm);                   // rows and the original mass: router summary
            if (ca && A.progress) {
                // streamed (physical layer step): the executed routing of this event's rows
                // replaces the router's standard top-k in place before the layer is published
                // (the FFN builds its token lists from these rows; routing.py:147-160)
                const int64_t b0 = tr.row_offset[ev] * p.K;
                for (int i = p.lane; i < T * p.K; i += 32) {
                    R.row_sel[b0 + i] = p.ca_sel[i];
                    R.row_w[b0 + i] = p.ca_w[i];
                }
                __threadfence();
                __syncwarp();
            }
            }
            if (cfg->prefetch != ESIM_PF_NONE && l + 1 < p.L) submit_prefetches(p, R, ev + 1);
            advance_to(p, p.now + (Tm)cfg->compute_us);
            pblocked += blocked;
            if (A.progress && p.lane == 0) {             // publish this layer's decisions to the host
                __threadfence_system();
                A.progress[1 + ev] = p.n_recs;
                __threadfence_system();
                A.progress[0] = ev + 1;
            }
        }
        if (p.err) break;
        emit(p, ESIM_REC_PASS, 0, tr.pass_kind[pass], tr.pass_tokens[pass], 0, 0, 0, pstart, p.now, pblocked, 0.0);
        if (p.lane == 0) {
            Ctr* c = p.ctr;
            c->passes++;
            if (pass == 0) c->ttft = p.now;
            c->total = p.now;
            if (tr.pass_kind[pass] == 1) { c->decode_passes++; c->decode_us += p.now - pstart; }
        }
        rows_before += tr.pass_tokens[pass];
    }
    __syncwarp();
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) p.digest += __shfl_xor_sync(FULL, p.digest, o);   // fold the lane partials
    p.digest += p.digest_u;
    if (A.progress && p.lane == 0) {
        __threadfence_system();
        A.progress[0] = p.err ? -1 : (int64_t)tr.n_passes * p.L + 1;    // +1: final PassRec written
    }
    if (p.lane == 0) {
        const Ctr* c = p.ctr;
        EsimCounters* o = &A.counters[orow];
        for (int i = 0; i < 8; i++) {
            int64_t t = 0;
            for (int l = 0; l < p.L; l++) t += p.pl[l * ESIM_PL_FIELDS + i];
            o->totals[i] = t;
        }
        o->totals[8] = p.n_evict;
        o->totals[9] = p.n_forced;
        for (int i = 0; i < 5; i++) o->totals[10 + i] = p.pf_ev[i];
        o->ttft_us = c->ttft; o->total_us = c->total; o->decode_us = c->decode_us;
        o->sync_overhead_us = c->sync_overhead; o->passes = c->passes; o->decode_passes = c->decode_passes;
        // router-only parts from the summary (router.cu route_totals_kernel)
        const EsimRouteSummary& S = *R.summary;
        o->rows_total = S.rows_total;
        o->faithful_rows = GEN ? (int64_t)c->faithful : S.rows_total;
        o->modified_rows = GEN ? (int64_t)c->modified : 0;
        double fc[8] = {S.orig_f, S.orig_c, S.orig_f, S.orig_c, S.prec_f, S.prec_c, S.rec_f, S.rec_c};
        if (GEN) { fc[2] = c->ps[2]; fc[3] = c->ps[3]; }
        if (ca) {
            o->pf_tp = c->pf_tp; o->pf_pred_total = c->pf_pred; o->pf_dem_total = c->pf_dem;
            o->pf_records = c->pf_records; o->pf_empty = c->pf_empty; o->pf_prec_parts = c->pf_prec_parts;
            o->pf_rec_parts = c->pf_rec_parts;
            for (int i = 4; i < 8; i++) fc[i] = c->ps[i];
        } else {
            o->pf_tp = S.pf_tp; o->pf_pred_total = S.pf_pred; o->pf_dem_total = S.pf_dem;
            o->pf_records = S.pf_records; o->pf_empty = S.pf_empty; o->pf_prec_parts = S.pf_prec_parts;
            o->pf_rec_parts = S.pf_rec_parts;
        }
        o->ls_forced = c->ls_forced; o->ls_unforced = 0; o->ls_refusals = c->ls_refusals;
        o->n_recs = p.n_recs; o->n_pred_experts = p.n_pe; o->digest = p.digest;
        double* vo = &o->original_mass;
        for (int i = 0; i < 4; i++) {
            const double f = fc[2 * i], cc = fc[2 * i + 1];
            vo[i] = (cc != 0.0 && isfinite(cc)) ? __dadd_rn(f, cc) : f;
        }
        o->status = p.err;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        o->pad[0] = t_begin;                 // scheduling diagnostics: globaltimer ns at start / end, SM id
        o->pad[1] = t_end;
        o->pad[2] = smid;
    }
    int64_t* plo = A.per_layer + orow * A.Lmax * ESIM_PL_FIELDS;
    for (int i = p.lane; i < A.Lmax * ESIM_PL_FIELDS; i += 32) {
        int64_t v = 0;
        if (i < p.L * ESIM_PL_FIELDS) {
            const int l = i / ESIM_PL_FIELDS, f = i - l * ESIM_PL_FIELDS;
            v = f < 8 ? (int64_t)p.pl[i] : R.layer_pred[2 * l + (f - 8)];   // 8, 9: predicted-set sizes (router)
        }
        plo[i] = v;
    }
}

template <int POL, int GEN, int LOG, int T32>
__global__ void __launch_bounds__(GEN ? 128 : 32 * kPersistWarps, 1) replay_kernel(ReplayArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int wid = threadIdx.x >> 5;
    unsigned char* base = smem_raw + (size_t)wid * A.point_bytes;
    if (A.work == nullptr) {                         // one point per warp
        const int pid = blockIdx.x * A.warps_per_cta + wid;
        if (pid < A.n_points) replay_point<POL, GEN, LOG, T32>(A, pid, base);
        return;
    }
    // persistent: every warp pulls the next point of the launch order (longest
    // first) as soon as it is free -- greedy LPT packing across the whole grid
    for (;;) {
        int pid = 0;
        if ((threadIdx.x & 31) == 0) pid = atomicAdd(A.work, 1);
        pid = __shfl_sync(FULL, pid, 0);
        if (pid >= A.n_points) break;
        replay_point<POL, GEN, LOG, T32>(A, pid, base);
        __syncwarp();
    }
}

}  // namespace esim

// one work counter per stream (launches on a stream are ordered, so they share it)
static cudaError_t work_counter(cudaStream_t st, int** out) {
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, int*> ctr;
    std::lock_guard<std::mutex> lock(mu);
    int*& c = ctr[st];
    if (!c) {
        const cudaError_t e = cudaMalloc((void**)&c, sizeof(int));
        if (e != cudaSuccess) { c = nullptr; return e; }
    }
    *out = c;
    return cudaSuccess;
}

int esim_replay_smem_bytes(int N, int S, int Q, int L, int E, int T, int K, bool ca, bool has_cnt, bool gen) {
    return esim::make_layout(N, S, Q, L, E, T, K, ca, has_cnt, gen).total;
}

cudaError_t esim_replay_launch_impl(const EsimConfig* d_cfg, int n, const EsimTraceDesc* d_traces,
                                    const EsimRouterOut* d_routers, EsimCounters* d_counters,
                                    int64_t* d_per_layer, EsimRec* d_recs, int64_t rec_cap, int32_t* d_pexp,
                                    int64_t pe_cap, int N, int S, int Q, int Lmax, int Emax, int Tmax, int Kmax,
                                    bool has_cnt, int warps_per_cta, cudaStream_t st, int64_t* progress,
                                    int policy, bool general, const int32_t* out_index, bool log_rt,
                                    int max_ctas, bool time32) {
    esim::ReplayArgs a;
    a.progress = progress;
    a.out_index = out_index;
    a.cfg = d_cfg; a.n_points = n; a.traces = d_traces; a.routers = d_routers;
    a.counters = d_counters; a.per_layer = d_per_layer; a.recs = d_recs; a.rec_cap = rec_cap;
    a.pexp = d_pexp; a.pe_cap = pe_cap;
    a.N = N; a.S = S; a.Q = Q; a.Lmax = Lmax; a.Emax = Emax; a.Tmax = Tmax; a.Kmax = Kmax;
    a.has_cnt = has_cnt ? 1 : 0;
    a.warps_per_cta = warps_per_cta;
    a.lay = esim::make_layout(N, S, Q, Lmax, Emax, Tmax, Kmax, Tmax > 0, has_cnt, general);
    a.point_bytes = a.lay.total;
    a.work = nullptr;
    const size_t smem = (size_t)a.point_bytes * warps_per_cta;
    int blocks = (n + warps_per_cta - 1) / warps_per_cta;
    void (*k)(esim::ReplayArgs) = nullptr;
#define ESIM_PICK(P)                                                                   \
    case P: k = general ? esim::replay_kernel<P, 1, 1, 0>                              \
                        : (log_rt ? (time32 ? esim::replay_kernel<P, 0, 1, 1> : esim::replay_kernel<P, 0, 1, 0>) \
                                  : (time32 ? esim::replay_kernel<P, 0, 0, 1> : esim::replay_kernel<P, 0, 0, 0>)); \
        break;
    switch (policy) {
        ESIM_PICK(ESIM_EV_LRU) ESIM_PICK(ESIM_EV_LFU) ESIM_PICK(ESIM_EV_LHU)
        ESIM_PICK(ESIM_EV_FLD) ESIM_PICK(ESIM_EV_SB) ESIM_PICK(ESIM_EV_LS)
        default: return cudaErrorInvalidValue;
    }
#undef ESIM_PICK
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // Shared-memory carveout experiment hook (percent; unset = driver default).
    // Forcing one carveout on every specialisation lets the concurrent group
    // launches co-reside from the start, but measured slower overall on the
    // C5 step (72 ms at 100 %, 73 at 72 %, 80 at 58 % vs 66 ms default).
    static const int carve = getenv("ESIM_CARVEOUT") ? atoi(getenv("ESIM_CARVEOUT")) : -1;
    if (carve >= 0) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        if (e != cudaSuccess) return e;
    }
    if (!general && !progress) {
        // persistent: one resident wave of warps pulls the points (launch order =
        // longest estimated first) from a per-stream work counter; as many warps
        // per CTA as shared memory allows, up to one SM's worth
        int w = esim::kPersistWarps;
        while (w > 1 && (size_t)a.point_bytes * w > 227 * 1024) w--;
        a.warps_per_cta = w;
        warps_per_cta = w;
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t psmem = (size_t)a.point_bytes * w;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem)) != cudaSuccess)
            return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32 * w, psmem)) != cudaSuccess) return e;
        blocks = (n + w - 1) / w;
        const int wave = sms * (per > 0 ? per : 1);
        if (blocks > wave) blocks = wave;
        if (max_ctas > 0 && blocks > max_ctas) blocks = max_ctas;   // this launch's share of the SMs
        if ((e = work_counter(st, &a.work)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(a.work, 0, sizeof(int), st)) != cudaSuccess) return e;
    }
    k<<<blocks, 32 * warps_per_cta, (size_t)a.point_bytes * warps_per_cta, st>>>(a);
    return cudaGetLastError();
}

int esim_replay_set_sum_plain(int plain) {          // see esim_set_host_sum
    return cudaMemcpyToSymbol(esim::g_pysum_plain, &plain, sizeof(int)) == cudaSuccess ? 0 : -2;
}
