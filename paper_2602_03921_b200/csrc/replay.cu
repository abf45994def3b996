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
// Device-native structures instead of the reference's containers: the
// directory is flat shared-memory arrays indexed by ident = layer*E+expert
// plus a slot table of residents carrying one 64-bit policy key; every
// victim choice is a warp argmin over the slot table (LS: class bit | gen,
// LRU: stamp, LFU: count then touch, FLD: cyclic distance, SB: fp64 signal).
// The channel is a ring buffer whose retiming is a warp max-plus scan.
// Scalars are computed redundantly by all 32 lanes (warp-uniform control
// flow); lane 0 owns counters and record output.
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/specmd_b200.h"
#include "numpy_f32.cuh"

namespace esim {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t FNV_OFFSET = 0xcbf29ce484222325ULL;
constexpr uint64_t FNV_PRIME = 0x100000001b3ULL;

struct ReplayArgs {
    const EsimConfig* cfg;
    int n_points;
    const EsimTraceDesc* traces;   // device copies of the descriptors (device pointers inside)
    const EsimRouterOut* routers;
    EsimCounters* counters;
    int64_t* per_layer;            // [n][Lmax][ESIM_PL_FIELDS]
    EsimRec* recs;
    int64_t rec_cap;
    int32_t* pexp;
    int64_t pe_cap;
    int N, S, Q, Lmax, Emax, Tmax, Kmax;  // smem sizing (max over points)
    int warps_per_cta;
    int point_bytes;
};

// shared-memory layout of one point (offsets in bytes, 8-byte aligned blocks)
struct Layout {
    int key, q_submit, q_start, q_comp, dsum;          // 8-byte arrays
    int cnt, rscore, q_score, pl, demmask, ca_w, dem_gate, dem_summed;  // 4/8-byte
    int hist, slot_of, res_ident, q_ident, ca_sel;     // 2-byte
    int st, q_flags, tofetch, ca_mod, dem_rank;        // 1-byte
    int ca_row, dem_expert, dem_tokens, lsc;
    int total;
};

__host__ __device__ inline int al8(int x) { return (x + 7) & ~7; }

__host__ __device__ inline Layout make_layout(int N, int S, int Q, int L, int E, int T, int K, bool ca) {
    Layout l;
    int o = 0;
    l.key = o; o += al8(S * 8);
    l.q_submit = o; o += al8(Q * 8);
    l.q_start = o; o += al8(Q * 8);
    l.q_comp = o; o += al8(Q * 8);
    l.dsum = o; o += al8(L * 8);
    l.dem_summed = o; o += al8(ca ? E * 8 : 0);
    l.cnt = o; o += al8(N * 4);
    l.rscore = o; o += al8(S * 4);
    l.q_score = o; o += al8(Q * 4);
    l.pl = o; o += al8(L * ESIM_PL_FIELDS * 4);
    l.demmask = o; o += al8(((E + 31) / 32) * 4);
    l.lsc = o; o += al8(E * 4);
    l.ca_w = o; o += al8(ca ? T * K * 4 : 0);
    l.ca_row = o; o += al8(ca ? E * 4 : 0);
    l.dem_gate = o; o += al8(ca ? E * 4 : 0);
    l.dem_tokens = o; o += al8(ca ? E * 4 : 0);
    l.dem_expert = o; o += al8(ca ? E * 4 : 0);
    l.hist = o; o += al8(N * 2);
    l.slot_of = o; o += al8(N * 2);
    l.res_ident = o; o += al8(S * 2);
    l.q_ident = o; o += al8(Q * 2);
    l.ca_sel = o; o += al8(ca ? T * K * 2 : 0);
    l.st = o; o += al8(N);
    l.q_flags = o; o += al8(Q);
    l.tofetch = o; o += al8(E);
    l.ca_mod = o; o += al8(ca ? T : 0);
    l.dem_rank = o; o += al8(ca ? E * 4 : 0);
    l.total = o;
    return l;
}

// status bits in st[]: bits 0-2 = resident precision + 1, bit 7 = in flight
constexpr uint8_t ST_INFLIGHT = 0x80;

struct Pt {
    // config
    const EsimConfig* c;
    int L, E, K, N, S, Q;
    int pol, lane;
    int64_t cap, bw;
    int64_t dur[4];
    // smem arrays
    uint8_t* st;
    int16_t* hist;
    int16_t* slot_of;
    int32_t* cnt;
    int16_t* res_ident;
    uint64_t* key;
    float* rscore;
    int16_t* q_ident;
    uint8_t* q_flags;
    float* q_score;
    int64_t *q_submit, *q_start, *q_comp;
    int32_t* pl;
    uint32_t* demmask;
    uint8_t* tofetch;
    double* dsum;
    float* lsc;
    // cache-aware scratch
    int16_t* ca_sel;
    float* ca_w;
    uint8_t* ca_mod;
    float* ca_row;
    int32_t* dem_expert_s;
    int32_t* dem_rank_s;
    float* dem_gate_s;
    double* dem_summed_s;
    int32_t* dem_tokens_s;
    // scalars (warp-uniform)
    int64_t now, resident_bytes, reserved_bytes;
    int qh, qn, nA;
    uint64_t seq;        // LRU stamp / LFU touch / LS gen counter
    int pass_id, layer;
    // outputs
    EsimCounters* C;     // global, lane 0 writes at the end
    EsimCounters acc;    // lane-0 accumulators live in registers of every lane (uniform)
    EsimRec* recs;
    int64_t rec_cap;
    int32_t* pexp;
    int64_t pe_cap;
    bool full;
    int err;
    PySum ps_orig, ps_exec, ps_prec, ps_rec;
};

__device__ __forceinline__ int qphys(const Pt& p, int i) {
    int x = p.qh + i;
    return x >= p.Q ? x - p.Q : x;
}

__device__ __forceinline__ uint64_t fnv_word(uint64_t h, uint64_t w) { return (h ^ w) * FNV_PRIME; }

// ---------------------------------------------------------------------------
// record output
// ---------------------------------------------------------------------------
__device__ void emit(Pt& p, EsimRec& r, const int32_t* pe, int npe) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(&r);
    uint64_t h = p.acc.digest;
    #pragma unroll
    for (int i = 0; i < 8; i++) {
        if (r.kind == ESIM_REC_PREDICTION && i == 4) continue;
        h = fnv_word(h, w[i]);
    }
    for (int j = 0; j < npe; j++) h = fnv_word(h, (uint64_t)(uint32_t)pe[j]);
    p.acc.digest = h;
    if (p.full) {
        int64_t n = p.acc.n_recs, m = p.acc.n_pred_experts;
        if (n < p.rec_cap && m + npe <= p.pe_cap) {
            if (r.kind == ESIM_REC_PREDICTION) r.t0 = m;
            if (p.lane == 0) p.recs[n] = r;
            for (int j = p.lane; j < npe; j += 32) p.pexp[m + j] = pe[j];
        } else if (!p.err) {
            p.err = -4;
        }
    }
    p.acc.n_recs++;
    p.acc.n_pred_experts += npe;
}

__device__ __forceinline__ void rec_prefetch(Pt& p, int ev, int target, int expert, int64_t t, float score,
                                             int reason) {
    EsimRec r;
    r.kind = ESIM_REC_PREFETCH; r.pass_id = p.pass_id; r.layer = p.layer;
    r.i0 = ev; r.i1 = target; r.i2 = expert; r.i3 = reason; r.i4 = 0;
    r.t0 = t; r.t1 = 0; r.t2 = 0; r.x0 = (double)score;
    emit(p, r, nullptr, 0);
    p.acc.totals[10 + ev]++;
}

// ---------------------------------------------------------------------------
// policies: note_* update the slot key; victim = warp argmin
// ---------------------------------------------------------------------------
constexpr uint64_t LS_CURRENT = 1ull << 62;

__device__ __forceinline__ uint64_t order_double(double d) {
    uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}

// admit / access / prefetch-hit bookkeeping on a resident's slot (all lanes call; lane 0 writes)
__device__ void pol_touch_ls(Pt& p, int slot) {
    uint64_t k = p.key[slot];
    if (k & LS_CURRENT) return;                              // first touch of the pass fixed it
    uint64_t nk = LS_CURRENT | (p.seq++);
    __syncwarp();
    if (p.lane == 0) p.key[slot] = nk;
    __syncwarp();
}

__device__ void pol_note_admit(Pt& p, int ident, int slot) {
    uint64_t nk = 0;
    switch (p.pol) {
    case ESIM_EV_LRU: nk = p.seq++; break;                    // move_to_end
    case ESIM_EV_LFU: case ESIM_EV_LHU: nk = p.seq++; break;  // touch; count setdefault 0
    case ESIM_EV_FLD: nk = 0; break;
    case ESIM_EV_SB: nk = __double_as_longlong(0.0); break;   // new residency starts at 0
    case ESIM_EV_LS: nk = LS_CURRENT | (p.seq++); break;      // untracked -> current
    }
    if (p.lane == 0) p.key[slot] = nk;
    __syncwarp();
}

__device__ void pol_note_access(Pt& p, int ident, int slot, bool has_gate, double gate, int prec) {
    switch (p.pol) {
    case ESIM_EV_LRU: {
        uint64_t nk = p.seq++;
        if (p.lane == 0) p.key[slot] = nk;
        break;
    }
    case ESIM_EV_LFU: case ESIM_EV_LHU: {
        int step = 1;
        if (p.pol == ESIM_EV_LHU) step = (prec == p.c->precisions[0]) ? 1 : 0;
        uint64_t nk = p.seq++;
        if (p.lane == 0) { p.cnt[ident] += step; p.key[slot] = nk; }
        break;
    }
    case ESIM_EV_FLD: break;
    case ESIM_EV_SB:
        if (has_gate) {
            double s = __longlong_as_double((long long)p.key[slot]);
            double ns = __dadd_rn(s, gate);
            __syncwarp();
            if (p.lane == 0) p.key[slot] = (uint64_t)__double_as_longlong(ns);
        }
        break;
    case ESIM_EV_LS: pol_touch_ls(p, slot); break;
    }
    __syncwarp();
}

// warp argmin over residents. Returns the victim slot or -1.
__device__ int select_victim(Pt& p, bool forced) {
    uint64_t bk = ~0ull;
    uint32_t bi = 0xffffffffu;
    int c = p.layer;
    for (int s = p.lane; s < p.S; s += 32) {
        int id = p.res_ident[s];
        if (id < 0) continue;
        uint64_t k;
        uint32_t tie = (uint32_t)id;
        switch (p.pol) {
        case ESIM_EV_LRU: case ESIM_EV_LS: k = p.key[s]; break;
        case ESIM_EV_LFU: case ESIM_EV_LHU:
            k = ((uint64_t)(uint32_t)p.cnt[id] << 32) | (uint32_t)p.key[s];
            break;
        case ESIM_EV_FLD: {
            int l = id / p.E, e = id - l * p.E;
            int d = ((l - c) % p.L + p.L) % p.L;
            k = (uint64_t)(p.L - 1 - d);
            tie = (uint32_t)(e * p.L + l);
            break;
        }
        default: k = order_double(__longlong_as_double((long long)p.key[s])); break;  // SB
        }
        if (k < bk || (k == bk && tie < bi)) { bk = k; bi = tie; }
    }
    int bs = -1;
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t ok = __shfl_xor_sync(FULL, bk, o);
        uint32_t oi = __shfl_xor_sync(FULL, bi, o);
        if (ok < bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
    }
    if (bi == 0xffffffffu) return -1;
    int ident = (int)bi;
    if (p.pol == ESIM_EV_FLD) { int e = ident / p.L, l = ident - e * p.L; ident = l * p.E + e; }
    if (p.pol == ESIM_EV_LS) {
        if (bk & LS_CURRENT) {                               // no stale resident left
            if (!forced) { p.acc.ls_refusals++; return -1; }
            p.acc.ls_forced++;
        }
    }
    bs = p.slot_of[ident];
    return bs;
}

// ---------------------------------------------------------------------------
// cache + history
// ---------------------------------------------------------------------------
__device__ int alloc_slot(Pt& p) {
    for (int base = 0; base < p.S; base += 32) {
        int s = base + p.lane;
        bool fr = s < p.S && p.res_ident[s] < 0;
        unsigned m = __ballot_sync(FULL, fr);
        if (m) return base + __ffs(m) - 1;
    }
    return -1;
}

__device__ void evict(Pt& p, int slot, int cause, bool forced) {          // engine.py:451-460
    int ident = p.res_ident[slot];
    int prec = (p.st[ident] & 7) - 1;
    p.resident_bytes -= p.c->expert_bytes[prec];
    __syncwarp();
    if (p.lane == 0) {
        p.st[ident] = 0;
        p.hist[ident] = (int16_t)p.pass_id;
        p.res_ident[slot] = -1;
        p.slot_of[ident] = -1;
    }
    __syncwarp();
    EsimRec r;
    r.kind = ESIM_REC_EVICT; r.pass_id = p.pass_id; r.layer = p.layer;
    r.i0 = ident / p.E; r.i1 = ident % p.E; r.i2 = prec; r.i3 = cause; r.i4 = forced ? 1 : 0;
    r.t0 = r.t1 = r.t2 = 0; r.x0 = 0.0;
    emit(p, r, nullptr, 0);
    p.acc.totals[8]++;
    if (forced) p.acc.totals[9]++;
}

// ---------------------------------------------------------------------------
// channel: ring buffer [head][A: demands/promoted][B: pending prefetches]
// ---------------------------------------------------------------------------
struct QEntry { int16_t ident; uint8_t flags; float score; int64_t submit, start, comp; };

__device__ __forceinline__ QEntry q_load(const Pt& p, int i) {
    int x = qphys(p, i);
    QEntry e;
    e.ident = p.q_ident[x]; e.flags = p.q_flags[x]; e.score = p.q_score[x];
    e.submit = p.q_submit[x]; e.start = p.q_start[x]; e.comp = p.q_comp[x];
    return e;
}
__device__ __forceinline__ void q_store(Pt& p, int i, const QEntry& e) {
    int x = qphys(p, i);
    p.q_ident[x] = e.ident; p.q_flags[x] = e.flags; p.q_score[x] = e.score;
    p.q_submit[x] = e.submit; p.q_start[x] = e.start; p.q_comp[x] = e.comp;
}

// open a hole at logical index `at` (shift [at, qn) right by one)
__device__ void q_open(Pt& p, int at) {
    for (int hi = p.qn; hi > at; hi -= 32) {
        int lo = max(at, hi - 32);
        int i = lo + p.lane;
        QEntry e;
        bool act = i < hi;
        if (act) e = q_load(p, i);
        __syncwarp();
        if (act) q_store(p, i + 1, e);
        __syncwarp();
    }
    p.qn++;
}

// close logical index `at` (shift (at, qn) left by one)
__device__ void q_close(Pt& p, int at) {
    for (int lo = at + 1; lo < p.qn; lo += 32) {
        int i = lo + p.lane;
        QEntry e;
        bool act = i < p.qn;
        if (act) e = q_load(p, i);
        __syncwarp();
        if (act) q_store(p, i - 1, e);
        __syncwarp();
    }
    p.qn--;
}

__device__ __forceinline__ int64_t entry_dur(const Pt& p, uint8_t flags) { return p.dur[(flags >> 2) & 3]; }

// start_i = max(comp_{i-1}, submit_i); comp_i = start_i + dur_i for i >= from (>=1):
// a warp inclusive scan of x -> max(x + a, b) maps (engine.py:283-288)
__device__ void retime(Pt& p, int from) {
    if (from < 1) from = 1;
    if (from >= p.qn) return;
    int64_t carry = p.q_comp[qphys(p, from - 1)];
    for (int base = from; base < p.qn; base += 32) {
        int i = base + p.lane;
        bool act = i < p.qn;
        int64_t a = 0, b = INT64_MIN / 4, d = 0, sub = 0;
        if (act) {
            int x = qphys(p, i);
            d = entry_dur(p, p.q_flags[x]);
            sub = p.q_submit[x];
            a = d;
            b = sub + d;
        }
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t pa = __shfl_up_sync(FULL, a, o);
            int64_t pb = __shfl_up_sync(FULL, b, o);
            if (p.lane >= o) { b = max(pb + a, b); a = pa + a; }
        }
        int64_t comp = max(carry + a, b);
        __syncwarp();
        if (act) {
            int x = qphys(p, i);
            p.q_comp[x] = comp;
            p.q_start[x] = comp - d;
        }
        int last = min(31, p.qn - 1 - base);
        carry = __shfl_sync(FULL, comp, last);
        __syncwarp();
    }
}

__device__ int q_find(const Pt& p, int ident) {
    for (int base = 0; base < p.qn; base += 32) {
        int i = base + p.lane;
        bool hit = i < p.qn && p.q_ident[qphys(p, i)] == ident;
        unsigned m = __ballot_sync(FULL, hit);
        if (m) return base + __ffs(m) - 1;
    }
    return -1;
}

__device__ void settle(Pt& p) {                                           // engine.py:422-442
    while (p.qn > 0) {
        int h = p.qh;
        int64_t comp = p.q_comp[h];
        if (comp > p.now) break;
        int ident = p.q_ident[h];
        uint8_t fl = p.q_flags[h];
        float score = p.q_score[h];
        int prec = (fl >> 2) & 3;
        int64_t nb = p.c->expert_bytes[prec];
        __syncwarp();
        p.qh = (p.qh + 1 == p.Q) ? 0 : p.qh + 1;
        p.qn--;
        if (p.nA > 0) p.nA--;
        p.reserved_bytes -= nb;
        p.resident_bytes += nb;
        int slot = alloc_slot(p);
        if (slot < 0) { p.err = -2; return; }
        if (p.lane == 0) {
            p.st[ident] = (uint8_t)(prec + 1);
            p.slot_of[ident] = (int16_t)slot;
            p.res_ident[slot] = (int16_t)ident;
            p.rscore[slot] = score;
            if (p.hist[ident] == -2) p.hist[ident] = -1;
        }
        __syncwarp();
        if (p.resident_bytes + p.reserved_bytes > p.cap && !p.err) p.err = -2;
        pol_note_admit(p, ident, slot);
        if (fl & 1) rec_prefetch(p, 2, ident / p.E, ident % p.E, comp, score, 0);
    }
}

__device__ __forceinline__ void advance_to(Pt& p, int64_t t) { p.now = t; settle(p); }

// _fetch (engine.py:463-510). Returns blocked us, or -1 for None.
__device__ int64_t do_fetch(Pt& p, int ident, float gate, int prec, bool final) {
    int64_t nb = p.c->expert_bytes[prec];
    if (nb > p.cap) {
        if (!final) return -1;
        p.err = -1;
        return 0;
    }
    while (p.cap - p.resident_bytes - p.reserved_bytes < nb && !p.err) {
        int v = select_victim(p, final);
        if (v >= 0) { evict(p, v, 0, final); continue; }
        if (!final) return -1;
        int nB = p.qn - 1 - p.nA;                                 // pending prefetches
        if (p.qn > 1 && nB > 0) {                                 // cancel newest (= queue tail)
            QEntry e = q_load(p, p.qn - 1);
            __syncwarp();
            p.qn--;
            p.reserved_bytes -= p.c->expert_bytes[(e.flags >> 2) & 3];
            if (p.lane == 0) p.st[e.ident] &= (uint8_t)~ST_INFLIGHT;
            __syncwarp();
            rec_prefetch(p, 4, e.ident / p.E, e.ident % p.E, p.now, e.score, 4);
            continue;
        }
        if (p.qn == 0) { p.err = -2; return 0; }
        int64_t nd = p.q_comp[p.qh];
        advance_to(p, nd > p.now ? nd : p.now);
    }
    if (p.err) return 0;
    p.reserved_bytes += nb;
    int at = p.qn > 0 ? 1 + p.nA : 0;
    q_open(p, at);
    QEntry e;
    e.ident = (int16_t)ident; e.flags = (uint8_t)(prec << 2); e.score = gate;
    e.submit = p.now;
    e.start = p.now; e.comp = p.now + p.dur[prec];
    if (p.lane == 0) { q_store(p, at, e); p.st[ident] |= ST_INFLIGHT; }
    __syncwarp();
    if (at > 0) p.nA++;
    retime(p, at);
    int64_t comp = p.q_comp[qphys(p, at)];
    int64_t blocked = comp - p.now;
    advance_to(p, comp);
    return blocked;
}

__device__ void access_rec(Pt& p, int expert, int tokens, int rank, int outcome, int mclass, int64_t blocked,
                           double wd, int prec, int sub) {
    EsimRec r;
    r.kind = ESIM_REC_ACCESS; r.pass_id = p.pass_id; r.layer = p.layer;
    r.i0 = expert; r.i1 = tokens; r.i2 = rank;
    r.i3 = outcome | ((mclass < 0 ? 0xFF : mclass) << 8) | ((prec + 1) << 16);
    r.i4 = sub; r.t0 = blocked; r.t1 = 0; r.t2 = 0; r.x0 = wd;
    emit(p, r, nullptr, 0);
    p.acc.totals[0]++;
    p.acc.sync_overhead_us += blocked;
    int32_t* pl = p.pl + p.layer * ESIM_PL_FIELDS;
    int f = outcome == 0 ? 1 : (outcome <= 2 ? 2 : (outcome == 3 ? 6 : 7));
    if (outcome == 0) p.acc.totals[1]++;
    else if (outcome <= 2) { p.acc.totals[2]++; p.acc.totals[3 + mclass]++; }
    else if (outcome == 3) p.acc.totals[6]++;
    else p.acc.totals[7]++;
    if (p.lane == 0) {
        pl[0]++;
        pl[f]++;
        if (outcome == 1 || outcome == 2) pl[3 + mclass]++;
    }
}

// _handle_demand + resolve_miss. Returns outcome code (0 hit 1 fetch 2 wait 3 drop 4 subst), -1 error.
__device__ int handle_demand(Pt& p, int expert, int rank, float gate, double summed, int tokens,
                             const float* layer_scores, int nd, int64_t& blocked, double& wd) {
    const EsimConfig* cfg = p.c;
    int ident = p.layer * p.E + expert;
    blocked = 0; wd = 0.0;
    uint8_t st = p.st[ident];
    if (st & 7) {
        int prec = (st & 7) - 1;
        int slot = p.slot_of[ident];
        pol_note_access(p, ident, slot, true, (double)gate, prec);
        if (p.lane == 0) p.rscore[slot] = gate;
        __syncwarp();
        access_rec(p, expert, tokens, rank, 0, -1, 0, 0.0, prec, -1);
        return 0;
    }
    int h = p.hist[ident];
    int mclass = h == -2 ? 0 : (h == p.pass_id ? 1 : 2);
    if (st & ST_INFLIGHT) {                                              // promote + wait
        int idx = q_find(p, ident);
        QEntry e = q_load(p, idx);
        e.flags |= 2;
        __syncwarp();
        int at = idx;
        if (idx == 0) {
            if (p.lane == 0) p.q_flags[qphys(p, 0)] = e.flags;
            __syncwarp();
        } else {
            bool inA = idx <= p.nA;
            q_close(p, idx);
            if (inA) p.nA--;
            at = 1 + p.nA;
            q_open(p, at);
            if (p.lane == 0) q_store(p, at, e);
            __syncwarp();
            p.nA++;
            retime(p, min(idx, at));
        }
        int prec = (e.flags >> 2) & 3;
        int64_t comp = p.q_comp[qphys(p, at)];
        blocked = comp - p.now;
        advance_to(p, comp);
        int slot = p.slot_of[ident];
        pol_note_access(p, ident, slot, true, (double)gate, prec);
        if (p.lane == 0) p.rscore[slot] = gate;
        __syncwarp();
        access_rec(p, expert, tokens, rank, 2, mclass, blocked, 0.0, prec, -1);
        return 2;
    }
    if (cfg->miss == ESIM_MISS_DROP && rank > cfg->drop_rank_threshold) {
        wd = -summed;
        access_rec(p, expert, tokens, rank, 3, -1, 0, wd, -1, -1);
        return 3;
    }
    if (cfg->miss == ESIM_MISS_SUBST) {                                  // find_substitute miss.py:66-79
        double bd = 0.0;
        int be = -1;
        for (int e0 = 0; e0 < p.E; e0 += 32) {
            int e = e0 + p.lane;
            double diff = 0.0;
            bool ok = false;
            if (e < p.E) {
                int id = p.layer * p.E + e;
                if (p.st[id] & 7) {
                    diff = fabs((double)p.rscore[p.slot_of[id]] - (double)gate);
                    ok = diff <= cfg->subst_tolerance;
                }
            }
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                double od = __shfl_xor_sync(FULL, diff, o);
                int oe = __shfl_xor_sync(FULL, ok ? e : -1, o);
                bool ook = oe >= 0;
                if (ook && (!ok || od < diff || (od == diff && oe < e))) { diff = od; e = oe; ok = true; }
            }
            if (ok && (be < 0 || diff < bd)) { bd = diff; be = e; }
        }
        if (be >= 0) {
            int sid = p.layer * p.E + be;
            int sp = (p.st[sid] & 7) - 1;
            pol_note_access(p, sid, p.slot_of[sid], false, 0.0, sp);
            wd = -summed;
            access_rec(p, expert, tokens, rank, 4, -1, 0, wd, sp, be);
            return 4;
        }
    }
    int prec = cfg->working_prec;
    int64_t b = -1;
    if (cfg->miss == ESIM_MISS_FETCH_LOW) {
        prec = cfg->precisions[cfg->n_precisions - 1];
        b = do_fetch(p, ident, gate, prec, true);
    } else if (cfg->miss == ESIM_MISS_FETCH_PRIORITY) {
        int start = 0;
        if (cfg->n_precisions > 1 && nd > 0) {
            // nearest-rank percentile of layer_scores (float64 compare)
            long rk = (long)ceil(cfg->degrade_percentile / 100.0 * (double)nd);
            if (rk < 1) rk = 1;
            float thr = 0.0f;
            bool found = false;
            for (int i = p.lane; i < nd; i += 32) {
                float v = layer_scores[i];
                int less = 0, le = 0;
                for (int j = 0; j < nd; j++) { float u = layer_scores[j]; less += u < v; le += u <= v; }
                if (less <= rk - 1 && rk - 1 < le) { thr = v; found = true; }
            }
            unsigned who = __ballot_sync(FULL, found);
            thr = __shfl_sync(FULL, thr, __ffs(who) - 1);
            if ((double)gate < (double)thr) start = 1;
        }
        for (int i = start; i < cfg->n_precisions; i++) {
            bool fin = i == cfg->n_precisions - 1;
            prec = cfg->precisions[i];
            b = do_fetch(p, ident, gate, prec, fin);
            if (b >= 0 || p.err) break;
        }
        if (b < 0 && !p.err) p.err = -2;
    } else {
        b = do_fetch(p, ident, gate, prec, true);
    }
    if (p.err) return -1;
    int slot = p.slot_of[ident];
    pol_note_access(p, ident, slot, true, (double)gate, prec);
    if (p.lane == 0) p.rscore[slot] = gate;
    __syncwarp();
    blocked = b;
    access_rec(p, expert, tokens, rank, 1, mclass, b, 0.0, prec, -1);
    return 1;
}

// _submit_prefetches + watchdog_step for submitting layer `layer`
__device__ void submit_prefetches(Pt& p, const EsimRouterOut& R, int64_t tev) {
    int target = p.layer + 1;
    int n = R.n_pred[tev];
    const int32_t* pe = R.pred_expert + tev * p.E;
    const float* ps = R.pred_score + tev * p.E;
    EsimRec r;
    r.kind = ESIM_REC_PREDICTION; r.pass_id = p.pass_id; r.layer = p.layer;
    r.i0 = target; r.i1 = n; r.i2 = R.pred_clamped[tev]; r.i3 = 0; r.i4 = 0;
    r.t0 = 0; r.t1 = 0; r.t2 = 0; r.x0 = 0.0;
    emit(p, r, pe, n);
    if (p.lane == 0) { p.pl[target * ESIM_PL_FIELDS + 8] += n; p.pl[target * ESIM_PL_FIELDS + 9] += 1; }
    for (int j = 0; j < n; j++) rec_prefetch(p, 0, target, pe[j], p.now, ps[j], 0);
    int wp = p.c->working_prec;
    int64_t nb = p.c->expert_bytes[wp];
    // sweep 1 (FIFO): residents are marked (LS touch), in-flight skipped
    int nt = 0;
    for (int j = 0; j < n; j++) {
        int e = pe[j];
        int ident = target * p.E + e;
        uint8_t st = p.st[ident];
        if (st & 7) {
            if (p.pol == ESIM_EV_LS) pol_touch_ls(p, p.slot_of[ident]);
            rec_prefetch(p, 3, target, e, p.now, ps[j], 1);
        } else if (st & ST_INFLIGHT) {
            rec_prefetch(p, 3, target, e, p.now, ps[j], 2);
        } else {
            if (p.lane == 0) p.tofetch[nt] = (uint8_t)j;
            nt++;
        }
    }
    __syncwarp();
    // sweep 2: evict unforced or drop; reserve; append behind the tail
    for (int t = 0; t < nt && !p.err; t++) {
        int j = p.tofetch[t];
        int e = pe[j];
        float sc = ps[j];
        int ident = target * p.E + e;
        bool refused = false;
        while (p.cap - p.resident_bytes - p.reserved_bytes < nb) {
            int v = select_victim(p, false);
            if (v < 0) { rec_prefetch(p, 4, target, e, p.now, sc, 3); refused = true; break; }
            evict(p, v, 1, false);
        }
        if (refused) continue;
        p.reserved_bytes += nb;
        QEntry q;
        q.ident = (int16_t)ident; q.flags = (uint8_t)(1 | (wp << 2)); q.score = sc; q.submit = p.now;
        int64_t tail = p.qn ? p.q_comp[qphys(p, p.qn - 1)] : p.now;
        q.start = p.qn ? (p.now > tail ? p.now : tail) : p.now;
        q.comp = q.start + p.dur[wp];
        int at = p.qn;
        __syncwarp();
        if (p.lane == 0) { q_store(p, at, q); p.st[ident] |= ST_INFLIGHT; }
        __syncwarp();
        p.qn++;
        rec_prefetch(p, 1, target, e, p.now, sc, 0);
    }
}

// ---- cache-aware routing in the loop (routing.py:143-161) ----------------
// Per row: original softmax/top-k, bias = f32(lam * mean) on this layer's
// resident experts, re-softmax, re-top-k; DeltaAvg mean updated after the
// row with the fp64 pairwise row sum. Fills the smem demand arrays and the
// per-row selection; returns the demand count.
__device__ float warp_softmax(float* buf, int E, int lane) {
    float m = -__int_as_float(0x7f800000);
    for (int i = lane; i < E; i += 32) m = fmaxf(m, buf[i]);
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    __syncwarp();
    for (int i = lane; i < E; i += 32) buf[i] = np_expf(__fsub_rn(buf[i], m));
    __syncwarp();
    float S = __fadd_rn(0.0f, warp_pw_sum(buf, E, lane));
    __syncwarp();
    for (int i = lane; i < E; i += 32) buf[i] = __fdiv_rn(buf[i], S);
    __syncwarp();
    return S;
}

__device__ int warp_topk(const float* s, int E, int K, int lane, int16_t* out) {
    uint32_t taken = 0;
    for (int j = 0; j < K; j++) {
        float bv = -1.0f;
        int bi = 0x7fffffff;
        for (int i = lane, t = 0; i < E; i += 32, t++) {
            if (taken & (1u << t)) continue;
            float v = s[i];
            if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            float ov = __shfl_xor_sync(FULL, bv, o);
            int oi = __shfl_xor_sync(FULL, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == 0) out[j] = (int16_t)bi;
    }
    __syncwarp();
    return 0;
}

// numpy DOUBLE_pairwise_sum of one float32 row cast to float64 (lanes 0..7
// accumulate); n <= 256 splits at most once, so no recursion.
__device__ __forceinline__ double warp_pw_block_f64(const float* a, int n, int lane) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, (double)a[i]);
        return res;
    }
    int lim = n - (n % 8);
    double r = 0.0;
    if (lane < 8) {
        r = (double)a[lane];
        for (int i = 8; i < lim; i += 8) r = __dadd_rn(r, (double)a[i + lane]);
    }
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
    double res = __shfl_sync(FULL, r, 0);
    for (int i = lim; i < n; i++) res = __dadd_rn(res, (double)a[i]);
    return res;
}

__device__ __forceinline__ double warp_pw_sum_f64(const float* a, int n, int lane) {
    if (n <= 128) return warp_pw_block_f64(a, n, lane);
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(warp_pw_block_f64(a, n2, lane), warp_pw_block_f64(a + n2, n - n2, lane));
}

__device__ int route_cache_aware(Pt& p, const EsimTraceDesc& tr, int64_t ev, int T, int64_t rows_before) {
    const int E = p.E, K = p.K, l = p.layer;
    const float* X = tr.logits + tr.row_offset[ev] * (int64_t)E;
    float* buf = p.ca_row;
    bool any_cached = false;
    for (int e = p.lane; e < E; e += 32) any_cached |= (p.st[l * E + e] & 7) != 0;
    any_cached = __any_sync(FULL, any_cached);
    int16_t orig[ESIM_MAX_K];
    for (int r = 0; r < T; r++) {
        const float* x = X + (int64_t)r * E;
        // original scores and top-k
        for (int i = p.lane; i < E; i += 32) buf[i] = x[i];
        __syncwarp();
        warp_softmax(buf, E, p.lane);
        warp_topk(buf, E, K, p.lane, p.ca_sel + r * K);       // temp: original selection
        for (int j = 0; j < K; j++) orig[j] = p.ca_sel[r * K + j];
        const int64_t dcount = (rows_before + r) * (int64_t)E;
        double mean = dcount ? __ddiv_rn(p.dsum[l], (double)dcount) : 0.0;
        // keep the original scores (weights are read at the biased selection)
        __syncwarp();
        for (int i = p.lane; i < E; i += 32) p.dem_gate_s[i] = buf[i];
        __syncwarp();
        for (int i = p.lane; i < E; i += 32) {
            float v = x[i];
            if (p.c->lam != 0.0 && mean != 0.0 && any_cached && (p.st[l * E + i] & 7)) {
                float bias = __double2float_rn(__dmul_rn(p.c->lam, mean));
                v = __fadd_rn(v, bias);
            }
            buf[i] = v;
        }
        __syncwarp();
        warp_softmax(buf, E, p.lane);
        warp_topk(buf, E, K, p.lane, p.ca_sel + r * K);
        // DeltaAvg update with this row (after the bias)
        for (int i = p.lane; i < E; i += 32) buf[i] = x[i];
        __syncwarp();
        double rs = __dadd_rn(0.0, warp_pw_sum_f64(buf, E, p.lane));
        if (p.lane == 0) p.dsum[l] = __dadd_rn(p.dsum[l], rs);
        bool same = true;
        for (int a = 0; a < K; a++) {
            int s = p.ca_sel[r * K + a];
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
    // aggregate demands (engine.py:578-594) from the biased selection
    int nd = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
        int e = e0 + p.lane;
        int rank = 0x7fffffff, tok = 0;
        float gate = -1.0f;
        double summed = 0.0;
        if (e < E) {
            for (int r = 0; r < T; r++)
                for (int j = 0; j < K; j++)
                    if (p.ca_sel[r * K + j] == e) {
                        float wv = p.ca_w[r * K + j];
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
    }
    __syncwarp();
    // order by (rank, -gate, expert): position of each present expert
    int cnt = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
        int e = e0 + p.lane;
        int pos = -1;
        if (e < E && p.dem_rank_s[e] != 0x7fffffff) {
            int rk = p.dem_rank_s[e];
            float g = p.dem_gate_s[e];
            pos = 0;
            for (int j = 0; j < E; j++) {
                int rj = p.dem_rank_s[j];
                if (rj == 0x7fffffff || j == e) continue;
                float gj = p.dem_gate_s[j];
                pos += (rj < rk) || (rj == rk && (gj > g || (gj == g && j < e)));
            }
        }
        cnt += __popc(__ballot_sync(FULL, pos >= 0));
        if (e < E) reinterpret_cast<int*>(p.ca_row)[e] = pos;   // routing done: reuse as int scratch
    }
    __syncwarp();
    nd = cnt;
    // scatter into sorted order: dem_expert_s holds the sorted expert list
    for (int e = p.lane; e < E; e += 32) {
        int pos = reinterpret_cast<int*>(p.ca_row)[e];
        if (pos >= 0) p.dem_expert_s[pos] = e;
    }
    __syncwarp();
    return nd;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) replay_kernel(ReplayArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int wid = threadIdx.x >> 5;
    const int pid = blockIdx.x * A.warps_per_cta + wid;
    if (pid >= A.n_points) return;
    const EsimConfig* cfg = &A.cfg[pid];
    const EsimTraceDesc tr = A.traces[cfg->trace_id];
    const EsimRouterOut R = A.routers[cfg->trace_id];
    unsigned char* base = smem_raw + (size_t)wid * A.point_bytes;
    const bool ca = cfg->routing == ESIM_ROUTE_CACHE_AWARE;
    Layout lay = make_layout(A.N, A.S, A.Q, A.Lmax, A.Emax, A.Tmax, A.Kmax, A.Tmax > 0);

    Pt p;
    p.c = cfg;
    p.L = cfg->num_layers; p.E = cfg->experts; p.K = cfg->top_k; p.N = p.L * p.E;
    p.lane = threadIdx.x & 31;
    p.pol = cfg->eviction;
    p.cap = cfg->capacity_bytes; p.bw = cfg->bandwidth;
    int64_t minb = INT64_MAX;
    for (int i = 0; i < 4; i++) {
        int64_t nb = cfg->expert_bytes[i];
        p.dur[i] = (p.bw == 0 || nb == 0) ? 0 : (nb * 1000000 + p.bw - 1) / p.bw;
        if (nb > 0 && nb < minb) minb = nb;
    }
    int64_t slots = p.cap / minb;
    if (slots > p.N) slots = p.N;
    if (slots > A.S) slots = A.S;
    p.S = (int)slots;
    p.Q = p.S + 1;
    if (p.Q > A.Q) p.Q = A.Q;
    p.key = reinterpret_cast<uint64_t*>(base + lay.key);
    p.q_submit = reinterpret_cast<int64_t*>(base + lay.q_submit);
    p.q_start = reinterpret_cast<int64_t*>(base + lay.q_start);
    p.q_comp = reinterpret_cast<int64_t*>(base + lay.q_comp);
    p.dsum = reinterpret_cast<double*>(base + lay.dsum);
    p.dem_summed_s = reinterpret_cast<double*>(base + lay.dem_summed);
    p.cnt = reinterpret_cast<int32_t*>(base + lay.cnt);
    p.rscore = reinterpret_cast<float*>(base + lay.rscore);
    p.q_score = reinterpret_cast<float*>(base + lay.q_score);
    p.pl = reinterpret_cast<int32_t*>(base + lay.pl);
    p.demmask = reinterpret_cast<uint32_t*>(base + lay.demmask);
    p.lsc = reinterpret_cast<float*>(base + lay.lsc);
    p.ca_w = reinterpret_cast<float*>(base + lay.ca_w);
    p.ca_row = reinterpret_cast<float*>(base + lay.ca_row);
    p.dem_gate_s = reinterpret_cast<float*>(base + lay.dem_gate);
    p.dem_tokens_s = reinterpret_cast<int32_t*>(base + lay.dem_tokens);
    p.dem_expert_s = reinterpret_cast<int32_t*>(base + lay.dem_expert);
    p.hist = reinterpret_cast<int16_t*>(base + lay.hist);
    p.slot_of = reinterpret_cast<int16_t*>(base + lay.slot_of);
    p.res_ident = reinterpret_cast<int16_t*>(base + lay.res_ident);
    p.q_ident = reinterpret_cast<int16_t*>(base + lay.q_ident);
    p.ca_sel = reinterpret_cast<int16_t*>(base + lay.ca_sel);
    p.st = base + lay.st;
    p.q_flags = base + lay.q_flags;
    p.tofetch = base + lay.tofetch;
    p.ca_mod = base + lay.ca_mod;
    p.dem_rank_s = reinterpret_cast<int32_t*>(base + lay.dem_rank);

    for (int i = p.lane; i < p.N; i += 32) { p.st[i] = 0; p.hist[i] = -2; p.slot_of[i] = -1; p.cnt[i] = 0; }
    for (int i = p.lane; i < p.S; i += 32) { p.res_ident[i] = -1; p.key[i] = 0; }
    for (int i = p.lane; i < p.L * ESIM_PL_FIELDS; i += 32) p.pl[i] = 0;
    for (int i = p.lane; i < p.L; i += 32) p.dsum[i] = 0.0;
    __syncwarp();
    p.now = 0; p.resident_bytes = 0; p.reserved_bytes = 0;
    p.qh = 0; p.qn = 0; p.nA = 0; p.seq = 0;
    p.err = 0;
    p.full = (cfg->flags & ESIM_FLAG_FULL_LOG) && A.recs != nullptr;
    p.recs = A.recs + (int64_t)pid * A.rec_cap;
    p.rec_cap = A.rec_cap;
    p.pexp = A.pexp + (int64_t)pid * A.pe_cap;
    p.pe_cap = A.pe_cap;
    memset(&p.acc, 0, sizeof(p.acc));
    p.acc.digest = FNV_OFFSET;
    p.ps_orig.init(); p.ps_exec.init(); p.ps_prec.init(); p.ps_rec.init();
    if (ca && (p.E > A.Emax || A.Tmax == 0)) p.err = -1;
    int64_t rows_before = 0;   // token rows of earlier passes (DeltaAvg counts, routing.py:83-90)

    for (int pass = 0; pass < tr.n_passes && !p.err; pass++) {
        p.pass_id = pass;
        // begin_pass (eviction.py:37-45): LS current -> stale, SB decay
        if (p.pol == ESIM_EV_LS) {
            for (int s = p.lane; s < p.S; s += 32) p.key[s] &= ~LS_CURRENT;
        } else if (p.pol == ESIM_EV_SB) {
            for (int s = p.lane; s < p.S; s += 32)
                if (p.res_ident[s] >= 0)
                    p.key[s] = (uint64_t)__double_as_longlong(
                        __dmul_rn(__longlong_as_double((long long)p.key[s]), cfg->sb_decay));
        }
        __syncwarp();
        int64_t pstart = p.now, pblocked = 0;
        for (int l = 0; l < p.L && !p.err; l++) {
            p.layer = l;
            const int64_t ev = (int64_t)pass * p.L + l;
            settle(p);
            const int T = (int)(tr.row_offset[ev + 1] - tr.row_offset[ev]);
            int nd;
            const int32_t *d_exp, *d_rank, *d_tok;
            const float* d_gate;
            const double* d_sum;
            if (ca) {
                nd = route_cache_aware(p, tr, ev, T, rows_before);
                d_exp = p.dem_expert_s;
                // gather sorted arrays (rank/gate/sum/tokens are indexed by expert)
                d_rank = p.dem_rank_s; d_gate = p.dem_gate_s; d_sum = p.dem_summed_s; d_tok = p.dem_tokens_s;
            } else {
                nd = R.n_dem[ev];
                d_exp = R.dem_expert + ev * p.E;
                d_rank = R.dem_rank + ev * p.E;
                d_gate = R.dem_gate + ev * p.E;
                d_sum = R.dem_summed + ev * p.E;
                d_tok = R.dem_tokens + ev * p.E;
            }
            // layer scores in demand order (for fetch_priority); reuse the tofetch area? use a
            // register-free path: read gate by position
            float* lscores = p.lsc;
            if (cfg->miss == ESIM_MISS_FETCH_PRIORITY) {
                for (int i = p.lane; i < nd; i += 32) {
                    int e = d_exp[i];
                    lscores[i] = ca ? d_gate[e] : d_gate[i];
                }
                __syncwarp();
            }
            // prefetch precision/recall for this (pass, layer) as a target (metrics.py:150-187)
            if (cfg->prefetch != ESIM_PF_NONE && l >= 1) {
                for (int i = p.lane; i < (p.E + 31) / 32; i += 32) p.demmask[i] = 0;
                __syncwarp();
                for (int i = p.lane; i < nd; i += 32) atomicOr(&p.demmask[d_exp[i] >> 5], 1u << (d_exp[i] & 31));
                __syncwarp();
                int np = R.n_pred[ev];
                int inter = 0;
                for (int j = p.lane; j < np; j += 32) {
                    int e = R.pred_expert[ev * p.E + j];
                    inter += (p.demmask[e >> 5] >> (e & 31)) & 1;
                }
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(FULL, inter, o);
                p.acc.pf_tp += inter;
                p.acc.pf_pred_total += np;
                p.acc.pf_dem_total += nd;
                p.acc.pf_records++;
                if (np) { p.ps_prec.add(__ddiv_rn((double)inter, (double)np)); p.acc.pf_prec_parts++; }
                else p.acc.pf_empty++;
                p.ps_rec.add(__ddiv_rn((double)inter, (double)nd));
                p.acc.pf_rec_parts++;
            }
            int64_t blocked = 0;
            double wdelta = 0.0;
            bool any_aff = false;
            if (cfg->miss == ESIM_MISS_DROP || cfg->miss == ESIM_MISS_SUBST) {
                for (int i = p.lane; i < (p.E + 31) / 32; i += 32) p.demmask[i] = 0;
                __syncwarp();
            }
            for (int i = 0; i < nd && !p.err; i++) {
                int e = d_exp[i];
                int k = ca ? e : i;
                int64_t b;
                double wd;
                int oc = handle_demand(p, e, d_rank[k], d_gate[k], d_sum[k], d_tok[k], lscores, nd, b, wd);
                blocked += b;
                wdelta = __dadd_rn(wdelta, wd);
                if (oc == 3 || oc == 4) {
                    any_aff = true;
                    if (p.lane == 0) p.demmask[e >> 5] |= 1u << (e & 31);
                    __syncwarp();
                }
            }
            if (p.err) break;
            // RouteRec (engine.py:625-643)
            int faithful = T, nmod = 0;
            if (ca) {
                int bad = 0;
                for (int r = p.lane; r < T; r += 32) {
                    bool hit = p.ca_mod[r] != 0;
                    nmod += p.ca_mod[r];
                    if (any_aff)
                        for (int j = 0; j < p.K; j++) { int s = p.ca_sel[r * p.K + j]; hit |= (p.demmask[s >> 5] >> (s & 31)) & 1; }
                    bad += hit;
                }
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) { bad += __shfl_xor_sync(FULL, bad, o); nmod += __shfl_xor_sync(FULL, nmod, o); }
                faithful = T - bad;
            } else if (any_aff) {
                int bad = 0;
                const int16_t* rs = R.row_sel + tr.row_offset[ev] * p.K;
                for (int r = p.lane; r < T; r += 32) {
                    bool hit = false;
                    for (int j = 0; j < p.K; j++) { int s = rs[r * p.K + j]; hit |= (p.demmask[s >> 5] >> (s & 31)) & 1; }
                    bad += hit;
                }
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(FULL, bad, o);
                faithful = T - bad;
            }
            double origm = R.sel_mass[ev];
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
            double exm = __dadd_rn(selm, wdelta);
            {
                EsimRec r;
                r.kind = ESIM_REC_ROUTE; r.pass_id = pass; r.layer = l;
                r.i0 = T; r.i1 = faithful; r.i2 = nmod; r.i3 = 0; r.i4 = 0;
                r.t0 = 0; r.t1 = __double_as_longlong(origm); r.t2 = __double_as_longlong(exm); r.x0 = selm;
                emit(p, r, nullptr, 0);
            }
            p.acc.rows_total += T; p.acc.faithful_rows += faithful; p.acc.modified_rows += nmod;
            p.ps_orig.add(origm);
            p.ps_exec.add(exm);
            if (cfg->prefetch != ESIM_PF_NONE && l + 1 < p.L) submit_prefetches(p, R, ev + 1);
            advance_to(p, p.now + cfg->compute_us);
            pblocked += blocked;
        }
        if (p.err) break;
        EsimRec r;
        r.kind = ESIM_REC_PASS; r.pass_id = pass; r.layer = 0;
        r.i0 = tr.pass_kind[pass]; r.i1 = tr.pass_tokens[pass]; r.i2 = 0; r.i3 = 0; r.i4 = 0;
        r.t0 = pstart; r.t1 = p.now; r.t2 = pblocked; r.x0 = 0.0;
        emit(p, r, nullptr, 0);
        p.acc.passes++;
        if (pass == 0) p.acc.ttft_us = p.now;
        p.acc.total_us = p.now;
        if (tr.pass_kind[pass] == 1) { p.acc.decode_passes++; p.acc.decode_us += p.now - pstart; }
        rows_before += tr.pass_tokens[pass];
    }
    p.acc.original_mass = p.ps_orig.value();
    p.acc.executed_mass = p.ps_exec.value();
    p.acc.pf_prec_sum = p.ps_prec.value();
    p.acc.pf_rec_sum = p.ps_rec.value();
    p.acc.status = p.err;
    __syncwarp();
    if (p.lane == 0) A.counters[pid] = p.acc;
    int64_t* plo = A.per_layer + (int64_t)pid * A.Lmax * ESIM_PL_FIELDS;
    for (int i = p.lane; i < p.L * ESIM_PL_FIELDS; i += 32) plo[i] = p.pl[i];
}

}  // namespace esim

int esim_replay_smem_bytes(int N, int S, int Q, int L, int E, int T, int K, bool ca) {
    return esim::make_layout(N, S, Q, L, E, T, K, ca).total;
}

cudaError_t esim_replay_launch_impl(const EsimConfig* d_cfg, int n, const EsimTraceDesc* d_traces,
                                    const EsimRouterOut* d_routers, EsimCounters* d_counters,
                                    int64_t* d_per_layer, EsimRec* d_recs, int64_t rec_cap, int32_t* d_pexp,
                                    int64_t pe_cap, int N, int S, int Q, int Lmax, int Emax, int Tmax, int Kmax,
                                    int warps_per_cta, cudaStream_t st) {
    esim::ReplayArgs a;
    a.cfg = d_cfg; a.n_points = n; a.traces = d_traces; a.routers = d_routers;
    a.counters = d_counters; a.per_layer = d_per_layer; a.recs = d_recs; a.rec_cap = rec_cap;
    a.pexp = d_pexp; a.pe_cap = pe_cap;
    a.N = N; a.S = S; a.Q = Q; a.Lmax = Lmax; a.Emax = Emax; a.Tmax = Tmax; a.Kmax = Kmax;
    a.warps_per_cta = warps_per_cta;
    a.point_bytes = esim::make_layout(N, S, Q, Lmax, Emax, Tmax, Kmax, Tmax > 0).total;
    size_t smem = (size_t)a.point_bytes * warps_per_cta;
    cudaError_t e = cudaFuncSetAttribute(esim::replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int blocks = (n + warps_per_cta - 1) / warps_per_cta;
    esim::replay_kernel<<<blocks, 32 * warps_per_cta, smem, st>>>(a);
    return cudaGetLastError();
}
