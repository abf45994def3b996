// report.cu -- native report assembly for sweeps.
//
// The result-dependent columns of metrics.flatten_report (totals, rates,
// timing, fidelity, prefetch; reference metrics.py:190-316, 348-362) for many
// grid points at once, written exactly as the reference's csv emission writes
// them (Python's csv module: str() of each value, i.e. the shortest
// round-trip repr for floats, True/False for bools). The config columns are
// fixed per point, so the host formats them once; per step only these
// columns change. Host code (no kernel): a few hundred bytes per point,
// ~1 us instead of ~180 us of Python report assembly; large sweeps format
// in parallel row chunks.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <thread>
#include <vector>

extern const char* esim_set_error(const char* msg);

#include "../../include/specmd_b200.h"

namespace {

// Python repr(float): shortest round-trip digits, fixed notation for
// 1e-4 <= |x| < 1e16 (with ".0" when integral), else d.ddde+XX
struct Out {
    char* p;
    char* end;
    bool ok = true;
    void put(const char* s, size_t n) {
        if (p + n > end) { ok = false; return; }
        std::memcpy(p, s, n);
        p += n;
    }
    void put(const char* s) { put(s, std::strlen(s)); }
    void put_int(int64_t v) {
        char b[32];
        auto r = std::to_chars(b, b + sizeof b, v);
        put(b, (size_t)(r.ptr - b));
    }
    void put_bool(bool v) { put(v ? "True" : "False"); }
    void put_float(double x) {
        if (std::isnan(x)) { put("nan"); return; }
        if (std::isinf(x)) { put(x > 0 ? "inf" : "-inf"); return; }
        if (x == 0.0) { put(std::signbit(x) ? "-0.0" : "0.0"); return; }
        char b[64];
        auto r = std::to_chars(b, b + sizeof b - 1, x, std::chars_format::scientific);   // shortest round-trip
        *r.ptr = 0;                                  // to_chars does not terminate
        const char* q = b;
        char s[64];
        int m = 0;
        if (*q == '-') { s[m++] = '-'; q++; }
        char digits[32];
        int n = 0;
        for (; q < r.ptr && *q != 'e'; q++)
            if (*q != '.') digits[n++] = *q;
        const int exp10 = std::atoi(q + 1);
        const int decpt = exp10 + 1;                 // value = 0.d1d2... x 10^decpt
        if (decpt <= -4 || decpt > 16) {
            s[m++] = digits[0];
            if (n > 1) { s[m++] = '.'; std::memcpy(s + m, digits + 1, n - 1); m += n - 1; }
            m += std::snprintf(s + m, sizeof s - m, "e%c%02d", exp10 < 0 ? '-' : '+', std::abs(exp10));
        } else if (decpt <= 0) {
            s[m++] = '0'; s[m++] = '.';
            for (int k = 0; k < -decpt; k++) s[m++] = '0';
            std::memcpy(s + m, digits, n); m += n;
        } else if (decpt >= n) {
            std::memcpy(s + m, digits, n); m += n;
            for (int k = 0; k < decpt - n; k++) s[m++] = '0';
            s[m++] = '.'; s[m++] = '0';
        } else {
            std::memcpy(s + m, digits, decpt); m += decpt;
            s[m++] = '.';
            std::memcpy(s + m, digits + decpt, n - decpt); m += n - decpt;
        }
        put(s, (size_t)m);
    }
};

double ratio(double a, double b) { return b != 0.0 ? a / b : 0.0; }


// rows [lo, hi) into o; offsets relative to `base`
int format_rows(const EsimCounters* cs, const int64_t* per_layer, int32_t pl_stride, const int32_t* num_layers,
                const int64_t* per_layer_compute_us, int lo, int hi, const char* prefixes,
                const int64_t* prefix_offsets, Out& o, const char* base, int64_t* offsets) {
    for (int i = lo; i < hi; i++) {
        offsets[i] = o.p - base;
        if (prefixes) o.put(prefixes + prefix_offsets[i], (size_t)(prefix_offsets[i + 1] - prefix_offsets[i]));
        const EsimCounters& c = cs[i];
        const int64_t* t = c.totals;            // TOTAL_FIELDS order
        const int64_t demanded = t[0], hits = t[1], misses = t[2], comp = t[3], coll = t[4], capm = t[5];
        const int64_t dropped = t[6], subst = t[7];
        // check_identities (metrics.py:319-336)
        if (hits + misses + dropped + subst != demanded || comp + coll + capm != misses) return -1;
        const int64_t* pl = per_layer + (int64_t)i * pl_stride * ESIM_PL_FIELDS;
        for (int l = 0; l < num_layers[i]; l++) {
            const int64_t* r = pl + (int64_t)l * ESIM_PL_FIELDS;
            if (r[1] + r[2] + r[6] + r[7] != r[0]) return -2;
        }
        for (int k = 0; k < 15; k++) { o.put_int(t[k]); o.put(","); }                       // totals
        const double d = (double)demanded;
        o.put_float(ratio((double)hits, d)); o.put(",");                                     // rates
        o.put_float(ratio((double)misses, d)); o.put(",");
        o.put_float(ratio((double)coll, d)); o.put(",");
        o.put_float(ratio((double)coll, (double)misses)); o.put(",");
        o.put_float(ratio((double)dropped, d)); o.put(",");
        o.put_float(ratio((double)subst, d)); o.put(",");
        o.put_int(c.ttft_us); o.put(","); o.put_int(c.total_us); o.put(",");                // timing
        o.put_int(c.decode_us); o.put(","); o.put_int(c.sync_overhead_us); o.put(",");
        o.put_int(c.passes); o.put(","); o.put_int(c.decode_passes); o.put(",");
        o.put_int(per_layer_compute_us[i]); o.put(",");
        o.put_float(c.decode_us > 0 ? (double)(c.decode_passes * 1000000) / (double)c.decode_us : 0.0); o.put(",");
        o.put_float(c.rows_total ? ratio((double)c.faithful_rows, (double)c.rows_total) : 1.0); o.put(",");  // fidelity
        o.put_float(c.original_mass != 0.0 ? ratio(c.executed_mass, c.original_mass) : 1.0); o.put(",");
        o.put_int(c.modified_rows); o.put(","); o.put_int(c.rows_total); o.put(",");
        const bool zero_den = c.pf_pred_total == 0;                                          // prefetch
        o.put_float(zero_den ? 1.0 : (double)c.pf_tp / (double)c.pf_pred_total); o.put(",");
        o.put_float(c.pf_dem_total == 0 ? 1.0 : ratio((double)c.pf_tp, (double)c.pf_dem_total)); o.put(",");
        o.put_float(c.pf_prec_parts ? ratio(c.pf_prec_sum, (double)c.pf_prec_parts) : 1.0); o.put(",");
        o.put_float(c.pf_rec_parts ? ratio(c.pf_rec_sum, (double)c.pf_rec_parts) : 1.0); o.put(",");
        o.put_int(c.pf_records); o.put(","); o.put_int(c.pf_pred_total); o.put(",");
        o.put_int(c.pf_tp); o.put(","); o.put_int(c.pf_empty); o.put(",");
        o.put_bool(zero_den);
        if (prefixes) o.put("\r\n", 2);
        if (!o.ok) return -4;
    }
    return 0;
}

}  // namespace

extern "C" int esim_report_csv(const EsimCounters* cs, const int64_t* per_layer, int32_t pl_stride,
                               const int32_t* num_layers, const int64_t* per_layer_compute_us, int32_t n,
                               const char* prefixes, const int64_t* prefix_offsets, char* out, int64_t cap,
                               int64_t* offsets) {
    // rows are independent: large sweeps format in parallel chunks (each into
    // its own buffer, bounded by its prefixes + 512 B per row), then the chunks
    // are concatenated in row order
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nth = n >= 512 ? std::min(hw, std::min(16, n / 256)) : 1;
    int rc = 0;
    if (nth <= 1) {
        Out o{out, out + cap};
        rc = format_rows(cs, per_layer, pl_stride, num_layers, per_layer_compute_us, 0, n, prefixes, prefix_offsets,
                         o, out, offsets);
        if (rc == 0) offsets[n] = o.p - out;
    } else {
        std::vector<std::vector<char>> bufs(nth);
        std::vector<int> rcs(nth, 0), lo(nth + 1);
        std::vector<int64_t> used(nth, 0);
        for (int k = 0; k <= nth; k++) lo[k] = (int)((int64_t)n * k / nth);
        std::vector<std::thread> th;
        for (int k = 0; k < nth; k++)
            th.emplace_back([&, k] {
                const int64_t pb = prefixes ? prefix_offsets[lo[k + 1]] - prefix_offsets[lo[k]] : 0;
                bufs[k].resize((size_t)(pb + 512 * (int64_t)(lo[k + 1] - lo[k]) + 64));
                Out o{bufs[k].data(), bufs[k].data() + bufs[k].size()};
                rcs[k] = format_rows(cs, per_layer, pl_stride, num_layers, per_layer_compute_us, lo[k], lo[k + 1],
                                     prefixes, prefix_offsets, o, bufs[k].data(), offsets);
                used[k] = o.p - bufs[k].data();
            });
        for (auto& t : th) t.join();
        int64_t pos = 0;
        for (int k = 0; k < nth && rc == 0; k++) {
            if ((rc = rcs[k])) break;
            if (pos + used[k] > cap) { rc = -4; break; }
            std::memcpy(out + pos, bufs[k].data(), (size_t)used[k]);
            for (int i = lo[k]; i < lo[k + 1]; i++) offsets[i] += pos;
            pos += used[k];
        }
        if (rc == 0) offsets[n] = pos;
    }
    if (rc == -1) { esim_set_error("accounting identity broken in a replay's totals"); return -1; }
    if (rc == -2) { esim_set_error("per-layer accounting identity broken in a replay"); return -1; }
    return rc;
}
