// trace_io.cu -- trace ingestion without per-event Python objects
// (reference trace.py:219-279 read_trace).
//
// Reference JSON-lines traces: the event lines (line 2 onwards, one layer
// event each: {"record": "event", "pass_id", "kind", "layer", "logits":
// [[...], ...]}) are parsed natively, in parallel line blocks, straight
// into float32 rows. Each number goes through a correctly rounded decimal ->
// double conversion (std::from_chars) and a double -> float32 cast, which is
// exactly what json.loads + np.asarray(dtype=np.float32) compute, so the
// logits are bit-identical to the reference reader's. The fast path accepts
// only well-formed, in-order, finite events; anything else (bad JSON, an
// unexpected record, a wrong pass/layer/kind/row count, NaN/Infinity, huge
// integer literals) returns ESIM_TRACE_SLOW with the first offending line so
// the host re-parses with the reference-exact reader and raises its
// TraceFormatError message.
//
// Device consumption: esim_trace_check_finite scans uploaded logits in HBM
// (binary traces arrive file -> pinned -> HBM with no host pass over them).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "../../include/specmd_b200.h"

extern const char* esim_set_error(const char* msg);

namespace {

struct EventLine {
    int64_t line;          // 1-based line number in the file
    int32_t pass_id, layer, kind, rows;
    int64_t first;         // first row in the block's float buffer
};

struct Block {
    std::vector<float> vals;
    std::vector<EventLine> ev;
    int64_t bad_line = 0;  // first line the fast path refuses (0: none)
};

// Correctly rounded decimal -> double for w * 10^q (w < 2^64, |q| <= 27):
// one extended-precision operation (w and 10^|q| are exact in a 64-bit (x87)
// or 113-bit (quad) significand, so L = RN_ext(w * 10^q)), then RN_double(L),
// accepted only when L is not within one extended ulp of a double midpoint
// (then the exact value sits on the same side of that midpoint as L). The
// libstdc++ from_chars conversion is exact too, but serialises across
// threads; this keeps the parallel blocks independent.
long double pow10l_exact(int k) {
    long double r = 1.0L;
    for (int i = 0; i < k; i++) r *= 10.0L;
    return r;
}

bool decimal_to_double(uint64_t w, int q, bool neg, double* out) {
    static_assert(std::numeric_limits<long double>::digits >= 64, "needs an extended long double");
    static const long double P[28] = {
        pow10l_exact(0), pow10l_exact(1), pow10l_exact(2), pow10l_exact(3), pow10l_exact(4), pow10l_exact(5),
        pow10l_exact(6), pow10l_exact(7), pow10l_exact(8), pow10l_exact(9), pow10l_exact(10), pow10l_exact(11),
        pow10l_exact(12), pow10l_exact(13), pow10l_exact(14), pow10l_exact(15), pow10l_exact(16),
        pow10l_exact(17), pow10l_exact(18), pow10l_exact(19), pow10l_exact(20), pow10l_exact(21),
        pow10l_exact(22), pow10l_exact(23), pow10l_exact(24), pow10l_exact(25), pow10l_exact(26),
        pow10l_exact(27)};
    if (w == 0) { *out = neg ? -0.0 : 0.0; return true; }
    if (q < -27 || q > 27) return false;
    const long double L = q < 0 ? (long double)w / P[-q] : (long double)w * P[q];
    const double d = (double)L;
    const double ad = std::fabs(d);
    if (!std::isfinite(d) || ad < 2.2250738585072014e-308) return false;
    const long double r = L - (long double)d;                       // exact (L, d within one double ulp)
    // spacing of doubles on the side of d where L lies
    const double nb = r > 0 ? std::nextafter(ad, INFINITY) : std::nextafter(ad, 0.0);
    const long double half = std::fabs((long double)nb - (long double)ad) / 2;
    const long double eps = std::ldexp(1.0L, std::ilogb(L) - (std::numeric_limits<long double>::digits - 1));
    if (std::fabs(std::fabs(r) - half) <= eps) return false;
    *out = neg ? -d : d;
    return true;
}

struct Cursor {
    const char* p;
    const char* end;
    void ws() { while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) p++; }
    bool lit(char c) { ws(); if (p < end && *p == c) { p++; return true; } return false; }
    // a JSON string without escapes (the reference writer never needs them)
    bool str(const char** s, size_t* n) {
        ws();
        if (p >= end || *p != '"') return false;
        const char* b = ++p;
        while (p < end && *p != '"') { if (*p == '\\') return false; p++; }
        if (p >= end) return false;
        *s = b; *n = (size_t)(p - b); p++;
        return true;
    }
    bool integer(int64_t* v) {
        ws();
        auto r = std::from_chars(p, end, *v);
        if (r.ec != std::errc() ) return false;
        if (r.ptr < end && (*r.ptr == '.' || *r.ptr == 'e' || *r.ptr == 'E')) return false;   // int() of a float: slow path
        p = r.ptr;
        return true;
    }
    // one JSON number -> float32 exactly as float(text) -> np.float32
    bool number(float* v) {
        ws();
        const char* b = p;
        bool neg = false;
        if (p < end && *p == '-') { neg = true; p++; }
        // digits (significand) / fraction / exponent, JSON grammar
        uint64_t w = 0;
        int nd = 0, dexp = 0;
        bool frac = false, any = false;
        while (p < end && *p >= '0' && *p <= '9') {
            any = true;
            if (w || *p != '0') { if (nd < 19) { w = w * 10 + (uint64_t)(*p - '0'); nd++; } else { nd = 99; dexp++; } }
            p++;
        }
        if (!any) return false;                           // NaN / Infinity / garbage: slow path
        const int int_digits_len = (int)(p - b) - (neg ? 1 : 0);
        if (p < end && *p == '.') {
            frac = true;
            p++;
            const char* f0 = p;
            while (p < end && *p >= '0' && *p <= '9') {
                if (w || *p != '0') { if (nd < 19) { w = w * 10 + (uint64_t)(*p - '0'); nd++; dexp--; } else nd = 99; }
                else dexp--;
                p++;
            }
            if (p == f0) return false;
        }
        if (p < end && (*p == 'e' || *p == 'E')) {
            frac = true;
            p++;
            bool eneg = false;
            if (p < end && (*p == '+' || *p == '-')) eneg = *p++ == '-';
            const char* e0 = p;
            int ev = 0;
            while (p < end && *p >= '0' && *p <= '9') { if (ev < 100000) ev = ev * 10 + (*p - '0'); p++; }
            if (p == e0) return false;
            dexp += eneg ? -ev : ev;
        }
        if (!frac && int_digits_len > 15) return false;  // big int literal: numpy's int path, slow path
        if (!frac) neg = neg && w != 0;                   // "-0" is the Python int 0 -> +0.0f
        double x;
        if (nd > 19 || !decimal_to_double(w, dexp, neg, &x)) {
            // rare: > 19 significant digits, far exponents, or a decimal within
            // one extended-precision ulp of a double midpoint -- the libstdc++
            // correctly rounded conversion decides
            auto r = std::from_chars(b, p, x);
            if (r.ec != std::errc() || r.ptr != p) return false;
        }
        *v = (float)x;
        return std::isfinite(*v);                         // the reference rejects non-finite logits
    }
};

// parse one event line; false = hand the file to the reference-exact reader
bool parse_event(const char* b, const char* e, int32_t experts, EventLine& ev, std::vector<float>& vals) {
    Cursor c{b, e};
    if (!c.lit('{')) return false;
    bool have_rec = false, have_pass = false, have_kind = false, have_layer = false, have_logits = false;
    for (bool first = true;; first = false) {
        c.ws();
        if (c.lit('}')) break;
        if (!first && !c.lit(',')) return false;
        const char* k; size_t kn;
        if (!c.str(&k, &kn) || !c.lit(':')) return false;
        auto key = [&](const char* s) { return kn == std::strlen(s) && std::memcmp(k, s, kn) == 0; };
        if (key("record")) {
            const char* v; size_t vn;
            if (!c.str(&v, &vn) || vn != 5 || std::memcmp(v, "event", 5) != 0) return false;
            have_rec = true;
        } else if (key("pass_id")) {
            int64_t v;
            if (!c.integer(&v) || v < 0 || v > INT32_MAX) return false;
            ev.pass_id = (int32_t)v; have_pass = true;
        } else if (key("layer")) {
            int64_t v;
            if (!c.integer(&v) || v < 0 || v > INT32_MAX) return false;
            ev.layer = (int32_t)v; have_layer = true;
        } else if (key("kind")) {
            const char* v; size_t vn;
            if (!c.str(&v, &vn)) return false;
            if (vn == 7 && std::memcmp(v, "prefill", 7) == 0) ev.kind = 0;
            else if (vn == 6 && std::memcmp(v, "decode", 6) == 0) ev.kind = 1;
            else return false;
            have_kind = true;
        } else if (key("logits")) {
            if (have_logits || !c.lit('[')) return false;
            ev.first = (int64_t)vals.size() / experts;
            int32_t rows = 0;
            c.ws();
            if (!c.lit(']')) {
                for (;;) {
                    if (!c.lit('[')) return false;
                    for (int32_t j = 0; j < experts; j++) {
                        float v;
                        if (j && !c.lit(',')) return false;
                        if (!c.number(&v)) return false;
                        vals.push_back(v);
                    }
                    if (!c.lit(']')) return false;          // wrong row width: slow path names the shape
                    rows++;
                    if (c.lit(']')) break;
                    if (!c.lit(',')) return false;
                }
            }
            ev.rows = rows;
            have_logits = true;
        } else {
            return false;                                   // unknown key: let the reference reader judge
        }
    }
    c.ws();
    return c.p == c.end && have_rec && have_pass && have_kind && have_layer && have_logits && ev.rows > 0;
}

struct Parsed {
    std::vector<Block> blocks;
    int64_t rows = 0;
    int32_t passes = 0;
    int32_t experts = 0;
};

}  // namespace

extern "C" int esim_trace_jsonl_parse(const char* text, int64_t len, int32_t num_layers, int32_t experts,
                                      int32_t n_threads, void** handle, int64_t* n_rows, int32_t* n_passes,
                                      int64_t* bad_line) {
    *handle = nullptr;
    *bad_line = 0;
    if (num_layers <= 0 || experts <= 0) { esim_set_error("trace parse: bad geometry"); return -1; }
    // line starts (line 1 is the spec record, parsed by the host)
    std::vector<int64_t> starts;
    int64_t pos = 0;
    while (pos < len && text[pos] != '\n') pos++;
    for (pos = pos + 1; pos < len;) {
        starts.push_back(pos);
        const void* nl = std::memchr(text + pos, '\n', (size_t)(len - pos));
        pos = nl ? (const char*)nl - text + 1 : len;
    }
    const int64_t nlines = (int64_t)starts.size();
    int nth = std::max(1, std::min<int>(n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency(), 32));
    nth = (int)std::max<int64_t>(1, std::min<int64_t>(nth, len >> 16));          // >= 64 KiB per block
    auto* P = new Parsed;
    P->experts = experts;
    P->blocks.resize(nth);
    auto work = [&](int k) {
        Block& B = P->blocks[k];
        // byte-balanced blocks (a prefill line can be megabytes, a decode line
        // a few KB): lines whose start falls in this block's byte range
        const int64_t b0 = len * k / nth, b1 = len * (k + 1) / nth;
        const int64_t lo = std::lower_bound(starts.begin(), starts.end(), b0) - starts.begin();
        const int64_t hi = k + 1 == nth ? nlines : std::lower_bound(starts.begin(), starts.end(), b1) - starts.begin();
        // every value takes >= 2 bytes of text ("0,"): reserve once (untouched
        // pages cost nothing) instead of growing -- regrowth remaps memory,
        // which serialises the threads on the address-space lock
        const int64_t bytes = (hi < nlines ? starts[hi] : len) - (lo < nlines ? starts[lo] : len);
        B.vals.reserve((size_t)std::max<int64_t>(bytes / 2, 0));
        for (int64_t i = lo; i < hi; i++) {
            const char* b = text + starts[i];
            const char* e = i + 1 < nlines ? text + starts[i + 1] : text + len;
            const char* t = b;
            while (t < e && (*t == ' ' || *t == '\t' || *t == '\r' || *t == '\n')) t++;
            if (t == e) continue;                                // blank line (skipped, trace.py:258)
            EventLine ev{i + 2, 0, 0, 0, 0, 0};
            if (!parse_event(b, e, experts, ev, B.vals)) { B.bad_line = i + 2; return; }
            B.ev.push_back(ev);
        }
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nth; k++) th.emplace_back(work, k);
    work(0);
    for (auto& t : th) t.join();
    // sequence validation (trace.py:62-95): passes 0,1,..; layers 0..L-1 per
    // pass; one kind and one row count per pass
    int32_t want_pass = 0, want_layer = 0, pass_kind = 0, pass_rows = 0;
    int64_t rows = 0;
    for (auto& B : P->blocks) {
        for (auto& ev : B.ev) {
            const bool new_pass = want_layer == 0;
            if (ev.pass_id != want_pass || ev.layer != want_layer ||
                (!new_pass && (ev.kind != pass_kind || ev.rows != pass_rows))) {
                *bad_line = ev.line;
                delete P;
                return ESIM_TRACE_SLOW;
            }
            if (new_pass) { pass_kind = ev.kind; pass_rows = ev.rows; }
            rows += ev.rows;
            if (++want_layer == num_layers) { want_layer = 0; want_pass++; }
        }
        if (B.bad_line) { *bad_line = B.bad_line; delete P; return ESIM_TRACE_SLOW; }
    }
    if (want_layer != 0 || want_pass == 0) {           // truncated last pass / no events
        *bad_line = -1;
        delete P;
        return ESIM_TRACE_SLOW;
    }
    P->rows = rows;
    P->passes = want_pass;
    *n_rows = rows;
    *n_passes = want_pass;
    *handle = P;
    return 0;
}

extern "C" int esim_trace_jsonl_take(void* handle, float* logits, int32_t* pass_tokens, int32_t* pass_kind) {
    auto* P = static_cast<Parsed*>(handle);
    if (!P) return -1;
    if (logits) {
        // blocks hold consecutive rows in file order: copy in parallel
        std::vector<int64_t> off(P->blocks.size() + 1, 0);
        for (size_t k = 0; k < P->blocks.size(); k++) off[k + 1] = off[k] + (int64_t)P->blocks[k].vals.size();
        std::vector<std::thread> th;
        for (size_t k = 0; k < P->blocks.size(); k++)
            th.emplace_back([&, k] {
                std::memcpy(logits + off[k], P->blocks[k].vals.data(), P->blocks[k].vals.size() * sizeof(float));
            });
        for (auto& t : th) t.join();
    }
    if (pass_tokens || pass_kind) {
        for (auto& B : P->blocks)
            for (auto& ev : B.ev)
                if (ev.layer == 0) {
                    if (pass_tokens) pass_tokens[ev.pass_id] = ev.rows;
                    if (pass_kind) pass_kind[ev.pass_id] = ev.kind;
                }
    }
    delete P;
    return 0;
}

extern "C" int esim_trace_jsonl_free(void* handle) {
    delete static_cast<Parsed*>(handle);
    return 0;
}

// ---------------------------------------------------------------------------
// device-side validation of uploaded logits: the first non-finite element
// (trace.py:94-95 "non-finite logit value"), grid-stride float4 loads
// ---------------------------------------------------------------------------
namespace {

__global__ void __launch_bounds__(256) check_finite_kernel(const float* __restrict__ x, int64_t n,
                                                           unsigned long long* first_bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 v = __ldg(x4 + i);
        const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (!isfinite(a[j])) atomicMin(first_bad, (unsigned long long)(4 * i + j));
    }
    for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        if (!isfinite(x[i])) atomicMin(first_bad, (unsigned long long)i);
}

}  // namespace

extern "C" int esim_trace_check_finite(const float* d_logits, int64_t n, int64_t* d_first_bad, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return 0;
    if (((uintptr_t)d_logits & 15) != 0) { esim_set_error("trace logits not 16-byte aligned"); return -1; }
    cudaError_t e = cudaMemsetAsync(d_first_bad, 0xff, sizeof(int64_t), st);     // INT64 "none" = all ones
    if (e != cudaSuccess) { esim_set_error(cudaGetErrorString(e)); return -2; }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t want = (n / 4 + 255) / 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
    check_finite_kernel<<<grid, 256, 0, st>>>(d_logits, n, reinterpret_cast<unsigned long long*>(d_first_bad));
    e = cudaGetLastError();
    if (e != cudaSuccess) { esim_set_error(cudaGetErrorString(e)); return -2; }
    return 0;
}
