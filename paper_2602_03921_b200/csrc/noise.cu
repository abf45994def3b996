// noise.cu -- prediction noise on the device: prefetch.apply_prediction_noise
// (prefetch.py:110-136) over a routed trace's whole prediction stream, drawn
// from numpy's np.random.default_rng(seed) (engine.py:413) in the
// reference's submission order (engine.py:653-666: pass by pass, layer
// 0..L-2 predicting layer+1).
//
// The generator is numpy's, restated bit for bit:
//   SeedSequence(seed)           entropy = seed as little-endian uint32 words,
//                                pool of 4 (hashmix / mix), generate_state(4,
//                                uint64) (numpy/random/bit_generator.pyx)
//   PCG64                        128-bit LCG, XSL-RR output, seeded with
//                                pcg_setseq_128_srandom_r(state = w0:w1,
//                                seq = w2:w3) (numpy/random/src/pcg64)
//   Generator.random()           (next64 >> 11) * 2^-53
//   Generator.integers(n)        n == 1: no draw; else Lemire's bounded
//                                uint32 on next_uint32 (which buffers the
//                                high half of a 64-bit draw; random() does
//                                not touch that buffer)
// A prediction event is a serial stream of draws, so one thread walks it;
// the unchosen-candidate list (ascending expert ids) is a 256-bit mask and
// the j-th candidate a popcount walk. Scores ride along with the swap; the
// prediction count per event is unchanged (the chosen set keeps its size).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/specmd_b200.h"

namespace esim {
namespace {

struct Pcg64 {
    uint64_t shi, slo, ihi, ilo;   // 128-bit state and increment
    uint32_t buf;                  // next_uint32's buffered high half
    bool has_buf;
};

__device__ __forceinline__ void pcg_step(Pcg64& g) {
    const uint64_t mhi = 2549297995355413924ULL, mlo = 4865540595714422341ULL;
    const uint64_t lo = g.slo * mlo;
    uint64_t hi = __umul64hi(g.slo, mlo) + g.slo * mhi + g.shi * mlo;
    const uint64_t nlo = lo + g.ilo;
    hi += g.ihi + (nlo < lo ? 1ULL : 0ULL);
    g.slo = nlo;
    g.shi = hi;
}

__device__ __forceinline__ uint64_t pcg_next64(Pcg64& g) {
    pcg_step(g);
    const uint64_t x = g.shi ^ g.slo;
    const unsigned rot = (unsigned)(g.shi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint32_t pcg_next32(Pcg64& g) {
    if (g.has_buf) {
        g.has_buf = false;
        return g.buf;
    }
    const uint64_t n = pcg_next64(g);
    g.has_buf = true;
    g.buf = (uint32_t)(n >> 32);
    return (uint32_t)n;
}

__device__ __forceinline__ double pcg_random(Pcg64& g) {
    return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Generator.integers(n), 1 <= n <= 2^32 (bounded by ESIM_MAX_E here)
__device__ __forceinline__ uint32_t pcg_integers(Pcg64& g, uint32_t n) {
    const uint32_t rng = n - 1;
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)pcg_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        const uint32_t threshold = (0xFFFFFFFFu - rng) % excl;
        while (left < threshold) {
            m = (uint64_t)pcg_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

// np.random.default_rng(seed): SeedSequence(seed).generate_state(4, uint64) -> PCG64
__device__ void pcg_seed(Pcg64& g, uint64_t seed) {
    const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
    const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
    uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int n_ent = (seed >> 32) ? 2 : 1;
    uint32_t hc = INIT_A;
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= MULT_A;
        v *= hc;
        return v ^ (v >> 16);
    };
    auto mix = [&](uint32_t x, uint32_t y) {
        uint32_t r = MIX_L * x - MIX_R * y;
        return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    uint32_t hb = INIT_B, w[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3] ^ hb;
        hb *= MULT_B;
        v *= hb;
        w[i] = v ^ (v >> 16);
    }
    uint64_t v64[4];
    for (int i = 0; i < 4; i++) v64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    // pcg_setseq_128_srandom_r(initstate = v0:v1, initseq = v2:v3)
    g.ihi = (v64[2] << 1) | (v64[3] >> 63);
    g.ilo = (v64[3] << 1) | 1ULL;
    g.shi = 0;
    g.slo = 0;
    pcg_step(g);
    const uint64_t lo = g.slo + v64[1];
    g.shi = g.shi + v64[0] + (lo < g.slo ? 1ULL : 0ULL);
    g.slo = lo;
    pcg_step(g);
    g.has_buf = false;
    g.buf = 0;
}

// one thread: the stream is serial by construction (every draw depends on
// the previous state and on whether the previous prediction drew twice)
__global__ void noise_kernel(int n_passes, int L, int E, EsimRouterOut o, double noise, uint64_t seed) {
    if (threadIdx.x != 0) return;
    Pcg64 g;
    pcg_seed(g, seed);
    for (int p = 0; p < n_passes; p++) {
        for (int l = 1; l < L; l++) {
            const int64_t ev = (int64_t)p * L + l;
            const int n = o.n_pred[ev];
            if (n == 0) continue;                           // empty prediction: no draws
            int32_t* pe = o.pred_expert + ev * E;
            uint32_t chosen[ESIM_MAX_E / 32];
            #pragma unroll
            for (int w = 0; w < ESIM_MAX_E / 32; w++) chosen[w] = 0;
            for (int i = 0; i < n; i++) chosen[pe[i] >> 5] |= 1u << (pe[i] & 31);
            const uint32_t n_cand = (uint32_t)(E - n);      // |chosen| stays n through every swap
            for (int i = 0; i < n; i++) {
                if (!(pcg_random(g) < noise)) continue;
                if (n_cand == 0) continue;                  // no candidates: no integers() draw
                uint32_t j = pcg_integers(g, n_cand);       // j-th unchosen expert, ascending
                int pick = -1;
                for (int w = 0; w < (E + 31) / 32 && pick < 0; w++) {
                    const int bits = E - 32 * w < 32 ? E - 32 * w : 32;
                    const uint32_t valid = bits == 32 ? 0xffffffffu : ((1u << bits) - 1u);
                    uint32_t free_ = ~chosen[w] & valid;
                    const uint32_t c = (uint32_t)__popc(free_);
                    if (j >= c) { j -= c; continue; }
                    for (uint32_t k = 0; k < j; k++) free_ &= free_ - 1;   // drop the j lowest
                    pick = 32 * w + (__ffs(free_) - 1);
                }
                const int e = pe[i];
                chosen[e >> 5] &= ~(1u << (e & 31));
                chosen[pick >> 5] |= 1u << (pick & 31);
                pe[i] = pick;
            }
        }
    }
}

}  // namespace
}  // namespace esim

extern "C" int esim_route_summary_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode,
                                         void* stream);
const char* esim_set_error(const char* msg);

extern "C" int esim_noise_launch(const EsimTraceDesc* tr, const EsimRouterOut* out, int32_t pred_mode,
                                 double noise, uint64_t seed, void* stream) {
    if (!tr || !out) { esim_set_error("null argument"); return -1; }
    if (!(noise >= 0.0 && noise <= 1.0)) { esim_set_error("prediction noise must be in [0, 1]"); return -1; }
    if (tr->experts < 1 || tr->experts > ESIM_MAX_E) { esim_set_error("experts out of range"); return -1; }
    if (noise == 0.0 || pred_mode == ESIM_PF_NONE || tr->n_events == 0) return 0;   // consumes nothing
    cudaStream_t st = (cudaStream_t)stream;
    esim::noise_kernel<<<1, 32, 0, st>>>(tr->n_passes, tr->num_layers, tr->experts, *out, noise, seed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { esim_set_error(cudaGetErrorString(e)); return -3; }
    return esim_route_summary_launch(tr, out, pred_mode, stream);
}
