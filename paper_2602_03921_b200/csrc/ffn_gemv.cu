// ffn_gemv.cu -- decode expert FFN (<= 4 tokens per expert) as a streaming
// GEMV over the cache slots, bf16 or quantised (int8 / int4 / int2 codes +
// fp32 per-row scales), dequantisation fused into the dot products.
//
// Why not tensor cores here: a decode expert is M = 1..4 tokens against
// 3*H*I weights, 2*T flop per weight element -- two orders of magnitude below
// the HBM ridge. The tcgen05 decode kernels (ffn_gemm.cu) pay a per-tile
// producer -> converter -> MMA hand-off (~280 ns per 128 x 64 tile, DESIGN
// section 4) that bounds them well above the weight-streaming time; here
// every thread streams its own 16-byte code vectors straight from HBM with
// 16 loads in flight, converts them in registers and accumulates in fp32
// (packed FFMA2), so the kernel is bound by the slot bytes it reads.
//
// Unit = (executed expert e, 64-row intermediate slice mt), one CTA:
//   phase 1  g_i, u_i (i in the slice) = rows of the w1 tiles (mt, k = 0..H/64)
//            -- one contiguous block of H * 128 * BITS / 8 bytes -- . x_tok
//   act      a_i = silu(s_g g_i) * (s_u u_i)               (fp32, smem)
//   phase 2  y[tok][h] += w_tok * s_d[h] * sum_i Wd[h][i] a_i  for all H rows:
//            the w2 tiles (mt, ht = 0..H/128), one contiguous block of
//            H * 64 * BITS / 8 bytes, bulk-prefetched into L2 at unit start
//            so its HBM reads overlap phase 1.
// Slot layout (layer_step.cu / ffn.py): tile-major w1 [I/64][H/64][64 gate +
// 64 up][64], w2 [I/64][H/128][128][64]; int4 / int2 words interleaved (even
// elements in the low half-word); then (quantised) fp32 scales [2I + H].
// No token gather: x rows are read through tok_index directly.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../include/specmd_b200.h"

namespace esim {
namespace gemv {

#ifndef GEMV_NT
#define GEMV_NT 512
#endif
constexpr int NT = GEMV_NT; // compute threads per CTA (+ one producer warp)
#ifndef GEMV_STAGES
#define GEMV_STAGES 4           // ring chunks in flight per CTA (two CTAs fit an SM)
#endif
#ifndef GEMV_PAIR_UNITS
#define GEMV_PAIR_UNITS -1      // at most this many units: a CTA pair per unit (-1: the device's SM count)
#endif
#ifndef GEMV_CHUNK
#define GEMV_CHUNK 16384        // bytes per ring chunk (one bulk copy; holds whole w1 tiles)
#endif

struct GemvArgs {
    const uint8_t* slots;
    int64_t slot_bytes;
    const __nv_bfloat16* x;     // [T][H]
    const int32_t* exec_slot;   // [n_exec]
    const int32_t* tok_index;   // [n_exec][npad]
    const float* tok_weight;    // [n_exec][npad]
    float* y;                   // [T][H]
    int I, H, n_exec, npad;
};

// padded fp32 staging: every EPV-element chunk (one code vector's span) is
// followed by 4 floats, so the VPR chunks a warp reads at once sit in
// distinct banks
template <int EPV>
__host__ __device__ __forceinline__ int padded(int col) { return col + (col / EPV) * 4; }

__device__ __forceinline__ float2 bf2_to_f2(uint32_t h) {
    return make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u));
}

// Per-token accumulators of one thread's rows. int4 / int2: one float2 per
// code position j inside the half-word (the element pair (2j, 2j+1) carries a
// 2^(BITS*j) factor, removed once in acc_total).
template <int BITS>
struct NAcc { static constexpr int N = BITS <= 4 ? 16 / BITS : 1; };

template <int BITS, int NTOK>
__device__ __forceinline__ void acc_zero(float2 (&acc)[NTOK][NAcc<BITS>::N]) {
#pragma unroll
    for (int n = 0; n < NTOK; n++)
#pragma unroll
        for (int j = 0; j < NAcc<BITS>::N; j++) acc[n][j] = make_float2(0.0f, 0.0f);
}
template <int BITS, int NTOK>
__device__ __forceinline__ float acc_total(const float2 (&acc)[NTOK][NAcc<BITS>::N], int n) {
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < NAcc<BITS>::N; j++) s += (acc[n][j].x + acc[n][j].y) * __int_as_float((127 - BITS * j) << 23);
    return BITS <= 4 ? s : acc[n][0].x + acc[n][0].y;
}

// acc[n] += (the 16-byte vector's elements) . xs[n][col0 ...]   for n < NTOK
// (xs: padded fp32 rows of length ld; elements in memory order of the vector)
template <int BITS, int NTOK>
__device__ __forceinline__ void dot_vec(const uint4 q, const float* xs, int ld, int col0,
                                        float2 (&acc)[NTOK][NAcc<BITS>::N]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    if constexpr (BITS == 16) {                  // 8 bf16
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const float2 f = bf2_to_f2(w[c]);
#pragma unroll
            for (int n = 0; n < NTOK; n++) {
                const float2 xv = *reinterpret_cast<const float2*>(xs + n * ld + col0 + 2 * c);
                acc[n][0] = __ffma2_rn(f, xv, acc[n][0]);
            }
        }
    } else if constexpr (BITS == 8) {            // 16 int8, byte order; fp32 magic 2^23 + (q + 128)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t o = w[c] ^ 0x80808080u;
            float2 f01, f23;
            f01.x = __uint_as_float(__byte_perm(o, 0x4B000000u, 0x7650));   // 0x4B0000 | byte k
            f01.y = __uint_as_float(__byte_perm(o, 0x4B000000u, 0x7651));
            f23.x = __uint_as_float(__byte_perm(o, 0x4B000000u, 0x7652));
            f23.y = __uint_as_float(__byte_perm(o, 0x4B000000u, 0x7653));
            const float2 m = make_float2(-8388736.0f, -8388736.0f);   // -(2^23 + 128)
            f01 = __fadd2_rn(f01, m);
            f23 = __fadd2_rn(f23, m);
#pragma unroll
            for (int n = 0; n < NTOK; n++) {
                const float4 xv = *reinterpret_cast<const float4*>(xs + n * ld + col0 + 4 * c);
                acc[n][0] = __ffma2_rn(f01, make_float2(xv.x, xv.y), acc[n][0]);
                acc[n][0] = __ffma2_rn(f23, make_float2(xv.z, xv.w), acc[n][0]);
            }
        }
    } else {                                     // int4 / int2, interleaved words
        // element 2j sits at bits [BITS*j, BITS*j + BITS) of the low half-word,
        // 2j+1 at the same position of the high one. (w & m_j) ^ (2^23 | half << BITS*j)
        // is the fp32 2^23 + (q + half) * 2^(BITS*j) (one LOP3, no shift); one packed
        // add of -(2^23 + half * 2^(BITS*j)) leaves q * 2^(BITS*j) exactly.
        constexpr uint32_t QM = (1u << BITS) - 1, HALF = 1u << (BITS - 1);
        constexpr int PAIRS = 16 / BITS;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t wl = w[c], wh = w[c] >> 16;
#pragma unroll
            for (int j = 0; j < PAIRS; j++) {
                const uint32_t m = QM << (BITS * j), cst = 0x4B000000u | (HALF << (BITS * j));
                uint32_t lo, hi;                 // (w & m) ^ cst: one LOP3 each
                asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(lo) : "r"(wl), "r"(m), "r"(cst));
                asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(hi) : "r"(wh), "r"(m), "r"(cst));
                float2 f = make_float2(__uint_as_float(lo), __uint_as_float(hi));
                const float b = -(8388608.0f + (float)(HALF << (BITS * j)));
                f = __fadd2_rn(f, make_float2(b, b));
                const int col = col0 + c * 2 * PAIRS + 2 * j;
#pragma unroll
                for (int n = 0; n < NTOK; n++) {
                    const float2 xv = *reinterpret_cast<const float2*>(xs + n * ld + col);
                    acc[n][j] = __ffma2_rn(f, xv, acc[n][j]);
                }
            }
        }
    }
}

template <int BITS>
struct Geo {
    static constexpr int RB = 64 * BITS / 8;            // bytes per tile row (64 elements)
    static constexpr int VPR = RB / 16;                 // 16-byte vectors per tile row
    static constexpr int EPV = 128 / BITS;              // elements per vector
    static constexpr int IPT = 128 * VPR;               // vectors per w1 tile (128 rows)
    static constexpr int NI = IPT >= NT ? IPT / NT : 1; // w1 items per thread per tile
    static constexpr int G = IPT >= NT ? 1 : NT / IPT;  // tiles a chunk's threads split (int2: two)
    static constexpr int TILE = 128 * RB;               // bytes per w1 tile
    static constexpr int TPC = GEMV_CHUNK / TILE;       // w1 tiles per ring chunk
    static_assert(TPC >= 1 && TPC % G == 0, "ring chunk must hold whole tiles");
};

// ---- mbarrier / bulk-copy ring ---------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}

__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_peer(const float* p, uint32_t rank) {   // DSMEM read of the peer CTA
    uint32_t a;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(p)), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}

// A unit is processed by CL CTAs (a thread-block cluster when CL = 2, so a
// decode layer's units cover every SM twice): CTA rank r takes the k-tiles
// [r*KT/CL, (r+1)*KT/CL) of the w1 block and the rows [r*H/CL, (r+1)*H/CL)
// of the w2 block; the gate/up partial sums are exchanged through
// distributed shared memory before the activation.
// Warps 0..NT/32-1 compute; the last warp (one lane) streams the CTA's weight
// bytes -- its part of the w1 block, then of the w2 block -- through a ring
// of GEMV_STAGES chunks of GEMV_CHUNK bytes (cp.async.bulk, mbarrier
// complete_tx), so HBM reads run continuously ahead of the dot products,
// across the phase-1 -> phase-2 boundary, with no registers held by loads;
// it also bulk-loads the CTA's down-row scales.
template <int BITS, int NTOK, int CL>
__global__ void __launch_bounds__(NT + 32) ffn_gemv_kernel(const __grid_constant__ GemvArgs g) {
    using Q = Geo<BITS>;
    constexpr int VPR = Q::VPR, EPV = Q::EPV, NI = Q::NI, G = Q::G, IPT = Q::IPT, RB = Q::RB, TPC = Q::TPC;
    constexpr int NS = GEMV_STAGES, CH = GEMV_CHUNK;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int H = g.H, I = g.I, KT = H / 64, m1 = I / 64;
    const int ldx = padded<EPV>(H), lda = padded<EPV>(64);
    unsigned char* ring = smraw;                                   // [NS][CH]
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + NS * CH); // [NS]
    uint64_t* empty = full + NS;                                   // [NS]
    uint64_t* sbar = empty + NS;                                   // down-row scales landed
    float* xs = reinterpret_cast<float*>(sbar + 2);                // [NTOK][ldx]
    float* acts = xs + NTOK * ldx;                                 // [NTOK][lda]
    float* red = acts + NTOK * lda;                                // [G][128][NTOK]
    float* ssc = red + G * 128 * NTOK;                             // down-row scales [H / CL] (quantised)
    const int tid = threadIdx.x;
    const int r = CL > 1 ? (int)(blockIdx.x % CL) : 0, u = blockIdx.x / CL;
#ifdef GEMV_STAMPS
    unsigned long long ts[6];
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[0]));
#define GSTAMP(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[i]))
#else
#define GSTAMP(i) do {} while (0)
#endif
    const int e = u / m1, mt = u - e * m1;
    const uint8_t* base = g.slots + (int64_t)g.exec_slot[e] * g.slot_bytes;
    const int64_t n1b = (int64_t)2 * I * H * BITS / 8;             // w1 bytes
    const int kt0 = r * (KT / CL), h0 = r * (H / CL);              // this CTA's k-tiles / down rows
    const uint8_t* w1 = base + ((int64_t)mt * KT + kt0) * Q::TILE;
    const uint8_t* w2 = base + n1b + (int64_t)mt * H * RB + (int64_t)h0 * RB;
    const float* scl = reinterpret_cast<const float*>(base + (int64_t)3 * I * H * BITS / 8);
    const int w1_bytes = (KT / CL) * Q::TILE, w2_bytes = (H / CL) * RB;
    const int n1c = (w1_bytes + CH - 1) / CH, n2c = (w2_bytes + CH - 1) / CH;
    if (tid == 0) {
        for (int i = 0; i < NS; i++) { bar_init(&full[i], 1); bar_init(&empty[i], NT / 32); }
        bar_init(sbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid >= NT) {                                               // ---- producer warp
        if (CL > 1) cluster_arrive();                              // nothing of its own to publish
        if (tid == NT) {
            if constexpr (BITS < 16) {
                bar_expect(sbar, (uint32_t)(H / CL) * 4);
                bulk_g2s(ssc, scl + 2 * I + h0, (uint32_t)(H / CL) * 4, sbar);
            }
            for (int c = 0; c < n1c + n2c; c++) {
                const int st = c % NS;
                if (c >= NS) bar_wait(&empty[st], ((c / NS) - 1) & 1);
                const bool p1 = c < n1c;
                const int off = (p1 ? c : c - n1c) * CH, tot = p1 ? w1_bytes : w2_bytes;
                const uint32_t nb = (uint32_t)(tot - off < CH ? tot - off : CH);
                bar_expect(&full[st], nb);
                bulk_g2s(ring + st * CH, (p1 ? w1 : w2) + off, nb, &full[st]);
            }
        }
        __syncwarp();
        if (CL > 1) {
            cluster_wait();
            cluster_arrive();                                      // peers done with our smem
            cluster_wait();
        }
        return;
    }
    int ti[NTOK];
    float tw[NTOK];
#pragma unroll
    for (int n = 0; n < NTOK; n++) {
        ti[n] = n < g.npad ? g.tok_index[e * g.npad + n] : -1;
        tw[n] = ti[n] >= 0 ? g.tok_weight[e * g.npad + n] : 0.0f;
    }
    // tokens -> padded fp32 rows (this CTA's columns)
#pragma unroll
    for (int n = 0; n < NTOK; n++) {
        const __nv_bfloat16* xr = g.x + (int64_t)(ti[n] < 0 ? 0 : ti[n]) * H;
        for (int c8 = kt0 * 8 + tid; c8 < (kt0 + KT / CL) * 8; c8 += NT) {
            const uint4 v = ti[n] < 0 ? make_uint4(0, 0, 0, 0) : *reinterpret_cast<const uint4*>(xr + c8 * 8);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            float* d = xs + n * ldx + padded<EPV>(c8 * 8);            // 8 | EPV: one chunk
#pragma unroll
            for (int c = 0; c < 4; c++) *reinterpret_cast<float2*>(d + 2 * c) = bf2_to_f2(w[c]);
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");         // compute warps only
    GSTAMP(1);

    // ---- phase 1: 128 rows (64 gate + 64 up) of the slice . x, tile by tile from the ring
    constexpr int NA = NAcc<BITS>::N;
    float2 acc[NI][NTOK][NA];
#pragma unroll
    for (int i = 0; i < NI; i++) acc_zero<BITS, NTOK>(acc[i]);
    const int it0 = G > 1 ? tid % IPT : tid, kg = G > 1 ? tid / IPT : 0;
    const int v = it0 % VPR;                                       // same for every item (NT % VPR == 0)
    const int lane = tid & 31;
    for (int c = 0; c < n1c; c++) {
        const int st = c % NS;
        bar_wait(&full[st], (c / NS) & 1);
        const unsigned char* chunk = ring + st * CH;
#pragma unroll
        for (int t = kg; t < TPC; t += G) {
            const int kl = c * TPC + t;                            // tile within this CTA's part
            if (kl < KT / CL) {
                uint4 q[NI];
#pragma unroll
                for (int i = 0; i < NI; i++)
                    q[i] = *reinterpret_cast<const uint4*>(chunk + (t * IPT + it0 + i * NT) * 16);
#pragma unroll
                for (int i = 0; i < NI; i++)
                    dot_vec<BITS, NTOK>(q[i], xs, ldx, padded<EPV>((kt0 + kl) * 64 + v * EPV), acc[i]);
            }
        }
        __syncwarp();
        if (lane == 0) bar_arrive(&empty[st]);
    }
#pragma unroll
    for (int i = 0; i < NI; i++) {
        const int row = (it0 + i * NT) / VPR;                      // tile row: gate 0-63, up 64-127
#pragma unroll
        for (int n = 0; n < NTOK; n++) {
            float s = acc_total<BITS, NTOK>(acc[i], n);
#pragma unroll
            for (int o = 1; o < VPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (v == 0) red[(kg * 128 + row) * NTOK + n] = s;
        }
    }
    GSTAMP(2);
    if (CL > 1) {                                                  // partial sums visible to the peer
        cluster_arrive();
        cluster_wait();
    } else {
        asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
    }
    if (tid < 64 * NTOK) {
        const int i = tid & 63, n = tid >> 6;
        float gs = 0.0f, us = 0.0f;
#pragma unroll
        for (int k = 0; k < G; k++) {
            gs += red[(k * 128 + i) * NTOK + n];
            us += red[(k * 128 + 64 + i) * NTOK + n];
            if (CL > 1) {
                gs += ld_peer(&red[(k * 128 + i) * NTOK + n], (uint32_t)(r ^ 1));
                us += ld_peer(&red[(k * 128 + 64 + i) * NTOK + n], (uint32_t)(r ^ 1));
            }
        }
        if constexpr (BITS < 16) {
            gs *= scl[mt * 64 + i];
            us *= scl[I + mt * 64 + i];
        }
        acts[n * lda + padded<EPV>(i)] = gs / (1.0f + __expf(-gs)) * us;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
    GSTAMP(3);
    if constexpr (BITS < 16) bar_wait(sbar, 0);

    // ---- phase 2: y[tok][h] += w * s_h * (Wd[h][slice] . act), chunk by chunk
    constexpr int VPC = CH / 16;                                   // vectors per chunk
    const int v2 = tid % VPR;
    for (int c = 0; c < n2c; c++) {
        const int cc = n1c + c, st = cc % NS;
        bar_wait(&full[st], (cc / NS) & 1);
        const unsigned char* chunk = ring + st * CH;
        const int nvec = (w2_bytes - c * CH < CH ? w2_bytes - c * CH : CH) / 16;
#pragma unroll
        for (int j = 0; j < (VPC + NT - 1) / NT; j++) {
            const int fl = j * NT + tid;                           // vector within the chunk
            float2 a2[NTOK][NA];
            acc_zero<BITS, NTOK>(a2);
            if (j * NT < nvec) {                                   // block-uniform
                const uint4 q = fl < nvec ? *reinterpret_cast<const uint4*>(chunk + fl * 16) : make_uint4(0, 0, 0, 0);
                dot_vec<BITS, NTOK>(q, acts, lda, padded<EPV>(v2 * EPV), a2);
                const int hl = (c * VPC + fl) / VPR;               // row within this CTA's part
#pragma unroll
                for (int n = 0; n < NTOK; n++) {
                    float sum = acc_total<BITS, NTOK>(a2, n);
#pragma unroll
                    for (int o = 1; o < VPR; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    if (BITS < 16 && fl < nvec) sum *= ssc[hl];
                    if (v2 == 0 && fl < nvec && ti[n] >= 0)
                        atomicAdd(&g.y[(int64_t)ti[n] * H + h0 + hl], tw[n] * sum);
                }
            }
        }
        __syncwarp();
        if (lane == 0) bar_arrive(&empty[st]);
    }
#ifdef GEMV_STAMPS
    GSTAMP(4);
    if (tid == 0 && (u == 0 || u == 64 || u == gridDim.x / CL - 1))
        printf("gemv blk %d r %d start %llu setup %llu ph1 %llu act %llu ph2 %llu (ns)\n", u, r, ts[0] % 100000000ull,
               ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3]);
#endif
    if (CL > 1) {                                                  // the peer has read our partial sums
        cluster_arrive();
        cluster_wait();
    }
}
#undef GSTAMP

template <int BITS, int NTOK>
static size_t gemv_smem(int H) {
    using Q = Geo<BITS>;
    return (size_t)GEMV_STAGES * GEMV_CHUNK + (2 * GEMV_STAGES + 2) * 8 +
           ((size_t)NTOK * padded<Q::EPV>(H) + (size_t)NTOK * padded<Q::EPV>(64) + (size_t)Q::G * 128 * NTOK +
            (BITS < 16 ? H : 0)) * 4;
}

template <int BITS, int NTOK>
static cudaError_t launch(const GemvArgs& a, cudaStream_t st) {
    const size_t smem = gemv_smem<BITS, NTOK>(a.H);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    const int units = a.n_exec * (a.I / 64);
    // fewer units than SMs: split each across a CTA pair (cluster), both SMs' worth of warps
    static int pair_units = -1;
    if (pair_units < 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        pair_units = GEMV_PAIR_UNITS >= 0 ? GEMV_PAIR_UNITS : sms;
    }
    const bool pair = units <= pair_units && (a.H / 64) % 2 == 0;
    cudaLaunchConfig_t lc{};
    lc.blockDim = dim3(NT + 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    cudaError_t e;
    // the smem opt-in is raised once per instantiation (to the largest request so far)
    static int set_pair = 0, set_one = 0;
    if (pair) {
        if ((int)smem > set_pair) {
            e = cudaFuncSetAttribute(ffn_gemv_kernel<BITS, NTOK, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            if (e != cudaSuccess) return e;
            set_pair = (int)smem;
        }
        lc.gridDim = dim3(2 * units);
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        return cudaLaunchKernelEx(&lc, ffn_gemv_kernel<BITS, NTOK, 2>, a);
    }
    if ((int)smem > set_one) {
        e = cudaFuncSetAttribute(ffn_gemv_kernel<BITS, NTOK, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        set_one = (int)smem;
    }
    lc.gridDim = dim3(units);
    return cudaLaunchKernelEx(&lc, ffn_gemv_kernel<BITS, NTOK, 1>, a);
}

template <int BITS>
static cudaError_t launch_bits(const GemvArgs& a, int max_tok, cudaStream_t st) {
    if (max_tok <= 1) return launch<BITS, 1>(a, st);
    if (max_tok <= 2) return launch<BITS, 2>(a, st);
    return launch<BITS, 4>(a, st);
}

}  // namespace gemv
}  // namespace esim

// y[t] += w * Wd (silu(Wg x_t) * (Wu x_t)) for every executed expert with at
// most 4 tokens (decode), straight from the slots (bits 16 = bf16 slots).
extern "C" int esim_ffn_experts_gemv(const void* d_slots, int64_t slot_bytes, int32_t bits, const void* d_x,
                                     const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                     const float* d_tok_weight, float* d_y, int32_t n_exec, int32_t npad,
                                     int32_t max_tok, int32_t I, int32_t H, void* stream) {
    using namespace esim::gemv;
    if (n_exec <= 0) return 0;
    if (I <= 0 || H <= 0 || I % 64 || H % 128 || H > 8192 || max_tok < 1 || max_tok > 4 || npad < max_tok ||
        (slot_bytes & 15))
        return -1;
    GemvArgs a{(const uint8_t*)d_slots, slot_bytes, (const __nv_bfloat16*)d_x, d_exec_slot, d_tok_index,
               d_tok_weight, d_y, I, H, n_exec, npad};
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    switch (bits) {
    case 16: e = launch_bits<16>(a, max_tok, st); break;
    case 8: e = launch_bits<8>(a, max_tok, st); break;
    case 4: e = launch_bits<4>(a, max_tok, st); break;
    case 2: e = launch_bits<2>(a, max_tok, st); break;
    default: return -1;
    }
    return e == cudaSuccess ? 0 : -3;
}
