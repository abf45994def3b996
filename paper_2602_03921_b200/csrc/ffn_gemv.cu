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

#include "../../include/specmd_b200.h"

namespace esim {
namespace gemv {

constexpr int NT = 256;     // threads per CTA
template <int NTOK>
struct Ld { static constexpr int N = NTOK == 1 ? 16 : NTOK == 2 ? 8 : 4; };   // 16-byte code vectors in flight per thread

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

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// padded fp32 staging: every EPV-element chunk (one code vector's span) is
// followed by 4 floats, so the VPR chunks a warp reads at once sit in
// distinct banks
template <int EPV>
__device__ __forceinline__ int padded(int col) { return col + (col / EPV) * 4; }

__device__ __forceinline__ float2 bf2_to_f2(uint32_t h) {
    return make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u));
}

// acc[n] += (the 16-byte vector's elements) . xs[n][col0 ...]   for n < NTOK
// (xs: padded fp32 rows of length ld; elements in memory order of the vector)
template <int BITS, int NTOK>
__device__ __forceinline__ void dot_vec(const uint4 q, const float* xs, int ld, int col0, float2 (&acc)[NTOK]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    if constexpr (BITS == 16) {                  // 8 bf16
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const float2 f = bf2_to_f2(w[c]);
#pragma unroll
            for (int n = 0; n < NTOK; n++) {
                const float2 xv = *reinterpret_cast<const float2*>(xs + n * ld + col0 + 2 * c);
                acc[n] = __ffma2_rn(f, xv, acc[n]);
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
                acc[n] = __ffma2_rn(f01, make_float2(xv.x, xv.y), acc[n]);
                acc[n] = __ffma2_rn(f23, make_float2(xv.z, xv.w), acc[n]);
            }
        }
    } else {                                     // int4 / int2, interleaved words
        constexpr uint32_t MASK = BITS == 4 ? 0x000F000Fu : 0x00030003u;
        constexpr uint32_t BIAS = BITS == 4 ? 0x43084308u : 0x43024302u;   // bf16x2 of 128 + 2^(BITS-1)
        constexpr int PAIRS = 16 / BITS;                                  // element pairs per word
#pragma unroll
        for (int c = 0; c < 4; c++) {
#pragma unroll
            for (int j = 0; j < PAIRS; j++) {
                uint32_t h, qq;
                asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(h) : "r"(w[c] >> (BITS * j)), "r"(MASK), "r"(BIAS));
                asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(qq) : "r"(h), "r"(BIAS));
                const float2 f = bf2_to_f2(qq);  // elements (2j, 2j+1) of the word
                const int col = col0 + c * 2 * PAIRS + 2 * j;
#pragma unroll
                for (int n = 0; n < NTOK; n++) {
                    const float2 xv = *reinterpret_cast<const float2*>(xs + n * ld + col);
                    acc[n] = __ffma2_rn(f, xv, acc[n]);
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
    static constexpr int NI = IPT >= NT ? IPT / NT : 1; // w1 items per thread
    static constexpr int G = IPT >= NT ? 1 : NT / IPT;  // k groups (int2: two)
};

template <int BITS, int NTOK>
__global__ void __launch_bounds__(NT, 2) ffn_gemv_kernel(const __grid_constant__ GemvArgs g) {
    using Q = Geo<BITS>;
    constexpr int VPR = Q::VPR, EPV = Q::EPV, NI = Q::NI, G = Q::G, IPT = Q::IPT, RB = Q::RB;
    constexpr int NLD = Ld<NTOK>::N;
    constexpr int U = NLD / NI > 0 ? NLD / NI : 1;       // k tiles per load batch
    extern __shared__ __align__(16) float sm[];
    const int H = g.H, I = g.I, KT = H / 64, m1 = I / 64;
    const int ldx = padded<EPV>(H), lda = padded<EPV>(64);
    float* xs = sm;                                     // [NTOK][ldx]
    float* acts = xs + NTOK * ldx;                      // [NTOK][lda]
    float* red = acts + NTOK * lda;                     // [G][128][NTOK]
    float* ssc = red + G * 128 * NTOK;                  // down-row scales [H] (quantised)
    const int tid = threadIdx.x, u = blockIdx.x;
    const int e = u / m1, mt = u - e * m1;
    const uint8_t* base = g.slots + (int64_t)g.exec_slot[e] * g.slot_bytes;
    const int64_t n1b = (int64_t)2 * I * H * BITS / 8;  // w1 bytes
    const uint8_t* w1 = base + (int64_t)mt * KT * 128 * RB;
    const uint8_t* w2 = base + n1b + (int64_t)mt * H * RB;
    const float* scl = reinterpret_cast<const float*>(base + (int64_t)3 * I * H * BITS / 8);
    if (tid == 0) {
        for (int64_t off = 0; off < (int64_t)H * RB; off += 65536)
            prefetch_l2(w2 + off, (uint32_t)((int64_t)H * RB - off < 65536 ? (int64_t)H * RB - off : 65536));
    }
    int ti[NTOK];
    float tw[NTOK];
#pragma unroll
    for (int n = 0; n < NTOK; n++) {
        ti[n] = n < g.npad ? g.tok_index[e * g.npad + n] : -1;
        tw[n] = ti[n] >= 0 ? g.tok_weight[e * g.npad + n] : 0.0f;
    }
    // tokens -> padded fp32 rows; down-row scales -> smem
    for (int n = 0; n < NTOK; n++) {
        const __nv_bfloat16* xr = g.x + (int64_t)(ti[n] < 0 ? 0 : ti[n]) * H;
        for (int c8 = tid; c8 < H / 8; c8 += NT) {
            uint4 v = ti[n] < 0 ? make_uint4(0, 0, 0, 0) : *reinterpret_cast<const uint4*>(xr + c8 * 8);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            float* d = xs + n * ldx + padded<EPV>(c8 * 8);    // 8 | EPV: one chunk
#pragma unroll
            for (int c = 0; c < 4; c++) *reinterpret_cast<float2*>(d + 2 * c) = bf2_to_f2(w[c]);
        }
    }
    if constexpr (BITS < 16)
        for (int h = tid; h < H; h += NT) ssc[h] = scl[2 * I + h];
    __syncthreads();

    // ---- phase 1: 128 rows (64 gate + 64 up) of the slice . x
    float2 acc[NI][NTOK];
#pragma unroll
    for (int i = 0; i < NI; i++)
#pragma unroll
        for (int n = 0; n < NTOK; n++) acc[i][n] = make_float2(0.0f, 0.0f);
    const int it0 = G > 1 ? tid % IPT : tid, kg = G > 1 ? tid / IPT : 0;
    const int v = it0 % VPR;                            // same for every item of the thread (NT % VPR == 0)
    for (int k0 = kg; k0 < KT; k0 += U * G) {
        uint4 q[U][NI];
#pragma unroll
        for (int b = 0; b < U; b++) {
            const int k = k0 + b * G;
#pragma unroll
            for (int i = 0; i < NI; i++)
                q[b][i] = k < KT ? ld_stream(w1 + ((int64_t)k * IPT + it0 + i * NT) * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int b = 0; b < U; b++) {
            const int k = k0 + b * G;
            if (k < KT) {
#pragma unroll
                for (int i = 0; i < NI; i++) dot_vec<BITS, NTOK>(q[b][i], xs, ldx, padded<EPV>(k * 64 + v * EPV), acc[i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NI; i++) {
        const int r = (it0 + i * NT) / VPR;             // tile row: gate 0-63, up 64-127
#pragma unroll
        for (int n = 0; n < NTOK; n++) {
            float s = acc[i][n].x + acc[i][n].y;
#pragma unroll
            for (int o = 1; o < VPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (v == 0) red[(kg * 128 + r) * NTOK + n] = s;
        }
    }
    __syncthreads();
    if (tid < 64 * NTOK) {
        const int i = tid & 63, n = tid >> 6;
        float gs = 0.0f, us = 0.0f;
#pragma unroll
        for (int k = 0; k < G; k++) {
            gs += red[(k * 128 + i) * NTOK + n];
            us += red[(k * 128 + 64 + i) * NTOK + n];
        }
        if constexpr (BITS < 16) {
            gs *= scl[mt * 64 + i];
            us *= scl[I + mt * 64 + i];
        }
        acts[n * lda + padded<EPV>(i)] = gs / (1.0f + __expf(-gs)) * us;
    }
    __syncthreads();

    // ---- phase 2: y[tok][h] += w * s_h * (Wd[h][slice] . act) for every h
    const int n2 = H * VPR;                             // w2 vectors of the slice
    const int v2 = tid % VPR;
    for (int f0 = 0; f0 < n2; f0 += NT * NLD) {
        uint4 q[NLD];
#pragma unroll
        for (int b = 0; b < NLD; b++) {
            const int f = f0 + b * NT + tid;
            q[b] = f < n2 ? ld_stream(w2 + (int64_t)f * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int b = 0; b < NLD; b++) {
            const int f = f0 + b * NT + tid;
            if (f0 + b * NT < n2) {                     // block-uniform
            float2 a2[NTOK];
#pragma unroll
            for (int n = 0; n < NTOK; n++) a2[n] = make_float2(0.0f, 0.0f);
            dot_vec<BITS, NTOK>(q[b], acts, lda, padded<EPV>(v2 * EPV), a2);
            const int h = f / VPR;
#pragma unroll
            for (int n = 0; n < NTOK; n++) {
                float s = a2[n].x + a2[n].y;
#pragma unroll
                for (int o = 1; o < VPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (BITS < 16) s *= ssc[h];
                if (v2 == 0 && f < n2 && ti[n] >= 0) atomicAdd(&g.y[(int64_t)ti[n] * H + h], tw[n] * s);
            }
            }
        }
    }
}

template <int BITS, int NTOK>
static size_t gemv_smem(int H) {
    using Q = Geo<BITS>;
    return ((size_t)NTOK * padded<Q::EPV>(H) + (size_t)NTOK * padded<Q::EPV>(64) + (size_t)Q::G * 128 * NTOK +
            (BITS < 16 ? H : 0)) * 4;
}

template <int BITS, int NTOK>
static cudaError_t launch(const GemvArgs& a, cudaStream_t st) {
    const size_t smem = gemv_smem<BITS, NTOK>(a.H);
    cudaError_t e = cudaFuncSetAttribute(ffn_gemv_kernel<BITS, NTOK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    ffn_gemv_kernel<BITS, NTOK><<<a.n_exec * (a.I / 64), NT, smem, st>>>(a);
    return cudaGetLastError();
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
