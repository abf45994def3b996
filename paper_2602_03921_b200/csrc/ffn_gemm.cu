// ffn_gemm.cu -- grouped bf16 SwiGLU expert FFN on tcgen05 / TMEM / TMA.
//
// The reference models expert compute as a constant (engine.py:648,
// models.py:129); this is the physical layer step's compute (SURVEY.md
// section 8 row a17): for each executed expert e with token set T_e,
//     y[t] += w[t,e] * Wd_e ( silu(Wg_e x_t) * (Wu_e x_t) )
// with weights read straight from the HBM cache slot the expert lives in.
//
// Swap-AB tiling (tiny M = tokens per expert): the weight rows are the MMA
// M side (128 per tile), tokens are N (padded to a multiple of 16).
//   gemm1: tile = (expert, 128 intermediate rows). Two accumulators in TMEM:
//          gate rows -> columns [0,N), up rows -> columns [N,2N), so the
//          epilogue thread owning TMEM lane r holds g and u of the same row
//          and writes act = silu(g)*u (bf16) without any exchange.
//   gemm2: tile = (expert, 128 hidden rows), K = I; epilogue scales by the
//          routing weight and scatter-adds into the fp32 layer output.
// Warp roles: warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer,
// warps 0-3 = epilogue (TMEM lanes 32w..32w+31). 4-stage mbarrier ring.
//
// Roofline: HBM (weight streaming). Per executed expert 12,582,912 B of
// weights (3 * 2048 * 1024 * 2) + activations; arithmetic intensity =
// 2 * T_e flop/B << the ridge (~250 flop/B), so decode and prefill-64 are
// bandwidth bound.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "../../include/specmd_b200.h"

namespace esim {
namespace ffn {

constexpr int BM = 128;          // weight rows per tile (UMMA M)
constexpr int BK = 64;           // 64 bf16 = 128 B = one swizzle-128B atom row

// ---- PTX wrappers ----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef MBAR_SPIN
#define MBAR_SPIN 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if MBAR_SPIN
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#endif
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// smem matrix descriptor: K-major, SWIZZLE_128B, rows of 128 B, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t umma_desc(const void* smem_tile) {
    const uint32_t a = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);            // start address
    d |= (uint64_t)1 << 16;                        // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;              // stride byte offset: 8 rows * 128 B
    d |= (uint64_t)1 << 46;                        // version = 1 (sm100)
    d |= (uint64_t)2 << 61;                        // layout: SWIZZLE_128B
    return d;
}

// instruction descriptor: kind::f16, bf16 x bf16 -> f32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4)                 // D format f32
           | (1u << 7)               // A bf16
           | (1u << 10)              // B bf16
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
// 32 lanes x 16 columns of 32-bit: thread t of warp w gets row 32w+t, columns col..col+15
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

__host__ __device__ inline uint32_t tmem_cols(uint32_t n) {
    uint32_t c = 32;
    while (c < n) c <<= 1;
    return c;
}

// ---- device sync helpers (gemm1 tiles -> gemm2 units across CTAs) ----------
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// programmatic dependent launch: the kernel starts while the previous one (token
// gather) finishes; what reads the gathered tokens waits here first
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- one persistent kernel for the whole layer's experts -------------------
// Work units, in this order (every CTA walks units blockIdx.x, +gridDim.x, ...):
//   gemm1 unit (e, mt): 64 gate rows + 64 up rows of expert e stacked into one
//     M = 128 tile (TMEM lanes 0-63 gate, 64-127 up), K = H; epilogue
//     act = silu(g) * u (bf16) for intermediate rows [64 mt, 64 mt + 64);
//   gemm2 unit (e, ht, kc): down rows [128 ht, +128), K chunk kc of I/n_kc;
//     epilogue y[t] += w[t,e] * partial (fp32 atomics, so split-K is free).
// A gemm2 unit needs only the gemm1 tiles of its K chunk: a per-(e, kc) counter
// (release/acquire at gpu scope) gates its act loads, while its weight tiles
// are already streaming into the ring. All gemm1 units precede all gemm2
// units and every CTA walks its units in increasing order, so a waiting unit
// always depends on units that are running or done (grid <= one CTA per SM,
// all resident): no deadlock. TMEM holds two accumulators, so the epilogue
// of one unit overlaps the MMAs of the next.
// Warps: 0 TMA producer, 1 MMA issuer, 2-5 epilogue (TMEM lane quarter w % 4).
constexpr int kFfnThreads = 192;

__host__ __device__ constexpr int ffn_xchg_bytes(int npad) {   // xchg + act tile + scatter staging
    return 64 * npad * 4 + npad * 128 + 4 * 16 * 36 * 4;
}
__host__ __device__ constexpr int ffn_stage_bytes(int npad) { return (BM * BK + npad * BK) * 2; }
__host__ __device__ constexpr int ffn_stages(int npad) {
    return (220 * 1024 - ffn_xchg_bytes(npad)) / ffn_stage_bytes(npad) > 12
               ? 12
               : (220 * 1024 - ffn_xchg_bytes(npad)) / ffn_stage_bytes(npad);
}

template <int NPAD>
struct FfnSmem {
    static constexpr int STAGES = ffn_stages(NPAD);
    alignas(1024) __nv_bfloat16 a[STAGES][BM * BK];
    alignas(1024) __nv_bfloat16 b[STAGES][NPAD * BK];
    alignas(1024) __nv_bfloat16 act_tile[NPAD * 64];   // act box [NPAD tokens][64 rows], 128B-swizzled (TMA store)
    float xchg[64][NPAD];                 // up-row accumulators -> the gate-row threads
    alignas(16) float red[4][16][36];     // per epilogue warp: 16 tokens x 32 rows, transposed for v4 reductions
    uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
    uint32_t tmem;
};

struct FfnArgs {
    const CUtensorMap* w1_maps;      // [n_slots]: tile-major [I/64][H/64][64 gate + 64 up][64] as 2-D [2IH/64][64], box 128 rows
    const CUtensorMap* w2_maps;      // [n_slots]: tile-major [I/64][H/128][128][64] as 2-D [IH/64][64], box 128 rows
    const CUtensorMap* x_map;        // gathered tokens [n_exec*NPAD rows, H cols], box NPAD rows
    const CUtensorMap* act_map;      // [n_exec*NPAD rows, I cols], box NPAD rows
    const int32_t* exec_slot;        // [n_exec] cache slot of each executed expert
    const int32_t* tok_index;        // [n_exec][NPAD] token row or -1
    const float* tok_weight;         // [n_exec][NPAD]
    __nv_bfloat16* act;              // [n_exec][NPAD][I]
    float* y;                        // [T][H] fp32 accumulator
    uint32_t* sync;                  // [n_exec * n_kc] tile counters, [n_exec * n_kc] done counter (self-resetting)
    int I, H, n_exec, n_kc;
    unsigned long long* trace;       // optional [n_units][8] globaltimer ns: [0] first stage ready, [2] accumulator ready, [3] epilogue end
    const uint8_t* qslots;           // quantised decode kernel: slot pool (codes + fp32 row scales per slot)
    int64_t slot_bytes;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct Unit { int kind, e, tile, kc; };

__device__ __forceinline__ Unit ffn_unit(const FfnArgs& g, int u) {
    const int m1 = g.I / 64, u1 = g.n_exec * m1;
    Unit x;
    if (u < u1) { x.kind = 0; x.e = u / m1; x.tile = u - x.e * m1; x.kc = 0; return x; }
    const int v = u - u1, per = (g.H / BM) * g.n_kc;
    x.kind = 1; x.e = v / per;
    const int r = v - x.e * per;
    x.tile = r / g.n_kc; x.kc = r - x.tile * g.n_kc;
    return x;
}

template <int NPAD>
__global__ void __launch_bounds__(kFfnThreads, 1) ffn_fused_kernel(const __grid_constant__ FfnArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    using S = FfnSmem<NPAD>;
    constexpr int STAGES = S::STAGES;
    auto& s = *reinterpret_cast<S*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_units = g.n_exec * (g.I / 64) + g.n_exec * (g.H / BM) * g.n_kc;
    const int kc_len = g.I / g.n_kc;                      // gemm2 K chunk (multiple of 64)
    const int KT = g.H / 64, HT = g.H / BM;               // tile-major weights: k tiles per w1 row tile, w2 row tiles
    const int tiles_per_kc = kc_len / 64;                 // gemm1 tiles feeding one chunk
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1); }
        for (int i = 0; i < 2; i++) { mbar_init(&s.tfull[i], 1); mbar_init(&s.tempty[i], 4); }
        fence_barrier_init();
        prefetch_tmap(g.x_map);
        prefetch_tmap(g.act_map);
    }
    if (warp == 0) tmem_alloc(&s.tmem, tmem_cols(2 * NPAD));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;

    if (warp == 0) {
        if (lane == 0) {                                  // ---- TMA producer
            int k_all = 0;                                // ring position over every unit
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const Unit x = ffn_unit(g, u);
                const int slot = g.exec_slot[x.e];
                if (x.kind == 0) {
                    const CUtensorMap* wm = g.w1_maps + slot;
                    const int nk = g.H / BK;
                    int kb = 0;
                    if (k_all == 0) {   // first unit: weight tiles stream before the gathered tokens exist
                        const int pre = STAGES < nk ? STAGES : nk;
                        for (int k = 0; k < pre; k++) {
                            mbar_expect_tx(&s.full[k], ffn_stage_bytes(NPAD));
                            tma_load_2d(s.a[k], wm, &s.full[k], 0, (x.tile * KT + k) * BM);
                        }
                        pdl_wait();
                        for (int k = 0; k < pre; k++) tma_load_2d(s.b[k], g.x_map, &s.full[k], k * BK, x.e * NPAD);
                        kb = pre;
                        k_all = pre;
                    }
                    for (int k = kb; k < nk; k++, k_all++) {
                        const int st = k_all % STAGES;
                        if (k_all >= STAGES) mbar_wait(&s.empty[st], ((k_all / STAGES) - 1) & 1);
                        mbar_expect_tx(&s.full[st], ffn_stage_bytes(NPAD));
                        tma_load_2d(s.a[st], wm, &s.full[st], 0, (x.tile * KT + k) * BM);    // [64 gate; 64 up] rows
                        tma_load_2d(s.b[st], g.x_map, &s.full[st], k * BK, x.e * NPAD);
                    }
                } else {
                    const CUtensorMap* wm = g.w2_maps + slot;
                    const int nk = kc_len / BK, k0 = x.kc * kc_len;
                    const int pre = nk < STAGES ? nk : STAGES;
                    // weights first: they do not depend on gemm1
                    for (int k = 0; k < pre; k++) {
                        const int st = (k_all + k) % STAGES;
                        if (k_all + k >= STAGES) mbar_wait(&s.empty[st], (((k_all + k) / STAGES) - 1) & 1);
                        mbar_expect_tx(&s.full[st], ffn_stage_bytes(NPAD));
                        tma_load_2d(s.a[st], wm, &s.full[st], 0, (((k0 + k * BK) / 64) * HT + x.tile) * BM);
                    }
                    const uint32_t* cnt = g.sync + x.e * g.n_kc + x.kc;
                    while (ld_acquire(cnt) < (uint32_t)tiles_per_kc) __nanosleep(64);
                    fence_proxy_async_global();
                    for (int k = 0; k < pre; k++) {
                        const int st = (k_all + k) % STAGES;
                        tma_load_2d(s.b[st], g.act_map, &s.full[st], k0 + k * BK, x.e * NPAD);
                    }
                    for (int k = pre; k < nk; k++) {
                        const int st = (k_all + k) % STAGES;
                        if (k_all + k >= STAGES) mbar_wait(&s.empty[st], (((k_all + k) / STAGES) - 1) & 1);
                        mbar_expect_tx(&s.full[st], ffn_stage_bytes(NPAD));
                        tma_load_2d(s.a[st], wm, &s.full[st], 0, (((k0 + k * BK) / 64) * HT + x.tile) * BM);
                        tma_load_2d(s.b[st], g.act_map, &s.full[st], k0 + k * BK, x.e * NPAD);
                    }
                    k_all += nk;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                  // ---- MMA issuer
            constexpr uint32_t idesc = idesc_bf16(BM, NPAD);
            int k_all = 0, j = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
                const Unit x = ffn_unit(g, u);
                const int buf = j & 1, use = j >> 1;
                if (use >= 1) mbar_wait(&s.tempty[buf], (use - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * NPAD);
                const int nk = x.kind == 0 ? g.H / BK : kc_len / BK;
                for (int k = 0; k < nk; k++, k_all++) {
                    const int st = k_all % STAGES;
                    mbar_wait(&s.full[st], (k_all / STAGES) & 1);
                    if (g.trace && k == 0) g.trace[8 * u] = gtimer();
                    tc_fence_after();
                    const uint64_t a = umma_desc(s.a[st]), b = umma_desc(s.b[st]);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++) umma_bf16(d, a + 2 * kk, b + 2 * kk, idesc, (k | kk) ? 1u : 0u);
                    umma_commit(&s.empty[st]);
                }
                umma_commit(&s.tfull[buf]);
            }
        }
    } else {                                              // ---- epilogue, warps 2..5
        pdl_wait();
        const int q = warp & 3;                           // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;                    // accumulator row (TMEM lane)
        int j = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
            const Unit x = ffn_unit(g, u);
            const int buf = j & 1, use = j >> 1;
            // token table of the unit, loaded before the accumulator wait: under
            // full HBM streaming a global load costs microseconds, hidden here
            constexpr int NR = (NPAD + 31) / 32;
            int tiv[NR];
            float twv[NR];
            int ncol = 0;
#pragma unroll
            for (int r = 0; r < NR; r++) {
                const int c = r * 32 + lane;
                tiv[r] = c < NPAD ? g.tok_index[x.e * NPAD + c] : -1;
                twv[r] = (x.kind == 1 && c < NPAD) ? g.tok_weight[x.e * NPAD + c] : 0.0f;
                ncol = tiv[r] >= 0 ? c + 1 : ncol;
            }
            ncol = __reduce_max_sync(0xffffffffu, ncol);   // token columns in use (padding is never read back)
            mbar_wait(&s.tfull[buf], use & 1);
            __syncwarp();
            tc_fence_after();
            if (g.trace && threadIdx.x == 64) g.trace[8 * u + 2] = gtimer();
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * NPAD);
            if (x.kind == 0) {
                if (row >= 64) {                          // up rows -> exchange
                    for (int c0 = 0; c0 < ncol; c0 += 16) {
                        float v[16];
                        tmem_ld16(taddr + c0, v);
#pragma unroll
                        for (int jj = 0; jj < 16; jj++) s.xchg[row - 64][c0 + jj] = v[jj];
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.tempty[buf]);
                }
                epi_bar();
                if (row < 64) {                           // act = silu(gate) * up -> the swizzled box
                    unsigned char* tile = reinterpret_cast<unsigned char*>(s.act_tile);
                    const int cb = row * 2;
                    for (int c0 = 0; c0 < ncol; c0 += 16) {
                        float gv[16];
                        tmem_ld16(taddr + c0, gv);
#pragma unroll
                        for (int jj = 0; jj < 16; jj++) {
                            const int n = c0 + jj;
                            const float gg = gv[jj];
                            const float a = gg / (1.0f + __expf(-gg)) * s.xchg[row][n];
                            *reinterpret_cast<__nv_bfloat16*>(tile + n * 128 + ((((cb >> 4) ^ (n & 7)) << 4) | (cb & 15))) =
                                __float2bfloat16(a);
                        }
                    }
                    fence_proxy_async_smem();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.tempty[buf]);
                }
                epi_bar();                                // tile written; xchg free again
                if (threadIdx.x == 64) {
                    // one TMA store of the act box, complete before the release; the
                    // consuming producer acquires, then fences the async proxy
                    tma_store_2d(g.act_map, s.act_tile, x.tile * 64, x.e * NPAD);
                    fence_proxy_async_global();
                    red_release_add(g.sync + x.e * g.n_kc + (x.tile * 64) / kc_len, 1u);
                    if (g.trace) g.trace[8 * u + 3] = gtimer();
                }
            } else {
                // y[t][h] += w * v: the warp's 32 rows x 16 token columns are transposed
                // through smem so each lane issues 4-wide vector reductions
                // (red.global.add.v4.f32) over 4 consecutive rows of one token
                float (*rb)[36] = s.red[warp - 2];
                const int hbase = x.tile * BM + q * 32;
                for (int c0 = 0; c0 < ncol; c0 += 16) {
                    float v[16];
                    tmem_ld16(taddr + c0, v);
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) {
                        const int c = c0 + jj;
                        const float w = __shfl_sync(0xffffffffu, twv[c >> 5], c & 31);
                        rb[jj][lane] = w * v[jj];
                    }
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        const int pr = lane + 32 * r, jj = pr >> 3, h4 = (pr & 7) * 4;
                        const int c = c0 + jj;
                        const int t = __shfl_sync(0xffffffffu, tiv[c >> 5], c & 31);
                        if (t >= 0) {
                            const float4 a = *reinterpret_cast<const float4*>(&rb[jj][h4]);
                            float* dst = g.y + (size_t)t * g.H + hbase + h4;
                            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a.x),
                                         "f"(a.y), "f"(a.z), "f"(a.w)
                                         : "memory");
                        }
                    }
                    __syncwarp();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.tempty[buf]);
                if (g.trace && threadIdx.x == 64) g.trace[8 * u + 3] = gtimer();
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols(2 * NPAD));
    // self-resetting counters: the last CTA out zeroes them for the next launch
    if (threadIdx.x == 0) {
        const int nc = g.n_exec * g.n_kc;
        __threadfence();
        if (atomicAdd(g.sync + nc, 1u) == gridDim.x - 1) {
            for (int i = 0; i <= nc; i++) g.sync[i] = 0u;
            __threadfence();
        }
    }
}

// ---- decode path: one unit = one expert's 64-row intermediate slice, fused ----
// With ~1 token per expert the two-phase kernel's critical path is the act
// handoff between CTAs (a globally visible write under full HBM streaming
// costs microseconds). Here a unit computes its slice end to end:
//   gemm1: [64 gate; 64 up] x tokens, K = H             (512 KB of weights)
//   act = silu(g) * u -> a swizzled smem tile, used directly as the B operand of
//   gemm2 partial: Wd[:, 64 mt : 64 mt + 64] x act, K = 64, all H/128 row tiles
//                                                       (256 KB of weights)
//   y[t] += w * partial (fp32 atomics; I/64 partial sums per output element)
// so units never wait on each other. The producer streams the down-projection
// tiles right behind the gate/up tiles (they do not depend on act).
// TMEM: columns [0, 16) gemm1 accumulator, [256, 256 + 16 * H/128) gemm2.
struct DecSmem {
    static constexpr int STAGES = 12;
    alignas(1024) __nv_bfloat16 a[STAGES][BM * BK];
    alignas(1024) __nv_bfloat16 b[STAGES][16 * BK];
    alignas(1024) __nv_bfloat16 act_tile[16 * 64];
    float xchg[64][17];
    uint64_t full[STAGES], empty[STAGES], t1full, t1empty, actrdy, t2full, t2empty;
    uint32_t tmem;
};

__global__ void __launch_bounds__(kFfnThreads, 1) ffn_decode_kernel(const __grid_constant__ FfnArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    using S = DecSmem;
    constexpr int STAGES = S::STAGES;
    constexpr int NPAD = 16;
    auto& s = *reinterpret_cast<S*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m1 = g.I / 64, n_units = g.n_exec * m1, n_ht = g.H / BM;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1); }
        mbar_init(&s.t1full, 1); mbar_init(&s.t1empty, 4); mbar_init(&s.actrdy, 2);   // one per act-writing warp
        mbar_init(&s.t2full, 1); mbar_init(&s.t2empty, 4);
        fence_barrier_init();
        prefetch_tmap(g.x_map);
    }
    if (warp == 0) tmem_alloc(&s.tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = NPAD * BK * 2;

    if (warp == 0) {
        if (lane == 0) {                                  // ---- TMA producer
            int k_all = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const int e = u / m1, mt = u - e * m1;
                const int slot = g.exec_slot[e];
                const CUtensorMap* w1 = g.w1_maps + slot;
                const CUtensorMap* w2 = g.w2_maps + slot;
                const int KT = g.H / 64;
                int k0 = 0;
                if (k_all == 0) {       // first unit: its weight tiles stream before the gathered tokens exist
                    const int pre = STAGES < g.H / BK ? STAGES : g.H / BK;
                    for (int k = 0; k < pre; k++) {
                        mbar_expect_tx(&s.full[k], A_BYTES + B_BYTES);
                        tma_load_2d(s.a[k], w1, &s.full[k], 0, (mt * KT + k) * BM);
                    }
                    pdl_wait();
                    for (int k = 0; k < pre; k++) tma_load_2d(s.b[k], g.x_map, &s.full[k], k * BK, e * NPAD);
                    k0 = pre;
                    k_all = pre;
                }
                for (int k = k0; k < g.H / BK; k++, k_all++) {
                    const int st = k_all % STAGES;
                    if (k_all >= STAGES) mbar_wait(&s.empty[st], ((k_all / STAGES) - 1) & 1);
                    mbar_expect_tx(&s.full[st], A_BYTES + B_BYTES);
                    tma_load_2d(s.a[st], w1, &s.full[st], 0, (mt * KT + k) * BM);          // [64 gate; 64 up] rows
                    tma_load_2d(s.b[st], g.x_map, &s.full[st], k * BK, e * NPAD);
                }
                for (int ht = 0; ht < n_ht; ht++, k_all++) {
                    const int st = k_all % STAGES;
                    if (k_all >= STAGES) mbar_wait(&s.empty[st], ((k_all / STAGES) - 1) & 1);
                    mbar_expect_tx(&s.full[st], A_BYTES);
                    tma_load_2d(s.a[st], w2, &s.full[st], 0, (mt * n_ht + ht) * BM);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                  // ---- MMA issuer
            constexpr uint32_t idesc = idesc_bf16(BM, NPAD);
            const uint64_t bact = umma_desc(s.act_tile);
            int k_all = 0, j = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
                if (j >= 1) mbar_wait(&s.t1empty, (j - 1) & 1);     // gemm1 accumulator drained
                tc_fence_after();
                for (int k = 0; k < g.H / BK; k++, k_all++) {
                    const int st = k_all % STAGES;
                    mbar_wait(&s.full[st], (k_all / STAGES) & 1);
                    tc_fence_after();
                    const uint64_t a = umma_desc(s.a[st]), b = umma_desc(s.b[st]);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++) umma_bf16(tmem, a + 2 * kk, b + 2 * kk, idesc, (k | kk) ? 1u : 0u);
                    umma_commit(&s.empty[st]);
                }
                umma_commit(&s.t1full);
                mbar_wait(&s.actrdy, j & 1);                       // act tile of this unit in smem
                if (j >= 1) mbar_wait(&s.t2empty, (j - 1) & 1);    // gemm2 accumulators drained
                tc_fence_after();
                for (int ht = 0; ht < n_ht; ht++, k_all++) {
                    const int st = k_all % STAGES;
                    mbar_wait(&s.full[st], (k_all / STAGES) & 1);
                    tc_fence_after();
                    const uint64_t a = umma_desc(s.a[st]);
                    const uint32_t d = tmem + 256u + (uint32_t)(ht * NPAD);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++) umma_bf16(d, a + 2 * kk, bact + 2 * kk, idesc, kk ? 1u : 0u);
                    umma_commit(&s.empty[st]);
                }
                umma_commit(&s.t2full);
            }
        }
    } else {                                              // ---- epilogue, warps 2..5
        pdl_wait();                                       // (the token tables / y precede the gather: belt and braces)
        const int q = warp & 3, row = q * 32 + lane;
        const uint32_t lanebase = (uint32_t)(q * 32) << 16;
        int j = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
            const int e = u / m1;
            const int ti = lane < NPAD ? g.tok_index[e * NPAD + lane] : -1;
            const float tw = lane < NPAD ? g.tok_weight[e * NPAD + lane] : 0.0f;
            const int ncol = __reduce_max_sync(0xffffffffu, ti >= 0 ? lane + 1 : 0);
            // gemm1 epilogue: act = silu(gate) * up -> act_tile (swizzled, the gemm2 B operand)
            mbar_wait(&s.t1full, j & 1);
            __syncwarp();
            tc_fence_after();
            float v[16];
            tmem_ld16(tmem + lanebase, v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.t1empty);
            if (row >= 64) {
#pragma unroll
                for (int c = 0; c < 16; c++) s.xchg[row - 64][c] = v[c];
            }
            epi_bar();
            if (row < 64) {
                unsigned char* tile = reinterpret_cast<unsigned char*>(s.act_tile);
                const int cb = row * 2;
#pragma unroll
                for (int n = 0; n < 16; n++) {
                    const float gg = v[n];
                    const float a = n < ncol ? gg / (1.0f + __expf(-gg)) * s.xchg[row][n] : 0.0f;
                    *reinterpret_cast<__nv_bfloat16*>(tile + n * 128 + ((((cb >> 4) ^ (n & 7)) << 4) | (cb & 15))) =
                        __float2bfloat16(a);
                }
                fence_proxy_async_smem();                 // generic smem writes -> the tensor core's view
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.actrdy);
            }
            // gemm2 epilogue: partial sums of the H rows, scaled, into y
            mbar_wait(&s.t2full, j & 1);
            __syncwarp();
            tc_fence_after();
            for (int ht = 0; ht < n_ht; ht++) {
                float p[16];
                tmem_ld16(tmem + lanebase + 256u + (uint32_t)(ht * NPAD), p);
                const int h = ht * BM + row;
#pragma unroll
                for (int c = 0; c < 16; c++) {            // static index: p stays in registers
                    if (c >= ncol) break;                 // (ncol is warp-uniform)
                    const int t = __shfl_sync(0xffffffffu, ti, c);
                    const float w = __shfl_sync(0xffffffffu, tw, c);
                    if (t >= 0) atomicAdd(&g.y[(size_t)t * g.H + h], w * p[c]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.t2empty);
            epi_bar();                                    // xchg / act_tile reuse by the next unit
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int NPAD>
size_t ffn_smem() { return sizeof(FfnSmem<NPAD>) + 1024; }

static int ffn_grid_cap() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

// ---- decode path over quantised slots: dequantisation fused into the A operand ----
// Same units and epilogue as ffn_decode_kernel, but the weight tiles stay in
// their quantised form all the way into shared memory: the producer bulk-copies
// each 128 x 64 tile's codes (8192 * BITS / 8 contiguous bytes of the
// tile-major slot, layer_step.cu) into a code ring, four converter warps turn
// them into the 128B-swizzled bf16 A tile (w = bf16(q * s_row), the row
// scales read through L1), fence the generic writes into the async proxy and
// arrive on the A ring's full barrier; the MMA issuer is unchanged. HBM reads
// per expert: 3*H*I*BITS/8 + scales instead of the dequantise-to-scratch
// path's codes + 2 x 3*H*I*2 B (scratch write + FFN read).
// The unit's gathered tokens (NPAD x H bf16 <= 64 KB) are loaded once per
// unit into their own buffer (every gemm1 step reuses them); the row scales (64 gate + 64 up + all H down rows,
// double-buffered by unit) are applied by the epilogue to the fp32
// accumulators (the A tile carries the integer codes, exact in bf16).
// Warps: 0 code producer, 1 MMA, 2-5 epilogue, 6-13 converters (two per SMSP:
// the conversion is ALU work on the tile's critical path: int4 / int2 pairs are
// one LOP3 + one bf16x2 subtract).
constexpr int kDecQConv = 256;
constexpr int kDecQThreads = 192 + kDecQConv;

#ifndef DECQ_DIAG
#define DECQ_DIAG 0   // A/B diagnostics: 1 no conversion, 2 no gemm1 MMAs, 3 phase stamps, 5 no conversion
                      // and no proxy fence, 6 = 5 + no gemm1 MMAs (the hand-off skeleton)
#endif
#ifndef DECQ_AS
#define DECQ_AS 4                                         // A (bf16) ring stages
#endif
#ifndef DECQ_QRING
#define DECQ_QRING (32 * 1024)                            // code ring bytes
#endif
template <int BITS>
struct DecQSmem {
    static constexpr int AS = DECQ_AS;
    static constexpr int QBYTES = BM * BK * BITS / 8;
    static constexpr int QS = DECQ_QRING / QBYTES;
    alignas(1024) __nv_bfloat16 a[AS][BM * BK];
    alignas(1024) __nv_bfloat16 xs[32][16 * BK];          // the unit's tokens, one 16 x 64 box per k (H <= 2048)
    alignas(1024) __nv_bfloat16 act_tile[16 * 64];
    alignas(128) uint8_t q[QS][QBYTES];
    alignas(16) float sc[2][128 + 2048];                  // per unit: gate, up, then the H down-row scales
    float xchg[64][17];
    uint64_t full[AS], empty[AS], qfull[QS], qempty[QS], xfull, xempty, sfull[2], sempty[2];
    uint64_t t1full, t1empty, actrdy, t2full, t2empty;
    uint32_t tmem;
};

template <int BITS>
__global__ void __launch_bounds__(kDecQThreads, 1) ffn_decode_q_kernel(const __grid_constant__ FfnArgs g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
#if DECQ_DIAG == 3
    __shared__ unsigned long long dq_t[16];
#define DQ_STAMP(i) do { unsigned long long _t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t)); dq_t[i] = _t; } while (0)
#else
#define DQ_STAMP(i) do {} while (0)
#endif
    using S = DecQSmem<BITS>;
    constexpr int AS = S::AS, QS = S::QS;
    constexpr uint32_t QBYTES = S::QBYTES;
    constexpr int NPAD = 16;
    auto& s = *reinterpret_cast<S*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m1 = g.I / 64, n_units = g.n_exec * m1, n_ht = g.H / BM, KT = g.H / BK;
    if (threadIdx.x == 0) DQ_STAMP(0);
    if (threadIdx.x == 0) {
        // converter hand-offs arrive once per warp
        for (int i = 0; i < AS; i++) { mbar_init(&s.full[i], kDecQConv / 32); mbar_init(&s.empty[i], 1); }
        for (int i = 0; i < QS; i++) { mbar_init(&s.qfull[i], 1); mbar_init(&s.qempty[i], kDecQConv / 32); }
        mbar_init(&s.xfull, 1); mbar_init(&s.xempty, 1);
        for (int i = 0; i < 2; i++) { mbar_init(&s.sfull[i], 1); mbar_init(&s.sempty[i], 4); }
        mbar_init(&s.t1full, 1); mbar_init(&s.t1empty, 4); mbar_init(&s.actrdy, 2);   // one per act-writing warp
        mbar_init(&s.t2full, 1); mbar_init(&s.t2empty, 4);
        fence_barrier_init();
        prefetch_tmap(g.x_map);
    }
    if (warp == 0) tmem_alloc(&s.tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    const int64_t n1 = 2LL * g.I * g.H;                   // w1 codes; then the w2 codes
    const int64_t soff = 3LL * g.I * g.H * BITS / 8;      // fp32 scales: 2I gate/up rows, H down rows

    if (warp == 0) {
        if (lane == 0) {                                  // ---- producer: code tiles + row scales
            int kq = 0, j = 0;
            auto code_tile = [&](const uint8_t* src) {
                const int st = kq % QS;
                if (kq >= QS) mbar_wait(&s.qempty[st], ((kq / QS) - 1) & 1);
                mbar_expect_tx(&s.qfull[st], QBYTES);
                bulk_load(s.q[st], src, QBYTES, &s.qfull[st]);
                kq++;
            };
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
                const int e = u / m1, mt = u - e * m1;
                const uint8_t* base = g.qslots + (int64_t)g.exec_slot[e] * g.slot_bytes;
                const float* s1 = reinterpret_cast<const float*>(base + soff);
                const int sb = j & 1;
                if (j >= 2) mbar_wait(&s.sempty[sb], ((j >> 1) - 1) & 1);
                mbar_expect_tx(&s.sfull[sb], (uint32_t)(128 + g.H) * 4);
                bulk_load(s.sc[sb], s1 + mt * 64, 256, &s.sfull[sb]);
                bulk_load(s.sc[sb] + 64, s1 + g.I + mt * 64, 256, &s.sfull[sb]);
                bulk_load(s.sc[sb] + 128, s1 + 2 * g.I, (uint32_t)g.H * 4, &s.sfull[sb]);
                int k0 = 0;
                if (j == 0) {                             // weights stream before the gathered tokens exist
                    k0 = QS < KT ? QS : KT;
                    for (int k = 0; k < k0; k++) code_tile(base + (int64_t)(mt * KT + k) * QBYTES);
                    pdl_wait();
                    DQ_STAMP(1);
                }
                if (j >= 1) mbar_wait(&s.xempty, (j - 1) & 1);
                mbar_expect_tx(&s.xfull, (uint32_t)(KT * NPAD * BK * 2));
                for (int k = 0; k < KT; k++) tma_load_2d(s.xs[k], g.x_map, &s.xfull, k * BK, e * NPAD);
                for (int k = k0; k < KT; k++) code_tile(base + (int64_t)(mt * KT + k) * QBYTES);
                for (int ht = 0; ht < n_ht; ht++)
                    code_tile(base + n1 * BITS / 8 + (int64_t)(mt * n_ht + ht) * QBYTES);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                  // ---- MMA issuer
            constexpr uint32_t idesc = idesc_bf16(BM, NPAD);
            const uint64_t bact = umma_desc(s.act_tile);
            int ka = 0, j = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
                if (j >= 1) mbar_wait(&s.t1empty, (j - 1) & 1);
                mbar_wait(&s.xfull, j & 1);
                if (j == 0) DQ_STAMP(2);
                tc_fence_after();
                for (int k = 0; k < KT; k++, ka++) {
                    const int st = ka % AS;
                    mbar_wait(&s.full[st], (ka / AS) & 1);
                    tc_fence_after();
                    const uint64_t a = umma_desc(s.a[st]), b = umma_desc(s.xs[k]);
#pragma unroll
                    for (int kk = 0; kk < ((DECQ_DIAG == 2 || DECQ_DIAG == 6) ? 0 : BK / 16); kk++)
                        umma_bf16(tmem, a + 2 * kk, b + 2 * kk, idesc, (k | kk) ? 1u : 0u);
                    umma_commit(&s.empty[st]);
                }
                if (j == 0) DQ_STAMP(3);
                umma_commit(&s.t1full);
                umma_commit(&s.xempty);
                mbar_wait(&s.actrdy, j & 1);
                if (j == 0) DQ_STAMP(6);
                if (j >= 1) mbar_wait(&s.t2empty, (j - 1) & 1);
                tc_fence_after();
                for (int ht = 0; ht < n_ht; ht++, ka++) {
                    const int st = ka % AS;
                    mbar_wait(&s.full[st], (ka / AS) & 1);
                    tc_fence_after();
                    const uint64_t a = umma_desc(s.a[st]);
                    const uint32_t d = tmem + 256u + (uint32_t)(ht * NPAD);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++) umma_bf16(d, a + 2 * kk, bact + 2 * kk, idesc, kk ? 1u : 0u);
                    umma_commit(&s.empty[st]);
                }
                umma_commit(&s.t2full);
            }
        }
    } else if (warp >= 6) {                               // ---- converters: codes -> swizzled bf16 A tiles
        // The A tile holds the integer codes themselves (exact in bf16); the
        // per-row scale is applied to the fp32 accumulator in the epilogue
        // (the TMEM lane is the weight row: y = s_row * (q . x)).
        // int4 / int2 words are interleaved (layer_step.py code_positions):
        // (w >> BITS*j) & 0x000F000F (0x00030003) holds elements (2j, 2j+1) in
        // its two half-words, so one LOP3 makes the pair's bf16x2 128 + u
        // (u = q + 2^(BITS-1), offset binary) and one bf16x2 subtract gives q.
        const int ct = threadIdx.x - 192;
        constexpr int NI = BM * BK / 16 / kDecQConv;      // 16-code items per thread per tile
        int kq = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            for (int t = 0; t < KT + n_ht; t++, kq++) {
                const int qs = kq % QS, st = kq % AS;
                mbar_wait(&s.qfull[qs], (kq / QS) & 1);
                if (kq >= AS) mbar_wait(&s.empty[st], ((kq / AS) - 1) & 1);
                const uint32_t dst = smem_u32(s.a[st]);
#pragma unroll
                for (int i = 0; i < ((DECQ_DIAG == 1 || DECQ_DIAG >= 5) ? 0 : NI); i++) {
                    const int it = ct + kDecQConv * i, r = it >> 2, c0 = (it & 3) * 2;   // row, first 16-B chunk
                    uint32_t o[8];                         // bf16 pairs, element 2c in the low half
                    if (BITS == 8) {
                        const uint4 v = *reinterpret_cast<const uint4*>(s.q[qs] + it * 16);
                        const uint32_t wq[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int c = 0; c < 8; c++) {
                            const uint32_t w = wq[c >> 1], sh = (c & 1) * 16;
                            // (float)q exactly: bits(1.5 * 2^23) + q, minus 1.5 * 2^23
                            const int q0 = (int)(w << (24 - sh)) >> 24, q1 = (int)(w << (16 - sh)) >> 24;
                            const float f0 = __int_as_float(0x4B400000 + q0) - 12582912.0f;
                            const float f1 = __int_as_float(0x4B400000 + q1) - 12582912.0f;
                            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(o[c]) : "f"(f1), "f"(f0));
                        }
                    } else {
                        constexpr uint32_t MASK = BITS == 4 ? 0x000F000Fu : 0x00030003u;
                        constexpr uint32_t BIAS = BITS == 4 ? 0x43084308u : 0x43024302u;   // 128 + 2^(BITS-1)
                        constexpr int PAIRS = 16 / BITS;                                  // pairs per word
                        uint32_t wq[2];
                        if (BITS == 4) {
                            const uint2 v = *reinterpret_cast<const uint2*>(s.q[qs] + it * 8);
                            wq[0] = v.x; wq[1] = v.y;
                        } else {
                            wq[0] = *reinterpret_cast<const uint32_t*>(s.q[qs] + it * 4);
                        }
#pragma unroll
                        for (int c = 0; c < 8; c++) {
                            const uint32_t w = wq[c / PAIRS] >> (BITS * (c % PAIRS));
                            uint32_t h;                    // ((w & MASK) ^ BIAS): 128 + u in each half
                            asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(h) : "r"(w), "r"(MASK), "r"(BIAS));
                            asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(o[c]) : "r"(h), "r"(BIAS));
                        }
                    }
                    const uint32_t row = dst + r * 128;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((c0 ^ (r & 7)) << 4)),
                                 "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]) : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + (((c0 + 1) ^ (r & 7)) << 4)),
                                 "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]) : "memory");
                }
                if (DECQ_DIAG < 5) fence_proxy_async_smem();   // generic smem writes -> the tensor core's view
                __syncwarp();                             // the warp's codes read, its tile rows written + fenced
                if (lane == 0) {
                    mbar_arrive(&s.qempty[qs]);
                    mbar_arrive(&s.full[st]);
                }
                if (ct == 0 && kq == 0) DQ_STAMP(9);
                if (ct == 0 && kq == KT - 1) DQ_STAMP(10);
            }
        }
    } else {                                              // ---- epilogue, warps 2..5 (ffn_decode_kernel's)
        pdl_wait();
        const int q = warp & 3, row = q * 32 + lane;
        const uint32_t lanebase = (uint32_t)(q * 32) << 16;
        int j = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, j++) {
            const int e = u / m1;
            const int ti = lane < NPAD ? g.tok_index[e * NPAD + lane] : -1;
            const float tw = lane < NPAD ? g.tok_weight[e * NPAD + lane] : 0.0f;
            const int ncol = __reduce_max_sync(0xffffffffu, ti >= 0 ? lane + 1 : 0);
            const int sb = j & 1;
            mbar_wait(&s.sfull[sb], (j >> 1) & 1);        // this unit's row scales
            const float s1 = s.sc[sb][row];               // gate rows 0-63, up rows 64-127
            mbar_wait(&s.t1full, j & 1);
            if (j == 0 && threadIdx.x == 64) DQ_STAMP(4);
            __syncwarp();
            tc_fence_after();
            float v[16];
            tmem_ld16(tmem + lanebase, v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.t1empty);
#pragma unroll
            for (int c = 0; c < 16; c++) v[c] *= s1;      // w = q * s_row
            if (row >= 64) {
#pragma unroll
                for (int c = 0; c < 16; c++) s.xchg[row - 64][c] = v[c];
            }
            epi_bar();
            if (row < 64) {
                unsigned char* tile = reinterpret_cast<unsigned char*>(s.act_tile);
                const int cb = row * 2;
#pragma unroll
                for (int n = 0; n < 16; n++) {
                    const float gg = v[n];
                    const float a = n < ncol ? gg / (1.0f + __expf(-gg)) * s.xchg[row][n] : 0.0f;
                    *reinterpret_cast<__nv_bfloat16*>(tile + n * 128 + ((((cb >> 4) ^ (n & 7)) << 4) | (cb & 15))) =
                        __float2bfloat16(a);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.actrdy);
                if (j == 0 && threadIdx.x == 64) DQ_STAMP(5);
            }
            mbar_wait(&s.t2full, j & 1);
            if (j == 0 && threadIdx.x == 64) DQ_STAMP(7);
            __syncwarp();
            tc_fence_after();
            for (int ht = 0; ht < n_ht; ht++) {
                float p[16];
                tmem_ld16(tmem + lanebase + 256u + (uint32_t)(ht * NPAD), p);
                const int h = ht * BM + row;
                const float s2 = s.sc[sb][128 + h];       // down row h
#pragma unroll
                for (int c = 0; c < 16; c++) {            // static index: p stays in registers
                    if (c >= ncol) break;                 // (ncol is warp-uniform)
                    const int t = __shfl_sync(0xffffffffu, ti, c);
                    const float w = __shfl_sync(0xffffffffu, tw, c);
                    if (t >= 0) atomicAdd(&g.y[(size_t)t * g.H + h], w * (p[c] * s2));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.sempty[sb]);    // this unit's scales consumed (one per warp)
            if (j == 0 && threadIdx.x == 64) DQ_STAMP(8);
            if (lane == 0) mbar_arrive(&s.t2empty);
            epi_bar();
        }
    }
    tc_fence_before();
    __syncthreads();
#if DECQ_DIAG == 3
    if (threadIdx.x == 0 && blockIdx.x < 3) {
        DQ_STAMP(11);
        printf("dq blk %d: pdl %lld xfull %lld g1issued %lld t1full %lld act %lld mma_act %lld t2full %lld unitend %lld conv0 %lld convKT %lld end %lld (ns from entry)\n",
               blockIdx.x, dq_t[1] - dq_t[0], dq_t[2] - dq_t[0], dq_t[3] - dq_t[0], dq_t[4] - dq_t[0], dq_t[5] - dq_t[0],
               dq_t[6] - dq_t[0], dq_t[7] - dq_t[0], dq_t[8] - dq_t[0], dq_t[9] - dq_t[0], dq_t[10] - dq_t[0], dq_t[11] - dq_t[0]);
    }
#endif
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int BITS>
cudaError_t launch_decode_q(const FfnArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(DecQSmem<BITS>) + 1024;
    cudaError_t e = cudaFuncSetAttribute(ffn_decode_q_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int units = a.n_exec * (a.I / 64);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(units < ffn_grid_cap() ? units : ffn_grid_cap());
    lc.blockDim = dim3(kDecQThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, ffn_decode_q_kernel<BITS>, a);
}

template <int NPAD>
cudaError_t launch_ffn(const FfnArgs& a, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(ffn_fused_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)ffn_smem<NPAD>());
    if (e != cudaSuccess) return e;
    const int n_units = a.n_exec * (a.I / 64) + a.n_exec * (a.H / BM) * a.n_kc;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(n_units < ffn_grid_cap() ? n_units : ffn_grid_cap());
    lc.blockDim = dim3(kFfnThreads);
    lc.dynamicSmemBytes = ffn_smem<NPAD>();
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // prologue overlaps the gather
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, ffn_fused_kernel<NPAD>, a);
}

// gather token rows per executed expert: xg[e][n][:] = x[tok_index[e][n]][:] (zero for padding)
__global__ void gather_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ tok_index,
                              __nv_bfloat16* __restrict__ xg, int npad, int H) {
    pdl_launch_dependents();                          // let the FFN kernel start its prologue now
    const int row = blockIdx.x;                       // e * npad + n
    const int t = tok_index[row];
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)(t < 0 ? 0 : t) * H);
    uint4* dst = reinterpret_cast<uint4*>(xg + (size_t)row * H);
    for (int i = threadIdx.x; i < H / 8; i += blockDim.x) dst[i] = t < 0 ? make_uint4(0, 0, 0, 0) : src[i];
}

// x += bf16(y); y = 0   (residual update between layers)
__global__ void residual_kernel(__nv_bfloat16* __restrict__ x, float* __restrict__ y, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        x[i] = __float2bfloat16(__bfloat162float(x[i]) + y[i]);
        y[i] = 0.0f;
    }
}

}  // namespace ffn
}  // namespace esim

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace esim::ffn;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D bf16 tensor map, row-major [rows][cols], box [box_rows][64 cols], 128B swizzle
extern "C" int esim_tmap_bf16(void* out_map, const void* base, int64_t rows, int64_t cols, int32_t box_rows) {
    auto enc = get_encode();
    if (!enc) return -3;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

extern "C" int esim_ffn_gather(const void* d_x, const int32_t* d_tok_index, void* d_xg, int32_t n_exec, int32_t npad,
                               int32_t H, void* stream) {
    if (n_exec <= 0) return 0;
    gather_kernel<<<n_exec * npad, 128, 0, (cudaStream_t)stream>>>(
        (const __nv_bfloat16*)d_x, d_tok_index, (__nv_bfloat16*)d_xg, npad, H);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

extern "C" int esim_ffn_residual(void* d_x, float* d_y, int64_t n, void* stream) {
    residual_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>((__nv_bfloat16*)d_x, d_y, (int)n);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// per-stream counters for the gemm1 -> gemm2 handoff (zeroed once, then
// self-resetting at the end of every launch; launches on one stream are ordered)
static cudaError_t ffn_sync_buf(cudaStream_t st, size_t n, uint32_t** out) {
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, std::pair<uint32_t*, size_t>> bufs;
    std::lock_guard<std::mutex> lock(mu);
    auto& b = bufs[st];
    if (b.second < n) {
        if (b.first) { cudaStreamSynchronize(st); cudaFree(b.first); b = {nullptr, 0}; }
        cudaError_t e = cudaMalloc((void**)&b.first, n * 4);
        if (e != cudaSuccess) return e;
        if ((e = cudaMemset(b.first, 0, n * 4)) != cudaSuccess) return e;
        b.second = n;
    }
    *out = b.first;
    return cudaSuccess;
}

static unsigned long long* g_ffn_trace = nullptr;   // diagnostics: per-unit timestamps of the next launches
extern "C" int esim_ffn_set_trace(void* d_trace) {
    g_ffn_trace = (unsigned long long*)d_trace;
    return 0;
}

// act = silu(Xg Wg^T) * (Xg Wu^T); y[t] += w * (act Wd^T)   for n_exec experts,
// one persistent launch (gemm1 tiles, then split-K gemm2 units)
extern "C" int esim_ffn_experts_ex(const void* d_w1_maps, const void* d_w2_maps, const void* d_x_map,
                                   const void* d_act_map, const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                   const float* d_tok_weight, void* d_act, float* d_y, int32_t n_exec, int32_t npad,
                                   int32_t I, int32_t H, int32_t max_tok, void* stream) {
    if (n_exec <= 0) return 0;
    if (I % BM || H % BM || H % BK || I % BK) return -1;
    cudaStream_t st = (cudaStream_t)stream;
    // decode-like layers (<= 4 tokens per expert): the fused per-slice kernel
    // (I/64 partial sums per output element; bounded atomics), TMEM 256 + 16 * H/128 columns
    if (npad == 16 && max_tok >= 1 && max_tok <= 4 && H / BM <= 16) {
        FfnArgs a{(const CUtensorMap*)d_w1_maps, (const CUtensorMap*)d_w2_maps, (const CUtensorMap*)d_x_map,
                  (const CUtensorMap*)d_act_map, d_exec_slot, d_tok_index, d_tok_weight, (__nv_bfloat16*)d_act, d_y,
                  nullptr, I, H, n_exec, 1, nullptr};
        const size_t smem = sizeof(DecSmem) + 1024;
        if (cudaFuncSetAttribute(ffn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return -3;
        const int units = n_exec * (I / 64);
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(units < ffn_grid_cap() ? units : ffn_grid_cap());
        lc.blockDim = dim3(kFfnThreads);
        lc.dynamicSmemBytes = smem;
        lc.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        return cudaLaunchKernelEx(&lc, ffn_decode_kernel, a) == cudaSuccess ? 0 : -3;
    }
    // gemm2 split-K: enough units to cover the SMs, chunks of >= 256 columns
    int n_kc = 1;
    while (n_kc < 4 && (I / (2 * n_kc)) % 256 == 0 && n_exec * (H / BM) * n_kc < 2 * ffn_grid_cap()) n_kc *= 2;
    uint32_t* sync = nullptr;
    if (ffn_sync_buf(st, (size_t)n_exec * n_kc + 1, &sync) != cudaSuccess) return -3;
    FfnArgs a{(const CUtensorMap*)d_w1_maps, (const CUtensorMap*)d_w2_maps, (const CUtensorMap*)d_x_map,
              (const CUtensorMap*)d_act_map, d_exec_slot, d_tok_index, d_tok_weight, (__nv_bfloat16*)d_act, d_y,
              sync, I, H, n_exec, n_kc, g_ffn_trace};
    cudaError_t e;
    switch (npad) {
    case 16: e = launch_ffn<16>(a, st); break;
    case 32: e = launch_ffn<32>(a, st); break;
    case 64: e = launch_ffn<64>(a, st); break;
    case 128: e = launch_ffn<128>(a, st); break;
    default: return -1;
    }
    return e == cudaSuccess ? 0 : -3;
}

// decode-like layers over quantised slots (BITS 8 / 4 / 2, the layout of
// layer_step.cu): dequantisation fused into the FFN's A operand
extern "C" int esim_ffn_experts_q(const void* d_slots, int64_t slot_bytes, int32_t bits, const void* d_x_map,
                                  const int32_t* d_exec_slot, const int32_t* d_tok_index, const float* d_tok_weight,
                                  float* d_y, int32_t n_exec, int32_t I, int32_t H, void* stream) {
    if (n_exec <= 0) return 0;
    if (I % BM || H % BM || H / BK > 32 || (slot_bytes & 127)) return -1;
    FfnArgs a{nullptr, nullptr, (const CUtensorMap*)d_x_map, nullptr, d_exec_slot, d_tok_index, d_tok_weight,
              nullptr, d_y, nullptr, I, H, n_exec, 1, nullptr, (const uint8_t*)d_slots, slot_bytes};
    cudaError_t e;
    switch (bits) {
    case 8: e = launch_decode_q<8>(a, (cudaStream_t)stream); break;
    case 4: e = launch_decode_q<4>(a, (cudaStream_t)stream); break;
    case 2: e = launch_decode_q<2>(a, (cudaStream_t)stream); break;
    default: return -1;
    }
    return e == cudaSuccess ? 0 : -3;
}

extern "C" int esim_ffn_experts(const void* d_w1_maps, const void* d_w2_maps, const void* d_x_map,
                                const void* d_act_map, const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                const float* d_tok_weight, void* d_act, float* d_y, int32_t n_exec, int32_t npad,
                                int32_t I, int32_t H, void* stream) {
    return esim_ffn_experts_ex(d_w1_maps, d_w2_maps, d_x_map, d_act_map, d_exec_slot, d_tok_index, d_tok_weight,
                               d_act, d_y, n_exec, npad, I, H, npad, stream);
}
