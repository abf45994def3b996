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
#include <cstdint>

#include "../../include/specmd_b200.h"

namespace esim {
namespace ffn {

constexpr int BM = 128;          // weight rows per tile (UMMA M)
constexpr int BK = 64;           // 64 bf16 = 128 B = one swizzle-128B atom row

// Pipeline depth from the shared-memory budget: with tiny token tiles the
// stage is almost all weight tile, and a deep ring keeps enough bytes in
// flight per SM (Little's law) for one CTA to stream at a high rate.
__host__ __device__ constexpr int stages_for(int npad, int na) {
    return (200 * 1024) / ((na * BM * BK + npad * BK) * 2) > 12 ? 12
                                                                 : (200 * 1024) / ((na * BM * BK + npad * BK) * 2);
}

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
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

// ---- shared layout ----------------------------------------------------------
template <int NPAD, int NA>   // NA = number of A tiles per stage (2 for gemm1: gate + up)
struct Smem {
    static constexpr int STAGES = stages_for(NPAD, NA);
    alignas(1024) __nv_bfloat16 a[STAGES][NA][BM * BK];
    alignas(1024) __nv_bfloat16 b[STAGES][NPAD * BK];
    uint64_t full[STAGES], empty[STAGES], done;
    uint32_t tmem;
};

struct Gemm1Args {
    const CUtensorMap* w1_maps;      // [n_slots]: [2I rows, H cols] gate rows then up rows
    const CUtensorMap* x_map;        // gathered tokens [n_exec*NPAD rows, H cols]
    const int32_t* exec_slot;        // [n_exec] cache slot of each executed expert
    __nv_bfloat16* act;              // [n_exec][NPAD][I]
    int I, H, n_mtiles;              // n_mtiles = I / BM
};

template <int NPAD>
__global__ void __launch_bounds__(128, 1) gemm1_kernel(const __grid_constant__ Gemm1Args g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    using S = Smem<NPAD, 2>;
    constexpr int STAGES = S::STAGES;
    auto& s = *reinterpret_cast<S*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int e = blockIdx.x / g.n_mtiles, mt = blockIdx.x % g.n_mtiles;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const CUtensorMap* wmap = g.w1_maps + g.exec_slot[e];
    const int nk = g.H / BK;
    constexpr uint32_t NCOL = 2 * NPAD;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1); }
        mbar_init(&s.done, 1);
        fence_barrier_init();
        prefetch_tmap(wmap);
        prefetch_tmap(g.x_map);
    }
    if (warp == 0) tmem_alloc(&s.tmem, tmem_cols(NCOL));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    if (warp == 0 && lane == 0) {                      // TMA producer
        for (int k = 0; k < nk; k++) {
            const int st = k % STAGES;
            if (k >= STAGES) mbar_wait(&s.empty[st], ((k / STAGES) - 1) & 1);
            mbar_expect_tx(&s.full[st], (2 * BM * BK + NPAD * BK) * 2);
            tma_load_2d(s.a[st][0], wmap, &s.full[st], k * BK, mt * BM);               // gate rows
            tma_load_2d(s.a[st][1], wmap, &s.full[st], k * BK, g.I + mt * BM);         // up rows
            tma_load_2d(s.b[st], g.x_map, &s.full[st], k * BK, e * NPAD);              // tokens
        }
    } else if (warp == 1 && lane == 0) {               // MMA issuer
        constexpr uint32_t idesc = idesc_bf16(BM, NPAD);
        for (int k = 0; k < nk; k++) {
            const int st = k % STAGES;
            mbar_wait(&s.full[st], (k / STAGES) & 1);
            tc_fence_after();
            const uint64_t ag = umma_desc(s.a[st][0]), au = umma_desc(s.a[st][1]), b = umma_desc(s.b[st]);
#pragma unroll
            for (int kk = 0; kk < BK / 16; kk++) {      // +32 B per K=16 step inside the swizzle atom
                const uint32_t acc = (k | kk) ? 1u : 0u;
                umma_bf16(tmem, ag + 2 * kk, b + 2 * kk, idesc, acc);
                umma_bf16(tmem + NPAD, au + 2 * kk, b + 2 * kk, idesc, acc);
            }
            umma_commit(&s.empty[st]);
        }
        umma_commit(&s.done);
    }
    __syncwarp();
    // epilogue: all 4 warps; thread owns intermediate row r = mt*BM + 32*warp + lane
    mbar_wait(&s.done, 0);
    __syncwarp();
    tc_fence_after();
    const int r = mt * BM + warp * 32 + lane;
    __nv_bfloat16* out = g.act + (size_t)e * NPAD * g.I;
#pragma unroll
    for (int c0 = 0; c0 < NPAD; c0 += 16) {
        float gv[16], uv[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, gv);
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + NPAD + c0, uv);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const float gg = gv[j];
            const float a = gg / (1.0f + __expf(-gg)) * uv[j];
            out[(size_t)(c0 + j) * g.I + r] = __float2bfloat16(a);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols(NCOL));
}

struct Gemm2Args {
    const CUtensorMap* w2_maps;      // [n_slots]: [H rows, I cols]
    const CUtensorMap* act_map;      // [n_exec*NPAD rows, I cols]
    const int32_t* exec_slot;        // [n_exec]
    const int32_t* tok_index;        // [n_exec][NPAD] token row or -1
    const float* tok_weight;         // [n_exec][NPAD]
    float* y;                        // [T][H] fp32 accumulator
    int I, H, n_mtiles;              // n_mtiles = H / BM
};

template <int NPAD>
__global__ void __launch_bounds__(128, 1) gemm2_kernel(const __grid_constant__ Gemm2Args g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    using S = Smem<NPAD, 1>;
    constexpr int STAGES = S::STAGES;
    auto& s = *reinterpret_cast<S*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int e = blockIdx.x / g.n_mtiles, mt = blockIdx.x % g.n_mtiles;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const CUtensorMap* wmap = g.w2_maps + g.exec_slot[e];
    const int nk = g.I / BK;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; i++) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1); }
        mbar_init(&s.done, 1);
        fence_barrier_init();
        prefetch_tmap(wmap);
        prefetch_tmap(g.act_map);
    }
    if (warp == 0) tmem_alloc(&s.tmem, tmem_cols(NPAD));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    if (warp == 0 && lane == 0) {
        for (int k = 0; k < nk; k++) {
            const int st = k % STAGES;
            if (k >= STAGES) mbar_wait(&s.empty[st], ((k / STAGES) - 1) & 1);
            mbar_expect_tx(&s.full[st], (BM * BK + NPAD * BK) * 2);
            tma_load_2d(s.a[st][0], wmap, &s.full[st], k * BK, mt * BM);
            tma_load_2d(s.b[st], g.act_map, &s.full[st], k * BK, e * NPAD);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = idesc_bf16(BM, NPAD);
        for (int k = 0; k < nk; k++) {
            const int st = k % STAGES;
            mbar_wait(&s.full[st], (k / STAGES) & 1);
            tc_fence_after();
            const uint64_t a = umma_desc(s.a[st][0]), b = umma_desc(s.b[st]);
#pragma unroll
            for (int kk = 0; kk < BK / 16; kk++) umma_bf16(tmem, a + 2 * kk, b + 2 * kk, idesc, (k | kk) ? 1u : 0u);
            umma_commit(&s.empty[st]);
        }
        umma_commit(&s.done);
    }
    __syncwarp();
    mbar_wait(&s.done, 0);
    __syncwarp();
    tc_fence_after();
    const int h = mt * BM + warp * 32 + lane;
    const int32_t* ti = g.tok_index + e * NPAD;
    const float* tw = g.tok_weight + e * NPAD;
#pragma unroll
    for (int c0 = 0; c0 < NPAD; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int t = ti[c0 + j];
            if (t >= 0) atomicAdd(&g.y[(size_t)t * g.H + h], tw[c0 + j] * v[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols(NPAD));
}

// gather token rows per executed expert: xg[e][n][:] = x[tok_index[e][n]][:] (zero for padding)
__global__ void gather_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ tok_index,
                              __nv_bfloat16* __restrict__ xg, int npad, int H) {
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

template <int NPAD>
size_t smem1() { return sizeof(Smem<NPAD, 2>) + 1024; }
template <int NPAD>
size_t smem2() { return sizeof(Smem<NPAD, 1>) + 1024; }

template <int NPAD>
cudaError_t launch_ffn(const Gemm1Args& a1, const Gemm2Args& a2, int n_exec, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(gemm1_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem1<NPAD>());
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm2_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2<NPAD>());
    if (e != cudaSuccess) return e;
    gemm1_kernel<NPAD><<<n_exec * a1.n_mtiles, 128, smem1<NPAD>(), st>>>(a1);
    gemm2_kernel<NPAD><<<n_exec * a2.n_mtiles, 128, smem2<NPAD>(), st>>>(a2);
    return cudaGetLastError();
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

// act = silu(Xg Wg^T) * (Xg Wu^T); y[t] += w * (act Wd^T)   for n_exec experts
extern "C" int esim_ffn_experts(const void* d_w1_maps, const void* d_w2_maps, const void* d_x_map,
                                const void* d_act_map, const int32_t* d_exec_slot, const int32_t* d_tok_index,
                                const float* d_tok_weight, void* d_act, float* d_y, int32_t n_exec, int32_t npad,
                                int32_t I, int32_t H, void* stream) {
    if (n_exec <= 0) return 0;
    if (I % BM || H % BM || H % BK || I % BK) return -1;
    Gemm1Args a1{(const CUtensorMap*)d_w1_maps, (const CUtensorMap*)d_x_map, d_exec_slot, (__nv_bfloat16*)d_act, I, H,
                 I / BM};
    Gemm2Args a2{(const CUtensorMap*)d_w2_maps, (const CUtensorMap*)d_act_map, d_exec_slot, d_tok_index, d_tok_weight,
                 d_y, I, H, H / BM};
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    switch (npad) {
    case 16: e = launch_ffn<16>(a1, a2, n_exec, st); break;
    case 32: e = launch_ffn<32>(a1, a2, n_exec, st); break;
    case 64: e = launch_ffn<64>(a1, a2, n_exec, st); break;
    case 128: e = launch_ffn<128>(a1, a2, n_exec, st); break;
    default: return -1;
    }
    return e == cudaSuccess ? 0 : -3;
}
