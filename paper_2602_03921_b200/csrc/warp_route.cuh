// warp_route.cuh -- warp-level routing helpers shared by the replay kernel
// (cache-aware routing in the loop) and the standalone cache-aware
// route_event kernel: numpy-exact softmax of one row, stable top-k, and
// numpy's float64 pairwise row sum (DeltaAvgState.update, routing.py:88).
#pragma once
#include <cstdint>

#include "numpy_f32.cuh"

#ifndef DFI
#define DFI __device__ __forceinline__
#endif

namespace esim {

DFI void warp_softmax(float* buf, int E, int lane) {
    float m = -__int_as_float(0x7f800000);
    for (int i = lane; i < E; i += 32) m = fmaxf(m, buf[i]);
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncwarp();
    for (int i = lane; i < E; i += 32) buf[i] = np_expf(__fsub_rn(buf[i], m));
    __syncwarp();
    const float S = __fadd_rn(0.0f, warp_pw_sum(buf, E, lane));
    __syncwarp();
    for (int i = lane; i < E; i += 32) buf[i] = __fdiv_rn(buf[i], S);
    __syncwarp();
}

DFI void warp_topk(const float* s, int E, int K, int lane, int16_t* out) {
    uint32_t taken = 0;
    for (int j = 0; j < K; j++) {
        float bv = -1.0f;
        int bi = 0x7fffffff;
        for (int i = lane, t = 0; i < E; i += 32, t++) {
            if (taken & (1u << t)) continue;
            const float v = s[i];
            if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == 0) out[j] = (int16_t)bi;
    }
    __syncwarp();
}

// numpy DOUBLE_pairwise_sum of a float32 row cast to float64 (block of <= 128)
DFI double warp_pw_block_f64(const float* a, int n, int lane) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, (double)a[i]);
        return res;
    }
    const int lim = n - (n % 8);
    double r = 0.0;
    if (lane < 8) {
        r = (double)a[lane];
        for (int i = 8; i < lim; i += 8) r = __dadd_rn(r, (double)a[i + lane]);
    }
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    double res = __shfl_sync(0xffffffffu, r, 0);
    for (int i = lim; i < n; i++) res = __dadd_rn(res, (double)a[i]);
    return res;
}

DFI double warp_pw_mid_f64(const float* a, int n, int lane) {   // n <= 256: the halves are <= 128
    if (n <= 128) return warp_pw_block_f64(a, n, lane);
    const int n2 = pw_split(n);
    return __dadd_rn(warp_pw_block_f64(a, n2, lane), warp_pw_block_f64(a + n2, n - n2, lane));
}

// numpy's recursion: the upper half of n in 249..255 (129..135) splits again
DFI double warp_pw_sum_f64(const float* a, int n, int lane) {
    if (n <= 128) return warp_pw_block_f64(a, n, lane);
    const int n2 = pw_split(n);
    return __dadd_rn(warp_pw_block_f64(a, n2, lane), warp_pw_mid_f64(a + n2, n - n2, lane));
}


}  // namespace esim
