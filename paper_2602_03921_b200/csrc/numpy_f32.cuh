// numpy_f32.cuh -- bit-exact device restatement of numpy's float32 softmax
// pieces used by the reference router (routing.py:22-29):
//   np.exp(float32)            numpy simd_exp_FLOAT (AVX2/AVX-512 hosts)
//   e.sum(axis=1, float32)     numpy FLOAT_pairwise_sum (8 accumulators)
//   x - max, e / S             IEEE single, round to nearest
// Every operation is an explicit _rn intrinsic so nvcc cannot contract a
// multiply-add into an FMA where numpy does not (and vice versa); the
// translation unit is built without --use_fast_math and with FTZ off.
#pragma once
#include <cstdint>

namespace esim {

// 2^q * y, correctly rounded (one rounding), for |q| within float range.
__device__ __forceinline__ float ldexp_exact(float y, int q) {
    if (q >= -126) {
        if (q > 127) return __int_as_float(0x7f800000);
        return __fmul_rn(y, __int_as_float((q + 127) << 23));
    }
    // y * 2^(q+64) is exact (normal range), then one rounding into the subnormals
    float t = __fmul_rn(y, __int_as_float((q + 64 + 127) << 23));
    return __fmul_rn(t, __int_as_float((-64 + 127) << 23));
}

__device__ __forceinline__ float np_expf(float x) {
    if (x >= 88.72283935546875f) return __int_as_float(0x7f800000);
    if (x <= -103.97208404541015625f) return 0.0f;
    const float log2e = 1.44269504088896341f;
    const float magic = 0x1.8p23f;
    float q = __fsub_rn(__fadd_rn(__fmul_rn(x, log2e), magic), magic);
    float r = __fmaf_rn(q, -6.93145752e-1f, x);
    r = __fmaf_rn(q, -1.42860677e-6f, r);
    r = __fmaf_rn(q, 0.0f, r);
    float num = __fmaf_rn(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
    num = __fmaf_rn(num, r, 5.114512081637298353406e-02f);
    num = __fmaf_rn(num, r, 2.473615434895520810817e-01f);
    num = __fmaf_rn(num, r, 7.257664613233124478488e-01f);
    num = __fmaf_rn(num, r, 9.999999999980870924916e-01f);
    float den = __fmaf_rn(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
    den = __fmaf_rn(den, r, 1.0f);
    return ldexp_exact(__fdiv_rn(num, den), (int)q);
}

// numpy pairwise sum of a[0..n) (n <= 128 block) computed by one warp:
// lanes 0..7 own accumulator r[lane] (strided sequential adds), a shuffle
// butterfly over xor 1,2,4 reproduces ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// exactly (IEEE addition is commutative), lane 0 adds the tail. Returns the
// same value in every lane. `a` is shared memory.
__device__ __forceinline__ float warp_pw_block(const float* a, int n, int lane) {
    const unsigned full = 0xffffffffu;
    if (n < 8) {
        float res = 0.0f;
        for (int i = 0; i < n; i++) res = __fadd_rn(res, a[i]);
        return res;
    }
    int lim = n - (n % 8);
    float r = 0.0f;
    if (lane < 8) {
        r = a[lane];
        for (int i = 8; i < lim; i += 8) r = __fadd_rn(r, a[i + lane]);
    }
    r = __fadd_rn(r, __shfl_xor_sync(full, r, 1));
    r = __fadd_rn(r, __shfl_xor_sync(full, r, 2));
    r = __fadd_rn(r, __shfl_xor_sync(full, r, 4));
    float res = __shfl_sync(full, r, 0);
    for (int i = lim; i < n; i++) res = __fadd_rn(res, a[i]);
    return res;
}

// numpy pairwise sum for n <= 256 (ESIM_MAX_E): blocks of <= 128 are
// summed directly; larger n split at n2 = n/2 - (n/2)%8 as numpy does. For
// n in 249..255 the upper half (129..135 elements) is itself over the block
// size and numpy splits it again; for n <= 256 the recursion never goes
// deeper than that (the lower half is always <= 128). No recursion on the
// device: the stack size stays statically known.
__device__ __forceinline__ int pw_split(int n) {
    int n2 = n / 2;
    return n2 - n2 % 8;
}

__device__ __forceinline__ float warp_pw_mid(const float* a, int n, int lane) {   // n <= 256, hi half <= 128
    if (n <= 128) return warp_pw_block(a, n, lane);
    const int n2 = pw_split(n);
    return __fadd_rn(warp_pw_block(a, n2, lane), warp_pw_block(a + n2, n - n2, lane));
}

__device__ __forceinline__ float warp_pw_sum(const float* a, int n, int lane) {
    if (n <= 128) return warp_pw_block(a, n, lane);
    const int n2 = pw_split(n);
    return __fadd_rn(warp_pw_block(a, n2, lane), warp_pw_mid(a + n2, n - n2, lane));
}

// The host interpreter's builtin sum() over floats (bltinmodule.c
// builtin_sum_impl float path): CPython >= 3.12 adds Neumaier compensation,
// earlier versions a plain left fold. Which one is a per-translation-unit
// device global set by esim_set_host_sum() (the Python wrapper passes
// sys.version_info at load), default 3.12+.
static __device__ int g_pysum_plain = 0;

struct PySum {
    double f, c;
    __device__ __forceinline__ void init() { f = 0.0; c = 0.0; }
    __device__ __forceinline__ void add(double x) {
        if (g_pysum_plain) { f = __dadd_rn(f, x); return; }
        double t = __dadd_rn(f, x);
        if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
        else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
        f = t;
    }
    __device__ __forceinline__ double value() const {
        return (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f;
    }
};

}  // namespace esim
