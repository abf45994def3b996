// digest.cuh -- the per-record word mix of the decision-log digest, shared by
// the replay kernel (records it emits) and the router's per-event summary
// (records whose content is fixed by the router output alone: RouteRec under
// standard routing with no drop/substitution, PredictionRec). Both sides must
// produce the identical 32-bit word; tests/golden digests pin it
// (records.digest_records is the host restatement).
//
// mix = sum_i w_i * K_i (mod 2^32) over the record's sixteen 32-bit words
// (t0 skipped for predictions) + sum_j (e_j + 1) * G * (j + 1) over a
// prediction's experts. The replay then folds it in with the record index:
// x = (mix ^ idx * C) * P, digest += x ^ (x >> 31).
#pragma once
#include <cstdint>

#include "../../include/specmd_b200.h"

namespace esim {

#define KM(i) (i == 0 ? 0x9E3779B1u : i == 1 ? 0x85EBCA77u : i == 2 ? 0xC2B2AE3Du : i == 3 ? 0x27D4EB2Fu : \
               i == 4 ? 0x165667B1u : i == 5 ? 0xD3A2646Bu : i == 6 ? 0xFD7046C5u : i == 7 ? 0xB55A4F09u : \
               i == 8 ? 0x68E31DA5u : i == 9 ? 0x2C1B3C6Du : i == 10 ? 0x297A2D39u : i == 11 ? 0x95E4A8F1u : \
               i == 12 ? 0x7FEB352Du : i == 13 ? 0x846CA68Bu : i == 14 ? 0x2545F491u : 0x9E6C63D1u)

constexpr uint32_t PE_MIX_G = 0x9E3779B1u;

__device__ __forceinline__ uint32_t rec_mix(int kind, int pass_id, int layer, int i0, int i1, int i2, int i3, int i4,
                                            int64_t t0, int64_t t1, int64_t t2, double x0) {
    const uint64_t x0b = (uint64_t)__double_as_longlong(x0);
    uint32_t mix = (uint32_t)kind * KM(0) + (uint32_t)pass_id * KM(1) + (uint32_t)layer * KM(2) +
                   (uint32_t)i0 * KM(3) + (uint32_t)i1 * KM(4) + (uint32_t)i2 * KM(5) + (uint32_t)i3 * KM(6) +
                   (uint32_t)i4 * KM(7) + (uint32_t)t1 * KM(10) + (uint32_t)((uint64_t)t1 >> 32) * KM(11) +
                   (uint32_t)t2 * KM(12) + (uint32_t)((uint64_t)t2 >> 32) * KM(13) + (uint32_t)x0b * KM(14) +
                   (uint32_t)(x0b >> 32) * KM(15);
    if (kind != ESIM_REC_PREDICTION) mix += (uint32_t)t0 * KM(8) + (uint32_t)((uint64_t)t0 >> 32) * KM(9);
    return mix;
}

// the expert-list term of a PredictionRec: position j (0-based) holds expert e
__device__ __forceinline__ uint32_t pe_mix_term(int j, int e) {
    return (uint32_t)(e + 1) * (PE_MIX_G * (uint32_t)(j + 1));
}

}  // namespace esim
