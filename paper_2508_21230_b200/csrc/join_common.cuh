// Pieces shared by the two join kernels: arguments, the reference distance
// combine, and warp-aggregated pair compaction.
#pragma once
#include "common.cuh"

namespace fasted {

struct JoinArgs {
    const float* norms;
    int64_t n_logical, n_pad, d_pad;
    int64_t row_begin, row_end, col_begin, col_end;
    float eps_sq;
    int count_only;
    uint32_t* out_i;
    uint32_t* out_j;
    float* out_d;
    unsigned long long capacity;
    unsigned long long* count;
};

// ((-2 a) + s_i) + s_j in FP32 round-to-nearest, clamped at 0
// (mma.py:143-157).  -2a is exact, so the first step is one RN FMA.
__device__ __forceinline__ float combine_rn(float a, float si, float sj) {
    const float t = __fmaf_rn(-2.0f, a, si);
    const float d2 = __fadd_rn(t, sj);
    return fmaxf(d2, 0.0f);
}

// Emit the (<= 8) qualifying pairs of one thread's row segment; the column
// of bit c is col0 + (c < 4 ? tx*4 + c : 64 + tx*4 + c - 4).  All 32 lanes
// of the warp must call this (warp-aggregated reservation).
__device__ __forceinline__ void emit_pairs8(const JoinArgs& a, uint32_t mask, int64_t i,
                                            int64_t col0, int tx, const float* dv) {
    if (!__any_sync(0xffffffffu, mask != 0)) return;
    const uint32_t cnt = __popc(mask);
    unsigned long long pos = warp_reserve(a.count, cnt);
    if (a.count_only) return;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        if (mask & (1u << c)) {
            if (pos < a.capacity) {
                const int64_t j = col0 + (c < 4 ? tx * 4 + c : 64 + tx * 4 + (c - 4));
                a.out_i[pos] = (uint32_t)(i + 1);
                a.out_j[pos] = (uint32_t)(j + 1);
                a.out_d[pos] = dv[c];
            }
            pos++;
        }
    }
}

int launch_join_exact(const __half* X, const JoinArgs& a, cudaStream_t s);
int launch_join_tc(const __half* X, const JoinArgs& a, cudaStream_t s);

}  // namespace fasted
