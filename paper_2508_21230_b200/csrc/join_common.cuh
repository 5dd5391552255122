// Pieces shared by the two join kernels: arguments, the reference distance
// combine, and the chunked pair writer.
#pragma once
#include "common.cuh"

namespace fasted {

struct JoinArgs {
    const float* norms;
    int64_t n_logical, n_pad, d_pad;
    int64_t row_begin, row_end, col_begin, col_end;
    float eps_sq;
    int count_only;
    int diag_flags;                    // FASTED_JOIN_DIAG_* (experiments only)
    int symmetric;                     // FASTED_JOIN_SYMMETRIC: upper tiles, mirrored records
    uint4* out;                        // records {i, j, dist_sq bits, 0}
    unsigned long long capacity;       // record slots available in out
    unsigned long long* count;         // [0] exact pair total, [1] chunks taken
    float* gram_diag;                  // diagonal pre-pass output (tcgen05 kernel), else null
};

// ((-2 a) + s_i) + s_j in FP32 round-to-nearest, clamped at 0
// (mma.py:143-157).  -2a is exact, so the first step is one RN FMA.
__device__ __forceinline__ float combine_rn(float a, float si, float sj) {
    const float t = __fmaf_rn(-2.0f, a, si);
    const float d2 = __fadd_rn(t, sj);
    return fmaxf(d2, 0.0f);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Chunked pair writer.  Every warp appends into private runs of
// FASTED_RECORD_CHUNK record slots taken from a global chunk counter (one
// atomic per 256 records), so different SMs write different cache lines and
// no shared "next slot" counter sits on the critical path.  An append of up
// to 32 records (one per lane) is one coalesced 16-byte store per lane.
// The tail of a warp's last chunk is marked unused (i == 0) by
// writer_finish; the sort drops those slots.
constexpr uint32_t WRITER_CHUNK = FASTED_RECORD_CHUNK;

struct PairWriter {
    unsigned long long base;   // first slot of the current chunk
    uint32_t fill;             // slots used in it (WRITER_CHUNK = none open)
    unsigned long long total;  // pairs found by this warp
};

__device__ __forceinline__ void writer_init(PairWriter& w) {
    w.base = 0;
    w.fill = WRITER_CHUNK;
    w.total = 0;
}

// Warp collective.  `ballot` (warp-uniform) holds the lanes that append one
// record each; `mine` is this lane's bit.
__device__ __forceinline__ void writer_append(PairWriter& w, const JoinArgs& a, uint32_t ballot,
                                              bool mine, uint32_t i1, uint32_t j1, float d2) {
    const uint32_t n = __popc(ballot);
    w.total += n;
    if (a.count_only || n == 0) return;
    const uint32_t room = WRITER_CHUNK - w.fill;
    unsigned long long next = 0;
    if (n > room) {
        unsigned long long c = 0;
        if (lane_id() == 0) c = atomicAdd(a.count + 1, 1ull);
        next = __shfl_sync(0xffffffffu, c, 0) * WRITER_CHUNK;
    }
    if (mine) {
        const uint32_t r = __popc(ballot & lanemask_lt());
        const unsigned long long slot = r < room ? w.base + w.fill + r : next + (r - room);
        if (slot < a.capacity) a.out[slot] = make_uint4(i1, j1, __float_as_uint(d2), 0u);
    }
    if (n > room) {
        w.base = next;
        w.fill = n - room;
    } else {
        w.fill += n;
    }
}

// Warp collective: mark the open chunk's unused tail (i == 0), publish the total.
__device__ __forceinline__ void writer_finish(PairWriter& w, const JoinArgs& a) {
    if (!a.count_only) {
        for (uint32_t s = w.fill + lane_id(); s < WRITER_CHUNK; s += 32)
            if (w.base + s < a.capacity) a.out[w.base + s] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (lane_id() == 0 && w.total) atomicAdd(a.count, w.total);
}

int launch_join_exact(const __half* X, const JoinArgs& a, cudaStream_t s);
int launch_join_tc(const __half* X, const JoinArgs& a, cudaStream_t s);
const char* join_tc_kernel_name(int64_t d_pad);

}  // namespace fasted
