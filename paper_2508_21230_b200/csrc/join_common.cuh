// Pieces shared by the two join kernels: arguments, the reference distance
// combine, and the chunked pair writer.
#pragma once
#include "common.cuh"
#include "experiments.h"

namespace fasted {

struct JoinArgs {
    const float* norms;
    int64_t n_logical, n_pad, d_pad;
    int64_t row_begin, row_end, col_begin, col_end;
    float eps_sq;
    int count_only;
    int diag_flags;                    // diagnostic flags (libfasted_exp.so only; 0 here)
    int symmetric;                     // FASTED_JOIN_SYMMETRIC: upper tiles, mirrored records
    int low_output;                    // FASTED_JOIN_LOW_OUTPUT hint (kernel choice only)
    int sparse;                        // FASTED_JOIN_SPARSE hint (kernel choice only)
    uint4* out;                        // records {i, j, dist_sq bits, 0}
    unsigned long long capacity;       // record slots available in out
    unsigned long long* count;         // [0] exact pair total, [1] chunks taken
    float* gram_diag;                  // diagonal pre-pass output (tcgen05 kernel), else null
    unsigned long long* trace;         // FASTED_JOIN_DIAG_TRACE timeline (CTA 0), else null
    unsigned long long* pace;          // resident kernel: units issued by all CTAs (zeroed per launch)
};

// FASTED_JOIN_DIAG_TRACE layout (resident kernel, CTA 0, first TRACE_TILES
// accumulator tiles, SM clock64): [t][2] MMA warp {tempty passed, tfull
// committed}, then [t][w][8] per epilogue warp {tfull passed, TMEM loads
// landed, tempty arrived, tile done, slice vote done, rare chunk: hit masks
// built, rare chunk: records appended, 1 if a rare chunk ran}.
// Then, with hit warps, [h][e][4] per hit warp h < TRACE_HIT_WARPS and
// queue entry e < TRACE_HIT_ENTRIES {wait for the entry started, entry
// visible, entry done, kind | records << 8}.
constexpr int TRACE_TILES = 256;
constexpr int TRACE_EPI_WARPS = 16;
constexpr int TRACE_HIT_WARPS = 2;
constexpr int TRACE_HIT_ENTRIES = 512;
constexpr unsigned long long TRACE_HIT_BASE =
    (unsigned long long)TRACE_TILES * (2 + 8 * TRACE_EPI_WARPS);
constexpr unsigned long long TRACE_WORDS =
    TRACE_HIT_BASE + (unsigned long long)TRACE_HIT_WARPS * TRACE_HIT_ENTRIES * 4;

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

// Staged pair writer (the tcgen05 kernels).  Same chunk protocol as
// PairWriter (private 256-slot chunks, one atomic per chunk, unused tail
// slots zeroed), but a hit costs one 16-byte SHARED store: each warp stages
// records in two STAGE-record buffers in shared memory and ships a full
// buffer with one bulk async copy (cp.async.bulk shared -> global, TMA
// engine), double-buffered.  Per-record 16-byte global stores measured
// +36% join time at S ~ 4096 (5M x 384) against the count-only join.
template <int STAGE>
struct StagedWriter {
    static_assert(WRITER_CHUNK % STAGE == 0, "chunk must hold whole staging buffers");
    static constexpr uint32_t kStage = STAGE;
    static constexpr bool kDirect = false;
    unsigned long long base;    // first slot of the current chunk (~0: none open)
    uint32_t flushed;           // staging buffers shipped into the current chunk
    uint32_t fill;              // records in the current staging buffer
    uint32_t sb;                // current staging buffer (0/1)
    uint32_t sbuf;              // shared address of this warp's 2 x STAGE x 16 bytes
    unsigned long long total;   // pairs found by this warp
    uint64_t policy;            // L2 evict_first cache policy for the record stream
};

// Per-warp row stash of the resident kernel's epilogue (epi_chunk_res's
// transposed hit search: one lane's 32 accumulator words), placed right after
// the warp's two staging buffers.
constexpr int EPI_STASH_BYTES = 128;

template <int STAGE>
__device__ __forceinline__ void writer_init(StagedWriter<STAGE>& w, uint32_t sbuf) {
    w.base = ~0ull;
    w.flushed = 0;
    w.fill = 0;
    w.sb = 0;
    w.sbuf = sbuf;
    w.total = 0;
    // Records are written once and read back only by the sort: keep them from
    // evicting the join's operand panels from L2 (measured at S ~ 4096: with
    // default policy the join re-read 861 GB from HBM per 75K-row slice
    // against 40 GB count-only, L2 hit rate 61% vs 97%).
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(w.policy));
}

__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Warp collective: ship the current staging buffer (all STAGE slots) to the
// next STAGE slots of the warp's chunk (grabbing a chunk when needed).
template <int STAGE>
__device__ __forceinline__ void writer_flush(StagedWriter<STAGE>& w, const JoinArgs& a) {
    // the lanes' generic shared stores -> visible to the async (bulk copy) proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (w.base == ~0ull || w.flushed == WRITER_CHUNK / STAGE) {
        unsigned long long c = 0;
        if (lane_id() == 0) c = atomicAdd(a.count + 1, 1ull);
        w.base = __shfl_sync(0xffffffffu, c, 0) * WRITER_CHUNK;
        w.flushed = 0;
    }
    const unsigned long long dst = w.base + (unsigned long long)w.flushed * STAGE;
    w.flushed++;
    if (lane_id() == 0 && dst < a.capacity) {
        const unsigned long long room = a.capacity - dst;
        const uint32_t recs = room < (unsigned long long)STAGE ? (uint32_t)room : (uint32_t)STAGE;
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(a.out + dst)),
            "r"(w.sbuf + w.sb * STAGE * 16u), "r"(recs * 16u), "l"(w.policy)
            : "memory");
    }
    w.sb ^= 1u;
    w.fill = 0;
    // the buffer written next was shipped two flushes ago: wait until that
    // copy has READ it (the one just issued may stay in flight)
    if (lane_id() == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
}

// Warp collective.  `ballot` (warp-uniform) holds the lanes that append one
// record each; `mine` is this lane's bit.
template <int STAGE>
__device__ __forceinline__ void writer_append(StagedWriter<STAGE>& w, const JoinArgs& a,
                                              uint32_t ballot, bool mine, uint32_t i1,
                                              uint32_t j1, float d2) {
    const uint32_t n = __popc(ballot);
    w.total += n;
    if (a.count_only || n == 0) return;
    const uint32_t rank = __popc(ballot & lanemask_lt());
    const uint4 rec = make_uint4(i1, j1, __float_as_uint(d2), 0u);
    uint32_t done = 0;
    while (done < n) {   // warp-uniform: usually one pass
        const uint32_t room = STAGE - w.fill;
        const uint32_t take = n - done < room ? n - done : room;
        if (mine && rank >= done && rank < done + take)
            st_shared_v4(w.sbuf + (w.sb * STAGE + w.fill + (rank - done)) * 16u, rec);
        w.fill += take;
        done += take;
        if (w.fill == STAGE) writer_flush(w, a);
    }
}

// Warp collective: zero the rest of the open chunk (unused slots, i == 0),
// wait for every bulk copy to land, publish the total.
template <int STAGE>
__device__ __forceinline__ void writer_finish(StagedWriter<STAGE>& w, const JoinArgs& a) {
    if (!a.count_only) {
        const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
        if (w.fill > 0) {
            for (uint32_t s = w.fill + lane_id(); s < STAGE; s += 32)
                st_shared_v4(w.sbuf + (w.sb * STAGE + s) * 16u, zero);
            writer_flush(w, a);
        }
        while (w.base != ~0ull && w.flushed < WRITER_CHUNK / STAGE) {
            for (uint32_t s = lane_id(); s < STAGE; s += 32)
                st_shared_v4(w.sbuf + (w.sb * STAGE + s) * 16u, zero);
            writer_flush(w, a);
        }
        if (lane_id() == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    if (lane_id() == 0 && w.total) atomicAdd(a.count, w.total);
}

// Direct pair writer (the resident kernel's sparse-output form): PairWriter's
// chunk protocol, each record one 16-byte global store with an L2
// evict_first hint straight from the epilogue warp's registers -- no shared
// memory on the hit path.  The shared-memory staging and hand-off round trips
// wait behind the tensor core's operand reads from the same shared memory
// (profiles/round2/c3_session3_epilogue_analysis.txt); at ~1 pair per 10^4
// examined the uncoalesced stores cost nothing measurable in bandwidth.
struct DirectWriter {
    static constexpr bool kDirect = true;
    unsigned long long base;   // first slot of the current chunk
    uint32_t fill;             // slots used in it (WRITER_CHUNK = none open)
    unsigned long long total;  // pairs found by this warp
    uint64_t policy;           // L2 evict_first for the record stream
};

__device__ __forceinline__ void writer_init(DirectWriter& w) {
    w.base = 0;
    w.fill = WRITER_CHUNK;
    w.total = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(w.policy));
}

__device__ __forceinline__ void st_global_v4_hint(uint4* p, uint4 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;"
                 ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}

// Warp collective (same contract as the other writers).
__device__ __forceinline__ void writer_append(DirectWriter& w, const JoinArgs& a, uint32_t ballot,
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
        if (slot < a.capacity)
            st_global_v4_hint(a.out + slot, make_uint4(i1, j1, __float_as_uint(d2), 0u), w.policy);
    }
    if (n > room) {
        w.base = next;
        w.fill = n - room;
    } else {
        w.fill += n;
    }
}

__device__ __forceinline__ void writer_finish(DirectWriter& w, const JoinArgs& a) {
    if (!a.count_only) {
        for (uint32_t s = w.fill + lane_id(); s < WRITER_CHUNK; s += 32)
            if (w.base + s < a.capacity) a.out[w.base + s] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (lane_id() == 0 && w.total) atomicAdd(a.count, w.total);
}

int launch_join_exact(const __half* X, const JoinArgs& a, cudaStream_t s);
int launch_join_tc(const __half* X, const JoinArgs& a, cudaStream_t s);
const char* join_tc_kernel_name(int64_t d_pad, int64_t rows, int64_t cols, bool low_output,
                                bool sparse);

}  // namespace fasted
