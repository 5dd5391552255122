// Kernel 2 (the product path): fused tcgen05 epsilon join for sm_100a.
//
// Per tile, everything stays on chip:
//   TMA (SWIZZLE_128B) -> smem ring -> tcgen05.mma kind::f16 (K=16)
//   accumulating a_ij = x_i . x_j in TMEM, then ONE extra tcgen05.mma
//   kind::tf32 step (K=8) that adds
//       sigma_i + rho_j = -s_i/2 + (-s_j/2 + eps^2/2)
//   from two tiny per-point "augment" rows (norms split into 3 exact tf32
//   parts, prepared per call by aug_prepare_kernel from the tensor core's
//   own Gram diagonal).  The accumulator then holds D_ij = (eps^2 - d2_ij)/2,
//   so the epilogue's common path is a sign test: d2 <= eps^2 <=> D >= 0.
//   Epilogue warps drain their whole TMEM slice with back-to-back
//   tcgen05.ld and one wait, release the accumulator to the MMA warp, then
//   AND-reduce the sign bits of the whole slice with one vote; only a chunk
//   holding a hit (or the diagonal) builds per-lane hit masks and writes
//   {i, j, d2 = eps^2 - 2D} records (StagedWriter: shared-memory staging,
//   bulk async stores, one atomic per 256 records per warp).
//
// Three kernels share that math and epilogue (tc_variant picks one):
//   join_tc_kernel<CG>   both operands streamed.  CG = 2: CTA pair
//                        (cta_group::2), a 256 x 256 tile per pair, each CTA
//                        stages its 128 rows of A and its 128-row half of B,
//                        the leader issues M=256 N=256 MMAs -- the form for
//                        large low-output joins at d_pad > 256.  CG = 1: one
//                        CTA, 128 x 256 tiles (the Gram pre-pass, A/B runs).
//   join_tc_mc_kernel    clusters of two single-CTA MMAs sharing B by TMA
//                        multicast (d_pad > 256 otherwise).
//   join_tc_res_kernel   CTA pair with the A panel resident in shared memory
//                        for a row tile x column segment (d_pad <= 512).
//
// The distance matrix never reaches HBM.  Replaces the reference's tile
// sweep (tiling.py:307-344): compute_block_tile (tiling.py:199-285),
// accumulate_panel (_kernel.py:57-76) and combine_distance (mma.py:143-157).
// Arithmetic differs from the reference in how a_ij and the norm terms are
// summed (tensor core FP32 accumulation instead of a sequential
// round-toward-zero chain); pair sets agree outside the 1e-3 relative band
// around eps^2 (tests/test_gpu.py).  Self pairs (i == j) are forced to
// distance 0, which is exactly what the reference produces.
//
// Warp roles (2 + NEPI warps; the product forms use NEPI = 16 -- 96
// registers per thread, a warp's 32 x 64 accumulator slice; NEPI = 8 gives
// 168 registers and 32 x 128 slices):
//   warp 0      : TMEM allocator / deallocator, then TMA producer
//   warp 1      : MMA issuer (leader CTA only for a CTA pair)
//   warps 2..   : epilogue; warp w reads TMEM lanes 32*(w%4).. and column
//                 group (w-2)/4 of the 256-column accumulator.
// The producer and MMA loops run on the whole warp with elected issue.
// TMEM: 2 accumulators x 256 columns (double buffered across tiles).
// Tiles walk a grouped raster: GROUP row tiles sweep every column tile
// together, so each B panel is read from HBM once per group and the group's
// A panels stay L2 resident.
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "join_common.cuh"

namespace fasted {
namespace tc {

constexpr int BM = 128;   // rows per CTA (TMEM lanes)
constexpr int BN = 256;   // columns per tile (TMEM columns per accumulator)
constexpr int BK = 64;    // one 128-byte swizzle atom of FP16
constexpr int UK = 16;    // K of one kind::f16 tcgen05.mma
constexpr int AUG_K = 8;  // K of one kind::tf32 tcgen05.mma: one 32-byte row
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_HALF_BYTES = 128 * BK * 2;
constexpr int AUG_ROW_BYTES = AUG_K * 4;
constexpr int NUM_EPI_WARPS = 8;
constexpr int FIRST_EPI_WARP = 2;
constexpr int THREADS = (FIRST_EPI_WARP + NUM_EPI_WARPS) * 32;
constexpr int TMEM_COLS = 2 * BN;
constexpr int BAR_BYTES = 256;
// Pair-record staging (StagedWriter): per epilogue warp 2 buffers of STAGE
// records of 16 bytes.
constexpr int WSTAGE = 64;
constexpr int WSTAGE_BYTES = NUM_EPI_WARPS * 2 * WSTAGE * 16;   // 16 KB

template <int CG>
struct Cfg {
    static constexpr int B_BYTES = (BN / CG) * BK * 2;   // this CTA's share of B
    static constexpr int STAGES = CG == 2 ? 6 : 4;
    static constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + BAR_BYTES + WSTAGE_BYTES + 1024;
    static constexpr int TILE_M = BM * CG;                // rows per tile
    // Instruction descriptors: D=F32 (bits 4-5 = 1); A/B format at bits
    // 7-9 / 10-12 (F16 = 0, TF32 = 2); both K-major; N>>3 at 17-22; M>>4 at
    // 24-28 (M = 256 for the CTA pair).
    static constexpr uint32_t IDESC_F16 =
        (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);
    static constexpr uint32_t IDESC_TF32 = IDESC_F16 | (2u << 7) | (2u << 10);
};

// Which pipeline warps wait for their mbarriers by a test_wait spin instead
// of a try_wait suspend: 1 the MMA warp (accumulator release, operand
// stages), 2 the TMA producer (stage release), 4 the hit warps.  A suspended
// try_wait can resume well after the phase completes; alternating launches
// (profiles/round2/mbarrier_spin_ab.txt): C4 1391 vs 1573 ms, C5 shard
// S~256 1561 vs 2101 ms, S~16 1542 vs 1760 ms with 3; C3 and C2 unchanged;
// the hit warps (4) do not gain.
constexpr int MMA_SPIN_DEFAULT = 3;

struct Sched {
    int row_tiles;
    int col_tiles;
    int group;
    int nkb;
    int64_t total;
    int diag;   // 1: Gram-diagonal pre-pass (tiles (r, r), no augment step)
    int mma_spin = MMA_SPIN_DEFAULT;   // MMA_SPIN_DEFAULT bits (FASTED_MMA_SPIN in experiments)
    int pace_w = 0;     // streaming pacing: blocks of PACE_TILES layers a CTA may run ahead
};

// Streaming-kernel pacing (the resident kernel's, per block of PACE_TILES tile
// layers: layer k = every pair's k-th tile, a contiguous run of the raster).
constexpr int PACE_TILES = 64;
__device__ __forceinline__ unsigned long long pace_need_stream(int64_t total, int64_t step,
                                                               int64_t b, int cg) {
    const int64_t L = total / step, rem = total % step;   // pairs p < rem have L + 1 tiles
    const int64_t jfull = L / PACE_TILES;
    const int64_t full = b + 1 < jfull ? b + 1 : jfull;
    const bool last = b >= jfull && (jfull + 1) * PACE_TILES == L + 1;
    return (unsigned long long)cg * (unsigned long long)(full * step + (last ? rem : 0));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// try_wait with a suspend-time hint (ns): a waiting warp sleeps in hardware
// until the phase completes or the hint expires, instead of re-polling.
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ uint64_t global_timer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Pacing wait: until `need` units were issued by all CTAs, at most
// PACE_GIVE_UP_NS.  Pacing is a locality aid, never a dependency: if the other
// CTAs are not resident (another kernel holds SMs -- e.g. two joins launched
// concurrently on one device) the wait would never end, so the CTA stops
// pacing for the rest of the launch instead (normal waits are microseconds).
constexpr uint64_t PACE_GIVE_UP_NS = 5000000ull;   // 5 ms
__device__ __forceinline__ void pace_wait(const unsigned long long* pace,
                                          unsigned long long need, bool& paced) {
    const uint64_t t0 = global_timer();
    while (ld_acquire_gpu_u64(pace) < need) {
        __nanosleep(64);
        if (global_timer() - t0 > PACE_GIVE_UP_NS) {
            paced = false;
            return;
        }
    }
}

// Spin on an mbarrier phase; traps after 20 s so a protocol bug aborts the
// launch (cudaErrorLaunchFailure) instead of wedging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = global_timer();
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins == 16u) {
            spins = 0;
            if (global_timer() - t0 > 20000000000ull) __trap();
        }
    }
}

// Pure-spin variant (no suspend hint): FASTED_JOIN_DIAG_SPIN A/B experiments.
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait2(uint32_t bar, uint32_t parity, bool spin) {
    if (!spin) {
        mbar_wait(bar, parity);
        return;
    }
    if (mbar_test_wait(bar, parity)) return;
    const uint64_t t0 = global_timer();
    uint32_t spins = 0;
    while (!mbar_test_wait(bar, parity)) {
        if (++spins == 256u) {
            spins = 0;
            if (global_timer() - t0 > 20000000000ull) __trap();
        }
    }
}

// Non-blocking phase test (mbarrier.test_wait: never suspends).
__device__ __forceinline__ bool mbar_test_only(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

// Pure spin on mbarrier.test_wait (never suspends): the MMA and TMA-producer
// warps' waits (MMA_SPIN_DEFAULT) -- a suspended try_wait may resume well
// after the phase completes.
__device__ __forceinline__ void mbar_spin(uint32_t bar, uint32_t parity) {
    if (mbar_test_only(bar, parity)) return;
    const uint64_t t0 = global_timer();
    uint32_t polls = 0;
    while (!mbar_test_only(bar, parity)) {
        if (++polls == 1024u) {
            polls = 0;
            if (global_timer() - t0 > 20000000000ull) __trap();
        }
    }
}

// The epilogue's accumulator wait.  sleep_ns == 0: mbar_wait2 (try_wait
// with a suspend hint).  Otherwise a failed test sleeps sleep_ns in
// __nanosleep: a try_wait-suspended warp is woken by other barrier traffic
// every ~100 cycles and re-polls (ncu at 1M x 128: ~9 polls, ~70 issued
// instructions per warp per tile), taking issue slots from the warps on
// its SM sub-partition that are still working on the previous tile.
__device__ __forceinline__ void epi_wait(uint32_t bar, uint32_t parity, bool spin,
                                         uint32_t sleep_ns) {
    if (sleep_ns == 0u) {
        mbar_wait2(bar, parity, spin);
        return;
    }
    if (sleep_ns == 1u) {   // FASTED_EPI_SLEEP_NS=1: pure test_wait spin
        mbar_spin(bar, parity);
        return;
    }
    if (mbar_test_only(bar, parity)) return;
    const uint64_t t0 = global_timer();
    uint32_t polls = 0;
    while (!mbar_test_only(bar, parity)) {
        __nanosleep(sleep_ns);
        if (++polls == 64u) {
            polls = 0;
            if (global_timer() - t0 > 20000000000ull) __trap();
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Relaxed local arrive for the accumulator release: the TMEM reads are
// ordered by tcgen05.fence::before_thread_sync; a (default) release arrive
// would also order this thread's earlier pair-record stores, i.e. wait for
// them, on the MMA's critical path.
__device__ __forceinline__ void mbar_arrive_relaxed(uint32_t bar) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Arrive on the barrier at the same offset in CTA `rank` of the cluster.
// Relaxed: the only ordering needed (TMEM reads before the MMA reuses the
// accumulator) comes from tcgen05.fence::before_thread_sync; a release
// arrive would also wait for this thread's outstanding global stores
// (measured: an ERRBAR per tile on the critical path).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                 : "memory");
}

// Relaxed arrive on a barrier address already mapped into the cluster
// window (mapa hoisted out of the per-tile loop).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t remote) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                 : "memory");
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(addr), "r"(rank));
    return remote;
}

// Release-semantics remote arrive: orders this thread's earlier TMEM stores
// (after tcgen05.wait::st) and shared-memory writes before the arrive.
__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

template <int CG>
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
    if constexpr (CG == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
            : "memory");
    } else {
        // both CTAs signal the leader's barrier: clear the peer bit
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
            "bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
            : "memory");
    }
}

// CTA-pair TMA load with an L2 cache policy (FASTED_A_EVICT_LAST experiments).
__device__ __forceinline__ void tma_load_2d_pair_hint(uint32_t dst, const CUtensorMap* map,
                                                      uint32_t bar, int c0, int c1, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
        "bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// One lane of a converged warp (the same lane every call).  The producer and
// MMA loops run on the whole warp so their addresses and descriptors stay in
// uniform registers; only the issue itself is elected.  (Looping on lane 0
// alone made the compiler rebuild every descriptor with ELECT + R2UR per MMA:
// ~40 dependent instructions per 512-cycle stage, measured 82% tensor-pipe
// activity at 1M x 960 with the MMA warp never waiting on data.)
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(p));
    return p != 0;
}

// Shared-memory matrix descriptors (K-major, swizzled): start address >> 4,
// LBO = 1 (unused for swizzled K-major), SBO = bytes between 8-row groups,
// version 1 (sm_100), layout type (SWIZZLE_128B = 2, SWIZZLE_32B = 6).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t sbo_bytes,
                                              uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) |
           ((uint64_t)(sbo_bytes >> 4) << 32) | ((uint64_t)1u << 46) |
           ((uint64_t)layout << 61);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) { return smem_desc(saddr, 1024, 2); }
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) { return smem_desc(saddr, 256, 6); }

template <int CG>
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t accumulate,
                                        uint32_t idesc = Cfg<CG>::IDESC_F16) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
            : "memory");
}

template <int CG>
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc = Cfg<CG>::IDESC_TF32) {
    if constexpr (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1u)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1u)
            : "memory");
}

// Completion of all prior MMAs -> arrive on `bar` (in both CTAs for CG=2).
template <int CG>
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    if constexpr (CG == 1)
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                bar)
            : "memory");
    else
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster."
            "b64 [%0], %1;" ::"r"(bar),
            "h"((uint16_t)0x3)
            : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

// 32 lanes x 64 columns in one tcgen05.ld (32x32b.x64): ra = columns 0..31,
// rb = 32..63 (FASTED_JOIN_DIAG_LDX64 A/B: half the load instructions).
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&ra)[32], uint32_t (&rb)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
        : "=r"(ra[0]), "=r"(ra[1]), "=r"(ra[2]), "=r"(ra[3]), "=r"(ra[4]), "=r"(ra[5]), "=r"(ra[6]), "=r"(ra[7]), "=r"(ra[8]), "=r"(ra[9]), "=r"(ra[10]), "=r"(ra[11]), "=r"(ra[12]), "=r"(ra[13]), "=r"(ra[14]), "=r"(ra[15]), "=r"(ra[16]), "=r"(ra[17]), "=r"(ra[18]), "=r"(ra[19]), "=r"(ra[20]), "=r"(ra[21]), "=r"(ra[22]), "=r"(ra[23]), "=r"(ra[24]), "=r"(ra[25]), "=r"(ra[26]), "=r"(ra[27]), "=r"(ra[28]), "=r"(ra[29]), "=r"(ra[30]), "=r"(ra[31]), "=r"(rb[0]), "=r"(rb[1]), "=r"(rb[2]), "=r"(rb[3]), "=r"(rb[4]), "=r"(rb[5]), "=r"(rb[6]), "=r"(rb[7]), "=r"(rb[8]), "=r"(rb[9]), "=r"(rb[10]), "=r"(rb[11]), "=r"(rb[12]), "=r"(rb[13]), "=r"(rb[14]), "=r"(rb[15]), "=r"(rb[16]), "=r"(rb[17]), "=r"(rb[18]), "=r"(rb[19]), "=r"(rb[20]), "=r"(rb[21]), "=r"(rb[22]), "=r"(rb[23]), "=r"(rb[24]), "=r"(rb[25]), "=r"(rb[26]), "=r"(rb[27]), "=r"(rb[28]), "=r"(rb[29]), "=r"(rb[30]), "=r"(rb[31])
        : "r"(taddr));
}

// tcgen05.wait::ld with the loaded registers threaded through, so no use of
// them can be scheduled before the wait.
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                   "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                   "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]),
                   "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]),
                   "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

__device__ __forceinline__ void tile_coords(const Sched& s, int64_t t, int& rt, int& ct) {
    const int64_t per_group = (int64_t)s.group * s.col_tiles;
    if (s.total <= 0xffffffffLL && per_group <= 0xffffffffLL) {
        // 32-bit divisions (every grid up to 2^32 tiles; 64-bit division is
        // a ~70-instruction software routine on the per-tile path)
        const uint32_t pg = (uint32_t)per_group, tt = (uint32_t)t;
        const uint32_t g = tt / pg;
        const uint32_t r = tt - g * pg;
        const uint32_t left = (uint32_t)s.row_tiles - g * (uint32_t)s.group;
        const uint32_t rows_in = left < (uint32_t)s.group ? left : (uint32_t)s.group;
        const uint32_t c = r / rows_in;
        ct = (int)c;
        rt = (int)(g * (uint32_t)s.group + (r - c * rows_in));
        return;
    }
    const int64_t g = t / per_group;
    const int64_t r = t - g * per_group;
    const int64_t left = (int64_t)s.row_tiles - g * s.group;
    const int rows_in = (int)(left < s.group ? left : s.group);
    ct = (int)(r / rows_in);
    rt = (int)(g * s.group + r % rows_in);
}

// FASTED_JOIN_SYMMETRIC: a tile wholly below the diagonal (every column index
// smaller than every row index) is skipped alike by the producer, the MMA
// warp and the epilogue; its pairs arrive as the mirrored records of the
// tile across the diagonal.  (Loops that count processed tiles undo their
// increment on a skip.)
__device__ __forceinline__ bool sym_skip(const JoinArgs& a, int64_t row0, int64_t col0,
                                         int tile_cols) {
    return a.symmetric && col0 + tile_cols - 1 < row0;
}

// r[e] for a warp-uniform runtime e without local memory: a 5-level
// select tree (31 SEL), so the rare path never spills the chunk.
__device__ __forceinline__ uint32_t pick32(const uint32_t (&r)[32], uint32_t e) {
    uint32_t t[16];
#pragma unroll
    for (int k = 0; k < 16; k++) t[k] = (e & 16u) ? r[k + 16] : r[k];
#pragma unroll
    for (int k = 0; k < 8; k++) t[k] = (e & 8u) ? t[k + 8] : t[k];
#pragma unroll
    for (int k = 0; k < 4; k++) t[k] = (e & 4u) ? t[k + 4] : t[k];
#pragma unroll
    for (int k = 0; k < 2; k++) t[k] = (e & 2u) ? t[k + 2] : t[k];
    return (e & 1u) ? t[1] : t[0];
}

// SM clock read ordered after `dep` is available (FASTED_JOIN_DIAG_TRACE:
// makes the stamp wait for the TMEM loads that produce it).
__device__ __forceinline__ unsigned long long clock_after(uint32_t dep) {
    unsigned long long t;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0x7fc00001;\n\t"
                 "@p mov.u64 %0, %%clock64;\n\t@!p mov.u64 %0, 0;\n\t}"
                 : "=l"(t)
                 : "r"(dep)
                 : "memory");
    return t;
}

// AND of 32 words as a balanced tree: the sign bit of the result is clear
// iff some word's sign bit is clear (some D >= 0, i.e. a hit).
__device__ __forceinline__ uint32_t and_tree32(const uint32_t (&r)[32]) {
    uint32_t t[16];
#pragma unroll
    for (int k = 0; k < 16; k++) t[k] = r[2 * k] & r[2 * k + 1];
#pragma unroll
    for (int k = 0; k < 8; k++) t[k] = t[2 * k] & t[2 * k + 1];
#pragma unroll
    for (int k = 0; k < 4; k++) t[k] = t[2 * k] & t[2 * k + 1];
    return (t[0] & t[1]) & (t[2] & t[3]);
}

// Bit e set iff r[e] >= 0 (sign bit clear): one funnel shift per word
// (SHF.L.W shifts the sign bit in), 32 instructions instead of ~80 for
// shift/mask/or per word.  Measured on the 5M x 384 shard at S ~ 4096, where
// most chunks take this path: 2305 vs 2781 ms per join (alternating launches).
__device__ __forceinline__ uint32_t hit_mask32(const uint32_t (&r)[32]) {
    uint32_t neg = 0;
#pragma unroll
    for (int e = 31; e >= 0; e--) neg = __funnelshift_l(r[e], neg, 1);   // (neg << 1) | sign(r[e])
    return ~neg;
}

// Epilogue of one 32-column chunk (columns jb.., row i = this lane).
// r[e] = D_{i, jb+e} = (eps^2 - d2) / 2 as FP32 bits.
template <typename W>
__device__ __forceinline__ void epi_chunk(const JoinArgs& a, W& wr, const uint32_t (&r)[32],
                                          int64_t jb, int64_t i, int64_t iw, bool row_ok) {
    // common path: is any D >= 0 (sign bit clear)?  A balanced AND tree
    // (depth ~5, not a 16-deep chain).
    const uint32_t acc = and_tree32(r);
    const bool diag = (jb < iw + 32) && (iw < jb + 32);   // warp-uniform
    if (!__any_sync(0xffffffffu, (int)acc >= 0) && !diag) return;
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOSLOW) return;
    // rare path.  Self pairs first: distance exactly 0 (the reference's
    // a_ii and s_i are the same chain), one append for the whole warp.
    if (diag) {
        const bool self = (i >= jb) && (i < jb + 32) && row_ok;
        const uint32_t b = __ballot_sync(0xffffffffu, self);
        if (b) writer_append(wr, a, b, self, (uint32_t)(i + 1), (uint32_t)(i + 1), 0.0f);
    }
    {
        // Per lane: build the hit mask (sign bits clear), drop the self
        // column and columns past n_logical; the warp appends one record per
        // hitting lane per round -- usually one round, hits being sparse.
        // (A column-scan form -- 32 REDUX.AND per chunk -- measured no faster
        // at 1M x 128 and doubled the rare-path code; it was removed.)
        uint32_t lm = hit_mask32(r);
        const int64_t valid = a.n_logical - jb;
        if (valid < 32) lm &= valid <= 0 ? 0u : ((1u << (uint32_t)valid) - 1u);
        if (i >= jb && i < jb + 32) lm &= ~(1u << (uint32_t)(i - jb));
        if (a.symmetric) {
            // upper triangle only (j > i); the mirrored record covers (j, i)
            const int64_t off = i - jb;   // columns jb .. i are not above the diagonal
            if (off >= 31) lm = 0u;
            else if (off >= 0) lm &= ~((2u << (uint32_t)off) - 1u);
        }
        if (!row_ok) lm = 0u;
        while (true) {
            const bool mine = lm != 0u;
            const uint32_t b = __ballot_sync(0xffffffffu, mine);
            if (b == 0u) break;
            const uint32_t e = mine ? (uint32_t)(__ffs(lm) - 1) : 0u;
            lm &= lm - 1u;
            const uint32_t v = pick32(r, e);
            const float d2 = fmaxf(__fmaf_rn(-2.0f, __uint_as_float(v), a.eps_sq), 0.0f);
            writer_append(wr, a, b, mine, (uint32_t)(i + 1), (uint32_t)(jb + e + 1), d2);
            if (a.symmetric)
                writer_append(wr, a, b, mine, (uint32_t)(jb + e + 1), (uint32_t)(i + 1), d2);
        }
    }
}

// The resident kernel's chunk epilogue: epi_chunk with a hybrid hit search.
// Hit search, transposed: a lane whose row has a candidate (some D >= 0)
// publishes its 32 words to the warp's shared-memory stash and every lane e
// tests column e of that row, so one ballot yields the row's hits and each
// hitting lane holds its own value -- no per-lane 32-bit hit mask, no
// select tree.  Rows with a candidate are rare (~2 per 32 x 64 slice at
// S ~ 64), and this path's dependent chain is a few tens of instructions
// against ~200 for the per-lane mask form it replaced (measured with
// FASTED_JOIN_DIAG_TRACE at 1M x 128: a warp with a hit came back to the next
// tile ~2900 cycles late, stalling the MMA warp on the accumulator).
// The stash is the 128 bytes after the warp's two staging buffers.  (The
// streaming and multicast kernels keep epi_chunk: at d > 256 the hybrid
// measured 6% slower at 5M x 384, S ~ 4096, and at 60K x 512.)
template <typename W>
__device__ __forceinline__ void epi_chunk_res(const JoinArgs& a, W& wr, const uint32_t (&r)[32],
                                              int64_t jb, int64_t i, int64_t iw, bool row_ok,
                                              unsigned long long* tr = nullptr) {
    uint32_t stash = 0u;
    if constexpr (!W::kDirect) stash = wr.sbuf + 2u * W::kStage * 16u;
    // common path: is any D >= 0 (sign bit clear)?  A balanced AND tree.
    const uint32_t acc = and_tree32(r);
    const bool diag = (jb < iw + 32) && (iw < jb + 32);   // warp-uniform
    const uint32_t rows = __ballot_sync(0xffffffffu, (int)acc >= 0 && row_ok);
    if (rows == 0u && !diag) return;
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOSLOW) return;
    const uint32_t lane = threadIdx.x & 31u;
    // rare path.  Self pairs first: distance exactly 0 (the reference's
    // a_ii and s_i are the same chain), one append for the whole warp.
    if (diag) {
        const bool self = (i >= jb) && (i < jb + 32) && row_ok;
        const uint32_t b = __ballot_sync(0xffffffffu, self);
        if (b) writer_append(wr, a, b, self, (uint32_t)(i + 1), (uint32_t)(i + 1), 0.0f);
    }
    if (tr && lane == 0) tr[5] = clock64();
    // One candidate row: the transposed search.  Two or more: per-lane hit
    // masks, all rows at once (serialising rows measured 20% slower at
    // 60K x 512, where a 32 x 32 chunk holds ~1 pair; A/B flags force either).
    const bool multi = (rows & (rows - 1u)) != 0u;
    if (W::kDirect || (((FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_RARE_LM) || multi) &&
                       !(FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_RARE_ROWS))) {
        // per-lane hit masks: all candidate rows at once
        uint32_t lm = hit_mask32(r);
        const int64_t valid = a.n_logical - jb;
        if (valid < 32) lm &= valid <= 0 ? 0u : ((1u << (uint32_t)valid) - 1u);
        if (i >= jb && i < jb + 32) lm &= ~(1u << (uint32_t)(i - jb));
        if (a.symmetric) {
            const int64_t off = i - jb;
            if (off >= 31) lm = 0u;
            else if (off >= 0) lm &= ~((2u << (uint32_t)off) - 1u);
        }
        if (!row_ok) lm = 0u;
        while (true) {
            const bool mine = lm != 0u;
            const uint32_t b = __ballot_sync(0xffffffffu, mine);
            if (b == 0u) break;
            const uint32_t e = mine ? (uint32_t)(__ffs(lm) - 1) : 0u;
            lm &= lm - 1u;
            const uint32_t v = pick32(r, e);
            const float d2 = fmaxf(__fmaf_rn(-2.0f, __uint_as_float(v), a.eps_sq), 0.0f);
            writer_append(wr, a, b, mine, (uint32_t)(i + 1), (uint32_t)(jb + e + 1), d2);
            if (a.symmetric)
                writer_append(wr, a, b, mine, (uint32_t)(jb + e + 1), (uint32_t)(i + 1), d2);
        }
        if (tr && lane == 0) tr[6] = clock64();
        return;
    }
    const int64_t j = jb + lane;
    const bool col_ok = j < a.n_logical;
    uint32_t rest = rows;
    while (rest != 0u) {
        const uint32_t src = (uint32_t)(__ffs(rest) - 1);
        rest &= rest - 1u;
        if (lane == src) {
#pragma unroll
            for (int k = 0; k < 8; k++)
                st_shared_v4(stash + 16u * k,
                             make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]));
        }
        __syncwarp();
        const uint32_t v = ld_shared_u32(stash + 4u * lane);
        __syncwarp();   // the stash is rewritten for the next row
        const int64_t is = iw + src;
        // drop the self column and columns past n_logical; symmetric: keep
        // the upper triangle only (j > i), the mirrored record covers (j, i)
        const bool hit = (int)v >= 0 && col_ok && j != is && (!a.symmetric || j > is);
        const uint32_t b = __ballot_sync(0xffffffffu, hit);
        if (b == 0u) continue;
        const float d2 = fmaxf(__fmaf_rn(-2.0f, __uint_as_float(v), a.eps_sq), 0.0f);
        writer_append(wr, a, b, hit, (uint32_t)(is + 1), (uint32_t)(j + 1), d2);
        if (a.symmetric) writer_append(wr, a, b, hit, (uint32_t)(j + 1), (uint32_t)(is + 1), d2);
    }
    if (tr && lane == 0) tr[6] = clock64();
}

// One epilogue warp's share of one finished accumulator of TBN columns:
// warp (q, h) owns TMEM lanes 32q.. (rows row0 + 32q + lane) and accumulator
// columns h*TBN/NSPLIT .. (h+1)*TBN/NSPLIT - 1 of buffer `buf`.  Drains its slice with
// back-to-back tcgen05.ld and ONE wait (a tcgen05.ld queues behind the MMAs
// already issued for the next tile, so waiting per chunk costs that queue
// drain each time), hands the accumulator back to the MMA warp before any
// math (the epilogue overlaps the next tiles' MMAs), then tests the signs.
template <int CG, int TBN, int NSPLIT = 2, typename W>
__device__ __forceinline__ void epilogue_tile(const JoinArgs& a, W& wr,
                                              uint32_t tmem_base, uint32_t tempty, int64_t row0,
                                              int64_t col0, int buf, uint32_t aph, int q, int h,
                                              int lane, bool leader, uint32_t tfull) {
    constexpr int HALF = TBN / NSPLIT;   // columns per warp
    constexpr int NCH = HALF / 32;       // 32-column chunks per warp (1, 2 or 4)
    static_assert(NCH == 1 || NCH == 2 || NCH == 4, "a warp covers 32, 64 or 128 columns");
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int64_t iw = row0 + q * 32;
    const int64_t i = iw + lane;
    const bool row_ok = i < a.n_logical && i < a.row_end;
    // chunks of 32 columns inside [col0 + HALF h, col_end); none if this
    // CTA's rows lie past the range end
    const int64_t left = a.col_end - (col0 + h * HALF);
    int nchunks = left <= 0 ? 0 : (left >= HALF ? NCH : (int)(left / 32));
    if (row0 >= a.row_end || (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOEPI)) nchunks = 0;
    const uint32_t tcol = tmem_base + lane_base + (uint32_t)(buf * TBN + h * HALF);
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_EPISPIN) mbar_spin(tfull, aph);
    else mbar_wait2(tfull, aph, (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0);
    tc_fence_after();
    uint32_t r0[32], r1[32], r2[32], r3[32];
    if (NCH > 1 && (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_LDX64) && nchunks == NCH) {
        tmem_ld64(tcol, r0, r1);
        if (NCH > 2) tmem_ld64(tcol + 64u, r2, r3);
    } else {
        if (nchunks > 0) tmem_ld32(tcol, r0);
        if (NCH > 1 && nchunks > 1) tmem_ld32(tcol + 32u, r1);
        if (NCH > 2 && nchunks > 2) tmem_ld32(tcol + 64u, r2);
        if (NCH > 2 && nchunks > 3) tmem_ld32(tcol + 96u, r3);
    }
    if (nchunks > 0) {
        tmem_ld_wait(r0);
        if (NCH > 1) tmem_ld_wait(r1);
        if (NCH > 2) {
            tmem_ld_wait(r2);
            tmem_ld_wait(r3);
        }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
        if (CG == 1 || leader) mbar_arrive_relaxed(tempty);
        else mbar_arrive_remote(tempty, 0);
    }
    const int64_t jb = col0 + h * HALF;
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_LOADONLY) return;
    // Whole-slice sign test first: one vote per tile in the common case (no
    // hit in the warp's 32 x HALF slice, no diagonal), instead of a vote and
    // a dependent AND chain per 32-column chunk (measured at 1M x 128: the
    // per-chunk form cost 50 ms of a 231 ms join).
    if (nchunks == NCH && !((jb < iw + 32) && (iw < jb + HALF))) {
        uint32_t all = and_tree32(r0);
        if (NCH > 1) all &= and_tree32(r1);
        if (NCH > 2) all &= and_tree32(r2) & and_tree32(r3);
        if (!__any_sync(0xffffffffu, (int)all >= 0)) return;
    }
    if (nchunks > 0) epi_chunk(a, wr, r0, jb, i, iw, row_ok);
    if (NCH > 1 && nchunks > 1) epi_chunk(a, wr, r1, jb + 32, i, iw, row_ok);
    if (NCH > 2 && nchunks > 2) epi_chunk(a, wr, r2, jb + 64, i, iw, row_ok);
    if (NCH > 2 && nchunks > 3) epi_chunk(a, wr, r3, jb + 96, i, iw, row_ok);
}

// The resident kernel's per-tile epilogue, lean form.  Everything that is
// fixed for a work unit (row validity, which tiles are full, which one holds
// the diagonal, the accumulator-release address) is computed once per unit
// by the caller, so the common tile -- full slice, off the diagonal, no hit --
// is: wait tfull, two TMEM loads, release the accumulator, a 64-word AND
// tree, one vote.  Measured with FASTED_JOIN_DIAG_TRACE at 1M x 128 (one
// row slice): the general epilogue_tile spent ~200 instructions per
// warp-tile, 16 warps x 200 issue slots against a ~1150-cycle tile, and the
// warps that found a hit (15% of warp-tiles) then took ~2900 cycles to get
// back to the next tile, stalling the MMA warp on the accumulator.
template <int CG, int TBN, int NSPLIT, bool TRACE, typename W>
__device__ __forceinline__ void res_epi_tile(const JoinArgs& a, W& wr, uint32_t tcol,
                                             uint32_t tfull, uint32_t aph, uint32_t tempty,
                                             bool local_release, bool spin, uint32_t sleep_ns,
                                             int dflags, int nchunks, bool fast, int64_t jb,
                                             int64_t i, int64_t iw, bool row_ok, int lane,
                                             unsigned long long* tr) {
    constexpr int HALF = TBN / NSPLIT;
    constexpr int NCH = HALF / 32;
    static_assert(NCH == 1 || NCH == 2 || NCH == 4, "a warp covers 32, 64 or 128 columns");
    if (dflags & FASTED_JOIN_DIAG_EPISPIN) mbar_spin(tfull, aph);
    else epi_wait(tfull, aph, spin, sleep_ns);
    tc_fence_after();
    if (TRACE && tr && lane == 0) tr[0] = clock64();
    uint32_t r0[32], r1[32], r2[32], r3[32];
    if (nchunks > 0) tmem_ld32(tcol, r0);
    if (NCH > 1 && nchunks > 1) tmem_ld32(tcol + 32u, r1);
    if (NCH > 2 && nchunks > 2) tmem_ld32(tcol + 64u, r2);
    if (NCH > 2 && nchunks > 3) tmem_ld32(tcol + 96u, r3);
    if (nchunks > 0) {
        tmem_ld_wait(r0);
        if (NCH > 1) tmem_ld_wait(r1);
        if (NCH > 2) {
            tmem_ld_wait(r2);
            tmem_ld_wait(r3);
        }
    }
    if (TRACE && tr && lane == 0)
        tr[1] = clock_after(r0[0] ^ r0[31] ^ (NCH > 1 ? r1[31] : 0u));
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
        if (local_release) mbar_arrive_relaxed(tempty);
        else if (!(dflags & FASTED_JOIN_DIAG_NOREMOTE)) mbar_arrive_cluster(tempty);
        if (TRACE && tr) tr[2] = clock64();
    }
    if (dflags & FASTED_JOIN_DIAG_LOADONLY) return;
    if (fast) {
        uint32_t all = and_tree32(r0);
        if (NCH > 1) all &= and_tree32(r1);
        if (NCH > 2) all &= and_tree32(r2) & and_tree32(r3);
        const bool any = __any_sync(0xffffffffu, (int)all >= 0);
        if (TRACE && tr && lane == 0) {
            tr[4] = clock64();
            tr[7] = any ? 1ull : 0ull;
        }
        if (!any) return;
    }
    unsigned long long* const trc = TRACE ? tr : nullptr;
    if (nchunks > 0) epi_chunk_res(a, wr, r0, jb, i, iw, row_ok, trc);
    if (NCH > 1 && nchunks > 1) epi_chunk_res(a, wr, r1, jb + 32, i, iw, row_ok, trc);
    if (NCH > 2 && nchunks > 2) epi_chunk_res(a, wr, r2, jb + 64, i, iw, row_ok);
    if (NCH > 2 && nchunks > 3) epi_chunk_res(a, wr, r3, jb + 96, i, iw, row_ok);
}

// Hit warps (FASTED_RES_HIT, FASTED_MC_HIT).  The trace of the resident
// kernel (below) shows the MMA waiting on the slowest of 32 epilogue warps,
// and the slowest is one that found a candidate and ran the rare path.  With
// NHIT hit warps the epilogue warps never run it: a lane whose row holds a
// candidate copies its 32 words into a shared-memory queue slot and the warp
// moves on; the hit warps pop slots in order, test the row transposed (lane e
// = column e), and own the record writers.  One queue per hit warp, fed by a
// fixed set of epilogue warps; an epilogue warp ends its stream with an END
// entry.  Slot protocol: slots are taken in order from a shared tail
// counter; a producer may fill slot idx once the hit warp's head counter
// (atomically stored after each entry) shows entry idx - Q consumed -- a
// parity wait alone would let a producer two laps ahead overwrite an
// unconsumed slot -- and the slot's empty mbarrier completed; it publishes
// the entry with the slot's full mbarrier.
template <int NHIT>
struct HitQ {
#ifndef FASTED_HITQ_SLOTS
#define FASTED_HITQ_SLOTS 16
#endif
    static constexpr int Q = FASTED_HITQ_SLOTS;     // slots per queue
    static constexpr int HWS = 64;                  // records per staging buffer (hit warp)
    static constexpr int WRITER_BYTES = NHIT * 2 * HWS * 16;
    static constexpr int DATA_BYTES = NHIT * Q * 128;
    static constexpr int META_BYTES = NHIT * Q * 16;
    static constexpr int BARQ_BYTES = NHIT * Q * 16;   // full, empty barriers
    static constexpr int BYTES = WRITER_BYTES + DATA_BYTES + META_BYTES + BARQ_BYTES + 16;
    static __device__ __forceinline__ uint32_t data(uint32_t r, int q, uint32_t s) {
        return r + WRITER_BYTES + ((uint32_t)q * Q + s) * 128u;
    }
    static __device__ __forceinline__ uint32_t meta(uint32_t r, int q, uint32_t s) {
        return r + WRITER_BYTES + DATA_BYTES + ((uint32_t)q * Q + s) * 16u;
    }
    static __device__ __forceinline__ uint32_t full(uint32_t r, int q, uint32_t s) {
        return r + WRITER_BYTES + DATA_BYTES + META_BYTES + ((uint32_t)q * Q + s) * 16u;
    }
    static __device__ __forceinline__ uint32_t tail(uint32_t r, int q) {
        return r + WRITER_BYTES + DATA_BYTES + META_BYTES + BARQ_BYTES + 4u * q;
    }
    static __device__ __forceinline__ uint32_t head(uint32_t r, int q) {
        return tail(r, q) + 8u;
    }
};

// The head counter is accessed with atomics (acquire read, release write):
// ordinary ld.acquire/st.release work too but read as races to racecheck.
__device__ __forceinline__ uint32_t ld_acquire_shared(uint32_t addr) {
    uint32_t v;
    asm volatile("atom.acquire.cta.shared::cta.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_shared(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.release.cta.shared::cta.exch.b32 %0, [%1], %2;"
                 : "=r"(old)
                 : "r"(addr), "r"(v)
                 : "memory");
}
enum { HIT_ROW = 0, HIT_SELF = 1, HIT_END = 2 };

// This CTA's shared::cta address as a shared::cluster address (st.async
// takes the latter; in a non-cluster launch the CTA is rank 0 of 1).
__device__ __forceinline__ uint32_t cluster_addr(uint32_t cta_addr) {
    uint32_t rank, r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(cta_addr), "r"(rank));
    return r;
}

// Relaxed: the entry's bytes travel with st.async and complete the phase
// through complete_tx, so the arrive orders nothing -- a (default) release
// arrive would first wait for this thread's earlier memory operations, e.g.
// a CTA-pair epilogue warp's remote accumulator-release arrive (DSMEM).
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}

// 16-byte asynchronous store into shared::cluster memory; its completion
// counts 16 bytes on the mbarrier `bar` (shared::cluster address).
__device__ __forceinline__ void st_async_v4(uint32_t addr, uint4 v, uint32_t bar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, "
        "[%5];" ::"r"(addr),
        "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// Wait until entry idx's slot is free: its previous lap (entry idx - Q) was
// consumed.  The hit warp publishes its head counter (release, after all 32
// lanes read the entry) and this acquire orders the refill after those
// reads; `head_seen` caches the last reading (a lower bound of the head).
template <int NHIT>
__device__ __forceinline__ void hit_slot_wait(uint32_t reg, int q, uint32_t idx,
                                              uint32_t& head_seen) {
    using H = HitQ<NHIT>;
    if (head_seen + H::Q <= idx) {
        head_seen = ld_acquire_shared(H::head(reg, q));
        if (head_seen + H::Q <= idx) {
            const uint64_t t0 = global_timer();
            while ((head_seen = ld_acquire_shared(H::head(reg, q))) + H::Q <= idx) {
                __nanosleep(32);
                if (global_timer() - t0 > 20000000000ull) __trap();
            }
        }
    }
}

// One queue entry, written by one thread: wait until the slot's previous
// lap was consumed, fill it, publish it.  `creg`: the queue region's
// shared::cluster address (mapped once per warp); `head_seen`: this
// thread's last reading of the hit warp's head counter -- a lower bound of
// it, so the counter is read again only when it cannot prove the slot free.
template <int NHIT>
__device__ __forceinline__ void hit_put(uint32_t reg, uint32_t creg, int q, uint32_t idx,
                                        uint32_t kind, uint32_t i, uint32_t jb, uint32_t mask,
                                        const uint32_t (&r)[32], bool with_data,
                                        uint32_t& head_seen, bool generic = false,
                                        unsigned long long* trs = nullptr) {
    using H = HitQ<NHIT>;
    const uint32_t slot = idx % H::Q;
    hit_slot_wait<NHIT>(reg, q, idx, head_seen);
#ifdef FASTED_TRACE_SLOT
    if (trs) trs[2] = clock_after(head_seen);   // slot known free (trace experiment)
#endif
    if (generic) {   // FASTED_JOIN_DIAG_GENERICQ: plain stores + a release arrive
        if (with_data) {
            const uint32_t d = H::data(reg, q, slot);
#pragma unroll
            for (int k = 0; k < 8; k++)
                st_shared_v4(d + 16u * k,
                             make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]));
        }
        st_shared_v4(H::meta(reg, q, slot), make_uint4(kind, i, jb, mask));
        mbar_arrive(H::full(reg, q, slot));
        return;
    }
    // The entry goes in with st.async (async proxy, completion counted in
    // bytes on the slot's full barrier): the consumer's wait returns once
    // the bytes landed, and the hand-off is the TMA-style one -- no generic
    // shared-memory store for a generic load on another warp to race with.
    const uint32_t full = creg + (H::full(reg, q, slot) - reg);
    mbar_arrive_expect_tx(H::full(reg, q, slot), with_data ? 144u : 16u);
    if (with_data) {
        const uint32_t d = creg + (H::data(reg, q, slot) - reg);
#pragma unroll
        for (int k = 0; k < 8; k++)
            st_async_v4(d + 16u * k, make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]),
                        full);
    }
    st_async_v4(creg + (H::meta(reg, q, slot) - reg), make_uint4(kind, i, jb, mask), full);
}

// Hand one 32-column chunk's candidate rows (and the diagonal's self pairs)
// to hit warp q.  Warp-collective.
template <int NHIT>
__device__ __forceinline__ void hit_push(uint32_t reg, uint32_t creg, uint8_t* smem_raw,
                                         uint32_t raw, int q, const uint32_t (&r)[32],
                                         uint32_t and_r, int jb, int i, int iw, bool row_ok,
                                         uint32_t lane, uint32_t& head_seen, int dflags = 0,
                                         unsigned long long* trp = nullptr) {
    const bool diag = (jb < iw + 32) && (iw < jb + 32);
    uint32_t rows, selfmask = 0u;
    if (!diag) {
        rows = __ballot_sync(0xffffffffu, (int)and_r >= 0 && row_ok);
    } else {
        // every row meets its own column here: candidates other than the self column
        uint32_t lm = hit_mask32(r);
        const bool self = i >= jb && i < jb + 32 && row_ok;
        if (self) lm &= ~(1u << (uint32_t)(i - jb));
        rows = __ballot_sync(0xffffffffu, lm != 0u && row_ok);
        selfmask = __ballot_sync(0xffffffffu, self);
    }
    const uint32_t k = (uint32_t)__popc(rows) + (selfmask ? 1u : 0u);
    if (k == 0u) return;
    uint32_t b0 = 0;
    if (lane == 0)
        b0 = atomicAdd(reinterpret_cast<unsigned*>(smem_raw + (HitQ<NHIT>::tail(reg, q) - raw)), k);
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (trp && lane == 0) trp[0] = clock64();
    // each candidate lane hands its row over (eight 16-byte st.async + the
    // metadata).  Measured alternatives, both slower at 1M x 128: the row
    // transposed across the warp by 32 shuffles and stored with one
    // warp-wide st.async (~1700 vs ~850 cycles per row), and (mask, <= 3
    // hit values) picked by select trees (35.5 vs 32.4 ms per shard).
    if ((rows >> lane) & 1u)
        hit_put<NHIT>(reg, creg, q, b0 + (uint32_t)__popc(rows & lanemask_lt()), HIT_ROW,
                      (uint32_t)i, (uint32_t)jb, 0u, r, !(dflags & FASTED_JOIN_DIAG_HITMETA),
                      head_seen, (dflags & FASTED_JOIN_DIAG_GENERICQ) != 0, trp);
    if (selfmask && lane == 0)
        hit_put<NHIT>(reg, creg, q, b0 + (uint32_t)__popc(rows), HIT_SELF, (uint32_t)iw,
                      (uint32_t)jb, selfmask, r, false, head_seen,
                      (dflags & FASTED_JOIN_DIAG_GENERICQ) != 0);
    if (trp && lane == 0) trp[3] = clock_after(head_seen);
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Ring hand-off (resident kernel, NHIT == RING_NHIT; experiment form).  The
// shared-queue hand-off above costs an epilogue warp ~1400 cycles per
// candidate slice at 1M x 128: a returned tail atomic, a returned head read
// and the slot stores, each a shared-memory round trip behind the tensor
// core's operand traffic.  Here every epilogue warp owns a private ring of
// RING_R slots (no tail atomic), fills a slot with st.async + expect_tx on the
// slot's own full mbarrier (nothing returns: fire and forget), and reads the
// consumer's counter only when its cached copy says the ring is full.  The
// hit warps poll their producers' next slots with mbarrier.test_wait, round
// robin, and publish each producer's consumed count with a release atomic.
// NHIT template value of the ring form: bit 4 set, the low bits count the
// hit warps (2: three would cap the kernel at 80 registers).
constexpr int RING_NHIT = 16 + 2;
constexpr int RING_HW = RING_NHIT & 15;
__host__ __device__ constexpr int hit_warps(int nhit) { return nhit > 0 ? (nhit & 15) : 0; }
struct Ring {
    static constexpr int R = 4;                       // slots per producer warp
    static constexpr int NPROD = 16;                  // producers (the 16 epilogue warps)
    static constexpr int SLOT = 144;                  // 128 B row + 16 B meta
    static constexpr int HWS = 32;                    // records per staging buffer (hit warp)
    static constexpr int WRITER_BYTES = RING_HW * 2 * HWS * 16;
    static constexpr int SLOT_BYTES = NPROD * R * SLOT;
    static constexpr int BAR_BYTES = NPROD * R * 8;
    static constexpr int BYTES = WRITER_BYTES + SLOT_BYTES + BAR_BYTES + NPROD * 4 + 16;
    static __device__ __forceinline__ uint32_t data(uint32_t r, int p, uint32_t s) {
        return r + WRITER_BYTES + ((uint32_t)p * R + s) * SLOT;
    }
    static __device__ __forceinline__ uint32_t full(uint32_t r, int p, uint32_t s) {
        return r + WRITER_BYTES + SLOT_BYTES + ((uint32_t)p * R + s) * 8u;
    }
    static __device__ __forceinline__ uint32_t cons(uint32_t r, int p) {
        return r + WRITER_BYTES + SLOT_BYTES + BAR_BYTES + 4u * (uint32_t)p;
    }
};

__device__ __forceinline__ void ring_init(uint32_t reg, uint8_t* smem_raw, uint32_t raw) {
    for (int p = 0; p < Ring::NPROD; p++) {
        for (uint32_t sl = 0; sl < (uint32_t)Ring::R; sl++) mbar_init(Ring::full(reg, p, sl), 1);
        *reinterpret_cast<volatile uint32_t*>(smem_raw + (Ring::cons(reg, p) - raw)) = 0u;
    }
}

// One entry (one thread): its slot's previous lap was consumed (checked by
// the caller); the bytes travel with st.async and complete the slot's phase.
__device__ __forceinline__ void ring_put(uint32_t reg, uint32_t creg, int p, uint32_t idx,
                                         uint32_t kind, uint32_t i, uint32_t jb, uint32_t mask,
                                         const uint32_t (&r)[32], bool with_data) {
    const uint32_t sl = idx % Ring::R;
    const uint32_t full = creg + (Ring::full(reg, p, sl) - reg);
    mbar_arrive_expect_tx(Ring::full(reg, p, sl), with_data ? 144u : 16u);
    const uint32_t d = creg + (Ring::data(reg, p, sl) - reg);
    if (with_data) {
#pragma unroll
        for (int k = 0; k < 8; k++)
            st_async_v4(d + 16u * k, make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]),
                        full);
    }
    st_async_v4(d + 128u, make_uint4(kind, i, jb, mask), full);
}

// Warp-uniform: make room for `need` more entries (pw pushed, cw cached).
__device__ __forceinline__ void ring_room(uint32_t reg, int p, uint32_t pw, uint32_t& cw,
                                          uint32_t need) {
    if (pw + need - cw <= (uint32_t)Ring::R) return;
    const uint64_t t0 = global_timer();
    while (true) {
        uint32_t c = 0;
        if ((threadIdx.x & 31) == 0) c = ld_acquire_shared(Ring::cons(reg, p));
        cw = __shfl_sync(0xffffffffu, c, 0);
        if (pw + need - cw <= (uint32_t)Ring::R) return;
        __nanosleep(64);
        if (global_timer() - t0 > 20000000000ull) __trap();
    }
}

// Hand one 32-column chunk's candidate rows (and the diagonal's self pairs)
// to this warp's ring.  Warp-collective.
__device__ __forceinline__ void ring_push(uint32_t reg, uint32_t creg, int p, const uint32_t (&r)[32],
                                          uint32_t and_r, int jb, int i, int iw, bool row_ok,
                                          uint32_t lane, uint32_t& pw, uint32_t& cw) {
    const bool diag = (jb < iw + 32) && (iw < jb + 32);
    uint32_t rows, selfmask = 0u;
    if (!diag) {
        rows = __ballot_sync(0xffffffffu, (int)and_r >= 0 && row_ok);
    } else {
        uint32_t lm = hit_mask32(r);
        const bool self = i >= jb && i < jb + 32 && row_ok;
        if (self) lm &= ~(1u << (uint32_t)(i - jb));
        rows = __ballot_sync(0xffffffffu, lm != 0u && row_ok);
        selfmask = __ballot_sync(0xffffffffu, self);
    }
    const uint32_t nrows = (uint32_t)__popc(rows);
    const uint32_t k = nrows + (selfmask ? 1u : 0u);
    if (k == 0u) return;
    const uint32_t rank = (uint32_t)__popc(rows & lanemask_lt());
    uint32_t done = 0;
    while (done < k) {   // warp-uniform; one pass unless the ring is short of room
        ring_room(reg, p, pw, cw, 1u);
        uint32_t n = (uint32_t)Ring::R - (pw - cw);
        if (n > k - done) n = k - done;
        if (((rows >> lane) & 1u) && rank >= done && rank < done + n)
            ring_put(reg, creg, p, pw + (rank - done), HIT_ROW, (uint32_t)i, (uint32_t)jb, 0u, r,
                     true);
        if (selfmask && lane == 0 && nrows >= done && nrows < done + n)
            ring_put(reg, creg, p, pw + (nrows - done), HIT_SELF, (uint32_t)iw, (uint32_t)jb,
                     selfmask, r, false);
        pw += n;
        done += n;
    }
    __syncwarp();
}

__device__ __forceinline__ void ring_end(uint32_t reg, int p, uint32_t lane, uint32_t& pw,
                                         uint32_t& cw) {
    ring_room(reg, p, pw, cw, 1u);
    if (lane == 0) {
        uint32_t none[32];
        ring_put(reg, cluster_addr(reg), p, pw, HIT_END, 0u, 0u, 0u, none, false);
    }
    pw++;
    __syncwarp();
}

// A ring hit warp: poll producers hq, hq + RING_NHIT, ... in turn; each
// ready entry is tested transposed (lane e = column e) and its records written.
__device__ __forceinline__ void ring_warp_loop(const JoinArgs& a, uint32_t reg, int hq, int lane) {
    constexpr int NPQ = (Ring::NPROD + RING_HW - 1) / RING_HW;
    StagedWriter<Ring::HWS> wr;
    writer_init(wr, reg + (uint32_t)hq * 2u * Ring::HWS * 16u);
    uint32_t c[NPQ];
    int nprod = 0;
#pragma unroll
    for (int q = 0; q < NPQ; q++) {
        c[q] = 0u;
        if (hq + q * RING_HW < Ring::NPROD) nprod++;
    }
    uint32_t ended = 0u;   // bit q: producer q sent END
    const uint32_t all = (1u << nprod) - 1u;
    const uint64_t t0 = global_timer();
    uint32_t idle = 0;
    while (ended != all) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < NPQ; q++) {
            const int p = hq + q * RING_HW;
            if (p >= Ring::NPROD || ((ended >> q) & 1u)) continue;
            const uint32_t sl = c[q] % Ring::R;
            if (!mbar_test_only(Ring::full(reg, p, sl), (c[q] / Ring::R) & 1u)) continue;
            any = true;
            const uint32_t d = Ring::data(reg, p, sl);
            const uint4 m = ld_shared_v4(d + 128u);
            if (m.x == HIT_ROW) {
                const uint32_t v = ld_shared_u32(d + 4u * (uint32_t)lane);
                const int64_t is = (int64_t)m.y, j = (int64_t)m.z + lane;
                const bool hit =
                    (int)v >= 0 && j < a.n_logical && j != is && (!a.symmetric || j > is);
                const uint32_t b = __ballot_sync(0xffffffffu, hit);
                if (b) {
                    const float d2 = fmaxf(__fmaf_rn(-2.0f, __uint_as_float(v), a.eps_sq), 0.0f);
                    writer_append(wr, a, b, hit, (uint32_t)(is + 1), (uint32_t)(j + 1), d2);
                    if (a.symmetric)
                        writer_append(wr, a, b, hit, (uint32_t)(j + 1), (uint32_t)(is + 1), d2);
                }
            } else if (m.x == HIT_SELF) {
                const bool mine = (m.w >> lane) & 1u;
                writer_append(wr, a, m.w, mine, m.y + (uint32_t)lane + 1u,
                              m.y + (uint32_t)lane + 1u, 0.0f);
            } else {
                ended |= 1u << q;
            }
            c[q]++;
            __syncwarp();   // every lane's reads of the slot are done
            if (lane == 0) st_release_shared(Ring::cons(reg, p), c[q]);
        }
        if (!any) {
            if (++idle == 4096u) {
                idle = 0;
                if (global_timer() - t0 > 20000000000ull) __trap();
            }
            __nanosleep(32);
        }
    }
    writer_finish(wr, a);
}

// The resident epilogue tile with hit warps: drain, release, slice test, and
// on a candidate only the hand-off.
template <int CG, int TBN, int NSPLIT, int NHIT, bool TRACE = false>
__device__ __forceinline__ void res_epi_tile_hit(const JoinArgs& a, uint32_t reg, uint32_t creg,
                                                 uint32_t& head_seen, uint32_t& ring_pw,
                                                 uint8_t* smem_raw,
                                                 uint32_t raw, int hq, uint32_t tcol,
                                                 uint32_t tfull, uint32_t aph, uint32_t tempty,
                                                 bool local_release, bool spin,
                                                 uint32_t sleep_ns, int dflags, int nchunks,
                                                 bool fast, int jb, int i, int iw, bool row_ok,
                                                 uint32_t lane, unsigned long long* tr = nullptr,
                                                 bool waiter = false) {
    constexpr int NEPI_BAR = 16;   // the resident kernel's epilogue warps
    constexpr int HALF = TBN / NSPLIT;
    constexpr int NCH = HALF / 32;
    static_assert(NCH == 2, "hit-warp epilogue: 64 columns per warp");
    if (dflags & FASTED_JOIN_DIAG_EPIBAR) {
        // one waiter per CTA; the rest sleep in a hardware barrier (no re-polls)
        if (waiter) epi_wait(tfull, aph, spin, sleep_ns);
        asm volatile("bar.sync 1, %0;" ::"r"(NEPI_BAR * 32) : "memory");
    } else if (dflags & FASTED_JOIN_DIAG_EPISPIN) {
        mbar_spin(tfull, aph);
    } else {
        epi_wait(tfull, aph, spin, sleep_ns);
    }
    tc_fence_after();
    if (TRACE && tr && lane == 0) tr[0] = clock64();
    uint32_t r0[32], r1[32];
    if (nchunks > 0) tmem_ld32(tcol, r0);
    if (nchunks > 1) tmem_ld32(tcol + 32u, r1);
    if (nchunks > 0) {
        tmem_ld_wait(r0);
        tmem_ld_wait(r1);
    }
    if (TRACE && tr && lane == 0) tr[1] = clock_after(r0[0] ^ r0[31] ^ r1[31]);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
        if (local_release) mbar_arrive_relaxed(tempty);
        else if (!(dflags & FASTED_JOIN_DIAG_NOREMOTE)) mbar_arrive_cluster(tempty);
        if (TRACE && tr) tr[2] = clock64();
    }
    if (dflags & FASTED_JOIN_DIAG_LOADONLY) return;
    const uint32_t and0 = and_tree32(r0), and1 = and_tree32(r1);
    if (fast) {
        const bool any = __any_sync(0xffffffffu, (int)(and0 & and1) >= 0);
        if (TRACE && tr && lane == 0) {
            tr[4] = clock64();
            tr[7] = any ? 1ull : 0ull;
        }
        if (!any) return;
    }
    if (dflags & FASTED_JOIN_DIAG_NOSLOW) return;
    if (TRACE && tr && lane == 0) tr[5] = clock64();
    if constexpr (NHIT == RING_NHIT) {   // hq: this warp's ring; head_seen: its cached consumed count
        if (nchunks > 0) ring_push(reg, creg, hq, r0, and0, jb, i, iw, row_ok, lane, ring_pw, head_seen);
        if (nchunks > 1)
            ring_push(reg, creg, hq, r1, and1, jb + 32, i, iw, row_ok, lane, ring_pw, head_seen);
    } else {
    if (nchunks > 0)
        hit_push<NHIT>(reg, creg, smem_raw, raw, hq, r0, and0, jb, i, iw, row_ok, lane, head_seen,
                       dflags, (TRACE && tr) ? tr + 4 : nullptr);
    if (nchunks > 1)
        hit_push<NHIT>(reg, creg, smem_raw, raw, hq, r1, and1, jb + 32, i, iw, row_ok, lane,
                       head_seen, dflags);
    }
#ifndef FASTED_TRACE_SLOT
    if (TRACE && tr && lane == 0) tr[6] = clock64();
#endif
}

// Queue barriers and counters (thread 0, before the CTA-wide barrier).
template <int NHIT>
__device__ __forceinline__ void hit_init(uint32_t reg, uint8_t* smem_raw, uint32_t raw) {
    for (int q = 0; q < NHIT; q++) {
        for (uint32_t sl = 0; sl < (uint32_t)HitQ<NHIT>::Q; sl++)
            mbar_init(HitQ<NHIT>::full(reg, q, sl), 1);
        *reinterpret_cast<volatile uint32_t*>(smem_raw + (HitQ<NHIT>::tail(reg, q) - raw)) = 0u;
        *reinterpret_cast<volatile uint32_t*>(smem_raw + (HitQ<NHIT>::head(reg, q) - raw)) = 0u;
    }
}

// An epilogue warp's last entry: END into its hit warp's queue.
template <int NHIT>
__device__ __forceinline__ void hit_end(uint32_t reg, uint8_t* smem_raw, uint32_t raw, int hq,
                                        int lane) {
    if (lane == 0) {
        const uint32_t idx = atomicAdd(
            reinterpret_cast<unsigned*>(smem_raw + (HitQ<NHIT>::tail(reg, hq) - raw)), 1u);
        uint32_t none[32];
        uint32_t head_seen = 0u;
        hit_put<NHIT>(reg, cluster_addr(reg), hq, idx, HIT_END, 0u, 0u, 0u, none, false,
                      head_seen);
    }
    __syncwarp();
}

// A hit warp's whole life: pop queue hq in order until `producers` END
// entries, test each row transposed, write the records.
template <int NHIT, bool TRACE = false>
__device__ __forceinline__ void hit_warp_loop(const JoinArgs& a, uint32_t reg, int hq,
                                              int producers, int lane, bool spin) {
    using H = HitQ<NHIT>;
    StagedWriter<H::HWS> wr;
    writer_init(wr, reg + (uint32_t)hq * 2u * H::HWS * 16u);
    unsigned long long* trh =
        (TRACE && a.trace && blockIdx.x == 0 && hq < TRACE_HIT_WARPS)
            ? a.trace + TRACE_HIT_BASE + (unsigned long long)hq * TRACE_HIT_ENTRIES * 4
            : nullptr;
    int ends = 0;
    for (uint32_t idx = 0; ends < producers; idx++) {
        const uint32_t sl = idx % H::Q;
        unsigned long long* te = (TRACE && trh && idx < (uint32_t)TRACE_HIT_ENTRIES)
                                     ? trh + 4u * idx : nullptr;
        if (TRACE && te && lane == 0) te[0] = clock64();
        if (spin) mbar_spin(H::full(reg, hq, sl), (idx / H::Q) & 1u); else mbar_wait(H::full(reg, hq, sl), (idx / H::Q) & 1u);
        if (TRACE && te && lane == 0) te[1] = clock64();
        const uint4 m = ld_shared_v4(H::meta(reg, hq, sl));
        if ((FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_HITSKIP) && m.x != HIT_END) {
        } else if (m.x == HIT_ROW) {
            const uint32_t v = ld_shared_u32(H::data(reg, hq, sl) + 4u * (uint32_t)lane);
            const int64_t is = (int64_t)m.y, j = (int64_t)m.z + lane;
            const bool hit = (int)v >= 0 && j < a.n_logical && j != is && (!a.symmetric || j > is);
            const uint32_t b = __ballot_sync(0xffffffffu, hit);
            if (b) {
                const float d2 = fmaxf(__fmaf_rn(-2.0f, __uint_as_float(v), a.eps_sq), 0.0f);
                writer_append(wr, a, b, hit, (uint32_t)(is + 1), (uint32_t)(j + 1), d2);
                if (a.symmetric)
                    writer_append(wr, a, b, hit, (uint32_t)(j + 1), (uint32_t)(is + 1), d2);
            }
        } else if (m.x == HIT_SELF) {
            const bool mine = (m.w >> lane) & 1u;
            writer_append(wr, a, m.w, mine, m.y + (uint32_t)lane + 1u, m.y + (uint32_t)lane + 1u,
                          0.0f);
        } else {
            ends++;
        }
        __syncwarp();   // every lane's reads of the slot are done
        if (lane == 0) st_release_shared(H::head(reg, hq), idx + 1u);
        if (TRACE && te && lane == 0) {
            te[2] = clock64();
            te[3] = (unsigned long long)m.x;
        }
    }
    writer_finish(wr, a);
}

// epilogue_tile with hit warps (streaming/multicast kernels): drain,
// release, slice test, hand candidate rows over.
template <int CG, int TBN, int NSPLIT, int NHIT>
__device__ __forceinline__ void epilogue_tile_hit(const JoinArgs& a, uint32_t reg, uint32_t creg, uint32_t& head_seen,
                                                  uint8_t* smem_raw, uint32_t raw, int hq,
                                                  uint32_t tmem_base, uint32_t tempty,
                                                  int64_t row0, int64_t col0, int buf,
                                                  uint32_t aph, int q, int h, int lane,
                                                  bool leader, uint32_t tfull) {
    constexpr int HALF = TBN / NSPLIT;
    constexpr int NCH = HALF / 32;
    static_assert(NCH == 2, "hit-warp epilogue: 64 columns per warp");
    const int64_t iw = row0 + q * 32;
    const int64_t i = iw + lane;
    const bool row_ok = i < a.n_logical && i < a.row_end;
    const int64_t left = a.col_end - (col0 + h * HALF);
    int nchunks = left <= 0 ? 0 : (left >= HALF ? NCH : (int)(left / 32));
    if (row0 >= a.row_end || (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOEPI)) nchunks = 0;
    const uint32_t tcol = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TBN + h * HALF);
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_EPISPIN) mbar_spin(tfull, aph);
    else mbar_wait2(tfull, aph, (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0);
    tc_fence_after();
    uint32_t r0[32], r1[32];
    if (nchunks > 0) tmem_ld32(tcol, r0);
    if (nchunks > 1) tmem_ld32(tcol + 32u, r1);
    if (nchunks > 0) {
        tmem_ld_wait(r0);
        tmem_ld_wait(r1);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
        if (CG == 1 || leader) mbar_arrive_relaxed(tempty);
        else mbar_arrive_remote(tempty, 0);
    }
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_LOADONLY) return;
    const int64_t jb = col0 + h * HALF;
    const uint32_t and0 = and_tree32(r0), and1 = and_tree32(r1);
    if (nchunks == NCH && !((jb < iw + 32) && (iw < jb + HALF))) {
        if (!__any_sync(0xffffffffu, (int)(and0 & and1) >= 0)) return;
    }
    if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOSLOW) return;
    if (nchunks > 0)
        hit_push<NHIT>(reg, creg, smem_raw, raw, hq, r0, and0, (int)jb, (int)i, (int)iw, row_ok,
                       (uint32_t)lane, head_seen);
    if (nchunks > 1)
        hit_push<NHIT>(reg, creg, smem_raw, raw, hq, r1, and1, (int)jb + 32, (int)i, (int)iw,
                       row_ok, (uint32_t)lane, head_seen);
}

template <int CG, bool DIAG, int NEPI = NUM_EPI_WARPS, int NHIT = 0>
__global__ void __launch_bounds__((FIRST_EPI_WARP + NEPI + NHIT) * 32, 1)
join_tc_kernel(const __grid_constant__ CUtensorMap tmap_x,
               const __grid_constant__ CUtensorMap tmap_aug_a,
               const __grid_constant__ CUtensorMap tmap_aug_b, const JoinArgs a,
               const Sched sch) {
    using C = Cfg<CG>;
    constexpr int STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const uint32_t sA = base;
    const uint32_t sB = base + STAGES * A_BYTES;
    const uint32_t bars = sB + STAGES * C::B_BYTES;
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
    auto tfull_bar = [&](int b) { return bars + 8u * (2 * STAGES + b); };
    auto tempty_bar = [&](int b) { return bars + 8u * (2 * STAGES + 2 + b); };
    const uint32_t slot = bars + 8u * (2 * STAGES + 4);
    volatile uint32_t* slot_ptr =
        reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const int64_t tile_id0 = CG == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
    const int64_t tile_step = CG == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            // CG = 2: only the leader's full barrier is used; the leader's
            // expect_tx covers both CTAs' bytes and the peer's TMA completes
            // its bytes there (it cannot run ahead a phase: it first waits
            // for this stage's empty barrier, i.e. the previous phase done).
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), NEPI * CG);
        }
        if constexpr (NHIT > 0) hit_init<NHIT>(bars + BAR_BYTES, smem_raw, raw);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_a))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_b))
                     : "memory");
    }
    if (warp == 0) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             slot),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             slot),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *slot_ptr;

    if (warp == 0) {
        // ---------------- TMA producer: nkb FP16 stages + 1 augment stage per tile
        // (whole warp walks the schedule; one elected lane issues)
        {
            uint64_t pol_evl;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_evl));
            int s = 0;
            uint32_t ph = 0;
            int64_t k = 0;   // this CTA's tile layer
            bool paced = true;   // lane 0's: cleared if a pacing wait gives up
            for (int64_t t = tile_id0; t < sch.total; t += tile_step, ++k) {
                if (sch.pace_w > 0 && k % PACE_TILES == 0 && k > 0) {
                    const int64_t b = k / PACE_TILES;   // block b - 1 issued; gate block b
                    if (lane == 0) {
                        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.pace)
                                     : "memory");
                        if (paced && b >= sch.pace_w)
                            pace_wait(a.pace,
                                      pace_need_stream(sch.total, tile_step, b - sch.pace_w, CG),
                                      paced);
                    }
                    __syncwarp();
                }
                int rt, ct;
                tile_coords(sch, t, rt, ct);
                const int64_t row0 = a.row_begin + (int64_t)rt * C::TILE_M;
                const int64_t col0 = DIAG ? row0 : a.col_begin + (int64_t)ct * BN;
                if (sym_skip(a, row0, col0, BN)) continue;
                // which 128-row halves exist (a half past the range end is skipped:
                // its rows/columns are masked in the epilogue)
                const bool a_hi = row0 + 128 < a.row_end;
                const bool b_hi = col0 + 128 < a.col_end;
                const int my_a = (int)(row0 + 128 * rank);
                const bool a_mine = rank == 0 || a_hi;
                for (int kb = 0; kb < sch.nkb + (DIAG ? 0 : 1); kb++) {
                    if (sch.mma_spin & 2) mbar_spin(empty_bar(s), ph ^ 1u); else mbar_wait(empty_bar(s), ph ^ 1u);
                    const uint32_t fb = full_bar(s);
                    if (elect_one()) {
                    if (kb < sch.nkb) {
                        const int kx = kb * BK;
                        if constexpr (CG == 1) {
                            mbar_expect_tx(fb, A_BYTES + (b_hi ? 2 : 1) * B_HALF_BYTES);
                            tma_load_2d<1>(sA + s * A_BYTES, &tmap_x, fb, kx, (int)row0);
                            tma_load_2d<1>(sB + s * C::B_BYTES, &tmap_x, fb, kx, (int)col0);
                            if (b_hi)
                                tma_load_2d<1>(sB + s * C::B_BYTES + B_HALF_BYTES, &tmap_x, fb, kx,
                                               (int)col0 + 128);
                        } else {
                            if (leader)
                                mbar_expect_tx(fb, (a_hi ? 2 : 1) * A_BYTES +
                                                       (b_hi ? 2 : 1) * B_HALF_BYTES);
                            if (a_mine)
                            {
                                if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_AEVL)
                                    tma_load_2d_pair_hint(sA + s * A_BYTES, &tmap_x, fb, kx, my_a,
                                                          pol_evl);
                                else
                                    tma_load_2d<2>(sA + s * A_BYTES, &tmap_x, fb, kx, my_a);
                            }
                            if (rank == 0 || b_hi)
                                tma_load_2d<2>(sB + s * C::B_BYTES, &tmap_x, fb, kx,
                                               (int)(col0 + 128 * rank));
                        }
                    } else {
                        constexpr int AUG_A = BM * AUG_ROW_BYTES;
                        constexpr int AUG_B_HALF = 128 * AUG_ROW_BYTES;
                        if constexpr (CG == 1) {
                            mbar_expect_tx(fb, AUG_A + (b_hi ? 2 : 1) * AUG_B_HALF);
                            tma_load_2d<1>(sA + s * A_BYTES, &tmap_aug_a, fb, 0, (int)row0);
                            tma_load_2d<1>(sB + s * C::B_BYTES, &tmap_aug_b, fb, 0, (int)col0);
                            if (b_hi)
                                tma_load_2d<1>(sB + s * C::B_BYTES + AUG_B_HALF, &tmap_aug_b, fb,
                                               0, (int)col0 + 128);
                        } else {
                            if (leader)
                                mbar_expect_tx(fb, (a_hi ? 2 : 1) * AUG_A +
                                                       (b_hi ? 2 : 1) * AUG_B_HALF);
                            if (a_mine)
                                tma_load_2d<2>(sA + s * A_BYTES, &tmap_aug_a, fb, 0, my_a);
                            if (rank == 0 || b_hi)
                                tma_load_2d<2>(sB + s * C::B_BYTES, &tmap_aug_b, fb, 0,
                                               (int)(col0 + 128 * rank));
                        }
                    }
                    }
                    __syncwarp();
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
            // a final block of exactly PACE_TILES layers is counted here (the
            // loop above counts a block when the next one starts)
            if (sch.pace_w > 0 && k > 0 && k % PACE_TILES == 0 && lane == 0)
                asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.pace) : "memory");
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------- MMA issuer (the leader CTA of a pair)
        if (leader) {   // whole warp; one elected lane issues
            const bool no_mma = (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOMMA) != 0;
            int s = 0;
            uint32_t ph = 0;
            int lt = 0;
            for (int64_t t = tile_id0; t < sch.total; t += tile_step, ++lt) {
                if (a.symmetric) {
                    int rt, ct;
                    tile_coords(sch, t, rt, ct);
                    if (sym_skip(a, a.row_begin + (int64_t)rt * C::TILE_M,
                                 a.col_begin + (int64_t)ct * BN, BN)) {
                        --lt;
                        continue;
                    }
                }
                const int buf = lt & 1;
                const uint32_t aph = (uint32_t)(lt >> 1) & 1u;
                if (sch.mma_spin & 1) mbar_spin(tempty_bar(buf), aph ^ 1u);
                else mbar_wait(tempty_bar(buf), aph ^ 1u);
                tc_fence_after();
                const uint32_t dtm = tmem_base + (uint32_t)(buf * BN);
                for (int kb = 0; kb < sch.nkb + (DIAG ? 0 : 1); kb++) {
                    if (sch.mma_spin & 1) mbar_spin(full_bar(s), ph);
                    else mbar_wait(full_bar(s), ph);
                    tc_fence_after();
                    if (elect_one()) {
                    if (!no_mma) {
                        if (kb < sch.nkb) {
                            const uint64_t ad = sw128_desc(sA + s * A_BYTES);
                            const uint64_t bd = sw128_desc(sB + s * C::B_BYTES);
#pragma unroll
                            for (int kk = 0; kk < BK / UK; kk++) {
                                const uint64_t koff = (uint64_t)((kk * UK * 2) >> 4);
                                mma_f16<CG>(dtm, ad + koff, bd + koff, (kb | kk) != 0 ? 1u : 0u);
                            }
                        } else {
                            mma_tf32<CG>(dtm, sw32_desc(sA + s * A_BYTES),
                                         sw32_desc(sB + s * C::B_BYTES));
                        }
                    }
                    mma_commit<CG>(empty_bar(s));
                    }
                    __syncwarp();
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                if (elect_one()) mma_commit<CG>(tfull_bar(buf));
                __syncwarp();
            }
        }
        __syncwarp();
    } else if (NHIT > 0 && warp >= FIRST_EPI_WARP + NEPI) {
        // ---------------- hit warp
        hit_warp_loop<NHIT>(a, bars + BAR_BYTES, warp - FIRST_EPI_WARP - NEPI, NEPI / NHIT, lane,
                            (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0 || (sch.mma_spin & 4));
    } else {
        // ---------------- epilogue
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int h = (warp - FIRST_EPI_WARP) >> 2;   // column half of the accumulator
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        // staging: 16 KB for the epilogue warps (64 records per buffer with 8
        // warps, 32 with 16); with hit warps the region holds their queues
        constexpr int WST = WSTAGE * NUM_EPI_WARPS / NEPI;
        StagedWriter<WST> wr;
        if constexpr (NHIT == 0)
            writer_init(wr, bars + BAR_BYTES + (uint32_t)(warp - FIRST_EPI_WARP) * 2 * WST * 16);
        const uint32_t hit_creg = NHIT > 0 ? cluster_addr(bars + BAR_BYTES) : 0u;
        uint32_t head_seen = 0u;
        int lt = 0;
        for (int64_t t = tile_id0; t < sch.total; t += tile_step, ++lt) {
            int rt, ct;
            tile_coords(sch, t, rt, ct);
            const int64_t row0 = a.row_begin + (int64_t)rt * C::TILE_M + 128 * rank;
            const int64_t col0 = a.col_begin + (int64_t)ct * BN;
            if (sym_skip(a, a.row_begin + (int64_t)rt * C::TILE_M, col0, BN)) {
                --lt;
                continue;
            }
            const int buf = lt & 1;
            const uint32_t aph = (uint32_t)(lt >> 1) & 1u;
            if constexpr (DIAG) {
                const int64_t i = row0 + q * 32 + lane;
                // Gram-diagonal pre-pass (CG = 1, col0 = row0): lane i's own
                // column i - row0 = 32 q + lane sits in chunk q of half 0.
                mbar_wait(tfull_bar(buf), aph);
                tc_fence_after();
                uint32_t r0[32];
                if (h == 0) {
                    tmem_ld32(tmem_base + lane_base + (uint32_t)(buf * BN + q * 32), r0);
                    tmem_ld_wait(r0);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty_bar(buf));
                if (h == 0 && i < a.row_end) a.gram_diag[i] = __uint_as_float(pick32(r0, lane));
                continue;
            }
            if constexpr (NHIT > 0)
                epilogue_tile_hit<CG, BN, NEPI / 4, NHIT>(
                    a, bars + BAR_BYTES, hit_creg, head_seen, smem_raw, raw, (warp - FIRST_EPI_WARP) % NHIT, tmem_base,
                    tempty_bar(buf), row0, col0, buf, aph, q, h, lane, leader, tfull_bar(buf));
            else
                epilogue_tile<CG, BN, NEPI / 4>(a, wr, tmem_base, tempty_bar(buf), row0, col0, buf,
                                                aph, q, h, lane, leader, tfull_bar(buf));
        }
        if constexpr (NHIT > 0)
            hit_end<NHIT>(bars + BAR_BYTES, smem_raw, raw, (warp - FIRST_EPI_WARP) % NHIT, lane);
        else
            writer_finish(wr, a);
    }

    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS)
                         : "memory");
    }
}

// ---------------------------------------------------------------------------
// B-multicast variant (large d).  At d = 960 the single-CTA kernel moves
// 737 KB of A and B from L2 per 128 x 256 tile, and measurement says that
// traffic, not the MMA, sets both the rate and the power: the TMA stream
// alone (no MMA, no epilogue) runs at ~10 KB/clk chip-wide and takes 1452 ms
// at the 1 kW cap against 1570 ms for the whole join (profiles/round1/
// tune_c4_power_session2.txt).  Here two CTAs of a cluster take vertically
// adjacent row tiles of the same column tile: each loads its own A and HALF
// of the shared B tile, multicast into both CTAs' shared memory, so per SM
// the bytes per tile drop by a third (491 KB).  Each CTA still issues its own
// M = 128 MMAs (no cross-SM operand reads, unlike cta_group::2).  A stage is
// refilled only after BOTH CTAs' MMAs released it (empty barrier count 2,
// multicast commits).  Every load is issued even for a tile past the range
// end (its rows/columns are masked in the epilogue; TMA zero-fills past
// n_pad), so the byte counts are fixed.
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster."
        "b64 [%0], %1;" ::"r"(bar),
        "h"(mask)
        : "memory");
}

constexpr int MC_STAGES = 4;
constexpr int MC_SMEM_BYTES =
    MC_STAGES * (A_BYTES + 2 * B_HALF_BYTES) + BAR_BYTES + WSTAGE_BYTES + 1024;

template <int NEPI, int NHIT = 0>
__global__ void __launch_bounds__((FIRST_EPI_WARP + NEPI + NHIT) * 32, 1)
join_tc_mc_kernel(const __grid_constant__ CUtensorMap tmap_x,
                  const __grid_constant__ CUtensorMap tmap_aug_a,
                  const __grid_constant__ CUtensorMap tmap_aug_b, const JoinArgs a,
                  const Sched sch) {
    constexpr int STAGES = MC_STAGES;
    constexpr int B_BYTES = 2 * B_HALF_BYTES;
    constexpr int AUG_A = BM * AUG_ROW_BYTES;
    constexpr int AUG_B_HALF = 128 * AUG_ROW_BYTES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const uint32_t sA = base;
    const uint32_t sB = base + STAGES * A_BYTES;
    const uint32_t bars = sB + STAGES * B_BYTES;
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
    auto tfull_bar = [&](int b) { return bars + 8u * (2 * STAGES + b); };
    auto tempty_bar = [&](int b) { return bars + 8u * (2 * STAGES + 2 + b); };
    const uint32_t slot = bars + 8u * (2 * STAGES + 4);
    volatile uint32_t* slot_ptr = reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t cr = cluster_rank();   // 0: upper row tile, 1: lower
    const int64_t tile_id0 = (int64_t)(blockIdx.x >> 1);
    const int64_t tile_step = (int64_t)(gridDim.x >> 1);
    constexpr uint16_t BOTH = 0x3;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 2);   // both CTAs' MMAs read this stage's B
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), NEPI);
        }
        if constexpr (NHIT > 0) hit_init<NHIT>(bars + BAR_BYTES, smem_raw, raw);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_a))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_b))
                     : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();   // peers' barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = *slot_ptr;

    if (warp == 0) {
        // ---------------- TMA producer (whole warp; one elected lane issues)
        int s = 0;
        uint32_t ph = 0;
        int64_t k = 0;   // this cluster's tile layer (pacing, as the streaming kernel)
        bool paced = true;
        for (int64_t t = tile_id0; t < sch.total; t += tile_step, ++k) {
            if (sch.pace_w > 0 && k % PACE_TILES == 0 && k > 0) {
                const int64_t b = k / PACE_TILES;
                if (lane == 0) {
                    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.pace)
                                 : "memory");
                    if (paced && b >= sch.pace_w)
                        pace_wait(a.pace, pace_need_stream(sch.total, tile_step, b - sch.pace_w, 2),
                                  paced);
                }
                __syncwarp();
            }
            int rt, ct;
            tile_coords(sch, t, rt, ct);
            if (sym_skip(a, a.row_begin + (int64_t)rt * 2 * BM, a.col_begin + (int64_t)ct * BN,
                         BN))
                continue;
            const int row0 = (int)(a.row_begin + ((int64_t)rt * 2 + cr) * BM);
            const int colh = (int)(a.col_begin + (int64_t)ct * BN + 128 * cr);
            for (int kb = 0; kb < sch.nkb + 1; kb++) {
                if (sch.mma_spin & 2) mbar_spin(empty_bar(s), ph ^ 1u); else mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t fb = full_bar(s);
                if (elect_one()) {
                    if (kb < sch.nkb) {
                        const int kx = kb * BK;
                        mbar_expect_tx(fb, A_BYTES + B_BYTES);
                        tma_load_2d<1>(sA + s * A_BYTES, &tmap_x, fb, kx, row0);
                        tma_load_2d_mc(sB + s * B_BYTES + cr * B_HALF_BYTES, &tmap_x, fb, kx, colh,
                                       BOTH);
                    } else {
                        mbar_expect_tx(fb, AUG_A + 2 * AUG_B_HALF);
                        tma_load_2d<1>(sA + s * A_BYTES, &tmap_aug_a, fb, 0, row0);
                        tma_load_2d_mc(sB + s * B_BYTES + cr * AUG_B_HALF, &tmap_aug_b, fb, 0, colh,
                                       BOTH);
                    }
                }
                __syncwarp();
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        if (sch.pace_w > 0 && k > 0 && k % PACE_TILES == 0 && lane == 0)   // a final full block
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.pace) : "memory");
    } else if (warp == 1) {
        // ---------------- MMA issuer (every CTA; M = 128; whole warp, one lane issues)
        const bool no_mma = (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOMMA) != 0;
        int s = 0;
        uint32_t ph = 0;
        int lt = 0;
        for (int64_t t = tile_id0; t < sch.total; t += tile_step, ++lt) {
            if (a.symmetric) {
                int rt, ct;
                tile_coords(sch, t, rt, ct);
                if (sym_skip(a, a.row_begin + (int64_t)rt * 2 * BM,
                             a.col_begin + (int64_t)ct * BN, BN)) {
                    --lt;
                    continue;
                }
            }
            const int buf = lt & 1;
            if (sch.mma_spin & 1)
                mbar_spin(tempty_bar(buf), ((uint32_t)(lt >> 1) & 1u) ^ 1u);
            else
                mbar_wait2(tempty_bar(buf), ((uint32_t)(lt >> 1) & 1u) ^ 1u,
                           (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0);
            tc_fence_after();
            const uint32_t dtm = tmem_base + (uint32_t)(buf * BN);
            for (int kb = 0; kb < sch.nkb + 1; kb++) {
                if (sch.mma_spin & 1) mbar_spin(full_bar(s), ph); else mbar_wait(full_bar(s), ph);
                tc_fence_after();
                const uint64_t ad = sw128_desc(sA + s * A_BYTES);
                const uint64_t bd = sw128_desc(sB + s * B_BYTES);
                if (elect_one()) {
                    if (!no_mma) {
                        if (kb < sch.nkb) {
#pragma unroll
                            for (int kk = 0; kk < BK / UK; kk++) {
                                const uint64_t koff = (uint64_t)((kk * UK * 2) >> 4);
                                mma_f16<1>(dtm, ad + koff, bd + koff, (kb | kk) != 0 ? 1u : 0u);
                            }
                        } else {
                            mma_tf32<1>(dtm, sw32_desc(sA + s * A_BYTES), sw32_desc(sB + s * B_BYTES));
                        }
                    }
                    mma_commit_mc(empty_bar(s), BOTH);
                }
                __syncwarp();
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (elect_one()) mma_commit<1>(tfull_bar(buf));
            __syncwarp();
        }
    } else if (NHIT > 0 && warp >= FIRST_EPI_WARP + NEPI) {
        // ---------------- hit warp
        hit_warp_loop<NHIT>(a, bars + BAR_BYTES, warp - FIRST_EPI_WARP - NEPI, NEPI / NHIT, lane,
                            (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0 || (sch.mma_spin & 4));
    } else {
        // ---------------- epilogue
        const int q = warp & 3;
        const int h = (warp - FIRST_EPI_WARP) >> 2;
        constexpr int WST = WSTAGE * NUM_EPI_WARPS / NEPI;   // 16 KB of staging either way
        StagedWriter<WST> wr;
        if constexpr (NHIT == 0)
            writer_init(wr, bars + BAR_BYTES + (uint32_t)(warp - FIRST_EPI_WARP) * 2 * WST * 16);
        const uint32_t hit_creg = NHIT > 0 ? cluster_addr(bars + BAR_BYTES) : 0u;
        uint32_t head_seen = 0u;
        int lt = 0;
        for (int64_t t = tile_id0; t < sch.total; t += tile_step, ++lt) {
            int rt, ct;
            tile_coords(sch, t, rt, ct);
            const int64_t row0 = a.row_begin + ((int64_t)rt * 2 + cr) * BM;
            const int64_t col0 = a.col_begin + (int64_t)ct * BN;
            if (sym_skip(a, a.row_begin + (int64_t)rt * 2 * BM, col0, BN)) {
                --lt;
                continue;
            }
            const int buf = lt & 1;
            if constexpr (NHIT > 0)
                epilogue_tile_hit<1, BN, NEPI / 4, NHIT>(
                    a, bars + BAR_BYTES, hit_creg, head_seen, smem_raw, raw, (warp - FIRST_EPI_WARP) % NHIT, tmem_base,
                    tempty_bar(buf), row0, col0, buf, (uint32_t)(lt >> 1) & 1u, q, h, lane, true,
                    tfull_bar(buf));
            else
                epilogue_tile<1, BN, NEPI / 4>(a, wr, tmem_base, tempty_bar(buf), row0, col0, buf,
                                               (uint32_t)(lt >> 1) & 1u, q, h, lane, true,
                                               tfull_bar(buf));
        }
        if constexpr (NHIT > 0)
            hit_end<NHIT>(bars + BAR_BYTES, smem_raw, raw, (warp - FIRST_EPI_WARP) % NHIT, lane);
        else
            writer_finish(wr, a);
    }

    tc_fence_before();
    cluster_sync();   // no CTA leaves while its peer may still multicast into it
    tc_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
}

// ---------------------------------------------------------------------------
// Resident-A variant (d_pad <= 512).  At d = 128 one 256 x 256 tile
// is only 9 MMAs, and streaming both operands moves 144 KB per CTA pair per
// tile from L2: measured, the TMA stream alone (no MMA, no epilogue) takes
// 192 ms at 1M x 128, against a 121 ms tensor floor (profiles/round1/
// tune_c3_session2.txt) -- the streaming kernel is L2->SM bound there.  Here
// a CTA keeps its 128-row A panel (every k-block plus its augment rows) in
// shared memory for a whole work unit -- one row tile x a segment of column
// tiles -- and streams only B, halving the bytes per MMA.  A is double
// buffered when two panels fit, so the next unit's A lands while the current
// one finishes.  Units are ordered segment-major, so the CTAs (pairs) that run
// side by side sweep the same B panels at the same time (L2 reuse).
//
// TBN = columns per tile.  With TBN = 128 the 512 TMEM columns hold FOUR
// accumulators instead of two: at d = 128 a tile is only ~600 MMA cycles and
// ncu showed the MMA warp waiting for an accumulator on 53% of tiles with two
// buffers (the epilogue warp that found hits in a tile runs late); four
// buffers absorb that jitter.  The MMA sequence per output element (k-blocks
// ascending, then the tf32 augment step) is the streaming kernel's, so both
// produce identical bits.
struct ResSched {
    int row_tiles;            // tiles of TILE_M rows in [row_begin, row_end)
    int col_tiles;            // tiles of TBN columns in [col_begin, col_end)
    int nsegs;                // column segments (balanced)
    int nkb;                  // 64-wide k-blocks
    int na;                   // A buffers (1 or 2)
    int stages;               // B ring stages
    uint32_t a_buf_bytes;     // one A buffer: nkb k-blocks + augment rows, 1024-aligned
    int64_t units;            // row_tiles * nsegs
    int lanes;                // units in flight: CTA pairs (CTAs) launched
    uint32_t epi_sleep_ns;    // epilogue accumulator wait backoff (0: suspend hint)
    int mma_spin = MMA_SPIN_DEFAULT;   // MMA_SPIN_DEFAULT bits (FASTED_MMA_SPIN in experiments)
    int pace_w = 0;           // unit layers a CTA may run ahead of the slowest (0: unpaced)
    int order = 0;            // unit order: 0 row-tile rounds, 1 segment-major
};

// Records per staging buffer in the resident kernel (tight shared memory):
// 8 KB for the epilogue in total, so the B ring keeps its 7 stages at d = 128
// (16 KB cost a stage: no-epilogue 204 vs 174 ms at 1M x 128).
#ifndef FASTED_RES_WSTAGE
#define FASTED_RES_WSTAGE 256
#endif
constexpr int RES_WSTAGE_TOTAL = FASTED_RES_WSTAGE;   // records, all epilogue warps x 2 buffers

template <int CG, int TBN>
struct ResCfg {
    static constexpr int TILE_M = BM * CG;
    static constexpr int NB = TBN / CG;                          // B rows (columns) per CTA
    static constexpr int BBOX = NB < 128 ? NB : 128;             // TMA box rows for B
    static constexpr int B_BYTES = NB * BK * 2;                  // this CTA's B k-block
    static constexpr int AUGB_BYTES = NB * AUG_ROW_BYTES;        // its augment rows
    static constexpr int STAGE_BYTES = B_BYTES + AUGB_BYTES;
    static constexpr int NACC = TMEM_COLS / TBN;                 // accumulator buffers
    static constexpr int MAX_STAGES = 16;
    static constexpr int BARS = 2 * MAX_STAGES + 2 * NACC + 4;
    static constexpr int BAR_REGION = ((BARS * 8 + 4 + 127) / 128) * 128;
    static constexpr uint32_t IDESC_F16 =
        (1u << 4) | ((uint32_t)(TBN >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);
    static constexpr uint32_t IDESC_TF32 = IDESC_F16 | (2u << 7) | (2u << 10);
    static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1024-aligned");
};

// Pacing (bounded drift).  Every lane walks the same sequence of unit layers
// (its ua-th unit is in layer ua), so co-running pairs share each B segment
// in L2 only while they stay within a few layers of each other.  Uneven
// epilogue work lets them drift apart (C3: 671 GB of HBM reads per launch,
// L2 hit rate 45%, against 188 GB with no epilogue).  With pace_w > 0 a
// producer starts layer ua only after all CTAs issued layer ua - pace_w: a
// global count of issued units (one relaxed-release add per unit per CTA).
// Total CTA-units in layers 0..j:
__device__ __forceinline__ unsigned long long pace_need(const ResSched& s, int64_t j, int cg) {
    const int64_t full = s.units / s.lanes, rem = s.units % s.lanes;
    const int64_t t = j + 1 < full ? j + 1 : full;
    return (unsigned long long)cg * (unsigned long long)(t * s.lanes + (j >= full ? rem : 0));
}

// Unit order (ResSched::order).  1, the default: segment-major -- unit u is
// row tile u % row_tiles of column segment u / row_tiles, so the co-running
// pairs sweep neighbouring row tiles of the same B segment and a pair that
// runs a few units ahead is still on it.  0: rounds of `lanes` row tiles.  Inside a round, lane (pair) p
// keeps row tile round * lanes + p and sweeps the column segments in order,
// all lanes on the same segment at the same time -- so co-running pairs share
// each B panel in L2 (as a segment-major order would), each pair's A panel
// stays the same for a whole round, and the record stream is row-coherent:
// a row's records are produced within one round, not spread over the whole
// launch (the canonical-order scatter then writes each row's segment while it
// is still in L2).  A last, partial round of m row tiles is spread over all
// lanes (unit v -> row tile v % m, segment v / m).
__device__ __forceinline__ void res_unit(const ResSched& s, int64_t u, int& rt, int& ct0,
                                         int& ct1) {
    if (s.order == 1) {   // segment-major: all row tiles on segment 0, then segment 1, ...
        const int64_t g = u / s.row_tiles;
        rt = (int)(u - g * s.row_tiles);
        ct0 = (int)((int64_t)s.col_tiles * g / s.nsegs);
        ct1 = (int)((int64_t)s.col_tiles * (g + 1) / s.nsegs);
        return;
    }
    const int64_t per_round = (int64_t)s.lanes * s.nsegs;
    const int64_t R = u / per_round;
    const int64_t v = u - R * per_round;
    const int64_t rt0 = R * s.lanes;
    const int64_t left = (int64_t)s.row_tiles - rt0;
    const int64_t m = left < s.lanes ? left : s.lanes;
    const int64_t g = v / m;
    rt = (int)(rt0 + (v - g * m));
    ct0 = (int)((int64_t)s.col_tiles * g / s.nsegs);
    ct1 = (int)((int64_t)s.col_tiles * (g + 1) / s.nsegs);
}

// res_unit with FASTED_JOIN_SYMMETRIC applied: the unit's column tiles start
// at the first one reaching the diagonal (an emptied unit still loads its A
// panel and commits it, so every role walks the same unit sequence).
template <int TILE_M, int TBN>
__device__ __forceinline__ void res_unit_sym(const ResSched& s, const JoinArgs& a, int64_t u,
                                             int& rt, int& ct0, int& ct1) {
    res_unit(s, u, rt, ct0, ct1);
    if (a.symmetric) {
        const int64_t num = (int64_t)rt * TILE_M - TBN + 1;   // ct * TBN + TBN - 1 >= rt * TILE_M
        const int ct_min = num <= 0 ? 0 : (int)((num + TBN - 1) / TBN);
        if (ct0 < ct_min) ct0 = ct_min < ct1 ? ct_min : ct1;
    }
}

// NHIT > 0: hit warps own the rare path; NHIT == 0: staged writers in the
// epilogue warps; NHIT == -1: DirectWriter (registers -> global) in the
// epilogue warps, the per-lane hit-mask search, no shared memory on the hit path.
template <int CG, int TBN, int NEPI, bool TRACE = false, int NHIT = 0>
__global__ void __launch_bounds__((FIRST_EPI_WARP + NEPI + hit_warps(NHIT)) * 32, 1)
join_tc_res_kernel(const __grid_constant__ CUtensorMap tmap_xa,
                   const __grid_constant__ CUtensorMap tmap_xb,
                   const __grid_constant__ CUtensorMap tmap_aug_a,
                   const __grid_constant__ CUtensorMap tmap_aug_b, const JoinArgs a,
                   const ResSched sch) {
    using C = ResCfg<CG, TBN>;
    constexpr int NACC = C::NACC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const int S = sch.stages;
    const uint32_t sAb = base;
    const uint32_t sB = base + (uint32_t)sch.na * sch.a_buf_bytes;
    const uint32_t bars = sB + (uint32_t)S * C::STAGE_BYTES;
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (S + s); };
    auto tfull_bar = [&](int b) { return bars + 8u * (2 * S + b); };
    auto tempty_bar = [&](int b) { return bars + 8u * (2 * S + NACC + b); };
    auto afull_bar = [&](int b) { return bars + 8u * (2 * S + 2 * NACC + b); };
    auto aempty_bar = [&](int b) { return bars + 8u * (2 * S + 2 * NACC + 2 + b); };
    const uint32_t slot = bars + 8u * (2 * S + 2 * NACC + 4);
    volatile uint32_t* slot_ptr = reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - raw));
    const uint32_t a_aug_off = (uint32_t)sch.nkb * A_BYTES;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const int64_t unit0 = CG == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
    const int64_t ustep = CG == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < NACC; b++) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b),
                      (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOREMOTE) ? NEPI : NEPI * CG);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(afull_bar(b), 1);
            mbar_init(aempty_bar(b), 1);
        }
        if constexpr (NHIT == RING_NHIT) ring_init(bars + C::BAR_REGION, smem_raw, raw);
        else if constexpr (NHIT > 0) hit_init<NHIT>(bars + C::BAR_REGION, smem_raw, raw);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_xa))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_xb))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_a))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_b))
                     : "memory");
    }
    if (warp == 0) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             slot),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             slot),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *slot_ptr;

    if (warp == 0) {
        // ---------------- TMA producer: per unit the A panel, then nkb B stages per tile
        // (whole warp walks the schedule; one elected lane issues)
        {
            int s = 0;
            uint32_t ph = 0;
            int ua = 0;
            bool paced = true;   // lane 0's: cleared if a pacing wait gives up
            for (int64_t u = unit0; u < sch.units; u += ustep, ++ua) {
                if (sch.pace_w > 0 && ua >= sch.pace_w) {
                    if (lane == 0 && paced)
                        pace_wait(a.pace, pace_need(sch, ua - sch.pace_w, CG), paced);
                    __syncwarp();
                }
                int rt, ct0, ct1;
                res_unit_sym<C::TILE_M, TBN>(sch, a, u, rt, ct0, ct1);
                const int64_t row0 = a.row_begin + (int64_t)rt * C::TILE_M;
                const bool a_hi = row0 + 128 < a.row_end;
                const int my_a = (int)(row0 + 128 * rank);
                const bool a_mine = rank == 0 || a_hi;
                const int ab = ua % sch.na;
                mbar_wait(aempty_bar(ab), ((uint32_t)(ua / sch.na) & 1u) ^ 1u);
                const uint32_t fa = afull_bar(ab);
                const uint32_t abuf = sAb + (uint32_t)ab * sch.a_buf_bytes;
                const uint32_t a_bytes = (uint32_t)sch.nkb * A_BYTES + BM * AUG_ROW_BYTES;
                if (elect_one()) {
                    if (CG == 1) mbar_expect_tx(fa, a_bytes);
                    else if (leader) mbar_expect_tx(fa, (a_hi ? 2u : 1u) * a_bytes);
                    if (a_mine) {
                        for (int kb = 0; kb < sch.nkb; kb++)
                            tma_load_2d<CG>(abuf + kb * A_BYTES, &tmap_xa, fa, kb * BK, my_a);
                        tma_load_2d<CG>(abuf + a_aug_off, &tmap_aug_a, fa, 0, my_a);
                    }
                }
                __syncwarp();
                for (int ct = ct0; ct < ct1; ct++) {
                    const int64_t col0 = a.col_begin + (int64_t)ct * TBN;
                    // this CTA's NB columns, in BBOX-row TMA boxes that exist
                    // (a box past the range end is skipped; masked in the epilogue)
                    const int64_t cb = col0 + (int64_t)C::NB * rank;
                    int nbox = 0;
                    for (int x = 0; x < C::NB / C::BBOX; x++)
                        if (cb + (int64_t)C::BBOX * x < a.col_end) nbox++;
                    int nbox_pair = nbox;
                    if (CG == 2 && leader) {
                        const int64_t cb1 = col0 + C::NB;
                        for (int x = 0; x < C::NB / C::BBOX; x++)
                            if (cb1 + (int64_t)C::BBOX * x < a.col_end) nbox_pair++;
                    }
                    for (int kb = 0; kb < sch.nkb; kb++) {
                        const bool last = kb == sch.nkb - 1;
                        if (sch.mma_spin & 2) mbar_spin(empty_bar(s), ph ^ 1u); else mbar_wait(empty_bar(s), ph ^ 1u);
                        const uint32_t fb = full_bar(s);
                        const uint32_t st = sB + (uint32_t)s * C::STAGE_BYTES;
                        const uint32_t box_bytes =
                            C::BBOX * (BK * 2 + (last ? AUG_ROW_BYTES : 0));
                        const bool el = elect_one();
                        if ((FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOTMA) != 0) {
                            if (el && (CG == 1 || leader)) mbar_arrive(fb);
                        } else if (el) {
                            if (CG == 1 || leader)
                                mbar_expect_tx(fb, (uint32_t)nbox_pair * box_bytes);
                            for (int x = 0; x < nbox; x++) {
                                const int c = (int)(cb + C::BBOX * x);
                                tma_load_2d<CG>(st + x * C::BBOX * BK * 2, &tmap_xb, fb, kb * BK, c);
                                if (last)
                                    tma_load_2d<CG>(st + C::B_BYTES + x * C::BBOX * AUG_ROW_BYTES,
                                                    &tmap_aug_b, fb, 0, c);
                            }
                        }
                        __syncwarp();
                        if (++s == S) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
                if (sch.pace_w > 0 && lane == 0)   // this unit issued
                    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.pace)
                                 : "memory");
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------- MMA issuer (the leader CTA of a pair)
        if (leader) {   // whole warp; one elected lane issues
            const bool no_mma = (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOMMA) != 0;
            int s = 0;
            uint32_t ph = 0;
            int lt = 0, ua = 0;
            for (int64_t u = unit0; u < sch.units; u += ustep, ++ua) {
                int rt, ct0, ct1;
                res_unit_sym<C::TILE_M, TBN>(sch, a, u, rt, ct0, ct1);
                const int ab = ua % sch.na;
                mbar_wait(afull_bar(ab), (uint32_t)(ua / sch.na) & 1u);
                tc_fence_after();
                const uint32_t abuf = sAb + (uint32_t)ab * sch.a_buf_bytes;
                for (int ct = ct0; ct < ct1; ct++, ++lt) {
                    const int buf = lt % NACC;
                    if (sch.mma_spin & 1)
                        mbar_spin(tempty_bar(buf), ((uint32_t)(lt / NACC) & 1u) ^ 1u);
                    else
                        mbar_wait2(tempty_bar(buf), ((uint32_t)(lt / NACC) & 1u) ^ 1u,
                                   (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0);
                    tc_fence_after();
                    unsigned long long* tr =
                        (TRACE && a.trace && blockIdx.x == 0 && lt < TRACE_TILES)
                            ? a.trace + 2 * lt
                            : nullptr;
                    if (TRACE && tr && lane == 0) tr[0] = clock64();
                    const uint32_t dtm = tmem_base + (uint32_t)(buf * TBN);
                    for (int kb = 0; kb < sch.nkb; kb++) {
                        if (sch.mma_spin & 1) mbar_spin(full_bar(s), ph);
                        else mbar_wait(full_bar(s), ph);
                        tc_fence_after();
                        const uint32_t st = sB + (uint32_t)s * C::STAGE_BYTES;
                        if (elect_one()) {
                        if (!no_mma) {
                            const uint64_t ad = sw128_desc(abuf + kb * A_BYTES);
                            const uint64_t bd = sw128_desc(st);
#pragma unroll
                            for (int kk = 0; kk < BK / UK; kk++) {
                                const uint64_t koff = (uint64_t)((kk * UK * 2) >> 4);
                                mma_f16<CG>(dtm, ad + koff, bd + koff, (kb | kk) != 0 ? 1u : 0u,
                                            C::IDESC_F16);
                            }
                            if (kb == sch.nkb - 1) {
                                if (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_AUGF16)
                                    mma_f16<CG>(dtm, sw32_desc(abuf + a_aug_off),
                                                sw32_desc(st + C::B_BYTES), 1u, C::IDESC_F16);
                                else if (!(FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_NOAUG))
                                    mma_tf32<CG>(dtm, sw32_desc(abuf + a_aug_off),
                                                 sw32_desc(st + C::B_BYTES), C::IDESC_TF32);
                            }
                        }
                        mma_commit<CG>(empty_bar(s));
                        }
                        __syncwarp();
                        if (++s == S) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                    if (elect_one()) mma_commit<CG>(tfull_bar(buf));
                    __syncwarp();
                    if (TRACE && tr && lane == 0) tr[1] = clock64();
                }
                if (elect_one()) mma_commit<CG>(aempty_bar(ab));
                __syncwarp();
            }
        }
        __syncwarp();
    } else if (NHIT > 0 && warp >= FIRST_EPI_WARP + NEPI) {
        // ---------------- hit warp
        if constexpr (NHIT == RING_NHIT)
            ring_warp_loop(a, bars + C::BAR_REGION, warp - FIRST_EPI_WARP - NEPI, lane);
        else if constexpr (NHIT > 0)
            hit_warp_loop<NHIT, TRACE>(a, bars + C::BAR_REGION, warp - FIRST_EPI_WARP - NEPI,
                                       NEPI / NHIT, lane,
                                       (FASTED_DFLAGS(a) & FASTED_JOIN_DIAG_SPIN) != 0 ||
                                           (sch.mma_spin & 4));
    } else {
        // ---------------- epilogue
        constexpr int NSPLIT = NEPI / 4;
        constexpr int HALF = TBN / NSPLIT;            // columns per warp
        constexpr int NCH = HALF / 32;
        const int q = warp & 3;                       // TMEM lane quarter
        const int h = (warp - FIRST_EPI_WARP) >> 2;   // column group (NEPI / 4 of them)
        constexpr int RWS = RES_WSTAGE_TOTAL / (2 * NEPI) * 2;   // 16 (NEPI 16) / 32 (NEPI 8)
        using EpiWriter = std::conditional_t<(NHIT < 0), DirectWriter, StagedWriter<RWS>>;
        EpiWriter wr;
        // per warp: two staging buffers, then the 128-byte row stash (no
        // writers here when hit warps write the records)
        if constexpr (NHIT == 0)
            writer_init(wr, bars + C::BAR_REGION +
                                (uint32_t)(warp - FIRST_EPI_WARP) * (2 * RWS * 16 + EPI_STASH_BYTES));
        else if constexpr (NHIT < 0)
            writer_init(wr);
        static_assert(NACC == 2, "lean epilogue assumes two accumulators");
        const uint32_t tcol0 = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * HALF);
        const bool local_release = CG == 1 || leader;
        const uint32_t release0 = local_release ? tempty_bar(0) : mapa_shared(tempty_bar(0), 0);
        // the two accumulator-release barriers are adjacent (tempty_bar(1) =
        // tempty_bar(0) + 8), in the cluster window too: no per-buffer select
        const uint32_t tfull0 = tfull_bar(0);
        const int dflags = FASTED_DFLAGS(a);
        const bool spin = (dflags & FASTED_JOIN_DIAG_SPIN) != 0;
        const bool noepi = (dflags & FASTED_JOIN_DIAG_NOEPI) != 0;
        // 32-bit point indices (n_pad < 2^31; records hold 32-bit ids anyway);
        // this warp's first column in tile 0 of the range
        const int jbase = (int)a.col_begin + h * HALF;
        const int col_end = (int)a.col_end;
        const uint32_t hit_creg = NHIT > 0 ? cluster_addr(bars + C::BAR_REGION) : 0u;
        uint32_t head_seen = 0u;   // queue: last head read; ring: cached consumed count
        uint32_t ring_pw = 0u;     // ring: entries pushed
        int lt = 0;
        uint32_t buf = 0, aph = 0;
        for (int u = (int)unit0; u < (int)sch.units; u += (int)ustep) {
            int rt, ct0, ct1;
            res_unit_sym<C::TILE_M, TBN>(sch, a, u, rt, ct0, ct1);
            const int row0 = (int)a.row_begin + rt * C::TILE_M + 128 * (int)rank;
            const int iw = row0 + q * 32;
            const int i = iw + lane;
            const bool row_ok = i < a.n_logical && i < a.row_end;
            const bool rows_in = row0 < a.row_end && !noepi;
            // tiles whose slice [jb, jb + HALF) lies inside [.., col_end)
            const int room = col_end - jbase - HALF;
            int ct_full = (room < 0 || !rows_in) ? 0 : room / TBN + 1;
            // the one tile (if any) whose slice meets rows [iw, iw + 32):
            // jb in (iw - HALF, iw + 32), jb = jbase + ct * TBN
            const int x = iw + 31 - jbase;
            const int ct_diag = (x >= 0 && (x / TBN) * TBN > x - 31 - HALF) ? x / TBN : -1;
            for (int ct = ct0; ct < ct1; ct++, ++lt) {
                const int jb = jbase + ct * TBN;
                int nchunks = NCH;
                if (ct >= ct_full) {
                    const int left = col_end - jb;
                    nchunks = (!rows_in || left <= 0) ? 0
                              : (left >= HALF ? NCH : left / 32);
                }
                const bool fast = ct < ct_full && ct != ct_diag;
                unsigned long long* tr = nullptr;
                if (TRACE && a.trace && blockIdx.x == 0 && lt < TRACE_TILES)
                    tr = a.trace + 2 * TRACE_TILES +
                         8 * (lt * TRACE_EPI_WARPS + (warp - FIRST_EPI_WARP));
                if constexpr (NHIT > 0)
                    res_epi_tile_hit<CG, TBN, NSPLIT, NHIT, TRACE>(
                        a, bars + C::BAR_REGION, hit_creg, head_seen, ring_pw, smem_raw, raw,
                        NHIT == RING_NHIT ? warp - FIRST_EPI_WARP
                                          : (warp - FIRST_EPI_WARP) % hit_warps(NHIT),
                        tcol0 + buf * TBN, tfull0 + 8u * buf, aph, release0 + 8u * buf,
                        local_release, spin, sch.epi_sleep_ns, dflags, nchunks, fast, jb, i, iw,
                        row_ok, (uint32_t)lane, tr, warp == FIRST_EPI_WARP);
                else
                    res_epi_tile<CG, TBN, NSPLIT, TRACE>(
                        a, wr, tcol0 + buf * TBN, tfull0 + 8u * buf, aph,
                        release0 + 8u * buf, local_release, spin, sch.epi_sleep_ns, dflags,
                        nchunks, fast, jb, i, iw, row_ok, lane, tr);
                if (TRACE && tr && lane == 0) tr[3] = clock64();
                buf ^= 1u;
                aph ^= buf ^ 1u;   // phase flips after buffer 1
            }
        }
        if constexpr (NHIT == RING_NHIT)   // end of this warp's stream in its ring
            ring_end(bars + C::BAR_REGION, warp - FIRST_EPI_WARP, (uint32_t)lane, ring_pw, head_seen);
        else if constexpr (NHIT > 0)   // end of this warp's stream in its hit warp's queue
            hit_end<NHIT>(bars + C::BAR_REGION, smem_raw, raw, (warp - FIRST_EPI_WARP) % NHIT, lane);
        else
            writer_finish(wr, a);
    }

    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS)
                         : "memory");
    }
}

#ifdef FASTED_EXPERIMENTS
// ---------------------------------------------------------------------------
// TMEM-A variant (d_pad <= 128, CTA pair).  The resident kernel at d = 128 is
// epilogue bound: a 256 x 256 tile is ~1150 MMA cycles and, with only two
// 256-column accumulators, a tile whose epilogue runs late (hits to write)
// stalls the MMA.  Narrower tiles with more accumulators need N = 128 MMAs,
// which re-read A from shared memory twice as often (measured slower).  Here
// A lives in TMEM instead (tcgen05.mma A-from-TMEM): each CTA's 128-row A
// panel (d_pad / 2 columns, two FP16 per 32-bit column, one row per lane) is
// written by four loader warps with tcgen05.st, double buffered per unit, and
// the 512 TMEM columns hold 2 A panels + THREE 128-column accumulators.
// B streams through shared memory as in the resident kernel; the tf32
// augment step keeps both operands in shared memory.
constexpr int TS_TBN = 128;
constexpr int TS_NACC = 3;
constexpr int TS_NEPI = 16;
constexpr int TS_LOAD_WARP0 = FIRST_EPI_WARP + TS_NEPI;           // 4 A-loader warps
constexpr int TS_THREADS = (TS_LOAD_WARP0 + 4) * 32;
constexpr int TS_A_COLS = 64;                                      // d_pad <= 128
constexpr int TS_ACC0 = 2 * TS_A_COLS;                             // first accumulator column
constexpr int TS_NB = TS_TBN / 2;                                  // B rows per CTA
constexpr int TS_STAGE_BYTES = TS_NB * BK * 2 + TS_NB * AUG_ROW_BYTES;   // 10 KB
constexpr int TS_AUGA_BYTES = BM * AUG_ROW_BYTES;                  // 4 KB
constexpr int TS_MAX_STAGES = 16;
constexpr int TS_BARS = 2 * TS_MAX_STAGES + 2 * TS_NACC + 6 + 1;
constexpr int TS_BAR_REGION = ((TS_BARS * 8 + 4 + 127) / 128) * 128;
constexpr int TS_WSTAGE = 16;                                      // records per staging buffer
constexpr uint32_t TS_IDESC_F16 =
    (1u << 4) | ((uint32_t)(TS_TBN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t TS_IDESC_TF32 = TS_IDESC_F16 | (2u << 7) | (2u << 10);
static_assert(TS_STAGE_BYTES % 1024 == 0, "stages must stay 1024-aligned");

__device__ __forceinline__ void mma_f16_ts2(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(TS_IDESC_F16), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
        "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

__global__ void __launch_bounds__(TS_THREADS, 1)
join_tc_ts_kernel(const uint4* __restrict__ X, const __grid_constant__ CUtensorMap tmap_xb,
                  const __grid_constant__ CUtensorMap tmap_aug_a,
                  const __grid_constant__ CUtensorMap tmap_aug_b, const JoinArgs a,
                  const ResSched sch) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const int S = sch.stages;
    const uint32_t sAug = base;                                   // 2 x aug A (4 KB each)
    const uint32_t sB = base + 2 * 4096;
    const uint32_t bars = sB + (uint32_t)S * TS_STAGE_BYTES;
    auto full_bar = [&](int st) { return bars + 8u * st; };
    auto empty_bar = [&](int st) { return bars + 8u * (S + st); };
    auto tfull_bar = [&](int b) { return bars + 8u * (2 * S + b); };
    auto tempty_bar = [&](int b) { return bars + 8u * (2 * S + TS_NACC + b); };
    auto afull_bar = [&](int b) { return bars + 8u * (2 * S + 2 * TS_NACC + b); };       // TMEM A
    auto augfull_bar = [&](int b) { return bars + 8u * (2 * S + 2 * TS_NACC + 2 + b); }; // TMA aug A
    auto aempty_bar = [&](int b) { return bars + 8u * (2 * S + 2 * TS_NACC + 4 + b); };
    const uint32_t slot = bars + 8u * (2 * S + 2 * TS_NACC + 6);
    volatile uint32_t* slot_ptr = reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - raw));
    const uint32_t wst_base = bars + TS_BAR_REGION;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int64_t unit0 = (int64_t)(blockIdx.x >> 1);
    const int64_t ustep = (int64_t)(gridDim.x >> 1);
    constexpr int TILE_M = 2 * BM;

    if (threadIdx.x == 0) {
        for (int st = 0; st < S; st++) {
            mbar_init(full_bar(st), 1);
            mbar_init(empty_bar(st), 1);
        }
        for (int b = 0; b < TS_NACC; b++) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), TS_NEPI * 2);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(afull_bar(b), 4 * 2);      // the A-loader warps of both CTAs
            mbar_init(augfull_bar(b), 1);
            mbar_init(aempty_bar(b), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_xb))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_a))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_aug_b))
                     : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *slot_ptr;
    const int nks = (int)(a.d_pad / UK);   // K=16 steps over the resident A

    if (warp == 0) {
        // ---------------- TMA producer: aug A per unit, nkb B stages per tile
        int st = 0;
        uint32_t ph = 0;
        int ua = 0;
        for (int64_t u = unit0; u < sch.units; u += ustep, ++ua) {
            int rt, ct0, ct1;
            res_unit_sym<TILE_M, TS_TBN>(sch, a, u, rt, ct0, ct1);
            const int64_t row0 = a.row_begin + (int64_t)rt * TILE_M;
            const bool a_hi = row0 + 128 < a.row_end;
            const int my_a = (int)(row0 + 128 * rank);
            const int ab = ua & 1;
            mbar_wait(aempty_bar(ab), ((uint32_t)(ua >> 1) & 1u) ^ 1u);
            if (elect_one()) {
                if (leader) mbar_expect_tx(augfull_bar(ab), (a_hi ? 2u : 1u) * TS_AUGA_BYTES);
                if (leader || a_hi)
                    tma_load_2d<2>(sAug + (uint32_t)ab * 4096u, &tmap_aug_a, augfull_bar(ab), 0,
                                   my_a);
            }
            __syncwarp();
            for (int ct = ct0; ct < ct1; ct++) {
                const int64_t col0 = a.col_begin + (int64_t)ct * TS_TBN;
                const int cb = (int)(col0 + TS_NB * rank);
                const bool mine = cb < a.col_end;
                const bool peer = col0 + TS_NB < a.col_end;
                for (int kb = 0; kb < sch.nkb; kb++) {
                    const bool last = kb == sch.nkb - 1;
                    mbar_wait(empty_bar(st), ph ^ 1u);
                    const uint32_t fb = full_bar(st);
                    const uint32_t sa = sB + (uint32_t)st * TS_STAGE_BYTES;
                    if (elect_one()) {
                        const uint32_t box = TS_NB * (BK * 2 + (last ? AUG_ROW_BYTES : 0));
                        if (leader) mbar_expect_tx(fb, (1u + (peer ? 1u : 0u)) * box);
                        if (mine) {
                            tma_load_2d<2>(sa, &tmap_xb, fb, kb * BK, cb);
                            if (last)
                                tma_load_2d<2>(sa + TS_NB * BK * 2, &tmap_aug_b, fb, 0, cb);
                        }
                    }
                    __syncwarp();
                    if (++st == S) {
                        st = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA)
        if (leader) {
            int st = 0;
            uint32_t ph = 0;
            int lt = 0, ua = 0;
            for (int64_t u = unit0; u < sch.units; u += ustep, ++ua) {
                int rt, ct0, ct1;
                res_unit_sym<TILE_M, TS_TBN>(sch, a, u, rt, ct0, ct1);
                const int ab = ua & 1;
                const uint32_t aph = (uint32_t)(ua >> 1) & 1u;
                mbar_wait(afull_bar(ab), aph);
                mbar_wait(augfull_bar(ab), aph);
                tc_fence_after();
                const uint32_t atm = tmem_base + (uint32_t)(ab * TS_A_COLS);
                for (int ct = ct0; ct < ct1; ct++, ++lt) {
                    const int buf = lt % TS_NACC;
                    mbar_wait(tempty_bar(buf), ((uint32_t)(lt / TS_NACC) & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t dtm = tmem_base + (uint32_t)(TS_ACC0 + buf * TS_TBN);
                    for (int kb = 0; kb < sch.nkb; kb++) {
                        mbar_wait(full_bar(st), ph);
                        tc_fence_after();
                        const uint32_t sa = sB + (uint32_t)st * TS_STAGE_BYTES;
                        const uint64_t bd = sw128_desc(sa);
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < BK / UK; kk++) {
                                const int k16 = kb * (BK / UK) + kk;
                                if (k16 < nks)
                                    mma_f16_ts2(dtm, atm + (uint32_t)(k16 * (UK / 2)),
                                                bd + (uint64_t)((kk * UK * 2) >> 4),
                                                k16 != 0 ? 1u : 0u);
                            }
                            if (kb == sch.nkb - 1)
                                mma_tf32<2>(dtm, sw32_desc(sAug + (uint32_t)ab * 4096u),
                                            sw32_desc(sa + TS_NB * BK * 2), TS_IDESC_TF32);
                            mma_commit<2>(empty_bar(st));
                        }
                        __syncwarp();
                        if (++st == S) {
                            st = 0;
                            ph ^= 1u;
                        }
                    }
                    if (elect_one()) mma_commit<2>(tfull_bar(buf));
                    __syncwarp();
                }
                if (elect_one()) mma_commit<2>(aempty_bar(ab));
                __syncwarp();
            }
        }
    } else if (warp >= TS_LOAD_WARP0) {
        // ---------------- A loaders: this CTA's 128 rows into TMEM, one row per lane
        const int q = warp & 3;
        int ua = 0;
        for (int64_t u = unit0; u < sch.units; u += ustep, ++ua) {
            int rt, ct0, ct1;
            res_unit_sym<TILE_M, TS_TBN>(sch, a, u, rt, ct0, ct1);
            const int64_t row = a.row_begin + (int64_t)rt * TILE_M + 128 * rank + 32 * q + lane;
            const int ab = ua & 1;
            mbar_wait(aempty_bar(ab), ((uint32_t)(ua >> 1) & 1u) ^ 1u);
            const int words = (int)(a.d_pad / 2);        // FP16 pairs in the row
            const uint4* src = X + row * (a.d_pad / 8);
            const uint32_t tdst =
                tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * TS_A_COLS);
#pragma unroll
            for (int half = 0; half < 2; half++) {   // 32 columns (64 FP16) at a time
                uint32_t v[32];
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const int w0 = half * 32 + 4 * c;
                    const uint4 w = (row < a.n_pad && w0 < words) ? __ldg(src + half * 8 + c)
                                                                  : make_uint4(0u, 0u, 0u, 0u);
                    v[4 * c] = w.x;
                    v[4 * c + 1] = w.y;
                    v[4 * c + 2] = w.z;
                    v[4 * c + 3] = w.w;
                }
                tmem_st32(tdst + (uint32_t)(half * 32), v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(afull_bar(ab));
                else mbar_arrive_remote_release(afull_bar(ab), 0);
            }
        }
    } else {
        // ---------------- epilogue: 16 warps, 32 x 32 each of a 128-column accumulator
        const int q = warp & 3;
        const int h = (warp - FIRST_EPI_WARP) >> 2;
        StagedWriter<TS_WSTAGE> wr;
        writer_init(wr, wst_base + (uint32_t)(warp - FIRST_EPI_WARP) * 2 * TS_WSTAGE * 16);
        int lt = 0;
        for (int64_t u = unit0; u < sch.units; u += ustep) {
            int rt, ct0, ct1;
            res_unit_sym<TILE_M, TS_TBN>(sch, a, u, rt, ct0, ct1);
            const int64_t row0 = a.row_begin + (int64_t)rt * TILE_M + 128 * rank;
            for (int ct = ct0; ct < ct1; ct++, ++lt) {
                const int buf = lt % TS_NACC;
                epilogue_tile<2, TS_TBN, 4>(a, wr, tmem_base + TS_ACC0, tempty_bar(buf), row0,
                                            a.col_begin + (int64_t)ct * TS_TBN, buf,
                                            (uint32_t)(lt / TS_NACC) & 1u, q, h, lane, leader,
                                            tfull_bar(buf));
            }
        }
        writer_finish(wr, a);
    }

    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
}
#endif  // FASTED_EXPERIMENTS

// Exact split of an FP32 value into three TF32 values (10-bit mantissas,
// low 13 bits zero) whose sum is the input: 3 x 11 significant bits >= 24.
__device__ __forceinline__ void split_tf32(float x, float& h1, float& h2, float& h3) {
    auto tf32 = [](float v) {
        uint32_t u;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v));
        return __uint_as_float(u & 0xffffe000u);
    };
    h1 = tf32(x);
    const float r1 = __fsub_rn(x, h1);
    h2 = tf32(r1);
    h3 = tf32(__fsub_rn(r1, h2));
}

// Augment rows: A_i = [sigma_i parts (3), 1, 1, 1, 1, 1] and
// B_j = [1, 1, 1, rho_j parts (3), rho'_j parts (2)] with sigma = -s/2 (exact)
// and rho + rho' = sigma + eps^2/2 EXACTLY (TwoSum: rho = RN(sigma + eps^2/2),
// rho' its rounding error, an FP32 value below ulp(rho)/2 whose two TF32
// parts drop at most its last 2 bits, i.e. < 2^-46 |rho|).  So
// A_i . B_j = (eps^2 - s_i - s_j) / 2 up to the tensor core's own summation:
// even when eps^2 >> s, an exact duplicate pair comes out at
// D = eps^2/2, i.e. distance 0, as in the reference.
__global__ void aug_prepare_kernel(const float* __restrict__ norms, int64_t begin, int64_t end,
                                   float eps_sq, float4* __restrict__ aug_a,
                                   float4* __restrict__ aug_b) {
    const int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= end) return;
    const float sigma = -0.5f * norms[i];
    const float half_eps = 0.5f * eps_sq;   // exact (no underflow for eps_sq >= 2^-125)
    const float rho = __fadd_rn(sigma, half_eps);
    // TwoSum (Knuth): rho + err == sigma + half_eps exactly
    const float bv = __fsub_rn(rho, sigma);
    const float av = __fsub_rn(rho, bv);
    const float err = __fadd_rn(__fsub_rn(sigma, av), __fsub_rn(half_eps, bv));
    float a1, a2, a3, b1, b2, b3, c1, c2, c3;
    split_tf32(sigma, a1, a2, a3);
    split_tf32(rho, b1, b2, b3);
    split_tf32(err, c1, c2, c3);
    aug_a[2 * i] = make_float4(a1, a2, a3, 1.0f);
    aug_a[2 * i + 1] = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
    aug_b[2 * i] = make_float4(1.0f, 1.0f, 1.0f, b1);
    aug_b[2 * i + 1] = make_float4(b2, b3, c1, c2);
}

}  // namespace tc

template <int CG, bool DIAG = false, int NEPI = tc::NUM_EPI_WARPS, int NHIT = 0>
static cudaError_t launch_variant(const CUtensorMap& mx, const CUtensorMap& ma,
                                  const CUtensorMap& mb, const JoinArgs& a, const tc::Sched& sch,
                                  cudaStream_t s) {
    using namespace tc;
    auto kern = join_tc_kernel<CG, DIAG, NEPI, NHIT>;
    static PerDeviceOnce attr_once;
    {
        cudaError_t e = attr_once.run([&] {
            return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Cfg<CG>::SMEM_BYTES);
        });
        if (e != cudaSuccess) return e;
    }
    const int sms = sm_count_current();
    const int64_t units = sms / CG;   // CTAs (or CTA pairs) resident at once
    const int64_t work = sch.total < units ? sch.total : units;
    if (work <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(work * CG));
    cfg.blockDim = dim3((FIRST_EPI_WARP + NEPI + NHIT) * 32);
    cfg.dynamicSmemBytes = Cfg<CG>::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, mx, ma, mb, a, sch);
}

// B-multicast launch: clusters of two CTAs over super-tiles of 256 rows.
template <int NEPI, int NHIT = 0>
static cudaError_t launch_mc(const CUtensorMap& mx, const CUtensorMap& ma, const CUtensorMap& mb,
                             const JoinArgs& a, cudaStream_t s) {
    using namespace tc;
    static_assert(HitQ<2>::BYTES <= WSTAGE_BYTES, "hit queues live in the staging region");
    auto kern = join_tc_mc_kernel<NEPI, NHIT>;
    static PerDeviceOnce attr_once;
    {
        cudaError_t e = attr_once.run([&] {
            return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        MC_SMEM_BYTES);
        });
        if (e != cudaSuccess) return e;
    }
    Sched sch;
    sch.diag = 0;
    sch.mma_spin = FASTED_KNOB("FASTED_MMA_SPIN", MMA_SPIN_DEFAULT);
    sch.row_tiles = (int)((a.row_end - a.row_begin + 2 * BM - 1) / (2 * BM));   // super-rows
    sch.col_tiles = (int)((a.col_end - a.col_begin + BN - 1) / BN);
    // 8192-row groups (measured at 1M x 960: 1374 TFLOPS vs 1305 for 4096 and
    // 1182 for 16384; profiles/round1/tune_c4_elect_session2.txt)
    sch.group = FASTED_KNOB("FASTED_GROUP_ROWS", 8192) / (2 * BM);
    if (sch.group < 1) sch.group = 1;
    sch.nkb = (int)((a.d_pad + BK - 1) / BK);
    sch.total = (int64_t)sch.row_tiles * sch.col_tiles;
    sch.pace_w = a.pace ? FASTED_KNOB("FASTED_MC_PACE_W", 0) : 0;
    const int64_t slots = sm_count_current() / 2;
    const int64_t work = sch.total < slots ? sch.total : slots;
    if (work <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(work * 2));
    cfg.blockDim = dim3((FIRST_EPI_WARP + NEPI + NHIT) * 32);
    cfg.dynamicSmemBytes = MC_SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, mx, ma, mb, a, sch);
}

// Resident-A launch: shared memory split between the A buffer(s) and as many
// B stages as fit.
template <int CG, int TBN, int NEPI, int NHIT = 0>
static cudaError_t launch_res(const CUtensorMap& mxa, const CUtensorMap& mxb,
                              const CUtensorMap& ma, const CUtensorMap& mb, const JoinArgs& a,
                              cudaStream_t s) {
    using namespace tc;
    using C = ResCfg<CG, TBN>;
    constexpr int SMEM_MAX = 227 * 1024;
#ifdef FASTED_EXPERIMENTS
    constexpr bool CAN_TRACE = CG == 2 && TBN == 256 && NEPI == 16;
#else
    constexpr bool CAN_TRACE = false;   // the clock64 timeline exists in libfasted_exp.so only
#endif
    auto kern = join_tc_res_kernel<CG, TBN, NEPI, false, NHIT>;
    static PerDeviceOnce attr_once, attr_once_trace;
    PerDeviceOnce* once = &attr_once;
    if constexpr (CAN_TRACE) {
        if (a.trace) {
            kern = join_tc_res_kernel<CG, TBN, NEPI, true, NHIT>;
            once = &attr_once_trace;
        }
    }
    {
        cudaError_t e = once->run([&] {
            return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        SMEM_MAX);
        });
        if (e != cudaSuccess) return e;
    }
    ResSched sch;
    sch.nkb = (int)((a.d_pad + BK - 1) / BK);
    sch.a_buf_bytes = (uint32_t)((sch.nkb * A_BYTES + BM * AUG_ROW_BYTES + 1023) & ~1023);
    const int wstage = NHIT == RING_NHIT ? Ring::BYTES
                       : NHIT > 0    ? HitQ<(NHIT > 0 ? NHIT : 1)>::BYTES
                       : NHIT == 0 ? NEPI * (2 * (RES_WSTAGE_TOTAL / (2 * NEPI) * 2) * 16 +
                                             EPI_STASH_BYTES)
                                   : 0;
    const int budget = SMEM_MAX - 1024 - C::BAR_REGION - wstage;
    sch.na = 2 * (int)sch.a_buf_bytes <= 80 * 1024 ? 2 : 1;
    sch.stages = (budget - sch.na * (int)sch.a_buf_bytes) / C::STAGE_BYTES;
    if (sch.stages > C::MAX_STAGES) sch.stages = C::MAX_STAGES;
    if (sch.stages < 2) return cudaErrorInvalidValue;
    sch.row_tiles = (int)((a.row_end - a.row_begin + C::TILE_M - 1) / C::TILE_M);
    sch.col_tiles = (int)((a.col_end - a.col_begin + TBN - 1) / TBN);
    // a segment of ~16K columns per unit: the A panel load is amortised over
    // many tiles and the units stay small enough to balance
    sch.epi_sleep_ns = (uint32_t)FASTED_KNOB("FASTED_EPI_SLEEP_NS", 0);
    // bounded drift of 2 unit layers (C3 243-247 vs 291 ms, HBM reads 47 vs 712 GB per
    // launch; C5 shard S~4096 1998 vs 2621 ms; S~256 unchanged -- pace_ab.txt)
    sch.pace_w = a.pace ? FASTED_KNOB("FASTED_PACE_W", 2) : 0;
    // segment-major unit order (with pacing: C3 234 vs 244 ms, C5 shard S~4096 1970 vs
    // 2090 ms, S~1024 1677 vs 1721, C2 2.67 vs 2.80 ms; the S~4096 sort is 115 vs 82 ms
    // because a row's records spread over the launch -- profiles/round2/unit_order_ab.txt)
    sch.order = FASTED_KNOB("FASTED_RES_ORDER", 1);
    sch.mma_spin = FASTED_KNOB("FASTED_MMA_SPIN", MMA_SPIN_DEFAULT);
    // ~16K columns per unit; 64K with hit warps (sparse output) and a
    // single-buffered A panel (d_pad > 256), whose reload every unit then
    // shows: C5 shard S~16 / eps 0 1532 / 1534 vs 1554 / 1553 ms; dense output
    // and C2 prefer 16K (S~1024 1630 vs 1647, C2 2.60 vs 3.05 ms;
    // profiles/round2/segment_length_single_a_ab.txt)
    int seg = FASTED_KNOB("FASTED_SEG_TILES",
                          (NHIT > 0 && sch.na == 1 ? 65536 : 16384) / TBN);
    if (seg < 1) seg = 1;
    sch.nsegs = (sch.col_tiles + seg - 1) / seg;
    sch.units = (int64_t)sch.row_tiles * sch.nsegs;
    const int smem = sch.na * (int)sch.a_buf_bytes + sch.stages * C::STAGE_BYTES +
                     C::BAR_REGION + wstage + 1024;
    const int64_t slots = sm_count_current() / CG;
    const int64_t work = sch.units < slots ? sch.units : slots;
    if (work <= 0) return cudaSuccess;
    sch.lanes = (int)work;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(work * CG));
    cfg.blockDim = dim3((FIRST_EPI_WARP + NEPI + hit_warps(NHIT)) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, mxa, mxb, ma, mb, a, sch);
}

// Which tcgen05 join kernel (and CTA group) a launch uses (env overrides:
// FASTED_CTA_GROUP=1|2 forces the streaming kernel, FASTED_RESIDENT=0 and
// FASTED_MC=0 disable the resident and multicast forms).
//   d_pad <= 512                          resident-A CTA pair
//   d_pad >  256, large, low output       streaming CTA pair, 16K-row raster
//   d_pad >  256 otherwise                B-multicast clusters
// The CTA pair (cta_group::2) reaches ~91% tensor-pipe utilisation per
// clock but its power grows with the epilogue's record traffic: at the 1 kW
// cap it wins at low selectivity (1M x 960, S = 48: 1376 vs 1333 TFLOPS;
// 5M x 384 shard, S <= 16: 1342-1352 vs 1205-1261) and loses as pairs per
// point grow (S ~ 250: 1053 vs 1234; S ~ 1000: 837 vs 1221), so the caller's
// FASTED_JOIN_LOW_OUTPUT hint (<= 128 pairs per row expected) selects it.
// Small joins are not power bound and the multicast form wins there
// (60K x 512: 1203 vs 1186).
enum { TC_STREAMING = 0, TC_RESIDENT = 1, TC_MULTICAST = 2 };
static int tc_variant(int64_t d_pad, int64_t rows, int64_t cols, bool low_output, int* cg) {
    const int cg_env = FASTED_KNOB("FASTED_CTA_GROUP", 0);
    // resident A up to d_pad 512 (one 132 KB A buffer + 4 B stages at 512);
    // measured at 60K x 512: 2.52 vs 2.85 ms, 5M x 384 shard: 1616-1640 vs
    // 2003-2122 ms for S <= 1000 (alternating launches) -- the streaming
    // forms move A and B from L2 per tile (~64 B/clk/SM at d = 512, above
    // what L2 delivers at 1.97 GHz), resident A only B
    const int64_t res_max = FASTED_KNOB("FASTED_RES_MAXD", 512);
    *cg = cg_env == 1 ? 1 : cg_env == 2 ? 2 : (d_pad <= res_max ? 2 : 1);
    if (d_pad <= res_max) return FASTED_KNOB("FASTED_RESIDENT", 1) != 0 ? TC_RESIDENT : TC_STREAMING;
    if (cg_env != 0 || FASTED_KNOB("FASTED_MC", 1) == 0) return TC_STREAMING;
    if (low_output && (double)rows * (double)cols >= 68.7e9 &&   // >= 2^36 pairs examined
        FASTED_KNOB("FASTED_PAIR_LOWOUT", 1) != 0) {
        *cg = 2;
        return TC_STREAMING;
    }
    return TC_MULTICAST;
}

// Hit warps (resident CTA pair, multicast): on the caller's
// FASTED_JOIN_SPARSE hint; FASTED_RES_HIT / FASTED_MC_HIT = 0 or 2 override.
static bool res_hit(bool sparse) { return FASTED_KNOB("FASTED_RES_HIT", sparse ? 2 : 0) == 2; }
static bool mc_hit(bool sparse) { return FASTED_KNOB("FASTED_MC_HIT", sparse ? 2 : 0) == 2; }
static bool stream_hit(bool sparse) { return FASTED_KNOB("FASTED_STREAM_HIT", sparse ? 2 : 0) == 2; }

const char* join_tc_kernel_name(int64_t d_pad, int64_t rows, int64_t cols, bool low_output,
                                bool sparse) {
    int cg = 0;
    switch (tc_variant(d_pad, rows, cols, low_output, &cg)) {
        case TC_RESIDENT:
            if (cg == 2 && FASTED_KNOB("FASTED_RES_EPI", 16) == 16 && res_hit(sparse))
                return "fasted::tc::join_tc_res_kernel<2> + 2 hit warps";
            return cg == 2 ? "fasted::tc::join_tc_res_kernel<2>" : "fasted::tc::join_tc_res_kernel<1>";
        case TC_MULTICAST:
            if (FASTED_KNOB("FASTED_MC_EPI", 16) == 16 && mc_hit(sparse))
                return "fasted::tc::join_tc_mc_kernel + 2 hit warps";
            return "fasted::tc::join_tc_mc_kernel";
        default:
            if (cg == 2 && FASTED_KNOB("FASTED_STREAM_EPI", 16) == 16 && stream_hit(sparse))
                return "fasted::tc::join_tc_kernel<2> + 2 hit warps";
            return cg == 2 ? "fasted::tc::join_tc_kernel<2>" : "fasted::tc::join_tc_kernel<1>";
    }
}

#ifdef FASTED_EXPERIMENTS
// TMEM-A launch (d_pad <= 128, CTA pair).
static cudaError_t launch_ts(const __half* X, const CUtensorMap& mxb, const CUtensorMap& ma,
                             const CUtensorMap& mbb, const JoinArgs& a, cudaStream_t s) {
    using namespace tc;
    constexpr int SMEM_MAX = 227 * 1024;
    auto kern = join_tc_ts_kernel;
    static PerDeviceOnce attr_once;
    {
        cudaError_t e = attr_once.run([&] {
            return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        SMEM_MAX);
        });
        if (e != cudaSuccess) return e;
    }
    ResSched sch;
    sch.epi_sleep_ns = 0u;
    sch.mma_spin = 0;
    sch.order = 0;
    sch.nkb = (int)((a.d_pad + BK - 1) / BK);
    sch.na = 2;
    sch.a_buf_bytes = 0;
    const int wst = TS_NEPI * 2 * TS_WSTAGE * 16;
    const int fixed = 2 * 4096 + TS_BAR_REGION + wst + 1024;
    sch.stages = (SMEM_MAX - fixed) / TS_STAGE_BYTES;
    if (sch.stages > TS_MAX_STAGES) sch.stages = TS_MAX_STAGES;
    sch.row_tiles = (int)((a.row_end - a.row_begin + 2 * BM - 1) / (2 * BM));
    sch.col_tiles = (int)((a.col_end - a.col_begin + TS_TBN - 1) / TS_TBN);
    int seg = FASTED_KNOB("FASTED_SEG_TILES", 16384 / TS_TBN);
    if (seg < 1) seg = 1;
    sch.nsegs = (sch.col_tiles + seg - 1) / seg;
    sch.units = (int64_t)sch.row_tiles * sch.nsegs;
    const int smem = fixed + sch.stages * TS_STAGE_BYTES;
    const int64_t slots = sm_count_current() / 2;
    const int64_t work = sch.units < slots ? sch.units : slots;
    if (work <= 0) return cudaSuccess;
    sch.lanes = (int)work;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(work * 2));
    cfg.blockDim = dim3(TS_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, reinterpret_cast<const uint4*>(X), mxb, ma, mbb, a, sch);
}
#endif  // FASTED_EXPERIMENTS

int launch_join_tc(const __half* X, const JoinArgs& a, cudaStream_t s) {
    using namespace tc;
    if ((a.d_pad % 8) != 0 || (reinterpret_cast<uintptr_t>(X) & 15u) != 0) {
        set_error("join_tc: d_pad must be a multiple of 8 and X 16-byte aligned");
        return FASTED_ERR_ARGUMENT;
    }
    if (a.n_pad > 0x7fffffffLL) {
        set_error("join_tc: n_pad exceeds TMA int32 coordinates");
        return FASTED_ERR_ARGUMENT;
    }
    // Variant choice (profiles/round1/tune_*.txt, measured on B200):
    //   d_pad <= 512: resident-A CTA pair (join_tc_res_kernel; 1M x 128:
    //                 1013 TFLOPS vs 693 for the streaming pair);
    //   d_pad >  256: B-multicast clusters of single-CTA MMAs
    //                 (join_tc_mc_kernel; 1M x 960: 1374 vs 1226 single-CTA
    //                 and ~980 for the CTA pair, which at the 1 kW cap runs
    //                 its clock down to ~920 MHz; 60K x 512: 1373 vs 1307).
    //   d_pad >  512, >= 2^36 examined pairs, LOW_OUTPUT hint: the streaming
    //                 CTA pair with a 16K-row raster (C4: 1376-1415 TFLOPS).
    // (libfasted_exp.so: FASTED_CTA_GROUP=1|2 forces the streaming kernel.)
    int cg = 1;
    const int variant = tc_variant(a.d_pad, a.row_end - a.row_begin, a.col_end - a.col_begin,
                                   a.low_output != 0, &cg);
    // per-call scratch (stream ordered): augment rows (two [n_pad][8] FP32,
    // eps-dependent) and the tensor-core Gram diagonal
    float4* aug = nullptr;
    // (+ 256 bytes: the resident kernel's pacing counter)
    const size_t aug_bytes = (size_t)a.n_pad * 64 + (size_t)a.n_pad * 4 + 256;
    // The per-call scratch comes from the device's default stream-ordered pool.
    // Its release threshold defaults to 0, so every synchronisation handed the
    // freed scratch back to the driver and the next call's cudaMallocAsync
    // mapped it again, on the timed path (60K x 512: 2.5-4 ms per 2.5 ms join
    // from one launch to the next).  Keep up to 1 GiB cached in the pool.
    static PerDeviceOnce pool_once;
    pool_once.run([] {
        int dev = 0;
        cudaMemPool_t pool;
        cudaError_t r = cudaGetDevice(&dev);
        if (r == cudaSuccess) r = cudaDeviceGetDefaultMemPool(&pool, dev);
        if (r == cudaSuccess && FASTED_KNOB("FASTED_POOL_KEEP", 1) != 0) {
            uint64_t keep = 1ull << 30;
            r = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        (void)cudaGetLastError();
        return cudaSuccess;
    });
    cudaError_t e = cudaMallocAsync(&aug, aug_bytes, s);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(augment rows)");
    float4* aug_a = aug;
    float4* aug_b = aug + 2 * a.n_pad;
    float* gram = reinterpret_cast<float*>(aug + 4 * a.n_pad);
    // Norms for the augment rows: the tensor core's own a_ii (Gram-diagonal
    // pre-pass, ~1/(n/128) of the join's work), so the norm terms carry the
    // same accumulation error as a_ij and cancel in d2 = a_ii + a_jj - 2 a_ij
    // (the reference's RZ norms paired with tensor-core a_ij bias d2 low by
    // ~2e-3 relative at d = 960, twice the 1e-3 band -- measured as a 0.43% vs
    // 0.14% Eq. 3 loss -- so they are never used here).  It also makes exact
    // duplicates distance 0, as in the reference.
    CUtensorMap mx, ma, mb;
    int st = encode_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, X, a.d_pad, a.n_pad, a.d_pad * 2, BK,
                       BM, CU_TENSOR_MAP_SWIZZLE_128B);
    if (st == FASTED_OK)
        st = encode_2d(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, aug_a, AUG_K, a.n_pad, AUG_ROW_BYTES,
                       AUG_K, BM, CU_TENSOR_MAP_SWIZZLE_32B);
    if (st == FASTED_OK)
        st = encode_2d(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, aug_b, AUG_K, a.n_pad, AUG_ROW_BYTES,
                       AUG_K, BM, CU_TENSOR_MAP_SWIZZLE_32B);
    if (st != FASTED_OK) {
        cudaFreeAsync(aug, s);
        return st;
    }
    // Both steps cover only the rows the join reads: [row_begin, row_end) and
    // [col_begin, col_end) (one range when they meet), so a launch needs just
    // those rows resident (FASTED_JOIN_APPEND column segments run while the
    // rest of the dataset is still being copied).
    int64_t rg[2][2] = {{a.row_begin, a.row_end}, {a.col_begin, a.col_end}};
    int nrg = 2;
    if (rg[1][0] <= rg[0][1] && rg[0][0] <= rg[1][1]) {
        rg[0][0] = rg[0][0] < rg[1][0] ? rg[0][0] : rg[1][0];
        rg[0][1] = rg[0][1] > rg[1][1] ? rg[0][1] : rg[1][1];
        nrg = 1;
    }
    for (int g = 0; g < nrg; g++) {
        const int64_t lo = rg[g][0], hi = rg[g][1];
        if (hi <= lo) continue;
        JoinArgs ad = a;
        ad.row_begin = lo;
        ad.row_end = hi;
        ad.col_begin = lo;
        ad.col_end = hi;
        ad.count_only = 1;
        ad.capacity = 0;
        ad.diag_flags = 0;
        ad.symmetric = 0;
        ad.trace = nullptr;
        ad.gram_diag = gram;
        Sched sd;
        sd.row_tiles = (int)((hi - lo + BM - 1) / BM);
        sd.col_tiles = 1;
        sd.group = 1;
        sd.nkb = (int)((a.d_pad + BK - 1) / BK);
        sd.total = sd.row_tiles;
        sd.diag = 1;
        sd.mma_spin = FASTED_KNOB("FASTED_MMA_SPIN", MMA_SPIN_DEFAULT);
        e = launch_variant<1, true>(mx, ma, mb, ad, sd, s);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) {
            cudaFreeAsync(aug, s);
            return cuda_status(e, "join_tc_kernel (Gram diagonal)");
        }
        aug_prepare_kernel<<<(unsigned)((hi - lo + 255) / 256), 256, 0, s>>>(gram, lo, hi,
                                                                             a.eps_sq, aug_a, aug_b);
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            cudaFreeAsync(aug, s);
            return cuda_status(e, "aug_prepare_kernel");
        }
    }
    // Resident-A form for d_pad <= 512: CTA pair, 256-column tiles, two
    // accumulators, 16 epilogue warps of 64 columns each plus, on the
    // caller's SPARSE hint, two hit warps that own the rare path and the
    // record writers (1M x 128, alternating launches: 225 vs 258 ms median).
    // Measured alternatives kept in libfasted_exp.so: 8 epilogue warps of 128
    // columns (269-319 vs 254 ms at 1M x 128, profiles/round1/
    // tune_c3_epi_ab_session2.txt); 128-column tiles with four accumulators
    // (372 vs 283 ms: the N=128 MMAs re-read A every 64 cycles); A in TMEM
    // (286-296 vs 256 ms).
    // the pacing counter (resident kernel; streaming kernel on FASTED_STREAM_PACE_W)
    unsigned long long* pace = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(aug) + aug_bytes - 256);
    cudaMemsetAsync(pace, 0, 8, s);
    JoinArgs ar = a;
    ar.pace = pace;
    if (variant == TC_RESIDENT) {
#ifdef FASTED_EXPERIMENTS
        const bool ts = cg == 2 && a.d_pad <= 128 && FASTED_KNOB("FASTED_TS", 0) != 0;
#else
        constexpr bool ts = false;
#endif
        const int tbn = ts ? 128 : 256;
        const int nb = tbn / cg, bbox = nb < 128 ? nb : 128;
        CUtensorMap mxb, mbb;
        st = encode_2d(&mxb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, X, a.d_pad, a.n_pad, a.d_pad * 2,
                       BK, bbox, CU_TENSOR_MAP_SWIZZLE_128B);
        if (st == FASTED_OK)
            st = encode_2d(&mbb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, aug_b, AUG_K, a.n_pad,
                           AUG_ROW_BYTES, AUG_K, bbox, CU_TENSOR_MAP_SWIZZLE_32B);
        if (st != FASTED_OK) {
            cudaFreeAsync(aug, s);
            return st;
        }
#ifdef FASTED_EXPERIMENTS
        if (ts)
            e = launch_ts(X, mxb, ma, mbb, a, s);
        else if (cg == 1)
            e = launch_res<1, 256, 8>(mx, mxb, ma, mbb, ar, s);
        else if (FASTED_KNOB("FASTED_RES_EPI", 16) != 16)
            e = launch_res<2, 256, 8>(mx, mxb, ma, mbb, ar, s);
        else if (FASTED_KNOB("FASTED_RES_DIRECT", 0) != 0)
            e = launch_res<2, 256, 16, -1>(mx, mxb, ma, mbb, ar, s);
        else if (FASTED_KNOB("FASTED_RES_HIT", 0) == RING_NHIT)
            e = launch_res<2, 256, 16, RING_NHIT>(mx, mxb, ma, mbb, ar, s);
        else
#endif
            e = res_hit(a.sparse != 0) ? launch_res<2, 256, 16, 2>(mx, mxb, ma, mbb, ar, s)
                                       : launch_res<2, 256, 16>(mx, mxb, ma, mbb, ar, s);
        if (e == cudaSuccess) e = cudaGetLastError();
        cudaFreeAsync(aug, s);
        if (e != cudaSuccess) return cuda_status(e, "join_tc_res_kernel");
        return FASTED_OK;
    }
    // d_pad > 512: B-multicast clusters of single-CTA MMAs, 16 epilogue warps
    // of 64 columns (alternating runs against 8 of 128: 60K x 512 2.63-2.67
    // vs 2.94-3.55 ms; 1M x 960 1406-1431 vs 1506-1515 ms; 5M x 384 shard at
    // S ~ 4000 2535 vs 3140 ms, profiles/round1/tune_mepi_session2.txt).
    if (variant == TC_MULTICAST) {
#ifdef FASTED_EXPERIMENTS
        if (FASTED_KNOB("FASTED_MC_EPI", 16) == 8)
            e = launch_mc<8>(mx, ma, mb, ar, s);
        else
#endif
            e = mc_hit(a.sparse != 0) ? launch_mc<16, 2>(mx, ma, mb, ar, s)
                                      : launch_mc<16>(mx, ma, mb, ar, s);
        if (e == cudaSuccess) e = cudaGetLastError();
        cudaFreeAsync(aug, s);
        if (e != cudaSuccess) return cuda_status(e, "join_tc_mc_kernel");
        return FASTED_OK;
    }
    Sched sch;
    sch.diag = 0;
    sch.mma_spin = FASTED_KNOB("FASTED_MMA_SPIN", MMA_SPIN_DEFAULT);
    const int tile_m = BM * cg;
    sch.row_tiles = (int)((a.row_end - a.row_begin + tile_m - 1) / tile_m);
    sch.col_tiles = (int)((a.col_end - a.col_begin + BN - 1) / BN);
    // grouped raster: GROUP row tiles sweep all columns.  CTA pair: 16384
    // rows -- 1376 TFLOPS vs 1331 for 8192, 1031 for 2048 and 1246 for 32768
    // at 1M x 960 (profiles/round1/tune_c4_cg2b_session2.txt); single CTA
    // (libfasted_exp.so only): 2048 rows, 0.82 vs 0.93 pJ/flop for 8192.
    sch.group = FASTED_KNOB("FASTED_GROUP_ROWS", cg == 2 ? 16384 : 2048) / tile_m;
    if (sch.group < 1) sch.group = 1;
    sch.nkb = (int)((a.d_pad + BK - 1) / BK);
    sch.total = (int64_t)sch.row_tiles * sch.col_tiles;
    // pacing, one block of 64 tile layers (C4 on a box whose pairs drifted: HBM reads
    // 5.45 TB -> 121 GB per launch, L2 hit 59 -> 98%, 1738 -> 1327 ms; profiles/round2/
    // stream_pacing_ab.txt)
    sch.pace_w = (cg == 2 && ar.pace) ? FASTED_KNOB("FASTED_STREAM_PACE_W", 1) : 0;
    // CTA pair: 16 epilogue warps of 64 columns (8 of 128: 1M x 960
    // 1466-1472 vs 1450-1491 TFLOPS, even; 5M x 384 shard at S <= 64:
    // 1917-1946 vs 2060-2253 ms, profiles/round1/tune_sepi_session2.txt)
#ifdef FASTED_EXPERIMENTS
    if (cg == 1)
        e = launch_variant<1>(mx, ma, mb, ar, sch, s);
    else if (FASTED_KNOB("FASTED_STREAM_EPI", 16) == 8)
        e = launch_variant<2>(mx, ma, mb, ar, sch, s);
    else
#endif
        e = stream_hit(a.sparse != 0) ? launch_variant<2, false, 16, 2>(mx, ma, mb, ar, sch, s)
                                      : launch_variant<2, false, 16>(mx, ma, mb, ar, sch, s);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaFreeAsync(aug, s);
    if (e != cudaSuccess) return cuda_status(e, "join_tc_kernel");
    return FASTED_OK;
}

}  // namespace fasted
