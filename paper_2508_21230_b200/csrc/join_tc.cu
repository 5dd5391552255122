// Kernel 2 (the product path): fused tcgen05 epsilon join for sm_100a.
//
//   TMA (SWIZZLE_128B) -> 4-stage smem ring -> tcgen05.mma kind::f16
//   (M=128, N=256, K=16; FP32 accumulators in TMEM, double buffered: 2 x 256
//   columns) -> epilogue warps: tcgen05.ld -> ((-2a)+s_i)+s_j -> <= eps^2 ->
//   warp-ballot compaction with one global atomic per warp.
//
// The distance matrix never reaches HBM.  Replaces the reference's tile
// sweep (tiling.py:307-344): compute_block_tile (tiling.py:199-285),
// accumulate_panel (_kernel.py:57-76) and combine_distance (mma.py:143-157).
// Arithmetic differs from the reference only in how the tensor core sums
// the FP32 products of a_ij (the reference sums sequentially with RZ); the
// epilogue uses the reference's combine order and threshold.  Self pairs
// (i == j) are forced to distance 0, which is exactly what the reference
// produces (its a_ii and s_i are the same RZ chain).
//
// Persistent CTAs (one per SM, 384 threads):
//   warp 0      : TMA producer (one lane)
//   warp 1      : MMA issuer   (one lane)
//   warp 2      : TMEM allocator / deallocator
//   warp 3      : idle
//   warps 4..11 : epilogue; warp w reads TMEM lanes 32*(w%4).. and column
//                 half (w-4)/4 of the 256-column accumulator.
// Tiles are (128 rows x 256 columns) walked in a grouped raster: GROUP row
// blocks sweep every column tile together, so each 256-row B panel is read
// from HBM once per group and the group's A panels stay L2 resident.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "join_common.cuh"

namespace fasted {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;   // one 128-byte swizzle atom of FP16
constexpr int UK = 16;   // K of one kind::f16 tcgen05.mma
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int NUM_EPI_WARPS = 8;
constexpr int THREADS = 128 + NUM_EPI_WARPS * 32;
constexpr int TMEM_COLS = 2 * BN;
constexpr int BAR_BYTES = 256;
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + BAR_BYTES + 1024;
constexpr int GROUP = 16;

// Instruction descriptor, kind::f16: D=F32 (bits 4-5 = 1), A=B=F16 (0),
// both K-major (bits 15,16 = 0), N>>3 at bits 17-22, M>>4 at bits 24-28.
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

struct Sched {
    int row_blocks;
    int col_tiles;
    int group;
    int nkb;
    int64_t total;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
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

__device__ __forceinline__ uint64_t global_timer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin on an mbarrier phase; traps after 20 s so a protocol bug aborts the
// launch (cudaErrorLaunchFailure) instead of wedging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = global_timer();
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins == 2048u) {
            spins = 0;
            if (global_timer() - t0 > 20000000000ull) __trap();
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand, 128-byte swizzle: rows of 128 B, 8-row core groups
// 1024 B apart (SBO), LBO unused (1), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) |
           ((uint64_t)(1024u >> 4) << 32) | ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}

#define FASTED_R32(X)                                                                        \
    X[0], X[1], X[2], X[3], X[4], X[5], X[6], X[7], X[8], X[9], X[10], X[11], X[12], X[13],  \
        X[14], X[15], X[16], X[17], X[18], X[19], X[20], X[21], X[22], X[23], X[24], X[25], \
        X[26], X[27], X[28], X[29], X[30], X[31]

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

// Packed FP32x2 (sm_100): two IEEE RN ops per instruction.
__device__ __forceinline__ uint64_t pk(float x, float y) {
    return (uint64_t)__float_as_uint(x) | ((uint64_t)__float_as_uint(y) << 32);
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }

__device__ __forceinline__ void tile_coords(const Sched& s, int64_t t, int& rb, int& ct) {
    const int64_t per_group = (int64_t)s.group * s.col_tiles;
    const int64_t g = t / per_group;
    const int64_t r = t - g * per_group;
    const int64_t left = (int64_t)s.row_blocks - g * s.group;
    const int rows_in = (int)(left < s.group ? left : s.group);
    ct = (int)(r / rows_in);
    rb = (int)(g * s.group + r % rows_in);
}

__global__ void __launch_bounds__(THREADS, 1)
join_tc_kernel(const __grid_constant__ CUtensorMap tmap, const JoinArgs a, const Sched sch) {
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
    volatile uint32_t* slot_ptr =
        reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), NUM_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap))
                     : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         slot),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *slot_ptr;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < sch.total; t += gridDim.x) {
                int rb, ct;
                tile_coords(sch, t, rb, ct);
                const int row0 = (int)(a.row_begin + (int64_t)rb * BM);
                const int col0 = (int)(a.col_begin + (int64_t)ct * BN);
                const bool second = (int64_t)col0 + 128 < a.col_end;
                const uint32_t bytes = A_BYTES + (second ? B_BYTES : B_BYTES / 2);
                for (int kb = 0; kb < sch.nkb; kb++) {
                    mbar_wait(empty_bar(s), ph ^ 1u);
                    mbar_expect_tx(full_bar(s), bytes);
                    const int kx = kb * BK;
                    tma_load_2d(sA + s * A_BYTES, &tmap, full_bar(s), kx, row0);
                    tma_load_2d(sB + s * B_BYTES, &tmap, full_bar(s), kx, col0);
                    if (second)
                        tma_load_2d(sB + s * B_BYTES + B_BYTES / 2, &tmap, full_bar(s), kx,
                                    col0 + 128);
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            int lt = 0;
            for (int64_t t = blockIdx.x; t < sch.total; t += gridDim.x, ++lt) {
                const int buf = lt & 1;
                const uint32_t aph = (uint32_t)(lt >> 1) & 1u;
                mbar_wait(tempty_bar(buf), aph ^ 1u);
                tc_fence_after();
                const uint32_t dtm = tmem_base + (uint32_t)(buf * BN);
                for (int kb = 0; kb < sch.nkb; kb++) {
                    mbar_wait(full_bar(s), ph);
                    tc_fence_after();
                    const uint64_t ad = sw128_desc(sA + s * A_BYTES);
                    const uint64_t bd = sw128_desc(sB + s * B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / UK; kk++) {
                        const uint64_t koff = (uint64_t)((kk * UK * 2) >> 4);
                        mma_f16(dtm, ad + koff, bd + koff, (kb | kk) != 0 ? 1u : 0u);
                    }
                    mma_commit(empty_bar(s));
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                mma_commit(tfull_bar(buf));
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------- epilogue
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int h = (warp - 4) >> 2;   // column half of the 256-wide accumulator
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const float eps_sq = a.eps_sq;
        const uint64_t neg2 = pk(-2.0f, -2.0f);
        int lt = 0;
        for (int64_t t = blockIdx.x; t < sch.total; t += gridDim.x, ++lt) {
            int rb, ct;
            tile_coords(sch, t, rb, ct);
            const int64_t row0 = a.row_begin + (int64_t)rb * BM;
            const int64_t col0 = a.col_begin + (int64_t)ct * BN;
            const int64_t iw = row0 + q * 32;
            const int64_t i = iw + lane;
            const float si = __ldg(a.norms + i);
            const uint64_t si2 = pk(si, si);
            const bool row_ok = i < a.n_logical;
            const int buf = lt & 1;
            const uint32_t aph = (uint32_t)(lt >> 1) & 1u;
            mbar_wait(tfull_bar(buf), aph);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 4; c++) {
                const int64_t jb = col0 + h * 128 + c * 32;
                if (jb >= a.col_end) break;
                uint32_t r[32];
                tmem_ld32(tmem_base + lane_base + (uint32_t)(buf * BN + h * 128 + c * 32), r);
                tmem_ld_wait(r);
                const float4* sj4 = reinterpret_cast<const float4*>(a.norms + jb);
                bool hit = false;
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    const float4 s4 = __ldg(sj4 + (e >> 2));
                    uint64_t d01 = ffma2(pk(__uint_as_float(r[e]), __uint_as_float(r[e + 1])),
                                         neg2, si2);
                    uint64_t d23 = ffma2(pk(__uint_as_float(r[e + 2]), __uint_as_float(r[e + 3])),
                                         neg2, si2);
                    d01 = fadd2(d01, pk(s4.x, s4.y));
                    d23 = fadd2(d23, pk(s4.z, s4.w));
                    hit |= (lo_f(d01) <= eps_sq) | (hi_f(d01) <= eps_sq) |
                           (lo_f(d23) <= eps_sq) | (hi_f(d23) <= eps_sq);
                }
                const bool diag = (jb < iw + 32) && (iw < jb + 32);
                if (__any_sync(0xffffffffu, hit) || diag) {
                    uint32_t m = 0;
                    float dv[32];
#pragma unroll
                    for (int e = 0; e < 32; e++) {
                        const int64_t j = jb + e;
                        float d2 = combine_rn(__uint_as_float(r[e]), si, __ldg(a.norms + j));
                        if (i == j) d2 = 0.0f;
                        dv[e] = d2;
                        if (row_ok && j < a.n_logical && d2 <= eps_sq) m |= 1u << e;
                    }
                    const uint32_t cnt = __popc(m);
                    unsigned long long pos = warp_reserve(a.count, cnt);
                    if (!a.count_only) {
#pragma unroll
                        for (int e = 0; e < 32; e++) {
                            if (m & (1u << e)) {
                                if (pos < a.capacity) {
                                    a.out_i[pos] = (uint32_t)(i + 1);
                                    a.out_j[pos] = (uint32_t)(jb + e + 1);
                                    a.out_d[pos] = dv[e];
                                }
                                pos++;
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(buf));
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
    }
}

}  // namespace tc

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int launch_join_tc(const __half* X, const JoinArgs& a, cudaStream_t s) {
    using namespace tc;
    auto encode = tensor_map_encoder();
    if (!encode) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return FASTED_ERR_CUDA;
    }
    if ((a.d_pad % 8) != 0 || (reinterpret_cast<uintptr_t>(X) & 15u) != 0) {
        set_error("join_tc: d_pad must be a multiple of 8 and X 16-byte aligned");
        return FASTED_ERR_ARGUMENT;
    }
    if (a.n_pad > 0x7fffffffLL) {
        set_error("join_tc: n_pad exceeds TMA int32 coordinates");
        return FASTED_ERR_ARGUMENT;
    }
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)a.d_pad, (cuuint64_t)a.n_pad};
    cuuint64_t gstride[1] = {(cuuint64_t)a.d_pad * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
    cuuint32_t estride[2] = {1, 1};
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(X), gdim,
                         gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)cr);
        return FASTED_ERR_CUDA;
    }
    Sched sch;
    sch.row_blocks = (int)((a.row_end - a.row_begin) / BM);
    sch.col_tiles = (int)((a.col_end - a.col_begin + BN - 1) / BN);
    sch.group = GROUP;
    sch.nkb = (int)((a.d_pad + BK - 1) / BK);
    sch.total = (int64_t)sch.row_blocks * sch.col_tiles;
    if (sch.total <= 0) return FASTED_OK;
    const int sms = sm_count_current();
    const int64_t grid = sch.total < sms ? sch.total : sms;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(join_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             SMEM_BYTES);
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(join_tc_kernel)");
        attr_set = true;
    }
    join_tc_kernel<<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(map, a, sch);
    FASTED_CHECK_LAUNCH("join_tc_kernel");
    return FASTED_OK;
}

}  // namespace fasted
