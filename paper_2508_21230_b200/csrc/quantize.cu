// Kernel 1: FP32 -> FP16 (RNE) quantisation, zero padding and RZ squared
// norms -- the GPU to_half (reference dataset.py:164-193 with
// _kernel.squared_norms_rz, _kernel.py:79-93).
//
// HBM-bound: reads n*d*4 bytes, writes n_pad*d_pad*2 + n_pad*4 bytes.
// The norm of a row is ONE sequential chain of __fmaf_rz(v, v, acc) in
// ascending k -- the exact op sequence of the reference (product exact in
// FP32, RZ add) -- so one thread owns one row and the data movement is what
// has to be fast.
//
// quantize_tma_kernel (rows of 16-byte multiple pitch, d % 4 == 0): a CTA
// owns 128 rows; 128 x 32 FP32 boxes stream into a QSTAGES-deep shared-memory
// ring by TMA (SWIZZLE_128B: thread t reads its row's 16-byte chunks
// j ^ (t % 8), conflict free), each thread casts and chains its row's 32
// values and writes the FP16 row segment to a padded staging tile, which the
// CTA then stores coalesced.  The loads of chunks c+1..c+QSTAGES-1 are in
// flight while chunk c is chained, so the stream never waits on the chain.
// quantize_kernel (any d): the earlier form -- coalesced register loads of
// a 128 x 32 block, a widened copy in shared memory, then the chains.
#include "common.cuh"

namespace fasted {

constexpr int QROWS = 128;
constexpr int QCOLS = 32;
constexpr int QSTAGES = 4;
constexpr int QIN_BYTES = QROWS * QCOLS * 4;          // one FP32 box, 16 KB
constexpr int QOUT_PITCH = QCOLS * 2 + 16;            // FP16 row segment + pad, 80 B
constexpr int QOUT_BYTES = QROWS * QOUT_PITCH;        // 10 KB
constexpr int QSMEM = 1024 + QSTAGES * QIN_BYTES + 2 * QOUT_BYTES + 64;

__device__ __forceinline__ uint32_t q_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void q_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void q_load(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                       int c1) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)QIN_BYTES)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

__global__ void __launch_bounds__(QROWS)
quantize_tma_kernel(const __grid_constant__ CUtensorMap tmap, int64_t n, int64_t d,
                    __half* __restrict__ out, int64_t n_pad, int64_t d_pad,
                    float* __restrict__ norms, unsigned long long* __restrict__ first_overflow) {
    extern __shared__ uint8_t q_raw[];
    const uint32_t raw = q_smem(q_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;          // SWIZZLE_128B: 1 KB aligned
    uint8_t* const gbase = q_raw + (base - raw);
    const uint32_t sin = base;
    uint8_t* const sout = gbase + QSTAGES * QIN_BYTES;
    const uint32_t bars = base + QSTAGES * QIN_BYTES + 2 * QOUT_BYTES;
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * QROWS;
    const int nch = (int)((d_pad + QCOLS - 1) / QCOLS);
    if (t == 0) {
        for (int s = 0; s < QSTAGES; s++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8u * s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap))
                     : "memory");
    }
    __syncthreads();
    if (t == 0)
        for (int s = 0; s < QSTAGES && s < nch; s++)
            q_load(sin + s * QIN_BYTES, &tmap, bars + 8u * s, s * QCOLS, (int)r0);
    const int64_t r = r0 + t;
    const bool row_in = r < n;
    const uint32_t sw = (uint32_t)(t & 7);
    float acc = 0.0f;
    for (int c = 0; c < nch; c++) {
        const int s = c % QSTAGES;
        q_wait(bars + 8u * s, (uint32_t)(c / QSTAGES) & 1u);
        const int64_t k0 = (int64_t)c * QCOLS;
        uint8_t* const orow = sout + (c & 1) * QOUT_BYTES + t * QOUT_PITCH;
        const uint8_t* const irow = gbase + s * QIN_BYTES + t * 128;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const float4 v = *reinterpret_cast<const float4*>(irow + ((j ^ sw) << 4));
            const __half h0 = __float2half_rn(v.x), h1 = __float2half_rn(v.y);
            const __half h2 = __float2half_rn(v.z), h3 = __float2half_rn(v.w);
            if (row_in && (__hisinf(h0) || __hisinf(h1) || __hisinf(h2) || __hisinf(h3))) {
                const int e = __hisinf(h0) ? 0 : __hisinf(h1) ? 1 : __hisinf(h2) ? 2 : 3;
                atomicMin(first_overflow, (unsigned long long)(r * d + k0 + 4 * j + e));
            }
            const float w0 = __half2float(h0), w1 = __half2float(h1);
            const float w2 = __half2float(h2), w3 = __half2float(h3);
            acc = __fmaf_rz(w0, w0, acc);   // RZ(acc + v*v), v*v exact; columns past
            acc = __fmaf_rz(w1, w1, acc);   // d_pad are TMA zero fill: RZ(acc + 0) == acc
            acc = __fmaf_rz(w2, w2, acc);
            acc = __fmaf_rz(w3, w3, acc);
            __half2 p0 = __halves2half2(h0, h1), p1 = __halves2half2(h2, h3);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&p0);
            pk.y = *reinterpret_cast<uint32_t*>(&p1);
            *reinterpret_cast<uint2*>(orow + 8 * j) = pk;
        }
        __syncthreads();   // stage s consumed by every thread; FP16 tile complete
        if (t == 0 && c + QSTAGES < nch)
            q_load(sin + s * QIN_BYTES, &tmap, bars + 8u * s, (c + QSTAGES) * QCOLS, (int)r0);
        // coalesced store of the 128 x 32 FP16 tile: 4 threads per row, 16 B each
        const uint8_t* const tile = sout + (c & 1) * QOUT_BYTES;
        const int64_t kcols = d_pad - k0 < QCOLS ? d_pad - k0 : QCOLS;   // multiple of 8
#pragma unroll
        for (int it = 0; it < 4; it++) {
            const int idx = it * QROWS + t;
            const int rl = idx >> 2, q = idx & 3;
            const int64_t rr = r0 + rl;
            if (rr < n_pad && 8 * q < kcols)
                *reinterpret_cast<uint4*>(out + rr * d_pad + k0 + 8 * q) =
                    *reinterpret_cast<const uint4*>(tile + rl * QOUT_PITCH + 16 * q);
        }
    }
    if (r < n_pad) norms[r] = acc;
}

__global__ void __launch_bounds__(QROWS)
quantize_kernel(const float* __restrict__ x, int64_t n, int64_t d, __half* __restrict__ out,
                int64_t n_pad, int64_t d_pad, float* __restrict__ norms,
                unsigned long long* __restrict__ first_overflow) {
    __shared__ float tile[QROWS][QCOLS + 1];
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * QROWS;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < d_pad; k0 += QCOLS) {
        // load + cast + store: element e of this thread is (row e*4 + t/32, col t%32)
#pragma unroll 8
        for (int e = 0; e < QROWS * QCOLS / QROWS; e++) {
            const int rl = e * (QROWS / QCOLS) + t / QCOLS;
            const int cl = t % QCOLS;
            const int64_t r = r0 + rl, k = k0 + cl;
            __half h = __float2half_rn(0.0f);
            if (r < n && k < d) {
                const float v = x[r * d + k];
                h = __float2half_rn(v);
                if (__hisinf(h)) atomicMin(first_overflow, (unsigned long long)(r * d + k));
            }
            if (r < n_pad && k < d_pad) out[r * d_pad + k] = h;
            tile[rl][cl] = __half2float(h);
        }
        __syncthreads();
        const int kmax = (int)((d_pad - k0) < QCOLS ? (d_pad - k0) : QCOLS);
        for (int c = 0; c < kmax; c++) {
            const float v = tile[t][c];
            acc = __fmaf_rz(v, v, acc);   // RZ(acc + v*v), v*v exact
        }
        __syncthreads();
    }
    if (r0 + t < n_pad) norms[r0 + t] = acc;
}

// Norms of an already-quantised matrix (compute_squared_norms).
__global__ void __launch_bounds__(QROWS)
norms_kernel(const __half* __restrict__ v16, int64_t n_pad, int64_t d_pad,
             float* __restrict__ norms) {
    __shared__ float tile[QROWS][QCOLS + 1];
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * QROWS;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < d_pad; k0 += QCOLS) {
#pragma unroll 8
        for (int e = 0; e < QCOLS; e++) {
            const int rl = e * (QROWS / QCOLS) + t / QCOLS;
            const int cl = t % QCOLS;
            const int64_t r = r0 + rl, k = k0 + cl;
            tile[rl][cl] = (r < n_pad && k < d_pad) ? __half2float(v16[r * d_pad + k]) : 0.0f;
        }
        __syncthreads();
        const int kmax = (int)((d_pad - k0) < QCOLS ? (d_pad - k0) : QCOLS);
        for (int c = 0; c < kmax; c++) {
            const float v = tile[t][c];
            acc = __fmaf_rz(v, v, acc);
        }
        __syncthreads();
    }
    if (r0 + t < n_pad) norms[r0 + t] = acc;
}

}  // namespace fasted

using namespace fasted;

// Stream-ordered quantise: no allocation, no synchronisation.  The caller
// initialises *first_overflow_dev to ~0 (all ones) before the launch; the
// kernel atomicMin's the flat index of every overflowing value into it.
extern "C" int fasted_quantize_async(const float* x, int64_t n, int64_t d, uint16_t* values16,
                                     int64_t n_pad, int64_t d_pad, float* norms,
                                     unsigned long long* first_overflow_dev, void* stream) {
    if (!x || !values16 || !norms || !first_overflow_dev || n < 1 || d < 1 || n_pad < n ||
        d_pad < d || (d_pad % 8) != 0) {
        set_error("fasted_quantize: bad arguments (n=%lld d=%lld n_pad=%lld d_pad=%lld)",
                  (long long)n, (long long)d, (long long)n_pad, (long long)d_pad);
        return FASTED_ERR_ARGUMENT;
    }
    cudaStream_t s = as_stream(stream);
    const int64_t blocks = (n_pad + QROWS - 1) / QROWS;
    // TMA form: 16-byte row pitch and base, 16-byte aligned output rows
    const bool tma = (d % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(values16) & 15u) == 0 && n <= 0x7fffffffLL;
    CUtensorMap map;
    if (tma && encode_2d(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, x, (uint64_t)d, (uint64_t)n,
                         (uint64_t)d * 4, QCOLS, QROWS, CU_TENSOR_MAP_SWIZZLE_128B) == FASTED_OK) {
        static PerDeviceOnce attr_once;
        cudaError_t e = attr_once.run([&] {
            return cudaFuncSetAttribute(quantize_tma_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, QSMEM);
        });
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(quantize)");
        quantize_tma_kernel<<<(unsigned)blocks, QROWS, QSMEM, s>>>(
            map, n, d, reinterpret_cast<__half*>(values16), n_pad, d_pad, norms,
            first_overflow_dev);
        FASTED_CHECK_LAUNCH("quantize_tma_kernel");
    } else {
        quantize_kernel<<<(unsigned)blocks, QROWS, 0, s>>>(
            x, n, d, reinterpret_cast<__half*>(values16), n_pad, d_pad, norms,
            first_overflow_dev);
        FASTED_CHECK_LAUNCH("quantize_kernel");
    }
    return FASTED_OK;
}

extern "C" int fasted_quantize(const float* x, int64_t n, int64_t d, uint16_t* values16,
                               int64_t n_pad, int64_t d_pad, float* norms,
                               int64_t* first_overflow_host, void* stream) {
    if (first_overflow_host) *first_overflow_host = -1;
    if (!x || !values16 || !norms || n < 1 || d < 1 || n_pad < n || d_pad < d ||
        (d_pad % 8) != 0) {
        set_error("fasted_quantize: bad arguments (n=%lld d=%lld n_pad=%lld d_pad=%lld)",
                  (long long)n, (long long)d, (long long)n_pad, (long long)d_pad);
        return FASTED_ERR_ARGUMENT;
    }
    cudaStream_t s = as_stream(stream);
    unsigned long long* flag = nullptr;
    cudaError_t e = cudaMallocAsync(&flag, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(overflow flag)");
    cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), s);
    const int st = fasted_quantize_async(x, n, d, values16, n_pad, d_pad, norms, flag, stream);
    if (st != FASTED_OK) {
        cudaFreeAsync(flag, s);
        return st;
    }
    unsigned long long h = ~0ull;
    cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(flag, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "quantize sync");
    if (h != ~0ull) {
        if (first_overflow_host) *first_overflow_host = (int64_t)h;
        set_error("FP16 overflow at flat index %llu", h);
        return FASTED_ERR_RANGE;
    }
    return FASTED_OK;
}

extern "C" int fasted_norms(const uint16_t* values16, int64_t n_pad, int64_t d_pad, float* norms,
                            void* stream) {
    if (!values16 || !norms || n_pad < 1 || d_pad < 1) {
        set_error("fasted_norms: bad arguments");
        return FASTED_ERR_ARGUMENT;
    }
    const int64_t blocks = (n_pad + QROWS - 1) / QROWS;
    norms_kernel<<<(unsigned)blocks, QROWS, 0, as_stream(stream)>>>(
        reinterpret_cast<const __half*>(values16), n_pad, d_pad, norms);
    FASTED_CHECK_LAUNCH("norms_kernel");
    return FASTED_OK;
}
