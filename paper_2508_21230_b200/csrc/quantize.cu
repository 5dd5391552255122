// Kernel 1: FP32 -> FP16 (RNE) quantisation, zero padding and RZ squared
// norms -- the GPU to_half (reference dataset.py:164-193 with
// _kernel.squared_norms_rz, _kernel.py:79-93).
//
// HBM-bound: reads n*d*4 bytes, writes n_pad*d_pad*2 + n_pad*4 bytes.
// A CTA owns 128 rows.  Per 32-column chunk the 128x32 FP32 block is read
// with warp-contiguous (coalesced) loads, cast, written back as FP16, and
// staged widened in shared memory (row pitch 33 words: conflict free) so
// each thread can run its row's norm as one sequential chain of
// __fmaf_rz(v, v, acc) -- the exact op sequence of the reference
// (product exact in FP32, RZ add, ascending k).
#include "common.cuh"

namespace fasted {

constexpr int QROWS = 128;
constexpr int QCOLS = 32;

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
    const int64_t blocks = (n_pad + QROWS - 1) / QROWS;
    quantize_kernel<<<(unsigned)blocks, QROWS, 0, s>>>(x, n, d, reinterpret_cast<__half*>(values16),
                                                      n_pad, d_pad, norms, flag);
    FASTED_CHECK_LAUNCH("quantize_kernel");
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
