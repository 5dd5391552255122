// FP64 ground truth for sampled query rows -- the GPU form of the
// reference's accuracy oracle (oracle.py:26-64: pairwise_sqdist_fp64 +
// brute_force_fp64), used to report pair accuracy against FP64 (Eq. 3,
// PAPER.md) at sizes where the CPU oracle cannot run (it took 324 s at
// 16K x 128).
//
// Per (query row q, point j): acc = 0; for k ascending: t = x_qk - x_jk
// (FP64), acc = RN(acc + RN(t * t)) -- numpy's `acc += t * t` order, no FMA
// contraction -- and the pair is kept iff sqrt(acc) <= eps in FP64.  Input
// is the ORIGINAL FP32 dataset (not the FP16 copy), as in the reference.
//
// CUDA-core FP64 kernel: a CTA owns 16 query rows x 128 points; k runs in
// 32-wide slabs staged (widened to FP64) in shared memory; each thread keeps
// 2 x 4 FP64 accumulators.
#include "common.cuh"

namespace fasted {

constexpr int F_Q = 16, F_J = 128, F_K = 32, F_THREADS = 256;

__global__ void __launch_bounds__(F_THREADS)
fp64_rows_kernel(const float* __restrict__ x, int64_t n, int64_t d,
                 const int64_t* __restrict__ qrows, int64_t nq, double eps,
                 uint4* __restrict__ out, unsigned long long capacity,
                 unsigned long long* __restrict__ count) {
    __shared__ double Qs[F_K][F_Q + 1];
    __shared__ double Xs[F_K][F_J + 1];
    const int t = threadIdx.x;
    const int tq = t / 32;          // 0..7 -> query rows tq*2 .. tq*2+1
    const int tj = t % 32;          // 0..31 -> points tj + 32*c, c < 4
    const int64_t q0 = (int64_t)blockIdx.y * F_Q;
    const int64_t j0 = (int64_t)blockIdx.x * F_J;
    double acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[a][c] = 0.0;
    for (int64_t k0 = 0; k0 < d; k0 += F_K) {
        // stage query slab [F_Q x F_K] and point slab [F_J x F_K] (transposed)
        for (int e = t; e < F_Q * F_K; e += F_THREADS) {
            const int qi = e / F_K, kk = e % F_K;
            const int64_t q = q0 + qi, k = k0 + kk;
            Qs[kk][qi] = (q < nq && k < d) ? (double)x[qrows[q] * d + k] : 0.0;
        }
        for (int e = t; e < F_J * F_K; e += F_THREADS) {
            const int ji = e / F_K, kk = e % F_K;
            const int64_t j = j0 + ji, k = k0 + kk;
            Xs[kk][ji] = (j < n && k < d) ? (double)x[j * d + k] : 0.0;
        }
        __syncthreads();
        const int kmax = (int)((d - k0) < F_K ? (d - k0) : F_K);
        for (int kk = 0; kk < kmax; kk++) {
            const double qa = Qs[kk][tq * 2], qb = Qs[kk][tq * 2 + 1];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const double xv = Xs[kk][tj + 32 * c];
                const double ta = __dsub_rn(qa, xv), tb = __dsub_rn(qb, xv);
                acc[0][c] = __dadd_rn(acc[0][c], __dmul_rn(ta, ta));
                acc[1][c] = __dadd_rn(acc[1][c], __dmul_rn(tb, tb));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 2; a++) {
        const int64_t q = q0 + tq * 2 + a;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int64_t j = j0 + tj + 32 * c;
            if (q < nq && j < n && __dsqrt_rn(acc[a][c]) <= eps) {
                const unsigned long long p = atomicAdd(count, 1ull);
                if (p < capacity) {
                    const unsigned long long bits = (unsigned long long)__double_as_longlong(acc[a][c]);
                    out[p] = make_uint4((uint32_t)(qrows[q] + 1), (uint32_t)(j + 1),
                                        (uint32_t)bits, (uint32_t)(bits >> 32));
                }
            }
        }
    }
}

}  // namespace fasted

using namespace fasted;

extern "C" int fasted_fp64_rows(const float* x, int64_t n, int64_t d, const int64_t* qrows,
                                int64_t nq, double epsilon, void* out_records,
                                uint64_t capacity, unsigned long long* count, void* stream) {
    if (!x || !qrows || !count || n < 1 || d < 1 || nq < 0 || !(epsilon >= 0.0) ||
        (capacity > 0 && !out_records)) {
        set_error("fasted_fp64_rows: bad arguments");
        return FASTED_ERR_ARGUMENT;
    }
    cudaStream_t s = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(count)");
    if (nq == 0) return FASTED_OK;
    dim3 grid((unsigned)((n + F_J - 1) / F_J), (unsigned)((nq + F_Q - 1) / F_Q));
    fp64_rows_kernel<<<grid, F_THREADS, 0, s>>>(x, n, d, qrows, nq, epsilon,
                                                reinterpret_cast<uint4*>(out_records), capacity,
                                                count);
    FASTED_CHECK_LAUNCH("fp64_rows_kernel");
    return FASTED_OK;
}
