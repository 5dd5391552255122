// Kernel 0: CUDA-core epsilon join that reproduces the reference BIT FOR BIT.
//
// Per pair, a_ij = RZ-sum over k ascending of exact FP32 products of the
// widened FP16 coordinates -- one __fmaf_rz(p, q, acc) per k, which is the
// reference's _rz_add(acc, p*q) (_kernel.py:39-54,66-70) because p*q is exact
// in FP32.  Epilogue ((-2a)+s_i)+s_j in RN, clamp, inclusive eps_sq test and
// index filter as tiling.py:273-285 / mma.py:143-157.  Self-distances come
// out exactly 0 with no special case (a_ii and s_i are the same RZ chain).
//
// Used for the parity tests (the sha256 of the C1 pair file must equal the
// reference's) and for self_join(..., mode="exact").  Not the product path:
// that is the tcgen05 kernel in join_tc.cu.
//
// Classic 128x128 CTA tile, 16-wide k slabs widened to FP32 in shared
// memory, 256 threads with an 8x8 register micro-tile each.
#include "common.cuh"
#include "join_common.cuh"

namespace fasted {

constexpr int EX_BM = 128, EX_BN = 128, EX_BK = 16, EX_THREADS = 256;

__global__ void __launch_bounds__(EX_THREADS)
join_exact_kernel(const __half* __restrict__ X, const JoinArgs a) {
    __shared__ float As[EX_BK][EX_BM + 4];
    __shared__ float Bs[EX_BK][EX_BN + 4];
    const int t = threadIdx.x;
    const int tx = t % 16, ty = t / 16;
    const int64_t n_row_tiles = (a.row_end - a.row_begin) / EX_BM;
    const int64_t n_col_tiles = (a.col_end - a.col_begin + EX_BN - 1) / EX_BN;
    const int64_t n_tiles = n_row_tiles * n_col_tiles;
    PairWriter wr;
    writer_init(wr);

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t row0 = a.row_begin + (tile / n_col_tiles) * EX_BM;
        const int64_t col0 = a.col_begin + (tile % n_col_tiles) * EX_BN;
        float acc[8][8];
#pragma unroll
        for (int r = 0; r < 8; r++)
#pragma unroll
            for (int c = 0; c < 8; c++) acc[r][c] = 0.0f;

        // loader: thread t stages 8 consecutive k of one row of A and of B
        const int lrow = t / 2, lk = (t % 2) * 8;
        for (int64_t k0 = 0; k0 < a.d_pad; k0 += EX_BK) {
            {
                const int64_t ra = row0 + lrow;
                const int64_t rb = col0 + lrow;
                uint4 va = make_uint4(0, 0, 0, 0), vb = make_uint4(0, 0, 0, 0);
                if (k0 + lk < a.d_pad) {
                    va = *reinterpret_cast<const uint4*>(X + ra * a.d_pad + k0 + lk);
                    if (rb < a.col_end)
                        vb = *reinterpret_cast<const uint4*>(X + rb * a.d_pad + k0 + lk);
                }
                const __half* ha = reinterpret_cast<const __half*>(&va);
                const __half* hb = reinterpret_cast<const __half*>(&vb);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    As[lk + q][lrow] = __half2float(ha[q]);
                    Bs[lk + q][lrow] = __half2float(hb[q]);
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < EX_BK; k++) {
                float ar[8], br[8];
                const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
                const float4 a1 = *reinterpret_cast<const float4*>(&As[k][64 + ty * 4]);
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
                const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][64 + tx * 4]);
                ar[0] = a0.x; ar[1] = a0.y; ar[2] = a0.z; ar[3] = a0.w;
                ar[4] = a1.x; ar[5] = a1.y; ar[6] = a1.z; ar[7] = a1.w;
                br[0] = b0.x; br[1] = b0.y; br[2] = b0.z; br[3] = b0.w;
                br[4] = b1.x; br[5] = b1.y; br[6] = b1.z; br[7] = b1.w;
#pragma unroll
                for (int r = 0; r < 8; r++)
#pragma unroll
                    for (int c = 0; c < 8; c++) acc[r][c] = __fmaf_rz(ar[r], br[c], acc[r][c]);
            }
            __syncthreads();
        }

        // epilogue: reference combine + threshold + compaction
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int64_t i = row0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + (r - 4));
            const bool row_ok = i < a.n_logical;
            const float si = a.norms[i];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int64_t j = col0 + (c < 4 ? tx * 4 + c : 64 + tx * 4 + (c - 4));
                float d2 = 0.0f;
                bool hit = false;
                if (row_ok && j < a.n_logical && j < a.col_end) {
                    d2 = combine_rn(acc[r][c], si, a.norms[j]);
                    hit = d2 <= a.eps_sq;
                }
                const uint32_t b = __ballot_sync(0xffffffffu, hit);
                if (b) writer_append(wr, a, b, hit, (uint32_t)(i + 1), (uint32_t)(j + 1), d2);
            }
        }
    }
    writer_finish(wr, a);
}

}  // namespace fasted

namespace fasted {
int launch_join_exact(const __half* X, const JoinArgs& a, cudaStream_t s) {
    const int64_t n_tiles = ((a.row_end - a.row_begin) / EX_BM) *
                            ((a.col_end - a.col_begin + EX_BN - 1) / EX_BN);
    const int64_t grid = n_tiles < (int64_t)sm_count_current() * 8 ? n_tiles
                                                                  : (int64_t)sm_count_current() * 8;
    if (grid <= 0) return FASTED_OK;
    join_exact_kernel<<<(unsigned)grid, EX_THREADS, 0, s>>>(X, a);
    FASTED_CHECK_LAUNCH("join_exact_kernel");
    return FASTED_OK;
}
}  // namespace fasted
