// Canonical (i, j) ordering of the join's pair records -- the GPU
// make_result_set (reference tiling.py:116-122, np.lexsort((j, i))) and the
// merge at tiling.py:346-351.
//
// The join emits records in arbitrary order.  Ordering is a counting sort
// on the row (i) followed by a per-row sort on the column (j):
//   1. row histogram (atomics, one per record)
//   2. exclusive scan of the counts -> 64-bit row offsets
//   3. scatter into row segments
//   4. per-row ordering by j (j values of a row are distinct):
//        - rows <= SHORT_MAX records: one warp per row, rank by comparison
//          against the row staged in shared memory;
//        - rows <= RANK_MAX: one CTA per row, a bucketed rank sort in shared
//          memory (rank_sort_segment): ~len/4 buckets over the row's
//          [j_min, j_max] by a monotone float map, counts + scan + scatter,
//          then each element's rank inside its bucket by comparison -- about
//          a dozen shared-memory operations per record instead of the
//          ~300 of a bitonic network (the high-selectivity case: S ~ 1000-4000
//          at 5M x 384, where central points of uniform data have several
//          times the mean neighbour count);
//        - longer rows: one CTA per row splits the row into column
//          super-buckets of <= RANK_MAX (shared-memory counts, scatter in
//          place), then rank-sorts each;
//        - fallbacks, for adversarially clustered j: a bucket above
//          RANK_BUCKET_MAX sends the row to a bitonic sort of (j << 32 | d)
//          keys in shared memory (O(len log^2 len)); a super-bucket above
//          RANK_MAX sends it to a bitmap of the column range with prefix
//          popcounts, O(n_cols/32 + len).
//          (This was the path for every row > 1024 before: at S = 4096 it
//          cleared and scanned a 625 KB bitmap per row, 3.1 s for 2.56e9
//          records; profiles/round1/c5_sweep_session2.jsonl.)
#include "common.cuh"

namespace fasted {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
constexpr int SHORT_MAX = 256;
constexpr int SHORT_WARPS = 4;
constexpr int MID_MAX = 4096;                  // rank sort, small tier (~37 KB smem, 6 CTAs/SM)
constexpr int BIG_MAX = 16384;                 // rank sort, large tier (~148 KB smem)
constexpr int RANK_THREADS = 256;              // small tier (several CTAs per SM)
constexpr int BIG_THREADS = 1024;              // large tier and long rows (one CTA per SM)
constexpr int RANK_BUCKET_MAX = 64;            // a fuller bucket: bitonic fallback
constexpr int RANK_PER = 16;                   // records per thread held in registers
static_assert(MID_MAX == RANK_THREADS * RANK_PER && BIG_MAX == BIG_THREADS * RANK_PER,
              "each rank-sort tier holds one row segment in registers");
constexpr int MID_THREADS = 512;
constexpr int LONG_BLOCKS = 32;
constexpr int LONG_THREADS = 512;

struct SortWs {
    uint32_t* counts;            // n_rows
    uint32_t* cursor;            // n_rows
    unsigned long long* offsets; // n_rows + 1
    unsigned long long* bsum;    // n_scan_blocks + 1
    uint32_t* long_rows;         // n_rows
    uint32_t* long_count;        // 1
    uint32_t* mid_rows;          // n_rows
    uint32_t* mid_count;         // 1
    uint32_t* big_rows;          // n_rows
    uint32_t* big_count;         // 1
    uint32_t* fb_rows;           // n_rows (long rows whose buckets overflow: bitmap path)
    uint32_t* fb_count;          // 1
    uint32_t* bitmap;            // LONG_BLOCKS * 2 * words
};

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t carve(void* base, int64_t n_rows, int64_t n_cols, SortWs* ws) {
    const int64_t nsb = (n_rows + SCAN_TILE - 1) / SCAN_TILE;
    const int64_t words = (n_cols + 31) / 32 + 1;
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t bytes) {
        char* p = b ? b + off : nullptr;
        off += align256(bytes);
        return p;
    };
    SortWs w;
    w.counts = reinterpret_cast<uint32_t*>(take(n_rows * 4));
    w.cursor = reinterpret_cast<uint32_t*>(take(n_rows * 4));
    w.offsets = reinterpret_cast<unsigned long long*>(take((n_rows + 1) * 8));
    w.bsum = reinterpret_cast<unsigned long long*>(take((nsb + 1) * 8));
    w.long_rows = reinterpret_cast<uint32_t*>(take(n_rows * 4));
    w.long_count = reinterpret_cast<uint32_t*>(take(4));
    w.mid_rows = reinterpret_cast<uint32_t*>(take(n_rows * 4));
    w.mid_count = reinterpret_cast<uint32_t*>(take(4));
    w.big_rows = reinterpret_cast<uint32_t*>(take(n_rows * 4));
    w.big_count = reinterpret_cast<uint32_t*>(take(4));
    w.fb_rows = reinterpret_cast<uint32_t*>(take(n_rows * 4));
    w.fb_count = reinterpret_cast<uint32_t*>(take(4));
    w.bitmap = reinterpret_cast<uint32_t*>(take((size_t)LONG_BLOCKS * 2 * words * 4));
    if (ws) *ws = w;
    return off;
}

// The record array is read twice, once per pass, as a stream: its loads
// carry an L2 evict_first policy so the 10s of GB flowing through L2 do not
// evict the working sets the passes write into (the per-row counters and
// cursors, and the row segments' partially written sectors -- with default
// loads the scatter wrote 1.8x and read 1.4x the payload: sectors evicted
// half-filled and merged in DRAM; profiles/round2/sort_launches_c5_s4096_r2.csv).
__device__ __forceinline__ uint64_t stream_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(p), "l"(pol));
    return v;
}

// Records per thread in flight (hist / scatter): SORT_ILP independent
// coalesced loads (and cursor atomics) before any result is used.
constexpr int SORT_ILP = 4;

__device__ __forceinline__ uint32_t sort_lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Row-segment readers: the scatter's scratch is AoS (j, dist_sq bits) in 8
// bytes (one store per record instead of two scattered 4-byte stores, each
// an L2 request and a partial 32-byte sector); the super-bucket path sorts
// the final SoA arrays in place.
struct JdAoS {
    const uint2* p;
    __device__ __forceinline__ uint32_t j(uint64_t e) const { return p[e].x; }
    __device__ __forceinline__ void jd(uint64_t e, uint32_t& j, float& d) const {
        const uint2 v = p[e];
        j = v.x;
        d = __uint_as_float(v.y);
    }
    __device__ __forceinline__ JdAoS at(uint64_t o) const { return JdAoS{p + o}; }
};
struct JdSoA {
    const uint32_t* pj;
    const float* pd;
    __device__ __forceinline__ uint32_t j(uint64_t e) const { return pj[e]; }
    __device__ __forceinline__ void jd(uint64_t e, uint32_t& j, float& d) const {
        j = pj[e];
        d = pd[e];
    }
    __device__ __forceinline__ JdSoA at(uint64_t o) const { return JdSoA{pj + o, pd + o}; }
};

__global__ void __launch_bounds__(256)
hist_kernel(const uint4* __restrict__ rec, uint64_t count, int64_t row_begin,
            uint32_t* __restrict__ counts) {
    const uint64_t pol = stream_policy();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count (the match below needs the whole warp)
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
         p - (threadIdx.x & 31) < count; p += stride * SORT_ILP) {
        uint32_t iv[SORT_ILP];
#pragma unroll
        for (int k = 0; k < SORT_ILP; k++) {
            const uint64_t q = p + (uint64_t)k * stride;
            iv[k] = q < count ? ld_stream_u32(reinterpret_cast<const uint32_t*>(rec + q), pol) : 0u;
        }
        // lanes holding the same row add once (a warp reads 32 consecutive
        // records: one join warp's staging buffer, a few rows repeated)
#pragma unroll
        for (int k = 0; k < SORT_ILP; k++) {   // i == 0: unused slot
            const uint32_t g = __match_any_sync(0xffffffffu, iv[k]);
            if (iv[k] && (g & sort_lanemask_lt()) == 0u)
                atomicAdd(&counts[iv[k] - 1 - row_begin], (uint32_t)__popc(g));
        }
    }
}

// Block-level exclusive scan of SCAN_TILE counts; writes local offsets and
// the block total.
__global__ void __launch_bounds__(SCAN_THREADS)
scan_local_kernel(const uint32_t* __restrict__ counts, int64_t n, unsigned long long* __restrict__ offsets,
                  unsigned long long* __restrict__ bsum) {
    __shared__ unsigned long long warp_tot[SCAN_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    unsigned long long v[SCAN_ITEMS];
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        v[k] = (base + k < n) ? counts[base + k] : 0ull;
        s += v[k];
    }
    // warp inclusive scan of s
    unsigned long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((threadIdx.x & 31) >= (unsigned)o) incl += t;
    }
    if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long w = warp_tot[threadIdx.x];
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
            if (threadIdx.x >= (unsigned)o) wi += t;
        }
        warp_tot[threadIdx.x] = wi - w;   // exclusive warp offsets
        if (threadIdx.x == 31) bsum[blockIdx.x] = wi;
    }
    __syncthreads();
    unsigned long long run = warp_tot[threadIdx.x >> 5] + incl - s;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        if (base + k < n) offsets[base + k] = run;
        run += v[k];
    }
}

// Exclusive scan of the block totals in place (single block, serial chunks).
__global__ void __launch_bounds__(SCAN_THREADS)
scan_blocks_kernel(unsigned long long* __restrict__ bsum, int64_t nb) {
    __shared__ unsigned long long warp_tot[SCAN_THREADS / 32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < nb; c0 += SCAN_THREADS) {
        const int64_t idx = c0 + threadIdx.x;
        const unsigned long long v = idx < nb ? bsum[idx] : 0ull;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((threadIdx.x & 31) >= (unsigned)o) incl += t;
        }
        if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = incl;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long w = warp_tot[threadIdx.x];
            unsigned long long wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
                if (threadIdx.x >= (unsigned)o) wi += t;
            }
            warp_tot[threadIdx.x] = wi - w;
        }
        __syncthreads();
        const unsigned long long excl = carry + warp_tot[threadIdx.x >> 5] + incl - v;
        __syncthreads();
        if (idx < nb) bsum[idx] = excl;
        if (threadIdx.x == SCAN_THREADS - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void scan_add_kernel(unsigned long long* __restrict__ offsets, int64_t n,
                                const unsigned long long* __restrict__ bsum) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < n) offsets[idx] += bsum[idx / SCAN_TILE];
    if (idx == 0) offsets[n] = bsum[(n + SCAN_TILE - 1) / SCAN_TILE];
}

__global__ void __launch_bounds__(256)
scatter_kernel(const uint4* __restrict__ rec, uint64_t count, int64_t row_begin,
               const unsigned long long* __restrict__ offsets, uint32_t* __restrict__ cursor,
               uint2* __restrict__ tjd, unsigned long long tjd_cap) {
    const uint64_t pol = stream_policy();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
         p - (threadIdx.x & 31) < count; p += stride * SORT_ILP) {
        uint4 v[SORT_ILP];
#pragma unroll
        for (int k = 0; k < SORT_ILP; k++) {
            const uint64_t q = p + (uint64_t)k * stride;
            v[k] = q < count ? ld_stream_u4(rec + q, pol) : make_uint4(0u, 0u, 0u, 0u);
        }
        // one cursor atomic per distinct row of the warp's 32 records; each
        // lane takes the next slot after its lower lanes of the same row
        uint32_t c[SORT_ILP], g[SORT_ILP];
#pragma unroll
        for (int k = 0; k < SORT_ILP; k++) {
            g[k] = __match_any_sync(0xffffffffu, v[k].x);
            const bool lead = v[k].x && (g[k] & sort_lanemask_lt()) == 0u;
            c[k] = lead ? atomicAdd(&cursor[(int64_t)v[k].x - 1 - row_begin],
                                    (uint32_t)__popc(g[k]))
                        : 0u;
        }
#pragma unroll
        for (int k = 0; k < SORT_ILP; k++)
            c[k] = __shfl_sync(0xffffffffu, c[k], __ffs(g[k]) - 1) +
                   (uint32_t)__popc(g[k] & sort_lanemask_lt());
#pragma unroll
        for (int k = 0; k < SORT_ILP; k++) {
            if (v[k].x == 0) continue;
            const unsigned long long pos = offsets[(int64_t)v[k].x - 1 - row_begin] + c[k];
            if (pos < tjd_cap) tjd[pos] = make_uint2(v[k].y, v[k].z);
        }
    }
}

// One warp per row: rank-by-comparison inside shared memory.
__global__ void __launch_bounds__(SHORT_WARPS * 32)
short_rows_kernel(const uint2* __restrict__ tjd,
                  const unsigned long long* __restrict__ offsets, int64_t n_rows,
                  int64_t row_begin, uint32_t* __restrict__ oi, uint32_t* __restrict__ oj,
                  float* __restrict__ od, uint32_t* __restrict__ long_rows,
                  uint32_t* __restrict__ long_count, uint32_t* __restrict__ mid_rows,
                  uint32_t* __restrict__ mid_count, uint32_t* __restrict__ big_rows,
                  uint32_t* __restrict__ big_count) {
    __shared__ uint32_t keys[SHORT_WARPS][SHORT_MAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t r = (int64_t)blockIdx.x * SHORT_WARPS + w; r < n_rows;
         r += (int64_t)gridDim.x * SHORT_WARPS) {
        const unsigned long long s0 = offsets[r], s1 = offsets[r + 1];
        const uint32_t len = (uint32_t)(s1 - s0);
        if (len == 0) continue;
        if (len > SHORT_MAX) {
            if (lane == 0) {
                if (len <= (uint32_t)MID_MAX) mid_rows[atomicAdd(mid_count, 1u)] = (uint32_t)r;
                else if (len <= (uint32_t)BIG_MAX) big_rows[atomicAdd(big_count, 1u)] = (uint32_t)r;
                else long_rows[atomicAdd(long_count, 1u)] = (uint32_t)r;
            }
            continue;
        }
        for (uint32_t e = lane; e < len; e += 32) keys[w][e] = tjd[s0 + e].x;
        __syncwarp();
        for (uint32_t e = lane; e < len; e += 32) {
            const uint32_t k = keys[w][e];
            uint32_t rank = 0;
            for (uint32_t q = 0; q < len; q++) rank += keys[w][q] < k;
            oi[s0 + rank] = (uint32_t)(row_begin + r + 1);
            oj[s0 + rank] = k;
            od[s0 + rank] = __uint_as_float(tjd[s0 + e].y);
        }
        __syncwarp();
    }
}

// Bitonic sort of n (power of 2) keys in shared memory, block-wide.
__device__ __forceinline__ void block_bitonic(unsigned long long* key, uint32_t n) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
            for (uint32_t t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
                const uint32_t i = ((t & ~(jj - 1)) << 1) | (t & (jj - 1));
                const uint32_t l = i + jj;
                const unsigned long long a = key[i], b = key[l];
                if ((a > b) == ((i & k) == 0)) {
                    key[i] = b;
                    key[l] = a;
                }
            }
            __syncthreads();
        }
    }
}

// Shared memory of one bucketed rank sort of up to CAP records: bucketed
// copies of j and d (bj then bd: together the 8-byte key array of the
// bitonic fallback), bucket offsets and cursors.
template <int CAP>
struct RankSmem {
    static constexpr int NB = CAP / 8;   // <= 8 records per bucket on average
    uint32_t bj[CAP];
    float bd[CAP];
    uint32_t off[NB + 1];
    uint32_t cur[NB];
    uint32_t red[64];
    uint32_t flag;
    static constexpr size_t BYTES = ((sizeof(uint32_t) * (2 * CAP + 2 * NB + 1 + 64 + 1)) + 15) &
                                    ~(size_t)15;
};

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide exclusive scan of a[0..n) in place (n <= 8 * blockDim.x);
// a[n] = total.  Returns the largest a[k] before the scan.
__device__ uint32_t block_scan_excl(uint32_t* a, uint32_t n, uint32_t* red) {
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t sum = 0, mx = 0;
    for (uint32_t k = 0; k < per; k++)
        if (b0 + k < n) {
            sum += a[b0 + k];
            mx = max(mx, a[b0 + k]);
        }
    const uint32_t incl = warp_inclusive_scan(sum);
    mx = warp_max_u32(mx);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 31) red[w] = incl;
    if ((threadIdx.x & 31) == 0) red[32 + w] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t t = threadIdx.x < (uint32_t)nw ? red[threadIdx.x] : 0u;
        const uint32_t m = threadIdx.x < (uint32_t)nw ? red[32 + threadIdx.x] : 0u;
        const uint32_t ti = warp_inclusive_scan(t);
        const uint32_t mm = warp_max_u32(m);
        red[threadIdx.x] = ti - t;
        if (threadIdx.x == 0) red[32] = mm;
    }
    __syncthreads();
    uint32_t run = red[w] + incl - sum;
    for (uint32_t k = 0; k < per; k++)
        if (b0 + k < n) {
            const uint32_t v = a[b0 + k];
            a[b0 + k] = run;
            run += v;
        }
    if (threadIdx.x == blockDim.x - 1) a[n] = run;
    const uint32_t res = red[32];
    __syncthreads();
    return res;
}

// Canonical order of one row segment of L records (distinct j): reads
// (sj, sd), writes (dj, dd) and, if di, the row id -- dst may alias src.
// Buckets: a monotone map of [j_min, j_max] onto nb ~ L/4 buckets (a float
// product: rounding is monotone, so bucket order is j order); counts, scan,
// scatter into shared memory, then each record's rank inside its bucket by
// comparison.  Returns false (nothing written) if some bucket holds more
// than RANK_BUCKET_MAX records (clustered j): the caller sorts otherwise.
template <int CAP, typename Src>
__device__ bool rank_sort_segment(const Src src, uint32_t L, uint32_t* dj,
                                  float* dd, uint32_t* di, uint32_t row1, RankSmem<CAP>& S) {
    // the row is read from global memory ONCE, into registers (element
    // threadIdx.x + k * blockDim.x in slot k; every launch of a CAP tier
    // has CAP / blockDim.x == RANK_PER), then min/max, bucket counts and the
    // bucket scatter all work from the registers
    uint32_t vj[RANK_PER];
    float vd[RANK_PER];
    uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
    for (int k = 0; k < RANK_PER; k++) {
        const uint32_t e = threadIdx.x + (uint32_t)k * blockDim.x;
        vj[k] = 0u;
        vd[k] = 0.0f;
        if (e < L) src.jd(e, vj[k], vd[k]);
        if (e < L) {
            mn = min(mn, vj[k]);
            mx = max(mx, vj[k]);
        }
    }
    mn = warp_min_u32(mn);
    mx = warp_max_u32(mx);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        S.red[w] = mn;
        S.red[32 + w] = mx;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t a = threadIdx.x < (uint32_t)nw ? S.red[threadIdx.x] : 0xffffffffu;
        const uint32_t b = threadIdx.x < (uint32_t)nw ? S.red[32 + threadIdx.x] : 0u;
        const uint32_t am = warp_min_u32(a), bm = warp_max_u32(b);
        __syncwarp();   // every lane's read of red[lane] before lane 0 overwrites red[0..1]
        if (threadIdx.x == 0) {
            S.red[0] = am;
            S.red[1] = bm;
        }
    }
    __syncthreads();
    mn = S.red[0];
    mx = S.red[1];
    __syncthreads();
    uint32_t nb = 1;
    while (nb < (uint32_t)RankSmem<CAP>::NB && nb * 4u < L) nb <<= 1;
    const float scale = (float)nb / ((float)(mx - mn) + 1.0f);
    auto bucket = [&](uint32_t j) {
        const uint32_t b = (uint32_t)((float)(j - mn) * scale);
        return b < nb ? b : nb - 1u;
    };
    for (uint32_t b = threadIdx.x; b <= nb; b += blockDim.x) S.off[b] = 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RANK_PER; k++)
        if (threadIdx.x + (uint32_t)k * blockDim.x < L) atomicAdd(&S.off[bucket(vj[k])], 1u);
    __syncthreads();
    const uint32_t fullest = block_scan_excl(S.off, nb, S.red);
    if (fullest > (uint32_t)RANK_BUCKET_MAX) return false;   // block-uniform
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) S.cur[b] = S.off[b];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RANK_PER; k++) {
        if (threadIdx.x + (uint32_t)k * blockDim.x < L) {
            const uint32_t p = atomicAdd(&S.cur[bucket(vj[k])], 1u);
            S.bj[p] = vj[k];
            S.bd[p] = vd[k];
        }
    }
    __syncthreads();   // every read of (sj, sd) done: dst may alias src
    for (uint32_t x = threadIdx.x; x < L; x += blockDim.x) {
        const uint32_t j = S.bj[x];
        const uint32_t b = bucket(j);
        const uint32_t lo = S.off[b], hi = S.off[b + 1];
        uint32_t rank = 0;
        for (uint32_t y = lo; y < hi; y++) rank += S.bj[y] < j;
        dj[lo + rank] = j;
        dd[lo + rank] = S.bd[x];
        if (di) di[lo + rank] = row1;
    }
    __syncthreads();
    return true;
}

// Bitonic fallback for a segment of L <= CAP records (dst may alias src):
// (j << 32 | d bits) keys in the rank sort's shared memory.
template <int CAP, typename Src>
__device__ void bitonic_segment(const Src src, uint32_t L, uint32_t* dj,
                                float* dd, uint32_t* di, uint32_t row1, RankSmem<CAP>& S) {
    unsigned long long* key = reinterpret_cast<unsigned long long*>(S.bj);
    uint32_t n = 1;
    while (n < L) n <<= 1;
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
        uint32_t j = 0u;
        float d = 0.0f;
        if (e < L) src.jd(e, j, d);
        key[e] = e < L ? ((unsigned long long)j << 32) | (unsigned long long)__float_as_uint(d)
                       : ~0ull;
    }
    __syncthreads();
    block_bitonic(key, n);
    for (uint32_t e = threadIdx.x; e < L; e += blockDim.x) {
        const unsigned long long v = key[e];
        dj[e] = (uint32_t)(v >> 32);
        dd[e] = __uint_as_float((uint32_t)v);
        if (di) di[e] = row1;
    }
    __syncthreads();
}

// One CTA per listed row (SHORT_MAX < len <= CAP): rank sort, bitonic if a
// bucket overflows.
template <int CAP, int THREADS>
__global__ void __launch_bounds__(THREADS)
rank_rows_kernel(const uint2* __restrict__ tjd,
                 const unsigned long long* __restrict__ offsets, int64_t row_begin,
                 const uint32_t* __restrict__ rows, const uint32_t* __restrict__ nrows,
                 uint32_t* __restrict__ oi, uint32_t* __restrict__ oj, float* __restrict__ od) {
    extern __shared__ __align__(16) uint8_t rank_raw[];
    RankSmem<CAP>& S = *reinterpret_cast<RankSmem<CAP>*>(rank_raw);
    const uint32_t nm = *nrows;
    for (uint32_t mi = blockIdx.x; mi < nm; mi += gridDim.x) {
        const int64_t r = rows[mi];
        const unsigned long long s0 = offsets[r];
        const uint32_t len = (uint32_t)(offsets[r + 1] - s0);
        const uint32_t row1 = (uint32_t)(row_begin + r + 1);
        const JdAoS src{tjd + s0};
        if (!rank_sort_segment<CAP>(src, len, oj + s0, od + s0, oi + s0, row1, S))
            bitonic_segment<CAP>(src, len, oj + s0, od + s0, oi + s0, row1, S);
    }
}

constexpr int BUCKETS_MAX = 1024;
constexpr uint32_t SUPER_TARGET = BIG_MAX / 2;   // expected records per column super-bucket

// One CTA per long row (> BIG_MAX records): column super-buckets (counts,
// scatter in place into the row's final slots of out_j/out_d), then a rank
// sort of each, in place.
__global__ void __launch_bounds__(BIG_THREADS)
bucket_rows_kernel(const uint2* __restrict__ tjd,
                   const unsigned long long* __restrict__ offsets, int64_t row_begin,
                   int64_t n_cols, const uint32_t* __restrict__ long_rows,
                   const uint32_t* __restrict__ long_count, uint32_t* __restrict__ fb_rows,
                   uint32_t* __restrict__ fb_count, uint32_t* __restrict__ oi,
                   uint32_t* __restrict__ oj, float* __restrict__ od) {
    extern __shared__ __align__(16) uint8_t rank_raw[];
    RankSmem<BIG_MAX>& S = *reinterpret_cast<RankSmem<BIG_MAX>*>(rank_raw);
    __shared__ uint32_t cnt[BUCKETS_MAX], boff[BUCKETS_MAX + 1], cur[BUCKETS_MAX];
    __shared__ uint32_t overflow;
    const uint32_t nl = *long_count;
    for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
        const int64_t r = long_rows[li];
        const unsigned long long s0 = offsets[r];
        const uint32_t len = (uint32_t)(offsets[r + 1] - s0);
        uint32_t nb = 2;
        while (nb < BUCKETS_MAX && (uint64_t)nb * SUPER_TARGET < len) nb <<= 1;
        const uint32_t bw = (uint32_t)(((uint64_t)n_cols + nb - 1) / nb);   // columns per bucket
        for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
        if (threadIdx.x == 0) overflow = 0;
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < len; e += blockDim.x)
            atomicAdd(&cnt[(tjd[s0 + e].x - 1u) / bw], 1u);
        __syncthreads();
        if (threadIdx.x == 0) {   // nb <= 1024: a serial scan is cheap next to the row
            uint32_t run = 0;
            for (uint32_t b = 0; b < nb; b++) {
                boff[b] = run;
                cur[b] = run;
                if (cnt[b] > (uint32_t)BIG_MAX) overflow = 1;
                run += cnt[b];
            }
            boff[nb] = run;
        }
        __syncthreads();
        if (overflow) {
            if (threadIdx.x == 0) fb_rows[atomicAdd(fb_count, 1u)] = (uint32_t)r;
            __syncthreads();
            continue;
        }
        for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) {
            const uint2 v = tjd[s0 + e];
            const uint32_t pos = atomicAdd(&cur[(v.x - 1u) / bw], 1u);
            oj[s0 + pos] = v.x;
            od[s0 + pos] = __uint_as_float(v.y);
        }
        __syncthreads();   // the block's own global writes are visible to it after this
        const uint32_t row1 = (uint32_t)(row_begin + r + 1);
        for (uint32_t b = 0; b < nb; b++) {
            const uint32_t b0 = boff[b], bl = boff[b + 1] - b0;
            if (bl == 0) continue;
            uint32_t* sj = oj + s0 + b0;
            float* sd = od + s0 + b0;
            const JdSoA src{sj, sd};
            if (!rank_sort_segment<BIG_MAX>(src, bl, sj, sd, oi + s0 + b0, row1, S))
                bitonic_segment<BIG_MAX>(src, bl, sj, sd, oi + s0 + b0, row1, S);
        }
    }
}

// One block per long row: bitmap ranks over the column range.
__global__ void __launch_bounds__(LONG_THREADS)
long_rows_kernel(const uint2* __restrict__ tjd,
                 const unsigned long long* __restrict__ offsets, int64_t row_begin,
                 int64_t n_cols, const uint32_t* __restrict__ long_rows,
                 const uint32_t* __restrict__ long_count, uint32_t* __restrict__ bitmap_all,
                 uint32_t* __restrict__ oi, uint32_t* __restrict__ oj, float* __restrict__ od) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t carry;
    constexpr int NW = LONG_THREADS / 32;
    const int64_t words = (n_cols + 31) / 32 + 1;
    uint32_t* bits = bitmap_all + (int64_t)blockIdx.x * 2 * words;
    uint32_t* pref = bits + words;
    const uint32_t nl = *long_count;
    for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
        const int64_t r = long_rows[li];
        const unsigned long long s0 = offsets[r], s1 = offsets[r + 1];
        for (int64_t w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0;
        __syncthreads();
        for (unsigned long long e = s0 + threadIdx.x; e < s1; e += blockDim.x) {
            const uint32_t j0 = tjd[e].x - 1;
            atomicOr(&bits[j0 >> 5], 1u << (j0 & 31));
        }
        __syncthreads();
        if (threadIdx.x == 0) carry = 0;
        __syncthreads();
        for (int64_t c0 = 0; c0 < words; c0 += blockDim.x) {
            const int64_t w = c0 + threadIdx.x;
            const uint32_t v = w < words ? (uint32_t)__popc(bits[w]) : 0u;
            const uint32_t incl = warp_inclusive_scan(v);
            if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = incl;
            __syncthreads();
            if (threadIdx.x < 32) {
                const uint32_t t = threadIdx.x < NW ? warp_tot[threadIdx.x] : 0u;
                const uint32_t ti = warp_inclusive_scan(t);
                warp_tot[threadIdx.x] = ti - t;
            }
            __syncthreads();
            const uint32_t excl = carry + warp_tot[threadIdx.x >> 5] + incl - v;
            __syncthreads();
            if (w < words) pref[w] = excl;
            if (threadIdx.x == blockDim.x - 1) carry = excl + v;
            __syncthreads();
        }
        for (unsigned long long e = s0 + threadIdx.x; e < s1; e += blockDim.x) {
            const uint2 v = tjd[e];
            const uint32_t j = v.x;
            const uint32_t j0 = j - 1;
            const uint32_t rank =
                pref[j0 >> 5] + (uint32_t)__popc(bits[j0 >> 5] & ((1u << (j0 & 31)) - 1u));
            oi[s0 + rank] = (uint32_t)(row_begin + r + 1);
            oj[s0 + rank] = j;
            od[s0 + rank] = __uint_as_float(v.y);
        }
        __syncthreads();
    }
}

}  // namespace fasted

using namespace fasted;

extern "C" size_t fasted_sort_workspace_bytes(int64_t n_rows, int64_t n_cols) {
    if (n_rows < 1 || n_cols < 1) return 0;
    return carve(nullptr, n_rows, n_cols, nullptr);
}

extern "C" int fasted_sort_pairs(const void* records, uint64_t count, int64_t row_begin,
                                 int64_t row_end, int64_t n_cols, uint32_t* out_i,
                                 uint32_t* out_j, float* out_d, void* tmp, size_t tmp_bytes,
                                 void* workspace, size_t workspace_bytes, void* stream) {
    const int64_t n_rows = row_end - row_begin;
    if (count == 0) return FASTED_OK;
    const uint4* rec = static_cast<const uint4*>(records);
    uint2* tjd = static_cast<uint2*>(tmp);
    if (!rec || !out_i || !out_j || !out_d || !tmp || (reinterpret_cast<uintptr_t>(tmp) & 7u) ||
        tmp_bytes < 8 || !workspace || n_rows < 1 ||
        n_cols < 1 || n_cols > 0xffffffffLL) {
        set_error("fasted_sort_pairs: bad arguments");
        return FASTED_ERR_ARGUMENT;
    }
    const size_t need = carve(nullptr, n_rows, n_cols, nullptr);
    if (workspace_bytes < need) {
        set_error("fasted_sort_pairs: workspace %zu < %zu bytes", workspace_bytes, need);
        return FASTED_ERR_ARGUMENT;
    }
    SortWs ws;
    carve(workspace, n_rows, n_cols, &ws);
    cudaStream_t s = as_stream(stream);
    cudaMemsetAsync(ws.counts, 0, n_rows * 4, s);
    cudaMemsetAsync(ws.cursor, 0, n_rows * 4, s);
    cudaMemsetAsync(ws.long_count, 0, 4, s);
    cudaMemsetAsync(ws.mid_count, 0, 4, s);
    cudaMemsetAsync(ws.big_count, 0, 4, s);
    cudaMemsetAsync(ws.fb_count, 0, 4, s);
    const int sms = sm_count_current();
    // one resident wave (8 x 256 threads per SM), SORT_ILP records per thread in flight
    const uint64_t rec_blocks = (count + 256 * SORT_ILP - 1) / (256 * SORT_ILP);
    const unsigned rec_grid =
        (unsigned)(rec_blocks < (uint64_t)sms * 8 ? rec_blocks : (uint64_t)sms * 8);
    hist_kernel<<<rec_grid, 256, 0, s>>>(rec, count, row_begin, ws.counts);
    FASTED_CHECK_LAUNCH("hist_kernel");
    const int64_t nsb = (n_rows + SCAN_TILE - 1) / SCAN_TILE;
    scan_local_kernel<<<(unsigned)nsb, SCAN_THREADS, 0, s>>>(ws.counts, n_rows, ws.offsets,
                                                              ws.bsum);
    FASTED_CHECK_LAUNCH("scan_local_kernel");
    scan_blocks_kernel<<<1, SCAN_THREADS, 0, s>>>(ws.bsum, nsb);
    FASTED_CHECK_LAUNCH("scan_blocks_kernel");
    scan_add_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(ws.offsets, n_rows, ws.bsum);
    FASTED_CHECK_LAUNCH("scan_add_kernel");
    scatter_kernel<<<rec_grid, 256, 0, s>>>(rec, count, row_begin, ws.offsets, ws.cursor, tjd,
                                            (unsigned long long)(tmp_bytes / 8));
    FASTED_CHECK_LAUNCH("scatter_kernel");
    const int64_t sgrid = (n_rows + SHORT_WARPS - 1) / SHORT_WARPS;
    short_rows_kernel<<<(unsigned)(sgrid < (int64_t)sms * 64 ? sgrid : (int64_t)sms * 64),
                        SHORT_WARPS * 32, 0, s>>>(tjd, ws.offsets, n_rows, row_begin,
                                                  out_i, out_j, out_d, ws.long_rows,
                                                  ws.long_count, ws.mid_rows, ws.mid_count,
                                                  ws.big_rows, ws.big_count);
    FASTED_CHECK_LAUNCH("short_rows_kernel");
    static PerDeviceOnce rank_once;
    {
        cudaError_t e = rank_once.run([&] {
            cudaError_t r = cudaFuncSetAttribute(rank_rows_kernel<MID_MAX, RANK_THREADS>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)RankSmem<MID_MAX>::BYTES);
            if (r == cudaSuccess)
                r = cudaFuncSetAttribute(rank_rows_kernel<BIG_MAX, BIG_THREADS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)RankSmem<BIG_MAX>::BYTES);
            if (r == cudaSuccess)
                r = cudaFuncSetAttribute(bucket_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)RankSmem<BIG_MAX>::BYTES);
            return r;
        });
        if (e != cudaSuccess) return cuda_status(e, "rank sort attributes");
    }
    rank_rows_kernel<MID_MAX, RANK_THREADS><<<(unsigned)(sms * 6), RANK_THREADS, RankSmem<MID_MAX>::BYTES, s>>>(
        tjd, ws.offsets, row_begin, ws.mid_rows, ws.mid_count, out_i, out_j, out_d);
    FASTED_CHECK_LAUNCH("rank_rows_kernel<4096>");
    rank_rows_kernel<BIG_MAX, BIG_THREADS><<<(unsigned)sms, BIG_THREADS, RankSmem<BIG_MAX>::BYTES, s>>>(
        tjd, ws.offsets, row_begin, ws.big_rows, ws.big_count, out_i, out_j, out_d);
    FASTED_CHECK_LAUNCH("rank_rows_kernel<16384>");
    bucket_rows_kernel<<<(unsigned)sms, BIG_THREADS, RankSmem<BIG_MAX>::BYTES, s>>>(
        tjd, ws.offsets, row_begin, n_cols, ws.long_rows, ws.long_count, ws.fb_rows,
        ws.fb_count, out_i, out_j, out_d);
    FASTED_CHECK_LAUNCH("bucket_rows_kernel");
    long_rows_kernel<<<LONG_BLOCKS, LONG_THREADS, 0, s>>>(tjd, ws.offsets, row_begin,
                                                          n_cols, ws.fb_rows, ws.fb_count,
                                                          ws.bitmap, out_i, out_j, out_d);
    FASTED_CHECK_LAUNCH("long_rows_kernel");
    return FASTED_OK;
}
