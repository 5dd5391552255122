// C ABI entry points of libfasted.so (declared in include/fasted.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"
#include "join_common.cuh"

namespace fasted {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return FASTED_ERR_CUDA;
}

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

int encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                     uint64_t rows, uint64_t row_bytes, uint32_t box_inner, uint32_t box_rows,
                     CUtensorMapSwizzle swz) {
    auto encode = tensor_map_encoder();
    if (!encode) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return FASTED_ERR_CUDA;
    }
    cuuint64_t gdim[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult cr = encode(map, dt, 2, const_cast<void*>(base), gdim, gstride, box, estride,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)cr);
        return FASTED_ERR_CUDA;
    }
    return FASTED_OK;
}

int sm_count_current() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

}  // namespace fasted

using namespace fasted;

extern "C" int fasted_abi_version(void) { return FASTED_ABI_VERSION; }

extern "C" const char* fasted_strerror(int status) {
    switch (status) {
        case FASTED_OK: return "ok";
        case FASTED_ERR_ARGUMENT: return "argument error";
        case FASTED_ERR_RANGE: return "value out of FP16 range";
        case FASTED_ERR_CAPACITY: return "result buffer too small";
        case FASTED_ERR_CUDA: return "CUDA error";
        case FASTED_ERR_UNSUPPORTED: return "unsupported device (needs sm_100)";
        default: return "unknown status";
    }
}

extern "C" const char* fasted_last_error(void) { return g_err; }

extern "C" int fasted_device_check(int device) {
    int major = 0, minor = 0;
    cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0) {
        set_error("device %d is sm_%d%d; libfasted is built for sm_100a only", device, major,
                  minor);
        return FASTED_ERR_UNSUPPORTED;
    }
    return FASTED_OK;
}

extern "C" const char* fasted_join_kernel_name(int64_t d_pad, int64_t rows, int64_t cols,
                                               int flags) {
    if ((flags & 1) == FASTED_JOIN_EXACT) return "fasted::join_exact_kernel";
    return join_tc_kernel_name(d_pad, rows, cols, (flags & FASTED_JOIN_LOW_OUTPUT) != 0,
                               (flags & FASTED_JOIN_SPARSE) != 0);
}

extern "C" int fasted_device_info(int* sm_count, char* name, int name_len) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    cudaDeviceProp p;
    e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties");
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (name && name_len > 0) {
        strncpy(name, p.name, (size_t)name_len - 1);
        name[name_len - 1] = 0;
    }
    return FASTED_OK;
}

extern "C" int fasted_join(const uint16_t* values16, const float* norms, int64_t n_logical,
                           int64_t n_pad, int64_t d_pad, int64_t row_begin, int64_t row_end,
                           int64_t col_begin, int64_t col_end, float eps_sq, int flags,
                           void* out_records, uint64_t capacity, unsigned long long* count,
                           void* stream) {
    const bool count_only = (flags & FASTED_JOIN_COUNT) != 0;
    const int kind = flags & 1;
    constexpr int kPublicFlags = FASTED_JOIN_EXACT | FASTED_JOIN_COUNT | FASTED_JOIN_SYMMETRIC |
                                 FASTED_JOIN_LOW_OUTPUT | FASTED_JOIN_APPEND | FASTED_JOIN_SPARSE;
    if (flags & ~(kPublicFlags | FASTED_JOIN_DIAG_ALL)) {
        set_error("fasted_join: unknown flag bits 0x%x", flags & ~(kPublicFlags | FASTED_JOIN_DIAG_ALL));
        return FASTED_ERR_ARGUMENT;
    }
    if (!values16 || !norms || !count || n_pad < 128 || (n_pad % 128) != 0 || d_pad < 16 ||
        (d_pad % 16) != 0 || n_logical < 1 || n_logical > n_pad || n_pad > 0xffffffffLL) {
        set_error("fasted_join: bad dataset geometry (n_logical=%lld n_pad=%lld d_pad=%lld)",
                  (long long)n_logical, (long long)n_pad, (long long)d_pad);
        return FASTED_ERR_ARGUMENT;
    }
    auto bad_bound = [&](int64_t b) { return b < 0 || b > n_pad || (b % 128 != 0 && b != n_pad); };
    if (bad_bound(row_begin) || bad_bound(row_end) || bad_bound(col_begin) ||
        bad_bound(col_end) || row_end < row_begin || col_end < col_begin) {
        set_error("fasted_join: ranges must be 128-aligned within [0, n_pad]");
        return FASTED_ERR_ARGUMENT;
    }
    if (!(eps_sq >= 0.0f) || !(eps_sq <= 3.402823466e38f)) {
        set_error("fasted_join: eps_sq must be finite and >= 0");
        return FASTED_ERR_ARGUMENT;
    }
    if (!count_only && capacity > 0 &&
        (!out_records || (reinterpret_cast<uintptr_t>(out_records) & 15u) != 0)) {
        set_error("fasted_join: 16-byte aligned record buffer required unless count-only");
        return FASTED_ERR_ARGUMENT;
    }
    const bool symmetric = (flags & FASTED_JOIN_SYMMETRIC) != 0;
    if (symmetric && (kind == FASTED_JOIN_EXACT || row_begin != col_begin || row_end != col_end)) {
        set_error("fasted_join: the symmetric schedule needs the tcgen05 kernel and row range == "
                  "column range");
        return FASTED_ERR_ARGUMENT;
    }
    cudaStream_t s = as_stream(stream);
    if (!(flags & FASTED_JOIN_APPEND)) {
        cudaError_t e = cudaMemsetAsync(count, 0, 2 * sizeof(unsigned long long), s);
        if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(count)");
    }
    if (row_end == row_begin || col_end == col_begin) return FASTED_OK;
    JoinArgs a;
    a.norms = norms;
    a.n_logical = n_logical;
    a.n_pad = n_pad;
    a.d_pad = d_pad;
    a.row_begin = row_begin;
    a.row_end = row_end;
    a.col_begin = col_begin;
    a.col_end = col_end;
    a.eps_sq = eps_sq;
    a.count_only = count_only ? 1 : 0;
    a.symmetric = symmetric ? 1 : 0;
    a.low_output = (flags & FASTED_JOIN_LOW_OUTPUT) != 0 ? 1 : 0;
    a.sparse = (flags & FASTED_JOIN_SPARSE) != 0 ? 1 : 0;
    a.diag_flags = flags & FASTED_JOIN_DIAG_ALL;   // always 0 in libfasted.so
    a.out = reinterpret_cast<uint4*>(out_records);
    a.capacity = count_only ? 0ull : (unsigned long long)capacity;
    a.count = count;
    a.gram_diag = nullptr;
    a.trace = nullptr;
    a.pace = nullptr;
#ifdef FASTED_EXPERIMENTS
    if (flags & FASTED_JOIN_DIAG_TRACE) {
        const unsigned long long trace_recs = TRACE_WORDS / 2;
        if (count_only || a.capacity < trace_recs) {
            set_error("fasted_join: the trace flag needs a record buffer with room for the "
                      "timeline");
            return FASTED_ERR_ARGUMENT;
        }
        a.capacity -= trace_recs;
        a.trace = reinterpret_cast<unsigned long long*>(a.out + a.capacity);
    }
#endif
    const __half* X = reinterpret_cast<const __half*>(values16);
    return kind == FASTED_JOIN_EXACT ? launch_join_exact(X, a, s) : launch_join_tc(X, a, s);
}
