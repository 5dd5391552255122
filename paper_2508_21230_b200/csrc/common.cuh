// Shared device/host helpers for libfasted (sm_100a only).
#pragma once

#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fasted.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libfasted is written for sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace fasted {

// ---------------------------------------------------------------- host side

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define FASTED_CHECK_LAUNCH(what)                                      \
    do {                                                               \
        cudaError_t _e = cudaGetLastError();                           \
        if (_e != cudaSuccess) return ::fasted::cuda_status(_e, what); \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count_current();

// A 2-D TMA tensor map: `rows` x `inner` elements of type dt, row pitch
// row_bytes (multiple of 16), box box_rows x box_inner, given swizzle;
// out-of-range elements load as zero.  Returns a FASTED_* status.
int encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
              uint64_t rows, uint64_t row_bytes, uint32_t box_inner, uint32_t box_rows,
              CUtensorMapSwizzle swz);

// cudaFuncSetAttribute applies per device context: a launcher keeps one of
// these per kernel and sets the attribute once for each device it runs on
// (one host thread per GPU in self_join(devices=[...])).
struct PerDeviceOnce {
    static constexpr int MAX_DEVICES = 64;
    volatile bool done[MAX_DEVICES] = {};
    template <typename F>
    cudaError_t run(F&& f) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= MAX_DEVICES) return f();
        if (done[dev]) return cudaSuccess;
        e = f();
        if (e == cudaSuccess) done[dev] = true;
        return e;
    }
};

// ---------------------------------------------------------------- device side

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= (uint32_t)o) v += t;
    }
    return v;
}

// Warp-aggregated reservation of `cnt` slots per lane in a global counter:
// one atomic per warp (north star: "one global atomic per warp").  Returns
// the first slot of this lane.  Must be called by all 32 lanes.
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* counter,
                                                            uint32_t cnt) {
    uint32_t incl = warp_inclusive_scan(cnt);
    uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane_id() == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + (incl - cnt);
}

}  // namespace fasted
