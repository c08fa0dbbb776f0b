// Shared device helpers for the adjamr B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "../../include/adjamr_b200.h"

#define ADJ_HD __host__ __device__ __forceinline__
#define ADJ_D __device__ __forceinline__

namespace adj {

// Programmatic dependent launch: kernels of a level sweep are launched with
// programmatic stream serialisation so a grid is scheduled while its
// predecessor drains; every such kernel waits for the predecessor's memory
// (griddepcontrol.wait) before touching anything, then lets its own
// successor launch.  Without the launch attribute both are no-ops.
ADJ_D void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
ADJ_D void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" :::); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// Record the last CUDA error for adj_last_error(); returns ADJ_ERR_CUDA on error.
int record_cuda(cudaError_t e, const char* where);
int check_launch(const char* where);

// Non-negative doubles order like their bit patterns, so an unsigned 64-bit
// atomicMax on the bits is a max on the values (speeds are |s| >= 0).
ADJ_D void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

ADJ_D double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// View of one patch inside a level store.
struct PatchView {
    const double* q;     // component 0 plane base + patch offset
    const double* aux;   // aux plane 0 base + patch offset
    int64_t cs, as;      // component / aux plane strides
    int pitch;           // x-row pitch (1 in 1D)
    ADJ_D double Q(int c, int i, int j) const { return q[c * cs + (int64_t)i * pitch + j]; }
    ADJ_D double A(int k, int i, int j) const { return aux[k * as + (int64_t)i * pitch + j]; }
};

// Reference limiter phi(theta), solver.py:65-77 (same min/max nesting).
ADJ_D double limiter_phi(int lim, double th) {
    switch (lim) {
        case ADJ_LIM_MINMOD: return fmax(0.0, fmin(1.0, th));
        case ADJ_LIM_MC: return fmax(0.0, fmin(fmin((1.0 + th) / 2.0, 2.0), 2.0 * th));
        case ADJ_LIM_SUPERBEE: return fmax(0.0, fmax(fmin(1.0, 2.0 * th), fmin(2.0, th)));
        default: return 1.0;
    }
}

}  // namespace adj
