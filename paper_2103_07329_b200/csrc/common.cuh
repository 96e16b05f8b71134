// common.cuh -- shared device helpers for the mrsolve-b200 kernels (sm_100a).
//
// Arithmetic contract (reference kernels/python_ref.py:1-15,
// kernels/_ckernels.pyx): every multiply-add on the solve path is a
// separately rounded multiply then add/sub.  We spell that with
// __dmul_rn/__dadd_rn/__dsub_rn so nvcc can never contract to FMA, which is
// what makes per-(row, column) SpMM results bitwise equal to the reference.
#pragma once

#include <cuda_runtime.h>

// Checked build (MRS_CHECKS=1 python -m paper_2103_07329_b200.build ->
// libmrsolve_b200_checked.so, loaded with MRS_LIB=...): device-side asserts on
// the index arithmetic and the synchronisation protocols (ticket folds,
// cluster barriers) -- the in-house substitute for compute-sanitizer, which
// this GPU pool does not allow.
#ifdef MRS_CHECKS
#include <cassert>
#define MRS_DCHECK(cond) assert(cond)
#else
#define MRS_DCHECK(cond) ((void)0)
#endif
#include <stdint.h>

#include "../../include/mrsolve_b200.h"

namespace mrs {

constexpr int kThreads = 256;          // every kernel in this library
constexpr int kMaxGridPerSM = 8;       // persistent-grid cap: 148 * 8 CTAs

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double divd(double a, double b) { return __ddiv_rn(a, b); }

template <typename T> __device__ __forceinline__ double widen(T v) { return (double)v; }

// Read-only streaming loads (matrix arrays are read once per product).
template <typename T> __device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// Column block of CPL consecutive doubles at p (p aligned to CPL*8 when CPL>=2).
template <int CPL> struct Vec { double v[CPL]; };

template <int CPL>
__device__ __forceinline__ Vec<CPL> load_vec(const double* __restrict__ p) {
    Vec<CPL> r;
    if constexpr (CPL == 1) {
        r.v[0] = __ldg(p);
    } else {
#pragma unroll
        for (int i = 0; i < CPL; i += 2) {
            double2 t = __ldg(reinterpret_cast<const double2*>(p + i));
            r.v[i] = t.x; r.v[i + 1] = t.y;
        }
    }
    return r;
}

// Plain (coherent) load: for operands written earlier in the same kernel chain
// by other CTAs we never read through the non-coherent path inside one kernel,
// so __ldg is safe everywhere a buffer is read-only for the kernel's lifetime.
template <int CPL>
__device__ __forceinline__ Vec<CPL> load_vec_rw(const double* p) {
    Vec<CPL> r;
    if constexpr (CPL == 1) {
        r.v[0] = *p;
    } else {
#pragma unroll
        for (int i = 0; i < CPL; i += 2) {
            double2 t = *reinterpret_cast<const double2*>(p + i);
            r.v[i] = t.x; r.v[i + 1] = t.y;
        }
    }
    return r;
}

template <int CPL>
__device__ __forceinline__ void store_vec(double* p, const Vec<CPL>& a) {
    if constexpr (CPL == 1) {
        *p = a.v[0];
    } else {
#pragma unroll
        for (int i = 0; i < CPL; i += 2)
            *reinterpret_cast<double2*>(p + i) = make_double2(a.v[i], a.v[i + 1]);
    }
}

// Compiler-only memory fence: loads before it are issued before loads/uses
// after it (keeps batches of independent loads together in SASS).
__device__ __forceinline__ void compiler_fence() { asm volatile("" ::: "memory"); }

// Programmatic dependent launch (PDL): every kernel waits for its stream
// predecessor's memory before touching it, then lets its own successor start
// launching.  Both are no-ops when the kernel was launched without the PDL
// attribute.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Launch with the PDL attribute (see launch_ex in kernels.cu).
bool pdl_enabled();

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

inline int grid_for(long long work_items, int items_per_cta) {
    long long g = (work_items + items_per_cta - 1) / items_per_cta;
    long long cap = (long long)num_sms() * kMaxGridPerSM;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace mrs

#define MRS_CUDA_OK(expr)                                  \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return MRS_ERR_CUDA;        \
    } while (0)
