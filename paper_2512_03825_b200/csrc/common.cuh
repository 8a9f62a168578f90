// common.cuh -- error plumbing shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "ptmh.h"

namespace ptmh {

void set_error(const std::string& msg);

#define PTMH_CHECK_ARG(cond, msg)                     \
    do {                                              \
        if (!(cond)) {                                \
            ::ptmh::set_error(std::string("argument: ") + (msg)); \
            return PTMH_ERR_ARG;                      \
        }                                             \
    } while (0)

#define PTMH_CUDA(call)                                                        \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) {                                               \
            cudaGetLastError(); /* a non-sticky error must not fail the next call */ \
            ::ptmh::set_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
            return PTMH_ERR_CUDA;                                              \
        }                                                                      \
    } while (0)

#define PTMH_LAUNCH_CHECK() PTMH_CUDA(cudaGetLastError())

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace ptmh
