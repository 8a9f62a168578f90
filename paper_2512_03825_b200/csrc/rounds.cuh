// rounds.cuh -- the point-to-point exchange-round words shared by the
// resident kernels (resident.cu, resident_smem.cu): one 64-bit (S, Bond,
// round stamp) word per slot in a kRing-deep ring, stored and polled with
// relaxed accesses (gpu scope on one GPU, system scope across GPUs).
#pragma once
#include <cstdint>

namespace ptmh {

constexpr int kRing = 4;

__device__ __forceinline__ uint64_t p2p_pack(int64_t S, int64_t Bd, int64_t round) {
    const uint64_t st = (uint64_t)((round & 0x7fff) | 0x8000);
    return st | (((uint64_t)S & 0xffffffull) << 16) | (((uint64_t)Bd & 0xffffffull) << 40);
}
__device__ __forceinline__ int64_t p2p_field(uint64_t v, int shift) {
    return (int64_t)(((int64_t)(v << (40 - shift))) >> 40);  // sign-extended 24-bit field at `shift`
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// across GPUs (NVLink peer memory): system scope
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// The reference exchange rule for one pair (kernels.py:116-148): x =
// (beta_i - beta_j) * (E_i - E_j), p = logistic(x) evaluated on the stable
// side, accept iff u < p.  near: |u - p| within 4 ulp of p, where a last-ulp
// difference between the device exp and glibc's could flip the decision.
//
// Fast path (the decision sits on a resident round's critical path: the FP64
// exp and division are ~550 cycles): p in FP32 from the same x, |p32 - p| <
// 1e-6, so wherever |u - p32| > 1e-5 the FP32 comparison IS the FP64 one.
// The rest (probability ~2e-5 per pair, and every near tie, since a near tie
// has |u - p| <= 4 ulp) takes the exact FP64 evaluation below.
__device__ __forceinline__ bool swap_decide(double bd, double Ei, double Ej, double u, bool& near) {
    const double x = __dmul_rn(bd, __dsub_rn(Ei, Ej));
    {
        const float xf = (float)x;
        const float pf = xf >= 0.0f ? __frcp_rn(1.0f + __expf(-xf)) : __fdividef(__expf(xf), 1.0f + __expf(xf));
        const double d = __dsub_rn(u, (double)pf);
        if (fabs(d) > 1e-5) {
            near = false;
            return d < 0.0;
        }
    }
    double prob;
    if (x >= 0.0) {
        prob = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
    } else {
        const double ex = exp(x);
        prob = __ddiv_rn(ex, __dadd_rn(1.0, ex));
    }
    near = fabs(u - prob) <= 4.0 * 2.220446049250313e-16 * fmax(prob, 2.2250738585072014e-308);
    return u < prob;
}

// The rounds and observations of a run segment without a 64-bit division per
// sweep: (done / every, done % every) are kept incrementally (done = t + 1).
struct RunSchedule {
    int64_t every, q, r;  // every > 0: done = q * every + r
    __device__ void init(int64_t ev, int64_t done0) {
        every = ev;
        q = ev > 0 ? done0 / ev : 0;
        r = ev > 0 ? done0 - q * ev : 1;
    }
    __device__ bool hit() const { return every > 0 && r == 0; }  // done % every == 0
    __device__ int64_t index() const { return q - 1; }           // done / every - 1 at a hit
    __device__ void step() {
        if (every > 0 && ++r == every) {
            r = 0;
            ++q;
        }
    }
};

}  // namespace ptmh
