// pf_log.h -- binary64 natural log for the PARITY tracers.
//
// The reference's tracking step is `t -= std::log(1 - u) * inv_sigma_max`
// (proj/src/volume.cpp:217, 247) with glibc's log, which is accurate to about
// half an ulp.  CUDA's log() is a ~55-instruction, <= 1 ulp routine and was
// 30% of the binary64 tracer's instructions (profiles/r02a_hot_trace_parity.md).
// This one is table-driven and cheaper (~30 instructions) and more accurate
// (~0.5 ulp), so it agrees with glibc at least as often as CUDA's did:
//
//   y = 2^k z, z in [OFF, 2 OFF) (OFF ~ 1/sqrt 2); i = top 7 mantissa bits
//   of bits(z) - bits(OFF); invc_i has <= 8 significant bits, so
//   r = fma(z, invc_i, -1) is EXACT (|r| < 2^-7); logc_i = -ln(invc_i) is a
//   double-double whose high part is a multiple of 2^-46, so
//   w = k ln2hi + logc_hi is exact;  log y = TwoSum(w, r) + (k ln2lo + logc_lo
//   + r^2 P(r)),  P = Taylor terms of log1p to r^8 (truncation < 2^-59 rel).
//
// Domain: positive normal doubles (the tracers call it on 1 - u, u a 53-bit
// uniform, i.e. y in [2^-53, 1]); log(1) = +0 exactly.  Host and device
// builds are identical operation-for-operation (explicit fma, no contraction),
// so tests/test_log.py checks this very code against glibc on the CPU.
#pragma once

#include <stdint.h>

#include "pf_log_table.h"

#ifndef PF_LOG_I2F
#define PF_LOG_I2F 1  // 0: round-1 instruction choices (A/B)
#endif

#if defined(__CUDACC__)
#define PF_LOG_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define PF_LOG_HD static inline
#endif

namespace pfk {

#if defined(__CUDACC__)
// one table per translation unit; 2 KB, L1-resident
static __device__ const pf_log_entry pf_log_tab_dev[1 << PF_LOG_BITS] = PF_LOG_TABLE_INIT;
#endif
static const pf_log_entry pf_log_tab_host[1 << PF_LOG_BITS] = PF_LOG_TABLE_INIT;

// Polynomial / ln2 constants.  On the device they live in the constant bank so
// the DFMAs take them as c[][] operands (64-bit immediates would cost two
// uniform moves each, every step).
#define PF_LOG_CONSTS                                                                                  \
    {-0x1p-3, 0x1.2492492492492p-3, -0x1.5555555555555p-3, 0x1.999999999999ap-3, -0x1p-2,              \
     0x1.5555555555555p-2, -0x1p-1, PF_LOG_LN2HI, PF_LOG_LN2LO}
#if defined(__CUDACC__)
static __constant__ double pf_log_c_dev[9] = PF_LOG_CONSTS;
#endif
static const double pf_log_c_host[9] = PF_LOG_CONSTS;
#if defined(__CUDA_ARCH__) && !defined(PF_LOG_IMM)
#define PF_LOG_C(i) pf_log_c_dev[i]
#elif defined(__CUDA_ARCH__)
#define PF_LOG_C(i) ((const double[9])PF_LOG_CONSTS)[i]
#else
#define PF_LOG_C(i) pf_log_c_host[i]
#endif

PF_LOG_HD uint64_t pf_log_bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
PF_LOG_HD double pf_log_dbl(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}
PF_LOG_HD double pf_log_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}
PF_LOG_HD double pf_log_add(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
PF_LOG_HD double pf_log_sub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
PF_LOG_HD double pf_log_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}

// log(y * 2^escale) for y a positive normal double and y * 2^escale normal: the same
// operations as pf_log(y * 2^escale), with escale folded into the exponent k only, so
// the result is bit-identical (z, r and the table index do not depend on escale).
#if defined(__CUDACC__)
// Shared-memory copy of the table with the two hi-word constants expanded to
// full doubles (32-byte entries: two loads and no register assembly per log).
struct __align__(32) pf_log_wide {
    double logc_hi, invc, logc_lo, pad;
};
__device__ __forceinline__ void pf_log_fill_wide(pf_log_wide *t, int tid, int nthreads) {
    for (int i = tid; i < (1 << PF_LOG_BITS); i += nthreads) {
        const pf_log_entry e = pf_log_tab_dev[i];
        t[i] = {e.logc_hi, pf_log_dbl((uint64_t)e.invc_hi << 32), pf_log_dbl((uint64_t)e.logc_lo_hi << 32), 0.0};
    }
}
#endif

template <bool SMEM = false>
PF_LOG_HD double pf_log_scaled(double y, int escale, uint32_t tab = 0u) {
    const uint64_t ix = pf_log_bits(y);
    const uint32_t hx = (uint32_t)(ix >> 32);
    const uint32_t tmp = hx - PF_LOG_OFF_HI;
    const int kraw = (int32_t)tmp >> 20;
    const int k = kraw + escale;
    const uint32_t i = (tmp >> (20 - PF_LOG_BITS)) & ((1u << PF_LOG_BITS) - 1u);
    double logc_hi, invc, logc_lo;
#if defined(__CUDA_ARCH__)
    if constexpr (SMEM) {  // pf_log_wide entries at byte address tab
        asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(logc_hi), "=d"(invc) : "r"(tab + 32u * i));
        asm("ld.shared.f64 %0, [%1];" : "=d"(logc_lo) : "r"(tab + 32u * i + 16u));
    } else {  // one 16-byte load of the compact entry
        const double2 v = __ldg(reinterpret_cast<const double2 *>(pf_log_tab_dev) + i);
        const unsigned long long u = (unsigned long long)__double_as_longlong(v.y);
        logc_hi = v.x;
        invc = pf_log_dbl((uint64_t)(uint32_t)u << 32);
        logc_lo = pf_log_dbl((u >> 32) << 32);
    }
#else
    (void)tab;
    const pf_log_entry e = pf_log_tab_host[i];
    logc_hi = e.logc_hi;
    invc = pf_log_dbl((uint64_t)e.invc_hi << 32);
    logc_lo = pf_log_dbl((uint64_t)e.logc_lo_hi << 32);
#endif
    const double z = pf_log_dbl(((uint64_t)(hx - ((uint32_t)kraw << 20)) << 32) | (ix & 0xffffffffull));
#if defined(__CUDA_ARCH__) && PF_LOG_I2F
    const double kd = __int2double_rn(k);  // exact; one I2F on the XU pipe (~20% busy) beats 3 ALU/DP ops
#else
    // kd = (double)k without a conversion instruction: 2^52 + (k + 1024) - (2^52 + 1024)
    const double kd = pf_log_sub(pf_log_dbl(0x4330000000000000ull | (uint32_t)(k + 1024)), 0x1.0000000000400p52);
#endif
    const double r = pf_log_fma(z, invc, -1.0);                    // exact
    const double w = pf_log_fma(kd, PF_LOG_C(7), logc_hi);       // exact
    // TwoSum(w, r)
    const double hi = pf_log_add(w, r);
    const double bb = pf_log_sub(hi, w);
    const double lo = pf_log_add(pf_log_sub(w, pf_log_sub(hi, bb)), pf_log_sub(r, bb));
    // log1p(r) - r = r^2 (c2 + c3 r + ... + c8 r^6)
    const double r2 = pf_log_mul(r, r);
    // -1/8 as a literal: an exact short DFMA immediate, so the first step needs
    // no register copy of a constant-bank operand
#if PF_LOG_I2F
    double p = pf_log_fma(r, -0.125, PF_LOG_C(1));  // -1/8 r + 1/7
#else
    double p = PF_LOG_C(0);                 // -1/8
    p = pf_log_fma(p, r, PF_LOG_C(1));      // 1/7
#endif
    p = pf_log_fma(p, r, PF_LOG_C(2));      // -1/6
    p = pf_log_fma(p, r, PF_LOG_C(3));      // 1/5
    p = pf_log_fma(p, r, PF_LOG_C(4));      // -1/4
    p = pf_log_fma(p, r, PF_LOG_C(5));      // 1/3
    p = pf_log_fma(p, r, PF_LOG_C(6));      // -1/2
    double tail = pf_log_fma(kd, PF_LOG_C(8), logc_lo);
    tail = pf_log_fma(r2, p, tail);
    return pf_log_add(hi, pf_log_add(lo, tail));
}

PF_LOG_HD double pf_log(double y) { return pf_log_scaled<false>(y, 0); }

}  // namespace pfk
