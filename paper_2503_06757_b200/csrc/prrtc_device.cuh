// prrtc_device.cuh — sm_100a device routines of the B200 pRRTC planner.
//
// Everything here runs inside one CTA (default 128 threads = 4 warps):
//   * exact FP64 restatements of the reference scalar arithmetic where the
//     reference's result must be reproduced bit-for-bit (Halton, lerp,
//     squared distance, the sphere predicates' guard-band fallback);
//   * the FP32 fast paths (forward kinematics, predicates) that do the bulk
//     of the work on the FP32 FMA pipe;
//   * the CTA-wide routines: nearest-neighbour scan (warp-shuffle argmin),
//     SIMT edge validation (states split over threads, two-stage spheres,
//     shared-memory-staged primitives, ballot/flag early exit).
//
// Reference cross-references are given as file:line of /root/reference/proj.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "prrtc_internal.h"

namespace prrtc_b200 {
namespace dev {

constexpr int kMaxDof = 32;
constexpr int kNoBad = 0x7fffffff;
constexpr int kTTab = 128;  // edge-sample fraction table covers n_cc <= 128
#ifndef PRRTC_NN_PAIRS
#define PRRTC_NN_PAIRS 2
#endif
constexpr int kNnPairs = PRRTC_NN_PAIRS;  // node pairs per NN scan trip (1, 2, 4 or 8; measured: 2)

// ---------------------------------------------------------------------------
// memory-model helpers (gpu scope)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// exact FP64 scalar arithmetic (no FMA contraction: __d*_rn are never fused)
// ---------------------------------------------------------------------------

// kernels_scalar.cpp:18-22 (lerp) — a + t*(b-a), one element.
__device__ __forceinline__ double lerp_exact(double a, double b, double t) {
    return __dadd_rn(a, __dmul_rn(t, __dsub_rn(b, a)));
}

// sampling.cpp:8-18 (halton_value): f /= b; r += f*(i mod b); i /= b.
__device__ __forceinline__ double halton_exact(unsigned base, unsigned long long index) {
    double f = 1.0, r = 0.0;
    const double b = static_cast<double>(base);
    if (index >> 32) {
        while (index > 0) {
            f = __ddiv_rn(f, b);
            r = __dadd_rn(r, __dmul_rn(f, static_cast<double>(index % base)));
            index /= base;
        }
    } else {
        unsigned i = static_cast<unsigned>(index);  // same digits, 32-bit divide
        while (i > 0) {
            f = __ddiv_rn(f, b);
            const unsigned q = i / base;
            r = __dadd_rn(r, __dmul_rn(f, static_cast<double>(i - q * base)));
            i = q;
        }
    }
    return r;
}

// halton_exact with the reciprocal powers f_k = (((1/b)/b).../b) taken from a
// table (the same IEEE divisions, computed once per CTA) and the digit
// division done by multiply-high with M = ceil(2^64 / b) (exact for 32-bit
// indices): bit-identical to halton_exact, without the per-digit FP64 and
// integer divides.
constexpr int kHaltonTab = HALTON_TAB;
__device__ __forceinline__ double halton_tab(unsigned base, unsigned long long magic, const double* ftab,
                                             unsigned long long index) {
    if (index >> 32) return halton_exact(base, index);
    unsigned i = static_cast<unsigned>(index);
    double r = 0.0;
    for (int k = 0; i > 0; ++k) {
        const unsigned q = (unsigned)__umul64hi((unsigned long long)i, magic);
        const double f = k < kHaltonTab ? ftab[k] : 0.0;
        if (k >= kHaltonTab) return halton_exact(base, index);
        r = __dadd_rn(r, __dmul_rn(f, static_cast<double>(i - q * base)));
        i = q;
    }
    return r;
}

// ---------------------------------------------------------------------------
// SamplerKind::Uniform (sampling.hpp:40-54): std::mt19937_64 seeded with
// params.seed * 0x9e3779b97f4a7c15 + worker (planner.cpp:194) and libstdc++'s
// uniform_real_distribution<double>(lo, hi): generate_canonical<double, 53>
// takes one 64-bit draw x (mt19937_64's range is 2^64), ret = double(x) /
// 2^64 (nextafter(1, 0) if it rounds to 1), value = ret * (hi - lo) + lo —
// the same IEEE operations here (__ull2double_rn, exact power-of-two
// scaling, __dmul_rn, __dadd_rn). One generator per CTA in shared memory
// (312 words + position); the twist runs CTA-wide in its three dependency
// phases, the tempering of a block's draws in parallel.
// ---------------------------------------------------------------------------
constexpr int kMtN = 312, kMtM = 156;
constexpr unsigned long long kMtA = 0xB5026F5AA96619E9ull;
constexpr unsigned long long kMtUpper = ~0ull << 31, kMtLower = ~kMtUpper;

__device__ __forceinline__ unsigned long long mt_mix(unsigned long long xk, unsigned long long xk1) {
    const unsigned long long y = (xk & kMtUpper) | (xk1 & kMtLower);
    return (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

// std::mersenne_twister_engine::seed(value) (one thread; CTA-uniform state)
__device__ __noinline__ void mt_seed(unsigned long long* mt, unsigned long long seed) {
    mt[0] = seed;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (unsigned)i;
    mt[kMtN] = kMtN;  // position: the first draw twists
}

// _M_gen_rand in its dependency phases (CTA-wide; all threads call; at most
// two elements per thread and phase, so nthreads >= 78)
__device__ __noinline__ void mt_twist(unsigned long long* mt, int nthreads) {
    const int tid = threadIdx.x, k0 = tid, k1 = tid + nthreads;
    constexpr int n1 = kMtN - kMtM;  // phase 1: k in [0, 156), old values only
    unsigned long long v0 = 0, v1 = 0;
    if (k0 < n1) v0 = mt[k0 + kMtM] ^ mt_mix(mt[k0], mt[k0 + 1]);
    if (k1 < n1) v1 = mt[k1 + kMtM] ^ mt_mix(mt[k1], mt[k1 + 1]);
    __syncthreads();
    if (k0 < n1) mt[k0] = v0;
    if (k1 < n1) mt[k1] = v1;
    __syncthreads();
    // phase 2: k in [156, 311): x[k - 156] is new, x[k], x[k + 1] old
    const int j0 = n1 + k0, j1 = n1 + k1;
    if (j0 < kMtN - 1) v0 = mt[j0 - n1] ^ mt_mix(mt[j0], mt[j0 + 1]);
    if (j1 < kMtN - 1) v1 = mt[j1 - n1] ^ mt_mix(mt[j1], mt[j1 + 1]);
    __syncthreads();
    if (j0 < kMtN - 1) mt[j0] = v0;
    if (j1 < kMtN - 1) mt[j1] = v1;
    __syncthreads();
    if (tid == 0) {  // the last element wraps to the new x[0]
        mt[kMtN - 1] = mt[kMtM - 1] ^ mt_mix(mt[kMtN - 1], mt[0]);
        mt[kMtN] = 0;
    }
    __syncthreads();
}

// uniform_real_distribution<double>(lo, hi)(rng) from one raw draw
__device__ __forceinline__ double uniform_dim(unsigned long long x, double lo, double hi) {
    double ret = __dmul_rn(__ull2double_rn(x), 0x1p-64);
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return __dadd_rn(__dmul_rn(ret, __dsub_rn(hi, lo)), lo);
}

// The next `count` draws of the CTA's generator as scaled samples, draw j =
// (sample j / dof, dimension j % dof), into out[j] (CTA-wide).
__device__ __noinline__ void mt_fill(unsigned long long* mt, const double* limits, int dof, double* out, int count,
                                    int nthreads) {
    int done = 0;
    while (done < count) {
        if (mt[kMtN] >= (unsigned long long)kMtN) mt_twist(mt, nthreads);
        const int pos = (int)mt[kMtN];
        const int take = min(count - done, kMtN - pos);
        for (int j = threadIdx.x; j < take; j += nthreads) {
            const int g = done + j, d = g % dof;
            out[g] = uniform_dim(mt_temper(mt[pos + j]), limits[2 * d], limits[2 * d + 1]);
        }
        __syncthreads();
        if (threadIdx.x == 0) mt[kMtN] = pos + take;
        __syncthreads();
        done += take;
    }
}

// sampling.cpp:39-51 (sample_config), one dimension.
__device__ __forceinline__ double sample_dim(double h, double lo, double hi) {
    double v = __dadd_rn(lo, __dmul_rn(h, __dsub_rn(hi, lo)));
    if (v >= hi) v = nextafter(hi, lo);
    return v;
}

// ---------------------------------------------------------------------------
// exact FP64 predicates — kernels_detail.hpp:17-50, same operation order
// ---------------------------------------------------------------------------
__device__ __forceinline__ double clamp01_exact(double t) {
    if (t < 0.0) t = 0.0;
    if (t > 1.0) t = 1.0;
    return t;
}

// kernels_detail.hpp:17-23
__device__ __noinline__ bool sphere_sphere_exact(double px, double py, double pz, double pr,
                                                 double sx, double sy, double sz, double sr) {
    const double dx = __dsub_rn(px, sx), dy = __dsub_rn(py, sy), dz = __dsub_rn(pz, sz);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const double rr = __dadd_rn(pr, sr);
    return d2 < __dmul_rn(rr, rr);
}

// kernels_detail.hpp:25-35
__device__ __noinline__ bool sphere_capsule_exact(double px, double py, double pz, double pr,
                                                  const double* c /* a, ab, inv, r */) {
    const double pax = __dsub_rn(px, c[0]), pay = __dsub_rn(py, c[1]), paz = __dsub_rn(pz, c[2]);
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(pax, c[3]), __dmul_rn(pay, c[4])),
                                 __dmul_rn(paz, c[5]));
    const double t = clamp01_exact(__dmul_rn(dot, c[6]));
    const double dx = __dsub_rn(pax, __dmul_rn(t, c[3]));
    const double dy = __dsub_rn(pay, __dmul_rn(t, c[4]));
    const double dz = __dsub_rn(paz, __dmul_rn(t, c[5]));
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const double rr = __dadd_rn(pr, c[7]);
    return d2 < __dmul_rn(rr, rr);
}

// kernels_detail.hpp:37-50
__device__ __noinline__ bool sphere_box_exact(double px, double py, double pz, double pr,
                                              const double* b /* m[9], t[3], h[3] */) {
    const double wx = __dsub_rn(px, b[9]), wy = __dsub_rn(py, b[10]), wz = __dsub_rn(pz, b[11]);
    const double lx = __dadd_rn(__dadd_rn(__dmul_rn(b[0], wx), __dmul_rn(b[1], wy)), __dmul_rn(b[2], wz));
    const double ly = __dadd_rn(__dadd_rn(__dmul_rn(b[3], wx), __dmul_rn(b[4], wy)), __dmul_rn(b[5], wz));
    const double lz = __dadd_rn(__dadd_rn(__dmul_rn(b[6], wx), __dmul_rn(b[7], wy)), __dmul_rn(b[8], wz));
    const double hx = b[12], hy = b[13], hz = b[14];
    const double cx = lx < -hx ? -hx : (lx > hx ? hx : lx);
    const double cy = ly < -hy ? -hy : (ly > hy ? hy : ly);
    const double cz = lz < -hz ? -hz : (lz > hz ? hz : lz);
    const double dx = __dsub_rn(lx, cx), dy = __dsub_rn(ly, cy), dz = __dsub_rn(lz, cz);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return d2 < __dmul_rn(pr, pr);
}

// Cylinder extension (no reference counterpart; restated bit-for-bit in
// oracle/prrtc_oracle.c sphere_cylinder_hit): local coordinates like the box
// test, radial excess max(rho - r, 0), axial excess max(|z| - h, 0),
// d2 = er^2 + ez^2 < pr^2, in this exact operation order.
__device__ __noinline__ bool sphere_cylinder_exact(double px, double py, double pz, double pr,
                                                   const double* y /* m[9], t[3], r, h */) {
    const double wx = __dsub_rn(px, y[9]), wy = __dsub_rn(py, y[10]), wz = __dsub_rn(pz, y[11]);
    const double lx = __dadd_rn(__dadd_rn(__dmul_rn(y[0], wx), __dmul_rn(y[1], wy)), __dmul_rn(y[2], wz));
    const double ly = __dadd_rn(__dadd_rn(__dmul_rn(y[3], wx), __dmul_rn(y[4], wy)), __dmul_rn(y[5], wz));
    const double lz = __dadd_rn(__dadd_rn(__dmul_rn(y[6], wx), __dmul_rn(y[7], wy)), __dmul_rn(y[8], wz));
    const double rho = __dsqrt_rn(__dadd_rn(__dmul_rn(lx, lx), __dmul_rn(ly, ly)));
    double er = __dsub_rn(rho, y[12]);
    if (er < 0.0) er = 0.0;
    double ez = __dsub_rn(fabs(lz), y[13]);
    if (ez < 0.0) ez = 0.0;
    const double d2 = __dadd_rn(__dmul_rn(er, er), __dmul_rn(ez, ez));
    return d2 < __dmul_rn(pr, pr);
}

// ---------------------------------------------------------------------------
// FP32 fast predicates. Each returns the squared distance d2 and the
// combined radius rr of the test "d2 < rr*rr" evaluated in FP32.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sph_d2(float px, float py, float pz, float4 s, float& d2) {
    const float dx = px - s.x, dy = py - s.y, dz = pz - s.z;
    d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}
// Primitive records are 16-byte aligned in shared memory (scene words:
// 12-word header, float4 spheres, 16-float boxes, 8-float capsules), so each
// is fetched with 128-bit loads (2 / 4 LDS.128 instead of 8 / 15 LDS.32).
__device__ __forceinline__ void cap_d2(float px, float py, float pz, const float* c, float& d2) {
    const float4 c0 = reinterpret_cast<const float4*>(c)[0];  // a.xyz, ab.x
    const float4 c1 = reinterpret_cast<const float4*>(c)[1];  // ab.yz, 1/|ab|^2, r
    const float pax = px - c0.x, pay = py - c0.y, paz = pz - c0.z;
    float t = fmaf(pax, c0.w, fmaf(pay, c1.x, paz * c1.y)) * c1.z;
    t = fminf(fmaxf(t, 0.0f), 1.0f);
    const float dx = fmaf(-t, c0.w, pax), dy = fmaf(-t, c1.x, pay), dz = fmaf(-t, c1.y, paz);
    d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}
__device__ __forceinline__ void box_d2(float px, float py, float pz, const float* b, float& d2) {
    const float4 b0 = reinterpret_cast<const float4*>(b)[0];  // M00 M01 M02 M10
    const float4 b1 = reinterpret_cast<const float4*>(b)[1];  // M11 M12 M20 M21
    const float4 b2 = reinterpret_cast<const float4*>(b)[2];  // M22 tx ty tz
    const float4 b3 = reinterpret_cast<const float4*>(b)[3];  // hx hy hz -
    const float wx = px - b2.y, wy = py - b2.z, wz = pz - b2.w;
    const float lx = fmaf(b0.x, wx, fmaf(b0.y, wy, b0.z * wz));
    const float ly = fmaf(b0.w, wx, fmaf(b1.x, wy, b1.y * wz));
    const float lz = fmaf(b1.z, wx, fmaf(b1.w, wy, b2.x * wz));
    const float dx = lx - fminf(fmaxf(lx, -b3.x), b3.x);
    const float dy = ly - fminf(fmaxf(ly, -b3.y), b3.y);
    const float dz = lz - fminf(fmaxf(lz, -b3.z), b3.z);
    d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}
__device__ __forceinline__ void cyl_d2(float px, float py, float pz, const float* y, float& d2) {
    const float4 y0 = reinterpret_cast<const float4*>(y)[0];  // M00 M01 M02 M10
    const float4 y1 = reinterpret_cast<const float4*>(y)[1];  // M11 M12 M20 M21
    const float4 y2 = reinterpret_cast<const float4*>(y)[2];  // M22 tx ty tz
    const float4 y3 = reinterpret_cast<const float4*>(y)[3];  // r h - -
    const float wx = px - y2.y, wy = py - y2.z, wz = pz - y2.w;
    const float lx = fmaf(y0.x, wx, fmaf(y0.y, wy, y0.z * wz));
    const float ly = fmaf(y0.w, wx, fmaf(y1.x, wy, y1.y * wz));
    const float lz = fmaf(y1.z, wx, fmaf(y1.w, wy, y2.x * wz));
    const float er = fmaxf(sqrtf(fmaf(lx, lx, ly * ly)) - y3.x, 0.0f);
    const float ez = fmaxf(fabsf(lz) - y3.y, 0.0f);
    d2 = fmaf(er, er, ez * ez);
}

// Guard band: returns 1 = certainly hit, 0 = certainly free, -1 = undecided
// (|distance - rr| <= eps: re-evaluate in exact FP64).
__device__ __forceinline__ int band(float d2, float rr, float eps) {
    const float hi = rr + eps;
    if (d2 > hi * hi) return 0;
    const float lo = rr - eps;
    if (lo > 0.0f && d2 < lo * lo) return 1;
    return -1;
}

// ---------------------------------------------------------------------------
// CTA context: pointers into dynamic shared memory
//
// SIMT mapping (PAPER.md:178-180 re-designed for 32-wide warps): a chunk holds
// NS = 32/64/128 edge states; lane i of every warp owns states i, i+32, ...;
// warps split the per-state work by link (FK), by (link, primitive group)
// (coarse stage) and by flagged entry (fine stage), so the primitive data
// is a warp-uniform shared-memory broadcast and each state's data is
// conflict-free (state is the fastest smem index).
// ---------------------------------------------------------------------------
// A pointer into the dynamic shared-memory window held as a 32-bit offset
// (every CTA-context buffer lives there): an access costs one add, where a
// generic pointer needs two generic->shared conversions (sh()) to let the
// compiler emit LDS/STS — ~22M instructions and ~3 KB of hot code per
// headline launch (ncu source view, r2d).
extern __shared__ __align__(16) unsigned char g_dsmem[];
template <class T>
struct SPtr {
    unsigned off;
    __device__ __forceinline__ T* get() const { return reinterpret_cast<T*>(g_dsmem + off); }
    __device__ __forceinline__ operator T*() const { return get(); }
    __device__ __forceinline__ SPtr& operator=(T* p) {
        off = (unsigned)__cvta_generic_to_shared(p) - (unsigned)__cvta_generic_to_shared(g_dsmem);
        return *this;
    }
};

// The CTA's fixed-size buffers sit at constant offsets at the start of the
// dynamic window (sizes for NS <= 128, nthreads <= 512): an access is an
// immediate shared address, where an SPtr first loads its offset from the
// shared Ctx — a dependent LDS the compiler must repeat after every barrier
// (ncu source view, r2i: 11.7% of plan_kernel's stall samples on those
// offset loads).
enum : unsigned {
    FX_ICTL = 0,        // [IC_COUNT] int
    FX_T0 = 128,        // [T0_COUNT] u64
    FX_RED_D = 192,     // [16] double
    FX_RED_I = 320,     // [16] int
    FX_MNN_D = 384,     // [32] double
    FX_MNN_I = 640,     // [32] int
    FX_MNN_OK = 768,    // [32] int
    FX_DCFG = 896,      // [8][kMaxDof] double
    FX_SGROUP = 2944,   // [128] int
    FX_SBAD = 3456,     // [128] int
    FX_TTAB = 3968,     // [kTTab + 1] double
    FX_PANY = 5008,     // [8] u64: self pairs coarse-flagged for any state of the chunk
    FX_LANY = 5072,     // u64: links coarse-flagged for any state of the chunk
    FX_END = 5088
};
static_assert(FX_DCFG + 8 * 8 * kMaxDof == FX_SGROUP && FX_TTAB + 8 * (kTTab + 1) <= FX_PANY &&
                  FX_PANY + 8 * 8 == FX_LANY && FX_LANY + 8 <= FX_END && FX_END % 16 == 0,
              "fixed shared-memory region");
template <class T, unsigned OFF>
struct FPtr {
    __device__ __forceinline__ T* get() const { return reinterpret_cast<T*>(g_dsmem + OFF); }
    __device__ __forceinline__ operator T*() const { return get(); }
};

struct Ctx {
    // robot (shared memory copy of the packed words)
    int L, dof, S, NP, MF, mflog;  // mflog: log2 of MF rounded up to a power of two
    SPtr<const int4> info;      // kind, parent, q_index, fine_off
    SPtr<const int> nfine;
    SPtr<const float> geo;      // [L][GEO_STRIDE]
    SPtr<const float4> fine;    // [S]
    SPtr<const int2> pairs;     // [NP]
    SPtr<const unsigned> bases; // [dof]
    SPtr<const unsigned long long> magic;  // [dof] ceil(2^64 / base)
    SPtr<const double> htab;    // [dof][kHaltonTab] Halton reciprocal powers (shared copy of the host table)
    SPtr<const int> flink;      // [S] link of each fine sphere
    SPtr<const int2> funits;    // [NFU] fine-stage units: (link, first sphere | count << 16)
    int NFU;
    const double* fine_r64;  // global
    SPtr<const double> limits;    // [dof][2] (shared copy, before the Halton table)
    unsigned fkflops;        // per-state FK + coarse posing flops
    long long* prof;         // per-phase clock64 stamps (debug hook only, else null)
    FPtr<double, FX_TTAB> ttab;   // [kTTab + 1]: i / ttab_n for i = 0..ttab_n (edge sample fractions)
    int ttab_n;              // n_cc the table was built for (0 = none)
    // scene (shared memory copy)
    int ns, nb, nc, ny, P;
    SPtr<const float4> sph;
    SPtr<const float> box;
    SPtr<const float> cap;
    SPtr<const float> cyl;
    float eps, cpad;
    SceneF64 s64;  // global FP64 mirror
    // per-chunk buffers
    int NS, nslog;   // states per chunk (32, 64 or 128)
    SPtr<float> pose;     // [L][12][NS]
    SPtr<float> ccen;     // [L][3][NS]
    SPtr<float> qf;       // [dof][NS]
    FPtr<int, FX_SGROUP> sgroup;  // [NS] group id, -1 = inactive
    FPtr<int, FX_SBAD> sbad;      // [NS]
    FPtr<unsigned long long, FX_PANY> pany;  // [8] pairs flagged for any state (then lany at [8])
    FPtr<unsigned long long, FX_LANY> lany;  // links flagged for any state
    SPtr<unsigned long long> lmask;  // [L][NS] coarse-flagged primitives per (link, state)
    SPtr<unsigned long long> pmask;  // [ceil(NP/64)][NS] coarse-flagged self pairs per state
    SPtr<double> ends;    // [NS + 2][dof] chain points of the chunk
    // CTA scalars
    FPtr<int, FX_ICTL> ictl;      // [32] misc ints
    FPtr<double, FX_DCFG> dcfg;   // [8][kMaxDof] scratch configs
    SPtr<double> sbuf;    // [32][dof] Halton samples of the CTA's current ticket block
    FPtr<double, FX_MNN_D> mnn_d; // [32] multi-sample NN: squared distance per evaluated sample
    FPtr<int, FX_MNN_I> mnn_i;    // [32]                  nearest index per evaluated sample
    FPtr<int, FX_MNN_OK> mnn_ok;  // [32]                  accepted (not duplicate, inside its dynamic domain)
    FPtr<double, FX_RED_D> red_d; // [nwarps]
    FPtr<int, FX_RED_I> red_i;    // [nwarps]
    int nthreads;
    // stats: per-thread slots [nthreads][2] in shared memory (sphere tests,
    // algorithmic FP32 flops), summed when a CTA leaves a problem
    SPtr<unsigned long long> stat;
    // the planner loop's thread-0 state (ticket block, iteration and CheckStats
    // counters): kept in shared memory so it does not occupy registers
    // (spilled around every call) in all threads of the CTA
    FPtr<unsigned long long, FX_T0> t0;
    // exact-CheckStats mode (deterministic planning): counters follow the
    // reference's sequential semantics (ref_state_count); per-state scratch
    int ref_stats;
    SPtr<unsigned long long> mt;      // [kMtN + 1] SamplerKind::Uniform generator state + position
    SPtr<unsigned long long> rcount;  // [NS] reference sphere_tests of each state
    SPtr<int> rfine;                  // [NS] 1 if the state enters the fine stage
};

enum : int {
    T0_TKBASE = 0, T0_TKPOS, T0_TKCNT, T0_USED, T0_LITER, T0_FK, T0_FINE,
    T0_RTESTS,  // exact-CheckStats mode: reference-semantics sphere tests
    T0_COUNT = 8
};

// The planner keeps its Ctx in shared memory (plan_kernel): every field is
// CTA-uniform, so reads are broadcast LDS instead of local-memory loads that
// the acquire fences' L1 invalidations would send to L2. The helpers below
// that fill it write through thread 0 only in that case (ctx_writer).
__device__ __forceinline__ bool ctx_writer(const Ctx& c) { return !__isShared(&c) || threadIdx.x == 0; }

// The Ctx lives in the kernel's local-memory frame, so a pointer read from it
// is generic: loads through it become LD.E (not LDS) and every store through
// it may alias the frame, forcing the other fields to be re-read. sh()
// re-derives the pointer from the dynamic shared-memory symbol, which lets the
// compiler prove the shared address space (LDS/STS, no aliasing with local
// memory). Hot routines take their pointers into registers through it once.
template <class T>
__device__ __forceinline__ T* sh(const SPtr<T>& p) {
    return p.get();
}
template <class T, unsigned OFF>
__device__ __forceinline__ T* sh(const FPtr<T, OFF>& p) {
    return p.get();
}
template <class T>
__device__ __forceinline__ T* sh(T* p) {
    // integer offsets in the shared window (no cross-object pointer arithmetic)
    const unsigned off = (unsigned)__cvta_generic_to_shared(p) - (unsigned)__cvta_generic_to_shared(g_dsmem);
    return reinterpret_cast<T*>(g_dsmem + off);
}

// Register-resident view of the scene (shared-memory pointers + scalars).
struct SceneV {
    const float4* sph;
    const float* box;
    const float* cap;
    const float* cyl;
    int ns, nb, nsbc, P;  // primitive order: spheres [0, ns), boxes, capsules, cylinders [nsbc, P)
    float eps;
    SceneF64 s64;
};
__device__ __forceinline__ SceneV scene_view(const Ctx& c) {
    return SceneV{sh(c.sph), sh(c.box), sh(c.cap), sh(c.cyl), c.ns, c.nb, c.ns + c.nb + c.nc, c.P, c.eps, c.s64};
}

// ictl slots
enum : int {
    IC_QN = 0,      // env queue length
    IC_PQN,         // pair queue length
    IC_OVF,         // queue overflow
    IC_FIRSTBAD,    // min bad group
    IC_FLAGGED,     // states entering the fine stage
    IC_TMP0,
    IC_TMP1,
    IC_TMP2,
    IC_TMP3,
    IC_TMP4,
    IC_TMP5,
    IC_TMP6,
    IC_TMP7,
    IC_KLO,         // first chain point held in `ends`
    IC_KNOWN0,      // per tree: published prefix this CTA holds acquire-ordered (or wrote itself);
    IC_KNOWN1,      //   a snapshot within it needs no fence (thread 0 only)
    IC_DIRTY,       // force a fence at the next header (set when the CTA joins a problem)
    IC_STOP,        // the problem's done flag as sampled by gen_chain_states (planner.cpp:112)
    IC_COUNT = 32
};

// dcfg rows
enum : int { DC_A = 0, DC_B, DC_SAMPLE, DC_NEW, DC_NN, DC_TARGET, DC_TMP, DC_TMP2 };

__device__ __forceinline__ double* dc(Ctx& c, int row) { return sh(c.dcfg) + row * kMaxDof; }

// Posed point R*p + t from a pose stored as [12][NS] column (state s).
// Explicit fmaf order: identical bits wherever it is used (FK parity).
__device__ __forceinline__ float3 pose_pt(const float* pose, int N, int l, int s, float px, float py,
                                          float pz) {
    const float* P = pose + l * 12 * N + s;
    float3 o;
    o.x = __fmaf_rn(P[0 * N], px, __fmaf_rn(P[1 * N], py, __fmaf_rn(P[2 * N], pz, P[9 * N])));
    o.y = __fmaf_rn(P[3 * N], px, __fmaf_rn(P[4 * N], py, __fmaf_rn(P[5 * N], pz, P[10 * N])));
    o.z = __fmaf_rn(P[6 * N], px, __fmaf_rn(P[7 * N], py, __fmaf_rn(P[8 * N], pz, P[11 * N])));
    return o;
}
__device__ __forceinline__ float3 pose_point(const Ctx& c, int l, int s, float px, float py,
                                             float pz) {
    return pose_pt(sh(c.pose), c.NS, l, s, px, py, pz);
}

// A link pose (3x4) of one state held in registers, applied with the same
// fmaf order as pose_pt (identical bits).
struct PoseR {
    float m[12];
};
__device__ __forceinline__ PoseR pose_load(const float* pose, int N, int l, int s) {
    const float* P = pose + l * 12 * N + s;
    PoseR r;
#pragma unroll
    for (int k = 0; k < 12; ++k) r.m[k] = P[k * N];
    return r;
}
__device__ __forceinline__ float3 pose_apply(const PoseR& P, float px, float py, float pz) {
    float3 o;
    o.x = __fmaf_rn(P.m[0], px, __fmaf_rn(P.m[1], py, __fmaf_rn(P.m[2], pz, P.m[9])));
    o.y = __fmaf_rn(P.m[3], px, __fmaf_rn(P.m[4], py, __fmaf_rn(P.m[5], pz, P.m[10])));
    o.z = __fmaf_rn(P.m[6], px, __fmaf_rn(P.m[7], py, __fmaf_rn(P.m[8], pz, P.m[11])));
    return o;
}

// ---------------------------------------------------------------------------
// forward kinematics for the chunk's states (kinematics.cpp:92-103), FP32,
// one pass: row r of world_l = row r of world_parent * local_l depends only
// on row r of the parent, so warps take (row, 32-state group) tasks and
// every lane walks its state's chain link by link in registers:
//   local_l = origin_tf * motion(q) (Rodrigues folded: cos M1 + sin M2 +
//             (1 - cos) M3, see prrtc_internal.h; recomputed by each of the
//             three row lanes of a state instead of staged through smem)
//   row r of world_l, stored to pose[l][3r..3r+2 | 9+r][s]
//   coordinate r of the posed coarse centre, stored to ccen[l][r][s]
// State is the fastest smem index: every access is conflict-free. A branch
// point (parent != previous link) reads the parent row this lane stored.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sincos_joint(float q, float* sn, float* cs) {
    // |q| within a few turns (joint limits): 2-constant Cody-Waite reduction
    // to [-pi, pi], then the SFU pair (abs error ~2^-21 there; FK stays well
    // inside the 1e-5 m sphere-centre tolerance)
    const float k = rintf(q * 0.15915494309189535f);
    const float r = __fmaf_rn(-k, 6.28318548202514648f, __fmaf_rn(-k, -1.7484555314695172e-7f, q));
    __sincosf(r, sn, cs);
}

__device__ __forceinline__ void fk_chunk(Ctx& c, int cnt) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = c.nthreads >> 5;
    const int NS = c.NS, L = c.L;
    float* const pose = sh(c.pose);
    const float* const qf = sh(c.qf);
    const int4* const info = sh(c.info);
    const float* const geo = sh(c.geo);
    float* const ccen = sh(c.ccen);
    const int groups = (cnt + 31) >> 5;
    {
        // the warps FK leaves idle (all warps if none is) reset the chunk's
        // verdict state and flag masks meanwhile; check_chunk's stages read
        // them after the closing barrier
        const int busy = 3 * groups < nw ? 3 * groups * 32 : 0;
        if (tid >= busy) {
            const int PW = (c.NP + 63) >> 6, t0 = tid - busy, nt = c.nthreads - busy;
            int* const sbad = sh(c.sbad);
            unsigned long long* const lmask = sh(c.lmask);
            for (int s = t0; s < NS; s += nt) sbad[s] = 0;
            for (int i = t0; i < (L + PW) * NS; i += nt) lmask[i] = 0ull;  // pmask follows lmask
            if (t0 < 9) sh(c.pany)[t0] = 0ull;  // pany[8] and lany
            if (t0 == 0) {
                sh(c.ictl)[IC_QN] = 0;
                sh(c.ictl)[IC_FIRSTBAD] = kNoBad;
            }
        }
        if (!busy) __syncthreads();  // no idle warp: the reset precedes FK
    }
    for (int task = warp; task < 3 * groups; task += nw) {
        const int r = task % 3;
        const int s = (task / 3) * 32 + lane;
        const bool act = s < cnt;
        const int sr = act ? s : 0;
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, wt = 0.f;  // row r of the previous link's world pose
        for (int l = 0; l < L; ++l) {
            const int4 inf = info[l];  // warp-uniform
            float g[36];  // the link's geometry record, 9 x 128-bit broadcast loads
#pragma unroll
            for (int k = 0; k < 9; ++k)
                reinterpret_cast<float4*>(g)[k] = reinterpret_cast<const float4*>(geo + l * GEO_STRIDE)[k];
            float R[9], t0, t1, t2;
            if (inf.x == PRRTC_JOINT_REVOLUTE) {
                float sn, cs;
                sincos_joint(qf[inf.z * NS + sr], &sn, &cs);
                const float omc = 1.0f - cs;
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = __fmaf_rn(cs, g[k], __fmaf_rn(sn, g[9 + k], __fmul_rn(omc, g[18 + k])));
                t0 = g[27];
                t1 = g[28];
                t2 = g[29];
            } else {
#pragma unroll
                for (int k = 0; k < 9; ++k) R[k] = g[k];
                if (inf.x == PRRTC_JOINT_PRISMATIC) {
                    const float q = qf[inf.z * NS + sr];
                    t0 = __fmaf_rn(g[30], q, g[27]);
                    t1 = __fmaf_rn(g[31], q, g[28]);
                    t2 = __fmaf_rn(g[32], q, g[29]);
                } else {
                    t0 = g[27];
                    t1 = g[28];
                    t2 = g[29];
                }
            }
            float n0, n1, n2, nt;
            if (inf.y < 0) {  // root: world = local
                // row r by selects (a runtime index into R would put it in local memory)
                n0 = r == 0 ? R[0] : (r == 1 ? R[3] : R[6]);
                n1 = r == 0 ? R[1] : (r == 1 ? R[4] : R[7]);
                n2 = r == 0 ? R[2] : (r == 1 ? R[5] : R[8]);
                nt = r == 0 ? t0 : (r == 1 ? t1 : t2);
            } else {
                float a0 = w0, a1 = w1, a2 = w2, tp = wt;
                if (inf.y != l - 1) {  // branch point: the parent row this lane stored
                    // (its own column s even when inactive: no lane reads another's row)
                    const float* Q = pose + inf.y * 12 * NS + s;
                    a0 = Q[(3 * r + 0) * NS];
                    a1 = Q[(3 * r + 1) * NS];
                    a2 = Q[(3 * r + 2) * NS];
                    tp = Q[(9 + r) * NS];
                }
                n0 = __fmaf_rn(a0, R[0], __fmaf_rn(a1, R[3], __fmul_rn(a2, R[6])));
                n1 = __fmaf_rn(a0, R[1], __fmaf_rn(a1, R[4], __fmul_rn(a2, R[7])));
                n2 = __fmaf_rn(a0, R[2], __fmaf_rn(a1, R[5], __fmul_rn(a2, R[8])));
                nt = __fmaf_rn(a0, t0, __fmaf_rn(a1, t1, __fmaf_rn(a2, t2, tp)));
            }
            if (act) {
                float* W = pose + l * 12 * NS + s;
                W[(3 * r + 0) * NS] = n0;
                W[(3 * r + 1) * NS] = n1;
                W[(3 * r + 2) * NS] = n2;
                W[(9 + r) * NS] = nt;
                // coordinate r of the coarse centre: same expression as pose_pt
                ccen[l * 3 * NS + r * NS + s] = __fmaf_rn(n0, g[33], __fmaf_rn(n1, g[34], __fmaf_rn(n2, g[35], nt)));
            }
            w0 = n0;
            w1 = n1;
            w2 = n2;
            wt = nt;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// exact fine-sphere vs primitive (p indexes spheres, boxes, capsules in that
// order). FP32 with guard band, FP64 exact fallback on the same inputs.
// ---------------------------------------------------------------------------
// cylinder extension, out of line: scenes without cylinders (every bench
// scene) keep the hot loop's instruction footprint
// (scalars and pointers by value: no local-memory copy of the scene view)
__device__ __noinline__ bool fine_vs_cyl(const float* cyl, const double* y64, float eps, float3 x, float rf,
                                         double rd) {
    float d2;
    cyl_d2(x.x, x.y, x.z, cyl, d2);
    const int b = band(d2, rf, eps);
    if (b >= 0) return b != 0;
    return sphere_cylinder_exact(x.x, x.y, x.z, rd, y64);
}
__device__ __noinline__ unsigned long long coarse_mask_cyl(const float* cyl, int nsbc, float x, float y, float z,
                                                           float rc, int p0, int p1) {
    unsigned long long m = 0;
    for (int p = p0; p < p1; ++p) {
        float d2;
        cyl_d2(x, y, z, cyl + (p - nsbc) * CYL_STRIDE, d2);
        if (d2 < rc * rc) m |= 1ull << p;
    }
    return m;
}

__device__ __forceinline__ bool fine_vs_prim(const SceneV& v, float3 x, float rf, double rd, int p) {
    float d2, rr;
    int b;
    if (p < v.ns) {
        const float4 s = v.sph[p];
        sph_d2(x.x, x.y, x.z, s, d2);
        rr = rf + s.w;
        b = band(d2, rr, v.eps);
        if (b >= 0) return b != 0;
        // the FP64 mirror is global: __ldg pins the address space (a plain
        // load here was mis-inferred as shared next to the sh() pointers)
        const double* S = v.s64.s + 4 * p;
        return sphere_sphere_exact(x.x, x.y, x.z, rd, __ldg(S), __ldg(S + 1), __ldg(S + 2), __ldg(S + 3));
    } else if (p < v.ns + v.nb) {
        const int k = p - v.ns;
        box_d2(x.x, x.y, x.z, v.box + k * BOX_STRIDE, d2);
        b = band(d2, rf, v.eps);
        if (b >= 0) return b != 0;
        return sphere_box_exact(x.x, x.y, x.z, rd, v.s64.b + BOX_STRIDE * k);
    } else if (p < v.nsbc) {
        const int k = p - v.ns - v.nb;
        const float* C = v.cap + k * CAP_STRIDE;
        cap_d2(x.x, x.y, x.z, C, d2);
        rr = rf + C[7];
        b = band(d2, rr, v.eps);
        if (b >= 0) return b != 0;
        return sphere_capsule_exact(x.x, x.y, x.z, rd, v.s64.c + CAP_STRIDE * k);
    } else {
        const int k = p - v.nsbc;
        return fine_vs_cyl(v.cyl + k * CYL_STRIDE, v.s64.y + CYL_STRIDE * k, v.eps, x, rf, rd);
    }
}

// 64-bit OR into shared memory as two native 32-bit ATOMS.OR (the 64-bit
// form compiles to a CAS spin loop)
__device__ __forceinline__ void or64_shared(unsigned long long* p, unsigned long long v) {
    unsigned* w = reinterpret_cast<unsigned*>(p);
    if ((unsigned)v) atomicOr(w, (unsigned)v);
    if ((unsigned)(v >> 32)) atomicOr(w + 1, (unsigned)(v >> 32));
}

// algorithmic flops of one sphere test (kernels_detail.hpp:17-50 counted:
// mul/add/sub = 1, FMA = 2): sphere 10, box 27, capsule 22
__device__ __forceinline__ int test_flops(const SceneV& v, int p) {
    return p < v.ns ? 10 : (p < v.ns + v.nb ? 27 : (p < v.nsbc ? 22 : 26));
}

#ifndef PRRTC_COARSE_UNROLL
#define PRRTC_COARSE_UNROLL 1
#endif
#define PRRTC_PRAGMA(x) _Pragma(#x)
#define PRRTC_UNROLL(n) PRRTC_PRAGMA(unroll n)

// coarse (padded) sphere vs primitives [p0, p1): hit bitmask, FP32 only
// (conservative: the padding covers FP32 error, so no fine hit is missed)
__device__ __forceinline__ unsigned long long coarse_mask(const SceneV& v, float x, float y, float z,
                                                          float rc, int p0, int p1) {
    unsigned long long m = 0;
    const int e1 = min(p1, v.ns), e2 = min(p1, v.ns + v.nb);
    int p = p0;
PRRTC_UNROLL(PRRTC_COARSE_UNROLL)
    for (; p < e1; ++p) {
        float d2;
        const float4 s = v.sph[p];
        sph_d2(x, y, z, s, d2);
        const float rr = rc + s.w;
        if (d2 < rr * rr) m |= 1ull << p;
    }
PRRTC_UNROLL(PRRTC_COARSE_UNROLL)
    for (; p < e2; ++p) {
        float d2;
        box_d2(x, y, z, v.box + (p - v.ns) * BOX_STRIDE, d2);
        if (d2 < rc * rc) m |= 1ull << p;
    }
    const int e3 = min(p1, v.nsbc);
PRRTC_UNROLL(PRRTC_COARSE_UNROLL)
    for (; p < e3; ++p) {
        float d2;
        const float* C = v.cap + (p - v.ns - v.nb) * CAP_STRIDE;
        cap_d2(x, y, z, C, d2);
        const float rr = rc + C[7];
        if (d2 < rr * rr) m |= 1ull << p;
    }
    if (p < p1) m |= coarse_mask_cyl(v.cyl, v.nsbc, x, y, z, rc, p, p1);  // cylinders (extension)
    return m;
}
// coarse_mask unrolled 4x (independent primitive tests in flight): the
// brute-force checkers' FP32 pre-mask over every primitive per fine sphere
// (dense checking only, so the planner's hot loop keeps the compact form)
__device__ __forceinline__ unsigned long long coarse_mask_dense(const SceneV& v, float x, float y, float z,
                                                          float rc, int p0, int p1) {
    unsigned long long m = 0;
    const int e1 = min(p1, v.ns), e2 = min(p1, v.ns + v.nb);
    int p = p0;
PRRTC_UNROLL(4)
    for (; p < e1; ++p) {
        float d2;
        const float4 s = v.sph[p];
        sph_d2(x, y, z, s, d2);
        const float rr = rc + s.w;
        if (d2 < rr * rr) m |= 1ull << p;
    }
PRRTC_UNROLL(4)
    for (; p < e2; ++p) {
        float d2;
        box_d2(x, y, z, v.box + (p - v.ns) * BOX_STRIDE, d2);
        if (d2 < rc * rc) m |= 1ull << p;
    }
    const int e3 = min(p1, v.nsbc);
PRRTC_UNROLL(4)
    for (; p < e3; ++p) {
        float d2;
        const float* C = v.cap + (p - v.ns - v.nb) * CAP_STRIDE;
        cap_d2(x, y, z, C, d2);
        const float rr = rc + C[7];
        if (d2 < rr * rr) m |= 1ull << p;
    }
    if (p < p1) m |= coarse_mask_cyl(v.cyl, v.nsbc, x, y, z, rc, p, p1);  // cylinders (extension)
    return m;
}

__device__ __forceinline__ int range_flops(const SceneV& v, int p0, int p1) {
    const int e1 = min(p1, v.ns), e2 = min(p1, v.ns + v.nb), e3 = min(p1, v.nsbc);
    return 10 * max(0, e1 - p0) + 27 * max(0, e2 - max(p0, e1)) + 22 * max(0, e3 - max(p0, e2)) +
           26 * max(0, p1 - max(p0, e3));
}

// self pair fine spheres (collision.cpp:89-98 / kernels_detail.hpp:17-23)
__device__ __forceinline__ bool fine_pair(float eps, const double* fine_r64, float3 a, float ra, int ja,
                                          float3 b, float rb, int jb) {
    float d2;
    sph_d2(a.x, a.y, a.z, make_float4(b.x, b.y, b.z, 0.f), d2);
    const int v = band(d2, ra + rb, eps);
    if (v >= 0) return v != 0;
    return sphere_sphere_exact(a.x, a.y, a.z, __ldg(fine_r64 + ja), b.x, b.y, b.z, __ldg(fine_r64 + jb));
}

// Per-chunk state arrays in registers (shared-memory pointers).
struct ChunkV {
    int* sbad;
    int* sgroup;
    int* ictl;
    int strict;  // exact-CheckStats mode: evaluate every state of the first bad group (see skip_state)
};
__device__ __forceinline__ ChunkV chunk_view(const Ctx& c) {
    return ChunkV{sh(c.sbad), sh(c.sgroup), sh(c.ictl), c.ref_stats};
}

__device__ __forceinline__ void mark_bad(const ChunkV& k, int s) {
    k.sbad[s] = 1;
    atomicMin(&k.ictl[IC_FIRSTBAD], k.sgroup[s]);
}

// skip test for early exit: chain mode skips groups >= first bad (a state
// of a later or the same sub-edge cannot change the outcome); independent
// mode skips states already known bad.
// (In the exact-CheckStats mode only later groups are skipped, so the first
// bad state of the first bad group is known: the reference's sequential
// validation stops exactly there.)
__device__ __forceinline__ bool skip_state(const ChunkV& k, int s, bool early_exit, bool indep) {
    if (!early_exit) return false;
    if (indep) return *(volatile int*)&k.sbad[s] != 0;
    const int fb = *(volatile int*)&k.ictl[IC_FIRSTBAD];
    return k.strict ? k.sgroup[s] > fb : k.sgroup[s] >= fb;
}

// i / n for i = 0..n (edge_sample's t, collision.cpp:19) tabulated once per
// CTA with the same IEEE division, so a state costs no FP64 divide.
__device__ void build_ttab(Ctx& c, int n_cc) {
    const bool ok = n_cc >= 1 && n_cc <= kTTab;
    if (ok) {
        double* tt = sh(c.ttab);
        for (int i = threadIdx.x; i <= n_cc; i += c.nthreads) tt[i] = __ddiv_rn((double)i, (double)n_cc);
    }
    __syncthreads();  // every reader of ttab_n is past here before it changes
    if (ctx_writer(c)) c.ttab_n = ok ? n_cc : 0;
    __syncthreads();
}

// ---------------------------------------------------------------------------
// brute-force fine-only check of the chunk (collision.cpp:100-128): warps
// split fine spheres (resp. self pairs), lanes states.
// ---------------------------------------------------------------------------
// Per-thread test / flop counters kept in registers for the duration of a
// chunk and folded into the context once (the context lives in local memory).
struct StatAcc {
    Ctx& c;
    unsigned long long t = 0, f = 0;
    __device__ explicit StatAcc(Ctx& cc) : c(cc) {}
    __device__ ~StatAcc() {
        unsigned long long* st = sh(c.stat) + 2 * threadIdx.x;
        st[0] += t;
        st[1] += f;
    }
};

// (its own StatAcc: a reference to the caller's would put the caller's
// counters in local memory)
__device__ __noinline__ void brute_chunk(Ctx& c, int cnt, bool early_exit, bool indep) {
    StatAcc acc(c);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = c.nthreads >> 5;
    const int NS = c.NS, S = c.S, NP = c.NP;
    const SceneV v = scene_view(c);
    const ChunkV k = chunk_view(c);
    const float* const pose = sh(c.pose);
    const float4* const fine = sh(c.fine);
    const int* const flink = sh(c.flink);
    const int4* const info = sh(c.info);
    const int* const nfine = sh(c.nfine);
    const int2* const pairs = sh(c.pairs);
    const double* const fine_r64 = c.fine_r64;
    const int pflops = range_flops(v, 0, v.P);
    for (int j = warp; j < S; j += nw) {
        const int l = flink[j];
        const float4 f = fine[j];
        const double rd = __ldg(fine_r64 + j);
        for (int s = lane; s < cnt; s += 32) {
            if (k.sgroup[s] < 0 || skip_state(k, s, early_exit, indep)) continue;
            const float3 x = pose_pt(pose, NS, l, s, f.x, f.y, f.z);
            // every primitive in FP32 first (a mask, as the coarse stage):
            // only those within two guard bands go through the banded test
            // and its exact fallback — the rest are certainly free (band()
            // would return 0), so the verdicts are unchanged
            unsigned long long m = coarse_mask_dense(v, x.x, x.y, x.z, f.w + 2.0f * v.eps, 0, v.P);
            acc.t += v.P;
            acc.f += 18 + pflops;
            while (m) {
                const int p = __ffsll((long long)m) - 1;
                m &= m - 1;
                if (fine_vs_prim(v, x, f.w, rd, p)) {
                    mark_bad(k, s);
                    if (early_exit) {  // the tests after the first hit were not executed
                        acc.t -= v.P - 1 - p;
                        acc.f -= range_flops(v, p + 1, v.P);
                        break;
                    }
                }
            }
        }
    }
    for (int pr = warp; pr < NP; pr += nw) {
        const int2 ab = pairs[pr];
        const int na = nfine[ab.x], nb = nfine[ab.y];
        const int ja0 = info[ab.x].w, jb0 = info[ab.y].w;
        for (int s = lane; s < cnt; s += 32) {
            if (k.sgroup[s] < 0 || skip_state(k, s, early_exit, indep)) continue;
            bool hit = false;
            const PoseR PA = pose_load(pose, NS, ab.x, s), PB = pose_load(pose, NS, ab.y, s);
            for (int i = 0; i < na && !(hit && early_exit); ++i) {
                const float4 fa = fine[ja0 + i];
                const float3 xa = pose_apply(PA, fa.x, fa.y, fa.z);
                for (int q = 0; q < nb; ++q) {
                    const float4 fb = fine[jb0 + q];
                    const float3 xb = pose_apply(PB, fb.x, fb.y, fb.z);
                    ++acc.t;
                    acc.f += 28;
                    if (fine_pair(v.eps, fine_r64, xa, fa.w, ja0 + i, xb, fb.w, jb0 + q)) {
                        hit = true;
                        if (early_exit) break;
                    }
                }
            }
            if (hit) mark_bad(k, s);
        }
    }
}

// ---------------------------------------------------------------------------
// validate the chunk's states (qf/sgroup already set): FK + collision.
// Two-stage (collision.cpp:130-204): padded coarse spheres flag primitives
// per (link, state) into 64-bit masks and self pairs per state into pair
// masks (collision.cpp:155-183); the fine stage re-tests only what flagged
// (collision.cpp:189-203): warps over fine spheres / pairs, lanes over
// states, iterating the set bits. Masks cannot overflow, so no fallback is
// ever needed. Result: sbad[], IC_FIRSTBAD, IC_QN (= anything flagged).
// ---------------------------------------------------------------------------
// stop_flag (nullable): thread 0 samples it once the poses are built and
// publishes it in ictl[IC_STOP] at the stage-1 barrier (or the brute-force
// path's final one), for callers that abandon the chain when the problem
// has been settled meanwhile; the load's latency hides behind stage 1.
// check_chunk_inl is inlined into the planner's single chain-validation site
// (no call boundary per chunk); check_chunk is the out-of-line copy for the
// cold callers (endpoint checks, the batched checking kernels).
__device__ __forceinline__ void check_chunk_inl(Ctx& c, int cnt, bool two_stage, bool early_exit, bool indep,
                                                const int* stop_flag = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = c.nthreads >> 5;
    const int NS = c.NS, L = c.L, NP = c.NP;
    const ChunkV k = chunk_view(c);
    unsigned long long* const lmask = sh(c.lmask);
    unsigned long long* const pmask = sh(c.pmask);
    long long* const prof = c.prof;
    StatAcc acc(c);
    if (prof && tid == 0) prof[1] = clock64();
    fk_chunk(c, cnt);  // also resets sbad / lmask / pmask / IC_QN / IC_FIRSTBAD; ends with __syncthreads
    if (prof && tid == 0) prof[4] = clock64();
    const int stop = (stop_flag && tid == 0) ? ld_relaxed(stop_flag) : 0;
    if (!two_stage) {
        brute_chunk(c, cnt, early_exit, indep);
        if (stop_flag && tid == 0) k.ictl[IC_STOP] = stop;
        __syncthreads();
        return;
    }
    const SceneV v = scene_view(c);
    const float* const pose = sh(c.pose);
    const float* const ccen = sh(c.ccen);
    const float* const geo = sh(c.geo);
    const float4* const fine = sh(c.fine);
    const int* const flink = sh(c.flink);
    const int4* const info = sh(c.info);
    const int* const nfine = sh(c.nfine);
    const int2* const pairs = sh(c.pairs);
    const double* const fine_r64 = c.fine_r64;
    const float cpad = c.cpad;
    // stage 1: the L x P (link, primitive) tests split into nw equal
    // contiguous ranges, one per warp (a warp walks its links' primitive
    // sub-ranges), states over lanes
    int flagged = 0;
    {
        unsigned long long lbits = 0;  // links this thread flagged: the chunk's summary in lany
        const int T = L * v.P, nwlog = 31 - __clz(nw);  // nw: 4, 8 or 16
        const int lo = (T * warp) >> nwlog, hi = (T * (warp + 1)) >> nwlog;
        int l = v.P ? lo / v.P : 0, p0 = lo - l * v.P;  // one division per warp, then walk
        for (int i = lo; i < hi; ++l, p0 = 0) {
            const int p1 = min(v.P, p0 + (hi - i));
            i += p1 - p0;
            const float rc = geo[l * GEO_STRIDE + 36] + cpad;
            const int fl = range_flops(v, p0, p1);
            for (int s = lane; s < cnt; s += 32) {
                if (k.sgroup[s] < 0) continue;
                const float* C = ccen + l * 3 * NS + s;
                const unsigned long long m = coarse_mask(v, C[0], C[NS], C[2 * NS], rc, p0, p1);
                acc.t += p1 - p0;
                acc.f += fl;
                if (m) {
                    or64_shared(&lmask[l * NS + s], m);
                    lbits |= 1ull << l;
                }
            }
        }
        if (lbits) {
            or64_shared(sh(c.lany), lbits);
            flagged = 1;
        }
    }
    if (prof && tid == 0) prof[10] = clock64();  // warp 0's share of the coarse env tests done
    // coarse self pairs (collision.cpp:174-183): pairs over warps, states
    // over lanes; a lane collects its state's pair bits of each 64-pair word
    // in a register and ORs them once
    for (int s = lane; s < cnt; s += 32) {
        if (k.sgroup[s] < 0) continue;
        unsigned long long pm = 0;
        int blk = warp >> 6;
        for (int pr = warp; pr < NP; pr += nw) {
            if ((pr >> 6) != blk) {
                if (pm) {
                    or64_shared(&pmask[blk * NS + s], pm);
                    or64_shared(sh(c.pany) + blk, pm);
                }
                flagged |= pm != 0;
                pm = 0;
                blk = pr >> 6;
            }
            const int2 ab = pairs[pr];
            const float rr = geo[ab.x * GEO_STRIDE + 36] + geo[ab.y * GEO_STRIDE + 36] + 2.0f * cpad;
            const float* A = ccen + ab.x * 3 * NS + s;
            const float* B = ccen + ab.y * 3 * NS + s;
            const float dx = A[0] - B[0], dy = A[NS] - B[NS], dz = A[2 * NS] - B[2 * NS];
            ++acc.t;
            acc.f += 10;
            if (fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr) pm |= 1ull << (pr & 63);
        }
        if (pm) {
            or64_shared(&pmask[blk * NS + s], pm);
            or64_shared(sh(c.pany) + blk, pm);
        }
        flagged |= pm != 0;
    }
    if (stop_flag && tid == 0) k.ictl[IC_STOP] = stop;
    if (prof && tid == 0) prof[11] = clock64();  // warp 0's self pairs done
    const int any_flag = __syncthreads_or(flagged);
    if (prof && tid == 0) prof[5] = clock64();
    if (!any_flag) return;  // nothing flagged: every state free
    if (stop_flag && k.ictl[IC_STOP]) return;  // settled: the caller abandons the chunk
    if (tid == 0) k.ictl[IC_QN] = 1;
    // stage 2a: fine spheres of flagged links vs the primitives that flagged
    // them. Work units of up to three consecutive fine spheres of one link
    // (host-built) over warps, states over lanes: an unflagged (link, state)
    // costs one mask read per unit, a flagged one loads the link pose into
    // registers once for the unit's spheres; small units keep warps balanced
    // when one link collects most of the flags.
    {
        const int2* const funits = sh(c.funits);
        const unsigned long long lany = *sh(c.lany);  // (a unit of a link no state flagged is skipped whole)
        for (int u = warp; u < c.NFU; u += nw) {
            const int2 un = funits[u];
            const int l = un.x, j0 = un.y & 0xffff, j1 = j0 + (un.y >> 16);
            if (!((lany >> l) & 1ull)) continue;
            for (int s = lane; s < cnt; s += 32) {
                const unsigned long long m0 = lmask[l * NS + s];
                if (!m0 || skip_state(k, s, early_exit, indep)) continue;
                const PoseR P = pose_load(pose, NS, l, s);
                for (int j = j0; j < j1; ++j) {
                    if (skip_state(k, s, early_exit, indep)) break;
                    const float4 f = fine[j];
                    const float3 x = pose_apply(P, f.x, f.y, f.z);
                    const double rd = __ldg(fine_r64 + j);
                    acc.f += 18;
                    unsigned long long m = m0;
                    while (m) {
                        const int p = __ffsll((long long)m) - 1;
                        m &= m - 1;
                        ++acc.t;
                        acc.f += test_flops(v, p);
                        if (fine_vs_prim(v, x, f.w, rd, p)) {
                            mark_bad(k, s);
                            break;
                        }
                    }
                }
            }
        }
    }
    if (prof) {
        __syncthreads();
        if (tid == 0) prof[6] = clock64();
    }
    // stage 2b: flagged (pair, state): fine x fine (collision.cpp:89-98);
    // a pair no state flagged is skipped whole
    // (the pairs some state flagged, pany, dealt to the warps round-robin)
    const unsigned long long* const pany = sh(c.pany);
    int pidx = 0;
    for (int w = 0; w < ((NP + 63) >> 6); ++w)
    for (unsigned long long pb = pany[w]; pb; pb &= pb - 1, ++pidx) {
        if ((pidx & (nw - 1)) != warp) continue;
        const int pr = (w << 6) + __ffsll((long long)pb) - 1;
        const int2 ab = pairs[pr];
        const int na = nfine[ab.x], nb = nfine[ab.y];
        const int ja0 = info[ab.x].w, jb0 = info[ab.y].w;
        const float rcb = geo[ab.y * GEO_STRIDE + 36] + 2.0f * cpad;
        for (int s = lane; s < cnt; s += 32) {
            if (!((pmask[(pr >> 6) * NS + s] >> (pr & 63)) & 1ull) || skip_state(k, s, early_exit, indep))
                continue;
            bool hit = false;
            // fine spheres of a that cannot reach b's (padded) coarse sphere
            // cannot hit any fine sphere of b (coarse contains fine,
            // kinematics.cpp:56-57): skip them before the fine x fine loop
            const float* CB = ccen + ab.y * 3 * NS + s;
            const float cbx = CB[0], cby = CB[NS], cbz = CB[2 * NS];
            const PoseR PA = pose_load(pose, NS, ab.x, s), PB = pose_load(pose, NS, ab.y, s);
            for (int i = 0; i < na && !hit; ++i) {
                const float4 fa = fine[ja0 + i];
                const float3 xa = pose_apply(PA, fa.x, fa.y, fa.z);
                {
                    const float dx = xa.x - cbx, dy = xa.y - cby, dz = xa.z - cbz;
                    const float rr = fa.w + rcb;
                    acc.f += 10;
                    if (!(fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr)) continue;
                }
                for (int q = 0; q < nb; ++q) {
                    const float4 fb = fine[jb0 + q];
                    const float3 xb = pose_apply(PB, fb.x, fb.y, fb.z);
                    ++acc.t;
                    acc.f += 28;
                    if (fine_pair(v.eps, fine_r64, xa, fa.w, ja0 + i, xb, fb.w, jb0 + q)) {
                        hit = true;
                        break;
                    }
                }
            }
            if (hit) mark_bad(k, s);
        }
    }
    __syncthreads();
}

__device__ __noinline__ void check_chunk(Ctx& c, int cnt, bool two_stage, bool early_exit, bool indep,
                                         const int* stop_flag = nullptr) {
    check_chunk_inl(c, cnt, two_stage, early_exit, indep, stop_flag);
}

// ---------------------------------------------------------------------------
// Exact CheckStats (collision.hpp:14-37): the reference's counters for one
// checked state, from the chunk's poses and flag masks, following its
// sequential order exactly — two-stage (collision.cpp:130-204): L x P coarse
// tests + one per self pair; if anything flagged, a fine-stage entry and, per
// flagged link in order, fine.n tests per flagging primitive in the order
// spheres, capsules, boxes (fine_link_vs_flagged, collision.cpp:67-87), then
// n_a x n_b per flagged pair (fine_pair_collides, :89-98), stopping at the
// first collision when early_exit; brute force (:100-128): P per fine sphere,
// stopping after the first colliding sphere when early_exit, then n_a x n_b
// per self pair while nothing collided. Cylinders (an extension the reference
// lacks) count as primitives after the boxes. One thread per state; only the
// deterministic (single-CTA replay) mode calls it.
// ---------------------------------------------------------------------------
__device__ bool link_hits_prim(const Ctx& c, const SceneV& v, int l, int p, int s) {
    const int4 inf = sh(c.info)[l];
    const PoseR P = pose_load(sh(c.pose), c.NS, l, s);
    const float4* fine = sh(c.fine);
    for (int j = inf.w; j < inf.w + sh(c.nfine)[l]; ++j) {
        const float4 f = fine[j];
        if (fine_vs_prim(v, pose_apply(P, f.x, f.y, f.z), f.w, __ldg(c.fine_r64 + j), p)) return true;
    }
    return false;
}

__device__ bool pair_hits(const Ctx& c, const SceneV& v, int a, int b, int s) {
    const int ja0 = sh(c.info)[a].w, jb0 = sh(c.info)[b].w, na = sh(c.nfine)[a], nb = sh(c.nfine)[b];
    const PoseR PA = pose_load(sh(c.pose), c.NS, a, s), PB = pose_load(sh(c.pose), c.NS, b, s);
    const float4* fine = sh(c.fine);
    for (int i = 0; i < na; ++i) {
        const float4 fa = fine[ja0 + i];
        const float3 xa = pose_apply(PA, fa.x, fa.y, fa.z);
        for (int q = 0; q < nb; ++q) {
            const float4 fb = fine[jb0 + q];
            if (fine_pair(v.eps, c.fine_r64, xa, fa.w, ja0 + i, pose_apply(PB, fb.x, fb.y, fb.z), fb.w, jb0 + q))
                return true;
        }
    }
    return false;
}

// The reference's coarse flag (kernels_detail.hpp:17-50 in FP64, no padding)
// for link l vs primitive p on the device's posed coarse centre; the FP64
// coarse radii follow the fine radii in fine_r64 (prrtc_robot_create).
__device__ bool coarse_hits_exact(const Ctx& c, const SceneV& v, int l, int p, int s) {
    const float* C = sh(c.ccen) + l * 3 * c.NS + s;
    const double x = C[0], y = C[c.NS], z = C[2 * c.NS], r = __ldg(c.fine_r64 + c.S + l);
    if (p < v.ns) {
        const double* S = v.s64.s + 4 * p;
        return sphere_sphere_exact(x, y, z, r, __ldg(S), __ldg(S + 1), __ldg(S + 2), __ldg(S + 3));
    }
    if (p < v.ns + v.nb) return sphere_box_exact(x, y, z, r, v.s64.b + BOX_STRIDE * (p - v.ns));
    if (p < v.nsbc) return sphere_capsule_exact(x, y, z, r, v.s64.c + CAP_STRIDE * (p - v.ns - v.nb));
    return sphere_cylinder_exact(x, y, z, r, v.s64.y + CYL_STRIDE * (p - v.nsbc));
}

__device__ bool coarse_pair_exact(const Ctx& c, int a, int b, int s) {  // collision.cpp:178-181
    const int NS = c.NS;
    const float* A = sh(c.ccen) + a * 3 * NS + s;
    const float* B = sh(c.ccen) + b * 3 * NS + s;
    const double dx = __dsub_rn(A[0], B[0]), dy = __dsub_rn(A[NS], B[NS]), dz = __dsub_rn(A[2 * NS], B[2 * NS]);
    const double rr = __dadd_rn(__ldg(c.fine_r64 + c.S + a), __ldg(c.fine_r64 + c.S + b));
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)) < __dmul_rn(rr, rr);
}

__device__ __noinline__ unsigned long long ref_state_count(const Ctx& c, int s, bool two_stage, bool early_exit,
                                                          int* fine_entry) {
    const SceneV v = scene_view(c);
    const int L = c.L, NP = c.NP, NS = c.NS;
    const int2* pairs = sh(c.pairs);
    const int* nfine = sh(c.nfine);
    unsigned long long n = 0;
    *fine_entry = 0;
    if (!two_stage) {
        bool hit = false;
        for (int l = 0; l < L && !(hit && early_exit); ++l) {
            const int j0 = sh(c.info)[l].w;
            const PoseR P = pose_load(sh(c.pose), NS, l, s);
            for (int j = j0; j < j0 + nfine[l]; ++j) {
                n += (unsigned long long)v.P;
                const float4 f = sh(c.fine)[j];
                const float3 x = pose_apply(P, f.x, f.y, f.z);
                bool h = false;
                for (int p = 0; p < v.P && !h; ++p) h = fine_vs_prim(v, x, f.w, __ldg(c.fine_r64 + j), p);
                if (h) {
                    hit = true;
                    if (early_exit) break;
                }
            }
        }
        for (int pr = 0; pr < NP && !(hit && early_exit); ++pr) {
            const int2 ab = pairs[pr];
            n += (unsigned long long)nfine[ab.x] * nfine[ab.y];
            if (pair_hits(c, v, ab.x, ab.y, s)) hit = true;
        }
        return n;
    }
    n = (unsigned long long)L * v.P + NP;
    const unsigned long long* lmask = sh(c.lmask);
    const unsigned long long* pmask = sh(c.pmask);
    // the device's coarse masks are padded (a superset): keep the flags the
    // reference's unpadded FP64 coarse tests raise
    bool any = false;
    for (int l = 0; l < L && !any; ++l) {
        unsigned long long m = lmask[l * NS + s];
        while (m && !any) {
            const int p = __ffsll((long long)m) - 1;
            m &= m - 1;
            any = coarse_hits_exact(c, v, l, p, s);
        }
    }
    for (int pr = 0; pr < NP && !any; ++pr)
        any = ((pmask[(pr >> 6) * NS + s] >> (pr & 63)) & 1ull) && coarse_pair_exact(c, pairs[pr].x, pairs[pr].y, s);
    if (!any) return n;
    *fine_entry = 1;
    const int ns = v.ns, nb = v.nb, nsbc = v.nsbc;
    // reference kind order: spheres [0, ns), capsules [ns + nb, nsbc), boxes [ns, ns + nb), then cylinders
    const unsigned long long msph = ns >= 64 ? ~0ull : ((1ull << ns) - 1);
    const unsigned long long mbox = (nb + ns >= 64 ? ~0ull : ((1ull << (ns + nb)) - 1)) & ~msph;
    const unsigned long long mcap = (nsbc >= 64 ? ~0ull : ((1ull << nsbc) - 1)) & ~msph & ~mbox;
    const unsigned long long mcyl = ~(msph | mbox | mcap);
    for (int l = 0; l < L; ++l) {
        const unsigned long long m = lmask[l * NS + s];
        if (!m) continue;
        // fine_link_vs_flagged returns at its first colliding primitive in
        // either mode; early_exit then also ends the whole check
        const unsigned long long order[4] = {m & msph, m & mcap, m & mbox, m & mcyl};
        bool link_hit = false;
        for (int k = 0; k < 4 && !link_hit; ++k) {
            unsigned long long mm = order[k];
            while (mm) {
                const int p = __ffsll((long long)mm) - 1;
                mm &= mm - 1;
                if (!coarse_hits_exact(c, v, l, p, s)) continue;
                n += (unsigned long long)nfine[l];
                if (link_hits_prim(c, v, l, p, s)) {
                    if (early_exit) return n;
                    link_hit = true;
                    break;
                }
            }
        }
    }
    for (int pr = 0; pr < NP; ++pr) {
        const int2 ab = pairs[pr];
        if (!((pmask[(pr >> 6) * NS + s] >> (pr & 63)) & 1ull) || !coarse_pair_exact(c, ab.x, ab.y, s)) continue;
        n += (unsigned long long)nfine[ab.x] * nfine[ab.y];
        if (early_exit && pair_hits(c, v, ab.x, ab.y, s)) return n;
    }
    return n;
}

// ---------------------------------------------------------------------------
// chain states. Points p_0 = A, p_k = lerp(A, B, k/n) (k < n), p_n = B
// (planner.cpp:35-44 step_target; extend is the n = 1 case). State g covers
// sample i = g % n_cc + 1 of sub-edge k = g / n_cc (collision.cpp:13-21:
// the far endpoint is copied exactly); a bitwise-equal sub-edge collapses to
// one check of its far end (collision.cpp:215). The chunk's chain points are
// computed once into `ends` (each is a full lerp with one FP64 division)
// and reused by the states and by the appends.
// ---------------------------------------------------------------------------
__device__ __noinline__ double chain_point(const double* A, const double* B, int d, long long k,
                                           long long n) {
    if (k == 0) return A[d];
    if (k >= n) return B[d];
    return lerp_exact(A[d], B[d], __ddiv_rn((double)k, (double)n));
}

// Returns the number of active states (each thread owns at most one: NS <= nthreads).
__device__ __noinline__ double frac_div(int i, int n) { return __ddiv_rn((double)i, (double)n); }

// Chain indices are 32-bit: a chain holds n_sub * n_cc < 2^30 states (the
// caller rejects longer ones; joint limits bound n_sub to a few dozen).
// stop_flag (nullable): thread 0 issues a relaxed load of it on entry and
// publishes the value in ictl[IC_STOP] just before the final barrier, so the
// caller can abandon the chunk without a barrier pair of its own.
__device__ __forceinline__ int gen_chain_states_inl(Ctx& c, const double* A, const double* B, long long n_sub,
                                                    int n_cc, long long g0l, int cnt, const int* stop_flag) {
    const int tid = threadIdx.x, dof = c.dof, NS = c.NS, nthreads = c.nthreads;
    const int stop = (stop_flag && tid == 0) ? ld_relaxed(stop_flag) : 0;
    double* const ends = sh(c.ends);
    int* const sgroup = sh(c.sgroup);
    float* const qf = sh(c.qf);
    const double* const ttab = n_cc == c.ttab_n ? sh(c.ttab) : nullptr;
    const unsigned ncc = (unsigned)n_cc, g0 = (unsigned)g0l;
    if (n_sub == 1) {
        // a single edge (extend, path checks): states straight from A and B,
        // one (state, dimension) item per thread, no chain-point staging
        const double* As = sh(A);
        const double* Bs = sh(B);
        bool eq = true;  // bitwise-equal edge: one check of the far end (collision.cpp:215)
        for (int d = 0; d < dof; ++d) eq &= As[d] == Bs[d];
        for (int idx = tid; idx < dof * NS; idx += nthreads) {
            const int d = idx >> c.nslog, s = idx & (NS - 1);
            const int i = (int)g0 + s + 1;
            const bool act = s < cnt && !(eq && i != n_cc);
            if (d == 0) sgroup[s] = act ? 0 : -1;
            if (!act) continue;
            qf[idx] = i == n_cc ? (float)Bs[d]
                                : (float)lerp_exact(As[d], Bs[d], ttab ? ttab[i] : frac_div(i, n_cc));
        }
        if (tid == 0) sh(c.ictl)[IC_STOP] = stop;
        __syncthreads();
        return eq ? ((int)g0 + cnt == n_cc ? 1 : 0) : cnt;
    }
    const unsigned k_lo = g0 / ncc;
    const int npts = (int)((g0 + cnt - 1) / ncc - k_lo) + 2;
    for (int idx = tid; idx < npts * dof; idx += nthreads) {
        const int j = idx / dof, d = idx - j * dof;
        ends[idx] = chain_point(A, B, d, (long long)(k_lo + j), n_sub);
    }
    if (tid == 0) sh(c.ictl)[IC_KLO] = (int)k_lo;
    __syncthreads();
    int mine = 0;
    for (int s = tid; s < NS; s += nthreads) {
        if (s >= cnt) {
            sgroup[s] = -1;
            continue;
        }
        const unsigned g = g0 + s;
        const unsigned k = g / ncc;
        const int i = (int)(g - k * ncc) + 1;
        const int j = (int)(k - k_lo);
        const double* F = ends + j * dof;
        const double* T = F + dof;
        bool eq = i != n_cc;  // a bitwise-equal sub-edge: only its far end is checked
        for (int d = 0; eq && d < dof; ++d) eq = F[d] == T[d];
        if (eq) {
            sgroup[s] = -1;
            continue;
        }
        if (i == n_cc) {
            for (int d = 0; d < dof; ++d) qf[d * NS + s] = (float)T[d];
        } else {
            const double t = ttab ? ttab[i] : frac_div(i, n_cc);
            for (int d = 0; d < dof; ++d) qf[d * NS + s] = (float)lerp_exact(F[d], T[d], t);
        }
        sgroup[s] = (int)k;
        ++mine;
    }
    if (tid == 0) sh(c.ictl)[IC_STOP] = stop;
    return __syncthreads_count(mine);
}

__device__ __noinline__ int gen_chain_states(Ctx& c, const double* A, const double* B, long long n_sub, int n_cc,
                                             long long g0l, int cnt, const int* stop_flag) {
    return gen_chain_states_inl(c, A, B, n_sub, n_cc, g0l, cnt, stop_flag);
}

// ---------------------------------------------------------------------------
// nearest neighbour over the published prefix of a tree (nn.cpp:22-29,
// kernels_scalar.cpp:9-37): exact FP64 keys in the scalar summation order
// over SoA rows, 128-bit loads (two nodes per load; plain L1-allocating
// loads: every slot below the snapshot was released before the caller's
// acquire of `published`, which also invalidates stale L1 lines, so the
// follow-up reads of the winner's config and dynamic-domain flag — both
// prefetched into L1 here — hit L1), per-thread strict-< argmin over
// increasing indices, then warp-shuffle and cross-warp argmin with ties to
// the lowest index. One routine serves one sample (m = 1) and the planner's
// multi-sample passes: m <= 32 samples over the same published prefix in one
// pass, g = nthreads / next_pow2(m) threads per sample striding the node
// pairs, then a segmented shuffle argmin (ties to the lowest index) — or, for
// g > 32, the cross-warp step. Results for sample j land in mnn_d[j] /
// mnn_i[j]; ends with a barrier.
// ---------------------------------------------------------------------------
// With `accept` set, the reducing thread of sample j also evaluates the
// planner's acceptance right away (duplicate, planner.cpp:218; dynamic
// domain with radius R when ddf is given, sampling.hpp:61-75) into
// mnn_ok[j], saving the caller a pass and a barrier.
__device__ __noinline__ void nn_scan_multi(Ctx& c, const double* cfg, long long cap, int count,
                                           const double* Q, int m, const int* ddf, bool accept = false,
                                           double R = 0.0) {
    __shared__ double s_md[32];
    __shared__ int s_mi[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, dof = c.dof, nt = c.nthreads;
    Q = sh(Q);
    double* const out_d = sh(c.mnn_d);
    int* const out_i = sh(c.mnn_i);
    int mplog = 0;
    while ((1 << mplog) < m) ++mplog;
    const int glog = (31 - __clz(nt)) - mplog;  // threads per sample g = nt / next_pow2(m) (a power of two)
    const int g = 1 << glog;
    const int j = tid >> glog, sub = tid & (g - 1);
    double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int bi = 0x7fffffff;
    const int npairs = (count + 1) >> 1;
    if (j < m) {
        const double* q = Q + j * dof;
        // kNnPairs node pairs per trip (pi, pi + g, ...: 2 x kNnPairs
        // independent FP64 accumulation chains), dimensions loaded
        // 8 / kNnPairs at a time for all of them (8 double2 of registers, as
        // one pair 8 at a time); the pairs are still visited in increasing
        // index order, so strict-< keeps the lowest index on ties
        constexpr int NP = kNnPairs, ND = 8 / kNnPairs;
        for (int pi = sub; pi < npairs; pi += NP * g) {
            int nn_[NP];
            bool in_[NP];
#pragma unroll
            for (int r = 0; r < NP; ++r) {
                in_[r] = pi + r * g < npairs;
                nn_[r] = in_[r] ? (pi + r * g) * 2 : pi * 2;  // (a clamped duplicate load when absent)
                if (ddf && in_[r]) asm volatile("prefetch.global.L1 [%0];" ::"l"(ddf + nn_[r]));
            }
            double acc[NP][2];
#pragma unroll
            for (int r = 0; r < NP; ++r) acc[r][0] = acc[r][1] = 0.0;
            for (int d0 = 0; d0 < dof; d0 += ND) {
                double2 v[NP][ND];
#pragma unroll
                for (int k = 0; k < ND; ++k)  // every slot assigned: v stays in registers
#pragma unroll
                    for (int r = 0; r < NP; ++r)
                        v[r][k] = d0 + k < dof ? *reinterpret_cast<const double2*>(cfg + (d0 + k) * cap + nn_[r])
                                               : make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 0; k < ND; ++k) {
                    if (d0 + k < dof) {
                        const double qd = q[d0 + k];
#pragma unroll
                        for (int r = 0; r < NP; ++r) {
                            const double e0 = __dsub_rn(v[r][k].x, qd), e1 = __dsub_rn(v[r][k].y, qd);
                            acc[r][0] = __dadd_rn(acc[r][0], __dmul_rn(e0, e0));
                            acc[r][1] = __dadd_rn(acc[r][1], __dmul_rn(e1, e1));
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < NP; ++r) {
                if (!in_[r]) continue;
                if (acc[r][0] < best) {
                    best = acc[r][0];
                    bi = nn_[r];
                }
                if (nn_[r] + 1 < count && acc[r][1] < best) {
                    best = acc[r][1];
                    bi = nn_[r] + 1;
                }
            }
        }
    }
    for (int o = min(g, 32) >> 1; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (g <= 32) {
        if (sub == 0 && j < m) {
            out_d[j] = best;
            out_i[j] = bi;
            if (accept) sh(c.mnn_ok)[j] = best != 0.0 && !(ddf && ddf[bi] && !(__dsqrt_rn(best) <= R));
        }
    } else {
        if (lane == 0) {
            s_md[w] = best;
            s_mi[w] = bi;
        }
        __syncthreads();
        const int wpg = g >> 5;  // warps per sample
        if (tid < m) {
            double b = s_md[tid * wpg];
            int i = s_mi[tid * wpg];
            for (int k = 1; k < wpg; ++k) {
                const double ob = s_md[tid * wpg + k];
                const int oi = s_mi[tid * wpg + k];
                if (ob < b || (ob == b && oi < i)) {
                    b = ob;
                    i = oi;
                }
            }
            out_d[tid] = b;
            out_i[tid] = i;
            if (accept) sh(c.mnn_ok)[tid] = b != 0.0 && !(ddf && ddf[i] && !(__dsqrt_rn(b) <= R));
        }
    }
    __syncthreads();
}

}  // namespace dev
}  // namespace prrtc_b200
