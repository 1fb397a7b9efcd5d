// prrtc_warp.cuh — the warp-worker batch planner (included by prrtc_kernels.cu).
//
// plan_kernel (prrtc_kernels.cu) runs one RRT-Connect worker per CTA: every
// phase of an iteration (sample, NN, steer, FK, coarse, fine, append, connect)
// is a CTA-wide step between barriers, which is what a single problem needs
// (148 CTAs x 16 warps on one search) but leaves a batch latency-bound: ncu of
// the headline batch shows 16 warps per SM, 38% issue, the barrier and
// L2-round-trip stalls on top (profiles/r2b_plan_kernel.md), and the phase
// tracer ~20k SM cycles per 32-state validation chunk.
//
// plan_warp_kernel gives every WARP its own worker (planner.cpp:186-242):
// one CTA per SM holds as many warp workers as the shared memory allows
// (14 for Panda), each with its own problem, scene copy and buffers, synced
// by __syncwarp only. A validation chunk is 32 states, one per lane, and a
// lane runs its state end to end in registers:
//   forward kinematics link by link (kinematics.cpp:92-103; the same FP32
//   fmaf sequence as fk_chunk, so posed spheres are bit-identical),
//   the link's coarse sphere against every primitive (collision.cpp:155-170)
//   right after its pose exists, the link's fine spheres against the
//   primitives that flagged (collision.cpp:189-196) while the pose is still
//   in registers, and the self pairs whose higher link it is (coarse,
//   collision.cpp:174-183; fine x fine, :197-203) against the stored pose of
//   the lower link;
// early exit is a ballot per link (the first bad sub-edge, collision.cpp:
// 216-222, is the group of the lowest bad lane: groups grow with the lane).
// Verdicts are the same function of the state as check_chunk's (the coarse
// stage is padded, the fine predicates and their FP64 fallback are shared),
// so the planner's search semantics are unchanged; only the schedule is.
//
// The tree protocol (reserve, write, release, publishing CAS, carry),
// tickets, help mode and termination are plan_kernel's, at warp scope.
#pragma once

// (included inside namespace prrtc_b200, after the CTA planner's helpers)

constexpr unsigned kFull = 0xffffffffu;

// CTA-shared view of the robot and the per-warp layout (shared memory,
// written by thread 0): byte offsets into the dynamic shared memory window.
struct WCtx {
    int L, dof, S, NP, nstore, fkflops;
    unsigned o_info, o_nfine, o_geo, o_fine, o_bases, o_magic;  // robot words
    unsigned o_lim, o_htab, o_ttab;  // [dof][2] limits, [dof][kHaltonTab] Halton table, [n_cc + 1] i / n_cc
    unsigned o_pstart, o_plo, o_slot;  // self pairs by higher link: [L + 1] starts; [NP] (lower link | its
                                       // store slot << 16, coarse radius sum bits); [L] store slot
    int ttab_n;
    unsigned warp0, per_warp;           // first warp region, region size
    unsigned w_scene, w_pose, w_ccen, w_qf, w_sbuf, w_dcfg;  // offsets inside a warp region
    int walk_cap;                       // ints of the pose store usable by path assembly
};
__shared__ WCtx g_w;

template <class T>
__device__ __forceinline__ T* smo(unsigned off) {
    return reinterpret_cast<T*>(g_dsmem + off);
}

struct WarpLayout {
    size_t robot, lim, htab, ttab, pstart, plo, slot, shared_end;
    size_t scene, pose, ccen, qf, sbuf, dcfg, per_warp;
};

// dcfg rows of a warp region
enum : int { WD_A = 0, WD_NEW, WD_TGT, WD_NN, WD_COUNT };

__host__ __device__ inline WarpLayout warp_layout(int robot_words, int L, int dof, int NP, int nstore,
                                                  int scene_words) {
    WarpLayout w;
    size_t o = 0;
    w.robot = o; o = al16(o + 4 * (size_t)robot_words);
    w.lim = o;   o = al16(o + 8 * (size_t)dof * 2);
    w.htab = o;  o = al16(o + 8 * (size_t)dof * kHaltonTab);
    w.ttab = o;  o = al16(o + 8 * (size_t)(kTTab + 1));
    w.pstart = o; o = al16(o + 4 * (size_t)(L + 1));
    w.plo = o;   o = al16(o + 8 * (size_t)(NP > 0 ? NP : 1));
    w.slot = o;  o = al16(o + 4 * (size_t)L);
    w.shared_end = o;
    size_t p = 0;
    w.scene = p; p = al16(p + 4 * (size_t)scene_words);
    w.pose = p;  p = al16(p + 4 * (size_t)nstore * 12 * 32);
    w.ccen = p;  p = al16(p + 4 * (size_t)nstore * 3 * 32);
    w.qf = p;    p = al16(p + 4 * (size_t)dof * 32);
    w.sbuf = p;  p = al16(p + 8 * (size_t)32 * dof);
    w.dcfg = p;  p = al16(p + 8 * (size_t)WD_COUNT * dof);
    w.per_warp = p;
    return w;
}

// Links whose pose a lane keeps in its store: the lower link of every self
// pair (read when the higher link is posed) and every parent that is not the
// previous link (branch points of a kinematic tree, e.g. Baxter's torso).
__host__ __device__ inline int warp_store_count(const int4* info, const int2* pairs, int L, int NP, int* slot) {
    int n = 0;
    for (int l = 0; l < L; ++l) {
        bool need = false;
        for (int m = l + 1; m < L && !need; ++m) need = info[m].y == l && l != m - 1;
        for (int p = 0; p < NP && !need; ++p) need = (pairs[p].x < pairs[p].y ? pairs[p].x : pairs[p].y) == l;
        if (slot) slot[l] = need ? n : -1;
        n += need;
    }
    return n;
}

// ---------------------------------------------------------------------------
// per-warp scene view (registers)
// ---------------------------------------------------------------------------
__device__ __forceinline__ SceneV warp_scene(const uint32_t* sw, SceneF64 f64, float* cpad) {
    SceneV v;
    v.ns = sw[SH_NS];
    v.nb = sw[SH_NB];
    v.nsbc = v.ns + v.nb + sw[SH_NC];
    v.P = v.nsbc + sw[SH_NY];
    v.sph = reinterpret_cast<const float4*>(sw + sw[SH_OFF_S]);
    v.box = reinterpret_cast<const float*>(sw + sw[SH_OFF_B]);
    v.cap = reinterpret_cast<const float*>(sw + sw[SH_OFF_C]);
    v.cyl = reinterpret_cast<const float*>(sw + sw[SH_OFF_Y]);
    v.eps = __uint_as_float(sw[SH_EPS]);
    v.s64 = f64;
    *cpad = __uint_as_float(sw[SH_CPAD]);
    return v;
}

__device__ __forceinline__ void warp_load_scene(uint32_t* sw, const uint32_t* scene_g, int lane) {
    __syncwarp();
    const int words = __ldg(scene_g + SH_WORDS);
    for (int i = lane; i < words; i += 32) sw[i] = __ldg(scene_g + i);
    __syncwarp();
}

// ---------------------------------------------------------------------------
// one lane, one state: FK + two-stage collision, early exit by ballot.
// q: this lane's column of the warp's qf[dof][32]. group: the state's
// sub-edge (chain mode) — lanes hold increasing groups; indep: states are
// independent (endpoint checks), a lane stops only at its own hit.
// Returns whether the lane's state collides (undefined for inactive lanes).
// ---------------------------------------------------------------------------
struct LaneAcc {
    unsigned long long t = 0, f = 0;  // sphere tests, algorithmic flops
};

__device__ __forceinline__ bool lane_check(const SceneV& v, float cpad, const double* fine_r64, const float* qf,
                                           float* pstore, float* cstore, bool active, int group, bool early_exit,
                                           bool indep, bool two_stage, LaneAcc& acc, bool* flagged) {
    const int lane = threadIdx.x & 31;
    const int L = g_w.L;
    const int4* const info = smo<int4>(g_w.o_info);
    const int* const nfine = smo<int>(g_w.o_nfine);
    const float* const geo = smo<float>(g_w.o_geo);
    const float4* const fine = smo<float4>(g_w.o_fine);
    const int* const pstart = smo<int>(g_w.o_pstart);
    const int2* const plo = smo<int2>(g_w.o_plo);
    const int* const slot = smo<int>(g_w.o_slot);
    const int pflops = range_flops(v, 0, v.P);
    bool bad = false, live = active, flag = false;
    PoseR W;  // the previous link's world pose (rows: R 0..8, t 9..11)
#pragma unroll
    for (int k = 0; k < 12; ++k) W.m[k] = 0.f;
    for (int l = 0; l < L; ++l) {
        if (early_exit) {
            const unsigned bm = __ballot_sync(kFull, bad);
            if (bm) {
                if (indep) {
                    live = live && !bad;
                } else {
                    const int fg = __shfl_sync(kFull, group, __ffs(bm) - 1);
                    live = live && group < fg;
                }
            }
            if (!__any_sync(kFull, live)) break;
        }
        const int4 inf = info[l];
        float g[37];
#pragma unroll
        for (int k = 0; k < 9; ++k)
            reinterpret_cast<float4*>(g)[k] = reinterpret_cast<const float4*>(geo + l * GEO_STRIDE)[k];
        g[36] = geo[l * GEO_STRIDE + 36];
        // local transform (fk_chunk's expressions)
        float R[9], t0, t1, t2;
        if (inf.x == PRRTC_JOINT_REVOLUTE) {
            float sn, cs;
            sincos_joint(qf[inf.z * 32 + lane], &sn, &cs);
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
                const float q = qf[inf.z * 32 + lane];
                t0 = __fmaf_rn(g[30], q, g[27]);
                t1 = __fmaf_rn(g[31], q, g[28]);
                t2 = __fmaf_rn(g[32], q, g[29]);
            } else {
                t0 = g[27];
                t1 = g[28];
                t2 = g[29];
            }
        }
        // world = world_parent * local, row by row (fk_chunk's fmaf order)
        if (inf.y < 0) {
#pragma unroll
            for (int k = 0; k < 9; ++k) W.m[k] = R[k];
            W.m[9] = t0;
            W.m[10] = t1;
            W.m[11] = t2;
        } else {
            if (inf.y != l - 1) {  // branch point: the parent's stored pose
                const float* Q = pstore + slot[inf.y] * 12 * 32 + lane;
#pragma unroll
                for (int k = 0; k < 12; ++k) W.m[k] = Q[k * 32];
            }
            float n[12];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const float a0 = W.m[3 * r], a1 = W.m[3 * r + 1], a2 = W.m[3 * r + 2], tp = W.m[9 + r];
                n[3 * r + 0] = __fmaf_rn(a0, R[0], __fmaf_rn(a1, R[3], __fmul_rn(a2, R[6])));
                n[3 * r + 1] = __fmaf_rn(a0, R[1], __fmaf_rn(a1, R[4], __fmul_rn(a2, R[7])));
                n[3 * r + 2] = __fmaf_rn(a0, R[2], __fmaf_rn(a1, R[5], __fmul_rn(a2, R[8])));
                n[9 + r] = __fmaf_rn(a0, t0, __fmaf_rn(a1, t1, __fmaf_rn(a2, t2, tp)));
            }
#pragma unroll
            for (int k = 0; k < 12; ++k) W.m[k] = n[k];
        }
        // coarse centre: pose_pt's expression
        const float cx = __fmaf_rn(W.m[0], g[33], __fmaf_rn(W.m[1], g[34], __fmaf_rn(W.m[2], g[35], W.m[9])));
        const float cy = __fmaf_rn(W.m[3], g[33], __fmaf_rn(W.m[4], g[34], __fmaf_rn(W.m[5], g[35], W.m[10])));
        const float cz = __fmaf_rn(W.m[6], g[33], __fmaf_rn(W.m[7], g[34], __fmaf_rn(W.m[8], g[35], W.m[11])));
        const int sl = slot[l];
        if (sl >= 0) {
            float* Pw = pstore + sl * 12 * 32 + lane;
#pragma unroll
            for (int k = 0; k < 12; ++k) Pw[k * 32] = W.m[k];
            float* Cw = cstore + sl * 3 * 32 + lane;
            Cw[0] = cx;
            Cw[32] = cy;
            Cw[64] = cz;
        }
        if (!live) continue;
        const int j0 = inf.w, j1 = inf.w + nfine[l];
        if (two_stage) {
            // stage 1: this link's padded coarse sphere vs every primitive
            const unsigned long long m = coarse_mask(v, cx, cy, cz, g[36] + cpad, 0, v.P);
            acc.t += v.P;
            acc.f += pflops;
            if (m) {
                flag = true;
                // stage 2a: the link's fine spheres vs the flagging primitives
                for (int j = j0; j < j1 && !bad; ++j) {
                    const float4 f = fine[j];
                    const float3 x = pose_apply(W, f.x, f.y, f.z);
                    const double rd = __ldg(fine_r64 + j);
                    acc.f += 18;
                    unsigned long long mm = m;
                    while (mm) {
                        const int p = __ffsll((long long)mm) - 1;
                        mm &= mm - 1;
                        ++acc.t;
                        acc.f += test_flops(v, p);
                        if (fine_vs_prim(v, x, f.w, rd, p)) {
                            bad = true;
                            break;
                        }
                    }
                }
            }
        } else {
            // brute force (collision.cpp:100-128): every fine sphere vs every
            // primitive (an FP32 pre-mask, as brute_chunk: verdicts unchanged)
            for (int j = j0; j < j1 && !(bad && early_exit); ++j) {
                const float4 f = fine[j];
                const float3 x = pose_apply(W, f.x, f.y, f.z);
                const double rd = __ldg(fine_r64 + j);
                unsigned long long mm = coarse_mask_dense(v, x.x, x.y, x.z, f.w + 2.0f * v.eps, 0, v.P);
                acc.t += v.P;
                acc.f += 18 + pflops;
                while (mm) {
                    const int p = __ffsll((long long)mm) - 1;
                    mm &= mm - 1;
                    if (fine_vs_prim(v, x, f.w, rd, p)) {
                        bad = true;
                        break;
                    }
                }
            }
        }
        // self pairs whose higher link is l (collision.cpp:174-183, 197-203)
        for (int e = pstart[l]; e < pstart[l + 1] && !(bad && early_exit); ++e) {
            const int2 pe = plo[e];
            const int a = pe.x & 0xffff, sa = pe.x >> 16;
            const float* CA = cstore + sa * 3 * 32 + lane;
            const float ax = CA[0], ay = CA[32], az = CA[64];
            if (two_stage) {
                const float rr = __int_as_float(pe.y) + 2.0f * cpad;  // (r_a + r_l) + 2 cpad
                const float dx = ax - cx, dy = ay - cy, dz = az - cz;
                ++acc.t;
                acc.f += 10;
                if (!(fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr)) continue;
                flag = true;
            }
            // fine x fine: spheres of l that cannot reach a's padded coarse
            // sphere cannot hit any of a's fine spheres (kinematics.cpp:56-57)
            const PoseR PA = pose_load(pstore + lane, 32, sa, 0);
            const int ja0 = info[a].w, na = nfine[a];
            const float rca = geo[a * GEO_STRIDE + 36] + 2.0f * cpad;
            // (brute force without early exit runs every fine x fine test,
            // collision.cpp:89-98 as the dense CheckStats count them)
            const bool all_tests = !two_stage && !early_exit;
            bool hit = false;
            for (int i = j0; i < j1 && !(hit && !all_tests); ++i) {
                const float4 fb = fine[i];
                const float3 xb = pose_apply(W, fb.x, fb.y, fb.z);
                if (two_stage) {
                    const float dx = xb.x - ax, dy = xb.y - ay, dz = xb.z - az;
                    const float rr = fb.w + rca;
                    acc.f += 10;
                    if (!(fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rr * rr)) continue;
                }
                for (int q = 0; q < na; ++q) {
                    const float4 fa = fine[ja0 + q];
                    const float3 xa = pose_apply(PA, fa.x, fa.y, fa.z);
                    ++acc.t;
                    acc.f += 28;
                    if (fine_pair(v.eps, fine_r64, xa, fa.w, ja0 + q, xb, fb.w, i)) {
                        hit = true;
                        if (!all_tests) break;
                    }
                }
            }
            bad = bad || hit;
        }
    }
    *flagged = flag;
    return bad;
}

// ---------------------------------------------------------------------------
// warp-scope helpers of the planner loop
// ---------------------------------------------------------------------------
struct WarpRegion {
    uint32_t* scene;
    float* pose;
    float* ccen;
    float* qf;
    double* sbuf;
    double* dcfg;
};

__device__ __forceinline__ WarpRegion warp_region(int wid) {
    const unsigned base = g_w.warp0 + (unsigned)wid * g_w.per_warp;
    WarpRegion r;
    r.scene = smo<uint32_t>(base + g_w.w_scene);
    r.pose = smo<float>(base + g_w.w_pose);
    r.ccen = smo<float>(base + g_w.w_ccen);
    r.qf = smo<float>(base + g_w.w_qf);
    r.sbuf = smo<double>(base + g_w.w_sbuf);
    r.dcfg = smo<double>(base + g_w.w_dcfg);
    return r;
}

__device__ void finish_problem_w(const PlanArgs& a, int prob, int done, int msg) {
    ProbCtl& C = a.ctl[prob];
    if (atomicCAS(&C.done, DONE_RUNNING, -1) == DONE_RUNNING) {  // claim
        C.msg = msg;
        C.t_end_ns = globaltimer();
        __threadfence();
        st_release(&C.done, done);
        atomicAdd(a.n_done, 1);
    }
}

// Chain states g0 .. g0 + 31 of the chain A -> B in n_sub sub-edges (lane =
// state; gen_chain_states_inl's arithmetic per lane): writes the lane's qf
// column, returns whether the lane holds an active state and its group.
__device__ __forceinline__ bool warp_gen_state(const double* A, const double* B, long long n_sub, int n_cc,
                                               long long total, long long g0, float* qf, int* group) {
    const int lane = threadIdx.x & 31, dof = g_w.dof;
    const long long g = g0 + lane;
    if (g >= total) {
        *group = 0x7fffffff;
        return false;
    }
    const unsigned ncc = (unsigned)n_cc;
    const unsigned k = (unsigned)g / ncc;
    const int i = (int)((unsigned)g - k * ncc) + 1;
    *group = (int)k;
    const double* const ttab = n_cc == g_w.ttab_n ? smo<double>(g_w.o_ttab) : nullptr;
    const double ti = i == n_cc ? 1.0 : (ttab ? ttab[i] : __ddiv_rn((double)i, (double)n_cc));
    // chain points p_k, p_{k+1} (chain_point: k / n_sub by one IEEE division)
    const bool kin = k > 0 && (long long)k < n_sub, k1in = (long long)k + 1 < n_sub;
    const double tk = kin ? __ddiv_rn((double)k, (double)n_sub) : 0.0;
    const double tk1 = k1in ? __ddiv_rn((double)(k + 1), (double)n_sub) : 0.0;
    bool eq = true;
    for (int d = 0; d < dof; ++d) {
        const double ad = A[d], bd = B[d];
        const double F = k == 0 ? ad : ((long long)k >= n_sub ? bd : lerp_exact(ad, bd, tk));
        const double T = k1in ? lerp_exact(ad, bd, tk1) : bd;
        eq = eq && F == T;
        qf[d * 32 + lane] = (float)(i == n_cc ? T : lerp_exact(F, T, ti));
    }
    // a bitwise-equal sub-edge is one check of its far end (collision.cpp:215)
    return !(eq && i != n_cc);
}

// Append `count` chained nodes p_{k0}, p_{k0+1}, ... of the chain A -> B
// (n_sub sub-edges; count = 1 with n_sub = 1 appends B) — tree_append_many
// at warp scope: one reservation, lanes write, one publishing CAS, carry.
__device__ int warp_append(const PlanArgs& a, const TreeRef& T, const double* A, const double* B, long long n_sub,
                           long long k0, int count, int parent0, int* last, int* known) {
    const int lane = threadIdx.x & 31, dof = g_w.dof;
    long long s0 = 0;
    if (lane == 0) s0 = atomicAdd(T.reserved, count);
    s0 = __shfl_sync(kFull, s0, 0);
    const int ok = (int)max(0ll, min((long long)count, a.cap - s0));
    for (int idx = lane; idx < ok * dof; idx += 32) {
        const int j = idx / dof, d = idx - j * dof;
        T.cfg[(size_t)d * a.stride + s0 + j] = n_sub == 1 ? B[d] : chain_point(A, B, d, k0 + j, n_sub);
    }
    for (int j = lane; j < ok; j += 32) {
        T.parent[s0 + j] = j == 0 ? parent0 : (int)(s0 + j - 1);
        T.dd[s0 + j] = 0;
        T.ready[s0 + j] = a.epoch;
    }
    __threadfence();  // data and flags before the publishing CAS
    __syncwarp();
    if (ok > 0) {
        int won = 0;
        if (lane == 0) won = atomicCAS(T.published, (int)s0, (int)(s0 + ok)) == s0;
        won = __shfl_sync(kFull, won, 0);
        if (won && *known == (int)s0) *known = (int)(s0 + ok);
        if (won) {  // carry `published` over successors that finished first (see tree_append_many)
            int p = (int)(s0 + ok);
            while (p < a.cap) {
                __threadfence();
                const long long idx = (long long)p + lane;
                const bool r = idx < a.cap && ld_acquire_u(&T.ready[idx]) == a.epoch;
                const bool settled = lane == 0 && ld_relaxed(T.done) != 0;
                const unsigned m = __ballot_sync(kFull, r);
                const int run = (m == kFull) ? 32 : (__ffs(~m) - 1);
                if (run == 0 || __any_sync(kFull, settled)) break;
                int old = 0;
                fence_acq_rel();
                if (lane == 0) old = atomicCAS(T.published, p, p + run);
                old = __shfl_sync(kFull, old, 0);
                if (old != p) break;
                p += run;
            }
        }
    }
    *last = ok > 0 ? (int)(s0 + ok - 1) : parent0;
    return ok;
}

// nearest neighbour(s) over the published prefix (nn_scan_multi at warp
// scope): m <= 32 samples, g = 32 / next_pow2(m) lanes per sample striding
// node pairs, FP64 keys in the scalar order, strict-< per lane over
// increasing indices, segmented shuffle argmin (ties to the lowest index).
// With accept, *first = the first sample that is not a duplicate and lies in
// its node's dynamic domain (planner.cpp:216-219, sampling.hpp:61-75), m if
// none; its node index and d2 are returned (sample 0's without accept).
__device__ __forceinline__ void warp_nn(const double* cfg, long long stride, int count, const double* Q, int m,
                                        const int* ddf, bool accept, double R, int* first, int* nn, double* d2) {
    const int lane = threadIdx.x & 31, dof = g_w.dof;
    int mplog = 0;
    while ((1 << mplog) < m) ++mplog;
    const int glog = 5 - mplog, gsz = 1 << glog;
    const int j = lane >> glog, sub = lane & (gsz - 1);
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int bi = 0x7fffffff;
    const int npairs = (count + 1) >> 1;
    if (j < m) {
        const double* q = Q + j * dof;
        for (int pi = sub; pi < npairs; pi += gsz) {
            const int n0 = pi * 2;
            double a0 = 0.0, a1 = 0.0;
            if (ddf) asm volatile("prefetch.global.L1 [%0];" ::"l"(ddf + n0));
            for (int d0 = 0; d0 < dof; d0 += 8) {
                double2 v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    v[k] = d0 + k < dof ? *reinterpret_cast<const double2*>(cfg + (d0 + k) * stride + n0)
                                        : make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (d0 + k < dof) {
                        const double qd = q[d0 + k];
                        const double e0 = __dsub_rn(v[k].x, qd), e1 = __dsub_rn(v[k].y, qd);
                        a0 = __dadd_rn(a0, __dmul_rn(e0, e0));
                        a1 = __dadd_rn(a1, __dmul_rn(e1, e1));
                    }
                }
            }
            if (a0 < best) {
                best = a0;
                bi = n0;
            }
            if (n0 + 1 < count && a1 < best) {
                best = a1;
                bi = n0 + 1;
            }
        }
    }
    for (int o = gsz >> 1; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(kFull, best, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        if (ob < best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    int src = 0;
    if (accept) {
        const bool ok = sub == 0 && j < m && best != 0.0 && !(ddf && ddf[bi] && !(__dsqrt_rn(best) <= R));
        const unsigned om = __ballot_sync(kFull, ok);
        *first = om ? (__ffs(om) - 1) >> glog : m;
        src = om ? __ffs(om) - 1 : 0;
    } else {
        *first = 0;
    }
    *nn = __shfl_sync(kFull, bi, src);
    *d2 = __shfl_sync(kFull, best, src);
}

// Validation of a chain A -> B (n_sub sub-edges) with appends — validate_chain
// at warp scope: 32 states per round up to the first invalid sub-edge, then
// the leading valid sub-edges' far points appended as one chained block.
// Returns the sub-edges appended, -1 - appended if the tree filled up.
__device__ long long warp_validate_chain(const PlanArgs& a, const WarpRegion& wr, const SceneV& v, float cpad,
                                         const double* A, const double* B, long long n_sub, const TreeRef& T,
                                         int parent0, int* last, bool* stopped, int* known, LaneAcc& acc,
                                         unsigned long long& fk_count, unsigned long long& fine_count) {
    const int lane = threadIdx.x & 31, n_cc = a.p.n_cc;
    const long long total = n_sub * (long long)n_cc;
    long long good = 0;
    *stopped = false;
    *last = parent0;
    if (total >= (1ll << 30)) return 0;  // beyond the 32-bit chain indexing: never valid
    for (long long g0 = 0; g0 < total; g0 += 32) {
        // the problem's done flag, read while the states are generated
        // (planner.cpp:112: a settled problem's chain is abandoned)
        int dn = 0;
        if (lane == 0) dn = ld_relaxed(T.done);
        int group;
        const bool act = warp_gen_state(A, B, n_sub, n_cc, total, g0, wr.qf, &group);
        if (__shfl_sync(kFull, dn, 0) != 0) {
            *stopped = true;
            return 0;
        }
        const unsigned am = __ballot_sync(kFull, act);
        fk_count += __popc(am);
        acc.f += act ? g_w.fkflops : 0u;
        bool fl;
        const bool bad = lane_check(v, cpad, a.fine_r64, wr.qf, wr.pose, wr.ccen, act, group, a.p.early_exit != 0,
                                    false, a.p.two_stage != 0, acc, &fl) && act;
        if (__any_sync(kFull, fl)) ++fine_count;
        const unsigned bm = __ballot_sync(kFull, bad);
        const long long cnt = min(32ll, total - g0);
        if (bm) {
            good = __shfl_sync(kFull, group, __ffs(bm) - 1);
            break;
        }
        good = (g0 + cnt) / n_cc;
    }
    if (good == 0) return 0;
    long long appended = 0;
    int prev = parent0;
    while (appended < good) {  // (a reservation holds at most INT_MAX nodes; chains are far shorter)
        const int cntk = (int)min(good - appended, 1ll << 20);
        const int got = warp_append(a, T, A, B, n_sub, appended + 1, cntk, prev, &prev, known);
        appended += got;
        if (got < cntk) {
            *last = prev;
            return -1 - appended;
        }
    }
    *last = prev;
    return appended;
}

// Path assembly (planner.cpp:125-150) by the winning warp: lane 0 walks the
// start tree from meet_a, lane 1 the goal tree from meet_b, recording the
// walks in the warp's pose store (a second walk writes the rows directly
// when one does not fit); then the lanes copy the rows into the arena.
// Returns the path length, -1 (arena full) or -2 (meeting configs differ).
__device__ int warp_assemble(const PlanArgs& a, const WarpRegion& wr, int prob, int meet_a, int meet_b) {
    const int lane = threadIdx.x & 31, dof = g_w.dof;
    const TreeRef Ta = tree_ref(a, prob, 0, dof), Tb = tree_ref(a, prob, 1, dof);
    int* ib = reinterpret_cast<int*>(wr.pose);
    const int half = g_w.walk_cap >> 1;
    int n = 0;
    if (lane < 2) {
        const int* par = lane == 0 ? Ta.parent : Tb.parent;
        int* w = ib + (lane == 0 ? 0 : half);
        for (int i = lane == 0 ? meet_a : meet_b;;) {
            if (n < half) w[n] = i;
            ++n;
            const int p = __ldcg(par + i);
            if (p < 0) break;
            i = p;
        }
    }
    const int la = __shfl_sync(kFull, n, 0), lb = __shfl_sync(kFull, n, 1);
    const int len = la + lb - 1;  // the meeting configuration once (planner.cpp:139-147)
    long long off = 0;
    int rc = len;
    if (lane == 0) {
        // planner.cpp:127-129: the meeting configurations must agree
        double acc = 0.0;
        for (int d = 0; d < dof; ++d) {
            const double e = __dsub_rn(__ldcg(&Ta.cfg[(size_t)d * a.stride + meet_a]),
                                       __ldcg(&Tb.cfg[(size_t)d * a.stride + meet_b]));
            acc = __dadd_rn(acc, __dmul_rn(e, e));
        }
        if (__dsqrt_rn(acc) > 1e-12) {
            rc = -2;
        } else {
            const unsigned long long need = (unsigned long long)len * dof;
            off = (long long)atomicAdd(a.arena_used, need);
            if ((unsigned long long)off + need > a.arena_cap) rc = -1;
            else a.ctl[prob].path_off = (unsigned long long)off;
        }
    }
    rc = __shfl_sync(kFull, rc, 0);
    off = __shfl_sync(kFull, off, 0);
    if (rc < 0) return rc;
    __syncwarp();
    if (la <= half && lb <= half) {
        for (int e = lane; e < len * dof; e += 32) {
            const int k = e / dof, d = e - k * dof;
            const bool inA = k < la;
            const int vtx = inA ? ib[la - 1 - k] : ib[half + (k - la + 1)];
            a.arena[off + e] = __ldcg(&(inA ? Ta : Tb).cfg[(size_t)d * a.stride + vtx]);
        }
    } else if (lane < 2) {  // long branches: walk again, one row per hop
        const TreeRef& T = lane == 0 ? Ta : Tb;
        int k = lane == 0 ? la - 1 : la - 1;  // tree A rows la-1 .. 0; tree B rows la-1 (meet, skipped) ..
        for (int i = lane == 0 ? meet_a : meet_b;;) {
            if (lane == 0 || k >= la)
                for (int d = 0; d < dof; ++d) a.arena[off + (long long)k * dof + d] = __ldcg(&T.cfg[(size_t)d * a.stride + i]);
            k += lane == 0 ? -1 : 1;
            const int p = __ldcg(T.parent + i);
            if (p < 0) break;
            i = p;
        }
    }
    __threadfence();
    __syncwarp();
    return len;
}

// Help mode (pick_help at warp scope): the running problem with the fewest
// active workers (ties to the lowest index); -1 once every problem is done.
__device__ int warp_pick_help(const PlanArgs& a) {
    const int lane = threadIdx.x & 31;
    for (int attempt = 0;; ++attempt) {
        if (attempt > 0) {
            int nd = 0;
            if (lane == 0) nd = ld_acquire(a.n_done);
            if (__shfl_sync(kFull, nd, 0) >= a.n_problems) return -1;
            __nanosleep(200);
        }
        int bk = 0x7fffffff, bp = -1, pending = 0;
        if (a.n_problems > 2 * kHelpWindow) {  // a rotating window first (see kHelpWindow)
            int start = 0;
            if (lane == 0) start = help_window_start(a.n_problems, attempt, blockIdx.x * 32 + (threadIdx.x >> 5));
            start = __shfl_sync(kFull, start, 0);
            help_scan(a, lane, 32, start, kHelpWindow, bk, bp, pending);
            pending = 0;
        }
        if (!__any_sync(kFull, bp >= 0)) help_scan(a, lane, 32, 0, a.n_problems, bk, bp, pending);
        // every problem is claimed (the claim loop ran dry) and every running
        // one has handed out its whole iteration budget: nothing can ever be
        // joined again, so leave instead of spinning (idle workers' scans
        // would take issue slots and L2 bandwidth from the working ones)
        if (!__any_sync(kFull, pending) && __all_sync(kFull, bp < 0)) return -1;
        for (int o = 16; o > 0; o >>= 1) {
            const int ok = __shfl_xor_sync(kFull, bk, o);
            const int op = __shfl_xor_sync(kFull, bp, o);
            if (ok < bk || (ok == bk && op >= 0 && (bp < 0 || op < bp))) {
                bk = ok;
                bp = op;
            }
        }
        int p = bp;
        if (lane == 0 && p >= 0) {
            atomicAdd(&a.ctl[p].active, 1);
            ld_acquire(&a.ctl[p].started);  // the roots are visible from here on
            if (ld_acquire(&a.ctl[p].done) != DONE_RUNNING) {
                atomicSub(&a.ctl[p].active, 1);
                p = -2;  // raced with completion: rescan
            }
        }
        p = __shfl_sync(kFull, p, 0);
        if (p >= 0) return p;
    }
}

// Endpoint checks and roots of a freshly claimed problem (init_problem at
// warp scope: lane 0 checks the start, lane 1 the goal, planner.cpp:263-293).
// Returns true if the search should run.
__device__ bool warp_init_problem(const PlanArgs& a, const WarpRegion& wr, const SceneV& v, float cpad, int prob,
                                  LaneAcc& acc, unsigned long long& fk_count) {
    const int lane = threadIdx.x & 31, dof = g_w.dof;
    ProbCtl& C = a.ctl[prob];
    const double* S = a.starts + (size_t)prob * dof;
    const double* G = a.goals + (size_t)prob * dof;
    if (lane == 0) C.t_start_ns = globaltimer();
    if (lane < 2)
        for (int d = 0; d < dof; ++d) wr.qf[d * 32 + lane] = (float)(lane == 0 ? S[d] : G[d]);
    bool fl;
    const bool bad = lane_check(v, cpad, a.fine_r64, wr.qf, wr.pose, wr.ccen, lane < 2, lane, a.p.early_exit != 0,
                                true, a.p.two_stage != 0, acc, &fl) && lane < 2;
    fk_count += 2;
    acc.f += lane < 2 ? g_w.fkflops : 0u;
    const unsigned bm = __ballot_sync(kFull, bad);
    int verdict = 0;
    if (lane == 0) {
        const double* lim = smo<double>(g_w.o_lim);
        bool sl = true, gl = true, eq = true;
        for (int d = 0; d < dof; ++d) {  // within_limits (planner.cpp:25-31): inclusive
            const double lo = lim[2 * d], hi = lim[2 * d + 1];
            const double s = S[d], g = G[d];
            sl &= !(s < lo || s > hi);
            gl &= !(g < lo || g > hi);
            eq &= s == g;
        }
        if (!sl || (bm & 1u)) verdict = 1;
        else if (!gl || (bm & 2u)) verdict = 2;
        else if (eq) verdict = 3;
        if (verdict == 1 || verdict == 2) {
            C.started = 1;
            finish_problem_w(a, prob, DONE_INFEASIBLE, verdict == 1 ? MSG_START : MSG_GOAL);
        } else if (verdict == 3) {  // start == goal: path [start], cost 0 (planner.cpp:279-285)
            const unsigned long long off = atomicAdd(a.arena_used, (unsigned long long)dof);
            C.started = 1;
            if (off + dof <= a.arena_cap) {
                for (int d = 0; d < dof; ++d) a.arena[off + d] = S[d];
                C.path_off = off;
                C.path_len = 1;
                C.winner = 1;
                __threadfence();
                finish_problem_w(a, prob, DONE_SOLVED, MSG_NONE);
            } else {
                finish_problem_w(a, prob, DONE_FAILED, MSG_ARENA);
            }
        }
    }
    verdict = __shfl_sync(kFull, verdict, 0);
    if (verdict) return false;
    for (int t = 0; t < 2; ++t) {  // roots (planner.cpp:292-293)
        const TreeRef T = tree_ref(a, prob, t, dof);
        if (lane < dof) T.cfg[(size_t)lane * a.stride] = (t == 0 ? S : G)[lane];
        if (lane == 0) {
            T.parent[0] = -1;
            T.dd[0] = 0;
            T.ready[0] = a.epoch;
            *T.reserved = 1;
            *T.published = 1;
        }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(&C.started, 1);
    return true;
}

// CTA setup of the warp-worker kernels: robot words, limits + Halton table,
// i / n_cc table, self pairs grouped by their higher link, store slots, and
// the per-warp layout in g_w.
__device__ void warp_cta_setup(const uint32_t* rg, const double* limits, int n_cc, int scene_words_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    const int robot_words = reinterpret_cast<const int*>(rg)[RH_WORDS];
    const int L = (int)rg[RH_NLINKS], dof = (int)rg[RH_DOF], NP = (int)rg[RH_NPAIRS];
    {
        const WarpLayout lay = warp_layout(robot_words, L, dof, NP, 0, 0);
        uint32_t* rw = reinterpret_cast<uint32_t*>(smem + lay.robot);
        for (int i = tid; i < robot_words / 4; i += blockDim.x)
            reinterpret_cast<uint4*>(rw)[i] = __ldg(reinterpret_cast<const uint4*>(rg) + i);
        double* lim = reinterpret_cast<double*>(smem + lay.lim);
        for (int i = tid; i < dof * (kHaltonTab + 2); i += blockDim.x) lim[i] = limits[i];  // limits, then table
        const bool tt = n_cc >= 1 && n_cc <= kTTab;
        double* ttab = reinterpret_cast<double*>(smem + lay.ttab);
        if (tt)
            for (int i = tid; i <= n_cc; i += blockDim.x) ttab[i] = __ddiv_rn((double)i, (double)n_cc);
        __syncthreads();
        if (tid == 0) {
            const int4* info = reinterpret_cast<const int4*>(rw + rw[RH_OFF_INFO]);
            const int2* pairs = reinterpret_cast<const int2*>(rw + rw[RH_OFF_PAIRS]);
            int* pstart = reinterpret_cast<int*>(smem + lay.pstart);
            int2* plo = reinterpret_cast<int2*>(smem + lay.plo);
            const float* geo = reinterpret_cast<const float*>(rw + rw[RH_OFF_GEO]);
            int* slot = reinterpret_cast<int*>(smem + lay.slot);
            const int nstore = warp_store_count(info, pairs, L, NP, slot);
            int e = 0;
            for (int l = 0; l < L; ++l) {  // self pairs grouped by their higher link
                pstart[l] = e;
                for (int p = 0; p < NP; ++p)
                    if (max(pairs[p].x, pairs[p].y) == l) {
                        // one 64-bit record per pair: the lower link, its pose
                        // store slot, and r_a + r_l (the coarse test's sum)
                        const int a = min(pairs[p].x, pairs[p].y);
                        plo[e++] = make_int2(a | (slot[a] << 16),
                                             __float_as_int(geo[a * GEO_STRIDE + 36] + geo[l * GEO_STRIDE + 36]));
                    }
            }
            pstart[L] = e;
            const WarpLayout wl = warp_layout(robot_words, L, dof, NP, nstore, scene_words_max);
            WCtx& w = g_w;
            const unsigned base = (unsigned)__cvta_generic_to_shared(smem) - (unsigned)__cvta_generic_to_shared(g_dsmem);
            w.L = L;
            w.dof = dof;
            w.S = (int)rw[RH_NFINE];
            w.NP = NP;
            w.nstore = nstore;
            w.fkflops = (int)rw[RH_FKFLOPS];
            w.o_info = base + (unsigned)lay.robot + 4u * rw[RH_OFF_INFO];
            w.o_nfine = base + (unsigned)lay.robot + 4u * rw[RH_OFF_NFINE];
            w.o_geo = base + (unsigned)lay.robot + 4u * rw[RH_OFF_GEO];
            w.o_fine = base + (unsigned)lay.robot + 4u * rw[RH_OFF_FINE];
            w.o_bases = base + (unsigned)lay.robot + 4u * rw[RH_OFF_BASES];
            w.o_magic = base + (unsigned)lay.robot + 4u * rw[RH_OFF_MAGIC];
            w.o_lim = base + (unsigned)lay.lim;
            w.o_htab = base + (unsigned)lay.htab;
            w.o_ttab = base + (unsigned)lay.ttab;
            w.ttab_n = tt ? n_cc : 0;
            w.o_pstart = base + (unsigned)lay.pstart;
            w.o_plo = base + (unsigned)lay.plo;
            w.o_slot = base + (unsigned)lay.slot;
            w.warp0 = base + (unsigned)al16(lay.shared_end);
            w.per_warp = (unsigned)wl.per_warp;
            w.w_scene = (unsigned)wl.scene;
            w.w_pose = (unsigned)wl.pose;
            w.w_ccen = (unsigned)wl.ccen;
            w.w_qf = (unsigned)wl.qf;
            w.w_sbuf = (unsigned)wl.sbuf;
            w.w_dcfg = (unsigned)wl.dcfg;
            w.walk_cap = nstore * 12 * 32;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// MAXW: the most warps the instantiation is launched with (one CTA per SM;
// fewer warps fit the shared memory for larger robots and scenes). The
// register cap follows: 128 at 16 warps, 136 at 14, 160 at 12 (a full 64K
// split, 144 x 14 warps, is refused at launch: "too many resources")
template <int MAXW>
__global__ void __maxnreg__(MAXW >= 16 ? 128 : (MAXW >= 14 ? 136 : 160)) plan_warp_kernel(PlanArgs a) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t* rg = a.robot;
    const int dof = (int)rg[RH_DOF];
    warp_cta_setup(rg, a.limits, a.p.n_cc, a.scene_words_max);
    const WarpRegion wr = warp_region(wid);
    const double R = a.p.dd_radius, delta = a.p.delta;
    const unsigned* const bases = smo<unsigned>(g_w.o_bases);
    const unsigned long long* const magic = smo<unsigned long long>(g_w.o_magic);
    const double* const lim = smo<double>(g_w.o_lim);
    const double* const htab = smo<double>(g_w.o_htab);
    if (tid == 0 && a.trace) atomicMax(&a.trace[0], 0x7fffffffffffffffull - (unsigned long long)globaltimer());
    LaneAcc acc;
    for (;;) {
        int prob = -1;
        unsigned long long fk_count = 0, fine_count = 0;
        SceneV v;
        float cpad = 0.f;
        // unstarted problems first: claim, stage its scene, initialise
        for (;;) {
            int p = 0;
            if (lane == 0) p = atomicAdd(a.next_problem, 1);
            p = __shfl_sync(kFull, p, 0);
            if (p >= a.n_problems) break;
            const int si = a.prob_scene[p];
            warp_load_scene(wr.scene, a.scene_words[si], lane);
            v = warp_scene(wr.scene, a.scene_f64[si], &cpad);
            if (lane == 0) atomicAdd(&a.ctl[p].active, 1);
            if (warp_init_problem(a, wr, v, cpad, p, acc, fk_count)) {
                prob = p;
                break;
            }
            // the endpoint checks' counters, then leave the settled problem
            unsigned long long t = acc.t, f = acc.f;
            for (int o = 16; o > 0; o >>= 1) {
                t += __shfl_xor_sync(kFull, t, o);
                f += __shfl_xor_sync(kFull, f, o);
            }
            acc = LaneAcc();
            if (lane == 0) {
                ProbCtl& C = a.ctl[p];
                if (t) atomicAdd(&C.sphere_tests, t);
                if (f) atomicAdd(&C.flops, f);
                atomicAdd(&C.fk_calls, fk_count);
                atomicSub(&C.active, 1);
            }
            fk_count = 0;
        }
        if (prob < 0) {
            prob = warp_pick_help(a);
            if (prob < 0) break;
            const int si = a.prob_scene[prob];
            warp_load_scene(wr.scene, a.scene_words[si], lane);
            v = warp_scene(wr.scene, a.scene_f64[si], &cpad);
        }
        ProbCtl& C = a.ctl[prob];
        // the roots: written by this warp, or acquired through `started`;
        // known0/1: the published prefix of each tree this warp holds
        // acquire-ordered (or wrote itself); dirty forces the first fence
        int known0 = 1, known1 = 1, dirty = 1;
        unsigned long long tk_base = 0, tk_pos = 0, tk_cnt = 0, used = 0;
        const int kblk = 32;
        int leave_msg = MSG_NONE;
        for (;;) {
            // ---- iteration header (lane 0's atomics and loads, broadcast) ----
            int dn = 0, la = 0, lb = 0;
            unsigned long long claimed = 0;
            const bool refill = tk_pos == tk_cnt;
            unsigned long long want = kblk;
            if (lane == 0) {
                dn = ld_relaxed(&C.done);
                if (refill) {
                    // near the end of the budget, smaller blocks (a.tail_claim)
                    if (a.tail_claim) {
                        const unsigned long long seen = tk_cnt ? tk_base + tk_cnt : __ldcg(&C.iters);
                        const int act = max(1, ld_relaxed(&C.active));
                        if (seen < a.p.budget)
                            want = max((unsigned long long)a.tail_min,
                                       min((unsigned long long)kblk, (a.p.budget - seen) / ((unsigned long long)a.tail_div * act)));
                    }
                    claimed = atomicAdd(&C.iters, want);
                }
                la = ld_relaxed(&C.published[0]);
                lb = ld_relaxed(&C.published[1]);
                if (la > known0 || lb > known1 || dirty) fence_acq_rel();
            }
            dn = __shfl_sync(kFull, dn, 0);
            la = __shfl_sync(kFull, la, 0);
            lb = __shfl_sync(kFull, lb, 0);
            if (refill) {
                tk_base = __shfl_sync(kFull, claimed, 0);
                tk_cnt = __shfl_sync(kFull, want, 0);
                tk_pos = 0;
            }
            known0 = max(known0, la);
            known1 = max(known1, lb);
            dirty = 0;
            const unsigned long long it = tk_base + tk_pos;
            const int leave = dn != DONE_RUNNING ? 1 : (it >= a.p.budget ? 2 : 0);
            if (leave) {
                leave_msg = leave == 2 ? MSG_BUDGET : MSG_NONE;
                break;
            }
            ++used;
            // extend_start_tree (planner.hpp:62-65)
            const int from_start = a.p.balance ? (la <= lb) : (int)((used & 1) == 1);
            const int ts = from_start ? 0 : 1;
            const int snap = from_start ? la : lb;
            const int slot = (int)tk_pos++;
            const int rem = (int)min(tk_cnt - (unsigned long long)slot, a.p.budget - it);
            const TreeRef Ts = tree_ref(a, prob, ts, dof);
            const TreeRef To = tree_ref(a, prob, 1 - ts, dof);
            // ---- sample (sampling.cpp:39-51): the ticket block at once,
            // Halton index 1 + seed + ticket ----
            if (refill) {
                const int nblk = (int)tk_cnt;
                __syncwarp();  // the previous block's samples are read before they are overwritten
                if (tk_base + nblk <= a.stab_n) {
                    // the block is one contiguous run of the per-launch table:
                    // up to four independent loads in flight per lane
                    const double* src = a.stab + tk_base * dof;
                    const int tot = nblk * dof;
                    for (int j0 = lane; j0 < tot; j0 += 128) {
                        double v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] = j0 + 32 * u < tot ? __ldg(src + j0 + 32 * u) : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (j0 + 32 * u < tot) wr.sbuf[j0 + 32 * u] = v[u];
                    }
                } else
                for (int j = lane; j < nblk * dof; j += 32) {
                    const int k = j / dof, d = j - k * dof;
                    const unsigned long long t = tk_base + k;  // (the per-launch sample table, see plan_kernel)
                    wr.sbuf[j] = t < a.stab_n ? __ldg(a.stab + t * dof + d)
                                              : sample_dim(halton_tab(bases[d], magic[d], htab + d * kHaltonTab, 1ull + a.p.seed + t),
                                                           lim[2 * d], lim[2 * d + 1]);
                }
                __syncwarp();
            }
            // ---- nearest neighbour(s) + acceptance: while the tree is
            // unchanged the block's next samples meet the same snapshot, so up
            // to 32 are scanned in one pass; the rejected ones before the
            // first accepted one count as iterations (planner.cpp:216-219) ----
            int m = 1;
            if (a.p.balance) m = max(1, min(rem, a.mnn_nodes / max(1, snap)));
            int first, nn;
            double d2;
            warp_nn(Ts.cfg, a.stride, snap, wr.sbuf + slot * dof, m, a.p.dynamic_domain ? Ts.dd : nullptr, true, R,
                    &first, &nn, &d2);
            {
                const int extra = (first < m ? first + 1 : m) - 1;
                tk_pos += extra;
                used += extra;
            }
            if (first == m) continue;
            const double* smp = wr.sbuf + (slot + first) * dof;
            const double dist = __dsqrt_rn(d2);
            // ---- steer (planner.cpp:48-64) ----
            double* nnc = wr.dcfg + WD_NN * dof;
            double* cnew = wr.dcfg + WD_NEW * dof;
            __syncwarp();  // every lane's reads of the previous chain's endpoints precede the rewrite
            if (lane < dof) {
                const double vv = Ts.cfg[(size_t)lane * a.stride + nn];  // L1: the scan read it
                nnc[lane] = vv;
                cnew[lane] = dist <= delta ? smp[lane] : lerp_exact(vv, smp[lane], __ddiv_rn(delta, dist));
            }
            __syncwarp();
            // ---- validation nn -> c_new + append (phase 0), then greedy
            // connect c_new -> the opposite tree (phase 1): one chain
            // validation call site for both ----
            const double* VA = nnc;
            const double* VB = cnew;
            long long nsub = 1;
            int par0 = nn, phase = 0, new_idx = nn, nno = -1, meet_self = nn;
            int outcome = 0;  // 0 next iteration, 1 reached, 2 tree full
#pragma unroll 1
            for (;;) {
                int last = par0;
                bool stopped = false;
                int kts = ts ? known1 : known0;
                const long long got = warp_validate_chain(a, wr, v, cpad, VA, VB, nsub, Ts, par0, &last, &stopped,
                                                          &kts, acc, fk_count, fine_count);
                if (ts) known1 = kts;
                else known0 = kts;
                if (got < 0) {
                    outcome = 2;
                    break;
                }
                if (phase == 1) {
                    outcome = (got == nsub && !stopped) ? 1 : 0;
                    meet_self = last;
                    break;
                }
                if (stopped) break;  // the header sees the done flag and leaves
                if (got == 0) {
                    if (a.p.dynamic_domain && lane == 0) Ts.dd[nn] = 1;  // record_failure
                    break;
                }
                new_idx = meet_self = last;
                int po = 0, settled = 0;
                const int kto = ts ? known0 : known1;
                if (lane == 0) {
                    po = ld_relaxed(To.published);
                    settled = ld_relaxed(&C.done);
                    if (po > kto) fence_acq_rel();
                }
                po = __shfl_sync(kFull, po, 0);
                settled = __shfl_sync(kFull, settled, 0);
                if (ts) known0 = max(known0, po);
                else known1 = max(known1, po);
                if (settled != DONE_RUNNING) break;  // the header leaves
                int f0;
                double d2o;
                warp_nn(To.cfg, a.stride, po, cnew, 1, nullptr, false, 0.0, &f0, &nno, &d2o);
                if (d2o == 0.0) {
                    outcome = 1;
                    break;
                }
                const double disto = __dsqrt_rn(d2o);
                double* tgt = wr.dcfg + WD_TGT * dof;
                double* A = wr.dcfg + WD_A * dof;
                __syncwarp();  // (as at the steer: reads of the old rows first)
                if (lane < dof) {
                    tgt[lane] = To.cfg[(size_t)lane * a.stride + nno];
                    A[lane] = cnew[lane];
                }
                __syncwarp();
                VA = A;
                VB = tgt;
                nsub = (long long)ceil(__ddiv_rn(disto, delta));
                par0 = new_idx;
                phase = 1;
            }
            if (outcome == 2) {
                leave_msg = MSG_CAPACITY;
                break;
            }
            if (outcome == 0) continue;
            // ---- winner (planner.cpp:232-238) ----
            int won = 0;
            if (lane == 0) won = atomicCAS(&C.winner, 0, 1 + (int)(blockIdx.x * (blockDim.x >> 5) + wid)) == 0;
            won = __shfl_sync(kFull, won, 0);
            if (won) {
                const int meet_a = ts == 0 ? meet_self : nno;
                const int meet_b = ts == 0 ? nno : meet_self;
                if (lane == 0) {
                    C.meet[0] = meet_a;
                    C.meet[1] = meet_b;
                }
                const int len = warp_assemble(a, wr, prob, meet_a, meet_b);
                if (lane == 0) {
                    if (len < 0) {
                        finish_problem_w(a, prob, DONE_FAILED, len == -2 ? MSG_MEET : MSG_ARENA);
                    } else {
                        C.path_len = len;
                        __threadfence();
                        finish_problem_w(a, prob, DONE_SOLVED, MSG_NONE);
                    }
                }
            }
            break;
        }
        // ---- leave: counters, then the last worker out of an unsolved problem fails it ----
        unsigned long long t = acc.t, f = acc.f;
        for (int o = 16; o > 0; o >>= 1) {
            t += __shfl_xor_sync(kFull, t, o);
            f += __shfl_xor_sync(kFull, f, o);
        }
        acc = LaneAcc();
        if (lane == 0) {
            if (used) atomicAdd(&C.iters_used, used);
            if (t) atomicAdd(&C.sphere_tests, t);
            if (f) atomicAdd(&C.flops, f);
            if (fk_count) atomicAdd(&C.fk_calls, fk_count);
            if (fine_count) atomicAdd(&C.fine_entries, fine_count);
            const int prev = atomicSub(&C.active, 1);
            if (leave_msg == MSG_CAPACITY) finish_problem_w(a, prob, DONE_FAILED, MSG_CAPACITY);
            else if (prev == 1 && ld_acquire(&C.done) == DONE_RUNNING) finish_problem_w(a, prob, DONE_FAILED, MSG_BUDGET);
        }
        __syncwarp();
    }
    if (lane == 0 && a.trace) atomicMax(&a.trace[1], (unsigned long long)globaltimer());
}

// ---------------------------------------------------------------------------
// batched edge validation (the product API prrtc_validate_edges and the
// collision microbenchmark) on the warp planner's checker: one edge per warp,
// one state per lane end to end (FK, two-stage or brute-force collision,
// early exit by ballot) — the same verdicts as check_chunk's (the planner's
// own edge test, collision.cpp:206-224), without the CTA-wide barriers.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) validate_edges_warp_kernel(RobotArgs r, SceneArgs sa, const double* from,
                                                                     const double* to, int n_edges, int n_cc,
                                                                     int two_stage, int early_exit, uint8_t* out,
                                                                     unsigned long long* counters) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_cta_setup(r.words, r.limits, n_cc, sa.n_words);
    const WarpRegion wr = warp_region(wid);
    const int dof = g_w.dof;
    warp_load_scene(wr.scene, sa.words, lane);
    float cpad = 0.f;
    const SceneV v = warp_scene(wr.scene, sa.f64, &cpad);
    LaneAcc acc;
    double* const A = wr.dcfg + WD_A * dof;
    double* const B = wr.dcfg + WD_NEW * dof;
    for (int e = blockIdx.x * nw + wid; e < n_edges; e += gridDim.x * nw) {
        __syncwarp();  // the previous edge's endpoints are read before they are rewritten
        if (lane < dof) {
            A[lane] = from[(size_t)e * dof + lane];
            B[lane] = to[(size_t)e * dof + lane];
        }
        __syncwarp();
        bool bad = false;
        for (int g0 = 0; g0 < n_cc && !(bad && early_exit); g0 += 32) {
            int group;
            const bool act = warp_gen_state(A, B, 1, n_cc, n_cc, g0, wr.qf, &group);
            acc.f += act ? (unsigned)g_w.fkflops : 0u;
            bool fl;
            const bool b = lane_check(v, cpad, r.fine_r64, wr.qf, wr.pose, wr.ccen, act, group, early_exit != 0,
                                      false, two_stage != 0, acc, &fl) && act;
            bad = __any_sync(kFull, b) || bad;
        }
        if (lane == 0) out[e] = bad ? 0 : 1;
    }
    if (counters) {  // measurement: executed sphere tests and algorithmic flops
        unsigned long long t = acc.t, f = acc.f;
        for (int o = 16; o > 0; o >>= 1) {
            t += __shfl_xor_sync(kFull, t, o);
            f += __shfl_xor_sync(kFull, f, o);
        }
        if (lane == 0) {
            atomicAdd(&counters[0], t);
            atomicAdd(&counters[1], f);
        }
    }
}

// Sound mode's path re-validation (validate_paths_kernel's job) on the warp
// checker: one path edge per warp, 4 n_cc states in rounds of 32 lanes,
// two-stage with early exit (the verdict of the reference's fine-only, no
// early exit check: see validate_paths_kernel), a warp re-stages its scene
// only when the next edge's problem has another one.
__global__ void __launch_bounds__(512, 1) validate_paths_warp_kernel(PlanArgs a, const int* prefix, int n_cc4) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_cta_setup(a.robot, a.limits, n_cc4, a.scene_words_max);
    const WarpRegion wr = warp_region(wid);
    const int dof = g_w.dof;
    double* const A = wr.dcfg + WD_A * dof;
    double* const B = wr.dcfg + WD_NEW * dof;
    const int total = prefix[a.n_problems];
    int cur_scene = -1;
    SceneV v{};
    float cpad = 0.f;
    LaneAcc acc;
    for (int E = blockIdx.x * nw + wid; E < total; E += gridDim.x * nw) {
        int lo = 0, hi = a.n_problems - 1;  // last p with prefix[p] <= E
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= E) lo = mid;
            else hi = mid - 1;
        }
        const int p = lo, e = E - prefix[p];
        const int si = a.prob_scene[p];
        if (si != cur_scene) {
            warp_load_scene(wr.scene, a.scene_words[si], lane);
            v = warp_scene(wr.scene, a.scene_f64[si], &cpad);
            cur_scene = si;
        }
        const double* P = a.arena + a.ctl[p].path_off + (size_t)e * dof;
        __syncwarp();
        if (lane < dof) {
            A[lane] = P[lane];
            B[lane] = P[dof + lane];
        }
        __syncwarp();
        bool bad = false;
        for (int g0 = 0; g0 < n_cc4 && !bad; g0 += 32) {
            int group;
            const bool act = warp_gen_state(A, B, 1, n_cc4, n_cc4, g0, wr.qf, &group);
            bool fl;
            const bool b = lane_check(v, cpad, a.fine_r64, wr.qf, wr.pose, wr.ccen, act, group, true, false, true, acc,
                                      &fl) && act;
            bad = __any_sync(kFull, b);
        }
        if (lane == 0 && bad) atomicOr(&a.ctl[p].path_bad, 1);
    }
}

// Warps per CTA for a warp-worker launch (one CTA per SM): as many workers
// as the shared memory holds, at most 16 (128 registers each); 0 when not
// even one fits (the CTA planner then runs the batch).
int warp_workers_per_sm(const uint32_t* robot_words_host, int scene_words_max, int max_smem) {
    const int rw = (int)robot_words_host[RH_WORDS];
    const int L = (int)robot_words_host[RH_NLINKS], dof = (int)robot_words_host[RH_DOF];
    const int NP = (int)robot_words_host[RH_NPAIRS];
    const int4* info = reinterpret_cast<const int4*>(robot_words_host + robot_words_host[RH_OFF_INFO]);
    const int2* pairs = reinterpret_cast<const int2*>(robot_words_host + robot_words_host[RH_OFF_PAIRS]);
    const int nstore = warp_store_count(info, pairs, L, NP, nullptr);
    const WarpLayout w = warp_layout(rw, L, dof, NP, nstore, scene_words_max);
    const long long room = (long long)max_smem - (long long)al16(w.shared_end);
    if (room < (long long)w.per_warp) return 0;
    return (int)std::min<long long>(16, room / (long long)w.per_warp);
}

size_t warp_smem_bytes(const uint32_t* robot_words_host, int scene_words_max, int warps) {
    const int rw = (int)robot_words_host[RH_WORDS];
    const int L = (int)robot_words_host[RH_NLINKS], dof = (int)robot_words_host[RH_DOF];
    const int NP = (int)robot_words_host[RH_NPAIRS];
    const int4* info = reinterpret_cast<const int4*>(robot_words_host + robot_words_host[RH_OFF_INFO]);
    const int2* pairs = reinterpret_cast<const int2*>(robot_words_host + robot_words_host[RH_OFF_PAIRS]);
    const int nstore = warp_store_count(info, pairs, L, NP, nullptr);
    const WarpLayout w = warp_layout(rw, L, dof, NP, nstore, scene_words_max);
    return al16(w.shared_end) + (size_t)warps * w.per_warp;
}

cudaError_t launch_plan_warp(const RobotArgs& r, const uint32_t* robot_words_host, PlanArgs a, int grid, int warps,
                             cudaStream_t st) {
    const size_t sm = warp_smem_bytes(robot_words_host, a.scene_words_max, warps);
    const void* fn = warps <= 12 ? reinterpret_cast<const void*>(plan_warp_kernel<12>)
                     : warps <= 14 ? reinterpret_cast<const void*>(plan_warp_kernel<14>)
                                   : reinterpret_cast<const void*>(plan_warp_kernel<16>);
    cudaFuncAttributes fa;  // (the 128-register instantiation if the device refuses the wider one)
    if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess || fa.maxThreadsPerBlock < 32 * warps)
        fn = reinterpret_cast<const void*>(plan_warp_kernel<16>);
    cudaError_t e = raise_smem_limit(fn, (int)sm);
    if (e != cudaSuccess) return e;
    void* args[] = {&a};
    return cudaLaunchKernel(fn, dim3(grid), dim3(32 * warps), args, sm, st);
}

cudaError_t launch_validate_edges_warp(const RobotArgs& r, const SceneArgs& s, const double* from, const double* to,
                                       int n_edges, int n_cc, int two_stage, int early_exit, uint8_t* out,
                                       cudaStream_t st, unsigned long long* counters, int sms, int max_smem) {
    const int warps = warp_workers_per_sm(r.host_words, s.n_words, max_smem);
    if (warps <= 0) return cudaErrorInvalidConfiguration;
    const size_t sm = warp_smem_bytes(r.host_words, s.n_words, warps);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(validate_edges_warp_kernel), (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<long long>(sms, ((long long)n_edges + warps - 1) / warps);
    if (grid > 0)
        validate_edges_warp_kernel<<<grid, 32 * warps, sm, st>>>(r, s, from, to, n_edges, n_cc, two_stage, early_exit,
                                                                out, counters);
    return cudaGetLastError();
}
