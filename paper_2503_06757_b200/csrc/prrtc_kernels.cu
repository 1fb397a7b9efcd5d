// prrtc_kernels.cu — sm_100a kernels of the B200 pRRTC planner.
//
// plan_kernel is the whole reference worker loop (planner.cpp:186-242) as one
// persistent kernel: every CTA is a "worker"; it takes an unstarted problem
// from a global ticket (initialising it: endpoint checks, roots), or joins the
// running problem with the fewest workers, and iterates
//   balanced pick -> Halton sample -> NN -> dynamic domain -> steer ->
//   SIMT edge validation -> atomic append -> NN in the opposite tree ->
//   greedy connect (chunked SIMT validation, appends) -> winner CAS ->
//   on-device path assembly
// until the problem is solved / fails, with no host round-trip. Trees are
// shared by all CTAs on a problem through gpu-scope atomics in HBM.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "prrtc_b200.h"
#include "prrtc_device.cuh"
#include "prrtc_launch.h"

namespace prrtc_b200 {

using namespace dev;

// ---------------------------------------------------------------------------
// shared memory carve-up (host and device agree through smem_layout)
// ---------------------------------------------------------------------------
struct SmemLayout {
    size_t robot, scene, pose, ccen, qf, sgroup, sbad, lmask, ictl, dcfg, red_d, red_i,
        ends, ttab, sbuf, mnn, stat, htab, t0, rcount, rfine, mt, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// scene_words: room for the largest scene the launch stages (the planner
// sizes it from its batch, other kernels take the maximum); with_mt: the
// Uniform sampler's generator state (2.5 KB) only when that sampler runs —
// trimmed so five 128-thread planner CTAs fit one SM's shared memory
__host__ __device__ inline SmemLayout smem_layout(int robot_words, int L, int dof, int NS,
                                                  int nthreads, int scene_words = SCENE_MAX_WORDS,
                                                  bool with_mt = true) {
    SmemLayout s;
    // the fixed-offset CTA buffers first (prrtc_device.cuh FX_*), then the
    // robot- and scene-sized ones
    s.ictl = FX_ICTL;
    s.t0 = FX_T0;
    s.red_d = FX_RED_D;
    s.red_i = FX_RED_I;
    s.mnn = FX_MNN_D;
    s.dcfg = FX_DCFG;
    s.sgroup = FX_SGROUP;
    s.sbad = FX_SBAD;
    s.ttab = FX_TTAB;
    size_t o = FX_END;
    s.robot = o; o = al16(o + 4 * (size_t)robot_words);
    s.scene = o; o = al16(o + 4 * (size_t)scene_words);
    s.pose = o;  o = al16(o + 4 * (size_t)L * 12 * NS);
    s.ccen = o;  o = al16(o + 4 * (size_t)L * 3 * NS);
    s.qf = o;    o = al16(o + 4 * (size_t)dof * NS);
    // lmask [L][NS] then pmask [ceil(NP/64)][NS] (PRRTC_MAX_SELF_PAIRS = 512)
    s.lmask = o; o = al16(o + 8 * (size_t)(L + 8) * NS);
    s.ends = o;  o = al16(o + 8 * (size_t)(NS + 2) * dof);
    s.sbuf = o;  o = al16(o + 8 * (size_t)32 * dof);  // one ticket block of 32 samples
    s.stat = o;  o = al16(o + 16 * (size_t)nthreads);
    s.htab = o;  o = al16(o + 8 * (size_t)dof * (kHaltonTab + 2));  // + the [dof][2] limits
    s.rcount = o; o = al16(o + 8 * (size_t)NS);
    s.rfine = o; o = al16(o + 4 * (size_t)NS);
    s.mt = o;    o = al16(o + (with_mt ? 8 * (size_t)(kMtN + 1) : 0));
    s.total = o;
    return s;
}

size_t smem_bytes(const RobotArgs& r, int ns_max, int nthreads, int scene_words, bool with_mt) {
    return smem_layout(r.n_words, r.n_links, r.dof, ns_max, nthreads, scene_words, with_mt).total;
}

// scene words the planner stages per CTA: the launch's largest scene (the
// host sets a.scene_words_max), else the maximum
__host__ __device__ inline int plan_scene_words(const PlanArgs& a) {
    return a.scene_words_max > 0 && a.scene_words_max <= SCENE_MAX_WORDS ? a.scene_words_max : SCENE_MAX_WORDS;
}

// Copies the packed robot into shared memory and wires the context.
__device__ void setup_ctx(Ctx& c, unsigned char* smem, const uint32_t* robot_g, int robot_words,
                          const double* fine_r64, const double* limits, int NS,
                          int scene_words = SCENE_MAX_WORDS, bool with_mt = true) {
    const int tid = threadIdx.x, nthreads = blockDim.x;
    uint32_t* rw = reinterpret_cast<uint32_t*>(smem + FX_END);  // the robot words (smem_layout: s.robot)
    // 16-byte vector copy (buffer padded to a multiple of 4 words on host)
    for (int i = tid; i < robot_words / 4; i += nthreads) {
        reinterpret_cast<uint4*>(rw)[i] = __ldg(reinterpret_cast<const uint4*>(robot_g) + i);
    }
    __syncthreads();
    const SmemLayout lay = smem_layout(robot_words, rw[RH_NLINKS], rw[RH_DOF], NS, nthreads, scene_words, with_mt);
    unsigned long long* stat = reinterpret_cast<unsigned long long*>(smem + lay.stat);
    stat[2 * tid] = 0;
    stat[2 * tid + 1] = 0;
    // Halton reciprocal table (host-built, after the limits) staged in shared
    // memory: the sampler reads it per digit, and global reads would often
    // miss the L1 the tree protocol's acquires keep invalidating
    double* htab = reinterpret_cast<double*>(smem + lay.htab);
    for (int i = tid; i < (int)rw[RH_DOF] * (kHaltonTab + 2); i += nthreads) htab[i] = limits[i];
    if (tid < T0_COUNT) reinterpret_cast<unsigned long long*>(smem + lay.t0)[tid] = 0;
    if (ctx_writer(c)) {
        c.nthreads = nthreads;
        c.L = rw[RH_NLINKS];
        c.dof = rw[RH_DOF];
        c.S = rw[RH_NFINE];
        c.NP = rw[RH_NPAIRS];
        c.MF = rw[RH_MAXFINE];
        c.info = reinterpret_cast<const int4*>(rw + rw[RH_OFF_INFO]);
        c.nfine = reinterpret_cast<const int*>(rw + rw[RH_OFF_NFINE]);
        c.geo = reinterpret_cast<const float*>(rw + rw[RH_OFF_GEO]);
        c.fine = reinterpret_cast<const float4*>(rw + rw[RH_OFF_FINE]);
        c.pairs = reinterpret_cast<const int2*>(rw + rw[RH_OFF_PAIRS]);
        c.bases = rw + rw[RH_OFF_BASES];
        c.magic = reinterpret_cast<const unsigned long long*>(rw + rw[RH_OFF_MAGIC]);
        c.flink = reinterpret_cast<const int*>(rw + rw[RH_OFF_FLINK]);
        c.funits = reinterpret_cast<const int2*>(rw + rw[RH_OFF_FUNITS]);
        c.NFU = rw[RH_NFUNITS];
        c.fine_r64 = fine_r64;
        c.limits = htab;  // shared copy: [dof][2] limits, then the Halton table
        c.NS = NS;
        c.pose = reinterpret_cast<float*>(smem + lay.pose);
        c.ccen = reinterpret_cast<float*>(smem + lay.ccen);
        c.qf = reinterpret_cast<float*>(smem + lay.qf);
        c.lmask = reinterpret_cast<unsigned long long*>(smem + lay.lmask);
        c.pmask = c.lmask + (size_t)c.L * NS;
        c.ends = reinterpret_cast<double*>(smem + lay.ends);
        c.htab = htab + 2 * c.dof;
        c.sbuf = reinterpret_cast<double*>(smem + lay.sbuf);
        c.stat = stat;
        c.ref_stats = 0;  // the planner turns it on in deterministic mode
        c.rcount = reinterpret_cast<unsigned long long*>(smem + lay.rcount);
        c.rfine = reinterpret_cast<int*>(smem + lay.rfine);
        c.mt = reinterpret_cast<unsigned long long*>(smem + lay.mt);
        c.ttab_n = 0;
        c.nslog = 31 - __clz(NS);
        c.mflog = c.MF > 1 ? 32 - __clz(c.MF - 1) : 0;
        c.fkflops = rw[RH_FKFLOPS];
        c.prof = nullptr;
        c.ns = c.nb = c.nc = c.ny = c.P = 0;  // scene pointers are wired by load_scene
    }
    __syncthreads();
}

// Stages one scene's primitives in shared memory (the full
// primitive set is cached in low-latency memory for the whole plan).
__device__ void load_scene(Ctx& c, unsigned char* sbase, const uint32_t* scene_g, SceneF64 f64) {
    uint32_t* sw = reinterpret_cast<uint32_t*>(sbase);
    __syncthreads();
    const int words = __ldg(scene_g + SH_WORDS);
    for (int i = threadIdx.x; i < words; i += c.nthreads) sw[i] = __ldg(scene_g + i);
    __syncthreads();
    if (ctx_writer(c)) {
        c.ns = sw[SH_NS];
        c.nb = sw[SH_NB];
        c.nc = sw[SH_NC];
        c.ny = sw[SH_NY];
        c.P = c.ns + c.nb + c.nc + c.ny;
        c.sph = reinterpret_cast<const float4*>(sw + sw[SH_OFF_S]);
        c.box = reinterpret_cast<const float*>(sw + sw[SH_OFF_B]);
        c.cap = reinterpret_cast<const float*>(sw + sw[SH_OFF_C]);
        c.cyl = reinterpret_cast<const float*>(sw + sw[SH_OFF_Y]);
        c.eps = __uint_as_float(sw[SH_EPS]);
        c.cpad = __uint_as_float(sw[SH_CPAD]);
        c.s64 = f64;
    }
    __syncthreads();
}

// the scene words live right after the robot in shared memory; load_scene
// needs the base, which setup_ctx stored in c.sph. Keep it in a helper.
__device__ __forceinline__ unsigned char* scene_base(unsigned char* smem, int robot_words, int L,
                                                     int dof, int NS, int nthreads) {
    return smem + smem_layout(robot_words, L, dof, NS, nthreads).scene;
}

// ---------------------------------------------------------------------------
// tree helpers (tree.hpp:27-53 semantics with device-scope atomics)
// ---------------------------------------------------------------------------
struct TreeRef {
    double* cfg;       // [dof][cap]
    int* parent;       // [cap]
    unsigned* ready;   // [cap]
    int* dd;           // [cap]
    int* reserved;
    int* published;
    const int* done;   // the problem's done flag (a settled problem's trees are never read again)
    int which;         // 0 start tree, 1 goal tree
};

// PRRTC_TRACE: last phase entered + when, iterations, and a ring of the
// last 11 (phase, time) events per CTA (slots 8..29); slots 32..47 sum the
// SM cycles spent in each phase code, 48..63 count the entries (a phase
// lasts until the next marker). Codes: 1 header, 2 NN (extend), 3 dynamic
// domain + steer, 4 NN (connect), 5 validation chunk, 6 winner/assembly,
// 7 sample, 8 append, 9 chain states + FK + collision bookkeeping, 10 leave.
// The row lives in shared memory while the CTA runs (global read-modify-
// writes would cost an L2 round trip per marker) and is copied out at exit.
constexpr int kTraceStride = 64;
__shared__ long long g_trace[kTraceStride];
__device__ __noinline__ void trace_phase_rec(int code);
template <bool TR = true>
__device__ __forceinline__ void trace_phase(const PlanArgs& a, int code) {
    if constexpr (!TR) return;  // production instantiation: no trace code in the loop
    // out of line: ten call sites of the recorder would otherwise bloat the
    // hot loop's instruction footprint even with tracing off
    if (threadIdx.x == 0 && a.cta_trace) trace_phase_rec(code);
}
__device__ __noinline__ void trace_phase_rec(int code) {
    long long* t = g_trace;
    const long long now = globaltimer();
    const long long cyc = clock64();
    const int prev = (int)t[6];
    if (prev > 0 && prev < 16) {
        t[32 + prev] += cyc - t[30];  // slot 30: clock64 of the last marker
        t[48 + prev] += 1;
    }
    t[30] = cyc;
    t[6] = code;
    t[7] = now;
    if (code == 1) t[5] += 1;
    const long long k = t[4]++;
    t[8 + 2 * (k % 11)] = code;
    t[9 + 2 * (k % 11)] = now;
}

__device__ __forceinline__ TreeRef tree_ref(const PlanArgs& a, int prob, int t, int dof) {
    TreeRef r;
    const size_t pt = (size_t)prob * 2 + t;
    r.cfg = a.cfg + pt * dof * a.stride;
    r.parent = a.parent + pt * a.stride;
    r.ready = a.ready + pt * a.stride;
    r.dd = a.dd + pt * a.stride;
    r.reserved = &a.ctl[prob].reserved[t];
    r.published = &a.ctl[prob].published[t];
    r.done = &a.ctl[prob].done;
    r.which = t;
    return r;
}

// Append `count` chained nodes (pts[j], parent of node 0 = parent0, of node
// j = node j-1): reserve a contiguous block (one fetch_add, tree.hpp:29),
// write configs/parents in parallel, set the slots' ready flags, then publish
// the block with one CAS published: s0 -> s0 + ok. Lock-free: unlike
// tree.hpp:36-43 no writer waits for a predecessor (that would deadlock CTAs
// that are not co-resident). If a predecessor block is still being written
// the CAS fails and that predecessor's writer, after publishing its own
// block, carries `published` forward over every ready slot. Returns the
// number appended (< count when the tree filled up, tree.hpp:30) and the
// last appended slot in *last.
__device__ int tree_append_many(Ctx& c, const PlanArgs& a, const TreeRef& T, const double* pts,
                                int count, int parent0, int* last) {
    const int tid = threadIdx.x, dof = c.dof;
    if (tid == 0) sh(c.ictl)[IC_TMP2] = atomicAdd(T.reserved, count);
    __syncthreads();
    const long long s0 = sh(c.ictl)[IC_TMP2];
    const int ok = (int)max(0ll, min((long long)count, a.cap - s0));
    for (int idx = tid; idx < ok * dof; idx += c.nthreads) {
        const int j = idx / dof, d = idx - j * dof;
        T.cfg[(size_t)d * a.stride + s0 + j] = pts[idx];
    }
    for (int j = tid; j < ok; j += c.nthreads) {
        T.parent[s0 + j] = j == 0 ? parent0 : (int)(s0 + j - 1);
        T.dd[s0 + j] = 0;
        T.ready[s0 + j] = a.epoch;
    }
    __threadfence();  // data and flags before the publishing CAS
    __syncthreads();
    if (tid < 32 && ok > 0) {  // warp 0 publishes
        const int lane = tid;
        int won = 0;
        if (lane == 0) {
            won = atomicCAS(T.published, (int)s0, (int)(s0 + ok)) == s0;
            // a block that starts at the CTA's known prefix extends it: the
            // new nodes are its own writes
            int* known = sh(c.ictl) + IC_KNOWN0 + T.which;
            if (won && *known == (int)s0) *known = (int)(s0 + ok);
        }
        won = __shfl_sync(0xffffffffu, won, 0);
        if (won) {
            // our block is published; carry `published` over the successors
            // that finished first: 32 ready flags per step, one CAS per run
            // (a burst of concurrent appends otherwise costs one acquire load +
            // CAS round trip per slot)
            int p = (int)(s0 + ok);
            while (p < a.cap) {
                // store->load (Dekker) ordering against a successor that set
                // its flags and then failed its CAS: our last CAS must be
                // visible before we read its flags (it fenced the other way
                // round). After every successful CAS the flags are read
                // again: a successor whose CAS lost to that one is only seen
                // here (stopping early would strand its block)
                __threadfence();
                const long long idx = (long long)p + lane;
                const bool r = idx < a.cap && ld_acquire_u(&T.ready[idx]) == a.epoch;
                // under a burst of appends the carrier can stay behind its
                // successors for a long time; once the problem has settled
                // (done != DONE_RUNNING) nobody reads its trees again, so
                // stop carrying (it held the last CTA out for ~30 us)
                const bool settled = lane == 0 && ld_relaxed(T.done) != 0;
                const unsigned m = __ballot_sync(0xffffffffu, r);
                const int run = (m == 0xffffffffu) ? 32 : (__ffs(~m) - 1);
                if (run == 0 || __any_sync(0xffffffffu, settled)) break;
                int old = 0;
                fence_acq_rel();  // release for the carried slots (acquired through their flags)
                if (lane == 0) old = atomicCAS(T.published, p, p + run);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old != p) break;  // another writer is advancing
                p += run;
            }
        }
    }
    *last = ok > 0 ? (int)(s0 + ok - 1) : parent0;
    return ok;
}

// Exact-CheckStats mode (deterministic planning): the reference validates the
// chain's states one by one and stops at the first collision (early_exit) or
// at the end of the first invalid sub-edge (collision.cpp:206-224,
// planner.cpp:111-117), so it counts exactly the states up to there; each
// state's counters follow ref_state_count. Every state of the first bad
// group was evaluated (skip_state is strict in this mode).
__device__ __noinline__ void ref_count_chain_chunk(Ctx& c, int cnt, bool two_stage, bool early_exit, int fb) {
    const int* sgroup = sh(c.sgroup);
    for (int s = threadIdx.x; s < cnt; s += c.nthreads) {
        int fe = 0;
        const bool counted = sgroup[s] >= 0 && (fb == kNoBad || sgroup[s] <= fb);
        sh(c.rcount)[s] = counted ? ref_state_count(c, s, two_stage, early_exit, &fe) : 0ull;
        sh(c.rfine)[s] = fe;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tests = 0, fk = 0, fine = 0;
        for (int s = 0; s < cnt; ++s) {
            if (sgroup[s] < 0) continue;
            if (fb != kNoBad && sgroup[s] > fb) break;
            tests += sh(c.rcount)[s];
            fine += sh(c.rfine)[s];
            ++fk;
            if (early_exit && sh(c.sbad)[s]) break;
        }
        unsigned long long* t0 = sh(c.t0);
        t0[T0_RTESTS] += tests;
        t0[T0_FK] += fk;
        t0[T0_FINE] += fine;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// chain validation with appends (extend: n_sub = 1; greedy connect:
// planner.cpp:66-123). Sub-edges are validated chunk by chunk (NS states of
// the whole chain at a time) up to the first invalid one; then the leading
// valid sub-edges' far points are appended as one chained block — exactly
// the nodes and parents the reference's sequential validate/append loop
// adds, published in one step instead of one by one. Returns the number of
// sub-edges appended, or -1 - appended if the tree filled up; the last
// appended slot in *last.
// ---------------------------------------------------------------------------
template <bool TR>
__device__ long long validate_chain(Ctx& c, const PlanArgs& a, const double* A, const double* B,
                                    long long n_sub, const TreeRef* T, int parent0, int* last,
                                    const int* done_flag, bool* stopped) {
    const int n_cc = a.p.n_cc;
    const long long total = n_sub * (long long)n_cc;
    long long good = 0;
    *stopped = false;
    *last = parent0;
    if (total >= (1ll << 30)) return 0;  // beyond the 32-bit chain indexing: never valid (see gen_chain_states)
    for (long long g0 = 0; g0 < total; g0 += c.NS) {
        trace_phase<TR>(a, 9);  // PRRTC_TRACE: chain states
        const int cnt = (int)min((long long)c.NS, total - g0);
        // (the problem's done flag, planner.cpp:112, is sampled once per chunk
        // by check_chunk after FK, where its L2 round trip is hidden; sampled
        // here too it held every chunk's state-generation barrier for it)
        const int act = gen_chain_states_inl(c, A, B, n_sub, n_cc, g0, cnt, nullptr);
        if (threadIdx.x == 0) {
            if (!c.ref_stats) sh(c.t0)[T0_FK] += act;
            sh(c.stat)[1] += (unsigned long long)act * c.fkflops;  // thread 0's flop slot
        }
        trace_phase<TR>(a, 5);  // FK + collision
        check_chunk_inl(c, cnt, a.p.two_stage != 0, a.p.early_exit != 0, false, done_flag);
        trace_phase<TR>(a, 9);
        if (done_flag && sh(c.ictl)[IC_STOP] != 0) {  // settled while this chunk was checked
            *stopped = true;
            return 0;
        }
        if (threadIdx.x == 0 && sh(c.ictl)[IC_QN] && !c.ref_stats) ++sh(c.t0)[T0_FINE];
        // (IC_FIRSTBAD is next reset inside the next chunk's FK, after the
        // state-generation barrier: every thread has read it by then)
        const int fb = sh(c.ictl)[IC_FIRSTBAD];
        if (c.ref_stats) ref_count_chain_chunk(c, cnt, a.p.two_stage != 0, a.p.early_exit != 0, fb);
        good = (fb != kNoBad) ? (long long)fb : (g0 + cnt) / n_cc;
        if (fb != kNoBad) break;
    }
    long long appended = 0;
    int prev = parent0;
    trace_phase<TR>(a, 8);  // append
    while (appended < good) {
        const int cntk = (int)min(good - appended, (long long)c.NS + 1);
        const double* pts = B;  // a single edge appends its far end as is (collision.cpp:19)
        if (n_sub > 1) {
            for (int idx = threadIdx.x; idx < cntk * c.dof; idx += c.nthreads) {
                const int j = idx / c.dof, d = idx - j * c.dof;
                sh(c.ends)[idx] = chain_point(A, B, d, appended + 1 + j, n_sub);
            }
            __syncthreads();
            pts = sh(c.ends);
        }
        // (tree_append_many reads pts and the shared scalars before its own
        // barriers, so the next round may overwrite them right away)
        const int got = tree_append_many(c, a, *T, pts, cntk, prev, &prev);
        appended += got;
        if (got < cntk) {
            *last = prev;
            return -1 - appended;
        }
    }
    *last = prev;
    return appended;
}

// ---------------------------------------------------------------------------
// device path assembly (planner.cpp:125-150): walk meet_a -> root of the
// start tree (reversed), then meet_b's parents -> root of the goal tree.
// ---------------------------------------------------------------------------
__device__ void assemble_path_serial(Ctx& c, const PlanArgs& a, int prob, int meet_a, int meet_b) {
    const int tid = threadIdx.x;
    const int dof = c.dof;
    const TreeRef Ta = tree_ref(a, prob, 0, dof), Tb = tree_ref(a, prob, 1, dof);
    int* ib = reinterpret_cast<int*>(c.pose.get());
    const int ib_cap = c.L * 12 * c.NS;
    if (tid == 0) {
        int la = 1, lb = 1;
        for (int i = meet_a; __ldcg(&Ta.parent[i]) >= 0; i = __ldcg(&Ta.parent[i])) ++la;
        for (int i = meet_b; __ldcg(&Tb.parent[i]) >= 0; i = __ldcg(&Tb.parent[i])) ++lb;
        const int len = la + lb - 1;
        const unsigned long long need = (unsigned long long)len * dof;
        const unsigned long long off = atomicAdd(a.arena_used, need);
        sh(c.ictl)[IC_TMP4] = len;
        if (off + need > a.arena_cap || len > ib_cap) {
            sh(c.ictl)[IC_TMP4] = -1;
        } else {
            a.ctl[prob].path_off = off;
            int pos = la - 1;
            for (int i = meet_a;; i = __ldcg(&Ta.parent[i])) {
                ib[pos--] = i;  // tree 0
                if (__ldcg(&Ta.parent[i]) < 0) break;
            }
            pos = la;
            for (int i = __ldcg(&Tb.parent[meet_b]); i >= 0; i = __ldcg(&Tb.parent[i])) {
                ib[pos++] = i | (1 << 30);  // tree 1
            }
        }
    }
    __syncthreads();
    const int len = sh(c.ictl)[IC_TMP4];
    if (len < 0) return;
    const unsigned long long off = a.ctl[prob].path_off;
    for (int e = tid; e < len * dof; e += c.nthreads) {
        const int k = e / dof, d = e % dof;
        const int v = ib[k];
        const TreeRef& T = (v >> 30) ? Tb : Ta;
        a.arena[off + e] = __ldcg(&T.cfg[(size_t)d * a.stride + (v & ((1 << 30) - 1))]);
    }
    __threadfence();
    __syncthreads();
}

// The same path with one walk per tree, both trees at once: thread 0 walks
// meet_a -> root of the start tree, thread 32 meet_b -> root of the goal
// tree (one dependent L2 load per hop, instead of four passes by one
// thread); the walks are recorded in the shared pose buffer and read back
// reversed / shifted by all threads. Falls back to the serial walk when a
// branch is longer than half the buffer.
__device__ void assemble_path(Ctx& c, const PlanArgs& a, int prob, int meet_a, int meet_b) {
    const int tid = threadIdx.x;
    const int dof = c.dof;
    const TreeRef Ta = tree_ref(a, prob, 0, dof), Tb = tree_ref(a, prob, 1, dof);
    int* ib = reinterpret_cast<int*>(c.pose.get());
    const int half = (c.L * 12 * c.NS) >> 1;
    if (tid == 0 || tid == 32) {
        const bool ta = tid == 0;
        const int* par = ta ? Ta.parent : Tb.parent;
        int* w = ib + (ta ? 0 : half);
        int n = 0;
        for (int i = ta ? meet_a : meet_b;;) {
            if (n < half) w[n] = i;
            ++n;
            const int p = __ldcg(par + i);
            if (p < 0) break;
            i = p;
        }
        sh(c.ictl)[ta ? IC_TMP2 : IC_TMP3] = n;
    }
    __syncthreads();
    const int la = sh(c.ictl)[IC_TMP2], lb = sh(c.ictl)[IC_TMP3];
    __syncthreads();  // read before thread 0 may reuse the slots
    if (la > half || lb > half) {
        assemble_path_serial(c, a, prob, meet_a, meet_b);
        return;
    }
    const int len = la + lb - 1;  // the meeting configuration once (planner.cpp:139-147)
    if (tid == 0) {
        // planner.cpp:127-129: the meeting configurations must agree (the
        // reference throws logic_error; here the problem fails with that message)
        double acc = 0.0;
        for (int d = 0; d < dof; ++d) {
            const double e = __dsub_rn(__ldcg(&Ta.cfg[(size_t)d * a.stride + meet_a]),
                                       __ldcg(&Tb.cfg[(size_t)d * a.stride + meet_b]));
            acc = __dadd_rn(acc, __dmul_rn(e, e));
        }
        if (__dsqrt_rn(acc) > 1e-12) {
            sh(c.ictl)[IC_TMP4] = -2;
        } else {
            const unsigned long long need = (unsigned long long)len * dof;
            const unsigned long long off = atomicAdd(a.arena_used, need);
            sh(c.ictl)[IC_TMP4] = len;
            if (off + need > a.arena_cap) sh(c.ictl)[IC_TMP4] = -1;
            else a.ctl[prob].path_off = off;
        }
    }
    __syncthreads();
    if (sh(c.ictl)[IC_TMP4] < 0) return;
    const unsigned long long off = a.ctl[prob].path_off;
    for (int e = tid; e < len * dof; e += c.nthreads) {
        const int k = e / dof, d = e - k * dof;
        const bool inA = k < la;
        const int v = inA ? ib[la - 1 - k] : ib[half + (k - la + 1)];
        const TreeRef& T = inA ? Ta : Tb;
        a.arena[off + e] = __ldcg(&T.cfg[(size_t)d * a.stride + v]);
    }
    __threadfence();
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Debug mode (PRRTC_DEBUG_FLAGS bit 2): the tree invariants of SPEC.md:368 /
// tree.hpp:27-53 checked at every snapshot the CTA acquires — every slot
// below the published count of either tree has its ready flag at this
// launch's epoch, a parent below itself (the root: -1), and an edge to its
// parent no longer than delta (extend steps and connect sub-edges are <= delta,
// planner.cpp:35-64). Violations are counted into ctl[prob].inv_bad.
// ---------------------------------------------------------------------------
// (fields by value: a reference to the kernel's parameter block would make
// the compiler copy it to local memory)
__device__ __noinline__ void check_tree_invariants(Ctx& c, ProbCtl* ctl, const double* cfg0, const int* parent0,
                                                   const unsigned* ready0, long long stride, unsigned epoch,
                                                   double delta) {
    const int dof = c.dof;
    const double lim = delta * (1.0 + 1e-9) + 1e-12;
    int bad = 0;
    for (int t = 0; t < 2; ++t) {
        const int n = ld_acquire(&ctl->published[t]);  // (the header fenced: a fresh snapshot)
        const double* cfg = cfg0 + (size_t)t * dof * stride;
        const int* parent = parent0 + (size_t)t * stride;
        const unsigned* ready = ready0 + (size_t)t * stride;
        for (int i = threadIdx.x; i < n; i += c.nthreads) {
            if (__ldcg(ready + i) != epoch) {
                ++bad;
                continue;
            }
            const int p = __ldcg(parent + i);
            if (i == 0 ? p != -1 : (p < 0 || p >= i)) {
                ++bad;
                continue;
            }
            if (i == 0) continue;
            double acc = 0.0;
            for (int d = 0; d < dof; ++d) {
                const double e = __ldcg(cfg + (size_t)d * stride + i) - __ldcg(cfg + (size_t)d * stride + p);
                acc += e * e;
            }
            if (!(sqrt(acc) <= lim)) ++bad;
        }
    }
    if (bad) atomicAdd(&ctl->inv_bad, bad);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// the persistent planner kernel
// ---------------------------------------------------------------------------
enum : int { DONE_RUNNING = 0, DONE_SOLVED = 1, DONE_FAILED = 2, DONE_INFEASIBLE = 3 };
enum : int {
    MSG_NONE = 0,
    MSG_START = 1,
    MSG_GOAL = 2,
    MSG_CAPACITY = 3,
    MSG_BUDGET = 4,
    MSG_ARENA = 5,
    MSG_MEET = 6
};

// set by the CTA whose finish_problem settled the problem (single-problem
// launches publish the result from that CTA, see publish_result)
__shared__ int g_finisher;

__device__ void finish_problem(const PlanArgs& a, int prob, int done, int msg) {
    ProbCtl& C = a.ctl[prob];
    if (atomicCAS(&C.done, DONE_RUNNING, -1) == DONE_RUNNING) {  // claim
        C.msg = msg;
        C.t_end_ns = globaltimer();
        __threadfence();
        st_release(&C.done, done);
        atomicAdd(a.n_done, 1);
        g_finisher = 1;
    }
}

// Initialise a freshly claimed problem: endpoint checks (planner.cpp:263-285)
// and roots (planner.cpp:292-293). Returns true if the search should run.
__device__ bool init_problem(Ctx& c, const PlanArgs& a, int prob) {
    const int tid = threadIdx.x, dof = c.dof;
    ProbCtl& C = a.ctl[prob];
    double* S = dc(c, DC_A);
    double* G = dc(c, DC_B);
    if (tid < dof) {
        S[tid] = a.inline_inputs ? a.in_sg[tid] : a.starts[(size_t)prob * dof + tid];
        G[tid] = a.inline_inputs ? a.in_sg[dof + tid] : a.goals[(size_t)prob * dof + tid];
    }
    if (tid == 0) C.t_start_ns = globaltimer();
    __syncthreads();
    // states: 0 = start, 1 = goal (independent, early exit per state)
    for (int s = tid; s < c.NS; s += c.nthreads) {
        sh(c.sgroup)[s] = s < 2 ? s : -1;
        if (s < 2) {
            for (int d = 0; d < dof; ++d) sh(c.qf)[d * c.NS + s] = (float)(s == 0 ? S[d] : G[d]);
        }
    }
    __syncthreads();
    check_chunk(c, 2, a.p.two_stage != 0, a.p.early_exit != 0, true);
    if (c.ref_stats && tid < 2) {  // exact-CheckStats mode: the two endpoint checks (planner.cpp:263-277)
        int fe = 0;
        sh(c.rcount)[tid] = ref_state_count(c, tid, a.p.two_stage != 0, a.p.early_exit != 0, &fe);
        sh(c.rfine)[tid] = fe;
    }
    __syncthreads();
    if (tid == 0) {
        if (!c.ref_stats) sh(c.t0)[T0_FK] += 2;
        sh(c.stat)[1] += 2ull * c.fkflops;  // thread 0's flop slot
        // within_limits (planner.cpp:25-31): inclusive bounds
        bool sl = true, gl = true;
        for (int d = 0; d < dof; ++d) {
            const double lo = c.limits[2 * d], hi = c.limits[2 * d + 1];
            sl &= !(S[d] < lo || S[d] > hi);
            gl &= !(G[d] < lo || G[d] > hi);
        }
        int verdict = 0;
        if (!sl || sh(c.sbad)[0]) verdict = 1;
        else if (!gl || sh(c.sbad)[1]) verdict = 2;
        else {
            bool eq = true;
            for (int d = 0; d < dof; ++d) eq &= (S[d] == G[d]);
            if (eq) verdict = 3;
        }
        if (c.ref_stats && (verdict == 0 || verdict == 3)) {
            // the reference reports the endpoint checks' counters only when
            // both endpoints are feasible (planner.cpp:263-285, :308-311)
            unsigned long long* t0 = sh(c.t0);
            t0[T0_RTESTS] += sh(c.rcount)[0] + sh(c.rcount)[1];
            t0[T0_FK] += 2;
            t0[T0_FINE] += sh(c.rfine)[0] + sh(c.rfine)[1];
        }
        sh(c.ictl)[IC_TMP5] = verdict;
    }
    __syncthreads();
    const int verdict = sh(c.ictl)[IC_TMP5];
    if (verdict == 1 || verdict == 2) {
        if (tid == 0) {
            C.started = 1;
            finish_problem(a, prob, DONE_INFEASIBLE, verdict == 1 ? MSG_START : MSG_GOAL);
        }
        __syncthreads();
        return false;
    }
    if (verdict == 3) {  // start == goal: path [start], cost 0 (planner.cpp:279-285)
        if (tid == 0) {
            const unsigned long long off = atomicAdd(a.arena_used, (unsigned long long)dof);
            if (off + dof <= a.arena_cap) {
                for (int d = 0; d < dof; ++d) a.arena[off + d] = S[d];
                C.path_off = off;
                C.path_len = 1;
                C.winner = 1;
                __threadfence();
                C.started = 1;
                finish_problem(a, prob, DONE_SOLVED, MSG_NONE);
            } else {
                C.started = 1;
                finish_problem(a, prob, DONE_FAILED, MSG_ARENA);
            }
        }
        __syncthreads();
        return false;
    }
    // roots
    for (int t = 0; t < 2; ++t) {
        const TreeRef T = tree_ref(a, prob, t, dof);
        if (tid < dof) T.cfg[(size_t)tid * a.stride] = (t == 0 ? S : G)[tid];
        if (tid == 0) {
            T.parent[0] = -1;
            T.dd[0] = 0;
            T.ready[0] = a.epoch;
            *T.reserved = 1;
            *T.published = 1;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&C.started, 1);
    return true;
}

// Which running problem a free worker joins (lower key first, ties to the
// lowest index): help_policy 1 = the most unclaimed budget per worker
// (budget - tickets claimed) / (active + 1) — the longest remaining work,
// which is what bounds a batch's makespan (the hardest problems are its long
// poles and they parallelise: tools/scale_one.py); 0 = the fewest active
// workers.
__device__ __forceinline__ int help_key(const PlanArgs& a, int active, unsigned long long claimed) {
    if (a.help_policy == 0) return active;
    const unsigned long long rem = a.p.budget - claimed;  // (claimed < budget)
    const unsigned long long per = rem * 16ull / (unsigned long long)(active + 1);
    return 0x7ffffffe - (int)min(per, 0x7ffffff0ull);
}

// One pass of the help scan over problems start + i (mod n), i = t0, t0 +
// step, ... < count: an L2 read of every visited problem's (started, done,
// winner, active) word and ticket count, two independent 16 / 8-byte loads
// per problem so they pipeline (a hint only: the chosen problem is acquired
// by the caller; an acquire per problem would invalidate L1 a thousand
// times). Keeps the best help_key in bk / bp; pending: a claimed problem
// whose endpoints are still being checked.
__device__ __forceinline__ void help_scan(const PlanArgs& a, int t0, int step, int start, int count, int& bk, int& bp,
                                          int& pending) {
    for (int i = t0; i < count; i += step) {
        int q = start + i;
        if (q >= a.n_problems) q -= a.n_problems;
        const ProbCtl& C = a.ctl[q];
        const int4 hdr = __ldcg(reinterpret_cast<const int4*>(&C));  // started, done, winner, active
        const unsigned long long it = __ldcg(&C.iters);
        pending |= hdr.x == 0 && hdr.y == DONE_RUNNING;
        if (hdr.x == 1 && hdr.y == DONE_RUNNING && it < a.p.budget && (a.help_cap == 0 || hdr.w < a.help_cap)) {
            const int key = help_key(a, hdr.w, it);
            if (key < bk || (key == bk && q < bp)) {
                bk = key;
                bp = q;
            }
        }
    }
}

// Large batches scan a rotating window of kHelpWindow problems first (every
// freed worker reading all n headers cost the warp planner ~30% of its stall
// samples on a 10k-problem batch); the full scan runs when the window holds
// nothing joinable, so leaving (nothing joinable anywhere) stays exact.
constexpr int kHelpWindow = 1024;
__device__ __forceinline__ int help_window_start(int n, int attempt, int who) {
    return (int)(((unsigned)who * 2654435761u + (unsigned)attempt * 40503u + (unsigned)(clock64() & 0xffff)) %
                 (unsigned)n);
}

// Help mode: join the running problem chosen by help_key. The parallel RRT-Connect iteration is elastic: any
// number of workers may join a problem at any time. -1 when none is left.
__device__ int pick_help(Ctx& c, const PlanArgs& a) {
    const int tid = threadIdx.x;
    // help mode: running problem with the fewest active CTAs (ties -> lowest);
    // wait while problems are claimed but not yet initialised, exit when all
    // problems are finished
    for (int attempt = 0;; ++attempt) {
        if (attempt > 0) {
            if (tid == 0) sh(c.ictl)[IC_TMP1] = ld_acquire(a.n_done);
            __syncthreads();
            const bool all_done = sh(c.ictl)[IC_TMP1] >= a.n_problems;
            __syncthreads();
            if (all_done) return -1;
            __nanosleep(200);
        }
        int bk = 0x7fffffff, bp = -1, pending = 0;
        if (a.n_problems > 2 * kHelpWindow) {
            if (tid == 0) sh(c.ictl)[IC_TMP1] = help_window_start(a.n_problems, attempt, blockIdx.x);
            __syncthreads();
            const int start = sh(c.ictl)[IC_TMP1];
            __syncthreads();
            help_scan(a, tid, c.nthreads, start, kHelpWindow, bk, bp, pending);
            pending = 0;  // (the full scan below decides waiting / leaving)
        }
        if (!__syncthreads_or(bp >= 0)) help_scan(a, tid, c.nthreads, 0, a.n_problems, bk, bp, pending);
        // every problem is claimed (the claim loop ran dry) and every running
        // one has handed out its whole iteration budget: nothing can ever be
        // joined again, so leave instead of spinning (the scans of idle CTAs
        // take issue slots and L2 bandwidth from the ones still working)
        if (!__syncthreads_or(pending || bp >= 0)) return -1;
        for (int o = 16; o > 0; o >>= 1) {
            const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (ok < bk || (ok == bk && op >= 0 && (bp < 0 || op < bp))) {
                bk = ok;
                bp = op;
            }
        }
        if ((tid & 31) == 0) {
            sh(c.red_i)[tid >> 5] = bp;
            sh(c.sgroup)[tid >> 5] = bk;
        }
        __syncthreads();
        if (tid == 0) {
            int k = sh(c.sgroup)[0], p = sh(c.red_i)[0];
            for (int w = 1; w < c.nthreads / 32; ++w) {
                if (sh(c.sgroup)[w] < k || (sh(c.sgroup)[w] == k && sh(c.red_i)[w] >= 0 && (p < 0 || sh(c.red_i)[w] < p))) {
                    k = sh(c.sgroup)[w];
                    p = sh(c.red_i)[w];
                }
            }
            if (p >= 0) {
                atomicAdd(&a.ctl[p].active, 1);
                ld_acquire(&a.ctl[p].started);  // the roots are visible from here on
                if (ld_acquire(&a.ctl[p].done) != DONE_RUNNING) {
                    atomicSub(&a.ctl[p].active, 1);
                    p = -2;  // raced with completion: rescan
                }
            }
            sh(c.ictl)[IC_TMP1] = p;
        }
        __syncthreads();
        const int p = sh(c.ictl)[IC_TMP1];
        __syncthreads();
        if (p >= 0) return p;
    }
}

// CheckStats counters (collision.hpp:17-25), reduced per warp then per CTA.
__device__ void flush_stats(Ctx& c, ProbCtl& C) {
    unsigned long long* st = sh(c.stat) + 2 * threadIdx.x;
    unsigned long long tests = st[0], flops = st[1];
    st[0] = 0;
    st[1] = 0;
    for (int o = 16; o > 0; o >>= 1) {
        tests += __shfl_xor_sync(0xffffffffu, tests, o);
        flops += __shfl_xor_sync(0xffffffffu, flops, o);
    }
    if ((threadIdx.x & 31) == 0 && tests && !c.ref_stats) atomicAdd(&C.sphere_tests, tests);
    if ((threadIdx.x & 31) == 0 && flops) atomicAdd(&C.flops, flops);
    if (threadIdx.x == 0) {
        unsigned long long* t0 = sh(c.t0);
        if (t0[T0_FK]) atomicAdd(&C.fk_calls, t0[T0_FK]);
        if (t0[T0_FINE]) atomicAdd(&C.fine_entries, t0[T0_FINE]);
        if (t0[T0_RTESTS]) atomicAdd(&C.sphere_tests, t0[T0_RTESTS]);
        t0[T0_FK] = 0;
        t0[T0_FINE] = 0;
        t0[T0_RTESTS] = 0;
    }
}

// Leaving a problem: the last worker out of an unsolved problem fails it
// (planner.cpp:317-320: all workers exhausted their budgets).
__device__ void leave_problem(const PlanArgs& a, int prob, int reason_msg) {
    ProbCtl& C = a.ctl[prob];
    const int prev = atomicSub(&C.active, 1);
    if (reason_msg == MSG_CAPACITY) {
        finish_problem(a, prob, DONE_FAILED, MSG_CAPACITY);
    } else if (prev == 1 && ld_acquire(&C.done) == DONE_RUNNING) {
        finish_problem(a, prob, DONE_FAILED, MSG_BUDGET);
    }
}

#define TRACE_PHASE(code) trace_phase<TR>(a, code)

__shared__ Ctx g_ctx;  // the planner's CTA context (see ctx_writer)

// Single-problem launches: the CTA that settled the problem (the winner, the
// last worker out of a failed problem, or the endpoint check) copies the
// out-header, controls and used path arena into mapped pinned host memory as
// soon as it has left the problem, and raises a flag there (out_map[0] =
// epoch, out_map[1] = 1 if it fit): the host reads the result without a D2H
// copy and without waiting for the other CTAs to notice the settled problem
// and retire. (CheckStats / iteration counters of CTAs still leaving are not
// in that snapshot; with one CTA — deterministic mode — they are exact.)
__device__ void publish_result(Ctx& c, const PlanArgs& a) {
    const int tid = threadIdx.x;
    __syncthreads();
    if (!g_finisher) return;
    __threadfence();
    const unsigned long long used = min(__ldcg(a.arena_used), a.arena_cap);
    const unsigned long long words = (a.out_hdr_bytes >> 3) + used;  // 8-byte words: header, controls, arena
    const bool fits = 64 + 8 * words <= a.out_map_bytes;
    if (fits) {
        const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.out_dev);
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.out_map + 64);
        for (unsigned long long i = tid; i < words; i += blockDim.x) dst[i] = __ldcg(src + i);
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
        volatile unsigned* f = reinterpret_cast<volatile unsigned*>(a.out_map);
        f[1] = fits ? 1u : 0u;
        __threadfence_system();
        f[0] = a.epoch;
    }
}

// TR: the PRRTC_TRACE instantiation (phase ring, per-CTA stamps); the
// production one carries no trace code in its loop (hot code above the
// 32 KB L1.5 instruction cache stalls on fetch)
template <int NT, int MINB, bool TR>
__global__ void __launch_bounds__(NT, MINB) plan_kernel(PlanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx& c = g_ctx;
    setup_ctx(c, smem, a.robot, reinterpret_cast<const int*>(a.robot)[RH_WORDS], a.fine_r64,
              a.limits, a.ns_max, plan_scene_words(a), a.p.uniform != 0);
    const int tid = threadIdx.x;
    const int dof = c.dof;
    const int robot_words = reinterpret_cast<const int*>(a.robot)[RH_WORDS];
    unsigned char* sbase = scene_base(smem, robot_words, c.L, dof, c.NS, c.nthreads);
    build_ttab(c, a.p.n_cc);
    if (tid == 0) c.ref_stats = a.ref_stats;
    __syncthreads();
    if (tid == 0) g_finisher = 0;
    if (a.inline_inputs) {
        // no H2D copy: CTA 0 zeroes the out-header and the problem's
        // controls, then releases the init word (its own buffer); the other
        // CTAs acquire it before they touch either (all CTAs of a
        // single-problem launch are co-resident)
        if (blockIdx.x == 0) {
            unsigned* hdr = const_cast<unsigned*>(reinterpret_cast<const unsigned*>(a.out_dev));
            const int hwords = (int)(a.out_hdr_bytes >> 2);
            for (int i = tid; i < hwords; i += c.nthreads) hdr[i] = 0u;
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release_u(a.init_flag, a.epoch);
        } else {
            if (tid == 0)
                while (ld_acquire_u(a.init_flag) != a.epoch) __nanosleep(32);
            __syncthreads();
        }
    }
    const double R = a.p.dd_radius, delta = a.p.delta;
    if (tid == 0 && a.trace) atomicMax(&a.trace[0], 0x7fffffffffffffffull - (unsigned long long)globaltimer());
    if (TR && tid == 0 && a.cta_trace) {
        for (int k = 0; k < kTraceStride; ++k) g_trace[k] = 0;
        g_trace[3] = globaltimer();
    }

    for (;;) {
        int prob = -1;
        // unstarted problems first: claim, stage its scene, initialise
        for (;;) {
            if (tid == 0) sh(c.ictl)[IC_TMP1] = atomicAdd(a.next_problem, 1);
            __syncthreads();
            const int p = sh(c.ictl)[IC_TMP1];
            __syncthreads();
            if (p >= a.n_problems) break;
            if (a.inline_inputs) {
                load_scene(c, sbase, a.scene_words1, a.scene_f64_1);
            } else {
                const int si = a.prob_scene[p];
                load_scene(c, sbase, a.scene_words[si], a.scene_f64[si]);
            }
            if (tid == 0) atomicAdd(&a.ctl[p].active, 1);
            if (init_problem(c, a, p)) {
                prob = p;
                break;
            }
            flush_stats(c, a.ctl[p]);
            if (tid == 0) atomicSub(&a.ctl[p].active, 1);
            __syncthreads();
        }
        if (prob < 0) {
            if (a.p.deterministic) break;
            prob = pick_help(c, a);
            if (prob < 0) break;
            if (a.inline_inputs) {
                load_scene(c, sbase, a.scene_words1, a.scene_f64_1);
            } else {
                const int si = a.prob_scene[prob];
                load_scene(c, sbase, a.scene_words[si], a.scene_f64[si]);
            }
        }
        ProbCtl& C = a.ctl[prob];
        if (tid == 0) {  // the roots: written by this CTA, or acquired through `started` (pick_help)
            sh(c.ictl)[IC_KNOWN0] = 1;
            sh(c.ictl)[IC_KNOWN1] = 1;
            sh(c.ictl)[IC_DIRTY] = 1;
        }
        // Halton tickets are claimed in blocks of kblk (one atomic per block,
        // every ticket still used once, in order within the CTA); the block's
        // samples are computed by all threads at once into sbuf. The ticket
        // state and iteration counters are thread 0's, in shared memory (t0).
        const int kblk = 32;
        if (tid == 0) {
            unsigned long long* t0 = sh(c.t0);
            t0[T0_TKBASE] = t0[T0_TKPOS] = t0[T0_TKCNT] = t0[T0_USED] = t0[T0_LITER] = 0;
            // Uniform sampler: a fresh generator per (problem, worker), seeded as
            // the reference's worker `blockIdx` (worker 0 in deterministic mode)
            if (a.p.uniform)
                mt_seed(sh(c.mt), a.p.seed * 0x9e3779b97f4a7c15ull + (a.p.deterministic ? 0u : blockIdx.x));
        }
        int leave_msg = MSG_NONE;
        for (;;) {
            // ---- iteration header (lead thread) ----
            TRACE_PHASE(1);
            if (tid == 0) {
                unsigned long long* t0 = sh(c.t0);
                unsigned long long tk_base = t0[T0_TKBASE], tk_pos = t0[T0_TKPOS], tk_cnt = t0[T0_TKCNT];
                const unsigned long long local_iter = t0[T0_LITER];
                // the done flag and both published counts are read back to
                // back (relaxed done, acquire counts)
                const int dn = ld_relaxed(&C.done);
                int refill = 0;
                if (tk_pos == tk_cnt) {
                    // near the end of the problem's budget, smaller blocks: the
                    // last tickets spread over more CTAs instead of a few CTAs
                    // holding 32 each while the others idle (a.tail_claim)
                    unsigned long long want = kblk;
                    if (a.tail_claim && !a.p.deterministic) {
                        const unsigned long long seen = tk_cnt ? tk_base + tk_cnt : __ldcg(&C.iters);
                        const int act = max(1, ld_relaxed(&C.active));
                        if (seen < a.p.budget)
                            want = max((unsigned long long)a.tail_min,
                                       min((unsigned long long)kblk, (a.p.budget - seen) / ((unsigned long long)a.tail_div * act)));
                    }
                    tk_base = a.p.deterministic ? tk_base + tk_cnt : atomicAdd(&C.iters, want);
                    tk_pos = 0;
                    tk_cnt = want;
                    refill = 1;
                }
                const unsigned long long it = tk_base + tk_pos;
                const int la = ld_relaxed(&C.published[0]);
                const int lb = ld_relaxed(&C.published[1]);
                // a snapshot beyond what the CTA already holds needs acquire
                // ordering (fence after the relaxed reads, which also drops
                // the SM's L1 lines) before plain loads of the new slots; a
                // CTA working alone never pays it — its own stores are
                // coherent with its SM's L1 (program order), so its own
                // appends and dynamic-domain flags need no fence (IC_DIRTY
                // only forces one when the CTA joins a problem)
                int* known = sh(c.ictl) + IC_KNOWN0;
                if (la > known[0] || lb > known[1] || sh(c.ictl)[IC_DIRTY] || (a.dbg & 5)) {
                    fence_acq_rel();
                    known[0] = max(known[0], la);
                    known[1] = max(known[1], lb);
                    sh(c.ictl)[IC_DIRTY] = 0;
                }
                const int leave = dn != DONE_RUNNING ? 1 : (it >= a.p.budget ? 2 : 0);
                // extend_start_tree (planner.hpp:62-65)
                const int from_start = a.p.balance ? (la <= lb) : ((local_iter & 1) == 0);
                const int snap = from_start ? la : lb;
                t0[T0_LITER] = local_iter + 1;
                t0[T0_USED] += leave == 0;
                sh(c.ictl)[IC_TMP0] = leave;
                sh(c.ictl)[IC_TMP1] = from_start;
                sh(c.ictl)[IC_TMP2] = snap;
                sh(c.ictl)[IC_TMP3] = refill;
                // tickets of the block from this one on that are within the
                // budget: the samples a multi-sample NN pass may consume
                const unsigned long long rem = tk_cnt - tk_pos;
                sh(c.ictl)[IC_TMP5] = (int)(it < a.p.budget ? min(rem, a.p.budget - it) : 1ull);
                sh(c.ictl)[IC_TMP4] = (int)tk_pos++;
                sh(c.ictl)[IC_TMP7] = (int)tk_cnt;
                reinterpret_cast<unsigned long long*>(sh(c.red_d))[0] = tk_base;
                t0[T0_TKBASE] = tk_base;
                t0[T0_TKPOS] = tk_pos;
                t0[T0_TKCNT] = tk_cnt;
            }
            __syncthreads();
            const int leave = sh(c.ictl)[IC_TMP0];
            if (leave) {
                leave_msg = leave == 2 ? MSG_BUDGET : MSG_NONE;
                break;
            }
            if (a.dbg & 4)
                check_tree_invariants(c, &C, a.cfg + (size_t)prob * 2 * dof * a.stride, a.parent + (size_t)prob * 2 * a.stride,
                                      a.ready + (size_t)prob * 2 * a.stride, a.stride, a.epoch, a.p.delta);
            const int ts = sh(c.ictl)[IC_TMP1] ? 0 : 1;
            const int snap = sh(c.ictl)[IC_TMP2];
            const int refill = sh(c.ictl)[IC_TMP3];
            const int slot = sh(c.ictl)[IC_TMP4];
            const TreeRef Ts = tree_ref(a, prob, ts, dof);
            const TreeRef To = tree_ref(a, prob, 1 - ts, dof);
            // ---- sample (sampling.cpp:39-51): a whole ticket block at once,
            // one thread per (ticket, dimension), Halton index 1 + seed + ticket
            if (refill) {
                TRACE_PHASE(7);
                const unsigned long long base = reinterpret_cast<unsigned long long*>(sh(c.red_d))[0];
                const int nblk = sh(c.ictl)[IC_TMP7];
                __syncthreads();  // header scalars read before they are reused
                if (a.p.uniform) {  // the CTA's own stream, in draw order (sampling.hpp:44-48)
                    mt_fill(sh(c.mt), sh(c.limits), dof, sh(c.sbuf), nblk * dof, c.nthreads);
                } else if (base + nblk <= a.stab_n) {
                    // every problem of the launch draws the same samples (same
                    // robot limits, seed and ticket range): the block is one
                    // contiguous run of the per-launch table, copied with up
                    // to four independent loads in flight per thread (one L2
                    // round trip per block instead of one per element)
                    const double* src = a.stab + base * dof;
                    double* dst = sh(c.sbuf);
                    const int tot = nblk * dof, nt = c.nthreads;
                    for (int j0 = tid; j0 < tot; j0 += 4 * nt) {
                        double v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] = j0 + u * nt < tot ? __ldg(src + j0 + u * nt) : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (j0 + u * nt < tot) dst[j0 + u * nt] = v[u];
                    }
                } else
                for (int j = tid; j < nblk * dof; j += c.nthreads) {
                    const int k = j / dof, d = j - k * dof;
                    // every problem of the launch draws the same samples (same
                    // robot limits, seed and ticket range): the per-launch
                    // table holds them, computed by this same routine
                    const unsigned long long t = base + k;
                    sh(c.sbuf)[j] = t < a.stab_n ? __ldg(a.stab + t * dof + d)
                                                 : sample_dim(halton_tab(sh(c.bases)[d], sh(c.magic)[d],
                                                                         sh(c.htab) + d * kHaltonTab, 1ull + a.p.seed + t),
                                                              sh(c.limits)[2 * d], sh(c.limits)[2 * d + 1]);
                }
            }
            __syncthreads();
            // ---- nearest neighbour(s) in the extended tree ----
            // While the tree is unchanged the samples of the block that the
            // sequential loop would draw next meet the same snapshot, so
            // (balanced mode: the extended tree does not alternate) up to 32
            // of them are evaluated in one pass, bounded to ~8 node pairs per
            // thread; the loop then continues with the first accepted one and
            // the rejected ones count as iterations — the same outcome as
            // one NN scan and accept test per iteration (planner.cpp:216-219).
            TRACE_PHASE(2);
            int m = 1;
            if (a.p.balance) m = max(1, min(sh(c.ictl)[IC_TMP5], a.mnn_nodes / max(1, snap)));
            // (the scan also evaluates each sample's acceptance: duplicate,
            // planner.cpp:218 / DynamicDomain::accept, sampling.hpp:61-75)
            nn_scan_multi(c, Ts.cfg, a.stride, snap, sh(c.sbuf) + slot * dof, m,
                          a.p.dynamic_domain ? Ts.dd : nullptr, true, R);
            TRACE_PHASE(3);
            const unsigned okm = __ballot_sync(0xffffffffu, (tid & 31) < m && sh(c.mnn_ok)[tid & 31]);
            const int first = okm ? __ffs(okm) - 1 : m;
            if (tid == 0) {  // the rejected samples before `first` were iterations too
                const int extra = (first < m ? first + 1 : m) - 1;
                unsigned long long* t0 = sh(c.t0);
                t0[T0_TKPOS] += extra;
                t0[T0_USED] += extra;
                t0[T0_LITER] += extra;
            }
            if (first == m) continue;
            const double* smp = sh(c.sbuf) + (slot + first) * dof;
            const int nn = sh(c.mnn_i)[first];
            const double d2 = sh(c.mnn_d)[first];
            const double dist = __dsqrt_rn(d2);
            const double v = tid < dof ? Ts.cfg[(size_t)tid * a.stride + nn] : 0.0;  // L1: the scan read it
            // ---- steer (planner.cpp:48-64) ----
            double* nnc = dc(c, DC_NN);
            double* cnew = dc(c, DC_NEW);
            if (tid < dof) {
                nnc[tid] = v;
                cnew[tid] = dist <= delta ? smp[tid] : lerp_exact(v, smp[tid], __ddiv_rn(delta, dist));
            }
            __syncthreads();
            // ---- SIMT edge validation nn -> c_new, then append (phase 0),
            // then greedy connect c_new -> the opposite tree (phase 1): one
            // validate_chain call site for both, so the chain/chunk code is
            // inlined once (no ABI register saves per chunk)
            // (the done flag is sampled in every chunk: a CTA still working
            // when another one solved the problem leaves at the next chunk
            // instead of finishing the iteration — the result is settled)
            const double* VA = nnc;
            const double* VB = cnew;
            long long nsub = 1;
            int par0 = nn, phase = 0, new_idx = nn, nno = -1, meet_self = nn;
            int outcome = 0;  // 0 next iteration, 1 reached, 2 tree full
#pragma unroll 1
            for (;;) {
                int last = par0;
                bool stopped = false;
                const long long got = validate_chain<TR>(c, a, VA, VB, nsub, &Ts, par0, &last, &C.done, &stopped);
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
                    if (a.p.dynamic_domain && tid == 0) Ts.dd[nn] = 1;  // record_failure
                    break;
                }
                new_idx = meet_self = last;
                // ---- greedy connect toward the opposite tree ----
                TRACE_PHASE(4);
                if (tid == 0) {
                    const int po = ld_relaxed(To.published);
                    sh(c.ictl)[IC_TMP3] = ld_relaxed(&C.done);  // settled meanwhile: skip the connect
                    int* known = sh(c.ictl) + IC_KNOWN0 + To.which;
                    if (po > *known || (a.dbg & 5)) {
                        fence_acq_rel();
                        *known = po;
                    }
                    sh(c.ictl)[IC_TMP2] = po;
                }
                __syncthreads();
                const int snap_o = sh(c.ictl)[IC_TMP2];
                const int settled = sh(c.ictl)[IC_TMP3];
                __syncthreads();
                if (settled != DONE_RUNNING) break;  // the header leaves
                nn_scan_multi(c, To.cfg, a.stride, snap_o, cnew, 1, nullptr);
                nno = sh(c.mnn_i)[0];
                const double d2o = sh(c.mnn_d)[0];
                if (d2o == 0.0) {
                    outcome = 1;
                    break;
                }
                const double disto = __dsqrt_rn(d2o);
                double* tgt = dc(c, DC_TARGET);
                double* A = dc(c, DC_A);
                if (tid < dof) {
                    tgt[tid] = To.cfg[(size_t)tid * a.stride + nno];
                    A[tid] = cnew[tid];
                }
                __syncthreads();
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
            TRACE_PHASE(6);
            if (tid == 0) sh(c.ictl)[IC_TMP6] = (atomicCAS(&C.winner, 0, blockIdx.x + 1) == 0);
            __syncthreads();
            if (sh(c.ictl)[IC_TMP6]) {
                const int meet_a = ts == 0 ? meet_self : nno;
                const int meet_b = ts == 0 ? nno : meet_self;
                if (tid == 0) {
                    C.meet[0] = meet_a;
                    C.meet[1] = meet_b;
                }
                assemble_path(c, a, prob, meet_a, meet_b);
                if (tid == 0) {
                    if (sh(c.ictl)[IC_TMP4] < 0) {
                        finish_problem(a, prob, DONE_FAILED, sh(c.ictl)[IC_TMP4] == -2 ? MSG_MEET : MSG_ARENA);
                    } else {
                        C.path_len = sh(c.ictl)[IC_TMP4];
                        __threadfence();
                        finish_problem(a, prob, DONE_SOLVED, MSG_NONE);
                    }
                }
            }
            break;
        }
        // ---- leave ----
        TRACE_PHASE(10);
        if (tid == 0 && sh(c.t0)[T0_USED]) atomicAdd(&C.iters_used, sh(c.t0)[T0_USED]);
        if (TR && tid == 0 && a.cta_trace) g_trace[0] = globaltimer();
        flush_stats(c, C);
        if (tid == 0) leave_problem(a, prob, leave_msg);
        __syncthreads();
        if (TR && tid == 0 && a.cta_trace) g_trace[1] = globaltimer();
        // a single problem: nothing left to claim or help once it is left
        // (skips the claim / help-scan round trips on the way out)
        if (a.n_problems == 1) break;
    }
    if (tid == 0 && a.trace) atomicMax(&a.trace[1], (unsigned long long)globaltimer());
    if (TR && tid == 0 && a.cta_trace) {
        TRACE_PHASE(0);  // close the last phase
        g_trace[2] = globaltimer();
        for (int k = 0; k < kTraceStride; ++k) a.cta_trace[blockIdx.x * kTraceStride + k] = g_trace[k];
    }
    if (a.out_map) publish_result(c, a);
}

// ---------------------------------------------------------------------------
// device re-validation of the returned paths (SURVEY.md §8f
// rank 1): every edge of every solved problem's path (already in the arena)
// is checked at 4 * n_cc states, fine spheres only, no early exit — the
// reference's soundness criterion — by a second kernel on the planner's
// stream. path_edges_scan_kernel lays the edges out (exclusive prefix over
// problems, one CTA); validate_paths_kernel takes edges grid-stride, finds
// the problem by binary search and ORs a collision into ctl[p].path_bad.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) path_edges_scan_kernel(const ProbCtl* ctl, int n, int* prefix) {
    __shared__ int part[1024];
    const int tid = threadIdx.x, per = (n + 1023) / 1024;
    const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
    int sum = 0;
    for (int p = b0; p < b1; ++p) sum += (ctl[p].done == 1 && ctl[p].path_len > 1) ? ctl[p].path_len - 1 : 0;
    part[tid] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan
        const int v = tid >= o ? part[tid - o] : 0;
        __syncthreads();
        part[tid] += v;
        __syncthreads();
    }
    int run = tid ? part[tid - 1] : 0;
    for (int p = b0; p < b1; ++p) {
        prefix[p] = run;
        run += (ctl[p].done == 1 && ctl[p].path_len > 1) ? ctl[p].path_len - 1 : 0;
    }
    if (tid == 1023) prefix[n] = part[1023];
}

__global__ void __launch_bounds__(128) validate_paths_kernel(PlanArgs a, const int* prefix, int n_cc4) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx c;
    setup_ctx(c, smem, a.robot, reinterpret_cast<const int*>(a.robot)[RH_WORDS], a.fine_r64, a.limits,
              a.ns_max);
    unsigned char* sbase = scene_base(smem, reinterpret_cast<const int*>(a.robot)[RH_WORDS], c.L, c.dof,
                                      c.NS, c.nthreads);
    const int total = prefix[a.n_problems];
    int cur_scene = -1;
    for (int E = blockIdx.x; E < total; E += gridDim.x) {
        int lo = 0, hi = a.n_problems - 1;  // last p with prefix[p] <= E
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= E) lo = mid;
            else hi = mid - 1;
        }
        const int p = lo, e = E - prefix[p];
        const int si = a.prob_scene[p];
        if (si != cur_scene) {
            load_scene(c, sbase, a.scene_words[si], a.scene_f64[si]);
            cur_scene = si;
        }
        const double* A = a.arena + a.ctl[p].path_off + (size_t)e * c.dof;
        double* sa = dc(c, DC_A);
        double* sb = dc(c, DC_B);
        if (threadIdx.x < c.dof) {
            sa[threadIdx.x] = A[threadIdx.x];
            sb[threadIdx.x] = A[c.dof + threadIdx.x];
        }
        __syncthreads();
        // the reference's soundness check is fine-only with early exit off
        // (SPEC.md:367); the verdict is the same with the two-stage checker
        // (its padded coarse stage never hides a fine hit: two-stage == brute
        // force, test_check_configs_bitexact_on_device_spheres) stopping at
        // the first colliding chunk — only CheckStats would differ, and none
        // are reported here (~5x fewer sphere tests on a sound path)
        int bad = 0;
        for (int g0 = 0; g0 < n_cc4 && !bad; g0 += c.NS) {
            const int cnt = min(c.NS, n_cc4 - g0);
            gen_chain_states(c, sa, sb, 1, n_cc4, g0, cnt, nullptr);
            check_chunk(c, cnt, true, true, false);
            bad = sh(c.ictl)[IC_FIRSTBAD] != kNoBad;
            __syncthreads();
        }
        if (threadIdx.x == 0 && bad) atomicOr(&a.ctl[p].path_bad, 1);
    }
}

// cudaFuncSetAttribute costs microseconds per call: raise the dynamic shared
// memory limit of a (kernel, device) only when a launch needs more than it
// was last set to
cudaError_t raise_smem_limit(const void* fn, int sm) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> set;
    int dev = 0;
    cudaGetDevice(&dev);
    // per-thread fast path: the limits only ever grow, so a (kernel, device)
    // this thread has seen at >= sm needs no lock
    thread_local const void* last_fn = nullptr;
    thread_local int last_dev = -1, last_sm = 0;
    if (fn == last_fn && dev == last_dev && sm <= last_sm) return cudaSuccess;
    std::lock_guard<std::mutex> lk(mu);
    int& cur = set[{fn, dev}];
    cudaError_t e = cudaSuccess;
    if (sm > cur) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        if (e == cudaSuccess) cur = sm;
    }
    if (e == cudaSuccess) {
        last_fn = fn;
        last_dev = dev;
        last_sm = cur;
    }
    return e;
}

#include "prrtc_warp.cuh"  // the warp-worker batch planner (plan_warp_kernel)

cudaError_t launch_validate_paths(const RobotArgs& r, const PlanArgs& a, int* prefix, int grid, cudaStream_t st) {
    path_edges_scan_kernel<<<1, 1024, 0, st>>>(a.ctl, a.n_problems, prefix);
    // the warp checker (one edge per warp) when the robot and the launch's
    // largest scene fit a warp region; the CTA-wide kernel otherwise
    if (r.host_words && a.scene_words_max > 0) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int warps = warp_workers_per_sm(r.host_words, a.scene_words_max, optin);
        if (warps > 0) {
            const size_t sm = warp_smem_bytes(r.host_words, a.scene_words_max, warps);
            cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(validate_paths_warp_kernel), (int)sm);
            if (e != cudaSuccess) return e;
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            validate_paths_warp_kernel<<<sms, 32 * warps, sm, st>>>(a, prefix, 4 * a.p.n_cc);
            return cudaGetLastError();
        }
    }
    const size_t sm = smem_bytes(r, a.ns_max, 128, SCENE_MAX_WORDS, true);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(validate_paths_kernel), (int)sm);
    if (e != cudaSuccess) return e;
    validate_paths_kernel<<<grid, 128, sm, st>>>(a, prefix, 4 * a.p.n_cc);
    return cudaGetLastError();
}

// CTA size variants: 128 threads (4 warps, up to 4 CTAs/SM) and 256 threads
// (8 warps, 2 CTAs/SM: each iteration's parallel phases finish faster).
using PlanFn = void (*)(PlanArgs);
// (5 or 6 CTAs of 128 threads per SM, 96 / 80 registers, spill and were
// measured 12-25% slower: DESIGN.md §9)
static PlanFn plan_fn(int nthreads, bool trace) {
    if (trace) {
        if (nthreads == 256) return plan_kernel<256, 2, true>;
        if (nthreads == 512) return plan_kernel<512, 1, true>;
        return plan_kernel<128, 4, true>;
    }
    if (nthreads == 256) return plan_kernel<256, 2, false>;
    if (nthreads == 512) return plan_kernel<512, 1, false>;
    return plan_kernel<128, 4, false>;
}

cudaError_t launch_plan(const RobotArgs& r, PlanArgs a, int grid, cudaStream_t st) {
    const size_t sm = smem_bytes(r, a.ns_max, a.nthreads, plan_scene_words(a), a.p.uniform != 0);
    const PlanFn fn = plan_fn(a.nthreads, a.cta_trace != nullptr);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(fn), (int)sm);
    if (e != cudaSuccess) return e;
    void* args[] = {&a};
    return cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(a.nthreads), args, sm, st);
}

int plan_occupancy(const RobotArgs& r, int ns_max, int nthreads, int scene_words, bool with_mt) {
    const size_t sm = smem_bytes(r, ns_max, nthreads, scene_words, with_mt);
    const PlanFn fn = plan_fn(nthreads, false);
    raise_smem_limit(reinterpret_cast<const void*>(fn), (int)sm);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, nthreads, sm) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

// ---------------------------------------------------------------------------
// batched collision checking kernels (product API) and parity hooks
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) check_configs_kernel(RobotArgs r, SceneArgs sa, const double* q,
                                                             int n, int two_stage, uint8_t* out,
                                                             int NS) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx c;
    setup_ctx(c, smem, r.words, r.n_words, r.fine_r64, r.limits, NS);
    load_scene(c, scene_base(smem, r.n_words, c.L, c.dof, NS, c.nthreads), sa.words, sa.f64);
    for (long long base = (long long)blockIdx.x * NS; base < n; base += (long long)gridDim.x * NS) {
        const int cnt = (int)min((long long)NS, n - base);
        for (int s = threadIdx.x; s < NS; s += c.nthreads) {
            sh(c.sgroup)[s] = s < cnt ? s : -1;
            if (s < cnt)
                for (int d = 0; d < c.dof; ++d) sh(c.qf)[d * NS + s] = (float)q[(base + s) * c.dof + d];
        }
        __syncthreads();
        check_chunk(c, cnt, two_stage != 0, true, true);
        for (int s = threadIdx.x; s < cnt; s += c.nthreads) out[base + s] = sh(c.sbad)[s] ? 0 : 1;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(128) validate_edges_kernel(RobotArgs r, SceneArgs sa, const double* from,
                                                              const double* to, int n_edges, int n_cc,
                                                              int two_stage, int early_exit,
                                                              uint8_t* out, int NS, long long* prof,
                                                              unsigned long long* counters) {
    extern __shared__ __align__(16) unsigned char smem[];
    const long long t0 = clock64();
    Ctx c;
    setup_ctx(c, smem, r.words, r.n_words, r.fine_r64, r.limits, NS);
    load_scene(c, scene_base(smem, r.n_words, c.L, c.dof, NS, c.nthreads), sa.words, sa.f64);
    build_ttab(c, n_cc);
    c.prof = nullptr;
    if (prof && blockIdx.x == 0) {
        // debug hook: phase stamps of the first chunk, warm: the chunk is
        // checked three times untimed (instruction cache, robot and scene
        // lines), then once with stamps
        long long* p = prof;
        prof = nullptr;
        for (int rep = 0; rep < 4; ++rep) {
            double* A = dc(c, DC_A);
            double* B = dc(c, DC_B);
            if (threadIdx.x < c.dof) {
                A[threadIdx.x] = from[threadIdx.x];
                B[threadIdx.x] = to[threadIdx.x];
            }
            __syncthreads();
            if (rep == 3) {
                c.prof = p;
                if (threadIdx.x == 0) {
                    p[0] = t0;
                    p[7] = clock64();
                }
            }
            gen_chain_states(c, A, B, 1, n_cc, 0, (int)min((long long)NS, (long long)n_cc), nullptr);
            if (c.prof && threadIdx.x == 0) c.prof[8] = clock64();
            check_chunk(c, (int)min((long long)NS, (long long)n_cc), two_stage != 0, early_exit != 0, false);
            __syncthreads();
            if (c.prof && threadIdx.x == 0) c.prof[9] = clock64();
            c.prof = nullptr;
        }
    }
    for (int e = blockIdx.x; e < n_edges; e += gridDim.x) {
        double* A = dc(c, DC_A);
        double* B = dc(c, DC_B);
        if (threadIdx.x < c.dof) {
            A[threadIdx.x] = from[(size_t)e * c.dof + threadIdx.x];
            B[threadIdx.x] = to[(size_t)e * c.dof + threadIdx.x];
        }
        __syncthreads();
        bool bad = false;
        for (long long g0 = 0; g0 < n_cc && !(bad && early_exit); g0 += NS) {
            const int cnt = (int)min((long long)NS, n_cc - g0);
            const int act = gen_chain_states(c, A, B, 1, n_cc, g0, cnt, nullptr);
            if (counters && threadIdx.x == 0) sh(c.stat)[1] += (unsigned long long)act * c.fkflops;
            check_chunk(c, cnt, two_stage != 0, early_exit != 0, false);
            bad |= sh(c.ictl)[IC_FIRSTBAD] != kNoBad;
            __syncthreads();
        }
        if (threadIdx.x == 0) out[e] = bad ? 0 : 1;
        __syncthreads();
    }
    if (counters) {  // measurement: executed sphere tests and algorithmic flops
        unsigned long long t = sh(c.stat)[2 * threadIdx.x], f = sh(c.stat)[2 * threadIdx.x + 1];
        for (int o = 16; o > 0; o >>= 1) {
            t += __shfl_xor_sync(0xffffffffu, t, o);
            f += __shfl_xor_sync(0xffffffffu, f, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&counters[0], t);
            atomicAdd(&counters[1], f);
        }
    }
}

// Edge-level parity hook: every sample of every edge checked (no early exit,
// independent states), per-state verdicts and posed fine spheres written out.
__global__ void __launch_bounds__(128) debug_check_edges_kernel(RobotArgs r, SceneArgs sa, const double* from,
                                                                 const double* to, int n_edges, int n_cc,
                                                                 int two_stage, uint8_t* state_valid,
                                                                 float* fine_out, int NS) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx c;
    setup_ctx(c, smem, r.words, r.n_words, r.fine_r64, r.limits, NS);
    load_scene(c, scene_base(smem, r.n_words, c.L, c.dof, NS, c.nthreads), sa.words, sa.f64);
    build_ttab(c, n_cc);
    const double* tt = n_cc == c.ttab_n ? sh(c.ttab) : nullptr;
    for (int e = blockIdx.x; e < n_edges; e += gridDim.x) {
        const double* A = from + (size_t)e * c.dof;
        const double* B = to + (size_t)e * c.dof;
        for (int g0 = 0; g0 < n_cc; g0 += NS) {
            const int cnt = min(NS, n_cc - g0);
            for (int idx = threadIdx.x; idx < c.dof * NS; idx += c.nthreads) {
                const int d = idx / NS, s = idx - d * NS;
                const int i = g0 + s + 1;
                if (d == 0) sh(c.sgroup)[s] = s < cnt ? 0 : -1;
                if (s >= cnt) continue;
                sh(c.qf)[idx] = i == n_cc ? (float)B[d]
                                          : (float)lerp_exact(A[d], B[d], tt ? tt[i] : frac_div(i, n_cc));
            }
            __syncthreads();
            check_chunk(c, cnt, two_stage != 0, false, true);
            for (int s = threadIdx.x; s < cnt; s += c.nthreads)
                state_valid[(size_t)e * n_cc + g0 + s] = sh(c.sbad)[s] ? 0 : 1;
            if (fine_out) {
                for (int it = threadIdx.x; it < cnt * c.S; it += c.nthreads) {
                    const int s = it % cnt, j = it / cnt;
                    const float4 f = c.fine[j];
                    const float3 x = pose_point(c, c.flink[j], s, f.x, f.y, f.z);
                    float* o = fine_out + (((size_t)e * n_cc + g0 + s) * c.S + j) * 3;
                    o[0] = x.x;
                    o[1] = x.y;
                    o[2] = x.z;
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(128) debug_fk_kernel(RobotArgs r, const double* q, int n, float* fine_out,
                                                        float* coarse_out, int NS) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx c;
    setup_ctx(c, smem, r.words, r.n_words, r.fine_r64, r.limits, NS);
    for (long long base = (long long)blockIdx.x * NS; base < n; base += (long long)gridDim.x * NS) {
        const int cnt = (int)min((long long)NS, n - base);
        for (int s = threadIdx.x; s < NS; s += c.nthreads) {
            if (s < cnt)
                for (int d = 0; d < c.dof; ++d) sh(c.qf)[d * NS + s] = (float)q[(base + s) * c.dof + d];
        }
        __syncthreads();
        fk_chunk(c, cnt);
        if (fine_out) {
            for (int it = threadIdx.x; it < cnt * c.S; it += c.nthreads) {
                const int s = it % cnt, j = it / cnt;
                const float4 f = c.fine[j];
                const float3 x = pose_point(c, c.flink[j], s, f.x, f.y, f.z);
                float* o = fine_out + ((base + s) * c.S + j) * 3;
                o[0] = x.x;
                o[1] = x.y;
                o[2] = x.z;
            }
        }
        if (coarse_out) {
            for (int it = threadIdx.x; it < cnt * c.L; it += c.nthreads) {
                const int s = it % cnt, l = it / cnt;
                float* o = coarse_out + ((base + s) * c.L + l) * 3;
                const float* C = sh(c.ccen) + (size_t)l * 3 * NS + s;
                o[0] = C[0];
                o[1] = C[NS];
                o[2] = C[2 * NS];
            }
        }
        __syncthreads();
    }
}

__global__ void debug_hits_kernel(SceneArgs sa, const float* centers, const double* radii, int n,
                                  int n_prims, uint8_t* hits) {
    __shared__ __align__(16) uint32_t sw[SCENE_MAX_WORDS];
    const int words = sa.words[SH_WORDS];
    for (int i = threadIdx.x; i < words; i += blockDim.x) sw[i] = sa.words[i];
    __syncthreads();
    // static shared memory: the view is built directly (sh() is for the
    // dynamic window only)
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
    v.s64 = sa.f64;
    for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < (long long)n * n_prims;
         it += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(it / n_prims), p = (int)(it % n_prims);
        const float3 x = make_float3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
        hits[it] = fine_vs_prim(v, x, (float)radii[i], radii[i], p) ? 1 : 0;
    }
}

// nn_scan_multi over groups of `group` queries (the planner's multi-sample
// pass): the parity tests run it against the reference's nearest_serial
__global__ void debug_nn_multi_kernel(const double* soa, long long cap, int count, int dof, const double* q,
                                      int nq, int group, uint32_t* idx, double* d2) {
    double* qs = reinterpret_cast<double*>(g_dsmem + FX_END);  // [32][kMaxDof], after the fixed region (mnn_*)
    Ctx c;
    c.dof = dof;
    c.nthreads = blockDim.x;
    for (int b = blockIdx.x * group; b < nq; b += gridDim.x * group) {
        const int m = min(group, nq - b);
        for (int k = threadIdx.x; k < m * dof; k += blockDim.x) qs[k] = q[(size_t)b * dof + k];
        __syncthreads();
        nn_scan_multi(c, soa, cap, count, qs, m, nullptr);
        if (threadIdx.x < m) {
            idx[b + threadIdx.x] = sh(c.mnn_i)[threadIdx.x];
            d2[b + threadIdx.x] = sh(c.mnn_d)[threadIdx.x];
        }
        __syncthreads();
    }
}

// planner's Halton path: reciprocal-power table + multiply-high digits
__device__ double halton_planner(unsigned base, unsigned long long index) {
    double ftab[kHaltonTab];
    double f = 1.0;
    for (int k = 0; k < kHaltonTab; ++k) {
        f = __ddiv_rn(f, (double)base);
        ftab[k] = f;
    }
    return halton_tab(base, ~0ull / base + 1, ftab, index);
}

__global__ void debug_halton_kernel(const uint32_t* bases, const uint64_t* idx, int n, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = halton_planner(bases[i], idx[i]);
}

__global__ void debug_sample_kernel(RobotArgs r, uint64_t index0, int n, double* out) {
    const uint32_t* rw = r.words;
    const int dof = rw[RH_DOF];
    const uint32_t* bases = rw + rw[RH_OFF_BASES];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * dof) return;
    const int k = i / dof, d = i % dof;
    // the planner's own path: host-built reciprocal table after the limits
    const double* ftab = r.limits + 2 * dof + d * kHaltonTab;
    out[i] = sample_dim(halton_tab(bases[d], ~0ull / bases[d] + 1, ftab, index0 + k), r.limits[2 * d],
                        r.limits[2 * d + 1]);
}

// FP32 FFMA-chain microbenchmark: the roofline denominator for the FK /
// collision work (MEASURED_PEAKS.json carries no FP32 figure). 8 independent
// dependency chains per thread, 256 threads x 8 CTAs per SM.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], 0.9999999f, 1e-7f);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5f) out[blockIdx.x] = s;  // keeps the chains alive
}

double measure_fp32_peak(int sms, cudaStream_t st) {
    float* out = nullptr;
    cudaMalloc(&out, 4 * 8 * sms);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048, grid = 8 * sms;
    ffma_peak_kernel<<<grid, 256, 0, st>>>(out, iters);  // warm-up
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) ffma_peak_kernel<<<grid, 256, 0, st>>>(out, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 5.0 * grid * 256.0 * iters * 16 * 8 * 2;
    return ms > 0 ? flops / (ms * 1e-3) / 1e12 : 0.0;
}

// FP64 DMUL/DADD-chain microbenchmark: the roofline denominator of the NN
// scan, whose keys are un-fused FP64 multiplies and adds in the reference's
// order (kernels_scalar.cpp:9-16; an FMA would change the bits). 8
// independent chains per thread; 2 flops per step (one DMUL, one DADD).
__global__ void __launch_bounds__(256) dpeak_kernel(double* out, int iters) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(__dmul_rn(a[k], 0.9999999), 1e-9);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5) out[blockIdx.x] = s;
}

double measure_fp64_peak(int sms, cudaStream_t st) {
    double* out = nullptr;
    cudaMalloc(&out, 8 * 8 * sms);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 512, grid = 8 * sms;
    dpeak_kernel<<<grid, 256, 0, st>>>(out, iters);  // warm-up
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) dpeak_kernel<<<grid, 256, 0, st>>>(out, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 5.0 * grid * 256.0 * iters * 8 * 8 * 2;
    return ms > 0 ? flops / (ms * 1e-3) / 1e12 : 0.0;
}

// L2 read bandwidth: every CTA streams float4s over a buffer that fits in
// L2 (after one warm pass), several passes per launch
__global__ void __launch_bounds__(512) l2_read_kernel(const float4* buf, long long n4, int passes, float* out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        // each pass starts at a CTA-dependent offset so CTAs spread over the slices
        const long long off = ((long long)blockIdx.x * 7919 + p * 104729) % n4;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            long long k = i + off;
            if (k >= n4) k -= n4;
            const float4 v = __ldcg(buf + k);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1.2345f) out[0] = acc;  // keeps the loads live
}

double measure_l2_gbs(int sms, cudaStream_t st) {
    const long long bytes = 32ll << 20;  // 32 MiB: well inside the 126 MB L2
    float4* buf = nullptr;
    float* out = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 0.0;
    cudaMalloc(&out, 4);
    cudaMemsetAsync(buf, 0, bytes, st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const long long n4 = bytes / 16;
    const int grid = 4 * sms, passes = 8;
    l2_read_kernel<<<grid, 512, 0, st>>>(buf, n4, 2, out);  // warm: lines resident in L2
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) l2_read_kernel<<<grid, 512, 0, st>>>(buf, n4, passes, out);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(out);
    return ms > 0 ? 5.0 * passes * (double)bytes / (ms * 1e-3) / 1e9 : 0.0;
}

static int chunk_states() { return 32; }

// SM count of the current device (grids are sized from it, not hard-coded)
static int cur_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 1;
    }
    return cache[dev];
}

cudaError_t launch_check_configs(const RobotArgs& r, const SceneArgs& s, const double* q, int n,
                                 int two_stage, uint8_t* out, cudaStream_t st) {
    const int NS = chunk_states();
    const size_t sm = smem_bytes(r, NS, 128, SCENE_MAX_WORDS, true);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(check_configs_kernel), (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)min((long long)(n + NS - 1) / NS, (long long)cur_sms() * 16);
    if (grid > 0) check_configs_kernel<<<grid, 128, sm, st>>>(r, s, q, n, two_stage, out, NS);
    return cudaGetLastError();
}

cudaError_t launch_validate_edges(const RobotArgs& r, const SceneArgs& s, const double* from,
                                  const double* to, int n_edges, int n_cc, int two_stage,
                                  int early_exit, uint8_t* out, cudaStream_t st, long long* prof,
                                  unsigned long long* counters) {
    // the warp-per-edge checker unless the chunk-profile debug hook asks for
    // the CTA one (prof) or the robot does not fit a warp region
    if (!prof && r.host_words && s.n_words > 0) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (warp_workers_per_sm(r.host_words, s.n_words, optin) > 0)
            return launch_validate_edges_warp(r, s, from, to, n_edges, n_cc, two_stage, early_exit, out, st,
                                              counters, cur_sms(), optin);
    }
    const int NS = chunk_states();
    const size_t sm = smem_bytes(r, NS, 128, SCENE_MAX_WORDS, true);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(validate_edges_kernel), (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)min((long long)n_edges, (long long)cur_sms() * 16);
    if (grid > 0)
        validate_edges_kernel<<<grid, 128, sm, st>>>(r, s, from, to, n_edges, n_cc, two_stage,
                                                     early_exit, out, NS, prof, counters);
    return cudaGetLastError();
}

cudaError_t launch_debug_check_edges(const RobotArgs& r, const SceneArgs& s, const double* from,
                                     const double* to, int n_edges, int n_cc, int two_stage,
                                     uint8_t* state_valid, float* fine_out, cudaStream_t st) {
    const int NS = chunk_states();
    const size_t sm = smem_bytes(r, NS, 128, SCENE_MAX_WORDS, true);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(debug_check_edges_kernel), (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)min((long long)n_edges, (long long)cur_sms() * 8);
    if (grid > 0)
        debug_check_edges_kernel<<<grid, 128, sm, st>>>(r, s, from, to, n_edges, n_cc, two_stage, state_valid,
                                                        fine_out, NS);
    return cudaGetLastError();
}

cudaError_t launch_debug_fk(const RobotArgs& r, const double* q, int n, float* fine_out,
                            float* coarse_out, cudaStream_t st) {
    const int NS = chunk_states();
    const size_t sm = smem_bytes(r, NS, 128, SCENE_MAX_WORDS, true);
    cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(debug_fk_kernel), (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = (int)min((long long)(n + NS - 1) / NS, (long long)cur_sms() * 16);
    if (grid > 0) debug_fk_kernel<<<grid, 128, sm, st>>>(r, q, n, fine_out, coarse_out, NS);
    return cudaGetLastError();
}

cudaError_t launch_debug_hits(const SceneArgs& s, const float* centers, const double* radii,
                              int n, int n_prims, uint8_t* hits, cudaStream_t st) {
    const long long items = (long long)n * n_prims;
    const int grid = (int)min((items + 127) / 128, (long long)cur_sms() * 8);
    if (grid > 0) debug_hits_kernel<<<grid, 128, 0, st>>>(s, centers, radii, n, n_prims, hits);
    return cudaGetLastError();
}

cudaError_t launch_debug_nn_multi(const double* soa, long long cap, int count, int dof, const double* q,
                                  int nq, int group, uint32_t* idx, double* d2, cudaStream_t st) {
    const int grid = min((nq + group - 1) / group, cur_sms() * 8);
    if (grid > 0)
        debug_nn_multi_kernel<<<grid, 128, FX_END + 8 * 32 * kMaxDof, st>>>(soa, cap, count, dof, q, nq,
                                                                                       group, idx, d2);
    return cudaGetLastError();
}

cudaError_t launch_debug_halton(const uint32_t* bases, const uint64_t* idx, int n, double* out,
                                cudaStream_t st) {
    if (n > 0) debug_halton_kernel<<<(n + 127) / 128, 128, 0, st>>>(bases, idx, n, out);
    return cudaGetLastError();
}

cudaError_t launch_debug_sample(const RobotArgs& r, uint64_t index0, int n, double* out,
                                cudaStream_t st) {
    const int items = n * r.dof;
    if (items > 0) debug_sample_kernel<<<(items + 127) / 128, 128, 0, st>>>(r, index0, n, out);
    return cudaGetLastError();
}

}  // namespace prrtc_b200
