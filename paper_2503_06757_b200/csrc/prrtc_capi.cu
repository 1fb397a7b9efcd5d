// prrtc_capi.cu — host side of the C-ABI declared in include/prrtc_b200.h.
//
// Validation mirrors the reference (RobotModel::finalize kinematics.cpp:15-74,
// Scene::validate geometry.cpp:10-39, plan() preconditions planner.cpp:248-252)
// and reports through return codes + prrtc_last_error instead of exceptions.
// All planning runs on the device; there is no CPU fallback: without an
// sm_100 device every compute entry point fails with PRRTC_ENODEV.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "prrtc_b200.h"
#include "prrtc_internal.h"
#include "prrtc_launch.h"

using namespace prrtc_b200;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return set_err(PRRTC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Device capability check, cached per ordinal (cudaGetDeviceProperties costs
// milliseconds; a plan call must not pay it).
std::atomic<int> g_dev_state[64];  // 0 unknown, 1 ok, 2 not sm_100

int check_device(int device) {
    if (device >= 0 && device < 64) {
        const int st = g_dev_state[device].load(std::memory_order_relaxed);
        if (st == 1) return PRRTC_OK;
        if (st == 2)
            return set_err(PRRTC_ENODEV, "device is not sm_100 (Blackwell); kernels are built for sm_100a only");
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return set_err(PRRTC_ENODEV, "no CUDA device: the B200 planner has no CPU fallback");
    if (device < 0 || device >= n || device >= 64) return set_err(PRRTC_ENODEV, "device ordinal out of range");
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess)
        return set_err(PRRTC_ENODEV, "cudaDeviceGetAttribute failed");
    g_dev_state[device].store(major == 10 ? 1 : 2, std::memory_order_relaxed);
    if (major != 10)
        return set_err(PRRTC_ENODEV, "device is not sm_100 (Blackwell); kernels are built for sm_100a only");
    return PRRTC_OK;
}

// Diagnostic / A-B environment switches, read once and
// cached: a getenv per switch per plan call cost microseconds of a ~0.1 ms
// single-problem call. prrtc_debug_reload_env() re-reads them (tests that
// change a switch in-process).
struct EnvKnobs {
    bool ns32 = false, ns64 = false, ns128 = false, trace = false, host_trace = false, no_map = false;
    unsigned debug_flags = 0;
    int tail_claim = 1, mnn_nodes = 0;
    int tail_min = 4, tail_div = 4;  // PRRTC_TAIL_MIN / PRRTC_TAIL_DIV (sweeps)
    int warp = -1;  // PRRTC_WARP=1: eligible batches on the warp-worker planner (A/B runs)
    int warps_cap = 0;  // PRRTC_WARPS=k: at most k warp workers per SM (sweeps)
    int help_cap = 0;  // PRRTC_HELP_CAP: most workers a help join may bring a problem to (sweeps)
    int help_policy = 1;  // PRRTC_HELP_POLICY: 1 most unclaimed budget per worker, 0 fewest workers (A/B)
    bool no_stab = false;  // PRRTC_NO_SAMPLE_TABLE: compute every Halton sample in the loop (A/B)
    long long map_bytes = -1;
    std::string dump_ctl;
};
std::atomic<const EnvKnobs*> g_env{nullptr};
std::mutex g_env_mu;

const EnvKnobs* read_env() {
    auto* k = new EnvKnobs();
    auto on = [](const char* n) { return std::getenv(n) != nullptr; };
    k->ns32 = on("PRRTC_NS32");
    k->ns64 = on("PRRTC_NS64");
    k->ns128 = on("PRRTC_NS128");
    k->trace = on("PRRTC_TRACE");
    k->host_trace = on("PRRTC_HOST_TRACE");
    k->no_map = on("PRRTC_NO_MAP");
    if (const char* e = std::getenv("PRRTC_DEBUG_FLAGS")) k->debug_flags = (unsigned)std::atoi(e);
    if (const char* e = std::getenv("PRRTC_TAIL_CLAIM")) k->tail_claim = std::atoi(e);
    if (const char* e = std::getenv("PRRTC_TAIL_MIN")) k->tail_min = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PRRTC_TAIL_DIV")) k->tail_div = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PRRTC_WARP")) k->warp = std::atoi(e);
    if (const char* e = std::getenv("PRRTC_WARPS")) k->warps_cap = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("PRRTC_HELP_CAP")) k->help_cap = std::atoi(e);
    if (const char* e = std::getenv("PRRTC_HELP_POLICY")) k->help_policy = std::atoi(e);
    k->no_stab = on("PRRTC_NO_SAMPLE_TABLE");
    if (const char* e = std::getenv("PRRTC_MNN_NODES")) k->mnn_nodes = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("PRRTC_MAP_BYTES")) k->map_bytes = std::strtoll(e, nullptr, 10);
    if (const char* e = std::getenv("PRRTC_DUMP_CTL")) k->dump_ctl = e;
    return k;
}

const EnvKnobs& env() {
    const EnvKnobs* k = g_env.load(std::memory_order_acquire);
    if (k) return *k;
    std::lock_guard<std::mutex> lk(g_env_mu);
    k = g_env.load(std::memory_order_relaxed);
    if (!k) {
        k = read_env();
        g_env.store(k, std::memory_order_release);
    }
    return *k;
}

// ---- small FP64 math in the reference's operation order (transform.hpp) ----
struct M3 {
    double m[9];
};
// Quat::to_mat3 (transform.hpp:97-103) on the raw (unnormalised) quaternion.
M3 quat_to_mat3(double w, double x, double y, double z) {
    return {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
             2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
             2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
}
M3 transposed(const M3& a) {
    return {{a.m[0], a.m[3], a.m[6], a.m[1], a.m[4], a.m[7], a.m[2], a.m[5], a.m[8]}};
}
M3 mul(const M3& a, const M3& b) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[3 * i + j] = a.m[3 * i] * b.m[j] + a.m[3 * i + 1] * b.m[3 + j] + a.m[3 * i + 2] * b.m[6 + j];
    return r;
}
double norm3(double x, double y, double z) { return std::sqrt(x * x + y * y + z * z); }

std::vector<unsigned> first_primes(size_t n) {  // sampling.cpp:20-37
    std::vector<unsigned> p;
    for (unsigned c = 2; p.size() < n; ++c) {
        bool ok = true;
        for (unsigned q : p) {
            if (q * q > c) break;
            if (c % q == 0) {
                ok = false;
                break;
            }
        }
        if (ok) p.push_back(c);
    }
    return p;
}

uint32_t fbits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

// Synchronous upload of setup data (robots, scenes) on a per-device
// non-blocking stream, waited on before returning: a cudaMemcpy from pageable
// memory may return before its DMA lands, and the planner's streams are not
// ordered after the legacy default stream.
std::mutex g_up_mu[64];
cudaStream_t g_up_stream[64];

cudaError_t upload_sync(int device, const std::pair<void*, std::pair<const void*, size_t>>* copies, int n) {
    if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_up_mu[device]);
    cudaSetDevice(device);
    if (!g_up_stream[device]) {
        cudaError_t e = cudaStreamCreateWithFlags(&g_up_stream[device], cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
    }
    for (int i = 0; i < n; ++i) {
        if (copies[i].second.second == 0) continue;
        cudaError_t e = cudaMemcpyAsync(copies[i].first, copies[i].second.first, copies[i].second.second,
                                        cudaMemcpyHostToDevice, g_up_stream[device]);
        if (e != cudaSuccess) return e;
    }
    return cudaStreamSynchronize(g_up_stream[device]);
}

// A completion marker of planner launches: an event recorded on a launch's
// stream after its last kernel. Workspaces own one (re-recorded per launch,
// so waiting on it is conservative: it covers every earlier launch on that
// stream); a scene keeps the markers of the workspaces that have read it, so
// prrtc_scene_update can wait for exactly those launches instead of the
// whole device.
struct UseMark {
    cudaEvent_t ev = nullptr;
    int device = 0;
    ~UseMark() {
        if (ev) {
            cudaSetDevice(device);
            cudaEventDestroy(ev);
        }
    }
};
using UseMarkP = std::shared_ptr<UseMark>;

}  // namespace

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct prrtc_robot {
    int device = 0;
    int dof = 0, n_links = 0, n_fine = 0, n_pairs = 0;
    std::vector<uint32_t> words;
    std::vector<double> limits;   // [dof][2]
    std::vector<double> fine_r64;
    uint32_t* d_words = nullptr;
    double* d_fine_r64 = nullptr;
    double* d_limits = nullptr;
    double reach = 0.0;           // bound on |posed sphere| (m)
    // planner CTAs per SM, by (ns_max / 32, CTA size) x (Uniform sampler) x (scene-size bucket)
    mutable std::atomic<int> occ[15 * 2 * 5] = {};
    // Halton sample tables per seed (sample_table): [kSampleTab][dof] doubles
    mutable std::mutex stab_mu;
    mutable std::vector<std::pair<uint64_t, double*>> stab;
    RobotArgs args() const {
        RobotArgs r;
        r.words = d_words;
        r.n_words = (int)words.size();
        r.fine_r64 = d_fine_r64;
        r.limits = d_limits;
        r.n_links = n_links;
        r.dof = dof;
        r.n_fine = n_fine;
        r.host_words = words.data();
        return r;
    }
};

struct prrtc_scene {
    int device = 0;
    std::vector<uint32_t> words;
    std::vector<double> f64;  // spheres, boxes, capsules, cylinders
    int ns = 0, nb = 0, nc = 0, ny = 0;
    double extent = 0.0;
    uint32_t* d_words = nullptr;
    double* d_f64 = nullptr;
    size_t cap_words = 0, cap_f64 = 0;  // device allocation sizes (elements)
    // bumped by every prrtc_scene_update: a persistent batch re-stages the
    // scene's device pointers and FP64 section offsets when it changed
    std::atomic<uint64_t> generation{0};
    // completion markers of the launches that read this scene (see UseMark)
    mutable std::mutex mark_mu;
    mutable std::vector<UseMarkP> marks;
    mutable std::atomic<const UseMark*> last_mark{nullptr};  // fast path: the marker most recently added
    void mark_use(const UseMarkP& m) const {
        if (last_mark.load(std::memory_order_acquire) == m.get()) return;  // (markers are never removed)
        std::lock_guard<std::mutex> lk(mark_mu);
        last_mark.store(m.get(), std::memory_order_release);
        for (const auto& x : marks)
            if (x == m) return;
        marks.push_back(m);
    }
    // wait until no launch that read the scene is still running
    cudaError_t wait_unused() const {
        std::vector<UseMarkP> ms;
        {
            std::lock_guard<std::mutex> lk(mark_mu);
            ms = marks;
        }
        for (const auto& m : ms) {
            const cudaError_t e = cudaEventSynchronize(m->ev);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    SceneArgs args() const {
        SceneArgs s;
        s.words = d_words;
        s.f64.s = d_f64;
        s.f64.b = d_f64 + 4 * ns;
        s.f64.c = d_f64 + 4 * ns + BOX_STRIDE * nb;
        s.f64.y = d_f64 + 4 * ns + BOX_STRIDE * nb + CAP_STRIDE * nc;
        s.n_words = (int)((words.size() + 3) & ~size_t(3));
        return s;
    }
};

extern "C" {

int prrtc_api_version(void) { return PRRTC_API_VERSION; }

int prrtc_last_error(char* buf, size_t len) {
    if (!buf || len == 0) return PRRTC_EINVAL;
    std::snprintf(buf, len, "%s", g_err.c_str());
    return PRRTC_OK;
}

int prrtc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    int ok = 0;
    for (int d = 0; d < n; ++d) {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10)
            ++ok;
    }
    return ok;
}

int prrtc_default_workers(int device) {
    int rc = check_device(device);
    if (rc) return rc;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n > 0 ? n : 1;  // one 512-thread CTA per SM (batch_setup)
}

void prrtc_params_default(prrtc_params* p) {  // planner.hpp:21-40
    std::memset(p, 0, sizeof(*p));
    p->delta = 0.5;
    p->n_cc = 32;
    p->workers = 0;
    p->max_iters_per_worker = 2000;
    p->tree_capacity = 200000;
    p->dd_radius = 0.0;
    p->dynamic_domain = 1;
    p->balance = 1;
    p->early_exit = 1;
    p->two_stage = 1;
    p->batched_cc = 0;
    p->nn_partitions = 1;
    p->sampler = PRRTC_SAMPLER_HALTON;
    p->seed = 0;
}

// ---- robot: RobotModel::finalize (kinematics.cpp:15-74) + upload ----
int prrtc_robot_create(const prrtc_robot_desc* d, int device, prrtc_robot** out) {
    if (!d || !out) return set_err(PRRTC_EINVAL, "prrtc_robot_create: null argument");
    const int n = (int)d->n_links;
    if (n == 0) return set_err(PRRTC_EINVAL, "robot: joints must be non-empty");
    if (n > PRRTC_MAX_LINKS) return set_err(PRRTC_EINVAL, "robot: too many links for the device layout");
    auto where = [](const char* what, int i) { return std::string("robot joints[") + std::to_string(i) + "]" + what; };
    int dof = 0;
    std::vector<int> qidx(n, -1);
    for (int i = 0; i < n; ++i) {
        if (d->parent[i] >= i) return set_err(PRRTC_EINVAL, where(".parent: must be smaller than the joint index", i));
        if (d->parent[i] < -1) return set_err(PRRTC_EINVAL, where(".parent: out of range", i));
        const double* q = d->origin_quat + 4 * i;
        const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (std::abs(qn - 1.0) > 1e-6)
            return set_err(PRRTC_EINVAL, where(".origin.quaternion: norm deviates from 1 by more than 1e-6", i));
        if (d->kind[i] < 0 || d->kind[i] > 2) return set_err(PRRTC_EINVAL, where(".kind: unknown joint kind", i));
        if (d->kind[i] != PRRTC_JOINT_FIXED) {
            const double* a = d->axis + 3 * i;
            if (std::abs(norm3(a[0], a[1], a[2]) - 1.0) > 1e-9)
                return set_err(PRRTC_EINVAL, where(".axis: must be unit length", i));
            if (!(d->lo[i] <= d->hi[i])) return set_err(PRRTC_EINVAL, where(".limits: lo must be <= hi", i));
            qidx[i] = dof++;
        }
    }
    if (dof > PRRTC_MAX_DOF) return set_err(PRRTC_EINVAL, "robot: too many degrees of freedom for the device layout");
    const uint32_t S = d->fine_offset[n];
    if (S > PRRTC_MAX_FINE) return set_err(PRRTC_EINVAL, "robot: too many fine spheres for the device layout");
    int maxf = 1;
    for (int l = 0; l < n; ++l) {
        const std::string w = "robot spheres[" + std::to_string(l) + "]";
        const double* c = d->coarse + 4 * l;
        if (!(c[3] > 0.0)) return set_err(PRRTC_EINVAL, w + ".coarse.radius: must be positive");
        if (d->fine_offset[l + 1] < d->fine_offset[l]) return set_err(PRRTC_EINVAL, w + ": bad fine offsets");
        const int nf = (int)(d->fine_offset[l + 1] - d->fine_offset[l]);
        if (nf > PRRTC_MAX_FINE_PER_LINK) return set_err(PRRTC_EINVAL, w + ": too many fine spheres");
        maxf = std::max(maxf, nf);
        for (uint32_t k = d->fine_offset[l]; k < d->fine_offset[l + 1]; ++k) {
            const double* f = d->fine + 4 * k;
            if (!(f[3] > 0.0)) return set_err(PRRTC_EINVAL, w + ".fine[" + std::to_string(k - d->fine_offset[l]) + "].radius: must be positive");
            const double reach = norm3(f[0] - c[0], f[1] - c[1], f[2] - c[2]) + f[3];
            if (reach > c[3] + 1e-9)
                return set_err(PRRTC_EINVAL, w + ".fine[" + std::to_string(k - d->fine_offset[l]) + "]: escapes the coarse bounding sphere");
        }
    }
    if (d->n_self_pairs > PRRTC_MAX_SELF_PAIRS) return set_err(PRRTC_EINVAL, "robot: too many self pairs");
    for (uint32_t p = 0; p < d->n_self_pairs; ++p) {
        const int a = d->self_pairs[2 * p], b = d->self_pairs[2 * p + 1];
        const std::string w = "robot self_pairs[" + std::to_string(p) + "]";
        if (a < 0 || b < 0 || a >= n || b >= n) return set_err(PRRTC_EINVAL, w + ": link index out of range");
        if (a == b) return set_err(PRRTC_EINVAL, w + ": a link cannot pair with itself");
        if (d->parent[a] == b || d->parent[b] == a)
            return set_err(PRRTC_EINVAL, w + ": adjacent parent-child links must not be tested");
    }
    int rc = check_device(device);
    if (rc) return rc;

    auto* r = new prrtc_robot();
    r->device = device;
    r->dof = dof;
    r->n_links = n;
    r->n_fine = (int)S;
    r->n_pairs = (int)d->n_self_pairs;
    // packed words
    std::vector<uint32_t>& w = r->words;
    w.assign(RH_COUNT, 0);
    auto align4 = [&]() { while (w.size() % 4) w.push_back(0); };
    w[RH_NLINKS] = n;
    w[RH_DOF] = dof;
    w[RH_NFINE] = S;
    w[RH_NPAIRS] = d->n_self_pairs;
    w[RH_MAXFINE] = maxf;
    align4();
    w[RH_OFF_INFO] = (uint32_t)w.size();
    for (int l = 0; l < n; ++l) {
        w.push_back((uint32_t)d->kind[l]);
        w.push_back((uint32_t)d->parent[l]);
        w.push_back((uint32_t)qidx[l]);
        w.push_back(d->fine_offset[l]);
    }
    w[RH_OFF_NFINE] = (uint32_t)w.size();
    for (int l = 0; l < n; ++l) w.push_back(d->fine_offset[l + 1] - d->fine_offset[l]);
    align4();
    w[RH_OFF_GEO] = (uint32_t)w.size();
    double reach_sum = 0.0;
    for (int l = 0; l < n; ++l) {
        const double* q = d->origin_quat + 4 * l;
        const M3 Ro = quat_to_mat3(q[0], q[1], q[2], q[3]);
        const double* a = d->axis + 3 * l;
        const M3 ax = {{0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0}};
        const M3 M2 = mul(Ro, ax);
        double v[3];
        for (int i = 0; i < 3; ++i) v[i] = Ro.m[3 * i] * a[0] + Ro.m[3 * i + 1] * a[1] + Ro.m[3 * i + 2] * a[2];
        float g[GEO_STRIDE] = {0};
        for (int k = 0; k < 9; ++k) {
            g[k] = (float)Ro.m[k];
            g[9 + k] = (float)M2.m[k];
            g[18 + k] = (float)(v[k / 3] * a[k % 3]);
        }
        for (int k = 0; k < 3; ++k) {
            g[27 + k] = (float)d->origin_xyz[3 * l + k];
            g[30 + k] = (float)v[k];
            g[33 + k] = (float)d->coarse[4 * l + k];
        }
        g[36] = (float)d->coarse[4 * l + 3];
        for (int k = 0; k < GEO_STRIDE; ++k) w.push_back(fbits(g[k]));
        reach_sum += norm3(d->origin_xyz[3 * l], d->origin_xyz[3 * l + 1], d->origin_xyz[3 * l + 2]) +
                     norm3(d->coarse[4 * l], d->coarse[4 * l + 1], d->coarse[4 * l + 2]) + d->coarse[4 * l + 3];
    }
    align4();
    w[RH_OFF_FINE] = (uint32_t)w.size();
    for (uint32_t k = 0; k < S; ++k)
        for (int i = 0; i < 4; ++i) w.push_back(fbits((float)d->fine[4 * k + i]));
    w[RH_OFF_PAIRS] = (uint32_t)w.size();
    for (uint32_t p = 0; p < d->n_self_pairs; ++p) {
        w.push_back((uint32_t)d->self_pairs[2 * p]);
        w.push_back((uint32_t)d->self_pairs[2 * p + 1]);
    }
    w[RH_OFF_BASES] = (uint32_t)w.size();
    const std::vector<unsigned> bases = first_primes(dof);
    for (unsigned b : bases) w.push_back(b);
    if (w.size() % 2) w.push_back(0);
    w[RH_OFF_MAGIC] = (uint32_t)w.size();
    for (unsigned b : bases) {  // ceil(2^64 / b): q = umul64hi(n, M) is exact for n < 2^32
        const uint64_t m = UINT64_MAX / b + 1;
        w.push_back((uint32_t)(m & 0xffffffffu));
        w.push_back((uint32_t)(m >> 32));
    }
    w[RH_OFF_FLINK] = (uint32_t)w.size();
    for (int l = 0; l < n; ++l)
        for (uint32_t k = d->fine_offset[l]; k < d->fine_offset[l + 1]; ++k) w.push_back((uint32_t)l);
    if (w.size() % 2) w.push_back(0);
    w[RH_OFF_FUNITS] = (uint32_t)w.size();
    uint32_t nunits = 0;
    for (int l = 0; l < n; ++l)
        for (uint32_t k = d->fine_offset[l]; k < d->fine_offset[l + 1]; k += 3, ++nunits) {
            w.push_back((uint32_t)l);
            w.push_back(k | (std::min<uint32_t>(3, d->fine_offset[l + 1] - k) << 16));
        }
    w[RH_NFUNITS] = nunits;
    align4();
    w[RH_WORDS] = (uint32_t)w.size();
    {   // 3 dof (lerp) + 63 per non-root link + 70 per revolute
        // + 21 per prismatic + 18 per posed (coarse) sphere
        unsigned nonroot = 0, rev = 0, pri = 0;
        for (int l = 0; l < n; ++l) {
            nonroot += d->parent[l] >= 0;
            rev += d->kind[l] == PRRTC_JOINT_REVOLUTE;
            pri += d->kind[l] == PRRTC_JOINT_PRISMATIC;
        }
        w[RH_FKFLOPS] = 3 * dof + 63 * nonroot + 70 * rev + 21 * pri + 18 * n;
    }
    r->reach = reach_sum;
    for (int l = 0; l < n; ++l) {
        if (d->kind[l] != PRRTC_JOINT_FIXED) {
            r->limits.push_back(d->lo[l]);
            r->limits.push_back(d->hi[l]);
            if (d->kind[l] == PRRTC_JOINT_PRISMATIC) r->reach += std::max(std::abs(d->lo[l]), std::abs(d->hi[l]));
        }
    }
    // Halton reciprocal powers f_k = (((1/b)/b).../b) (halton_value's f /= b,
    // sampling.cpp:12) after the [dof][2] limits: the same IEEE divisions as
    // on the device, read through the read-only path by the sampler
    for (unsigned b : first_primes(dof)) {
        double f = 1.0;
        for (int k = 0; k < HALTON_TAB; ++k) {
            f = f / (double)b;
            r->limits.push_back(f);
        }
    }
    // FP64 radii: the fine spheres', then the coarse spheres' (exact CheckStats mode)
    r->fine_r64.resize(S + n);
    for (uint32_t k = 0; k < S; ++k) r->fine_r64[k] = d->fine[4 * k + 3];
    for (int l = 0; l < n; ++l) r->fine_r64[S + l] = d->coarse[4 * l + 3];

    cudaSetDevice(device);
    if (cudaMalloc(&r->d_words, 4 * w.size()) != cudaSuccess ||
        cudaMalloc(&r->d_fine_r64, 8 * r->fine_r64.size()) != cudaSuccess ||
        cudaMalloc(&r->d_limits, 8 * std::max<size_t>(2, r->limits.size())) != cudaSuccess) {
        prrtc_robot_destroy(r);
        return set_err(PRRTC_ENOMEM, "prrtc_robot_create: device allocation failed");
    }
    const std::pair<void*, std::pair<const void*, size_t>> copies[3] = {
        {r->d_words, {w.data(), 4 * w.size()}},
        {r->d_fine_r64, {r->fine_r64.data(), 8 * r->fine_r64.size()}},
        {r->d_limits, {r->limits.data(), 8 * r->limits.size()}}};
    if (upload_sync(device, copies, 3) != cudaSuccess) {
        prrtc_robot_destroy(r);
        return set_err(PRRTC_ECUDA, "prrtc_robot_create: upload failed");
    }
    *out = r;
    return PRRTC_OK;
}

int prrtc_robot_destroy(prrtc_robot* r) {
    if (!r) return PRRTC_OK;
    cudaSetDevice(r->device);
    cudaFree(r->d_words);
    cudaFree(r->d_fine_r64);
    cudaFree(r->d_limits);
    for (auto& t : r->stab) cudaFree(t.second);
    delete r;
    return PRRTC_OK;
}

int prrtc_robot_dof(const prrtc_robot* r) { return r ? r->dof : PRRTC_EINVAL; }
int prrtc_robot_fine_count(const prrtc_robot* r) { return r ? r->n_fine : PRRTC_EINVAL; }
int prrtc_robot_limits(const prrtc_robot* r, double* lim) {
    if (!r || !lim) return PRRTC_EINVAL;
    std::copy(r->limits.begin(), r->limits.begin() + 2 * r->dof, lim);  // [dof][2]; the Halton table follows
    return PRRTC_OK;
}

// ---- scene: Scene::validate (geometry.cpp:10-39) + SceneIndex layout ----
static int build_scene(const prrtc_scene_desc* d, prrtc_scene* s) {
    const uint32_t ny = d->cylinders ? d->n_cylinders : 0;
    const uint32_t P = d->n_spheres + d->n_boxes + d->n_capsules + ny;
    if (P > PRRTC_MAX_PRIMS) return set_err(PRRTC_EINVAL, "scene: more than PRRTC_MAX_PRIMS primitives");
    int idx = 0;
    auto where = [&](int i) { return std::string("scene primitives[") + std::to_string(i) + "]"; };
    for (uint32_t i = 0; i < d->n_spheres; ++i, ++idx)
        if (!(d->spheres[4 * i + 3] > 0.0)) return set_err(PRRTC_EINVAL, where(idx) + ".radius: must be positive");
    for (uint32_t i = 0; i < d->n_boxes; ++i, ++idx) {
        const double* b = d->boxes + 10 * i;
        if (!(b[7] > 0.0 && b[8] > 0.0 && b[9] > 0.0))
            return set_err(PRRTC_EINVAL, where(idx) + ".half_extents: must be componentwise positive");
        const double qn = std::sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2] + b[3] * b[3]);
        if (std::abs(qn - 1.0) > 1e-6)
            return set_err(PRRTC_EINVAL, where(idx) + ".pose.quaternion: norm deviates from 1 by more than 1e-6");
    }
    for (uint32_t i = 0; i < d->n_capsules; ++i, ++idx)
        if (!(d->capsules[7 * i + 6] > 0.0)) return set_err(PRRTC_EINVAL, where(idx) + ".radius: must be positive");
    for (uint32_t i = 0; i < ny; ++i, ++idx) {  // cylinder extension, validated like boxes / capsules
        const double* y = d->cylinders + 9 * i;
        if (!(y[7] > 0.0)) return set_err(PRRTC_EINVAL, where(idx) + ".radius: must be positive");
        if (!(y[8] > 0.0)) return set_err(PRRTC_EINVAL, where(idx) + ".half_length: must be positive");
        const double qn = std::sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2] + y[3] * y[3]);
        if (std::abs(qn - 1.0) > 1e-6)
            return set_err(PRRTC_EINVAL, where(idx) + ".pose.quaternion: norm deviates from 1 by more than 1e-6");
    }

    s->ns = d->n_spheres;
    s->nb = d->n_boxes;
    s->nc = d->n_capsules;
    s->ny = ny;
    std::vector<uint32_t>& w = s->words;
    std::vector<double>& f = s->f64;
    w.assign(SH_COUNT, 0);
    f.clear();
    double ext = 0.0;
    auto upd = [&](double x) { ext = std::max(ext, std::abs(x)); };
    w[SH_NS] = s->ns;
    w[SH_NB] = s->nb;
    w[SH_NC] = s->nc;
    w[SH_OFF_S] = (uint32_t)w.size();
    for (int i = 0; i < s->ns; ++i) {
        const double* p = d->spheres + 4 * i;
        for (int k = 0; k < 4; ++k) {
            w.push_back(fbits((float)p[k]));
            f.push_back(p[k]);
            upd(p[k]);
        }
        upd(std::abs(p[0]) + p[3]);
    }
    w[SH_OFF_B] = (uint32_t)w.size();
    for (int i = 0; i < s->nb; ++i) {
        const double* b = d->boxes + 10 * i;
        // BoxPrim -> SceneIndex: world-to-box rotation R^T, t, h (geometry.cpp:87-97)
        const M3 rt = transposed(quat_to_mat3(b[0], b[1], b[2], b[3]));
        double v[BOX_STRIDE] = {0};
        for (int k = 0; k < 9; ++k) v[k] = rt.m[k];
        for (int k = 0; k < 3; ++k) {
            v[9 + k] = b[4 + k];
            v[12 + k] = b[7 + k];
            upd(std::abs(b[4 + k]) + norm3(b[7], b[8], b[9]));
        }
        for (int k = 0; k < BOX_STRIDE; ++k) {
            w.push_back(fbits((float)v[k]));
            f.push_back(v[k]);
        }
    }
    w[SH_OFF_C] = (uint32_t)w.size();
    for (int i = 0; i < s->nc; ++i) {
        const double* c = d->capsules + 7 * i;
        // CapsulePrim -> SceneIndex: a, ab = b - a, inv_ab2 (geometry.cpp:75-86)
        const double abx = c[3] - c[0], aby = c[4] - c[1], abz = c[5] - c[2];
        const double ab2 = abx * abx + aby * aby + abz * abz;
        double v[CAP_STRIDE] = {c[0], c[1], c[2], abx, aby, abz, ab2 > 0.0 ? 1.0 / ab2 : 0.0, c[6]};
        for (int k = 0; k < CAP_STRIDE; ++k) {
            w.push_back(fbits((float)v[k]));
            f.push_back(v[k]);
        }
        for (int k = 0; k < 6; ++k) upd(std::abs(c[k]) + c[6]);
    }
    w[SH_NY] = s->ny;
    w[SH_OFF_Y] = (uint32_t)w.size();
    for (int i = 0; i < s->ny; ++i) {
        const double* y = d->cylinders + 9 * i;
        // like a box: world-to-cylinder rotation R^T, t, then radius, half length
        const M3 rt = transposed(quat_to_mat3(y[0], y[1], y[2], y[3]));
        double v[CYL_STRIDE] = {0};
        for (int k = 0; k < 9; ++k) v[k] = rt.m[k];
        for (int k = 0; k < 3; ++k) {
            v[9 + k] = y[4 + k];
            upd(std::abs(y[4 + k]) + y[7] + y[8]);
        }
        v[12] = y[7];
        v[13] = y[8];
        for (int k = 0; k < CYL_STRIDE; ++k) {
            w.push_back(fbits((float)v[k]));
            f.push_back(v[k]);
        }
    }
    while (w.size() % 4) w.push_back(0);
    w[SH_WORDS] = (uint32_t)w.size();
    s->extent = ext;
    return PRRTC_OK;
}

// Guard band for the FP32 predicates: 16 ulps of the largest coordinate
// magnitude the test can see (robot reach + scene extent), floor 8 m.
static void finish_scene_words(prrtc_scene* s, double robot_reach) {
    const double M = std::max(8.0, 2.0 * (s->extent + robot_reach));
    const float eps = (float)(M * std::ldexp(1.0, -20));
    s->words[SH_EPS] = fbits(eps);
    s->words[SH_CPAD] = fbits(4.0f * eps + 1e-8f);
}

// Uploads a built scene (words, f64 and counts already in `s`). With
// `prev_words`/`prev_f64` (prrtc_scene_update) the existing device buffers are
// rewritten in place when they are large enough, once every launch that read
// the scene has finished (its completion markers, not the whole device);
// otherwise new buffers are allocated, filled, and the old ones freed after
// those launches. Returns with the data on the device (the copies are waited
// for). On failure the previous device buffers stay as they were.
static int upload_scene(prrtc_scene* s, const prrtc_scene* prev) {
    cudaSetDevice(s->device);
    const size_t nf = std::max<size_t>(1, s->f64.size());
    const bool in_place = prev && prev->d_words && s->words.size() <= prev->cap_words && nf <= prev->cap_f64;
    if (prev && prev->wait_unused() != cudaSuccess) return set_err(PRRTC_ECUDA, "scene: waiting for running plans failed");
    uint32_t* dw = in_place ? prev->d_words : nullptr;
    double* df = in_place ? prev->d_f64 : nullptr;
    if (!in_place) {
        if (cudaMalloc(&dw, 4 * s->words.size()) != cudaSuccess) return set_err(PRRTC_ENOMEM, "scene: device allocation failed");
        if (cudaMalloc(&df, 8 * nf) != cudaSuccess) {
            cudaFree(dw);
            return set_err(PRRTC_ENOMEM, "scene: device allocation failed");
        }
    }
    const std::pair<void*, std::pair<const void*, size_t>> copies[2] = {
        {dw, {s->words.data(), 4 * s->words.size()}}, {df, {s->f64.data(), 8 * s->f64.size()}}};
    if (upload_sync(s->device, copies, 2) != cudaSuccess) {
        if (!in_place) {
            cudaFree(dw);
            cudaFree(df);
        }
        return set_err(PRRTC_ECUDA, "scene: upload failed");
    }
    s->d_words = dw;
    s->d_f64 = df;
    s->cap_words = in_place ? prev->cap_words : s->words.size();
    s->cap_f64 = in_place ? prev->cap_f64 : nf;
    return PRRTC_OK;
}

// default reach used for the guard band before a robot is known (m)
static constexpr double kDefaultReach = 4.0;

int prrtc_scene_create(const prrtc_scene_desc* d, int device, prrtc_scene** out) {
    if (!d || !out) return set_err(PRRTC_EINVAL, "prrtc_scene_create: null argument");
    int rc = check_device(device);
    if (rc) return rc;
    auto* s = new prrtc_scene();
    s->device = device;
    rc = build_scene(d, s);
    if (rc) {
        delete s;
        return rc;
    }
    finish_scene_words(s, kDefaultReach);
    rc = upload_scene(s, nullptr);
    if (rc) {
        prrtc_scene_destroy(s);
        return rc;
    }
    *out = s;
    return PRRTC_OK;
}

int prrtc_scene_update(prrtc_scene* s, const prrtc_scene_desc* d) {
    if (!s || !d) return set_err(PRRTC_EINVAL, "prrtc_scene_update: null argument");
    // build and upload into a temporary; the handle changes only on success
    prrtc_scene tmp;
    tmp.device = s->device;
    int rc = build_scene(d, &tmp);
    if (rc) return rc;
    finish_scene_words(&tmp, kDefaultReach);
    rc = upload_scene(&tmp, s);
    if (rc) return rc;
    if (tmp.d_words != s->d_words) {  // reallocated: the old buffers are no longer read (upload_scene waited)
        cudaFree(s->d_words);
        cudaFree(s->d_f64);
    }
    s->words.swap(tmp.words);
    s->f64.swap(tmp.f64);
    s->ns = tmp.ns;
    s->nb = tmp.nb;
    s->nc = tmp.nc;
    s->ny = tmp.ny;
    s->extent = tmp.extent;
    s->d_words = tmp.d_words;
    s->d_f64 = tmp.d_f64;
    s->cap_words = tmp.cap_words;
    s->cap_f64 = tmp.cap_f64;
    tmp.d_words = nullptr;
    tmp.d_f64 = nullptr;
    s->generation.fetch_add(1, std::memory_order_release);
    return PRRTC_OK;
}

int prrtc_scene_destroy(prrtc_scene* s) {
    if (!s) return PRRTC_OK;
    cudaSetDevice(s->device);
    s->wait_unused();  // a launch that reads the scene may still be running
    cudaFree(s->d_words);
    cudaFree(s->d_f64);
    delete s;
    return PRRTC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// planning workspace and batches
//
// A workspace owns every device buffer a launch needs, laid out so one call
// costs one packed H2D copy, one kernel and one D2H copy:
//   io   (pinned host) : starts | goals | scene-word ptrs | scene-f64 ptrs | prob_scene
//                        | pad to 128 B | zeroed out-header for n problems
//   d_in (device)      : the same layout, then the path arena right after
//                        the out-header: d_out = d_in + out_offset(n) is
//                        [hdr 128 B: arena_used u64, next_problem, n_done]
//                        [ProbCtl x n][path arena]
// so the inputs and the zeroed controls go up in one copy, and the controls
// and paths come back in one. (A persistent prrtc_batch uploads its inputs
// once and zeroes the out-header with a memset per launch.)
//   trees              : cfg [n][2][dof][stride], parent/ready/dd [n][2][stride]
// Workspaces grow monotonically and are cached per device for prrtc_plan /
// prrtc_plan_batch (allocation is setup, not part of a plan call).
// ---------------------------------------------------------------------------
namespace {

struct Workspace {
    int device = -1;
    size_t n_cap = 0, dof_cap = 0, nodes_cap = 0, arena_cap = 0;
    unsigned epoch = 0;
    void* h_io = nullptr;
    size_t io_bytes = 0;
    void* h_out = nullptr;
    size_t out_bytes = 0;
    // mapped pinned block the kernel publishes single-problem results into
    // (publish_result): flag words, then header, controls and arena
    static constexpr size_t kMapBytes = 64 << 10;
    void* h_map = nullptr;
    unsigned char* d_map = nullptr;
    size_t h_out_arena = 0;  // arena doubles h_out holds past the header
    double path_hint = 0.0;  // recent arena doubles used per problem (sizes the D2H prefix)
    uint64_t last_h2d = 0, last_d2h = 0;  // bytes copied by the last plan call
    unsigned char* d_in = nullptr;  // inputs, then the out-header and arena (see above)
    double* d_cfg = nullptr;
    int* d_parent = nullptr;
    int* d_dd = nullptr;
    unsigned* d_ready = nullptr;
    int* d_vprefix = nullptr;  // [n + 1] path-edge prefix (validate_path)
    unsigned* d_init = nullptr;  // inline-input launches: the init word (epoch of the last zeroing)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t stream = nullptr;
    UseMarkP mark;  // recorded after every launch (scenes it read wait on it before an update)

    static size_t in_bytes(size_t n, size_t dof) {
        return 8 * 2 * n * dof + sizeof(void*) * n + sizeof(SceneF64) * n + 4 * n + 64;
    }
    static size_t out_hdr(size_t n) { return 128 + sizeof(ProbCtl) * n; }

    void release() {
        if (device < 0) return;
        cudaSetDevice(device);
        cudaFreeHost(h_io);
        cudaFreeHost(h_out);
        if (h_map) cudaFreeHost(h_map);
        cudaFree(d_in);
        cudaFree(d_cfg);
        cudaFree(d_parent);
        cudaFree(d_dd);
        cudaFree(d_ready);
        cudaFree(d_vprefix);
        cudaFree(d_init);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (stream) cudaStreamDestroy(stream);
        UseMarkP m = std::move(mark);  // scenes may still hold it; the event dies with the last holder
        *this = Workspace();
    }

    // Grow the pinned result buffer to hold `need` arena doubles past the header.
    void grow_h_out(size_t need) {
        if (need <= h_out_arena) return;
        need = std::min(arena_cap, std::max(need, 2 * h_out_arena));
        void* h = nullptr;
        if (cudaMallocHost(&h, out_hdr(n_cap) + 8 * need) != cudaSuccess) return;  // keep the old one
        cudaFreeHost(h_out);
        h_out = h;
        h_out_arena = need;
    }
    ~Workspace() { release(); }

    // Grow to hold n problems of dof with the given tree stride and arena.
    int reserve(int dev, size_t n, size_t dof, size_t stride, size_t arena) {
        const size_t nodes = n * 2 * stride;
        if (device == dev && n <= n_cap && dof <= dof_cap && nodes * dof <= nodes_cap * dof_cap &&
            nodes <= nodes_cap && arena <= arena_cap)
            return PRRTC_OK;
        const size_t nn = std::max(n, n_cap), nd = std::max(dof, dof_cap);
        const size_t nnodes = std::max(nodes, nodes_cap), narena = std::max(arena, arena_cap);
        release();
        device = dev;
        cudaSetDevice(dev);
        io_bytes = in_bytes(nn, nd);
        out_bytes = out_hdr(nn) + 8 * narena;
        if (cudaMallocHost(&h_io, io_bytes + 128 + out_hdr(nn)) != cudaSuccess ||
            cudaMallocHost(&h_out, out_hdr(nn) + 8 * (h_out_arena = std::min<size_t>(narena, 1 << 16))) != cudaSuccess ||
            cudaMalloc(&d_in, io_bytes + 128 + out_bytes) != cudaSuccess ||
            cudaMalloc(&d_cfg, 8 * nnodes * nd) != cudaSuccess ||
            cudaMalloc(&d_parent, 4 * nnodes) != cudaSuccess ||
            cudaMalloc(&d_dd, 4 * nnodes) != cudaSuccess ||
            cudaMalloc(&d_ready, 4 * nnodes) != cudaSuccess ||
            cudaMalloc(&d_vprefix, 4 * (nn + 1)) != cudaSuccess ||
            cudaMalloc(&d_init, 4) != cudaSuccess) {
            release();
            return set_err(PRRTC_ENOMEM, "plan: device workspace allocation failed (" +
                                             std::to_string((8 * nd + 12) * nnodes) + " bytes of trees)");
        }
        // ready flags are epoch tagged: zero once, launches use epoch >= 1
        cudaMemset(d_ready, 0, 4 * nnodes);
        cudaMemset(d_init, 0, 4);  // epochs start at 1
        // optional: without a mapped block results come back by D2H copy
        if (cudaHostAlloc(&h_map, kMapBytes, cudaHostAllocMapped) == cudaSuccess) {
            std::memset(h_map, 0, kMapBytes);
            void* dm = nullptr;
            if (cudaHostGetDevicePointer(&dm, h_map, 0) == cudaSuccess) {
                d_map = static_cast<unsigned char*>(dm);
            } else {
                cudaFreeHost(h_map);
                h_map = nullptr;
            }
        } else {
            h_map = nullptr;
            cudaGetLastError();
        }
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
        mark = std::make_shared<UseMark>();
        mark->device = dev;
        cudaEventCreateWithFlags(&mark->ev, cudaEventDisableTiming);
        n_cap = nn;
        dof_cap = nd;
        nodes_cap = nnodes;
        arena_cap = narena;
        epoch = 0;
        if (cudaDeviceSynchronize() != cudaSuccess) {
            release();
            return set_err(PRRTC_ECUDA, "plan: workspace initialisation failed");
        }
        return PRRTC_OK;
    }
};

std::mutex g_ws_mu[64];
Workspace g_ws[64];

}  // namespace

struct prrtc_batch {
    const prrtc_robot* robot = nullptr;
    Workspace own;
    Workspace* ws = nullptr;
    int device = 0;
    int n = 0, dof = 0;
    prrtc_params params{};
    long long cap = 0, stride = 0;
    int grid = 0, nthreads = 128, ns_max = 32;
    // warp-worker planner (plan_warp_kernel): eligible batches run one worker
    // per warp, `warps` warps in one CTA per SM (0: the CTA planner runs it)
    bool warp_ok = false, warp_auto = false;
    int warps = 0, cta_grid = 0, scene_words_max = 0;
    unsigned long long budget = 0, arena = 0;
    cudaStream_t last_stream = 0;
    int launches = 0;
    unsigned char* d_out = nullptr;  // ws->d_in + out_offset: out-header, controls, arena
    bool timed = true;  // bracket the kernel with events (batch results report the kernel time)
    bool use_map = false;  // the kernel publishes the result into the workspace's mapped block
    // device views into ws->d_in / d_out
    double *d_starts = nullptr, *d_goals = nullptr;
    const uint32_t** d_scene_words = nullptr;
    SceneF64* d_scene_f64 = nullptr;
    int* d_prob_scene = nullptr;
    unsigned long long* d_arena_used = nullptr;
    int *d_next = nullptr, *d_ndone = nullptr;
    long long* cta_trace = nullptr;  // PRRTC_TRACE only
    ProbCtl* d_ctl = nullptr;
    double* d_arena = nullptr;
    // persistent batches: the bound scenes and their generations at staging
    std::vector<const prrtc_scene*> scenes;
    std::vector<uint64_t> scene_gen;
};

namespace {

int check_params(const prrtc_params* p) {  // planner.cpp:250-252
    if (!(p->delta > 0.0)) return set_err(PRRTC_EINVAL, "plan: delta must be positive");
    if (p->n_cc < 1) return set_err(PRRTC_EINVAL, "plan: n_cc must be >= 1");
    if (p->tree_capacity < 2) return set_err(PRRTC_EINVAL, "plan: tree_capacity too small");
    if (p->threads_per_cta != 0 && p->threads_per_cta != 32 && p->threads_per_cta != 128 &&
        p->threads_per_cta != 256 && p->threads_per_cta != 512)
        return set_err(PRRTC_EINVAL, "plan: threads_per_cta must be 0, 32, 128, 256 or 512");
    if (p->sampler != PRRTC_SAMPLER_HALTON && p->sampler != PRRTC_SAMPLER_UNIFORM)
        return set_err(PRRTC_EINVAL, "plan: unknown sampler");
    return PRRTC_OK;
}

// The Halton samples of tickets [0, kSampleTab) for (robot, seed): every
// problem of a batch draws the same ones (sample index 1 + seed + ticket in
// the robot's limits), so they are computed once — by debug_sample_kernel,
// the planner's own sampler (bit-exact, test_sample_config_bitexact) — and
// read from L2 by every CTA instead of recomputed per ticket block (the
// sample phase was ~5.6% of planner CTA cycles). Built synchronously on first
// use and kept for the robot's lifetime (a launch may still read an older
// table, so none is freed early); at most kSampleTabs seeds per robot.
constexpr unsigned long long kSampleTab = 4096;
constexpr size_t kSampleTabs = 16;
const double* sample_table(const prrtc_robot* r, uint64_t seed, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(r->stab_mu);
    for (const auto& t : r->stab)
        if (t.first == seed) return t.second;
    if (r->stab.size() >= kSampleTabs) return nullptr;
    double* d = nullptr;
    if (cudaMalloc(&d, sizeof(double) * kSampleTab * r->dof) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (launch_debug_sample(r->args(), 1 + seed, (int)kSampleTab, d, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d);
        return nullptr;
    }
    r->stab.emplace_back(seed, d);
    return d;
}

// the largest dynamic shared memory a CTA may opt into (cached per device)
int smem_optin(int device) {
    static std::atomic<int> cache[64];
    if (device < 0 || device >= 64) return 48 * 1024;
    int v = cache[device].load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        if (v <= 0) v = 48 * 1024;
        cache[device].store(v, std::memory_order_relaxed);
    }
    return v;
}

int sm_count(int device) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n > 0 ? n : 1;
}

template <class T>
int dmalloc(T** p, size_t count) {
    if (cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(1, count)) != cudaSuccess)
        return set_err(PRRTC_ENOMEM, "device allocation of " + std::to_string(sizeof(T) * count) + " bytes failed");
    return PRRTC_OK;
}

// Validates the request and fills the batch sizing (no device work).
int batch_setup(prrtc_batch* b, const prrtc_robot* robot, const prrtc_scene* const* scenes,
                uint32_t n_problems, const double* starts, const double* goals, uint32_t dof,
                const prrtc_params* params) {
    if (!robot || !scenes || !starts || !goals || !params)
        return set_err(PRRTC_EINVAL, "plan: null argument");
    if ((int)dof != robot->dof)  // require_dim (types.hpp:16-21)
        return set_err(PRRTC_EINVAL, "plan.start: expected dimension " + std::to_string(robot->dof) +
                                         ", got " + std::to_string(dof));
    int rc = check_params(params);
    if (rc) return rc;
    if (n_problems == 0) return set_err(PRRTC_EINVAL, "plan: empty batch");
    for (uint32_t i = 0; i < n_problems; ++i)
        if (!scenes[i] || scenes[i]->device != robot->device)
            return set_err(PRRTC_EINVAL, "plan: scene missing or on another device");
    rc = check_device(robot->device);
    if (rc) return rc;
    b->robot = robot;
    b->device = robot->device;
    b->n = (int)n_problems;
    b->dof = (int)dof;
    b->params = *params;
    b->cap = std::max<long long>(2, (long long)(params->tree_capacity / 2));  // planner.cpp:290
    b->stride = (b->cap + 31) / 32 * 32;
    // CTA size (threads_per_cta = 0): a single problem gets 512-thread CTAs
    // (the extra warps split the chunk's links / primitives / pairs: lower
    // latency per iteration); batches use 128-thread CTAs (more independent
    // workers per SM) unless the robot is large (many fine spheres or self
    // pairs, e.g. the dual-arm Baxter), where the split pays again
    // a single problem: 512-thread CTAs, one per SM (16 warps split each
    // chunk's links / primitives / pairs: measured -3% / -6% / -21% median
    // latency for Panda / Fetch / Baxter against 256, tools/lat_variants.py)
    // (batches of large robots used 256-thread CTAs until this round's hot
    // code changes; 128 is now faster for Baxter too: 1000 problems 12.7 ->
    // 11.7 ms, 3333 problems 41.0 -> 37.2 ms)
    b->nthreads = params->threads_per_cta && params->threads_per_cta != 32
                      ? (int)params->threads_per_cta
                      : (n_problems == 1 ? 512 : 128);
    const EnvKnobs& ekw = env();
    // The warp-worker planner (one RRT-Connect worker per warp,
    // plan_warp_kernel) for batches whose mode allows it (not deterministic
    // replay with its exact CheckStats, not the Uniform sampler's per-CTA
    // generator, no phase tracer or debug flags): asked for with
    // threads_per_cta = 32, and chosen automatically (threads_per_cta = 0)
    // when the batch holds at least as many problems as the device has warp
    // workers, and at least 2048 (batch_bind): its weakness is per-problem
    // latency, which only a long tail of problems exposes.
    // PRRTC_WARP=1 / 0 force it on / off for every eligible batch (A/B).
    const bool warp_mode_ok = n_problems > 1 && !params->deterministic &&
                              params->sampler == PRRTC_SAMPLER_HALTON && !ekw.trace && ekw.debug_flags == 0;
    b->warp_ok = warp_mode_ok && (params->threads_per_cta == 32 ||
                                  (params->threads_per_cta == 0 && ekw.warp != 0));
    b->warp_auto = b->warp_ok && params->threads_per_cta == 0 && ekw.warp < 0;
    // states per validation chunk: one n_cc = 32 edge; a 256-thread CTA uses
    // its extra warps to split links / pairs / primitives of the same chunk.
    // A single problem (latency-bound, one CTA per SM) takes wider chunks: a
    // connect chain needs fewer chunk rounds. 64 states on 256-thread CTAs
    // (Panda median wall latency 0.141 -> 0.121 ms); 128 on the default
    // 512-thread CTAs when they fit the shared memory (Panda median 0.097 ->
    // 0.089 ms, Fetch and Baxter +-0; tools/lat.py). PRRTC_NS32 / PRRTC_NS64 /
    // PRRTC_NS128 force a width (64-state chunks in the Panda batch: 159k ->
    // 137k problems/s).
    const EnvKnobs& ek = env();
    const bool wide = !ek.ns32 && ((n_problems == 1 && b->nthreads >= 256) || ek.ns64 || ek.ns128);
    bool ns128 = wide && (ek.ns128 || (n_problems == 1 && b->nthreads >= 512 && !ek.ns64));
    if (ns128 && !ek.ns128) {
        size_t swm1 = 0;
        for (uint32_t i = 0; i < n_problems; ++i) swm1 = std::max(swm1, scenes[i]->words.size());
        ns128 = smem_bytes(robot->args(), 128, b->nthreads, (int)swm1 + 4,
                           params->sampler == PRRTC_SAMPLER_UNIFORM) <= (size_t)smem_optin(robot->device);
    }
    b->ns_max = wide ? (ns128 ? 128 : 64) : 32;
    // shared memory per CTA follows the largest scene of the launch and the
    // sampler (the Uniform generator's state); occupancy is cached per
    // scene-size bucket, computed at the bucket's upper bound
    size_t swm = 0;
    for (uint32_t i = 0; i < n_problems; ++i) swm = std::max(swm, scenes[i]->words.size());
    static const int kSceneBucket[5] = {256, 512, 768, 1024, SCENE_MAX_WORDS};
    int bk = 0;
    while (bk < 4 && (int)swm > kSceneBucket[bk]) ++bk;
    const bool uni = params->sampler == PRRTC_SAMPLER_UNIFORM;
    const int okey = (b->ns_max / 32 + (b->nthreads == 256 ? 5 : (b->nthreads == 512 ? 10 : 0))) * 10 +
                     (uni ? 5 : 0) + bk;
    int occ = robot->occ[okey].load(std::memory_order_relaxed);
    if (occ == 0) {
        occ = plan_occupancy(robot->args(), b->ns_max, b->nthreads, kSceneBucket[bk], uni);
        robot->occ[okey].store(occ, std::memory_order_relaxed);
    }
    const int sms = sm_count(robot->device);
    unsigned workers_eff;
    if (params->deterministic) {
        b->grid = 1;
        workers_eff = 1;
    } else if (n_problems == 1) {
        // workers = 0: one CTA per SM (measured: ~64-148 CTAs give
        // the lowest time-to-solution; 2 per SM only adds redundant work)
        b->grid = (int)(params->workers ? std::min<unsigned>(params->workers, sms * occ)
                                        : (b->nthreads >= 256 ? sms : 2 * sms));
        workers_eff = b->grid;
    } else {
        const unsigned per_sm = params->ctas_per_sm ? std::min<unsigned>(params->ctas_per_sm, occ) : occ;
        b->grid = sms * per_sm;
        // batch budget: workers=0 gives every problem the iteration budget of
        // kBatchWorkers reference workers (the reference's default is
        // workers = hardware concurrency, planner.cpp:287-288); CTAs are
        // shared elastically, so this is a budget, not a CTA count
        constexpr unsigned kBatchWorkers = 32;
        workers_eff = params->workers ? params->workers : kBatchWorkers;
    }
    b->budget = params->max_iters_per_worker * (unsigned long long)workers_eff;
    b->cta_grid = b->grid;
    // path arena: room for a 4096-config path per problem on average
    b->arena = (unsigned long long)dof * std::min<long long>(4096, 2 * b->cap) * n_problems;
    return PRRTC_OK;
}

// Binds the batch to a workspace and stages the inputs into its pinned buffer.
size_t io_used(const prrtc_batch* b) {
    const size_t n = b->n, dof = b->dof;
    return 8 * 2 * n * dof + sizeof(void*) * n + sizeof(SceneF64) * n + 4 * n;
}

// offset of the out-header in the device block (and of its zeroed image in h_io)
size_t out_offset(const prrtc_batch* b) { return (io_used(b) + 127) / 128 * 128; }

int batch_bind(prrtc_batch* b, Workspace* ws, const prrtc_scene* const* scenes, const double* starts,
               const double* goals) {
    int rc = ws->reserve(b->device, b->n, b->dof, b->stride, b->arena);
    if (rc) return rc;
    b->ws = ws;
    const size_t n = b->n, dof = b->dof;
    unsigned char* h = static_cast<unsigned char*>(ws->h_io);
    unsigned char* d = ws->d_in;
    size_t o = 0;
    if (starts) std::memcpy(h + o, starts, 8 * n * dof);  // (null: re-staging, inputs already in h_io)
    b->d_starts = reinterpret_cast<double*>(d + o);
    o += 8 * n * dof;
    if (goals) std::memcpy(h + o, goals, 8 * n * dof);
    b->d_goals = reinterpret_cast<double*>(d + o);
    o += 8 * n * dof;
    auto** sw = reinterpret_cast<const uint32_t**>(h + o);
    b->d_scene_words = reinterpret_cast<const uint32_t**>(d + o);
    o += sizeof(void*) * n;
    auto* sf = reinterpret_cast<SceneF64*>(h + o);
    b->d_scene_f64 = reinterpret_cast<SceneF64*>(d + o);
    o += sizeof(SceneF64) * n;
    auto* ps = reinterpret_cast<int*>(h + o);
    b->d_prob_scene = reinterpret_cast<int*>(d + o);
    o += 4 * n;
    b->scenes.assign(scenes, scenes + n);
    b->scene_gen.resize(n);
    for (size_t i = 0; i < n; ++i) {
        b->scene_gen[i] = scenes[i]->generation.load(std::memory_order_acquire);
        const SceneArgs sa = scenes[i]->args();
        sw[i] = sa.words;
        sf[i] = sa.f64;
        ps[i] = (int)i;
        scenes[i]->mark_use(ws->mark);
    }
    std::memset(h + out_offset(b), 0, Workspace::out_hdr(n));  // the zeroed controls ride the upload
    b->d_out = d + out_offset(b);
    b->d_arena_used = reinterpret_cast<unsigned long long*>(b->d_out);
    b->d_next = reinterpret_cast<int*>(b->d_out + 8);
    b->d_ndone = reinterpret_cast<int*>(b->d_out + 12);
    b->d_ctl = reinterpret_cast<ProbCtl*>(b->d_out + 128);
    b->d_arena = reinterpret_cast<double*>(b->d_out + Workspace::out_hdr(n));
    // warp-worker sizing: every warp holds a copy of its problem's scene,
    // so the per-warp region follows the largest bound scene
    b->warps = 0;
    b->grid = b->cta_grid;
    size_t mx = 0;
    for (size_t i = 0; i < n; ++i) mx = std::max(mx, scenes[i]->words.size());
    b->scene_words_max = (int)((mx + 3) & ~size_t(3));
    if (b->warp_ok) {
        b->warps = warp_workers_per_sm(b->robot->words.data(), b->scene_words_max, smem_optin(b->device));
        if (env().warps_cap > 0) b->warps = std::min(b->warps, env().warps_cap);
        const int sms = sm_count(b->device);
        // (crossover measured with windowed help scans: Panda ~2500
        // problems, Fetch < 2500, Baxter ~2000; below it the per-problem
        // latency of a warp worker sets the batch's tail)
        if (b->warp_auto && (long long)b->n < std::max(2048ll, (long long)b->warps * sms)) b->warps = 0;
        if (b->warps > 0) b->grid = sms;
    }
    return PRRTC_OK;
}


constexpr int kMnnNodesSingle = 2048;

// Enqueues: inputs H2D (optional), header memset, the planner kernel.
int batch_enqueue(prrtc_batch* b, cudaStream_t st, bool upload) {
    const auto q0 = std::chrono::steady_clock::now();
    Workspace* ws = b->ws;
    cudaSetDevice(b->device);
    b->last_stream = st;
    if (++ws->epoch == 0) ++ws->epoch;
    const size_t up = out_offset(b) + Workspace::out_hdr(b->n);
    // a single problem published through mapped memory needs no copy at all:
    // start, goal and scene travel in the kernel parameters and the kernel
    // zeroes its own controls (PlanArgs::inline_inputs)
    const bool inline_in = upload && b->n == 1 && b->use_map && ws->d_map && b->dof <= 32 && !env().trace;
    ws->last_h2d = upload && !inline_in ? up : 0;
    if (inline_in) {
        // (no copy)
    } else if (upload) {  // inputs + zeroed out-header in one copy
        CUDA_TRY(cudaMemcpyAsync(ws->d_in, ws->h_io, up, cudaMemcpyHostToDevice, st));
    } else {
        CUDA_TRY(cudaMemsetAsync(b->d_out, 0, Workspace::out_hdr(b->n), st));
    }
    PlanArgs a{};
    if (inline_in) {
        const unsigned char* h = static_cast<const unsigned char*>(ws->h_io);  // batch_bind's staging
        std::memcpy(a.in_sg, h, 8 * 2 * (size_t)b->dof);
        size_t o = 8 * 2 * (size_t)b->dof;
        std::memcpy(&a.scene_words1, h + o, sizeof(void*));
        o += sizeof(void*);
        std::memcpy(&a.scene_f64_1, h + o, sizeof(SceneF64));
        a.inline_inputs = 1;
        a.init_flag = ws->d_init;
    }
    a.robot = b->robot->d_words;
    a.fine_r64 = b->robot->d_fine_r64;
    a.limits = b->robot->d_limits;
    a.scene_words = b->d_scene_words;
    a.scene_f64 = b->d_scene_f64;
    a.prob_scene = b->d_prob_scene;
    a.starts = b->d_starts;
    a.goals = b->d_goals;
    a.n_problems = b->n;
    a.ctl = b->d_ctl;
    a.cfg = ws->d_cfg;
    a.parent = ws->d_parent;
    a.ready = ws->d_ready;
    a.dd = ws->d_dd;
    a.cap = b->cap;
    a.stride = b->stride;
    a.arena = b->d_arena;
    a.arena_used = b->d_arena_used;
    a.arena_cap = b->arena;
    a.next_problem = b->d_next;
    a.n_done = b->d_ndone;
    a.trace = inline_in ? nullptr : reinterpret_cast<unsigned long long*>(b->d_out + 16);
    a.cta_trace = nullptr;
    const EnvKnobs& ek = env();
    if (ek.trace) {
        static long long* d_ct = nullptr;
        static int ct_cap = 0;
        if (ct_cap < b->grid) {
            cudaFree(d_ct);
            cudaMalloc(&d_ct, sizeof(long long) * 64 * b->grid);
            ct_cap = b->grid;
        }
        cudaMemsetAsync(d_ct, 0, sizeof(long long) * 64 * b->grid, st);
        a.cta_trace = d_ct;
        b->cta_trace = d_ct;
    }
    a.epoch = ws->epoch;
    a.dbg = ek.debug_flags;
    a.p.delta = b->params.delta;
    a.p.dd_radius = b->params.dd_radius > 0.0 ? b->params.dd_radius : 4.0 * b->params.delta;
    a.p.n_cc = b->params.n_cc;
    a.p.dynamic_domain = b->params.dynamic_domain;
    a.p.balance = b->params.balance;
    a.p.early_exit = b->params.early_exit;
    a.p.two_stage = b->params.two_stage;
    a.p.deterministic = b->params.deterministic;
    a.ref_stats = b->params.deterministic ? 1 : 0;
    a.tail_claim = ek.tail_claim;
    a.tail_min = ek.tail_min;
    a.tail_div = ek.tail_div;
    // help joins stop at the problem's worker cap (an env override for sweeps)
    a.help_cap = ek.help_cap ? ek.help_cap : (int)b->params.max_workers_per_problem;
    a.help_policy = ek.help_policy;
    a.stab = nullptr;
    a.stab_n = 0;
    if (b->params.sampler == PRRTC_SAMPLER_HALTON && !ek.no_stab) {
        a.stab = sample_table(b->robot, b->params.seed, st);
        a.stab_n = a.stab ? kSampleTab : 0;
    }
    a.p.budget = b->budget;
    a.p.seed = b->params.seed;
    a.p.uniform = b->params.sampler == PRRTC_SAMPLER_UNIFORM ? 1 : 0;
    a.ns_max = b->ns_max;
    a.nthreads = b->nthreads;
    // multi-sample NN bound (samples x tree nodes per pass, ~4-8 node pairs
    // per thread): batches trade a longer pass for fewer passes; a single
    // problem is latency-bound (PRRTC_MNN_NODES overrides, for sweeps)
    a.mnn_nodes = b->n == 1 ? kMnnNodesSingle : 2048;
    if (ek.mnn_nodes) a.mnn_nodes = ek.mnn_nodes;
    if (b->use_map && ws->d_map) {
        a.out_map = ws->d_map;
        a.out_map_bytes = Workspace::kMapBytes;
        if (ek.map_bytes >= 0)  // tests: force the copy-back fallback
            a.out_map_bytes = std::min<unsigned long long>(a.out_map_bytes, (unsigned long long)ek.map_bytes);
        a.out_dev = b->d_out;
        a.out_hdr_bytes = Workspace::out_hdr(b->n);
        a.exit_count = reinterpret_cast<unsigned*>(b->d_out + 32);
    } else {
        b->use_map = false;
    }
    const auto e0 = std::chrono::steady_clock::now();
    a.scene_words_max = b->scene_words_max;  // per-CTA (per-warp) scene region size
    if (b->warps) {
        // warp workers: a multi-sample NN pass bounded to ~2 node pairs per
        // lane (128 nodes: 10k batches Baxter -3%, Fetch -2% vs 512)
        a.mnn_nodes = ek.mnn_nodes ? ek.mnn_nodes : 128;
    }
    if (b->timed) CUDA_TRY(cudaEventRecord(ws->ev0, st));
    const auto e1 = std::chrono::steady_clock::now();
    if (b->warps)
        CUDA_TRY(launch_plan_warp(b->robot->args(), b->robot->words.data(), a, b->grid, b->warps, st));
    else
        CUDA_TRY(launch_plan(b->robot->args(), a, b->grid, st));
    const auto e2 = std::chrono::steady_clock::now();
    if (b->timed) CUDA_TRY(cudaEventRecord(ws->ev1, st));
    if (ek.host_trace) {
        auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
        std::fprintf(stderr, "prrtc enqueue: copies %.1f ev0 %.1f launch %.1f ev1 %.1f us\n", us(q0, e0),
                     us(e0, e1), us(e1, e2), us(e2, std::chrono::steady_clock::now()));
    }
    if (b->params.validate_path)  // stream-ordered after the planner, outside its timing
        CUDA_TRY(launch_validate_paths(b->robot->args(), a, ws->d_vprefix, 4 * sm_count(b->device), st));
    CUDA_TRY(cudaEventRecord(ws->mark->ev, st));  // the scenes' completion marker
    b->launches = 1;
    return PRRTC_OK;
}

const char* message_for(int msg) {
    switch (msg) {  // planner.cpp:270-276, 317-320
        case 1: return "start configuration is out of limits or in collision";
        case 2: return "goal configuration is out of limits or in collision";
        case 3: return "tree capacity exhausted";
        case 4: return "all workers exhausted their iteration budgets";
        case 5: return "path arena exhausted";
        case 6: return "assemble_path: meeting configurations disagree";
        default: return "";
    }
}

// path_cost (planner.cpp:152-158) with the scalar distance (nn.cpp:12-20).
// path_cost (planner.cpp:152-158) and, in the same pass, assemble_path's
// zero-length check (planner.cpp:144-148: no bitwise-equal consecutive
// configs; a zero distance is confirmed bitwise, so +0 / -0 pairs pass).
double path_cost(const double* path, uint32_t len, uint32_t dof, bool* zero_segment) {
    double cost = 0.0;
    *zero_segment = false;
    for (uint32_t i = 1; i < len; ++i) {
        double acc = 0.0;
        const double* a = path + (size_t)(i - 1) * dof;
        const double* b = path + (size_t)i * dof;
        for (uint32_t d = 0; d < dof; ++d) {
            const double e = a[d] - b[d];
            acc += e * e;
        }
        if (acc == 0.0 && std::memcmp(a, b, sizeof(double) * dof) == 0) *zero_segment = true;
        cost += std::sqrt(acc);
    }
    return cost;
}

// Copies the header, controls and used arena back and fills out[].
std::chrono::steady_clock::time_point g_sync_time;  // PRRTC_HOST_TRACE

// ---------------------------------------------------------------------------
// result path blocks: a batch's paths stay in the pinned block the D2H copy
// of the path arena landed in; every result of the batch points into it and
// holds one reference (prrtc_result_free drops it), so a 1000-problem call
// costs no per-path allocation or host copy (fill was ~0.17 ms of a ~2 ms
// call). Blocks are pooled: cudaHostAlloc / cudaFreeHost are slow and the
// latter can synchronise the device.
// ---------------------------------------------------------------------------
struct PathBlock {
    double* data = nullptr;
    size_t cap = 0;  // doubles
    std::atomic<int> refs{0};
};
constexpr int kMaxPathBlocks = 4096;
std::atomic<PathBlock*> g_path_blocks[kMaxPathBlocks];
std::mutex g_path_mu;
std::vector<PathBlock*> g_path_pool;  // free blocks (refs 0, no slot)
int g_path_hint = 0;

// A block of >= doubles capacity in a free slot: returns the slot id (1-based)
// or 0 (no slot or no pinned memory: the caller falls back to copies).
int path_block_acquire(size_t doubles, PathBlock** out) {
    std::lock_guard<std::mutex> lk(g_path_mu);
    int slot = -1;
    for (int k = 0; k < kMaxPathBlocks; ++k) {
        const int i = (g_path_hint + k) % kMaxPathBlocks;
        if (!g_path_blocks[i].load(std::memory_order_relaxed)) {
            slot = i;
            break;
        }
    }
    if (slot < 0) return 0;
    PathBlock* pb = nullptr;
    size_t best = SIZE_MAX;
    int bi = -1;
    for (int i = 0; i < (int)g_path_pool.size(); ++i)
        if (g_path_pool[i]->cap >= doubles && g_path_pool[i]->cap < best) {
            best = g_path_pool[i]->cap;
            bi = i;
        }
    if (bi >= 0) {
        pb = g_path_pool[bi];
        g_path_pool.erase(g_path_pool.begin() + bi);
    } else {
        size_t cap = size_t(1) << 17;  // 1 MB at least, powers of two
        while (cap < doubles) cap <<= 1;
        pb = new PathBlock();
        if (cudaHostAlloc(reinterpret_cast<void**>(&pb->data), 8 * cap, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            delete pb;
            return 0;
        }
        pb->cap = cap;
    }
    pb->refs.store(0, std::memory_order_relaxed);
    g_path_blocks[slot].store(pb, std::memory_order_release);
    g_path_hint = slot + 1;
    *out = pb;
    return slot + 1;
}

void path_block_release(int id) {  // refs reached 0 (or never handed out)
    std::lock_guard<std::mutex> lk(g_path_mu);
    PathBlock* pb = g_path_blocks[id - 1].exchange(nullptr, std::memory_order_acq_rel);
    if (!pb) return;
    g_path_pool.push_back(pb);
    while (g_path_pool.size() > 8) {  // keep a few; free the oldest
        cudaFreeHost(g_path_pool.front()->data);
        delete g_path_pool.front();
        g_path_pool.erase(g_path_pool.begin());
    }
}

void path_block_unref(int id) {
    if (id <= 0 || id > kMaxPathBlocks) return;
    PathBlock* pb = g_path_blocks[id - 1].load(std::memory_order_acquire);
    if (pb && pb->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) path_block_release(id);
}

int fill_results(prrtc_batch* b, prrtc_result* out, const unsigned char* h, const double* arena,
                 unsigned long long used, int block_id = 0, PathBlock* pb = nullptr);

int batch_collect(prrtc_batch* b, prrtc_result* out) {
    Workspace* ws = b->ws;
    cudaSetDevice(b->device);
    if (b->use_map) {
        // wait for publish_result's flag (not for the grid to retire); poll
        // the stream now and then so a failed launch cannot hang the caller
        const volatile unsigned* f = static_cast<const volatile unsigned*>(ws->h_map);
        for (unsigned spins = 1; f[0] != ws->epoch; ++spins) {
            if ((spins & 1023) == 0) {
                const cudaError_t q = cudaStreamQuery(b->last_stream);
                if (q == cudaErrorNotReady) continue;
                if (f[0] == ws->epoch) break;
                if (q != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("plan: ") + cudaGetErrorString(q));
                break;  // retired without the flag: read back below
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        g_sync_time = std::chrono::steady_clock::now();
        b->use_map = false;
        if (f[0] == ws->epoch && f[1] == 1u) {
            const unsigned char* h = static_cast<const unsigned char*>(ws->h_map) + 64;
            const size_t hdr = Workspace::out_hdr(b->n);
            const unsigned long long used =
                std::min<unsigned long long>(*reinterpret_cast<const unsigned long long*>(h), b->arena);
            ws->last_d2h = hdr + 8 * used;
            ws->path_hint = (double)used / b->n;
            return fill_results(b, out, h, reinterpret_cast<const double*>(h + hdr), used);
        }
        // did not fit (very long path): the regular copy-back
    }
    const size_t hdr = Workspace::out_hdr(b->n);
    // one D2H of header + controls + an arena prefix sized from the paths of
    // recent calls (a single problem reads back a few KB, not the whole
    // arena); a second copy only when the paths overflow the prefix
    size_t prefix = std::min<size_t>(b->arena, 1 << 16);
    if (ws->path_hint > 0.0) {
        const size_t want = (size_t)(1.5 * ws->path_hint * b->n) + 64 * (size_t)b->dof;
        ws->grow_h_out(std::min<size_t>(want, b->arena));
        prefix = std::min({(size_t)b->arena, want, ws->h_out_arena});
    }
    ws->last_d2h = hdr + 8 * prefix;
    // batches: the arena prefix goes straight into a pooled pinned path block
    // that the results will point into (a single problem keeps its one copy)
    PathBlock* pb = nullptr;
    int bid = b->n > 1 ? path_block_acquire(prefix, &pb) : 0;
    if (bid) {
        CUDA_TRY(cudaMemcpyAsync(ws->h_out, b->d_out, hdr, cudaMemcpyDeviceToHost, b->last_stream));
        CUDA_TRY(cudaMemcpyAsync(pb->data, b->d_arena, 8 * prefix, cudaMemcpyDeviceToHost, b->last_stream));
    } else {
        CUDA_TRY(cudaMemcpyAsync(ws->h_out, b->d_out, hdr + 8 * prefix, cudaMemcpyDeviceToHost, b->last_stream));
    }
    const cudaError_t se = cudaStreamSynchronize(b->last_stream);
    if (se != cudaSuccess) {
        if (bid) path_block_release(bid);
        return set_err(PRRTC_ECUDA, std::string("plan: ") + cudaGetErrorString(se));
    }
    g_sync_time = std::chrono::steady_clock::now();
    const unsigned char* h = static_cast<const unsigned char*>(ws->h_out);
    unsigned long long used = *reinterpret_cast<const unsigned long long*>(h);
    used = std::min<unsigned long long>(used, b->arena);
    {
        const double per = (double)used / b->n;
        ws->path_hint = per >= ws->path_hint ? per : 0.9 * ws->path_hint + 0.1 * per;
    }
    if (bid) {
        if (used > prefix) {  // fetch the rest, into a block that holds all of it
            ws->last_d2h += 8 * (used - prefix);
            if (used > pb->cap) {
                PathBlock* nb = nullptr;
                const int nid = path_block_acquire(used, &nb);
                if (!nid) {
                    path_block_release(bid);
                    return set_err(PRRTC_ENOMEM, "plan: pinned path block allocation failed");
                }
                std::memcpy(nb->data, pb->data, 8 * prefix);
                path_block_release(bid);
                bid = nid;
                pb = nb;
            }
            if (cudaMemcpy(pb->data + prefix, b->d_arena + prefix, 8 * (used - prefix), cudaMemcpyDeviceToHost) !=
                cudaSuccess) {
                path_block_release(bid);
                return set_err(PRRTC_ECUDA, "plan: path read-back failed");
            }
        }
        return fill_results(b, out, h, pb->data, used, bid, pb);
    }
    const double* arena = reinterpret_cast<const double*>(h + hdr);
    std::vector<double> big;
    if (used > prefix) {
        big.resize(used);  // prefix already on the host; fetch only the rest
        ws->last_d2h += 8 * (used - prefix);
        std::memcpy(big.data(), arena, 8 * prefix);
        CUDA_TRY(cudaMemcpy(big.data() + prefix, b->d_arena + prefix, 8 * (used - prefix),
                            cudaMemcpyDeviceToHost));
        arena = big.data();
    }
    return fill_results(b, out, h, arena, used);
}

// Parses a host copy of the out-header (h), controls and arena into out[].
int fill_results(prrtc_batch* b, prrtc_result* out, const unsigned char* h, const double* arena,
                 unsigned long long used, int block_id, PathBlock* pb) {
    Workspace* ws = b->ws;
    int block_refs = 0;
    const ProbCtl* ctl = reinterpret_cast<const ProbCtl*>(h + 128);
    float ms = 0.f;
    if (b->timed) cudaEventElapsedTime(&ms, ws->ev0, ws->ev1);
    if (env().trace) {  // kernel span vs per-problem span (globaltimer)
        const auto* tr = reinterpret_cast<const unsigned long long*>(h + 16);
        const long long k0 = (long long)(0x7fffffffffffffffull - tr[0]), k1 = (long long)tr[1];
        long long p0 = ctl[0].t_start_ns, p1 = ctl[0].t_end_ns;
        for (int i = 1; i < b->n; ++i) {
            p0 = std::min(p0, ctl[i].t_start_ns);
            p1 = std::max(p1, ctl[i].t_end_ns);
        }
        std::fprintf(stderr,
                     "prrtc trace: events %.3f ms | first CTA -> first init %.3f | inits -> last done %.3f | "
                     "last done -> last CTA exit %.3f | grid %d x %d\n",
                     ms, (p0 - k0) * 1e-6, (p1 - p0) * 1e-6, (k1 - p1) * 1e-6, b->grid, b->nthreads);
        if (!env().dump_ctl.empty()) {  // per-problem timeline (analysis tools)
            if (FILE* o = std::fopen(env().dump_ctl.c_str(), "w")) {
                for (int i = 0; i < b->n; ++i)
                    std::fprintf(o, "%d %.6f %.6f %llu %d %d\n", i, (ctl[i].t_start_ns - k0) * 1e-6,
                                 (ctl[i].t_end_ns - k0) * 1e-6, (unsigned long long)ctl[i].iters_used, ctl[i].done,
                                 ctl[i].winner);
                std::fclose(o);
            }
        }
        if (b->cta_trace) {
            std::vector<long long> ct(64 * b->grid);
            cudaMemcpy(ct.data(), b->cta_trace, 8 * ct.size(), cudaMemcpyDeviceToHost);
            {  // per-phase SM cycles summed over CTAs (kernels.cu trace_phase codes)
                static const char* names[16] = {"-", "header", "nn_extend", "dd+steer", "nn_connect", "fk+collide",
                                                 "winner", "sample", "append", "chain_book", "leave", "", "", "",
                                                 "", ""};
                double cyc[16] = {0}, cnt[16] = {0}, tot = 0;
                for (int g = 0; g < b->grid; ++g)
                    for (int k = 0; k < 16; ++k) {
                        cyc[k] += (double)ct[64 * g + 32 + k];
                        cnt[k] += (double)ct[64 * g + 48 + k];
                    }
                for (int k = 0; k < 16; ++k) tot += cyc[k];
                std::fprintf(stderr, "prrtc phases (share of CTA cycles, mean cycles/entry):");
                for (int k = 1; k < 16; ++k)
                    if (cnt[k] > 0)
                        std::fprintf(stderr, " %s %.1f%% %.0f", names[k], 100.0 * cyc[k] / tot, cyc[k] / cnt[k]);
                std::fprintf(stderr, "\n");
            }
            long long max_start = 0, max_leave = 0, max_flush = 0, max_exit = 0;
            int slow = -1;
            for (int g = 0; g < b->grid; ++g) {
                const long long* t = &ct[64 * g];
                max_start = std::max(max_start, t[3] - k0);
                if (t[0]) {
                    if (t[0] - p1 > max_leave) { max_leave = t[0] - p1; slow = g; }
                    max_flush = std::max(max_flush, t[1] - t[0]);
                    max_exit = std::max(max_exit, t[2] - t[1]);
                }
            }
            {  // when the CTAs left the kernel (t[2], globaltimer): the share of CTA time a batch's tail idles
                std::vector<long long> ex;
                for (int g = 0; g < b->grid; ++g)
                    if (ct[64 * g + 2]) ex.push_back(ct[64 * g + 2] - k0);
                std::sort(ex.begin(), ex.end());
                if (!ex.empty()) {
                    double busy = 0;
                    for (long long e : ex) busy += (double)e;
                    auto q = [&](double f) { return ex[std::min(ex.size() - 1, (size_t)(f * ex.size()))] * 1e-6; };
                    std::fprintf(stderr,
                                 "prrtc trace: CTA exits (ms) p10 %.3f p50 %.3f p90 %.3f max %.3f | CTA-time used %.1f%%\n",
                                 q(0.1), q(0.5), q(0.9), ex.back() * 1e-6, 100.0 * busy / ((double)ex.back() * ex.size()));
                }
            }
            std::fprintf(stderr,
                         "prrtc trace: latest CTA start +%.3f ms | latest leave after last done %.3f (CTA %d) | "
                         "max flush+leave %.3f | max leave->exit %.3f\n",
                         max_start * 1e-6, max_leave * 1e-6, slow, max_flush * 1e-6, max_exit * 1e-6);
            if (slow >= 0) {
                const long long* t = &ct[64 * slow];
                std::fprintf(stderr, "prrtc trace: slow CTA %d: iterations %lld, last phase %lld entered %.3f ms "
                                     "before leaving (%.3f ms after last done)\n",
                             slow, t[5], t[6], (t[0] - t[7]) * 1e-6, (t[7] - p1) * 1e-6);
                std::fprintf(stderr, "prrtc trace: slow CTA events (phase@ms rel. first init):");
                const long long nev = std::min<long long>(t[4], 11);
                for (long long e = t[4] - nev; e < t[4]; ++e)
                    std::fprintf(stderr, " %lld@%.3f", t[8 + 2 * (e % 11)], (t[9 + 2 * (e % 11)] - p0) * 1e-6);
                std::fprintf(stderr, " | start@%.3f leave@%.3f done@%.3f\n", (t[3] - p0) * 1e-6,
                             (t[0] - p0) * 1e-6, (p1 - p0) * 1e-6);
            }
        }
    }
    for (int i = 0; i < b->n; ++i) {
        prrtc_result& r = out[i];
        std::memset(&r, 0, sizeof(r));
        const ProbCtl& C = ctl[i];
        r.dof = b->dof;
        r.status = C.done == 1 ? PRRTC_SOLVED : C.done == 3 ? PRRTC_INFEASIBLE_ENDPOINT : PRRTC_FAILED;
        {  // (no snprintf per result: ~0.1 ms per 1000-problem batch)
            const char* msg = C.done == 0 ? "problem did not finish" : message_for(C.msg);
            if (msg[0]) std::strncpy(r.message, msg, sizeof(r.message) - 1);
        }
        if (r.status == PRRTC_SOLVED && C.path_len > 0 &&
            C.path_off + (unsigned long long)C.path_len * b->dof <= used) {
            r.path_len = C.path_len;
            if (pb) {  // a view into the batch's path block (one reference per path)
                r.path = const_cast<double*>(arena) + C.path_off;
                r.path_block = (uint32_t)block_id;
                ++block_refs;
            } else {
                r.path = static_cast<double*>(std::malloc(sizeof(double) * b->dof * C.path_len));
                std::memcpy(r.path, arena + C.path_off, sizeof(double) * b->dof * C.path_len);
            }
            bool zero_segment = false;
            r.cost = path_cost(r.path, r.path_len, b->dof, &zero_segment);
            // planner.cpp:144-148: no zero-length (bitwise-equal) segment
            if (zero_segment) {
                if (r.path_block) {  // not handed out: drop the view
                    r.path = nullptr;
                    r.path_len = 0;
                    r.path_block = 0;
                    --block_refs;
                } else {
                    prrtc_result_free(&r);
                }
                r.status = PRRTC_FAILED;
                r.cost = 0.0;
                std::snprintf(r.message, sizeof(r.message), "assemble_path: zero-length segment in assembled path");
            }
        } else if (r.status == PRRTC_SOLVED) {
            r.status = PRRTC_FAILED;
            std::snprintf(r.message, sizeof(r.message), "path unavailable");
        }
        if (C.inv_bad)  // PRRTC_DEBUG_FLAGS bit 2 only
            std::snprintf(r.message, sizeof(r.message), "debug: %d tree invariant violations", C.inv_bad);
        // per-problem device time (globaltimer: initialisation -> finish)
        r.device_time_ms = (C.t_end_ns > C.t_start_ns) ? (C.t_end_ns - C.t_start_ns) * 1e-6 : 0.0;
        r.wall_time_ms = ms;  // launch time; prrtc_plan overwrites with the host wall clock
        r.iterations_total = C.iters_used;
        r.sphere_tests = C.sphere_tests;
        r.fk_calls = C.fk_calls;
        r.fine_stage_entries = C.fine_entries;
        r.flops = C.flops;
        r.tree_nodes[0] = (uint64_t)std::max(0, C.published[0]);
        r.tree_nodes[1] = (uint64_t)std::max(0, C.published[1]);
        r.solving_worker = C.winner - 1;
        if (b->params.validate_path && r.status == PRRTC_SOLVED) r.path_check = C.path_bad ? 2 : 1;
    }
    if (pb) {  // the block lives until the last of its paths is freed
        if (block_refs > 0) pb->refs.store(block_refs, std::memory_order_release);
        else path_block_release(block_id);
    }
    return PRRTC_OK;
}

}  // namespace

extern "C" {

int prrtc_batch_create(const prrtc_robot* robot, const prrtc_scene* const* scenes,
                       uint32_t n_problems, const double* starts, const double* goals,
                       uint32_t dof, const prrtc_params* params, prrtc_batch** out) {
    if (!out) return set_err(PRRTC_EINVAL, "prrtc_batch_create: null argument");
    auto* b = new prrtc_batch();
    int rc = batch_setup(b, robot, scenes, n_problems, starts, goals, dof, params);
    if (!rc) rc = batch_bind(b, &b->own, scenes, starts, goals);
    if (!rc) {  // inputs uploaded once
        cudaSetDevice(b->device);
        if (cudaMemcpy(b->own.d_in, b->own.h_io, io_used(b), cudaMemcpyHostToDevice) != cudaSuccess)
            rc = set_err(PRRTC_ECUDA, "prrtc_batch_create: input upload failed");
    }
    if (rc) {
        delete b;
        return rc;
    }
    *out = b;
    return PRRTC_OK;
}

int prrtc_batch_launch(prrtc_batch* b, void* stream) {
    if (!b) return set_err(PRRTC_EINVAL, "prrtc_batch_launch: null batch");
    // a scene updated since the batch staged it (prrtc_scene_update may have
    // moved its buffers or changed its per-kind counts, i.e. the FP64 section
    // offsets): re-stage the scene table before launching
    bool stale = false;
    for (size_t i = 0; i < b->scenes.size() && !stale; ++i)
        stale = b->scenes[i]->generation.load(std::memory_order_acquire) != b->scene_gen[i];
    if (stale) {
        cudaSetDevice(b->device);
        // the previous launch (if any) must not see the table change under it
        if (b->last_stream && cudaStreamSynchronize(b->last_stream) != cudaSuccess)
            return set_err(PRRTC_ECUDA, "prrtc_batch_launch: sync before re-staging failed");
        const std::vector<const prrtc_scene*> sc = b->scenes;
        int rc = batch_bind(b, &b->own, sc.data(), nullptr, nullptr);
        if (rc) return rc;
        if (cudaMemcpy(b->own.d_in, b->own.h_io, io_used(b), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess)
            return set_err(PRRTC_ECUDA, "prrtc_batch_launch: scene re-staging failed");
    }
    return batch_enqueue(b, reinterpret_cast<cudaStream_t>(stream), false);
}

int prrtc_batch_launch_count(const prrtc_batch* b) { return b ? b->launches : 0; }

int prrtc_batch_results(prrtc_batch* b, prrtc_result* out) {
    if (!b || !out) return set_err(PRRTC_EINVAL, "prrtc_batch_results: null argument");
    return batch_collect(b, out);
}

int prrtc_batch_destroy(prrtc_batch* b) {
    delete b;
    return PRRTC_OK;
}

// Host-buffer entry point (the e2e path): packed H2D, kernel, D2H on the
// device's cached workspace.
namespace {
// Sound mode (params.validate_path): a problem whose path fails the device's
// 4 x n_cc re-validation is planned again with the next seed,
// up to kSoundRetries times; a problem that never yields a sound path is
// reported Failed. Planning at n_cc resolution (the reference's semantics)
// can return an edge whose collision lies between two of its 32 samples;
// this mode never returns one.
constexpr int kSoundRetries = 4;
constexpr uint64_t kRetrySeedStride = 1ull << 28;
int plan_batch_once(const prrtc_robot* robot, const prrtc_scene* const* scenes, uint32_t n_problems,
                    const double* starts, const double* goals, uint32_t dof, const prrtc_params* params,
                    prrtc_result* out);
}  // namespace

int prrtc_plan_batch(const prrtc_robot* robot, const prrtc_scene* const* scenes,
                     uint32_t n_problems, const double* starts, const double* goals,
                     uint32_t dof, const prrtc_params* params, prrtc_result* out) {
    const auto t0 = std::chrono::steady_clock::now();
    int rc = plan_batch_once(robot, scenes, n_problems, starts, goals, dof, params, out);
    if (rc || !params->validate_path) return rc;
    prrtc_params p = *params;
    for (int attempt = 0; attempt < kSoundRetries; ++attempt) {
        std::vector<uint32_t> bad;
        for (uint32_t i = 0; i < n_problems; ++i)
            if (out[i].status == PRRTC_SOLVED && out[i].path_check == 2) bad.push_back(i);
        if (bad.empty()) break;
        std::vector<const prrtc_scene*> sc;
        std::vector<double> s, g;
        for (uint32_t i : bad) {
            sc.push_back(scenes[i]);
            s.insert(s.end(), starts + (size_t)i * dof, starts + (size_t)(i + 1) * dof);
            g.insert(g.end(), goals + (size_t)i * dof, goals + (size_t)(i + 1) * dof);
        }
        // a different sample set per attempt: the seed offsets the Halton
        // index (1 + seed + ticket), so +1 would replay the same sequence
        // shifted by one sample; a 2^28 stride keeps indices below 2^32
        p.seed += kRetrySeedStride;
        std::vector<prrtc_result> re(bad.size());
        rc = plan_batch_once(robot, sc.data(), (uint32_t)bad.size(), s.data(), g.data(), dof, &p, re.data());
        if (rc) return rc;
        for (size_t k = 0; k < bad.size(); ++k) {
            prrtc_result& o = out[bad[k]];
            const uint64_t iters = o.iterations_total, tests = o.sphere_tests, fk = o.fk_calls,
                           fine = o.fine_stage_entries, flops = o.flops;
            prrtc_result_free(&o);
            o = re[k];  // takes ownership of the new path
            o.iterations_total += iters;
            o.sphere_tests += tests;
            o.fk_calls += fk;
            o.fine_stage_entries += fine;
            o.flops += flops;
        }
    }
    for (uint32_t i = 0; i < n_problems; ++i)
        if (out[i].status == PRRTC_SOLVED && out[i].path_check == 2) {
            prrtc_result_free(&out[i]);
            out[i].status = PRRTC_FAILED;
            std::snprintf(out[i].message, sizeof(out[i].message), "no path passed the 4 x n_cc re-validation");
        }
    if (n_problems == 1)
        out[0].wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return PRRTC_OK;
}

namespace {
int plan_batch_once(const prrtc_robot* robot, const prrtc_scene* const* scenes, uint32_t n_problems,
                    const double* starts, const double* goals, uint32_t dof, const prrtc_params* params,
                    prrtc_result* out) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!out) return set_err(PRRTC_EINVAL, "plan: null result");
    prrtc_batch b;
    int rc = batch_setup(&b, robot, scenes, n_problems, starts, goals, dof, params);
    if (rc) return rc;
    if (b.device < 0 || b.device >= 64) return set_err(PRRTC_ENODEV, "device ordinal out of range");
    std::lock_guard<std::mutex> lk(g_ws_mu[b.device]);
    Workspace& ws = g_ws[b.device];
    // a single problem reports the host wall clock: no kernel events
    const EnvKnobs& ek = env();
    b.timed = n_problems > 1 || ek.trace || ek.host_trace;
    // a single problem's result is published by the kernel into mapped host
    // memory (no D2H, no wait for the grid to retire); path re-validation runs
    // a second kernel after the planner, so it keeps the copy-back
    b.use_map = n_problems == 1 && !params->validate_path && !ek.trace && !ek.no_map;
    const auto t1 = std::chrono::steady_clock::now();
    rc = batch_bind(&b, &ws, scenes, starts, goals);
    const auto t2 = std::chrono::steady_clock::now();
    if (!rc) rc = batch_enqueue(&b, ws.stream, true);
    const auto t3 = std::chrono::steady_clock::now();
    if (!rc) rc = batch_collect(&b, out);
    if (rc) return rc;
    const auto t4 = std::chrono::steady_clock::now();
    const double wall = std::chrono::duration<double, std::milli>(t4 - t0).count();
    if (ek.host_trace) {
        auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
        float ev = 0.f;
        cudaEventElapsedTime(&ev, ws.ev0, ws.ev1);
        std::fprintf(stderr,
                     "prrtc host: setup %.1f bind %.1f enqueue %.1f wait+d2h %.1f fill %.1f us | kernel %.1f problem %.1f us\n",
                     us(t0, t1), us(t1, t2), us(t2, t3), us(t3, g_sync_time), us(g_sync_time, t4), ev * 1e3,
                     out[0].device_time_ms * 1e3);
    }
    if (n_problems == 1) out[0].wall_time_ms = wall;
    if (ek.trace) std::fprintf(stderr, "prrtc trace: host wall %.3f ms\n", wall);
    return PRRTC_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// multi-device batches: a host thread per device, a shared
// chunk queue, no collective
// ---------------------------------------------------------------------------
}  // extern "C"
namespace {
uint32_t auto_chunk(uint32_t n, uint32_t n_dev) {
    const uint32_t c = (n + 4 * n_dev - 1) / (4 * n_dev);
    return std::max<uint32_t>(64, c);
}

// Runs `work(worker, begin, count)` for consecutive chunks handed out by one
// atomic counter to n_workers threads (thread 0 is the caller); stops handing
// out chunks once some work returns nonzero and returns the first such code.
template <class F>
int run_chunk_queue(uint32_t n_workers, uint32_t n, uint32_t chunk, F work) {
    std::atomic<uint32_t> next{0};
    std::atomic<int> err{0};
    auto loop = [&](uint32_t w) {
        for (;;) {
            if (err.load(std::memory_order_relaxed)) return;
            const uint32_t b = next.fetch_add(chunk, std::memory_order_relaxed);
            if (b >= n) return;
            const int rc = work(w, b, std::min(chunk, n - b));
            if (rc) {
                int z = 0;
                err.compare_exchange_strong(z, rc);
                return;
            }
        }
    };
    std::vector<std::thread> th;
    for (uint32_t w = 1; w < n_workers; ++w) th.emplace_back(loop, w);
    loop(0);
    for (auto& t : th) t.join();
    return err.load();
}
}  // namespace
extern "C" {

int prrtc_plan_batch_multi(const prrtc_robot* const* robots, const prrtc_scene* const* scenes,
                           uint32_t n_devices, uint32_t n_problems, const double* starts,
                           const double* goals, uint32_t dof, const prrtc_params* params,
                           uint32_t chunk, prrtc_result* out) {
    if (!robots || !scenes || !starts || !goals || !params || !out)
        return set_err(PRRTC_EINVAL, "prrtc_plan_batch_multi: null argument");
    if (n_devices == 0) return set_err(PRRTC_EINVAL, "prrtc_plan_batch_multi: no devices");
    if (n_problems == 0) return set_err(PRRTC_EINVAL, "plan: empty batch");
    for (uint32_t d = 0; d < n_devices; ++d) {
        if (!robots[d]) return set_err(PRRTC_EINVAL, "prrtc_plan_batch_multi: null robot");
        if ((int)dof != robots[d]->dof)
            return set_err(PRRTC_EINVAL, "plan.start: expected dimension " + std::to_string(robots[d]->dof) +
                                             ", got " + std::to_string(dof));
        for (uint32_t e = 0; e < d; ++e)
            if (robots[e]->device == robots[d]->device)
                return set_err(PRRTC_EINVAL, "prrtc_plan_batch_multi: two entries on the same device");
        for (uint32_t i = 0; i < n_problems; ++i) {
            const prrtc_scene* sc = scenes[(size_t)d * n_problems + i];
            if (!sc || sc->device != robots[d]->device)
                return set_err(PRRTC_EINVAL, "plan: scene missing or on another device");
        }
    }
    int rc = check_params(params);
    if (rc) return rc;
    if (!chunk) chunk = auto_chunk(n_problems, n_devices);
    std::vector<std::string> errs(n_devices);
    rc = run_chunk_queue(n_devices, n_problems, chunk, [&](uint32_t d, uint32_t b, uint32_t cnt) {
        const int r = prrtc_plan_batch(robots[d], scenes + (size_t)d * n_problems + b, cnt,
                                       starts + (size_t)b * dof, goals + (size_t)b * dof, dof, params, out + b);
        if (r) errs[d] = g_err;  // thread-local message of the worker's thread
        return r;
    });
    if (rc) {
        for (const auto& e : errs)
            if (!e.empty()) return set_err(rc, e);
        return set_err(rc, "prrtc_plan_batch_multi failed");
    }
    return PRRTC_OK;
}

int prrtc_debug_chunk_queue(uint32_t n_workers, uint32_t n_problems, uint32_t chunk, const uint32_t* delay_us,
                            int32_t* owner, uint32_t* chunks_taken) {
    if (!owner || !chunks_taken || n_workers == 0) return set_err(PRRTC_EINVAL, "prrtc_debug_chunk_queue: bad argument");
    if (!chunk) chunk = auto_chunk(n_problems, n_workers);
    for (uint32_t i = 0; i < n_problems; ++i) owner[i] = -1;
    for (uint32_t w = 0; w < n_workers; ++w) chunks_taken[w] = 0;
    return run_chunk_queue(n_workers, n_problems, chunk, [&](uint32_t w, uint32_t b, uint32_t cnt) {
        for (uint32_t i = b; i < b + cnt; ++i) {
            if (owner[i] != -1) return PRRTC_EINVAL;  // handed out twice
            owner[i] = (int32_t)w;
        }
        ++chunks_taken[w];
        if (delay_us && delay_us[w]) std::this_thread::sleep_for(std::chrono::microseconds(delay_us[w] * cnt));
        return PRRTC_OK;
    });
}

int prrtc_debug_reload_env(void) {
    std::lock_guard<std::mutex> lk(g_env_mu);
    g_env.store(read_env(), std::memory_order_release);  // (the previous snapshot is leaked: readers may hold it)
    return PRRTC_OK;
}

int prrtc_last_transfer_bytes(int device, uint64_t* h2d, uint64_t* d2h) {
    if (device < 0 || device >= 64) return set_err(PRRTC_ENODEV, "device ordinal out of range");
    std::lock_guard<std::mutex> lk(g_ws_mu[device]);
    if (h2d) *h2d = g_ws[device].last_h2d;
    if (d2h) *d2h = g_ws[device].last_d2h;
    return PRRTC_OK;
}

int prrtc_plan(const prrtc_robot* robot, const prrtc_scene* scene, const double* start,
               const double* goal, uint32_t dof, const prrtc_params* params, prrtc_result* result) {
    if (!scene) return set_err(PRRTC_EINVAL, "prrtc_plan: null scene");
    return prrtc_plan_batch(robot, &scene, 1, start, goal, dof, params, result);
}

void prrtc_result_free(prrtc_result* r) {
    if (r && r->path) {
        if (r->path_block) path_block_unref((int)r->path_block);  // a view into its batch's block
        else std::free(r->path);
        r->path = nullptr;
        r->path_len = 0;
        r->path_block = 0;
    }
}

void prrtc_results_free(prrtc_result* r, uint32_t n) {
    if (!r) return;
    for (uint32_t i = 0; i < n; ++i) prrtc_result_free(r + i);
}

int prrtc_results_pack_paths(const prrtc_result* r, uint32_t n, double* out, uint64_t* offsets) {
    if (!r || !offsets) return set_err(PRRTC_EINVAL, "prrtc_results_pack_paths: null argument");
    uint64_t o = 0;
    for (uint32_t i = 0; i < n; ++i) {
        offsets[i] = o;
        const uint64_t k = r[i].path ? (uint64_t)r[i].path_len * r[i].dof : 0;
        if (k && out) std::memcpy(out + o, r[i].path, 8 * k);
        o += k;
    }
    offsets[n] = o;
    return PRRTC_OK;
}

// ---------------------------------------------------------------------------
// batched collision checking + parity hooks
// ---------------------------------------------------------------------------
int prrtc_validate_edges(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                         const double* to, uint32_t n_edges, uint32_t dof, int32_t n_cc,
                         int two_stage, int early_exit, uint8_t* valid) {
    if (!robot || !scene || !valid || (n_edges && (!from || !to)))
        return set_err(PRRTC_EINVAL, "prrtc_validate_edges: null argument");
    if ((int)dof != robot->dof) return set_err(PRRTC_EINVAL, "validate_edge.from: expected dimension " + std::to_string(robot->dof));
    if (n_cc < 1) return set_err(PRRTC_EINVAL, "validate_edge: resolution_count must be >= 1");
    if (n_edges == 0) return PRRTC_OK;
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double *df = nullptr, *dt = nullptr;
    uint8_t* dv = nullptr;
    const size_t nb = sizeof(double) * n_edges * dof;
    if ((rc = dmalloc(&df, n_edges * dof)) || (rc = dmalloc(&dt, n_edges * dof)) || (rc = dmalloc(&dv, n_edges))) {
        cudaFree(df);
        cudaFree(dt);
        return rc;
    }
    cudaMemcpy(df, from, nb, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, to, nb, cudaMemcpyHostToDevice);
    cudaError_t e = launch_validate_edges(robot->args(), scene->args(), df, dt, (int)n_edges, n_cc,
                                          two_stage, early_exit, dv, 0);
    if (e == cudaSuccess) e = cudaMemcpy(valid, dv, n_edges, cudaMemcpyDeviceToHost);
    cudaFree(df);
    cudaFree(dt);
    cudaFree(dv);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_validate_edges: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_check_configs(const prrtc_robot* robot, const prrtc_scene* scene, const double* q,
                        uint32_t n, uint32_t dof, int two_stage, uint8_t* valid) {
    if (!robot || !scene || !valid || (n && !q)) return set_err(PRRTC_EINVAL, "prrtc_check_configs: null argument");
    if ((int)dof != robot->dof) return set_err(PRRTC_EINVAL, "check_config: expected dimension " + std::to_string(robot->dof));
    if (n == 0) return PRRTC_OK;
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double* dq = nullptr;
    uint8_t* dv = nullptr;
    if ((rc = dmalloc(&dq, (size_t)n * dof)) || (rc = dmalloc(&dv, n))) {
        cudaFree(dq);
        return rc;
    }
    cudaMemcpy(dq, q, sizeof(double) * n * dof, cudaMemcpyHostToDevice);
    cudaError_t e = launch_check_configs(robot->args(), scene->args(), dq, (int)n, two_stage, dv, 0);
    if (e == cudaSuccess) e = cudaMemcpy(valid, dv, n, cudaMemcpyDeviceToHost);
    cudaFree(dq);
    cudaFree(dv);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_check_configs: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_fk(const prrtc_robot* robot, const double* q, uint32_t n, uint32_t dof,
                   float* fine_out, float* coarse_out) {
    if (!robot || (n && !q)) return set_err(PRRTC_EINVAL, "prrtc_debug_fk: null argument");
    if ((int)dof != robot->dof) return set_err(PRRTC_EINVAL, "forward_kinematics: expected dimension " + std::to_string(robot->dof));
    if (n == 0) return PRRTC_OK;
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double* dq = nullptr;
    float *df = nullptr, *dc = nullptr;
    const size_t nf = (size_t)n * robot->n_fine * 3, nc = (size_t)n * robot->n_links * 3;
    if ((rc = dmalloc(&dq, (size_t)n * dof)) || (rc = dmalloc(&df, nf)) || (rc = dmalloc(&dc, nc))) {
        cudaFree(dq);
        cudaFree(df);
        return rc;
    }
    cudaMemcpy(dq, q, sizeof(double) * n * dof, cudaMemcpyHostToDevice);
    cudaError_t e = launch_debug_fk(robot->args(), dq, (int)n, df, dc, 0);
    if (e == cudaSuccess && fine_out) e = cudaMemcpy(fine_out, df, 4 * nf, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && coarse_out) e = cudaMemcpy(coarse_out, dc, 4 * nc, cudaMemcpyDeviceToHost);
    cudaFree(dq);
    cudaFree(df);
    cudaFree(dc);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_fk: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_check_edges(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                            const double* to, uint32_t n_edges, uint32_t dof, int32_t n_cc, int two_stage,
                            uint8_t* state_valid, float* fine_out) {
    if (!robot || !scene || !state_valid || (n_edges && (!from || !to)))
        return set_err(PRRTC_EINVAL, "prrtc_debug_check_edges: null argument");
    if ((int)dof != robot->dof) return set_err(PRRTC_EINVAL, "validate_edge.from: expected dimension " + std::to_string(robot->dof));
    if (n_cc < 1) return set_err(PRRTC_EINVAL, "validate_edge: resolution_count must be >= 1");
    if (scene->device != robot->device) return set_err(PRRTC_EINVAL, "scene on another device");
    if (n_edges == 0) return PRRTC_OK;
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double *df = nullptr, *dt = nullptr;
    uint8_t* dv = nullptr;
    float* dfo = nullptr;
    const size_t ns = (size_t)n_edges * n_cc, nf = fine_out ? ns * robot->n_fine * 3 : 0;
    if ((rc = dmalloc(&df, (size_t)n_edges * dof)) || (rc = dmalloc(&dt, (size_t)n_edges * dof)) ||
        (rc = dmalloc(&dv, ns)) || (fine_out && (rc = dmalloc(&dfo, nf)))) {
        cudaFree(df);
        cudaFree(dt);
        cudaFree(dv);
        return rc;
    }
    cudaMemcpy(df, from, 8 * (size_t)n_edges * dof, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, to, 8 * (size_t)n_edges * dof, cudaMemcpyHostToDevice);
    cudaError_t e = launch_debug_check_edges(robot->args(), scene->args(), df, dt, (int)n_edges, n_cc, two_stage, dv,
                                             dfo, 0);
    if (e == cudaSuccess) e = cudaMemcpy(state_valid, dv, ns, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && fine_out) e = cudaMemcpy(fine_out, dfo, 4 * nf, cudaMemcpyDeviceToHost);
    cudaFree(df);
    cudaFree(dt);
    cudaFree(dv);
    cudaFree(dfo);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_check_edges: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_sphere_hits(const prrtc_scene* scene, const float* centers, const double* radii,
                            uint32_t n, uint8_t* hits) {
    if (!scene || !hits || (n && (!centers || !radii))) return set_err(PRRTC_EINVAL, "prrtc_debug_sphere_hits: null argument");
    if (n == 0) return PRRTC_OK;
    int rc = check_device(scene->device);
    if (rc) return rc;
    cudaSetDevice(scene->device);
    const int P = scene->ns + scene->nb + scene->nc + scene->ny;
    float* dcn = nullptr;
    double* dr = nullptr;
    uint8_t* dh = nullptr;
    if ((rc = dmalloc(&dcn, (size_t)n * 3)) || (rc = dmalloc(&dr, n)) || (rc = dmalloc(&dh, (size_t)n * P))) {
        cudaFree(dcn);
        cudaFree(dr);
        return rc;
    }
    cudaMemcpy(dcn, centers, 12 * (size_t)n, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, radii, 8 * (size_t)n, cudaMemcpyHostToDevice);
    cudaError_t e = launch_debug_hits(scene->args(), dcn, dr, (int)n, P, dh, 0);
    if (e == cudaSuccess && P) e = cudaMemcpy(hits, dh, (size_t)n * P, cudaMemcpyDeviceToHost);
    cudaFree(dcn);
    cudaFree(dr);
    cudaFree(dh);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_sphere_hits: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_nn(const double* tree, uint32_t count, uint32_t dof, const double* q,
                   uint32_t n_queries, int device, uint32_t* index, double* sq_dist) {
    // the planner's scan, one query per pass
    return prrtc_debug_nn_multi(tree, count, dof, q, n_queries, 1, device, index, sq_dist);
}

int prrtc_debug_nn_multi(const double* tree, uint32_t count, uint32_t dof, const double* q,
                         uint32_t n_queries, uint32_t group, int device, uint32_t* index, double* sq_dist) {
    if (group > 32) return set_err(PRRTC_EINVAL, "prrtc_debug_nn_multi: group must be <= 32");
    if (!tree || !q || !index || !sq_dist) return set_err(PRRTC_EINVAL, "prrtc_debug_nn: null argument");
    if (count == 0) return set_err(PRRTC_EINVAL, "nearest_serial: empty tree snapshot");
    if (dof == 0 || dof > PRRTC_MAX_DOF) return set_err(PRRTC_EINVAL, "prrtc_debug_nn: bad dof");
    int rc = check_device(device);
    if (rc) return rc;
    cudaSetDevice(device);
    const long long cap = ((long long)count + 31) / 32 * 32;
    std::vector<double> soa((size_t)cap * dof, 0.0);  // the planner's SoA tree layout
    for (uint32_t i = 0; i < count; ++i)
        for (uint32_t d = 0; d < dof; ++d) soa[(size_t)d * cap + i] = tree[(size_t)i * dof + d];
    double *ds = nullptr, *dq = nullptr, *dd = nullptr;
    uint32_t* di = nullptr;
    if ((rc = dmalloc(&ds, soa.size())) || (rc = dmalloc(&dq, (size_t)n_queries * dof)) ||
        (rc = dmalloc(&dd, n_queries)) || (rc = dmalloc(&di, n_queries))) {
        cudaFree(ds);
        cudaFree(dq);
        cudaFree(dd);
        return rc;
    }
    cudaMemcpy(ds, soa.data(), 8 * soa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dq, q, 8 * (size_t)n_queries * dof, cudaMemcpyHostToDevice);
    cudaError_t e = launch_debug_nn_multi(ds, cap, (int)count, (int)dof, dq, (int)n_queries, (int)std::max(1u, group),
                                          di, dd, 0);
    if (e == cudaSuccess) e = cudaMemcpy(index, di, 4 * (size_t)n_queries, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(sq_dist, dd, 8 * (size_t)n_queries, cudaMemcpyDeviceToHost);
    cudaFree(ds);
    cudaFree(dq);
    cudaFree(dd);
    cudaFree(di);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_nn: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_halton(const uint32_t* bases, const uint64_t* indices, uint32_t n, int device,
                       double* out) {
    if (!bases || !indices || !out) return set_err(PRRTC_EINVAL, "prrtc_debug_halton: null argument");
    for (uint32_t i = 0; i < n; ++i)
        if (bases[i] < 2) return set_err(PRRTC_EINVAL, "halton_value: base must be >= 2");
    if (n == 0) return PRRTC_OK;
    int rc = check_device(device);
    if (rc) return rc;
    cudaSetDevice(device);
    uint32_t* db = nullptr;
    uint64_t* di = nullptr;
    double* dout = nullptr;
    if ((rc = dmalloc(&db, n)) || (rc = dmalloc(&di, n)) || (rc = dmalloc(&dout, n))) {
        cudaFree(db);
        cudaFree(di);
        return rc;
    }
    cudaMemcpy(db, bases, 4 * (size_t)n, cudaMemcpyHostToDevice);
    cudaMemcpy(di, indices, 8 * (size_t)n, cudaMemcpyHostToDevice);
    cudaError_t e = launch_debug_halton(db, di, (int)n, dout, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, 8 * (size_t)n, cudaMemcpyDeviceToHost);
    cudaFree(db);
    cudaFree(di);
    cudaFree(dout);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_halton: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_chunk_profile(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                              const double* to, uint32_t dof, int32_t n_cc, int two_stage,
                              long long* stamps) {
    if (!robot || !scene || !from || !to || !stamps) return set_err(PRRTC_EINVAL, "prrtc_debug_chunk_profile: null argument");
    if ((int)dof != robot->dof) return set_err(PRRTC_EINVAL, "prrtc_debug_chunk_profile: dimension");
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double *df = nullptr, *dt = nullptr;
    uint8_t* dv = nullptr;
    long long* dp = nullptr;
    if ((rc = dmalloc(&df, dof)) || (rc = dmalloc(&dt, dof)) || (rc = dmalloc(&dv, 1)) || (rc = dmalloc(&dp, 16))) {
        cudaFree(df);
        cudaFree(dt);
        cudaFree(dv);
        return rc;
    }
    cudaMemcpy(df, from, 8 * dof, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, to, 8 * dof, cudaMemcpyHostToDevice);
    cudaMemset(dp, 0, 16 * 8);
    cudaError_t e = launch_validate_edges(robot->args(), scene->args(), df, dt, 1, n_cc, two_stage, 1, dv, 0, dp);
    if (e == cudaSuccess) e = cudaMemcpy(stamps, dp, 16 * 8, cudaMemcpyDeviceToHost);
    cudaFree(df);
    cudaFree(dt);
    cudaFree(dv);
    cudaFree(dp);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_chunk_profile: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

double prrtc_fp32_peak_tflops(int device) {
    if (check_device(device)) return 0.0;
    cudaSetDevice(device);
    return measure_fp32_peak(sm_count(device), 0);
}

double prrtc_fp64_peak_tflops(int device) {
    if (check_device(device)) return 0.0;
    cudaSetDevice(device);
    return measure_fp64_peak(sm_count(device), 0);
}

double prrtc_l2_peak_gbs(int device) {
    if (check_device(device)) return 0.0;
    cudaSetDevice(device);
    return measure_l2_gbs(sm_count(device), 0);
}

}  // extern "C"

namespace {
// mean ms per launch of `launch` over `reps` launches after one warm-up (CUDA events, stream 0)
template <class F>
cudaError_t time_launches(F launch, int reps, double* ms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t e = launch();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaEventRecord(e0, 0);
    for (int r = 0; r < reps && e == cudaSuccess; ++r) e = launch();
    if (e == cudaSuccess) e = cudaEventRecord(e1, 0);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, e0, e1);
    *ms = t / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return e;
}
}  // namespace

extern "C" {

int prrtc_bench_validate_edges(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                               const double* to, uint32_t n_edges, uint32_t dof, int32_t n_cc, int two_stage,
                               int early_exit, int reps, double* ms, double* flops, double* tests) {
    if (!robot || !scene || !from || !to || !ms || n_edges == 0 || reps < 1)
        return set_err(PRRTC_EINVAL, "prrtc_bench_validate_edges: bad argument");
    if ((int)dof != robot->dof) return set_err(PRRTC_EINVAL, "prrtc_bench_validate_edges: dimension");
    if (n_cc < 1) return set_err(PRRTC_EINVAL, "validate_edge: resolution_count must be >= 1");
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double *df = nullptr, *dt = nullptr;
    uint8_t* dv = nullptr;
    unsigned long long* dc = nullptr;
    if ((rc = dmalloc(&df, (size_t)n_edges * dof)) || (rc = dmalloc(&dt, (size_t)n_edges * dof)) ||
        (rc = dmalloc(&dv, n_edges)) || (rc = dmalloc(&dc, 2))) {
        cudaFree(df);
        cudaFree(dt);
        cudaFree(dv);
        return rc;
    }
    cudaMemcpy(df, from, 8 * (size_t)n_edges * dof, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, to, 8 * (size_t)n_edges * dof, cudaMemcpyHostToDevice);
    const RobotArgs ra = robot->args();
    const SceneArgs sa = scene->args();
    cudaError_t e = time_launches(
        [&] { return launch_validate_edges(ra, sa, df, dt, (int)n_edges, n_cc, two_stage, early_exit, dv, 0); },
        reps, ms);
    unsigned long long cnt[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemset(dc, 0, 16);  // one counted launch (outside the timing)
    if (e == cudaSuccess)
        e = launch_validate_edges(ra, sa, df, dt, (int)n_edges, n_cc, two_stage, early_exit, dv, 0, nullptr, dc);
    if (e == cudaSuccess) e = cudaMemcpy(cnt, dc, 16, cudaMemcpyDeviceToHost);
    cudaFree(df);
    cudaFree(dt);
    cudaFree(dv);
    cudaFree(dc);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_bench_validate_edges: ") + cudaGetErrorString(e));
    if (tests) *tests = (double)cnt[0];
    if (flops) *flops = (double)cnt[1];
    return PRRTC_OK;
}

int prrtc_bench_nn(const double* tree, uint32_t count, uint32_t dof, const double* q, uint32_t n_queries,
                   uint32_t group, int device, int reps, double* ms) {
    if (!tree || !q || !ms || count == 0 || n_queries == 0 || reps < 1 || group < 1 || group > 32)
        return set_err(PRRTC_EINVAL, "prrtc_bench_nn: bad argument");
    if (dof == 0 || dof > PRRTC_MAX_DOF) return set_err(PRRTC_EINVAL, "prrtc_bench_nn: bad dof");
    int rc = check_device(device);
    if (rc) return rc;
    cudaSetDevice(device);
    const long long cap = ((long long)count + 31) / 32 * 32;
    std::vector<double> soa((size_t)cap * dof, 0.0);  // the planner's SoA tree layout
    for (uint32_t i = 0; i < count; ++i)
        for (uint32_t d = 0; d < dof; ++d) soa[(size_t)d * cap + i] = tree[(size_t)i * dof + d];
    double *ds = nullptr, *dq = nullptr, *dd = nullptr;
    uint32_t* di = nullptr;
    if ((rc = dmalloc(&ds, soa.size())) || (rc = dmalloc(&dq, (size_t)n_queries * dof)) ||
        (rc = dmalloc(&dd, n_queries)) || (rc = dmalloc(&di, n_queries))) {
        cudaFree(ds);
        cudaFree(dq);
        cudaFree(dd);
        return rc;
    }
    cudaMemcpy(ds, soa.data(), 8 * soa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dq, q, 8 * (size_t)n_queries * dof, cudaMemcpyHostToDevice);
    cudaError_t e = time_launches(
        [&] { return launch_debug_nn_multi(ds, cap, (int)count, (int)dof, dq, (int)n_queries, (int)group, di, dd, 0); },
        reps, ms);
    cudaFree(ds);
    cudaFree(dq);
    cudaFree(dd);
    cudaFree(di);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_bench_nn: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

int prrtc_debug_sample(const prrtc_robot* robot, uint64_t index0, uint32_t n, double* out) {
    if (!robot || !out) return set_err(PRRTC_EINVAL, "prrtc_debug_sample: null argument");
    if (n == 0) return PRRTC_OK;
    int rc = check_device(robot->device);
    if (rc) return rc;
    cudaSetDevice(robot->device);
    double* dout = nullptr;
    if ((rc = dmalloc(&dout, (size_t)n * robot->dof))) return rc;
    cudaError_t e = launch_debug_sample(robot->args(), index0, (int)n, dout, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, 8 * (size_t)n * robot->dof, cudaMemcpyDeviceToHost);
    cudaFree(dout);
    if (e != cudaSuccess) return set_err(PRRTC_ECUDA, std::string("prrtc_debug_sample: ") + cudaGetErrorString(e));
    return PRRTC_OK;
}

}  // extern "C"
