/*
 * oracle/prrtc_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's planning hot path
 * (/root/reference/proj), used as the checker when the compiled reference
 * (oracle/_ref) is not available. Every function cites the reference
 * file:line it restates; arithmetic follows the reference's scalar operation
 * order exactly and the file is compiled with -ffp-contract=off, so results
 * are bit-identical to the reference built the same way with the scalar
 * backend forced (kernels.hpp:107-110). Pinned by tests/test_oracle_port.py
 * against oracle/_ref and the golden fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.
 */
#define _GNU_SOURCE
#include <math.h>
#include <unistd.h>
#include <pthread.h>
#include <sched.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "prrtc_b200.h"

static _Thread_local char g_err[256];

int orc_last_error(char* buf, size_t len) {
    if (buf && len) snprintf(buf, len, "%s", g_err);
    return 0;
}

/* ---------------- math core (transform.hpp) ---------------- */
typedef struct { double x, y, z; } V3;
typedef struct { double m[9]; } M3;
typedef struct { M3 r; V3 t; } TF;

static M3 m3_id(void) { M3 a = {{1, 0, 0, 0, 1, 0, 0, 0, 1}}; return a; }
/* Mat3::apply (transform.hpp:28-32) */
static V3 m3_apply(const M3* a, V3 v) {
    V3 o = {a->m[0] * v.x + a->m[1] * v.y + a->m[2] * v.z,
            a->m[3] * v.x + a->m[4] * v.y + a->m[5] * v.z,
            a->m[6] * v.x + a->m[7] * v.y + a->m[8] * v.z};
    return o;
}
/* Mat3::operator* (transform.hpp:33-44) */
static M3 m3_mul(const M3* a, const M3* b) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[i * 3 + j] = a->m[i * 3 + 0] * b->m[0 * 3 + j] + a->m[i * 3 + 1] * b->m[1 * 3 + j] +
                             a->m[i * 3 + 2] * b->m[2 * 3 + j];
    return r;
}
static M3 m3_T(const M3* a) {
    M3 r = {{a->m[0], a->m[3], a->m[6], a->m[1], a->m[4], a->m[7], a->m[2], a->m[5], a->m[8]}};
    return r;
}
/* Mat3::axis_angle (transform.hpp:56-66) */
static M3 axis_angle(V3 axis, double angle) {
    const double c = cos(angle), s = sin(angle), t = 1.0 - c;
    const double ax = axis.x, ay = axis.y, az = axis.z;
    M3 r = {{t * ax * ax + c, t * ax * ay - s * az, t * ax * az + s * ay,
             t * ax * ay + s * az, t * ay * ay + c, t * ay * az - s * ax,
             t * ax * az - s * ay, t * ay * az + s * ax, t * az * az + c}};
    return r;
}
/* Transform::apply / operator* (transform.hpp:77-80) */
static V3 tf_apply(const TF* a, V3 p) {
    V3 v = m3_apply(&a->r, p);
    V3 o = {v.x + a->t.x, v.y + a->t.y, v.z + a->t.z};
    return o;
}
static TF tf_mul(const TF* a, const TF* b) {
    TF o;
    o.r = m3_mul(&a->r, &b->r);
    o.t = tf_apply(a, b->t);
    return o;
}
/* Quat::to_mat3 (transform.hpp:97-103) */
static M3 quat_mat(const double* q) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    M3 r = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
             2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
             2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    return r;
}
static double v3_norm(V3 v) { return sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }

/* ---------------- robot (robot.hpp, kinematics.cpp) ---------------- */
typedef struct {
    int L, dof, S, NP;
    int* kind;
    int* parent;
    int* qidx;
    TF* origin;
    V3* axis;
    double* lo;
    double* hi;
    V3* cc;
    double* cr;
    int* foff;     /* [L+1] */
    V3* fc;
    double* fr;
    int* pairs;    /* [NP*2] */
} Robot;

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

void orc_robot_destroy(void* p) {
    Robot* r = (Robot*)p;
    if (!r) return;
    free(r->kind); free(r->parent); free(r->qidx); free(r->origin); free(r->axis);
    free(r->lo); free(r->hi); free(r->cc); free(r->cr); free(r->foff); free(r->fc);
    free(r->fr); free(r->pairs); free(r);
}

/* RobotModel::finalize (kinematics.cpp:15-74) */
void* orc_robot_create(const prrtc_robot_desc* d) {
    const int n = (int)d->n_links;
    if (n == 0) { fail("robot: joints must be non-empty"); return NULL; }
    Robot* r = (Robot*)calloc(1, sizeof(Robot));
    r->L = n;
    r->kind = malloc(sizeof(int) * n); r->parent = malloc(sizeof(int) * n);
    r->qidx = malloc(sizeof(int) * n); r->origin = malloc(sizeof(TF) * n);
    r->axis = malloc(sizeof(V3) * n); r->lo = malloc(sizeof(double) * n);
    r->hi = malloc(sizeof(double) * n); r->cc = malloc(sizeof(V3) * n);
    r->cr = malloc(sizeof(double) * n); r->foff = malloc(sizeof(int) * (n + 1));
    const int S = (int)d->fine_offset[n];
    r->S = S;
    r->fc = malloc(sizeof(V3) * (S ? S : 1)); r->fr = malloc(sizeof(double) * (S ? S : 1));
    r->NP = (int)d->n_self_pairs;
    r->pairs = malloc(sizeof(int) * 2 * (r->NP ? r->NP : 1));
    int dof = 0;
    for (int i = 0; i < n; ++i) {
        r->kind[i] = d->kind[i];
        r->parent[i] = d->parent[i];
        if (d->parent[i] >= i) { fail("robot joints: parent must be smaller than the joint index"); goto bad; }
        if (d->parent[i] < -1) { fail("robot joints: parent out of range"); goto bad; }
        const double* q = d->origin_quat + 4 * i;
        const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (fabs(qn - 1.0) > 1e-6) { fail("robot joints: origin.quaternion norm deviates from 1 by more than 1e-6"); goto bad; }
        r->origin[i].r = quat_mat(q);
        r->origin[i].t = (V3){d->origin_xyz[3 * i], d->origin_xyz[3 * i + 1], d->origin_xyz[3 * i + 2]};
        r->axis[i] = (V3){d->axis[3 * i], d->axis[3 * i + 1], d->axis[3 * i + 2]};
        r->lo[i] = d->lo[i];
        r->hi[i] = d->hi[i];
        r->qidx[i] = -1;
        if (d->kind[i] != PRRTC_JOINT_FIXED) {
            if (fabs(v3_norm(r->axis[i]) - 1.0) > 1e-9) { fail("robot joints: axis must be unit length"); goto bad; }
            if (!(d->lo[i] <= d->hi[i])) { fail("robot joints: limits lo must be <= hi"); goto bad; }
            r->qidx[i] = dof++;
        }
    }
    r->dof = dof;
    for (int l = 0; l <= n; ++l) r->foff[l] = (int)d->fine_offset[l];
    for (int l = 0; l < n; ++l) {
        r->cc[l] = (V3){d->coarse[4 * l], d->coarse[4 * l + 1], d->coarse[4 * l + 2]};
        r->cr[l] = d->coarse[4 * l + 3];
        if (!(r->cr[l] > 0.0)) { fail("robot spheres: coarse.radius must be positive"); goto bad; }
        for (int k = r->foff[l]; k < r->foff[l + 1]; ++k) {
            r->fc[k] = (V3){d->fine[4 * k], d->fine[4 * k + 1], d->fine[4 * k + 2]};
            r->fr[k] = d->fine[4 * k + 3];
            if (!(r->fr[k] > 0.0)) { fail("robot spheres: fine radius must be positive"); goto bad; }
            V3 dv = {r->fc[k].x - r->cc[l].x, r->fc[k].y - r->cc[l].y, r->fc[k].z - r->cc[l].z};
            if (v3_norm(dv) + r->fr[k] > r->cr[l] + 1e-9) { fail("robot spheres: fine sphere escapes the coarse bounding sphere"); goto bad; }
        }
    }
    for (int p = 0; p < r->NP; ++p) {
        const int a = d->self_pairs[2 * p], b = d->self_pairs[2 * p + 1];
        if (a < 0 || b < 0 || a >= n || b >= n) { fail("robot self_pairs: link index out of range"); goto bad; }
        if (a == b) { fail("robot self_pairs: a link cannot pair with itself"); goto bad; }
        if (d->parent[a] == b || d->parent[b] == a) { fail("robot self_pairs: adjacent parent-child links must not be tested"); goto bad; }
        r->pairs[2 * p] = a;
        r->pairs[2 * p + 1] = b;
    }
    return r;
bad:
    orc_robot_destroy(r);
    return NULL;
}

int orc_robot_dof(void* r) { return ((Robot*)r)->dof; }

/* forward_kinematics (kinematics.cpp:78-103) */
static void fk(const Robot* r, const double* q, TF* out) {
    for (int i = 0; i < r->L; ++i) {
        const double qi = r->qidx[i] >= 0 ? q[r->qidx[i]] : 0.0;
        TF motion;
        if (r->kind[i] == PRRTC_JOINT_REVOLUTE) {
            motion.r = axis_angle(r->axis[i], qi);
            motion.t = (V3){0, 0, 0};
        } else if (r->kind[i] == PRRTC_JOINT_PRISMATIC) {
            motion.r = m3_id();
            motion.t = (V3){r->axis[i].x * qi, r->axis[i].y * qi, r->axis[i].z * qi};
        } else {
            motion.r = m3_id();
            motion.t = (V3){0, 0, 0};
        }
        const TF local = tf_mul(&r->origin[i], &motion);
        out[i] = r->parent[i] < 0 ? local : tf_mul(&out[r->parent[i]], &local);
    }
}

int orc_fk_poses(void* rp, const double* q, double* out) {
    const Robot* r = (const Robot*)rp;
    TF* P = malloc(sizeof(TF) * r->L);
    fk(r, q, P);
    for (int l = 0; l < r->L; ++l) {
        for (int k = 0; k < 9; ++k) out[12 * l + k] = P[l].r.m[k];
        out[12 * l + 9] = P[l].t.x;
        out[12 * l + 10] = P[l].t.y;
        out[12 * l + 11] = P[l].t.z;
    }
    free(P);
    return 0;
}

/* sphere_positions (kinematics.cpp:111-126) */
int orc_fk_spheres(void* rp, const double* q, int level, double* out) {
    const Robot* r = (const Robot*)rp;
    TF* P = malloc(sizeof(TF) * r->L);
    fk(r, q, P);
    int n = 0;
    for (int l = 0; l < r->L; ++l) {
        if (level == 0) {
            V3 c = tf_apply(&P[l], r->cc[l]);
            out[4 * n] = c.x; out[4 * n + 1] = c.y; out[4 * n + 2] = c.z; out[4 * n + 3] = r->cr[l];
            ++n;
        } else {
            for (int k = r->foff[l]; k < r->foff[l + 1]; ++k) {
                V3 c = tf_apply(&P[l], r->fc[k]);
                out[4 * n] = c.x; out[4 * n + 1] = c.y; out[4 * n + 2] = c.z; out[4 * n + 3] = r->fr[k];
                ++n;
            }
        }
    }
    free(P);
    return n;
}

/* ---------------- scene (geometry.hpp/.cpp) ---------------- */
typedef struct {
    int ns, nb, nc, ny;
    double* s;  /* [ns][4] */
    double* b;  /* [nb][15]: world->box rotation m[9], t[3], h[3] (SceneIndex) */
    double* c;  /* [nc][8]: a[3], ab[3], inv_ab2, r */
    double* y;  /* [ny][14]: world->cylinder rotation m[9], t[3], r, h — EXTENSION, no
                   reference counterpart (geometry.hpp:35); parity unpinned */
} SceneI;

void orc_scene_destroy(void* p) {
    SceneI* s = (SceneI*)p;
    if (!s) return;
    free(s->s); free(s->b); free(s->c); free(s->y); free(s);
}

/* Scene::validate (geometry.cpp:10-39) + SceneIndex (geometry.cpp:68-99) */
void* orc_scene_create(const prrtc_scene_desc* d) {
    SceneI* s = (SceneI*)calloc(1, sizeof(SceneI));
    s->ns = d->n_spheres; s->nb = d->n_boxes; s->nc = d->n_capsules;
    s->ny = d->cylinders ? (int)d->n_cylinders : 0;
    s->y = malloc(sizeof(double) * 14 * (s->ny + 1));
    for (int i = 0; i < s->ny; ++i) {
        const double* p = d->cylinders + 9 * i;
        if (!(p[7] > 0.0) || !(p[8] > 0.0)) { fail("scene cylinder radius and half_length must be positive"); orc_scene_destroy(s); return NULL; }
        const double qn = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2] + p[3] * p[3]);
        if (fabs(qn - 1.0) > 1e-6) { fail("scene cylinder pose.quaternion norm deviates from 1 by more than 1e-6"); orc_scene_destroy(s); return NULL; }
        M3 R = quat_mat(p);
        M3 rt = m3_T(&R);
        for (int k = 0; k < 9; ++k) s->y[14 * i + k] = rt.m[k];
        for (int k = 0; k < 3; ++k) s->y[14 * i + 9 + k] = p[4 + k];
        s->y[14 * i + 12] = p[7];
        s->y[14 * i + 13] = p[8];
    }
    s->s = malloc(sizeof(double) * 4 * (s->ns + 1));
    s->b = malloc(sizeof(double) * 15 * (s->nb + 1));
    s->c = malloc(sizeof(double) * 8 * (s->nc + 1));
    for (int i = 0; i < s->ns; ++i) {
        for (int k = 0; k < 4; ++k) s->s[4 * i + k] = d->spheres[4 * i + k];
        if (!(s->s[4 * i + 3] > 0.0)) { fail("scene primitive radius must be positive"); orc_scene_destroy(s); return NULL; }
    }
    for (int i = 0; i < s->nb; ++i) {
        const double* p = d->boxes + 10 * i;
        if (!(p[7] > 0.0 && p[8] > 0.0 && p[9] > 0.0)) { fail("scene box half_extents must be componentwise positive"); orc_scene_destroy(s); return NULL; }
        const double qn = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2] + p[3] * p[3]);
        if (fabs(qn - 1.0) > 1e-6) { fail("scene box pose.quaternion norm deviates from 1 by more than 1e-6"); orc_scene_destroy(s); return NULL; }
        M3 R = quat_mat(p);
        M3 rt = m3_T(&R);
        for (int k = 0; k < 9; ++k) s->b[15 * i + k] = rt.m[k];
        for (int k = 0; k < 3; ++k) {
            s->b[15 * i + 9 + k] = p[4 + k];
            s->b[15 * i + 12 + k] = p[7 + k];
        }
    }
    for (int i = 0; i < s->nc; ++i) {
        const double* p = d->capsules + 7 * i;
        if (!(p[6] > 0.0)) { fail("scene primitive radius must be positive"); orc_scene_destroy(s); return NULL; }
        const double abx = p[3] - p[0], aby = p[4] - p[1], abz = p[5] - p[2];
        const double ab2 = abx * abx + aby * aby + abz * abz;
        double* c = s->c + 8 * i;
        c[0] = p[0]; c[1] = p[1]; c[2] = p[2]; c[3] = abx; c[4] = aby; c[5] = abz;
        c[6] = ab2 > 0.0 ? 1.0 / ab2 : 0.0;
        c[7] = p[6];
    }
    return s;
}

/* ---------------- predicates (kernels_detail.hpp:11-58) ---------------- */
static double clamp01(double t) {
    if (t < 0.0) t = 0.0;
    if (t > 1.0) t = 1.0;
    return t;
}
static int sphere_sphere_hit(double px, double py, double pz, double pr, double sx, double sy,
                             double sz, double sr) {
    const double dx = px - sx, dy = py - sy, dz = pz - sz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double rr = pr + sr;
    return d2 < rr * rr;
}
static int sphere_capsule_hit(double px, double py, double pz, double pr, const double* c) {
    const double pax = px - c[0], pay = py - c[1], paz = pz - c[2];
    const double t = clamp01((pax * c[3] + pay * c[4] + paz * c[5]) * c[6]);
    const double dx = pax - t * c[3], dy = pay - t * c[4], dz = paz - t * c[5];
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double rr = pr + c[7];
    return d2 < rr * rr;
}
static int sphere_box_hit(double px, double py, double pz, double pr, const double* b) {
    const double* m = b;
    const double wx = px - b[9], wy = py - b[10], wz = pz - b[11];
    const double lx = m[0] * wx + m[1] * wy + m[2] * wz;
    const double ly = m[3] * wx + m[4] * wy + m[5] * wz;
    const double lz = m[6] * wx + m[7] * wy + m[8] * wz;
    const double hx = b[12], hy = b[13], hz = b[14];
    const double cx = lx < -hx ? -hx : (lx > hx ? hx : lx);
    const double cy = ly < -hy ? -hy : (ly > hy ? hy : ly);
    const double cz = lz < -hz ? -hz : (lz > hz ? hz : lz);
    const double dx = lx - cx, dy = ly - cy, dz = lz - cz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    return d2 < pr * pr;
}

/* Cylinder EXTENSION (the reference has none, geometry.hpp:35): solid
   cylinder about its local z axis; the same operation order as the device's
   sphere_cylinder_exact (paper_2503_06757_b200/csrc/prrtc_device.cuh). */
static int sphere_cylinder_hit(double px, double py, double pz, double pr, const double* y) {
    const double wx = px - y[9], wy = py - y[10], wz = pz - y[11];
    const double lx = y[0] * wx + y[1] * wy + y[2] * wz;
    const double ly = y[3] * wx + y[4] * wy + y[5] * wz;
    const double lz = y[6] * wx + y[7] * wy + y[8] * wz;
    const double rho = sqrt(lx * lx + ly * ly);
    double er = rho - y[12];
    if (er < 0.0) er = 0.0;
    double ez = fabs(lz) - y[13];
    if (ez < 0.0) ez = 0.0;
    const double d2 = er * er + ez * ez;
    return d2 < pr * pr;
}

/* sphere_vs_primitive (geometry.cpp:41-66), primitive order spheres, boxes,
   capsules (+ cylinders, extension) */
int orc_sphere_hits(void* sp, double x, double y, double z, double r, uint8_t* hits) {
    const SceneI* s = (const SceneI*)sp;
    int any = 0, k = 0;
    for (int i = 0; i < s->ns; ++i, ++k) {
        const double* p = s->s + 4 * i;
        hits[k] = (uint8_t)sphere_sphere_hit(x, y, z, r, p[0], p[1], p[2], p[3]);
        any |= hits[k];
    }
    for (int i = 0; i < s->nb; ++i, ++k) {
        hits[k] = (uint8_t)sphere_box_hit(x, y, z, r, s->b + 15 * i);
        any |= hits[k];
    }
    for (int i = 0; i < s->nc; ++i, ++k) {
        hits[k] = (uint8_t)sphere_capsule_hit(x, y, z, r, s->c + 8 * i);
        any |= hits[k];
    }
    for (int i = 0; i < s->ny; ++i, ++k) {
        hits[k] = (uint8_t)sphere_cylinder_hit(x, y, z, r, s->y + 14 * i);
        any |= hits[k];
    }
    return any;
}

int orc_force_scalar(int on) { (void)on; return 1; }

/* ---------------- collision checker (collision.cpp) ---------------- */
typedef struct {
    uint64_t tests, fk_calls, fine_entries;
} Stats;

typedef struct {
    const Robot* r;
    const SceneI* s;
    TF* poses;
    V3* cc;           /* posed coarse */
    V3* fp;           /* posed fine */
    char* fine_posed;
    uint8_t* flag;    /* [L][P]: flagged primitive per link (order spheres, capsules, boxes) */
    int* flagged_links;
    int* flagged_pairs;
    double* sample;
} Checker;

static void checker_init(Checker* c, const Robot* r, const SceneI* s) {
    c->r = r;
    c->s = s;
    c->poses = malloc(sizeof(TF) * r->L);
    c->cc = malloc(sizeof(V3) * r->L);
    c->fp = malloc(sizeof(V3) * (r->S + 1));
    c->fine_posed = malloc(r->L);
    c->flag = malloc((size_t)r->L * (s->ns + s->nb + s->nc + s->ny + 1));
    c->flagged_links = malloc(sizeof(int) * r->L);
    c->flagged_pairs = malloc(sizeof(int) * (r->NP + 1));
    c->sample = malloc(sizeof(double) * (r->dof + 1));
}
static void checker_free(Checker* c) {
    free(c->poses); free(c->cc); free(c->fp); free(c->fine_posed); free(c->flag);
    free(c->flagged_links); free(c->flagged_pairs); free(c->sample);
}

/* posed_fine (collision.cpp:49-65) */
static void posed_fine(Checker* c, int l) {
    if (c->fine_posed[l]) return;
    for (int k = c->r->foff[l]; k < c->r->foff[l + 1]; ++k) c->fp[k] = tf_apply(&c->poses[l], c->r->fc[k]);
    c->fine_posed[l] = 1;
}

/* fine_pair_collides (collision.cpp:89-98) */
static int fine_pair_collides(Checker* c, int li, int lj, Stats* st) {
    const Robot* r = c->r;
    posed_fine(c, li);
    posed_fine(c, lj);
    const int ni = r->foff[li + 1] - r->foff[li], nj = r->foff[lj + 1] - r->foff[lj];
    st->tests += (uint64_t)ni * nj;
    for (int s = r->foff[li]; s < r->foff[li + 1]; ++s)
        for (int k = r->foff[lj]; k < r->foff[lj + 1]; ++k)
            if (sphere_sphere_hit(c->fp[s].x, c->fp[s].y, c->fp[s].z, r->fr[s], c->fp[k].x, c->fp[k].y,
                                  c->fp[k].z, r->fr[k]))
                return 1;
    return 0;
}

/* check_config_brute (collision.cpp:100-128) */
static int check_brute(Checker* c, Stats* st, int early_exit) {
    const Robot* r = c->r;
    const SceneI* S = c->s;
    const int P = S->ns + S->nb + S->nc + S->ny;
    int colliding = 0;
    for (int l = 0; l < r->L && !(colliding && early_exit); ++l) {
        posed_fine(c, l);
        for (int k = r->foff[l]; k < r->foff[l + 1]; ++k) {
            st->tests += P;
            const V3 x = c->fp[k];
            int hit = 0;
            for (int i = 0; i < S->ns && !hit; ++i)
                hit = sphere_sphere_hit(S->s[4 * i], S->s[4 * i + 1], S->s[4 * i + 2], S->s[4 * i + 3], x.x, x.y, x.z, r->fr[k]);
            for (int i = 0; i < S->nc && !hit; ++i) hit = sphere_capsule_hit(x.x, x.y, x.z, r->fr[k], S->c + 8 * i);
            for (int i = 0; i < S->nb && !hit; ++i) hit = sphere_box_hit(x.x, x.y, x.z, r->fr[k], S->b + 15 * i);
            for (int i = 0; i < S->ny && !hit; ++i) hit = sphere_cylinder_hit(x.x, x.y, x.z, r->fr[k], S->y + 14 * i);
            if (hit) {
                colliding = 1;
                if (early_exit) break;
            }
        }
    }
    for (int p = 0; p < r->NP && !(colliding && early_exit); ++p)
        if (fine_pair_collides(c, r->pairs[2 * p], r->pairs[2 * p + 1], st)) colliding = 1;
    return !colliding;
}

/* CollisionChecker::check_config (collision.cpp:130-204) */
static int check_config(Checker* c, const double* q, Stats* st, int two_stage, int early_exit) {
    const Robot* r = c->r;
    const SceneI* S = c->s;
    fk(r, q, c->poses);
    st->fk_calls += 1;
    memset(c->fine_posed, 0, r->L);
    if (!two_stage) return check_brute(c, st, early_exit);
    const int P = S->ns + S->nb + S->nc + S->ny;
    for (int l = 0; l < r->L; ++l) c->cc[l] = tf_apply(&c->poses[l], r->cc[l]);
    int nfl = 0, nfp = 0;
    for (int l = 0; l < r->L; ++l) {
        uint8_t* f = c->flag + (size_t)l * (P + 1);
        int any = 0;
        st->tests += P;
        const V3 x = c->cc[l];
        /* stage 1 kernels record sphere, capsule, box flags (collision.cpp:155-176);
           sphere_vs_spheres(scene spheres, coarse): px = coarse, s = scene */
        for (int i = 0; i < S->ns; ++i) {
            f[i] = (uint8_t)sphere_sphere_hit(x.x, x.y, x.z, r->cr[l], S->s[4 * i], S->s[4 * i + 1], S->s[4 * i + 2], S->s[4 * i + 3]);
            any |= f[i];
        }
        for (int i = 0; i < S->nc; ++i) {
            f[S->ns + i] = (uint8_t)sphere_capsule_hit(x.x, x.y, x.z, r->cr[l], S->c + 8 * i);
            any |= f[S->ns + i];
        }
        for (int i = 0; i < S->nb; ++i) {
            f[S->ns + S->nc + i] = (uint8_t)sphere_box_hit(x.x, x.y, x.z, r->cr[l], S->b + 15 * i);
            any |= f[S->ns + S->nc + i];
        }
        for (int i = 0; i < S->ny; ++i) {  /* cylinder extension */
            f[S->ns + S->nc + S->nb + i] = (uint8_t)sphere_cylinder_hit(x.x, x.y, x.z, r->cr[l], S->y + 14 * i);
            any |= f[S->ns + S->nc + S->nb + i];
        }
        if (any) c->flagged_links[nfl++] = l;
    }
    for (int p = 0; p < r->NP; ++p) {
        const int a = r->pairs[2 * p], b = r->pairs[2 * p + 1];
        st->tests += 1;
        const double dx = c->cc[a].x - c->cc[b].x, dy = c->cc[a].y - c->cc[b].y, dz = c->cc[a].z - c->cc[b].z;
        const double rr = r->cr[a] + r->cr[b];
        if (dx * dx + dy * dy + dz * dz < rr * rr) c->flagged_pairs[nfp++] = p;
    }
    if (nfl == 0 && nfp == 0) return 1;
    st->fine_entries += 1;
    int colliding = 0;
    /* fine_link_vs_flagged (collision.cpp:67-87): spheres, then capsules, then boxes */
    for (int u = 0; u < nfl; ++u) {
        const int l = c->flagged_links[u];
        const uint8_t* f = c->flag + (size_t)l * (P + 1);
        posed_fine(c, l);
        const int n = r->foff[l + 1] - r->foff[l];
        int hit = 0;
        for (int i = 0; i < S->ns && !hit; ++i) {
            if (!f[i]) continue;
            st->tests += n;
            for (int k = r->foff[l]; k < r->foff[l + 1] && !hit; ++k)
                hit = sphere_sphere_hit(S->s[4 * i], S->s[4 * i + 1], S->s[4 * i + 2], S->s[4 * i + 3], c->fp[k].x, c->fp[k].y, c->fp[k].z, r->fr[k]);
        }
        for (int i = 0; i < S->nc && !hit; ++i) {
            if (!f[S->ns + i]) continue;
            st->tests += n;
            for (int k = r->foff[l]; k < r->foff[l + 1] && !hit; ++k)
                hit = sphere_capsule_hit(c->fp[k].x, c->fp[k].y, c->fp[k].z, r->fr[k], S->c + 8 * i);
        }
        for (int i = 0; i < S->nb && !hit; ++i) {
            if (!f[S->ns + S->nc + i]) continue;
            st->tests += n;
            for (int k = r->foff[l]; k < r->foff[l + 1] && !hit; ++k)
                hit = sphere_box_hit(c->fp[k].x, c->fp[k].y, c->fp[k].z, r->fr[k], S->b + 15 * i);
        }
        for (int i = 0; i < S->ny && !hit; ++i) {
            if (!f[S->ns + S->nc + S->nb + i]) continue;
            st->tests += n;
            for (int k = r->foff[l]; k < r->foff[l + 1] && !hit; ++k)
                hit = sphere_cylinder_hit(c->fp[k].x, c->fp[k].y, c->fp[k].z, r->fr[k], S->y + 14 * i);
        }
        if (hit) {
            colliding = 1;
            if (early_exit) return 0;
        }
    }
    for (int u = 0; u < nfp; ++u) {
        const int p = c->flagged_pairs[u];
        if (fine_pair_collides(c, r->pairs[2 * p], r->pairs[2 * p + 1], st)) {
            colliding = 1;
            if (early_exit) return 0;
        }
    }
    return !colliding;
}

/* lerp (kernels_scalar.cpp:18-22) */
static void lerp(const double* a, const double* b, double t, double* out, int n) {
    for (int i = 0; i < n; ++i) out[i] = a[i] + t * (b[i] - a[i]);
}
static int bitwise_equal(const double* a, const double* b, int n) {
    for (int i = 0; i < n; ++i)
        if (a[i] != b[i]) return 0;
    return 1;
}

/* edge_sample (collision.cpp:13-21) */
static void edge_sample(const double* from, const double* to, int i, int n, double* out, int dof) {
    if (i == n) memcpy(out, to, sizeof(double) * dof);
    else lerp(from, to, (double)i / n, out, dof);
}

/* validate_edge (collision.cpp:206-224) */
static int validate_edge(Checker* c, const double* from, const double* to, int n, Stats* st,
                         int two_stage, int early_exit) {
    const int dof = c->r->dof;
    if (bitwise_equal(from, to, dof)) return check_config(c, to, st, two_stage, early_exit);
    int ok = 1;
    for (int i = 1; i <= n; ++i) {
        edge_sample(from, to, i, n, c->sample, dof);
        if (!check_config(c, c->sample, st, two_stage, early_exit)) {
            ok = 0;
            if (early_exit) break;
        }
    }
    return ok;
}

static void put_stats(const Stats* s, uint64_t* out) {
    if (!out) return;
    out[0] = s->tests;
    out[1] = s->fk_calls;
    out[2] = s->fine_entries;
}

int orc_check_config(void* rp, void* sp, const double* q, int two_stage, int early_exit, uint64_t* stats) {
    Checker c;
    checker_init(&c, rp, sp);
    Stats st = {0, 0, 0};
    int ok = check_config(&c, q, &st, two_stage, early_exit);
    put_stats(&st, stats);
    checker_free(&c);
    return ok;
}

int orc_check_configs(void* rp, void* sp, const double* q, uint32_t n, int two_stage, uint8_t* out) {
    Checker c;
    checker_init(&c, rp, sp);
    Stats st = {0, 0, 0};
    const int dof = ((Robot*)rp)->dof;
    for (uint32_t i = 0; i < n; ++i) out[i] = (uint8_t)check_config(&c, q + (size_t)i * dof, &st, two_stage, 1);
    checker_free(&c);
    return 0;
}

int orc_validate_edge(void* rp, void* sp, const double* from, const double* to, int n, int two_stage,
                      int early_exit, uint64_t* stats) {
    if (n < 1) return fail("validate_edge: resolution_count must be >= 1");
    Checker c;
    checker_init(&c, rp, sp);
    Stats st = {0, 0, 0};
    int ok = validate_edge(&c, from, to, n, &st, two_stage, early_exit);
    put_stats(&st, stats);
    checker_free(&c);
    return ok;
}

int orc_validate_edges(void* rp, void* sp, const double* from, const double* to, uint32_t ne, int n,
                       int two_stage, int early_exit, uint8_t* out) {
    if (n < 1) return fail("validate_edge: resolution_count must be >= 1");
    Checker c;
    checker_init(&c, rp, sp);
    Stats st = {0, 0, 0};
    const int dof = ((Robot*)rp)->dof;
    for (uint32_t e = 0; e < ne; ++e)
        out[e] = (uint8_t)validate_edge(&c, from + (size_t)e * dof, to + (size_t)e * dof, n, &st, two_stage, early_exit);
    checker_free(&c);
    return 0;
}

/* validate_edge_batched (collision.cpp:226-262) */
int orc_validate_edge_batched(void* rp, void* sp, const double* from, const double* to, uint32_t ne,
                              int n, int two_stage, int early_exit, uint8_t* out, uint64_t* stats) {
    if (n < 1) return fail("validate_edge_batched: resolution_count must be >= 1");
    Checker c;
    checker_init(&c, rp, sp);
    Stats st = {0, 0, 0};
    const int dof = ((Robot*)rp)->dof;
    uint8_t* done = calloc(ne + 1, 1);
    int* counts = malloc(sizeof(int) * (ne + 1));
    int max_n = 0;
    for (uint32_t e = 0; e < ne; ++e) {
        out[e] = 1;
        counts[e] = bitwise_equal(from + (size_t)e * dof, to + (size_t)e * dof, dof) ? 1 : n;
        if (counts[e] > max_n) max_n = counts[e];
    }
    for (int i = 1; i <= max_n; ++i) {
        int open = 0;
        for (uint32_t e = 0; e < ne; ++e) {
            if (done[e] || i > counts[e]) continue;
            edge_sample(from + (size_t)e * dof, to + (size_t)e * dof, i, counts[e], c.sample, dof);
            if (!check_config(&c, c.sample, &st, two_stage, early_exit)) {
                out[e] = 0;
                if (early_exit) {
                    done[e] = 1;
                    continue;
                }
            }
            if (i < counts[e]) open = 1;
        }
        if (!open) break;
    }
    free(done);
    free(counts);
    put_stats(&st, stats);
    checker_free(&c);
    return 0;
}

/* ---------------- nearest neighbour (nn.cpp, kernels_scalar.cpp) ---------------- */
static double sq_distance(const double* a, const double* b, int n) {  /* kernels_scalar.cpp:9-16 */
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}
static uint64_t argmin_sq(const double* cfg, uint64_t count, int dof, const double* q, double* bd2) {
    uint64_t best = 0;  /* kernels_scalar.cpp:24-37 */
    double b = sq_distance(cfg, q, dof);
    for (uint64_t i = 1; i < count; ++i) {
        const double d2 = sq_distance(cfg + i * dof, q, dof);
        if (d2 < b) {
            b = d2;
            best = i;
        }
    }
    *bd2 = b;
    return best;
}

double orc_sq_distance(const double* a, const double* b, uint32_t dof) { return sq_distance(a, b, (int)dof); }

int64_t orc_nearest_serial(const double* cfg, uint64_t count, uint32_t dof, const double* q, double* dist) {
    if (count == 0) return fail("nearest_serial: empty tree snapshot");
    double d2;
    const uint64_t i = argmin_sq(cfg, count, (int)dof, q, &d2);
    if (dist) *dist = sqrt(d2);
    return (int64_t)i;
}

/* nearest_parallel (nn.cpp:31-69) */
int64_t orc_nearest_parallel(const double* cfg, uint64_t count, uint32_t dof, const double* q,
                             uint64_t partitions, double* dist) {
    if (count == 0) return fail("nearest_parallel: empty tree snapshot");
    if (partitions == 0) return fail("nearest_parallel: partitions must be >= 1");
    uint64_t lanes = 1;
    while (lanes < partitions) lanes <<= 1;
    double* ld = malloc(sizeof(double) * lanes);
    uint64_t* li = malloc(sizeof(uint64_t) * lanes);
    for (uint64_t l = 0; l < lanes; ++l) {
        ld[l] = INFINITY;
        li[l] = UINT64_MAX;
    }
    const uint64_t chunk = (count + partitions - 1) / partitions;
    for (uint64_t l = 0; l < partitions; ++l) {
        const uint64_t begin = l * chunk;
        if (begin >= count) break;
        const uint64_t len = chunk < count - begin ? chunk : count - begin;
        double d2;
        const uint64_t local = argmin_sq(cfg + begin * dof, len, (int)dof, q, &d2);
        ld[l] = d2;
        li[l] = begin + local;
    }
    for (uint64_t s = lanes / 2; s >= 1; s /= 2)
        for (uint64_t l = 0; l < s; ++l)
            if (ld[l + s] < ld[l] || (ld[l + s] == ld[l] && li[l + s] < li[l])) {
                ld[l] = ld[l + s];
                li[l] = li[l + s];
            }
    if (dist) *dist = sqrt(ld[0]);
    const int64_t r = (int64_t)li[0];
    free(ld);
    free(li);
    return r;
}

/* ---------------- sampling (sampling.cpp) ---------------- */
double orc_halton_value(unsigned base, uint64_t index) {  /* sampling.cpp:8-18 */
    double f = 1.0, r = 0.0;
    while (index > 0) {
        f /= base;
        r += f * (double)(index % base);
        index /= base;
    }
    return r;
}

int orc_halton_bases(uint32_t n, uint32_t* out) {  /* sampling.cpp:20-37 */
    uint32_t k = 0;
    for (unsigned c = 2; k < n; ++c) {
        int prime = 1;
        for (uint32_t j = 0; j < k; ++j) {
            if (out[j] * out[j] > c) break;
            if (c % out[j] == 0) {
                prime = 0;
                break;
            }
        }
        if (prime) out[k++] = c;
    }
    return 0;
}

static void limits_of(const Robot* r, double* lo, double* hi) {  /* robot.hpp:57-64 */
    int k = 0;
    for (int i = 0; i < r->L; ++i)
        if (r->kind[i] != PRRTC_JOINT_FIXED) {
            lo[k] = r->lo[i];
            hi[k] = r->hi[i];
            ++k;
        }
}

/* sample_config (sampling.cpp:39-51) */
static void sample_halton(const uint32_t* bases, uint64_t index, const double* lo, const double* hi,
                          int dof, double* out) {
    for (int d = 0; d < dof; ++d) {
        const double h = orc_halton_value(bases[d], index);
        double v = lo[d] + h * (hi[d] - lo[d]);
        if (v >= hi[d]) v = nextafter(hi[d], lo[d]);
        out[d] = v;
    }
}

int orc_sample_config(void* rp, uint64_t offset, uint64_t stride, uint32_t n, double* out) {
    const Robot* r = (const Robot*)rp;
    uint32_t bases[PRRTC_MAX_DOF];
    double lo[PRRTC_MAX_DOF], hi[PRRTC_MAX_DOF];
    orc_halton_bases(r->dof, bases);
    limits_of(r, lo, hi);
    for (uint32_t i = 0; i < n; ++i) sample_halton(bases, offset + i * stride, lo, hi, r->dof, out + (size_t)i * r->dof);
    return 0;
}

/* UniformSampler (sampling.hpp:40-54): std::mt19937_64 + libstdc++
   uniform_real_distribution(generate_canonical<double,53>) */
typedef struct {
    uint64_t mt[312];
    int i;
} Mt64;
static void mt_seed(Mt64* m, uint64_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 312; ++i) m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}
static uint64_t mt_next(Mt64* m) {
    if (m->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t x = (m->mt[k] & 0xFFFFFFFF80000000ULL) | (m->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            m->mt[k] = m->mt[(k + 156) % 312] ^ xa;
        }
        m->i = 0;
    }
    uint64_t x = m->mt[m->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
static double uniform(Mt64* m, double a, double b) {
    const long double r = 18446744073709551616.0L;
    double ret = (double)mt_next(m) / (double)r;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret * (b - a) + a;
}

/* ---------------- planner (planner.cpp) ---------------- */
typedef struct {
    int dof;
    uint64_t cap;
    double* cfg;
    uint64_t* parent;
    _Atomic uint64_t reserved;
    _Atomic uint64_t published;
} Tree;

#define K_FULL UINT64_MAX
#define K_ROOT UINT64_MAX

static void tree_init(Tree* t, uint64_t cap, int dof) {
    t->dof = dof;
    t->cap = cap;
    t->cfg = malloc(sizeof(double) * cap * dof);
    t->parent = malloc(sizeof(uint64_t) * cap);
    atomic_init(&t->reserved, 0);
    atomic_init(&t->published, 0);
}
static void tree_free(Tree* t) {
    free(t->cfg);
    free(t->parent);
}
/* Tree::append (tree.hpp:27-44) */
static uint64_t tree_append(Tree* t, const double* c, uint64_t parent) {
    const uint64_t slot = atomic_fetch_add_explicit(&t->reserved, 1, memory_order_relaxed);
    if (slot >= t->cap) return K_FULL;
    memcpy(t->cfg + slot * t->dof, c, sizeof(double) * t->dof);
    t->parent[slot] = parent;
    int spins = 0;
    while (atomic_load_explicit(&t->published, memory_order_acquire) != slot) {
        if (++spins > 64) {
            sched_yield();
            spins = 0;
        }
    }
    atomic_store_explicit(&t->published, slot + 1, memory_order_release);
    return slot;
}

typedef struct {
    const Robot* r;
    const SceneI* s;
    const prrtc_params* p;
    Tree ta, tb;
    _Atomic uint64_t* dda;   /* dynamic-domain radii as double bits, +inf = unset */
    _Atomic uint64_t* ddb;
    double dd_r;
    _Atomic int stop;
    _Atomic int winner;
    _Atomic uint64_t iterations;
    _Atomic uint64_t tests, fk_calls, fine_entries;
    double* path;
    uint32_t path_len;
    int path_error;
    unsigned workers;
} Shared;

static uint64_t dbits(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}
static double bitsd(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}

typedef struct {
    uint64_t index;
    double distance;
} Nn;

static Nn nearest(const Tree* t, uint64_t snapshot, const double* q, unsigned partitions) {
    Nn o;
    double d;
    o.index = (uint64_t)orc_nearest_parallel(t->cfg, snapshot, (uint32_t)t->dof, q, partitions ? partitions : 1, &d);
    o.distance = d;
    return o;
}

/* assemble_path (planner.cpp:125-150) */
static int assemble(Shared* sh, uint64_t ma, uint64_t mb) {
    const int dof = sh->r->dof;
    const double* A = sh->ta.cfg + ma * dof;
    const double* B = sh->tb.cfg + mb * dof;
    if (sqrt(sq_distance(A, B, dof)) > 1e-12) return -1;
    uint32_t la = 1, lb = 1;
    for (uint64_t i = ma; sh->ta.parent[i] != K_ROOT; i = sh->ta.parent[i]) ++la;
    for (uint64_t i = mb; sh->tb.parent[i] != K_ROOT; i = sh->tb.parent[i]) ++lb;
    const uint32_t len = la + lb - 1;
    double* path = malloc(sizeof(double) * dof * len);
    uint32_t pos = la - 1;
    for (uint64_t i = ma;; i = sh->ta.parent[i]) {
        memcpy(path + (size_t)pos * dof, sh->ta.cfg + i * dof, sizeof(double) * dof);
        if (sh->ta.parent[i] == K_ROOT) break;
        --pos;
    }
    pos = la;
    for (uint64_t i = sh->tb.parent[mb]; mb != 0 && 1; i = sh->tb.parent[i]) {
        if (sh->tb.parent[mb] == K_ROOT) break;
        memcpy(path + (size_t)pos * dof, sh->tb.cfg + i * dof, sizeof(double) * dof);
        ++pos;
        if (sh->tb.parent[i] == K_ROOT) break;
    }
    for (uint32_t i = 1; i < len; ++i)
        if (bitwise_equal(path + (size_t)(i - 1) * dof, path + (size_t)i * dof, dof)) {
            free(path);
            return -1;
        }
    sh->path = path;
    sh->path_len = len;
    return 0;
}

typedef struct {
    Shared* sh;
    unsigned w;
} WorkerArg;

/* worker_main (planner.cpp:186-242) */
static void* worker_main(void* argp) {
    WorkerArg* arg = (WorkerArg*)argp;
    Shared* sh = arg->sh;
    const prrtc_params* p = sh->p;
    const Robot* r = sh->r;
    const int dof = r->dof;
    const unsigned W = sh->workers;
    double lo[PRRTC_MAX_DOF], hi[PRRTC_MAX_DOF];
    uint32_t bases[PRRTC_MAX_DOF];
    limits_of(r, lo, hi);
    orc_halton_bases(dof, bases);
    Checker ck;
    checker_init(&ck, r, sh->s);
    Stats st = {0, 0, 0};
    uint64_t hidx = 1 + p->seed + arg->w;
    Mt64 mt;
    mt_seed(&mt, p->seed * 0x9e3779b97f4a7c15ULL + arg->w);
    double sample[PRRTC_MAX_DOF], cnew[PRRTC_MAX_DOF], prev[PRRTC_MAX_DOF], next[PRRTC_MAX_DOF],
        target[PRRTC_MAX_DOF], nnc[PRRTC_MAX_DOF];
    uint64_t local = 0;
    for (uint64_t iter = 0; iter < p->max_iters_per_worker; ++iter) {
        if (atomic_load_explicit(&sh->stop, memory_order_acquire)) break;
        ++local;
        const uint64_t la = atomic_load_explicit(&sh->ta.published, memory_order_acquire);
        const uint64_t lb = atomic_load_explicit(&sh->tb.published, memory_order_acquire);
        const int from_start = p->balance ? la <= lb : (iter % 2 == 0);  /* planner.hpp:62-65 */
        Tree* ts = from_start ? &sh->ta : &sh->tb;
        Tree* to = from_start ? &sh->tb : &sh->ta;
        _Atomic uint64_t* dd = from_start ? sh->dda : sh->ddb;
        if (p->sampler == PRRTC_SAMPLER_HALTON) {
            sample_halton(bases, hidx, lo, hi, dof, sample);
            hidx += W;
        } else {
            for (int d = 0; d < dof; ++d) sample[d] = uniform(&mt, lo[d], hi[d]);
        }
        const uint64_t snap = atomic_load_explicit(&ts->published, memory_order_acquire);
        const Nn nn = nearest(ts, snap, sample, p->nn_partitions);
        if (nn.distance == 0.0) continue;
        if (p->dynamic_domain &&
            !(nn.distance <= bitsd(atomic_load_explicit(&dd[nn.index], memory_order_relaxed))))
            continue;
        /* extend_step (planner.cpp:48-64) */
        memcpy(nnc, ts->cfg + nn.index * dof, sizeof(double) * dof);
        if (nn.distance <= p->delta) memcpy(cnew, sample, sizeof(double) * dof);
        else lerp(nnc, sample, p->delta / nn.distance, cnew, dof);
        const int valid = validate_edge(&ck, nnc, cnew, p->n_cc, &st, p->two_stage, p->early_exit);
        if (!valid) {
            if (p->dynamic_domain) {
                uint64_t expected = dbits(INFINITY);
                atomic_compare_exchange_strong_explicit(&dd[nn.index], &expected, dbits(sh->dd_r),
                                                        memory_order_relaxed, memory_order_relaxed);
            }
            continue;
        }
        const uint64_t new_index = tree_append(ts, cnew, nn.index);
        if (new_index == K_FULL) break;
        /* greedy_connect (planner.cpp:66-123) */
        int reached = 0;
        uint64_t last_added = new_index;
        const uint64_t snap_o = atomic_load_explicit(&to->published, memory_order_acquire);
        const Nn nno = nearest(to, snap_o, cnew, p->nn_partitions);
        if (nno.distance == 0.0) {
            reached = 1;
        } else {
            const uint64_t n_ext = (uint64_t)ceil(nno.distance / p->delta);
            memcpy(target, to->cfg + nno.index * dof, sizeof(double) * dof);
            if (p->batched_cc) {
                double* from = malloc(sizeof(double) * dof * n_ext);
                double* tos = malloc(sizeof(double) * dof * n_ext);
                uint8_t* ok = malloc(n_ext);
                memcpy(prev, cnew, sizeof(double) * dof);
                for (uint64_t k = 1; k <= n_ext; ++k) {
                    memcpy(from + (k - 1) * dof, prev, sizeof(double) * dof);
                    if (k >= n_ext) memcpy(tos + (k - 1) * dof, target, sizeof(double) * dof);
                    else lerp(cnew, target, (double)k / (double)n_ext, tos + (k - 1) * dof, dof);
                    memcpy(prev, tos + (k - 1) * dof, sizeof(double) * dof);
                }
                Stats bst = {0, 0, 0};
                /* validate_edge_batched via a private checker keeps the stats separate */
                {
                    uint8_t* done = calloc(n_ext, 1);
                    int* counts = malloc(sizeof(int) * n_ext);
                    int max_n = 0;
                    for (uint64_t e = 0; e < n_ext; ++e) {
                        ok[e] = 1;
                        counts[e] = bitwise_equal(from + e * dof, tos + e * dof, dof) ? 1 : p->n_cc;
                        if (counts[e] > max_n) max_n = counts[e];
                    }
                    for (int i = 1; i <= max_n; ++i) {
                        int open = 0;
                        for (uint64_t e = 0; e < n_ext; ++e) {
                            if (done[e] || i > counts[e]) continue;
                            edge_sample(from + e * dof, tos + e * dof, i, counts[e], ck.sample, dof);
                            if (!check_config(&ck, ck.sample, &bst, p->two_stage, p->early_exit)) {
                                ok[e] = 0;
                                if (p->early_exit) {
                                    done[e] = 1;
                                    continue;
                                }
                            }
                            if (i < counts[e]) open = 1;
                        }
                        if (!open) break;
                    }
                    free(done);
                    free(counts);
                }
                st.tests += bst.tests;
                st.fk_calls += bst.fk_calls;
                st.fine_entries += bst.fine_entries;
                uint64_t prev_idx = new_index;
                reached = 1;
                for (uint64_t k = 0; k < n_ext; ++k) {
                    if (!ok[k]) { reached = 0; break; }
                    const uint64_t idx = tree_append(ts, tos + k * dof, prev_idx);
                    if (idx == K_FULL) { reached = 0; break; }
                    prev_idx = idx;
                    last_added = idx;
                }
                free(from);
                free(tos);
                free(ok);
            } else {
                memcpy(prev, cnew, sizeof(double) * dof);
                uint64_t prev_idx = new_index;
                reached = 1;
                for (uint64_t k = 1; k <= n_ext; ++k) {
                    if (atomic_load_explicit(&sh->stop, memory_order_relaxed)) { reached = 0; break; }
                    if (k >= n_ext) memcpy(next, target, sizeof(double) * dof);
                    else lerp(cnew, target, (double)k / (double)n_ext, next, dof);
                    if (!validate_edge(&ck, prev, next, p->n_cc, &st, p->two_stage, p->early_exit)) { reached = 0; break; }
                    const uint64_t idx = tree_append(ts, next, prev_idx);
                    if (idx == K_FULL) { reached = 0; break; }
                    prev_idx = idx;
                    last_added = idx;
                    memcpy(prev, next, sizeof(double) * dof);
                }
            }
        }
        if (!reached) continue;
        int expected = -1;
        if (atomic_compare_exchange_strong(&sh->winner, &expected, (int)arg->w)) {
            const uint64_t ma = from_start ? last_added : nno.index;
            const uint64_t mb = from_start ? nno.index : last_added;
            if (assemble(sh, ma, mb) != 0) sh->path_error = 1;
            atomic_store_explicit(&sh->stop, 1, memory_order_release);
        }
        break;
    }
    atomic_fetch_add_explicit(&sh->iterations, local, memory_order_relaxed);
    atomic_fetch_add(&sh->tests, st.tests);
    atomic_fetch_add(&sh->fk_calls, st.fk_calls);
    atomic_fetch_add(&sh->fine_entries, st.fine_entries);
    checker_free(&ck);
    return NULL;
}

static int within_limits(const Robot* r, const double* q) {  /* planner.cpp:25-31 */
    double lo[PRRTC_MAX_DOF], hi[PRRTC_MAX_DOF];
    limits_of(r, lo, hi);
    for (int d = 0; d < r->dof; ++d)
        if (q[d] < lo[d] || q[d] > hi[d]) return 0;
    return 1;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static double path_cost(const double* path, uint32_t len, int dof) {  /* planner.cpp:152-158 */
    double c = 0.0;
    for (uint32_t i = 1; i < len; ++i) c += sqrt(sq_distance(path + (size_t)(i - 1) * dof, path + (size_t)i * dof, dof));
    return c;
}

/* plan (planner.cpp:246-322) */
int orc_plan(void* rp, void* sp, const double* start, const double* goal, const prrtc_params* p,
             prrtc_result* out) {
    const Robot* r = (const Robot*)rp;
    const int dof = r->dof;
    if (!(p->delta > 0.0)) return fail("plan: delta must be positive");
    if (p->n_cc < 1) return fail("plan: n_cc must be >= 1");
    if (p->tree_capacity < 2) return fail("plan: tree_capacity too small");
    const double t0 = now_ms();
    memset(out, 0, sizeof(*out));
    out->dof = dof;
    out->solving_worker = -1;
    Stats est = {0, 0, 0};
    {
        Checker ck;
        checker_init(&ck, r, sp);
        int bad_s = !within_limits(r, start) || !check_config(&ck, start, &est, p->two_stage, p->early_exit);
        int bad_g = !bad_s && (!within_limits(r, goal) || !check_config(&ck, goal, &est, p->two_stage, p->early_exit));
        checker_free(&ck);
        if (bad_s || bad_g) {
            out->status = PRRTC_INFEASIBLE_ENDPOINT;
            snprintf(out->message, sizeof out->message, "%s configuration is out of limits or in collision",
                     bad_s ? "start" : "goal");
            out->sphere_tests = est.tests;
            out->fk_calls = est.fk_calls;
            out->fine_stage_entries = est.fine_entries;
            out->wall_time_ms = now_ms() - t0;
            return 0;
        }
    }
    if (bitwise_equal(start, goal, dof)) {
        out->status = PRRTC_SOLVED;
        out->path_len = 1;
        out->path = malloc(sizeof(double) * dof);
        memcpy(out->path, start, sizeof(double) * dof);
        out->sphere_tests = est.tests;
        out->fk_calls = est.fk_calls;
        out->fine_stage_entries = est.fine_entries;
        out->wall_time_ms = now_ms() - t0;
        return 0;
    }
    unsigned W = p->workers;
    if (W == 0) {
        long n = sysconf(_SC_NPROCESSORS_ONLN);
        W = n > 0 ? (unsigned)n : 1;
    }
    const uint64_t cap = p->tree_capacity / 2 > 2 ? p->tree_capacity / 2 : 2;
    Shared* sh = calloc(1, sizeof(Shared));
    sh->r = r;
    sh->s = sp;
    sh->p = p;
    sh->workers = W;
    tree_init(&sh->ta, cap, dof);
    tree_init(&sh->tb, cap, dof);
    sh->dd_r = p->dd_radius > 0.0 ? p->dd_radius : 4.0 * p->delta;
    sh->dda = malloc(sizeof(_Atomic uint64_t) * cap);
    sh->ddb = malloc(sizeof(_Atomic uint64_t) * cap);
    for (uint64_t i = 0; i < cap; ++i) {
        atomic_init(&sh->dda[i], dbits(INFINITY));
        atomic_init(&sh->ddb[i], dbits(INFINITY));
    }
    atomic_init(&sh->stop, 0);
    atomic_init(&sh->winner, -1);
    tree_append(&sh->ta, start, K_ROOT);
    tree_append(&sh->tb, goal, K_ROOT);
    if (W == 1) {
        WorkerArg a = {sh, 0};
        worker_main(&a);
    } else {
        pthread_t* th = malloc(sizeof(pthread_t) * W);
        WorkerArg* args = malloc(sizeof(WorkerArg) * W);
        for (unsigned w = 0; w < W; ++w) {
            args[w].sh = sh;
            args[w].w = w;
            pthread_create(&th[w], NULL, worker_main, &args[w]);
        }
        for (unsigned w = 0; w < W; ++w) pthread_join(th[w], NULL);
        free(th);
        free(args);
    }
    out->iterations_total = atomic_load(&sh->iterations);
    out->sphere_tests = atomic_load(&sh->tests) + est.tests;
    out->fk_calls = atomic_load(&sh->fk_calls) + est.fk_calls;
    out->fine_stage_entries = atomic_load(&sh->fine_entries) + est.fine_entries;
    out->solving_worker = atomic_load(&sh->winner);
    out->tree_nodes[0] = atomic_load(&sh->ta.published);
    out->tree_nodes[1] = atomic_load(&sh->tb.published);
    if (out->solving_worker >= 0 && !sh->path_error) {
        out->status = PRRTC_SOLVED;
        out->path = sh->path;
        out->path_len = sh->path_len;
        out->cost = path_cost(sh->path, sh->path_len, dof);
    } else {
        out->status = PRRTC_FAILED;
        snprintf(out->message, sizeof out->message, "all workers exhausted their iteration budgets");
        free(sh->path);
    }
    tree_free(&sh->ta);
    tree_free(&sh->tb);
    free(sh->dda);
    free(sh->ddb);
    free(sh);
    out->wall_time_ms = now_ms() - t0;
    return 0;
}

void orc_result_free(prrtc_result* r) {
    if (r && r->path) {
        free(r->path);
        r->path = NULL;
    }
}

typedef struct {
    void* robot;
    void* const* scenes;
    const double* starts;
    const double* goals;
    const prrtc_params* p;
    prrtc_result* out;
    uint32_t n;
    _Atomic uint32_t next;
} Many;

static void* many_worker(void* a) {
    Many* m = (Many*)a;
    const int dof = ((Robot*)m->robot)->dof;
    for (;;) {
        const uint32_t i = atomic_fetch_add(&m->next, 1);
        if (i >= m->n) break;
        if (orc_plan(m->robot, m->scenes[i], m->starts + (size_t)i * dof, m->goals + (size_t)i * dof, m->p, &m->out[i]) != 0) {
            memset(&m->out[i], 0, sizeof(prrtc_result));
            m->out[i].status = -1;
            snprintf(m->out[i].message, sizeof m->out[i].message, "%s", g_err);
        }
    }
    return NULL;
}

double orc_plan_many(void* robot, void* const* scenes, uint32_t n, const double* starts,
                     const double* goals, const prrtc_params* p, uint32_t n_threads, prrtc_result* out) {
    Many m = {robot, scenes, starts, goals, p, out, n, 0};
    const double t0 = now_ms();
    const uint32_t T = n_threads ? n_threads : 1;
    pthread_t* th = malloc(sizeof(pthread_t) * T);
    for (uint32_t t = 1; t < T; ++t) pthread_create(&th[t], NULL, many_worker, &m);
    many_worker(&m);
    for (uint32_t t = 1; t < T; ++t) pthread_join(th[t], NULL);
    free(th);
    return now_ms() - t0;
}

/* soundness re-validation: fine-only, early exit off */
int orc_path_valid(void* rp, void* sp, const double* path, uint32_t len, int n) {
    const Robot* r = (const Robot*)rp;
    if (len == 0) return 0;
    Checker c;
    checker_init(&c, r, sp);
    Stats st = {0, 0, 0};
    int ok = check_config(&c, path, &st, 0, 0);
    for (uint32_t i = 1; ok && i < len; ++i)
        ok = validate_edge(&c, path + (size_t)(i - 1) * r->dof, path + (size_t)i * r->dof, n, &st, 0, 0);
    checker_free(&c);
    return ok;
}

double orc_path_cost(const double* path, uint32_t len, uint32_t dof) { return path_cost(path, len, (int)dof); }
