/*
 * sdfgi_oracle.c — TEST INFRASTRUCTURE (see sdfgi_oracle.h). Plain C99 restatement
 * of the reference's probe path, one scalar function per reference function, in
 * the reference's operation order (compile with -ffp-contract=off).
 */
#include "sdfgi_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORA_PI 3.14159265358979323846
#define ORA_INF INFINITY
#define MAXCAS 8

/* ------------------------------------------------------------------ vec.hpp */
typedef struct { double x, y, z; } v3;
typedef struct { double x, y; } v2;

static inline v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 add(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 sub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 muls(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static inline v3 divs(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static inline v3 mulv(v3 a, v3 b) { return V(a.x * b.x, a.y * b.y, a.z * b.z); }
static inline double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }  /* vec.hpp:50 */
static inline double len(v3 v) { return sqrt(dot(v, v)); }
static inline v3 norm(v3 v) { return divs(v, len(v)); }                            /* vec.hpp:56 */
static inline v3 lerp3(v3 a, v3 b, double t) { return add(a, muls(sub(b, a), t)); } /* vec.hpp:64 */
/* std::min / std::max / std::clamp */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double sclamp(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
static inline int iclamp(int v, int lo, int hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
static inline double maxc(v3 v) { return smax(v.x, smax(v.y, v.z)); }

/* ------------------------------------------------------------------ rng.hpp */
static inline uint64_t hashU64(uint64_t x) { /* rng.hpp:10-15 */
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e9b5ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static inline uint64_t hashCombine(uint64_t a, uint64_t b) { /* rng.hpp:17 */
    return hashU64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}
typedef struct { uint64_t s; } rng_t;
static inline rng_t rng_key(uint64_t key) { rng_t r; r.s = hashU64(key); return r; } /* rng.hpp:28 */
static inline uint64_t rng_next(rng_t* r) {                                          /* rng.hpp:31-38 */
    r->s += 0x9e3779b97f4a7c15ull;
    uint64_t z = r->s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e9b5ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static inline double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; } /* rng.hpp:41 */

/* ---------------------------------------------------------------- scene state */
typedef struct {
    int res[3], level, base, oct;
    double spacing, origin[3];
} cascade_t;

typedef struct {
    v3 rest, pos, last;
    int reject, alive, last_frame;
} probe_t;

struct ora_stage {
    int np, nk, nl, nm;
    sdfgi_prim* prims;
    sdfgi_cluster* clusters;
    int32_t* mstart;
    int32_t* midx;
    sdfgi_light* lights;
    v3 sky;
    int ncas, nprobes, oct;
    cascade_t cas[MAXCAS];
    probe_t* probes;
    float* atlas[2];
    int front;
};

typedef struct { uint64_t q, cv, cs, pe, steps, sphere, shadow, vis; } stats_t;

/* ------------------------------------------------------------ primitives.hpp */
static double evalPrimitive(const sdfgi_prim* pr, v3 p) { /* primitives.hpp:73-86 */
    const double* m = pr->rot;
    v3 q = sub(p, V(pr->trans[0], pr->trans[1], pr->trans[2]));
    if (!(m[0] == 1.0 && m[4] == 1.0 && m[8] == 1.0))
        q = V(m[0] * q.x + m[3] * q.y + m[6] * q.z, m[1] * q.x + m[4] * q.y + m[7] * q.z,
              m[2] * q.x + m[5] * q.y + m[8] * q.z); /* transposeMul, vec.hpp:113-117 */
    switch (pr->kind) {
        case SDFGI_SPHERE: return len(q) - pr->size[0];                        /* :42 */
        case SDFGI_BOX: {                                                      /* :44-49 */
            v3 a = V(fabs(q.x) - pr->size[0], fabs(q.y) - pr->size[1], fabs(q.z) - pr->size[2]);
            double outside = len(V(smax(a.x, 0.0), smax(a.y, 0.0), smax(a.z, 0.0)));
            double inside = smin(maxc(a), 0.0);
            return outside + inside;
        }
        case SDFGI_PLANE: return q.z;                                          /* :51 */
        case SDFGI_CYLINDER: {                                                 /* :53-60 */
            double dx = sqrt(q.x * q.x + q.y * q.y) - pr->size[0];
            double dy = fabs(q.z) - pr->size[1];
            double outside = sqrt(smax(dx, 0.0) * smax(dx, 0.0) + smax(dy, 0.0) * smax(dy, 0.0));
            double inside = smin(smax(dx, dy), 0.0);
            return outside + inside;
        }
        default: {                                                              /* :62-65 */
            v3 c = V(q.x, q.y, q.z - sclamp(q.z, -pr->size[1], pr->size[1]));
            return len(c) - pr->size[0];
        }
    }
}

static v3 evalGradient(const sdfgi_prim* pr, v3 p) { /* primitives.hpp:96-108, h = 1e-3 */
    const double h = 1e-3;
    v3 g = V(evalPrimitive(pr, V(p.x + h, p.y, p.z)) - evalPrimitive(pr, V(p.x - h, p.y, p.z)),
             evalPrimitive(pr, V(p.x, p.y + h, p.z)) - evalPrimitive(pr, V(p.x, p.y - h, p.z)),
             evalPrimitive(pr, V(p.x, p.y, p.z + h)) - evalPrimitive(pr, V(p.x, p.y, p.z - h)));
    double n = len(g);
    if (n < 1e-6 * 2 * h) return V(1, 0, 0);
    return divs(g, n);
}

/* ------------------------------------------------------------------ scene.hpp */
/* queryCore scalar path (scene.hpp:214-332, the #else branch :293-305) */
static double query(const ora_stage* s, v3 p, double initD, stats_t* st, int* owner) {
    double d = initD;
    int own = -1;
    if (st) ++st->q;
    for (int c = 0; c < s->nk; ++c) {
        const sdfgi_cluster* cl = &s->clusters[c];
        double dx = smax(smax(cl->lo[0] - p.x, p.x - cl->hi[0]), 0.0);
        double dy = smax(smax(cl->lo[1] - p.y, p.y - cl->hi[1]), 0.0);
        double dz = smax(smax(cl->lo[2] - p.z, p.z - cl->hi[2]), 0.0);
        double boxSq = dx * dx + dy * dy + dz * dz;
        if (!cl->unbounded && (d > 0 ? boxSq >= d * d : boxSq > 0)) {
            if (st) ++st->cs;
            continue;
        }
        int end = s->mstart[c + 1];
        if (st) {
            ++st->cv;
            st->pe += (uint64_t)(end - s->mstart[c]);
        }
        for (int m = s->mstart[c]; m < end; ++m) {
            int idx = s->midx[m];
            double pd = evalPrimitive(&s->prims[idx], p);
            if (pd < d) {
                d = pd;
                own = idx;
            }
        }
    }
    if (owner) *owner = own;
    return d;
}

typedef struct {
    int converged, miss, prim, steps;
    double t;
    v3 pos, normal;
} hit_t;

/* sphereTrace, scene.hpp:391-435 */
static hit_t sphereTrace(const ora_stage* s, v3 o, v3 dir, double tMax, double eps, int maxSteps, stats_t* st,
                         double startBound) {
    if (st) ++st->sphere;
    hit_t h;
    memset(&h, 0, sizeof(h));
    h.normal = V(0, 0, 1);
    h.prim = -1;
    double t = 0, lastD = startBound * 0.5;
    for (int step = 0; step < maxSteps; ++step) {
        if (st) ++st->steps;
        v3 p = add(o, muls(dir, t));
        double d = query(s, p, 2 * lastD, st, NULL);
        if (d < eps) {
            int owner = -1;
            d = query(s, p, d + 1e-9, st, &owner);
            for (int i = 0; i < 8 && fabs(d) > 0.25 * eps; ++i) {
                t += d;
                p = add(o, muls(dir, t));
                int o2 = -1;
                d = query(s, p, 2 * fabs(d) + 1e-9, st, &o2);
                if (o2 >= 0) owner = o2;
            }
            h.converged = 1;
            h.t = t;
            h.pos = p;
            h.prim = owner;
            h.steps = step + 1;
            if (owner >= 0) h.normal = evalGradient(&s->prims[owner], p);
            return h;
        }
        if (d >= tMax - t) {
            h.miss = 1;
            h.steps = step + 1;
            return h;
        }
        t += d;
        lastD = d;
    }
    h.miss = 2;
    h.steps = maxSteps;
    return h;
}

/* softShadowTrace, scene.hpp:459-476 */
static double softShadowTrace(const ora_stage* s, v3 o, v3 dir, double tMin, double tMax, double k, stats_t* st,
                              int maxSteps) {
    const double minStep = 5e-4;
    if (st) ++st->shadow;
    double v = 1.0, t = tMin, lastD = ORA_INF;
    for (int step = 0; step < maxSteps && t < tMax; ++step) {
        if (st) ++st->steps;
        double d = query(s, add(o, muls(dir, t)), lastD == ORA_INF ? ORA_INF : 2 * lastD, st, NULL);
        v = smin(v, sclamp(k * d / t, 0.0, 1.0));
        if (v < 1e-3) return 0.0;
        t += smax(d, minStep);
        lastD = smax(d, minStep);
    }
    return v;
}

/* ------------------------------------------------------------- octahedral.hpp */
static inline double signNotZero(double v) { return v >= 0.0 ? 1.0 : -1.0; }
static v2 octEncode(v3 d) { /* octahedral.hpp:13-24 */
    double n = fabs(d.x) + fabs(d.y) + fabs(d.z);
    double px = d.x / n, py = d.y / n;
    if (d.z < 0) {
        double ox = (1.0 - fabs(py)) * signNotZero(px);
        double oy = (1.0 - fabs(px)) * signNotZero(py);
        px = ox;
        py = oy;
    }
    v2 r = {px * 0.5 + 0.5, py * 0.5 + 0.5};
    return r;
}
static v3 octDecode(v2 uv) { /* octahedral.hpp:26-36 */
    double fx = uv.x * 2.0 - 1.0, fy = uv.y * 2.0 - 1.0;
    v3 n = V(fx, fy, 1.0 - fabs(fx) - fabs(fy));
    if (n.z < 0) {
        double t = -n.z;
        n.x += n.x >= 0 ? -t : t;
        n.y += n.y >= 0 ? -t : t;
    }
    return norm(n);
}

/* ------------------------------------------------------------------ atlas.hpp */
static inline size_t tileFloats(int oct) { return (size_t)(oct + 2) * (oct + 2) * 3; }
static inline float* at(float* a, int oct, int probe, int x, int y) {
    int T = oct + 2;
    return a + (((size_t)probe * T + y) * T + x) * 3; /* atlas.hpp:119-124 */
}
static v3 sampleBilinear(const float* a, int oct, int probe, v2 uv) { /* atlas.hpp:59-75 */
    int T = oct + 2;
    double cx = sclamp(uv.x, 0.0, 1.0) * oct + 1.0;
    double cy = sclamp(uv.y, 0.0, 1.0) * oct + 1.0;
    int x0 = (int)floor(cx - 0.5), y0 = (int)floor(cy - 0.5);
    double tx = cx - 0.5 - x0, ty = cy - 0.5 - y0;
    x0 = iclamp(x0, 0, T - 2);
    y0 = iclamp(y0, 0, T - 2);
    const float* p00 = at((float*)a, oct, probe, x0, y0);
    const float* p10 = at((float*)a, oct, probe, x0 + 1, y0);
    const float* p01 = at((float*)a, oct, probe, x0, y0 + 1);
    const float* p11 = at((float*)a, oct, probe, x0 + 1, y0 + 1);
    v3 A = lerp3(V(p00[0], p00[1], p00[2]), V(p10[0], p10[1], p10[2]), tx);
    v3 B = lerp3(V(p01[0], p01[1], p01[2]), V(p11[0], p11[1], p11[2]), tx);
    return lerp3(A, B, ty);
}
static void copyTexel(float* a, int oct, int probe, int dx, int dy, int sx, int sy) {
    memcpy(at(a, oct, probe, dx, dy), at(a, oct, probe, sx, sy), 3 * sizeof(float));
}
static void fillBorder(float* a, int oct, int probe) { /* atlas.hpp:44-56 */
    int r = oct;
    for (int i = 1; i <= r; ++i) {
        copyTexel(a, oct, probe, i, 0, r + 1 - i, 1);
        copyTexel(a, oct, probe, i, r + 1, r + 1 - i, r);
        copyTexel(a, oct, probe, 0, i, 1, r + 1 - i);
        copyTexel(a, oct, probe, r + 1, i, r, r + 1 - i);
    }
    copyTexel(a, oct, probe, 0, 0, r, r);
    copyTexel(a, oct, probe, r + 1, 0, 1, r);
    copyTexel(a, oct, probe, 0, r + 1, r, 1);
    copyTexel(a, oct, probe, r + 1, r + 1, 1, 1);
}

/* ------------------------------------------------------------- mean_value.hpp */
static int mvcWeightsHex(const v3* corners, v3 x, double* w) { /* mean_value.hpp:16-107 */
    static const int faces[6][4] = {{0, 2, 3, 1}, {4, 5, 7, 6}, {0, 1, 5, 4}, {2, 6, 7, 3}, {0, 4, 6, 2}, {1, 3, 7, 5}};
    const double eps = 1e-10;
    double dist[8];
    v3 unit[8];
    for (int i = 0; i < 8; ++i) w[i] = 0.0;
    for (int i = 0; i < 8; ++i) {
        v3 v = sub(corners[i], x);
        dist[i] = len(v);
        if (dist[i] < eps) {
            w[i] = 1.0;
            return 1;
        }
        unit[i] = divs(v, dist[i]);
    }
    int any = 0;
    for (int f = 0; f < 6; ++f) {
        int tris[2][3] = {{faces[f][0], faces[f][1], faces[f][2]}, {faces[f][0], faces[f][2], faces[f][3]}};
        for (int tr = 0; tr < 2; ++tr) {
            const int* tri = tris[tr];
            double d[3], theta[3], c[3], sn[3];
            v3 u[3];
            for (int i = 0; i < 3; ++i) {
                d[i] = dist[tri[i]];
                u[i] = unit[tri[i]];
            }
            for (int i = 0; i < 3; ++i) {
                double l = len(sub(u[(i + 1) % 3], u[(i + 2) % 3]));
                theta[i] = 2.0 * asin(sclamp(l * 0.5, 0.0, 1.0));
            }
            double h = (theta[0] + theta[1] + theta[2]) * 0.5;
            if (ORA_PI - h < 1e-8) {
                double total = 0, ww[3];
                for (int i = 0; i < 8; ++i) w[i] = 0.0;
                for (int i = 0; i < 3; ++i) {
                    ww[i] = sin(theta[i]) * d[(i + 1) % 3] * d[(i + 2) % 3];
                    total += ww[i];
                }
                if (total < eps) return 0;
                for (int i = 0; i < 3; ++i) w[tri[i]] = ww[i] / total;
                return 1;
            }
            v3 cr = V(u[1].y * u[2].z - u[1].z * u[2].y, u[1].z * u[2].x - u[1].x * u[2].z,
                      u[1].x * u[2].y - u[1].y * u[2].x); /* cross, vec.hpp:51-53 */
            double det = dot(u[0], cr);
            double sign = det >= 0 ? 1.0 : -1.0;
            int skip = 0;
            for (int i = 0; i < 3; ++i) {
                double denom = sin(theta[(i + 1) % 3]) * sin(theta[(i + 2) % 3]);
                if (fabs(denom) < eps) {
                    skip = 1;
                    break;
                }
                c[i] = (2.0 * sin(h) * sin(h - theta[i])) / denom - 1.0;
                sn[i] = sign * sqrt(smax(0.0, 1.0 - c[i] * c[i]));
                if (fabs(sn[i]) <= eps) {
                    skip = 1;
                    break;
                }
            }
            if (skip) continue;
            for (int i = 0; i < 3; ++i) {
                double wi = (theta[i] - c[(i + 1) % 3] * theta[(i + 2) % 3] - c[(i + 2) % 3] * theta[(i + 1) % 3]) /
                            (d[i] * sin(theta[(i + 1) % 3]) * sn[(i + 2) % 3]);
                w[tri[i]] += wi;
                any = 1;
            }
        }
    }
    if (!any) return 0;
    double total = 0;
    for (int i = 0; i < 8; ++i) total += w[i];
    if (fabs(total) < eps || !isfinite(total)) return 0;
    for (int i = 0; i < 8; ++i) w[i] /= total;
    return 1;
}

/* ------------------------------------------------------------ probe_volume.hpp */
typedef struct {
    int cascade; /* slot */
    int probe[8];
    double w[8];
    int count, sky;
} stencil_t;

/* interpolationStencil, probe_volume.hpp:224-310 */
static stencil_t interpolationStencil(const ora_stage* s, v3 point, double frac) {
    stencil_t st;
    memset(&st, 0, sizeof(st));
    int chosen = -1, cell[3] = {0, 0, 0}, containing = 0;
    for (int ci = 0; ci < s->ncas; ++ci) {
        const cascade_t* c = &s->cas[ci];
        v3 f = divs(sub(point, V(c->origin[0], c->origin[1], c->origin[2])), c->spacing);
        int ix = (int)floor(f.x), iy = (int)floor(f.y), iz = (int)floor(f.z);
        int inside = ix >= 0 && ix + 1 < c->res[0] && iy >= 0 && iy + 1 < c->res[1] && iz >= 0 && iz + 1 < c->res[2];
        if (!inside) continue;
        ++containing;
        if (chosen < 0 || c->spacing < s->cas[chosen].spacing) {
            chosen = ci;
            cell[0] = ix;
            cell[1] = iy;
            cell[2] = iz;
        }
    }
    int insideCoarser = containing > 1;
    if (chosen < 0) {
        st.sky = 1;
        return st;
    }
    const cascade_t* c = &s->cas[chosen];
    v3 f = divs(sub(point, V(c->origin[0], c->origin[1], c->origin[2])), c->spacing);
    double tx = f.x - cell[0], ty = f.y - cell[1], tz = f.z - cell[2];
    v3 corners[8];
    int pidx[8];
    double maxDisp = 0, w[8];
    for (int k = 0; k < 8; ++k) {
        int ix = cell[0] + (k & 1), iy = cell[1] + ((k >> 1) & 1), iz = cell[2] + ((k >> 2) & 1);
        int pi = ix + c->res[0] * (iy + c->res[1] * iz);
        pidx[k] = pi;
        const probe_t* pr = &s->probes[c->base + pi];
        corners[k] = pr->pos;
        maxDisp = smax(maxDisp, len(sub(pr->pos, pr->rest)));
    }
    int boundary = insideCoarser && (cell[0] == 0 || cell[0] + 2 == c->res[0] || cell[1] == 0 ||
                                     cell[1] + 2 == c->res[1] || cell[2] == 0 || cell[2] + 2 == c->res[2]);
    int wantMvc = maxDisp > frac * c->spacing || boundary, haveMvc = 0;
    if (wantMvc) {
        haveMvc = mvcWeightsHex(corners, point, w);
        if (haveMvc)
            for (int k = 0; k < 8; ++k) w[k] = smax(0.0, w[k]);
    }
    if (!haveMvc)
        for (int k = 0; k < 8; ++k) {
            double wx = (k & 1) ? tx : 1 - tx;
            double wy = ((k >> 1) & 1) ? ty : 1 - ty;
            double wz = ((k >> 2) & 1) ? tz : 1 - tz;
            w[k] = wx * wy * wz;
        }
    double sum = 0;
    for (int k = 0; k < 8; ++k) {
        if (!s->probes[c->base + pidx[k]].alive) w[k] = 0;
        sum += w[k];
    }
    if (sum <= 1e-12) {
        st.sky = 1;
        return st;
    }
    for (int k = 0; k < 8; ++k) {
        st.probe[k] = pidx[k];
        st.w[k] = w[k] / sum;
    }
    st.cascade = chosen;
    st.count = 8;
    return st;
}

/* ------------------------------------------------------------ probe_update.hpp */
/* sampleBounceIrradiance, probe_update.hpp:63-92; prev = front atlas */
static int sampleBounce(const ora_stage* s, v3 pos, v3 normal, double frac, v3* out) {
    if (s->ncas <= 0) return 0;
    stencil_t st = interpolationStencil(s, pos, frac);
    if (st.sky || st.count == 0) return 0;
    const cascade_t* c = &s->cas[st.cascade];
    double wsum = 0, w[8] = {0};
    for (int i = 0; i < st.count; ++i) {
        if (st.w[i] <= 0) continue;
        v3 toProbe = sub(s->probes[c->base + st.probe[i]].pos, pos);
        double l = len(toProbe);
        double facing = l > 1e-9 ? dot(divs(toProbe, l), normal) : 1.0;
        double backface = (facing + 1.0) * 0.5;
        w[i] = st.w[i] * backface * backface;
        wsum += w[i];
    }
    if (wsum <= 1e-12) return 0;
    v3 acc = V(0, 0, 0);
    v2 uv = octEncode(normal);
    for (int i = 0; i < st.count; ++i) {
        if (w[i] <= 0) continue;
        acc = add(acc, muls(sampleBilinear(s->atlas[s->front], s->oct, c->base + st.probe[i], uv), w[i] / wsum));
    }
    *out = acc;
    return 1;
}

/* directIrradiance, probe_update.hpp:97-132 */
static v3 directIrradiance(const ora_stage* s, v3 pos, v3 normal, const sdfgi_cfg* cfg, stats_t* st) {
    v3 total = V(0, 0, 0);
    for (int li = 0; li < s->nl; ++li) {
        const sdfgi_light* L = &s->lights[li];
        v3 dir, unshadowed, I = V(L->intensity[0], L->intensity[1], L->intensity[2]);
        double tMax;
        if (L->kind == SDFGI_LIGHT_POINT) {
            v3 toLight = sub(V(L->position[0], L->position[1], L->position[2]), pos);
            double r2 = dot(toLight, toLight);
            if (r2 < 1e-12) continue;
            double r = sqrt(r2);
            dir = divs(toLight, r);
            double cosT = dot(normal, dir);
            if (cosT <= 0) continue;
            unshadowed = muls(I, cosT / r2);
            tMax = r;
        } else if (L->kind == SDFGI_LIGHT_DIRECTIONAL) {
            dir = V(-L->direction[0], -L->direction[1], -L->direction[2]);
            double cosT = dot(normal, dir);
            if (cosT <= 0) continue;
            unshadowed = muls(I, cosT);
            tMax = cfg->ray_tmax;
        } else {
            continue;
        }
        double cosT = dot(normal, dir);
        double bias = 2.0 * cfg->surface_epsilon / smax(0.1, cosT);
        double vis = 1.0;
        if (tMax - bias > bias)
            vis = softShadowTrace(s, add(pos, muls(normal, bias)), dir, bias, tMax - bias, cfg->shadow_k, st,
                                  (int)cfg->shadow_steps);
        total = add(total, muls(unshadowed, vis));
    }
    return total;
}

/* shadeHit, probe_update.hpp:136-149 */
static v3 shadeHit(const ora_stage* s, const hit_t* h, const sdfgi_cfg* cfg, stats_t* st) {
    if (h->prim < 0) return s->sky;
    const sdfgi_prim* pr = &s->prims[h->prim];
    v3 brdf = divs(V(pr->albedo[0], pr->albedo[1], pr->albedo[2]), ORA_PI);
    v3 radiance = add(V(pr->emission[0], pr->emission[1], pr->emission[2]),
                      mulv(brdf, directIrradiance(s, h->pos, h->normal, cfg, st)));
    if (cfg->bounce_coeff > 0) {
        v3 prev;
        if (sampleBounce(s, h->pos, h->normal, cfg->mvc_relocation_frac, &prev))
            radiance = add(radiance, mulv(brdf, muls(prev, cfg->bounce_coeff)));
    }
    return radiance;
}

/* sampleDirections, sampling.hpp:23-31 (randomRotation rng.hpp:72-90) */
static void sampleDirections(int n, int frame, uint64_t key, uint64_t seed, int rotatePerFrame, v3* dirs) {
    rng_t r = rng_key(hashCombine(hashCombine(hashCombine(seed, rotatePerFrame ? (uint64_t)(int64_t)frame : 0xf1b0u),
                                              key),
                                  0x5df6d1u));
    double u1 = rng_uniform(&r), u2 = rng_uniform(&r), u3 = rng_uniform(&r);
    double a = sqrt(1.0 - u1), b = sqrt(u1);
    double qx = a * sin(2 * ORA_PI * u2), qy = a * cos(2 * ORA_PI * u2);
    double qz = b * sin(2 * ORA_PI * u3), qw = b * cos(2 * ORA_PI * u3);
    double m[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw), 2 * (qx * qz + qy * qw),
                   2 * (qx * qy + qz * qw),     1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw),
                   2 * (qx * qz - qy * qw),     2 * (qy * qz + qx * qw), 1 - 2 * (qx * qx + qy * qy)};
    const double golden = ORA_PI * (3.0 - sqrt(5.0));
    for (int i = 0; i < n; ++i) { /* sphericalFibonacci, sampling.hpp:11-17 */
        double z = 1.0 - (2.0 * i + 1.0) / n;
        double rr = sqrt(smax(0.0, 1.0 - z * z));
        double phi = golden * i;
        v3 v = V(rr * cos(phi), rr * sin(phi), z);
        dirs[i] = V(m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
                    m[6] * v.x + m[7] * v.y + m[8] * v.z);
    }
}

static inline uint64_t probeKey(int cascade, int index) { /* probe_update.hpp:156-159 */
    return hashCombine((uint64_t)cascade + 0x9e1du, (uint64_t)index);
}

/* updateProbe, probe_update.hpp:166-211, writing the back atlas `curr` */
static void updateProbe(ora_stage* s, int slot, int pi, float* curr, const sdfgi_cfg* cfg, int frame,
                        stats_t* st, double* maxDelta, int* raysOut) {
    const cascade_t* c = &s->cas[slot];
    probe_t* probe = &s->probes[c->base + pi];
    int N = (int)cfg->n_rays_full;
    int rays = probe->reject ? N * 2 : N;
    v3* dirs = (v3*)malloc(sizeof(v3) * rays);
    v3* rad = (v3*)malloc(sizeof(v3) * rays);
    sampleDirections(rays, frame, probeKey(c->level, pi), cfg->seed, (int)cfg->rotate_per_frame, dirs);
    for (int i = 0; i < rays; ++i) {
        hit_t h = sphereTrace(s, probe->pos, dirs[i], cfg->ray_tmax, cfg->surface_epsilon, (int)cfg->max_trace_steps,
                              st, ORA_INF);
        rad[i] = h.converged ? shadeHit(s, &h, cfg, st) : s->sky;
    }
    *raysOut = rays;
    double alpha = probe->reject ? 1.0 : sclamp((1.0 - cfg->hysteresis) * rays / cfg->n_rays_full, cfg->alpha_min, 1.0);
    int r = s->oct;
    double md = 0;
    for (int y = 0; y < r; ++y)
        for (int x = 0; x < r; ++x) {
            v3 D = octDecode((v2){(x + 0.5) / r, (y + 0.5) / r}); /* octTexelDir */
            v3 acc = V(0, 0, 0);                                  /* convolveIrradiance :25-34 */
            for (int i = 0; i < rays; ++i) {
                double w = dot(D, dirs[i]);
                if (w > 0) acc = add(acc, muls(rad[i], w));
            }
            v3 fresh = muls(acc, 4.0 * ORA_PI / (double)rays);
            float* t = at(curr, s->oct, c->base + pi, x + 1, y + 1);
            v3 old = V(t[0], t[1], t[2]);
            v3 bl = lerp3(old, fresh, alpha);
            v3 df = sub(bl, old);
            md = smax(md, maxc(V(fabs(df.x), fabs(df.y), fabs(df.z))));
            t[0] = (float)bl.x;
            t[1] = (float)bl.y;
            t[2] = (float)bl.z;
        }
    fillBorder(curr, s->oct, c->base + pi);
    probe->reject = 0;
    probe->last_frame = frame;
    *maxDelta = md;
    free(dirs);
    free(rad);
}

/* ================================================================== C API */
ora_stage* ora_create(const sdfgi_prim* prims, int n_prims, const sdfgi_cluster* clusters, int n_clusters,
                      const int32_t* member_start, const int32_t* member_idx, const sdfgi_light* lights,
                      int n_lights, const double sky[3]) {
    ora_stage* s = (ora_stage*)calloc(1, sizeof(ora_stage));
    s->np = n_prims;
    s->nk = n_clusters;
    s->nl = n_lights;
    s->nm = n_clusters ? member_start[n_clusters] : 0;
    s->prims = (sdfgi_prim*)malloc(sizeof(sdfgi_prim) * (n_prims + 1));
    memcpy(s->prims, prims, sizeof(sdfgi_prim) * n_prims);
    s->clusters = (sdfgi_cluster*)malloc(sizeof(sdfgi_cluster) * (n_clusters + 1));
    memcpy(s->clusters, clusters, sizeof(sdfgi_cluster) * n_clusters);
    s->mstart = (int32_t*)malloc(4 * (n_clusters + 1));
    memcpy(s->mstart, member_start, 4 * (n_clusters + 1));
    s->midx = (int32_t*)malloc(4 * (s->nm + 1));
    memcpy(s->midx, member_idx, 4 * s->nm);
    s->lights = (sdfgi_light*)malloc(sizeof(sdfgi_light) * (n_lights + 1));
    memcpy(s->lights, lights, sizeof(sdfgi_light) * n_lights);
    s->sky = V(sky[0], sky[1], sky[2]);
    s->oct = 8;
    return s;
}

void ora_destroy(ora_stage* s) {
    if (!s) return;
    free(s->prims);
    free(s->clusters);
    free(s->mstart);
    free(s->midx);
    free(s->lights);
    free(s->probes);
    free(s->atlas[0]);
    free(s->atlas[1]);
    free(s);
}

int ora_add_cascade(ora_stage* s, int level, int rx, int ry, int rz, double spacing, const double origin[3],
                    int oct_res) {
    if (s->ncas >= MAXCAS || (s->ncas && oct_res != s->oct)) return 1;
    cascade_t* c = &s->cas[s->ncas];
    c->res[0] = rx;
    c->res[1] = ry;
    c->res[2] = rz;
    c->level = level;
    c->spacing = spacing;
    c->oct = oct_res;
    for (int k = 0; k < 3; ++k) c->origin[k] = origin[k];
    c->base = s->nprobes;
    int n = rx * ry * rz;
    s->oct = oct_res;
    s->probes = (probe_t*)realloc(s->probes, sizeof(probe_t) * (s->nprobes + n));
    for (int iz = 0; iz < rz; ++iz)
        for (int iy = 0; iy < ry; ++iy)
            for (int ix = 0; ix < rx; ++ix) { /* makeCascade, probe_volume.hpp:66-74 */
                probe_t* p = &s->probes[c->base + ix + rx * (iy + ry * iz)];
                p->rest = add(V(origin[0], origin[1], origin[2]), V(ix * spacing, iy * spacing, iz * spacing));
                p->pos = p->rest;
                p->last = p->rest;
                p->reject = 1;
                p->alive = 1;
                p->last_frame = -1;
            }
    s->nprobes += n;
    size_t nf = tileFloats(oct_res) * (size_t)s->nprobes;
    for (int b = 0; b < 2; ++b) {
        s->atlas[b] = (float*)realloc(s->atlas[b], nf * sizeof(float));
        memset(s->atlas[b] + tileFloats(oct_res) * c->base, 0, tileFloats(oct_res) * n * sizeof(float));
    }
    s->ncas++;
    return 0;
}

static void addStats(uint64_t* out, const stats_t* st) {
    if (!out) return;
    out[0] += st->q;
    out[1] += st->cv;
    out[2] += st->cs;
    out[3] += st->pe;
    out[4] += st->steps;
    out[5] += st->sphere;
    out[6] += st->shadow;
    out[7] += st->vis;
}

/* Row-parallel loops of the gather stages (the reference's parallelFor over image
 * rows, shading.hpp:45,288,356,437): worker w takes rows w, w+W, ...; every row's
 * outputs are its own and the per-worker TraceStats are summed (order-free). */
static int g_threads = 1;
void ora_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

typedef void (*row_fn)(void* ctx, int row, stats_t* st, int64_t* acc);
typedef struct {
    row_fn fn;
    void* ctx;
    int n, worker, workers;
    stats_t st;
    int64_t acc;
} rows_t;
static void* rowsWorker(void* arg) {
    rows_t* r = (rows_t*)arg;
    for (int row = r->worker; row < r->n; row += r->workers) r->fn(r->ctx, row, &r->st, &r->acc);
    return NULL;
}
static int64_t parRows(int n, row_fn fn, void* ctx, stats_t* total) {
    int W = g_threads < n ? g_threads : (n > 0 ? n : 1);
    rows_t* ws = (rows_t*)calloc((size_t)W, sizeof(rows_t));
    pthread_t* th = (pthread_t*)calloc((size_t)W, sizeof(pthread_t));
    for (int w = 0; w < W; ++w) {
        ws[w].fn = fn;
        ws[w].ctx = ctx;
        ws[w].n = n;
        ws[w].worker = w;
        ws[w].workers = W;
        if (W > 1)
            pthread_create(&th[w], NULL, rowsWorker, &ws[w]);
        else
            rowsWorker(&ws[w]);
    }
    int64_t acc = 0;
    for (int w = 0; w < W; ++w) {
        if (W > 1) pthread_join(th[w], NULL);
        acc += ws[w].acc;
        if (total) {
            total->q += ws[w].st.q;
            total->cv += ws[w].st.cv;
            total->cs += ws[w].st.cs;
            total->pe += ws[w].st.pe;
            total->steps += ws[w].st.steps;
            total->sphere += ws[w].st.sphere;
            total->shadow += ws[w].st.shadow;
            total->vis += ws[w].st.vis;
        }
    }
    free(ws);
    free(th);
    return acc;
}

int ora_relocate(ora_stage* s, int slot, double th1, double th2, int max_steps, double grad_step, int report[3],
                 uint64_t stats[8]) { /* updateProbePositions, probe_volume.hpp:99-143 */
    if (slot < 0 || slot >= s->ncas) return 1;
    const cascade_t* c = &s->cas[slot];
    int n = c->res[0] * c->res[1] * c->res[2];
    int rel = 0, rej = 0, dead = 0;
    stats_t st;
    memset(&st, 0, sizeof(st));
    double budgetTotal = 0.5 * c->spacing;
    for (int i = 0; i < n; ++i) {
        probe_t* p = &s->probes[c->base + i];
        v3 prev = p->pos, pos = p->rest;
        double d = query(s, pos, ORA_INF, &st, NULL);
        int alive = 1;
        if (d < th1) {
            double budget = budgetTotal, h = grad_step;
            for (int step = 0; step < max_steps && d < th1 && budget > 0; ++step) {
                /* sceneGradient, scene.hpp:360-371 */
                v3 g = V(query(s, V(pos.x + h, pos.y, pos.z), ORA_INF, &st, NULL) -
                             query(s, V(pos.x - h, pos.y, pos.z), ORA_INF, &st, NULL),
                         query(s, V(pos.x, pos.y + h, pos.z), ORA_INF, &st, NULL) -
                             query(s, V(pos.x, pos.y - h, pos.z), ORA_INF, &st, NULL),
                         query(s, V(pos.x, pos.y, pos.z + h), ORA_INF, &st, NULL) -
                             query(s, V(pos.x, pos.y, pos.z - h), ORA_INF, &st, NULL));
                double gn = len(g);
                v3 dir = gn < 1e-6 * 2 * h ? V(1, 0, 0) : divs(g, gn);
                double want = smin((th1 - d) * 1.25, budget);
                pos = add(pos, muls(dir, want));
                budget -= want;
                d = query(s, pos, ORA_INF, &st, NULL);
            }
            alive = d >= th1;
            if (alive && len(sub(pos, p->rest)) > 1e-12) ++rel;
        }
        if (!alive) {
            ++dead;
            p->alive = 0;
            p->last = prev;
            p->pos = pos;
            continue;
        }
        p->alive = 1;
        p->last = prev;
        p->pos = pos;
        int hadHistory = p->last_frame >= 0 && !p->reject;
        if (len(sub(pos, prev)) > th2) {
            p->reject = 1;
            if (hadHistory) ++rej;
        }
    }
    if (report) {
        report[0] = rel;
        report[1] = rej;
        report[2] = dead;
    }
    addStats(stats, &st);
    return 0;
}

typedef struct {
    ora_stage* s;
    const sdfgi_cfg* cfg;
    int frame, slot, stride, worker, workers;
    const int32_t* refs; /* (slot, index) pairs, or NULL: every stride-th probe of `slot` */
    int nrefs;
    double md;
    int64_t rays, updated;
    stats_t st;
} work_t;

/* parallelFor's strided split (parallel.hpp:19-36): worker w owns items w, w+W, ... */
static void* updateWorker(void* arg) {
    work_t* w = (work_t*)arg;
    const cascade_t* c = &w->s->cas[w->slot];
    int n = c->res[0] * c->res[1] * c->res[2];
    float* back = w->s->atlas[1 - w->s->front];
    if (w->refs) {
        for (int item = w->worker; item < w->nrefs; item += w->workers) {
            int slot = w->refs[2 * item], i = w->refs[2 * item + 1];
            if (!w->s->probes[w->s->cas[slot].base + i].alive) continue; /* pipeline.hpp:141 */
            double d;
            int r;
            updateProbe(w->s, slot, i, back, w->cfg, w->frame, &w->st, &d, &r);
            w->md = smax(w->md, d);
            w->rays += r;
            w->updated += 1;
        }
        return NULL;
    }
    for (int item = w->worker; item * w->stride < n; item += w->workers) {
        int i = item * w->stride;
        if (!w->s->probes[c->base + i].alive) continue; /* pipeline.hpp:141 */
        double d;
        int r;
        updateProbe(w->s, w->slot, i, back, w->cfg, w->frame, &w->st, &d, &r);
        w->md = smax(w->md, d);
        w->rays += r;
        w->updated += 1;
    }
    return NULL;
}

static int updateCommon(ora_stage* s, const sdfgi_cfg* cfg, int frame, int stride, const int32_t* refs, int nrefs,
                        int threads, double* max_delta, int64_t* rays, int64_t* updated, uint64_t stats[8]);

int ora_update(ora_stage* s, const sdfgi_cfg* cfg, int frame, int stride, int threads, double* max_delta,
               int64_t* rays, int64_t* updated, uint64_t stats[8]) {
    return updateCommon(s, cfg, frame, stride, NULL, 0, threads, max_delta, rays, updated, stats);
}

int ora_update_refs(ora_stage* s, const sdfgi_cfg* cfg, int frame, const int32_t* refs, int n_refs, int threads,
                    double* max_delta, int64_t* rays, int64_t* updated, uint64_t stats[8]) {
    for (int i = 0; i < n_refs; ++i) {
        int slot = refs[2 * i], idx = refs[2 * i + 1];
        if (slot < 0 || slot >= s->ncas) return 2;
        const cascade_t* c = &s->cas[slot];
        if (idx < 0 || idx >= c->res[0] * c->res[1] * c->res[2]) return 2;
    }
    return updateCommon(s, cfg, frame, 1, refs, n_refs, threads, max_delta, rays, updated, stats);
}

static int updateCommon(ora_stage* s, const sdfgi_cfg* cfg, int frame, int stride, const int32_t* refs, int nrefs,
                        int threads, double* max_delta, int64_t* rays, int64_t* updated, uint64_t stats[8]) {
    if (cfg->oct_res != s->oct) return 1;
    int front = s->front, back = 1 - front;
    size_t nf = tileFloats(s->oct) * (size_t)s->nprobes;
    memcpy(s->atlas[back], s->atlas[front], nf * sizeof(float)); /* pipeline.hpp:131 */
    if (stride < 1) stride = 1;
    if (threads < 1) threads = 1;
    double md = 0;
    int64_t nr = 0, nu = 0;
    stats_t tot;
    memset(&tot, 0, sizeof(tot));
    work_t* ws = (work_t*)calloc((size_t)threads, sizeof(work_t));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int slot = 0; slot < (refs ? 1 : s->ncas); ++slot) {
        for (int w = 0; w < threads; ++w) {
            memset(&ws[w], 0, sizeof(work_t));
            ws[w].s = s;
            ws[w].cfg = cfg;
            ws[w].frame = frame;
            ws[w].slot = slot;
            ws[w].refs = refs;
            ws[w].nrefs = nrefs;
            ws[w].stride = stride;
            ws[w].worker = w;
            ws[w].workers = threads;
            if (threads > 1)
                pthread_create(&th[w], NULL, updateWorker, &ws[w]);
            else
                updateWorker(&ws[w]);
        }
        for (int w = 0; w < threads; ++w) {
            if (threads > 1) pthread_join(th[w], NULL);
            md = smax(md, ws[w].md);
            nr += ws[w].rays;
            nu += ws[w].updated;
            tot.q += ws[w].st.q;
            tot.cv += ws[w].st.cv;
            tot.cs += ws[w].st.cs;
            tot.pe += ws[w].st.pe;
            tot.steps += ws[w].st.steps;
            tot.sphere += ws[w].st.sphere;
            tot.shadow += ws[w].st.shadow;
            tot.vis += ws[w].st.vis;
        }
    }
    free(ws);
    free(th);
    s->front = back; /* frame-end swap, pipeline.hpp:220 */
    if (max_delta) *max_delta = md;
    if (rays) *rays = nr;
    if (updated) *updated = nu;
    addStats(stats, &tot);
    return 0;
}

int ora_probes(const ora_stage* s, int slot, sdfgi_probe* out, int n) {
    if (slot < 0 || slot >= s->ncas) return 1;
    const cascade_t* c = &s->cas[slot];
    if (n != c->res[0] * c->res[1] * c->res[2]) return 1;
    for (int i = 0; i < n; ++i) {
        const probe_t* p = &s->probes[c->base + i];
        memset(&out[i], 0, sizeof(sdfgi_probe));
        double* dst[3] = {out[i].resting, out[i].pos, out[i].last_pos};
        const v3* src[3] = {&p->rest, &p->pos, &p->last};
        for (int k = 0; k < 3; ++k) {
            dst[k][0] = src[k]->x;
            dst[k][1] = src[k]->y;
            dst[k][2] = src[k]->z;
        }
        out[i].reject_history = p->reject;
        out[i].alive = p->alive;
        out[i].last_update_frame = p->last_frame;
    }
    return 0;
}

int ora_atlas(const ora_stage* s, int slot, float* out, int64_t n_floats) {
    if (slot < 0 || slot >= s->ncas) return 1;
    const cascade_t* c = &s->cas[slot];
    int64_t n = (int64_t)tileFloats(s->oct) * c->res[0] * c->res[1] * c->res[2];
    if (n != n_floats) return 1;
    memcpy(out, s->atlas[s->front] + tileFloats(s->oct) * c->base, (size_t)n * sizeof(float));
    return 0;
}

/* Test hooks for the sharded (multi-rank) decomposition, tests/test_multirank.py:
 * overwrite the front atlas of a cascade (the slab exchange), and mark probes as
 * updated this pass (probe_update.hpp:208-209) without tracing them. */
int ora_atlas_set(ora_stage* s, int slot, const float* src, int64_t n_floats) {
    if (slot < 0 || slot >= s->ncas) return 1;
    const cascade_t* c = &s->cas[slot];
    int64_t n = (int64_t)tileFloats(s->oct) * c->res[0] * c->res[1] * c->res[2];
    if (n != n_floats) return 1;
    memcpy(s->atlas[s->front] + tileFloats(s->oct) * c->base, src, (size_t)n * sizeof(float));
    return 0;
}

int ora_mark_updated(ora_stage* s, const int32_t* refs, int n_refs, int frame) {
    for (int i = 0; i < n_refs; ++i) {
        int slot = refs[2 * i], idx = refs[2 * i + 1];
        if (slot < 0 || slot >= s->ncas) return 1;
        probe_t* p = &s->probes[s->cas[slot].base + idx];
        if (!p->alive) continue;
        p->reject = 0;
        p->last_frame = frame;
    }
    return 0;
}

int ora_trace_rays(const ora_stage* s, const sdfgi_cfg* cfg, int frame, int slot, int probe, sdfgi_ray_record* out,
                   int cap) {
    if (slot < 0 || slot >= s->ncas) return -1;
    const cascade_t* c = &s->cas[slot];
    const probe_t* p = &s->probes[c->base + probe];
    int N = (int)cfg->n_rays_full, n = p->reject ? 2 * N : N;
    if (n > cap) return -1;
    v3* dirs = (v3*)malloc(sizeof(v3) * n);
    sampleDirections(n, frame, probeKey(c->level, probe), cfg->seed, (int)cfg->rotate_per_frame, dirs);
    for (int i = 0; i < n; ++i) {
        hit_t h = sphereTrace(s, p->pos, dirs[i], cfg->ray_tmax, cfg->surface_epsilon, (int)cfg->max_trace_steps,
                              NULL, ORA_INF);
        v3 L = h.converged ? shadeHit(s, &h, cfg, NULL) : s->sky;
        sdfgi_ray_record* r = &out[i];
        memset(r, 0, sizeof(*r));
        r->dir[0] = dirs[i].x;
        r->dir[1] = dirs[i].y;
        r->dir[2] = dirs[i].z;
        r->t = h.converged ? h.t : 0.0;
        r->radiance[0] = L.x;
        r->radiance[1] = L.y;
        r->radiance[2] = L.z;
        r->normal[0] = h.normal.x;
        r->normal[1] = h.normal.y;
        r->normal[2] = h.normal.z;
        r->converged = h.converged;
        r->miss = h.miss;
        r->prim_index = h.prim;
        r->steps = h.steps;
    }
    free(dirs);
    return n;
}

void ora_query(const ora_stage* s, const double* pts, const double* init, int n, double* d, int32_t* owner) {
    for (int i = 0; i < n; ++i) {
        int o = -1;
        d[i] = query(s, V(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]), init ? init[i] : ORA_INF, NULL, &o);
        owner[i] = o;
    }
}

/* ================================================================= gather (e) */
static v3 P3(const double* a) { return V(a[0], a[1], a[2]); }

/* Camera::rayDir / project, camera.hpp:29-48 */
static v3 camRayDir(const sdfgi_camera* c, double px, double py, int w, int h) {
    double tanHalf = tan(c->fov_y_deg * ORA_PI / 360.0);
    double aspect = (double)w / h;
    double ndcX = (2.0 * (px + 0.5) / w - 1.0) * tanHalf * aspect;
    double ndcY = (1.0 - 2.0 * (py + 0.5) / h) * tanHalf;
    return norm(add(add(P3(c->forward), muls(P3(c->right), ndcX)), muls(P3(c->up), ndcY)));
}
static int camProject(const sdfgi_camera* c, v3 world, int w, int h, double* ox, double* oy) {
    v3 rel = sub(world, P3(c->position));
    double z = dot(rel, P3(c->forward));
    if (z <= 1e-9) return 0;
    double tanHalf = tan(c->fov_y_deg * ORA_PI / 360.0);
    double aspect = (double)w / h;
    double ndcX = dot(rel, P3(c->right)) / (z * tanHalf * aspect);
    double ndcY = dot(rel, P3(c->up)) / (z * tanHalf);
    *ox = (ndcX + 1.0) * 0.5 * w - 0.5;
    *oy = (1.0 - ndcY) * 0.5 * h - 0.5;
    return 1;
}

typedef struct {
    const ora_stage* s;
    const sdfgi_camera* cam;
    int w, h;
    const sdfgi_cfg* cfg;
    sdfgi_gbuffer_pixel* out;
} gbctx_t;
static void gbufferRow(void* vc, int y, stats_t* st, int64_t* acc) {
    const gbctx_t* g = (const gbctx_t*)vc;
    const ora_stage* s = g->s;
    const sdfgi_camera* cam = g->cam;
    const int w = g->w, h = g->h;
    (void)acc;
    for (int x = 0; x < w; ++x) {
        sdfgi_gbuffer_pixel* px = &g->out[(size_t)y * w + x];
        memset(px, 0, sizeof(*px));
        px->depth = ORA_INF;
        px->normal[2] = 1.0;
        px->prim_index = -1;
        v3 dir = camRayDir(cam, x, (double)y, w, h);
        hit_t hit = sphereTrace(s, P3(cam->position), dir, g->cfg->ray_tmax, g->cfg->surface_epsilon,
                                (int)g->cfg->max_trace_steps, st, ORA_INF);
        if (!hit.converged) continue;
        px->depth = hit.t;
        px->normal[0] = hit.normal.x;
        px->normal[1] = hit.normal.y;
        px->normal[2] = hit.normal.z;
        px->world_pos[0] = hit.pos.x;
        px->world_pos[1] = hit.pos.y;
        px->world_pos[2] = hit.pos.z;
        px->prim_index = hit.prim;
        if (hit.prim >= 0) {
            memcpy(px->albedo, s->prims[hit.prim].albedo, sizeof(px->albedo));
            memcpy(px->emission, s->prims[hit.prim].emission, sizeof(px->emission));
        }
        double ppx, ppy;
        if (camProject(cam, hit.pos, w, h, &ppx, &ppy)) {
            px->motion[0] = ppx - x;
            px->motion[1] = ppy - y;
        }
    }
}

int ora_render_gbuffer(const ora_stage* s, const sdfgi_camera* cam, int w, int h, const sdfgi_cfg* cfg,
                       sdfgi_gbuffer_pixel* out, uint64_t stats[8]) { /* shading.hpp:39-72 */
    stats_t st;
    memset(&st, 0, sizeof(st));
    gbctx_t g = {s, cam, w, h, cfg, out};
    parRows(h, gbufferRow, &g, &st);
    addStats(stats, &st);
    return 0;
}

static int isSky(const sdfgi_gbuffer_pixel* p) { return !(p->depth < ORA_INF); } /* shading.hpp:22 */

/* orthonormalBasis vec.hpp:188-194; cosineHemisphereDir rng.hpp:58-69 */
static v3 cosineHemisphereDir(rng_t* r, v3 n) {
    double u1 = rng_uniform(r), u2 = rng_uniform(r);
    double rr = sqrt(u1), phi = 2.0 * ORA_PI * u2;
    double lx = rr * cos(phi), ly = rr * sin(phi), lz = sqrt(smax(0.0, 1.0 - u1));
    double sign = copysign(1.0, n.z);
    double a = -1.0 / (sign + n.z);
    double c = n.x * n.y * a;
    v3 t = V(1.0 + sign * n.x * n.x * a, sign * c, -sign * n.x);
    v3 b = V(c, sign + n.y * n.y * a, -n.y);
    return norm(add(add(muls(t, lx), muls(b, ly)), muls(n, lz)));
}

typedef struct {
    int key[5];
} tkey_t;

/* the state the gather's row loops share (ora_gather_frame) */
typedef struct {
    const ora_stage* s;
    const sdfgi_gbuffer_pixel* gb;
    int w, h, hw, hh, sw, sh, tilesX, nS;
    const sdfgi_cfg* cfg;
    const int *hs, *sl;
    double* sirr;
    int *svalid, *sanchor;
    const float* front;
    double* res;
    double* indirect;
    const double *hist_irr, *hist_depth;
    int hist_valid;
    double radius;
} gctx_t;

#define GCTX_ALIASES                                                                             \
    const gctx_t* g = (const gctx_t*)vc;                                                          \
    const ora_stage* s = g->s;                                                                    \
    const sdfgi_gbuffer_pixel* gb = g->gb;                                                        \
    const int w = g->w, h = g->h, sw = g->sw, sh = g->sh;                                         \
    const sdfgi_cfg* cfg = g->cfg;                                                                \
    (void)s; (void)gb; (void)w; (void)h; (void)sw; (void)sh; (void)cfg

/* buildVisibilityTasks (shading.hpp:185-259) + runVisibilityTasks (:281-300) +
   shadePixelGI (:319-338): per 4x4 half-res tile, dedup in insertion order; one
   row of tiles */
static void tilesRow(void* vc, int ty, stats_t* stp, int64_t* acc) {
    GCTX_ALIASES;
    const int *hs = g->hs, *sl = g->sl;
    double* sirr = g->sirr;
    int *svalid = g->svalid, *sanchor = g->sanchor;
    const float* front = g->front;
    for (int tx = 0; tx < g->tilesX; ++tx) {
            tkey_t keys[32];
            double tvis[32];
            int nk = 0;
            stencil_t stc[4];
            int cellOf[4], valid[4], tIdx[4][8];
            for (int q = 0; q < 4; ++q) {
                valid[q] = 0;
                cellOf[q] = -1;
                int cx = 2 * tx + (q & 1), cy = 2 * ty + (q >> 1);
                if (cx >= sw || cy >= sh) continue;
                int cell = cy * sw + cx;
                cellOf[q] = cell;
                int src = hs[sl[cell]];
                const sdfgi_gbuffer_pixel* px = &gb[src];
                if (isSky(px)) continue;
                stc[q] = interpolationStencil(s, P3(px->world_pos), cfg->mvc_relocation_frac);
                if (stc[q].sky || stc[q].count == 0) continue;
                valid[q] = 1;
                for (int e = 0; e < stc[q].count; ++e) {
                    if (stc[q].w[e] <= 0) {
                        tIdx[q][e] = -1;
                        continue;
                    }
                    double quant = cfg->dedup_quant_frac * s->cas[stc[q].cascade].spacing;
                    tkey_t k = {{stc[q].cascade, stc[q].probe[e], (int32_t)floor(px->world_pos[0] / quant),
                                 (int32_t)floor(px->world_pos[1] / quant), (int32_t)floor(px->world_pos[2] / quant)}};
                    int found = -1;
                    for (int i = 0; i < nk; ++i)
                        if (memcmp(&keys[i], &k, sizeof(k)) == 0) {
                            found = i;
                            break;
                        }
                    if (found < 0) {
                        /* probeVisibility, shading.hpp:264-279 */
                        const cascade_t* c = &s->cas[stc[q].cascade];
                        v3 sp = P3(px->world_pos), nn = P3(px->normal);
                        v3 toProbe = sub(s->probes[c->base + stc[q].probe[e]].pos, sp);
                        double dist = len(toProbe), vis = 1.0;
                        if (dist >= 1e-9) {
                            v3 dir = divs(toProbe, dist);
                            double cosT = dot(nn, dir);
                            double bias = 2.0 * cfg->surface_epsilon / smax(0.1, cosT);
                            double tMax = dist - cfg->threshold1_frac * c->spacing;
                            if (tMax > bias) {
                                ++stp->vis;
                                vis = softShadowTrace(s, add(sp, muls(nn, bias)), dir, bias, tMax,
                                                      cfg->probe_visibility_k, stp, (int)cfg->shadow_steps);
                            }
                        }
                        found = nk;
                        keys[nk] = k;
                        tvis[nk] = vis;
                        ++nk;
                        ++*acc;
                    }
                    tIdx[q][e] = found;
                }
            }
            for (int q = 0; q < 4; ++q) {
                int cell = cellOf[q];
                if (cell < 0) continue;
                sanchor[cell] = hs[sl[cell]];
                if (!valid[q]) continue;
                const sdfgi_gbuffer_pixel* px = &gb[sanchor[cell]];
                const cascade_t* c = &s->cas[stc[q].cascade];
                double wsum = 0;
                v2 uv = octEncode(P3(px->normal));
                v3 acc = V(0, 0, 0);
                for (int e = 0; e < stc[q].count; ++e) {
                    if (stc[q].w[e] <= 0 || tIdx[q][e] < 0) continue;
                    double ww = stc[q].w[e] * tvis[tIdx[q][e]];
                    if (ww <= 0) continue;
                    acc = add(acc, muls(sampleBilinear(front, s->oct, c->base + stc[q].probe[e], uv), ww));
                    wsum += ww;
                }
                if (wsum <= 1e-9) continue;
                v3 irr = divs(acc, wsum);
                sirr[3 * cell] = irr.x;
                sirr[3 * cell + 1] = irr.y;
                sirr[3 * cell + 2] = irr.z;
                svalid[cell] = 1;
            }
    }
}

/* upsampleAndResolve, shading.hpp:350-426: one image row */
static void resolveRow(void* vc, int y, stats_t* stp, int64_t* acc) {
    GCTX_ALIASES;
    (void)stp;
    (void)acc;
    const int* sanchor = g->sanchor;
    const int* svalid = g->svalid;
    const double* sirr = g->sirr;
    const float* front = g->front;
    const double *hist_irr = g->hist_irr, *hist_depth = g->hist_depth;
    const int hist_valid = g->hist_valid;
    double* res = g->res;
    for (int x = 0; x < w; ++x) {
            const sdfgi_gbuffer_pixel* px = &gb[(size_t)y * w + x];
            if (isSky(px)) continue;
            int qx = x / 4, qy = y / 4;
            v3 acc = V(0, 0, 0), cmin = V(ORA_INF, ORA_INF, ORA_INF), cmax = V(-ORA_INF, -ORA_INF, -ORA_INF);
            double wsum = 0;
            int anyN = 0;
            double sigma = smax(1e-6, cfg->depth_sigma_frac * px->depth);
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int nx = qx + dx, ny = qy + dy;
                    if (nx < 0 || ny < 0 || nx >= sw || ny >= sh) continue;
                    int cell = ny * sw + nx;
                    if (!svalid[cell]) continue;
                    const sdfgi_gbuffer_pixel* an = &gb[sanchor[cell]];
                    double ww = exp(-fabs(an->depth - px->depth) / sigma) *
                                pow(smax(0.0, dot(P3(an->normal), P3(px->normal))), 4.0);
                    if (ww <= 1e-6) continue;
                    v3 si = P3(&sirr[3 * cell]);
                    acc = add(acc, muls(si, ww));
                    wsum += ww;
                    cmin = V(smin(cmin.x, si.x), smin(cmin.y, si.y), smin(cmin.z, si.z));
                    cmax = V(smax(cmax.x, si.x), smax(cmax.y, si.y), smax(cmax.z, si.z));
                    anyN = 1;
                }
            v3 cur = V(0, 0, 0), hist = V(0, 0, 0), o = V(0, 0, 0);
            int haveCur = wsum > 1e-9, haveHist = 0;
            if (haveCur) cur = divs(acc, wsum);
            if (hist_valid) {
                int hx = (int)lround(x + px->motion[0]), hy = (int)lround(y + px->motion[1]);
                if (hx >= 0 && hy >= 0 && hx < w && hy < h) {
                    double hdp = hist_depth[(size_t)hy * w + hx];
                    if (isfinite(hdp) && fabs(hdp - px->depth) <= 0.1 * smax(hdp, px->depth)) {
                        hist = P3(&hist_irr[3 * ((size_t)hy * w + hx)]);
                        if (anyN)
                            hist = V(smin(smax(hist.x, cmin.x), cmax.x), smin(smax(hist.y, cmin.y), cmax.y),
                                     smin(smax(hist.z, cmin.z), cmax.z));
                        haveHist = 1;
                    }
                }
            }
            if (haveCur && haveHist)
                o = add(muls(cur, cfg->history_blend), muls(hist, 1.0 - cfg->history_blend));
            else if (haveCur)
                o = cur;
            else if (haveHist)
                o = hist;
            else {
                stencil_t st = interpolationStencil(s, P3(px->world_pos), cfg->mvc_relocation_frac);
                if (!st.sky) { /* sampleIrradianceRaw, probe_update.hpp:47-57 */
                    v2 uv = octEncode(P3(px->normal));
                    const cascade_t* c = &s->cas[st.cascade];
                    for (int e = 0; e < st.count; ++e) {
                        if (st.w[e] <= 0) continue;
                        o = add(o, muls(sampleBilinear(front, s->oct, c->base + st.probe[e], uv), st.w[e]));
                    }
                }
            }
            double* r = &res[3 * ((size_t)y * w + x)];
            r[0] = o.x;
            r[1] = o.y;
            r[2] = o.z;
    }
}

/* contactGI, shading.hpp:431-477: one image row */
static void contactRow(void* vc, int y, stats_t* stp, int64_t* acc) {
    GCTX_ALIASES;
    (void)acc;
    const double* res = g->res;
    double* indirect = g->indirect;
    const double radius = g->radius;
    const int nS = g->nS;
    for (int x = 0; x < w; ++x) {
                const sdfgi_gbuffer_pixel* px = &gb[(size_t)y * w + x];
                double* out = &indirect[3 * ((size_t)y * w + x)];
                out[0] = out[1] = out[2] = 0;
                if (isSky(px)) continue;
                v3 brdf = divs(P3(px->albedo), ORA_PI);
                v3 probeGi = mulv(brdf, P3(&res[3 * ((size_t)y * w + x)]));
                if (nS <= 0 || radius <= 0) {
                    out[0] = probeGi.x;
                    out[1] = probeGi.y;
                    out[2] = probeGi.z;
                    continue;
                }
                rng_t r = rng_key(hashCombine(hashCombine(cfg->seed, 0xc0417ffull), (uint64_t)y * w + x));
                int unocc = 0;
                v3 occ = V(0, 0, 0), nn = P3(px->normal), wp = P3(px->world_pos);
                for (int k = 0; k < nS; ++k) {
                    v3 dir = cosineHemisphereDir(&r, nn);
                    double cosT = smax(0.1, dot(dir, nn));
                    double bias = 2.0 * cfg->surface_epsilon / cosT;
                    hit_t hit = sphereTrace(s, add(wp, muls(nn, bias)), dir, radius, cfg->surface_epsilon,
                                            (int)cfg->max_trace_steps, stp, bias + cfg->surface_epsilon);
                    if (!hit.converged)
                        ++unocc;
                    else
                        occ = add(occ, shadeHit(s, &hit, cfg, stp));
                }
                double ao = (double)unocc / nS;
                v3 contact = mulv(muls(divs(P3(px->albedo), ORA_PI), ORA_PI / nS), occ);
                v3 o = add(muls(probeGi, ao), contact);
                out[0] = o.x;
                out[1] = o.y;
                out[2] = o.z;
    }
}

int ora_gather_frame(const ora_stage* s, const sdfgi_gbuffer_pixel* gb, int w, int h, int frame, const sdfgi_cfg* cfg,
                     const double* hist_irr, const double* hist_depth, int hist_valid, double* half_depth,
                     int32_t* half_src, int32_t* sel, double* sparse_irr, int32_t* sparse_valid,
                     int32_t* sparse_anchor, double* resolved, double* indirect, uint64_t vis_stats[8],
                     uint64_t contact_stats[8]) {
    const int hw = (w + 1) / 2, hh = (h + 1) / 2;
    const int sw = (hw + 1) / 2, sh = (hh + 1) / 2;
    double* hd = (double*)malloc(sizeof(double) * hw * hh);
    int* hs = (int*)malloc(sizeof(int) * hw * hh);
    /* downsampleDepthCheckerboard, shading.hpp:85-112 */
    for (int y = 0; y < hh; ++y)
        for (int x = 0; x < hw; ++x) {
            int takeMax = ((x + y) & 1) == 0;
            double best = takeMax ? -ORA_INF : ORA_INF;
            int bestSrc = 0;
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    int sx = 2 * x + dx < w - 1 ? 2 * x + dx : w - 1;
                    int sy = 2 * y + dy < h - 1 ? 2 * y + dy : h - 1;
                    double d = gb[(size_t)sy * w + sx].depth;
                    if (takeMax ? d > best : d < best) {
                        best = d;
                        bestSrc = sy * w + sx;
                    }
                }
            hd[y * hw + x] = best;
            hs[y * hw + x] = bestSrc;
        }
    /* selectVisibilityPixels, shading.hpp:125-161 */
    static const int offs[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    int* sl = (int*)malloc(sizeof(int) * sw * sh);
    int rot = frame & 3;
    for (int y = 0; y < sh; ++y)
        for (int x = 0; x < sw; ++x) {
            int hx0 = 2 * x, hy0 = 2 * y;
            double lo = ORA_INF, hi = -ORA_INF;
            int loIdx = -1, hiIdx = -1;
            for (int k = 0; k < 4; ++k) {
                int hx = hx0 + offs[k][0] < hw - 1 ? hx0 + offs[k][0] : hw - 1;
                int hy = hy0 + offs[k][1] < hh - 1 ? hy0 + offs[k][1] : hh - 1;
                double d = hd[hy * hw + hx];
                if (!isfinite(d)) continue;
                if (d < lo) { lo = d; loIdx = hy * hw + hx; }
                if (d > hi) { hi = d; hiIdx = hy * hw + hx; }
            }
            int hx = hx0 + offs[rot][0] < hw - 1 ? hx0 + offs[rot][0] : hw - 1;
            int hy = hy0 + offs[rot][1] < hh - 1 ? hy0 + offs[rot][1] : hh - 1;
            int pick = hy * hw + hx;
            if (loIdx >= 0) {
                int rotSky = !isfinite(hd[pick]);
                int spread = (hi - lo) > 0.1 * hi;
                if (spread)
                    pick = (frame & 1) == 0 ? loIdx : hiIdx;
                else if (rotSky)
                    pick = loIdx;
            }
            sl[y * sw + x] = pick;
        }
    int ncell = sw * sh;
    double* sirr = (double*)calloc((size_t)ncell * 3, sizeof(double));
    int* svalid = (int*)calloc((size_t)ncell, sizeof(int));
    int* sanchor = (int*)calloc((size_t)ncell, sizeof(int));
    double* res = (double*)calloc((size_t)w * h * 3, sizeof(double));
    gctx_t g;
    memset(&g, 0, sizeof(g));
    g.s = s;
    g.gb = gb;
    g.w = w;
    g.h = h;
    g.hw = hw;
    g.hh = hh;
    g.sw = sw;
    g.sh = sh;
    g.tilesX = (sw + 1) / 2;
    g.cfg = cfg;
    g.hs = hs;
    g.sl = sl;
    g.sirr = sirr;
    g.svalid = svalid;
    g.sanchor = sanchor;
    g.front = s->atlas[s->front];
    g.res = res;
    g.indirect = indirect;
    g.hist_irr = hist_irr;
    g.hist_depth = hist_depth;
    g.hist_valid = hist_valid;
    g.radius = cfg->contact_radius_frac * s->cas[0].spacing;
    g.nS = (int)cfg->contact_samples;
    stats_t vst, cst;
    memset(&vst, 0, sizeof(vst));
    memset(&cst, 0, sizeof(cst));
    int ntasks = (int)parRows((sh + 1) / 2, tilesRow, &g, &vst);
    parRows(h, resolveRow, &g, NULL);
    if (indirect) parRows(h, contactRow, &g, &cst);
    if (half_depth) memcpy(half_depth, hd, sizeof(double) * hw * hh);
    if (half_src) memcpy(half_src, hs, sizeof(int) * hw * hh);
    if (sel) memcpy(sel, sl, sizeof(int) * ncell);
    if (sparse_irr) memcpy(sparse_irr, sirr, sizeof(double) * 3 * ncell);
    if (sparse_valid) memcpy(sparse_valid, svalid, sizeof(int) * ncell);
    if (sparse_anchor) memcpy(sparse_anchor, sanchor, sizeof(int) * ncell);
    if (resolved) memcpy(resolved, res, sizeof(double) * 3 * w * h);
    addStats(vis_stats, &vst);
    addStats(contact_stats, &cst);
    free(hd);
    free(hs);
    free(sl);
    free(sirr);
    free(svalid);
    free(sanchor);
    free(res);
    return ntasks;
}

/* composeFrame, shading.hpp:480-504 (per pixel, row-major; statistics merged) */
int ora_compose(const ora_stage* s, const sdfgi_gbuffer_pixel* gb, int w, int h, const double* indirect,
                const sdfgi_cfg* cfg, double* out, uint64_t stats[8]) {
    stats_t st;
    memset(&st, 0, sizeof(st));
    for (int64_t i = 0; i < (int64_t)w * h; ++i) {
        const sdfgi_gbuffer_pixel* px = &gb[i];
        v3 o;
        if (!(px->depth < ORA_INF)) {
            o = s->sky;
        } else {
            v3 pos = V(px->world_pos[0], px->world_pos[1], px->world_pos[2]);
            v3 nrm = V(px->normal[0], px->normal[1], px->normal[2]);
            v3 direct = directIrradiance(s, pos, nrm, cfg, &st);
            v3 alb = V(px->albedo[0], px->albedo[1], px->albedo[2]);
            v3 em = V(px->emission[0], px->emission[1], px->emission[2]);
            o = add(add(em, mulv(divs(alb, ORA_PI), direct)), V(indirect[3 * i], indirect[3 * i + 1], indirect[3 * i + 2]));
        }
        out[3 * i] = o.x;
        out[3 * i + 1] = o.y;
        out[3 * i + 2] = o.z;
    }
    if (stats) {
        const uint64_t v[8] = {st.q, st.cv, st.cs, st.pe, st.steps, st.sphere, st.shadow, st.vis};
        for (int k = 0; k < 8; ++k) stats[k] += v[k];
    }
    return 0;
}

/* selectProbesForUpdate, probe_volume.hpp:154-198: priority favours near,
 * camera-facing, stale and history-rejected probes; probes at least one fair
 * period stale are forced (oldest first). std::stable_sort's order = this total
 * order with the candidate position as the final key. */
typedef struct {
    int slot, index, staleness, forced;
    double priority;
    int64_t pos;
} cand_t;

static int candCmp(const void* pa, const void* pb) {
    const cand_t* a = (const cand_t*)pa;
    const cand_t* b = (const cand_t*)pb;
    if (a->forced != b->forced) return a->forced ? -1 : 1;
    if (a->forced) {
        if (a->staleness != b->staleness) return a->staleness > b->staleness ? -1 : 1;
    } else if (a->priority != b->priority) {
        return a->priority > b->priority ? -1 : 1;
    }
    return a->pos < b->pos ? -1 : (a->pos > b->pos ? 1 : 0);
}

int ora_select(const ora_stage* s, const double cam_pos[3], const double cam_fwd[3], int budget, int frame,
               int32_t* out_refs) {
    int total = 0;
    for (int ci = 0; ci < s->ncas; ++ci) total += s->cas[ci].res[0] * s->cas[ci].res[1] * s->cas[ci].res[2];
    if (total == 0 || budget <= 0) return 0;
    int period = (total + budget - 1) / budget;
    int forceAge = period;
    cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)total);
    v3 cp = V(cam_pos[0], cam_pos[1], cam_pos[2]), cf = V(cam_fwd[0], cam_fwd[1], cam_fwd[2]);
    int64_t k = 0;
    for (int ci = 0; ci < s->ncas; ++ci) {
        const cascade_t* cs = &s->cas[ci];
        int n = cs->res[0] * cs->res[1] * cs->res[2];
        for (int i = 0; i < n; ++i) {
            const probe_t* p = &s->probes[cs->base + i];
            double dist = len(sub(p->pos, cp));
            int staleness = frame - p->last_frame;
            double angular = 0.25;
            if (dist > 1e-9) angular += 0.75 * smax(0.0, dot(divs(sub(p->pos, cp), dist), cf));
            double priority = (1.0 / (1.0 + dist / cs->spacing)) * angular * staleness;
            if (p->reject) priority *= 4.0;
            c[k].slot = ci;
            c[k].index = i;
            c[k].staleness = staleness;
            c[k].forced = staleness >= forceAge;
            c[k].priority = priority;
            c[k].pos = k;
            ++k;
        }
    }
    qsort(c, (size_t)total, sizeof(cand_t), candCmp);
    int n = budget < total ? budget : total;
    for (int i = 0; i < n; ++i) {
        out_refs[2 * i] = c[i].slot;
        out_refs[2 * i + 1] = c[i].index;
    }
    free(c);
    return n;
}
