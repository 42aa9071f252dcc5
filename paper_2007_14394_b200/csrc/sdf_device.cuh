// sdf_device.cuh — device-side SDF scene, tracing, shading and probe math.
//
// Templated on the arithmetic type R (double = parity mode, compiled with
// -fmad=false so every product/sum rounds exactly as the reference's
// -ffp-contract=off build; float = perf mode). Each function cites the
// reference function whose semantics it reproduces; the *structure* is GPU
// first: the scene is stored in cluster (CSR) order so a warp walks clusters
// and members in lock-step with warp-uniform (broadcast) loads, the probe update
// is one CTA per probe with rays across lanes, and the texel convolution reads
// the CTA's samples from shared memory.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sdfgi_dev {

constexpr double kPi = 3.14159265358979323846;

// std::min / std::max / std::clamp semantics (operand order, NaN and signed-zero
// behaviour) — vec.hpp uses the std versions, not fmin/fmax.
template <typename R> __device__ __forceinline__ R smin(R a, R b) { return (b < a) ? b : a; }
template <typename R> __device__ __forceinline__ R smax(R a, R b) { return (a < b) ? b : a; }
template <typename R> __device__ __forceinline__ R sclamp(R v, R lo, R hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}
__device__ __forceinline__ int iclamp(int v, int lo, int hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

template <typename R> __device__ __forceinline__ R rsqrt_exact(R v) { return sqrt(v); }

template <typename R> struct V3 {
    R x, y, z;
};
template <typename R> __device__ __forceinline__ V3<R> mk(R x, R y, R z) { return V3<R>{x, y, z}; }
template <typename R> __device__ __forceinline__ V3<R> operator+(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <typename R> __device__ __forceinline__ V3<R> operator-(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <typename R> __device__ __forceinline__ V3<R> operator-(V3<R> a) { return {-a.x, -a.y, -a.z}; }
template <typename R> __device__ __forceinline__ V3<R> operator*(V3<R> a, R s) { return {a.x * s, a.y * s, a.z * s}; }
template <typename R> __device__ __forceinline__ V3<R> operator/(V3<R> a, R s) { return {a.x / s, a.y / s, a.z / s}; }
template <typename R> __device__ __forceinline__ V3<R> operator*(V3<R> a, V3<R> b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
// vec.hpp:50 — (x*x + y*y) + z*z
template <typename R> __device__ __forceinline__ R dot(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <typename R> __device__ __forceinline__ R length(V3<R> v) { return sqrt(dot(v, v)); }
template <typename R> __device__ __forceinline__ V3<R> normalize(V3<R> v) { return v / length(v); }
template <typename R> __device__ __forceinline__ V3<R> lerp(V3<R> a, V3<R> b, R t) { return a + (b - a) * t; }
template <typename R> __device__ __forceinline__ R maxComponent(V3<R> v) { return smax(v.x, smax(v.y, v.z)); }

// ------------------------------------------------------------------ rng.hpp
__device__ __forceinline__ uint64_t hashU64(uint64_t x) {  // rng.hpp:10-15
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e9b5ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t hashCombine(uint64_t a, uint64_t b) {  // rng.hpp:17
    return hashU64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}
struct Rng {  // rng.hpp:22-48
    uint64_t s;
    __device__ explicit Rng(uint64_t key) : s(hashU64(key)) {}
    __device__ uint64_t next() {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e9b5ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    __device__ double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
// probeKey, probe_update.hpp:156-159
__device__ __forceinline__ uint64_t probeKey(int cascade, int index) {
    return hashCombine(static_cast<uint64_t>(cascade) + 0x9e1du, static_cast<uint64_t>(index));
}

// --------------------------------------------------------------- scene data
// One primitive in CSR (cluster) order. identity = the rotation's diagonal is all
// 1.0 (primitives.hpp:76-77 fast path). 128 B for double, ordered for 16-byte
// loads: translation, size, kind/identity and rot[0] in the first 64 B (four
// loads cover an unrotated primitive), the rest of the rotation in the next 64 B.
template <typename R> struct __align__(16) DPrim {
    R trans[3];
    R size[3];
    int kind;
    int identity;
    R rot[9];
};
// FP32 perf-mode record: every kind in one branch-free form (see evalPrim<float>):
// e = half extents of a box, or (e0, -1, e2) for a radial shape (cylinder r/h,
// capsule 0/h, sphere 0/0: e1 < 0 marks radial), rr = rounding radius (capsule,
// sphere); rr < 0 marks a plane. 64 B = four 16-byte loads.
template <> struct __align__(16) DPrim<float> {
    float rot[9];
    float trans[3];
    float e[3];
    float rr;
};
template <typename R> struct __align__(16) DCluster {
    R lo[3];
    R hi[3];
    int unbounded;
    int _pad;
};
struct DLight {  // sdfgi_light, kept in double in both modes (tiny)
    int kind;
    int _pad;
    double position[3];
    double direction[3];
    double intensity[3];
};

// Candidate grid (exact acceleration of the cluster walk). For every cell of a
// uniform grid over the bounded clusters, U = SDF(cell centre) + half the (padded)
// cell diagonal bounds the scene SDF anywhere in the cell (1-Lipschitz), so only
// primitives whose conservative AABB lies within max(U, 0) of the cell can hold
// the minimum — or tie with it — at any point of the cell; the cell's list holds
// exactly those (CSR positions, nearest first) and the query evaluates them
// without cluster tests. Points outside the grid (and queries still open at a
// truncated list's sentinel) walk a bounding-volume hierarchy over the bounded
// clusters nearest child first, then visit the unbounded clusters. Visiting order
// no longer follows cluster order, so the walks break distance ties explicitly
// towards the lowest CSR position — the primitive the reference's in-order walk
// keeps (scene.hpp:243) — and values and owners stay identical to the reference's.
//
// BVH node: the two children's boxes (padded outward, float) and their codes:
// code >= 0 an inner node, code < 0 the cluster -code - 1.
struct BNode {
    float lo[2][3];
    float hi[2][3];
    int child[2];
};
constexpr int kBvhStack = 24;  // median splits: depth <= ceil(log2(clusters)) (16M clusters)

struct GridDev {
    double lo[3];
    double invH;
    float flo[3];   // the same in float for the FP32 path
    float finvH;
    double h;       // cell size (cell centres: lo + (i + 1/2) h)
    int dim[3];
    int bvhRoot;    // code of the root (see BNode); meaningless when nBounded == 0
    const int* __restrict__ start;  // ncells + 1
    // per cell, one 16-byte load: x = start, y = end of its entries, (z, w) = its
    // first entry (bound bits, CSR position; (+inf, -1) for an empty list) — the
    // list range and the first candidate without a second dependent load
    const int4* __restrict__ cell;
    // per list entry, one 8-byte load: x = the bits of a float lower bound E on that
    // primitive's SDF at the cell centre c (minus the build margin, rounded down), y =
    // its CSR position (-1: sentinel). Every primitive SDF is 1-Lipschitz, so at a
    // query point p the primitive is at least E - |p - c| away; entries are sorted by
    // E, so a query stops at the first E - |p - c| > its running minimum.
    const int2* __restrict__ entry;
    const BNode* __restrict__ bvh;
    const int* __restrict__ unbounded;  // cluster ids of the unbounded clusters
    int nUnbounded;
    int nBounded;
    float walkSlack;  // FP64 walks' float box tests: > the float rounding of |p - box| at this scale
    // the union of the bounded clusters' boxes: every bounded primitive's SDF is at
    // least the distance to it from outside (the escape tests of accel mode 2)
    double geoLo[3], geoHi[3];
};

// softShadowTrace (scene.hpp:459-476) from t on can no longer lower v: outside the
// box holding every bounded primitive (no unbounded one in the scene) each
// remaining query returns d >= L, the distance to the box, which is convex along
// the ray: L(t') >= L(t) + L'(t) (t' - t). The lower bound (L + L' (t' - t)) / t' of
// the remaining terms d / t' is monotone in t', so its minimum over [t, tEnd] sits
// at an end; when k times it exceeds v (with a relative margin far above the FP64
// rounding of the terms), min(v, clamp(k d / t')) stays v for every remaining step
// and the march's result is v.
template <typename R>
__device__ __forceinline__ bool shadowSettled(const GridDev& g, V3<R> p, V3<R> dir, R t, R tEnd, R k, R v) {
    const double px = p.x, py = p.y, pz = p.z;
    if (px >= g.geoLo[0] && px <= g.geoHi[0] && py >= g.geoLo[1] && py <= g.geoHi[1] && pz >= g.geoLo[2] &&
        pz <= g.geoHi[2])
        return false;  // inside the geometry box: no bound
    const double dx = px - sclamp(px, g.geoLo[0], g.geoHi[0]);
    const double dy = py - sclamp(py, g.geoLo[1], g.geoHi[1]);
    const double dz = pz - sclamp(pz, g.geoLo[2], g.geoHi[2]);
    const double L2 = dx * dx + dy * dy + dz * dz;
    if (!(L2 > 0)) return false;
    const double L = sqrt(L2);
    const double dL = (double(dir.x) * dx + double(dir.y) * dy + double(dir.z) * dz) / L;
    const double f0 = L / double(t), f1 = (L + dL * (double(tEnd) - double(t))) / double(tEnd);
    return double(k) * fmin(f0, f1) * (1.0 - 1e-9) > double(v) * (1.0 + 1e-9);
}

template <typename R> struct SceneView {
    const DPrim<R>* __restrict__ prims;        // CSR order
    const DCluster<R>* __restrict__ clusters;
    const int* __restrict__ cstart;            // K+1
    const int* __restrict__ orig;              // CSR position -> ActiveScene primitive index
    const double* __restrict__ albedo;         // 3 per CSR position
    const double* __restrict__ emission;       // 3 per CSR position
    const int* __restrict__ kindId;            // kind | identity << 8 per CSR position (statistics)
    const DLight* __restrict__ lights;
    int n_prims, n_clusters, n_lights;
    double sky[3];
    GridDev grid;
    int useGrid;
    // the primitive records in the layout the tracing kernels stage in shared memory
    // (stageBytes == 0: the scene does not fit and the kernels read `prims`)
    const void* __restrict__ stage;
    int stageBytes;
    int stageRotOff;  // FP64: byte offset of the rotation rows (8 doubles per rotated primitive)
    // dynamic primitives (moved since the candidate grid was built; not in its lists):
    // CSR positions every on-grid query evaluates besides the cell's list
    const int* __restrict__ dyn;
    int nDyn;
};

// TraceStats (scene.hpp:16-36), per thread.
// ek[0..4]: primitive evaluations by PrimitiveKind, ek[5]: of those, rotated ones
// (the algorithmic-work accounting of SURVEY §8d weights evaluations by kind).
struct Counters {
    unsigned long long q, cv, cs, pe, steps, sphere, shadow, vis;
    unsigned long long ek[6];
    __device__ void zero() {
        q = cv = cs = pe = steps = sphere = shadow = vis = 0;
        for (int i = 0; i < 6; ++i) ek[i] = 0;
    }
};

// ------------------------------------------------------------ primitives.hpp
// evalPrimitive, primitives.hpp:73-86 (+ detail::*Sdf :42-65)
template <typename R>
__device__ __forceinline__ R evalPrim(const DPrim<R>& pr, V3<R> p) {
    V3<R> q = p - mk(pr.trans[0], pr.trans[1], pr.trans[2]);
    if (!pr.identity) {
        // transposeMul, vec.hpp:113-117
        const R* m = pr.rot;
        q = mk(m[0] * q.x + m[3] * q.y + m[6] * q.z,
               m[1] * q.x + m[4] * q.y + m[7] * q.z,
               m[2] * q.x + m[5] * q.y + m[8] * q.z);
    }
    switch (pr.kind) {
        case 0:  // sphere
            return length(q) - pr.size[0];
        case 1: {  // box
            V3<R> a = mk(fabs(q.x) - pr.size[0], fabs(q.y) - pr.size[1], fabs(q.z) - pr.size[2]);
            R outside = length(mk(smax(a.x, R(0)), smax(a.y, R(0)), smax(a.z, R(0))));
            R inside = smin(maxComponent(a), R(0));
            return outside + inside;
        }
        case 2:  // plane
            return q.z;
        case 3: {  // cylinder
            R dx = sqrt(q.x * q.x + q.y * q.y) - pr.size[0];
            R dy = fabs(q.z) - pr.size[1];
            R ox = smax(dx, R(0)), oy = smax(dy, R(0));
            R outside = sqrt(ox * ox + oy * oy);
            R inside = smin(smax(dx, dy), R(0));
            return outside + inside;
        }
        default: {  // capsule
            V3<R> c = mk(q.x, q.y, q.z - sclamp(q.z, -pr.size[1], pr.size[1]));
            return length(c) - pr.size[0];
        }
    }
}

// The per-kind tail of the FP64 evaluation (primitives.hpp:42-65) from the local
// point q: the branches only set up sqrt((vx*vx + vy*vy) + vz*vz) + post, and the
// one square root every kind ends in runs after they reconverge. SDFGI_EVAL_HOIST:
// the cylinder's radial square root is taken by every lane before the branches
// (same value; no divergent FP64 sqrt inside the cylinder branch) and max(x, 0)
// is (x + |x|) / 2 (exact, and only ever squared).
#ifndef SDFGI_EVAL_HOIST
#define SDFGI_EVAL_HOIST 1  // C2 step FP64 30.68 -> 30.42 ms
#endif
__device__ __forceinline__ double pos0(double x) { return SDFGI_EVAL_HOIST ? (x + fabs(x)) * 0.5 : smax(x, 0.0); }
__device__ __forceinline__ double evalKindTail(int kind, V3<double> q, double size0, double size1, double size2) {
    if (kind == 2) return q.z;  // plane
    double rho = 0.0;
    if (SDFGI_EVAL_HOIST) rho = sqrt(q.x * q.x + q.y * q.y);
    double vx, vy, vz, post;
    if (kind == 1) {  // box
        const double ax = fabs(q.x) - size0, ay = fabs(q.y) - size1, az = fabs(q.z) - size2;
        vx = pos0(ax);
        vy = pos0(ay);
        vz = pos0(az);
        post = smin(smax(ax, smax(ay, az)), 0.0);
    } else if (kind == 3) {  // cylinder
        if (!SDFGI_EVAL_HOIST) rho = sqrt(q.x * q.x + q.y * q.y);
        const double dx = rho - size0, dy = fabs(q.z) - size1;
        vx = pos0(dx);
        vy = pos0(dy);
        vz = 0.0;
        post = smin(smax(dx, dy), 0.0);
    } else {  // sphere (0) / capsule (4)
        vx = q.x;
        vy = q.y;
        vz = kind == 0 ? q.z : q.z - sclamp(q.z, -size1, size1);
        post = -size0;
    }
    return sqrt(vx * vx + vy * vy + vz * vz) + post;
}

// FP64 parity mode: the per-kind branches only set up sqrt((vx*vx + vy*vy) + vz*vz)
// + post, and the one square root every kind ends in runs after the branches have
// reconverged (lanes of a warp evaluate mixed kinds). Bit-identical to the switch
// above: s + (-r) is s - r, and the cylinder's + 0*0 leaves its 2-D sum unchanged.
// The record is read with 16-byte loads (four, plus four more for a rotation).
template <>
__device__ __forceinline__ double evalPrim<double>(const DPrim<double>& pr, V3<double> p) {
    const double2* v = reinterpret_cast<const double2*>(&pr);
    const double2 a0 = __ldg(v), a1 = __ldg(v + 1), a2 = __ldg(v + 2);
    const int4 a3 = __ldg(reinterpret_cast<const int4*>(v + 3));
    const double size0 = a1.y, size1 = a2.x, size2 = a2.y;
    V3<double> q = p - mk(a0.x, a0.y, a1.x);
    if (!a3.y) {  // transposeMul, vec.hpp:113-117
        const double m0 = __hiloint2double(a3.w, a3.z);
        const double2 r12 = __ldg(v + 4), r34 = __ldg(v + 5), r56 = __ldg(v + 6), r78 = __ldg(v + 7);
        q = mk(m0 * q.x + r34.x * q.y + r56.y * q.z, r12.x * q.x + r34.y * q.y + r78.x * q.z,
               r12.y * q.x + r56.x * q.y + r78.y * q.z);
    }
    return evalKindTail(a3.x, q, size0, size1, size2);
}

// FP32 perf mode: the five kinds as one branch-free formula so lanes evaluating
// different kinds do not serialise. With q = R^T (p - t):
//   u = (radial ? |q.xy| : |q.x|) - e0,  v = radial ? -inf : |q.y| - e1,  w = |q.z| - e2
//   d = |max((u, v, w), 0)| + min(max(u, v, w), 0) - rr      (plane: q.z)
// box (e = half extents), cylinder (radial, e = r, -, h), capsule (radial,
// e = 0, -, h, rr = r) and sphere (radial, e = 0, rr = r) are exactly the
// reference's formulas (primitives.hpp:42-65) in exact arithmetic.
template <>
__device__ __forceinline__ float evalPrim<float>(const DPrim<float>& pr, V3<float> p) {
    const float px = p.x - pr.trans[0], py = p.y - pr.trans[1], pz = p.z - pr.trans[2];
    const float* m = pr.rot;
    const float qx = fmaf(m[0], px, fmaf(m[3], py, m[6] * pz));
    const float qy = fmaf(m[1], px, fmaf(m[4], py, m[7] * pz));
    const float qz = fmaf(m[2], px, fmaf(m[5], py, m[8] * pz));
    const bool radial = pr.e[1] < 0.f;
    const float rho = sqrtf(fmaf(qx, qx, qy * qy));
    const float u = (radial ? rho : fabsf(qx)) - pr.e[0];
    const float v = radial ? -1e30f : fabsf(qy) - pr.e[1];
    const float w = fabsf(qz) - pr.e[2];
    const float ou = fmaxf(u, 0.f), ov = fmaxf(v, 0.f), ow = fmaxf(w, 0.f);
    const float outside = sqrtf(fmaf(ou, ou, fmaf(ov, ov, ow * ow)));
    const float inside = fminf(fmaxf(u, fmaxf(v, w)), 0.f);
    const float d = outside + inside - pr.rr;
    return pr.rr < 0.f ? qz : d;
}

// Primitive records staged in shared memory by the tracing kernels (stagePrims).
// FP64: per primitive the first 64 B of DPrim<double> (translation, size, kind, and
// rot[0]) with the identity flag replaced by the index of its rotation row (-1:
// identity), the rows rot[1..8] (64 B each) after the records; the arithmetic is
// evalPrim<double>'s, so the values are bit-identical. FP32: DPrim<float> as is.
extern __shared__ __align__(128) unsigned char sdfgiDynSmem[];
__device__ __forceinline__ double evalPrimStaged(const unsigned char* base, int rotOff, int j, V3<double> p) {
    const double2* v = reinterpret_cast<const double2*>(base + 64 * static_cast<size_t>(j));
    const double2 a0 = v[0], a1 = v[1], a2 = v[2];
    const int4 a3 = *reinterpret_cast<const int4*>(v + 3);
    const double size0 = a1.y, size1 = a2.x, size2 = a2.y;
    V3<double> q = p - mk(a0.x, a0.y, a1.x);
    if (a3.y >= 0) {  // transposeMul, vec.hpp:113-117
        const double m0 = __hiloint2double(a3.w, a3.z);
        const double2* r = reinterpret_cast<const double2*>(base + rotOff + 64 * static_cast<size_t>(a3.y));
        const double2 r12 = r[0], r34 = r[1], r56 = r[2], r78 = r[3];
        q = mk(m0 * q.x + r34.x * q.y + r56.y * q.z, r12.x * q.x + r34.y * q.y + r78.x * q.z,
               r12.y * q.x + r56.x * q.y + r78.y * q.z);
    }
    return evalKindTail(a3.x, q, size0, size1, size2);
}
// evalPrimitive of CSR primitive j: from the shared-memory copy in kernels that
// staged it (STG), else from global memory.
template <typename R, bool STG>
__device__ __forceinline__ R evalPrimAt(const SceneView<R>& s, int j, V3<R> p) {
    if constexpr (STG) {
        if constexpr (sizeof(R) == 8)
            return evalPrimStaged(sdfgiDynSmem, s.stageRotOff, j, p);
        else
            return evalPrim(reinterpret_cast<const DPrim<float>*>(sdfgiDynSmem)[j], p);
    } else {
        return evalPrim(s.prims[j], p);
    }
}

// evalGradientDetailed / evalGradient, primitives.hpp:96-108 (h = 1e-3)
template <typename R>
__device__ __forceinline__ V3<R> evalGradient(const DPrim<R>& pr, V3<R> p) {
    const R h = R(1e-3);
    V3<R> g = mk(evalPrim(pr, mk(p.x + h, p.y, p.z)) - evalPrim(pr, mk(p.x - h, p.y, p.z)),
                 evalPrim(pr, mk(p.x, p.y + h, p.z)) - evalPrim(pr, mk(p.x, p.y - h, p.z)),
                 evalPrim(pr, mk(p.x, p.y, p.z + h)) - evalPrim(pr, mk(p.x, p.y, p.z - h)));
    R n = length(g);
    if (n < R(1e-6) * R(2) * h) return mk(R(1), R(0), R(0));
    return g / n;
}

// ------------------------------------------------------------------ scene.hpp
// Skip test of queryCore (scene.hpp:231, 299): a cluster is skipped when its box is
// at least the running minimum away (d > 0) or does not contain p (d <= 0).
template <typename R>
__device__ __forceinline__ bool clusterSkipped(const DCluster<R>& cl, V3<R> p, R d) {
    R dx = smax(smax(cl.lo[0] - p.x, p.x - cl.hi[0]), R(0));
    R dy = smax(smax(cl.lo[1] - p.y, p.y - cl.hi[1]), R(0));
    R dz = smax(smax(cl.lo[2] - p.z, p.z - cl.hi[2]), R(0));
    R boxSq = dx * dx + dy * dy + dz * dz;
    return !cl.unbounded && (d > R(0) ? boxSq >= d * d : boxSq > R(0));
}

// queryCore (scene.hpp:214-332): exactly min(naive SDF, initD); owner = the first
// primitive in cluster order attaining it (or -1). Inside the candidate grid a lane
// walks its cell's ascending candidate list, elsewhere every cluster in order.
// The cluster -> member walk is flattened into ONE loop with one primitive
// evaluation per iteration (the next visited cluster's skip tests run when a
// member range is exhausted), so lanes whose lists and clusters differ in length
// stay converged on the evaluation instead of splitting over nested loops.
// Members of one visited cluster: in order with the reference's strict `<`
// (TIE = false), or with the explicit lowest-CSR-position tie-break (TIE = true)
// when clusters are visited out of order.
template <typename R, bool ST, bool TIE, bool STG = false>
__device__ __forceinline__ void visitMembers(const SceneView<R>& s, int k, V3<R> p, R& d, int& own, Counters* c) {
    const int b = s.cstart[k], e = s.cstart[k + 1];
    if (ST) {
        ++c->cv;
        c->pe += e - b;
    }
    for (int j = b; j < e; ++j) {
        if (ST) {
            ++c->ek[s.kindId[j] & 0xff];
            c->ek[5] += (s.kindId[j] >> 8) ? 0 : 1;
        }
        const R pd = evalPrimAt<R, STG>(s, j, p);
        if (pd < d || (TIE && pd == d && own >= 0 && j < own)) {
            d = pd;
            own = j;
        }
    }
}

// An SDF query in flight: the point, the running minimum/owner, and (inside the
// candidate grid) the cursor over the cell's candidate list. queryBegin either
// sets the cursor or — off the grid, or with the grid disabled — completes the
// whole query at once; query() then walks the cell list. Splitting the query
// lets the persistent kernels interleave one evaluation per loop iteration with
// per-lane ray state, so a lane whose query ends early moves on instead of
// waiting for the slowest lane of its warp.
template <typename R> struct QueryState {
    V3<R> p;
    R d;
    R r;  // an upper bound on |p - centre of its cell| (candidate-grid walks)
    int own;
    int cur, end;
    int2 first;  // the list's first entry (from the cell record)
    bool walk;  // the query completes through hierarchyWalk
};

// Off the grid (and behind a truncated cell list): the unbounded clusters, then the
// BVH nearest child first with a short stack. A subtree is dropped only when its
// padded box is strictly farther than the running minimum (ties are visited), so
// the value and (with the CSR tie-break) the owner are exact whatever the running
// minimum was on entry.
template <typename R>
__device__ __forceinline__ R boxDistSq(const float* lo, const float* hi, V3<R> p) {
    R dx = smax(smax(R(lo[0]) - p.x, p.x - R(hi[0])), R(0));
    R dy = smax(smax(R(lo[1]) - p.y, p.y - R(hi[1])), R(0));
    R dz = smax(smax(R(lo[2]) - p.z, p.z - R(hi[2])), R(0));
    return dx * dx + dy * dy + dz * dz;
}
template <typename R>
__device__ __forceinline__ bool boxReaches(R boxSq, R d) {
    return d > R(0) ? boxSq <= d * d : boxSq <= R(0);
}

// The node box tests in float for both precisions (the boxes are float already):
// with p rounded to float, the float box distance is within walkSlack of the exact
// one, so a subtree is kept whenever dist - walkSlack <= d. That keeps every
// subtree the exact test keeps (and a few more): the walk stays exact.
template <typename R, bool ST, bool STG = false>
__device__ __forceinline__ void hierarchyWalk(const SceneView<R>& s, QueryState<R>& q, Counters* c) {
    const GridDev& g = s.grid;
    const V3<R> p = q.p;
    for (int i = 0; i < g.nUnbounded; ++i) visitMembers<R, ST, true, STG>(s, g.unbounded[i], p, q.d, q.own, c);
    if (g.nBounded == 0) return;
    if constexpr (sizeof(R) == 8) {
        // FP64: float box tests with the slack (keep iff |p - box| <= max(d, 0) + slack)
        const V3<float> pf = mk(float(p.x), float(p.y), float(p.z));
        int stackN[kBvhStack];
        float stackB[kBvhStack];
        int sp = 0;
        int next = g.bvhRoot;
        auto reach = [&](float b) {
            const float r = fmaxf(float(q.d), 0.f) * 1.000001f + g.walkSlack;
            return b <= r * r;
        };
        while (true) {
            if (next >= 0) {
                const BNode& n = g.bvh[next];
                const float b0 = boxDistSq<float>(n.lo[0], n.hi[0], pf), b1 = boxDistSq<float>(n.lo[1], n.hi[1], pf);
                const bool k0 = reach(b0), k1 = reach(b1);
                if (k0 && k1) {
                    const int nr = b1 < b0 ? 1 : 0;
                    stackN[sp] = n.child[1 - nr];
                    stackB[sp] = nr ? b0 : b1;
                    ++sp;
                    next = n.child[nr];
                    continue;
                }
                if (k0 || k1) {
                    next = n.child[k0 ? 0 : 1];
                    continue;
                }
                if (ST) c->cs += 2;
            } else {
                visitMembers<R, ST, true, STG>(s, -next - 1, p, q.d, q.own, c);
            }
            bool more = false;
            while (sp > 0) {
                --sp;
                if (reach(stackB[sp])) {
                    next = stackN[sp];
                    more = true;
                    break;
                }
            }
            if (!more) break;
        }
        return;
    }
    int stackN[kBvhStack];
    R stackB[kBvhStack];
    int sp = 0;
    int next = g.bvhRoot;
    while (true) {
        if (next >= 0) {
            const BNode& n = g.bvh[next];
            const R b0 = boxDistSq(n.lo[0], n.hi[0], p), b1 = boxDistSq(n.lo[1], n.hi[1], p);
            const bool k0 = boxReaches(b0, q.d), k1 = boxReaches(b1, q.d);
            if (k0 && k1) {
                const int nr = b1 < b0 ? 1 : 0;
                stackN[sp] = n.child[1 - nr];
                stackB[sp] = nr ? b0 : b1;
                ++sp;
                next = n.child[nr];
                continue;
            }
            if (k0 || k1) {
                next = n.child[k0 ? 0 : 1];
                continue;
            }
            if (ST) c->cs += 2;
        } else {
            visitMembers<R, ST, true, STG>(s, -next - 1, p, q.d, q.own, c);
        }
        // pop the nearest pending subtree still within reach
        bool more = false;
        while (sp > 0) {
            --sp;
            if (boxReaches(stackB[sp], q.d)) {
                next = stackN[sp];
                more = true;
                break;
            }
        }
        if (!more) break;
    }
}

// The candidate-grid cell holding p, or -1 off the grid. With r: also an upper
// bound on p's distance to the cell centre (float, rounded outwards: 1e-5 relative
// covers every rounding of the float arithmetic and of the centre's position).
template <typename R>
__device__ __forceinline__ int gridCell(const GridDev& g, V3<R> p, R* r = nullptr) {
    const bool f32 = sizeof(R) == 4;
    const R lx = f32 ? R(g.flo[0]) : R(g.lo[0]), ly = f32 ? R(g.flo[1]) : R(g.lo[1]);
    const R lz = f32 ? R(g.flo[2]) : R(g.lo[2]), ih = f32 ? R(g.finvH) : R(g.invH);
    R fx = (p.x - lx) * ih;
    R fy = (p.y - ly) * ih;
    R fz = (p.z - lz) * ih;
    if (!(fx >= R(0) && fy >= R(0) && fz >= R(0) && fx < R(g.dim[0]) && fy < R(g.dim[1]) && fz < R(g.dim[2])))
        return -1;
    int ix = min(static_cast<int>(fx), g.dim[0] - 1);
    int iy = min(static_cast<int>(fy), g.dim[1] - 1);
    int iz = min(static_cast<int>(fz), g.dim[2] - 1);
    if (r) {  // (f - i - 1/2) h, in cell units first: no cancellation against the grid origin
        const float dx = static_cast<float>(fx - R(ix)) - 0.5f, dy = static_cast<float>(fy - R(iy)) - 0.5f,
                    dz = static_cast<float>(fz - R(iz)) - 0.5f;
        const float h = static_cast<float>(g.h);
        *r = R(sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) * h * 1.00001f);
    }
    return ix + g.dim[0] * (iy + g.dim[1] * iz);
}

constexpr int kCellUnknown = -2;  // queryBegin computes p's cell itself

// A lane's last cell record: consecutive steps of a march near a surface (and the
// owner / polish queries at a converged point) stay in one cell, and reuse its
// record instead of another dependent load.
struct CellCache {
    int cell = -1;
    int4 rec;
};

// cellHint / rHint: p's candidate-grid cell (-1 off the grid) and distance bound
// when the caller has them already (the persistent kernels' parking test).
template <typename R, bool ST>
__device__ __forceinline__ void queryBegin(const SceneView<R>& s, V3<R> p, R initD, QueryState<R>& q, Counters* c,
                                           int cellHint = kCellUnknown, R rHint = R(0), CellCache* cache = nullptr,
                                           const int4* preRec = nullptr) {
    q.p = p;
    q.d = initD;
    q.own = -1;
    q.cur = q.end = 0;
    q.walk = false;
    if (ST) ++c->q;
    if (!s.useGrid) {
        // the reference's walk: every cluster in order, strict `<`
        for (int k = 0; k < s.n_clusters; ++k) {
            if (clusterSkipped(s.clusters[k], p, q.d)) {
                if (ST) ++c->cs;
                continue;
            }
            visitMembers<R, ST, false>(s, k, p, q.d, q.own, c);
        }
        return;
    }
    const GridDev& g = s.grid;
    q.r = rHint;
    const int cell = cellHint == kCellUnknown ? gridCell<R>(g, p, &q.r) : cellHint;
    if (cell >= 0) {
        int4 rec;
        if (preRec) {
            rec = *preRec;  // loaded by the caller as soon as the cell was known
        } else if (cache && cache->cell == cell) {
            rec = cache->rec;
        } else {
            rec = __ldg(&g.cell[cell]);
            if (cache) {
                cache->cell = cell;
                cache->rec = rec;
            }
        }
        q.cur = rec.x;
        q.end = rec.y;
        q.first = make_int2(rec.z, rec.w);
        if (ST) c->pe += q.end - q.cur;
        return;
    }
    q.walk = true;
}

// The cell list walk (lowest-CSR-position tie-break: order-free), with the next
// entry loaded while the current candidate is evaluated. A truncated list ends in
// a sentinel (-1) whose bound covers every omitted candidate; a query still open
// there completes through the cluster hierarchy.
template <typename R, bool ST, bool STG = false>
__device__ __forceinline__ R query(const SceneView<R>& s, V3<R> p, R initD, int* owner, Counters* c, int seed = -1,
                                   int cellHint = kCellUnknown, R rHint = R(0), CellCache* cache = nullptr,
                                   const int4* preRec = nullptr) {
    QueryState<R> q;
    queryBegin<R, ST>(s, p, initD, q, c, cellHint, rHint, cache, preRec);
    // seed (candidate-grid walks only, which break ties by CSR position in any
    // visiting order): evaluate a likely owner first — e.g. the previous step's
    // — so the hierarchy prunes against a tight minimum from its first node
    if (seed >= 0 && s.useGrid) {
        if (ST) {
            ++c->ek[s.kindId[seed] & 0xff];
            c->ek[5] += (s.kindId[seed] >> 8) ? 0 : 1;
        }
        const R pd = evalPrimAt<R, STG>(s, seed, p);
        if (pd < q.d || (pd == q.d && q.own >= 0 && seed < q.own)) {
            q.d = pd;
            q.own = seed;
        }
    }
    // the dynamic primitives (not in the cell lists), lowest-CSR-position tie-break
    if (s.nDyn && !q.walk) {
        for (int i = 0; i < s.nDyn; ++i) {
            const int j = s.dyn[i];
            if (ST) {
                ++c->ek[s.kindId[j] & 0xff];
                c->ek[5] += (s.kindId[j] >> 8) ? 0 : 1;
            }
            const R pd = evalPrimAt<R, STG>(s, j, p);
            if (pd < q.d || (pd == q.d && q.own >= 0 && j < q.own)) {
                q.d = pd;
                q.own = j;
            }
        }
    }
    if (q.cur < q.end) {
        int2 e = q.first;
        while (true) {
            if (R(__int_as_float(e.x)) > q.d + q.r) break;  // this and every later candidate is farther
            ++q.cur;
            const bool more = q.cur < q.end;
            int2 en = make_int2(0, -1);
            if (more) en = __ldg(&s.grid.entry[q.cur]);
            const int j = e.y;
            if (j < 0) {
                q.walk = true;
                break;
            }
            if (ST) {
                ++c->ek[s.kindId[j] & 0xff];
                c->ek[5] += (s.kindId[j] >> 8) ? 0 : 1;
            }
            const R pd = evalPrimAt<R, STG>(s, j, q.p);
            if (pd < q.d || (pd == q.d && q.own >= 0 && j < q.own)) {
                q.d = pd;
                q.own = j;
            }
            if (!more) break;
            e = en;
        }
    }
    if (q.walk) hierarchyWalk<R, ST, STG>(s, q, c);
    if (owner) *owner = q.own;
    return q.d;
}

template <typename R> struct Hit {
    R t;
    V3<R> pos;
    V3<R> normal;
    int prim;      // CSR position, -1 if none
    int converged;
    int miss;      // 0 None, 1 TMax, 2 StepLimit
    int steps;
};

// Margins sized for the arithmetic: the reference's 1e-9 (scene.hpp:407,412) is
// below float resolution at scene scale.
template <typename R> __device__ __forceinline__ R polishPad(R d);
template <> __device__ __forceinline__ double polishPad<double>(double d) { return d + 1e-9; }
template <> __device__ __forceinline__ float polishPad<float>(float d) { return d + fmaxf(fabsf(d) * 1e-6f, 1e-9f); }

// sphereTrace, scene.hpp:391-435 (2*lastD seeding, polish, owner, normal)
template <typename R, bool ST>
__device__ Hit<R> sphereTrace(const SceneView<R>& s, V3<R> o, V3<R> dir, R tMax, R eps, int maxSteps,
                              Counters* c, R startBound) {
    if (ST) ++c->sphere;
    Hit<R> hit;
    hit.t = R(0);
    hit.pos = mk(R(0), R(0), R(0));
    hit.normal = mk(R(0), R(0), R(1));
    hit.prim = -1;
    hit.converged = 0;
    hit.miss = 0;
    R t = R(0);
    R lastD = startBound * R(0.5);
    for (int step = 0; step < maxSteps; ++step) {
        if (ST) ++c->steps;
        V3<R> p = o + dir * t;
        R d = query<R, ST>(s, p, R(2) * lastD, nullptr, c);
        if (d < eps) {
            int owner = -1;
            d = query<R, ST>(s, p, polishPad(d), &owner, c);
            for (int i = 0; i < 8 && fabs(d) > R(0.25) * eps; ++i) {
                t += d;
                p = o + dir * t;
                int o2 = -1;
                d = query<R, ST>(s, p, polishPad(R(2) * fabs(d)), &o2, c);
                if (o2 >= 0) owner = o2;
            }
            hit.converged = 1;
            hit.t = t;
            hit.pos = p;
            hit.prim = owner;
            hit.steps = step + 1;
            if (owner >= 0) hit.normal = evalGradient(s.prims[owner], p);
            return hit;
        }
        if (d >= tMax - t) {
            hit.miss = 1;
            hit.steps = step + 1;
            return hit;
        }
        t += d;
        lastD = d;
    }
    hit.miss = 2;
    hit.steps = maxSteps;
    return hit;
}

// softShadowTrace, scene.hpp:459-476
template <typename R, bool ST>
__device__ R softShadowTrace(const SceneView<R>& s, V3<R> o, V3<R> dir, R tMin, R tMax, R k, int maxSteps,
                             Counters* c) {
    const R minStep = R(5e-4);
    const R inf = R(INFINITY);
    if (ST) ++c->shadow;
    R v = R(1);
    R t = tMin;
    R lastD = inf;
    for (int step = 0; step < maxSteps && t < tMax; ++step) {
        if (ST) ++c->steps;
        R d = query<R, ST>(s, o + dir * t, lastD == inf ? inf : R(2) * lastD, nullptr, c);
        v = smin(v, sclamp(k * d / t, R(0), R(1)));
        if (v < R(1e-3)) return R(0);
        t += smax(d, minStep);
        lastD = smax(d, minStep);
    }
    return v;
}

// ------------------------------------------------------------- octahedral.hpp
template <typename R> struct V2 {
    R x, y;
};
template <typename R> __device__ __forceinline__ R signNotZero(R v) { return v >= R(0) ? R(1) : R(-1); }
// octEncode, octahedral.hpp:13-24
template <typename R> __device__ __forceinline__ V2<R> octEncode(V3<R> d) {
    R norm = fabs(d.x) + fabs(d.y) + fabs(d.z);
    R px = d.x / norm;
    R py = d.y / norm;
    if (d.z < R(0)) {
        R ox = (R(1) - fabs(py)) * signNotZero(px);
        R oy = (R(1) - fabs(px)) * signNotZero(py);
        px = ox;
        py = oy;
    }
    return V2<R>{px * R(0.5) + R(0.5), py * R(0.5) + R(0.5)};
}
// octDecode, octahedral.hpp:26-36
template <typename R> __device__ __forceinline__ V3<R> octDecode(V2<R> uv) {
    R fx = uv.x * R(2) - R(1);
    R fy = uv.y * R(2) - R(1);
    V3<R> n = mk(fx, fy, R(1) - fabs(fx) - fabs(fy));
    if (n.z < R(0)) {
        R t = -n.z;
        n.x += n.x >= R(0) ? -t : t;
        n.y += n.y >= R(0) ? -t : t;
    }
    return normalize(n);
}

// ------------------------------------------------------------ probe volume
struct CascadeDev {
    int res[3];
    int base;         // first probe of this cascade in the concatenated arrays
    double spacing;
    double origin[3];
    int level;
    int _pad;
};
constexpr int kMaxCascades = 8;

// Probe state, structure-of-arrays over all cascades (concatenated).
struct ProbesView {
    double* pos;       // 3 per probe (AoS xyz: stencil gathers read whole vectors)
    double* rest;      // 3 per probe
    double* last;      // 3 per probe
    int* alive;
    int* reject;
    int* lastFrame;
    double* clear;     // the scene SDF at pos, from the last relocation (its final query)
};

// ProbeAtlas layout (atlas.hpp:119-124): tile (R+2)^2 texels of 3 floats, probe-major.
struct AtlasView {
    const float* __restrict__ data;
    int res;
    int tile;
};

// sampleBilinear, atlas.hpp:59-75 (double arithmetic on float texels in both modes;
// the lookup is 8 per bounce, not a hot loop)
__device__ __forceinline__ V3<double> sampleBilinear(const AtlasView& a, int probe, V2<double> uv) {
    double cx = sclamp(uv.x, 0.0, 1.0) * a.res + 1.0;
    double cy = sclamp(uv.y, 0.0, 1.0) * a.res + 1.0;
    int x0 = static_cast<int>(floor(cx - 0.5));
    int y0 = static_cast<int>(floor(cy - 0.5));
    double tx = cx - 0.5 - x0;
    double ty = cy - 0.5 - y0;
    x0 = iclamp(x0, 0, a.tile - 2);
    y0 = iclamp(y0, 0, a.tile - 2);
    const float* base = a.data + static_cast<size_t>(probe) * a.tile * a.tile * 3;
    auto fetch = [&](int x, int y) {
        const float* p = base + (y * a.tile + x) * 3;
        return mk<double>(__ldg(p), __ldg(p + 1), __ldg(p + 2));
    };
    V3<double> A = lerp(fetch(x0, y0), fetch(x0 + 1, y0), tx);
    V3<double> B = lerp(fetch(x0, y0 + 1), fetch(x0 + 1, y0 + 1), tx);
    return lerp(A, B, ty);
}

// mvcWeightsHex, mean_value.hpp:16-107, in precision M (double in the parity
// mode, float in the perf mode). The same weights with the sines taken
// algebraically from the half angles a_i = asin(l_i / 2): sin(theta_i) =
// 2 sin a_i cos a_i, and sin(h), sin(h - theta_i) by angle addition over
// a_0 + a_1 + a_2 — 3 asin per triangle instead of 3 asin + 7 sin (the values
// agree with the reference's to a few ulps of M). Same degenerate-case branches.
template <typename M> __device__ __forceinline__ M mvcAsin(M v);
// asin on [0, 1] without branches (lanes of a warp fall on both sides of 0.5, and
// the library asin's two paths would run one after the other): z = x, or for
// x > 0.5 z = sqrt((1 - x) / 2) with asin x = pi/2 - 2 asin z; asin z = z + z t P(t),
// t = z^2 <= 1/4, P of degree 11 (Chebyshev fit on [0, 1/4], ~1e-16 relative; the
// fit: scripts/fit_asin.py). Within ~1-2 ulp of the correctly rounded asin.
__device__ __forceinline__ double asinSqrt(double x);  // mvcSqrt<double> (below)
__constant__ const double kAsinP[12] = {
    0.16666666666666624,
    0.07500000000029536,
    0.04464285709453126,
    0.030381947788153375,
    0.022372036498208864,
    0.017355440300771036,
    0.01392777380792154,
    0.011888341648348918,
    0.007745641486205083,
    0.016196107598564897,
    -0.011005663933853308,
    0.028347549339135487};
__device__ __forceinline__ double asin01(double x) {
    const bool big = x > 0.5;
    const double s = asinSqrt(0.5 - 0.5 * x);  // exact argument for x >= 0.5
    const double z = big ? s : x;
    const double t = z * z;
    double p = kAsinP[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) p = fma(p, t, kAsinP[k]);
    const double r = fma(z * t, p, z);
    return big ? 1.5707963267948966 - fma(2.0, r, -6.123233995736766e-17) : r;
}
template <> __device__ __forceinline__ double mvcAsin<double>(double v) { return asin01(v); }
// The same in float (FP32 perf mode): degree-4 P, ~1.5e-7 absolute on [0, 1].
__device__ __forceinline__ float asin01f(float x) {
    const bool big = x > 0.5f;
    const float s = sqrtf(0.5f - 0.5f * x);
    const float z = big ? s : x;
    const float t = z * z;
    const float p = fmaf(fmaf(fmaf(fmaf(0.038085025f, t, 0.026554542f), t, 0.04500138f), t, 0.07498855f), t,
                         0.16666673f);
    const float r = fmaf(z * t, p, z);
    return big ? fmaf(-2.0f, r, 1.57079637f) - 4.37113883e-8f : r;
}
template <> __device__ __forceinline__ float mvcAsin<float>(float v) { return asin01f(v); }
template <typename M> __device__ __forceinline__ M mvcDiv(M a, M b) { return a / b; }
template <> __device__ __forceinline__ float mvcDiv<float>(float a, float b) { return __fdividef(a, b); }
// MVC square roots and reciprocals in FP64: the MUFU seed (rsqrt/rcp.approx.ftz.f64)
// refined by Newton steps in DFMA — within ~1 ulp, branch-free and a third of the
// correctly rounded sequence (12 square roots per triangle). Arguments outside
// [1e-300, 1e300] (zero, denormal, inf, NaN, negative) take the IEEE path.
#ifndef SDFGI_MVC_FAST_SQRT
#define SDFGI_MVC_FAST_SQRT 1
#endif
__device__ __forceinline__ double rsqrtSeed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rcpSeed(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ bool mvcFastRange(double x) { return x > 1e-300 && x < 1e300; }
// the IEEE operations out of line: one copy for every call site, run only by the
// (degenerate) lanes outside the fast range
static __device__ __noinline__ double mvcSqrtIeee(double x) { return sqrt(x); }
static __device__ __noinline__ double mvcRcpIeee(double x) { return 1.0 / x; }
// 1 / sqrt(x): the seed's relative error e0 (~2^-22) -> ~e0^3 after one
// third-order step y (1 + e/2 + 3e^2/8), e = 1 - x y^2.
__device__ __forceinline__ double rsqrtRefined(double x) {
    const double y = rsqrtSeed(x);
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}
template <typename M> __device__ __forceinline__ M mvcSqrt(M x) { return sqrt(x); }
template <> __device__ __forceinline__ double mvcSqrt<double>(double x) {
    if (!SDFGI_MVC_FAST_SQRT) return sqrt(x);
    const double y = rsqrtRefined(x);
    double r = x * y;
    r = fma(fma(-r, r, x), 0.5 * y, r);  // one residual correction of x y
    if (!mvcFastRange(x)) r = mvcSqrtIeee(x);
    return r;
}
template <typename M> __device__ __forceinline__ M mvcRcp(M x) { return M(1) / x; }
template <> __device__ __forceinline__ double mvcRcp<double>(double x) {
    if (!SDFGI_MVC_FAST_SQRT) return 1.0 / x;
    const double a = fabs(x);
    double r = rcpSeed(x);
    r = fma(r, fma(-x, r, 1.0), r);  // e0 -> e0^2
    r = fma(r, fma(-x, r, 1.0), r);  // -> e0^4, below half an ulp
    if (!mvcFastRange(a)) r = mvcRcpIeee(x);
    return r;
}
__device__ __forceinline__ double asinSqrt(double x) { return mvcSqrt<double>(x); }

// The MVC working set (8 distances, unit vectors and weight sums, indexed by the
// triangle corners) lives in per-thread local memory, or — for kernels that pass
// a shared-memory slab (kMvcSlab values per thread, thread-interleaved) — in
// shared memory, which keeps it out of the local-memory traffic of a
// register-capped kernel.
template <typename M, bool SH>
struct MvcArrays;
template <typename M>
struct MvcArrays<M, false> {
    M ld[8], lx[8], ly[8], lz[8], lw[8];
    __device__ MvcArrays(M*) {}
    __device__ M& dist(int i) { return ld[i]; }
    __device__ M& ux(int i) { return lx[i]; }
    __device__ M& uy(int i) { return ly[i]; }
    __device__ M& uz(int i) { return lz[i]; }
    __device__ M& wts(int i) { return lw[i]; }
};
template <typename M>
struct MvcArrays<M, true> {
    M* b;  // this thread's column of the slab
    int s;
    __device__ explicit MvcArrays(M* slab) : b(slab + threadIdx.x), s(blockDim.x) {}
    __device__ M& dist(int i) { return b[i * s]; }
    __device__ M& ux(int i) { return b[(8 + i) * s]; }
    __device__ M& uy(int i) { return b[(16 + i) * s]; }
    __device__ M& uz(int i) { return b[(24 + i) * s]; }
    __device__ M& wts(int i) { return b[(32 + i) * s]; }
};
constexpr int kMvcSlab = 40;  // values per thread in a shared slab

// The 8 corners of a cascade cell: probe positions read straight from the probe
// array (corner k = cell + (k & 1, k >> 1 & 1, k >> 2 & 1)), no local copy.
struct CellCorners {
    const double* pos;  // probe positions, xyz per probe
    int p0, dy, dz;     // global index of corner 0, strides in y and z
    __device__ int index(int k) const { return p0 + (k & 1) + ((k >> 1) & 1) * dy + ((k >> 2) & 1) * dz; }
    __device__ V3<double> corner(int k) const {
        const double* P = pos + 3 * static_cast<size_t>(index(k));
        return mk(P[0], P[1], P[2]);
    }
};

// Triangulated hex faces (mean_value.hpp:18-20): warp-uniform loop index, so one
// broadcast constant load per corner instead of a local-memory table.
__constant__ const int kMvcFaces[6][4] = {{0, 2, 3, 1}, {4, 5, 7, 6}, {0, 1, 5, 4}, {2, 6, 7, 3}, {0, 4, 6, 2}, {1, 3, 7, 5}};

// The angle of one triangle edge (mean_value.hpp:53-55): theta = 2 asin(|u_a - u_b| / 2),
// returned as sin and cos of the half angle a = theta / 2 and theta itself. The
// value depends only on the unordered pair (u_a - u_b = -(u_b - u_a) exactly), so
// the two triangles sharing an edge can share it.
template <typename M>
__device__ __forceinline__ void mvcEdgeAngles(V3<M> ua, V3<M> ub, M& sa, M& ca, M& th) {
    const V3<M> e = ua - ub;
    const M l = mvcSqrt<M>(dot(e, e));
    sa = sclamp(l * M(0.5), M(0), M(1));
    ca = mvcSqrt<M>(smax(M(0), M(1) - sa * sa));
    th = M(2) * mvcAsin<M>(sa);
}
// sign(det(u0, u1, u2)) (mean_value.hpp:73-74)
template <typename M>
__device__ __forceinline__ M mvcSign(V3<M> u0, V3<M> u1, V3<M> u2) {
    V3<M> cr = mk(u1.y * u2.z - u1.z * u2.y, u1.z * u2.x - u1.x * u2.z, u1.x * u2.y - u1.y * u2.x);
    return dot(u0, cr) >= M(0) ? M(1) : M(-1);
}

// One triangle of mvcWeightsHex's loop (mean_value.hpp:45-97) from its corners'
// distances d, its edge angles (sa, ca, theta: the edge opposite corner i) and
// the orientation sign. Returns kTriSkip (degenerate, mean_value.hpp:80-89: no
// contribution), kTriAdd (w = the three weight contributions, :91-96), kTriOn (x
// on the triangle: w = its normalised 2D barycentric weights, :57-71) or kTriFail
// (on the triangle but degenerate: mvcWeightsHex returns false).
constexpr int kTriSkip = 0, kTriAdd = 1, kTriOn = 2, kTriFail = 3;
template <typename M>
__device__ __forceinline__ int mvcTriangleCore(const M d[3], const M sa[3], const M ca[3], const M theta[3], M sign,
                                               M w[3]) {
    const M eps = M(1e-10);
    const M pi = M(kPi);
    M st[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) st[i] = M(2) * sa[i] * ca[i];
    const M h = (theta[0] + theta[1] + theta[2]) * M(0.5);
    if (pi - h < M(1e-8)) {
        M total = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            w[i] = st[i] * d[(i + 1) % 3] * d[(i + 2) % 3];
            total += w[i];
        }
        if (total < eps) return kTriFail;
#pragma unroll
        for (int i = 0; i < 3; ++i) w[i] = w[i] / total;
        return kTriOn;
    }
    // sin h, h = a0 + a1 + a2
    const M sh = sa[0] * ca[1] * ca[2] + ca[0] * sa[1] * ca[2] + ca[0] * ca[1] * sa[2] - sa[0] * sa[1] * sa[2];
    M c[3], sv[3];
    bool skip = false;
    // FP64: the three divisions by st_j st_k through one reciprocal of
    // st_0 st_1 st_2 (1 / (st_j st_k) = st_i / P; a few ulps, far inside the
    // range: a triangle with a product below eps is skipped)
    const M invP = sizeof(M) == 8 ? mvcRcp<M>(st[0] * st[1] * st[2]) : M(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3, k = (i + 2) % 3;
        const M denom = st[j] * st[k];
        // sin(h - theta_i) = sin(a_j + a_k - a_i)
        const M sjk = sa[j] * ca[k] + ca[j] * sa[k], cjk = ca[j] * ca[k] - sa[j] * sa[k];
        const M shi = sjk * ca[i] - cjk * sa[i];
        if (sizeof(M) == 8)
            c[i] = M(2) * sh * shi * (st[i] * invP) - M(1);
        else
            c[i] = mvcDiv(M(2) * sh * shi, denom) - M(1);
        sv[i] = sign * mvcSqrt<M>(smax(M(0), M(1) - c[i] * c[i]));
        // the reference stops at the first degenerate i (mean_value.hpp:80-86);
        // the values after it are unused either way
        skip = skip || fabs(denom) < eps || fabs(sv[i]) <= eps;
    }
    if (skip) return kTriSkip;
    M D[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) D[i] = d[i] * st[(i + 1) % 3] * sv[(i + 2) % 3];
    const M invQ = sizeof(M) == 8 ? mvcRcp<M>(D[0] * D[1] * D[2]) : M(0);  // FP64: one reciprocal
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3, k = (i + 2) % 3;
        const M num = theta[i] - c[j] * theta[k] - c[k] * theta[j];
        w[i] = sizeof(M) == 8 ? num * (D[j] * D[k] * invQ) : mvcDiv(num, D[i]);
    }
    return kTriAdd;
}
template <typename M>
__device__ __forceinline__ int mvcTriangle(const M d[3], const V3<M> u[3], M w[3]) {
    M sa[3], ca[3], theta[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) mvcEdgeAngles(u[(i + 1) % 3], u[(i + 2) % 3], sa[i], ca[i], theta[i]);
    return mvcTriangleCore<M>(d, sa, ca, theta, mvcSign(u[0], u[1], u[2]), w);
}

// Result: the weights in a.wts(0..7) (precision M; the caller widens to double).
template <typename M, bool SH>
__device__ inline bool mvcWeightsHexImpl(const CellCorners& cc, V3<double> xd, MvcArrays<M, SH>& a) {
    const M eps = M(1e-10);
    for (int i = 0; i < 8; ++i) a.wts(i) = M(0);
    const V3<M> x = mk(M(xd.x), M(xd.y), M(xd.z));
    for (int i = 0; i < 8; ++i) {
        const V3<double> ci = cc.corner(i);
        V3<M> v = mk(M(ci.x), M(ci.y), M(ci.z)) - x;
        const M di = mvcSqrt<M>(dot(v, v));
        a.dist(i) = di;
        if (di < eps) {
            for (int k = 0; k < 8; ++k) a.wts(k) = M(0);
            a.wts(i) = M(1);
            return true;
        }
        const M inv = sizeof(M) == 8 ? mvcRcp<M>(di) : mvcDiv(M(1), di);
        a.ux(i) = v.x * inv;
        a.uy(i) = v.y * inv;
        a.uz(i) = v.z * inv;
    }
    bool any = false;
#pragma unroll 1
    for (int t = 0; t < 12; ++t) {
        const int f = t >> 1, tr = t & 1;
        const int tri[3] = {kMvcFaces[f][0], kMvcFaces[f][tr ? 2 : 1], kMvcFaces[f][tr ? 3 : 2]};
        M d[3], w[3];
        V3<M> u[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            d[i] = a.dist(tri[i]);
            u[i] = mk(a.ux(tri[i]), a.uy(tri[i]), a.uz(tri[i]));
        }
        const int r = mvcTriangle<M>(d, u, w);
        if (r == kTriFail) return false;
        if (r == kTriOn) {
            for (int k = 0; k < 8; ++k) a.wts(k) = M(0);
#pragma unroll
            for (int i = 0; i < 3; ++i) a.wts(tri[i]) = w[i];
            return true;
        }
        if (r == kTriSkip) continue;
#pragma unroll
        for (int i = 0; i < 3; ++i) a.wts(tri[i]) += w[i];
        any = true;
    }
    if (!any) return false;
    M total = 0;
    for (int i = 0; i < 8; ++i) total += a.wts(i);
    if (fabs(total) < eps || !isfinite(total)) return false;
    for (int i = 0; i < 8; ++i) a.wts(i) = a.wts(i) / total;
    return true;
}

struct Stencil {
    int cascade;      // chosen cascade slot (-1: sky fallback)
    int probe[8];     // probe index within the cascade
    double w[8];
    int count;
    int sky;
    int usedMvc;
};

// interpolationStencil's cell selection (probe_volume.hpp:224-278): the finest
// containing cascade, the cell, its trilinear coordinates and whether the MVC path
// is taken. chosen < 0: no cascade contains the point (sky fallback).
struct StencilCell {
    int chosen;
    CellCorners cc;
    double tx, ty, tz;
    bool wantMvc;
    bool boundary;  // InterpolationStencil::crossCascade (probe_volume.hpp:276)
};
// checkMvc = false: the caller knows the MVC test fails (wantMvc stays false).
__device__ inline StencilCell stencilCell(const CascadeDev* cas, int nCas, const ProbesView& pv, V3<double> point,
                                          double mvcFrac, bool checkMvc = true) {
    StencilCell sc;
    sc.chosen = -1;
    sc.wantMvc = false;
    sc.boundary = false;
    sc.tx = sc.ty = sc.tz = 0;
    int chosen = -1;
    int cell[3] = {0, 0, 0};
    int containing = 0;
    for (int ci = 0; ci < nCas; ++ci) {
        const CascadeDev& c = cas[ci];
        V3<double> f = (point - mk(c.origin[0], c.origin[1], c.origin[2])) / c.spacing;
        int ix = static_cast<int>(floor(f.x));
        int iy = static_cast<int>(floor(f.y));
        int iz = static_cast<int>(floor(f.z));
        bool inside = ix >= 0 && ix + 1 < c.res[0] && iy >= 0 && iy + 1 < c.res[1] && iz >= 0 && iz + 1 < c.res[2];
        if (!inside) continue;
        ++containing;
        if (chosen < 0 || c.spacing < cas[chosen].spacing) {
            chosen = ci;
            cell[0] = ix;
            cell[1] = iy;
            cell[2] = iz;
        }
    }
    if (chosen < 0) return sc;
    bool insideCoarser = containing > 1;
    const CascadeDev& c = cas[chosen];
    V3<double> f = (point - mk(c.origin[0], c.origin[1], c.origin[2])) / c.spacing;
    sc.chosen = chosen;
    sc.tx = f.x - cell[0];
    sc.ty = f.y - cell[1];
    sc.tz = f.z - cell[2];
    sc.cc = CellCorners{pv.pos, c.base + cell[0] + c.res[0] * (cell[1] + c.res[1] * cell[2]), c.res[0],
                        c.res[0] * c.res[1]};
    const CellCorners& cc = sc.cc;
    bool boundary = insideCoarser && (cell[0] == 0 || cell[0] + 2 == c.res[0] || cell[1] == 0 ||
                                      cell[1] + 2 == c.res[1] || cell[2] == 0 || cell[2] + 2 == c.res[2]);
    // maxDisp > mvcFrac * spacing (probe_volume.hpp:263-278) is "some corner's displacement
    // length exceeds the threshold": decided on the squared length with a 1e-9
    // relative margin either side of thr^2 (sqrt is correctly rounded and
    // monotone, so outside the margin the answer is the same), the exact sqrt only
    // inside it; NaN lengths never count, as in the max
    const double thr = mvcFrac * c.spacing;
    const double thr2 = thr * thr;
    const bool squared = thr > 0 && thr2 > 1e-280 && thr2 < 1e280;
    bool wantMvc = checkMvc && (boundary || thr < 0);  // maxDisp >= 0 > thr
    for (int k = 0; k < 8 && checkMvc && !wantMvc; ++k) {
        const double* Q = pv.rest + 3 * static_cast<size_t>(cc.index(k));
        const V3<double> dv = cc.corner(k) - mk(Q[0], Q[1], Q[2]);
        const double d2 = dot(dv, dv);
        if (squared && d2 > thr2 * (1 + 1e-9))
            wantMvc = true;
        else if (!squared || !(d2 < thr2 * (1 - 1e-9)))
            wantMvc = sqrt(d2) > thr;
    }
    sc.wantMvc = wantMvc;
    sc.boundary = boundary;
    return sc;
}

// trilinear weight of corner k (probe_volume.hpp:290-296)
__device__ __forceinline__ double trilinearWeight(const StencilCell& sc, int k) {
    double wx = (k & 1) ? sc.tx : 1 - sc.tx;
    double wy = ((k >> 1) & 1) ? sc.ty : 1 - sc.ty;
    double wz = ((k >> 2) & 1) ? sc.tz : 1 - sc.tz;
    return wx * wy * wz;
}

// interpolationStencil's ending (probe_volume.hpp:297-309) from the cell's 8
// weights: dead corners get 0, the sum must exceed 1e-12 (else sky fallback), the
// weights are normalised.
__device__ inline Stencil finishStencil(const CascadeDev* cas, const ProbesView& pv, const StencilCell& sc, double* w,
                                        int usedMvc) {
    Stencil st;
    st.count = 0;
    st.sky = 0;
    st.usedMvc = usedMvc;
    st.cascade = -1;
    const CellCorners& cc = sc.cc;
    double sum = 0;
    for (int k = 0; k < 8; ++k) {
        if (!pv.alive[cc.index(k)]) w[k] = 0;
        sum += w[k];
    }
    if (sum <= 1e-12) {
        st.sky = 1;
        return st;
    }
    const int base = cas[sc.chosen].base;
    for (int k = 0; k < 8; ++k) {
        st.probe[k] = cc.index(k) - base;
        st.w[k] = w[k] / sum;
    }
    st.cascade = sc.chosen;
    st.count = 8;
    return st;
}

// interpolationStencil, probe_volume.hpp:224-310 (cell and trilinear weights in
// double in both modes; MVC in precision M)
// SLAB_ONLY: the caller always passes a shared slab, so only that variant of the
// MVC is compiled in (a second inlined copy cost instruction-cache misses).
template <typename M = double, bool SLAB_ONLY = false>
__device__ inline Stencil interpolationStencil(const CascadeDev* cas, int nCas, const ProbesView& pv, V3<double> point,
                                        double mvcFrac, M* slab = nullptr) {
    Stencil st;
    st.count = 0;
    st.sky = 0;
    st.usedMvc = 0;
    st.cascade = -1;
    const StencilCell sc = stencilCell(cas, nCas, pv, point, mvcFrac);
    if (sc.chosen < 0) {
        st.sky = 1;
        return st;
    }
    const CellCorners& cc = sc.cc;
    double w[8];
    bool haveMvc = false;
    if (sc.wantMvc) {
        if (SLAB_ONLY || slab) {
            MvcArrays<M, true> a(slab);
            haveMvc = mvcWeightsHexImpl<M, true>(cc, point, a);
            if (haveMvc)
                for (int k = 0; k < 8; ++k) w[k] = double(a.wts(k));
        } else if (!SLAB_ONLY) {
            MvcArrays<M, false> a(slab);
            haveMvc = mvcWeightsHexImpl<M, false>(cc, point, a);
            if (haveMvc)
                for (int k = 0; k < 8; ++k) w[k] = double(a.wts(k));
        }
        if (haveMvc) {
            for (int k = 0; k < 8; ++k) w[k] = smax(0.0, w[k]);
            st.usedMvc = 1;
        }
    }
    if (!haveMvc)
        for (int k = 0; k < 8; ++k) w[k] = trilinearWeight(sc, k);
    return finishStencil(cas, pv, sc, w, st.usedMvc);
}

// sampleBounceIrradiance's lookup (probe_update.hpp:70-91) from a finished stencil:
// backface weight ((cos+1)/2)^2 per probe, renormalised, 8 bilinear lookups at
// octEncode(normal). Returns false when "empty".
template <typename M = double>
__device__ inline bool bounceFromStencil(const CascadeDev* cas, const ProbesView& pv, const float* atlas, int oct,
                                         const Stencil& st, V3<double> pos, V3<double> normal, V3<double>* out) {
    if (st.sky || st.count == 0) return false;
    const CascadeDev& c = cas[st.cascade];
    double wsum = 0;
    double w[8];
    // a finished stencil has 8 entries (count is 0 or 8): fixed trip counts keep
    // the arrays in registers
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w[i] = 0;
        if (st.w[i] <= 0) continue;
        const double* P = pv.pos + 3 * static_cast<size_t>(c.base + st.probe[i]);
        V3<double> toProbe = mk(P[0], P[1], P[2]) - pos;
        double facing;
        if constexpr (sizeof(M) == 4) {  // FP32 perf mode: one float reciprocal
            const V3<float> tp = mk(float(toProbe.x), float(toProbe.y), float(toProbe.z));
            const float len = length(tp);
            facing = len > 1e-9f ? double(dot(tp, mk(float(normal.x), float(normal.y), float(normal.z))) * (1.f / len))
                                 : 1.0;
        } else {
            double len = length(toProbe);
            facing = len > 1e-9 ? dot(toProbe / len, normal) : 1.0;
        }
        double backface = (facing + 1.0) * 0.5;
        w[i] = st.w[i] * backface * backface;
        wsum += w[i];
    }
    if (wsum <= 1e-12) return false;
    V3<double> acc = mk(0.0, 0.0, 0.0);
    V2<double> uv = octEncode(normal);
    AtlasView av{atlas, oct, oct + 2};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (w[i] <= 0) continue;
        acc = acc + sampleBilinear(av, c.base + st.probe[i], uv) * (w[i] / wsum);
    }
    *out = acc;
    return true;
}

// sampleBounceIrradiance, probe_update.hpp:63-92. Returns false when "empty".
template <typename M = double, bool SLAB_ONLY = false>
__device__ inline bool sampleBounceIrradiance(const CascadeDev* cas, int nCas, const ProbesView& pv,
                                       const float* atlas, int oct, V3<double> pos, V3<double> normal,
                                       double mvcFrac, V3<double>* out, M* slab = nullptr, int* usedMvc = nullptr) {
    if (nCas <= 0) return false;
    Stencil st = interpolationStencil<M, SLAB_ONLY>(cas, nCas, pv, pos, mvcFrac, slab);
    if (usedMvc) *usedMvc = st.usedMvc;
    return bounceFromStencil<M>(cas, pv, atlas, oct, st, pos, normal, out);
}

// Everything updateProbe / contactGI needs from RenderConfig (config.hpp:9-50).
struct TraceCfg {
    double eps;
    double rayTMax;
    double shadowK;
    double bounceCoeff;
    double mvcFrac;
    int maxSteps;
    int shadowSteps;
    double shadowMinStep;  // softShadowTrace's minStep (scene.hpp:462); 0 = the default 5e-4
};

// directIrradiance, probe_update.hpp:97-132
template <typename R, bool ST>
__device__ V3<double> directIrradiance(const SceneView<R>& s, V3<R> pos, V3<R> normal, const TraceCfg& cfg,
                                       Counters* c) {
    V3<double> total = mk(0.0, 0.0, 0.0);
    for (int li = 0; li < s.n_lights; ++li) {
        const DLight& L = s.lights[li];
        V3<R> dir;
        R tMax;
        V3<double> unshadowed;
        V3<double> I = mk(L.intensity[0], L.intensity[1], L.intensity[2]);
        if (L.kind == 0) {
            V3<R> toLight = mk(R(L.position[0]), R(L.position[1]), R(L.position[2])) - pos;
            R r2 = dot(toLight, toLight);
            if (r2 < R(1e-12)) continue;
            R r = sqrt(r2);
            dir = toLight / r;
            R cosT = dot(normal, dir);
            if (cosT <= R(0)) continue;
            unshadowed = I * static_cast<double>(cosT / r2);
            tMax = r;
        } else if (L.kind == 1) {
            dir = mk(R(-L.direction[0]), R(-L.direction[1]), R(-L.direction[2]));
            R cosT = dot(normal, dir);
            if (cosT <= R(0)) continue;
            unshadowed = I * static_cast<double>(cosT);
            tMax = R(cfg.rayTMax);
        } else {
            continue;
        }
        R cosT = dot(normal, dir);
        R bias = R(2.0) * R(cfg.eps) / smax(R(0.1), cosT);
        R vis = R(1);
        if (tMax - bias > bias)
            vis = softShadowTrace<R, ST>(s, pos + normal * bias, dir, bias, tMax - bias, R(cfg.shadowK),
                                         cfg.shadowSteps, c);
        total = total + unshadowed * static_cast<double>(vis);
    }
    return total;
}

// shadeHit, probe_update.hpp:136-149 (converged hit with owner `prim` in CSR order)
template <typename R, bool ST>
__device__ V3<double> shadeHit(const SceneView<R>& s, const Hit<R>& hit, const CascadeDev* cas, int nCas,
                               const ProbesView& pv, const float* prevAtlas, int oct, const TraceCfg& cfg,
                               Counters* c) {
    if (hit.prim < 0) return mk(s.sky[0], s.sky[1], s.sky[2]);
    const double* A = s.albedo + 3 * hit.prim;
    const double* E = s.emission + 3 * hit.prim;
    V3<double> brdf = mk(A[0], A[1], A[2]) / kPi;
    V3<double> direct = directIrradiance<R, ST>(s, hit.pos, hit.normal, cfg, c);
    V3<double> radiance = mk(E[0], E[1], E[2]) + brdf * direct;
    if (cfg.bounceCoeff > 0 && prevAtlas != nullptr) {
        V3<double> prev;
        V3<double> hp = mk<double>(hit.pos.x, hit.pos.y, hit.pos.z);
        V3<double> hn = mk<double>(hit.normal.x, hit.normal.y, hit.normal.z);
        if (sampleBounceIrradiance<R>(cas, nCas, pv, prevAtlas, oct, hp, hn, cfg.mvcFrac, &prev))
            radiance = radiance + brdf * (prev * cfg.bounceCoeff);
    }
    return radiance;
}

// randomRotation's matrix from its quaternion (rng.hpp:79-89), row-major into m.
// The quaternion's sines/cosines come from the host's libm (host_trig.h).
__device__ __forceinline__ void quatToRotation(double qx, double qy, double qz, double qw, double* m) {
    m[0] = 1 - 2 * (qy * qy + qz * qz);
    m[1] = 2 * (qx * qy - qz * qw);
    m[2] = 2 * (qx * qz + qy * qw);
    m[3] = 2 * (qx * qy + qz * qw);
    m[4] = 1 - 2 * (qx * qx + qz * qz);
    m[5] = 2 * (qy * qz - qx * qw);
    m[6] = 2 * (qx * qz - qy * qw);
    m[7] = 2 * (qy * qz + qx * qw);
    m[8] = 1 - 2 * (qx * qx + qy * qy);
}

// cosineHemisphereDir (rng.hpp:58-69) with orthonormalBasis (vec.hpp:188-194);
// lx = r cos(phi), ly = r sin(phi) come from the host's libm (host_trig.h).
__device__ __forceinline__ V3<double> cosineHemisphereDir(double lx, double ly, double u1, V3<double> n) {
    double lz = sqrt(smax(0.0, 1.0 - u1));
    double sign = copysign(1.0, n.z);
    double a = -1.0 / (sign + n.z);
    double c = n.x * n.y * a;
    V3<double> t = mk(1.0 + sign * n.x * n.x * a, sign * c, -sign * n.x);
    V3<double> b = mk(c, sign + n.y * n.y * a, -n.y);
    return normalize(t * lx + b * ly + n * lz);
}

}  // namespace sdfgi_dev
