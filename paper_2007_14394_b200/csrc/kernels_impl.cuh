// kernels_impl.cuh — kernel bodies, included once per precision translation unit.
#pragma once

#include "kernels.cuh"

namespace sdfgi_dev {

__device__ __forceinline__ int cascadeOf(const ProbeCommon& pc, int gp) {
    int ci = 0;
    for (int k = 1; k < pc.nCas; ++k)
        if (gp >= pc.cas[k].base) ci = k;
    return ci;
}

__device__ __forceinline__ void flushCounters(const Counters& c, unsigned long long* out) {
    // warp reduce then one atomic per warp per counter
    unsigned long long v[14] = {c.q,     c.cv,    c.cs,    c.pe,    c.steps, c.sphere, c.shadow,
                                c.vis,   c.ek[0], c.ek[1], c.ek[2], c.ek[3], c.ek[4],  c.ek[5]};
#pragma unroll
    for (int i = 0; i < 14; ++i) {
        unsigned long long x = v[i];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(out + i, x);
    }
}

// ------------------------------------------------------------ (d) relocation
// updateProbePositions, probe_volume.hpp:99-143, one thread per probe of one cascade.
template <bool ST>
__global__ void __launch_bounds__(128) k_relocate(RelocParams P) {
    const CascadeDev& c = P.pc.cas[P.cascade];
    const int n = c.res[0] * c.res[1] * c.res[2];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    Counters cnt;
    cnt.zero();
    int relocated = 0, rejected = 0, dead = 0;
    if (i < n) {
        const int gp = c.base + i;
        const ProbesView& pv = P.pc.probes;
        const SceneView<double>& s = P.scene;
        const double inf = INFINITY;
        V3<double> prev = mk(pv.pos[3 * gp], pv.pos[3 * gp + 1], pv.pos[3 * gp + 2]);
        V3<double> rest = mk(pv.rest[3 * gp], pv.rest[3 * gp + 1], pv.rest[3 * gp + 2]);
        V3<double> pos = rest;
        double budgetTotal = 0.5 * c.spacing;
        double d = query<double, ST>(s, pos, inf, nullptr, &cnt);
        bool alive = true;
        if (d < P.th1) {
            double budget = budgetTotal;
            const double h = P.gradStep;
            for (int step = 0; step < P.maxSteps && d < P.th1 && budget > 0; ++step) {
                // sceneGradient, scene.hpp:360-371
                V3<double> g = mk(query<double, ST>(s, mk(pos.x + h, pos.y, pos.z), inf, nullptr, &cnt) -
                                      query<double, ST>(s, mk(pos.x - h, pos.y, pos.z), inf, nullptr, &cnt),
                                  query<double, ST>(s, mk(pos.x, pos.y + h, pos.z), inf, nullptr, &cnt) -
                                      query<double, ST>(s, mk(pos.x, pos.y - h, pos.z), inf, nullptr, &cnt),
                                  query<double, ST>(s, mk(pos.x, pos.y, pos.z + h), inf, nullptr, &cnt) -
                                      query<double, ST>(s, mk(pos.x, pos.y, pos.z - h), inf, nullptr, &cnt));
                double gn = length(g);
                V3<double> dir = (gn < 1e-6 * 2 * h) ? mk(1.0, 0.0, 0.0) : g / gn;
                double want = smin((P.th1 - d) * 1.25, budget);
                pos = pos + dir * want;
                budget -= want;
                d = query<double, ST>(s, pos, inf, nullptr, &cnt);
            }
            alive = d >= P.th1;
            if (alive && length(pos - rest) > 1e-12) ++relocated;
        }
        pv.last[3 * gp] = prev.x;
        pv.last[3 * gp + 1] = prev.y;
        pv.last[3 * gp + 2] = prev.z;
        pv.pos[3 * gp] = pos.x;
        pv.pos[3 * gp + 1] = pos.y;
        pv.pos[3 * gp + 2] = pos.z;
        if (!alive) {
            ++dead;
            pv.alive[gp] = 0;
        } else {
            pv.alive[gp] = 1;
            bool hadHistory = pv.lastFrame[gp] >= 0 && !pv.reject[gp];
            if (length(pos - prev) > P.th2) {
                pv.reject[gp] = 1;
                if (hadHistory) ++rejected;
            }
        }
    }
    // block-aggregated report
    for (int o = 16; o > 0; o >>= 1) {
        relocated += __shfl_xor_sync(0xffffffffu, relocated, o);
        rejected += __shfl_xor_sync(0xffffffffu, rejected, o);
        dead += __shfl_xor_sync(0xffffffffu, dead, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (relocated) atomicAdd(P.report + 0, relocated);
        if (rejected) atomicAdd(P.report + 1, rejected);
        if (dead) atomicAdd(P.report + 2, dead);
    }
    if (ST) flushCounters(cnt, P.stats);
}

// ---------------------------------------------------------- (a)(b)(c) update
template <typename R, bool ST>
__device__ __forceinline__ V3<double> traceAndShade(const UpdateParams<R>& P, V3<double> origin, V3<double> dir,
                                                    Counters* cnt, Hit<R>* hitOut) {
    const TraceCfg& tc = P.tc;
    V3<R> o = mk(R(origin.x), R(origin.y), R(origin.z));
    V3<R> d = mk(R(dir.x), R(dir.y), R(dir.z));
    Hit<R> hit = sphereTrace<R, ST>(P.scene, o, d, R(tc.rayTMax), R(tc.eps), tc.maxSteps, cnt, R(INFINITY));
    if (hitOut) *hitOut = hit;
    if (hit.converged)
        return shadeHit<R, ST>(P.scene, hit, P.pc.cas, P.pc.nCas, P.pc.probes, P.prevAtlas, P.oct, tc, cnt);
    return mk(P.scene.sky[0], P.scene.sky[1], P.scene.sky[2]);
}

template <typename R, bool ST>
__global__ void __launch_bounds__(kUpdateThreads) k_probe_update(UpdateParams<R> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double rot[9];
    __shared__ __align__(16) float tile[12 * 12 * 3 + 4];
    __shared__ unsigned long long redDelta[kUpdateThreads / 32];

    const int gp = P.refs ? P.refs[blockIdx.x] : static_cast<int>(blockIdx.x);
    const ProbesView& pv = P.pc.probes;
    if (!pv.alive[gp]) return;  // pipeline.hpp:141; its back tile is the copied front tile
    const int ci = cascadeOf(P.pc, gp);
    const int level = P.pc.cas[ci].level;
    const int local = gp - P.pc.cas[ci].base;
    const int reject = pv.reject[gp];
    const int n = reject ? 2 * P.nRaysFull : P.nRaysFull;
    const V3<double> origin = mk(pv.pos[3 * gp], pv.pos[3 * gp + 1], pv.pos[3 * gp + 2]);

    R* sdir = reinterpret_cast<R*>(smem_raw);        // 3n
    R* srad = sdir + 3 * n;                           // 3n

    if (threadIdx.x == 0)
        probeRotation(P.seed, P.frame, P.rotatePerFrame != 0, probeKey(level, local), rot);
    __syncthreads();

    Counters cnt;
    cnt.zero();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        V3<double> dir = probeRayDir(rot, i, n);
        V3<double> L = traceAndShade<R, ST>(P, origin, dir, &cnt, nullptr);
        sdir[3 * i] = R(dir.x);
        sdir[3 * i + 1] = R(dir.y);
        sdir[3 * i + 2] = R(dir.z);
        srad[3 * i] = R(L.x);
        srad[3 * i + 1] = R(L.y);
        srad[3 * i + 2] = R(L.z);
    }
    __syncthreads();

    // convolveIrradiance + hysteresis blend (probe_update.hpp:25-34,192-206)
    const int res = P.oct;
    const int T = res + 2;
    const double alpha = reject ? 1.0
                                : sclamp((1.0 - P.hysteresis) * n / P.nRaysFull, P.alphaMin, 1.0);
    const double scale = 4.0 * kPi / static_cast<double>(n);
    const float* oldTile = P.prevAtlas + static_cast<size_t>(gp) * T * T * 3;
    double maxDelta = 0.0;
    for (int tx = threadIdx.x; tx < res * res; tx += blockDim.x) {
        const int y = tx / res, x = tx % res;
        V3<R> D;
        {
            V3<double> dd = octDecode(V2<double>{(x + 0.5) / res, (y + 0.5) / res});
            D = mk(R(dd.x), R(dd.y), R(dd.z));
        }
        R ax = 0, ay = 0, az = 0;
        for (int i = 0; i < n; ++i) {
            R w = D.x * sdir[3 * i] + D.y * sdir[3 * i + 1] + D.z * sdir[3 * i + 2];
            if (w > R(0)) {
                ax = ax + srad[3 * i] * w;
                ay = ay + srad[3 * i + 1] * w;
                az = az + srad[3 * i + 2] * w;
            }
        }
        V3<double> fresh = mk(double(ax), double(ay), double(az)) * scale;
        const float* o = oldTile + ((y + 1) * T + (x + 1)) * 3;
        V3<double> old = mk<double>(o[0], o[1], o[2]);
        V3<double> bl = lerp(old, fresh, alpha);
        V3<double> df = bl - old;
        maxDelta = smax(maxDelta, maxComponent(mk(fabs(df.x), fabs(df.y), fabs(df.z))));
        float* t = tile + ((y + 1) * T + (x + 1)) * 3;
        t[0] = static_cast<float>(bl.x);
        t[1] = static_cast<float>(bl.y);
        t[2] = static_cast<float>(bl.z);
    }
    __syncthreads();
    // fillBorder, atlas.hpp:44-56: edges copy the adjacent interior row/column
    // reversed, corners the diagonally opposite interior corner.
    for (int k = threadIdx.x; k < 4 * res + 4; k += blockDim.x) {
        int dx, dy, sx, sy;
        if (k < 4 * res) {
            const int i = k / 4 + 1, e = k % 4;
            if (e == 0) { dx = i; dy = 0; sx = res + 1 - i; sy = 1; }
            else if (e == 1) { dx = i; dy = res + 1; sx = res + 1 - i; sy = res; }
            else if (e == 2) { dx = 0; dy = i; sx = 1; sy = res + 1 - i; }
            else { dx = res + 1; dy = i; sx = res; sy = res + 1 - i; }
        } else {
            const int e = k - 4 * res;
            if (e == 0) { dx = 0; dy = 0; sx = res; sy = res; }
            else if (e == 1) { dx = res + 1; dy = 0; sx = 1; sy = res; }
            else if (e == 2) { dx = 0; dy = res + 1; sx = res; sy = 1; }
            else { dx = res + 1; dy = res + 1; sx = 1; sy = 1; }
        }
        const float* s = tile + (sy * T + sx) * 3;
        float* d = tile + (dy * T + dx) * 3;
        d[0] = s[0];
        d[1] = s[1];
        d[2] = s[2];
    }
    __syncthreads();
    // coalesced tile store: T*T*3 floats, 16-byte aligned when T*T*3 % 4 == 0
    float* dst = P.currAtlas + static_cast<size_t>(gp) * T * T * 3;
    const int nf = T * T * 3;
    if ((nf & 3) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(tile);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int k = threadIdx.x; k < nf / 4; k += blockDim.x) d4[k] = s4[k];
    } else {
        for (int k = threadIdx.x; k < nf; k += blockDim.x) dst[k] = tile[k];
    }
    // jitter metric and counters
    unsigned long long bits = __double_as_longlong(maxDelta);
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
        bits = other > bits ? other : bits;
    }
    if ((threadIdx.x & 31) == 0) redDelta[threadIdx.x >> 5] = bits;
    if (ST) flushCounters(cnt, P.stats);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x) / 32; ++w) m = redDelta[w] > m ? redDelta[w] : m;
        atomicMax(P.maxDeltaBits, m);
        atomicAdd(P.rays, static_cast<unsigned long long>(n));
        atomicAdd(P.updated, 1u);
        pv.reject[gp] = 0;  // probe_update.hpp:208-209
        pv.lastFrame[gp] = P.frame;
    }
}

// Per-ray records of the update's ray stage for the listed probes (no state change).
template <typename R>
__global__ void __launch_bounds__(kUpdateThreads) k_trace_debug(UpdateParams<R> P) {
    __shared__ double rot[9];
    const int gp = P.refs[blockIdx.x];
    const ProbesView& pv = P.pc.probes;
    const int ci = cascadeOf(P.pc, gp);
    const int level = P.pc.cas[ci].level;
    const int local = gp - P.pc.cas[ci].base;
    const int n = pv.reject[gp] ? 2 * P.nRaysFull : P.nRaysFull;
    const V3<double> origin = mk(pv.pos[3 * gp], pv.pos[3 * gp + 1], pv.pos[3 * gp + 2]);
    if (threadIdx.x == 0) probeRotation(P.seed, P.frame, P.rotatePerFrame != 0, probeKey(level, local), rot);
    __syncthreads();
    RayRecord* out = P.records + P.recordOffset[blockIdx.x];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        V3<double> dir = probeRayDir(rot, i, n);
        Hit<R> hit;
        V3<double> L = traceAndShade<R, false>(P, origin, dir, nullptr, &hit);
        RayRecord r;
        r.dir[0] = dir.x;
        r.dir[1] = dir.y;
        r.dir[2] = dir.z;
        r.t = hit.converged ? double(hit.t) : 0.0;
        r.radiance[0] = L.x;
        r.radiance[1] = L.y;
        r.radiance[2] = L.z;
        r.normal[0] = hit.normal.x;
        r.normal[1] = hit.normal.y;
        r.normal[2] = hit.normal.z;
        r.converged = hit.converged;
        r.miss = hit.miss;
        r.prim_index = hit.prim >= 0 ? P.scene.orig[hit.prim] : -1;
        r.steps = hit.steps;
        out[i] = r;
    }
}

template <typename R>
void launch_probe_update(const UpdateParams<R>& p, int nBlocks, int maxRays, bool stats, cudaStream_t st) {
    size_t smem = static_cast<size_t>(maxRays) * 6 * sizeof(R);
    if (stats) {
        auto k = k_probe_update<R, true>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<nBlocks, kUpdateThreads, smem, st>>>(p);
    } else {
        auto k = k_probe_update<R, false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<nBlocks, kUpdateThreads, smem, st>>>(p);
    }
}

template <typename R>
void launch_trace_debug(const UpdateParams<R>& p, int nBlocks, cudaStream_t st) {
    k_trace_debug<R><<<nBlocks, kUpdateThreads, 0, st>>>(p);
}

}  // namespace sdfgi_dev
