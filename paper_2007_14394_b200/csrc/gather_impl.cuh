// gather_impl.cuh — the per-pixel gather (e), included once per precision TU.
//
//   k_render_gbuffer   renderGBuffer (shading.hpp:39-72): one camera ray per pixel
//                      (the gather's input; f1 in SURVEY §8).
//   k_downsample       downsampleDepthCheckerboard (shading.hpp:85-112), thread per
//                      half-res pixel.
//   k_select           selectVisibilityPixels (shading.hpp:125-161), thread per cell.
//   k_tiles            buildVisibilityTasks + runVisibilityTasks + shadePixelGI
//                      (shading.hpp:185-338) fused: ONE WARP PER 4x4 half-res tile,
//                      lane = (selection cell, stencil slot) in the reference's
//                      insertion order; the per-tile dedup is a warp compare of the
//                      (cascade, probe, quantised position) keys, the first lane of a
//                      key traces the soft-shadow visibility, the others read it by
//                      shuffle, and each cell's weighted sum runs in slot order.
//   k_resolve          upsampleAndResolve (shading.hpp:350-426), thread per pixel.
// Contact GI (shading.hpp:431-477) runs as a wavefront of (pixel, sample) rays
// through the probe-update kernels (launch_contact, kernels_impl.cuh).
#pragma once

#include "kernels.cuh"

namespace sdfgi_dev {

// Camera::rayDir / project (camera.hpp:29-48)
__device__ __forceinline__ V3<double> camRayDir(const CameraDev& c, double px, double py, int w, int h) {
    double tanHalf = c.tanHalf;
    double aspect = static_cast<double>(w) / h;
    double ndcX = (2.0 * (px + 0.5) / w - 1.0) * tanHalf * aspect;
    double ndcY = (1.0 - 2.0 * (py + 0.5) / h) * tanHalf;
    V3<double> f = mk(c.fwd[0], c.fwd[1], c.fwd[2]), r = mk(c.right[0], c.right[1], c.right[2]),
               u = mk(c.up[0], c.up[1], c.up[2]);
    return normalize(f + r * ndcX + u * ndcY);
}
__device__ __forceinline__ bool camProject(const CameraDev& c, V3<double> world, int w, int h, double* ox, double* oy) {
    V3<double> rel = world - mk(c.pos[0], c.pos[1], c.pos[2]);
    double z = dot(rel, mk(c.fwd[0], c.fwd[1], c.fwd[2]));
    if (z <= 1e-9) return false;
    double tanHalf = c.tanHalf;
    double aspect = static_cast<double>(w) / h;
    double ndcX = dot(rel, mk(c.right[0], c.right[1], c.right[2])) / (z * tanHalf * aspect);
    double ndcY = dot(rel, mk(c.up[0], c.up[1], c.up[2])) / (z * tanHalf);
    *ox = (ndcX + 1.0) * 0.5 * w - 0.5;
    *oy = (1.0 - ndcY) * 0.5 * h - 0.5;
    return true;
}

__device__ __forceinline__ bool isSky(const GPix& p) { return !(p.depth < INFINITY); }

// ------------------------------------------------------------------ G-buffer
template <typename R>
__global__ void __launch_bounds__(128) k_render_gbuffer(GatherParams<R> P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.w * P.h) return;
    const int x = i % P.w, y = i / P.w;
    GPix px;
    px.depth = INFINITY;
    px.normal[0] = px.normal[1] = 0;
    px.normal[2] = 1;
    for (int k = 0; k < 3; ++k) px.albedo[k] = px.emission[k] = px.world_pos[k] = 0;
    px.motion[0] = px.motion[1] = 0;
    px.prim = -1;
    px._pad = 0;
    V3<double> d = camRayDir(P.cam, x, static_cast<double>(y), P.w, P.h);
    V3<R> o = mk(R(P.cam.pos[0]), R(P.cam.pos[1]), R(P.cam.pos[2]));
    Hit<R> hit = sphereTrace<R, false>(P.scene, o, mk(R(d.x), R(d.y), R(d.z)), R(P.tc.rayTMax), R(P.tc.eps),
                                       P.tc.maxSteps, nullptr, R(INFINITY));
    if (hit.converged) {
        px.depth = hit.t;
        px.normal[0] = hit.normal.x;
        px.normal[1] = hit.normal.y;
        px.normal[2] = hit.normal.z;
        px.world_pos[0] = hit.pos.x;
        px.world_pos[1] = hit.pos.y;
        px.world_pos[2] = hit.pos.z;
        if (hit.prim >= 0) {
            px.prim = P.scene.orig[hit.prim];
            for (int k = 0; k < 3; ++k) {
                px.albedo[k] = P.scene.albedo[3 * hit.prim + k];
                px.emission[k] = P.scene.emission[3 * hit.prim + k];
            }
        }
        double ox, oy;
        if (camProject(P.prevCam, mk<double>(hit.pos.x, hit.pos.y, hit.pos.z), P.w, P.h, &ox, &oy)) {
            px.motion[0] = ox - x;
            px.motion[1] = oy - y;
        }
    }
    P.gb[i] = px;
}

// ----------------------------------------------------------------- downsample
template <typename R>
__global__ void __launch_bounds__(128) k_downsample(GatherParams<R> P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.hw * P.hh) return;
    const int x = i % P.hw, y = i / P.hw;
    const bool takeMax = ((x + y) & 1) == 0;
    double best = takeMax ? -INFINITY : INFINITY;
    int bestSrc = 0;
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            int sx = min(2 * x + dx, P.w - 1), sy = min(2 * y + dy, P.h - 1);
            double d = P.gb[sy * P.w + sx].depth;
            if (takeMax ? d > best : d < best) {
                best = d;
                bestSrc = sy * P.w + sx;
            }
        }
    P.halfDepth[i] = best;
    P.halfSrc[i] = bestSrc;
}

template <typename R>
__global__ void __launch_bounds__(128) k_select(GatherParams<R> P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.sw * P.sh) return;
    const int x = i % P.sw, y = i / P.sw;
    const int ox[4] = {0, 1, 0, 1}, oy[4] = {0, 0, 1, 1};
    const int hx0 = 2 * x, hy0 = 2 * y;
    double lo = INFINITY, hi = -INFINITY;
    int loIdx = -1, hiIdx = -1;
    for (int k = 0; k < 4; ++k) {
        int hx = min(hx0 + ox[k], P.hw - 1), hy = min(hy0 + oy[k], P.hh - 1);
        double d = P.halfDepth[hy * P.hw + hx];
        if (!isfinite(d)) continue;
        if (d < lo) {
            lo = d;
            loIdx = hy * P.hw + hx;
        }
        if (d > hi) {
            hi = d;
            hiIdx = hy * P.hw + hx;
        }
    }
    const int rot = P.frame & 3;
    int pick = min(hy0 + oy[rot], P.hh - 1) * P.hw + min(hx0 + ox[rot], P.hw - 1);
    if (loIdx >= 0) {
        bool rotSky = !isfinite(P.halfDepth[pick]);
        bool spread = (hi - lo) > 0.1 * hi;
        if (spread)
            pick = (P.frame & 1) == 0 ? loIdx : hiIdx;
        else if (rotSky)
            pick = loIdx;
    }
    P.sel[i] = pick;
}

// --------------------------------------------------- tiles: tasks + vis + GI
template <typename R, bool ST>
__global__ void __launch_bounds__(128) k_tiles(GatherParams<R> P) {
    __shared__ Stencil sst[4][4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tilesX = (P.sw + 1) / 2, tilesY = (P.sh + 1) / 2;
    const int tile = blockIdx.x * 4 + warp;
    if (tile >= tilesX * tilesY) return;  // whole warp exits together
    const int tx = tile % tilesX, ty = tile / tilesX;
    const int q = lane >> 3, e = lane & 7;
    const int cx = 2 * tx + (q & 1), cy = 2 * ty + (q >> 1);
    const bool inb = cx < P.sw && cy < P.sh;
    const int cell = inb ? cy * P.sw + cx : 0;
    const int anchor = inb ? P.halfSrc[P.sel[cell]] : 0;
    const GPix& px = P.gb[anchor];
    const bool geo = inb && !isSky(px);
    const V3<double> wp = mk(px.world_pos[0], px.world_pos[1], px.world_pos[2]);
    const V3<double> nn = mk(px.normal[0], px.normal[1], px.normal[2]);
    if (e == 0 && geo) sst[warp][q] = interpolationStencil(P.pc.cas, P.pc.nCas, P.pc.probes, wp, P.tc.mvcFrac);
    __syncwarp();
    const Stencil& st = sst[warp][q];
    const bool valid = geo && !st.sky && st.count > 0;
    const double weight = valid ? st.w[e] : 0.0;
    const bool has = valid && weight > 0;
    int key[5] = {0, 0, 0, 0, 0};
    if (has) {
        const double quant = P.dedupFrac * P.pc.cas[st.cascade].spacing;
        key[0] = st.cascade;
        key[1] = st.probe[e];
        key[2] = static_cast<int>(floor(wp.x / quant));
        key[3] = static_cast<int>(floor(wp.y / quant));
        key[4] = static_cast<int>(floor(wp.z / quant));
    }
    // dedup: the first lane (insertion order) holding the same key owns the task
    // (every lane executes every shuffle: no short-circuit around __shfl_sync)
    int owner = lane;
    for (int j = 0; j < 32; ++j) {
        int same = __shfl_sync(kFull, has ? 1 : 0, j);
        for (int k = 0; k < 5; ++k) {
            const int kj = __shfl_sync(kFull, key[k], j);
            same &= kj == key[k] ? 1 : 0;
        }
        if (has && same && j < owner) owner = j;
    }
    Counters cnt;
    cnt.zero();
    double vis = 1.0;
    if (has && owner == lane) {
        // probeVisibility, shading.hpp:264-279
        const CascadeDev& c = P.pc.cas[st.cascade];
        const double* pp = P.pc.probes.pos + 3 * static_cast<size_t>(c.base + st.probe[e]);
        V3<double> toProbe = mk(pp[0], pp[1], pp[2]) - wp;
        double dist = length(toProbe);
        if (dist >= 1e-9) {
            V3<double> dir = toProbe / dist;
            double cosT = dot(nn, dir);
            double bias = 2.0 * P.tc.eps / smax(0.1, cosT);
            double tMax = dist - P.th1Frac * c.spacing;
            if (tMax > bias) {
                if (ST) ++cnt.vis;
                V3<double> so = wp + nn * bias;
                vis = double(softShadowTrace<R, ST>(P.scene, mk(R(so.x), R(so.y), R(so.z)),
                                                    mk(R(dir.x), R(dir.y), R(dir.z)), R(bias), R(tMax),
                                                    R(P.visK), P.tc.shadowSteps, &cnt));
            }
        }
    }
    const unsigned owners = __ballot_sync(kFull, has && owner == lane);
    if (lane == 0 && owners) atomicAdd(P.taskCount, static_cast<unsigned long long>(__popc(owners)));
    vis = __shfl_sync(kFull, vis, owner);
    // shadePixelGI (shading.hpp:319-338): slot-ordered sum by the cell's lane 0
    const double wv = has ? weight * vis : 0.0;
    V3<double> smp = mk(0.0, 0.0, 0.0);
    if (has && wv > 0) {
        AtlasView av{P.atlas, P.oct, P.oct + 2};
        smp = sampleBilinear(av, P.pc.cas[st.cascade].base + st.probe[e], octEncode(nn));
    }
    V3<double> acc = mk(0.0, 0.0, 0.0);
    double wsum = 0;
    for (int k = 0; k < 8; ++k) {
        const int src = (lane & ~7) + k;
        const double w = __shfl_sync(kFull, wv, src);
        const double sx = __shfl_sync(kFull, smp.x, src), sy = __shfl_sync(kFull, smp.y, src),
                     sz = __shfl_sync(kFull, smp.z, src);
        if (w > 0) {
            acc = acc + mk(sx, sy, sz) * w;
            wsum += w;
        }
    }
    if (e == 0 && inb) {
        P.sparseAnchor[cell] = anchor;
        const bool ok = valid && wsum > 1e-9;
        V3<double> irr = ok ? acc / wsum : mk(0.0, 0.0, 0.0);
        P.sparseValid[cell] = ok ? 1 : 0;
        P.sparseIrr[3 * cell] = irr.x;
        P.sparseIrr[3 * cell + 1] = irr.y;
        P.sparseIrr[3 * cell + 2] = irr.z;
    }
    if (ST) flushCounters(cnt, P.visStats);
}

// --------------------------------------------------------------------- resolve
template <typename R>
__global__ void __launch_bounds__(128) k_resolve(GatherParams<R> P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.w * P.h) return;
    const int x = i % P.w, y = i / P.w;
    const GPix& px = P.gb[i];
    double* out = P.resolved + 3 * static_cast<size_t>(i);
    if (isSky(px)) {
        out[0] = out[1] = out[2] = 0;
        return;
    }
    const int qx = x / 4, qy = y / 4;
    const double inf = INFINITY;
    V3<double> acc = mk(0.0, 0.0, 0.0), cmin = mk(inf, inf, inf), cmax = mk(-inf, -inf, -inf);
    double wsum = 0;
    bool any = false;
    const double sigma = smax(1e-6, P.depthSigmaFrac * px.depth);
    const V3<double> pn = mk(px.normal[0], px.normal[1], px.normal[2]);
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            const int nx = qx + dx, ny = qy + dy;
            if (nx < 0 || ny < 0 || nx >= P.sw || ny >= P.sh) continue;
            const int cell = ny * P.sw + nx;
            if (!P.sparseValid[cell]) continue;
            const GPix& an = P.gb[P.sparseAnchor[cell]];
            double w = exp(-fabs(an.depth - px.depth) / sigma) *
                       pow(smax(0.0, dot(mk(an.normal[0], an.normal[1], an.normal[2]), pn)), 4.0);
            if (w <= 1e-6) continue;
            V3<double> si = mk(P.sparseIrr[3 * cell], P.sparseIrr[3 * cell + 1], P.sparseIrr[3 * cell + 2]);
            acc = acc + si * w;
            wsum += w;
            cmin = mk(smin(cmin.x, si.x), smin(cmin.y, si.y), smin(cmin.z, si.z));
            cmax = mk(smax(cmax.x, si.x), smax(cmax.y, si.y), smax(cmax.z, si.z));
            any = true;
        }
    V3<double> cur = mk(0.0, 0.0, 0.0), hist = cur, o = cur;
    const bool haveCur = wsum > 1e-9;
    bool haveHist = false;
    if (haveCur) cur = acc / wsum;
    if (P.histValid) {
        const int hx = static_cast<int>(llround(x + px.motion[0])), hy = static_cast<int>(llround(y + px.motion[1]));
        if (hx >= 0 && hy >= 0 && hx < P.w && hy < P.h) {
            const double hd = P.histDepth[hy * P.w + hx];
            if (isfinite(hd) && fabs(hd - px.depth) <= 0.1 * smax(hd, px.depth)) {
                const double* hi = P.histIrr + 3 * (static_cast<size_t>(hy) * P.w + hx);
                hist = mk(hi[0], hi[1], hi[2]);
                if (any)
                    hist = mk(smin(smax(hist.x, cmin.x), cmax.x), smin(smax(hist.y, cmin.y), cmax.y),
                              smin(smax(hist.z, cmin.z), cmax.z));
                haveHist = true;
            }
        }
    }
    if (haveCur && haveHist)
        o = cur * P.historyBlend + hist * (1.0 - P.historyBlend);
    else if (haveCur)
        o = cur;
    else if (haveHist)
        o = hist;
    else {
        const V3<double> wp = mk(px.world_pos[0], px.world_pos[1], px.world_pos[2]);
        Stencil st = interpolationStencil(P.pc.cas, P.pc.nCas, P.pc.probes, wp, P.tc.mvcFrac);
        if (!st.sky) {  // sampleIrradianceRaw, probe_update.hpp:47-57
            V2<double> uv = octEncode(pn);
            AtlasView av{P.atlas, P.oct, P.oct + 2};
            for (int k = 0; k < st.count; ++k) {
                if (st.w[k] <= 0) continue;
                o = o + sampleBilinear(av, P.pc.cas[st.cascade].base + st.probe[k], uv) * st.w[k];
            }
        }
    }
    out[0] = o.x;
    out[1] = o.y;
    out[2] = o.z;
}

template <typename R>
void launch_gather(const GatherParams<R>& p, int stage, bool stats, cudaStream_t st) {
    const int np = p.w * p.h;
    switch (stage) {
        case 0: k_render_gbuffer<R><<<(np + 127) / 128, 128, 0, st>>>(p); break;
        case 1:
            k_downsample<R><<<(p.hw * p.hh + 127) / 128, 128, 0, st>>>(p);
            k_select<R><<<(p.sw * p.sh + 127) / 128, 128, 0, st>>>(p);
            break;
        case 2: {
            const int tiles = ((p.sw + 1) / 2) * ((p.sh + 1) / 2);
            if (stats)
                k_tiles<R, true><<<(tiles + 3) / 4, 128, 0, st>>>(p);
            else
                k_tiles<R, false><<<(tiles + 3) / 4, 128, 0, st>>>(p);
            break;
        }
        default: k_resolve<R><<<(np + 127) / 128, 128, 0, st>>>(p); break;
    }
}

}  // namespace sdfgi_dev
