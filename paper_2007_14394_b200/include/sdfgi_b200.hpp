// sdfgi_b200.hpp — C++ drop-in over the C-ABI (include/sdfgi_b200.h) that speaks the
// reference's own types (/root/reference/proj/include/sdfgi/*.hpp).
//
// Header-only adapter for code that already uses the reference library: include it
// after the reference headers and replace the probe stage of Renderer::renderFrame
// (pipeline.hpp:108-151) with
//
//     sdfgi::b200::Device gpu(0);                 // once
//     gpu.uploadScene(active_);                   // per frame (after cullAndLod)
//     gpu.syncCascades(cascades_, cfg_.octRes);   // once / after recenterCascade
//     for (ci...) m.relocated += gpu.updateProbePositions(ci, cascades_[ci], th1, th2, ...).relocated;
//     gpu.updateProbes(refs, cfg_, frame_, atlas_[writeIdx], &stats);   // replaces the parallelFor
//
// The probe state stays device-resident between calls; the host CascadeVolume /
// ProbeAtlas objects are refreshed from the device after each call so the rest
// of the reference pipeline (gather, dumps, metrics) keeps working unchanged.
// Errors: every non-zero ABI status throws std::runtime_error with the ABI's
// message (the reference's own convention for failures, scene_file.hpp:76-83).
#pragma once

#include <sdfgi/pipeline.hpp>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sdfgi_b200.h"

namespace sdfgi::b200 {

inline void check(int rc, const char* what) {
    if (rc != SDFGI_OK) throw std::runtime_error(std::string(what) + ": " + sdfgi_last_error());
}

inline sdfgi_cfg toCfg(const RenderConfig& c) {
    sdfgi_cfg o;
    std::memset(&o, 0, sizeof(o));
    o.surface_epsilon = c.surfaceEpsilon;
    o.max_trace_steps = c.maxTraceSteps;
    o.shadow_steps = c.shadowSteps;
    o.ray_tmax = c.rayTMax;
    o.shadow_k = c.shadowK;
    o.probe_visibility_k = c.probeVisibilityK;
    o.gradient_step = c.gradientStep;
    o.max_per_cluster = c.maxPerCluster;
    o.merge_radius = c.mergeRadius;
    o.threshold1_frac = c.threshold1Frac;
    o.threshold2_frac = c.threshold2Frac;
    o.max_descent_steps = c.maxDescentSteps;
    o.probe_budget = c.probeBudget;
    o.n_rays_full = c.nRaysFull;
    o.hysteresis = c.hysteresis;
    o.alpha_min = c.alphaMin;
    o.bounce_coeff = c.bounceCoeff;
    o.oct_res = c.octRes;
    o.rotate_per_frame = c.rotatePerFrame ? 1 : 0;
    o.seed = c.seed;
    o.mvc_relocation_frac = c.mvcRelocationFrac;
    o.dedup_quant_frac = c.dedupQuantFrac;
    o.contact_radius_frac = c.contactRadiusFrac;
    o.contact_samples = c.contactSamples;
    o.history_blend = c.historyBlend;
    o.depth_sigma_frac = c.depthSigmaFrac;
    o.exposure = c.exposure;
    o.fps = c.fps;
    return o;
}

class Device {
public:
    explicit Device(int device = 0, bool fp64 = true) {
        check(sdfgi_ctx_create(device, 0, 1, nullptr, fp64 ? SDFGI_F64 : SDFGI_F32, &ctx_), "sdfgi_ctx_create");
    }
    ~Device() { sdfgi_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    // ActiveScene (scene.hpp:88-103) -> device; replaces finalize() for the GPU side.
    void uploadScene(const ActiveScene& s) {
        std::vector<sdfgi_prim> prims(s.primitives.size());
        for (size_t i = 0; i < prims.size(); ++i) {
            const SdfPrimitive& p = s.primitives[i];
            sdfgi_prim& q = prims[i];
            std::memset(&q, 0, sizeof(q));
            q.id = p.id;
            q.kind = static_cast<int32_t>(p.kind);
            q.lod_tier = p.lodTier;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) q.rot[3 * a + b] = p.transform.rotation.m[a][b];
            for (int a = 0; a < 3; ++a) {
                q.trans[a] = p.transform.translation[a];
                q.size[a] = p.size[a];
                q.albedo[a] = p.material.albedo[a];
                q.emission[a] = p.material.emission[a];
            }
        }
        std::vector<sdfgi_cluster> cl(s.clusters.size());
        std::vector<int32_t> start{0}, idx;
        for (size_t k = 0; k < cl.size(); ++k) {
            std::memset(&cl[k], 0, sizeof(cl[k]));
            for (int a = 0; a < 3; ++a) {
                cl[k].lo[a] = s.clusters[k].cullAabb.lo[a];
                cl[k].hi[a] = s.clusters[k].cullAabb.hi[a];
            }
            cl[k].unbounded = s.clusters[k].unbounded ? 1 : 0;
            for (int m : s.clusters[k].members) idx.push_back(m);
            start.push_back(static_cast<int32_t>(idx.size()));
        }
        std::vector<sdfgi_light> lights(s.lights.size());
        for (size_t i = 0; i < lights.size(); ++i) {
            std::memset(&lights[i], 0, sizeof(lights[i]));
            lights[i].kind = static_cast<int32_t>(s.lights[i].kind);
            for (int a = 0; a < 3; ++a) {
                lights[i].position[a] = s.lights[i].position[a];
                lights[i].direction[a] = s.lights[i].direction[a];
                lights[i].intensity[a] = s.lights[i].intensity[a];
            }
        }
        const double sky[3] = {s.sky.x, s.sky.y, s.sky.z};
        check(sdfgi_scene_upload(ctx_, prims.data(), static_cast<int>(prims.size()), cl.data(),
                                 static_cast<int>(cl.size()), start.data(), idx.data(), lights.data(),
                                 static_cast<int>(lights.size()), sky),
              "sdfgi_scene_upload");
    }

    // Mirror the host cascades (makeCascade, probe_volume.hpp:57-76) and their probe
    // state on the device; atlases start from the given host atlases (or zero).
    void syncCascades(const std::vector<CascadeVolume>& cascades, int octRes,
                      const std::vector<ProbeAtlas>* front = nullptr) {
        check(sdfgi_cascades_clear(ctx_), "sdfgi_cascades_clear");
        for (const CascadeVolume& c : cascades) {
            const double o[3] = {c.origin.x, c.origin.y, c.origin.z};
            check(sdfgi_cascade_set(ctx_, c.level, c.resX, c.resY, c.resZ, c.spacing, o, octRes), "sdfgi_cascade_set");
            pushProbes(c);
        }
        if (front)
            for (size_t i = 0; i < cascades.size(); ++i)
                check(sdfgi_atlas_upload(ctx_, cascades[i].level, 0, (*front)[i].raw().data(), (*front)[i].raw().size()),
                      "sdfgi_atlas_upload");
    }

    // updateProbePositions (probe_volume.hpp:99-143), bit-exact; host probes refreshed.
    RelocationReport updateProbePositions(CascadeVolume& cascade, double th1, double th2, int maxDescentSteps = 16,
                                          TraceStats* stats = nullptr, double gradientStep = 1e-3) {
        sdfgi_reloc_report rep;
        sdfgi_stats st{};
        check(sdfgi_probes_relocate(ctx_, cascade.level, th1, th2, maxDescentSteps, gradientStep, &rep,
                                    stats ? &st : nullptr),
              "sdfgi_probes_relocate");
        pullProbes(cascade);
        if (stats) merge(*stats, st);
        return {rep.relocated, rep.rejected, rep.dead};
    }

    // The batched updateProbe (probe_update.hpp:166-211) over `refs` — the parallelFor
    // of pipeline.hpp:138-148. `curr` receives the back atlases; the device swaps.
    ProbeUpdateResult updateProbes(std::vector<CascadeVolume>& cascades, const std::vector<ProbeRef>& refs,
                                   const RenderConfig& cfg, int frameIndex, std::vector<ProbeAtlas>& curr,
                                   TraceStats* stats = nullptr) {
        std::vector<int32_t> r;
        r.reserve(2 * refs.size());
        for (const ProbeRef& ref : refs) {
            r.push_back(cascades[ref.cascade].level);
            r.push_back(ref.index);
        }
        sdfgi_cfg c = toCfg(cfg);
        sdfgi_update_result res;
        sdfgi_stats st{};
        check(sdfgi_probes_update(ctx_, r.data(), static_cast<int>(refs.size()), frameIndex, &c, &res,
                                  stats ? &st : nullptr),
              "sdfgi_probes_update");
        for (size_t i = 0; i < cascades.size(); ++i) {
            auto& raw = const_cast<std::vector<float>&>(curr[i].raw());
            check(sdfgi_atlas_download(ctx_, cascades[i].level, 1, raw.data(), raw.size()), "sdfgi_atlas_download");
            pullProbes(cascades[i]);
        }
        check(sdfgi_atlas_swap(ctx_), "sdfgi_atlas_swap");
        if (stats) merge(*stats, st);
        ProbeUpdateResult out;
        out.maxTexelDelta = res.max_texel_delta;
        out.raysTraced = static_cast<int>(res.rays_traced);
        return out;
    }

    void* handle() const { return ctx_; }

private:
    static void merge(TraceStats& a, const sdfgi_stats& b) {
        a.sdfQueries += b.sdf_queries;
        a.clustersVisited += b.clusters_visited;
        a.clustersSkipped += b.clusters_skipped;
        a.primitiveEvals += b.primitive_evals;
        a.traceSteps += b.trace_steps;
        a.sphereTraces += b.sphere_traces;
        a.shadowTraces += b.shadow_traces;
        a.visibilityTraces += b.visibility_traces;
    }
    void pushProbes(const CascadeVolume& c) {
        std::vector<sdfgi_probe> p(c.probes.size());
        for (size_t i = 0; i < p.size(); ++i) {
            std::memset(&p[i], 0, sizeof(p[i]));
            for (int a = 0; a < 3; ++a) {
                p[i].resting[a] = c.probes[i].restingPos[a];
                p[i].pos[a] = c.probes[i].pos[a];
                p[i].last_pos[a] = c.probes[i].lastPos[a];
            }
            p[i].reject_history = c.probes[i].rejectHistory ? 1 : 0;
            p[i].alive = c.probes[i].alive ? 1 : 0;
            p[i].last_update_frame = c.probes[i].lastUpdateFrame;
        }
        check(sdfgi_probes_upload(ctx_, c.level, p.data(), static_cast<int>(p.size())), "sdfgi_probes_upload");
    }
    void pullProbes(CascadeVolume& c) {
        std::vector<sdfgi_probe> p(c.probes.size());
        check(sdfgi_probes_download(ctx_, c.level, p.data(), static_cast<int>(p.size())), "sdfgi_probes_download");
        for (size_t i = 0; i < p.size(); ++i) {
            c.probes[i].restingPos = {p[i].resting[0], p[i].resting[1], p[i].resting[2]};
            c.probes[i].pos = {p[i].pos[0], p[i].pos[1], p[i].pos[2]};
            c.probes[i].lastPos = {p[i].last_pos[0], p[i].last_pos[1], p[i].last_pos[2]};
            c.probes[i].rejectHistory = p[i].reject_history != 0;
            c.probes[i].alive = p[i].alive != 0;
            c.probes[i].lastUpdateFrame = p[i].last_update_frame;
        }
    }

    void* ctx_ = nullptr;
};

}  // namespace sdfgi::b200
