// sdfgi_b200.hpp — C++ drop-in over the C-ABI (include/sdfgi_b200.h) that speaks the
// reference's own types (/root/reference/proj/include/sdfgi/*.hpp).
//
// Header-only adapter for code that already uses the reference library: include it
// after the reference headers. Three levels of replacement:
//
//  1. The whole frame loop: sdfgi::b200::Renderer has Renderer's constructor and
//     renderFrame() (pipeline.hpp:50-230) with every per-frame stage except scene
//     instancing/culling on the device.
//  2. The two stages of Renderer::renderFrame, inside the reference's own loop:
//       sdfgi::b200::Device gpu(0);                          // once
//       gpu.uploadScene(active_);                            // per frame (after cullAndLod)
//       gpu.syncCascades(cascades_, cfg_.octRes);            // once / after recenterCascade
//       for (auto& c : cascades_)                            // probe placement, :108-121
//           m.relocated += gpu.updateProbePositions(c, th1, th2, ...).relocated;
//       gpu.updateProbes(cascades_, refs, cfg_, frame_, atlas_[writeIdx], &stats);  // :126-151
//       gbuffer_ = gpu.renderGBuffer(camera_, prevCamera_, w, h, cfg_);            // :155
//       auto g = gpu.gather(frame_, cfg_, &stats);           // :161-207 (resolved + indirect)
//       image_ = gpu.composeFrame(cfg_, &stats);             // :209
//  3. The free functions, batched on the device: querySceneSdf, sphereTrace,
//     softShadowTrace, shadeHit, convolveIrradiance, interpolationStencil and the
//     per-probe updateProbe (a 1-probe batch).
//
// The probe state stays device-resident between calls; the host CascadeVolume /
// ProbeAtlas objects are refreshed from the device after each call so the rest
// of the reference pipeline (dumps, metrics) keeps working unchanged. Functions
// that read "the previous field" (shadeHit, updateProbe) take the reference's
// IrradianceField and upload it as the device's front atlas first.
// Errors: every non-zero ABI status throws std::runtime_error with the ABI's
// message (the reference's own convention for failures, scene_file.hpp:76-83).
#pragma once

#include <sdfgi/pipeline.hpp>

#include <algorithm>
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

    // ------------------------------------------------------------ free functions
    // (each runs on the scene last given to uploadScene)

    // querySceneSdf (scene.hpp:336-340): exact, with the owner primitive (index into
    // ActiveScene::primitives) when `owner` is given.
    std::vector<double> querySceneSdf(const std::vector<Vec3>& points, double initD = kInf,
                                      std::vector<int>* owner = nullptr) {
        const size_t n = points.size();
        std::vector<double> p(3 * n), init(n, initD), d(n);
        std::vector<int32_t> o(n);
        for (size_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) p[3 * i + a] = points[i][a];
        check(sdfgi_query_points(ctx_, p.data(), init.data(), static_cast<int>(n), d.data(), o.data()),
              "sdfgi_query_points");
        if (owner) owner->assign(o.begin(), o.end());
        return d;
    }
    double querySceneSdf(const ActiveScene&, const Vec3& p, double initD = kInf, TraceStats* = nullptr,
                         int* owner = nullptr) {
        std::vector<int> o;
        double d = querySceneSdf(std::vector<Vec3>{p}, initD, &o)[0];
        if (owner) *owner = o[0];
        return d;
    }

    // sphereTrace (scene.hpp:391-435) of a batch of rays with shared parameters.
    std::vector<Hit> sphereTrace(const ActiveScene& scene, const std::vector<Vec3>& origins,
                                 const std::vector<Vec3>& dirs, double tMax, double surfaceEpsilon = 1e-3,
                                 int maxSteps = 128, TraceStats* stats = nullptr, double startBound = kInf) {
        const size_t n = origins.size();
        std::vector<double> o(3 * n), d(3 * n);
        for (size_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) {
                o[3 * i + a] = origins[i][a];
                d[3 * i + a] = dirs[i][a];
            }
        std::vector<sdfgi_hit> h(n);
        sdfgi_stats st{};
        check(sdfgi_trace_rays(ctx_, o.data(), d.data(), static_cast<int>(n), tMax, surfaceEpsilon, maxSteps,
                               startBound, h.data(), stats ? &st : nullptr),
              "sdfgi_trace_rays");
        if (stats) merge(*stats, st);
        std::vector<Hit> out(n);
        for (size_t i = 0; i < n; ++i) {
            Hit& r = out[i];
            r.converged = h[i].converged != 0;
            r.miss = static_cast<MissReason>(h[i].miss);
            r.t = h[i].t;
            r.position = {h[i].pos[0], h[i].pos[1], h[i].pos[2]};
            r.normal = {h[i].normal[0], h[i].normal[1], h[i].normal[2]};
            r.primitiveIndex = h[i].prim_index;
            r.primitiveId = h[i].prim_index >= 0 ? scene.primitives[h[i].prim_index].id : -1;
        }
        return out;
    }
    Hit sphereTrace(const ActiveScene& scene, const Vec3& origin, const Vec3& dir, double tMax,
                    double surfaceEpsilon = 1e-3, int maxSteps = 128, TraceStats* stats = nullptr,
                    double startBound = kInf) {
        return sphereTrace(scene, std::vector<Vec3>{origin}, std::vector<Vec3>{dir}, tMax, surfaceEpsilon, maxSteps,
                           stats, startBound)[0];
    }

    // softShadowTrace (scene.hpp:459-476) of a batch of segments.
    std::vector<double> softShadowTrace(const std::vector<Vec3>& origins, const std::vector<Vec3>& dirs,
                                        const std::vector<double>& tMin, const std::vector<double>& tMax, double k,
                                        TraceStats* stats = nullptr, int maxSteps = 256, double minStep = 5e-4) {
        const size_t n = origins.size();
        std::vector<double> o(3 * n), d(3 * n), v(n);
        for (size_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) {
                o[3 * i + a] = origins[i][a];
                d[3 * i + a] = dirs[i][a];
            }
        sdfgi_stats st{};
        check(sdfgi_soft_shadow(ctx_, o.data(), d.data(), tMin.data(), tMax.data(), static_cast<int>(n), k, maxSteps,
                                minStep, v.data(), stats ? &st : nullptr),
              "sdfgi_soft_shadow");
        if (stats) merge(*stats, st);
        return v;
    }
    double softShadowTrace(const ActiveScene&, const Vec3& origin, const Vec3& dir, double tMin, double tMax,
                           double k, TraceStats* stats = nullptr, int maxSteps = 256, double minStep = 5e-4) {
        return softShadowTrace(std::vector<Vec3>{origin}, std::vector<Vec3>{dir}, std::vector<double>{tMin},
                               std::vector<double>{tMax}, k, stats, maxSteps, minStep)[0];
    }

    // shadeHit (probe_update.hpp:136-149) of a batch of hits against prevField.
    std::vector<Vec3> shadeHit(const std::vector<Hit>& hits, const IrradianceField& prevField, double bounceCoeff,
                               const RenderConfig& cfg, TraceStats* stats = nullptr) {
        if (prevField.valid()) syncField(prevField, cfg.octRes);
        const size_t n = hits.size();
        std::vector<sdfgi_hit> h(n);
        for (size_t i = 0; i < n; ++i) {
            std::memset(&h[i], 0, sizeof(h[i]));
            h[i].t = hits[i].t;
            for (int a = 0; a < 3; ++a) {
                h[i].pos[a] = hits[i].position[a];
                h[i].normal[a] = hits[i].normal[a];
            }
            h[i].prim_index = hits[i].primitiveIndex;
            h[i].converged = hits[i].converged ? 1 : 0;
        }
        sdfgi_cfg c = toCfg(cfg);
        std::vector<double> rgb(3 * n);
        sdfgi_stats st{};
        check(sdfgi_shade_hits(ctx_, h.data(), static_cast<int>(n), prevField.valid() ? bounceCoeff : 0.0, &c,
                               rgb.data(), stats ? &st : nullptr),
              "sdfgi_shade_hits");
        if (stats) merge(*stats, st);
        std::vector<Vec3> out(n);
        for (size_t i = 0; i < n; ++i) out[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
        return out;
    }
    Vec3 shadeHit(const ActiveScene&, const Hit& hit, const IrradianceField& prevField, double bounceCoeff,
                  const RenderConfig& cfg, TraceStats* stats = nullptr) {
        return shadeHit(std::vector<Hit>{hit}, prevField, bounceCoeff, cfg, stats)[0];
    }

    // convolveIrradiance (probe_update.hpp:25-34) of one sample set for many texel
    // directions.
    std::vector<ConvolveResult> convolveIrradiance(const std::vector<RadianceSample>& samples,
                                                   const std::vector<Vec3>& texelDirs) {
        std::vector<ConvolveResult> out(texelDirs.size());
        if (samples.empty()) {
            for (auto& r : out) r = {{0, 0, 0}, true};
            return out;
        }
        std::vector<double> sd(3 * samples.size()), sr(3 * samples.size()), td(3 * texelDirs.size()),
            rgb(3 * texelDirs.size());
        for (size_t i = 0; i < samples.size(); ++i)
            for (int a = 0; a < 3; ++a) {
                sd[3 * i + a] = samples[i].dir[a];
                sr[3 * i + a] = samples[i].radiance[a];
            }
        for (size_t i = 0; i < texelDirs.size(); ++i)
            for (int a = 0; a < 3; ++a) td[3 * i + a] = texelDirs[i][a];
        check(sdfgi_convolve_irradiance(ctx_, sd.data(), sr.data(), static_cast<int>(samples.size()), td.data(),
                                        static_cast<int>(texelDirs.size()), rgb.data()),
              "sdfgi_convolve_irradiance");
        for (size_t i = 0; i < out.size(); ++i) out[i] = {{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]}, false};
        return out;
    }
    ConvolveResult convolveIrradiance(const std::vector<RadianceSample>& samples, const Vec3& texelDir) {
        return convolveIrradiance(samples, std::vector<Vec3>{texelDir})[0];
    }

    // interpolationStencil (probe_volume.hpp:224-310) over the device cascades
    // (mirrored from `cascades`: pass the same vector syncCascades / the updates use).
    std::vector<InterpolationStencil> interpolationStencil(const std::vector<CascadeVolume>& cascades,
                                                           const std::vector<Vec3>& points,
                                                           double mvcRelocationFrac = 0.25) {
        const size_t n = points.size();
        std::vector<double> p(3 * n);
        for (size_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) p[3 * i + a] = points[i][a];
        std::vector<sdfgi_stencil> st(n);
        check(sdfgi_interpolation_stencil(ctx_, p.data(), static_cast<int>(n), mvcRelocationFrac, st.data()),
              "sdfgi_interpolation_stencil");
        std::vector<InterpolationStencil> out(n);
        for (size_t i = 0; i < n; ++i) {
            InterpolationStencil& s = out[i];
            s.count = st[i].count;
            s.crossCascade = st[i].cross_cascade != 0;
            s.skyFallback = st[i].sky_fallback != 0;
            s.usedMvc = st[i].used_mvc != 0;
            int slot = 0;
            for (size_t k = 0; k < cascades.size(); ++k)
                if (cascades[k].level == st[i].level) slot = static_cast<int>(k);
            for (int k = 0; k < s.count; ++k) s.entries[k] = {{slot, st[i].index[k]}, st[i].weight[k]};
        }
        return out;
    }
    InterpolationStencil interpolationStencil(const std::vector<CascadeVolume>& cascades, const Vec3& point,
                                              double mvcRelocationFrac = 0.25) {
        return interpolationStencil(cascades, std::vector<Vec3>{point}, mvcRelocationFrac)[0];
    }

    // updateProbe (probe_update.hpp:166-211) for one probe: prev's probe state and
    // atlases become the device's, the probe is updated as a 1-probe batch, its tile
    // lands in `curr` and its state in `cascade`.
    ProbeUpdateResult updateProbe(const ActiveScene&, CascadeVolume& cascade, int probeIndex,
                                  const IrradianceField& prev, ProbeAtlas& curr, int nRays, const RenderConfig& cfg,
                                  int frameIndex, TraceStats* stats = nullptr) {
        if (!prev.valid()) throw std::runtime_error("updateProbe: invalid previous field");
        syncField(prev, cfg.octRes);
        RenderConfig c2 = cfg;
        c2.nRaysFull = nRays;
        sdfgi_cfg c = toCfg(c2);
        const int32_t ref[2] = {cascade.level, probeIndex};
        sdfgi_update_result res;
        sdfgi_stats st{};
        check(sdfgi_probes_update(ctx_, ref, 1, frameIndex, &c, &res, stats ? &st : nullptr), "sdfgi_probes_update");
        std::vector<float> back(curr.raw().size());
        check(sdfgi_atlas_download(ctx_, cascade.level, 1, back.data(), back.size()), "sdfgi_atlas_download");
        const size_t tile = curr.raw().size() / static_cast<size_t>(std::max(cascade.probeCount(), 1));
        auto& raw = const_cast<std::vector<float>&>(curr.raw());
        std::copy(back.begin() + tile * probeIndex, back.begin() + tile * (probeIndex + 1), raw.begin() + tile * probeIndex);
        std::vector<sdfgi_probe> p(cascade.probes.size());
        check(sdfgi_probes_download(ctx_, cascade.level, p.data(), static_cast<int>(p.size())), "sdfgi_probes_download");
        Probe& q = cascade.probes[probeIndex];
        q.rejectHistory = p[probeIndex].reject_history != 0;
        q.lastUpdateFrame = p[probeIndex].last_update_frame;
        if (stats) merge(*stats, st);
        ProbeUpdateResult out;
        out.maxTexelDelta = res.max_texel_delta;
        out.raysTraced = static_cast<int>(res.rays_traced);
        return out;
    }

    // ------------------------------------------------------------- gather stage
    // renderGBuffer (shading.hpp:39-72) on the device; the G-buffer stays there for
    // gather() / composeFrame(), the returned copy is for the caller.
    GBuffer renderGBuffer(const Camera& camera, const Camera& prevCamera, int width, int height,
                          const RenderConfig& cfg) {
        sdfgi_camera c = toCamera(camera), pc = toCamera(prevCamera);
        sdfgi_cfg k = toCfg(cfg);
        check(sdfgi_gbuffer_render(ctx_, &c, &pc, width, height, &k), "sdfgi_gbuffer_render");
        return downloadGBuffer(width, height);
    }
    // a host G-buffer as the gather's input (instead of renderGBuffer)
    void uploadGBuffer(const GBuffer& gb) {
        std::vector<sdfgi_gbuffer_pixel> px(gb.pixels.size());
        for (size_t i = 0; i < px.size(); ++i) {
            const GBufferPixel& s = gb.pixels[i];
            sdfgi_gbuffer_pixel& d = px[i];
            std::memset(&d, 0, sizeof(d));
            d.depth = s.depth;
            for (int a = 0; a < 3; ++a) {
                d.normal[a] = s.normal[a];
                d.albedo[a] = s.albedo[a];
                d.emission[a] = s.emission[a];
                d.world_pos[a] = s.worldPos[a];
            }
            d.motion[0] = s.motion.x;
            d.motion[1] = s.motion.y;
            d.prim_index = s.primitiveIndex;
        }
        check(sdfgi_gbuffer_upload(ctx_, gb.width, gb.height, px.data()), "sdfgi_gbuffer_upload");
        gw_ = gb.width;
        gh_ = gb.height;
    }

    struct GatherResult {
        ImageRgb resolved;  // upsampleAndResolve's output (shading.hpp:350-426), next frame's history
        ImageRgb indirect;  // contactGI's output (shading.hpp:431-477)
        int64_t visibilityTasks = 0;
        double visTracesPerPixel = 0;
    };
    // The gather of pipeline.hpp:161-207 against the device's front atlas (prevField):
    // downsampleDepthCheckerboard, selectVisibilityPixels, buildVisibilityTasks,
    // runVisibilityTasks, shadePixelGI, upsampleAndResolve (with the device-held
    // history of the previous gather), contactGI; then the history roll of :213-218.
    GatherResult gather(int frameIndex, const RenderConfig& cfg, TraceStats* stats = nullptr) {
        sdfgi_cfg c = toCfg(cfg);
        sdfgi_stats vs{}, cs{};
        GatherResult g;
        check(sdfgi_gather(ctx_, frameIndex, &c, &g.visibilityTasks, &vs, &cs), "sdfgi_gather");
        if (stats) {
            merge(*stats, vs);
            merge(*stats, cs);
        }
        g.visTracesPerPixel = static_cast<double>(vs.visibility_traces) / (static_cast<double>(gw_) * gh_);
        g.resolved = downloadImage(0);
        g.indirect = downloadImage(1);
        return g;
    }
    void resetGatherHistory() { check(sdfgi_gather_reset_history(ctx_), "sdfgi_gather_reset_history"); }
    // composeFrame (shading.hpp:480-504) of the device G-buffer and the last gather's
    // indirect image (or one set with setIndirect).
    ImageRgb composeFrame(const RenderConfig& cfg, TraceStats* stats = nullptr) {
        sdfgi_cfg c = toCfg(cfg);
        sdfgi_stats st{};
        check(sdfgi_compose(ctx_, &c, stats ? &st : nullptr, nullptr), "sdfgi_compose");
        if (stats) merge(*stats, st);
        return downloadImage(8);
    }
    void setIndirect(const ImageRgb& img) {
        std::vector<double> v(3 * img.pixels.size());
        for (size_t i = 0; i < img.pixels.size(); ++i)
            for (int a = 0; a < 3; ++a) v[3 * i + a] = img.pixels[i][a];
        check(sdfgi_indirect_upload(ctx_, v.data(), v.size()), "sdfgi_indirect_upload");
    }

    // selectProbesForUpdate (probe_volume.hpp:154-198) on the device's probe state.
    std::vector<ProbeRef> selectProbesForUpdate(const std::vector<CascadeVolume>& cascades, const Vec3& camPos,
                                                const Vec3& camFwd, int budget, int frameIndex) {
        const double p[3] = {camPos.x, camPos.y, camPos.z}, f[3] = {camFwd.x, camFwd.y, camFwd.z};
        int total = 0;
        for (const auto& c : cascades) total += c.probeCount();
        std::vector<int32_t> r(2 * static_cast<size_t>(std::max(0, std::min(budget, total))) + 2);
        int n = 0;
        check(sdfgi_select_probes(ctx_, p, f, budget, frameIndex, r.data(), &n), "sdfgi_select_probes");
        std::vector<ProbeRef> out(n);
        for (int i = 0; i < n; ++i) {
            int slot = 0;
            for (size_t k = 0; k < cascades.size(); ++k)
                if (cascades[k].level == r[2 * i]) slot = static_cast<int>(k);
            out[i] = {slot, r[2 * i + 1]};
        }
        return out;
    }

    // recenterCascade (probe_volume.hpp:80-86) + the atlas clear of pipeline.hpp:110-113
    // for the device copy of `c` (call after the host recenterCascade returned true).
    void recenterCascade(const CascadeVolume& c, int octRes) {
        const double o[3] = {c.origin.x, c.origin.y, c.origin.z};
        check(sdfgi_cascade_set(ctx_, c.level, c.resX, c.resY, c.resZ, c.spacing, o, octRes), "sdfgi_cascade_set");
    }
    void swapAtlases() { check(sdfgi_atlas_swap(ctx_), "sdfgi_atlas_swap"); }
    // refresh host cascades / atlases from the device (front = the read side)
    void pullCascade(CascadeVolume& c) { pullProbes(c); }
    void pullAtlas(const CascadeVolume& c, ProbeAtlas& a, bool front = true) {
        auto& raw = const_cast<std::vector<float>&>(a.raw());
        check(sdfgi_atlas_download(ctx_, c.level, front ? 0 : 1, raw.data(), raw.size()), "sdfgi_atlas_download");
    }

    void* handle() const { return ctx_; }

private:
    static sdfgi_camera toCamera(const Camera& c) {
        sdfgi_camera o;
        for (int a = 0; a < 3; ++a) {
            o.position[a] = c.position[a];
            o.forward[a] = c.forward[a];
            o.right[a] = c.right[a];
            o.up[a] = c.up[a];
        }
        o.fov_y_deg = c.fovYDeg;
        return o;
    }
    GBuffer downloadGBuffer(int w, int h) {
        gw_ = w;
        gh_ = h;
        std::vector<sdfgi_gbuffer_pixel> px(static_cast<size_t>(w) * h);
        check(sdfgi_gbuffer_download(ctx_, px.data(), px.size()), "sdfgi_gbuffer_download");
        GBuffer gb(w, h);
        for (size_t i = 0; i < px.size(); ++i) {
            GBufferPixel& d = gb.pixels[i];
            const sdfgi_gbuffer_pixel& s = px[i];
            d.depth = s.depth;
            d.normal = {s.normal[0], s.normal[1], s.normal[2]};
            d.albedo = {s.albedo[0], s.albedo[1], s.albedo[2]};
            d.emission = {s.emission[0], s.emission[1], s.emission[2]};
            d.worldPos = {s.world_pos[0], s.world_pos[1], s.world_pos[2]};
            d.motion = {s.motion[0], s.motion[1]};
            d.primitiveIndex = s.prim_index;
        }
        return gb;
    }
    ImageRgb downloadImage(int which) {
        ImageRgb img(gw_, gh_);
        std::vector<double> v(3 * img.pixels.size());
        check(sdfgi_gather_download(ctx_, which, v.data(), v.size() * 8), "sdfgi_gather_download");
        for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
        return img;
    }
    // a reference IrradianceField as the device's probe state + front atlas
    void syncField(const IrradianceField& f, int octRes) {
        int n = 0;
        check(sdfgi_cascade_count(ctx_, &n), "sdfgi_cascade_count");
        bool same = n == static_cast<int>(f.cascades->size());
        if (!same) syncCascades(*f.cascades, octRes, f.atlases);
        else {
            for (size_t i = 0; i < f.cascades->size(); ++i) {
                pushProbes((*f.cascades)[i]);
                check(sdfgi_atlas_upload(ctx_, (*f.cascades)[i].level, 0, (*f.atlases)[i].raw().data(),
                                         (*f.atlases)[i].raw().size()),
                      "sdfgi_atlas_upload");
            }
        }
    }
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
    int gw_ = 0, gh_ = 0;
};

// Renderer (pipeline.hpp:50-230) with every per-frame stage but scene instancing
// and culling (the reference's own sceneAtTime + cullAndLod, host) on the device.
// Same constructor, accessors and renderFrame() as the reference's; the stage
// times in FrameMetrics are host wall-clock around each (synchronous) stage call.
class Renderer {
public:
    Renderer(SceneFile file, int width, int height, bool fp64 = true)
        : file_(std::move(file)), cfg_(file_.config), width_(width), height_(height), gpu_(0, fp64) {
        camera_ = buildCamera(file_.camera);
        prevCamera_ = camera_;
        for (int level = 0; level < file_.cascade.levels; ++level)
            cascades_.push_back(makeCascade(file_.cascade.resX, file_.cascade.resY, file_.cascade.resZ,
                                            file_.cascade.spacing, level, camera_.position));
        // the scene goes first: the device's acceleration grid grows over the cascades
        SceneState state = sceneAtTime(file_, 0.0);
        ActiveScene a = cullAndLod(state.primitives, camera_.position, file_.lodDistances,
                                   {cfg_.maxPerCluster, cfg_.mergeRadius});
        a.lights = state.lights;
        a.sky = state.sky;
        gpu_.uploadScene(a);
        gpu_.syncCascades(cascades_, cfg_.octRes);
        gpu_.resetGatherHistory();
    }

    const RenderConfig& config() const { return cfg_; }
    RenderConfig& config() { return cfg_; }
    int frameIndex() const { return frame_; }
    const Camera& camera() const { return camera_; }
    void setCamera(const Camera& cam) { camera_ = cam; }
    void setGiEnabled(bool on) { giEnabled_ = on; }
    const std::vector<CascadeVolume>& cascades() const { return cascades_; }
    const ActiveScene& activeScene() const { return active_; }
    const GBuffer& gbuffer() const { return gbuffer_; }
    const ImageRgb& image() const { return image_; }
    const ImageRgb& indirect() const { return indirect_; }
    const ImageRgb& resolvedIrradiance() const { return resolved_; }
    Device& device() { return gpu_; }

    FrameMetrics renderFrame() {
        using Clock = std::chrono::steady_clock;
        auto ms = [](Clock::time_point a, Clock::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        FrameMetrics m;
        m.frame = frame_;
        TraceStats stats;
        auto t0 = Clock::now();
        SceneState state = sceneAtTime(file_, static_cast<double>(frame_) / cfg_.fps);
        active_ = cullAndLod(state.primitives, camera_.position, file_.lodDistances,
                             {cfg_.maxPerCluster, cfg_.mergeRadius});
        active_.lights = state.lights;
        active_.sky = state.sky;
        active_.frameIndex = frame_;
        m.activePrimitives = static_cast<int>(active_.primitives.size());
        m.clusters = static_cast<int>(active_.clusters.size());
        gpu_.uploadScene(active_);
        auto t1 = Clock::now();
        m.tCullMs = ms(t0, t1);
        for (size_t ci = 0; ci < cascades_.size(); ++ci) {
            if (sdfgi::recenterCascade(cascades_[ci], camera_.position)) gpu_.recenterCascade(cascades_[ci], cfg_.octRes);
            auto rep = gpu_.updateProbePositions(cascades_[ci], cfg_.threshold1(cascades_[ci].spacing),
                                                 cfg_.threshold2(cascades_[ci].spacing), cfg_.maxDescentSteps, &stats,
                                                 cfg_.gradientStep);
            m.relocated += rep.relocated;
            m.rejected += rep.rejected;
            m.dead += rep.dead;
            m.probesTotal += cascades_[ci].probeCount();
        }
        auto t2 = Clock::now();
        m.tProbePosMs = ms(t1, t2);
        if (giEnabled_) {
            const int budget = cfg_.probeBudget > 0 ? cfg_.probeBudget : m.probesTotal;
            std::vector<ProbeRef> refs;
            if (budget < m.probesTotal) {
                refs = gpu_.selectProbesForUpdate(cascades_, camera_.position, camera_.forward, budget, frame_);
            } else {
                for (size_t ci = 0; ci < cascades_.size(); ++ci)
                    for (int i = 0; i < cascades_[ci].probeCount(); ++i) refs.push_back({static_cast<int>(ci), i});
            }
            m.probesUpdated = static_cast<int>(refs.size());
            std::vector<ProbeAtlas> back;
            for (const auto& c : cascades_) back.emplace_back(c.probeCount(), cfg_.octRes);
            auto r = gpu_.updateProbes(cascades_, refs, cfg_, frame_, back, &stats);  // swaps: back is the front now
            m.jitterMaxTexelDelta = r.maxTexelDelta;
            front_ = std::move(back);
        }
        auto t3 = Clock::now();
        m.tProbeUpdateMs = ms(t2, t3);
        // the gather reads the previous field: the front before this frame's update
        if (giEnabled_) gpu_.swapAtlases();
        gbuffer_ = gpu_.renderGBuffer(camera_, prevCamera_, width_, height_, cfg_);
        auto t4 = Clock::now();
        m.tGBufferMs = ms(t3, t4);
        if (giEnabled_) {
            auto g = gpu_.gather(frame_, cfg_, &stats);
            m.visTracesPerPixel = g.visTracesPerPixel;
            resolved_ = std::move(g.resolved);
            indirect_ = std::move(g.indirect);
        } else {
            indirect_ = ImageRgb(width_, height_);
            gpu_.setIndirect(indirect_);
        }
        auto t7 = Clock::now();
        m.tContactMs = ms(t4, t7);
        image_ = gpu_.composeFrame(cfg_, &stats);
        auto t8 = Clock::now();
        m.tComposeMs = ms(t7, t8);
        if (giEnabled_) gpu_.swapAtlases();  // readIdx_ = writeIdx (pipeline.hpp:224)
        prevCamera_ = camera_;
        ++frame_;
        m.stats = stats;
        return m;
    }

private:
    SceneFile file_;
    RenderConfig cfg_;
    int width_, height_;
    Device gpu_;
    Camera camera_, prevCamera_;
    std::vector<CascadeVolume> cascades_;
    std::vector<ProbeAtlas> front_;
    bool giEnabled_ = true;
    ActiveScene active_;
    GBuffer gbuffer_;
    ImageRgb indirect_, image_, resolved_;
    int frame_ = 0;
};

}  // namespace sdfgi::b200
