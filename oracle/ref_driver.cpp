// ref_driver.cpp — TEST INFRASTRUCTURE, not product code.
//
// A small driver that #includes the UNMODIFIED reference headers from
// /root/reference/proj/include and calls their public functions, so the
// reference itself produces the golden fixtures (tests/golden/) and the CPU
// baseline timing. Built by oracle/Makefile into oracle/_ref/ (git-ignored):
//   ref_parity : -O3 -march=x86-64-v3 -ffp-contract=off  (bit-exact goldens)
//   ref_perf   : -O3 -march=<v4|v3>                        (CPU baseline, shipped-like flags)
// No reference source is copied into this repository.
//
// Subcommands
//   scene  <file.scene> <out.sdfs>
//       loadSceneFile -> sceneAtTime(0) -> cullAndLod (scene_file.hpp:447,584;
//       scene.hpp:188) and write the SDFS interchange file (layout: include/sdfgi_b200.h).
//   passes <in.sdfs> <outdir> [options]
//       the probe stage of Renderer::renderFrame (pipeline.hpp:108-151) for P passes
//       (frame = pass index): updateProbePositions, atlas copy, updateProbe for every
//       alive probe; dumps probe state, SDFA atlas, per-ray records and a summary.
//   gather <in.sdfs> <outdir> [options]
//       C3: probe passes, then renderGBuffer and the gather stages of renderFrame
//       (pipeline.hpp:155-207) for the requested frames; dumps every stage buffer.
#include <sdfgi/pipeline.hpp>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "../include/sdfgi_b200.h"

using namespace sdfgi;

namespace {

struct SdfsHeader {
    char magic[4];
    uint32_t version;
    uint32_t nPrims, nLights, nClusters, nMembers;
    double sky[3];
    double camPos[3], camForward[3], camRight[3], camUp[3];
    double fovY;
    int32_t res[3];
    int32_t levels;
    double spacing;
};
static_assert(sizeof(SdfsHeader) == 176, "SDFS header layout");
static_assert(sizeof(sdfgi_prim) == 184, "prim layout");
static_assert(sizeof(sdfgi_light) == 80, "light layout");
static_assert(sizeof(sdfgi_cluster) == 56, "cluster layout");
static_assert(sizeof(sdfgi_cfg) == 224, "cfg layout");
static_assert(sizeof(sdfgi_probe) == 88, "probe layout");

struct Loaded {
    ActiveScene scene;
    Camera camera;
    CascadeSpec cascade;
    RenderConfig cfg;
};

void v3out(double* o, const Vec3& v) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
Vec3 v3in(const double* o) { return {o[0], o[1], o[2]}; }

sdfgi_cfg toCfg(const RenderConfig& c) {
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

RenderConfig fromCfg(const sdfgi_cfg& o) {
    RenderConfig c;
    c.surfaceEpsilon = o.surface_epsilon;
    c.maxTraceSteps = static_cast<int>(o.max_trace_steps);
    c.shadowSteps = static_cast<int>(o.shadow_steps);
    c.rayTMax = o.ray_tmax;
    c.shadowK = o.shadow_k;
    c.probeVisibilityK = o.probe_visibility_k;
    c.gradientStep = o.gradient_step;
    c.maxPerCluster = static_cast<int>(o.max_per_cluster);
    c.mergeRadius = o.merge_radius;
    c.threshold1Frac = o.threshold1_frac;
    c.threshold2Frac = o.threshold2_frac;
    c.maxDescentSteps = static_cast<int>(o.max_descent_steps);
    c.probeBudget = static_cast<int>(o.probe_budget);
    c.nRaysFull = static_cast<int>(o.n_rays_full);
    c.hysteresis = o.hysteresis;
    c.alphaMin = o.alpha_min;
    c.bounceCoeff = o.bounce_coeff;
    c.octRes = static_cast<int>(o.oct_res);
    c.rotatePerFrame = o.rotate_per_frame != 0;
    c.seed = o.seed;
    c.mvcRelocationFrac = o.mvc_relocation_frac;
    c.dedupQuantFrac = o.dedup_quant_frac;
    c.contactRadiusFrac = o.contact_radius_frac;
    c.contactSamples = static_cast<int>(o.contact_samples);
    c.historyBlend = o.history_blend;
    c.depthSigmaFrac = o.depth_sigma_frac;
    c.exposure = o.exposure;
    c.fps = static_cast<int>(o.fps);
    return c;
}

void writeSdfs(const std::string& path, const ActiveScene& s, const Camera& cam,
               const CascadeSpec& cs, const RenderConfig& cfg) {
    SdfsHeader h;
    std::memset(&h, 0, sizeof(h));
    std::memcpy(h.magic, "SDFS", 4);
    h.version = 1;
    h.nPrims = static_cast<uint32_t>(s.primitives.size());
    h.nLights = static_cast<uint32_t>(s.lights.size());
    h.nClusters = static_cast<uint32_t>(s.clusters.size());
    uint32_t nm = 0;
    for (auto& c : s.clusters) nm += static_cast<uint32_t>(c.members.size());
    h.nMembers = nm;
    v3out(h.sky, s.sky);
    v3out(h.camPos, cam.position);
    v3out(h.camForward, cam.forward);
    v3out(h.camRight, cam.right);
    v3out(h.camUp, cam.up);
    h.fovY = cam.fovYDeg;
    h.res[0] = cs.resX;
    h.res[1] = cs.resY;
    h.res[2] = cs.resZ;
    h.levels = cs.levels;
    h.spacing = cs.spacing;
    std::ofstream out(path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(&h), sizeof(h));
    sdfgi_cfg c = toCfg(cfg);
    out.write(reinterpret_cast<const char*>(&c), sizeof(c));
    for (auto& p : s.primitives) {
        sdfgi_prim q;
        std::memset(&q, 0, sizeof(q));
        q.id = p.id;
        q.kind = static_cast<int32_t>(p.kind);
        q.lod_tier = p.lodTier;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) q.rot[i * 3 + j] = p.transform.rotation.m[i][j];
        v3out(q.trans, p.transform.translation);
        v3out(q.size, p.size);
        v3out(q.albedo, p.material.albedo);
        v3out(q.emission, p.material.emission);
        out.write(reinterpret_cast<const char*>(&q), sizeof(q));
    }
    for (auto& l : s.lights) {
        sdfgi_light q;
        std::memset(&q, 0, sizeof(q));
        q.kind = static_cast<int32_t>(l.kind);
        v3out(q.position, l.position);
        v3out(q.direction, l.direction);
        v3out(q.intensity, l.intensity);
        out.write(reinterpret_cast<const char*>(&q), sizeof(q));
    }
    for (auto& c : s.clusters) {
        sdfgi_cluster q;
        std::memset(&q, 0, sizeof(q));
        v3out(q.lo, c.cullAabb.lo);
        v3out(q.hi, c.cullAabb.hi);
        q.unbounded = c.unbounded ? 1 : 0;
        out.write(reinterpret_cast<const char*>(&q), sizeof(q));
    }
    std::vector<int32_t> start{0}, idx;
    for (auto& c : s.clusters) {
        for (int m : c.members) idx.push_back(m);
        start.push_back(static_cast<int32_t>(idx.size()));
    }
    out.write(reinterpret_cast<const char*>(start.data()), start.size() * 4);
    out.write(reinterpret_cast<const char*>(idx.data()), idx.size() * 4);
    if ((start.size() + idx.size()) % 2) {
        int32_t z = 0;
        out.write(reinterpret_cast<const char*>(&z), 4);
    }
}

Loaded readSdfs(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    SdfsHeader h;
    in.read(reinterpret_cast<char*>(&h), sizeof(h));
    if (std::memcmp(h.magic, "SDFS", 4) != 0 || h.version != 1)
        throw std::runtime_error("bad SDFS file " + path);
    sdfgi_cfg c;
    in.read(reinterpret_cast<char*>(&c), sizeof(c));
    Loaded L;
    L.cfg = fromCfg(c);
    L.scene.sky = v3in(h.sky);
    L.camera.position = v3in(h.camPos);
    L.camera.forward = v3in(h.camForward);
    L.camera.right = v3in(h.camRight);
    L.camera.up = v3in(h.camUp);
    L.camera.fovYDeg = h.fovY;
    L.cascade.resX = h.res[0];
    L.cascade.resY = h.res[1];
    L.cascade.resZ = h.res[2];
    L.cascade.levels = h.levels;
    L.cascade.spacing = h.spacing;
    for (uint32_t i = 0; i < h.nPrims; ++i) {
        sdfgi_prim q;
        in.read(reinterpret_cast<char*>(&q), sizeof(q));
        SdfPrimitive p;
        p.id = q.id;
        p.kind = static_cast<PrimitiveKind>(q.kind);
        p.lodTier = q.lod_tier;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) p.transform.rotation.m[a][b] = q.rot[a * 3 + b];
        p.transform.translation = v3in(q.trans);
        p.size = v3in(q.size);
        p.material.albedo = v3in(q.albedo);
        p.material.emission = v3in(q.emission);
        L.scene.primitives.push_back(p);
    }
    for (uint32_t i = 0; i < h.nLights; ++i) {
        sdfgi_light q;
        in.read(reinterpret_cast<char*>(&q), sizeof(q));
        Light l;
        l.kind = static_cast<LightKind>(q.kind);
        l.position = v3in(q.position);
        l.direction = v3in(q.direction);
        l.intensity = v3in(q.intensity);
        L.scene.lights.push_back(l);
    }
    std::vector<sdfgi_cluster> cl(h.nClusters);
    in.read(reinterpret_cast<char*>(cl.data()), cl.size() * sizeof(sdfgi_cluster));
    std::vector<int32_t> start(h.nClusters + 1), idx(h.nMembers);
    in.read(reinterpret_cast<char*>(start.data()), start.size() * 4);
    in.read(reinterpret_cast<char*>(idx.data()), idx.size() * 4);
    if (!in) throw std::runtime_error("truncated SDFS file " + path);
    for (uint32_t k = 0; k < h.nClusters; ++k) {
        Cluster c;
        c.cullAabb.lo = v3in(cl[k].lo);
        c.cullAabb.hi = v3in(cl[k].hi);
        c.aabb = c.cullAabb;
        c.unbounded = cl[k].unbounded != 0;
        for (int m = start[k]; m < start[k + 1]; ++m) {
            c.members.push_back(idx[m]);
            c.memberIds.push_back(L.scene.primitives[idx[m]].id);
        }
        c.centroid = c.aabb.center();
        L.scene.clusters.push_back(std::move(c));
    }
    L.scene.finalize();
    return L;
}

template <typename T>
void writeVec(const std::string& path, const std::vector<T>& v) {
    std::ofstream out(path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
}

std::string statsJson(const TraceStats& s) {
    std::ostringstream o;
    o << "{\"sdf_queries\": " << s.sdfQueries << ", \"clusters_visited\": " << s.clustersVisited
      << ", \"clusters_skipped\": " << s.clustersSkipped
      << ", \"primitive_evals\": " << s.primitiveEvals << ", \"trace_steps\": " << s.traceSteps
      << ", \"sphere_traces\": " << s.sphereTraces << ", \"shadow_traces\": " << s.shadowTraces
      << ", \"visibility_traces\": " << s.visibilityTraces << "}";
    return o.str();
}

std::vector<sdfgi_probe> probeDump(const CascadeVolume& c) {
    std::vector<sdfgi_probe> out(c.probes.size());
    for (size_t i = 0; i < c.probes.size(); ++i) {
        const Probe& p = c.probes[i];
        sdfgi_probe& q = out[i];
        std::memset(&q, 0, sizeof(q));
        v3out(q.resting, p.restingPos);
        v3out(q.pos, p.pos);
        v3out(q.last_pos, p.lastPos);
        q.reject_history = p.rejectHistory ? 1 : 0;
        q.alive = p.alive ? 1 : 0;
        q.last_update_frame = p.lastUpdateFrame;
    }
    return out;
}

struct Opts {
    int passes = 1;
    int threads = 1;
    int res[3] = {0, 0, 0};
    double spacing = 0;
    int nRays = 0;
    int stride = 1;          // update every stride-th probe (bounded CPU-baseline sample)
    int reps = 1;            // timing repetitions of the whole run
    bool dump = true;
    std::vector<int> debugProbes;
    std::vector<std::string> sets;  // "key value" config overrides
    int width = 0, height = 0;  // gather
    int gatherFrames = 2;
    int budget = 0;  // probeBudget for selectProbesForUpdate (0 = every probe)
    int dumpEvery = 1;  // dynamic: probes/atlas dump period
};

void applySet(RenderConfig& c, const std::string& kv) {
    std::istringstream is(kv);
    std::string k;
    double v;
    is >> k >> v;
    if (k == "n_rays") c.nRaysFull = static_cast<int>(v);
    else if (k == "bounce_coeff") c.bounceCoeff = v;
    else if (k == "hysteresis") c.hysteresis = v;
    else if (k == "seed") c.seed = static_cast<uint64_t>(v);
    else if (k == "rotate_per_frame") c.rotatePerFrame = v != 0;
    else if (k == "oct_res") c.octRes = static_cast<int>(v);
    else if (k == "shadow_steps") c.shadowSteps = static_cast<int>(v);
    else if (k == "max_trace_steps") c.maxTraceSteps = static_cast<int>(v);
    else if (k == "contact_samples") c.contactSamples = static_cast<int>(v);
    else throw std::runtime_error("unknown --set key " + k);
}

Opts parseOpts(int argc, char** argv, int first) {
    Opts o;
    for (int i = first; i < argc; ++i) {
        std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
            return argv[++i];
        };
        if (a == "--passes") o.passes = std::stoi(next());
        else if (a == "--threads") o.threads = std::stoi(next());
        else if (a == "--res") {
            o.res[0] = std::stoi(next());
            o.res[1] = std::stoi(next());
            o.res[2] = std::stoi(next());
        } else if (a == "--spacing") o.spacing = std::stod(next());
        else if (a == "--nrays") o.nRays = std::stoi(next());
        else if (a == "--stride") o.stride = std::stoi(next());
        else if (a == "--reps") o.reps = std::stoi(next());
        else if (a == "--no-dump") o.dump = false;
        else if (a == "--debug-probe") o.debugProbes.push_back(std::stoi(next()));
        else if (a == "--set") o.sets.push_back(next());
        else if (a == "--size") {
            o.width = std::stoi(next());
            o.height = std::stoi(next());
        } else if (a == "--gather-frames") o.gatherFrames = std::stoi(next());
        else if (a == "--budget") o.budget = std::stoi(next());
        else if (a == "--dump-every") o.dumpEvery = std::stoi(next());
        else throw std::runtime_error("unknown option " + a);
    }
    return o;
}

// The probe-stage state of Renderer (pipeline.hpp:51-68) without the Renderer, so
// the cascade resolution / ray count can be overridden per config.
struct ProbeStage {
    ActiveScene scene;
    RenderConfig cfg;
    Camera camera;
    std::vector<CascadeVolume> cascades;
    std::vector<ProbeAtlas> atlas[2];
    int readIdx = 0;
};

void initStage(ProbeStage& st, const Loaded& L, const Opts& o) {
    st.scene = L.scene;
    st.cfg = L.cfg;
    for (auto& s : o.sets) applySet(st.cfg, s);
    if (o.nRays > 0) st.cfg.nRaysFull = o.nRays;
    st.camera = L.camera;
    CascadeSpec cs = L.cascade;
    if (o.res[0] > 0) {
        cs.resX = o.res[0];
        cs.resY = o.res[1];
        cs.resZ = o.res[2];
    }
    if (o.spacing > 0) cs.spacing = o.spacing;
    st.cascades.clear();
    for (int level = 0; level < cs.levels; ++level)
        st.cascades.push_back(
            makeCascade(cs.resX, cs.resY, cs.resZ, cs.spacing, level, st.camera.position));
    for (int b = 0; b < 2; ++b) {
        st.atlas[b].clear();
        for (auto& c : st.cascades) st.atlas[b].emplace_back(c.probeCount(), st.cfg.octRes);
    }
    st.readIdx = 0;
}

struct PassResult {
    RelocationReport rep;
    TraceStats relocStats, updateStats;
    long long rays = 0;
    int updated = 0;
    double jitter = 0;
    double relocMs = 0, updateMs = 0;
    std::vector<int32_t> refs;  // selected (cascade, index) pairs
};

// One probe pass of renderFrame (pipeline.hpp:108-151), frame = `frame`.
PassResult runPass(ProbeStage& st, int frame, const Opts& o, std::vector<sdfgi_ray_record>* rays) {
    using Clock = std::chrono::steady_clock;
    PassResult r;
    auto t0 = Clock::now();
    for (size_t ci = 0; ci < st.cascades.size(); ++ci) {
        auto rep = updateProbePositions(st.cascades[ci], st.scene,
                                        st.cfg.threshold1(st.cascades[ci].spacing),
                                        st.cfg.threshold2(st.cascades[ci].spacing),
                                        st.cfg.maxDescentSteps, &r.relocStats,
                                        st.cfg.gradientStep);
        r.rep.relocated += rep.relocated;
        r.rep.rejected += rep.rejected;
        r.rep.dead += rep.dead;
    }
    auto t1 = Clock::now();
    int writeIdx = 1 - st.readIdx;
    IrradianceField prevField{&st.cascades, &st.atlas[st.readIdx]};

    // per-ray records for the debug probes, exactly as updateProbe traces them
    // (probe_update.hpp:173-189), captured before the probe's state changes
    if (rays) {
        for (int pi : o.debugProbes) {
            CascadeVolume& c = st.cascades[0];
            const Probe& probe = c.probes[pi];
            int n = probe.rejectHistory ? st.cfg.nRaysFull * 2 : st.cfg.nRaysFull;
            ProbeRef ref{c.level, pi};
            auto dirs = sampleDirections(n, frame, probeKey(ref), st.cfg.seed, st.cfg.rotatePerFrame);
            for (int i = 0; i < n; ++i) {
                Hit hit = sphereTrace(st.scene, probe.pos, dirs[i], st.cfg.rayTMax,
                                      st.cfg.surfaceEpsilon, st.cfg.maxTraceSteps);
                sdfgi_ray_record rec;
                std::memset(&rec, 0, sizeof(rec));
                v3out(rec.dir, dirs[i]);
                Vec3 L = hit.converged ? shadeHit(st.scene, hit, prevField, st.cfg.bounceCoeff, st.cfg)
                                       : st.scene.sky;
                rec.t = hit.converged ? hit.t : 0.0;
                v3out(rec.radiance, L);
                v3out(rec.normal, hit.normal);
                rec.converged = hit.converged ? 1 : 0;
                rec.miss = static_cast<int32_t>(hit.miss);
                rec.prim_index = hit.primitiveIndex;
                rec.steps = 0;  // the reference Hit does not expose its step count
                rays->push_back(rec);
            }
        }
    }

    st.atlas[writeIdx] = st.atlas[st.readIdx];
    int total = 0;
    for (auto& c : st.cascades) total += c.probeCount();
    // pipeline.hpp:133-135: budget = probeBudget > 0 ? probeBudget : every probe
    auto refs = selectProbesForUpdate(st.cascades, st.camera.position, st.camera.forward,
                                      o.budget > 0 ? o.budget : total, frame);
    for (const ProbeRef& ref : refs) {
        r.refs.push_back(ref.cascade);
        r.refs.push_back(ref.index);
    }
    if (o.stride > 1) {
        std::vector<ProbeRef> sub;
        for (auto& ref : refs)
            if (ref.index % o.stride == 0) sub.push_back(ref);
        refs.swap(sub);
    }
    int threads = std::max(1, o.threads);
    std::vector<TraceStats> chunkStats(threads);
    std::vector<double> chunkJitter(threads, 0.0);
    std::vector<long long> chunkRays(threads, 0);
    std::vector<int> chunkUpdated(threads, 0);
    parallelFor(0, static_cast<int64_t>(refs.size()), threads, [&](int64_t i, int worker) {
        const ProbeRef& ref = refs[i];
        if (!st.cascades[ref.cascade].probes[ref.index].alive) return;
        auto res = updateProbe(st.scene, st.cascades[ref.cascade], ref.index, prevField,
                               st.atlas[writeIdx][ref.cascade], st.cfg.nRaysFull, st.cfg, frame,
                               &chunkStats[worker]);
        chunkJitter[worker] = std::max(chunkJitter[worker], res.maxTexelDelta);
        chunkRays[worker] += res.raysTraced;
        chunkUpdated[worker] += 1;
    });
    auto t2 = Clock::now();
    for (int w = 0; w < threads; ++w) {
        r.updateStats.merge(chunkStats[w]);
        r.jitter = std::max(r.jitter, chunkJitter[w]);
        r.rays += chunkRays[w];
        r.updated += chunkUpdated[w];
    }
    st.readIdx = writeIdx;  // frame-end swap (pipeline.hpp:220)
    r.relocMs = std::chrono::duration<double, std::milli>(t1 - t0).count();
    r.updateMs = std::chrono::duration<double, std::milli>(t2 - t1).count();
    return r;
}

int cmdScene(int argc, char** argv) {
    if (argc < 4) throw std::runtime_error("usage: scene <file.scene> <out.sdfs>");
    SceneFile f = loadSceneFile(argv[2]);
    SceneState state = sceneAtTime(f, 0);
    Camera cam = buildCamera(f.camera);
    ActiveScene active = cullAndLod(state.primitives, cam.position, f.lodDistances,
                                    {f.config.maxPerCluster, f.config.mergeRadius});
    active.lights = state.lights;
    active.sky = state.sky;
    writeSdfs(argv[3], active, cam, f.cascade, f.config);
    std::printf("{\"prims\": %zu, \"clusters\": %zu, \"lights\": %zu}\n", active.primitives.size(),
                active.clusters.size(), active.lights.size());
    return 0;
}

// Re-cluster an SDFS scene with the reference builder (buildClusters, scene.hpp:110-178),
// used for small synthetic fixtures so both sides see reference-built clusters.
int cmdRecluster(int argc, char** argv) {
    if (argc < 6) throw std::runtime_error("usage: recluster <in.sdfs> <out.sdfs> <maxPer> <mergeRadius>");
    Loaded L = readSdfs(argv[2]);
    L.scene.clusters = buildClusters(L.scene.primitives, std::stoi(argv[4]), std::stod(argv[5]));
    L.scene.finalize();
    writeSdfs(argv[3], L.scene, L.camera, L.cascade, L.cfg);
    std::printf("{\"prims\": %zu, \"clusters\": %zu}\n", L.scene.primitives.size(),
                L.scene.clusters.size());
    return 0;
}

int cmdPasses(int argc, char** argv) {
    if (argc < 4) throw std::runtime_error("usage: passes <in.sdfs> <outdir> [opts]");
    Loaded L = readSdfs(argv[2]);
    std::string dir = argv[3];
    Opts o = parseOpts(argc, argv, 4);
    std::ostringstream js;
    js << "{\"threads\": " << o.threads << ", \"stride\": " << o.stride << ", \"reps\": [";
    for (int rep = 0; rep < o.reps; ++rep) {
        ProbeStage st;
        initStage(st, L, o);
        if (rep) js << ", ";
        js << "[";
        for (int p = 0; p < o.passes; ++p) {
            std::vector<sdfgi_ray_record> rays;
            bool dump = o.dump && rep == 0;
            PassResult r = runPass(st, p, o, dump ? &rays : nullptr);
            if (dump) {
                std::string sfx = "_p" + std::to_string(p);
                for (size_t ci = 0; ci < st.cascades.size(); ++ci) {
                    std::string c = "_c" + std::to_string(ci);
                    writeVec(dir + "/probes" + sfx + c + ".bin", probeDump(st.cascades[ci]));
                    st.atlas[st.readIdx][ci].dump(dir + "/atlas" + sfx + c + ".sdfa");
                }
                if (!rays.empty()) writeVec(dir + "/rays" + sfx + ".bin", rays);
                if (o.budget > 0) writeVec(dir + "/refs" + sfx + ".bin", r.refs);
            }
            if (p) js << ", ";
            js << "{\"pass\": " << p << ", \"relocated\": " << r.rep.relocated
               << ", \"rejected\": " << r.rep.rejected << ", \"dead\": " << r.rep.dead
               << ", \"rays_traced\": " << r.rays << ", \"probes_updated\": " << r.updated
               << ", \"max_texel_delta\": " << r.jitter << ", \"reloc_ms\": " << r.relocMs
               << ", \"update_ms\": " << r.updateMs
               << ", \"reloc_stats\": " << statsJson(r.relocStats)
               << ", \"update_stats\": " << statsJson(r.updateStats) << "}";
        }
        js << "]";
    }
    js << "]}";
    std::cout << js.str() << std::endl;
    return 0;
}

void dumpImage(const std::string& path, const ImageRgb& img) {
    std::vector<double> v;
    v.reserve(img.pixels.size() * 3);
    for (const Vec3& p : img.pixels) {
        v.push_back(p.x);
        v.push_back(p.y);
        v.push_back(p.z);
    }
    writeVec(path, v);
}

// C5: a dynamic sequence. Per frame f: sceneAtTime(f / fps), cullAndLod with the
// scene's clustering (pipeline.hpp:92-103), then the probe pass of renderFrame with
// frame index f on the persistent cascades. Dumps every frame's active scene
// (frame<f>.sdfs) and, every --dump-every frames and on the last, probes + atlas.
int cmdDynamic(int argc, char** argv) {
    if (argc < 4) throw std::runtime_error("usage: dynamic <file.scene> <outdir> [opts]");
    SceneFile f = loadSceneFile(argv[2]);
    std::string dir = argv[3];
    Opts o = parseOpts(argc, argv, 4);
    Camera cam = buildCamera(f.camera);
    auto frameScene = [&](int frame) {
        double t = static_cast<double>(frame) / static_cast<double>(f.config.fps);
        SceneState state = sceneAtTime(f, t);
        ActiveScene a = cullAndLod(state.primitives, cam.position, f.lodDistances,
                                   {f.config.maxPerCluster, f.config.mergeRadius});
        a.lights = state.lights;
        a.sky = state.sky;
        a.frameIndex = frame;
        return a;
    };
    Loaded L;
    L.scene = frameScene(0);
    L.camera = cam;
    L.cascade = f.cascade;
    L.cfg = f.config;
    ProbeStage st;
    initStage(st, L, o);
    std::ostringstream js;
    js << "{\"frames\": [";
    for (int fr = 0; fr < o.passes; ++fr) {
        st.scene = frameScene(fr);
        std::string sfx = "_f" + std::to_string(fr);
        if (o.dump) writeSdfs(dir + "/frame" + sfx + ".sdfs", st.scene, cam, L.cascade, st.cfg);
        PassResult r = runPass(st, fr, o, nullptr);
        if (o.dump && (fr % std::max(1, o.dumpEvery) == 0 || fr + 1 == o.passes)) {
            for (size_t ci = 0; ci < st.cascades.size(); ++ci) {
                std::string c = "_c" + std::to_string(ci);
                writeVec(dir + "/probes" + sfx + c + ".bin", probeDump(st.cascades[ci]));
                st.atlas[st.readIdx][ci].dump(dir + "/atlas" + sfx + c + ".sdfa");
            }
        }
        if (fr) js << ", ";
        js << "{\"frame\": " << fr << ", \"relocated\": " << r.rep.relocated << ", \"rejected\": " << r.rep.rejected
           << ", \"dead\": " << r.rep.dead << ", \"rays_traced\": " << r.rays << ", \"probes_updated\": " << r.updated
           << ", \"max_texel_delta\": " << r.jitter << ", \"update_ms\": " << r.updateMs << "}";
    }
    js << "]}";
    std::cout << js.str() << std::endl;
    return 0;
}

// The whole reference frame loop: Renderer::renderFrame (pipeline.hpp:84-230) for
// --passes frames at --size W H; per frame the composed image (writeHdr, SDFI), and
// every FrameMetrics row (csvRow) into metrics.csv. --nrays overrides n_rays.
int cmdRender(int argc, char** argv) {
    if (argc < 4) throw std::runtime_error("usage: render <file.scene> <outdir> [opts]");
    SceneFile f = loadSceneFile(argv[2]);
    std::string dir = argv[3];
    Opts o = parseOpts(argc, argv, 4);
    if (o.width <= 0) throw std::runtime_error("--size W H required");
    if (o.nRays > 0) f.config.nRaysFull = o.nRays;
    for (auto& kv : o.sets) applySet(f.config, kv);
    Renderer r(f, o.width, o.height, std::max(1, o.threads));
    std::ofstream csv(dir + "/metrics.csv");
    csv << FrameMetrics::csvHeader() << "\n";
    std::ostringstream js;
    js << "{\"frames\": [";
    for (int fr = 0; fr < o.passes; ++fr) {
        FrameMetrics m = r.renderFrame();
        csv << m.csvRow() << "\n";
        if (o.dump) writeHdr(r.image(), dir + "/image_f" + std::to_string(fr) + ".sdfi");
        if (fr) js << ", ";
        js << "{\"frame\": " << m.frame << ", \"active_primitives\": " << m.activePrimitives
           << ", \"clusters\": " << m.clusters << ", \"probes_total\": " << m.probesTotal
           << ", \"probes_updated\": " << m.probesUpdated << ", \"relocated\": " << m.relocated
           << ", \"rejected\": " << m.rejected << ", \"dead\": " << m.dead
           << ", \"vis_traces_per_pixel\": " << m.visTracesPerPixel
           << ", \"jitter_max_texel_delta\": " << m.jitterMaxTexelDelta
           << ", \"ms\": " << (m.tCullMs + m.tProbePosMs + m.tProbeUpdateMs + m.tGBufferMs + m.tVisibilityMs +
                                m.tGiResolveMs + m.tContactMs + m.tComposeMs)
           << ", \"stats\": " << statsJson(m.stats) << "}";
    }
    js << "]}";
    std::cout << js.str() << std::endl;
    return 0;
}

// C3: probe passes, then renderGBuffer + the gather stages of renderFrame
// (pipeline.hpp:155-207) for --gather-frames frames against the final atlas.
int cmdGather(int argc, char** argv) {
    using Clock = std::chrono::steady_clock;
    if (argc < 4) throw std::runtime_error("usage: gather <in.sdfs> <outdir> [opts]");
    Loaded L = readSdfs(argv[2]);
    std::string dir = argv[3];
    Opts o = parseOpts(argc, argv, 4);
    if (o.width <= 0) throw std::runtime_error("--size W H required");
    ProbeStage st;
    initStage(st, L, o);
    for (int p = 0; p < o.passes; ++p) runPass(st, p, o, nullptr);
    const int W = o.width, H = o.height, T = std::max(1, o.threads);
    TraceStats gst;
    auto t0 = Clock::now();
    GBuffer gb = renderGBuffer(st.scene, st.camera, st.camera, W, H, st.cfg, &gst, T);
    double gbMs = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    if (o.dump) {
        std::vector<sdfgi_gbuffer_pixel> px(gb.pixels.size());
        for (size_t i = 0; i < px.size(); ++i) {
            const GBufferPixel& g = gb.pixels[i];
            sdfgi_gbuffer_pixel& q = px[i];
            std::memset(&q, 0, sizeof(q));
            q.depth = g.depth;
            v3out(q.normal, g.normal);
            v3out(q.albedo, g.albedo);
            v3out(q.emission, g.emission);
            v3out(q.world_pos, g.worldPos);
            q.motion[0] = g.motion.x;
            q.motion[1] = g.motion.y;
            q.prim_index = g.primitiveIndex;
        }
        writeVec(dir + "/gbuffer.bin", px);
        for (size_t ci = 0; ci < st.cascades.size(); ++ci) {
            std::string c = "_c" + std::to_string(ci);
            writeVec(dir + "/gprobes" + c + ".bin", probeDump(st.cascades[ci]));
            st.atlas[st.readIdx][ci].dump(dir + "/gatlas" + c + ".sdfa");
        }
    }
    IrradianceField field{&st.cascades, &st.atlas[st.readIdx]};
    HistoryBuffers history;
    std::ostringstream js;
    js << "{\"gbuffer_ms\": " << gbMs << ", \"gbuffer_stats\": " << statsJson(gst) << ", \"frames\": [";
    for (int f = 0; f < o.gatherFrames; ++f) {
        TraceStats vs, cs;
        auto a = Clock::now();
        HalfResDepth half = downsampleDepthCheckerboard(gb);
        SelectedPixels sel = selectVisibilityPixels(half, f);
        VisibilityWork work = buildVisibilityTasks(st.cascades, gb, half, sel, st.cfg);
        std::vector<double> vis = runVisibilityTasks(st.scene, st.cascades, work, st.cfg, &vs, T);
        SparseGi sparse;  // pipeline.hpp:173-185
        sparse.width = sel.width;
        sparse.height = sel.height;
        sparse.irradiance.resize(work.pixels.size());
        sparse.anchorPixel.resize(work.pixels.size());
        sparse.valid.assign(work.pixels.size(), 0);
        for (size_t i = 0; i < work.pixels.size(); ++i) {
            int anchor = half.srcPixel[sel.halfResIndex[i]];
            sparse.anchorPixel[i] = anchor;
            PixelGiResult r = shadePixelGI(work.pixels[i], vis, gb.pixels[anchor].normal, field);
            sparse.irradiance[i] = r.irradiance;
            sparse.valid[i] = r.valid ? 1 : 0;
        }
        auto b = Clock::now();
        ImageRgb resolved = upsampleAndResolve(sparse, gb, history, st.cascades, field, st.cfg, T);
        auto c = Clock::now();
        double radius = st.cfg.contactRadiusFrac * st.cascades[0].spacing;
        ImageRgb indirect = contactGI(st.scene, gb, resolved, field, radius, st.cfg.contactSamples, st.cfg, &cs, T);
        auto d = Clock::now();
        TraceStats ps;
        ImageRgb composed = composeFrame(st.scene, gb, indirect, st.cfg, &ps, T);  // pipeline.hpp:209
        auto e = Clock::now();
        if (o.dump) {
            std::string sfx = "_f" + std::to_string(f);
            writeVec(dir + "/half_depth" + sfx + ".bin", half.depth);
            writeVec(dir + "/half_src" + sfx + ".bin", half.srcPixel);
            writeVec(dir + "/sel" + sfx + ".bin", sel.halfResIndex);
            std::vector<double> irr;
            std::vector<int32_t> valid(sparse.valid.begin(), sparse.valid.end());
            for (const Vec3& v : sparse.irradiance) {
                irr.push_back(v.x);
                irr.push_back(v.y);
                irr.push_back(v.z);
            }
            writeVec(dir + "/sparse_irr" + sfx + ".bin", irr);
            writeVec(dir + "/sparse_valid" + sfx + ".bin", valid);
            writeVec(dir + "/sparse_anchor" + sfx + ".bin", sparse.anchorPixel);
            writeVec(dir + "/vis" + sfx + ".bin", vis);
            dumpImage(dir + "/resolved" + sfx + ".bin", resolved);
            dumpImage(dir + "/indirect" + sfx + ".bin", indirect);
            dumpImage(dir + "/composed" + sfx + ".bin", composed);
        }
        if (f) js << ", ";
        js << "{\"frame\": " << f << ", \"tasks\": " << work.tasks.size()
           << ", \"visibility_ms\": " << std::chrono::duration<double, std::milli>(b - a).count()
           << ", \"resolve_ms\": " << std::chrono::duration<double, std::milli>(c - b).count()
           << ", \"contact_ms\": " << std::chrono::duration<double, std::milli>(d - c).count()
           << ", \"compose_ms\": " << std::chrono::duration<double, std::milli>(e - d).count()
           << ", \"vis_stats\": " << statsJson(vs) << ", \"contact_stats\": " << statsJson(cs)
           << ", \"compose_stats\": " << statsJson(ps) << "}";
        history.irradiance = std::move(resolved);  // pipeline.hpp:214-218
        history.depth.resize(gb.pixels.size());
        for (size_t i = 0; i < gb.pixels.size(); ++i) history.depth[i] = gb.pixels[i].depth;
        history.valid = true;
    }
    js << "]}";
    std::cout << js.str() << std::endl;
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) {
            std::fprintf(stderr, "usage: %s scene|passes ...\n", argv[0]);
            return 2;
        }
        std::string cmd = argv[1];
        if (cmd == "scene") return cmdScene(argc, argv);
        if (cmd == "passes") return cmdPasses(argc, argv);
        if (cmd == "recluster") return cmdRecluster(argc, argv);
        if (cmd == "gather") return cmdGather(argc, argv);
        if (cmd == "dynamic") return cmdDynamic(argc, argv);
        if (cmd == "render") return cmdRender(argc, argv);
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
