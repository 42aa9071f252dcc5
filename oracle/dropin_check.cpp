// dropin_check.cpp — TEST INFRASTRUCTURE: the drop-in demonstration.
//
// Built against the UNMODIFIED reference headers (/root/reference/proj/include) and
// libsdfgi_b200.so by oracle/Makefile (target `dropin`, output oracle/_ref/). It
// runs the probe stage of Renderer::renderFrame (pipeline.hpp:108-151) twice on the
// same ActiveScene: once with the reference's own updateProbePositions +
// parallelFor(updateProbe), once with those calls replaced by the B200 drop-in
// (paper_2007_14394_b200/include/sdfgi_b200.hpp). It prints one JSON line with the
// comparison; tests/test_dropin.py asserts on it.
//
// usage: dropin_check <scene.sdfs> <passes> <resX> <resY> <resZ> <spacing> <nRays>
//        dropin_check render <file.scene> <frames> <width> <height> [nRays]
//            the whole Renderer::renderFrame loop: the reference's Renderer vs
//            sdfgi::b200::Renderer (every per-frame stage on the device)
//        dropin_check funcs <scene.sdfs> <resX> <resY> <resZ> <spacing> <nRays>
//            the free functions (querySceneSdf, sphereTrace, softShadowTrace,
//            interpolationStencil, convolveIrradiance, shadeHit, per-probe updateProbe)
//            against the reference's, after one reference probe pass
#include <sdfgi/pipeline.hpp>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>

#include "../paper_2007_14394_b200/include/sdfgi_b200.hpp"

using namespace sdfgi;

namespace {

struct Hdr {
    char magic[4];
    uint32_t version, nPrims, nLights, nClusters, nMembers;
    double sky[3], camPos[3], camF[3], camR[3], camU[3], fov;
    int32_t res[3], levels;
    double spacing;
};

ActiveScene readScene(const char* path, Vec3& cam, RenderConfig& cfg) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open scene");
    Hdr h;
    in.read(reinterpret_cast<char*>(&h), sizeof(h));
    sdfgi_cfg c;
    in.read(reinterpret_cast<char*>(&c), sizeof(c));
    cfg.surfaceEpsilon = c.surface_epsilon;
    cfg.maxTraceSteps = static_cast<int>(c.max_trace_steps);
    cfg.shadowSteps = static_cast<int>(c.shadow_steps);
    cfg.rayTMax = c.ray_tmax;
    cfg.bounceCoeff = c.bounce_coeff;
    cfg.nRaysFull = static_cast<int>(c.n_rays_full);
    cam = {h.camPos[0], h.camPos[1], h.camPos[2]};
    ActiveScene s;
    s.sky = {h.sky[0], h.sky[1], h.sky[2]};
    for (uint32_t i = 0; i < h.nPrims; ++i) {
        sdfgi_prim q;
        in.read(reinterpret_cast<char*>(&q), sizeof(q));
        SdfPrimitive p;
        p.id = q.id;
        p.kind = static_cast<PrimitiveKind>(q.kind);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) p.transform.rotation.m[a][b] = q.rot[3 * a + b];
        p.transform.translation = {q.trans[0], q.trans[1], q.trans[2]};
        p.size = {q.size[0], q.size[1], q.size[2]};
        p.material.albedo = {q.albedo[0], q.albedo[1], q.albedo[2]};
        p.material.emission = {q.emission[0], q.emission[1], q.emission[2]};
        s.primitives.push_back(p);
    }
    for (uint32_t i = 0; i < h.nLights; ++i) {
        sdfgi_light q;
        in.read(reinterpret_cast<char*>(&q), sizeof(q));
        Light l;
        l.kind = static_cast<LightKind>(q.kind);
        l.position = {q.position[0], q.position[1], q.position[2]};
        l.direction = {q.direction[0], q.direction[1], q.direction[2]};
        l.intensity = {q.intensity[0], q.intensity[1], q.intensity[2]};
        s.lights.push_back(l);
    }
    std::vector<sdfgi_cluster> cl(h.nClusters);
    in.read(reinterpret_cast<char*>(cl.data()), cl.size() * sizeof(sdfgi_cluster));
    std::vector<int32_t> st(h.nClusters + 1), idx(h.nMembers);
    in.read(reinterpret_cast<char*>(st.data()), st.size() * 4);
    in.read(reinterpret_cast<char*>(idx.data()), idx.size() * 4);
    for (uint32_t k = 0; k < h.nClusters; ++k) {
        Cluster c;
        c.cullAabb.lo = {cl[k].lo[0], cl[k].lo[1], cl[k].lo[2]};
        c.cullAabb.hi = {cl[k].hi[0], cl[k].hi[1], cl[k].hi[2]};
        c.aabb = c.cullAabb;
        c.unbounded = cl[k].unbounded != 0;
        for (int m = st[k]; m < st[k + 1]; ++m) c.members.push_back(idx[m]);
        s.clusters.push_back(c);
    }
    s.finalize();
    return s;
}

}  // namespace

double relErr(double got, double want, double floor) { return std::fabs(got - want) / std::max(std::fabs(want), floor); }

// Renderer::renderFrame (pipeline.hpp:84-230), reference vs device, frame by frame.
int runRender(int argc, char** argv) {
    if (argc < 6) throw std::runtime_error("usage: render file.scene frames w h [nrays]");
    SceneFile file = loadSceneFile(argv[2]);
    if (argc > 6) file.config.nRaysFull = std::atoi(argv[6]);
    const int frames = std::atoi(argv[3]), w = std::atoi(argv[4]), h = std::atoi(argv[5]);
    Renderer ref(file, w, h, hardwareThreads());
    sdfgi::b200::Renderer gpu(file, w, h, true);
    long long metricMismatch = 0, px = 0, exact = 0;
    double maxRel = 0;
    for (int f = 0; f < frames; ++f) {
        FrameMetrics a = ref.renderFrame();
        FrameMetrics b = gpu.renderFrame();
        if (a.activePrimitives != b.activePrimitives || a.clusters != b.clusters || a.probesTotal != b.probesTotal ||
            a.probesUpdated != b.probesUpdated || a.relocated != b.relocated || a.rejected != b.rejected ||
            a.dead != b.dead)
            ++metricMismatch;
        const ImageRgb& ia = ref.image();
        const ImageRgb& ib = gpu.image();
        double mean = 0;
        for (const Vec3& v : ia.pixels) mean += (std::fabs(v.x) + std::fabs(v.y) + std::fabs(v.z)) / 3;
        mean /= std::max<size_t>(ia.pixels.size(), 1);
        for (size_t i = 0; i < ia.pixels.size(); ++i)
            for (int k = 0; k < 3; ++k) {
                ++px;
                if (ia.pixels[i][k] == ib.pixels[i][k]) ++exact;
                maxRel = std::max(maxRel, relErr(ib.pixels[i][k], ia.pixels[i][k], 0.05 * mean));
            }
    }
    std::printf("{\"frames\": %d, \"metric_mismatches\": %lld, \"channels\": %lld, \"exact_channels\": %lld, "
                "\"max_rel_err\": %.6g}\n",
                frames, metricMismatch, px, exact, maxRel);
    return 0;
}

// The free functions against the reference's, on the state after one reference pass.
int runFuncs(int argc, char** argv) {
    if (argc < 8) throw std::runtime_error("usage: funcs scene.sdfs rx ry rz spacing nrays");
    Vec3 cam;
    RenderConfig cfg;
    ActiveScene scene = readScene(argv[2], cam, cfg);
    const int rx = std::atoi(argv[3]), ry = std::atoi(argv[4]), rz = std::atoi(argv[5]);
    const double spacing = std::atof(argv[6]);
    cfg.nRaysFull = std::atoi(argv[7]);
    std::vector<CascadeVolume> cas{makeCascade(rx, ry, rz, spacing, 0, cam)};
    std::vector<ProbeAtlas> atl[2];
    for (auto& a : atl) a.emplace_back(cas[0].probeCount(), cfg.octRes);
    // one reference pass so the field has texels and relocated probes
    updateProbePositions(cas[0], scene, cfg.threshold1(spacing), cfg.threshold2(spacing), cfg.maxDescentSteps);
    IrradianceField f0{&cas, &atl[0]};
    for (int i = 0; i < cas[0].probeCount(); ++i)
        if (cas[0].probes[i].alive) updateProbe(scene, cas[0], i, f0, atl[1][0], cfg.nRaysFull, cfg, 0);
    IrradianceField prev{&cas, &atl[1]};

    sdfgi::b200::Device gpu(0, true);
    gpu.uploadScene(scene);
    gpu.syncCascades(cas, cfg.octRes, &atl[1]);
    Rng rng(7);
    const Vec3 lo = cas[0].origin, hi = cas[0].origin + Vec3(rx - 1, ry - 1, rz - 1) * spacing;
    auto randIn = [&] { return Vec3(rng.uniform(lo.x, hi.x), rng.uniform(lo.y, hi.y), rng.uniform(lo.z, hi.z)); };
    const int n = 4096;
    std::vector<Vec3> o(n), d(n);
    for (int i = 0; i < n; ++i) {
        o[i] = randIn();
        d[i] = uniformSphereDir(rng);
    }
    long long bad = 0;
    // querySceneSdf
    std::vector<int> own;
    std::vector<double> q = gpu.querySceneSdf(o, kInf, &own);
    for (int i = 0; i < n; ++i) {
        int ow = -1;
        double r = querySceneSdf(scene, o[i], kInf, nullptr, &ow);
        if (r != q[i] || ow != own[i]) ++bad;
    }
    const long long badQuery = bad;
    // sphereTrace (bit-exact in FP64)
    std::vector<Hit> hg = gpu.sphereTrace(scene, o, d, cfg.rayTMax, cfg.surfaceEpsilon, cfg.maxTraceSteps);
    std::vector<Hit> hr(n);
    long long badTrace = 0;
    for (int i = 0; i < n; ++i) {
        hr[i] = sphereTrace(scene, o[i], d[i], cfg.rayTMax, cfg.surfaceEpsilon, cfg.maxTraceSteps);
        const Hit& a = hr[i];
        const Hit& b = hg[i];
        if (a.converged != b.converged || a.miss != b.miss || a.primitiveIndex != b.primitiveIndex ||
            a.primitiveId != b.primitiveId || a.t != b.t || !(a.position == b.position) || !(a.normal == b.normal))
            ++badTrace;
    }
    // softShadowTrace
    std::vector<double> t0(n, 0.01), t1(n, 3.0);
    std::vector<double> vg = gpu.softShadowTrace(o, d, t0, t1, cfg.shadowK, nullptr, cfg.shadowSteps);
    long long badShadow = 0;
    for (int i = 0; i < n; ++i)
        if (softShadowTrace(scene, o[i], d[i], 0.01, 3.0, cfg.shadowK, nullptr, cfg.shadowSteps) != vg[i]) ++badShadow;
    // interpolationStencil (the MVC's sines are algebraic on the device: weights to ~1e-12)
    std::vector<InterpolationStencil> sg = gpu.interpolationStencil(cas, o, cfg.mvcRelocationFrac);
    long long badStencil = 0;
    double stencilErr = 0;
    for (int i = 0; i < n; ++i) {
        InterpolationStencil a = interpolationStencil(cas, o[i], cfg.mvcRelocationFrac);
        const InterpolationStencil& b = sg[i];
        if (a.count != b.count || a.skyFallback != b.skyFallback || a.usedMvc != b.usedMvc ||
            a.crossCascade != b.crossCascade)
            ++badStencil;
        for (int k = 0; k < a.count && k < b.count; ++k) {
            if (a.entries[k].ref.index != b.entries[k].ref.index || a.entries[k].ref.cascade != b.entries[k].ref.cascade)
                ++badStencil;
            stencilErr = std::max(stencilErr, std::fabs(a.entries[k].weight - b.entries[k].weight));
        }
    }
    // convolveIrradiance
    std::vector<RadianceSample> samples(300);
    for (auto& sm : samples) {
        sm.dir = uniformSphereDir(rng);
        sm.radiance = {rng.uniform(), rng.uniform(), rng.uniform()};
    }
    std::vector<ConvolveResult> cg = gpu.convolveIrradiance(samples, std::vector<Vec3>(d.begin(), d.begin() + 64));
    long long badConv = 0;
    for (int i = 0; i < 64; ++i) {
        ConvolveResult a = convolveIrradiance(samples, d[i]);
        if (!(a.irradiance == cg[i].irradiance) || a.empty != cg[i].empty) ++badConv;
    }
    // shadeHit on the converged hits, against the field (bounce through the MVC: 1e-9)
    std::vector<Hit> conv;
    for (const Hit& hh : hr)
        if (hh.converged) conv.push_back(hh);
    std::vector<Vec3> lg = gpu.shadeHit(conv, prev, cfg.bounceCoeff, cfg);
    double shadeErr = 0;
    for (size_t i = 0; i < conv.size(); ++i) {
        Vec3 a = shadeHit(scene, conv[i], prev, cfg.bounceCoeff, cfg);
        for (int k = 0; k < 3; ++k) shadeErr = std::max(shadeErr, relErr(lg[i][k], a[k], 1e-6));
    }
    // per-probe updateProbe of every 7th alive probe, frame 1, reading `prev`
    std::vector<CascadeVolume> casG = cas;
    ProbeAtlas currR = atl[1][0], currG = atl[1][0];
    long long badProbe = 0, texels = 0, exactTexels = 0;
    double probeErr = 0;
    double mean = 0;
    for (float v : atl[1][0].raw()) mean += std::fabs(v);
    mean /= atl[1][0].raw().size();
    for (int i = 0; i < cas[0].probeCount(); i += 7) {
        if (!cas[0].probes[i].alive) continue;
        auto ra = updateProbe(scene, cas[0], i, prev, currR, cfg.nRaysFull, cfg, 1);
        IrradianceField prevG{&casG, &atl[1]};
        auto rb = gpu.updateProbe(scene, casG[0], i, prevG, currG, cfg.nRaysFull, cfg, 1);
        if (ra.raysTraced != rb.raysTraced || casG[0].probes[i].rejectHistory != cas[0].probes[i].rejectHistory ||
            casG[0].probes[i].lastUpdateFrame != cas[0].probes[i].lastUpdateFrame)
            ++badProbe;
    }
    for (size_t k = 0; k < currR.raw().size(); ++k) {
        ++texels;
        if (currR.raw()[k] == currG.raw()[k]) ++exactTexels;
        probeErr = std::max(probeErr, relErr(currG.raw()[k], currR.raw()[k], 0.05 * mean));
    }
    std::printf("{\"query_mismatches\": %lld, \"trace_mismatches\": %lld, \"shadow_mismatches\": %lld, "
                "\"stencil_mismatches\": %lld, \"stencil_max_abs_err\": %.3g, \"convolve_mismatches\": %lld, "
                "\"shade_hits\": %zu, \"shade_max_rel_err\": %.3g, \"probe_mismatches\": %lld, "
                "\"texels\": %lld, \"exact_texels\": %lld, \"probe_max_rel_err\": %.3g}\n",
                badQuery, badTrace, badShadow, badStencil, stencilErr, badConv, conv.size(), shadeErr, badProbe, texels,
                exactTexels, probeErr);
    return 0;
}

int main(int argc, char** argv) {
    try {
        if (argc > 1 && std::string(argv[1]) == "render") return runRender(argc, argv);
        if (argc > 1 && std::string(argv[1]) == "funcs") return runFuncs(argc, argv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    if (argc < 8) {
        std::fprintf(stderr, "usage: %s scene.sdfs passes rx ry rz spacing nrays\n", argv[0]);
        return 2;
    }
    try {
        Vec3 cam;
        RenderConfig cfg;
        ActiveScene scene = readScene(argv[1], cam, cfg);
        int passes = std::atoi(argv[2]);
        int rx = std::atoi(argv[3]), ry = std::atoi(argv[4]), rz = std::atoi(argv[5]);
        double spacing = std::atof(argv[6]);
        cfg.nRaysFull = std::atoi(argv[7]);

        // reference side (pipeline.hpp:108-151)
        std::vector<CascadeVolume> refCas{makeCascade(rx, ry, rz, spacing, 0, cam)};
        std::vector<ProbeAtlas> ref[2];
        for (auto& a : ref) a.emplace_back(refCas[0].probeCount(), cfg.octRes);
        // drop-in side: identical host objects, GPU does the work
        std::vector<CascadeVolume> gpuCas = refCas;
        std::vector<ProbeAtlas> gpuAtlas{ProbeAtlas(refCas[0].probeCount(), cfg.octRes)};
        sdfgi::b200::Device gpu(0, true);
        gpu.uploadScene(scene);
        gpu.syncCascades(gpuCas, cfg.octRes);

        int readIdx = 0;
        long long mismatchProbe = 0, texels = 0, exact = 0;
        double maxRel = 0;
        for (int frame = 0; frame < passes; ++frame) {
            double th1 = cfg.threshold1(spacing), th2 = cfg.threshold2(spacing);
            RelocationReport a = updateProbePositions(refCas[0], scene, th1, th2, cfg.maxDescentSteps);
            RelocationReport b = gpu.updateProbePositions(gpuCas[0], th1, th2, cfg.maxDescentSteps);
            if (a.relocated != b.relocated || a.dead != b.dead || a.rejected != b.rejected) mismatchProbe += 1000000;
            int writeIdx = 1 - readIdx;
            ref[writeIdx] = ref[readIdx];
            IrradianceField prev{&refCas, &ref[readIdx]};
            std::vector<ProbeRef> refs;
            for (int i = 0; i < refCas[0].probeCount(); ++i) refs.push_back({0, i});
            parallelFor(0, static_cast<int64_t>(refs.size()), hardwareThreads(), [&](int64_t i, int) {
                if (!refCas[0].probes[refs[i].index].alive) return;
                updateProbe(scene, refCas[0], refs[i].index, prev, ref[writeIdx][0], cfg.nRaysFull, cfg, frame);
            });
            readIdx = writeIdx;
            gpu.updateProbes(gpuCas, refs, cfg, frame, gpuAtlas);
            for (int i = 0; i < refCas[0].probeCount(); ++i) {
                const Probe& p = refCas[0].probes[i];
                const Probe& q = gpuCas[0].probes[i];
                if (!(p.pos == q.pos) || p.alive != q.alive || p.rejectHistory != q.rejectHistory ||
                    p.lastUpdateFrame != q.lastUpdateFrame)
                    ++mismatchProbe;
            }
            const auto& ra = ref[readIdx][0].raw();
            const auto& ga = gpuAtlas[0].raw();
            double mean = 0;
            for (float v : ra) mean += std::fabs(v);
            mean /= ra.size();
            for (size_t k = 0; k < ra.size(); ++k) {
                ++texels;
                if (ra[k] == ga[k]) ++exact;
                double rel = std::fabs(double(ga[k]) - ra[k]) / std::max(std::fabs(double(ra[k])), 0.05 * mean);
                maxRel = std::max(maxRel, rel);
            }
        }
        std::printf("{\"probe_mismatches\": %lld, \"texels\": %lld, \"exact_texels\": %lld, \"max_rel_err\": %.6g}\n",
                    mismatchProbe, texels, exact, maxRel);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
