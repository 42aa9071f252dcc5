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
#include <sdfgi/pipeline.hpp>

#include <cmath>
#include <cstdio>
#include <fstream>

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

int main(int argc, char** argv) {
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
