// sdfgi_abi.cu — the C-ABI (include/sdfgi_b200.h): context, device-resident scene,
// probe state and double-buffered atlases, and the launch sequence of the probe
// stage. Host code only; kernels live in kernels_f64.cu / kernels_f32.cu.
//
// HBM layout (per context):
//   scene   prims in cluster (CSR) order, FP64 (128 B) and FP32 (64 B) copies;
//           cluster cull boxes (FP64 56 B / FP32 32 B); CSR starts; CSR->original
//           index; albedo/emission (FP64).
//   probes  all cascades concatenated (cascade c starts at base[c]); pos/rest/last
//           as xyz triples of double, alive/reject/lastFrame as int32.
//   atlas   two buffers (front = read, back = write), all cascades concatenated,
//           tile-major exactly as ProbeAtlas::raw() (atlas.hpp:119-124), so an
//           atlas download is one contiguous copy and a z-slab is one byte range.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sdfgi_b200.h"
#include "host_trig.h"
#include "kernels.cuh"

using namespace sdfgi_dev;

namespace sdfgi_dev {
double measure_fma_rate(bool f64, cudaStream_t st);
}

static_assert(sizeof(sdfgi_prim) == 184, "prim ABI");
static_assert(sizeof(sdfgi_light) == 80, "light ABI");
static_assert(sizeof(DPrim<double>) == 128 && offsetof(DPrim<double>, rot) == 56, "FP64 primitive record layout (evalPrim<double> loads)");
static_assert(sizeof(sdfgi_light) == sizeof(DLight), "light mirror");
static_assert(sizeof(sdfgi_cluster) == 56, "cluster ABI");
static_assert(sizeof(sdfgi_cfg) == 224, "cfg ABI");
static_assert(sizeof(sdfgi_probe) == 88, "probe ABI");
static_assert(sizeof(sdfgi_ray_record) == sizeof(RayRecord), "ray record mirror");
static_assert(sizeof(sdfgi_hit) == 72 && sizeof(sdfgi_stencil) == 120, "hit / stencil ABI");

namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw Error(e_ == cudaErrorMemoryAllocation ? SDFGI_ERR_OOM : SDFGI_ERR_CUDA,       \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                        \
    } while (0)
#define NK(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) throw Error(SDFGI_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)
#define REQ(cond, code, msg)                        \
    do {                                            \
        if (!(cond)) throw Error((code), (msg));    \
    } while (0)

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SDFGI_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SDFGI_ERR_INVALID;
    }
}

// Device buffer: n = the size asked for, cap = what is allocated (grow-only: a grid
// rebuild or a batch of another size reuses the memory instead of a cudaFree +
// cudaMalloc pair, each of which synchronises the device).
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    void alloc(size_t count) {
        if (count <= cap && p) {
            n = count;
            return;
        }
        free();
        if (count) CK(cudaMalloc(&p, count * sizeof(T)));
        n = cap = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = cap = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t s) {
        alloc(count);
        if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
};

struct CascadeHost {
    int res[3] = {0, 0, 0};
    int level = 0;
    double spacing = 1.0;
    double origin[3] = {0, 0, 0};
    int base = 0;
    int count() const { return res[0] * res[1] * res[2]; }
};

struct Ctx {
    int device = 0, rank = 0, world = 1, precision = SDFGI_F64;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // update start/end, relocate start/end
    cudaEvent_t kev[kWaveEvents] = {};  // the last update's stage boundaries (launch_wavefront)
    bool evUpdate = false, evReloc = false;
    double stageSum[kWaveEvents] = {};  // sdfgi_stage_ms_sum: stages + update total since the last reset
    // The probe stage's counters and stage events: the context's own (synchronous
    // calls) or, for sdfgi_probe_stage_async, pass slot k's until it is collected.
    unsigned long long* scr = nullptr;
    cudaEvent_t* kevCur = nullptr;
    static constexpr int kMaxPending = 8;
    static constexpr int kSlotWords = kShadowStats + 32;
    DBuf<unsigned long long> scratchAsync;           // kMaxPending x kSlotWords
    cudaEvent_t kevAsync[kMaxPending][kWaveEvents] = {};
    unsigned long long* hAsync = nullptr;            // pinned, per slot: 3 tail words + 2 * kMaxCascades report words
    int nPending = 0;
    bool pendingTimed[kMaxPending] = {};
    int pendingCascades[kMaxPending] = {};
    ncclComm_t comm = nullptr;
    long long launches = 0;
    // scene
    bool haveScene = false;
    int nPrims = 0, nClusters = 0, nLights = 0;
    double sky[3] = {0, 0, 0};
    DBuf<DPrim<double>> prim64;
    DBuf<DPrim<float>> prim32;
    // the records K1/K2 stage in shared memory (evalPrimStaged); 0 bytes: the scene
    // does not fit (or SDFGI_STAGE=0) and they read prim64 / prim32
    DBuf<unsigned char> stage64;
    int stage64Bytes = 0, stage64RotOff = 0, stage32Bytes = 0;
    DBuf<DCluster<double>> cl64;
    DBuf<DCluster<float>> cl32;
    DBuf<int> cstart, orig;
    DBuf<double> albedo, emission;
    DBuf<int> kindId;
    DBuf<DLight> lights;
    // candidate-cluster grid (GridDev, sdf_device.cuh)
    // 0 the reference's flat cluster walk (exact TraceStats), 1 the candidate grid
    // (exact march sequence), 2 (default) grid + escaped marches ended early
    int accel = 2;
    bool haveGrid = false;
    GridDev grid{};
    long long gridEntries = 0;
    DBuf<int> gridStart, gridList, gridCounts;
    DBuf<int2> gridEntry;
    DBuf<int4> gridCell;
    DBuf<int> brickCounts, brickStart, brickList, brickSeed;
    DBuf<unsigned char> scanTemp;
    DBuf<double> gridU, primBox;
    DBuf<BNode> bvh;
    DBuf<int> unbList;
    double gridBox[6] = {0, 0, 0, 0, 0, 0};  // region the cells cover
    int gridAccel = -1;
    uint64_t gridParams = 0;  // hash of the grid's build parameters (environment knobs)
    // dynamic primitives (original indices, sorted): left out of the grid lists (they
    // moved since it was built) and evaluated by every on-grid query (dynCsr: their
    // current CSR positions); gridCsrOrig: the CSR -> original map of the lists
    std::vector<int> gridDyn, gridCsrOrig;
    DBuf<int> dynCsr;
    int nDyn = 0;
    long long gridRefits = 0;
    bool escapeValid = false;  // every bounded primitive inside the grid box (escape tests)
    bool hintValid = false;
    double hint[6] = {0, 0, 0, 0, 0, 0};     // probe volumes the grid must cover
    // host copy of the uploaded scene (the grid is rebuilt when the hint grows)
    std::vector<sdfgi_prim> hPrims;
    // sdfgi_scene_upload's conversion buffers (reused across uploads)
    std::vector<DPrim<double>> up64;
    std::vector<DPrim<float>> up32;
    std::vector<int> upOrig, upKid;
    std::vector<double> upAlb, upEm;
    std::vector<unsigned char> upStage, upRows;
    // the cluster boxes and coordinate scale the BVH was built from (a re-sent scene
    // with the same boxes keeps it)
    std::vector<sdfgi_cluster> bvhClusters;
    double bvhScale = -1;
    double gridMargin = -1;  // the margin multiple the grid was built with
    std::vector<int32_t> hMember, hStart;
    std::vector<sdfgi_cluster> hClusters;
    std::vector<sdfgi_light> hLights;
    // probes
    std::vector<CascadeHost> cascades;
    int octRes = 8;
    int totalProbes = 0;
    DBuf<double> pos, rest, last, clear;
    // clearValid[slot]: clear holds the SDF at every probe's position of that cascade
    // (its relocation ran after the last scene, probe or cascade change)
    std::vector<char> clearValid;
    DBuf<int> alive, reject, lastFrame;
    DBuf<float> atlas[2];
    int front = 0;
    // atlasZero[b][slot]: cascade `slot` of atlas buffer b is known to be all zeros
    // (makeCascade / recenter state). While the whole front atlas is zero, every
    // bounce lookup returns exactly 0 and adds nothing (probe_update.hpp:143-147),
    // so the probe update skips it (SURVEY §7.7's exact saving: pass 0 of a fresh
    // volume).
    std::vector<char> atlasZero[2];
    bool frontZero() const {
        for (char z : atlasZero[front])
            if (!z) return false;
        return !atlasZero[front].empty();
    }
    // scratch
    // [0..7] TraceStats, [8..13] evaluations by kind + rotated, [16] maxDelta bits,
    // [17] rays, [18] probes updated
    DBuf<unsigned long long> scratch;
    unsigned long long lastWork[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long lastTrace[2][14] = {};  // the last stats update's K1 / K2 counters
    unsigned long long shadeWork[2] = {0, 0};
    DBuf<int> report;
    DBuf<int> refs, allRefs;
    DBuf<RayRecord> records;
    // wavefront scratch (kernels.cuh)
    DBuf<int> wRayCount, wHitList, wHitAt, wMvcList, wTriList;
    DBuf<long long> wRayStart;
    DBuf<double> wRot, fib;
    DBuf<int> perm;
    int fibN = -1;
    int* hReport = nullptr;  // pinned: relocation reports of sdfgi_probe_stage (read after its one sync)
    // pinned ring the host arrays of an upload are staged in, so their copies are
    // asynchronous DMA (a pageable cudaMemcpyAsync costs ~50 us of staging each);
    // arenaEv: the latest copy out of it
    char* arena = nullptr;
    size_t arenaCap = 0, arenaOff = 0;
    cudaEvent_t arenaEv = nullptr;
    DBuf<double> probeAos;  // sdfgi_probe records in transit (probes upload / download)
    // The per-pass quaternions (host_trig.h) in two slots: pinned host staging + a
    // device copy made on copyStream. A pass reads one slot; the other takes the
    // next frame's quaternions, computed on the host and copied while the current
    // pass runs on the device (a frame loop's next update finds them on the device).
    struct QuatSlot {
        double* h = nullptr;
        size_t hn = 0;
        DBuf<double> d;
        cudaEvent_t copied = nullptr;  // on copyStream: d holds h
        cudaEvent_t used = nullptr;    // on stream: the last pass reading d is done
        uint64_t key = 0;
    };
    QuatSlot qs[2];
    int qLast = 0;    // slot of the latest pass
    int qSpec = -1;   // slot holding the speculated next frame
    int qReady = -1;  // slot prepared for the coming pass (sdfgi_probe_stage: before relocation)
    const double* quatDev = nullptr;
    cudaStream_t copyStream = nullptr;
    // Contact GI's cosineHemisphereDir (lx, ly) per (pixel, sample), host libm; keyed
    // (seed, w, h, samples): the reference's stream has no frame index (shading.hpp:451)
    DBuf<double> cLocal;
    uint64_t cLocalSeed = 0;
    int cLocalW = 0, cLocalH = 0, cLocalS = -1;
    DBuf<unsigned char> wHits, wVis, wRad, wPark, wCRay, wPRay, wSRay, wSelTemp, wConv;
    DBuf<unsigned long long> wCtr;
    int persistCap = 0;  // 0 = occupancy-sized persistent grids
    // gather (e): G-buffer, stage buffers, history (pipeline.hpp:213-218)
    int gw = 0, gh = 0;
    DBuf<GPix> gbuf;
    DBuf<double> halfDepth, sparseIrr, resolved, indirect, histIrr, histDepth, composed;
    DBuf<int> halfSrc, sel, sparseValid, sparseAnchor;
    int histValid = 0;
    cudaEvent_t gev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t cev[2] = {nullptr, nullptr};  // compose
    bool gevValid = false;
    DBuf<unsigned char> selScratch;  // sdfgi_select_probes
    DBuf<double> qpts, qinit, qd;
    DBuf<int> qowner;

    ~Ctx() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        prim64.free(); prim32.free(); stage64.free(); cl64.free(); cl32.free(); cstart.free(); orig.free();
        albedo.free(); emission.free(); lights.free(); kindId.free();
        gridStart.free(); gridList.free(); gridCounts.free(); gridU.free(); gridEntry.free(); gridCell.free(); brickCounts.free(); brickStart.free(); brickList.free(); brickSeed.free(); scanTemp.free();
        bvh.free(); unbList.free(); primBox.free(); dynCsr.free();
        pos.free(); rest.free(); last.free(); clear.free(); alive.free(); reject.free(); lastFrame.free();
        atlas[0].free(); atlas[1].free(); scratch.free(); report.free(); refs.free(); allRefs.free();
        records.free(); selScratch.free(); qpts.free(); qinit.free(); qd.free(); qowner.free();
        wRayCount.free(); wHitList.free(); wMvcList.free(); wTriList.free(); wHitAt.free(); wSelTemp.free(); wRayStart.free(); wRot.free(); fib.free(); cLocal.free(); wHits.free();
        if (hReport) cudaFreeHost(hReport);
        if (hAsync) cudaFreeHost(hAsync);
        scratchAsync.free();
        for (auto& row : kevAsync)
            for (auto& e : row)
                if (e) cudaEventDestroy(e);
        if (arena) cudaFreeHost(arena);
        if (arenaEv) cudaEventDestroy(arenaEv);
        probeAos.free();
        for (auto& q : qs) {
            if (q.h) cudaFreeHost(q.h);
            q.d.free();
            if (q.copied) cudaEventDestroy(q.copied);
            if (q.used) cudaEventDestroy(q.used);
        }
        if (copyStream) cudaStreamDestroy(copyStream);
        wVis.free(); wPark.free(); wCRay.free(); wPRay.free(); wConv.free(); wSRay.free(); wCtr.free(); perm.free(); wRad.free();
        gbuf.free(); halfDepth.free(); sparseIrr.free(); resolved.free(); indirect.free(); histIrr.free(); composed.free();
        histDepth.free(); halfSrc.free(); sel.free(); sparseValid.free(); sparseAnchor.free();
        for (auto& e : gev)
            if (e) cudaEventDestroy(e);
        for (auto& e : cev)
            if (e) cudaEventDestroy(e);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : kev)
            if (e) cudaEventDestroy(e);
        if (comm) ncclCommDestroy(comm);
        if (stream) cudaStreamDestroy(stream);
    }

    size_t tileFloats() const { return static_cast<size_t>(octRes + 2) * (octRes + 2) * 3; }
    size_t atlasFloats() const { return tileFloats() * totalProbes; }

    ProbeCommon probeCommon() const {
        ProbeCommon pc;
        std::memset(&pc, 0, sizeof(pc));
        pc.nCas = static_cast<int>(cascades.size());
        for (int i = 0; i < pc.nCas; ++i) {
            const CascadeHost& c = cascades[i];
            for (int k = 0; k < 3; ++k) {
                pc.cas[i].res[k] = c.res[k];
                pc.cas[i].origin[k] = c.origin[k];
            }
            pc.cas[i].base = c.base;
            pc.cas[i].spacing = c.spacing;
            pc.cas[i].level = c.level;
        }
        pc.probes.pos = pos.p;
        pc.probes.rest = rest.p;
        pc.probes.last = last.p;
        pc.probes.alive = alive.p;
        pc.probes.reject = reject.p;
        pc.probes.lastFrame = lastFrame.p;
        pc.probes.clear = clear.p;
        return pc;
    }

    template <typename R>
    SceneView<R> sceneView() const;

    int slot(int level) const {
        for (size_t i = 0; i < cascades.size(); ++i)
            if (cascades[i].level == level) return static_cast<int>(i);
        throw Error(SDFGI_ERR_INVALID, "no cascade with level " + std::to_string(level));
    }
};

// Host array -> device through the pinned ring (stream-ordered; the ring wraps
// once every copy out of it has finished).
void stageCopy(Ctx* c, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    size_t off = (c->arenaOff + 255) & ~static_cast<size_t>(255);
    if (off + bytes > c->arenaCap) {
        CK(cudaEventSynchronize(c->arenaEv));
        off = 0;
        if (bytes > c->arenaCap) {
            if (c->arena) CK(cudaFreeHost(c->arena));
            c->arena = nullptr;
            c->arenaCap = 0;
            const size_t cap = std::max<size_t>(bytes, 8u << 20);
            CK(cudaMallocHost(&c->arena, cap));
            c->arenaCap = cap;
        }
    }
    std::memcpy(c->arena + off, src, bytes);
    CK(cudaMemcpyAsync(dst, c->arena + off, bytes, cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->arenaEv, c->stream));
    c->arenaOff = off + bytes;
}
template <class T>
void upload(Ctx* c, DBuf<T>& b, const T* h, size_t n) {
    b.alloc(n);
    stageCopy(c, b.p, h, n * sizeof(T));
}

template <>
SceneView<double> Ctx::sceneView<double>() const {
    SceneView<double> v;
    v.prims = prim64.p;
    v.clusters = cl64.p;
    v.cstart = cstart.p;
    v.orig = orig.p;
    v.albedo = albedo.p;
    v.emission = emission.p;
    v.kindId = kindId.p;
    v.lights = lights.p;
    v.n_prims = nPrims;
    v.n_clusters = nClusters;
    v.n_lights = nLights;
    for (int k = 0; k < 3; ++k) v.sky[k] = sky[k];
    v.grid = grid;
    v.useGrid = (accel && haveGrid) ? 1 : 0;
    v.stage = stage64.p;
    v.stageBytes = stage64Bytes;
    v.stageRotOff = stage64RotOff;
    v.dyn = dynCsr.p;
    v.nDyn = haveGrid ? nDyn : 0;
    return v;
}
template <>
SceneView<float> Ctx::sceneView<float>() const {
    SceneView<float> v;
    v.prims = prim32.p;
    v.clusters = cl32.p;
    v.cstart = cstart.p;
    v.orig = orig.p;
    v.albedo = albedo.p;
    v.emission = emission.p;
    v.kindId = kindId.p;
    v.lights = lights.p;
    v.n_prims = nPrims;
    v.n_clusters = nClusters;
    v.n_lights = nLights;
    for (int k = 0; k < 3; ++k) v.sky[k] = sky[k];
    v.grid = grid;
    v.useGrid = (accel && haveGrid) ? 1 : 0;
    v.stage = prim32.p;
    v.stageBytes = stage32Bytes;
    v.stageRotOff = 0;
    v.dyn = dynCsr.p;
    v.nDyn = haveGrid ? nDyn : 0;
    return v;
}

Ctx* C(void* p) {
    REQ(p != nullptr, SDFGI_ERR_INVALID, "null context");
    Ctx* c = static_cast<Ctx*>(p);
    CK(cudaSetDevice(c->device));
    return c;
}

void requireProbes(Ctx* c) {
    REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
    REQ(!c->cascades.empty(), SDFGI_ERR_STATE, "no cascade set");
}

void checkLaunch(Ctx* c) {
    ++c->launches;
    CK(cudaGetLastError());
}

// Probe range [lo, hi) of cascade slot `ci` owned by this rank: a z-slab of
// layers [resZ*r/W, resZ*(r+1)/W). Contiguous because
// index = ix + resX*(iy + resY*iz) (probe_volume.hpp:32).
void slabRange(const CascadeHost& c, int rank, int world, int* lo, int* hi) {
    int z0 = static_cast<int>((static_cast<long long>(c.res[2]) * rank) / world);
    int z1 = static_cast<int>((static_cast<long long>(c.res[2]) * (rank + 1)) / world);
    int layer = c.res[0] * c.res[1];
    *lo = c.base + z0 * layer;
    *hi = c.base + z1 * layer;
}

void resetProbes(Ctx* c, int slot) {
    c->clearValid.resize(c->cascades.size(), 0);
    c->clearValid[slot] = 0;
    const CascadeHost& cs = c->cascades[slot];
    const int n = cs.count();
    const size_t off = static_cast<size_t>(cs.base);
    // makeCascade's probes (restingAt, probe_volume.hpp:37-39) written on the device
    launch_probes_reset(c->probeCommon().probes, cs.base, cs.res, cs.origin, cs.spacing, c->stream);
    checkLaunch(c);
    for (int b = 0; b < 2; ++b) {
        CK(cudaMemsetAsync(c->atlas[b].p + off * c->tileFloats(), 0, n * c->tileFloats() * 4, c->stream));
        c->atlasZero[b].resize(c->cascades.size(), 0);
        c->atlasZero[b][slot] = 1;
    }
    CK(cudaStreamSynchronize(c->stream));
}

void reallocProbes(Ctx* c) {
    int total = 0;
    for (auto& cs : c->cascades) {
        cs.base = total;
        total += cs.count();
    }
    // preserve existing cascades' state is not needed: set() resets the touched one and
    // the concatenation may move, so reset all.
    c->totalProbes = total;
    c->pos.alloc(3 * static_cast<size_t>(total));
    c->clear.alloc(std::max(total, 1));
    c->clearValid.assign(c->cascades.size(), 0);
    c->rest.alloc(3 * static_cast<size_t>(total));
    c->last.alloc(3 * static_cast<size_t>(total));
    c->alive.alloc(total);
    c->reject.alloc(total);
    c->lastFrame.alloc(total);
    c->atlas[0].alloc(c->atlasFloats());
    c->atlas[1].alloc(c->atlasFloats());
    for (int b = 0; b < 2; ++b) c->atlasZero[b].assign(c->cascades.size(), 0);
    for (size_t i = 0; i < c->cascades.size(); ++i) resetProbes(c, static_cast<int>(i));
}

template <typename R>
void fillPrim(DPrim<R>& d, const sdfgi_prim& s) {
    for (int k = 0; k < 9; ++k) d.rot[k] = static_cast<R>(s.rot[k]);
    for (int k = 0; k < 3; ++k) {
        d.trans[k] = static_cast<R>(s.trans[k]);
        d.size[k] = static_cast<R>(s.size[k]);
    }
    d.kind = s.kind;
    // primitives.hpp:76: skip the rotation when the diagonal is exactly 1
    d.identity = (s.rot[0] == 1.0 && s.rot[4] == 1.0 && s.rot[8] == 1.0) ? 1 : 0;
}

// FP32 unified record (DPrim<float>, evalPrim<float>): the per-kind `size`
// meanings of primitives.hpp:25-30 mapped onto (e, rr); e1 < 0 marks radial
// shapes, rr < 0 a plane.
void fillPrim(DPrim<float>& d, const sdfgi_prim& s) {
    for (int k = 0; k < 9; ++k) d.rot[k] = static_cast<float>(s.rot[k]);
    for (int k = 0; k < 3; ++k) {
        d.trans[k] = static_cast<float>(s.trans[k]);
        d.e[k] = 0.f;
    }
    d.rr = 0.f;
    switch (s.kind) {
        case SDFGI_SPHERE: d.e[1] = -1.f; d.rr = static_cast<float>(s.size[0]); break;
        case SDFGI_BOX:
            for (int k = 0; k < 3; ++k) d.e[k] = static_cast<float>(s.size[k]);
            break;
        case SDFGI_PLANE: d.rr = -1.f; break;
        case SDFGI_CYLINDER:
            d.e[0] = static_cast<float>(s.size[0]);
            d.e[1] = -1.f;
            d.e[2] = static_cast<float>(s.size[1]);
            break;
        default:  // capsule
            d.e[1] = -1.f;
            d.e[2] = static_cast<float>(s.size[1]);
            d.rr = static_cast<float>(s.size[0]);
            break;
    }
}

// Build the candidate-cluster grid over the bounded clusters (exact; see GridDev).
// Conservative world AABB of a primitive's surface (primitiveAabb, primitives.hpp:112-151),
// widened by a small relative margin; planes are unbounded (+-inf).
void primAabb(const sdfgi_prim& s, double* out) {
    double lo[3], hi[3];
    auto fromHalf = [&](double hx, double hy, double hz) {
        for (int i = 0; i < 3; ++i) {
            double e = std::fabs(s.rot[3 * i]) * hx + std::fabs(s.rot[3 * i + 1]) * hy + std::fabs(s.rot[3 * i + 2]) * hz;
            lo[i] = s.trans[i] - e;
            hi[i] = s.trans[i] + e;
        }
    };
    switch (s.kind) {
        case SDFGI_SPHERE:
            for (int i = 0; i < 3; ++i) {
                lo[i] = s.trans[i] - s.size[0];
                hi[i] = s.trans[i] + s.size[0];
            }
            break;
        case SDFGI_BOX: fromHalf(s.size[0], s.size[1], s.size[2]); break;
        case SDFGI_CYLINDER: fromHalf(s.size[0], s.size[0], s.size[1]); break;
        case SDFGI_CAPSULE:
            for (int i = 0; i < 3; ++i) {
                double a = s.rot[3 * i + 2] * s.size[1];  // R * (0, 0, h)
                lo[i] = s.trans[i] - std::fabs(a) - s.size[0];
                hi[i] = s.trans[i] + std::fabs(a) + s.size[0];
            }
            break;
        default:
            for (int i = 0; i < 6; ++i) out[i] = i < 3 ? -INFINITY : INFINITY;
            return;
    }
    for (int i = 0; i < 3; ++i) {
        out[i] = lo[i] - (1e-7 * (std::fabs(lo[i]) + 1.0));
        out[3 + i] = hi[i] + (1e-7 * (std::fabs(hi[i]) + 1.0));
    }
}

// The cluster BVH for queries off the grid (and the grid build's exact queries),
// the unbounded-cluster list and the box of the bounded geometry (the escape
// tests of accel mode 2), for the context's current clusters. Median split of the
// box centres along the widest axis (depth <= ceil(log2 n) < kBvhStack), one
// cluster per leaf. Child boxes are padded like the FP32 cluster boxes and
// rounded outward to float, so the subtree tests are conservative in both
// precisions.
void buildBvh(Ctx* c, double scaleHint) {
    const sdfgi_cluster* clusters = c->hClusters.data();
    const int n = static_cast<int>(c->hClusters.size());
    if (c->bvhScale == scaleHint && c->bvhClusters.size() == c->hClusters.size() &&
        std::memcmp(c->bvhClusters.data(), clusters, n * sizeof(sdfgi_cluster)) == 0)
        return;  // same boxes: the same hierarchy (BNode refers to clusters by index)
    c->bvhClusters = c->hClusters;
    c->bvhScale = scaleHint;
    double glo[3] = {INFINITY, INFINITY, INFINITY}, ghi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double scale = 0;
    for (int k = 0; k < n; ++k) {
        if (clusters[k].unbounded) continue;
        for (int a = 0; a < 3; ++a) {
            glo[a] = std::min(glo[a], clusters[k].lo[a]);
            ghi[a] = std::max(ghi[a], clusters[k].hi[a]);
            scale = std::max(scale, std::max(std::fabs(clusters[k].lo[a]), std::fabs(clusters[k].hi[a])));
        }
    }
    scale = std::max(scale, scaleHint);  // the grid box's coordinate scale
    std::vector<int> unb, ids;
    for (int k = 0; k < n; ++k) (clusters[k].unbounded ? unb : ids).push_back(k);
    std::vector<BNode> nodes;
    nodes.reserve(ids.size());
    struct Box {
        double lo[3], hi[3];
    };
    auto boxOf = [&](int b, int e) {
        Box r;
        for (int a = 0; a < 3; ++a) {
            r.lo[a] = INFINITY;
            r.hi[a] = -INFINITY;
        }
        for (int i = b; i < e; ++i)
            for (int a = 0; a < 3; ++a) {
                r.lo[a] = std::min(r.lo[a], clusters[ids[i]].lo[a]);
                r.hi[a] = std::max(r.hi[a], clusters[ids[i]].hi[a]);
            }
        return r;
    };
    // returns the code of the subtree over ids[b, e)
    std::function<int(int, int, int)> build = [&](int b, int e, int depth) -> int {
        REQ(depth < kBvhStack, SDFGI_ERR_INVALID, "cluster BVH too deep");
        if (e - b == 1) return -ids[b] - 1;
        double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int i = b; i < e; ++i)
            for (int a = 0; a < 3; ++a) {
                const double m = 0.5 * (clusters[ids[i]].lo[a] + clusters[ids[i]].hi[a]);
                clo[a] = std::min(clo[a], m);
                chi[a] = std::max(chi[a], m);
            }
        int axis = 0;
        for (int a = 1; a < 3; ++a)
            if (chi[a] - clo[a] > chi[axis] - clo[axis]) axis = a;
        const int mid = (b + e) / 2;
        std::nth_element(ids.begin() + b, ids.begin() + mid, ids.begin() + e, [&](int x, int y) {
            const double mx = clusters[x].lo[axis] + clusters[x].hi[axis];
            const double my = clusters[y].lo[axis] + clusters[y].hi[axis];
            return mx < my || (mx == my && x < y);
        });
        const int self = static_cast<int>(nodes.size());
        nodes.emplace_back();
        const int range[2][2] = {{b, mid}, {mid, e}};
        for (int ch = 0; ch < 2; ++ch) {
            const Box bx = boxOf(range[ch][0], range[ch][1]);
            for (int a = 0; a < 3; ++a) {
                const double lo = bx.lo[a] - 2e-5 * (std::fabs(bx.lo[a]) + 1.0);
                const double hi = bx.hi[a] + 2e-5 * (std::fabs(bx.hi[a]) + 1.0);
                nodes[self].lo[ch][a] = std::nextafter(static_cast<float>(lo), -INFINITY);
                nodes[self].hi[ch][a] = std::nextafter(static_cast<float>(hi), INFINITY);
            }
            const int code = build(range[ch][0], range[ch][1], depth + 1);
            nodes[self].child[ch] = code;
        }
        return self;
    };
    int root = 0;
    if (!ids.empty()) root = build(0, static_cast<int>(ids.size()), 0);
    std::vector<int> unbPad(unb);
    if (nodes.empty()) nodes.emplace_back();  // never read (nBounded < 2 uses the root code only)
    if (unbPad.empty()) unbPad.push_back(0);
    upload(c, c->bvh, nodes.data(), nodes.size());
    upload(c, c->unbList, unbPad.data(), unbPad.size());
    CK(cudaStreamSynchronize(c->stream));
    c->grid.bvh = c->bvh.p;
    c->grid.bvhRoot = root;
    c->grid.nBounded = static_cast<int>(ids.size());
    // FP64 walks test node boxes in float; the slack bounds the float rounding of
    // a point-box distance at this coordinate scale (hierarchyWalk)
    c->grid.walkSlack = static_cast<float>(4e-5 * (scale + 1.0));
    c->grid.unbounded = c->unbList.p;
    c->grid.nUnbounded = static_cast<int>(unb.size());
    for (int a = 0; a < 3; ++a) {
        c->grid.geoLo[a] = glo[a];
        c->grid.geoHi[a] = ghi[a];
    }
}

double gridMargin(const Ctx* c, int precision) {
    const char* menv = std::getenv("SDFGI_GRID_MARGIN");
    if (menv) return std::atof(menv);
    bool unbounded = false;
    for (const auto& k : c->hClusters) unbounded = unbounded || k.unbounded;
    return !unbounded && precision == SDFGI_F64 ? 0.5 : 3.5;
}

// One build attempt at cellScale x the default cell count; false when the lists
// would overflow their 2^30-entry index (the caller retries coarser).
bool buildGridAt(Ctx* c, double cellScale) {
    const sdfgi_prim* prims = c->hPrims.data();
    const int32_t* member_idx = c->hMember.data();
    const sdfgi_cluster* clusters = c->hClusters.data();
    const int n = static_cast<int>(c->hClusters.size());
    c->haveGrid = false;
    c->gridEntries = 0;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int bounded = 0;
    for (int k = 0; k < n; ++k) {
        if (clusters[k].unbounded) continue;
        ++bounded;
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], clusters[k].lo[a]);
            hi[a] = std::max(hi[a], clusters[k].hi[a]);
        }
    }
    if (bounded == 0 || n < 2) return true;
    double ext[3], scale = 0;
    // the grid extends past the geometry so rays leaving the scene stay on the
    // (cheap) candidate lists for their first steps; SDFGI_GRID_MARGIN overrides.
    // It also covers the probe volumes (the hint box grown by sdfgi_cascade_set):
    // probes above an open scene would otherwise query off the grid every step.
    // The margin is a multiple of the geometry's SMALLEST extent on every axis: a
    // flat open scene (C4: 240 x 20 x 240) keeps the rays that leave it upwards on
    // the grid without spending cells on its far horizontal surroundings.
    // Sweep (profiles/README.md, 50M cells): C2 pass 0 FP64 margin 0.6 per-axis
    // 13.1 ms, 2.5 x min 12.0, 4 x min 12.3; C4 pass 1 0.235 -> 0.326 -> 0.374 Grays/s.
    // SDFGI_GRID_MARGIN sets the multiple, SDFGI_GRID_MARGIN_MIN=0 the per-axis extent.
    // With escape (accel mode 2, every cluster bounded) a march ends as soon as it
    // leaves the grid box, so cells beyond the geometry only delay that: FP64 takes
    // a 0.5x margin (C2 step 26.3 -> 25.1 ms at 240M cells; the same cells then sit
    // closer to the geometry). FP32 (per-lane cell cache) and scenes with unbounded
    // primitives (C4's ground plane: no escape, its marches stay on the grid) keep
    // 3.5x (FP32 C2 16.1 vs 16.8 ms; C4 pass 1 183 vs 217 ms at 2.5x).
    // profiles/r02_sweep_grid_cells.log
    const double marginFrac = gridMargin(c, c->precision);
    c->gridMargin = marginFrac;
    const char* mmode = std::getenv("SDFGI_GRID_MARGIN_MIN");
    const bool fromMin = !mmode || std::atoi(mmode) != 0;
    const double minExt = std::min(hi[0] - lo[0], std::min(hi[1] - lo[1], hi[2] - lo[2]));
    for (int a = 0; a < 3; ++a) {
        double e = fromMin ? minExt : hi[a] - lo[a];
        double m = marginFrac * e + 1e-3;
        lo[a] -= m;
        hi[a] += m;
        if (c->hintValid) {
            lo[a] = std::min(lo[a], c->hint[a]);
            hi[a] = std::max(hi[a], c->hint[3 + a]);
        }
        ext[a] = hi[a] - lo[a];
        scale = std::max(scale, std::max(std::fabs(lo[a]), std::fabs(hi[a])));
    }
    const char* env = std::getenv("SDFGI_GRID_CELLS");
    // finer cells -> smaller U -> shorter, more uniform candidate lists (and tighter
    // per-entry bounds); measured on C2 with the current kernels (pass 0, FP64, warm):
    // 2M cells 17.4 ms, 4M 16.6, 8M 15.9, 16M 15.5, 24M 15.3 (margin 0.6, round-1
    // kernels); with the SDF-bound lists and the min-extent margin 33M -> 50M -> 66M
    // cells: C2 13.9 / 12.3 / 12.9 ms, C4 0.28 / 0.37 / 0.34 Grays/s
    // Small scenes need far fewer cells: 120k cells per primitive, between 2M and
    // 240M (~12 GB of grid for C2, out of the 180 GB of HBM). With the round-1
    // final kernels 50M -> 66M: C2 pass 0 FP64 9.50 -> 9.36 ms; with the round-2
    // kernels (profiles/r02_sweep_grid_cells.log) C2 step 66M / 100M / 132M / 180M
    // / 240M = 27.58 / 27.11 / 26.73 / 26.49 / 26.34 ms FP64, C4 pass 1 199.9 /
    // 189.7 (132M) / 183.2 ms (240M). A grid build at 240M takes ~0.1 s (once per
    // static scene; an animated scene refits, see sdfgi_scene_upload).
    const double byPrims = std::min(240000000.0, std::max(2097152.0, 120000.0 * c->nPrims));
    double target = (env ? std::atof(env) : byPrims) * cellScale;
    if (target < 1) return true;
    double h = std::cbrt(ext[0] * ext[1] * ext[2] / target);
    int dim[3];
    for (int a = 0; a < 3; ++a) {
        h = std::max(h, ext[a] / 1024.0);
    }
    // rounding every axis up can overshoot the target: grow h until the cell count
    // is inside the 2^28 cells the grid allows (never fail for a size we chose)
    long long ncells = 1;
    for (int tries = 0;; ++tries) {
        ncells = 1;
        for (int a = 0; a < 3; ++a) {
            dim[a] = std::max(1, static_cast<int>(std::ceil(ext[a] / h)));
            ncells *= dim[a];
        }
        if (ncells < (1LL << 28)) break;
        REQ(tries < 64, SDFGI_ERR_INVALID, "candidate grid too large");
        h *= std::cbrt(static_cast<double>(ncells) / static_cast<double>(1LL << 28)) * 1.001;
    }
    buildBvh(c, scale);
    GridBuildParams p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<double>();
    // the bound kernel's exact queries walk the BVH: a grid of no cells puts every
    // point "off the grid"
    p.scene.useGrid = 1;
    p.scene.grid = c->grid;
    for (int a = 0; a < 3; ++a) p.scene.grid.dim[a] = 0;
    p.scene.grid.invH = 0.0;
    p.scene.grid.finvH = 0.f;
    for (int a = 0; a < 3; ++a) {
        p.lo[a] = lo[a];
        p.dim[a] = dim[a];
    }
    p.h = h;
    // pad the cells for FP32 point->cell rounding; slack covers every rounding on the way
    p.pad = 1e-4 * h + 4e-6 * scale;
    p.margin = 1e-5 * (scale + 1.0);
    // cells far from the geometry would list every primitive within their (large)
    // bound; lists keep the maxList nearest plus a sentinel carrying the omitted
    // candidates' lower bound (a query that cannot stop there walks the hierarchy)
    const char* lenv = std::getenv("SDFGI_GRID_MAXLIST");
    p.maxList = lenv ? std::max(8, std::atoi(lenv)) : 96;
    c->gridU.alloc(ncells);
    c->gridCounts.alloc(ncells + 1);  // [ncells] = 0: the exclusive scan's last entry is the total
    c->gridStart.alloc(ncells + 1);
    CK(cudaMemsetAsync(c->gridCounts.p + ncells, 0, 4, c->stream));
    {
        std::vector<double> boxes(6 * static_cast<size_t>(c->nPrims));
        for (int j = 0; j < c->nPrims; ++j) primAabb(prims[member_idx[j]], &boxes[6 * static_cast<size_t>(j)]);
        upload(c, c->primBox, boxes.data(), boxes.size());
    }
    p.primBox = c->primBox.p;
    p.U = c->gridU.p;
    p.counts = c->gridCounts.p;
    // bricks of kBrick^3 cells: the nearest primitive at each brick centre seeds the
    // exact queries of its cells' bounds (the BVH walk then prunes against a tight
    // minimum from its first node), and each brick lists its candidate clusters
    long long nbricks = 1;
    for (int a = 0; a < 3; ++a) {
        p.bdim[a] = (dim[a] + kBrick - 1) / kBrick;
        nbricks *= p.bdim[a];
    }
    c->brickSeed.alloc(nbricks);
    p.bSeed = c->brickSeed.p;
    launch_grid_seed(p, static_cast<int>(nbricks), c->stream);
    checkLaunch(c);
    launch_grid_bound(p, static_cast<int>(ncells), c->stream);
    checkLaunch(c);
    c->brickCounts.alloc(nbricks + 1);
    c->brickStart.alloc(nbricks + 1);
    CK(cudaMemsetAsync(c->brickCounts.p + nbricks, 0, 4, c->stream));
    p.bCounts = c->brickCounts.p;
    launch_brick_clusters(p, static_cast<int>(nbricks), false, c->stream);
    checkLaunch(c);
    // device prefix sums; only the totals come back to the host
    auto deviceScan = [&](const int* in, int* out, long long n) {
        const size_t need = scan_ints(in, out, static_cast<int>(n), nullptr, 0, c->stream);
        if (c->scanTemp.n < std::max<size_t>(need, 1)) c->scanTemp.alloc(std::max<size_t>(need, 1));
        scan_ints(in, out, static_cast<int>(n), c->scanTemp.p, c->scanTemp.n, c->stream);
        int tot = 0;
        CK(cudaMemcpyAsync(&tot, out + n - 1, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return static_cast<long long>(tot);
    };
    {
        const long long bt = deviceScan(c->brickCounts.p, c->brickStart.p, nbricks + 1);
        if (!(bt >= 0 && bt < (1LL << 30))) return false;  // brick cluster lists too large
        c->brickList.alloc(std::max<long long>(bt, 1));
    }
    p.bStart = c->brickStart.p;
    p.bList = c->brickList.p;
    launch_brick_clusters(p, static_cast<int>(nbricks), true, c->stream);
    checkLaunch(c);
    launch_grid_list(p, static_cast<int>(ncells), false, c->stream);
    checkLaunch(c);
    const long long total = deviceScan(c->gridCounts.p, c->gridStart.p, ncells + 1);
    if (!(total >= 0 && total < (1LL << 30))) return false;  // candidate lists too large
    c->gridEntry.alloc(std::max<long long>(total, 1));
    p.entry = c->gridEntry.p;
    p.start = c->gridStart.p;
    launch_grid_list(p, static_cast<int>(ncells), true, c->stream);
    checkLaunch(c);
    c->gridCell.alloc(ncells);
    launch_grid_cells(c->gridStart.p, c->gridEntry.p, c->gridCell.p, static_cast<int>(ncells), c->stream);
    checkLaunch(c);
    CK(cudaStreamSynchronize(c->stream));
    for (int a = 0; a < 3; ++a) {
        c->grid.lo[a] = lo[a];
        c->grid.dim[a] = dim[a];
        c->gridBox[a] = lo[a];
        c->gridBox[3 + a] = lo[a] + dim[a] * h;
    }
    c->grid.invH = 1.0 / h;
    c->grid.h = h;

    for (int a = 0; a < 3; ++a) c->grid.flo[a] = static_cast<float>(lo[a]);
    c->grid.finvH = static_cast<float>(1.0 / h);
    c->grid.start = c->gridStart.p;
    c->grid.cell = c->gridCell.p;
    c->grid.entry = c->gridEntry.p;
    c->gridEntries = total;

    c->haveGrid = true;
    return true;
}

// The candidate grid at the default size, coarser while its lists overflow.
void buildGrid(Ctx* c) {
    for (double f = 1.0;; f *= 0.5) {
        if (buildGridAt(c, f)) return;
        REQ(f > 1.0 / 64, SDFGI_ERR_INVALID, "candidate lists too large");
    }
}


void readCounters(Ctx* c, sdfgi_stats* stats, unsigned long long* tail, int ntail) {
    // [0..13] K1 (and relocation) counters, [16..] tail values, [kShadowStats..+13] K2's
    std::vector<unsigned long long> h(kShadowStats + 32);
    CK(cudaMemcpyAsync(h.data(), c->scr, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (stats) {
        const unsigned long long* k2 = h.data() + kShadowStats;
        for (int i = 0; i < 14; ++i) {
            c->lastTrace[0][i] = h[i];
            c->lastTrace[1][i] = k2[i];
        }
        for (int i = 0; i < 6; ++i) c->lastWork[i] = h[8 + i] + k2[8 + i];
        c->shadeWork[0] = h[20];  // shadeHit calls, MVC evaluations (K3a)
        c->shadeWork[1] = h[21];
        stats->sdf_queries += h[0] + k2[0];
        stats->clusters_visited += h[1] + k2[1];
        stats->clusters_skipped += h[2] + k2[2];
        stats->primitive_evals += h[3] + k2[3];
        stats->trace_steps += h[4] + k2[4];
        stats->sphere_traces += h[5] + k2[5];
        stats->shadow_traces += h[6] + k2[6];
        stats->visibility_traces += h[7] + k2[7];
    }
    for (int i = 0; i < ntail; ++i) tail[i] = h[16 + i];
}

// Trace order of the n Fibonacci samples: sorted along a Morton curve over their
// octahedral coordinates, so the 32 lanes of a warp march neighbouring directions
// (the per-probe random rotation is rigid and keeps neighbours neighbours). Only
// the scheduling order changes; samples are stored and summed by index.
std::vector<int> coherentOrder(int n) {
    const double golden = M_PI * (3.0 - std::sqrt(5.0));
    std::vector<std::pair<uint32_t, int>> keys(n);
    auto spread = [](uint32_t x) {
        x &= 0xffff;
        x = (x | (x << 8)) & 0x00ff00ff;
        x = (x | (x << 4)) & 0x0f0f0f0f;
        x = (x | (x << 2)) & 0x33333333;
        x = (x | (x << 1)) & 0x55555555;
        return x;
    };
    for (int i = 0; i < n; ++i) {
        double z = 1.0 - (2.0 * i + 1.0) / n, r = std::sqrt(std::max(0.0, 1.0 - z * z)), phi = golden * i;
        double x = r * std::cos(phi), y = r * std::sin(phi);
        double nrm = std::fabs(x) + std::fabs(y) + std::fabs(z);
        double px = x / nrm, py = y / nrm;
        if (z < 0) {
            double ox = (1.0 - std::fabs(py)) * (px >= 0 ? 1.0 : -1.0);
            double oy = (1.0 - std::fabs(px)) * (py >= 0 ? 1.0 : -1.0);
            px = ox;
            py = oy;
        }
        uint32_t u = static_cast<uint32_t>(std::min(65535.0, (px * 0.5 + 0.5) * 65535.0));
        uint32_t v = static_cast<uint32_t>(std::min(65535.0, (py * 0.5 + 0.5) * 65535.0));
        keys[i] = {spread(u) | (spread(v) << 1), i};
    }
    std::sort(keys.begin(), keys.end());
    std::vector<int> perm(n);
    for (int j = 0; j < n; ++j) perm[j] = keys[j].second;
    return perm;
}

// Wavefront scratch (kernels.cuh): grow-only so repeated passes never reallocate.
template <typename T>
void reserve(DBuf<T>& b, size_t count) {
    if (b.n < count) b.alloc(count);
}

// Parking buffer for off-grid marches (K1 / K2 far phases): room for every ray and
// every (ray, light) march, capped by SDFGI_PARK_MB (default 8192); marches that
// find it full are traced in place.
template <typename R>
void reservePark(Ctx* c, size_t rays, int lights) {
    const size_t need = std::max(rays * sizeof(ParkRay<R>), rays * lights * sizeof(ParkShadow<R>));
    const char* env = std::getenv("SDFGI_PARK_MB");
    const size_t cap = static_cast<size_t>(env ? std::max(0.0, std::atof(env)) : 8192.0) << 20;
    reserve(c->wPark, std::max<size_t>(std::min(need, cap), 64));
}

// The trace-order hit slots and the compaction's temporary storage for n items.
template <typename R>
void reserveHitAt(Ctx* c, WaveParams<R>& p, size_t n) {
    n = std::max<size_t>(n, 1);
    reserve(c->wHitAt, n);
    const size_t need = compact_hits(nullptr, nullptr, nullptr, static_cast<int>(n), nullptr, 0, c->stream);
    reserve(c->wSelTemp, std::max<size_t>(need, 16));
    p.hitAt = c->wHitAt.p;
    p.selTemp = c->wSelTemp.p;
    p.selTempBytes = c->wSelTemp.n;
    p.maxItems = static_cast<long long>(n);
}

// accel mode 2's escape test (WaveParams::escape) holds when the candidate grid
// exists and the scene has no unbounded primitive (a plane can be reached from
// anywhere outside the grid box)
int escapeOk(const Ctx* c) {
    return (c->accel == 2 && c->haveGrid && c->escapeValid && c->grid.nUnbounded == 0) ? 1 : 0;
}

template <typename R>
WaveParams<R> waveParams(Ctx* c, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand) {
    const int N = static_cast<int>(cfg->n_rays_full);
    const size_t maxRays = static_cast<size_t>(nCand) * 2 * N;
    const int L = std::max(c->nLights, 1);
    reserve(c->wRayCount, std::max(nCand, 1));
    reserve(c->wRayStart, static_cast<size_t>(nCand) + 1);
    reserve(c->wRot, 9 * static_cast<size_t>(std::max(nCand, 1)));
    reserve(c->wHits, std::max<size_t>(maxRays, 1) * sizeof(HitRec<R>));
    reserve(c->wHitList, std::max<size_t>(maxRays, 1));
    reserve(c->wMvcList, std::max<size_t>(maxRays, 1));
    reserve(c->wTriList, std::max<size_t>(maxRays, 1));
    reserve(c->wVis, std::max<size_t>(maxRays, 1) * L * sizeof(R));
    reserve(c->wRad, std::max<size_t>(maxRays, 1) * 3 * sizeof(R));
    reserve(c->wCtr, kLightCtr + L);
    reservePark<R>(c, maxRays, L);
    reserve(c->wSRay, std::max<size_t>(maxRays, 1) * L * sizeof(ShadowRay<R>));
    reserve(c->wPRay, std::max<size_t>(maxRays, 1) * sizeof(ProbeRay<R>));
    if (c->fibN != N) {
        // sphericalFibonacci tables for n = N and 2N from the host's libm (host_trig.h)
        std::vector<double> fib(9 * static_cast<size_t>(N));
        sdfgi_host::fibTable(N, fib.data());
        sdfgi_host::fibTable(2 * N, fib.data() + 3 * N);
        reserve(c->fib, fib.size());
        CK(cudaMemcpyAsync(c->fib.p, fib.data(), fib.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // fib is a local
        std::vector<int> perm = coherentOrder(N);
        std::vector<int> perm2 = coherentOrder(2 * N);
        perm.insert(perm.end(), perm2.begin(), perm2.end());
        upload(c, c->perm, perm.data(), perm.size());
        c->fibN = N;
    }
    WaveParams<R> p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<R>();
    p.pc = c->probeCommon();
    p.cand = cand;
    p.nCand = nCand;
    p.rayCount = c->wRayCount.p;
    p.rayStart = c->wRayStart.p;
    p.rot = c->wRot.p;
    p.quat = c->quatDev;
    p.pray = c->wPRay.p;
    p.fib = c->fib.p;
    p.perm = c->perm.p;
    p.nRaysDirect = -1;  // probe batch: ray count from the K0 prefix sum
    p.hits = reinterpret_cast<HitRec<R>*>(c->wHits.p);
    p.hitList = c->wHitList.p;
    p.mvcList = c->wMvcList.p;
    p.triList = c->wTriList.p;
    p.vis = reinterpret_cast<R*>(c->wVis.p);
    p.rad = reinterpret_cast<R*>(c->wRad.p);
    p.ctr = c->wCtr.p;
    p.sray = reinterpret_cast<ShadowRay<R>*>(c->wSRay.p);
    reserveHitAt<R>(c, p, maxRays);
    p.srayCap = std::max<size_t>(maxRays, 1);
    p.park = c->accel && c->haveGrid && c->wPark.n >= 4096 ? c->wPark.p : nullptr;  // SDFGI_PARK_MB=0: off
    p.parkBytes = p.park ? c->wPark.n : 0;
    p.prevAtlas = c->atlas[c->front].p;
    p.currAtlas = c->atlas[1 - c->front].p;
    p.prevZero = c->frontZero() ? 1 : 0;
    p.escape = escapeOk(c);
    p.settle = p.escape;
    p.ownerFromMarch = c->accel == 2 && c->haveGrid ? 1 : 0;
    p.useClear = c->accel == 2 && !c->clearValid.empty() &&
                 std::all_of(c->clearValid.begin(), c->clearValid.end(), [](char v) { return v != 0; });
    p.oct = c->octRes;
    p.frame = frame;
    p.tc.eps = cfg->surface_epsilon;
    p.tc.rayTMax = cfg->ray_tmax;
    p.tc.shadowK = cfg->shadow_k;
    p.tc.bounceCoeff = cfg->bounce_coeff;
    p.tc.mvcFrac = cfg->mvc_relocation_frac;
    p.tc.maxSteps = static_cast<int>(cfg->max_trace_steps);
    p.tc.shadowSteps = static_cast<int>(cfg->shadow_steps);
    p.hysteresis = cfg->hysteresis;
    p.alphaMin = cfg->alpha_min;
    p.nRaysFull = static_cast<int>(cfg->n_rays_full);
    p.seed = cfg->seed;
    p.rotatePerFrame = static_cast<int>(cfg->rotate_per_frame);
    p.stats = c->scr;
    p.maxDeltaBits = c->scr + 16;
    p.rays = c->scr + 17;
    p.updated = reinterpret_cast<unsigned int*>(c->scr + 18);
    return p;
}

// Everything a pass's quaternions depend on: seed, frame (or none), the
// candidates (null = every probe) and the cascades' levels and bases.
uint64_t quatKey(const Ctx* c, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i, v >>= 8) h = (h ^ (v & 0xff)) * 1099511628211ull;
    };
    mix(cfg->seed);
    mix(cfg->rotate_per_frame ? static_cast<uint64_t>(static_cast<int64_t>(frame)) : 0xf1b0ull);
    mix(static_cast<uint64_t>(nCand));
    mix(cand ? 1 : 0);
    if (cand)
        for (int s = 0; s < nCand; ++s) mix(static_cast<uint64_t>(cand[s]));
    for (const auto& cs : c->cascades) {
        mix(static_cast<uint64_t>(cs.level));
        mix(static_cast<uint64_t>(cs.base));
    }
    return h;
}

void ensurePinned(double*& p, size_t& n, size_t need) {
    if (n >= need) return;
    if (p) CK(cudaFreeHost(p));
    p = nullptr;
    n = 0;
    CK(cudaMallocHost(&p, need * sizeof(double)));
    n = need;
}

void computeQuats(Ctx* c, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand, double* out) {
    std::vector<uint64_t> keys(nCand);
    for (int s = 0; s < nCand; ++s) {
        const int g = cand ? cand[s] : s;
        int ci = 0;
        for (size_t k = 1; k < c->cascades.size(); ++k)
            if (g >= c->cascades[k].base) ci = static_cast<int>(k);
        keys[s] = sdfgi_host::probeKey(c->cascades[ci].level, g - c->cascades[ci].base);
    }
    sdfgi_host::probeQuats(cfg->seed, frame, cfg->rotate_per_frame != 0, keys.data(), nCand, out);
}

// Slot u <- the quaternions of (frame, cand): host libm into its pinned buffer
// (once the previous copy out of it is done), then copied on copyStream once no
// queued pass reads the slot's device buffer.
void fillQuatSlot(Ctx* c, int u, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand, uint64_t key) {
    Ctx::QuatSlot& q = c->qs[u];
    const size_t need = 4 * static_cast<size_t>(std::max(nCand, 1));
    CK(cudaEventSynchronize(q.copied));
    ensurePinned(q.h, q.hn, need);
    computeQuats(c, cfg, frame, cand, nCand, q.h);
    reserve(q.d, need);
    CK(cudaStreamWaitEvent(c->copyStream, q.used, 0));
    CK(cudaMemcpyAsync(q.d.p, q.h, 4 * static_cast<size_t>(nCand) * sizeof(double), cudaMemcpyHostToDevice,
                       c->copyStream));
    CK(cudaEventRecord(q.copied, c->copyStream));
    q.key = key;
}

// randomRotation's quaternion of every candidate for this pass (sampleDirections'
// key: seed, frame or 0xf1b0, probeKey(level, index)), evaluated with the host's
// libm (host_trig.h) — or the previous pass's speculation when it was for this
// frame — in a slot whose device copy runs beside the queued work. cand = null:
// every probe 0..nCand-1. Returns the slot; nothing waits on it yet.
int prepareQuats(Ctx* c, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand) {
    const uint64_t key = quatKey(c, cfg, frame, cand, nCand);
    if (c->qReady >= 0 && c->qs[c->qReady].key == key) return c->qReady;
    int u;
    if (c->qSpec >= 0 && c->qs[c->qSpec].key == key) {
        u = c->qSpec;
    } else {
        u = 1 - c->qLast;
        fillQuatSlot(c, u, cfg, frame, cand, nCand, key);
    }
    c->qSpec = -1;
    c->qReady = u;
    return u;
}

// This pass's quaternions on the device: the stream waits for the slot's copy.
void uploadQuats(Ctx* c, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand) {
    const int u = prepareQuats(c, cfg, frame, cand, nCand);
    CK(cudaStreamWaitEvent(c->stream, c->qs[u].copied, 0));
    c->quatDev = c->qs[u].d.p;
    c->qLast = u;
    c->qReady = -1;
}

// After the launches reading this pass's slot.
void quatsConsumed(Ctx* c) { CK(cudaEventRecord(c->qs[c->qLast].used, c->stream)); }

// The next frame's quaternions for the same candidates into the other slot, on the
// host while the device runs this pass; copied on copyStream.
void speculateQuats(Ctx* c, const sdfgi_cfg* cfg, int frame, const int* cand, int nCand) {
    if (!cfg->rotate_per_frame) return;  // frame-independent: the key matches the current slot's next time
    const int s = 1 - c->qLast;
    fillQuatSlot(c, s, cfg, frame + 1, cand, nCand, quatKey(c, cfg, frame + 1, cand, nCand));
    c->qSpec = s;
}

void validateCfg(Ctx* c, const sdfgi_cfg* cfg) {
    REQ(cfg != nullptr, SDFGI_ERR_INVALID, "null cfg");
    REQ(cfg->oct_res == c->octRes, SDFGI_ERR_INVALID, "cfg.oct_res differs from the cascade atlas resolution");
    // K3 keeps 2N direction+radiance samples in shared memory (<= 227 KB in FP64)
    REQ(cfg->n_rays_full > 0 && cfg->n_rays_full <= 2048, SDFGI_ERR_INVALID, "n_rays_full out of range [1, 2048]");
    REQ(cfg->max_trace_steps >= 0 && cfg->shadow_steps >= 0, SDFGI_ERR_INVALID, "negative step limits");
}

// Global probe ids (cascade base + index) for the update: the caller's refs, or
// every probe; restricted to this rank's z-slabs when world > 1.
std::vector<int> selectRefs(Ctx* c, const int32_t* refs, int nRefs) {
    std::vector<int> out;
    if (refs) {
        REQ(nRefs >= 0, SDFGI_ERR_INVALID, "negative n_refs");
        out.reserve(nRefs);
        for (int i = 0; i < nRefs; ++i) {
            int level = refs[2 * i], idx = refs[2 * i + 1];
            int s = c->slot(level);
            REQ(idx >= 0 && idx < c->cascades[s].count(), SDFGI_ERR_INVALID, "probe index out of range");
            out.push_back(c->cascades[s].base + idx);
        }
    } else {
        out.resize(c->totalProbes);
        for (int i = 0; i < c->totalProbes; ++i) out[i] = i;
    }
    if (c->world > 1) {
        std::vector<int> mine;
        for (int g : out) {
            int s = 0;
            for (size_t k = 0; k < c->cascades.size(); ++k)
                if (g >= c->cascades[k].base) s = static_cast<int>(k);
            int lo, hi;
            slabRange(c->cascades[s], c->rank, c->world, &lo, &hi);
            if (g >= lo && g < hi) mine.push_back(g);
        }
        out.swap(mine);
    }
    return out;
}

void rebuildGrid(Ctx* c);  // below (the grid's margin follows the precision)

}  // namespace

extern "C" {

int sdfgi_abi_version(void) { return SDFGI_ABI_VERSION; }
const char* sdfgi_last_error(void) { return g_err.c_str(); }

int sdfgi_device_count(int* out) {
    return guard([&] {
        REQ(out, SDFGI_ERR_INVALID, "null out");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *out = n;
    });
}

int sdfgi_nccl_unique_id(uint8_t out[128]) {
    return guard([&] {
        REQ(out, SDFGI_ERR_INVALID, "null out");
        static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
        ncclUniqueId id;
        NK(ncclGetUniqueId(&id));
        std::memcpy(out, &id, 128);
    });
}

int sdfgi_ctx_create(int device, int rank, int world, const uint8_t* nccl_uid, int precision, void** out_ctx) {
    return guard([&] {
        REQ(out_ctx, SDFGI_ERR_INVALID, "null out_ctx");
        REQ(world >= 1 && rank >= 0 && rank < world, SDFGI_ERR_INVALID, "bad rank/world");
        REQ(precision == SDFGI_F64 || precision == SDFGI_F32, SDFGI_ERR_INVALID, "bad precision");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        REQ(e == cudaSuccess && n > 0, SDFGI_ERR_CUDA, "no CUDA device: the B200 path has no CPU fallback");
        REQ(device >= 0 && device < n, SDFGI_ERR_INVALID, "device index out of range");
        CK(cudaSetDevice(device));
        Ctx* c = new Ctx();
        c->device = device;
        c->rank = rank;
        c->world = world;
        c->precision = precision;
        try {
            CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            for (auto& e : c->ev) CK(cudaEventCreate(&e));
            CK(cudaStreamCreateWithFlags(&c->copyStream, cudaStreamNonBlocking));
            for (auto& q : c->qs) {
                CK(cudaEventCreateWithFlags(&q.copied, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&q.used, cudaEventDisableTiming));
                CK(cudaEventRecord(q.copied, c->copyStream));
                CK(cudaEventRecord(q.used, c->stream));
            }
            for (auto& e : c->kev) CK(cudaEventCreate(&e));
            c->scratch.alloc(kShadowStats + 32);
            c->report.alloc(4 * kMaxCascades * (Ctx::kMaxPending + 1));
            c->scr = c->scratch.p;
            c->kevCur = c->kev;
            CK(cudaMallocHost(&c->hReport, 4 * kMaxCascades * sizeof(int)));
            CK(cudaEventCreateWithFlags(&c->arenaEv, cudaEventDisableTiming));
            CK(cudaEventRecord(c->arenaEv, c->stream));
            if (world > 1) {
                REQ(nccl_uid, SDFGI_ERR_INVALID, "world > 1 needs an NCCL unique id");
                ncclUniqueId id;
                std::memcpy(&id, nccl_uid, 128);
                NK(ncclCommInitRank(&c->comm, world, id, rank));
            }
        } catch (...) {
            delete c;
            throw;
        }
        *out_ctx = c;
    });
}

int sdfgi_ctx_destroy(void* ctx) {
    return guard([&] {
        if (!ctx) return;
        delete static_cast<Ctx*>(ctx);
    });
}

int sdfgi_ctx_set_precision(void* ctx, int precision) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(precision == SDFGI_F64 || precision == SDFGI_F32, SDFGI_ERR_INVALID, "bad precision");
        c->precision = precision;
        // the grid's margin depends on the precision (buildGridAt): rebuild when it changes
        if (c->haveScene && c->haveGrid && gridMargin(c, precision) != c->gridMargin) rebuildGrid(c);
    });
}

int sdfgi_ctx_stream(void* ctx, void** out) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        *out = c->stream;
    });
}

int sdfgi_ctx_synchronize(void* ctx) {
    return guard([&] {
        Ctx* c = C(ctx);
        CK(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"

namespace {

// The scene's device arrays (CSR order: device primitive j = prims[member_idx[j]])
// and their host copies; no acceleration structure.
void uploadSceneArrays(Ctx* c, const sdfgi_prim* prims, int n_prims, const sdfgi_cluster* clusters, int n_clusters,
                       const int32_t* member_start, const int32_t* member_idx, const sdfgi_light* lights,
                       int n_lights, const double sky[3]) {
    REQ(n_prims >= 0 && n_clusters >= 0 && n_lights >= 0, SDFGI_ERR_INVALID, "negative count");
    REQ(n_prims == 0 || prims, SDFGI_ERR_INVALID, "null prims");
    REQ(n_clusters == 0 || (clusters && member_start && member_idx), SDFGI_ERR_INVALID, "null clusters");
    REQ(n_lights == 0 || lights, SDFGI_ERR_INVALID, "null lights");
    REQ(sky, SDFGI_ERR_INVALID, "null sky");
    int nMembers = n_clusters ? member_start[n_clusters] : 0;
    REQ(n_clusters == 0 || member_start[0] == 0, SDFGI_ERR_INVALID, "member_start[0] != 0");
    for (int k = 0; k < n_clusters; ++k)
        REQ(member_start[k + 1] >= member_start[k], SDFGI_ERR_INVALID, "member_start not monotone");
    for (int m = 0; m < nMembers; ++m)
        REQ(member_idx[m] >= 0 && member_idx[m] < n_prims, SDFGI_ERR_INVALID, "member index out of range");
    for (int i = 0; i < n_prims; ++i)
        REQ(prims[i].kind >= 0 && prims[i].kind <= 4, SDFGI_ERR_INVALID, "bad primitive kind");
    // cluster (CSR) order: device primitive j = prims[member_idx[j]]
    // conversion buffers kept in the context (a re-sent scene touches no fresh pages)
    auto& p64 = c->up64;
    auto& p32 = c->up32;
    auto& orig = c->upOrig;
    auto& kid = c->upKid;
    auto& alb = c->upAlb;
    auto& em = c->upEm;
    p64.resize(nMembers);
    p32.resize(nMembers);
    orig.resize(nMembers);
    kid.resize(std::max(nMembers, 1));
    alb.resize(3 * static_cast<size_t>(nMembers));
    em.resize(3 * static_cast<size_t>(nMembers));
    for (int j = 0; j < nMembers; ++j) {
        const sdfgi_prim& s = prims[member_idx[j]];
        std::memset(&p64[j], 0, sizeof(p64[j]));
        std::memset(&p32[j], 0, sizeof(p32[j]));
        fillPrim(p64[j], s);
        fillPrim(p32[j], s);
        orig[j] = member_idx[j];
        kid[j] = s.kind | (p64[j].identity << 8);
        for (int k = 0; k < 3; ++k) {
            alb[3 * j + k] = s.albedo[k];
            em[3 * j + k] = s.emission[k];
        }
    }
    std::vector<DCluster<double>> c64(n_clusters);
    std::vector<DCluster<float>> c32(n_clusters);
    for (int k = 0; k < n_clusters; ++k) {
        std::memset(&c64[k], 0, sizeof(c64[k]));
        std::memset(&c32[k], 0, sizeof(c32[k]));
        for (int a = 0; a < 3; ++a) {
            c64[k].lo[a] = clusters[k].lo[a];
            c64[k].hi[a] = clusters[k].hi[a];
            // FP32 cull boxes: widened so float rounding of the box distance can
            // never skip a member the FP32 evaluation would have picked
            double lo = clusters[k].lo[a], hi = clusters[k].hi[a];
            double padLo = 1e-5 * (std::fabs(lo) + 1.0), padHi = 1e-5 * (std::fabs(hi) + 1.0);
            c32[k].lo[a] = std::nextafter(static_cast<float>(lo - padLo), -INFINITY);
            c32[k].hi[a] = std::nextafter(static_cast<float>(hi + padHi), INFINITY);
        }
        c64[k].unbounded = c32[k].unbounded = clusters[k].unbounded ? 1 : 0;
    }
    std::vector<int> starts(member_start, member_start + n_clusters + 1);
    if (n_clusters == 0) starts.assign(1, 0);
    upload(c, c->prim64, p64.data(), p64.size());
    upload(c, c->prim32, p32.data(), p32.size());
    upload(c, c->cl64, c64.data(), c64.size());
    upload(c, c->cl32, c32.data(), c32.size());
    upload(c, c->cstart, starts.data(), starts.size());
    upload(c, c->orig, orig.data(), orig.size());
    upload(c, c->albedo, alb.data(), alb.size());
    upload(c, c->emission, em.data(), em.size());
    upload(c, c->kindId, kid.data(), kid.size());
    upload(c, c->lights, reinterpret_cast<const DLight*>(lights), n_lights);
    // shared-memory staging of the primitive records for K1/K2 (evalPrimStaged):
    // FP64 64 B per primitive + 64 B per rotation row, FP32 the 64 B records as is
    {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
        const long long limit = static_cast<long long>(optin) - 1024;  // the kernels' static shared memory
        const char* senv = std::getenv("SDFGI_STAGE");
        const bool allow = !(senv && std::atoi(senv) == 0) && nMembers > 0;
        auto& st = c->upStage;
        auto& rows = c->upRows;
        st.resize(64 * static_cast<size_t>(nMembers));
        rows.clear();
        for (int j = 0; j < nMembers; ++j) {
            unsigned char* r = st.data() + 64 * static_cast<size_t>(j);
            std::memcpy(r, &p64[j], 64);
            int rotIdx = -1;
            if (!p64[j].identity) {
                rotIdx = static_cast<int>(rows.size() / 64);
                const unsigned char* src = reinterpret_cast<const unsigned char*>(&p64[j]) + 64;
                rows.insert(rows.end(), src, src + 64);
            }
            std::memcpy(r + 52, &rotIdx, 4);  // the identity flag's slot
        }
        const long long b64 = static_cast<long long>(st.size() + rows.size());
        c->stage64Bytes = 0;
        if (allow && b64 <= limit) {
            st.insert(st.end(), rows.begin(), rows.end());
            upload(c, c->stage64, st.data(), st.size());
            c->stage64Bytes = static_cast<int>(b64);
            c->stage64RotOff = 64 * nMembers;
        }
        const long long b32 = 64LL * nMembers;
        c->stage32Bytes = (allow && b32 <= limit) ? static_cast<int>(b32) : 0;
    }
    CK(cudaStreamSynchronize(c->stream));
    c->nPrims = nMembers;
    c->nClusters = n_clusters;
    c->nLights = n_lights;
    for (int k = 0; k < 3; ++k) c->sky[k] = sky[k];
    c->haveScene = true;
    c->hPrims.assign(prims, prims + n_prims);
    c->hMember.assign(member_idx, member_idx + (n_clusters ? member_start[n_clusters] : 0));
    c->hClusters.assign(clusters, clusters + n_clusters);
    c->hStart.assign(member_start, member_start + (n_clusters ? n_clusters + 1 : 0));
    c->hLights.assign(lights, lights + n_lights);
}

// Geometry of primitive a and b equal (the fields the SDF reads)
bool sameGeometry(const sdfgi_prim& a, const sdfgi_prim& b) {
    return a.kind == b.kind && std::memcmp(a.rot, b.rot, sizeof(a.rot)) == 0 &&
           std::memcmp(a.trans, b.trans, sizeof(a.trans)) == 0 && std::memcmp(a.size, b.size, sizeof(a.size)) == 0;
}

void checkEscape(Ctx* c);

// The grid's CSR positions -> the current ones (the caller re-clustered: same
// primitives, other cluster order), and the dynamic list's CSR positions.
void remapGrid(Ctx* c) {
    std::vector<int> csrOf(c->hPrims.size(), -1);
    for (size_t j = 0; j < c->hMember.size(); ++j)
        if (csrOf[c->hMember[j]] < 0) csrOf[c->hMember[j]] = static_cast<int>(j);
    if (c->gridCsrOrig != c->hMember) {
        std::vector<int> map(std::max<size_t>(c->gridCsrOrig.size(), 1));
        for (size_t j = 0; j < c->gridCsrOrig.size(); ++j) map[j] = csrOf[c->gridCsrOrig[j]];
        DBuf<int> dmap;
        upload(c, dmap, map.data(), map.size());
        launch_grid_remap(c->gridEntry.p, c->gridEntries, dmap.p, c->stream);
        checkLaunch(c);
        launch_grid_cells(c->gridStart.p, c->gridEntry.p, c->gridCell.p,
                          c->grid.dim[0] * c->grid.dim[1] * c->grid.dim[2], c->stream);
        checkLaunch(c);
        CK(cudaStreamSynchronize(c->stream));
        dmap.free();
        c->gridCsrOrig = c->hMember;
    }
    std::vector<int> dyn;
    for (int o : c->gridDyn)
        if (csrOf[o] >= 0) dyn.push_back(csrOf[o]);
    std::sort(dyn.begin(), dyn.end());
    c->nDyn = static_cast<int>(dyn.size());
    if (dyn.empty()) dyn.push_back(0);
    upload(c, c->dynCsr, dyn.data(), dyn.size());
    CK(cudaStreamSynchronize(c->stream));
}

// The candidate grid over every primitive not in gridDyn (the ones that moved since
// it was built): with dynamic primitives the lists and bounds are built on a scene
// of the static ones (clusters without their dynamic members), then mapped back to
// the full scene's CSR order; queries evaluate the dynamic list besides the cell
// list (query()). The cluster BVH is over the full scene.
void rebuildGrid(Ctx* c) {
    if (c->gridDyn.empty()) {
        buildGrid(c);
        c->gridCsrOrig = c->hMember;
    } else {
        const std::vector<sdfgi_prim> fp = c->hPrims;
        const std::vector<int32_t> fm = c->hMember, fs = c->hStart;
        const std::vector<sdfgi_cluster> fc = c->hClusters;
        const std::vector<sdfgi_light> fl = c->hLights;
        const double sky[3] = {c->sky[0], c->sky[1], c->sky[2]};
        std::vector<char> isDyn(fp.size(), 0);
        for (int o : c->gridDyn) isDyn[o] = 1;
        std::vector<sdfgi_cluster> sc;
        std::vector<int32_t> ss{0}, sm;
        for (size_t k = 0; k + 1 < fs.size(); ++k) {
            const size_t before = sm.size();
            for (int m = fs[k]; m < fs[k + 1]; ++m)
                if (!isDyn[fm[m]]) sm.push_back(fm[m]);
            if (sm.size() == before) continue;
            sc.push_back(fc[k]);
            ss.push_back(static_cast<int32_t>(sm.size()));
        }
        uploadSceneArrays(c, fp.data(), static_cast<int>(fp.size()), sc.data(), static_cast<int>(sc.size()), ss.data(),
                          sm.data(), fl.data(), static_cast<int>(fl.size()), sky);
        buildGrid(c);
        c->gridCsrOrig = sm;
        uploadSceneArrays(c, fp.data(), static_cast<int>(fp.size()), fc.data(), static_cast<int>(fc.size()), fs.data(),
                          fm.data(), fl.data(), static_cast<int>(fl.size()), sky);
    }
    double scale = 0;
    for (int a = 0; a < 6; ++a) scale = std::max(scale, std::fabs(c->gridBox[a]));
    buildBvh(c, scale);
    if (c->haveGrid) remapGrid(c);
    checkEscape(c);
}

// accel mode 2's escape tests need every bounded primitive inside the grid box
void checkEscape(Ctx* c) {
    bool inside = c->haveGrid;
    for (int a = 0; a < 3 && inside; ++a)
        inside = c->grid.geoLo[a] >= c->gridBox[a] && c->grid.geoHi[a] <= c->gridBox[3 + a];
    c->escapeValid = inside;
}

}  // namespace

extern "C" {

int sdfgi_scene_upload(void* ctx, const sdfgi_prim* prims, int n_prims, const sdfgi_cluster* clusters,
                       int n_clusters, const int32_t* member_start, const int32_t* member_idx,
                       const sdfgi_light* lights, int n_lights, const double sky[3]) {
    return guard([&] {
        Ctx* c = C(ctx);
        const auto T0 = std::chrono::steady_clock::now();
        std::vector<sdfgi_prim> prev;
        prev.swap(c->hPrims);  // uploadSceneArrays stores the new ones
        std::fill(c->clearValid.begin(), c->clearValid.end(), 0);  // the SDF may have changed
        uploadSceneArrays(c, prims, n_prims, clusters, n_clusters, member_start, member_idx, lights, n_lights, sky);
        const auto T1 = std::chrono::steady_clock::now();
        // The acceleration structures are a function of the geometry alone. A static
        // scene re-sent every frame keeps its grid; when primitives move, the ones
        // that moved become "dynamic" (left out of the grid lists, evaluated by every
        // query) and only a primitive moving for the first time rebuilds the grid
        // (without it); beyond kMaxDynamic moving primitives the grid is rebuilt over
        // all of them. A re-clustering of the same geometry remaps the lists.
        uint64_t ph = 1469598103934665603ull;
        for (const char* k : {"SDFGI_GRID_MARGIN", "SDFGI_GRID_CELLS", "SDFGI_GRID_MAXLIST", "SDFGI_GRID_HINT",
                              "SDFGI_DYNAMIC_MAX"}) {
            const char* v = std::getenv(k);  // the grid's build parameters
            const std::string t = v ? v : "-";
            for (unsigned char ch : t) ph = (ph ^ ch) * 1099511628211ull;
        }
        bool sameSet = c->haveGrid && prev.size() == static_cast<size_t>(n_prims) && c->gridParams == ph &&
                       (c->gridAccel != 0) == (c->accel != 0);
        for (int i = 0; sameSet && i < n_prims; ++i) sameSet = prev[i].id == prims[i].id;
        std::vector<int> moved;
        if (sameSet)
            for (int i = 0; i < n_prims; ++i)
                if (!sameGeometry(prev[i], prims[i])) moved.push_back(i);
        const char* denv = std::getenv("SDFGI_DYNAMIC_MAX");
        const int maxDyn = denv ? std::atoi(denv) : kMaxDynamic;
        if (!sameSet) {
            c->gridDyn.clear();
            c->gridParams = ph;
            c->gridAccel = c->accel;
            rebuildGrid(c);
            return;
        }
        std::vector<int> grow;
        std::set_difference(moved.begin(), moved.end(), c->gridDyn.begin(), c->gridDyn.end(), std::back_inserter(grow));
        if (grow.empty()) {  // the grid's static geometry is unchanged: refit
            double scale = 0;
            for (int a = 0; a < 6; ++a) scale = std::max(scale, std::fabs(c->gridBox[a]));
            const auto T2 = std::chrono::steady_clock::now();
            buildBvh(c, scale);
            const auto T3 = std::chrono::steady_clock::now();
            remapGrid(c);
            checkEscape(c);
            if (std::getenv("SDFGI_TIMING")) {
                auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
                std::fprintf(stderr, "scene_upload us: arrays %.1f compare %.1f bvh %.1f remap %.1f\n", us(T0, T1),
                             us(T1, T2), us(T2, T3), us(T3, std::chrono::steady_clock::now()));
            }
            ++c->gridRefits;
            return;
        }
        std::vector<int> dyn;
        std::set_union(c->gridDyn.begin(), c->gridDyn.end(), grow.begin(), grow.end(), std::back_inserter(dyn));
        c->gridDyn = (static_cast<int>(dyn.size()) <= maxDyn && 4 * dyn.size() < static_cast<size_t>(n_prims))
                         ? dyn : std::vector<int>();
        rebuildGrid(c);
    });
}

int sdfgi_lights_upload(void* ctx, const sdfgi_light* lights, int n_lights, const double sky[3]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(n_lights >= 0 && (n_lights == 0 || lights) && sky, SDFGI_ERR_INVALID, "bad lights");
        upload(c, c->lights, reinterpret_cast<const DLight*>(lights), n_lights);
        CK(cudaStreamSynchronize(c->stream));
        c->nLights = n_lights;
        for (int k = 0; k < 3; ++k) c->sky[k] = sky[k];
    });
}

int sdfgi_cascade_set(void* ctx, int level, int res_x, int res_y, int res_z, double spacing, const double origin[3],
                      int oct_res) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(res_x > 0 && res_y > 0 && res_z > 0, SDFGI_ERR_INVALID, "resolution must be positive");
        REQ(spacing > 0 && origin, SDFGI_ERR_INVALID, "bad spacing/origin");
        REQ(oct_res >= 1 && oct_res <= 10, SDFGI_ERR_INVALID, "oct_res must be in [1, 10]");
        REQ(c->cascades.empty() || oct_res == c->octRes, SDFGI_ERR_INVALID, "all cascades share one oct_res");
        REQ(static_cast<long long>(res_x) * res_y * res_z < (1LL << 30), SDFGI_ERR_INVALID, "too many probes");
        CascadeHost h;
        h.res[0] = res_x;
        h.res[1] = res_y;
        h.res[2] = res_z;
        h.level = level;
        h.spacing = spacing;
        for (int k = 0; k < 3; ++k) h.origin[k] = origin[k];
        bool replaced = false, sameShape = false;
        int slot = -1;
        for (size_t k = 0; k < c->cascades.size(); ++k) {
            CascadeHost& cs = c->cascades[k];
            if (cs.level == level) {
                sameShape = cs.count() == h.count();
                h.base = cs.base;
                cs = h;
                replaced = true;
                slot = static_cast<int>(k);
            }
        }
        if (!replaced) {
            REQ(static_cast<int>(c->cascades.size()) < kMaxCascades, SDFGI_ERR_INVALID, "too many cascades");
            c->cascades.push_back(h);
        }
        if (replaced && sameShape && oct_res == c->octRes) {
            // recenterCascade (probe_volume.hpp:80-86): this cascade's probes are
            // re-made and its atlas tiles cleared (pipeline.hpp:110-113); the other
            // cascades and the front/back roles are untouched
            resetProbes(c, slot);
        } else {
            c->octRes = oct_res;
            c->front = 0;
            reallocProbes(c);
        }
        // grow the grid over this volume (one probe spacing of slack, plus a quarter
        // of the volume so a scrolling cascade does not rebuild every frame)
        double box[6];
        bool covered = c->haveGrid;
        for (int a = 0; a < 3; ++a) {
            const int r = a == 0 ? res_x : (a == 1 ? res_y : res_z);
            box[a] = origin[a] - spacing;
            box[3 + a] = origin[a] + r * spacing;
            covered = covered && box[a] >= c->gridBox[a] && box[3 + a] <= c->gridBox[3 + a];
        }
        const char* henv = std::getenv("SDFGI_GRID_HINT");
        if (!covered && !(henv && std::atoi(henv) == 0)) {
            for (int a = 0; a < 3; ++a) {
                const double slack = 0.25 * (box[3 + a] - box[a]);
                const double blo = box[a] - slack, bhi = box[3 + a] + slack;
                c->hint[a] = c->hintValid ? std::min(c->hint[a], blo) : blo;
                c->hint[3 + a] = c->hintValid ? std::max(c->hint[3 + a], bhi) : bhi;
            }
            c->hintValid = true;
            if (c->haveScene) rebuildGrid(c);
        }
    });
}

int sdfgi_cascade_count(void* ctx, int* out) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        *out = static_cast<int>(c->cascades.size());
    });
}

int sdfgi_cascades_clear(void* ctx) {
    return guard([&] {
        Ctx* c = C(ctx);
        c->cascades.clear();
        c->front = 0;
        reallocProbes(c);
    });
}

int sdfgi_probes_reset(void* ctx, int level) {
    return guard([&] {
        Ctx* c = C(ctx);
        resetProbes(c, c->slot(level));
    });
}

static_assert(sizeof(sdfgi_probe) == 11 * sizeof(double), "sdfgi_probe is 11 doubles (k_probes_unpack)");

int sdfgi_probes_upload(void* ctx, int level, const sdfgi_probe* probes, int n) {
    return guard([&] {
        Ctx* c = C(ctx);
        int s = c->slot(level);
        c->clearValid.resize(c->cascades.size(), 0);
        c->clearValid[s] = 0;
        const CascadeHost& cs = c->cascades[s];
        REQ(probes && n == cs.count(), SDFGI_ERR_INVALID, "probe count mismatch");
        // the records in one copy, split into the device arrays there
        reserve(c->probeAos, 11 * static_cast<size_t>(n));
        stageCopy(c, c->probeAos.p, probes, static_cast<size_t>(n) * sizeof(sdfgi_probe));
        launch_probes_unpack(c->probeCommon().probes, cs.base, n, c->probeAos.p, c->stream);
        checkLaunch(c);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_probes_download(void* ctx, int level, sdfgi_probe* probes, int n) {
    return guard([&] {
        Ctx* c = C(ctx);
        int s = c->slot(level);
        const CascadeHost& cs = c->cascades[s];
        REQ(probes && n == cs.count(), SDFGI_ERR_INVALID, "probe count mismatch");
        reserve(c->probeAos, 11 * static_cast<size_t>(n));
        launch_probes_pack(c->probeCommon().probes, cs.base, n, c->probeAos.p, c->stream);
        checkLaunch(c);
        CK(cudaMemcpyAsync(probes, c->probeAos.p, static_cast<size_t>(n) * sizeof(sdfgi_probe), cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_select_probes(void* ctx, const double cam_pos[3], const double cam_fwd[3], int budget, int frame,
                        int32_t* out_refs, int* n_out) {
    return guard([&] {
        Ctx* c = C(ctx);
        requireProbes(c);
        REQ(cam_pos && cam_fwd && n_out, SDFGI_ERR_INVALID, "null argument");
        const int total = c->totalProbes;
        *n_out = 0;
        if (total == 0 || budget <= 0) return;  // probe_volume.hpp:171
        REQ(out_refs, SDFGI_ERR_INVALID, "null out_refs");
        SelectParams P;
        std::memset(&P, 0, sizeof(P));
        P.pc = c->probeCommon();
        P.total = total;
        P.frame = frame;
        P.forceAge = static_cast<int>((static_cast<long long>(total) + budget - 1) / budget);  // one fair period
        for (int k = 0; k < 3; ++k) {
            P.camPos[k] = cam_pos[k];
            P.camFwd[k] = cam_fwd[k];
        }
        const size_t n = static_cast<size_t>(total);
        const size_t tempBytes = select_scratch_bytes(total);
        size_t off = 0;
        auto carve = [&](size_t bytes) {
            size_t o = off;
            off += (bytes + 255) & ~static_cast<size_t>(255);
            return o;
        };
        const size_t oForced = carve(n), oOther = carve(n), oIds = carve(4 * n), oKeyF = carve(4 * n),
                     oKeyO = carve(8 * n), oIdsF = carve(4 * n), oIdsO = carve(4 * n), oIdsF2 = carve(4 * n),
                     oIdsO2 = carve(4 * n), oKF = carve(4 * n), oKF2 = carve(4 * n), oKO = carve(8 * n),
                     oKO2 = carve(8 * n), oCounts = carve(8), oRefs = carve(8 * n), oTemp = carve(tempBytes);
        reserve(c->selScratch, off);
        unsigned char* b = c->selScratch.p;
        P.forced = reinterpret_cast<char*>(b + oForced);
        P.other = reinterpret_cast<char*>(b + oOther);
        P.ids = reinterpret_cast<int*>(b + oIds);
        P.keyForced = reinterpret_cast<unsigned int*>(b + oKeyF);
        P.keyOther = reinterpret_cast<unsigned long long*>(b + oKeyO);
        P.idsF = reinterpret_cast<int*>(b + oIdsF);
        P.idsO = reinterpret_cast<int*>(b + oIdsO);
        P.idsF2 = reinterpret_cast<int*>(b + oIdsF2);
        P.idsO2 = reinterpret_cast<int*>(b + oIdsO2);
        P.kF = reinterpret_cast<unsigned int*>(b + oKF);
        P.kF2 = reinterpret_cast<unsigned int*>(b + oKF2);
        P.kO = reinterpret_cast<unsigned long long*>(b + oKO);
        P.kO2 = reinterpret_cast<unsigned long long*>(b + oKO2);
        P.counts = reinterpret_cast<int*>(b + oCounts);
        P.outRefs = reinterpret_cast<int*>(b + oRefs);
        P.temp = b + oTemp;
        P.tempBytes = tempBytes;
        const int sel = launch_select(P, budget, c->stream, &c->launches);
        checkLaunch(c);
        if (sel > 0)
            CK(cudaMemcpyAsync(out_refs, P.outRefs, 8 * static_cast<size_t>(sel), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *n_out = sel;
    });
}

// updateProbePositions for cascade slot s, enqueued on the context stream (no host
// synchronisation): counts land in rep[0..2] on the device.
void relocEnqueue(Ctx* c, int s, double threshold1, double threshold2, int max_descent_steps,
                  double gradient_step, bool stats, int* rep, bool clearCounters = true) {
    RelocParams p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<double>();
    p.pc = c->probeCommon();
    p.cascade = s;
    p.th1 = threshold1;
    p.th2 = threshold2;
    p.maxSteps = max_descent_steps;
    p.gradStep = gradient_step;
    p.report = rep;
    p.stats = c->scr;
    CK(cudaMemsetAsync(rep, 0, 4 * sizeof(int), c->stream));
    if (clearCounters) CK(cudaMemsetAsync(c->scr, 0, (kShadowStats + 32) * 8, c->stream));
    // relocation is replicated on every rank (deterministic, bit-exact): no exchange
    CK(cudaEventRecord(c->ev[2], c->stream));
    launch_relocate(p, c->cascades[s].count(), stats, c->stream);
    checkLaunch(c);
    c->clearValid.resize(c->cascades.size(), 0);
    c->clearValid[s] = 1;  // every probe's SDF at its new position (RelocParams: pv.clear)
    CK(cudaEventRecord(c->ev[3], c->stream));
    c->evReloc = true;
}

void fillReport(sdfgi_reloc_report* report, const int* rep) {
    report->relocated = rep[0];
    report->rejected = rep[1];
    report->dead = rep[2];
    report->_pad = 0;
}

int sdfgi_probes_relocate(void* ctx, int level, double threshold1, double threshold2, int max_descent_steps,
                          double gradient_step, sdfgi_reloc_report* report, sdfgi_stats* stats) {
    return guard([&] {
        Ctx* c = C(ctx);
        requireProbes(c);
        int s = c->slot(level);
        relocEnqueue(c, s, threshold1, threshold2, max_descent_steps, gradient_step, stats != nullptr, c->report.p);
        int rep[4];
        CK(cudaMemcpyAsync(rep, c->report.p, sizeof(rep), cudaMemcpyDeviceToHost, c->stream));
        readCounters(c, stats, nullptr, 0);
        if (report) fillReport(report, rep);
    });
}

// The update half of the probe stage (pipeline.hpp:126-151); ends with the one
// host synchronisation of the call (readCounters).
// noSync (sdfgi_probe_stage_async): the pass's tail counters are copied to the
// slot's pinned words instead, read by sdfgi_probe_stage_collect.
bool updateBody(Ctx* c, const int32_t* probe_refs, int n_refs, int frame, const sdfgi_cfg* cfg,
                sdfgi_update_result* result, sdfgi_stats* stats, unsigned long long* noSync = nullptr) {
    requireProbes(c);
    validateCfg(c, cfg);
    std::vector<int> refs = selectRefs(c, probe_refs, n_refs);
    float* back = c->atlas[1 - c->front].p;
    const float* frontp = c->atlas[c->front].p;
    // atlas_[write] = atlas_[read] (pipeline.hpp:131); updated tiles are overwritten
    CK(cudaMemcpyAsync(back, frontp, c->atlasFloats() * 4, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemsetAsync(c->scr, 0, (kShadowStats + 32) * 8, c->stream));
    const bool all = (probe_refs == nullptr && c->world == 1);
    // back <- front (copied above) + the updated tiles: still all-zero only if no
    // probe anywhere is updated this pass
    const bool anyUpdate = probe_refs == nullptr ? c->totalProbes > 0 : n_refs > 0;
    c->atlasZero[1 - c->front] = c->atlasZero[c->front];
    if (anyUpdate) std::fill(c->atlasZero[1 - c->front].begin(), c->atlasZero[1 - c->front].end(), 0);
    if (!all) upload(c, c->refs, refs.data(), refs.size());
    const int nCand = static_cast<int>(refs.size());
    if (nCand > 0) {
        const int* cand = all ? nullptr : c->refs.p;
        uploadQuats(c, cfg, frame, all ? nullptr : refs.data(), nCand);
        if (c->precision == SDFGI_F64) {
            WaveParams<double> p = waveParams<double>(c, cfg, frame, cand, nCand);
            launch_wavefront<double>(p, c->persistCap, stats != nullptr, c->stream, c->kevCur,
                                     &c->launches);
        } else {
            WaveParams<float> p = waveParams<float>(c, cfg, frame, cand, nCand);
            launch_wavefront<float>(p, c->persistCap, stats != nullptr, c->stream, c->kevCur,
                                    &c->launches);
        }
        CK(cudaGetLastError());
        c->evUpdate = true;
        quatsConsumed(c);
        speculateQuats(c, cfg, frame, all ? nullptr : refs.data(), nCand);
    }
    if (c->world > 1) {
        // all-gather the back atlas slabs in place (one broadcast per rank-owned
        // slab: slabs may be uneven), then sum counters / max the jitter metric.
        NK(ncclGroupStart());
        for (auto& cs : c->cascades)
            for (int r = 0; r < c->world; ++r) {
                int lo, hi;
                slabRange(cs, r, c->world, &lo, &hi);
                if (hi <= lo) continue;
                float* ptr = back + static_cast<size_t>(lo) * c->tileFloats();
                NK(ncclBroadcast(ptr, ptr, static_cast<size_t>(hi - lo) * c->tileFloats(), ncclFloat, r, c->comm,
                                 c->stream));
            }
        NK(ncclGroupEnd());
        NK(ncclAllReduce(c->scr, c->scr, 14, ncclUint64, ncclSum, c->comm, c->stream));
        NK(ncclAllReduce(c->scr + kShadowStats, c->scr + kShadowStats, 14, ncclUint64, ncclSum,
                         c->comm, c->stream));
        NK(ncclAllReduce(c->scr + 16, c->scr + 16, 1, ncclUint64, ncclMax, c->comm, c->stream));
        NK(ncclAllReduce(c->scr + 17, c->scr + 17, 2, ncclUint64, ncclSum, c->comm, c->stream));
    }
    if (c->world > 1) {
        // every rank marks every updated probe (probe_update.hpp:208-209) on the
        // device, so the replicated probe state stays identical without an exchange
        const int* ids = nullptr;
        int nAll = c->totalProbes;
        if (probe_refs) {
            std::vector<int> allRefs(n_refs);
            for (int i = 0; i < n_refs; ++i)
                allRefs[i] = c->cascades[c->slot(probe_refs[2 * i])].base + probe_refs[2 * i + 1];
            upload(c, c->allRefs, allRefs.data(), allRefs.size());
            ids = c->allRefs.p;
            nAll = n_refs;
        }
        launch_mark_updated(ids, nAll, frame, c->alive.p, c->reject.p, c->lastFrame.p, c->stream);
        checkLaunch(c);
    }
    if (noSync) {
        CK(cudaMemcpyAsync(noSync, c->scr + 16, 3 * 8, cudaMemcpyDeviceToHost, c->stream));
        return nCand > 0;
    }
    unsigned long long tail[3];
    readCounters(c, stats, tail, 3);
    if (nCand > 0) {  // this update's stage events are complete (readCounters synchronised)
        for (int i = 0; i + 1 < kWaveEvents; ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c->kev[i], c->kev[i + 1]));
            c->stageSum[i] += ms;
        }
        float tot = 0.f;
        CK(cudaEventElapsedTime(&tot, c->kev[0], c->kev[kWaveEvents - 1]));
        c->stageSum[kWaveEvents - 1] += tot;
    }
    if (result) {
        double md;
        std::memcpy(&md, &tail[0], 8);
        result->max_texel_delta = md;
        result->rays_traced = static_cast<int64_t>(tail[1]);
        result->probes_updated = static_cast<int64_t>(tail[2] & 0xffffffffull);
    }
    return nCand > 0;
}

int sdfgi_probes_update(void* ctx, const int32_t* probe_refs, int n_refs, int frame, const sdfgi_cfg* cfg,
                        sdfgi_update_result* result, sdfgi_stats* stats) {
    return guard([&] { updateBody(C(ctx), probe_refs, n_refs, frame, cfg, result, stats); });
}

int sdfgi_probe_stage(void* ctx, int frame, const sdfgi_cfg* cfg, const double cam_pos[3], const double cam_fwd[3],
                      sdfgi_reloc_report* reports, int n_reports, sdfgi_update_result* result, sdfgi_stats* stats) {
    return guard([&] {
        Ctx* c = C(ctx);
        requireProbes(c);
        validateCfg(c, cfg);
        const int nc = static_cast<int>(c->cascades.size());
        REQ(reports == nullptr || n_reports >= nc, SDFGI_ERR_INVALID, "reports: one per cascade");
        // probe placement for every cascade (pipeline.hpp:108-123), thresholds as
        // cfg_.threshold1/2(spacing): fraction x spacing
        CK(cudaMemsetAsync(c->scratch.p, 0, (kShadowStats + 32) * 8, c->stream));
        for (int s = 0; s < nc; ++s) {
            const double sp = c->cascades[s].spacing;
            relocEnqueue(c, s, cfg->threshold1_frac * sp, cfg->threshold2_frac * sp,
                         static_cast<int>(cfg->max_descent_steps), cfg->gradient_step, stats != nullptr,
                         c->report.p + 4 * s, false);
        }
        if (cfg->probe_budget <= 0 && c->totalProbes > 0) {
            // this pass's quaternions (unless speculated) on the host while the device
            // relocates, copied beside it; the update's stream waits for them
            const std::vector<int> cand = selectRefs(c, nullptr, 0);
            if (!cand.empty())
                prepareQuats(c, cfg, frame, c->world == 1 ? nullptr : cand.data(), static_cast<int>(cand.size()));
        }
        sdfgi_stats relocStats;
        std::memset(&relocStats, 0, sizeof(relocStats));
        if (stats) readCounters(c, &relocStats, nullptr, 0);  // the update clears the counters
        std::vector<int32_t> refs;
        const int32_t* pr = nullptr;
        int nr = 0;
        if (cfg->probe_budget > 0) {
            // selectProbesForUpdate after placement (pipeline.hpp:132-135)
            REQ(cam_pos && cam_fwd, SDFGI_ERR_INVALID, "a probe budget needs the camera");
            refs.resize(2 * static_cast<size_t>(std::min<int64_t>(cfg->probe_budget, c->totalProbes)));
            int rc = sdfgi_select_probes(ctx, cam_pos, cam_fwd, static_cast<int>(cfg->probe_budget), frame,
                                         refs.data(), &nr);
            REQ(rc == SDFGI_OK, rc, "probe selection failed");
            pr = refs.data();
        }
        // pinned destination: the copy stays asynchronous until the update's sync
        CK(cudaMemcpyAsync(c->hReport, c->report.p, sizeof(int) * 4 * nc, cudaMemcpyDeviceToHost, c->stream));
        static const int32_t kNoRefs[2] = {0, 0};
        if (cfg->probe_budget > 0 && nr == 0) pr = kNoRefs;  // budget selected nothing: not "every probe"
        updateBody(c, pr, nr, frame, cfg, result, stats);  // synchronises
        if (reports)
            for (int s = 0; s < nc; ++s) fillReport(&reports[s], c->hReport + 4 * s);
        if (stats) {
            stats->sdf_queries += relocStats.sdf_queries;
            stats->clusters_visited += relocStats.clusters_visited;
            stats->clusters_skipped += relocStats.clusters_skipped;
            stats->primitive_evals += relocStats.primitive_evals;
            stats->trace_steps += relocStats.trace_steps;
            stats->sphere_traces += relocStats.sphere_traces;
            stats->shadow_traces += relocStats.shadow_traces;
            stats->visibility_traces += relocStats.visibility_traces;
        }
    });
}

constexpr int kAsyncHostWords = 3 + 2 * kMaxCascades;  // tail counters + 4 int32 per cascade report

int sdfgi_probe_stage_async(void* ctx, int frame, const sdfgi_cfg* cfg, const double cam_pos[3],
                            const double cam_fwd[3]) {
    return guard([&] {
        Ctx* c = C(ctx);
        requireProbes(c);
        validateCfg(c, cfg);
        REQ(c->nPending < Ctx::kMaxPending, SDFGI_ERR_STATE, "too many passes in flight: collect them first");
        if (!c->hAsync) {
            CK(cudaMallocHost(&c->hAsync, Ctx::kMaxPending * kAsyncHostWords * sizeof(unsigned long long)));
            c->scratchAsync.alloc(static_cast<size_t>(Ctx::kMaxPending) * Ctx::kSlotWords);
            for (auto& row : c->kevAsync)
                for (auto& e : row) CK(cudaEventCreate(&e));
        }
        const int k = c->nPending;
        const int nc = static_cast<int>(c->cascades.size());
        // report region 0 belongs to the synchronous calls
        int* rep = c->report.p + 4 * kMaxCascades * (k + 1);
        unsigned long long* host = c->hAsync + k * kAsyncHostWords;
        struct Restore {
            Ctx* c;
            ~Restore() {
                c->scr = c->scratch.p;
                c->kevCur = c->kev;
            }
        } restore{c};
        c->scr = c->scratchAsync.p + static_cast<size_t>(k) * Ctx::kSlotWords;
        c->kevCur = c->kevAsync[k];
        CK(cudaMemsetAsync(c->scr, 0, Ctx::kSlotWords * 8, c->stream));
        for (int s = 0; s < nc; ++s) {
            const double sp = c->cascades[s].spacing;
            relocEnqueue(c, s, cfg->threshold1_frac * sp, cfg->threshold2_frac * sp,
                         static_cast<int>(cfg->max_descent_steps), cfg->gradient_step, false, rep + 4 * s, false);
        }
        std::vector<int32_t> refs;
        const int32_t* pr = nullptr;
        int nr = 0;
        static const int32_t kNoRefs[2] = {0, 0};
        if (cfg->probe_budget > 0) {  // the selection reads the relocated probes back: synchronous
            REQ(cam_pos && cam_fwd, SDFGI_ERR_INVALID, "a probe budget needs the camera");
            refs.resize(2 * static_cast<size_t>(std::min<int64_t>(cfg->probe_budget, c->totalProbes)));
            int rc = sdfgi_select_probes(ctx, cam_pos, cam_fwd, static_cast<int>(cfg->probe_budget), frame,
                                         refs.data(), &nr);
            REQ(rc == SDFGI_OK, rc, "probe selection failed");
            pr = nr > 0 ? refs.data() : kNoRefs;
        } else if (c->totalProbes > 0) {
            const std::vector<int> cand = selectRefs(c, nullptr, 0);
            if (!cand.empty())
                prepareQuats(c, cfg, frame, c->world == 1 ? nullptr : cand.data(), static_cast<int>(cand.size()));
        }
        CK(cudaMemcpyAsync(host + 3, rep, 4 * nc * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        c->pendingTimed[k] = updateBody(c, pr, nr, frame, cfg, nullptr, nullptr, host);
        c->pendingCascades[k] = nc;
        ++c->nPending;
    });
}

int sdfgi_probe_stage_collect(void* ctx, sdfgi_reloc_report* reports, int reports_per_pass,
                              sdfgi_update_result* results, int max_passes, int* n_passes) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(n_passes, SDFGI_ERR_INVALID, "null n_passes");
        CK(cudaStreamSynchronize(c->stream));
        const int np = c->nPending;
        REQ(results == nullptr || max_passes >= np, SDFGI_ERR_INVALID, "results: one per pass in flight");
        REQ(reports == nullptr || max_passes >= np, SDFGI_ERR_INVALID, "reports: one row per pass in flight");
        for (int k = 0; k < np; ++k) {
            const unsigned long long* host = c->hAsync + k * kAsyncHostWords;
            if (results) {
                double md;
                std::memcpy(&md, &host[0], 8);
                results[k].max_texel_delta = md;
                results[k].rays_traced = static_cast<int64_t>(host[1]);
                results[k].probes_updated = static_cast<int64_t>(host[2] & 0xffffffffull);
            }
            if (reports) {
                const int* r = reinterpret_cast<const int*>(host + 3);
                for (int s = 0; s < reports_per_pass; ++s) {
                    if (s < c->pendingCascades[k])
                        fillReport(&reports[static_cast<size_t>(k) * reports_per_pass + s], r + 4 * s);
                    else
                        std::memset(&reports[static_cast<size_t>(k) * reports_per_pass + s], 0, sizeof(sdfgi_reloc_report));
                }
            }
            if (c->pendingTimed[k]) {
                const cudaEvent_t* e = c->kevAsync[k];
                for (int i = 0; i + 1 < kWaveEvents; ++i) {
                    float ms = 0.f;
                    CK(cudaEventElapsedTime(&ms, e[i], e[i + 1]));
                    c->stageSum[i] += ms;
                }
                float tot = 0.f;
                CK(cudaEventElapsedTime(&tot, e[0], e[kWaveEvents - 1]));
                c->stageSum[kWaveEvents - 1] += tot;
            }
        }
        c->nPending = 0;
        *n_passes = np;
    });
}

int sdfgi_atlas_swap(void* ctx) {
    return guard([&] {
        Ctx* c = C(ctx);
        c->front = 1 - c->front;
    });
}

int sdfgi_atlas_download(void* ctx, int level, int which, float* dst, size_t n_floats) {
    return guard([&] {
        Ctx* c = C(ctx);
        int s = c->slot(level);
        REQ(which == 0 || which == 1, SDFGI_ERR_INVALID, "which must be 0 or 1");
        size_t n = c->tileFloats() * c->cascades[s].count();
        REQ(dst && n_floats == n, SDFGI_ERR_INVALID, "atlas size mismatch");
        const float* src = c->atlas[which == 0 ? c->front : 1 - c->front].p + c->tileFloats() * c->cascades[s].base;
        CK(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_atlas_upload(void* ctx, int level, int which, const float* src, size_t n_floats) {
    return guard([&] {
        Ctx* c = C(ctx);
        int s = c->slot(level);
        REQ(which == 0 || which == 1, SDFGI_ERR_INVALID, "which must be 0 or 1");
        size_t n = c->tileFloats() * c->cascades[s].count();
        REQ(src && n_floats == n, SDFGI_ERR_INVALID, "atlas size mismatch");
        float* dst = c->atlas[which == 0 ? c->front : 1 - c->front].p + c->tileFloats() * c->cascades[s].base;
        c->atlasZero[which == 0 ? c->front : 1 - c->front][s] = 0;
        CK(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_atlas_device_ptr(void* ctx, int level, int which, void** out_ptr, size_t* out_bytes) {
    return guard([&] {
        Ctx* c = C(ctx);
        int s = c->slot(level);
        REQ(which == 0 || which == 1, SDFGI_ERR_INVALID, "which must be 0 or 1");
        REQ(out_ptr && out_bytes, SDFGI_ERR_INVALID, "null out");
        *out_ptr = c->atlas[which == 0 ? c->front : 1 - c->front].p + c->tileFloats() * c->cascades[s].base;
        c->atlasZero[which == 0 ? c->front : 1 - c->front][s] = 0;  // the caller may write through it
        *out_bytes = c->tileFloats() * c->cascades[s].count() * 4;
    });
}

int sdfgi_probes_trace_debug(void* ctx, const int32_t* probe_refs, int n_refs, int frame, const sdfgi_cfg* cfg,
                             sdfgi_ray_record* out, int n_records_max, int* n_written) {
    return guard([&] {
        Ctx* c = C(ctx);
        requireProbes(c);
        validateCfg(c, cfg);
        REQ(probe_refs && n_refs > 0 && out && n_written, SDFGI_ERR_INVALID, "bad debug arguments");
        std::vector<int> g;
        for (int i = 0; i < n_refs; ++i) {
            int s = c->slot(probe_refs[2 * i]);
            REQ(probe_refs[2 * i + 1] >= 0 && probe_refs[2 * i + 1] < c->cascades[s].count(), SDFGI_ERR_INVALID,
                "probe index out of range");
            g.push_back(c->cascades[s].base + probe_refs[2 * i + 1]);
        }
        const size_t cap = static_cast<size_t>(n_refs) * 2 * static_cast<size_t>(cfg->n_rays_full);
        upload(c, c->refs, g.data(), g.size());
        uploadQuats(c, cfg, frame, g.data(), n_refs);
        reserve(c->records, cap);
        // the same K0..K3 wavefront in debug mode: per-ray records, no atlas/state writes
        if (c->precision == SDFGI_F64) {
            WaveParams<double> p = waveParams<double>(c, cfg, frame, c->refs.p, n_refs);
            p.records = c->records.p;
            p.debug = 1;
            p.escape = 0;  // per-ray records: the exact march (miss reason, steps)
            p.settle = 0;
            p.useClear = 0;
            launch_wavefront<double>(p, c->persistCap, false, c->stream, nullptr, &c->launches);
        } else {
            WaveParams<float> p = waveParams<float>(c, cfg, frame, c->refs.p, n_refs);
            p.records = c->records.p;
            p.debug = 1;
            p.escape = 0;
            p.settle = 0;
            launch_wavefront<float>(p, c->persistCap, false, c->stream, nullptr, &c->launches);
        }
        CK(cudaGetLastError());
        quatsConsumed(c);
        long long total = 0;
        CK(cudaMemcpyAsync(&total, c->wRayStart.p + n_refs, sizeof(total), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        REQ(total <= n_records_max, SDFGI_ERR_INVALID, "n_records_max too small");
        CK(cudaMemcpyAsync(out, c->records.p, total * sizeof(RayRecord), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *n_written = total;
    });
}

int sdfgi_query_points(void* ctx, const double* points_xyz, const double* init_d, int n, double* out_d,
                       int32_t* out_owner) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(n >= 0 && (n == 0 || (points_xyz && out_d && out_owner)), SDFGI_ERR_INVALID, "bad query arguments");
        if (n == 0) return;
        upload(c, c->qpts, points_xyz, 3 * static_cast<size_t>(n));
        if (init_d) upload(c, c->qinit, init_d, n);
        c->qd.alloc(n);
        c->qowner.alloc(n);
        QueryParams p;
        p.scene = c->sceneView<double>();
        p.pts = c->qpts.p;
        p.init = init_d ? c->qinit.p : nullptr;
        p.outD = c->qd.p;
        p.outOwner = c->qowner.p;
        p.n = n;
        launch_query_points(p, c->stream);
        checkLaunch(c);
        CK(cudaMemcpyAsync(out_d, c->qd.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(out_owner, c->qowner.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_last_kernel_ms(void* ctx, double* update_ms, double* relocate_ms) {
    return guard([&] {
        Ctx* c = C(ctx);
        CK(cudaStreamSynchronize(c->stream));
        float a = 0.f, b = 0.f;
        if (c->evUpdate) CK(cudaEventElapsedTime(&a, c->kev[0], c->kev[kWaveEvents - 1]));
        if (c->evReloc) CK(cudaEventElapsedTime(&b, c->ev[2], c->ev[3]));
        if (update_ms) *update_ms = a;
        if (relocate_ms) *relocate_ms = b;
    });
}

int sdfgi_last_stage_ms(void* ctx, double out[7]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        REQ(c->evUpdate, SDFGI_ERR_STATE, "no update timed yet");
        CK(cudaStreamSynchronize(c->stream));
        for (int i = 0; i + 1 < kWaveEvents; ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c->kev[i], c->kev[i + 1]));
            out[i] = ms;
        }
    });
}

int sdfgi_stage_ms_sum(void* ctx, double out[8], int reset) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        for (int i = 0; i < kWaveEvents; ++i) out[i] = c->stageSum[i];
        if (reset)
            for (double& v : c->stageSum) v = 0.0;
    });
}

int sdfgi_last_trace_counters(void* ctx, uint64_t out[28]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < 14; ++i) out[14 * k + i] = c->lastTrace[k][i];
    });
}

int sdfgi_last_shading_work(void* ctx, uint64_t out[2]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        out[0] = c->shadeWork[0];
        out[1] = c->shadeWork[1];
    });
}

int sdfgi_last_work(void* ctx, uint64_t out[6]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        for (int i = 0; i < 6; ++i) out[i] = c->lastWork[i];
    });
}

int sdfgi_measure_fp_peak(void* ctx, double* f64_fma_per_s, double* f32_fma_per_s) {
    return guard([&] {
        Ctx* c = C(ctx);
        if (f64_fma_per_s) *f64_fma_per_s = measure_fma_rate(true, c->stream);
        if (f32_fma_per_s) *f32_fma_per_s = measure_fma_rate(false, c->stream);
        CK(cudaGetLastError());
    });
}

int sdfgi_set_accel(void* ctx, int mode) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(mode >= 0 && mode <= 2, SDFGI_ERR_INVALID, "accel mode must be 0, 1 or 2");
        c->accel = mode;
    });
}

int sdfgi_accel_info(void* ctx, int64_t out[6]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        out[0] = c->accel;
        out[1] = c->haveGrid ? 1 : 0;
        out[2] = c->grid.dim[0];
        out[3] = c->grid.dim[1];
        out[4] = c->grid.dim[2];
        out[5] = c->gridEntries;
    });
}

}  // extern "C"

namespace {

CameraDev toCam(const sdfgi_camera& c) {
    CameraDev d;
    for (int k = 0; k < 3; ++k) {
        d.pos[k] = c.position[k];
        d.fwd[k] = c.forward[k];
        d.right[k] = c.right[k];
        d.up[k] = c.up[k];
    }
    d.fov = c.fov_y_deg;
    d.tanHalf = sdfgi_host::tanHalf(c.fov_y_deg);  // host libm (camera.hpp:30,42)
    return d;
}

void ensureGather(Ctx* c, int w, int h) {
    REQ(w > 0 && h > 0 && static_cast<long long>(w) * h < (1LL << 28), SDFGI_ERR_INVALID, "bad G-buffer size");
    if (w != c->gw || h != c->gh) c->histValid = 0;
    c->gw = w;
    c->gh = h;
    const size_t np = static_cast<size_t>(w) * h;
    const int hw = (w + 1) / 2, hh = (h + 1) / 2, sw = (hw + 1) / 2, sh = (hh + 1) / 2;
    c->gbuf.alloc(np);
    c->halfDepth.alloc(static_cast<size_t>(hw) * hh);
    c->halfSrc.alloc(static_cast<size_t>(hw) * hh);
    c->sel.alloc(static_cast<size_t>(sw) * sh);
    c->sparseIrr.alloc(3 * static_cast<size_t>(sw) * sh);
    c->sparseValid.alloc(static_cast<size_t>(sw) * sh);
    c->sparseAnchor.alloc(static_cast<size_t>(sw) * sh);
    c->resolved.alloc(3 * np);
    c->indirect.alloc(3 * np);
    c->composed.alloc(3 * np);
    c->histIrr.alloc(3 * np);
    c->histDepth.alloc(np);
    for (auto& e : c->gev)
        if (!e) CK(cudaEventCreate(&e));
}

// Wavefront parameters for the Contact GI batch: every (pixel, sample) ray of the
// current G-buffer; reuses the probe wavefront's scratch buffers.
template <typename R>
WaveParams<R> contactParams(Ctx* c, const sdfgi_cfg* cfg) {
    const long long nr = static_cast<long long>(c->gw) * c->gh * std::max<long long>(cfg->contact_samples, 0);
    const size_t cap = static_cast<size_t>(std::max<long long>(nr, 1));
    const int L = std::max(c->nLights, 1);
    reserve(c->wHits, cap * sizeof(HitRec<R>));
    reserve(c->wHitList, cap);
    reserve(c->wMvcList, cap);
    reserve(c->wTriList, cap);
    reserve(c->wVis, cap * L * sizeof(R));
    reserve(c->wRad, cap * 3 * sizeof(R));
    reserve(c->wCtr, kLightCtr + L);
    reservePark<R>(c, cap, L);
    reserve(c->wSRay, cap * L * sizeof(ShadowRay<R>));
    reserve(c->wCRay, cap * sizeof(ContactRay<R>));
    reserve(c->wConv, cap);
    const int S = static_cast<int>(std::max<long long>(cfg->contact_samples, 0));
    if (nr > 0 && (c->cLocalS != S || c->cLocalW != c->gw || c->cLocalH != c->gh || c->cLocalSeed != cfg->seed)) {
        // frame-invariant: built once per (seed, resolution, sample count)
        std::vector<double> tab(2 * static_cast<size_t>(nr));
        sdfgi_host::contactLocal(cfg->seed, c->gw, c->gh, S, tab.data());
        c->cLocal.alloc(tab.size());
        CK(cudaMemcpyAsync(c->cLocal.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // tab is a local
        c->cLocalS = S;
        c->cLocalW = c->gw;
        c->cLocalH = c->gh;
        c->cLocalSeed = cfg->seed;
    }
    WaveParams<R> p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<R>();
    p.pc = c->probeCommon();
    p.tc.eps = cfg->surface_epsilon;
    p.tc.rayTMax = cfg->ray_tmax;
    p.tc.shadowK = cfg->shadow_k;
    p.tc.bounceCoeff = cfg->bounce_coeff;
    p.tc.mvcFrac = cfg->mvc_relocation_frac;
    p.tc.maxSteps = static_cast<int>(cfg->max_trace_steps);
    p.tc.shadowSteps = static_cast<int>(cfg->shadow_steps);
    p.prevAtlas = c->atlas[c->front].p;
    p.oct = c->octRes;
    p.seed = cfg->seed;
    p.hits = reinterpret_cast<HitRec<R>*>(c->wHits.p);
    p.hitList = c->wHitList.p;
    p.mvcList = c->wMvcList.p;
    p.triList = c->wTriList.p;
    p.vis = reinterpret_cast<R*>(c->wVis.p);
    p.rad = reinterpret_cast<R*>(c->wRad.p);
    p.ctr = c->wCtr.p;
    p.sray = reinterpret_cast<ShadowRay<R>*>(c->wSRay.p);
    reserveHitAt<R>(c, p, cap);
    p.srayCap = cap;
    p.park = c->accel && c->haveGrid && c->wPark.n >= 4096 ? c->wPark.p : nullptr;  // SDFGI_PARK_MB=0: off
    p.parkBytes = p.park ? c->wPark.n : 0;
    p.stats = c->scratch.p + 32;  // contact counters: scratch[32..], the visibility ones stay at [0..]
    // short rays: neither the escape test nor the shared-memory primitive copy pays
    // off here (measured: contact +2.5% / +3% each, scripts/time_gather.py)
    p.escape = 0;
    {
        const char* e = std::getenv("SDFGI_CONTACT_SETTLE");
        p.settle = (!e || std::atoi(e) != 0) ? escapeOk(c) : 0;
    }
    p.scene.stageBytes = 0;
    p.ownerFromMarch = c->accel == 2 && c->haveGrid ? 1 : 0;  // exact (see waveParams)
    p.nRaysDirect = nr;
    p.cray = c->wCRay.p;
    p.conv = c->wConv.p;
    p.clocal = c->cLocal.p;
    p.gb = c->gbuf.p;
    p.gw = c->gw;
    p.gh = c->gh;
    p.contactSamples = static_cast<int>(cfg->contact_samples);
    double sp0 = 1.0;
    if (!c->cascades.empty()) sp0 = c->cascades[0].spacing / std::pow(2.0, c->cascades[0].level);
    p.contactRadius = cfg->contact_radius_frac * sp0;  // pipeline.hpp:200
    p.resolved = c->resolved.p;
    p.indirect = c->indirect.p;
    return p;
}

// Wavefront parameters for composeFrame: one shadow-ray item per (geometry pixel,
// light); hits/vis indexed by pixel.
template <typename R>
WaveParams<R> composeParams(Ctx* c, const sdfgi_cfg* cfg) {
    const size_t np = static_cast<size_t>(c->gw) * c->gh;
    const int L = std::max(c->nLights, 1);
    reserve(c->wHits, np * sizeof(HitRec<R>));
    reserve(c->wHitList, np);
    reserve(c->wVis, np * L * sizeof(R));
    reserve(c->wCtr, kLightCtr + L);
    reservePark<R>(c, np, L);
    reserve(c->wSRay, std::max<size_t>(np, 1) * L * sizeof(ShadowRay<R>));
    WaveParams<R> p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<R>();
    p.pc = c->probeCommon();
    p.tc.eps = cfg->surface_epsilon;
    p.tc.rayTMax = cfg->ray_tmax;
    p.tc.shadowK = cfg->shadow_k;
    p.tc.shadowSteps = static_cast<int>(cfg->shadow_steps);
    p.hits = reinterpret_cast<HitRec<R>*>(c->wHits.p);
    p.hitList = c->wHitList.p;
    p.vis = reinterpret_cast<R*>(c->wVis.p);
    p.ctr = c->wCtr.p;
    p.sray = reinterpret_cast<ShadowRay<R>*>(c->wSRay.p);
    p.srayCap = std::max<size_t>(np, 1);
    p.park = c->accel && c->haveGrid && c->wPark.n >= 4096 ? c->wPark.p : nullptr;
    p.parkBytes = p.park ? c->wPark.n : 0;
    p.stats = c->scratch.p;
    p.nRaysDirect = static_cast<long long>(np);
    p.gb = c->gbuf.p;
    p.gw = c->gw;
    p.gh = c->gh;
    p.resolved = c->indirect.p;  // input: the indirect image
    p.composed = c->composed.p;
    p.scene.stageBytes = 0;  // measured slower for the compose shadow rays (+2%)
    return p;
}

template <typename R>
GatherParams<R> gatherParams(Ctx* c, const sdfgi_cfg* cfg, int frame) {
    GatherParams<R> p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<R>();
    p.pc = c->probeCommon();
    p.tc.eps = cfg->surface_epsilon;
    p.tc.rayTMax = cfg->ray_tmax;
    p.tc.shadowK = cfg->shadow_k;
    p.tc.bounceCoeff = cfg->bounce_coeff;
    p.tc.mvcFrac = cfg->mvc_relocation_frac;
    p.tc.maxSteps = static_cast<int>(cfg->max_trace_steps);
    p.tc.shadowSteps = static_cast<int>(cfg->shadow_steps);
    p.atlas = c->cascades.empty() ? nullptr : c->atlas[c->front].p;
    p.oct = c->octRes;
    p.w = c->gw;
    p.h = c->gh;
    p.hw = (p.w + 1) / 2;
    p.hh = (p.h + 1) / 2;
    p.sw = (p.hw + 1) / 2;
    p.sh = (p.hh + 1) / 2;
    p.frame = frame;
    p.gb = c->gbuf.p;
    p.halfDepth = c->halfDepth.p;
    p.halfSrc = c->halfSrc.p;
    p.sel = c->sel.p;
    p.sparseIrr = c->sparseIrr.p;
    p.sparseValid = c->sparseValid.p;
    p.sparseAnchor = c->sparseAnchor.p;
    p.resolved = c->resolved.p;
    p.indirect = c->indirect.p;
    p.histIrr = c->histIrr.p;
    p.histDepth = c->histDepth.p;
    p.histValid = c->histValid;
    p.dedupFrac = cfg->dedup_quant_frac;
    p.th1Frac = cfg->threshold1_frac;
    p.visK = cfg->probe_visibility_k;
    p.depthSigmaFrac = cfg->depth_sigma_frac;
    p.historyBlend = cfg->history_blend;
    // contactRadiusFrac * cascade-0 spacing (pipeline.hpp:200)
    double sp0 = 1.0;
    if (!c->cascades.empty()) sp0 = c->cascades[0].spacing / std::pow(2.0, c->cascades[0].level);
    p.contactRadius = cfg->contact_radius_frac * sp0;
    p.contactSamples = static_cast<int>(cfg->contact_samples);
    p.seed = cfg->seed;
    // visibility counters at scratch[0..13] (contact: [32..], contactParams)
    p.visStats = c->scratch.p;
    p.contactStats = c->scratch.p + 32;
    p.taskCount = c->scratch.p + 19;
    return p;
}

}  // namespace

extern "C" {

int sdfgi_gbuffer_upload(void* ctx, int w, int h, const sdfgi_gbuffer_pixel* px) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(px, SDFGI_ERR_INVALID, "null pixels");
        ensureGather(c, w, h);
        static_assert(sizeof(GPix) == sizeof(sdfgi_gbuffer_pixel), "gbuffer mirror");
        CK(cudaMemcpyAsync(c->gbuf.p, px, sizeof(GPix) * static_cast<size_t>(w) * h, cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_gbuffer_render(void* ctx, const sdfgi_camera* cam, const sdfgi_camera* prev_cam, int w, int h,
                         const sdfgi_cfg* cfg) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(cam && cfg, SDFGI_ERR_INVALID, "null camera/cfg");
        ensureGather(c, w, h);
        if (c->precision == SDFGI_F64) {
            GatherParams<double> p = gatherParams<double>(c, cfg, 0);
            p.cam = toCam(*cam);
            p.prevCam = toCam(prev_cam ? *prev_cam : *cam);
            launch_gather<double>(p, 0, false, c->stream);
        } else {
            GatherParams<float> p = gatherParams<float>(c, cfg, 0);
            p.cam = toCam(*cam);
            p.prevCam = toCam(prev_cam ? *prev_cam : *cam);
            launch_gather<float>(p, 0, false, c->stream);
        }
        checkLaunch(c);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_gbuffer_download(void* ctx, sdfgi_gbuffer_pixel* out, size_t n_pixels) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out && n_pixels == static_cast<size_t>(c->gw) * c->gh && n_pixels > 0, SDFGI_ERR_INVALID,
            "G-buffer size mismatch");
        CK(cudaMemcpyAsync(out, c->gbuf.p, sizeof(GPix) * n_pixels, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_gather(void* ctx, int frame, const sdfgi_cfg* cfg, int64_t* n_tasks, sdfgi_stats* vis_stats,
                 sdfgi_stats* contact_stats) {
    return guard([&] {
        Ctx* c = C(ctx);
        requireProbes(c);
        REQ(cfg, SDFGI_ERR_INVALID, "null cfg");
        REQ(c->gw > 0 && c->gbuf.p, SDFGI_ERR_STATE, "no G-buffer (upload or render one first)");
        REQ(cfg->oct_res == c->octRes, SDFGI_ERR_INVALID, "cfg.oct_res differs from the atlas resolution");
        const bool st = vis_stats != nullptr || contact_stats != nullptr;
        CK(cudaMemsetAsync(c->scratch.p, 0, 64 * 8, c->stream));
        CK(cudaEventRecord(c->gev[0], c->stream));
        auto run = [&](auto p) {
            launch_gather(p, 1, st, c->stream);  // downsample + select
            CK(cudaEventRecord(c->gev[1], c->stream));
            launch_gather(p, 2, st, c->stream);  // tiles: tasks + visibility + shadePixelGI
            CK(cudaEventRecord(c->gev[2], c->stream));
            launch_gather(p, 3, st, c->stream);  // upsample + temporal resolve
            CK(cudaEventRecord(c->gev[3], c->stream));
            return p;
        };
        // Contact GI (shading.hpp:431-477) as a wavefront over (pixel, sample) rays; its
        // counters live at scratch[32..], so no host round trip between the stages
        if (c->precision == SDFGI_F64) {
            run(gatherParams<double>(c, cfg, frame));
            launch_contact<double>(contactParams<double>(c, cfg), st, c->stream, &c->launches);
        } else {
            run(gatherParams<float>(c, cfg, frame));
            launch_contact<float>(contactParams<float>(c, cfg), st, c->stream, &c->launches);
        }
        c->launches += 4;
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->gev[4], c->stream));
        c->gevValid = true;
        unsigned long long visH[64];
        CK(cudaMemcpyAsync(visH, c->scratch.p, sizeof(visH), cudaMemcpyDeviceToHost, c->stream));
        const unsigned long long* conH = visH + 32;
        // roll history (pipeline.hpp:213-218): resolved E and this frame's depth
        const size_t np = static_cast<size_t>(c->gw) * c->gh;
        CK(cudaMemcpyAsync(c->histIrr.p, c->resolved.p, 3 * np * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpy2DAsync(c->histDepth.p, sizeof(double), c->gbuf.p, sizeof(GPix), sizeof(double), np,
                             cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->histValid = 1;
        auto fill = [](sdfgi_stats* s, const unsigned long long* h) {
            if (!s) return;
            s->sdf_queries += h[0];
            s->clusters_visited += h[1];
            s->clusters_skipped += h[2];
            s->primitive_evals += h[3];
            s->trace_steps += h[4];
            s->sphere_traces += h[5];
            s->shadow_traces += h[6];
            s->visibility_traces += h[7];
        };
        fill(vis_stats, visH);
        fill(contact_stats, conH);
        if (n_tasks) *n_tasks = static_cast<int64_t>(visH[19]);
    });
}

int sdfgi_gather_reset_history(void* ctx) {
    return guard([&] {
        Ctx* c = C(ctx);
        c->histValid = 0;
    });
}

int sdfgi_gather_download(void* ctx, int which, void* dst, size_t bytes) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(dst, SDFGI_ERR_INVALID, "null dst");
        const void* src = nullptr;
        size_t n = 0;
        switch (which) {
            case 0: src = c->resolved.p; n = c->resolved.n * 8; break;
            case 1: src = c->indirect.p; n = c->indirect.n * 8; break;
            case 2: src = c->halfDepth.p; n = c->halfDepth.n * 8; break;
            case 3: src = c->halfSrc.p; n = c->halfSrc.n * 4; break;
            case 4: src = c->sel.p; n = c->sel.n * 4; break;
            case 5: src = c->sparseIrr.p; n = c->sparseIrr.n * 8; break;
            case 6: src = c->sparseValid.p; n = c->sparseValid.n * 4; break;
            case 7: src = c->sparseAnchor.p; n = c->sparseAnchor.n * 4; break;
            case 8: src = c->composed.p; n = c->composed.n * 8; break;
            default: throw Error(SDFGI_ERR_INVALID, "unknown gather buffer");
        }
        REQ(src && bytes == n, SDFGI_ERR_INVALID, "gather buffer size mismatch");
        CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_indirect_upload(void* ctx, const double* rgb, size_t n_doubles) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(rgb, SDFGI_ERR_INVALID, "null image");
        REQ(c->gw > 0 && n_doubles == 3 * static_cast<size_t>(c->gw) * c->gh, SDFGI_ERR_INVALID,
            "indirect image size mismatch (3 doubles per G-buffer pixel)");
        CK(cudaMemcpyAsync(c->indirect.p, rgb, n_doubles * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sdfgi_compose(void* ctx, const sdfgi_cfg* cfg, sdfgi_stats* stats, double* ms) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(cfg, SDFGI_ERR_INVALID, "null cfg");
        REQ(c->gw > 0 && c->gbuf.p, SDFGI_ERR_STATE, "no G-buffer (upload or render one first)");
        const bool st = stats != nullptr;
        CK(cudaMemsetAsync(c->scratch.p, 0, 32 * 8, c->stream));
        for (auto& e : c->cev)
            if (!e) CK(cudaEventCreate(&e));
        CK(cudaEventRecord(c->cev[0], c->stream));
        // settled shadows (exact) only without stats: the stats run keeps the
        // reference's query sequence, whose counts the parity tests compare
        const char* se = std::getenv("SDFGI_COMPOSE_SETTLE");
        const int settle = (!st && (!se || std::atoi(se) != 0)) ? escapeOk(c) : 0;
        if (c->precision == SDFGI_F64) {
            WaveParams<double> p = composeParams<double>(c, cfg);
            p.settle = settle;
            launch_compose<double>(p, st, c->stream, &c->launches);
        } else {
            WaveParams<float> p = composeParams<float>(c, cfg);
            p.settle = settle;
            launch_compose<float>(p, st, c->stream, &c->launches);
        }
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->cev[1], c->stream));
        unsigned long long h[32];
        CK(cudaMemcpyAsync(h, c->scratch.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (ms) {
            float e = 0;
            CK(cudaEventElapsedTime(&e, c->cev[0], c->cev[1]));
            *ms = e;
        }
        if (stats) {
            stats->sdf_queries += h[0];
            stats->clusters_visited += h[1];
            stats->clusters_skipped += h[2];
            stats->primitive_evals += h[3];
            stats->trace_steps += h[4];
            stats->sphere_traces += h[5];
            stats->shadow_traces += h[6];
            stats->visibility_traces += h[7];
        }
    });
}

int sdfgi_last_gather_ms(void* ctx, double out[4]) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out && c->gevValid, SDFGI_ERR_STATE, "no gather timed yet");
        CK(cudaStreamSynchronize(c->stream));
        for (int i = 0; i < 4; ++i) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, c->gev[i], c->gev[i + 1]));
            out[i] = ms;
        }
    });
}

int sdfgi_build_clusters(const sdfgi_prim* prims, int n, int max_per_cluster, sdfgi_cluster* out_clusters,
                         int* out_n_clusters, int32_t* member_start, int32_t* member_idx) {
    return guard([&] {
        REQ(n >= 0 && (n == 0 || prims) && out_clusters && out_n_clusters && member_start && member_idx,
            SDFGI_ERR_INVALID, "bad cluster-build arguments");
        REQ(max_per_cluster >= 1, SDFGI_ERR_INVALID, "max_per_cluster must be >= 1");
        // conservative surface boxes (primitiveAabb, primitives.hpp:112-151); planes
        // become their own unbounded clusters (buildClusters never merges them)
        std::vector<std::array<double, 6>> box(n);
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        std::vector<int> bounded, planes;
        for (int i = 0; i < n; ++i) {
            REQ(prims[i].kind >= 0 && prims[i].kind <= 4, SDFGI_ERR_INVALID, "bad primitive kind");
            primAabb(prims[i], box[i].data());
            if (prims[i].kind == SDFGI_PLANE) {
                planes.push_back(i);
                continue;
            }
            bounded.push_back(i);
            for (int a = 0; a < 3; ++a) {
                const double cc = 0.5 * (box[i][a] + box[i][3 + a]);
                lo[a] = std::min(lo[a], cc);
                hi[a] = std::max(hi[a], cc);
            }
        }
        // Morton order of the box centres, then runs of max_per_cluster
        auto spread10 = [](uint32_t x) {
            x &= 0x3ff;
            x = (x | (x << 16)) & 0x030000ff;
            x = (x | (x << 8)) & 0x0300f00f;
            x = (x | (x << 4)) & 0x030c30c3;
            x = (x | (x << 2)) & 0x09249249;
            return x;
        };
        std::vector<std::pair<uint32_t, int>> order;
        order.reserve(bounded.size());
        for (int i : bounded) {
            uint32_t code = 0;
            for (int a = 0; a < 3; ++a) {
                const double cc = 0.5 * (box[i][a] + box[i][3 + a]);
                const double ext = hi[a] - lo[a];
                const double u = ext > 0 ? std::min(1.0, std::max(0.0, (cc - lo[a]) / ext)) : 0.0;
                code |= spread10(static_cast<uint32_t>(u * 1023.0)) << a;
            }
            order.push_back({code, i});
        }
        std::sort(order.begin(), order.end());
        int k = 0, m = 0;
        member_start[0] = 0;
        auto emit = [&](const int* mem, int cnt, bool unbounded) {
            sdfgi_cluster& c = out_clusters[k];
            std::memset(&c, 0, sizeof(c));
            for (int a = 0; a < 3; ++a) {
                c.lo[a] = INFINITY;
                c.hi[a] = -INFINITY;
            }
            for (int t = 0; t < cnt; ++t) {
                member_idx[m++] = mem[t];
                for (int a = 0; a < 3; ++a) {
                    c.lo[a] = std::min(c.lo[a], box[mem[t]][a]);
                    c.hi[a] = std::max(c.hi[a], box[mem[t]][3 + a]);
                }
            }
            for (int a = 0; a < 3; ++a) {  // cullAabb = aabb.inflated(kClusterCullMargin), scene.hpp:165
                c.lo[a] -= 1e-9;
                c.hi[a] += 1e-9;
            }
            c.unbounded = unbounded ? 1 : 0;
            member_start[++k] = m;
        };
        std::vector<int> run;
        for (size_t t = 0; t < order.size(); t += max_per_cluster) {
            run.clear();
            for (size_t u = t; u < std::min(order.size(), t + max_per_cluster); ++u) run.push_back(order[u].second);
            emit(run.data(), static_cast<int>(run.size()), false);
        }
        for (int p : planes) emit(&p, 1, true);
        *out_n_clusters = k;
    });
}

int sdfgi_slab_range(int res_x, int res_y, int res_z, int rank, int world, int* lo, int* hi) {
    return guard([&] {
        REQ(res_x > 0 && res_y > 0 && res_z > 0 && world >= 1 && rank >= 0 && rank < world && lo && hi,
            SDFGI_ERR_INVALID, "bad slab arguments");
        CascadeHost c;
        c.res[0] = res_x;
        c.res[1] = res_y;
        c.res[2] = res_z;
        c.base = 0;
        slabRange(c, rank, world, lo, hi);
    });
}

}  // extern "C"

namespace {

// Wavefront parameters for a batch of n caller-given items (sdfgi_trace_rays,
// sdfgi_soft_shadow, sdfgi_shade_hits): the probe wavefront's scratch buffers.
template <typename R>
WaveParams<R> batchParams(Ctx* c, size_t n) {
    const size_t cap = std::max<size_t>(n, 1);
    const int L = std::max(c->nLights, 1);
    reserve(c->wHits, cap * sizeof(HitRec<R>));
    reserve(c->wHitList, cap);
    reserve(c->wMvcList, cap);
    reserve(c->wTriList, cap);
    reserve(c->wVis, cap * L * sizeof(R));
    reserve(c->wRad, cap * 3 * sizeof(R));
    reserve(c->wCtr, kLightCtr + L);
    reservePark<R>(c, cap, L);
    reserve(c->wSRay, cap * L * sizeof(ShadowRay<R>));
    reserve(c->wCRay, cap * sizeof(ContactRay<R>));
    WaveParams<R> p;
    std::memset(&p, 0, sizeof(p));
    p.scene = c->sceneView<R>();
    p.pc = c->probeCommon();
    p.hits = reinterpret_cast<HitRec<R>*>(c->wHits.p);
    p.hitList = c->wHitList.p;
    p.mvcList = c->wMvcList.p;
    p.triList = c->wTriList.p;
    p.vis = reinterpret_cast<R*>(c->wVis.p);
    p.rad = reinterpret_cast<R*>(c->wRad.p);
    p.ctr = c->wCtr.p;
    p.sray = reinterpret_cast<ShadowRay<R>*>(c->wSRay.p);
    p.srayCap = cap;
    reserveHitAt<R>(c, p, cap);
    p.park = c->accel && c->haveGrid && c->wPark.n >= 4096 ? c->wPark.p : nullptr;
    p.parkBytes = p.park ? c->wPark.n : 0;
    p.stats = c->scratch.p;
    p.nRaysDirect = static_cast<long long>(n);
    p.cray = c->wCRay.p;
    p.prevAtlas = c->cascades.empty() ? nullptr : c->atlas[c->front].p;
    p.oct = c->octRes;
    return p;
}

void fillStats(sdfgi_stats* s, const unsigned long long* h) {
    if (!s) return;
    s->sdf_queries += h[0];
    s->clusters_visited += h[1];
    s->clusters_skipped += h[2];
    s->primitive_evals += h[3];
    s->trace_steps += h[4];
    s->sphere_traces += h[5];
    s->shadow_traces += h[6];
    s->visibility_traces += h[7];
}

template <typename R>
void traceRays(Ctx* c, const double* o, const double* d, int n, double tMax, double eps, int maxSteps, double sb,
               sdfgi_hit* out, bool st) {
    WaveParams<R> p = batchParams<R>(c, n);
    p.tc.eps = eps;
    p.tc.maxSteps = maxSteps;
    p.tc.rayTMax = tMax;
    p.keepAll = 1;  // every ray's result is returned
    std::vector<ContactRay<R>> rays(n);
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) {
            rays[i].o[k] = R(o[3 * i + k]);
            rays[i].dir[k] = R(d[3 * i + k]);
        }
        rays[i].tMax = R(tMax);
        rays[i].startBound = R(sb);
    }
    CK(cudaMemcpyAsync(p.cray, rays.data(), rays.size() * sizeof(ContactRay<R>), cudaMemcpyHostToDevice, c->stream));
    launch_batch<R>(p, 0, st, c->stream, &c->launches);
    CK(cudaGetLastError());
    std::vector<HitRec<R>> h(n);
    std::vector<int> orig(c->nPrims);
    CK(cudaMemcpyAsync(h.data(), p.hits, n * sizeof(HitRec<R>), cudaMemcpyDeviceToHost, c->stream));
    if (c->nPrims) CK(cudaMemcpyAsync(orig.data(), c->orig.p, c->nPrims * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < n; ++i) {
        sdfgi_hit& r = out[i];
        std::memset(&r, 0, sizeof(r));
        const bool conv = h[i].status & 1;
        r.converged = conv ? 1 : 0;
        r.miss = (h[i].status >> 1) & 3;
        r.t = conv ? double(h[i].t) : 0.0;
        r.prim_index = conv && h[i].owner >= 0 ? orig[h[i].owner] : -1;
        for (int k = 0; k < 3; ++k) {
            r.pos[k] = conv ? double(h[i].p[k]) : 0.0;
            r.normal[k] = k == 2 ? 1.0 : 0.0;
            if (r.prim_index >= 0) r.normal[k] = double(h[i].n[k]);
        }
    }
}

template <typename R>
void softShadow(Ctx* c, const double* o, const double* d, const double* t0, const double* t1, int n, double k,
                int maxSteps, double minStep, double* out, bool st) {
    WaveParams<R> p = batchParams<R>(c, n);
    const int L = std::max(c->nLights, 1);
    p.scene.n_lights = 1;  // one list of segments (list 0); vis[i * 1]
    p.tc.shadowK = k;
    p.tc.shadowSteps = maxSteps;
    p.tc.shadowMinStep = minStep;
    std::vector<ShadowRay<R>> rays(n);
    for (int i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            rays[i].o[a] = R(o[3 * i + a]);
            rays[i].dir[a] = R(d[3 * i + a]);
        }
        rays[i].t = R(t0[i]);
        rays[i].tEnd = R(t1[i]);
        rays[i].rid = i;
        rays[i].li = 0;
    }
    std::vector<unsigned long long> ctr(kLightCtr + L, 0);
    ctr[kLightCtr] = static_cast<unsigned long long>(n);
    CK(cudaMemcpyAsync(p.ctr, ctr.data(), ctr.size() * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(p.sray, rays.data(), rays.size() * sizeof(ShadowRay<R>), cudaMemcpyHostToDevice, c->stream));
    launch_batch<R>(p, 1, st, c->stream, &c->launches);
    CK(cudaGetLastError());
    std::vector<R> v(n);
    CK(cudaMemcpyAsync(v.data(), p.vis, n * sizeof(R), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < n; ++i) out[i] = double(v[i]);
}

template <typename R>
void shadeHits(Ctx* c, const sdfgi_hit* hits, int n, double bounce, const sdfgi_cfg* cfg, double* out, bool st) {
    WaveParams<R> p = batchParams<R>(c, n);
    const int L = std::max(c->nLights, 1);
    p.tc.eps = cfg->surface_epsilon;
    p.tc.rayTMax = cfg->ray_tmax;
    p.tc.shadowK = cfg->shadow_k;
    p.tc.bounceCoeff = bounce;
    p.tc.mvcFrac = cfg->mvc_relocation_frac;
    p.tc.maxSteps = static_cast<int>(cfg->max_trace_steps);
    p.tc.shadowSteps = static_cast<int>(cfg->shadow_steps);
    p.prevZero = c->frontZero() ? 1 : 0;
    // original primitive index -> CSR position
    std::vector<int> csr(c->hPrims.size(), -1);
    for (size_t j = 0; j < c->hMember.size(); ++j)
        if (csr[c->hMember[j]] < 0) csr[c->hMember[j]] = static_cast<int>(j);
    std::vector<HitRec<R>> h(n);
    std::vector<int> list;
    std::vector<R> rad(3 * static_cast<size_t>(n), R(0));
    for (int i = 0; i < n; ++i) {
        std::memset(&h[i], 0, sizeof(h[i]));
        const int pi = hits[i].prim_index;
        REQ(pi < static_cast<int>(csr.size()), SDFGI_ERR_INVALID, "hit prim_index out of range");
        h[i].owner = pi >= 0 ? csr[pi] : -1;
        h[i].status = 1;
        h[i].t = R(hits[i].t);
        for (int k = 0; k < 3; ++k) {
            h[i].p[k] = R(hits[i].pos[k]);
            h[i].n[k] = R(hits[i].normal[k]);
        }
        if (h[i].owner >= 0)
            list.push_back(i);
        else
            for (int k = 0; k < 3; ++k) rad[3 * i + k] = R(c->sky[k]);  // shadeHit's miss branch
    }
    std::vector<unsigned long long> ctr(kLightCtr + L, 0);
    ctr[kCtrHits] = list.size();
    CK(cudaMemcpyAsync(p.ctr, ctr.data(), ctr.size() * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(p.hits, h.data(), n * sizeof(HitRec<R>), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(p.rad, rad.data(), rad.size() * sizeof(R), cudaMemcpyHostToDevice, c->stream));
    if (!list.empty())
        CK(cudaMemcpyAsync(p.hitList, list.data(), list.size() * 4, cudaMemcpyHostToDevice, c->stream));
    launch_batch<R>(p, 2, st, c->stream, &c->launches);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(rad.data(), p.rad, rad.size() * sizeof(R), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < rad.size(); ++i) out[i] = double(rad[i]);
}

template <typename F>
void withStats(Ctx* c, sdfgi_stats* stats, F&& f) {
    CK(cudaMemsetAsync(c->scratch.p, 0, 64 * 8, c->stream));
    f();
    unsigned long long h[32];
    CK(cudaMemcpyAsync(h, c->scratch.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    fillStats(stats, h);
}

}  // namespace

extern "C" {

int sdfgi_trace_rays(void* ctx, const double* origins, const double* dirs, int n, double t_max,
                     double surface_epsilon, int max_steps, double start_bound, sdfgi_hit* out, sdfgi_stats* stats) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(n >= 0 && (n == 0 || (origins && dirs && out)), SDFGI_ERR_INVALID, "bad ray arguments");
        if (n == 0) return;
        withStats(c, stats, [&] {
            if (c->precision == SDFGI_F64)
                traceRays<double>(c, origins, dirs, n, t_max, surface_epsilon, max_steps, start_bound, out, stats);
            else
                traceRays<float>(c, origins, dirs, n, t_max, surface_epsilon, max_steps, start_bound, out, stats);
        });
    });
}

int sdfgi_soft_shadow(void* ctx, const double* origins, const double* dirs, const double* t_min,
                      const double* t_max, int n, double k, int max_steps, double min_step, double* out_vis,
                      sdfgi_stats* stats) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(n >= 0 && (n == 0 || (origins && dirs && t_min && t_max && out_vis)), SDFGI_ERR_INVALID,
            "bad shadow arguments");
        REQ(min_step > 0, SDFGI_ERR_INVALID, "min_step must be > 0");
        if (n == 0) return;
        withStats(c, stats, [&] {
            if (c->precision == SDFGI_F64)
                softShadow<double>(c, origins, dirs, t_min, t_max, n, k, max_steps, min_step, out_vis, stats);
            else
                softShadow<float>(c, origins, dirs, t_min, t_max, n, k, max_steps, min_step, out_vis, stats);
        });
    });
}

int sdfgi_shade_hits(void* ctx, const sdfgi_hit* hits, int n, double bounce_coeff, const sdfgi_cfg* cfg,
                     double* out_rgb, sdfgi_stats* stats) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(c->haveScene, SDFGI_ERR_STATE, "scene not uploaded");
        REQ(cfg, SDFGI_ERR_INVALID, "null cfg");
        REQ(n >= 0 && (n == 0 || (hits && out_rgb)), SDFGI_ERR_INVALID, "bad hit arguments");
        if (n == 0) return;
        withStats(c, stats, [&] {
            if (c->precision == SDFGI_F64)
                shadeHits<double>(c, hits, n, bounce_coeff, cfg, out_rgb, stats);
            else
                shadeHits<float>(c, hits, n, bounce_coeff, cfg, out_rgb, stats);
        });
    });
}

int sdfgi_convolve_irradiance(void* ctx, const double* sample_dirs, const double* sample_radiance, int n_samples,
                              const double* texel_dirs, int n_texels, double* out_rgb) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(n_samples >= 0 && n_texels >= 0, SDFGI_ERR_INVALID, "negative count");
        REQ(n_texels == 0 || (texel_dirs && out_rgb), SDFGI_ERR_INVALID, "null texel arguments");
        REQ(n_samples == 0 || (sample_dirs && sample_radiance), SDFGI_ERR_INVALID, "null sample arguments");
        if (n_texels == 0) return;
        if (n_samples == 0) {  // ConvolveResult{0, empty}
            std::fill(out_rgb, out_rgb + 3 * static_cast<size_t>(n_texels), 0.0);
            return;
        }
        DBuf<double> buf;
        const size_t ns = 3 * static_cast<size_t>(n_samples), nt = 3 * static_cast<size_t>(n_texels);
        buf.alloc(2 * ns + 2 * nt);
        CK(cudaMemcpyAsync(buf.p, sample_dirs, ns * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(buf.p + ns, sample_radiance, ns * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(buf.p + 2 * ns, texel_dirs, nt * 8, cudaMemcpyHostToDevice, c->stream));
        launch_convolve_batch(buf.p, buf.p + ns, n_samples, buf.p + 2 * ns, n_texels, buf.p + 2 * ns + nt, c->stream);
        checkLaunch(c);
        CK(cudaMemcpyAsync(out_rgb, buf.p + 2 * ns + nt, nt * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        buf.free();
    });
}

int sdfgi_interpolation_stencil(void* ctx, const double* points, int n, double mvc_relocation_frac,
                                sdfgi_stencil* out) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(n >= 0 && (n == 0 || (points && out)), SDFGI_ERR_INVALID, "bad stencil arguments");
        if (n == 0) return;
        DBuf<double> pts, w;
        DBuf<int> idx, meta;
        upload(c, pts, points, 3 * static_cast<size_t>(n));
        w.alloc(8 * static_cast<size_t>(n));
        idx.alloc(8 * static_cast<size_t>(n));
        meta.alloc(5 * static_cast<size_t>(n));
        launch_stencil_batch(c->probeCommon(), pts.p, n, mvc_relocation_frac, idx.p, w.p, meta.p, c->stream);
        checkLaunch(c);
        std::vector<double> hw(8 * static_cast<size_t>(n));
        std::vector<int> hi(8 * static_cast<size_t>(n)), hm(5 * static_cast<size_t>(n));
        CK(cudaMemcpyAsync(hw.data(), w.p, hw.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hi.data(), idx.p, hi.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hm.data(), meta.p, hm.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int i = 0; i < n; ++i) {
            sdfgi_stencil& s = out[i];
            std::memset(&s, 0, sizeof(s));
            const int slot = hm[5 * i];
            s.level = slot >= 0 ? c->cascades[slot].level : -1;
            s.count = hm[5 * i + 1];
            s.cross_cascade = hm[5 * i + 2];
            s.sky_fallback = hm[5 * i + 3];
            s.used_mvc = hm[5 * i + 4];
            for (int k = 0; k < 8; ++k) {
                s.index[k] = hi[8 * i + k];
                s.weight[k] = hw[8 * i + k];
            }
        }
        pts.free();
        w.free();
        idx.free();
        meta.free();
    });
}

int sdfgi_launch_count(void* ctx, int64_t* out) {
    return guard([&] {
        Ctx* c = C(ctx);
        REQ(out, SDFGI_ERR_INVALID, "null out");
        *out = c->launches;
    });
}

}  // extern "C"
