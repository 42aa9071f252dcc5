// kernels.cuh — the probe-stage kernels and their launch parameter blocks.
//
// Probe update (a)(b)(c) = updateProbe (probe_update.hpp:166-211) for a batch of
// probes, as a wavefront of four kernels so that the expensive part — SDF
// queries — runs with full SIMT lanes:
//   k_ray_setup      K0: per selected probe its ray count (2N on history reject,
//                    N, 0 when dead) and the per-probe rotation of sampleDirections
//                    (sampling.hpp:23-31); block prefix sums give every ray an id.
//   k_trace_primary  K1: persistent, self-refilling lanes. Every loop iteration is
//                    one SDF query for every active lane, stepping a per-lane state
//                    machine (march / polish) that reproduces sphereTrace
//                    (scene.hpp:391-435) exactly; idle lanes fetch the next ray id
//                    with one warp-aggregated atomic. Converged hits are compacted.
//   k_trace_shadow   K2: same scheme over (hit x light) items: the penumbra march of
//                    softShadowTrace (scene.hpp:459-476) set up as directIrradiance
//                    (probe_update.hpp:97-132) does.
//   k_shade_convolve K3: one CTA per probe: shadeHit (emission + shadowed direct +
//                    bounce from the previous atlas through the 8-probe stencil),
//                    radiance samples in shared memory, the cosine convolution of
//                    every texel in the reference's summation order, hysteresis
//                    blend, octahedral border fill, coalesced 16-byte tile stores.
// Relocation (d): k_relocate, one thread per probe, FP64 in every mode.
#pragma once

#include "sdf_device.cuh"

namespace sdfgi_dev {

struct ProbeCommon {
    CascadeDev cas[kMaxCascades];
    int nCas;
    ProbesView probes;
};

struct RelocParams {
    SceneView<double> scene;
    ProbeCommon pc;
    int cascade;          // slot
    double th1, th2;
    int maxSteps;
    double gradStep;
    int* report;          // relocated, rejected, dead
    unsigned long long* stats;  // counters or null
};

// Mirror of sdfgi_ray_record (include/sdfgi_b200.h).
struct RayRecord {
    double dir[3];
    double t;
    double radiance[3];
    double normal[3];
    int converged, miss, prim_index, steps;
};

// One primary-ray result (K1 -> K2, K3).
template <typename R> struct __align__(16) HitRec {
    R p[3];
    R n[3];
    R t;
    int owner;   // CSR position or -1
    int status;  // bit0 converged, bits1-2 MissReason, bits 8.. steps
};

// A march parked by K1 when its next point leaves the candidate grid; the far
// phase of K1 resumes it (state exactly as before the parked query).
template <typename R> struct __align__(16) ParkRay {
    R o[3], dir[3];
    R t, lastD, d, tMax;
    int step, state, pol, owner;
    unsigned long long rid;
    int seed;  // last known nearest primitive (query seed of the far phase)
    int item;  // the ray's position in the trace order (its hitAt slot)
};
// A probe ray prepared by k_probe_ray_setup: origin (the probe), direction and its
// ray id, in trace order.
template <typename R> struct __align__(16) ProbeRay {
    R o[3], dir[3];
    int rid;
    R clear;  // the probe's SDF (relocation's final query), < 0: not known
};
// A Contact GI ray prepared by k_contact_setup (tMax < 0: sky pixel, no ray).
template <typename R> struct __align__(16) ContactRay {
    R o[3], dir[3];
    R tMax, startBound;
};
// The same for a shadow march of K2.
template <typename R> struct __align__(16) ParkShadow {
    R o[3], dir[3];
    R t, tEnd, v, lastD;
    int step, seed;  // seed: last known nearest primitive
    unsigned long long slot;
};

// A shadow march prepared by the hit setup (k_hit_normals / k_compose_setup): the
// directIrradiance set-up of one (hit, light) pair whose segment is traced
// (probe_update.hpp:100-128), compacted per light.
template <typename R> struct __align__(16) ShadowRay {
    R o[3], dir[3];
    R t, tEnd;
    int rid, li;
};

template <typename R> struct WaveParams {
    SceneView<R> scene;
    ProbeCommon pc;
    TraceCfg tc;
    const float* prevAtlas;   // front (read) atlas, all cascades concatenated
    float* currAtlas;         // back (write) atlas
    int prevZero;             // the whole front atlas is zero: every bounce lookup adds exactly 0 (skipped)
    int oct;
    int frame;
    double hysteresis, alphaMin;
    int nRaysFull;
    uint64_t seed;
    int rotatePerFrame;
    // batch
    const int* cand;          // global probe ids of the batch (null: 0..nCand-1)
    int nCand;
    int* rayCount;            // per candidate (K0)
    long long* rayStart;      // nCand + 1 exclusive prefix (K0 scan)
    double* rot;              // 9 per candidate (K0, from quat)
    const double* quat;       // 4 per candidate: randomRotation's quaternion, host libm (host_trig.h)
    const double* fib;        // sphericalFibonacci table: n=N (N xyz) then n=2N (2N xyz), host libm
    const int* perm;          // coherent trace order of the sample indices: n=N then n=2N
    HitRec<R>* hits;          // per ray
    int* hitList;             // compacted ray ids of converged hits with an owner, in trace order
    int* hitAt;               // per trace-order item: its ray id if a lit hit, else -1 (compacted to hitList)
    int* mvcList;             // K3a -> K3c: ray ids of hits whose bounce lookup takes the MVC path
    void* selTemp;            // CUB temporary storage of the compaction
    size_t selTempBytes;
    long long maxItems;       // hitAt slots (the batch's upper bound of rays)
    R* vis;                   // per (ray, light)
    R* rad;                   // per ray: shaded radiance (3)
    // [kCtrRay] K1 ray cursor, [kCtrHits] hit count, [kCtrShadow] K2 item cursor,
    // [kCtrParkRay] rays parked by K1, [kCtrFarRay] K1 far-phase cursor,
    // [kCtrParkShadow] shadow marches parked by K2, [kCtrFarShadow] K2 far cursor,
    // [kLightCtr + li] traced shadow marches toward light li
    unsigned long long* ctr;
    // off-grid marches are parked here and resumed together by a far phase, so
    // the hierarchy walks run side by side instead of stalling near-field warps
    // (null: no parking). K1 and K2 reuse the buffer (K1's far phase ends first).
    void* park;
    unsigned long long parkBytes;
    void* cray;  // contact batch: the prepared rays (ContactRay<R>)
    unsigned char* conv;  // contact batch: per ray, 1 = converged (the combine's AO count)
    int keepAll;          // K1 writes every ray's HitRec (sdfgi_trace_rays reads them all)
    void* pray;  // probe batch: the prepared rays (ProbeRay<R>) in trace order
    // accel mode 2: every probe's SDF from the relocation that just ran (clear) is its
    // rays' first query, the same query at the same point (k_probe_ray_setup)
    int useClear;
    // K3a: hits whose bounce lookup takes the trilinear stencil, finished by K3c
    // before its MVC list (null: K3a looks them up itself)
    int* triList;
    // a march query that lands within eps with an exact result (an owner found below
    // its bound) already holds the owner query's answer at that point (same value,
    // same lowest-CSR-position tie-break): the polish starts without re-querying
    int ownerFromMarch;
    // accel mode 2: a march whose point leaves the candidate grid (which holds every
    // bounded primitive) after starting inside it can never converge again (the grid
    // box is convex, no unbounded primitive): K1 ends it as a miss on the spot
    int escape;
    // accel mode 2: K2's settled-shadow test (the same conditions as escape; the
    // Contact GI and compose wavefronts keep it while K1's escape is off there)
    int settle;
    const double* clocal;  // contact batch: cosineHemisphereDir's (lx, ly) per (pixel, sample), host libm
    // the traced shadow marches, light li's at [li * srayCap, + ctr[kLightCtr + li])
    ShadowRay<R>* sray;
    unsigned long long srayCap;
    // results
    unsigned long long* stats;       // counters or null
    unsigned long long* maxDeltaBits;
    unsigned long long* rays;
    unsigned int* updated;
    // debug: per-ray records instead of atlas/state writes
    RayRecord* records;
    int debug;
    // contact batch (Contact GI rays, shading.hpp:431-477); nRaysDirect < 0 = probe batch
    long long nRaysDirect;
    const struct GPix* gb;
    int gw, gh, contactSamples;
    double contactRadius;
    const double* resolved;   // contact batch: resolved irradiance; compose: the indirect image
    double* indirect;
    double* composed;         // compose: the final image (3 per pixel)
};

// Mirror of sdfgi_gbuffer_pixel (GBufferPixel, shading.hpp:13-22).
struct GPix {
    double depth;
    double normal[3];
    double albedo[3];
    double emission[3];
    double world_pos[3];
    double motion[2];
    int prim;
    int _pad;
};

// Mirror of sdfgi_camera (Camera, camera.hpp:9-49).
struct CameraDev {
    double pos[3], fwd[3], right[3], up[3];
    double fov;
    double tanHalf;  // std::tan(fov * pi / 360) on the host (camera.hpp:30,42; host_trig.h)
};

// Gather (e) launch parameters: shading.hpp:85-477 over one G-buffer.
template <typename R> struct GatherParams {
    SceneView<R> scene;
    ProbeCommon pc;
    TraceCfg tc;
    const float* atlas;  // front (previous) atlas, prevField of pipeline.hpp:127
    int oct;
    int w, h, hw, hh, sw, sh;
    int frame;
    CameraDev cam, prevCam;
    GPix* gb;
    double* halfDepth;
    int* halfSrc;
    int* sel;
    double* sparseIrr;
    int* sparseValid;
    int* sparseAnchor;
    double* resolved;
    double* indirect;
    const double* histIrr;
    const double* histDepth;
    int histValid;
    double dedupFrac, th1Frac, visK, depthSigmaFrac, historyBlend, contactRadius;
    int contactSamples;
    uint64_t seed;
    unsigned long long* visStats;
    unsigned long long* contactStats;
    unsigned long long* taskCount;
};

// selectProbesForUpdate on the device (select.cu).
struct SelectParams {
    ProbeCommon pc;
    int total, frame, forceAge;
    double camPos[3], camFwd[3];
    char* forced;
    char* other;
    int* ids;
    unsigned int* keyForced;
    unsigned long long* keyOther;
    int *idsF, *idsO, *idsF2, *idsO2;
    unsigned int *kF, *kF2;
    unsigned long long *kO, *kO2;
    int* counts;   // [0] forced, [1] others
    int* outRefs;  // 2 per selected probe: cascade level, index
    void* temp;
    size_t tempBytes;
};
size_t select_scratch_bytes(int total);
int launch_select(const SelectParams& P, int budget, cudaStream_t st, long long* launches);

struct QueryParams {
    SceneView<double> scene;
    const double* pts;
    const double* init;
    double* outD;
    int* outOwner;
    int n;
};

// Candidate-grid build (see GridDev in sdf_device.cuh), FP64.
struct GridBuildParams {
    SceneView<double> scene;  // useGrid = 0: exact flat walk
    double lo[3];
    double h;
    int dim[3];
    double pad;     // cell boxes are padded by this much on every side
    double margin;  // absolute slack on the bound
    const double* primBox;  // conservative AABB per CSR primitive (lo xyz, hi xyz; -inf/+inf unbounded)
    double* U;
    int* counts;
    const int* start;
    int2* entry;  // per entry: (float bits of the candidate's SDF lower bound over the cell, CSR position)
    int maxList;  // longer lists keep the nearest maxList + a sentinel (list = -1)
    // bricks of kBrick^3 cells: the clusters any of the brick's cells can list
    // (a superset of every cell's, ascending cluster order), so a cell scans its
    // brick's clusters instead of all of them
    int bdim[3];
    int* bSeed;   // per brick: the nearest primitive (CSR) at its centre, seeds the cells' bound queries
    int* bCounts;
    const int* bStart;
    int* bList;
};
constexpr int kBrick = 4;
// at most this many moving primitives are kept out of the grid (evaluated by every
// query) before the grid is rebuilt over all of them (SDFGI_DYNAMIC_MAX overrides)
constexpr int kMaxDynamic = 32;

// Launch the whole wavefront for one batch (K0..K3) on `st`. `persistBlocks` sizes
// the persistent K1/K2 grids; `ev` (optional, 2 events) brackets K1..K3.
template <typename R>
void launch_contact(const WaveParams<R>& p, bool stats, cudaStream_t st, long long* launches);
template <typename R>
void launch_compose(const WaveParams<R>& p, bool stats, cudaStream_t st, long long* launches);
// kind 0: sphereTrace rays (P.cray), 1: softShadowTrace rays (light list 0), 2: shadeHit of P.hitList
template <typename R>
void launch_batch(const WaveParams<R>& p, int kind, bool stats, cudaStream_t st, long long* launches);
// convolveIrradiance (probe_update.hpp:25-34) of one sample set for many texel directions
void launch_convolve_batch(const double* sdir, const double* srad, int ns, const double* tdir, int nt, double* out,
                           cudaStream_t st);
// interpolationStencil (probe_volume.hpp:224-310) of many points, FP64:
// per point 8 probe indices, 8 weights and (cascade slot, count, crossCascade, skyFallback, usedMvc)
void launch_stencil_batch(const ProbeCommon& pc, const double* pts, int n, double mvcFrac, int* idx, double* w,
                          int* meta, cudaStream_t st);
// ev (optional, kWaveEvents events) marks the stage boundaries: before K1, after K1,
// its far phase, the compaction + normals, K2, its far phase, K3a + K3c, K3b.
constexpr int kWaveEvents = 8;
constexpr int kShadowStats = 64;  // K2's counters at stats + kShadowStats (stats runs)
template <typename R>
void launch_wavefront(const WaveParams<R>& p, int persistBlocks, bool stats, cudaStream_t st, const cudaEvent_t* ev,
                      long long* launches);
// stage 0 G-buffer, 1 downsample+select, 2 tiles (tasks+visibility+shadePixelGI),
// 3 resolve, 4 contact
template <typename R>
void launch_gather(const GatherParams<R>& p, int stage, bool stats, cudaStream_t st);
void launch_relocate(const RelocParams& p, int nProbes, bool stats, cudaStream_t st);
void launch_query_points(const QueryParams& p, cudaStream_t st);
// Probe state (ProbesView arrays at global index base..base+n): the makeCascade
// state (restingAt, probe_volume.hpp:37-39: origin + i * spacing per axis; alive,
// rejectHistory set, never updated), and the sdfgi_probe AoS <-> SoA conversions.
void launch_probes_reset(ProbesView pv, int base, const int res[3], const double origin[3], double spacing,
                         cudaStream_t st);
// aos: 11 doubles per probe (sdfgi_probe: resting, pos, last_pos, then 4 int32)
void launch_probes_unpack(ProbesView pv, int base, int n, const double* aos, cudaStream_t st);
void launch_probes_pack(ProbesView pv, int base, int n, double* aos, cudaStream_t st);
void launch_mark_updated(const int* ids, int n, int frame, const int* alive, int* reject, int* lastFrame,
                         cudaStream_t st);
void launch_grid_bound(const GridBuildParams& p, int ncells, cudaStream_t st);
void launch_grid_seed(const GridBuildParams& p, int nbricks, cudaStream_t st);
void launch_grid_list(const GridBuildParams& p, int ncells, bool fill, cudaStream_t st);
void launch_grid_cells(const int* start, const int2* entry, int4* cell, int ncells, cudaStream_t st);
// entry.y = map[entry.y] for every list entry (sentinels stay -1)
void launch_grid_remap(int2* entry, long long n, const int* map, cudaStream_t st);
void launch_brick_clusters(const GridBuildParams& p, int nbricks, bool fill, cudaStream_t st);
// exclusive prefix sum of n ints on the device (CUB); temp == null: returns the bytes needed
size_t scan_ints(const int* in, int* out, int n, void* temp, size_t tempBytes, cudaStream_t st);
// hitList = the ids >= 0 of hitAt in order, *count = their number (CUB select); temp == null: bytes needed
size_t compact_hits(const int* hitAt, int* hitList, unsigned long long* count, int n, void* temp, size_t tempBytes,
                    cudaStream_t st);

constexpr int kWaveThreads = 128;   // K1/K2 persistent CTAs
// WaveParams::ctr slots, each on its own 128-byte line: the work cursors and
// compaction counters are hit by atomics from every SM, and counters sharing a
// line would serialise there (and slow every read of the line); the per-light
// shadow-march counts follow, read-only while K2 runs.
constexpr int kCtrRay = 0, kCtrHits = 16, kCtrShadow = 32, kCtrParkRay = 48, kCtrFarRay = 64, kCtrParkShadow = 80,
              kCtrFarShadow = 96, kCtrMvc = 112, kCtrTri = 128;
constexpr int kLightCtr = 144;
// minimum resident K1/K2/K3a CTAs per SM (register cap = 64K / (128 * n)); the
// tracing kernels are latency bound at low occupancy (measured, profiles/)
#ifndef SDFGI_WAVE_MINB64
#define SDFGI_WAVE_MINB64 7  // C2 pass 0 FP64 (K1 / K2 CTAs): 6/7 9.80, 7/6 9.75-9.83, 7/7 9.49-9.57,
#endif                       // 7/8 9.51-9.55, 8/7 9.67-9.72, 8/8 9.68-9.73, 9/9 10.13-10.21 ms
#ifndef SDFGI_WAVE_MINB32
#define SDFGI_WAVE_MINB32 8  // C2 pass 0 FP32: 6 / 7 / 8 / 10 CTAs = 6.33 / 6.24 / 6.16 / 6.32 ms
#endif
#ifndef SDFGI_SHADE_MINB
#define SDFGI_SHADE_MINB 6  // 80 registers since the bounce lookups left K3a: 5 / 6 / 8 CTAs = 0.69 / 0.63 / 0.65 ms per step (ncu); round 1: 3 / 4 / 5 = 10.26 / 10.11 / 10.02 ms
#endif
#ifndef SDFGI_SHADOW_MINB64
#define SDFGI_SHADOW_MINB64 SDFGI_WAVE_MINB64
#endif
#ifndef SDFGI_SHADOW_MINB32
#define SDFGI_SHADOW_MINB32 SDFGI_WAVE_MINB32
#endif
// K1 / K2 with the primitive records staged in shared memory: one CTA per SM with
// as many threads as the register budget of the many-CTA form allows (FP64: 7 x 128
// at 72 registers, FP32: 8 x 128 at 64).
#ifndef SDFGI_STAGE_THREADS64
#define SDFGI_STAGE_THREADS64 896
#endif
#ifndef SDFGI_STAGE_THREADS32
#define SDFGI_STAGE_THREADS32 1024
#endif
template <typename R> struct StageOcc {
    static constexpr int threads = sizeof(R) == 8 ? SDFGI_STAGE_THREADS64 : SDFGI_STAGE_THREADS32;
};
template <typename R> struct WaveOcc {
    static constexpr int trace = sizeof(R) == 8 ? SDFGI_WAVE_MINB64 : SDFGI_WAVE_MINB32;
    static constexpr int shadow = sizeof(R) == 8 ? SDFGI_SHADOW_MINB64 : SDFGI_SHADOW_MINB32;
    static constexpr int shade = SDFGI_SHADE_MINB;
};
constexpr int kShadeThreads = 128;  // per-ray shading
#ifndef SDFGI_MVC_MINB
#define SDFGI_MVC_MINB 5
#endif
#ifndef SDFGI_MVC_THREADS
#define SDFGI_MVC_THREADS 128
#endif
// K3c: one MVC hit per thread, kMvcThreads per CTA, kMvcMinBlocks resident per SM
constexpr int kMvcThreads = SDFGI_MVC_THREADS;
constexpr int kMvcMinBlocks = SDFGI_MVC_MINB;
// K3b CTA per probe: one thread per texel summing its three channels over the
// rays (one cosine per (texel, ray) instead of three), or per (texel, channel)
#ifndef SDFGI_CONV_TEXEL
#define SDFGI_CONV_TEXEL 1
#endif
constexpr bool kConvPerTexel = SDFGI_CONV_TEXEL != 0;
// K3b streams a probe's rays through shared memory in chunks of kConvChunk
// (6 KB in FP64 instead of the whole 2N-ray set: 4x the resident CTAs)
#ifndef SDFGI_CONV_CHUNK
#define SDFGI_CONV_CHUNK 128
#endif
constexpr int kConvChunk = SDFGI_CONV_CHUNK;
constexpr int kConvThreads = kConvPerTexel ? 64 : 192;
constexpr int kScanThreads = 1024;  // K0 prefix sum

}  // namespace sdfgi_dev
