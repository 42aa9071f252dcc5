// kernels.cuh — the probe-stage kernels and their launch parameter blocks.
//
//   k_relocate       (d) updateProbePositions, probe_volume.hpp:99-143. One thread
//                    per probe, always FP64 (bit-exact relocation in every mode).
//   k_probe_update   (a)(b)(c) updateProbe, probe_update.hpp:166-211. One CTA per
//                    probe: rays strided over the CTA's lanes (sphere trace ->
//                    shadeHit), radiance samples in shared memory, one texel per
//                    lane for the cosine convolution + hysteresis blend, octahedral
//                    border fill in shared memory, the finished 1200-byte tile
//                    stored with coalesced 16-byte stores.
//   k_trace_debug    per-ray records of the same ray stage (parity tests).
//   k_query_points   querySceneSdf at arbitrary points (parity tests).
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
    unsigned long long* stats;  // 8 counters or null
};

template <typename R> struct UpdateParams {
    SceneView<R> scene;
    ProbeCommon pc;
    const float* prevAtlas;   // front (read) atlas, all cascades concatenated
    float* currAtlas;         // back (write) atlas
    int oct;
    const int* refs;          // global probe ids (cascade base + index); null = all
    int nRefs;
    int frame;
    TraceCfg tc;
    double hysteresis, alphaMin;
    int nRaysFull;
    uint64_t seed;
    int rotatePerFrame;
    unsigned long long* stats;       // 8 counters or null
    unsigned long long* maxDeltaBits;
    unsigned long long* rays;
    unsigned int* updated;
    // debug
    struct RayRecord* records;
    const int* recordOffset;
};

// Mirror of sdfgi_ray_record (include/sdfgi_b200.h).
struct RayRecord {
    double dir[3];
    double t;
    double radiance[3];
    double normal[3];
    int converged, miss, prim_index, steps;
};

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
    double* U;
    int* counts;
    const int* start;
    int* list;
};

template <typename R>
void launch_probe_update(const UpdateParams<R>& p, int nBlocks, int maxRays, bool stats, cudaStream_t st);
template <typename R>
void launch_trace_debug(const UpdateParams<R>& p, int nBlocks, cudaStream_t st);
void launch_relocate(const RelocParams& p, int nProbes, bool stats, cudaStream_t st);
void launch_query_points(const QueryParams& p, cudaStream_t st);
void launch_grid_bound(const GridBuildParams& p, int ncells, cudaStream_t st);
void launch_grid_list(const GridBuildParams& p, int ncells, bool fill, cudaStream_t st);

constexpr int kUpdateThreads = 128;

}  // namespace sdfgi_dev
