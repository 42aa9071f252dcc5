/*
 * sdfgi_b200.h — C-ABI of the B200-native SDFDDGI probe update.
 *
 * This is the drop-in boundary. Every entry point takes plain pointers and sizes
 * (no torch / CUDA / C++ types) and returns an int status (SDFGI_OK == 0). The
 * message for the last failure on the calling thread is sdfgi_last_error().
 * There is no CPU fallback: a context can only be created on a CUDA device.
 *
 * The reference (`/root/reference/proj/include/sdfgi/`, header-only C++20) has no
 * FFI; its hot path is a set of inline functions called from
 * Renderer::renderFrame (pipeline.hpp:108-151 probe stage, :161-207 gather).
 * Each entry point below cites the reference interface it replaces. The C++
 * shim `paper_2007_14394_b200/include/sdfgi_b200.hpp` and the Python mirror
 * `paper_2007_14394_b200/api.py` keep the reference's names over this ABI.
 *
 * Threading contract: one host thread per context; every call is ordered on
 * the context's CUDA stream and returns after the stream has drained unless
 * the function says otherwise.
 *
 * Structs are also the on-disk layout of the SDFS scene interchange file
 * (see paper_2007_14394_b200/scene_io.py); all fields are little-endian and
 * naturally aligned, no implicit padding.
 */
#ifndef SDFGI_B200_H
#define SDFGI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDFGI_ABI_VERSION 1

#if defined(__GNUC__)
#define SDFGI_API __attribute__((visibility("default")))
#else
#define SDFGI_API
#endif

enum sdfgi_status {
    SDFGI_OK = 0,
    SDFGI_ERR_INVALID = 1,   /* bad argument (null pointer, size mismatch, range) */
    SDFGI_ERR_CUDA = 2,      /* CUDA runtime failure, or no CUDA device */
    SDFGI_ERR_NCCL = 3,      /* collective failure */
    SDFGI_ERR_STATE = 4,     /* call out of order (e.g. update before scene upload) */
    SDFGI_ERR_OOM = 5
};

/* PrimitiveKind, primitives.hpp:9 */
enum sdfgi_prim_kind { SDFGI_SPHERE = 0, SDFGI_BOX = 1, SDFGI_PLANE = 2, SDFGI_CYLINDER = 3, SDFGI_CAPSULE = 4 };
/* LightKind, primitives.hpp:16 */
enum sdfgi_light_kind { SDFGI_LIGHT_POINT = 0, SDFGI_LIGHT_DIRECTIONAL = 1, SDFGI_LIGHT_SKY = 2 };
/* arithmetic of the device path */
enum sdfgi_precision { SDFGI_F64 = 0, SDFGI_F32 = 1 };

/* SdfPrimitive + Material, primitives.hpp:11-38 (rotation row-major, vec.hpp:75). 184 B. */
typedef struct sdfgi_prim {
    int32_t id;
    int32_t kind;
    int32_t lod_tier;
    int32_t _pad;
    double rot[9];
    double trans[3];
    double size[3];
    double albedo[3];
    double emission[3];
} sdfgi_prim;

/* Light, primitives.hpp:18-23. 80 B. */
typedef struct sdfgi_light {
    int32_t kind;
    int32_t _pad;
    double position[3];
    double direction[3];
    double intensity[3];
} sdfgi_light;

/* Cluster cull bounds (Cluster::cullAabb + unbounded, scene.hpp:38-46), already
 * inflated by kClusterCullMargin. Members are CSR: member_start[k+1], member_idx[]. 56 B. */
typedef struct sdfgi_cluster {
    double lo[3];
    double hi[3];
    int32_t unbounded;
    int32_t _pad;
} sdfgi_cluster;

/* RenderConfig, config.hpp:9-50. Every field 8 bytes; ints widened to int64. 224 B. */
typedef struct sdfgi_cfg {
    double surface_epsilon;
    int64_t max_trace_steps;
    int64_t shadow_steps;
    double ray_tmax;
    double shadow_k;
    double probe_visibility_k;
    double gradient_step;
    int64_t max_per_cluster;
    double merge_radius;
    double threshold1_frac;
    double threshold2_frac;
    int64_t max_descent_steps;
    int64_t probe_budget;
    int64_t n_rays_full;
    double hysteresis;
    double alpha_min;
    double bounce_coeff;
    int64_t oct_res;
    int64_t rotate_per_frame;
    uint64_t seed;
    double mvc_relocation_frac;
    double dedup_quant_frac;
    double contact_radius_frac;
    int64_t contact_samples;
    double history_blend;
    double depth_sigma_frac;
    double exposure;
    int64_t fps;
} sdfgi_cfg;

/* Probe, probe_volume.hpp:12-19, as stored on the host side of the ABI. 88 B. */
typedef struct sdfgi_probe {
    double resting[3];
    double pos[3];
    double last_pos[3];
    int32_t reject_history;
    int32_t alive;
    int32_t last_update_frame;
    int32_t _pad;
} sdfgi_probe;

/* TraceStats, scene.hpp:16-36 */
typedef struct sdfgi_stats {
    uint64_t sdf_queries;
    uint64_t clusters_visited;
    uint64_t clusters_skipped;
    uint64_t primitive_evals;
    uint64_t trace_steps;
    uint64_t sphere_traces;
    uint64_t shadow_traces;
    uint64_t visibility_traces;
} sdfgi_stats;

/* RelocationReport, probe_volume.hpp:88-92 */
typedef struct sdfgi_reloc_report {
    int32_t relocated;
    int32_t rejected;
    int32_t dead;
    int32_t _pad;
} sdfgi_reloc_report;

/* Sum over a batch of ProbeUpdateResult (probe_update.hpp:151-154). */
typedef struct sdfgi_update_result {
    double max_texel_delta;   /* max over updated probes */
    int64_t rays_traced;      /* sum of raysTraced */
    int64_t probes_updated;   /* alive probes that were updated */
} sdfgi_update_result;

/* Per-ray record (debug / parity), mirrors the Hit + RadianceSample pair built in
 * updateProbe (probe_update.hpp:177-189). 96 B. */
typedef struct sdfgi_ray_record {
    double dir[3];
    double t;              /* Hit::t when converged, else 0 */
    double radiance[3];
    double normal[3];
    int32_t converged;
    int32_t miss;          /* MissReason: 0 None, 1 TMax, 2 StepLimit */
    int32_t prim_index;    /* Hit::primitiveIndex */
    int32_t steps;         /* sphere-trace loop iterations */
} sdfgi_ray_record;

/* GBufferPixel (shading.hpp:13-22): depth along the view ray (+inf = sky), normal,
 * albedo, emission, world position, motion (pixel offset to last frame), owner. 128 B. */
typedef struct sdfgi_gbuffer_pixel {
    double depth;
    double normal[3];
    double albedo[3];
    double emission[3];
    double world_pos[3];
    double motion[2];
    int32_t prim_index;
    int32_t _pad;
} sdfgi_gbuffer_pixel;

/* Camera (camera.hpp:9-49): orthonormal frame + vertical fov in degrees. 104 B. */
typedef struct sdfgi_camera {
    double position[3];
    double forward[3];
    double right[3];
    double up[3];
    double fov_y_deg;
} sdfgi_camera;

/* Hit, scene.hpp:375-383: one sphereTrace result. prim_index indexes the uploaded
 * primitive array (ActiveScene::primitives); miss is MissReason (0 None, 1 TMax,
 * 2 StepLimit). 72 B. */
typedef struct sdfgi_hit {
    double t;
    double pos[3];
    double normal[3];
    int32_t prim_index;
    int32_t converged;
    int32_t miss;
    int32_t _pad;
} sdfgi_hit;

/* InterpolationStencil, probe_volume.hpp:205-217: 8 entries of one cascade
 * (level), weights normalised; count 0 with sky_fallback when no cascade holds the
 * point or every corner is dead. 120 B. */
typedef struct sdfgi_stencil {
    double weight[8];
    int32_t level;
    int32_t index[8];
    int32_t count;
    int32_t cross_cascade;
    int32_t sky_fallback;
    int32_t used_mvc;
    int32_t _pad;
} sdfgi_stencil;

/* ---------------------------------------------------------------- lifecycle */
SDFGI_API int sdfgi_abi_version(void);
SDFGI_API const char* sdfgi_last_error(void);
/* Number of CUDA devices visible (0 on a machine without a GPU). */
SDFGI_API int sdfgi_device_count(int* out);
/* NCCL unique id for a multi-GPU context (rank 0 creates, the caller broadcasts). */
SDFGI_API int sdfgi_nccl_unique_id(uint8_t out[128]);
/* rank/world: probe-slab sharding. nccl_uid may be NULL when world == 1. */
SDFGI_API int sdfgi_ctx_create(int device, int rank, int world, const uint8_t* nccl_uid, int precision,
                     void** out_ctx);
SDFGI_API int sdfgi_ctx_destroy(void* ctx);
SDFGI_API int sdfgi_ctx_set_precision(void* ctx, int precision);
/* Raw CUDA stream handle (cudaStream_t) of the context, for event timing. */
SDFGI_API int sdfgi_ctx_stream(void* ctx, void** out_stream);
SDFGI_API int sdfgi_ctx_synchronize(void* ctx);

/* -------------------------------------------------------------------- scene */
/* Replaces ActiveScene construction + finalize() (scene.hpp:88-103). Copied to
 * the device; the caller keeps ownership. `sky` = ActiveScene::sky. */
SDFGI_API int sdfgi_scene_upload(void* ctx, const sdfgi_prim* prims, int n_prims,
                       const sdfgi_cluster* clusters, int n_clusters,
                       const int32_t* member_start, const int32_t* member_idx,
                       const sdfgi_light* lights, int n_lights, const double sky[3]);
/* Lights and sky only (moving lights, C5); primitives unchanged. */
SDFGI_API int sdfgi_lights_upload(void* ctx, const sdfgi_light* lights, int n_lights, const double sky[3]);

/* ------------------------------------------------------------- probe volume */
/* makeCascade / CascadeVolume (probe_volume.hpp:24-76). Allocates probes (reset to
 * resting, rejectHistory=1, alive=1, lastUpdateFrame=-1) and both atlases (zero). */
SDFGI_API int sdfgi_cascade_set(void* ctx, int level, int res_x, int res_y, int res_z, double spacing,
                      const double origin[3], int oct_res);
SDFGI_API int sdfgi_cascade_count(void* ctx, int* out);
/* Drop every cascade (probes and atlases); the next cascade_set starts a new volume. */
SDFGI_API int sdfgi_cascades_clear(void* ctx);
SDFGI_API int sdfgi_probes_reset(void* ctx, int level);
SDFGI_API int sdfgi_probes_upload(void* ctx, int level, const sdfgi_probe* probes, int n);
SDFGI_API int sdfgi_probes_download(void* ctx, int level, sdfgi_probe* probes, int n);

/* selectProbesForUpdate (probe_volume.hpp:154-198) over every cascade's device
 * probes: priority = 1/(1 + dist/spacing) * (0.25 + 0.75 max(0, facing)) *
 * staleness (x4 if rejectHistory); probes stale for >= ceil(total/budget) frames
 * are forced first, oldest first; the first `budget` in the reference's
 * stable-sort order. out_refs: 2 * min(budget, total) int32 (cascade level,
 * index), ready for sdfgi_probes_update. budget <= 0 selects nothing (the caller
 * passes the probe count for "all", pipeline.hpp:133). */
SDFGI_API int sdfgi_select_probes(void* ctx, const double cam_pos[3], const double cam_fwd[3], int budget, int frame,
                                  int32_t* out_refs, int* n_out);

/* updateProbePositions (probe_volume.hpp:99-143) for one cascade, device-resident.
 * Bit-exact with the reference in SDFGI_F64 mode. */
SDFGI_API int sdfgi_probes_relocate(void* ctx, int level, double threshold1, double threshold2,
                          int max_descent_steps, double gradient_step,
                          sdfgi_reloc_report* report, sdfgi_stats* stats);

/* The probe stage of renderFrame (pipeline.hpp:126-151): back atlas <- front atlas,
 * then updateProbe (probe_update.hpp:166-211) for every selected alive probe, writing
 * the back atlas and reading the front atlas for bounce. probe_refs are (cascade,
 * index) pairs; NULL means every probe of every cascade (probeBudget 0). With
 * world > 1 each rank updates its z-slab and the back atlas is all-gathered. */
SDFGI_API int sdfgi_probes_update(void* ctx, const int32_t* probe_refs, int n_refs, int frame,
                        const sdfgi_cfg* cfg, sdfgi_update_result* result, sdfgi_stats* stats);
/* The whole probe stage of renderFrame (pipeline.hpp:108-151; the recenter of
 * :110-113 stays with the caller, sdfgi_cascade_set) in one call and one host
 * synchronisation:
 * updateProbePositions for every cascade with cfg's thresholds (threshold*_frac x
 * the cascade's spacing, max_descent_steps, gradient_step), then — with
 * cfg->probe_budget > 0 — selectProbesForUpdate from cam_pos/cam_fwd, and the
 * updateProbe pass of sdfgi_probes_update (NULL refs = every probe when the budget
 * is 0; cam_pos/cam_fwd may then be NULL). reports: one per cascade in the order
 * sdfgi_cascade_set created them (n_reports >= cascade count) or NULL; stats sum relocation and update.
 * Same results as the sequence of sdfgi_probes_relocate / sdfgi_select_probes /
 * sdfgi_probes_update calls it replaces. */
SDFGI_API int sdfgi_probe_stage(void* ctx, int frame, const sdfgi_cfg* cfg, const double cam_pos[3],
                                const double cam_fwd[3], sdfgi_reloc_report* reports, int n_reports,
                                sdfgi_update_result* result, sdfgi_stats* stats);
/* sdfgi_probe_stage without the host synchronisation: the pass is queued on the
 * context's stream and the call returns; up to 8 passes (with sdfgi_atlas_swap
 * between them) may be in flight, so the host prepares pass p+1 while the device
 * runs pass p. Their reports and results come from sdfgi_probe_stage_collect, in
 * pass order (reports: reports_per_pass per pass, cascade order; results: one per
 * pass); it synchronises, adds the passes' stage times to sdfgi_stage_ms_sum and
 * returns the pass count in *n_passes. No TraceStats in this form. A budgeted
 * pass (cfg->probe_budget > 0) synchronises for its selection. */
SDFGI_API int sdfgi_probe_stage_async(void* ctx, int frame, const sdfgi_cfg* cfg, const double cam_pos[3],
                                      const double cam_fwd[3]);
SDFGI_API int sdfgi_probe_stage_collect(void* ctx, sdfgi_reloc_report* reports, int reports_per_pass,
                                        sdfgi_update_result* results, int max_passes, int* n_passes);
/* readIdx swap at frame end (pipeline.hpp:220). */
SDFGI_API int sdfgi_atlas_swap(void* ctx);
/* which = 0: front (read) atlas, 1: back (write) atlas. Layout = ProbeAtlas::raw()
 * (atlas.hpp:119-124): ((probe*(R+2)+y)*(R+2)+x)*3 floats. */
SDFGI_API int sdfgi_atlas_download(void* ctx, int level, int which, float* dst, size_t n_floats);
SDFGI_API int sdfgi_atlas_upload(void* ctx, int level, int which, const float* src, size_t n_floats);
/* Pinned-free device pointer of an atlas (for collectives / zero-copy views). */
SDFGI_API int sdfgi_atlas_device_ptr(void* ctx, int level, int which, void** out_ptr, size_t* out_bytes);

/* Debug/parity: re-run the ray stage of updateProbe for the listed probes against
 * the front atlas and return one record per ray (2N when rejectHistory). Records are
 * written consecutively, probe by probe; n_records_max bounds the output. */
SDFGI_API int sdfgi_probes_trace_debug(void* ctx, const int32_t* probe_refs, int n_refs, int frame,
                             const sdfgi_cfg* cfg, sdfgi_ray_record* out, int n_records_max,
                             int* n_written);

/* Point queries (querySceneSdf, scene.hpp:336-340): d[i] = min(naive SDF, init_d[i]),
 * owner[i] = primitive index or -1. init_d may be NULL (= +inf). Host arrays. */
SDFGI_API int sdfgi_query_points(void* ctx, const double* points_xyz, const double* init_d, int n,
                       double* out_d, int32_t* out_owner);

/* Device time (CUDA events on the context stream, bracketing only the kernel) of the
 * most recent k_probe_update launch and of the most recent relocation launch, in ms. */
SDFGI_API int sdfgi_last_kernel_ms(void* ctx, double* update_ms, double* relocate_ms);

/* Primitive evaluations of the most recent stats-enabled relocate/update call, by
 * PrimitiveKind (sphere, box, plane, cylinder, capsule) and [5] how many of them
 * were rotated: with sdfgi_stats these define the algorithmic work. */
SDFGI_API int sdfgi_last_work(void* ctx, uint64_t out[6]);
/* Shading work of the last stats-enabled sdfgi_probes_update: {shadeHit calls
 * (converged hits with an owner), mvcWeightsHex evaluations} — the W_stencil
 * term of the algorithmic-work model. */
SDFGI_API int sdfgi_last_shading_work(void* ctx, uint64_t out[2]);
/* Device ms of the last sdfgi_probes_update's stages: {K1 primary rays, K1 far
 * phase, hit compaction + normals + shadow set-up, K2 shadow rays, K2 far phase,
 * K3a + K3c shading, K3b convolution + blend}. */
SDFGI_API int sdfgi_last_stage_ms(void* ctx, double out[7]);
/* The same stage times summed over every update since the last reset, out[7] = the
 * updates' total (first to last stage event); reset != 0 zeroes the sums after
 * reading. Lets a frame loop read its timings once instead of after every pass. */
SDFGI_API int sdfgi_stage_ms_sum(void* ctx, double out[8], int reset);
/* The last stats-enabled update's event counters per tracing kernel: out[0..13]
 * K1 (primary rays), out[14..27] K2 (shadow rays), each {sdf_queries,
 * clusters_visited, clusters_skipped, primitive_evals, trace_steps, sphere_traces,
 * shadow_traces, visibility_traces, evaluations by kind x5, rotated evaluations}. */
SDFGI_API int sdfgi_last_trace_counters(void* ctx, uint64_t out[28]);

/* FP pipe throughput microbenchmark on the context's device: FP64 and FP32 fused
 * multiply-add instructions per second (the roofline denominators for the tracing
 * kernels, which MEASURED_PEAKS.json does not carry). */
SDFGI_API int sdfgi_measure_fp_peak(void* ctx, double* f64_fma_per_s, double* f32_fma_per_s);

/* Cluster-walk strategy of every SDF query: 0 = the reference's flat walk in cluster
 * order (TraceStats identical to the reference), 1 = candidate-cluster grid (default;
 * identical query values and owners, far fewer cluster tests). */
SDFGI_API int sdfgi_set_accel(void* ctx, int mode);
/* {mode, grid built, dim x, dim y, dim z, candidate list entries} */
SDFGI_API int sdfgi_accel_info(void* ctx, int64_t out[6]);

/* Probe-index range [lo, hi) of a cascade that rank `rank` of `world` updates: the
 * z-slab of layers [res_z*rank/world, res_z*(rank+1)/world). Pure
 * function (no context, no device). */
SDFGI_API int sdfgi_slab_range(int res_x, int res_y, int res_z, int rank, int world, int* lo, int* hi);

/* ------------------------------------------------------------ gather (e) */
/* Input G-buffer (renderGBuffer, shading.hpp:39-72): upload the caller's, or render
 * it on the device from the camera (prev_cam NULL = same camera, motion 0). */
SDFGI_API int sdfgi_gbuffer_upload(void* ctx, int w, int h, const sdfgi_gbuffer_pixel* px);
SDFGI_API int sdfgi_gbuffer_render(void* ctx, const sdfgi_camera* cam, const sdfgi_camera* prev_cam, int w, int h,
                                   const sdfgi_cfg* cfg);
SDFGI_API int sdfgi_gbuffer_download(void* ctx, sdfgi_gbuffer_pixel* out, size_t n_pixels);
/* One gather frame of renderFrame (pipeline.hpp:161-207) against the FRONT atlas
 * (prevField): downsampleDepthCheckerboard, selectVisibilityPixels,
 * buildVisibilityTasks + runVisibilityTasks + shadePixelGI, upsampleAndResolve with
 * the context's history, contactGI; then rolls the history (pipeline.hpp:213-218). */
SDFGI_API int sdfgi_gather(void* ctx, int frame, const sdfgi_cfg* cfg, int64_t* n_tasks, sdfgi_stats* vis_stats,
                           sdfgi_stats* contact_stats);
SDFGI_API int sdfgi_gather_reset_history(void* ctx);
/* which: 0 resolved E, 1 indirect (contactGI output), 2 half-res depth, 3 half-res
 * source pixel, 4 selection, 5 sparse irradiance, 6 sparse valid, 7 sparse anchor,
 * 8 composed image (sdfgi_compose). Doubles for 0,1,2,5,8 (3 per pixel/cell for
 * 0,1,5,8), int32 otherwise. */
SDFGI_API int sdfgi_gather_download(void* ctx, int which, void* dst, size_t bytes);
/* Device ms of the last gather: {downsample+select, tiles, resolve, contact}. */
SDFGI_API int sdfgi_last_gather_ms(void* ctx, double out[4]);
/* Replace the indirect image (3 doubles per G-buffer pixel) — e.g. to compose an
 * externally computed indirect term. */
SDFGI_API int sdfgi_indirect_upload(void* ctx, const double* rgb, size_t n_doubles);
/* composeFrame (shading.hpp:480-504; pipeline.hpp:209): per G-buffer pixel, sky
 * radiance on sky pixels, else emission + albedo/pi * directIrradiance(worldPos,
 * normal) + indirect, with the direct term's soft shadows traced on the device.
 * Reads the context's G-buffer and indirect image (the last gather's, or the
 * uploaded one); the result is gather buffer 8. stats (may be NULL) += TraceStats
 * of the shadow traces; ms (may be NULL) = device time. */
SDFGI_API int sdfgi_compose(void* ctx, const sdfgi_cfg* cfg, sdfgi_stats* stats, double* ms);

/* Linear-time cluster builder for large scenes (replaces buildClusters,
 * scene.hpp:110-178, whose greedy agglomeration is O(N^3)): bounded primitives in
 * Morton order of their box centres, runs of max_per_cluster; each plane its own
 * unbounded cluster; cull boxes = surface boxes inflated by kClusterCullMargin.
 * Any conservative clustering yields identical query values (scene.hpp:205-211).
 * Host only (no context). Capacity: n clusters, n+1 starts, n members. */
SDFGI_API int sdfgi_build_clusters(const sdfgi_prim* prims, int n, int max_per_cluster, sdfgi_cluster* out_clusters,
                                   int* out_n_clusters, int32_t* member_start, int32_t* member_idx);

/* Launch counter: kernels this context has launched since creation. */
/* ---- the reference's free functions, batched (each call runs one device batch
 * over n items with the context's scene, cascades and front atlas) ---- */
/* sphereTrace (scene.hpp:391-435) of n rays (origins, dirs: 3 doubles each) with
 * the shared tMax, surfaceEpsilon, maxSteps and startBound. */
SDFGI_API int sdfgi_trace_rays(void* ctx, const double* origins, const double* dirs, int n, double t_max,
                               double surface_epsilon, int max_steps, double start_bound, sdfgi_hit* out,
                               sdfgi_stats* stats);
/* softShadowTrace (scene.hpp:459-476) of n segments [t_min[i], t_max[i]] with the
 * shared k, maxSteps and minStep; out_vis[i] in [0, 1]. */
SDFGI_API int sdfgi_soft_shadow(void* ctx, const double* origins, const double* dirs, const double* t_min,
                                const double* t_max, int n, double k, int max_steps, double min_step,
                                double* out_vis, sdfgi_stats* stats);
/* shadeHit (probe_update.hpp:136-149) of n hits against the context's front atlas
 * (the previous field) with the given bounceCoeff; out_rgb 3 doubles per hit. */
SDFGI_API int sdfgi_shade_hits(void* ctx, const sdfgi_hit* hits, int n, double bounce_coeff, const sdfgi_cfg* cfg,
                               double* out_rgb, sdfgi_stats* stats);
/* convolveIrradiance (probe_update.hpp:25-34): one sample set (directions and
 * radiance, 3 doubles each) convolved for n_texels directions into out_rgb. */
SDFGI_API int sdfgi_convolve_irradiance(void* ctx, const double* sample_dirs, const double* sample_radiance,
                                        int n_samples, const double* texel_dirs, int n_texels, double* out_rgb);
/* interpolationStencil (probe_volume.hpp:224-310) of n points over the context's
 * cascades and probe state. */
SDFGI_API int sdfgi_interpolation_stencil(void* ctx, const double* points, int n, double mvc_relocation_frac,
                                          sdfgi_stencil* out);

SDFGI_API int sdfgi_launch_count(void* ctx, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* SDFGI_B200_H */
