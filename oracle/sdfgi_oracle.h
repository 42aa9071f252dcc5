/*
 * sdfgi_oracle.h — TEST INFRASTRUCTURE: a plain-C restatement of the reference's
 * probe path, used only as the checker (tests/, __graft_entry__.smoke(), and the
 * bench's CPU-baseline leg). Never linked into or called by the product.
 *
 * Every function restates the reference function cited beside it
 * (/root/reference/proj/include/sdfgi/*.hpp). Built with -ffp-contract=off, the
 * same flag pinning as oracle/_ref/ref_parity, it is bit-exact with the reference
 * (checked against tests/golden/ by tests/test_oracle.py).
 *
 * Parity is pinned: the golden fixtures were produced by the reference itself.
 */
#ifndef SDFGI_ORACLE_H
#define SDFGI_ORACLE_H

#include <stdint.h>

#include "../include/sdfgi_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ora_stage ora_stage;

/* ActiveScene (scene.hpp:88-103) from the ABI arrays; the arrays are copied. */
ora_stage* ora_create(const sdfgi_prim* prims, int n_prims, const sdfgi_cluster* clusters, int n_clusters,
                      const int32_t* member_start, const int32_t* member_idx, const sdfgi_light* lights,
                      int n_lights, const double sky[3]);
void ora_destroy(ora_stage* s);

/* makeCascade-equivalent volume (probe_volume.hpp:57-76): fresh probes, zero atlases. */
int ora_add_cascade(ora_stage* s, int level, int rx, int ry, int rz, double spacing, const double origin[3],
                    int oct_res);

/* updateProbePositions (probe_volume.hpp:99-143) for cascade slot `slot`. */
int ora_relocate(ora_stage* s, int slot, double th1, double th2, int max_steps, double grad_step, int report[3],
                 uint64_t stats[8]);

/* The probe stage of renderFrame (pipeline.hpp:126-151): back <- front, updateProbe
 * (probe_update.hpp:166-211) for every alive probe whose index % stride == 0, using
 * `threads` OpenMP threads (results are thread-count independent), then swap. */
int ora_update(ora_stage* s, const sdfgi_cfg* cfg, int frame, int stride, int threads, double* max_delta,
               int64_t* rays, int64_t* updated, uint64_t stats[8]);

/* ora_update over an explicit (slot, index) list (e.g. ora_select's). */
int ora_update_refs(ora_stage* s, const sdfgi_cfg* cfg, int frame, const int32_t* refs, int n_refs, int threads,
                    double* max_delta, int64_t* rays, int64_t* updated, uint64_t stats[8]);

/* selectProbesForUpdate (probe_volume.hpp:154-198): up to `budget` (slot, index)
 * pairs into out_refs, in the reference's order; returns the count. */
int ora_select(const ora_stage* s, const double cam_pos[3], const double cam_fwd[3], int budget, int frame,
               int32_t* out_refs);

int ora_probes(const ora_stage* s, int slot, sdfgi_probe* out, int n);
int ora_atlas(const ora_stage* s, int slot, float* out, int64_t n_floats); /* front atlas */
/* test hooks of the sharded decomposition (tests/test_multirank.py) */
int ora_atlas_set(ora_stage* s, int slot, const float* src, int64_t n_floats);
int ora_mark_updated(ora_stage* s, const int32_t* refs, int n_refs, int frame);

/* Per-ray records of updateProbe's ray stage (probe_update.hpp:173-189) for one probe. */
int ora_trace_rays(const ora_stage* s, const sdfgi_cfg* cfg, int frame, int slot, int probe, sdfgi_ray_record* out,
                   int cap);

/* querySceneSdf (scene.hpp:336-340) at n points; init may be NULL (+inf). */
void ora_query(const ora_stage* s, const double* pts, const double* init, int n, double* d, int32_t* owner);

/* renderGBuffer (shading.hpp:39-72) with prevCamera == camera. out: w*h pixels. */
/* threads of the gather's row loops and renderGBuffer (default 1) */
void ora_set_threads(int n);
int ora_render_gbuffer(const ora_stage* s, const sdfgi_camera* cam, int w, int h, const sdfgi_cfg* cfg,
                       sdfgi_gbuffer_pixel* out, uint64_t stats[8]);

/* One gather frame of renderFrame (pipeline.hpp:161-207) against the front atlas:
 * downsampleDepthCheckerboard, selectVisibilityPixels, buildVisibilityTasks,
 * runVisibilityTasks, shadePixelGI, upsampleAndResolve (with the given history;
 * hist_valid = 0 for none), contactGI (radius = contactRadiusFrac * cascade-0
 * spacing). Outputs (any may be NULL): half depth/src ((w+1)/2 x (h+1)/2), selection
 * (quarter grid), sparse irradiance (3 per cell) / valid / anchor, resolved and
 * indirect (3 doubles per pixel). Returns the number of visibility tasks. */
int ora_gather_frame(const ora_stage* s, const sdfgi_gbuffer_pixel* gb, int w, int h, int frame, const sdfgi_cfg* cfg,
                     const double* hist_irr, const double* hist_depth, int hist_valid, double* half_depth,
                     int32_t* half_src, int32_t* sel, double* sparse_irr, int32_t* sparse_valid,
                     int32_t* sparse_anchor, double* resolved, double* indirect, uint64_t vis_stats[8],
                     uint64_t contact_stats[8]);

/* composeFrame (shading.hpp:480-504): sky radiance on sky pixels, else
 * emission + albedo/pi * directIrradiance(worldPos, normal) + indirect.
 * indirect / out: 3 doubles per pixel. */
int ora_compose(const ora_stage* s, const sdfgi_gbuffer_pixel* gb, int w, int h, const double* indirect,
                const sdfgi_cfg* cfg, double* out, uint64_t stats[8]);

#ifdef __cplusplus
}
#endif
#endif
