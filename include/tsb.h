/*
 * tsb.h — C ABI of libtsb.so, the B200 (sm_100a) textured-2DGS render path.
 *
 * The library allocates no device memory for frame data: the caller (PyTorch
 * in the Python host layer, or any C/C++ host) owns every buffer and passes
 * raw device pointers, a CUDA stream and a workspace sized by
 * tsb_frame_workspace_size(). The only library-owned device objects are the
 * cudaArray/texture objects behind a tsb_atlas_tex_t (tsb_atlas_tex_create).
 * Nothing synchronises the host; errors from launches are reported through
 * the return code (cudaGetLastError after each launch) and tsb_last_error().
 *
 * The reference (/root/reference/pkg/src/texsplat, pure numpy) has no FFI;
 * each entry point below replaces one Python callable of its hot path, cited
 * at the declaration. The Python binding is paper_2506_13348_b200/_lib.py
 * (ctypes); INTEGRATION.md shows the binding a texsplat maintainer would add.
 */
#ifndef TSB_H
#define TSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. The Python shim maps them to the reference's exceptions. */
#define TSB_OK 0
#define TSB_ERR_VALUE (-1)    /* ValueError   (bad mode, shapes, resolution) */
#define TSB_ERR_LOOKUP (-2)   /* LookupError  (bad atlas entry / page)       */
#define TSB_ERR_CUDA (-3)     /* RuntimeError (launch / CUDA API failure)     */
#define TSB_ERR_CAPACITY (-4) /* workspace smaller than tsb_frame_workspace_size */

/* Texture modes (rasterize.py:172-236 "perprim"/"atlas"/"flat").
 * HW: atlas fetched by the texture units (tex2DLayered, bilinear).
 * VERIFY: fp32 software bilinear from linear atlas pages (bit-exact with oracle).
 * FLAT: per-splat mean texels (rasterize.py:203-209). */
#define TSB_MODE_HW 0
#define TSB_MODE_VERIFY 1
#define TSB_MODE_FLAT 2

/* Atlas texel formats for the HW mode. */
#define TSB_TEXEL_RGBA32F 0
#define TSB_TEXEL_RGBA16F 1

/* splats.py:45-78 Camera. world_to_view is row-major 4x4. */
typedef struct tsb_camera {
  double world_to_view[16];
  double fx, fy, cx, cy, near_z, far_z;
  int32_t width, height;
} tsb_camera;

/* scene.py:52-77 Scene parameter arrays (float64, device pointers). */
typedef struct tsb_scene {
  int32_t num_splats;
  int32_t sh_degree;           /* 0..3; sh has (deg+1)^2 x 3 values per splat */
  const double* positions;     /* P x 3 */
  const double* tangent_u;     /* P x 3 */
  const double* tangent_v;     /* P x 3 */
  const double* scales;        /* P x 2 */
  const double* opacities;     /* P     */
  const double* sh;            /* P x K x 3 */
  const int32_t* record_slot;  /* P or NULL: where each splat's per-frame records
                                  live in the workspace (a storage permutation for
                                  locality, e.g. Morton order of position; it never
                                  changes a result). NULL = identity */
} tsb_scene;

typedef struct tsb_atlas_tex* tsb_atlas_tex_t;

/* atlas.py:35-105 AtlasSet: family A = [albedo.rgb, roughness],
 * family B = [normal.a, normal.b, metallic, 0], pages of page_h x page_w
 * RGBA float32 texels, indirection entries (chart_x, chart_y, page). */
typedef struct tsb_atlas {
  int32_t resolution;          /* T: texels per chart side */
  int32_t page_w, page_h, pages;
  const int32_t* entries;      /* P x 3 device */
  const float* family_a;       /* pages x page_h x page_w x 4 device (VERIFY) */
  const float* family_b;       /* same layout (VERIFY) */
  const float* flat_attrs;     /* P x 5: mean albedo rgb, metallic, roughness (FLAT) */
  tsb_atlas_tex_t tex;         /* from tsb_atlas_tex_create (HW), may be NULL otherwise */
  int32_t texel_stride;        /* float4s between consecutive texels of a family: 1 for
                                  separate family pages, 2 when A and B are interleaved
                                  per texel (family_b = family_a + 4 floats) */
} tsb_atlas;

/* environment.py:209-224 EnvironmentLight + BrdfLut (device, float32). */
#define TSB_ENV_MAX_LEVELS 16
typedef struct tsb_environment {
  int32_t levels;
  const float* spec_mips[TSB_ENV_MAX_LEVELS];  /* level l: mip_h[l] x mip_w[l] x 3 */
  int32_t mip_h[TSB_ENV_MAX_LEVELS];
  int32_t mip_w[TSB_ENV_MAX_LEVELS];
  const float* diffuse;                        /* diff_h x diff_w x 3 */
  int32_t diff_h, diff_w;
  const float* lut;                            /* lut_res x lut_res x 2 */
  int32_t lut_res;
} tsb_environment;

/* Per-pixel forward state (all H x W, device). Kept for the backward pass
 * (replaces the reference's Python tape, rasterize.py:383-384). */
typedef struct tsb_pixel_state {
  int32_t* n_contrib;   /* composited fragments per pixel */
  int32_t* last_entry;  /* sorted-entry index of the last contributor, -1 if none */
  float* final_T;       /* transmittance after the last contributor */
  float* T_last;        /* transmittance in front of the last contributor */
  uint8_t* splat_touched; /* optional (may be NULL), P bytes: set to 1 for every
                             splat with at least one composited fragment
                             (diagnostics: compulsory atlas bytes of a frame) */
} tsb_pixel_state;

/* Bytes of frame workspace for P splats at W x H with `max_entries`
 * splat x tile entries. The workspace persists from tsb_render_forward to
 * tsb_render_backward of the same frame. */
int tsb_frame_workspace_size(int32_t num_splats, int32_t width, int32_t height,
                             int32_t tile, int64_t max_entries, uint64_t* bytes);

/* Byte offset, inside the same workspace, of the int64 running maximum of
 * the entries needed by every frame binned into it since the caller last
 * zeroed it (the per-frame counters are reset by each frame; this word is
 * not). A frame graph replayed without a host check can compare it with
 * max_entries afterwards: larger means some frame overflowed (rendered with
 * empty tile lists) and must be re-rendered with a larger workspace. */
int tsb_frame_workspace_max_needed_offset(int32_t num_splats, int32_t width, int32_t height,
                                          int32_t tile, int64_t max_entries, uint64_t* offset);

/* Whole forward pass K1-K5 (replaces rasterize.prepare rasterize.py:172-243,
 * _tile_lists :246-258 and render_forward :395-438): preprocess, fp64
 * depth-rank sort, tile duplication, stable tile sort, tile ranges and the
 * per-tile compositor into a planar 13 x H x W float32 G-buffer
 * (rasterize.py:52-59 channel map, coverage-premultiplied).
 * entries_needed (device int64) receives the splat x tile entry count; if it
 * exceeds max_entries the frame is incomplete and must be re-rendered with a
 * larger workspace. tile is 8, 16 or 32. */
int tsb_render_forward(const tsb_scene* scene, const tsb_camera* camera,
                       const tsb_atlas* atlas, int32_t mode, int32_t tile,
                       void* workspace, uint64_t workspace_bytes,
                       int64_t max_entries, float* gbuf,
                       const tsb_pixel_state* pixels, int64_t* entries_needed,
                       void* stream);

/* The two halves of tsb_render_forward, for callers that time or overlap
 * them separately: binning = K1-K4 (prepare + _tile_lists, rasterize.py:
 * 172-258), composite = K5 (the _render_tile loop, rasterize.py:320-385)
 * reading the lists binning left in the workspace. */
int tsb_render_binning(const tsb_scene* scene, const tsb_camera* camera,
                       const tsb_atlas* atlas, int32_t mode, int32_t tile,
                       void* workspace, uint64_t workspace_bytes,
                       int64_t max_entries, int64_t* entries_needed, void* stream);
int tsb_render_composite(const tsb_scene* scene, const tsb_camera* camera,
                         const tsb_atlas* atlas, int32_t mode, int32_t tile,
                         void* workspace, uint64_t workspace_bytes,
                         int64_t max_entries, float* gbuf,
                         const tsb_pixel_state* pixels, void* stream);

/* Frame graph: tsb_render_forward (+ tsb_shade_forward when env is not
 * NULL) of one view captured once as a CUDA graph over fixed buffers; each
 * tsb_frame_graph_launch rewrites only the camera-dependent kernel
 * parameters (and optionally the colour output) and replays the graph —
 * the multi-view serving path (cli.py:63-68 per-view body) without ~20
 * host launches per view. The camera size must match the captured one.
 * create renders (and shades) the given view once, uncaptured, to validate
 * the arguments. */
typedef struct tsb_frame_graph* tsb_frame_graph_t;
int tsb_frame_graph_create(const tsb_scene* scene, const tsb_camera* camera,
                           const tsb_atlas* atlas, int32_t mode, int32_t tile,
                           void* workspace, uint64_t workspace_bytes, int64_t max_entries,
                           float* gbuf, const tsb_pixel_state* pixels, int64_t* entries_needed,
                           const tsb_environment* env, const float* background, float* color,
                           float* diffuse, float* specular, tsb_frame_graph_t* graph);
/* As tsb_frame_graph_create, with a caller-owned cudaEvent_t recorded by
 * every replay between binning and rasterisation (may be NULL): a copy
 * stream waiting on it overlaps the previous frame's read-back with this
 * frame's rasteriser instead of its latency-bound binning. */
int tsb_frame_graph_create_ev(const tsb_scene* scene, const tsb_camera* camera,
                              const tsb_atlas* atlas, int32_t mode, int32_t tile,
                              void* workspace, uint64_t workspace_bytes, int64_t max_entries,
                              float* gbuf, const tsb_pixel_state* pixels,
                              int64_t* entries_needed, const tsb_environment* env,
                              const float* background, float* color, float* diffuse,
                              float* specular, void* binned_event, tsb_frame_graph_t* graph);
int tsb_frame_graph_launch(tsb_frame_graph_t graph, const tsb_camera* camera, float* color,
                           void* stream);
int tsb_frame_graph_destroy(tsb_frame_graph_t graph);

/* Copy the frame's structural results out of the workspace (debug/parity):
 * sorted_ids (P, kept splats in draw order then culled ids), keys
 * (max_entries: (tile << 32) | depth_rank of every sorted entry, padding
 * entries = -1) and ranges (num_tiles x 2 [start, end)). Any may be NULL. */
int tsb_frame_export(int32_t num_splats, int32_t width, int32_t height, int32_t tile,
                     int64_t max_entries, const void* workspace,
                     int32_t* sorted_ids, int64_t* keys, int32_t* ranges,
                     int32_t* rects, void* stream);

/* Deferred split-sum shading (replaces shading.shade_gbuffer shading.py:126-183
 * with mesh=None). gbuf planar 13 x H x W; color/diffuse/specular H x W x 3
 * (diffuse/specular may be NULL). background: 3 floats (host). */
int tsb_shade_forward(const float* gbuf, const tsb_camera* camera,
                      const tsb_environment* env, const float* background,
                      float* color, float* diffuse, float* specular, void* stream);

/* K0: upload both atlas families (device linear pages, float32 RGBA) into
 * layered cudaArrays bound to bilinear texture objects (replaces the
 * 8-channel page concatenation of rasterize.py:225-236). */
int tsb_atlas_tex_create(const float* family_a, const float* family_b, int32_t page_w,
                         int32_t page_h, int32_t pages, int32_t texel_format,
                         tsb_atlas_tex_t* out, void* stream);
int tsb_atlas_tex_destroy(tsb_atlas_tex_t tex);

/* Measurement: `blocks` x `threads` threads each issue `iters` float atomic
 * adds to pseudo-random addresses of a 2^log2_floats-float buffer (the
 * gradient scatter of K8 without contention): the RED throughput peak the
 * training roofline divides by. */
int tsb_red_probe(float* buf, int32_t log2_floats, int32_t iters, int32_t blocks, int32_t threads,
                  void* stream);

/* TEX-unit throughput probe used by bench.py for the TEX roofline: `fetches`
 * bilinear RGBA fetches spread over an L1-resident window of the atlas.
 * Writes a checksum per thread into sink (grid*block floats). */
int tsb_tex_probe(tsb_atlas_tex_t tex, int32_t window, int32_t iters, float* sink,
                  int32_t blocks, int32_t threads, void* stream);

/* ---- Training backward (tsb_backward.cu) ---------------------------------- */

/* Gradient outputs. Scene parameter gradients are float64 like the
 * parameters (rasterize.py:441-451 SceneGrads); texel gradients are float32
 * in the reference's per-splat combined layout P x T x T x 7
 * (albedo.rgb, roughness, metallic, normal a, b). Accumulated into: the
 * caller zeroes them. */
typedef struct tsb_scene_grads {
  double* positions;   /* P x 3 */
  double* tangent_u;   /* P x 3 */
  double* tangent_v;   /* P x 3 */
  double* scales;      /* P x 2 */
  double* opacities;   /* P     */
  double* sh;          /* P x K x 3 */
  float* texels;       /* P x T x T x 7 (combined order), or x 8 (interleaved) */
  int32_t texel_layout; /* TSB_TEXELS_COMBINED (the reference's per-splat
                           [alb rgb, rough, metal, nrm a, nrm b]) or
                           TSB_TEXELS_INTERLEAVED (the 8-channel atlas order
                           [alb rgb, rough, nrm a, nrm b, metal, 0]) */
} tsb_scene_grads;

#define TSB_TEXELS_COMBINED 0
#define TSB_TEXELS_INTERLEAVED 1

/* environment.py:198-206 EnvGrads, float32, accumulated into. */
typedef struct tsb_env_grads {
  float* spec_mips[TSB_ENV_MAX_LEVELS];
  float* diffuse;
} tsb_env_grads;

/* Per-splat scratch bytes needed by tsb_render_backward. */
int tsb_backward_scratch_size(int32_t num_splats, uint64_t* bytes);

/* Scratch bytes for the sharded environment-gradient accumulation of
 * tsb_shade_backward (32 private copies of the env grids). */
int tsb_shade_backward_scratch_size(const tsb_environment* env, uint64_t* bytes);

/* K7: adjoint of tsb_shade_forward (replaces shading.shade_backward
 * shading.py:186-228). dcolor H x W x 3; writes every channel of the planar
 * dgbuf (13 x H x W) and accumulates environment gradients into env_grads
 * (may be NULL). With scratch (>= tsb_shade_backward_scratch_size bytes)
 * the env atomics go to per-CTA-group shards that are summed at the end;
 * scratch may be NULL (direct atomics). */
int tsb_shade_backward(const float* gbuf, const tsb_camera* camera,
                       const tsb_environment* env, const float* background,
                       const float* dcolor, float* dgbuf, tsb_env_grads* env_grads,
                       void* scratch, uint64_t scratch_bytes, void* stream);

/* K8 + K9: adjoint of the forward frame left in `workspace` by
 * tsb_render_forward in TSB_MODE_VERIFY (replaces rasterize.splat_backward
 * rasterize.py:472-593 and _finish_param_grads :642-676). dgbuf: planar
 * 13 x H x W gradient of the G-buffer; scratch: tsb_backward_scratch_size
 * bytes. Gradients are accumulated into `grads`. */
int tsb_render_backward(const tsb_scene* scene, const tsb_camera* camera,
                        const tsb_atlas* atlas, int32_t tile, const void* workspace,
                        uint64_t workspace_bytes, int64_t max_entries,
                        const tsb_pixel_state* pixels, const float* dgbuf, void* scratch,
                        tsb_scene_grads* grads, void* stream);

/* tsb_render_backward with a `deterministic` switch: the
 * reference reduces in a fixed tile order (rasterize.py:494, :646), so its
 * gradients are repeatable; the default path accumulates with float atomics
 * (order-dependent low bits). deterministic != 0 accumulates the per-splat
 * terms and texel gradients as int64 fixed point (2^-32 / 2^-40 resolution;
 * integer adds commute), so two runs give bitwise-equal gradients.
 * det_scratch: tsb_backward_det_scratch_size bytes (ignored otherwise). */
int tsb_render_backward_ex(const tsb_scene* scene, const tsb_camera* camera,
                           const tsb_atlas* atlas, int32_t tile, const void* workspace,
                           uint64_t workspace_bytes, int64_t max_entries,
                           const tsb_pixel_state* pixels, const float* dgbuf, void* scratch,
                           tsb_scene_grads* grads, int32_t deterministic, void* det_scratch,
                           uint64_t det_scratch_bytes, void* stream);

/* Diagnostics (synchronous): reads the number of global atomic adds the
 * backward rasterizer issued since the last call into *count (may be NULL),
 * resets it, and switches counting on (enable != 0) or off. */
int tsb_debug_red_count(int32_t enable, unsigned long long* count);

/* Scratch bytes of the deterministic backward for P splats at T x T texels
 * in `texel_layout` (TSB_TEXELS_COMBINED / TSB_TEXELS_INTERLEAVED). */
int tsb_backward_det_scratch_size(int32_t num_splats, int32_t T, int32_t texel_layout,
                                  uint64_t* bytes);

/* ---- Training-step glue (K10-K13) ------------------------------------- */

/* Scratch bytes of tsb_loss_image for a W x H image. */
int tsb_loss_scratch_size(int32_t width, int32_t height, uint64_t* bytes);

/* K10: image loss of a training step (replaces losses.image_loss
 * losses.py:120-134 composed with linear_to_display / _grad :24-37 as in
 * compute_step training.py:143-146). color: linear H x W x 3 (the shaded
 * image), target: display-space H x W x 3. Writes dcolor (H x W x 3) =
 * d loss / d color and ADDS into terms (device doubles, zero them first):
 * terms[0] += sum |disp - target|, terms[1] += sum SSIM map,
 * terms[2] += sum (clip(disp) - clip(target))^2 (for PSNR); each over the
 * 3 W H values. loss_image = (1-w) terms[0]/N + w (1 - terms[1]/N)/2. */
int tsb_loss_image(const float* color, const float* target, int32_t width, int32_t height,
                   float dssim_weight, float* dcolor, double* terms, void* scratch,
                   uint64_t scratch_bytes, void* stream);

/* K11: normal-consistency and smoothness regularisers of compute_step
 * (training.py:147-172; losses.py:147-277). gbuf: planar 13 x H x W G-buffer
 * of the step, target: display H x W x 3. ADDS their gradients into the
 * planar dgbuf (normal channels 5..7, depth 11, alpha 12) and into terms:
 * terms[3] += sum (1 - n.n_ref) and terms[4] += count over valid pixels,
 * terms[5] += sum w |dn| and terms[6] += pair count (the losses are
 * terms[3]/max(terms[4],1) and terms[5]/max(terms[6],1)). */
int tsb_loss_regularizers(const float* gbuf, const float* target, const tsb_camera* camera,
                          float normal_weight, float smooth_weight, float* dgbuf, double* terms,
                          void* stream);

/* K12: one Adam step (training.py:69-100 Adam.step) over up to
 * TSB_ADAM_MAX_GROUPS parameter groups in one launch, each followed by its
 * projection (clip to [0,1] or a floor, training.py:270-293). Gradients are
 * float32; parameters and moments are float32 or float64 (dtype). */
#define TSB_ADAM_MAX_GROUPS 24
#define TSB_F32 0
#define TSB_F64 1
/* float32 texels in the 8-channel interleaved order (count = P*T*T*8) with
 * float32 gradients in the 7-channel combined order (P*T*T*7) */
#define TSB_F32_TEX87 2
#define TSB_CLAMP_NONE 0
#define TSB_CLAMP_UNIT 1
#define TSB_CLAMP_FLOOR 2
typedef struct tsb_adam_group {
  void* param;          /* count elements of dtype */
  const float* grad;    /* count float32 */
  void* m;              /* first moment, dtype */
  void* v;              /* second moment, dtype */
  int64_t count;
  double lr;
  double floor;         /* TSB_CLAMP_FLOOR */
  int32_t dtype;
  int32_t clamp;
} tsb_adam_group;
int tsb_adam_step(const tsb_adam_group* groups, int32_t num_groups, int32_t step, double beta1,
                  double beta2, double eps, void* stream);

/* K12 with a divergence guard: no update when *halt != 0 (device int32, set
 * by tsb_guard_finite), so a diverged step leaves the parameters as the
 * reference's train() leaves them when it raises (training.py:263-265). */
int tsb_adam_step_ex(const tsb_adam_group* groups, int32_t num_groups, int32_t step,
                     double beta1, double beta2, double eps, const int32_t* halt, void* stream);

/* K13: Gram-Schmidt re-orthonormalisation of the tangent frames
 * (Scene.renormalize_tangents, splats.py:382-392), in place, float64. */
int tsb_orthonormalize_tangents(int32_t num_splats, double* tangent_u, double* tangent_v,
                                void* stream);
int tsb_orthonormalize_tangents_ex(int32_t num_splats, double* tangent_u, double* tangent_v,
                                   const int32_t* halt, void* stream);

/* ---- train() loop glue (training.py:187-322) -------------------------- */

/* Sets *halt = 1 if any of terms[0..n) is not finite (the loss guard of
 * training.py:263-265, evaluated on the device: no host sync per step). */
int tsb_guard_finite(const double* terms, int32_t n, int32_t* halt, void* stream);

/* Stage-2 chart growth (broadcast_textures, training.py:201-221) of texels in
 * the 8-channel interleaved (P, T, T, 8) float32 layout: T0 x T0 -> T x T,
 * each texel repeated T/T0 times per axis (or texel (0,0) repeated when T is
 * not a multiple of T0). src and dst must not overlap. */
int tsb_broadcast_texels(int32_t num_splats, int32_t T0, int32_t T, const float* src, float* dst,
                         void* stream);

/* Opacity pruning (_prune, training.py:187-198): keeps, in order, the rows
 * whose opacity > threshold, gathering each buffer's rows from src into dst
 * (parameters, texels, Adam moments: any row size); *kept (device int32)
 * receives the kept count. scratch: tsb_prune_scratch_size bytes. */
typedef struct tsb_row_buffer {
  const void* src;
  void* dst;
  int64_t row_bytes;
} tsb_row_buffer;
int tsb_prune_scratch_size(int32_t num_splats, uint64_t* bytes);
int tsb_prune_rows(int32_t num_splats, const double* opacities, double threshold,
                   const tsb_row_buffer* bufs, int32_t num_bufs, int32_t* kept, void* scratch,
                   uint64_t scratch_bytes, void* stream);

/* ---- Environment precompute (K15-K16) ---------------------------------- */

/* Scratch bytes of tsb_env_prefilter for a height x width base map. */
int tsb_env_scratch_size(int32_t height, int32_t width, uint64_t* bytes);

/* EnvironmentLight.from_base (environment.py:231-244) on the device: from a
 * float64 base radiance map (height x width x 3, device), level 0 = the base
 * (float32), level l >= 1 = GGX prefilter with roughness l/(levels-1)
 * (prefilter_specular :145-175) at mip_h[l] x mip_w[l], and the cosine
 * irradiance (diffuse_irradiance :178-195) at diff_h x diff_w, all over the
 * 2x-downsampled base, fp64 sums. Outputs float32 x 3; any may be NULL. */
int tsb_env_prefilter(const double* base, int32_t height, int32_t width, int32_t levels,
                      float* const* spec_mips, const int32_t* mip_h, const int32_t* mip_w,
                      float* diffuse, int32_t diff_h, int32_t diff_w, void* scratch,
                      uint64_t scratch_bytes, void* stream);

/* BrdfLut.build (environment.py:381-425) on the device: table (resolution x
 * resolution x 2, float64, device) of split-sum (A, B), GGX importance
 * sampling over `samples` Hammersley points per cell. */
int tsb_brdf_lut(int32_t resolution, int32_t samples, double* table, void* stream);

/* K14: the decomposition images of the render command (cli.py:52-96 with
 * --decompose) as 8-bit pixels: out holds, back to back, albedo (H x W x 3),
 * normal (H x W x 3), roughness (H x W), metallic (H x W), diffuse,
 * specular and final (H x W x 3 each) — 17 W H bytes — quantised like
 * write_png (imgio.py:13-21) after linear_to_display where the reference
 * applies it. gbuf planar 13 x H x W; colour/diffuse/specular H x W x 3. */
int tsb_decompose(const float* gbuf, const float* color, const float* diffuse,
                  const float* specular, int32_t width, int32_t height, uint8_t* out,
                  void* stream);

/* Last error message of the calling thread. */
const char* tsb_last_error(void);

/* Library version string. */
const char* tsb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TSB_H */
