/*
 * softmpm_b200.h -- C ABI of the B200-native MLS-MPM substep.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * package (softmpm, /root/reference/pkg/src/softmpm) has no native ABI: its
 * "operator ABI" is the set of numba kernels called by core.py with flat
 * numpy arrays.  Each entry point below names the reference interface it
 * replaces.  Conventions:
 *   - every function returns 0 on success, a negative MPM_E* code otherwise;
 *     mpm_last_error(ctx) holds the message;
 *   - host arrays are the reference's fp64 C-order numpy layouts
 *     (x/v (n,3), F/C (n,3,3) row-major, grid_mv (nx,ny,nz,3), grid_m
 *     (nx,ny,nz)); they are borrowed for the duration of the call only;
 *   - particle order on the host is always the caller's original order; the
 *     device keeps its own binned permutation;
 *   - calls are synchronous with respect to the host buffers passed in and
 *     may be made from any host thread (each call sets the device itself).
 */
#ifndef SOFTMPM_B200_H
#define SOFTMPM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPM_OK 0
#define MPM_EINVAL -1   /* invalid argument -> softmpm.errors.ParameterError */
#define MPM_ENOMEM -2   /* device/host allocation failed -> SimError */
#define MPM_ECUDA -3    /* CUDA runtime error -> SimError */
#define MPM_ESTATE -4   /* call out of order (e.g. no particles) -> SimError */
#define MPM_ESTENCIL -5 /* particle outside the 1.5-cell margin -> StencilError */

/* field masks for upload/download */
#define MPM_FIELD_X 1u
#define MPM_FIELD_V 2u
#define MPM_FIELD_F 4u
#define MPM_FIELD_C 8u
#define MPM_FIELD_ALL 15u

/* stress forms */
#define MPM_STRESS_KERNEL 0 /* P = mu F + ((lam lnJ - mu)/J) cof^T : kernels.py:253-262 */
#define MPM_STRESS_SPEC 1   /* P = mu (F - F^-T) + lam lnJ F^-T  : materials.py:59-60  */

typedef struct mpm_ctx mpm_ctx;

/* Mirrors Grid (core.py:24-56) + SimParams (core.py:59-79) + build options. */
typedef struct {
  int device;
  int res[3];           /* Grid.resolution */
  double dx;            /* Grid.dx (uniform) */
  double dt;            /* SimParams.dt */
  double gravity[3];    /* SimParams.gravity */
  int boundary_width;   /* SimParams.boundary_width */
  int stick;            /* SimParams.boundary == "stick" */
  double theta;         /* collision band; < 0 disables (core.py:290-291) */
  int stress_form;      /* MPM_STRESS_* */
  int mode_live;        /* 0: collider mode frozen at first pack (F7 compat), 1: live */
  int deterministic;    /* 1: sorted deterministic-order P2G (bit-exact grid mass) */
  int rebin_interval;   /* substeps between particle re-binning (fast mode), >= 1 */
  /* Batched independent environments (BASELINE config 4): the grid is
   * env_tiles[0] x env_tiles[1] x env_tiles[2] tiles of res/env_tiles nodes,
   * one environment per tile with its own domain walls and margins; the
   * collider table holds colliders_per_env colliders per tile, tile-major.
   * {0,0,0} or {1,1,1}: one environment. */
  int env_tiles[3];
  int colliders_per_env; /* 0: every collider acts on the whole grid */
} mpm_config;

/* ---- lifetime ---------------------------------------------------------- */
int mpm_create(mpm_ctx **out, const mpm_config *cfg);
int mpm_destroy(mpm_ctx *ctx);
/* Replace dt/gravity/boundary/theta/stress options (SimParams changes between calls). */
int mpm_set_config(mpm_ctx *ctx, const mpm_config *cfg);
const char *mpm_last_error(mpm_ctx *ctx);
const char *mpm_version(void);

/* ---- materials: replaces materials.pack_materials (materials.py:77-82) --- */
int mpm_set_materials(mpm_ctx *ctx, const double *mu, const double *lam, int count);

/* ---- particle state: SimState x/v/F/C/mass/vol0/material_id (core.py:92-143)
 * n = 0 is a valid (empty) state, as in the reference: substeps then run the
 * grid stages on an empty grid and particle transfers are no-ops. */
int mpm_upload_particles(mpm_ctx *ctx, int64_t n, const double *x, const double *v,
                         const double *F, const double *C, const double *mass,
                         const double *vol0, const int32_t *material_id);
/* Overwrite a subset of x/v/F/C (host-side edits of SimState fields).
 * mask bits 0..3 select x, v, F, C (NULL pointers are skipped).  Pageable
 * buffers and transfers of >= 2^20 values are narrowed to fp32 on host
 * worker threads and cross PCIe as fp32; small pinned ones cross as fp64 and
 * are converted on the device (option "host_xfer"; the same
 * round-to-nearest values either way). */
int mpm_upload_fields(mpm_ctx *ctx, uint32_t mask, const double *x, const double *v,
                      const double *F, const double *C);
/* Download a subset of x/v/F/C in the caller's particle order.  mask bit 4
 * (MPM_DOWNLOAD_KEEP_EQUAL): a destination value whose fp32 rounding equals
 * the device value is left as it is (the device left it unchanged: the
 * caller keeps its fp64 value), others get the device value. */
#define MPM_DOWNLOAD_KEEP_EQUAL 16u
int mpm_download_particles(mpm_ctx *ctx, uint32_t mask, double *x, double *v, double *F,
                           double *C);
int64_t mpm_particle_count(mpm_ctx *ctx);

/* ---- grid: SimState.grid_mv / grid_m (core.py:106-117) ------------------ */
/* target 0: the momentum buffer read by grid_update, 1: the velocity buffer
 * read by g2p_advect.  grid_m may be NULL (target 1). */
int mpm_upload_grid(mpm_ctx *ctx, int target, const double *grid_mv, const double *grid_m);
/* Download grid_mv as SimState shows it after the last stage, and grid_m. */
int mpm_download_grid(mpm_ctx *ctx, double *grid_mv, double *grid_m);

/* ---- colliders: replaces collision.pack_colliders / PackedColliders
 *      (collision.py:174-241).  Geometry is static; poses change per substep. */
int mpm_set_colliders(mpm_ctx *ctx, int count, const int32_t *kind, const double *half,
                      const double *rotation, const double *translation,
                      const double *linear_velocity, const double *angular_velocity,
                      const double *friction, const int32_t *mode, const double *sdf_values,
                      int64_t sdf_len, const int64_t *sdf_offset, const int32_t *sdf_resolution,
                      const double *sdf_bounds_min, const double *sdf_extent);
/* Pose table for the next `nsub` substeps (PackedColliders.refresh_poses per
 * substep, collision.py:192-197); arrays are (nsub, count, ...).  mode may be
 * NULL (keep the packed/frozen mode). */
int mpm_set_pose_table(mpm_ctx *ctx, int nsub, const double *rotation,
                       const double *translation, const double *linear_velocity,
                       const double *angular_velocity, const int32_t *mode);

/* ---- stage operators (core.py:211-258; kernels.py:198-534) --------------- */
/* p2g_scatter + p2g_reduce: F advanced in place; *inverted = det<=0 count. */
int mpm_p2g(mpm_ctx *ctx, int64_t *inverted);
/* kernels.grid_update with the collision field of build_collision_field
 * evaluated lazily at massive nodes; use_colliders selects pose row 0. */
int mpm_grid_update(mpm_ctx *ctx, int use_colliders);
/* kernels.g2p_advect */
int mpm_g2p(mpm_ctx *ctx);

/* ---- fused driver: core.substep x nsub (core.py:261-320) ---------------- */
/* Runs nsub substeps device-resident; colliders use pose row s at substep s
 * when use_colliders.  *inverted = summed det<=0 count; stage_ms (may be
 * NULL) receives device milliseconds of the whole sequence. */
int mpm_substeps(mpm_ctx *ctx, int nsub, int use_colliders, int64_t *inverted,
                 double *device_ms);

/* Peer-memory halo exchange (NVLink P2P / CUDA IPC), the device-side
 * alternative to mpm_halo_pack / unpack_* + a host transport.  Per side the
 * context exports its receive buffers and two interprocess events as an
 * mpm_ipc_blob_size() byte blob (mpm_ipc_export) that the neighbour maps
 * (mpm_ipc_import with its opposite side).  mpm_ipc_halo(phase, sides):
 * 0 packs our ghost momentum straight into each neighbour's buffers, 1 adds
 * what the neighbours wrote into ours, 2 writes the velocities of those
 * bricks back into the neighbours, 3 applies the velocities we received; all
 * stream-ordered with event waits, counts stay on the device.  The caller
 * orders each phase pair (0 before the neighbours' 1, 2 before their 3) with
 * a host barrier, so that every event wait follows the record it needs. */
int64_t mpm_ipc_blob_size(void);
int mpm_ipc_export(mpm_ctx *ctx, int side, void *blob);
int mpm_ipc_import(mpm_ctx *ctx, int side, const void *peer_blob);
int mpm_ipc_halo(mpm_ctx *ctx, int phase, int sides);
/* 1 when mpm_ipc_halo orders the neighbours' streams by itself (stream
 * memory operations: a wait on our counter, a write into the neighbour's,
 * no host barrier per substep); 0 on the interprocess-event fallback
 * (SOFTMPM_IPC_EVENTS set, or no driver entry points), where the caller
 * barriers between phases 0/1 and 2/3. */
int mpm_ipc_mode(mpm_ctx *ctx, int *device_ordered);
/* Same-process neighbours (several windows driven by one process, on one GPU
 * or on peer-accessible GPUs): wires window a's `side` neighbour to b (and
 * b's opposite side to a) with direct device pointers instead of IPC
 * handles.  mpm_ipc_halo then runs the same kernels with the streams ordered
 * by plain events (a stream-value wait could block a later-issued signal of
 * another stream of the process that aliases its hardware queue); the caller
 * issues each halo phase for every window before the next phase. */
int mpm_peer_connect(mpm_ctx *a, int side, mpm_ctx *b);

/* ---- slab decomposition (BASELINE config 5) ------------------------------
 * A context can own an x-window of a larger global grid: its res[0] nodes
 * start at global node offset[0] (multiple of 4) and include `ghost_bricks`
 * 4-node brick layers on each side owned by the neighbouring windows.  Walls,
 * colliders and margins use global coordinates; device particle positions
 * are window-local.  Per substep the driver calls
 *   mpm_stage_particles -> mpm_halo_pack (both sides) -> exchange ->
 *   mpm_halo_unpack_add -> mpm_stage_grid -> mpm_halo_pack_vel -> exchange ->
 *   mpm_halo_unpack_vel
 * (exchange = NCCL send/recv of the buffers of mpm_halo_buffers, or device
 * copies between contexts of one process), and at stretch boundaries
 * mpm_stage_end -> mpm_extract_migrants -> exchange -> mpm_append_particles ->
 * mpm_stage_begin.  Replaces nothing in the reference (single-process CPU). */
int mpm_set_slab(mpm_ctx *ctx, const int *global_res, const int *offset, int ghost_bricks);
int mpm_halo_buffers(mpm_ctx *ctx, int side, void **send_ids, void **send_data, void **recv_ids,
                     void **recv_data, int64_t *capacity);
int mpm_stage_begin(mpm_ctx *ctx, int nsub, int use_colliders);
int mpm_stage_particles(mpm_ctx *ctx, int first);
int mpm_stage_grid(mpm_ctx *ctx, int sub, int clear);
int mpm_stage_end(mpm_ctx *ctx, int64_t *inverted);
int mpm_halo_pack(mpm_ctx *ctx, int side, int64_t *count);
int mpm_halo_unpack_add(mpm_ctx *ctx, int side, int64_t n);
int mpm_halo_pack_vel(mpm_ctx *ctx, int side, int64_t *count);
int mpm_halo_unpack_vel(mpm_ctx *ctx, int side, int64_t n);
/* Migrants leave in two packed device row blocks (one per neighbour): field
 * q of migrant d at rows[q * n + d], n = that side's count, 28 fields (26
 * floats, material id, particle id) -- one contiguous copy per neighbour;
 * *rows_cap is set to 0 (the stride is the count).  An emptied window keeps
 * running (grid + halos) and can receive migrants. */
int mpm_extract_migrants(mpm_ctx *ctx, int own_lo, int own_hi, int64_t *n_lo, int64_t *n_hi,
                         void **rows_lo, void **rows_hi, int64_t *rows_cap);
int mpm_append_particles(mpm_ctx *ctx, const void *rows, int64_t m, int64_t rows_cap, int src_offset);
int mpm_reserve(mpm_ctx *ctx, int64_t capacity);
int mpm_download_ids(mpm_ctx *ctx, int32_t *ids, double *x);
int mpm_device_copy(void *dst, const void *src, int64_t bytes);
/* Slab windows identify particles by global id: */
int mpm_set_ids(mpm_ctx *ctx, const int32_t *ids);
int mpm_download_rows(mpm_ctx *ctx, int32_t *ids, double *x, double *v, double *F, double *C);

/* ---- diagnostics -------------------------------------------------------- */
/* update_collision_field (collision.py:244-272) over all nodes, current pose
 * row 0; dist (nx,ny,nz) f64, obj (nx,ny,nz) i32, cap = 2 theta. */
int mpm_collision_field(mpm_ctx *ctx, double theta, double *dist, int32_t *obj);
/* SimState.has_nan (core.py:149-151) on device. */
int mpm_has_nan(mpm_ctx *ctx, int *flag);

/* compute_metrics (scene.py:204-220) as a device reduction: out[5] =
 * {lifted_fraction (dy > 2 dx), detached_fraction (dy > dx),
 *  mean |det F - 1|, max |x - x0|, particle count}.  x0: the caller's
 * (n, 3) fp64 reference positions in caller order, uploaded into the context;
 * NULL reuses the last upload (MPM_ESTATE if none for this particle count). */
int mpm_metrics(mpm_ctx *ctx, const double *x0, double dx, double *out);

/* splat_density (surfacing.py:45-67 -> kernels.splat_mass / splat_reduce,
 * kernels.py:541-588): quadratic B-spline mass deposit on a dense res[0] x
 * res[1] x res[2] lattice of spacing field_dx, divided by field_dx^3; out is
 * the (res0, res1, res2) C-order fp64 density.  positions == NULL: the
 * context's particles (no download); else caller (n, 3) positions + (n,)
 * masses.  fp64 weights, fp64 atomic accumulation (node sums in arrival
 * order, not the reference's chunk order). */
int mpm_splat_density(mpm_ctx *ctx, const double *positions, const double *masses, int64_t n,
                      const int32_t *res, double field_dx, double *out);
/* The density field also stays on the device (out may be NULL) as the input
 * of mpm_marching_cubes(values = NULL). */
/* Same without a simulation context (temporary device buffers on `device`). */
int mpm_splat_density_host(int device, const double *positions, const double *masses, int64_t n,
                           const int32_t *res, double field_dx, double *out);

/* marching_cubes (surfacing.py:70-95; scikit-image's Lorensen tables in the
 * reference) on the device: isosurface at `iso` of the dense fp64 field
 * (values: host (res0, res1, res2) C-order array, or NULL for the context's
 * last splatted field).  Indexed mesh, one vertex per crossed lattice edge,
 * counter-clockwise triangles seen from the outside (value < iso) and unit
 * outward normals; the counts come back here, the arrays via mpm_mesh_fetch. */
int mpm_marching_cubes(mpm_ctx *ctx, const double *values, const int32_t *res, double dx, double iso,
                       int64_t *nverts, int64_t *ntris);
int mpm_mesh_fetch(mpm_ctx *ctx, double *verts, int32_t *tris, double *normals);
/* encode_frame (server.py:65-92) body from the last mesh, packed on the device:
 * f32 vertices (3V), f32 normals (3V), f32 planar UVs (2V; compute_uvs,
 * surfacing.py:92-101, against extent[3]) and u32 triangle indices (3T),
 * little-endian, back to back -- 32 V + 12 T bytes into out (host memory,
 * cap bytes).  *len receives the size; out = NULL only queries it.  The MPMF
 * header and collider records around it are assembled by the caller. */
int mpm_mesh_encode(mpm_ctx *ctx, const double *extent, uint8_t *out, int64_t cap, int64_t *len);
/* Per-kernel CUDA-event timing on the context stream (bench/roofline).
 * When enabled every fast-path launch is bracketed by events; mpm_get_timing
 * fills out[16] = {g2p_stress_ms, g2p_stress_launches, grid_op_ms,
 * grid_op_launches, rebin_ms, rebin_calls, g2p_ms, g2p_launches,
 * active_bricks_last, work_items_last, p2g_tile_ms, p2g_tile_launches,
 * fused_ms, fused_launches, substeps_kernel_ms, substeps_kernel_substeps}
 * accumulated since the last enable, and resets them. */
int mpm_set_timing(mpm_ctx *ctx, int enable);
int mpm_get_timing(mpm_ctx *ctx, double *out);
/* Runtime options: "graphs" (1 = replay fast-path frames as CUDA graphs,
 * default), "split" (1 = stage A + stage B every substep instead of the fused
 * kernel; A/B comparisons), "mega" (1 = substeps 2..L of a stretch as one
 * cooperative kernel with grid barriers between the fused and grid-op
 * phases; pays off for small scenes, e.g. +12% at 30 K particles), "pdl"
 * (1 = fused kernel and grid op launched with programmatic dependent launch,
 * each kernel's prologue overlapping its predecessor's tail; on by default:
 * +1% at C3 with the plain grid op, within noise at C4 / C5), "rebin_frames"
 * (k >= 1: a frame of an untouched state keeps the particle order of a
 * re-binning up to k - 1 frames old; default 1 -- k = 2 gains 1-1.6% on the
 * settling C4 / C5 scenes but loses 7% on the pressed C3 slab, whose cells
 * compress between re-binnings), "host_xfer" (1 = particle uploads /
 * downloads of pageable buffers or >= 2^20 values are converted on host
 * worker threads and cross PCIe as fp32, the default; 0 = always fp64 over
 * PCIe with device conversion; SOFTMPM_HOST_THREADS sets the worker count,
 * default min(16, hardware threads)), "gridop_simple"
 * (1 = warp-per-brick grid op, the default; 0 = the prefetching persistent
 * kernel), "fx_shift" (test hook, 0..8: loosen
 * the node-sum term of the fixed-point P2G scale by 2^value and divide the
 * per-cell count limit of its overflow guard by the same factor, so the
 * guard's float fallback is exercised on ordinary scenes; 0 in production). */
int mpm_set_option(mpm_ctx *ctx, const char *key, int value);
/* Cumulative device statistics of the context: index 0 = particles the
 * fixed-point overflow guard sent down the float scatter path (their base
 * cell already held the item's count limit, 2 x the densest cell at
 * re-binning).  No reference counterpart (the reference scatters in fp64,
 * kernels.py:296-313). */
int mpm_get_stat(mpm_ctx *ctx, int index, int64_t *out);
/* Kernel launches issued by this context so far (evidence counter; a graph
 * replay counts every kernel node it runs). */
int64_t mpm_launch_count(mpm_ctx *ctx);
/* Page-locked host buffer for fast uploads/downloads (e2e path). */
void *mpm_host_alloc(int64_t bytes);
void mpm_host_free(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* SOFTMPM_B200_H */
