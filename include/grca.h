/*
 * include/grca.h -- C ABI of the B200-native GRCA hot path (libgrca.so).
 *
 * The operation ("Problem Statement"): a LiDAR fires rays
 * into a scene of triangles; "for each ray the simulation must find the
 * closest triangle it intersects and its distance", with no acceleration
 * structure: each triangle's emitter-centric angular footprint selects the
 * channels and the ray range it can hit (Observations 1-2;
 * SURVEY.md 8(a) rows A0-A9), and only those (triangle, ray) pairs are tested.
 *
 * Conventions
 *  - Emitter n has gamma_n channels (elevations phi_j, ascending) and chi_n rays
 *    per channel; ray (n, j, i) has global index g = O_n + j*chi_n + i with
 *    O_n = sum_{m<n} gamma_m chi_m.  Direction (PAPER.md:418-435,
 *    Eq. ray_dir): d = RN32(cos(th_i)cos(phi_j) f + sin(th_i)cos(phi_j) r + sin(phi_j) u)
 *    evaluated in fp64, th_i = -floor(chi/2)*dth + i*dth, dth = H/chi, H = 2*pi (360 deg)
 *    or pi (180 deg).  The reported distance is the ray parameter t of that d.
 *  - Hit: closed triangle, 0 < t <= max_range, two-sided unless `faces` says
 *    otherwise; per ray the minimum t wins, equal fp32 t -> smaller triangle id.
 *    Miss: distance +inf, id -1.
 *  - Results are exact up to rounding: no culling approximation is applied
 *    (SURVEY 8(c)); see DESIGN.md for the precision contract.
 *
 * Errors: every call returns grca_status; nothing throws across the ABI.
 * grca_last_error(h) returns a message for the last failing call on h.
 * A handle is not thread-safe; distinct handles are independent.
 */
#ifndef GRCA_H
#define GRCA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct grca_ctx *grca_t;

typedef enum {
    GRCA_OK = 0,
    GRCA_E_INVALID = 1,  /* bad argument (see grca_last_error) */
    GRCA_E_STATE = 2,    /* call order: cast before set_emitters / update_triangles */
    GRCA_E_CAPACITY = 3, /* counts above the capacities fixed at create */
    GRCA_E_CUDA = 4,     /* a CUDA runtime error (message has cudaGetErrorString) */
    GRCA_E_NCCL = 5,     /* an NCCL call of the in-library collective failed (message has the NCCL error) */
    GRCA_E_OOM = 6       /* device allocation failed at create */
} grca_status;

/* Face modes (PAPER.md:614-620 back-face rule).  N = (v1-v0)x(v2-v0). */
enum {
    GRCA_FACES_TWO_SIDED = 0, /* default: both sides hit */
    GRCA_FACES_KEEP_POS = 1,  /* keep hits with d.N > 0  <=> (c - o).N > 0 */
    GRCA_FACES_KEEP_NEG = 2   /* keep hits with d.N < 0 */
};

/* Debug / instrumentation flags (grca_create_info.debug_flags). */
enum {
    GRCA_DEBUG_COUNT_ALL_HITS = 1u, /* per-ray count of every accepted hit (all-hits invariant) */
    GRCA_DEBUG_NO_CULL = 2u,        /* every (tri, emitter) pair tests the full ray grid */
    GRCA_PROFILE_KERNELS = 4u,      /* CUDA events around each kernel; see grca_kernel_times */
    GRCA_DEBUG_FORCE_FP64 = 8u,     /* every candidate takes the fp64 path (precision check) */
    GRCA_DEBUG_SPLIT_REFINE = 16u,  /* run K2b (bounds) and K4s (small work) as two kernels instead of
                                       the fused refine+small kernel (A/B measurement, same results) */
    GRCA_DEBUG_NO_REFINE = 32u,     /* K3 keeps whole rectangle rows (no A7 per-channel refinement) */
    GRCA_DEBUG_NO_PACKED = 128u,    /* K2 without the packed fp32x2 (two-emitter) path (A/B) */
    GRCA_USE_CUDA_GRAPH = 512u,      /* grca_cast runs its launch sequence as one CUDA graph (captured per cast,
                                        cudaGraphExecUpdate'd in place; needs a non-NULL stream; ignored with
                                        GRCA_PROFILE_KERNELS or inside a caller's stream capture, where the
                                        cast's launches are recorded into the caller's graph instead) */
    GRCA_DEBUG_VIRTUAL_RANKS = 256u, /* nranks > 1 without nccl_uid: the handle casts exactly rank's share of the
                                        partition (shard_mode / merge as with a communicator) and writes the
                                        outputs that rank would write, but runs no collective (the caller merges;
                                        one-GPU tests and per-rank timing of a P-rank run) */
    GRCA_L2_PERSIST = 64u           /* opt-in: reserve persisting L2 for the ray table + hit keys
                                       (raises cudaLimitPersistingL2CacheSize device-wide and sets a
                                       per-launch access-policy window on the gather kernels) */
};

/* Multi-GPU partition of a collective cast (the paper itself is single-GPU).
 * The per-ray closest hit is a min over triangles (a lattice), so any triangle partition merges exactly
 * by an element-wise min of the packed (t, id) keys. */
enum {
    GRCA_SHARD_AUTO = 0,      /* EMITTERS when n_emitters >= nranks and nranks | n_emitters, else TRIANGLES */
    GRCA_SHARD_TRIANGLES = 1, /* each rank passes its own triangle shard (global ids); grca_cast merges */
    GRCA_SHARD_EMITTERS = 2   /* each rank passes every triangle; emitter n is cast by rank n mod nranks */
};
/* How a triangle-sharded cast merges (in-stream, between K4 and K5). */
enum {
    GRCA_MERGE_ALLREDUCE = 0,      /* ncclAllReduce(keys, ncclUint64, ncclMin): every rank gets every ray */
    GRCA_MERGE_REDUCE_SCATTER = 1, /* ncclReduceScatter(ncclMin): rank r gets rays [r c, r c + c), c = ceil(n / P),
                                      half the traffic; only that slice of the outputs is written */
    GRCA_MERGE_NVLS = 2            /* fused: the intersection kernels record hits with multimem.red.min.u64 into
                                      an NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister + the lsa
                                      multimem pointer), no separate reduction (NEXT-f3); needs NVLS multicast */
};

typedef struct {
    int32_t device;          /* CUDA device ordinal */
    void *stream;            /* cudaStream_t all work is enqueued on (e.g. torch's current stream);
                                NULL -> the legacy default stream */
    int32_t nranks, rank;    /* collective cast over nranks processes (one GPU each); 1, 0 for one GPU */
    const void *nccl_uid;    /* 128-byte ncclUniqueId (grca_nccl_unique_id on one rank, broadcast by the caller;
                                the library copies it).  Non-NULL -> grca_create builds an NCCL communicator
                                (ncclCommInitRank: every rank must call grca_create) and grca_cast is collective.
                                Required when nranks > 1; allowed with nranks == 1 (a one-rank communicator) */
    int32_t shard_mode;      /* GRCA_SHARD_* (used with a communicator) */
    int32_t merge;           /* GRCA_MERGE_* (triangle shards) */
    int32_t gather_outputs;  /* emitter shards: 1 -> ncclBroadcast every emitter's keys from its owner so every
                                rank's outputs hold every ray; 0 -> each rank writes only its emitters' rays */
    int64_t max_triangles;   /* per handle; fixes scratch sizes so grca_cast never allocates */
    int64_t max_rays;        /* upper bound of sum_n gamma_n chi_n */
    int64_t max_large_items; /* capacity of the large-pair list (0 -> default); overflow is
                                handled inline (slower, never dropped) and counted in stats */
    int32_t faces;           /* GRCA_FACES_* */
    uint32_t debug_flags;    /* GRCA_DEBUG_* | GRCA_PROFILE_KERNELS */
    int32_t small_max;       /* pairs with <= small_max candidates (<= 1023) take the small-rectangle
                                path (K4s); larger ones are chunked (K3/K4).  0 -> default 512 */
    float apparent_area_eps; /* NEXT-f1 paper mode, APPROXIMATE: skip a (triangle, emitter) pair when
                                (A_T (c-o).n)^2 < eps^2 |c-o|^6 (eps_A = 1e-6 there;
                                |.| of (c-o).n in two-sided mode).  0 -> off (exact results) */
    int32_t reserved[4];
} grca_create_info;

/* One spinning LiDAR (ray origin); SPEC SensorConfig. */
typedef struct {
    float origin[3];
    float forward[3], right[3], up[3]; /* orthonormal within 1e-3 (any such frame is exact) */
    const float *channel_elev_rad;     /* host pointer, gamma entries, strictly ascending,
                                          |phi| <= RN32(pi/2); copied by grca_set_emitters */
    int32_t n_channels;                /* gamma_n in [1, 65535] */
    int32_t rays_per_channel;          /* chi_n in [1, 65535] */
    int32_t hfov_deg;                  /* 360 or 180 */
    float max_range;                   /* D_max > 0; <= 0 or +inf -> unlimited */
    const float *ray_azimuth_rad;      /* NULL -> grid theta_i = -floor(chi/2) dth + i dth; else the noise
                                          model's pre-stored perturbed azimuths theta*_i (chi entries,
                                          strictly ascending, |theta*_i - theta_i| < dth; PAPER.md:
                                          2276-2283).  Per-channel elevation noise = the elevation table */
} grca_emitter;

/* Per-cast counters (SURVEY 5 "Metrics"; Eq. 1 and 2131-2144 Eq. rtic_reduced). */
typedef struct {
    int64_t pairs;           /* (triangle, emitter) pairs considered = tau * Omega */
    int64_t range_culled;    /* dropped by Step 1.3 range cull */
    int64_t channel_culled;  /* no channel in the elevation interval */
    int64_t azimuth_culled;  /* no ray in the azimuth arc, degenerate, or face mode */
    int64_t survivors;       /* pairs with >= 1 candidate */
    int64_t small_pairs;     /* tested inline by the cull kernel */
    int64_t large_pairs;     /* binned to the large list */
    int64_t chunks;          /* load-balanced work chunks made from the large list */
    int64_t rtic_tested;     /* ray-triangle tests performed (candidates) */
    int64_t rtic_brute;      /* Eq. 1: sum gamma chi * tau */
    int64_t fp64_fallbacks;  /* candidates decided by the fp64 path */
    int64_t hits_recorded;   /* accepted intersections (before the closest-hit min) */
    int64_t overflow_inline; /* large pairs processed inline because the list was full */
    int64_t prefilter_survivors; /* pairs passed by the K2 elevation pre-test to K2b */
    int64_t rtic_small;      /* part of rtic_tested done by K4s (small rectangles) */
    int64_t sat_pairs;       /* paper classification of surviving pairs (Eq. sat_cond):
                                SAT = no seam wrap and gamma_span <= 64 and chi_span <= 64 ... */
    int64_t bat_pairs;       /* ... BAT = the rest (counts only; the build bins by item count) */
    int64_t area_culled;     /* pairs skipped by the apparent-area cull (paper mode) */
    int64_t hits_large;      /* part of hits_recorded (= RED.MIN key updates issued) made by K4 / the serial
                                fallback; the rest by the fused small-rectangle kernel */
    int32_t overflow;        /* 1 if any capacity fallback happened */
    float ms_total;          /* device time of the last cast if GRCA_PROFILE_KERNELS */
    float ms_k[8];           /* per kernel: K0 init, K2 cull, K2b refine (split mode only), K2b+K4s
                                refine+small (K4s in split mode), K3 bin, K4 large, K5 unpack */
} grca_stats;

/* Create a handle bound to ci->device.  Allocates all device scratch.  With ci->nccl_uid, also the NCCL
 * communicator of the collective cast (blocks until all ci->nranks ranks have called grca_create).
 * Errors: GRCA_E_INVALID (null/negative sizes, bad faces / shard / merge mode, rank outside [0, nranks),
 * nranks > 1 without nccl_uid), GRCA_E_CUDA, GRCA_E_OOM, GRCA_E_NCCL. */
grca_status grca_create(const grca_create_info *ci, grca_t *out);

/* Write a fresh 128-byte ncclUniqueId to out (host memory) for grca_create_info.nccl_uid: call on one
 * rank, broadcast the bytes to the others (e.g. over torch.distributed).  Errors: GRCA_E_INVALID (NULL),
 * GRCA_E_NCCL. */
grca_status grca_nccl_unique_id(void *out);

/* The partition this rank casts after grca_set_emitters: *shard_mode = GRCA_SHARD_TRIANGLES or
 * GRCA_SHARD_EMITTERS (0 without a communicator), and the rays of the outputs grca_cast writes:
 * [*first_ray, *first_ray + *n_written) for triangle shards (all rays, or this rank's reduce-scatter
 * slice); for emitter shards *first_ray = -1 and *n_written = the rays of this rank's emitters (n mod
 * nranks == rank; all rays when gather_outputs).  Any pointer may be NULL.  Errors: GRCA_E_STATE
 * (before grca_set_emitters). */
grca_status grca_get_shard(grca_t h, int32_t *shard_mode, int64_t *first_ray, int64_t *n_written);

/* Destroy the handle and free its memory (synchronizes its stream).  NULL is a no-op. */
grca_status grca_destroy(grca_t h);

/* Set the emitters (copies everything; host arrays may be freed after return).  With a communicator every
 * rank passes the SAME full emitter list (collective under GRCA_MERGE_NVLS, which (re)binds its symmetric
 * window here); under emitter sharding the handle casts only its own emitters (n mod nranks == rank) but
 * keeps the global ray layout.
 * Builds the fp32 ray table in fp64 on the host (O1 above; PAPER.md:2322-2325 ray setup)
 * and uploads it with the per-emitter records and sin(phi_j) tables (synchronous).
 * Errors: GRCA_E_INVALID for n_emitters not in [1, 255], gamma/chi out of range, an
 * unsorted or non-strict elevation table, |phi| > RN32(pi/2), a non-orthonormal frame,
 * hfov not 180/360, sum over emitters of (gamma_n + 2) > 4096 (each sin table carries two +inf sentinels);
 * GRCA_E_CAPACITY if sum gamma chi > max_rays. */
grca_status grca_set_emitters(grca_t h, const grca_emitter *em, int32_t n_emitters);

/* Borrow this frame's triangles (no copy).  d_vertices: device float4 (x, y, z, w unused),
 * 16-byte stride.  d_indices: device uint32, 3 per triangle, or NULL -> non-indexed: triangle
 * k is vertices 3k, 3k+1, 3k+2.  d_tri_ids: device int32 global id per triangle, or NULL ->
 * id = tri_id_base + k.  Ids must be in [0, 2^31 - 1).  Buffers must stay alive and
 * unmodified until the cast consuming them completes on the handle's stream.
 * Errors: GRCA_E_INVALID (null vertices with n_triangles > 0, indexed with n_vertices < 1),
 * GRCA_E_CAPACITY (n_triangles > max_triangles). */
grca_status grca_update_triangles(grca_t h, const float *d_vertices, int64_t n_vertices,
                                  const uint32_t *d_indices, int64_t n_triangles,
                                  const int32_t *d_tri_ids, int32_t tri_id_base);
/* Same as grca_update_triangles with the vertices as packed float3 (x, y, z: 12 bytes each, 4-byte
 * aligned) instead of float4 -- a quarter fewer bytes to upload per frame.  Same ownership,
 * layout of indices / ids and errors (alignment: 4 bytes). */
grca_status grca_update_triangles_f3(grca_t h, const float *d_xyz, int64_t n_vertices, const uint32_t *d_indices,
                                     int64_t n_triangles, const int32_t *d_tri_ids, int32_t tri_id_base);
/* Two-part triangle set in one call (same role as grca_update_triangles; PAPER.md:146-157 casts every
 * triangle of the frame, the split is only a storage layout): triangles [0, n_soup_triangles) are
 * non-indexed float4 triplets d_soup (vertex 3k..3k+2 = triangle k; 16-byte aligned; w ignored) --
 * scenery that needs no index indirection -- and triangles [n_soup_triangles, n_soup + n_mesh) are
 * the indexed packed-float3 mesh d_mesh_xyz (n_mesh_vertices x 12 bytes, 4-byte aligned) with
 * d_mesh_indices (uint32[3 * n_mesh_triangles], local to d_mesh_xyz).  Either part may be empty
 * (its pointers are then ignored).  Triangle k of the concatenation has id d_tri_ids[k] or
 * tri_id_base + k.  Ownership as grca_update_triangles.  Errors: GRCA_E_INVALID (negative counts,
 * misaligned or missing buffers of a non-empty part), GRCA_E_CAPACITY (n_soup + n_mesh >
 * max_triangles). */
grca_status grca_update_scene(grca_t h, const float *d_soup, int64_t n_soup_triangles, const float *d_mesh_xyz,
                              int64_t n_mesh_vertices, const uint32_t *d_mesh_indices, int64_t n_mesh_triangles,
                              const int32_t *d_tri_ids, int32_t tri_id_base);

/* Rigid instances (ABI extension named in SURVEY 8(a) row A1: "an optional per-instance 3x4 affine applied
 * inside K1"): the dynamic objects of the paper's motion modes (f.i; poses and per-axis scales
 * redrawn every frame) are instances of one mesh, so a frame's input is one 48-byte matrix per
 * instance instead of every posed vertex.  Appends part C to the triangle set of the last grca_update_scene /
 * grca_update_triangles[_f3] call (or to an empty set): triangle n_ab + i * n_faces + f (n_ab = that call's
 * triangle count) is face f of instance i, with vertices d_local_xyz[d_local_faces[3 f + c]] (packed float3,
 * object space; n_local_vertices of them) mapped by the row-major 3x4 matrix M_i = d_poses[12 i .. 12 i + 11]
 * (rows (m00 m01 m02 m03), (m10 ...), (m20 ...), 16-byte aligned): world_r = ((m_r0 x + m_r1 y) + m_r2 z) + m_r3
 * in fp32 with every product and sum rounded in this order (no FMA), so a host reproduces the world vertices bit
 * for bit.  Ids as the set's (d_tri_ids covering all parts, or tri_id_base + k).  Buffers borrowed as in
 * grca_update_triangles.  Every later grca_update_scene / grca_update_triangles[_f3] drops part C.
 * Errors: GRCA_E_INVALID (negative counts, n_faces or n_instances >= 2^31, missing or misaligned buffers),
 * GRCA_E_CAPACITY (n_ab + n_faces * n_instances > max_triangles). */
grca_status grca_update_instances(grca_t h, const float *d_local_xyz, int64_t n_local_vertices,
                                  const uint32_t *d_local_faces, int64_t n_faces, const float *d_poses,
                                  int64_t n_instances);

/* Hybrid static/dynamic mode (NEXT-f2; "GRCA on dynamic, static BVH on static,
 * per-ray min merge", here without any BVH): borrow a static triangle set (same conventions as
 * grca_update_triangles; buffers must stay alive and unmodified while set).  The next cast (and the
 * first cast after every grca_set_emitters) casts them once into a cached per-ray key buffer; every
 * cast then starts from those keys instead of MISS and culls only the grca_update_triangles set.
 * Exact: the per-ray closest hit is a min over triangles.  Ids of both sets share one space.
 * Errors: as grca_update_triangles. */
grca_status grca_set_static_triangles(grca_t h, const float *d_vertices, int64_t n_vertices,
                                      const uint32_t *d_indices, int64_t n_triangles,
                                      const int32_t *d_tri_ids, int32_t tri_id_base);
/* Leave hybrid mode (the static set is forgotten; nothing is freed). */
grca_status grca_clear_static(grca_t h);

/* Cast one frame: K0 init -> K2 cull (+ inline small work) -> K3 bin -> K4 intersect ->
 * [merge] -> K5 unpack, all enqueued on the handle's stream (no allocation, no host sync unless
 * h_stats != NULL).  d_out_dist: device float[n_rays] (+inf on a miss); d_out_tri: device
 * int32[n_rays] (-1 on a miss), n_rays = all emitters' rays (global layout).  Either output may be NULL
 * to skip K5.  With a communicator the call is COLLECTIVE (every rank, same sequence): triangle shards
 * merge in-stream (GRCA_MERGE_*) before K5; emitter shards cast their own emitters and optionally
 * broadcast them (gather_outputs).  grca_get_shard says which rays of the outputs are written.
 * Errors: GRCA_E_STATE (no emitters), GRCA_E_CUDA, GRCA_E_NCCL. */
grca_status grca_cast(grca_t h, float *d_out_dist, int32_t *d_out_tri, grca_stats *h_stats);

/* Split form: grca_cast_packed runs K0..K4 (and, with a communicator, the merge / gather) into the
 * handle's packed hit buffer (uint64 per ray: fp32 distance bits << 32 | triangle id; miss =
 * 0x7F800000FFFFFFFF; ordered like (t, id), positive as int64 so a signed or unsigned
 * min-allreduce merges shards exactly).  grca_hits_packed returns its device pointer.
 * grca_unpack runs K5 from that buffer (after the caller's merge). */
grca_status grca_cast_packed(grca_t h);
/* (Under emitter shards without gather_outputs only this rank's emitters' keys are initialised and valid; under a
 * reduce-scatter merge the buffer holds this rank's unmerged keys -- the merged slice is what grca_cast unpacks.) */
grca_status grca_hits_packed(grca_t h, uint64_t **d_hits, int64_t *n_rays);
grca_status grca_unpack(grca_t h, float *d_out_dist, int32_t *d_out_tri);
/* K5 over a slice of the rays, for ray-sharded merges (a reduce-scatter(MIN) leaves
 * each rank the merged keys of its own ray slice).  d_keys: device uint64[n] holding the packed keys
 * of global rays [first_ray, first_ray + n), or NULL for the handle's own buffer at first_ray.
 * d_out_dist / d_out_tri: device float[n] / int32[n] (slice-local), either may be NULL.  The distance
 * noise model (grca_set_distance_noise) keys its draws by the global ray index, so a slice gives
 * exactly the values the full unpack gives for those rays.  Counts as the cast's unpack (advances
 * the cast counter, like grca_unpack).  Errors: GRCA_E_INVALID (range outside [0, n_rays)),
 * GRCA_E_STATE (no emitters), GRCA_E_CUDA. */
grca_status grca_unpack_range(grca_t h, const uint64_t *d_keys, int64_t first_ray, int64_t n, float *d_out_dist,
                              int32_t *d_out_tri);

/* NEXT-f3: fused NVLS min-merge for triangle-sharded multi-GPU casts (the merge
 * of PAPER.md's per-ray closest hit over shards, P:2340-2356 f_sort).  d_uc is this rank's unicast
 * view and d_mc the multicast view (cuMulticastCreate/BindMem/cuMemMap, every rank's memory bound)
 * of one NVLS buffer of at least grca_nvls_status(..., bytes_needed) bytes: the per-ray packed keys
 * (n_rays u64, padded to 128 B) followed by a 128-byte barrier word.  Both views 128-byte aligned,
 * owned by the caller, valid until grca_set_nvls(h, NULL, NULL, 0) or grca_destroy.
 * After it, every grca_cast / grca_cast_packed on every rank: K0 initialises the rank's own keys,
 * a device-side barrier (multimem add + acquire spin on the flag) waits for all n_ranks, the
 * intersection kernels record hits with multimem.red.min.u64 on d_mc (the NVSwitch applies the
 * min to every rank's copy: no separate all-reduce), a second barrier, then K5 unpacks the merged
 * keys from d_uc.  Every rank must call grca_set_nvls before any rank casts, and all ranks must
 * cast the same sequence.  A barrier whose peers never arrive gives up after ~20 s and sets the
 * timed_out flag of grca_nvls_status (the result is then incomplete).  Errors: GRCA_E_INVALID
 * (one view missing, n_ranks < 1, misaligned), GRCA_E_STATE (before grca_set_emitters, with
 * GRCA_DEBUG_COUNT_ALL_HITS; casting with cached static triangles).  NULL, NULL -> merge off. */
grca_status grca_set_nvls(grca_t h, void *d_uc, void *d_mc, int32_t n_ranks);
/* Bytes the NVLS buffer needs for the current emitters; timed_out (synchronizes) = 1 if any
 * barrier of this handle gave up waiting.  Either pointer may be NULL. */
grca_status grca_nvls_status(grca_t h, int64_t *bytes_needed, int32_t *timed_out);

/* Distance noise (noise model: "a post-processing perturbation added after output
 * conversion"): K5 adds sigma * N(0,1) to every hit distance (clamped at 0; misses stay +inf), the
 * normal drawn from a counter-based generator keyed by (seed, cast index, ray).  sigma <= 0 -> off. */
grca_status grca_set_distance_noise(grca_t h, float sigma, uint64_t seed);

/* Counters of the last cast (synchronizes the stream). */
grca_status grca_get_stats(grca_t h, grca_stats *h_stats);

/* Sum of per-kernel device times over the last n_last casts (GRCA_PROFILE_KERNELS only;
 * n_last in [1, 64]; synchronizes).  ms_per_kernel[8]: [0] K0 init, [1] K2 cull (phase A),
 * [2] K2b refine, [3] K4s small-rectangle intersect, [4] K3 bin, [5] K4 large intersect,
 * [6] K5 unpack, [7] whole cast. */
grca_status grca_kernel_times(grca_t h, int32_t n_last, float *ms_per_kernel);

/* Per-ray all-hit counts of the last cast (GRCA_DEBUG_COUNT_ALL_HITS only):
 * device pointer to uint32[n_rays]. */
grca_status grca_debug_all_hits(grca_t h, const uint32_t **d_counts);

/* Test/diagnostic: copy up to cap entries of the last cast's large-pair list to host memory as
 * int32[4] {tri, emitter | c_from << 8, c_to, r_lo | r_len << 16}; *n_out = entries appended. */
grca_status grca_debug_large_list(grca_t h, int32_t *h_out, int64_t cap, int64_t *n_out);

/* Test-only, host: the azimuth approximation used by the cull (|error| <= 2.0e-6 rad),
 * evaluated with the same code on the host for n (y, x) pairs. */
grca_status grca_debug_fast_atan2(const float *h_y, const float *h_x, float *h_out, int64_t n);

/* n_rays_total and ray_offsets[n_emitters + 1] (O_n) of the current emitters. */
grca_status grca_get_layout(grca_t h, int64_t *n_rays_total, int64_t *ray_offsets);

/* Copy the fp32 ray table to host memory h_xyz[3 * n_rays] (test-only: bit-compare). */
grca_status grca_debug_ray_table(grca_t h, float *h_xyz);

/* Last error message of the handle (or of the last failed grca_create if h is NULL). */
const char *grca_last_error(grca_t h);

/* Library version string. */
const char *grca_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GRCA_H */
