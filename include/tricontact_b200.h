/*
 * tricontact_b200.h -- C ABI of the B200 (sm_100a) triangle-pair contact
 * kernels: the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/tricontact/kernels.py, "RK" below).
 *
 * Every entry point takes plain pointers and sizes; no torch types.  Two
 * families:
 *
 *  - device entry points (tc_<variant>_<dtype>): all array pointers are
 *    DEVICE pointers, work is enqueued on `stream` (a cudaStream_t passed as
 *    void*, NULL = legacy default stream) and the call returns without
 *    synchronising.  Return code reports argument/launch errors only;
 *    per-pair degenerate failures are reported through tc_stats.degenerate
 *    and kind == TC_KIND_DEGENERATE.
 *  - host entry points (tc_<variant>_host_<dtype>): all array pointers are
 *    HOST pointers (pinned memory makes the copies asynchronous DMA); the
 *    library pipelines H2D copy / kernel / D2H copy over chunks on its own
 *    streams and returns after the results are on the host.  The hybrid host
 *    call returns TC_EDEGENERATE when a fallback pair was degenerate (the
 *    reference raises DegenerateTriangle there, RK/kernels.py:598-600).
 *
 * Layout (flags & TC_SOA == 0, the reference's own, RK/geometry.py:35-42):
 *   tri_a, tri_b: (n, 3, 3) vertex-major triangles, 9 scalars per triangle;
 *   point_a/point_b: (n, 3); bary_a/bary_b: (n, 2); distance, kind: (n,).
 * With TC_SOA: tri_a / tri_b are planar [9][n] (plane 3*v + c holds vertex v
 * coordinate c of every pair); point_* are [3][n] and bary_* [2][n] planes.
 * Any output pointer may be NULL (not written); with all of them NULL the
 * call is reduce-only (tc_stats).
 */
#ifndef TRICONTACT_B200_H
#define TRICONTACT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ABI_VERSION 2

/* return codes */
#define TC_OK 0
#define TC_EINVAL 1          /* bad argument (n < 0, NULL input, bad params) */
#define TC_EDEGENERATE 2     /* host hybrid: some fallback pair was degenerate */
#define TC_ECUDA 3           /* CUDA runtime error (tc_last_error() has the text) */
#define TC_ENODEVICE 4       /* no usable sm_100 device */

/* kind values, RK/kernels.py:36-39 (+ DEGENERATE, set only by hybrid) */
#define TC_KIND_NO_CONTACT 0
#define TC_KIND_CONTACT 1
#define TC_KIND_NOT_TERMINATED 2
#define TC_KIND_DEGENERATE 3

/* flags (tc_params.flags) */
#define TC_SOA 1u       /* planar inputs/outputs, see above */
#define TC_STRICT 2u    /* numpy-order rounding: no FMA contraction, 3-term dot in the
                           reference's einsum order; bit-identical to the reference */
#define TC_EMIT_IDS 4u  /* write ids (4 bytes per pair, layout in DESIGN.md) */

/* RK/kernels.py:42-72 KernelParams, plus flags. */
typedef struct {
    double epsilon;            /* halo width used when eps == NULL */
    double c_factor;           /* functional-change settle factor */
    double alpha_iterative;    /* penalty weight factor (x max squared edge) */
    double alpha_regulariser;  /* diagonal regulariser factor (x max squared edge) */
    double move_factor;        /* contact-point-movement settle factor */
    double start_coord;        /* initial barycentric coordinate */
    int32_t n_iterative;       /* fixed sweep count */
    uint32_t flags;            /* TC_SOA | TC_STRICT | TC_EMIT_IDS */
} tc_params;

/* Device-resident tallies, accumulated atomically (monotone, like
 * KernelCounters RK/kernels.py:75-93) until reset with tc_stats_reset. */
typedef struct {
    int64_t iterative;    /* iterative_invocations */
    int64_t comparison;   /* comparison_invocations */
    int64_t fallback;     /* fallback_invocations */
    int64_t degenerate;   /* fallback pairs with a degenerate triangle */
    int64_t contacts;     /* pairs whose final kind is CONTACT */
    int64_t intersecting; /* comparison results that found a proper edge-face crossing */
    double min_distance;  /* min final distance over non-degenerate pairs (+inf if none) */
} tc_stats;

/* Fill p with the reference defaults (RK/kernels.py:56-62). */
void tc_params_default(tc_params* p);
int tc_abi_version(void);
const char* tc_last_error(void);

/* Zero the counters and set min_distance = +inf (device pointer). */
int tc_stats_reset(tc_stats* stats, void* stream);

/* ---- device entry points ------------------------------------------------
 * eps: per-pair halo (n,) or NULL for p->epsilon (RK/kernels.py:143-149).
 * allow_fb: per-pair fallback mask (n,) uint8 or NULL for "all" (RK/kernels.py:589-593).
 * stats: device tc_stats or NULL. */

/* RK/kernels.py:301 comparison_batch */
int tc_comparison_f64(const double* tri_a, const double* tri_b, int64_t n, const double* eps,
                      const tc_params* p, double* distance, double* point_a, double* point_b,
                      double* bary_a, double* bary_b, int8_t* kind, uint8_t* ids,
                      tc_stats* stats, void* stream);
int tc_comparison_f32(const float* tri_a, const float* tri_b, int64_t n, const float* eps,
                      const tc_params* p, float* distance, float* point_a, float* point_b,
                      float* bary_a, float* bary_b, int8_t* kind, uint8_t* ids,
                      tc_stats* stats, void* stream);

/* RK/kernels.py:447 iterative_batch */
int tc_iterative_f64(const double* tri_a, const double* tri_b, int64_t n, const double* eps,
                     const tc_params* p, double* distance, double* point_a, double* point_b,
                     double* bary_a, double* bary_b, int8_t* kind, uint8_t* ids,
                     tc_stats* stats, void* stream);
int tc_iterative_f32(const float* tri_a, const float* tri_b, int64_t n, const float* eps,
                     const tc_params* p, float* distance, float* point_a, float* point_b,
                     float* bary_a, float* bary_b, int8_t* kind, uint8_t* ids,
                     tc_stats* stats, void* stream);

/* RK/kernels.py:568 hybrid_batch: iterative, then in-kernel comparison fallback
 * for NOT_TERMINATED pairs with allow_fb set; degenerate fallback pairs keep
 * the iterative result with kind TC_KIND_DEGENERATE. */
int tc_hybrid_f64(const double* tri_a, const double* tri_b, int64_t n, const double* eps,
                  const uint8_t* allow_fb, const tc_params* p, double* distance,
                  double* point_a, double* point_b, double* bary_a, double* bary_b,
                  int8_t* kind, uint8_t* ids, tc_stats* stats, void* stream);
int tc_hybrid_f32(const float* tri_a, const float* tri_b, int64_t n, const float* eps,
                  const uint8_t* allow_fb, const tc_params* p, float* distance,
                  float* point_a, float* point_b, float* bary_a, float* bary_b,
                  int8_t* kind, uint8_t* ids, tc_stats* stats, void* stream);

/* RK/kernels.py:157 closest_point_triangle_batch: points (n,3), tris (n,3,3). */
int tc_closest_point_triangle_f64(const double* points, const double* tris, int64_t n,
                                  double* closest, double* bary, void* stream);
int tc_closest_point_triangle_f32(const float* points, const float* tris, int64_t n,
                                  float* closest, float* bary, void* stream);

/* Point-to-triangle distance for the surrogate halo checks
 * (RK/surrogate.py:237-257 conservative_epsilon, :463-505
 * validate_conservative): distance[i] = |points[i] - closest point of
 * tris[tri_index[i]]| (tri_index NULL = tris[i], then n <= n_tris), rounded
 * like np.linalg.norm(p - closest_point_triangle_batch(p, t)[0], axis=1);
 * closest (n,3) optional.  Always strict IEEE (bit-identical). */
int tc_point_triangle_distance_f64(const double* points, const double* tris, int64_t n_tris,
                                   const int32_t* tri_index, int64_t n, double* distance,
                                   double* closest, void* stream);
int tc_point_triangle_distance_f32(const float* points, const float* tris, int64_t n_tris,
                                   const int32_t* tri_index, int64_t n, float* distance,
                                   float* closest, void* stream);

/* RK/geometry.py:68 degenerate_mask(tris, rel_tol): tris (n,3,3) -> mask (n,);
 * flags sq_area < rel_tol * longest_sq^2 (rel_tol rounded to the dtype, like
 * the reference's Python float times a REAL array; the reference default is
 * 1e-12, which the hybrid's fallback screen always uses). */
int tc_degenerate_mask_f64(const double* tris, int64_t n, double rel_tol, uint8_t* mask, void* stream);
int tc_degenerate_mask_f32(const float* tris, int64_t n, double rel_tol, uint8_t* mask, void* stream);

/* ---- all-pairs particle blocks (BASELINE.json config 2) -------------------
 * meshes: [n_meshes][tris_per_mesh][9] world-space triangles (device), or
 * local-space ones when motions ([n_meshes][7]: unit quaternion w, x, y, z and
 * translation, RK/geometry.py:124-176) is given -- the rigid motion is then
 * applied while the mesh is staged (fused transform, no world-space copy);
 * blocks: [n_blocks][2] int32 mesh indices; every block runs the hybrid kernel
 * on all tris_per_mesh^2 triangle pairs (mesh A's triangle i, mesh B's j),
 * both meshes staged in shared memory -- the all-pairs meshgrid of
 * RK/stepping.py:285-308 / RK/contact.py:97-140.  mesh_tris: [n_meshes]
 * triangle count of each mesh (ragged meshes, each <= tris_per_mesh, padded
 * to that stride), NULL = all tris_per_mesh; a block (m, m) of a mesh
 * against itself skips the diagonal i == j (RK/contact.py:119-124), so it
 * runs n (n - 1) pairs.  block_eps: per-block halo
 * (NULL = p->epsilon).  CONTACT pairs are appended (unordered) to
 * contact_idx [max][3] = (block, tri_a, tri_b), contact_distance [max],
 * contact_point_a/b [max][3]; *n_contacts (device int64, caller-zeroed) counts
 * all contacts, also those beyond max_contacts.  tc_stats tallies every pair.
 * Degenerate fallback pairs are counted in stats->degenerate, never listed. */
int tc_blocks_hybrid_f64(const double* meshes, int32_t tris_per_mesh, int64_t n_meshes,
                         const int32_t* mesh_tris,
                         const double* motions, const int32_t* blocks, int64_t n_blocks, const double* block_eps,
                         const tc_params* p, int64_t max_contacts, int32_t* contact_idx,
                         double* contact_distance, double* contact_point_a,
                         double* contact_point_b, int64_t* n_contacts, tc_stats* stats,
                         void* stream);
int tc_blocks_hybrid_f32(const float* meshes, int32_t tris_per_mesh, int64_t n_meshes,
                         const int32_t* mesh_tris,
                         const float* motions, const int32_t* blocks, int64_t n_blocks, const float* block_eps,
                         const tc_params* p, int64_t max_contacts, int32_t* contact_idx,
                         float* contact_distance, float* contact_point_a,
                         float* contact_point_b, int64_t* n_contacts, tc_stats* stats,
                         void* stream);

/* ---- multiscale frontier traversal ---------------------
 * RK/stepping.py:311-368 multiscale_contacts for n_pairs particle pairs at
 * once.  The surrogate trees of all particles are concatenated FlatTree arrays
 * (RK/stepping.py:78-129) under one global id space (DEVICE pointers):
 * tris [n_total][9] world coordinates -- or local ones when motions
 * ([n_particles][7], as tc_blocks_hybrid_*) is given, node_owner [n_total]
 * naming each node's particle: the rigid motion is then applied to every
 * node as it is loaded (RK/stepping.py:157-159 world_tris) -- node_eps [n_total], child_off
 * [n_total + 1] / child_ids (CSR children, global ids; a leaf node lists its
 * mesh triangles), is_fine [n_total] (1 = mesh triangle), height [n_total]
 * (0 = mesh level).  roots: HOST [n_pairs][2] global root ids (i, j).
 * Every round runs the hybrid kernel on the frontier with the halo
 * 0.5 (eps_i + eps_j) and the comparison fallback only on mesh-level pairs,
 * then unfolds contact/unsettled non-mesh pairings into the meshgrid of their
 * children (a mesh-level side stays itself).  Mesh-level contacts are
 * appended (unordered) to contact_idx [max][3] = (pair, id_i, id_j) and
 * contact_point_a/b [max][3] (device); *n_contacts (HOST) counts all of them,
 * also those beyond max_contacts.  checks (HOST, may be NULL)
 * [max_height + 1] accumulates the pairings per max(height_i, height_j)
 * (StepStats.record_checks); stats (HOST, may be NULL) accumulates the
 * kernel tallies.  TC_EDEGENERATE when a mesh-level fallback pair holds a
 * degenerate triangle (the reference raises DegenerateTriangle).  Params
 * flags: TC_STRICT only.  Synchronous on `stream` (one 8-byte read-back per
 * round). */
int tc_multiscale_f64(const double* tris, const int32_t* node_owner, const double* motions,
                      const double* node_eps, const int32_t* child_off,
                      const int32_t* child_ids, const uint8_t* is_fine, const int32_t* height,
                      int32_t max_height, const int32_t* roots, int64_t n_pairs, const tc_params* p,
                      int64_t max_contacts, int32_t* contact_idx, double* contact_point_a,
                      double* contact_point_b, int64_t* n_contacts, int64_t* checks, tc_stats* stats,
                      void* stream);
int tc_multiscale_f32(const float* tris, const int32_t* node_owner, const float* motions,
                      const float* node_eps, const int32_t* child_off,
                      const int32_t* child_ids, const uint8_t* is_fine, const int32_t* height,
                      int32_t max_height, const int32_t* roots, int64_t n_pairs, const tc_params* p,
                      int64_t max_contacts, int32_t* contact_idx, float* contact_point_a,
                      float* contact_point_b, int64_t* n_contacts, int64_t* checks, tc_stats* stats,
                      void* stream);

/* ---- host entry points ----------------------------------------------------
 * Same arguments with HOST pointers; variant: 0 comparison, 1 iterative,
 * 2 hybrid.  stats (host, may be NULL) receives this call's tallies
 * (accumulated into *stats).  Synchronous. */
#define TC_VARIANT_COMPARISON 0
#define TC_VARIANT_ITERATIVE 1
#define TC_VARIANT_HYBRID 2
int tc_run_host_f64(int variant, const double* tri_a, const double* tri_b, int64_t n,
                    const double* eps, const uint8_t* allow_fb, const tc_params* p,
                    double* distance, double* point_a, double* point_b, double* bary_a,
                    double* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats);
int tc_run_host_f32(int variant, const float* tri_a, const float* tri_b, int64_t n,
                    const float* eps, const uint8_t* allow_fb, const tc_params* p,
                    float* distance, float* point_a, float* point_b, float* bary_a,
                    float* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats);

/* Pinned host memory for result arrays: tc_run_host_* writes pinned outputs
 * by DMA directly instead of staging them (the drop-in allocates its
 * BatchResult columns here).  Blocks are recycled by size; tc_host_alloc
 * returns NULL on failure (tc_last_error), tc_host_free TC_EINVAL for a
 * pointer it did not hand out. */
void* tc_host_alloc(int64_t bytes);
int tc_host_free(void* p);
/* Host-pointer versions of the two helpers above (synchronous). */
int tc_closest_point_triangle_host_f64(const double* points, const double* tris, int64_t n,
                                       double* closest, double* bary);
int tc_closest_point_triangle_host_f32(const float* points, const float* tris, int64_t n,
                                       float* closest, float* bary);
int tc_degenerate_mask_host_f64(const double* tris, int64_t n, double rel_tol, uint8_t* mask);
int tc_degenerate_mask_host_f32(const float* tris, int64_t n, double rel_tol, uint8_t* mask);

/* FMA-pipe throughput probe (fp64 != 0: DFMA, else FFMA): enqueues one launch
 * of `blocks` CTAs and returns its flop count (or -1); time it with events
 * to get the FP64/FP32 roofline denominator.  sink: device scratch, >= blocks
 * elements. */
int64_t tc_fma_probe(int fp64, int64_t blocks, int iters, void* sink, void* stream);

/* Benchmark / test workload: pairs [start, start + n) of the cfg0 distribution
 * (BASELINE.json: A ~ U[0,1]^9; B = A rotated about its centroid by a uniform
 * random rotation and shifted by s * (random unit vector), s ~ U[sep_lo,
 * sep_hi]) from a counter-based Philox4x32-10 stream keyed by (seed, pair
 * index), written as SoA planes [18][n] (device pointer): any shard is
 * generated independently.  Not numpy's stream: a device generator of the same
 * distribution (numpy mirror: workloads.philox_pairs). */
int tc_random_pairs_soa_f64(uint64_t seed, int64_t start, int64_t n, double sep_lo, double sep_hi,
                            double* planes, void* stream);
/* Test knob: cap the CTAs of every persistent launch (0 = the occupancy
 * maximum).  Changing the CTA count changes which pairs share a CTA's
 * fallback queues and batches, so result equality across caps exposes
 * ordering / synchronisation faults (tests/test_gpu_stress.py). */
void tc_debug_set_max_ctas(int64_t max_ctas);
/* The fast hybrid keeps, per device, a history of its recent launches
 * (cumulative counters the kernels update; no synchronisation): when the
 * iterative warps found the hand-over ring full, the next launches use the
 * instance whose iterative warps also serve their own open pairs.  Returns 1
 * if the calling thread's current device would get that instance now, 0 if
 * not (tests/test_gpu_stress.py). */
int tc_debug_fallback_rate_high(void);
/* The kernel the next fast hybrid launch on the current device gets: 0 the
 * warp-specialised kernel, 1 its self-serving instance, 2 the kernel for
 * batches with few fallbacks (every warp iterates and serves its own queue). */
int tc_debug_hybrid_mode(void);
/* The history's cumulative counters as last published by a kernel: pairs,
 * fallbacks, ring waits of the iterative warps (per lane and poll), self-served tiles. */
void tc_debug_fallback_history(uint64_t out[4]);
/* Number of kernel launches this library has enqueued since load. */
int64_t tc_launch_count(void);

/* reduce a device tc_stats over the ranks of an NCCL
 * communicator -- one ncclGroupStart/End with ncclAllReduce(int64[6], sum)
 * and ncclAllReduce(double[1], min), enqueued on `stream` (no host sync).
 * nccl_comm: an ncclComm_t the caller created.  libnccl.so.2 is dlopen'ed on
 * first use (TC_ENODEVICE if absent); the other entry points never need it.
 * Python hosts may use torch.distributed instead (paper_2105_12415_b200/shard.py). */
int tc_allreduce_stats(tc_stats* stats, void* nccl_comm, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TRICONTACT_B200_H */
