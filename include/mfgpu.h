/*
 * mfgpu.h -- C ABI of the B200 decimation / cluster-pooling library (libmfgpu.so).
 *
 * Drop-in boundary for the reference package `meshforge` (pure Python/numpy,
 * /root/reference/pkg/src/meshforge).  The reference has no native FFI, so
 * each entry point below replaces one Python function of its public API:
 *
 *   mf_decimate        <- decimate.decimate_parallel(mesh, config)   decimate.py:344-382
 *                         (TriMesh and BatchedMesh; round chain decimate.py:294-316;
 *                          batch merge decimate.py:319-341)
 *   mf_decimation_*    <- DecimationResult fields mesh / replace / mapping   decimate.py:74-92
 *   mf_decimate_into   <- decimate_parallel with the result arrays emitted into caller buffers
 *   mf_pool            <- pooling.pool(features, result, mode, weights)      pooling.py:49-71
 *   mf_unpool          <- pooling.unpool(coarse, result)                     pooling.py:74-77
 *   mf_pool_backward   <- pooling.pool_backward / unpool_backward            pooling.py:80-102
 *   mf_round_targets   <- decimate._round_targets                            decimate.py:294-316
 *   mf_validate_mesh   <- TriMesh.__init__ re-validation of outputs          mesh.py:25-31, validation.py:8-41
 *
 * Plain pointers and sizes only.  Array pointers may be host or device memory
 * (detected per pointer); offsets are always host arrays.  Integer outputs are
 * int64 like the reference.  Every call is stream-ordered on `stream`
 * (a cudaStream_t, NULL = legacy default stream) and returns once its outputs
 * are complete.  Error codes map to the reference exception types:
 *
 *   MF_OK                0
 *   MF_ERR_VALUE         1  -> ValueError            (decimate.py:365-370, pooling.py:19-32)
 *   MF_ERR_STRUCTURAL    2  -> StructuralError       (validation.py:59-65)
 *   MF_ERR_INFEASIBLE    3  -> InfeasibleTargetError (decimate.py:239-244, 268-273);
 *                              mf_status.achievable_vertices / .mesh_index filled
 *   MF_ERR_CUDA          4  -> CUDA runtime failure
 *   MF_ERR_RUNTIME       5  -> RuntimeError          (pooling.py:27-28 coverage check)
 *   MF_ERR_LIMIT         6  -> input exceeds a documented device limit
 */
#ifndef MFGPU_H
#define MFGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MF_OK 0
#define MF_ERR_VALUE 1
#define MF_ERR_STRUCTURAL 2
#define MF_ERR_INFEASIBLE 3
#define MF_ERR_CUDA 4
#define MF_ERR_RUNTIME 5
#define MF_ERR_LIMIT 6

#define MF_DTYPE_F64 0
#define MF_DTYPE_F32 1

#define MF_POOL_AVERAGE 0  /* pooling.py:15 POOL_MODES order */
#define MF_POOL_MAX 1
#define MF_POOL_WEIGHTED 2
#define MF_POOL_SUM 3

typedef struct mf_context mf_context;
typedef struct mf_decimation mf_decimation;

typedef struct mf_status {
    int32_t code;
    int32_t mesh_index;           /* batch entry the error refers to (-1 = none) */
    int64_t achievable_vertices;  /* MF_ERR_INFEASIBLE */
    int64_t target_vertices;      /* target of the failing round */
    int32_t no_edges;             /* infeasible because the round had no edges */
    int32_t reserved;
    char message[256];
} mf_status;

/* TriMesh (mesh.py:13-52) or BatchedMesh (mesh.py:137-205) view. */
typedef struct mf_mesh_view {
    const double *positions;        /* [n,3] float64 */
    const int64_t *facets;          /* [m,3] int64 */
    const void *features;           /* [n,c] float64/float32, or NULL = copy of positions (mesh.py:28-29) */
    int32_t features_dtype;         /* MF_DTYPE_* */
    int32_t facets_i32;             /* 1: facets is a DEVICE int32 [m,3] array (e.g. a previous result's,
                                       mf_decimation_device_arrays) -- a decimation with >= 1 round only */
    int64_t n, m, c;
    const int64_t *vertex_offsets;  /* host [n_meshes+1], or NULL for one mesh */
    const int64_t *facet_offsets;   /* host [n_meshes+1], or NULL */
    int64_t n_meshes;
} mf_mesh_view;

/* DecimationConfig (decimate.py:45-71). */
typedef struct mf_decimate_config {
    int64_t target_vertices;
    int32_t rounds;        /* -1 = 'auto' */
    int32_t placement;     /* 0 = 'average', 1 = 'inverse' (quadrics.py:89-114); other -> MF_ERR_VALUE */
    int32_t seeded;        /* shuffle_seed is not None */
    int32_t einsum_order;  /* 0 = numpy AVX-512 lane-split dot3, 1 = sequential dot3 */
    uint64_t pcg_state[4]; /* default_rng(seed).bit_generator.state: state_hi, state_lo, inc_hi, inc_lo */
} mf_decimate_config;

/* A context owns a device workspace, streams and the captured CUDA graphs of its calls: use one
 * context per calling thread (calls on distinct contexts may run concurrently; calls on the
 * same context must not overlap).  The graph cache is per thread as well, so a context should
 * stay with the thread that created it. */
int mf_context_create(int device, mf_context **out);
void mf_context_destroy(mf_context *ctx);

int mf_decimate(mf_context *ctx, const mf_mesh_view *mesh, const mf_decimate_config *cfg, void *stream,
                mf_decimation **out, mf_status *status);

/* Caller-owned result buffers for mf_decimate_into: device memory or pinned host memory (written
 * through its mapped device address); NULL skips an array.  facets needs room for the input facet
 * count (the output count is known only at the end); n_out = target_vertices * n_meshes. */
typedef struct mf_outputs {
    double *positions;         /* [n_out, 3] float64 */
    int64_t *facets;           /* [facets_capacity, 3] int64; rows [0, m_out) are written */
    int64_t facets_capacity;   /* rows available in facets (>= the input facet count) */
    void *features;            /* [n_out, c] of features_dtype */
    int32_t features_dtype;    /* MF_DTYPE_* */
    int32_t features_if_distinct; /* 1: leave `features` unwritten when the result's features are
                                     known to be the positions bitwise (omitted input features, or
                                     host features equal to the positions); the caller then shares
                                     the positions' array -- mf_decimation_device_arrays reports it */
    int64_t *replace;          /* [n_in] int64 */
    int64_t *mapping;          /* [n_in] int64 */
    int64_t *vertex_offsets;   /* host [n_meshes + 1] */
    int64_t *facet_offsets;    /* host [n_meshes + 1] */
} mf_outputs;

/* mf_decimate + mf_decimation_copy in one call: the outputs are emitted by the same launch that
 * fills the handle's arrays, before the call's single synchronisation.  The handle is still
 * returned (pooling reuses it). */
int mf_decimate_into(mf_context *ctx, const mf_mesh_view *mesh, const mf_decimate_config *cfg, void *stream,
                     const mf_outputs *outputs, mf_decimation **out, mf_status *status);

/* mf_decimate_into split in two: _begin validates, stages and launches the round chain and returns
 * without waiting; _end emits the results (into `outputs`, which may be NULL) and synchronises.
 * One begun call per context at a time; the mesh buffers must stay alive until _end. */
int mf_decimate_begin(mf_context *ctx, const mf_mesh_view *mesh, const mf_decimate_config *cfg, void *stream,
                      mf_status *status);
int mf_decimate_end(mf_context *ctx, const mf_outputs *outputs, mf_decimation **out, mf_status *status);

int mf_decimation_sizes(const mf_decimation *res, int64_t *n_in, int64_t *n_out, int64_t *m_out, int64_t *c,
                        int64_t *n_meshes);
/* Copy results into caller buffers (host or device; NULL skips an array).
 * facets / replace / mapping / offsets are written as int64. */
int mf_decimation_copy(const mf_decimation *res, double *positions, int64_t *facets, void *features,
                       int32_t features_dtype, int64_t *replace, int64_t *mapping, int64_t *vertex_offsets,
                       int64_t *facet_offsets, void *stream, mf_status *status);
void mf_decimation_free(mf_decimation *res);
/* Device views of a result's mesh (valid while `res` lives): positions float64 [n_out,3],
 * facets int32 [m_out,3]; *features_alias = 1 when the features are the positions bitwise.
 * Feeding them back as the next call's mesh_view (facets_i32 = 1) chains a decimation
 * hierarchy without a host round trip. */
int mf_decimation_device_arrays(const mf_decimation *res, const double **positions, const int32_t **facets,
                                int32_t *features_alias);
/* Per-round counts of the call (rows of 6: N, M, E, N_out, M_out, matching iterations);
 * returns the number of rounds. */
int32_t mf_decimation_round_stats(const mf_decimation *res, int64_t *out, int32_t cap_rounds);

/* pool over a replace tensor (host/device int64[n]) or over a decimation's
 * own replace (res != NULL, replace ignored: reuses its device cluster CSR). */
int mf_pool(mf_context *ctx, const mf_decimation *res, const int64_t *replace, int64_t n, int64_t n_out,
            const void *features, int32_t dtype, int64_t c, int32_t mode, const void *weights, void *out,
            void *stream, mf_status *status);
/* pooling.pool_backward (pooling.py:80-97).  out dtype follows numpy: average -> float64,
 * sum -> grad dtype, weighted -> promote(grad, features), max -> features dtype.
 * unpool_backward (pooling.py:100-102) = mf_pool(mode = MF_POOL_SUM). */
int mf_pool_backward(mf_context *ctx, const mf_decimation *res, const int64_t *replace, int64_t n, int64_t n_out,
                     const void *grad_output, int32_t grad_dtype, const void *features, int32_t features_dtype,
                     int64_t c, int32_t mode, const void *weights, void *out, int32_t out_dtype, void *stream,
                     mf_status *status);
int mf_unpool(mf_context *ctx, const mf_decimation *res, const int64_t *replace, int64_t n, int64_t n_out,
              const void *coarse, int32_t dtype, int64_t c, void *out, void *stream, mf_status *status);

int64_t mf_round_targets(int64_t n_in, int64_t target, int32_t rounds, int64_t *chain, int64_t cap);

/* Re-validation of a mesh on the device -- replaces TriMesh.__init__'s checks (mesh.py:25-31 ->
 * validation.py:8-41): finite positions, facet indices in [0, n) (and inside their own batch
 * entry when offsets are given), no facet repeating a vertex; with check_duplicates also no two
 * facets with the same vertex set (the dedupe invariant of decimate.py:153-157).  Errors:
 * MF_ERR_STRUCTURAL with the reference's messages, in its check order.  Host or device arrays.
 * Setting MF_DEBUG=1 in the environment runs this check (plus replace / mapping ranges) on every
 * mf_decimate result before it returns. */
int mf_validate_mesh(mf_context *ctx, const double *positions, int64_t n, const int64_t *facets, int64_t m,
                     const int64_t *vertex_offsets, const int64_t *facet_offsets, int64_t n_meshes,
                     int32_t check_duplicates, void *stream, mf_status *status);

/* Binary little-endian PLY bodies (io.py:226-431), decoded / encoded on the device.
 * Field types: MF_PLY_I1 .. MF_PLY_F8 = PLY char, uchar, short, ushort, int, uint, float, double. */
enum { MF_PLY_I1 = 0, MF_PLY_U1 = 1, MF_PLY_I2 = 2, MF_PLY_U2 = 3, MF_PLY_I4 = 4, MF_PLY_U4 = 5, MF_PLY_F4 = 6,
       MF_PLY_F8 = 7 };
typedef struct mf_ply_vertex_spec {
    int32_t record_size;  /* bytes per vertex record */
    int32_t offset[6];    /* byte offsets of x y z red green blue in a record (-1: absent) */
    int32_t type[6];      /* MF_PLY_* of each field */
} mf_ply_vertex_spec;
/* body: bytes after end_header (host or device).  Vertex records start at byte 0,
 * uniform-arity face records (uchar count + arity indices of index_type) at face_offset.
 * Outputs: positions float64[nv, 3]; features float64[nv, n_channels] (3 = copy of the
 * positions, 6 = + colours c / 255 * 2 - 1, io.py:390-392); facets int64[n_faces *
 * (arity - 2), 3] fan-triangulated (io.py:92-93).  Replaces io.py:277-306 + 329-344. */
int mf_ply_decode(mf_context *ctx, const uint8_t *body, int64_t body_len, int64_t n_vertices,
                  const mf_ply_vertex_spec *vertex_spec, int64_t face_offset, int64_t n_faces, int32_t arity,
                  int32_t index_type, double *positions, double *features, int32_t n_channels, int64_t *facets,
                  void *stream, mf_status *status);
/* _save_ply body (io.py:404-431): n vertex records (float32 xyz, + uchar rgb when
 * features has >= 6 channels) then m records (uchar 3, int32 x3); body must hold
 * n * (12 or 15) + m * 13 bytes (host or device). */
int mf_ply_encode(mf_context *ctx, const double *positions, int64_t n, const double *features, int64_t c,
                  const int64_t *facets, int64_t m, uint8_t *body, void *stream, mf_status *status);

/* vertex_facet_adjacency (mesh.py:114-122): offsets int64[n+1], facet_ids int64[3m]
 * (each vertex's facets ascending).  facets: int64[m, 3]; host or device pointers. */
int mf_vertex_facet_adjacency(mf_context *ctx, const int64_t *facets, int64_t m, int64_t n, int64_t *offsets,
                              int64_t *facet_ids, void *stream, mf_status *status);
/* facet2vertex_forward (conv.py:222-250), strided when vertex_ids != NULL (rows = len,
 * e.g. representative_vertices(result), decimate.py:118-123): out[rows, C*L] in the
 * features' dtype.  offsets / facet_ids: the adjacency over n vertices; features
 * [m, C] (MF_DTYPE_F32/F64); weights float64[T, C, L] already rounded to the features'
 * dtype (kernel.weights.astype(dtype), conv.py:241); coeff float64[m, T]. */
int mf_facet2vertex(mf_context *ctx, const int64_t *offsets, int64_t n, const int64_t *facet_ids,
                    const void *features, int32_t dtype, int64_t m, int64_t c, const double *weights, int64_t t,
                    int64_t multiplier, const double *coeff, const int64_t *vertex_ids, int64_t rows, void *out,
                    void *stream, mf_status *status);

/* quality_report's per-output-vertex error (replaces decimate.py:580-602 up to the
 * numpy reductions): cluster quadric of the ORIGINAL mesh's vertex quadrics (summed in
 * ascending member order, accumulate_quadrics quadrics.py:80-86) evaluated at the output
 * positions (Quadric.evaluate, quadrics.py:53-58).  `original`: the input mesh (host or
 * device pointers, offsets ignored); replace: host/device int64[n] or taken from `res`;
 * positions_out: float64[n_out, 3]; errors: float64[n_out] (host or device).  The caller
 * takes mean / max / bincount exactly like the reference (decimate.py:594-602). */
int mf_quality_errors(mf_context *ctx, const mf_mesh_view *original, const mf_decimation *res,
                      const int64_t *replace, int64_t n_out, const double *positions_out, int32_t einsum_order,
                      double *errors, void *stream, mf_status *status);

/* Per-kernel CUDA-event timing on the launching stream (mode 0 off, 1 all, 2 only `only`). */
void mf_profile(int32_t mode, const char *only);
int32_t mf_profile_read(char *names, int32_t name_cap, double *total_ms, int64_t *launches, int32_t cap);

/* Number of kernels this library launched on the calling thread since the last reset. */
int64_t mf_kernel_launch_count(int32_t reset);
const char *mf_version(void);

#ifdef __cplusplus
}
#endif
#endif
