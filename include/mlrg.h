/* Device C-ABI of the B200 build ("the thin C-ABI layer").
 *
 * Plain pointers and sizes only. Array arguments marked "dev" are device
 * pointers to complex64 data (interleaved float re, im) in the reference's
 * row-major layouts; they may come from any allocator (cudaMalloc, torch,
 * ...). Every call returns MLRG_OK or an MLR_* error code and records a
 * thread-local message for mlrg_last_error(), mirroring capi.cpp:37-47.
 * Work is enqueued on the context's stream; calls that return host values
 * synchronise it.
 */
#ifndef MLR_B200_MLRG_H
#define MLR_B200_MLRG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLRG_OK 0

typedef struct mlrg_ctx mlrg_ctx;     /* geometry + device tables + stream */
typedef struct mlrg_recon mlrg_recon; /* device reconstruction result */
typedef struct mlrg_memo mlrg_memo;   /* host memo client + store (decision logic) */

const char* mlrg_last_error(void);
void mlrg_free(char* text);
int mlrg_version(void);

/* ---- operator context (scalerun.hpp:61-116 OperatorEngine, per geometry) ---- */
/* stream: a cudaStream_t; NULL selects the legacy default stream (stream 0), which
 * orders the calls with work a host framework issued on its default stream. */
mlrg_ctx* mlrg_ctx_create(int64_t n1, int64_t n0, int64_t n2, int64_t n_theta, int64_t h, int64_t w,
                          double phi, void* stream);
/* Same with an explicit spreading kernel: 0 = es (10 taps, the default of
 * mlrg_ctx_create), 1 = gaussian (the reference's 24-tap plan, nufft.cpp:48-103).
 * Both evaluate the NUDFT of operators.cpp:87-200; see geometry.hpp. */
mlrg_ctx* mlrg_ctx_create_kernel(int64_t n1, int64_t n0, int64_t n2, int64_t n_theta, int64_t h, int64_t w,
                                 double phi, void* stream, int kernel);
void mlrg_ctx_destroy(mlrg_ctx* ctx);
int mlrg_sync(mlrg_ctx* ctx);
/* Plan figures for measurement (bench.py): {fu2d target classes per detector row,
 * kernel taps per dimension, oversampled grid extents M1, M2, gather CTAs and
 * classes per CTA per 16-row batch}. */
int mlrg_ctx_stats(mlrg_ctx* ctx, int64_t out[6]);

/* nufft::fu1d_gridding (nufft.cpp:107-134): dev u (d0, n0, n2) -> dev out (d0, h, n2). */
int mlrg_fu1d(mlrg_ctx* ctx, const void* u, void* out, int64_t d0);
/* nufft::fu1d_adj_gridding (nufft.cpp:136-162): (d0, h, n2) -> (d0, n0, n2). */
int mlrg_fu1d_adj(mlrg_ctx* ctx, const void* v, void* out, int64_t d0);
/* nufft::fu2d_gridding / fused_sub_fu2d (nufft.cpp:183-225, operators.cpp:285-299):
 * dev v (n1, d1, n2) -> dev out (n_theta, d1, w); d_hat (same shape as out) is
 * subtracted when non-NULL. */
int mlrg_fu2d(mlrg_ctx* ctx, const void* v, const void* d_hat, void* out, int64_t d1);
/* nufft::fu2d_adj_gridding (nufft.cpp:227-267): (n_theta, d1, w) -> (n1, d1, n2). */
int mlrg_fu2d_adj(mlrg_ctx* ctx, const void* p, void* out, int64_t d1);
/* f2d / f2d_adj (operators.cpp:39-74): centred unitary 2D DFT of d0 (h, w) planes. */
int mlrg_f2d(mlrg_ctx* ctx, const void* p, void* out, int64_t d0, int adjoint);
/* forward_L / adjoint_L (operators.cpp:301-309) on full arrays. */
int mlrg_forward_L(mlrg_ctx* ctx, const void* u, void* out);
int mlrg_adjoint_L(mlrg_ctx* ctx, const void* d, void* out);
/* grad / div (operators.cpp:311-352) on (n1, n0, n2) volumes. */
int mlrg_grad(mlrg_ctx* ctx, const void* u, void* g0, void* g1, void* g2);
int mlrg_div(mlrg_ctx* ctx, const void* g0, const void* g1, const void* g2, void* out);
/* Encoder::encode (encoder.cpp:386-422) of every chunk_extent slab of a full
 * operator input (op: 0 fu1d, 1 fu2d, 2 fu1d_adj, 3 fu2d_adj, 4 f2d, 5 f2d_adj):
 * host keys [n_slabs][key_dim] (slot-mixed) and host input norms [n_slabs]. */
int mlrg_encode(mlrg_ctx* ctx, int op, const void* x, int64_t chunk_extent, int key_dim, uint64_t seed,
                float* keys, double* norms, int64_t n_slabs);

/* The CNN key encoder (encoder_variant = cnn, encoder.cpp:95-197) with the seeded
 * initial weights (init_cnn): raw keys [n_slabs][key_dim] (before slot_mix) and
 * input norms of every chunk_extent slab of the op's input. */
int mlrg_encode_cnn(mlrg_ctx* ctx, int op, const void* x, int64_t chunk_extent, int key_dim, uint64_t seed,
                    float* keys, double* norms, int64_t n_slabs);
/* init_cnn (encoder.cpp:441-470): conv1 [32][2][5][5], conv2 [64][32][3][3], fc [key_dim][64]. */
int mlrg_cnn_weights(int key_dim, uint64_t seed, float* c1w, float* c2w, float* fcw);

/* ---- device reconstruction (admm.cpp:208-272) ----
 * config_text: the reference's key=value config text. dev d (n_theta, h, w)
 * space-domain data, optional dev reference (n1, n0, n2), dev u_out. */
mlrg_recon* mlrg_reconstruct(const char* config_text, const void* d, const void* reference, void* u_out,
                             void* stream);
char* mlrg_recon_csv(const mlrg_recon* r);
int mlrg_recon_aborted(const mlrg_recon* r);
char* mlrg_recon_abort_reason(const mlrg_recon* r);
/* Audit log (scalerun.hpp:45-54): per decision (iteration, op, location,
 * outcome 0 miss / 1 remote hit / 2 cache hit) and cs. Returns the entry
 * count; copies at most cap entries. */
int64_t mlrg_recon_audit(const mlrg_recon* r, int32_t* meta4, float* cs, int64_t cap);
/* MemoCounters (memoclient.hpp:42-54): lookups, cache_hits, remote_hits,
 * misses, cache_comparisons, cache_probes, timeouts, batches_sent,
 * inserts_enqueued, inserts_sent, inserts_dropped. */
int mlrg_recon_counters(const mlrg_recon* r, uint64_t out[11]);
/* Memo value tiers (cold_tier.hpp): out = {HBM ring arena bytes, values
 * spilled to pinned host memory, bytes spilled}. B200 extension: the
 * reference's store is one unbounded host array (memostore.cpp:112-120). */
int mlrg_recon_tiers(const mlrg_recon* r, uint64_t out[3]);
void mlrg_recon_free(mlrg_recon* r);

/* ---- steppable device solver (the outer loop of admm.cpp:208-272) ----
 * mlrg_solver_new runs the setup (engine, encoder matrices, d_hat = f2d(d));
 * each mlrg_solver_step runs exactly one ADMM outer iteration on `stream`
 * (NULL = the legacy default stream) and synchronises it. */
typedef struct mlrg_solver mlrg_solver;
mlrg_solver* mlrg_solver_new(const char* config_text, const void* d, const void* reference, void* stream);
int mlrg_solver_step(mlrg_solver* s, int* aborted);
int mlrg_solver_volume(mlrg_solver* s, void* u_out);
char* mlrg_solver_csv(const mlrg_solver* s);
int mlrg_solver_counters(const mlrg_solver* s, uint64_t out[11]);
int mlrg_solver_tiers(const mlrg_solver* s, uint64_t out[3]);
int64_t mlrg_solver_audit(const mlrg_solver* s, int32_t* meta4, float* cs, int64_t cap);
void mlrg_solver_free(mlrg_solver* s);

/* ---- z-slab sharded solver across the GPUs of one node ----
 * One process per GPU. mlrg_comm_create joins the node-local communicator
 * `name` (POSIX shared memory; rank 0 creates it, every rank passes the same
 * name and world; blocks until all ranks joined or timeout_s). Pure host: no
 * CUDA calls. The sharded solver splits the volume along axis 0 and the
 * detector rows along axis 1 in whole 16-slabs with the reference's assign()
 * (scalerun.cpp:14-27); d and reference are the FULL arrays on every rank's
 * device; mlrg_solver_volume then returns this rank's planes [a, b) and
 * mlrg_solver_shard reports {a, b, c, d}. The CSV, counters and audit are the
 * global ones on every rank. A comm of world 1 (or NULL) is mlrg_solver_new. */
typedef struct mlrg_comm mlrg_comm;
mlrg_comm* mlrg_comm_create(const char* name, int rank, int world, double timeout_s);
void mlrg_comm_free(mlrg_comm* c);
int mlrg_comm_barrier(mlrg_comm* c);
/* Marks the job failed: every rank in (or entering) a collective returns
 * MLR_ERR_RUNTIME instead of waiting (a failing mlrg_solver_step does this). */
int mlrg_comm_abort(mlrg_comm* c);
/* v[i] = sum over ranks, added in rank order (bit-identical on every rank). */
int mlrg_comm_allreduce(mlrg_comm* c, double* v, int n);
/* out = every rank's `bytes` bytes, concatenated in rank order (bytes <= 1 MiB). */
int mlrg_comm_allgather(mlrg_comm* c, const void* in, uint64_t bytes, void* out);
/* Per rank r: out[4r..4r+3] = {a, b, c, d}: planes [a, b) of axis 0 (n1) and
 * detector rows [c, d) of axis 1 (h). */
int mlrg_partition(int64_t n1, int64_t h, int64_t chunk, int world, int64_t* out);
mlrg_solver* mlrg_solver_new_sharded(const char* config_text, const void* d, const void* reference, void* stream,
                                     mlrg_comm* comm);
int mlrg_solver_shard(const mlrg_solver* s, int64_t out[4]);

/* ---- host memo decision logic (memoclient.cpp + memostore.cpp), for replay tests ---- */
mlrg_memo* mlrg_memo_new(float tau, int nprobe, uint64_t insert_cap, uint64_t coalesce_bytes, int global_cache,
                         int nlist, int train_size);
void mlrg_memo_free(mlrg_memo* m);
/* One lookup_batch: n keys of dim key_dim with (location, op, value_bytes);
 * writes outcome, cs and value id per key. */
int mlrg_memo_lookup(mlrg_memo* m, int64_t n, int key_dim, const float* keys, const int64_t* locations,
                     const int32_t* ops, const uint64_t* value_bytes, int32_t* outcome, float* cs,
                     uint64_t* value_id);
/* insert_async of one key with a value of value_bytes; returns 1 if staged. */
int mlrg_memo_insert(mlrg_memo* m, int key_dim, const float* key, uint64_t value_bytes);
int mlrg_memo_flush(mlrg_memo* m);
int mlrg_memo_counters(const mlrg_memo* m, uint64_t out[11]);
/* The store's IVF training (memostore.cpp:40-108): k-means++ seeding + Lloyd over
 * nk keys of dim floats, then each key's nearest centroid; on_device selects the
 * GPU trainer (memo_gpu.cu), which must equal the host's bit for bit. Writes
 * min(k, nk) x dim centroids and nk indices. */
int mlrg_kmeans(const float* keys, int64_t nk, int dim, int k, uint64_t seed, int iters, int on_device,
                float* centroids, int64_t* nearest);

/* ---- encoder matrix and slot mix (encoder.cpp:16-86, 369-379), host ---- */
int mlrg_projection_matrix(int64_t d0, int64_t d1, int64_t d2, int key_dim, uint64_t seed, float* out,
                           int64_t count);
int mlrg_slot_mix(float* key, int key_dim, uint64_t seed, int64_t location, int op);

/* ---- measurement hooks (bench.py) ----
 * Total kernel launches issued by this library since load, and opt-in CUDA
 * event timers around each launch of the named hot kernels (k_fu1d,
 * k_fu1d_adj, k_fu2d_rows, k_fu2d_cols, k_fu2d_gather, k_fu2d_adj_prep,
 * k_fu2d_adj_spread, k_fu2d_adj_cols, k_fu2d_adj_rows). */
uint64_t mlrg_launch_count(void);
void mlrg_prof_enable(int on);
void mlrg_prof_reset(void);
int mlrg_prof_query(const char* name, double* total_ms, int64_t* count);
/** Writes every profiled span since the last reset as "name stream start_ms end_ms"
 *  (times relative to the earliest span start). */
int mlrg_prof_dump(const char* path);

/* ---- the drop-in result's memo audit (extension of mlr.h) ---- */
struct mlr_result;
int64_t mlrg_result_audit(const struct mlr_result* r, int32_t* meta4, float* cs, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* MLR_B200_MLRG_H */
