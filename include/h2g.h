/*
 * h2g — C ABI of the B200-native adaptive H^2 x H^2 product (arXiv 2309.09061).
 *
 * Drop-in boundary for the reference package h2mul's hot path:
 *   h2g_multiply   replaces h2mul.multiply            (/root/reference/pkg/src/h2mul/induced.py:358-372)
 *                  i.e. cluster_basis_product (h2.py:127-145), basis_weights / total_weights
 *                  (weights.py:37-101), compress_induced_row/col_basis (induced.py:76-200),
 *                  build_product_block_tree (trees.py:314-359) and assemble_product (induced.py:220-355)
 *   h2g_coarsen    replaces h2mul.coarsen             (coarsening.py:408-422)
 *                  i.e. build_coarse_row/col_basis (coarsening.py:187-339) and project_final (:354-405)
 *   h2g_recompress replaces h2mul.recompress          (coarsening.py:437-445), the input preparation
 *
 * The reference has no FFI of its own (callers import the Python functions directly, bench.py:21-31);
 * these entry points are what a ctypes / cffi binding of that path binds.
 *
 * Data model: plain host arrays in the packed layout of paper_2309_09061_b200/packed.py —
 * cluster trees (start, stop, child CSR; preorder ids), block trees (row, col, child CSR, adm),
 * bases (rank, leaf_off, xfer_off, data; leaf = size x k, transfer = k_child x k_parent, row-major),
 * couplings / nearfield (per-block offsets into one float64 array, -1 where absent).
 *
 * Status codes: 0 ok, 1 invalid input (h2mul InvalidInputError), 2 structural invariant
 * (h2mul StructureError), 3 CUDA failure.  h2g_last_error() returns the message of the last failure
 * on the calling thread.  Calls on one context are serialised on its stream; contexts are independent.
 */
#ifndef H2G_H
#define H2G_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct h2g_ctx h2g_ctx;
typedef struct h2g_tree h2g_tree;
typedef struct h2g_blocks h2g_blocks;
typedef struct h2g_h2 h2g_h2;

/* context: device + stream (NULL stream -> a private non-blocking stream) */
int h2g_ctx_create(int device, void* stream, h2g_ctx** out);
int h2g_ctx_destroy(h2g_ctx* ctx);
int h2g_ctx_set_timing(h2g_ctx* ctx, int on);
/* Multi-GPU (one process per GPU): the ranks sharing each product.  Every rank holds the whole of
   X and Y; multiply / coarsen split the row (and column) cluster trees into subtrees at the first
   level with >= size clusters (h2g_tree_partition), compute their own subtrees' clusters and blocks
   plus the replicated top levels, and exchange the results with `fn`, an in-place all-gather of a
   device buffer: segment i = bytes [off[i], off[i+1]) is valid on rank i on entry and on every rank
   on return; issued on `stream`; channel 0 / 1 = the row / column pass (concurrent host threads;
   use one communicator each).  Returns 0 on success.  size 1 (default): single GPU. */
typedef int (*h2g_allgather_fn)(void* user, int channel, void* dbuf, const long long* off, int nseg,
                                void* stream);
int h2g_ctx_set_comm(h2g_ctx* ctx, int rank, int size, h2g_allgather_fn fn, void* user);
/* Optional variable all-to-all for the partitioned product (replaces h2mul's nothing: SURVEY 8(e)
   halo / transpose exchanges): rank i sends bytes [soff[j], soff[j+1]) of sbuf to rank j and
   receives rank j's bytes into [roff[j], roff[j+1]) of rbuf, device buffers ordered on `stream`;
   returns 0 on success.  Without it, those exchanges fall back to the all-gather. */
typedef int (*h2g_alltoall_fn)(void* user, int channel, const void* sbuf, const long long* soff, void* rbuf,
                               const long long* roff, int nseg, void* stream);
int h2g_ctx_set_alltoall(h2g_ctx* ctx, h2g_alltoall_fn fn, void* user);
/* ms per stage of the last multiply / coarsen: setup, t1_row, t1_col, t1_mat, t2_row, t2_col, t2_mat
   (the reference harness's stage split, bench.py:195-237) */
int h2g_ctx_stage_times(h2g_ctx* ctx, double* out7);
/* out[0..n) = {setup, t1_row, t1_col, t1_mat, t2_row, t2_col, t2_mat, setup_col, t1_span, t2_span,
   t2_norms} ms (bench.py:195-237 split; the row / column passes of a phase run concurrently, each
   t*_row / t*_col is its own stream span, t*_span the joint span) */
int h2g_ctx_stage_times_ext(h2g_ctx* ctx, double* out, int n);
/* device memory of the engine's arenas (the device's default cudaMallocAsync pool), bytes:
   out6 = {pool used high-water, used now, reserved high-water, reserved now, arena payload
   high-water, payload now} (payload: bytes handed out by the process's arenas, without the 64 MB
   chunk granularity); reset: restart the high-water marks */
int h2g_ctx_mem(h2g_ctx* ctx, long long* out6, int reset);
/* kernel launches and host synchronisations since the last reset: out2 = {launches, syncs} */
int h2g_ctx_counters(h2g_ctx* ctx, long long* out2, int reset);
int h2g_ctx_synchronize(h2g_ctx* ctx);
/* host-side time per named section in timing mode, as "name=ms;..." (returns the full length) */
int h2g_ctx_host_times(h2g_ctx* ctx, char* buf, int len, int reset);
/* profile mode: CUDA events around every batched launch, accumulated per kernel class
   (0 gsum, 1 qr_r, 2 svd, 3 norm, 4 gather, 5 mv); out24 = per class {launches, ms, algorithmic flops,
   bytes} */
int h2g_ctx_set_profile(h2g_ctx* ctx, int on);
/* serial mode (process-wide): the row and column passes and the auxiliary launches of a product run
   one after the other on the main stream, so profile-mode events time each launch by itself */
int h2g_set_serial(int on);
int h2g_ctx_kernel_stats(h2g_ctx* ctx, double* out24, int reset);
/* timeline: trace_begin turns on per-launch events; trace_dump writes a chrome://tracing JSON */
int h2g_ctx_trace_begin(h2g_ctx* ctx);
int h2g_ctx_trace_dump(h2g_ctx* ctx, const char* path);

/* cluster tree (reference ClusterTree, trees.py:34-97): n nodes in preorder */
int h2g_tree_create(h2g_ctx* ctx, int n, const long long* start, const long long* stop,
                    const long long* child_ptr, const long long* child_idx, h2g_tree** out);
void h2g_tree_destroy(h2g_tree* t);
/* Host-only: owner rank (or -1 = replicated top level) of every cluster for nparts ranks, and the
   partition level (-1: no level has nparts clusters, everything replicated). */
int h2g_tree_partition(h2g_tree* t, int nparts, long long* owner, int* level);

/* block tree (reference BlockTree, trees.py:176-227): nb blocks in preorder */
int h2g_blocks_create(h2g_ctx* ctx, h2g_tree* rows, h2g_tree* cols, int nb, const long long* row,
                      const long long* col, const long long* child_ptr, const long long* child_idx,
                      const unsigned char* adm, h2g_blocks** out);
void h2g_blocks_destroy(h2g_blocks* b);

/* H^2 matrix (reference H2Matrix, h2.py:148-194) uploaded from the packed host layout.
   share_bases != 0: the column basis is the row basis object (cb_* ignored). */
int h2g_h2_upload(h2g_ctx* ctx, h2g_blocks* bt,
                  const long long* rb_rank, const long long* rb_leaf_off, const long long* rb_xfer_off,
                  const double* rb_data, long long rb_len,
                  const long long* cb_rank, const long long* cb_leaf_off, const long long* cb_xfer_off,
                  const double* cb_data, long long cb_len, int share_bases,
                  const long long* coup_off, const double* coup_data, long long coup_len,
                  const long long* near_off, const double* near_data, long long near_len, h2g_h2** out);
/* same, but the nearfield array is copied asynchronously on the context's copy stream: the call
   returns once bases and couplings are enqueued; kernels that read the nearfield wait for it on
   the device. The nearfield copy itself is issued at the matrix's first use (so that a second
   operand's bases and couplings are not queued behind it) or by h2g_ctx_synchronize, whichever comes
   first. near_data must stay valid until h2g_ctx_synchronize returns (it starts a pending copy and
   drains the copy stream), or until a synchronising call that follows a use of the matrix
   (h2g_h2_download of a result computed from it). */
int h2g_h2_upload_async(h2g_ctx* ctx, h2g_blocks* bt,
                        const long long* rb_rank, const long long* rb_leaf_off, const long long* rb_xfer_off,
                        const double* rb_data, long long rb_len,
                        const long long* cb_rank, const long long* cb_leaf_off, const long long* cb_xfer_off,
                        const double* cb_data, long long cb_len, int share_bases,
                        const long long* coup_off, const double* coup_data, long long coup_len,
                        const long long* near_off, const double* near_data, long long near_len, h2g_h2** out);
void h2g_h2_destroy(h2g_h2* h);
/* out8 = {nblocks, row-tree nodes, col-tree nodes, rb_len, cb_len, coup_len, near_len, block child_idx len} */
int h2g_h2_sizes(h2g_h2* h, long long* out8);
/* per-cluster ranks of the row and column bases (ClusterBasis.rank, h2.py:32-72); no device work */
int h2g_h2_ranks(h2g_h2* h, long long* row_rank, long long* col_rank);
int h2g_h2_structure(h2g_h2* h, long long* row, long long* col, long long* child_ptr, long long* child_idx,
                     unsigned char* adm);
int h2g_h2_download(h2g_ctx* ctx, h2g_h2* h, long long* rb_rank, long long* rb_leaf_off,
                    long long* rb_xfer_off, double* rb_data, long long* cb_rank, long long* cb_leaf_off,
                    long long* cb_xfer_off, double* cb_data, long long* coup_off, double* coup_data,
                    long long* near_off, double* near_data);

/* Host-only structure: the refined product block tree T^XY of two block trees (trees.py:314-359),
   with counts of terminal triples {a, b, c}; no device work, usable without a GPU. */
int h2g_product_tree(h2g_blocks* bx, h2g_blocks* by, h2g_blocks** out, long long* ntriples3);
/* sizes2 = {nblocks, child_idx length}; arrays may be NULL to query sizes only */
int h2g_blocks_structure(h2g_blocks* b, long long* sizes2, long long* row, long long* col, long long* child_ptr,
                         long long* child_idx, unsigned char* adm);

/* Z = X * Y over the refined product tree T^XY (phase 1).  max_rank < 0: no cap. */
int h2g_multiply(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, double tol, int max_rank, int scaling, h2g_h2** g);
/* re-compression of g onto `coarse` (phase 2) */
int h2g_coarsen(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank, int scale_blocks,
                h2g_h2** z);
/* same, and the dense blocks of z that are dense blocks of g are copied, while phase 2 runs, into
   near_host at their offsets of z's packed nearfield layout; h2g_h2_download with near_data ==
   near_host then moves only the remaining blocks. near_host (pinned for overlap) holds near_len
   doubles (no prefetch when that is less than z's nearfield) and must stay valid until that
   download returns. */
int h2g_coarsen_prefetch(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank, int scale_blocks,
                         double* near_host, long long near_len, h2g_h2** z);
/* orthogonalise + coarsen onto the own block tree */
int h2g_recompress(h2g_ctx* ctx, h2g_h2* x, double tol, int max_rank, h2g_h2** z);
/* Interpolation H^2 matrix of a point-kernel problem with the couplings and nearfield blocks
   evaluated on the GPU (reference problems.py:295-332): kernel 0 = -log r, 1 = 1/(4 pi r),
   2 = 1/r, 3 = exp(-r)/r; points (n x dim) and weights (n) in cluster-tree order; the shared
   interpolation basis in the packed layout (rank / leaf_off / xfer_off / data); node_off / nodes =
   per-cluster Chebyshev grid (rank x dim, row-major) used for the couplings. Host arrays. */
int h2g_h2_build_kernel(h2g_ctx* ctx, h2g_blocks* bt, int kernel, int dim, const double* points,
                        const double* weights, const long long* rank, const long long* leaf_off,
                        const long long* xfer_off, const double* basis, long long basis_len,
                        const long long* node_off, const double* nodes, long long nodes_len, h2g_h2** out);
/* y <- (accumulate ? y : 0) + alpha * op(G) x, op = identity (trans = 0) or transpose (trans = 1);
   x and y are DEVICE vectors (length cols / rows of op(G)), computed on the context's stream.
   Replaces h2mul.h2_matvec / h2_matvec_adjoint (h2.py:224-267). */
int h2g_matvec(h2g_ctx* ctx, h2g_h2* g, int trans, const double* x, double* y, double alpha, int accumulate);

/* ---------------------------------------------------------------------------------------------
   Stage-level entry points: the reference's stage functions one call at a time, as its harness
   times them (bench.py:195-237) and as h2mul/__init__.py:11-32 exports them.  Results are opaque
   handles owning their device memory; each can be inspected (shapes / download) or fed to the
   next stage.  All calls run on the context's stream and return after the stage completes.
   --------------------------------------------------------------------------------------------- */
typedef struct h2g_basis h2g_basis;     /* ClusterBasis (h2.py:32-72) on the device */
typedef struct h2g_mats h2g_mats;       /* per-cluster / per-block small matrices: BasisProduct.p
                                           (h2.py:116-124), BasisWeights.r / TotalWeights.z
                                           (weights.py:20-34), basis_change / block_projections
                                           (induced.py:33-46), CoarsenState.r / .z (coarsening.py:36-50) */
typedef struct h2g_induced h2g_induced; /* InducedBasisResult (induced.py:33-46) */
typedef struct h2g_cstate h2g_cstate;   /* CoarsenState (coarsening.py:36-50) */

/* which = 0: row basis, 1: column basis of g (a view; keeps g's memory alive) */
int h2g_h2_basis(h2g_h2* g, int which, h2g_basis** out);
/* a basis uploaded from the packed layout (rank / leaf_off / xfer_off / data), host arrays */
int h2g_basis_upload(h2g_ctx* ctx, h2g_tree* tree, const long long* rank, const long long* leaf_off,
                     const long long* xfer_off, const double* data, long long len, h2g_basis** out);
/* out2 = {clusters, packed length}; then h2g_basis_download fills rank / leaf_off / xfer_off / data */
int h2g_basis_sizes(h2g_basis* b, long long* out2);
int h2g_basis_download(h2g_ctx* ctx, h2g_basis* b, long long* rank, long long* leaf_off, long long* xfer_off,
                       double* data);
void h2g_basis_destroy(h2g_basis* b);

/* n matrices (rows[i] x cols[i], row-major at data + off[i]; off[i] < 0 or an empty shape: none) */
int h2g_mats_upload(h2g_ctx* ctx, int n, const long long* rows, const long long* cols, const long long* off,
                    const double* data, long long len, h2g_mats** out);
/* *n = number of entries; rows / cols (may be NULL) receive the shapes (0 x 0 where absent) */
int h2g_mats_shapes(h2g_mats* m, int* n, long long* rows, long long* cols);
/* packed download: off[i] = offset of entry i in data (-1 if absent), row-major */
int h2g_mats_download(h2g_ctx* ctx, h2g_mats* m, long long* off, double* data);
void h2g_mats_destroy(h2g_mats* m);

/* cluster_basis_product(wx, vy) (h2.py:127-145): P_s = W_X,s^T V_Y,s for every cluster s */
int h2g_cluster_basis_product(h2g_ctx* ctx, h2g_basis* wx, h2g_basis* vy, h2g_mats** out);
/* basis_weights(w) (weights.py:37-57): R_r with W_r = Q_r R_r (R factor only) */
int h2g_basis_weights(h2g_ctx* ctx, h2g_basis* w, h2g_mats** out);
/* total_weights(y or y^T, rw, scaling) (weights.py:60-101): transposed = 1 condenses the columns
   of y^T (the reference's total_weights(x.transposed(), ...)) */
int h2g_total_weights(h2g_ctx* ctx, h2g_h2* y, int transposed, h2g_mats* rw, int scaling, h2g_mats** out);
/* compress_induced_row_basis(x, y, zy, pxy, tol, max_rank, scale_blocks, level_decay)
   (induced.py:76-184); max_rank < 0: none */
int h2g_compress_induced_row_basis(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_mats* zy, h2g_mats* pxy, double tol,
                                   int max_rank, int scale_blocks, double level_decay, h2g_induced** out);
/* compress_induced_col_basis(x, y, zx_adjoint, pxy, ...) (induced.py:187-200) */
int h2g_compress_induced_col_basis(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_mats* zxt, h2g_mats* pxy, double tol,
                                   int max_rank, int scale_blocks, double level_decay, h2g_induced** out);
/* parts of an InducedBasisResult: q (isometric basis), basis_change (per cluster, Q_t^T V_t) and
   block_projections (per block of X's block tree, or of Y^T's for a column basis, Q_t^T X|ts V_Y,s;
   absent for admissible leaves); any output may be NULL */
int h2g_induced_parts(h2g_induced* r, h2g_basis** q, h2g_mats** basis_change, h2g_mats** block_projections);
/* an InducedBasisResult from given parts (e.g. computed elsewhere); col = 1 for a column basis */
int h2g_induced_create(h2g_ctx* ctx, h2g_basis* q, h2g_mats* basis_change, h2g_mats* block_projections, int col,
                       h2g_induced** out);
void h2g_induced_destroy(h2g_induced* r);
/* assemble_product(x, y, qrow, qcol, pxy) (induced.py:220-355); T^XY built inside (trees.py:314-359) */
int h2g_assemble_product(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_induced* qrow, h2g_induced* qcol, h2g_mats* pxy,
                         h2g_h2** out);
/* _coupling_norms / _nearfield_norms (coarsening.py:342-351): spectral norms of g's admissible /
   inadmissible leaves into DEVICE arrays indexed by block id (nblocks doubles each; other entries 0) */
int h2g_block_norms(h2g_ctx* ctx, h2g_h2* g, double* coupling_norms, double* nearfield_norms);
/* build_coarse_row_basis / build_coarse_col_basis (coarsening.py:187-339); norms: device arrays from
   h2g_block_norms or NULL (computed when scale_blocks) */
int h2g_build_coarse_row_basis(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank,
                               int scale_blocks, const double* coupling_norms, const double* nearfield_norms,
                               h2g_cstate** out);
int h2g_build_coarse_col_basis(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank,
                               int scale_blocks, const double* coupling_norms, const double* nearfield_norms,
                               h2g_cstate** out);
/* parts of a CoarsenState: q, r (Q_t^T V_t), z (condensation weights), number of stored reps */
int h2g_cstate_parts(h2g_cstate* s, h2g_basis** q, h2g_mats** r, h2g_mats** z, long long* nreps);
void h2g_cstate_destroy(h2g_cstate* s);
/* project_final(g, rowstate, colstate, coarse) (coarsening.py:354-405) */
int h2g_project_final(h2g_ctx* ctx, h2g_h2* g, h2g_cstate* rowstate, h2g_cstate* colstate, h2g_blocks* coarse,
                      h2g_h2** out);

const char* h2g_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* H2G_H */
