/*
 * lapb200.h -- C ABI of the B200-native Laplacian-eigensolver hot path.
 *
 * The reference package (lapeig 0.1.0, /root/reference/pkg/src/lapeig) is
 * pure Python; its "plugin" seams are duck-typed Python functions.  Every
 * entry point below replaces one of those seams and is what a ctypes / cffi
 * binding in the reference would call:
 *
 *   lg_csr_create / lg_spmv*      <- sparse.py:26-139   (CsrMatrix, spmv)
 *   lg_build_laplacian            <- graphs.py:250-263  (build_laplacian)
 *   lg_ic0_factorize              <- ic0.py:48-116      (_attempt, ic0_factorize)
 *   lg_ic0_create / lg_ic0_apply  <- ic0.py:24-45,139-150 (Ic0Factor.apply)
 *   lg_fused                      <- pcg.py:55-60 (DeflationBasis.project_out),
 *                                    kernels.py:22-55 (Gram-Schmidt sweeps),
 *                                    dacg.py:36-96 / pcg.py:131-155 (dots, axpys)
 *   lg_gemm_small                 <- jd.py:67-73,89-90; irlm.py:166,192 (V @ y)
 *   lg_scalar                     <- the scalar recurrences of dacg.py:188-233,
 *                                    pcg.py:133-155 executed on the device
 *
 * Conventions
 *   - every function returns 0 on success and a negative LG_E* code on error;
 *     lg_last_error() returns a thread-local message for the last failure.
 *   - pointers named *_h are host pointers; every other double* / int* is a
 *     device pointer owned by the caller (torch tensors in the Python layer).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - handles (lg_csr, lg_ic0) are immutable after creation and may be used
 *     concurrently from several streams; lg_ws (reduction workspace) must be
 *     used by one stream at a time.
 *   - all reductions are deterministic (fixed partition + fixed tree order,
 *     no floating-point atomics): identical inputs give bitwise identical
 *     outputs run to run.
 */
#ifndef LAPB200_H
#define LAPB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LG_OK 0
#define LG_EINVAL -1      /* bad argument (maps to ValueError)              */
#define LG_ECUDA -2       /* CUDA runtime failure (maps to RuntimeError)    */
#define LG_ENOMEM -3      /* allocation failure                             */
#define LG_EBREAKDOWN -4  /* IC(0) pivot breakdown at every shift (Ic0Error) */
#define LG_EFORMAT -5     /* malformed graph file (GraphFormatError)         */

/* ---- library / device -------------------------------------------------- */
const char* lg_last_error(void);
int lg_version(void);                        /* 100 * major + minor        */
int lg_device_info(int* sm_count, int* l2_bytes, int* cc_major, int* cc_minor);
/* async D2H copy of `bytes` into pinned host memory followed by a stream
 * synchronisation: the single host<->device round trip a solver iteration
 * pays for its convergence test. */
int lg_readback(const void* dev, void* host_pinned, int64_t bytes, void* stream);
int lg_upload(void* dev, const void* host, int64_t bytes, void* stream);

/* ---- CUDA graphs --------------------------------------------------------- */
/* A solver iteration is a fixed launch sequence over fixed buffers: capture
 * it once on a (non-legacy) stream and replay it with one launch. */
int lg_capture_begin(void* stream);
int lg_capture_end(void* stream, void** exec_out);
int lg_graph_launch(void* exec, void* stream);
int lg_graph_destroy(void* exec);

/* ---- reduction workspace ---------------------------------------------- */
typedef struct lg_ws lg_ws;
int lg_ws_create(lg_ws** out);
int lg_ws_destroy(lg_ws* ws);

/* ---- CSR matrix + SpMV (sparse.py:26-139) ------------------------------ */
typedef struct lg_csr lg_csr;
/* Upload an n x n CSR (int64 row_ptr, int64 col, f64 val as held by the
 * reference CsrMatrix, sparse.py:39-41).  Columns are stored as int32 when
 * n < 2^31.  Builds the nnz-balanced row-block schedule and, when the
 * off-diagonal values take few distinct values, the packed value table.
 * flags: LG_CSR_PLAIN disables the packed-value format; LG_CSR_SKIP_EMPTY
 * leaves rows without stored entries out of the schedule (lg_spmv does not
 * write y there): one rank's row block of the row-partitioned SpMV. */
#define LG_CSR_PLAIN 1
#define LG_CSR_SKIP_EMPTY 2
int lg_csr_create(int64_t n, int64_t nnz, const int64_t* row_ptr_h,
                  const int64_t* col_h, const double* val_h, int flags,
                  lg_csr** out);
int lg_csr_destroy(lg_csr* a);
/* n, nnz, number of row blocks, long rows, packed format flag, and the
 * bytes one SpMV streams from HBM under the stored format. */
int lg_csr_info(const lg_csr* a, int64_t* n, int64_t* nnz, int64_t* nblocks,
                int64_t* nlong, int* packed, int64_t* stream_bytes);
/* Read the device arrays back (row_ptr, col, val in the canonical layout):
 * the byte-identity check of an upload. */
int lg_csr_download(const lg_csr* a, int64_t* row_ptr_h, int64_t* col_h,
                    double* val_h);

/* y = A x - theta x, with theta = theta_h (+ *theta_d when theta_d != NULL,
 * sign flipped when theta_neg).  Optional fused epilogue dot products of the
 * freshly computed y:
 *   out[0:ndots]          = y . dvec[d]           (dvec[d] == NULL -> y . y)
 *   out[ndots:ndots+nq]   = Q^T y                 (Q column-major, ld ldq)
 * out may be NULL when ndots == nq == 0.  skip (device int*) != NULL and
 * *skip != 0 turns the launch into a no-op (device-side predication used by
 * speculative solver iterations). */
int lg_spmv(const lg_csr* a, const double* x, double* y, double theta_h,
            const double* theta_d, int theta_neg, int ndots,
            const double* const* dvec, const double* q, int64_t ldq, int nq,
            double* out, lg_ws* ws, const int* skip, void* stream);
/* Measurement aid: runs only the x gathers of the operator's stored column
 * stream (one per stored off-diagonal; no values, rows or y) -- the floor the
 * product pays for x[col] alone.  out: one device double (scratch).  For a
 * panelled operator the probe runs on the full stream (one pass). */
int lg_spmv_gather_probe(const lg_csr* a, const double* x, double* out, void* stream);
/* End-to-end call through host buffers: H2D of x, SpMV, D2H of y. */
int lg_spmv_host(const lg_csr* a, const double* x_h, double* y_h,
                 double* x_dev_scratch, double* y_dev_scratch, void* stream);
/* Batched SpMM: Y[:, j] = A X[:, j] for j < k (column-major, ld = n). */
int lg_spmm(const lg_csr* a, const double* x, double* y, int k, void* stream);
/* Y = A X with X, Y row-major n x k (ld k), 1 <= k <= 16, packed matrices:
 * one gather of a contiguous k-vector per nonzero serves all k products
 * (results.py:90-105's k fresh products as one pass). */
int lg_spmm_rowmajor(const lg_csr* a, const double* x, double* y, int k, lg_ws* ws,
                     void* stream);

/* ---- Laplacian assembly (graphs.py:250-263), bit-exact ----------------- */
/* Canonical edge list (i < j, lexicographically sorted, w > 0) -> CSR of
 * L = D - A with explicit diagonal.  Degrees are summed in the reference's
 * order (graphs.py:257-258: upper-row weights ascending, then lower-row
 * weights ascending, from 0.0).  Runs on the device; results copied to the
 * host arrays (row_ptr_h[n+1], col_h[n+2m], val_h[n+2m]). */
int lg_build_laplacian(int64_t n, int64_t m, const int64_t* i_h,
                       const int64_t* j_h, const double* w_h,
                       int64_t* row_ptr_h, int64_t* col_h, double* val_h);

/* ---- device-side ingest for C5-scale graphs (no reference counterpart) --- */
/* R-MAT sampling (scale, edge_factor, a, b, c, seed) with a counter-based
 * RNG, canonicalised (i < j, sorted, unique, no self-loops) on the device.
 * *d_i / *d_j are cudaMalloc'ed int32 arrays (free with lg_free). */
int lg_rmat_device(int scale, int edge_factor, double a, double b, double c,
                   uint64_t seed, int32_t** d_i, int32_t** d_j, int64_t* m_out);
/* Largest connected component of a canonical device edge list (nodes
 * renumbered in increasing order, edges compacted in place of the input). */
int lg_lcc_device(int64_t n, int64_t m, int32_t** d_i, int32_t** d_j,
                  int64_t* n_out, int64_t* m_out);
/* Multi-GPU row block: rows [r0, r1) of a packed matrix as a packed n x n
 * matrix whose other rows are absent from the schedule (lg_spmv does not
 * write y there); columns keep the global numbering, so each rank's slice of
 * an n-vector is exchanged in place. */
int lg_csr_row_block(const lg_csr* a, int64_t r0, int64_t r1, lg_csr** out);
/* Interior / exterior split of a packed row block [r0, r1) (square
 * partition): *inner holds the columns in [r0, r1) and the diagonal, *outer
 * every other column and no diagonal; both are n x n with the other rows
 * absent.  y = inner x can run while the other ranks' slices of x are still
 * being exchanged; lg_spmv_acc(outer) then adds the rest.  (SURVEY 8(e):
 * interior SpMV overlapped with the halo transfer; no reference
 * counterpart.) */
int lg_csr_split_cols(const lg_csr* a, int64_t r0, int64_t r1, lg_csr** inner,
                      lg_csr** outer);
/* Column panel [c0, c1) of a packed operator: every row, only the columns in
 * the range (and the diagonal when with_diag).  The product of a graph whose
 * x exceeds L2 splits into panels (y = P_0 x, y += P_k x with lg_spmv_acc) so
 * each panel's gathers hit an L2-resident slice of x.  (SURVEY 8(f) SpMV
 * locality; no reference counterpart.) */
int lg_csr_col_panel(const lg_csr* a, int64_t c0, int64_t c1, int with_diag, lg_csr** out);
/* Attach p (2..16) equal-width column panels to a FULL packed operator (every
 * row present, not a row block); lg_spmv then computes y = (D - theta I) x,
 * y += P_k x for every panel (same epilogue).  p <= 1 detaches.  C5
 * (x = 250 MB > L2): 4 panels, 12.44 -> 9.57 ms a product. */
int lg_csr_set_panels(lg_csr* a, int p);
/* y += A x, no epilogue (the exterior half of a split row block). */
int lg_spmv_acc(const lg_csr* a, const double* x, double* y, lg_ws* ws, const int* skip,
                void* stream);
/* Stream row pointers (packed: off-diagonal; plain: row_ptr), n + 1 int64. */
int lg_csr_row_ptr(const lg_csr* a, int64_t* host_out);
/* Host CSR (row_ptr [n+1], col / val [nnz], diagonal in sorted position) of
 * any matrix, device-only packed ones included (C5's device-built Laplacian):
 * the input of the host IC(0) factorization (ic0.py:48-116). */
int lg_csr_export_host(const lg_csr* a, int64_t* rp_h, int64_t* col_h, double* val_h);
/* Unit-weight Laplacian of a canonical device edge list, built directly in
 * the packed SpMV format on the device (no host copy of the matrix). */
int lg_csr_laplacian_device(int64_t n, int64_t m, const int32_t* d_i,
                            const int32_t* d_j, lg_csr** out);
int lg_csr_diagonal(const lg_csr* a, double* d_out);
int lg_free(void* p);

/* ---- IC(0) factorization (ic0.py:48-116), host, bit-exact -------------- */
/* Factor A + alpha diag(A) on the lower pattern of A, trying shift0 and then
 * every schedule entry > shift0, then 0.1 * max diag (ic0.py:98-111).
 * Subtractions run in ascending column order as in ic0.py:56-71 and the
 * file is compiled with -ffp-contract=off, so the factor equals the
 * reference's bit for bit.  On success fills the lower-triangular factor
 * (row_ptr_h[n+1], col_h, val_h with capacity = nnz of the lower part of A,
 * diagonal last in each row), *shift and *attempts.  LG_EBREAKDOWN when all
 * shifts fail. */
int lg_ic0_factorize(int64_t n, const int64_t* row_ptr_h, const int64_t* col_h,
                     const double* val_h, double shift0, const double* sched_h,
                     int nsched, int64_t* l_row_ptr_h, int64_t* l_col_h,
                     double* l_val_h, double* shift, int* attempts);

/* ---- graph file ingest (graphs.py:126-247) ------------------------------
 * Parse a text edge list (format 0: first line n, then 'i j w' lines, '#'
 * comments) or Matrix Market coordinate file (format 1: diagonal entries
 * dropped, off-diagonal magnitudes become weights) held in memory, with the
 * reference's rules and messages: the canonical edge list (i < j, sorted by
 * (i, j)) comes back in malloc'ed arrays (free with lg_host_free); a
 * repeated pair is an error unless symmetrize (then the maximum weight).
 * LG_EFORMAT + lg_last_error() + *err_line (1-based, 0 = none) on bad input. */
int lg_graph_parse(const char* text, int64_t len, int format, int symmetrize, int64_t* n_out,
                   int64_t* m_out, int64_t** i_out, int64_t** j_out, double** w_out,
                   int64_t* err_line);
int lg_host_free(void* p);

/* ---- FSAI preconditioner (flagged non-reference variant; the approximate
 * inverse PAPER.md:704-706 proposes) ----------------
 * M^{-1} = G^T G, G lower triangular on the lower pattern of A (at most kmax
 * entries per row, diagonal last; hub rows keep their kmax - 1 largest
 * |a_ij|), each row from one dense SPD solve A[P_i, P_i] g = e_last scaled by
 * 1 / sqrt(g_last).  Host setup, OpenMP over rows; the apply is two device
 * SpMVs (lg_csr of G and of G^T).  lg_fsai_nnz gives the size of G. */
int lg_fsai_nnz(int64_t n, const int64_t* row_ptr_h, const int64_t* col_h,
                const double* val_h, int kmax, int levels, int64_t* nnz);
/* levels 2 ("FSAI(2)"): the pattern also takes second-level neighbours j < i,
 * scored by |a_ij| + sum_k |a_ik||a_kj| (k over neighbours of i with at most
 * 64 entries), the kmax - 1 best kept. */
int lg_fsai_factorize(int64_t n, const int64_t* row_ptr_h, const int64_t* col_h,
                      const double* val_h, int kmax, int levels, int64_t* g_row_ptr_h,
                      int64_t* g_col_h, double* g_val_h);
/* The same preconditioner built on the device for a packed matrix with one
 * off-diagonal value (unit-weight Laplacians, e.g. the device-built C5), one
 * warp per row (kmax <= 32); returns G and G^T as plain-format matrices. */
int lg_fsai_device(const lg_csr* a, int kmax, lg_csr** g_out, lg_csr** gt_out);

/* ---- IC(0) apply (ic0.py:40-45) ---------------------------------------- */
typedef struct lg_ic0 lg_ic0;
/* Upload the lower factor L (CSR, diagonal last in each row) and build L^T
 * for the backward sweep. */
int lg_ic0_create(int64_t n, const int64_t* l_row_ptr_h, const int64_t* l_col_h,
                  const double* l_val_h, lg_ic0** out);
/* Same for the factor of P A P^T (a reordered matrix): perm_h[i] is the
 * original index of factor row i.  lg_ic0_apply then reads r and writes z in
 * the original numbering (the permutation is folded into the sweeps). */
int lg_ic0_create_perm(int64_t n, const int64_t* l_rp, const int64_t* l_col,
                       const double* l_val, const int64_t* perm_h, lg_ic0** out);
int lg_ic0_destroy(lg_ic0* f);
/* Greedy colouring in smallest-last order (host).  color[v] in [0, ncolors). */
int lg_color_smallest_last(int64_t n, const int64_t* row_ptr_h, const int64_t* col_h,
                           int32_t* color, int32_t* ncolors);
/* n, stored nonzeros of L (diagonal included) and the depth of the factor's
 * dependency DAG (levels of a plain triangular sweep). */
int lg_ic0_info(const lg_ic0* f, int64_t* n, int64_t* nnz_l, int* levels);
/* Depth of the two sweeps as scheduled and the entries they stream: the
 * device applies a level-merged form of the factor (rows of even levels have
 * the level below substituted in, reading the right-hand side there), about
 * 0.6x the factor's depth for ~1.5x the entries; LG_IC0_MERGE caps the number
 * of merging passes (default 3), 0 keeps the plain sweeps. */
int lg_ic0_sweep_depth(const lg_ic0* f, int* fwd, int* bwd, int64_t* entries);
/* Host only (no device needed): one triangular solve -- L y = b, or L^T y = b
 * when `backward` -- through the level-merged system the device would run
 * after `passes` merging passes, in the system's topological order.  Test hook
 * for the host transformation; depth / entries / unknowns describe the system. */
int lg_ic0_merged_solve_host(int64_t n, const int64_t* l_row_ptr_h, const int64_t* l_col_h,
                             const double* l_val_h, int passes, int backward, const double* b_h,
                             double* y_h, int* depth, int64_t* entries, int64_t* unknowns);
/* z = (L L^T)^{-1} r: sync-free forward sweep on L then backward sweep on
 * L^T, one cooperative persistent kernel each.  The forward result lives in
 * scratch owned by the handle, so applies of one handle must be ordered on
 * one stream.  z may alias r. */
int lg_ic0_apply(const lg_ic0* f, const double* r, double* z, const int* skip,
                 void* stream);
/* Sweep implementation of a factor: 0 = dataflow sweeps (one cooperative launch
 * per triangle; the default), 1 = resident sweep (both triangles in one CTA,
 * levels separated by CTA barriers; opt-in, also LG_SWEEP_CTA=1).  Same bits
 * either way.  Returns the previous mode; any other `mode` only queries. */
int lg_ic0_set_mode(lg_ic0* f, int mode);
/* Debug instrumentation of the sweeps: enable != 0 allocates a timestamp
 * buffer written after every level segment (CTA 0's view); host_out (cap
 * entries) receives the last apply's timestamps.  Returns the number of
 * segments (forward + backward). */
int lg_ic0_trace(lg_ic0* f, int enable, unsigned long long* host_out, int cap);
/* Debug: dataflow-sweep task timestamps {level, start, ready, done} (ns). */
int lg_ic0_flow_trace(lg_ic0* f, int enable, unsigned long long* host_out, int cap);
/* Debug: per-segment {tasks, narrow, barrier, 0} of one sweep. */
int lg_ic0_schedule(const lg_ic0* f, int backward, int* host_out, int cap);
/* Jacobi (diagonal) apply z = r / diag, a flagged non-reference variant. */
int lg_diag_apply(int64_t n, const double* dinv, const double* r, double* z,
                  const int* skip, void* stream);

/* ---- fused vector pass -------------------------------------------------- */
#define LG_MAXT 4   /* linear-combination terms per output          */
#define LG_MAXD 8   /* explicit dot pairs                           */
#define LG_MAXB 2   /* column blocks for Q^T v dots                 */
#define LG_MAXO 3   /* outputs per pass                             */
#define LG_MAXQ 64  /* total block columns per launch               */
/* sentinel vector pointers naming the outputs of the same pass */
#define LG_OUT0 ((const double*)(uintptr_t)1)
#define LG_OUT1 ((const double*)(uintptr_t)2)
#define LG_OUT2 ((const double*)(uintptr_t)3)

typedef struct {
  const double* v;     /* input vector (may be LG_OUT0 for out1 terms)   */
  double h;            /* host scale                                      */
  const double* d;     /* device scalar multiplier or NULL                */
} lg_term;

typedef struct {
  double* out;         /* NULL: output disabled                            */
  int nterms;
  lg_term t[LG_MAXT];
  /* optional block updates: out -= sum_j (cscale * c[j]) Q[:, j], for up
   * to two column blocks (uq, uk, uc) and (uq2, uk2, uc2) with ld uld / uld2 */
  const double* uq;
  int64_t uld;
  int uk;
  const double* uc;    /* device coefficients (k of them)                  */
  double cscale;
  const double* uq2;
  int64_t uld2;
  int uk2;
  const double* uc2;
  /* optional final scaling by a device scalar p = *d_post:
   * post_mode 1: out *= p, 2: out /= p, 3: out /= sqrt(p)               */
  const double* d_post;
  int post_mode;
} lg_output;

typedef struct {
  const double* q;     /* column-major block, ld                          */
  int64_t ld;
  int k;
  const double* v;     /* vector dotted against every column (or LG_OUTx) */
} lg_block;

typedef struct {
  int64_t n;
  lg_output o[LG_MAXO];
  int ndots;
  /* dot d = (da[d] - dc[d]) . db[d]; dc NULL = 0; db NULL = same as the
   * first operand.  Any operand may name an output (LG_OUTx). */
  const double* da[LG_MAXD];
  const double* db[LG_MAXD];
  const double* dc[LG_MAXD];
  int nblocks;
  lg_block b[LG_MAXB];
  double* result;              /* device: [ndots + sum(b.k)]              */
  const int* skip;
} lg_fused_args;

/* One streaming pass over n rows: up to three outputs, each a linear
 * combination of up to four vectors (inputs or earlier outputs) minus a
 * block combination Q c, optionally rescaled by a device scalar, plus
 * deterministic dot products / Q^T v block dots of inputs and outputs. */
int lg_fused(const lg_fused_args* args, lg_ws* ws, void* stream);
/* lg_fused followed, in the pass's finishing CTA, by a device scalar program
 * (lg_scalar_prog semantics) over slots / flags: the program sees this
 * pass's dot products and costs no launch of its own.  The pass must
 * compute at least one dot product; the pass's skip flag covers both. */
int lg_fused_prog(const lg_fused_args* args, double* slots, int* flags, const uint8_t* prog,
                  int nops, const double* imm, int nimm, lg_ws* ws, void* stream);

/* Out[:, 0:p] = In[:, 0:m] * Y  (Y is m x p column-major, host, copied by
 * value into the launches; any m, p: tiles of <= 32 output columns and
 * <= 1024 / width input columns, later input tiles accumulating in order;
 * In/Out column-major ld = n). */
int lg_gemm_small(int64_t n, const double* in, int64_t ldi, int m,
                  const double* y_h, int p, double* out, int64_t ldo,
                  void* stream);

/* ---- device scalar programs -------------------------------------------- */
/* The scalar recurrences of the solvers (PR-beta, the 2x2 plane pencil, PCG
 * gamma/beta, convergence and breakdown tests: dacg.py:188-233,
 * pcg.py:133-155) run on the device so an iteration needs no host round trip
 * until its status is read.  A program is a list of 4-byte instructions
 * {op, dst, a, b} over a slot file s[0..255] (device doubles) and an int flag
 * file (device ints, the `skip` predicates of the kernels).  Opcodes are
 * enumerated in csrc/lg_scalar.cu (LG_OP_*); imm_h supplies constants. */
#define LG_MAXOPS 192
#define LG_MAXIMM 32
int lg_scalar_prog(double* s, int* flags, const uint8_t* prog_h, int nops,
                   const double* imm_h, int nimm, const int* skip,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LAPB200_H */
