/*
 * rgb200.h — C ABI of librgb200.so, the sm_100a hot path of block GCRO-DR
 * (block recycled GMRES, arXiv 1604.01713) behind the recgmres Python API.
 *
 * Conventions (every entry point):
 *   - Plain pointers and sizes; no torch / numpy types.  All pointers named
 *     d_* are DEVICE pointers owned by the caller; the library never
 *     allocates device memory.  Scratch memory is caller-provided and sized
 *     with rg_*_workspace_bytes().  The workspace counter word must be zero
 *     when first handed to the library (the kernels leave it zero again).
 *   - Dense blocks are column-major (Fortran order, like the reference's
 *     as_block, sparse_core.py:51-58) with a leading dimension ld >= n.
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     stream-ordered and asynchronous (no host synchronisation inside).
 *   - Return value: RG_OK (0) on success, RG_EBADARG (1) for bad shapes /
 *     arguments (the Python layer raises ShapeError/ValueError, as the
 *     reference does), RG_ECUDA (2) for a CUDA launch error.  The message of
 *     the last failure on the calling thread is available from
 *     rg_last_error().
 *   - Floating point is IEEE float64 throughout.
 */
#ifndef RGB200_H
#define RGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RG_OK 0
#define RG_EBADARG 1
#define RG_ECUDA 2

/* Library identification: returns a static string "rgb200 <version> sm_100a". */
const char* rg_version(void);

/* Message of the last failing call on this thread ("" when none). */
const char* rg_last_error(void);

/* Number of SMs of the current device (for grid sizing / diagnostics). */
int rg_device_sm_count(void);

/*
 * Y = A * X for a CSR matrix A and an n_cols x p block X.
 *
 * Replaces recgmres.sparse_core.spmm -> _spmm_kernel
 * (/root/reference/pkg/src/recgmres/sparse_core.py:132-149 and :25-40) and
 * spmv (:152-157).  Every output entry Y[i,c] is accumulated from 0.0 over
 * the row's stored nonzeros in ascending storage order with separately
 * rounded multiply and add (no FMA) — the reference kernel's exact
 * arithmetic, so results are bitwise identical to it.
 *
 * Rows [row_begin, row_end) are computed (row-range launches let the
 * distributed layer overlap interior rows with the halo exchange).  Column
 * indices j < n_local read X[j + c*ldx]; j >= n_local read the ghost block
 * Xg[(j - n_local) + c*ldg] (pass n_local = n_cols, d_xg = NULL on one GPU).
 * row_ptr / col_idx are int32 (nnz < 2^31).
 */
int rg_spmm_csr_f64(int64_t n_rows, int64_t row_begin, int64_t row_end,
                    const int32_t* d_row_ptr, const int32_t* d_col_idx,
                    const double* d_vals,
                    const double* d_x, int64_t ldx, int64_t n_local,
                    const double* d_xg, int64_t ldg,
                    int32_t p, double* d_y, int64_t ldy, void* stream);

/*
 * The same product for matrices whose nonzeros lie on <= 32 diagonals (the
 * stencil configurations), from a diagonal layout built once per matrix:
 *   d_dia   n_rows x ndiag column-major (ld_dia), value of row i on diagonal
 *           h_offsets[d] (column i + h_offsets[d]), 0 where i stores none
 *   d_mask  n_rows uint32 bit masks: bit d set iff row i stores that entry
 *   h_offsets ascending (host array)
 * Each row sums its stored entries in ascending column order with the
 * reference's separately rounded arithmetic: bitwise equal to
 * rg_spmm_csr_f64 on the same matrix.  X windows per block of rows stream in
 * by TMA; no column indices are read.  d_row_ptr (optional) is the CSR row
 * pointer, used only for the launch record's byte model.  Requires 16-byte
 * aligned operands with even leading dimensions; no ghost columns.
 */
int rg_spmm_dia_f64(int64_t n_rows, int64_t row_begin, int64_t row_end, int32_t ndiag, const int32_t* h_offsets,
                    const double* d_dia, int64_t ld_dia, const uint32_t* d_mask, int64_t n_cols,
                    const double* d_x, int64_t ldx, int32_t p, double* d_y, int64_t ldy, const int32_t* d_row_ptr,
                    void* stream);

/*
 * The diagonal layout built from the CSR arrays on the device, once per
 * matrix (no reference counterpart: the reference keeps CSR only).
 *   rg_dia_offsets   distinct offsets col - row of rows [row_begin, row_end)
 *                    into d_table (64 int32, preset to INT32_MIN);
 *                    *d_overflow (preset 0) = 1 if more exist
 *   rg_dia_fill_f64  values into d_dia (n_rows x ndiag, zeroed) and per-row
 *                    masks (zeroed) for those rows, given the ascending
 *                    offsets on the device.  A layout built over a sub-range
 *                    (the interior rows of a row partition, which reference
 *                    owned columns only) serves products inside that range.
 */
int rg_dia_offsets(int64_t n_rows, int64_t row_begin, int64_t row_end, const int32_t* d_rp, const int32_t* d_ci,
                   int32_t* d_table, int32_t* d_overflow, void* stream);
int rg_dia_fill_f64(int64_t n_rows, int64_t row_begin, int64_t row_end, const int32_t* d_rp, const int32_t* d_ci,
                    const double* d_vals, int32_t ndiag, const int32_t* d_offsets, double* d_dia, int64_t ld_dia,
                    uint32_t* d_mask, void* stream);

/*
 * Fused tall-skinny "update, triangular solve, Gram" pass over an n x p
 * block Z (one read of every operand, one write of Z):
 *
 *   z   = (d_zin ? Zin : 0)                       (n x p)
 *   z  += alpha1 * (X1 @ S1)                      X1: n x a1, S1: a1 x p
 *   z  += alpha2 * (X2 @ S2)                      X2: n x a2, S2: a2 x p
 *   z   = z @ inv(R1)   if d_r1                   R1: p x p upper triangular
 *   z   = z @ inv(R2)   if d_r2
 *   Zout = z            if d_zout (may alias Zin)
 *   gram_mode 1:  Gout = Gb^T @ z                 Gb: n x gc, Gout: gc x p
 *   gram_mode 2:  Gout = z^T @ z                  (gc must equal p)
 *   gram_mode 3:  Gout[c] = sum_i z[i,c]^2        (column sums of squares)
 *
 * S1/S2/R1/R2 and Gout are DEVICE arrays, column-major with ld = rows.
 * Gram sums are reduced in a fixed order (deterministic run to run).
 * When Gb aliases X1 (same pointer and ld, gc <= a1), and when X1 == X2
 * with a1 == a2, the operand is streamed once.
 *
 * Implementation: passes streaming >= 64 columns without norms run the
 * warp-specialised kernel (producer warps fill a CTA-shared ring of 64-row
 * stages, consumer warps run the DMMA update / Gram from it); narrower
 * passes, norms and p > 16 run the per-warp slab-ring kernel (v6, v5, v3).
 * RG_TALL_WS=0 in the environment forces the latter (A/B runs).
 *
 * Replaces the numpy/OpenBLAS products of the hot path:
 *   arnoldi.step CGS2 branch   arnoldi.py:172-180   (C^T Ahat, Ahat -= C S,
 *                                                    W^T Ahat, Ahat -= W c)
 *   reduced_qr Gram / apply    dense_kernels.py:41  (CholQR2 passes)
 *   C-scrubs                   solver.py:155, :266-267, :281, :297
 *   _apply_update              solver.py:175-179
 *   recycle products           recycling.py:119-120, :165-169, :186-188
 *   column norms               solver.py:214, :274, :299, :321
 */
int rg_tall_f64(int64_t n, int32_t p,
                const double* d_zin, int64_t ldzin,
                double* d_zout, int64_t ldzout,
                const double* d_x1, int64_t ldx1, int32_t a1,
                const double* d_s1, double alpha1,
                const double* d_x2, int64_t ldx2, int32_t a2,
                const double* d_s2, double alpha2,
                const double* d_r1, const double* d_r2,
                int32_t gram_mode, const double* d_gb, int64_t ldgb, int32_t gc,
                double* d_gout,
                void* d_work, int64_t work_bytes, void* stream);

/* Workspace bytes rg_tall_f64 needs for these shapes. */
int64_t rg_tall_workspace_bytes(int64_t n, int32_t p, int32_t a1, int32_t a2,
                                int32_t gram_mode, int32_t gc);

/*
 * Cholesky G = R^T R of a p x p SPD Gram (device, column-major, ld = p),
 * p <= 64.  Writes R (upper, ld = p; strictly-lower part zeroed) and
 * d_status[0]: 0 ok; 1 not positive definite / non-finite; 2 ill
 * conditioned (min_j R_jj^2 < cond_tol * max_j G_jj).  Used by the CholQR2
 * path of reduced_qr (dense_kernels.py:31-48); status != 0 sends the block
 * to the Householder TSQR path instead.
 */
int rg_chol_f64(int32_t p, const double* d_g, double* d_r, int32_t* d_status,
                double cond_tol, void* stream);

/*
 * Householder TSQR of an n x p block (p <= 32), in place:  X = Q R with Q
 * overwriting X and R (p x p, upper, ld = p) written to d_r.  Signs follow
 * the reference convention R_jj >= 0 (dense_kernels.py:42-45).  This is the
 * robust path of reduced_qr (np.linalg.qr, dense_kernels.py:41), used when
 * CholQR2 declines (near rank-deficient blocks, breakdown handling).
 */
int rg_tsqr_f64(int64_t n, int32_t p, double* d_x, int64_t ldx, double* d_r,
                void* d_work, int64_t work_bytes, void* stream);
int64_t rg_tsqr_workspace_bytes(int64_t n, int32_t p);

/*
 * One CGS2 projection of an n x p block Z (in place) against C (n x k) and
 * the basis W (n x w), in the reference's order (arnoldi.py:172-180: two
 * passes, each C then W), as the fused rg_tall_f64 schedule the Python
 * layer uses.  d_coef receives S1 (k x p) | c1 (w x p) | S2 | c2 packed
 * column-major (F = S1 + S2, H = c1 + c2 on the host, arnoldi.py:177,180);
 * if d_gram is non-NULL it receives Z^T Z of the projected block (the first
 * CholQR Gram).  p <= 16, k <= 128 and w <= 128 (each basis is one Gram
 * operand of rg_tall_f64; callers split wider bases).
 * joint != 0 (the solver's layout: W directly follows C in one allocation,
 * d_w == d_c + k*ldc, ldw == ldc, k + w <= 128, and C is orthogonal to W
 * -- the caller asserts this; the library cannot check it)
 * runs the projection against [C W] as one basis in three passes -- the
 * same CGS2 up to rounding -- and d_coef holds G1 = [S1; c1] | G2 =
 * [S2; c2], each (k+w) x p; the workspace must then cover gc = k + w.
 * joint == 0 always runs the sequential schedule (any C, W).
 */
int rg_cgs2_f64(int64_t n, int32_t p, double* d_z, int64_t ldz,
                const double* d_c, int64_t ldc, int32_t k,
                const double* d_w, int64_t ldw, int32_t w,
                double* d_coef, double* d_gram, int32_t joint,
                void* d_work, int64_t work_bytes, void* stream);

/*
 * CholQR2 of X (n x p, p <= 16) into Q (must not alias X): d_small holds
 * G1 | R1 | G2 | R2 (4 p x p column-major blocks; R = R2 R1 with r_jj > 0),
 * d_status[0..1] the two Cholesky statuses (non-zero: fall back to
 * rg_tsqr_f64 on X, as reduced_qr does).  gram_ready != 0 means G1 = X^T X
 * is already in d_small (e.g. from rg_cgs2_f64's d_gram).
 * Replaces np.linalg.qr in reduced_qr (dense_kernels.py:41).
 */
int rg_cholqr2_f64(int64_t n, int32_t p, const double* d_x, int64_t ldx, double* d_q, int64_t ldq,
                   double* d_small, int32_t* d_status, int32_t gram_ready,
                   void* d_work, int64_t work_bytes, void* stream);

/*
 * complex128 twins (BASELINE configs[4]; the reference is real-only, so these
 * follow the complex restatement of SURVEY.md §8c: conjugate transposes,
 * real non-negative r_jj).  Complex blocks are column-major arrays of
 * interleaved (re, im) doubles; ld counts complex elements.
 *   rg_spmm_csr_c128  as rg_spmm_csr_f64 (vals interleaved complex); every
 *                     partial product and sum of (a*x) is rounded separately
 *   rg_tall_c128      as rg_tall_f64 with Gout = Gb^H z / z^H z, p <= 16;
 *                     gc <= 48 (p <= 8) or 32 (p > 8; 64 for a pure Gram),
 *                     staged term columns <= 256 (p <= 8) or 128 (p > 8);
 *                     mode 3 writes p real sums of |z|^2
 *   rg_chol_c128      Hermitian Cholesky G = R^H R, p <= 64
 */
int rg_spmm_csr_c128(int64_t n_rows, int64_t row_begin, int64_t row_end,
                     const int32_t* d_row_ptr, const int32_t* d_col_idx, const double* d_vals,
                     const double* d_x, int64_t ldx, int64_t n_local, const double* d_xg, int64_t ldg,
                     int32_t p, double* d_y, int64_t ldy, void* stream);
int rg_tall_c128(int64_t n, int32_t p, const double* d_zin, int64_t ldzin, double* d_zout, int64_t ldzout,
                 const double* d_x1, int64_t ldx1, int32_t a1, const double* d_s1, double alpha1,
                 const double* d_x2, int64_t ldx2, int32_t a2, const double* d_s2, double alpha2,
                 const double* d_r1, const double* d_r2, int32_t gram_mode, const double* d_gb, int64_t ldgb,
                 int32_t gc, double* d_gout, void* d_work, int64_t work_bytes, void* stream);
int64_t rg_tall_c128_workspace_bytes(int64_t n, int32_t p, int32_t a1, int32_t a2, int32_t gram_mode, int32_t gc);
int rg_chol_c128(int32_t p, const double* d_g, double* d_r, int32_t* d_status, double cond_tol, void* stream);

/*
 * ILU(0) preconditioner (reference precond.py:33-90).
 *   rg_wave_schedule  HOST routine (host pointers, run once per factor): the
 *                     level schedule of the lower (upper = 0) or upper
 *                     (upper = 1) dependency graph of a CSR pattern with
 *                     diagonal positions diag_pos.  Writes the rows in level
 *                     order to order[n] and chunk offsets (chunks of <=
 *                     chunk_rows rows of one level, a multiple of 32) to
 *                     chunk[rg_wave_max_chunks(n)];
 *                     returns the chunk count (-1 on bad arguments);
 *                     *width = the most chunks in one level (the kernels
 *                     size their persistent grid from it).
 *   rg_ilu0_f64       in-place IKJ ILU(0) of d_vals on the lower schedule:
 *                     afterwards the strictly lower entries hold L (unit
 *                     diagonal implicit) and the rest U, bitwise as
 *                     precond.py:60-72.  *d_zero_row (caller sets INT64_MAX)
 *                     receives the first row whose pivot is 0 (the reference
 *                     raises ZeroPivotError there, precond.py:63-64, :71-72).
 *   rg_sptrsv_f64     X = L^-1 B (upper = 0, lower schedule) or X = U^-1 B
 *                     (upper = 1, upper schedule) on the combined LU pattern;
 *                     p <= 64 columns; X may alias B (replaces
 *                     precond.py:87-88's spsolve_triangular).
 * Both kernels are persistent, sync-free wavefronts: lanes wait on per-row
 * completion flags in d_work (rg_wave_workspace_bytes(n) bytes, zeroed once
 * at allocation; each call passes a new positive epoch).
 */
int64_t rg_wave_workspace_bytes(int64_t n);
int64_t rg_wave_max_chunks(int64_t n);
int32_t rg_wave_schedule(int64_t n, const int32_t* row_ptr, const int32_t* col_idx, const int32_t* diag_pos,
                         int32_t upper, int32_t chunk_rows, int32_t* order, int32_t* chunk, int32_t* n_levels,
                         int32_t* width);
int rg_ilu0_f64(int64_t n, const int32_t* d_row_ptr, const int32_t* d_col_idx, double* d_vals,
                const int32_t* d_diag_pos, const int32_t* d_order, const int32_t* d_chunk, int32_t nchunks,
                int32_t width, int64_t* d_zero_row, void* d_work, int64_t work_bytes, int32_t epoch, void* stream);
int rg_sptrsv_f64(int64_t n, const int32_t* d_row_ptr, const int32_t* d_col_idx, const double* d_vals,
                  const int32_t* d_diag_pos, const int32_t* d_order, const int32_t* d_chunk, int32_t nchunks,
                  int32_t width, int32_t upper, int32_t p, const double* d_b, int64_t ldb, double* d_x, int64_t ldx, void* d_work,
                  int64_t work_bytes, int32_t epoch, void* stream);
/*
 * Level-ordered solve (used by apply_precond):
 *   rg_wave_permute      HOST: renumber one triangle by its schedule (pos,
 *                        permuted rp/ci, entry map); returns its entry count
 *   rg_gather_f64        dst[j] = src[idx[j]] (permuted values, U diagonal)
 *   rg_permute_rows_f64  move a block between the column-major original
 *                        order (null pos) and a row-major level order
 *   rg_sptrsv_perm_f64   in-place solve on the row-major level-ordered block;
 *                        d_dval = U's diagonal in level order (null: unit L)
 */
int64_t rg_wave_permute(int64_t n, const int32_t* row_ptr, const int32_t* col_idx, const int32_t* diag_pos,
                        int32_t upper, const int32_t* order, int32_t* pos, int32_t* rp_out, int32_t* ci_out,
                        int64_t* emap);
int rg_gather_f64(int64_t m, const int64_t* d_idx, const double* d_src, double* d_dst, void* stream);
int rg_permute_rows_f64(int64_t n, int32_t p, const double* d_src, int64_t lds, const int32_t* d_pos_src,
                        double* d_dst, int64_t ldd, const int32_t* d_pos_dst, void* stream);
int rg_sptrsv_perm_f64(int64_t n, const int32_t* d_rp, const int32_t* d_ci, const double* d_vals,
                       const double* d_dval, const int32_t* d_chunk, int32_t nchunks, int32_t width, int32_t p,
                       double* d_xw, void* d_work, int64_t work_bytes, int32_t epoch, void* stream);

/*
 * Halo pack of the row-partitioned SpMM (the reference is
 * single-process, its product is sparse_core.py:25-40):
 *   out[i + c*ldo] = Z[idx[i] + c*ldz],  i < k, c < p
 * esz = 8 (float64) or 16 (complex128, ld in complex elements).  Each column
 * of out is one contiguous send; the peer receives it straight into column c
 * of its ghost block.
 */
int rg_halo_pack(int64_t k, int32_t p, int32_t esz, const int32_t* d_idx, const void* d_z, int64_t ldz,
                 void* d_out, int64_t ldo, void* stream);

/*
 * The same exchange without a transport library, for the ranks of one node:
 *   rg_halo_push  the gather of rg_halo_pack stored straight into the peer's
 *                 ghost block (d_peer_out: a CUDA IPC mapping, rg_ipc_alloc /
 *                 rg_peer_open; NVLink peer stores), then flag = epoch on the
 *                 peer (d_peer_flag, mapped) once every CTA's stores are
 *                 fenced (d_ticket: a zeroed local counter); k = 0 only
 *                 publishes the flag
 *   rg_halo_wait  one small kernel ahead of the boundary rows: waits until
 *                 d_flags[peers[i]] == epoch for every listed peer (host
 *                 array, <= 8), at most timeout_s, else *d_err = epoch
 * Ghost blocks alternate between two buffers with the epoch's parity, and
 * every pair of neighbours signals both ways each epoch, so a rank can be at
 * most one product ahead of a neighbour and never overwrites rows being read.
 */
int rg_halo_push(int64_t k, int32_t p, int32_t esz, const int32_t* d_idx, const void* d_z, int64_t ldz,
                 void* d_peer_out, int64_t ldo, uint32_t* d_peer_flag, uint32_t epoch, uint32_t* d_ticket,
                 void* stream);
int rg_halo_wait(const uint32_t* d_flags, const int32_t* peers, int32_t npeers, uint32_t epoch, double timeout_s,
                 uint32_t* d_err, void* stream);

/*
 * Gram reduction over the row partition through peer memory (SURVEY.md §8e:
 * "the (k+mp) x p Gram matrices are summed" across the GPUs; the reference is
 * single-process -- its products arnoldi.py:172-180 are the global sums).
 * One process per GPU on one node.  Each rank allocates an exchange buffer,
 * passes its 64-byte CUDA IPC handle to the others (any host transport) and
 * maps theirs; after rg_peer_set every Gram / norm pass of rg_tall_f64 /
 * rg_tall_c128 (and so rg_cgs2_f64, rg_cholqr2_f64) finishes the sum over
 * the ranks inside its own kernel: the CTA that sums the CTA partials stores
 * its rank's values into every peer's slot (NVLink peer stores), publishes an
 * epoch flag, waits for the peers' flags and adds the slots in rank order, so
 * every rank holds the same bits.  No NCCL call and no extra launch.
 *   rg_peer_buffer_bytes  size of one exchange buffer
 *   rg_peer_alloc         allocate + zero the local buffer, return its handle
 *   rg_peer_open/close    map / unmap a peer's buffer from its handle
 *   rg_peer_free          release the local buffer
 *   rg_peer_set           register the group (bufs[r] = rank r's buffer as
 *                         mapped here; bufs[rank] = the local one); all ranks
 *                         call it at the same point of their launch sequence;
 *                         timeout_s bounds the in-kernel wait (<= 0: 20 s)
 *   rg_peer_clear         back to single-process sums
 *   rg_peer_active        0, or the registered world size
 *   rg_peer_error         epoch at which a peer failed to arrive in time (0:
 *                         none); synchronises the stream
 *   rg_peer_allreduce_f64 in-place sum over the group of a small device
 *                         buffer (<= 4096 doubles) no rg_tall pass produced
 *   rg_peer_emulate_f64   tests: `world` ranks as one cooperative grid on one
 *                         GPU over local exchange buffers (same device code)
 * All reductions of a process go to one stream, in the same order on every
 * rank.
 */
int64_t rg_peer_buffer_bytes(void);
int rg_ipc_alloc(int64_t bytes, void** d_buf, void* handle64); /* any size (ghost blocks, halo flags) */
int rg_peer_alloc(void** d_buf, void* handle64);
int rg_peer_open(const void* handle64, void** d_buf);
int rg_peer_close(void* d_buf);
int rg_peer_free(void* d_buf);
int rg_peer_set(int32_t world, int32_t rank, void* const* bufs, double timeout_s);
void rg_peer_clear(void);
int32_t rg_peer_active(void);
int rg_peer_error(uint32_t* epoch, void* stream);
int rg_peer_allreduce_f64(double* d_buf, int64_t count, void* stream);
int rg_peer_emulate_f64(int32_t world, int32_t ne, int32_t rounds, uint32_t epoch0, double* d_vals, void* d_buf,
                        void* stream);

/*
 * Launch accounting and per-launch device timing (no reference counterpart:
 * the reference times whole Python calls with perf_counter, bench.py:58-67).
 *   rg_launch_count    kernels launched by this library since load
 *   rg_count_launches  add n (a host replaying a captured CUDA graph of
 *                      library calls reports the kernels each replay runs)
 *   rg_profile_enable  1: clear the records and bracket every kernel-launching
 *                      call (rg_tall_f64, rg_spmm_csr_f64, rg_chol_f64, ...,
 *                      including those the orchestrators make) with CUDA
 *                      events on its stream; 0: stop recording
 *   rg_profile_count   records so far
 *   rg_profile_record  record i: label, device ms (synchronises on its end
 *                      event), algorithmic bytes, FP64
 *                      tensor-core flops, kernels launched
 *   rg_profile_gap     device ms from the end of record i-1 to the start of
 *                      record i (work of other libraries + idle time)
 */
int64_t rg_launch_count(void);
void rg_count_launches(int64_t n);
void rg_profile_enable(int32_t on);
int32_t rg_profile_count(void);
int rg_profile_record(int32_t i, char* label, int32_t label_cap, double* ms, int64_t* bytes, double* flops,
                      int32_t* launches);
int rg_profile_gap(int32_t i, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* RGB200_H */
