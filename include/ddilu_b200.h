/*
 * ddilu_b200.h -- C ABI of libddilu_b200.so (hand-written sm_100a CUDA).
 *
 * The reference (`ddilu`, pure Python + numba) has no FFI layer; its boundary is
 * the public Python API (pkg/src/ddilu/__init__.py:11-59).  Each entry below
 * replaces one numba kernel (or a numpy expression around it) of that package;
 * the file:line it replaces is cited per function.  paper_2303_08881_b200/_lib.py
 * binds these symbols with ctypes (INTEGRATION.md shows the same stub a
 * maintainer of the reference would add).
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless the name ends in _h,
 *   - indices are int32 on the device (nnz < 2^31 is checked by the host side),
 *     values are fp64; CSR rows have strictly increasing columns,
 *   - `stream` is a cudaStream_t passed as void*; nothing synchronises the device,
 *   - the return value is 0 on success, -1000 for a bad argument, or
 *     -(cudaError_t) for a launch failure.
 */
#ifndef DDILU_B200_H
#define DDILU_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- primitives used by the count -> scan -> fill setup passes (the reference
 * uses np.cumsum: e.g. sparse.py:449, factor.py:254-257) */
long long ddilu_scan_tmp_elems(long long n);
/* out[0..n] = exclusive prefix sums of in[0..n-1], out[n] = total; in == out allowed */
int ddilu_exclusive_scan_i32(const int *in, int *out, long long n, int *tmp, void *stream);
long long ddilu_sort_tmp_elems(long long n);
/* stable LSD radix sort of (key, value) pairs on the low `bits` bits of the key */
int ddilu_sort_pairs_i32(int *keys, int *vals, int *keys_alt, int *vals_alt, long long n, int bits, int *tmp,
                         void *stream);

/* ---- sparse.py:219-225 `_spmv` (+ the `b - A x` residual expressions of
 * krylov.py:106,168 and precond.py:258,264,354,379).  Rows [row_begin,row_end).
 * mode 0: y = A x; 1: y = b - A x; 2: y = b + A x.  y/b are indexed by row. */
int ddilu_spmv_csr_f64(int row_begin, int row_end, const int *row_ptr, const int *col_idx, const double *values,
                       const double *x, const double *b, double *y, int mode, void *stream);
/* the same with the average row length of the range as a hint (0 = unknown): picks rows per CTA and the
 * shared-memory stage so that 27-point / ILUT-length rows still take the staged path and short rows get
 * full occupancy */
int ddilu_spmv_csr_f64_tuned(int row_begin, int row_end, const int *row_ptr, const int *col_idx, const double *values,
                             const double *x, const double *b, double *y, int mode, double avg_row_len, void *stream);

/* ---- level schedules (absent from the reference: SPEC.md:112; definition in
 * lev[i] = 1 + max lev[j] over the dependencies of row i) */
int ddilu_levels(int n, const int *row_ptr, const int *col_idx, int upper, int *lev, int *max_lev, void *stream);
/* rows sorted by (level, index) [index descending for upper] into `rows`;
 * level_ptr[n_levels+1]; slot_ptr[n_levels+1] = level starts padded to 32;
 * order[n + 32*n_levels] = padded schedule (-1 = empty slot). */
int ddilu_schedule_build(int n, const int *lev, int n_levels, int upper, int *keys, int *rows, int *keys_alt,
                         int *rows_alt, int *sort_tmp, int *level_ptr, int *slot_ptr, int *order, void *stream);

/* ---- sparse.py:228-249 `_lower_solve` / :252-272 `_upper_solve`.
 * *err must hold INT_MAX on entry; on a zero/missing diagonal it receives the
 * smallest failing row (the reference raises ZeroDivisionError for that row). */
int ddilu_sptrsv(int n, int n_slots, const int *order, const int *row_ptr, const int *col_idx, const double *values,
                 const double *b, double *x, int upper, int unit_diag, int *err, void *stream);
/* the same solve with a WARP per row: long rows (ILUT / ILU(k) / 27-point factors, 10-20 dependencies) -- one
 * coalesced load of the row, all dependencies polled at once, products added in storage order by one lane */
int ddilu_sptrsv_warprow(int n, int n_slots, const int *order, const int *row_ptr, const int *col_idx,
                         const double *values, const double *b, double *x, int upper, int unit_diag, int *err,
                         void *stream);

/* Schedule-ordered sliced-ELL form of a factor (group = 32 schedule slots = one
 * warp): gw32[g] = 32 * (longest dependency list in group g) -> scan -> goff;
 * entry k of lane l at goff[g] + 32*k + l (col -1 = padding); sdiag[slot] = pivot.
 * goff == NULL selects the uniform layout: every group has `uniform_width` entries
 * per lane at g * 32 * uniform_width (no descriptor load on the dependency chain).
 * gwait[g] (optional; pos_work = n scratch ints) = the dependency of group g that is latest
 * in the schedule: the warp spins on that one address before checking the others.
 * ddilu_sptrsv_sell is the production solve (same semantics as ddilu_sptrsv;
 * sdiag == NULL means unit diagonal). */
int ddilu_sell_width(int n_slots, const int *order, const int *row_ptr, const int *col_idx, const double *values,
                     int upper, int unit_diag, int *gw32, double *sdiag, int *bad_row, int *pos_work, int *gwait,
                     void *stream);
int ddilu_sell_fill(int n_slots, const int *order, const int *row_ptr, const int *col_idx, const double *values,
                    int upper, const int *goff, int uniform_width, int *scol, double *sval, void *stream);
/* out[g] = gwait[group of prev[g]]: the same kind of indicator one level further back */
int ddilu_compose_wait(int n_groups, const int *gwait, const int *pos, const int *prev, int *out, void *stream);
/* gwait / gfar1 / gfar2 (each optional): single addresses 1 / 2 / 3 levels back a warp waits on before
 * it polls its own dependencies ("trsv_stage_mask" selects which are used); avg_width = average padded
 * entries per lane (0: the uniform width): rows longer than 6 / 14 poll 8 / 16 dependencies per round */
int ddilu_sptrsv_sell(int n, int n_slots, int n_levels, const int *order, const int *goff, int uniform_width,
                      const int *scol, const double *sval, const double *sdiag, const int *gwait, const int *gfar1,
                      const int *gfar2, double avg_width, const double *b, double *x, void *stream);

/* ---- factor.py:270-369 `_iluk_symbolic`: level-of-fill pattern (levels <= klevel), rows >= n_elim keep
 * their trailing block un-eliminated.  Row slabs of row_cap entries: p_* = pivot (L) part, k_* = kept
 * (U / Schur) part with fill levels; *status != 0: a row outgrew row_cap (retry with a larger one).  order (NULL =
 * index order): processing order of the rows, any permutation in which a row follows its pivot rows.
 * ddilu_compact_cols: slab -> CSR columns; ddilu_prefill: factor.py:372-390 `_prefill`. */
long long ddilu_iluk_smem_bytes(int row_cap);
int ddilu_iluk_symbolic(int n, const int *a_rp, const int *a_ci, int n_elim, int klevel, int row_cap, int *p_cnt,
                        int *p_ci, int *k_cnt, int *k_ci, int *k_lv, int *done, int *status, const int *order,
                        void *stream);
int ddilu_compact_cols(int n, int cap, const int *cnt, const int *ci, const int *out_rp, int *out_ci, void *stream);
int ddilu_prefill(int n, const int *a_rp, const int *a_ci, const double *a_v, const int *rp, const int *ci, double *v,
                  int n_elim, int upper_part, void *stream);

/* ---- tiled triangular solve (csrc/tiled.cu): sparse.py:228-272 again, for factors whose
 * rows cluster into tiles (<= 1024 rows) with an ACYCLIC tile dependency graph.  A CTA
 * walks a tile's levels with the tile's x in shared memory; boundary dependencies go
 * through L2.  Setup passes (all device pointers unless *_h):
 *   tile_box_keys : key of row i = box of grid node nodes[i] (x fastest, like ordering.py:171-190),
 *                   + owner[node] * n_boxes when owner != NULL; *n_keys_h = boxes per owner
 *   tile_heads / tile_assign : from (key, row) pairs sorted by key: compact tile ids,
 *                   tile_of[row], tpos[row] (position in the sorted list), tile_ptr[n_tiles+1]
 *   tile_edges_*  : (producer tile, consumer tile) pairs of the cross-tile dependencies
 *   tile_relax    : `passes` sweeps of tlev[c] = max(tlev[c], tlev[p]+1); flags[0] = last sweep
 *                   changed something, flags[1] = cycle (a level reached n_tiles)
 *   tile_build    : item_warps = 4 (rotating-warp kernel), 1 (warp-per-tile kernel) or 0 (lean records, rows with <= 3 dependencies); fill = 0: size of every tile's static block (16-byte units) -> blk16[q],
 *                   stats[0..2] = max rows, max externals, max bytes, stats[4] = longest row (kmax); fill = 1: blk16 holds the
 *                   scanned offsets, blocks are written to blob, stats[3] = first bad pivot row
 *   sptrsv_tiled  : x = T^-1 b; one cooperative launch */
int ddilu_tile_box_keys(int n, const int *nodes, int nd, const int *dims_h, const int *tdims_h, const int *owner,
                        int *keys, long long *n_keys_h, void *stream);
int ddilu_tile_heads(int n, const int *sorted_keys, int *flags, void *stream);
int ddilu_tile_assign(int n, const int *sorted_keys, const int *head_scan, const int *sorted_rows, int *tile_of,
                      int *tpos, int *tile_ptr, void *stream);
int ddilu_tile_edges_count(int n, const int *row_ptr, const int *col_idx, int upper, const int *tile_of, int *cnt,
                           void *stream);
int ddilu_tile_edges_fill(int n, const int *row_ptr, const int *col_idx, int upper, const int *tile_of,
                          const int *off, int *edges, void *stream);
int ddilu_tile_relax(long long n_edges, const int *edges, int n_tiles, int *tlev, int *flags, int passes,
                     void *stream);
int ddilu_tile_build(int fill, int n_tiles, const int *tsched, const int *tile_ptr, const int *trows,
                     const int *tile_of, const int *tpos, const int *row_ptr, const int *col_idx,
                     const double *values, const int *glev, int upper, int has_diag, int item_warps, int *blk16,
                     int *stats, unsigned char *blob, void *stream);
long long ddilu_tiled_smem_bytes(int stat_max, int tmax, int emax);
/* self-check of the division the U solves use (pivot reciprocal + two FMA corrections) against the
 * IEEE division on n pseudo-random / adversarial operand pairs; *mismatch = pairs whose bits differ */
int ddilu_fastdiv_selftest(long long n_samples, unsigned long long seed, unsigned long long *mismatch, void *stream);
int ddilu_sptrsv_tiled(int n, int n_tiles, const int *blk_off16, const unsigned char *blob, int stat_max, int tmax,
                       int emax, int kmax, int has_diag, const double *b, double *x, void *stream);

/* ---- block sweep (csrc/sweep.cu): L^-1, U^-1 or U^-1 L^-1 on a block-diagonal factor pair with narrow levels --
 * the interface factors L_S / U_S, one diagonal block per subdomain (precond.py:239-249 `_schur_solve` inside
 * `reduced_matvec`, precond.py:361-366 `_coarse_precond`; arithmetic of sparse.py:228-272, bit-exact).  One CTA
 * per block, the block's x in a shared-memory window, the rows' operands streamed as 256-row pages in schedule
 * order through a TMA ring, L and U back to back in one launch.
 * ddilu_sweep_fill: operands of a factor into its pages (k = operand slots per row: 2, 3, 4, 8, or 16 / 24 for long rows, gpos / lpos = global padded /
 * block-local schedule position of every row, gpos_u = position of the row in the U schedule (lower factor only),
 * window = shared-memory window in doubles, a power of two).
 * ddilu_sweep_rhs: right-hand side in schedule order, out[i] = base[row] (row_ptr NULL), (A y)[row] (mode 0),
 * base[row] - (A y)[row] (mode 1: `r_ext - W fp`, precond.py:242-243) or base + A y (mode 2), row = rowof[i],
 * 0 where rowof[i] < 0 (page padding); with add_out also add_out[i] = add[rowof_u[i]], the vector the U phase
 * adds to its results, in U schedule order.
 * ddilu_sweep_solve: phases 1 = L, 2 = U, 3 = L then U; blocks = 8 ints per block {rows, first page, L levels,
 * U levels, offset into levtab, 0, 0, 0}; stages = ring depth (power of two), sets x nct compute threads that own
 * rows_per_thread (1, 2) rows of a level each; out[row] = x (+ add[U position of the row]: `y + S^-1 E y`,
 * precond.py:249). */
int ddilu_sweep_page_rows(int k);         /* rows per operand page: 256, or 64 for long rows (k > 8) */
int ddilu_sweep_helper_threads(void);   /* threads of a CTA that do not compute (TMA issuer, gate, writers) */
long long ddilu_sweep_page_bytes(int k, int upper);
long long ddilu_sweep_smem_bytes(int k, int stages, int window, int max_lev);
int ddilu_sweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                     const int *gpos, const int *lpos, const int *gpos_u, int window, unsigned char *pages,
                     int *bad_row, void *stream);
int ddilu_sweep_rhs(int npad, const int *rowof, const int *row_ptr, const int *col_idx, const double *values,
                    const double *y, const double *base, int mode, double *out, const int *rowof_u, const double *add,
                    double *add_out, void *stream);
int ddilu_sweep_solve(int n_blocks, const int *blocks, const int *levtab, const unsigned char *pages_l,
                      const unsigned char *pages_u, int k, int window, int stages, int sets, int nct,
                      int rows_per_thread, int max_lev, int phases, const double *rhs, double *tmp, double *out,
                      const double *add, void *stream);

/* ---- cluster sweep (csrc/csweep.cu): L^-1 or U^-1 on a block-diagonal factor with LARGE deep blocks -- the interior
 * factors L_B / U_B, one diagonal block per subdomain (precond.py:236-238, 244-246 `_interior_solve`; arithmetic of
 * sparse.py:228-272, bit-exact).  A thread-block cluster of cluster_size (<= 16) CTAs per block: every level is cut
 * into chunks, one per CTA; a CTA keeps the values it needs (own results and halo values of other CTAs) in a
 * shared-memory window; a producer pushes a result into the windows of the other CTAs that need it through
 * distributed shared memory (st.async completing bytes on the consumer's mbarrier); one mbarrier wait per level.
 * ddilu_csweep_fill: operands of a factor in CTA-local schedule order (k = operand slots per row: 3, 4 or 20;
 * gpos = position of the row in the operand arrays, dep_slot = per stored entry the window slot of that dependency
 * in the READER's CTA; np = length of the position space; coef[k][np]; code[code_words(k)][np]: the 16-bit halves
 * of a row's words are its k dependency slots (filled here) and then its max_push(k) push targets
 * slot << rank_bits(k) | rank, 0xffff = none (filled by the caller); rowid[np]; piv[np][2] = (pivot, reciprocal) pairs (upper only)).
 * ddilu_csweep_solve: ctas = 4 ints per CTA {first position, rows, first step, steps}; steps = 8 ints per step
 * {start (a multiple of 4), end (positions, at most `threads` rows), window slot of the first row, first row when
 * the rows are consecutive else -1 (rowid is read), halo bytes arriving for the level (first step of a level),
 * flags 1 = first | 2 = last step of its level, 0, 0}; depth = stages of the operand ring (2..4). */
int ddilu_csweep_threads(int k);      /* k selects the kernel shape: 3, 4 = short rows, 20 = long rows (27-point / ILUT) */
int ddilu_csweep_window(int k);
int ddilu_csweep_max_push(int k);
int ddilu_csweep_rank_bits(int k);    /* a push target is slot << rank_bits | rank: clusters of <= 1 << rank_bits CTAs */
int ddilu_csweep_code_words(int k);
long long ddilu_csweep_smem_bytes(int k, int upper, int depth, int max_steps);
int ddilu_csweep_active_clusters(int cluster_size, int k, int depth, int max_steps);
int ddilu_csweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                      const int *gpos, const int *dep_slot, long long np, double *coef, unsigned *code, int *rowid,
                      double *piv, int *bad_row, void *stream);
/* long rows (k = 20): the operands lie STEP BY STEP in one blob -- per step a block coef[k][r4] | piv[2][r4] (upper) |
 * words[code_words][r4] | row ids[r4] with r4 = rows of the step rounded up to 4, so that the feeder moves a step
 * with one bulk copy; steps[..][6] = byte offset of the block / 16.  ddilu_csweep_fill_long writes a row's operands
 * (blk_base / r4 / off: byte offset of its step's block, r4 of that step, its entry), push targets start as 0xffff. */
int ddilu_csweep_long_record_bytes(int k, int upper);
int ddilu_csweep_fill_long(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                           const long long *blk_base, const int *r4, const int *off, const int *dep_slot,
                           unsigned char *blob, int *bad_row, void *stream);
int ddilu_csweep_solve(int n_blocks, int cluster_size, const int *ctas, const int *steps, const double *coef,
                       const unsigned *code, const int *rowid, const double *piv, const unsigned char *blob,
                       long long np, int k, int upper, int max_steps, int depth, const double *b, double *out,
                       void *stream);

/* ---- peer-memory exchanges (csrc/peer.cu) for the multi-GPU path, SURVEY.md 8e / PAPER.md:701-705: the halo of
 * interface values and the sum of dot / norm scalars without a collective library call.  Every rank owns a mailbox
 * (flags, reduction slots red[2][size][kmax], halo buffers data[2][size][cap]) that all ranks of the node map through
 * CUDA IPC; the tables `slots` / `data` / `flags` / `acks` hold, per rank, the address of that rank's region in THIS
 * process.  seq = 1, 2, ... per exchange kind; waits are bounded by spin_cycles (*err != 0: a peer never arrived).
 * ddilu_peer_allreduce: out[i] = sum over ranks, in rank order, of partial_r[i] (i < k <= kmax); one launch.
 * ddilu_peer_send: message values off[d] .. off[d+1] (value j = send[j], or send[idx[j]]: the pack of the interface
 * values fused into the send) into rank d's data[seq & 1][rank][..], then its halo flag [rank] = seq (after rank d
 * acknowledged seq - 2: `ack` = my acknowledgement flags).
 * ddilu_peer_recv: recv[off[s] .. off[s+1]) from my data[seq & 1][s][..] once my halo flag [s] >= seq (the own part
 * from self_send + self_off), then rank s's acknowledgement flag [rank] = seq. */
int ddilu_peer_allreduce(int k, int kmax, const double *partial, double *out, const unsigned long long *slots,
                         const unsigned long long *flags, int rank, int size, long long seq, long long spin_cycles,
                         int *err, void *stream);
int ddilu_peer_send(int size, int rank, int total, const double *send, const int *idx, const int *off,
                    const unsigned long long *data,
                    const unsigned long long *flags, const long long *ack, long long cap, long long seq,
                    long long spin_cycles, unsigned int *counter, int *err, void *stream);
int ddilu_peer_recv(int size, int rank, int total, double *recv, const int *off, const double *mydata,
                    const long long *myflags, const unsigned long long *acks, const double *self_send,
                    const int *self_idx, int self_off, long long cap, long long seq, long long spin_cycles,
                    unsigned int *counter, int *err, void *stream);

/* ---- factor.py:198-216 `_split_counts` + :435-443 `_row_inf_norms` */
int ddilu_split_count(int n, const int *a_rp, const int *a_ci, const double *a_v, int n_elim, int *pc, int *kc,
                      double *rownorm, void *stream);
/* ---- factor.py:219-246 `_split_fill` */
int ddilu_split_fill(int n, const int *a_rp, const int *a_ci, const double *a_v, int n_elim, const int *p_rp,
                     int *p_ci, double *p_v, const int *k_rp, int *k_ci, double *k_v, void *stream);
/* ---- factor.py:397-432 `_factor_split`: ILU(0) / MILU(0) / partial ILU(0) on the
 * split pattern, rows visited in the level order `order` of the pivot pattern. */
int ddilu_ilu0_numeric(int n, int n_slots, const int *order, const int *p_rp, const int *p_ci, double *p_v,
                       const int *k_rp, const int *k_ci, double *k_v, int n_elim, int milu, const double *target,
                       const double *wvec, double delta, const double *rownorm, int *done, void *stream);
/* ---- factor.py:482-656 `_ilut_factor` + :465-479 `_select_largest`.  Rows are
 * written to fixed-capacity slabs: caps_h = {lcap, ucap, scap} from ddilu_ilut_caps;
 * L row i at i*lcap; U row i at i*ucap (i < n_elim, diagonal first) or
 * n_elim*ucap + (i-n_elim)*scap (Schur rows).  *status != 0: row_cap too small.
 * order (NULL = index order): processing order of the rows, any permutation in which a row comes after its pivot
 * rows -- callers interleave independent diagonal blocks so that all of them advance at once. */
long long ddilu_ilut_smem_bytes(int row_cap);
int ddilu_ilut_caps(int maxfill, int row_cap, int *caps_h);
int ddilu_ilut_factor(int n, const int *a_rp, const int *a_ci, const double *a_v, int n_elim, double tau, int maxfill,
                      double tau_s, double delta, int row_cap, int *l_cnt, int *l_ci, double *l_v, int *u_cnt,
                      int *u_ci, double *u_v, int *done, int *status, const int *order, void *stream);
/* slab rows (cap_a for rows < n_split, cap_b after) -> CSR with the given row_ptr */
int ddilu_compact_rows(int n, int n_split, int cap_a, int cap_b, const int *cnt, const int *ci, const double *v,
                       const int *out_rp, int *out_ci, double *out_v, void *stream);

/* ---- factor.py:756-803 `_col_split_*` / sparse.py:456-471 `extract_block` on
 * contiguous index ranges: rows [r0,r1) x cols [c0,c1), columns shifted by -c0 */
int ddilu_csr_block_count(const int *rp, const int *ci, int r0, int r1, int c0, int c1, int *counts, void *stream);
int ddilu_csr_block_fill(const int *rp, const int *ci, const double *v, int r0, int r1, int c0, int c1,
                         const int *out_rp, int *out_ci, double *out_v, void *stream);

/* ---- Krylov vector kernels: sparse.py:275-280 `_vdot`, :526-528 `vnorm2`,
 * krylov.py:74-77 `_axpy`, and the numpy expressions of krylov.py:122,156,160-167 */
long long ddilu_reduce_ws_bytes(void);
int ddilu_dot(long long n, const double *x, const double *y, double *out, void *ws, void *stream);
int ddilu_dot_dir(long long n, const double *x, const double *y, double *out, void *ws, int reverse, void *stream);
/* w += (alpha_dev ? alpha_host * *alpha_dev : alpha_host) * v; if u: *out = dot(u, w) */
int ddilu_axpy_dot(long long n, const double *alpha_dev, double alpha_host, const double *v, double *w,
                   const double *u, double *out, void *ws, void *stream);
/* the same walking the vectors from the end when reverse != 0: consecutive MGS steps alternate the direction
 * so that a step starts with the part of w and of the shared basis vector that is still in L2 */
int ddilu_axpy_dot_dir(long long n, const double *alpha_dev, double alpha_host, const double *v, double *w,
                       const double *u, double *out, void *ws, int reverse, void *stream);
/* Blocked modified Gram-Schmidt (krylov.py:131-136, the loop `h[i,j] = vdot(V[i], w); w -= h[i,j] V[i]`): one pass
 * (a) subtracts the previous block, w -= sum_{l<kp} h_l vprev[l*ld + :], with h solved from the raw sums of the
 * previous pass (raw_prev = [d_0..d_{kp-1}, G_10, G_20, G_21, ...]: h_i = d_i - sum_{l<i} h_l G_il) and stored to
 * hout[0..kp), and (b) writes the raw sums of vnext[0..kn) against the updated w to out; kn == 0: out[0] = <w, w>.
 * kp, kn <= ddilu_mgs_max_block().  Same values as the vector-by-vector loop up to the rounding of the dots. */
long long ddilu_mgs_ws_bytes(void);
int ddilu_mgs_max_block(void);
int ddilu_mgs_block(long long n, long long ld, int kp, const double *vprev, const double *raw_prev, double *hout,
                    double *w, int kn, const double *vnext, double *out, void *ws, int reverse, void *stream);
/* krylov.py:236-256, one Arnoldi step of `fixed_gmres` on a SHORT vector (the interface unknowns) in ONE cooperative
 * launch: w orthogonalised in place against v[0..k) (k <= ddilu_mgs_small_max(), leading dimension ld),
 * hout[0..k) = the MGS coefficients, hout[k] = <w, w>, vout = w / sqrt(<w, w>).  The phases are the three launches
 * it replaces -- ddilu_mgs_block(0, k), ddilu_mgs_block(k, 0), ddilu_scale -- with the same grid, loops and
 * reduction order (same bits), separated by grid barriers; falls back to those launches when the grid cannot be
 * resident at once.  raw: scratch of k + k(k-1)/2 doubles (fallback only); ws as for ddilu_mgs_block. */
int ddilu_mgs_small_max(void);
int ddilu_mgs_small_step(long long n, long long ld, int k, const double *v, double *w, double *hout, double *vout,
                         double *raw, void *ws, int reverse_dots, int reverse_update, void *stream);
/* krylov.py:226-232, the start of `fixed_gmres` on one rank: *out = <x, x>, y = x / sqrt(<x, x>) in ONE cooperative
 * launch (= ddilu_dot + ddilu_scale(take_sqrt), same bits; falls back to those when the grid cannot be resident at
 * once).  ws: workspace of ddilu_mgs_block, red_ws: workspace of ddilu_dot (fallback only). */
int ddilu_norm_scale_small(long long n, const double *x, double *out, double *y, void *ws, void *red_ws, void *stream);
/* y = x / s (mode 0) or x * s (mode 1); s = *alpha_dev or alpha_host, sqrt'ed if take_sqrt */
int ddilu_scale(long long n, const double *x, const double *alpha_dev, double alpha_host, int take_sqrt, int mode,
                double *y, void *stream);
/* krylov.py:233-268: the host arithmetic of `fixed_gmres` (Givens rotations, back substitution) for an m-step
 * inner solve (m <= ddilu_gmres_small_max()) on the device: H row j = [h_0j .. h_jj, |w_j|^2] with stride ldh,
 * *bb = <b, b>; coef[0..m) = coefficients of the basis combination.  *flag is set to 1 when the reference
 * would have left its loop early (zero right-hand side, happy breakdown) or a number is not finite: the caller
 * then redoes the application on the host-read path. */
int ddilu_gmres_small_max(void);
int ddilu_gmres_small_solve(int m, const double *H, int ldh, const double *bb, double happy_tol, double *coef,
                            int *flag, void *stream);
/* x (+)= sum_i coef[i] * basis[i*ld + :] in increasing i */
/* L2 residency hint for the Arnoldi work vector (stream access-policy window, persisting L2); bytes = 0 clears */
int ddilu_l2_persist_window(const void *ptr, long long bytes, void *stream);
int ddilu_multi_axpy(long long n, int k, const double *basis, long long ld, const double *coef, double *x,
                     int overwrite, void *stream);
/* z = a + b (0), a - b (1), -a (2) */
int ddilu_ewise(long long n, const double *a, const double *b, int op, double *z, void *stream);
/* dst[i] = src[idx[i]] / dst[idx[i]] = src[i]  (precond.py:190, 369, 384 fancy indexing) */
int ddilu_gather(long long n, const int *idx, const double *src, double *dst, void *stream);
int ddilu_scatter(long long n, const int *idx, const double *src, double *dst, void *stream);

/* ---- ordering.py:88-94 `_mark_exterior` on the symmetrised pattern (:32-81) */
int ddilu_mark_exterior(int n, const int *rp, const int *ci, const int *owner, int *exterior, void *stream);
/* keys = exterior * p + owner, vals = iota: sorting them gives DomainLayout.global_perm (ordering.py:273-293) */
int ddilu_layout_keys(int n, const int *owner, const int *exterior, int p, int *keys, int *vals, void *stream);
int ddilu_lower_bounds(const int *sorted, int n, int nkeys, int *out, void *stream);
/* ordering.py:171-187: structured box partition */
int ddilu_box_owner(int n, int nd, const int *dims_h, const int *factors_h, int *owner, void *stream);

/* ---- sparse.py:303-330 `_gather_rows_count/_fill` (take_submatrix / extract_block),
 * precond.py:154-170 `_keep_cross_block` folded in as a filter:
 * filter & 3: 0 all, 1 same-domain entries only, 2 cross-domain only; filter & 4: drop diagonal */
int ddilu_build_map(int n_nodes, const int *nodes, int offset, int *map, void *stream);
int ddilu_gather_rows_count(int n_sel, const int *rows, const int *rp, const int *ci, const int *colmap,
                            const int *dom, int filter, int *counts, void *stream);
int ddilu_gather_rows_fill(int n_sel, const int *rows, const int *rp, const int *ci, const double *v,
                           const int *colmap, const int *dom, int filter, const int *out_rp, int *out_ci,
                           double *out_v, int resort, void *stream);

/* ---- halo planning for the one-subdomain-block-per-GPU mapping (no reference
 * equivalent: the reference loops over domains in one process, precond.py:189-190).
 * flags[j] = 1 for every column of the selected rows with colmap[j] < 0;
 * flags[rank * n_ext + extmap[j]] = 1 when a row of another rank touches my exterior j. */
int ddilu_mark_foreign_cols(int n_sel, const int *rows, const int *rp, const int *ci, const int *colmap, int *flags,
                            void *stream);
int ddilu_mark_sends(int n, const int *rp, const int *ci, const int *owner, int doms_per_rank, int my_rank,
                     const int *extmap, int n_ext, int *flags, void *stream);

/* ---- ordering.py:32-81 `_sym_adjacency` (neighbour sets; order inside a row is unspecified) */
int ddilu_sym_adj_count(int n, const int *rp, const int *ci, int *counts, void *stream);
int ddilu_sym_adj_fill(int n, const int *rp, const int *ci, const int *out_rp, int *cursor, int *out_ci, void *stream);
int ddilu_row_lengths(int n, const int *rp, int *out, void *stream);

int ddilu_sort_rows_i32(int n, const int *rp, int *ci, void *stream);
/* ---- ordering.py:97-127 `_grow_regions` (serial greedy BFS growth; work = 2n ints) */
int ddilu_grow_regions(int n, const int *adj_rp, const int *adj_ci, int n_dom, const int *sizes, int *owner,
                       int *work, void *stream);
/* ---- sparse.py:333-370, 487-505 `sparse_matmul`: C = A B with the exact structural pattern (cancelled entries
 * kept), values bit-identical to the reference's marker/accumulator loop.  bound[i] = products of row i (scan it
 * into off[n_rows + 1]); expand writes the products of a row, stably sorted by column, into s_col / s_val at
 * off[i] and the number of distinct columns into counts[i] (scan it into out_rp); compact sums the runs. */
int ddilu_spgemm_bound(int n_rows, const int *a_rp, const int *a_ci, const int *b_rp, int *bound, void *stream);
int ddilu_spgemm_expand(int n_rows, const int *a_rp, const int *a_ci, const double *a_v, const int *b_rp,
                        const int *b_ci, const double *b_v, const int *off, int *s_col, double *s_val, int *counts,
                        void *stream);
int ddilu_spgemm_compact(int n_rows, const int *off, const int *s_col, const double *s_val, const int *out_rp,
                         int *out_ci, double *out_v, void *stream);
/* ---- precond.py:84-125 `_l1_row_shifts`, `_add_to_diagonal` (l1 block Jacobi) */
int ddilu_l1_row_shifts(int n_sel, const int *rows, const int *rp, const int *ci, const double *v, const int *owner,
                        double *out, void *stream);
int ddilu_add_to_diagonal(int n, const int *rp, const int *ci, double *v, const double *shifts, int *missing,
                          void *stream);
/* ---- factor.py:806-822 `_drop_small_rows` (schur_drop_tol thinning) */
int ddilu_drop_small_count(int n, const int *rp, const int *ci, const double *v, double tol, int *counts,
                           void *stream);
int ddilu_drop_small_fill(int n, const int *rp, const int *ci, const double *v, double tol, const int *out_rp,
                          int *out_ci, double *out_v, void *stream);

/* ---- ordering.py:304-397 `_bfs_ecc` + `_rcm_order`: Cuthill-McKee order (not reversed) */
long long ddilu_cm_work_elems(int n);
int ddilu_cm_order(int n, const int *adj_rp, const int *adj_ci, int *order, int *work, void *stream);
/* the same when the node ranges [seg_ptr[s], seg_ptr[s+1]) (device array, n_seg + 1 entries) are mutually
 * disconnected (one per subdomain, precond.py:141-144 calls rcm once per domain): disjoint CTA groups order
 * the ranges concurrently; identical output */
int ddilu_cm_order_segments(int n, const int *adj_rp, const int *adj_ci, int n_seg, const int *seg_ptr, int *order,
                            int *work, void *stream);
/* ordering.py:416 reversal, per domain segment */
int ddilu_reverse_segments(int n, const int *cm, int n_seg, const int *seg_ptr, int *out, void *stream);

/* ---- int64 <-> int32 index conversion at the API boundary (sparse.py:95-96 uses int64) */
int ddilu_narrow_i64(long long n, const long long *in, int *out, void *stream);
int ddilu_widen_i32(long long n, const int *in, long long *out, void *stream);

#ifdef __cplusplus
}
#endif

/* Measured-slower alternative kernels, tuning knobs and diagnostics are NOT part of the product ABI: they are
 * compiled only with -DDDILU_EXPERIMENTS (DDILU_EXPERIMENTS=1 python -m paper_2303_08881_b200.build) and declared
 * in ddilu_b200_experiments.h. */
#ifdef DDILU_EXPERIMENTS
#include "ddilu_b200_experiments.h"
#endif
#endif /* DDILU_B200_H */
