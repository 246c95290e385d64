/*
 * ddilu_b200_experiments.h -- entries of libddilu_b200.so that exist only in a -DDDILU_EXPERIMENTS build
 * (DDILU_EXPERIMENTS=1 python -m paper_2303_08881_b200.build): alternative triangular-solve kernels that were
 * measured slower than the production ones and are kept as recorded negative results, tuning
 * knobs and cycle-counter diagnostics of the probe scripts under scripts/.  None of them is on the product
 * path; the product ABI is include/ddilu_b200.h.  Same conventions as there (device pointers, int status,
 * stream last).
 */
#ifndef DDILU_B200_EXPERIMENTS_H
#define DDILU_B200_EXPERIMENTS_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- tuning knobs (no reference equivalent): "trsv_blocks_per_sm", "trsv_depth",
 * "trsv_stage_mask", "trsv_far_sleep_ns", "trsv_pipe", "trsv_pipe_warps_per_sm", "trsv_sleep_ns" */
int ddilu_set_tuning(const char *key, int value);

/* Block-local variant for small, deep, block-diagonal factors (interface factors L_S/U_S:
 * precond.py:239-245 `_schur_solve`, :361-366 `_coarse_precond`): one CTA per independent row
 * block seg_ptr[d]..seg_ptr[d+1], levels separated by a CTA barrier.  start/cnt[d*n_levels+l]
 * = first position / number of rows of block d in level l inside level_rows. */
int ddilu_blocklocal_table(int n, int n_blocks, const int *seg_ptr, int n_levels, const int *lev,
                           const int *level_rows, int *start, int *cnt, void *stream);
int ddilu_sptrsv_blocklocal(int n_blocks, int n_levels, const int *start, const int *cnt, const int *level_rows,
                            const int *row_ptr, const int *col_idx, const double *values, const double *b, double *x,
                            int upper, int unit_diag, int *err, void *stream);

/* same sweep on the SELL arrays; sstart[d*n_levels+l] = first SCHEDULE SLOT of block d in level l */
/* the same sweep with the block's part of x in a shared-memory window: scol_loc = block-local schedule position
 * of every dependency (-1 padding), lbase = first position of (block, level), wmask + 1 = window size (a power
 * of two, checked at setup against the furthest dependency), sdinv = RN(1/pivot) or 0 (see ddilu_fastdiv_selftest) */
int ddilu_sptrsv_blockwin_sell(int n_blocks, int n_levels, const int *sstart, const int *cnt, const int *lbase,
                               const int *order, const int *goff, int uniform_width, const int *scol_loc,
                               const double *sval,
                               const double *sdiag, const double *sdinv, int wmask, const double *b, double *x,
                               void *stream);
int ddilu_sptrsv_blocklocal_sell(int n_blocks, int n_levels, const int *sstart, const int *cnt, const int *order,
                                 const int *goff, int uniform_width, const int *scol, const double *sval,
                                 const double *sdiag, const double *b, double *x, void *stream);

/* diagnostics: same solve with per-group timestamps (8 int64 per group: start, spin done, deps
 * loaded, stored [globaltimer ns], SM id, spin count, re-poll rounds, warp id) */
int ddilu_sptrsv_sell_trace(int n, int n_slots, int blocks_per_sm, const int *order, const int *goff,
                            int uniform_width, const int *scol, const double *sval, const double *sdiag,
                            const int *gwait, const double *b, double *x, long long *stamps, void *stream);

int ddilu_tiled_set_tuning(const char *key, int value);
/* diagnostics: 8 int64 per CTA (life, wait static/rhs, wait boundary, tile time [cycles], levels, tiles); NULL = off */
int ddilu_tiled_set_debug(long long *device_buf);

/* "wavefront slab" tiles: key = (owner, box of the first two grid coordinates, lev[i] / delta) with lev =
 * the factor's level of row i; *n_keys_h = size of the key range */
int ddilu_tile_slab_keys(int n, const int *nodes, int nd, const int *dims_h, const int *tdims_h, const int *lev,
                         int n_levels, int delta, const int *owner, int n_owners, int *keys, long long *n_keys_h,
                         void *stream);

/* warp-per-tile variant of the same solve (static blocks built with item_warps = 1): every warp owns a
 * stream of tiles, no named barriers, no helper warps; as many independent warps per SM as shared
 * memory allows */
long long ddilu_warptile_smem_per_warp(int stat_max, int tmax, int emax);
/* lean variant for rows with <= 3 dependencies (static blocks built with item_warps = 0: pre-digested
 * 16-byte row records, ~40 instructions per level) */
int ddilu_sptrsv_lean(int n, int n_tiles, const int *blk_off16, const unsigned char *blob, int stat_max, int tmax,
                      int emax, int kmax, int has_diag, const double *b, double *x, void *stream);
int ddilu_sptrsv_warptile(int n, int n_tiles, const int *blk_off16, const unsigned char *blob, int stat_max, int tmax,
                          int emax, int kmax, int has_diag, const double *b, double *x, void *stream);

int ddilu_sweep_set_tuning(int writer_sleep_ns, int flags);   /* diagnostics */
int ddilu_sweep_set_debug(long long *buf);   /* diagnostics: 64 int64 cycle counters per block, NULL = off */
int ddilu_csweep_set_debug(long long *buf);  /* cluster sweep: 16 int64 cycle counters per CTA and probe thread (first, last), NULL = off */

/* ---- lattice triangular solve (csrc/experiments/lattice.cu): the fast path of sparse.py:228-272 for factors whose box
 * tiles are lattices with one-way axes and <= 3 dependencies per row (7-point ILU(0) factors).  One warp per
 * tile, results of a step handed to the next through the warp's shared-memory line buffer, row records streamed
 * through a per-warp cp.async ring, per-tile completion flags instead of a sentinel preset of x.
 * ddilu_lattice_build: fill = 0 checks the lattice property and sizes the blocks (blk16[q] in 16-byte units,
 * stats = {failed, max boundary values, max steps, first bad pivot row, max producer tiles, max block bytes,
 * max rows}); fill = 1 writes
 * the per-tile table `tab` (32 int4 per tile) and the blocks at blob + 16 * blk16[q] (scanned offsets).
 * nodes[row] = grid node of a row, dims3 / tdims3 = grid and tile dimensions (x fastest, padded with 1). */
int ddilu_lattice_build(int fill, int n_tiles, const int *tsched, const int *tile_pos, const int *tile_ptr,
                        const int *trows, const int *tile_of, const int *row_ptr, const int *col_idx,
                        const double *values, const int *nodes, const int *dims3, const int *tdims3, int upper,
                        int has_diag, void *tab, int *blk16, int *stats, unsigned char *blob, void *stream);
int ddilu_lattice_max_ext(void);
int ddilu_lattice_set_tuning(const char *key, int value);
long long ddilu_lattice_smem_bytes(int blkmax, int tmax, int xemax);
int ddilu_lattice_set_debug(long long *buf);
int ddilu_sptrsv_lattice(int n_tiles, const void *tab, const unsigned char *blob, int *flags, int n_slots,
                         int has_diag, int blkmax, int tmax, int xemax, const double *b, double *x, void *stream);

/* ---- tile sweep (csrc/experiments/tsweep.cu; measured, not adopted: DESIGN.md 5.7): sparse.py:228-272 for the INTERIOR factors of a structured problem, with
 * right-hand side and solution kept in TILE ORDER (tiles one after the other, padded to whole 256-row pages with
 * zeros, rows of a tile in level-major order of the L factor; the U factor walks the reverse order).  Pages of
 * operands and vector slices arrive by TMA, results leave by bulk stores, boundary values of neighbour tiles are
 * gathered one tile ahead; persistent CTAs of a cooperative launch take the tiles in a topological order.
 * ddilu_tsweep_fill: operands into pages (gpos / lpos = padded global / tile-local position of every row in the
 * factor's own position space, ecode[k] = boundary slot of entry k or -1).  ddilu_tsweep_permute: a vector
 * between row order and tile order.  ddilu_tsweep_solve: tiles = 16 ints per tile in schedule order {rows, first
 * page, levels, offset into levtab, boundary values, offset into extpos, producer tiles, offset into prods, pad
 * rows in front (U), 0 ...}; flags = one int per tile (scratch). */
long long ddilu_tsweep_page_bytes(int k, int upper);
long long ddilu_tsweep_smem_bytes(int k, int upper, int stages, int window, int xe_cap, int max_lev);
int ddilu_tsweep_fill(int n, const int *row_ptr, const int *col_idx, const double *values, int upper, int k,
                      const int *gpos, const int *lpos, const int *ecode, int window, unsigned char *pages,
                      int *bad_row, void *stream);
int ddilu_tsweep_permute(int n, const int *pos, const double *in, double *out, int to_tile, void *stream);
int ddilu_tsweep_solve(int n_tiles, const int *tiles, const int *levtab, const int *extpos, const int *prods,
                       const unsigned char *pages, int *flags, int k, int upper, int window, int xe_cap, int max_lev,
                       int stages, int sets, int nct, const double *b, double *x, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DDILU_B200_EXPERIMENTS_H */
