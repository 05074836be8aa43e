/*
 * hyperball_b200.h -- C-ABI of the B200 HyperBall hot path (libhyperball_b200.so).
 *
 * Plain pointers and sizes only; every pointer argument documented as "device" must be
 * a CUDA device pointer (the host side allocates with torch, the library allocates
 * nothing).  `stream` is a cudaStream_t passed as void*.  Every entry point returns 0
 * on success and a nonzero code otherwise; hb_last_error() describes the last failure
 * of the calling thread.  All launches are asynchronous on `stream`.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/hyperball):
 *
 *   hb_seed           engine.py:153-162 _ProbabilisticBackend.seed
 *                     (-> hll.py:79-88 hash_items, hll.py:147-158 register_values,
 *                         _kernels.py:43-51 scatter_max, _kernels.py:37-40
 *                         estimate_register_rows)
 *   hb_estimate_rows  _kernels.py:37-40 estimate_register_rows (+ 15-34 per row)
 *   hb_union_step     engine.py:164-169 _ProbabilisticBackend.union_range
 *                     (-> _kernels.py:67-114 hll_union_range) fused with
 *                     centrality.py:132-150 CentralityAccumulator.on_step/accumulate
 *   hb_finalize       centrality.py:153-171 finalize_closeness / finalize_harmonic /
 *                     finalize_lin (on the device-resident sums)
 *   hb_gather_changed / hb_scatter_rows / hb_refresh_rows
 *                     multi-GPU exchange of changed counter rows (no reference
 *                     counterpart: the reference shares `cur` between threads,
 *                     engine.py:377-390)
 *   hb_sample_flagged_arcs
 *                     share of arcs with a changed source, sampled (picks the dense
 *                     step; no reference counterpart)
 *   hb_relabel_csr / hb_relabel_csr_rows / hb_relabel_csr_src_rows
 *                     graph.py:145-155 transpose's output consumed in schedule order
 *                     (internal relabelling; no reference counterpart)
 *   hb_sort_rows      graph.py:52-80 keeps successor lists sorted; this restores that
 *                     order after the internal relabelling
 *   hb_gen_rmat_keys / hb_gen_degrees / hb_gen_blocks / hb_gen_arc_keys / hb_keys_to_csr
 *                     graph.py:52-80 (from_edges: sort, dedup, CSR) + 145-155 (transpose),
 *                     for the synthetic configs, on the device
 *   hb_transpose_csr  graph.py:145-155 transpose, on the device
 *   hb_pack_registers / hb_unpack_registers
 *                     hll.py:145-177 (CounterArray packing, to_blob / from_blob body),
 *                     for counters(), save() and load_state() (engine.py:254-327)
 *   hb_union_step_runs
 *                     cli.py:222-254 repeated runs (engine.run per seed), batched: R runs
 *                     in one union pass
 *   hb_exact_seed / hb_exact_union_step
 *                     engine.py:194-206 _ExactBackend.seed / union_range
 *                     (-> _kernels.py:117-172 bitset_union_range, weighted_popcount_row)
 *   hb_forward_csr / hb_mark_active / hb_mark_pull / hb_mark_pull_filtered
 *                     frontier of a sparse iteration (no reference counterpart: the
 *                     reference scans every node's successor list, _kernels.py:82-87)
 *   hb_hash_items     hll.py:79-88 hash_items (device twin, used by tests)
 *
 * Layout:
 *   regs / cur / nxt   uint8  [n, p] row-major, p = 2^b, row stride p bytes
 *                      (the reference's dense working registers, engine.py:147-148)
 *   offsets            int64  [n+1]   CSR of the transpose graph, internal ids
 *   succ               int32  [m]     in-neighbour ids (internal ids)
 *   chg_prev, chg_now  uint32 [ceil(n/32)] change bitmaps, bit (v & 31) of word v >> 5
 *   est                fp64   [n]     cached estimates, updated in place
 *   sum_dist,sum_recip fp64   [n]     CentralityAccumulator sums (either may be NULL)
 *   lc_table           fp64   [p+1]   lc_table[V] = p * log(p / V) built on the host with
 *                                     math.log (bit-identical to numba's np.log)
 */
#ifndef HYPERBALL_B200_H
#define HYPERBALL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Library version string and the last error message of the calling thread. */
const char *hb_version(void);
const char *hb_last_error(void);

/* Minimum / maximum supported log2m (b).  The reference accepts any b >= 4
 * (hll.py:117-122); this build instantiates kernels for HB_MIN_LOG2M..HB_MAX_LOG2M. */
int hb_min_log2m(void);
int hb_max_log2m(void);

/* Seed one counter per node (engine.py:153-162).  regs: device uint8 [n, 2^b] (fully
 * overwritten); est: device fp64 [n].  perm: device int32 [n] mapping internal id ->
 * original node id (the id that is hashed), or NULL for the identity.  weights: device
 * int64 [n] indexed by ORIGINAL id, or NULL for one item (v, replica=1) per node
 * (engine.py:100-119).  seed is the CounterParams.seed reduced mod 2^64. */
int hb_seed(uint8_t *regs, double *est, int64_t n, int b, int register_width, uint64_t seed,
            const int32_t *perm, const int64_t *weights, const double *lc_table,
            double alpha_p2, double lc_cut, void *stream);

/* out[v] = estimate(regs[v]) for v in [lo, hi) (_kernels.py:15-40). */
int hb_estimate_rows(const uint8_t *regs, int64_t lo, int64_t hi, int b,
                     const double *lc_table, double alpha_p2, double lc_cut, double *out,
                     void *stream);

/* One ball-growth step over internal ids [lo, hi) (_kernels.py:67-114), fused with the
 * accumulator fold (centrality.py:132-150):
 *   nxt[v] = cur[v] max (max over succ w of v with chg_prev[w] (or every w when dense))
 *   chg_now[v] = nxt[v] != cur[v];  est[v] = estimate(nxt[v]) where changed;
 *   sum_dist[v] += t * max(new - old, 0);  sum_recip[v] += max(new - old, 0) / t.
 * nxt rows are written only when chg_prev[v] or chg_now[v] (the other rows of the
 * recycled buffer already hold the right value).
 * The schedule splits [lo, hi) into:
 *   light nodes: in-degree <= light_max_deg, one lane group per node, every id in
 *                [lo, hi) visited (heavier ids are skipped);
 *   heavy nodes: heavy_nodes[0..n_heavy) (device int32), each split into work items
 *                item_first[j]..item_first[j+1] (device int32 [n_heavy+1]); item i covers
 *                arcs [item_beg[i], min(item_beg[i] + item_arcs, offsets[v+1])) of node
 *                item_node[i] (device int32 / int64 [n_items]) and leaves a partial row
 *                in partial (device uint8 [n_items, p]).  finish_order (device int32
 *                [n_heavy]) is a permutation of 0..n_heavy-1 whose first n_mega entries are
 *                the heavy nodes with many items (merged one warp per node), the rest one
 *                lane group per node.
 * chg_now words covering [lo, hi) must be zero on entry (hb_union_step clears the whole
 * bitmap when clear_chg_now != 0).  *nch_out (device uint64) receives the changed count
 * (zeroed by the call); *merged_out (device uint64, may be NULL) receives the number of
 * arcs whose source row was actually merged (source-skip aware).  dense != 0 treats
 * every source as changed (first iteration and
 * skip_stable_nodes=False; results are identical).  hot_rows > 0 marks rows
 * [0, hot_rows) of cur as persisting in L2 for the duration of the call (degree order:
 * the most-read rows); 0 leaves the cache policy alone.  Discounted-gain sums
 * (centrality.py:26-101,149-150), at most 8: disc (device fp64 [n_disc, disc_stride])
 * gets disc[k][v] += (bit k of disc_div) ? delta / t : disc_scale[k] * delta for every
 * changed v (n_disc <= 8); disc_scale is a HOST array of the n_disc factors f_k(t) for this step.
 * active (device uint32 bitmap, may be NULL): frontier mode -- only nodes whose bit is set
 * are visited (hb_mark_active); NULL visits every node.  Fused push (multi-GPU, DESIGN.md
 * section 6): n_peers > 0 (at most 7) additionally stores every written nxt row into
 * peer_nxt[q] (device addresses of the peers' nxt replicas, same layout) and sets its
 * change bit in peer_chg[q]; peer_nxt / peer_chg are HOST arrays of those pointers.  The
 * caller must not clear chg_now (clear_chg_now = 0) while peers may be pushing, and must
 * barrier all ranks before reading what the peers pushed. */
int hb_union_step(int64_t n, int64_t lo, int64_t hi, const int64_t *offsets,
                  const int32_t *succ, const uint8_t *cur, uint8_t *nxt,
                  const uint32_t *chg_prev, uint32_t *chg_now, int clear_chg_now,
                  double *est, double *sum_dist, double *sum_recip, int64_t t,
                  const double *lc_table, double alpha_p2, double lc_cut, int b, int dense,
                  int64_t light_max_deg, const int32_t *heavy_nodes, const int32_t *item_first,
                  int64_t n_heavy, const int32_t *finish_order, int64_t n_mega,
                  const int32_t *item_node, const int64_t *item_beg,
                  int64_t n_items, int64_t item_arcs, uint8_t *partial, uint64_t *nch_out,
                  uint64_t *merged_out, int64_t hot_rows, double *disc, int64_t disc_stride,
                  int n_disc, const double *disc_scale, int disc_div, const uint32_t *active,
                  int n_peers, uint8_t *const *peer_nxt, uint32_t *const *peer_chg,
                  void *stream);

/* The same step with its arguments in one struct (the form to bind from a non-Python
 * host: fields are named, and later versions only append fields, so a caller built
 * against this header keeps working -- struct_size tells the library which fields the
 * caller knows).  Field meanings are those of hb_union_step above; struct_size must be
 * at least hb_step_args_min_size().  hb_union_step is a thin wrapper that fills this struct. */
typedef struct hb_step_args {
  uint64_t struct_size;
  /* graph (internal ids) and the row range of this call */
  int64_t n, lo, hi;
  const int64_t *offsets;
  const int32_t *succ;
  /* counters, change flags, estimates */
  const uint8_t *cur;
  uint8_t *nxt;
  const uint32_t *chg_prev;
  uint32_t *chg_now;
  double *est;
  int32_t b, dense, clear_chg_now, n_disc;
  int64_t t;
  const double *lc_table;
  double alpha_p2, lc_cut;
  /* fused accumulator (each may be NULL) and discounted-gain sums */
  double *sum_dist, *sum_recip;
  double *disc;
  int64_t disc_stride;
  const double *disc_scale;
  int32_t disc_div, n_peers;
  /* heavy-node schedule */
  int64_t light_max_deg;
  const int32_t *heavy_nodes, *item_first;
  int64_t n_heavy;
  const int32_t *finish_order;
  int64_t n_mega;
  const int32_t *item_node;
  const int64_t *item_beg;
  int64_t n_items, item_arcs;
  uint8_t *partial;
  /* outputs and options */
  uint64_t *nch_out, *merged_out;
  int64_t hot_rows;
  const uint32_t *active;
  uint8_t *const *peer_nxt;
  uint32_t *const *peer_chg;
  void *stream;
  /* bounds for the checked build (libhyperball_b200_checked.so; ignored otherwise):
   * addressable register rows (0 = n) and successor ids in succ (0 = unchecked) */
  int64_t check_rows, check_m;
  /* appended (read only when struct_size covers it; a caller built before passes the
   * size up to check_m, hb_step_args_min_size()): with n_peers > 0, 0 stores the written
   * rows unpacked into peer_nxt[q]; hb_push_row_stride(b) stores the rows that changed
   * 5-bit packed into peer_nxt[q] = the peer's inbox of this step (register_width <= 5
   * only), which the peer unpacks with hb_unpack_inbox after the step's barrier
   * (DESIGN.md section 6). */
  int64_t peer_packed_stride;
  /* appended: device uint64 scratch, or NULL.  With it the light kernel deals its node
   * chunks to the warps in the order they ask (a ticket counter the call zeroes on the
   * stream) instead of grid-stride: warps that drew long chunks take fewer, the launch
   * ends without a tail.  Results do not depend on it.  One scratch
   * word per stream: calls that may run concurrently must not share it. */
  uint64_t *ticket;
  /* appended: die-affine heavy items, or NULL / 0: die_head is a
   * device buffer of die_rows rows whose 2 KB chunks hb_die_map has mapped, item_split
   * the per-item split hb_die_partition wrote for that map.  Used for 16- / 32-register
   * rows of an array >= 1 GB with hot_rows > 0, outside frontier mode: the call copies
   * the first die_rows rows of cur into die_head and merges every item in two passes, each
   * on the SMs of one die (the result does not depend on it).  The call then needs
   * `ticket` to hold 2 uint64 words and `partial` 2 * n_items rows. */
  uint8_t *die_head;
  int64_t die_rows;
  const int32_t *item_split;
} hb_step_args;

int hb_union_step_v2(const hb_step_args *args);
uint64_t hb_step_args_size(void);   /* sizeof(hb_step_args) as built */
uint64_t hb_step_args_min_size(void); /* smallest struct_size accepted (fields up to check_m) */

/* Packed push (multi-GPU, register_width <= 5): bytes per row of a peer inbox for 2^b
 * registers (12 for b = 4, 10 * 2^b / 16 above), -1 for a bad b.  The writer stores only
 * rows that changed this step.  hb_unpack_inbox, for every v in [0, n) outside [lo, hi):
 * bit v set in chg_now -> nxt row v = the unpacked inbox row v; else set in
 * chg_prev_copy (changed in the previous step only) -> nxt row v = cur row v. */
int hb_push_row_stride(int b);
int hb_unpack_inbox(int64_t n, int64_t lo, int64_t hi, int b, const uint32_t *chg_now,
                    const uint32_t *chg_prev_copy, const uint8_t *inbox, const uint8_t *cur,
                    uint8_t *nxt, void *stream);

/* L2 persistence (hot_rows above): on by default.  hb_set_l2_persist(0) stops the
 * library from touching the persisting-L2 set-aside and the stream's access-policy
 * window (for a host that manages them itself).  When on, the set-aside limit is raised
 * to the library's size only if the current limit is smaller. */
void hb_set_l2_persist(int enable);

/* L2 die map (B200: two dies, each homing half of the L2; a line read from both dies is
 * cached twice).  For the 2 KB chunks of [base, base + bytes) -- chunk 0 is the 2 KB block
 * holding base[0] -- writes bit c = home die of chunk c into bits_out (device uint32
 * [hb_die_map_words(base, bytes)]), measured from the latency of atomicOr(p, 0) (data is
 * not changed) from SMs of both dies; the first call on a device also classifies its SMs.
 * stats (host int64 [4]): SMs of die 0, SMs of die 1, chunks on die 1, chunks whose two
 * latencies differ by < 64 cycles.  stats[0] == 0: the device did not split into two dies,
 * or the mechanism is not enabled (it is opt-in: environment HB_DIE=1), and bits_out is
 * untouched.  Synchronises the stream. */
int hb_die_map(void *base, int64_t bytes, uint32_t *bits_out, int64_t *stats, void *stream);
int64_t hb_die_map_words(const void *base, int64_t bytes);
/* Once per graph and head buffer: reorder the ids inside every heavy item (slices of
 * <= item_arcs <= 512 arcs, hb_heavy_items) into the two passes of the die-affine merge
 * -- first the sources whose row of `head` (die_rows rows of 2^b bytes, mapped by
 * hb_die_map into die_bits) is homed on die 0 and the sources >= die_rows with an even
 * id, then the rest; item_split[i] (device int32 [n_items]) = ids of the first pass.
 * succ is rewritten in place (the order of a row's ids does not matter to the union). */
int hb_die_partition(int64_t n_items, const int32_t *item_node, const int64_t *item_beg,
                     const int64_t *offsets, int32_t *succ, int64_t item_arcs, int b,
                     const void *head, int64_t die_rows, const uint32_t *die_bits,
                     int32_t *item_split, void *stream);

/* Finalizers (centrality.py:153-171) over device sums in internal order, written in
 * original order: out[o] uses internal row rank[o] (rank NULL = identity).
 *   closeness[o] = 1 / sum_dist where sum_dist > 0, else 0
 *   harmonic[o]  = sum_recip
 *   lin[o]       = coreach^2 / sum_dist where sum_dist > 0, else 1
 * Any output pointer may be NULL (not computed). */
int hb_finalize(int64_t n, const int32_t *rank, const double *sum_dist, const double *sum_recip,
                const double *coreach, double *closeness, double *harmonic, double *lin,
                void *stream);

/* Multi-GPU exchange.
 * hb_gather_changed: for every v in [lo, hi) with chg_bits bit v set, append v to ids_out
 *   and rows[v] to rows_out -- p = 2^b bytes per row, or hb_packed_row_bytes(b) bytes of
 *   5-bit fields when packed != 0 (only valid for register_width <= 5); *count_out
 *   (device uint64, zeroed by the call) receives the number appended.  Order unspecified.
 * hb_scatter_rows: dst[ids[i]] = rows[i] (unpacked when packed != 0) for i < k and set bit
 *   ids[i] of chg_bits (chg_bits may be NULL).
 * hb_refresh_rows: dst[v] = src[v] for every v in [0, n) outside [lo, hi) whose bit is
 *   set in bits (keeps the lazy double buffer of rows owned by other ranks). */
int hb_packed_row_bytes(int b);
int hb_gather_changed(int64_t lo, int64_t hi, const uint32_t *chg_bits, const uint8_t *rows,
                      int b, int packed, int32_t *ids_out, uint8_t *rows_out,
                      uint64_t *count_out, void *stream);
int hb_scatter_rows(int64_t k, const int32_t *ids, const uint8_t *rows, int b, int packed,
                    uint8_t *dst, uint32_t *chg_bits, void *stream);
int hb_refresh_rows(int64_t n, int64_t lo, int64_t hi, const uint32_t *bits, const uint8_t *src,
                    uint8_t *dst, int b, void *stream);

/* Schedule setup on the device (schedule.py).
 * hb_max_degree: *out (host) = max in-degree offsets[v+1] - offsets[v] over v < n;
 *   scratch: device uint64 [1].  Synchronises the stream.
 * hb_schedule_order: node order of the `degree` (order 1: stable sort by descending
 *   in-degree; with world > 1 the ranking is dealt round-robin, position j to rank j % W,
 *   slot bounds[j % W] + j / W) or `window` (order 2: stable sort by descending in-degree
 *   inside each light-kernel chunk window of each rank's range) schedule: perm[i] = old
 *   row of internal id i, rank = its inverse, new_offsets [n+1] = the prefix sums of the
 *   permuted in-degrees.  bounds: host int64 [world + 1] rank ranges.  temp == NULL
 *   queries *temp_bytes (keys / values / cub scratch).
 * hb_heavy_items: work items of the heavy rows (in-degree > light_max_deg) among rows
 *   [lo, lo + nrows) whose offsets are row_offsets[0..nrows] (global or rank-local
 *   positions): heavy[j] = row id, item_first [n_heavy + 1], item_node / item_beg
 *   [n_items] (slices of <= item_arcs arcs), finish_order = heavy indices, those with
 *   more than mega_items items first.  counts (host int64 [4]) receives n_heavy, n_items,
 *   n_mega and the number of rows with in-degree > 0; a call with heavy == NULL only
 *   counts (the caller then allocates the outputs and calls again).  temp == NULL
 *   queries *temp_bytes.  Synchronises the stream. */
int hb_max_degree(int64_t n, const int64_t *offsets, uint64_t *scratch, int64_t *out,
                  void *stream);
int hb_schedule_order(int64_t n, const int64_t *offsets, int order, int b, int world,
                      const int64_t *bounds, int32_t *perm, int32_t *rank,
                      int64_t *new_offsets, void *temp, uint64_t *temp_bytes, void *stream);
int hb_heavy_items(int64_t nrows, int64_t lo, const int64_t *row_offsets, int64_t light_max_deg,
                   int64_t item_arcs, int64_t mega_items, int32_t *heavy, int32_t *item_first,
                   int32_t *item_node, int64_t *item_beg, int32_t *finish_order,
                   int64_t *counts, void *temp, uint64_t *temp_bytes, void *stream);

/* Relabel a CSR into schedule order: new row i is old row perm[i] with every id mapped
 * through rank (rank[perm[i]] == i).  new_offsets (device int64 [n+1]) must already hold
 * the prefix sums of the permuted degrees. */
int hb_relabel_csr(int64_t n, const int64_t *old_offsets, const int32_t *old_succ,
                   const int32_t *perm, const int32_t *rank, const int64_t *new_offsets,
                   int32_t *new_succ, void *stream);

/* hb_relabel_csr restricted to the new rows [r0, r1) (the other rows are left as they
 * are): the schedule relabels the CSR slice by slice while the rest of the successor ids
 * are still being uploaded, and iteration 1 starts on the slices already relabelled. */
int hb_relabel_csr_rows(int64_t n, int64_t r0, int64_t r1, const int64_t *old_offsets,
                        const int32_t *old_succ, const int32_t *perm, const int32_t *rank,
                        const int64_t *new_offsets, int32_t *new_succ, void *stream);

/* hb_relabel_csr by OLD rows [o0, o1) (old row o becomes new row rank[o]): the degree
 * relabel runs on every slice of the successor-id upload as soon as it has landed. */
int hb_relabel_csr_src_rows(int64_t n, int64_t o0, int64_t o1, const int64_t *old_offsets,
                            const int32_t *old_succ, const int32_t *rank,
                            const int64_t *new_offsets, int32_t *new_succ, void *stream);

/* *out (device uint64) = how many of `samples` pseudo-random arcs (arc splitmix64(seed + i)
 * mod m of succ, device int32 [m]) have their source flagged in bits (device uint32
 * [ceil(n/32)]): an estimate of the share of arcs whose source changed, which decides
 * whether the next step merges every source without the per-source test (engine.py). */
int hb_sample_flagged_arcs(int64_t m, const int32_t *succ, const uint32_t *bits,
                           int64_t samples, uint64_t seed, uint64_t *out, void *stream);

/* Sort the ids of every CSR row ascending (schedule setup, after hb_relabel_csr): offsets
 * (device int64 [n+1]) describe the rows of ids (device int32 [m]); alt (device int32 [m])
 * is scratch of the same size.  The rows are sorted in n_batches batches of < 2^31 arcs:
 * batch q covers rows [host_batch_rows[q], host_batch_rows[q+1]) whose arcs start at
 * host_batch_arcs[q] (= offsets[host_batch_rows[q]]; both HOST arrays of n_batches + 1).
 * Call with temp == NULL to get the scratch size in *temp_bytes, then again with that
 * buffer.  The sorted ids end in `ids` (*result_in_alt, if given, is set to 0). */
int hb_sort_rows(int64_t n, const int64_t *offsets, int64_t n_batches,
                 const int64_t *host_batch_rows, const int64_t *host_batch_arcs, int32_t *ids,
                 int32_t *alt, void *temp, uint64_t *temp_bytes, int *result_in_alt,
                 void *stream);

/* At-rest register format (hll.py:128-132 CounterArray.registers, hll.py:161-177 HLLA blob
 * body): every register's `width` low bits MSB-first, rows of p*width/8 bytes back to back.
 * hb_pack_registers: regs (device uint8 [*, p], p = 2^b) -> out (device uint8
 * [n, p*width/8]), packed row i taken from regs row order[i] (order: device int32 [n] or
 * NULL = identity; pass the schedule's rank to pack in original node order).
 * hb_unpack_registers: the inverse, regs row i from packed row order[i] (pass perm). */
int hb_pack_registers(int64_t n, int b, int width, const uint8_t *regs, const int32_t *order,
                      uint8_t *out, void *stream);
int hb_unpack_registers(int64_t n, int b, int width, const uint8_t *packed, const int32_t *order,
                        uint8_t *regs, void *stream);

/* Batched runs (run_multi, cli.py:222-254): R = 2^log2_runs runs with
 * the same log2m b share one CSR scan.  cur / nxt hold n rows of R * p bytes (run r's
 * registers at bytes [r*p, (r+1)*p) of a row; R * p <= 256), est / sum_dist / sum_recip
 * are [R, run_stride] fp64 (run r at + r * run_stride, run_stride >= n).  chg_prev /
 * chg_now are the OR over runs of the change flags (source skip and lazy double buffer,
 * as hb_union_step; chg_now is cleared by the call), chg_runs (device uint32 [R, ceil(n/32)],
 * cleared by the call) receives each run's change bits and run_nch_out (device uint64 [R])
 * each run's changed count; *nch_out counts nodes with any run changed.  Discounted sums
 * as hb_union_step, disc laid out [R, n_disc, disc_stride].  The schedule arrays are
 * those of build at log2m b + log2_runs (the wide row).  Every run's bits equal an
 * independent hb_union_step run with its own seed. */
int hb_union_step_runs(int64_t n, int64_t lo, int64_t hi, const int64_t *offsets,
                       const int32_t *succ, const uint8_t *cur, uint8_t *nxt,
                       const uint32_t *chg_prev, uint32_t *chg_now, uint32_t *chg_runs,
                       double *est, double *sum_dist, double *sum_recip, int64_t run_stride,
                       int64_t t, const double *lc_table, double alpha_p2, double lc_cut, int b,
                       int log2_runs, int dense, int64_t light_max_deg,
                       const int32_t *heavy_nodes, const int32_t *item_first, int64_t n_heavy,
                       const int32_t *finish_order, int64_t n_mega, const int32_t *item_node,
                       const int64_t *item_beg, int64_t n_items, int64_t item_arcs,
                       uint8_t *partial, uint64_t *nch_out, uint64_t *merged_out,
                       uint64_t *run_nch_out, int64_t hot_rows, double *disc,
                       int64_t disc_stride, int n_disc, const double *disc_scale, int disc_div,
                       const uint32_t *active, void *stream);

/* Exact backend (engine.py:178-213, _kernels.py:117-172): one bitset of n bits per node,
 * MSB-first bytes (the reference's rows), padded to row_stride bytes (multiple of 16,
 * >= ceil(n/8)).  hb_exact_seed: zero every row, set node v's own bit, est[v] = weight
 * (weights: device int64 [n] or NULL = 1).  hb_exact_union_step: one step over all nodes
 * with the source-skip rule -- OR of the changed sources' rows into nxt, change test,
 * est = weighted popcount (exact), fused accumulate and discounted sums as hb_union_step;
 * nch_out / merged_out as hb_union_step; chg_now is cleared by the call. */
int hb_exact_seed(int64_t n, int64_t row_stride, uint8_t *bits, double *est,
                  const int64_t *weights, void *stream);
int hb_exact_union_step(int64_t n, const int64_t *offsets, const int32_t *succ,
                        const uint8_t *cur, uint8_t *nxt, int64_t row_stride,
                        const uint32_t *chg_prev, uint32_t *chg_now, double *est,
                        double *sum_dist, double *sum_recip, int64_t t, int dense,
                        const int64_t *weights, double *disc, int64_t disc_stride, int n_disc,
                        const double *disc_scale, int disc_div, uint64_t *nch_out,
                        uint64_t *merged_out, void *stream);

/* Frontier mode for sparse iterations.
 * hb_mark_active: active = chg_prev | out-neighbours(chg_prev) (device bitmaps over n
 *   nodes), the only nodes the source-skip rule can touch this iteration. */
/* hb_forward_csr: the forward graph by counting sort -- fwd_offsets (device int64 [n+1]),
 *   cursor (device int64 [n], scratch), fwd_dst (device int32 [m]); rows unordered.
 *   temp == NULL queries *temp_bytes (scan scratch). */
int hb_forward_csr(int64_t n, const int64_t *offsets, const int32_t *succ, int64_t m,
                   int64_t *fwd_offsets, int64_t *cursor, int32_t *fwd_dst, void *temp,
                   uint64_t *temp_bytes, void *stream);
int hb_mark_active(int64_t n, const int64_t *fwd_offsets, const int32_t *fwd_succ,
                   const uint32_t *chg_prev, uint32_t *active, void *stream);
/* hb_mark_pull: the same active bitmap from the CSR of G^T alone (no forward graph): one
 *   streaming pass over the successor ids (short sparse tails).  Rows with in-degree >
 *   light_max_deg are marked through the schedule's work items (item_node / item_beg /
 *   n_items / item_arcs, as for hb_union_step), which must cover them. */
int hb_mark_pull(int64_t n, const int64_t *offsets, const int32_t *succ,
                 const uint32_t *chg_prev, uint32_t *active, int64_t light_max_deg,
                 const int32_t *item_node, const int64_t *item_beg, int64_t n_items,
                 int64_t item_arcs, void *stream);

/* hb_mark_pull with two speed-ups, same result.  heavy_lo < heavy_hi: the heavy rows are
 * exactly the row range [heavy_lo, heavy_hi) (degree order), so their ids are streamed
 * flat instead of item by item.  filter != NULL (nearly converged steps, a few thousand
 * changed nodes): a 2^18-bit hash filter of the changed nodes is built there (device
 * uint32 [hb_change_filter_words()]) and kept in shared memory by every block, so each
 * streamed id is tested there and the change bitmap is read only on a filter hit. */
int hb_mark_pull_filtered(int64_t n, const int64_t *offsets, const int32_t *succ,
                          const uint32_t *chg_prev, uint32_t *active, int64_t light_max_deg,
                          const int32_t *item_node, const int64_t *item_beg, int64_t n_items,
                          int64_t item_arcs, int64_t heavy_lo, int64_t heavy_hi,
                          uint32_t *filter, void *stream);
int64_t hb_change_filter_words(void);

/* GPU graph build.
 * hb_gen_rmat_keys: m R-MAT arcs (scale levels, 32-bit quadrant thresholds thr_a <= thr_ab
 *   <= thr_abc, counter-based splitmix RNG keyed by seed -- bit-identical to
 *   libhbgraph.so's hbg_rmat) as device uint64 keys (dst << 32 | src) of the transpose;
 *   self-loops are written as ~0.
 * hb_keys_to_csr: sort + deduplicate the keys (keys and alt: device uint64 [m], both
 *   clobbered), drop the self-loop sentinel, and write the CSR of the transpose:
 *   offsets (device int64 [n+1]) and succ (device int32 [>= unique arcs]); *m_out (HOST)
 *   receives the number of arcs.  temp == NULL queries *temp_bytes.  Synchronises
 *   `stream` once (to size the output). */
int hb_gen_rmat_keys(int scale, int64_t m, uint64_t thr_a, uint64_t thr_ab, uint64_t thr_abc,
                     uint64_t seed, uint64_t *keys, void *stream);
int hb_keys_to_csr(int64_t n, int64_t m, uint64_t *keys, uint64_t *alt, void *temp,
                   uint64_t *temp_bytes, int64_t *m_out, int64_t *offsets, int32_t *succ,
                   void *stream);

/* Device builders of the other synthetic configs (bit-identical to libhbgraph.so's hbg_er /
 * hbg_disconnected / hbg_weblike): kind 1 = ER, 3 = disconnected, 4 = web-like.
 * hb_gen_degrees: deg[u] (device int64 [n]) = out-degree of source u, drawn from the host
 *   built CDF table (device fp64 [cdf_len]: Poisson CDF for kinds 1 / 3, Zipf CDF on
 *   {kmin..} for kind 4 -- the same tables graphgen.c builds).
 * hb_gen_blocks: the disconnected config's blocks: the giant block [0, giant), then
 *   Geometric(geo_p) sized blocks; lo / hi (device int64 [n]) receive each node's block
 *   bounds.  size / start: device int64 scratch [n - giant]; temp == NULL queries
 *   *temp_bytes.
 * hb_gen_arc_keys: the arcs of every source u at offsets[u]..offsets[u+1] (device int64
 *   [n+1], exclusive prefix sum of the degrees) as transpose keys (dst << 32 | src),
 *   self-loops as ~0; feed them to hb_keys_to_csr. */
int hb_gen_degrees(int kind, int64_t n, uint64_t seed, const double *cdf, int64_t cdf_len,
                   int64_t kmin, int64_t *deg, void *stream);
int hb_gen_blocks(int64_t n, int64_t giant, double geo_p, uint64_t seed, int64_t *size,
                  int64_t *start, int64_t *lo, int64_t *hi, void *temp, uint64_t *temp_bytes,
                  void *stream);
int hb_gen_arc_keys(int kind, int64_t n, uint64_t seed, const int64_t *offsets,
                    const int64_t *block_lo, const int64_t *block_hi, double p_local,
                    int64_t window, uint64_t *keys, void *stream);

/* Transpose of a CSR on the device (graph.py:145-155 transpose: every arc reversed,
 * duplicates and self-loops kept, each new row listing its sources in ascending order --
 * the reference's stable argsort by target).  offsets / succ: device int64 [n+1] /
 * int32 [m]; keys, alt: device uint64 [m] scratch; out_offsets / out_succ: device int64
 * [n+1] / int32 [m].  temp == NULL queries *temp_bytes. */
int hb_transpose_csr(int64_t n, int64_t m, const int64_t *offsets, const int32_t *succ,
                     uint64_t *keys, uint64_t *alt, void *temp, uint64_t *temp_bytes,
                     int64_t *out_offsets, int32_t *out_succ, void *stream);

/* out[k] = rank[ids[k]] for k < m (device int32 arrays; out may alias ids): a rank-local
 * CSR's ids relabelled into the internal order (multi-GPU). */
int hb_map_ids(int64_t m, const int32_t *ids, const int32_t *rank, int32_t *out, void *stream);

/* out[i] = hash_items(items[i], replicas[i], seed) (hll.py:79-88), device arrays. */
int hb_hash_items(int64_t n, const uint64_t *items, const uint64_t *replicas, uint64_t seed,
                  uint64_t *out, void *stream);

/* Number of work items / recommended item size for heavy-node splitting at log2m b. */
int64_t hb_item_arcs(int b);
int64_t hb_light_max_deg(int b);
/* Light-kernel geometry at log2m b: nodes per warp round (npw) and nodes per grid-stride
 * chunk (window); the "window" schedule sorts nodes by in-degree inside each window. */
int64_t hb_light_npw(int b);
int64_t hb_light_window(int b);

#ifdef __cplusplus
}
#endif

#endif /* HYPERBALL_B200_H */
