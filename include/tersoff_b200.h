/*
 * tersoff_b200.h -- C ABI of the B200-native Tersoff energy/force/virial path.
 *
 * This is the drop-in boundary for the reference `tersoffmd` hot path
 * (/root/reference/pkg/src/tersoffmd).  The reference has no FFI; its plugin
 * point is the Python function kernels.compute() (kernels.py:517-527) fed by
 * neighbor.build_neighbor_list()/needs_rebuild() (neighbor.py:194-229).  Each
 * entry point below names the reference interface it replaces.  The Python
 * host package paper_1710_00882_b200 binds these symbols with ctypes
 * (paper_1710_00882_b200/_native.py); INTEGRATION.md shows the binding a
 * reference maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Array arguments may be HOST or DEVICE
 *    pointers (detected with cudaPointerGetAttributes); host arrays are copied
 *    on the context's stream, device arrays are used in place.
 *  - positions/forces are (n,3) row-major float64 in Angstrom / eV/A;
 *    species are int32 in [0, nspecies); box lengths float64[3]; periodic
 *    int32[3] (0/1).
 *  - Every call returns a TB_* status; tb_last_error() gives the message.
 *    TB_ERR_CONFIG maps to ConfigurationError, TB_ERR_INPUT to InputError
 *    (errors.py:9-14), with the reference's message wording.
 *  - A context is bound to one device and one CUDA stream and is not
 *    re-entrant.  Scratch memory is context-owned; outputs are caller-owned.
 */
#ifndef TERSOFF_B200_H
#define TERSOFF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_OK 0
#define TB_ERR_CONFIG 1 /* -> ConfigurationError */
#define TB_ERR_INPUT 2  /* -> InputError */
#define TB_ERR_CUDA 3   /* CUDA runtime failure */
#define TB_ERR_ARG 4    /* bad argument (null pointer, size) */
#define TB_ERR_UNSUPPORTED 5 /* tb_md_run cannot take this system: use tb_md_step */

#define TB_PREC_DOUBLE 0 /* fp64 everywhere ("double", kernels.py:154-165) */
#define TB_PREC_MIXED 1  /* fp64 positions/displacements/accumulators, fp32 potential math ("single") */

#define TB_SCATTER_ATOMIC 0 /* dzeta scatter to j/k with red.global.add.f64 */
#define TB_SCATTER_GATHER 1 /* per-entry force buffer + deterministic gather pass */

typedef struct tb_context tb_context;
typedef struct tb_nlist tb_nlist;

/* stats[] layout written by tb_compute */
#define TB_STAT_ZETA_VISITS 0 /* sum_i n_i^2 over packed rows (kernels.py:537-544) */
#define TB_STAT_PACKED_PAIRS 1 /* entries with r < r_cut at current positions */
#define TB_STAT_LIVE_PAIRS 2   /* packed pairs inside their own pair cutoff */
#define TB_STAT_LIVE_TRIPLETS 3 /* (i,j,k) with live j and f_C(r_ik) > 0 */
#define TB_STAT_TAPER_PAIRS 4   /* live pairs with R-D < r_ij (sin/cos taper evaluated) */
#define TB_STAT_TAPER_TRIPLETS 5 /* live triplets with R-D < r_ik */
#define TB_NSTATS 6

/* ---- context ---------------------------------------------------------- */

/* New context on `device`.  Replaces nothing in the reference (it has no
 * device state); owns the stream and scratch buffers. */
int tb_create(int device, tb_context **out);
void tb_destroy(tb_context *ctx);
const char *tb_last_error(const tb_context *ctx);
/* Use an external CUDA stream (cudaStream_t, e.g. torch's current stream);
 * NULL selects the legacy default stream.  Until this is called the context
 * uses its own non-blocking stream. */
int tb_set_stream(tb_context *ctx, void *stream);
/* Kernel-selection options.  TB_OPT_TILE_KERNEL = 1 forces the general
 * shared-memory tile kernel even when the warp-chunk kernel applies (rows of
 * <= 32 skin-list entries); used to cover both paths in the parity tests. */
#define TB_OPT_TILE_KERNEL 1
/* TB_OPT_LIST_MARGIN = p: neighbour lists built from now on reserve p percent
 * (default 25) of extra entries and warp chunks, the room tb_md_run's device
 * rebuild grows into before it has to replay from its entry state. */
#define TB_OPT_LIST_MARGIN 2
/* TB_OPT_LIVE_PACK = 0 / 1 / 2 (off / on / auto, default auto): before each
 * evaluation cut every skin-list row to its entries with r < r_cut at the
 * current positions (pack_adjacency, neighbor.py:330-360) and re-chunk the
 * rows on the device, so that dead entries occupy no warp lanes.  Auto: on for
 * atomic scatter over species-filtered rows (multi-species tables). */
#define TB_OPT_LIVE_PACK 3
/* TB_OPT_MD_LOOSE_SKIN = h: tb_md_run (one species, atomic scatter) keeps a
 * list with skin + h/100 A (default 30 = 0.3 A) that it rebuilds only when an
 * atom moved more than half of that; the reference's own rebuilds are still
 * decided, counted and their positions kept, and the exact list at the last of
 * them is rebuilt when the run ends.  0 = rebuild the exact list every time. */
#define TB_OPT_MD_LOOSE_SKIN 4
/* TB_OPT_REPACK_MARGIN = d: the live repack (TB_OPT_LIVE_PACK) cuts rows to
 * r < r_cut + d/1000 A (default 1 = 0.001 A) and is redone only when some atom
 * moved more than half of that since the last repack (decided on the device);
 * the kernel's exact r < r_cut test keeps every term identical.  0 = repack
 * exactly at every evaluation.  (Wider margins keep the repack across MD steps
 * but add dead lanes: config 3 step 261 / 276 / 331 us at 1 / 10 / 50 mA.) */
#define TB_OPT_REPACK_MARGIN 5
/* TB_OPT_STREAM_RANGE = r (default 131072, 0 = off): tb_compute called with
 * PINNED host positions / forces / per-atom energies on a system of at least
 * 8 r atoms (one species, atomic scatter) streams the call: the atoms are cut
 * into up to 32 index ranges of at least r atoms, a warp chunk runs as soon as
 * the ranges it references are on the device, and a range's forces go back
 * once the last chunk touching it has run -- host-to-device copy, kernel and
 * device-to-host copy overlap (PCIe is full duplex).  Same chunks, same
 * arithmetic as the unstreamed call; pays off when the atom order is
 * spatially coherent (lattice order), falls back to sequential otherwise. */
#define TB_OPT_STREAM_RANGE 6
/* TB_OPT_ROW_KERNEL = 0 / 1 / m (default 1): one-species, lam3 = 0 tables
 * evaluate rows of at most 4 skin-list entries with the atom-per-lane kernel
 * (one lane holds an atom's neighbours in registers; g(cos) once per unordered
 * pair) when the list has at least m such rows (1 = the default threshold,
 * 1000000: one lane per atom needs about that many atoms to beat the warp-chunk kernel); longer
 * rows keep the warp-chunk kernel.  0 = warp-chunk kernel for every row. */
#define TB_OPT_ROW_KERNEL 7
int tb_set_option(tb_context *ctx, int option, int value);

/* Synchronise the context's stream. */
int tb_synchronize(tb_context *ctx);

/* Parameter table, flattened exactly like ParamTable.views()
 * (potential.py:127-155): pair_mat[S*S*8] = [R,D,A,lam1,B,lam2,beta,eta] of
 * entry (i,j,j); trip_mat[S^3*8] = [R,D,gamma,c,d,h,lam3,m] of entry (i,j,k).
 * Host pointers.  1 <= nspecies <= 64 (1-4: compile-time kernels; 5-64: the
 * tile kernel with a runtime species count).  r_cut_out (may be NULL) receives
 * max(R+D) (potential.py:106). */
int tb_set_params(tb_context *ctx, int nspecies, const double *pair_mat,
                  const double *trip_mat, double *r_cut_out);

/* ---- neighbour list (neighbor.py:194-229) ------------------------------- */

int tb_nlist_create(tb_context *ctx, tb_nlist **out);
void tb_nlist_destroy(tb_nlist *nl);

/* build_neighbor_list(state, r_cut, skin) (neighbor.py:194-217): full
 * symmetric list at bc = r_cut + skin, rows ascending; the pair set equals the
 * reference's bit for bit.  Snapshots the positions for tb_needs_rebuild. */
int tb_build_neighbors(tb_context *ctx, tb_nlist *nl, int64_t n, const double *positions,
                       const double *box, const int32_t *periodic, double r_cut,
                       double skin);
/* Domain-decomposed variant: atoms [0, n_owned) are owned, [n_owned, n) are
 * ghosts (halo copies, unshifted coordinates).  Only owned atoms get rows, so
 * only their energy terms are evaluated; ghosts appear as neighbours j, k.
 * The pair set of every owned row equals the single-domain list's. */
int tb_build_neighbors_owned(tb_context *ctx, tb_nlist *nl, int64_t n, int64_t n_owned,
                             const double *positions, const double *box,
                             const int32_t *periodic, double r_cut, double skin);

/* Import a neighbour list built elsewhere -- the reference's NeighborList
 * (neighbor.py:170-191: offsets[n+1] / neighbors int64 CSR, its
 * reference_positions snapshot, build r_cut and skin) -- so the reference's
 * own ForceField / run_nve / verify suites evaluate on the B200 kernels
 * without rebuilding their list.  Rows are used as given
 * (the evaluation re-tests r < r_cut at the current positions, as
 * pack_adjacency does); tb_needs_rebuild works against ref_positions.
 * Host or device pointers.  Imported lists have no cell grid, so
 * tb_nlist_rebuild_device / tb_md_run return TB_ERR_UNSUPPORTED for them
 * (tb_build_neighbors replaces them with a native list). */
int tb_nlist_import(tb_context *ctx, tb_nlist *nl, int64_t n, const int64_t *offsets,
                    const int64_t *neighbors, const double *ref_positions, const double *box,
                    const int32_t *periodic, double r_cut, double skin);

/* Forget the species-pair compute filter (multi-species tables): the next
 * evaluation derives it again from the species it is given.  Needed only
 * after changing a device species array in place (see tb_compute_device). */
int tb_nlist_refilter(tb_context *ctx, tb_nlist *nl);

/* number of list entries (sum of row lengths) and the longest row */
int tb_nlist_info(const tb_nlist *nl, int64_t *n_atoms, int64_t *n_entries,
                  int64_t *max_row);
/* export the CSR (offsets[n+1], neighbors[n_entries]) as int64, host or
 * device pointers (NeighborList.offsets / .neighbors, neighbor.py:170-191) */
int tb_nlist_export(tb_context *ctx, const tb_nlist *nl, int64_t *offsets,
                    int64_t *neighbors);
/* needs_rebuild(state, nl) (neighbor.py:220-229): *out = 1 when any atom
 * moved more than skin/2 (min image) since the build. */
int tb_needs_rebuild(tb_context *ctx, const tb_nlist *nl, const double *positions,
                     int32_t *out);

/* ---- the Tersoff evaluation (kernels.py:517-527 compute()) ------------- */

/* One energy + force (+ virial) evaluation at the given positions:
 * re-packs the skin list at the current positions (pack_adjacency,
 * neighbor.py:330-360) and evaluates the Tersoff terms (ScalarOpt semantics,
 * kernels.py:250-315; math potential.py:167-290).
 *   forces    (n,3) out, required          per_atom (n) out, may be NULL
 *   energy    1 double out (host), required virial[6] xx,yy,zz,xy,xz,yz, may be NULL
 *   stats     TB_NSTATS int64 (host), may be NULL
 * r_cut must not exceed the list's build r_cut (neighbor.py:334-337).
 * Synchronises the stream before returning.  Host buffers that are pinned
 * (page-locked) are the fast path: small systems get their forces written
 * straight into host memory, large one-species systems are streamed in atom
 * ranges so that both copy directions and the kernel overlap
 * (TB_OPT_STREAM_RANGE); pageable buffers are staged and copied. */
int tb_compute(tb_context *ctx, const tb_nlist *nl, const double *positions,
               const int32_t *species, double r_cut, int precision, int scatter,
               double *forces, double *per_atom, double *energy, double *virial,
               int64_t *stats);

/* Asynchronous, device-resident variant for drivers, benchmarks and CUDA
 * graph capture: all pointers are DEVICE pointers; `result` receives
 * [energy, virial(6)] as 7 doubles; `dstats` TB_NSTATS uint64 (may be NULL).
 * Does not synchronise; validation errors are latched on the device and
 * reported by the next tb_check_errors().  With two or more species the
 * first call after a build (or after tb_set_params, or with a different
 * species pointer) derives a species-pair compute filter from d_species (one
 * host synchronisation).  Species changed IN PLACE afterwards are detected on
 * the device (a copy of the filter's species is compared every evaluation):
 * tb_compute then rebuilds the filter and re-evaluates; here the next
 * tb_check_errors() returns TB_ERR_INPUT -- call tb_nlist_refilter (or
 * rebuild the list) and evaluate again. */
int tb_compute_device(tb_context *ctx, const tb_nlist *nl, const double *d_positions,
                      const int32_t *d_species, double r_cut, int precision, int scatter,
                      double *d_forces, double *d_per_atom, double *d_result,
                      uint64_t *d_stats);
int tb_check_errors(tb_context *ctx);

/* Kernel timing for the roofline report: while enabled, CUDA events bracket
 * every Tersoff kernel launch on the context stream; tb_profile_read
 * synchronises, returns the summed kernel milliseconds and launch count since
 * the last read, and resets them. */
int tb_profile(tb_context *ctx, int enable);
int tb_profile_read(tb_context *ctx, double *total_ms, int64_t *launches);

/* ---- device-resident NVE (system.py:355-380, :427-460) ------------------ */

/* One velocity-Verlet step on device buffers (positions, velocities, forces
 * updated in place; mass per atom in amu, v += 0.5 dt accel F / m).  Rebuilds the list on the skin/2
 * trigger or when `force_rebuild` is set; *rebuilt (host, may be NULL)
 * reports it.  d_result (8 doubles) as in tb_compute_device plus the kinetic
 * energy 0.5 sum m v^2 / accel in d_result[7] (system.py:129-134). */
int tb_md_step(tb_context *ctx, tb_nlist *nl, int64_t n, double *d_positions,
               double *d_velocities, double *d_forces, const double *d_mass,
               const int32_t *d_species, const double *box, const int32_t *periodic,
               double dt, double accel, double r_cut, double skin, int precision,
               int scatter, int force_rebuild, double *d_per_atom, double *d_result,
               int32_t *rebuilt);

/* Rebuild nl in place at d_positions with the device-side builder of
 * tb_md_run (sizes kept in device memory, no host round trip between its
 * kernels; one synchronisation at the end to refresh the host-side counts).
 * Same pair set and row order as tb_build_neighbors (neighbor.py:157-212);
 * falls back to it when the list outgrows its capacity.  Requires a list
 * built by tb_build_neighbors for a periodic box with rows <= 32 entries
 * (else TB_ERR_UNSUPPORTED). */
int tb_nlist_rebuild_device(tb_context *ctx, tb_nlist *nl, const double *d_positions,
                            const int32_t *d_species, int scatter);

/* Warp-chunk layout of the list the Tersoff kernel runs on: *nchunks warps
 * of 32 lanes, *lanes_used of them holding a list entry (lane occupancy,
 * the B200 counterpart of the reference's lane_active / lane_total,
 * kernels.py:80-92).  Zero chunks when the general tile kernel is used. */
int tb_nlist_lanes(const tb_nlist *nl, int64_t *nchunks, int64_t *lanes_used);

/* Device-resident NVE run: `steps` velocity-Verlet steps (same semantics as
 * tb_md_step: skin/2 trigger plus a fixed cadence when rebuild_every > 0,
 * system.py:355-380, 427-460) as ONE CUDA-graph launch with no host
 * synchronisation inside -- the neighbour-list rebuild runs on the device in
 * a conditional graph node, its sizes kept in device memory.  On entry nl must
 * be built (tb_build_neighbors) for periodic boxes, d_forces / d_result[0] hold
 * F and E of the current positions.  Every `record_every` steps (step s =
 * 1..steps) [E_pot, E_kin] is written to d_series[2*(s/record_every)] (row 0 is
 * the caller's).  On return d_result holds E, W6 and E_kin (d_result[7]) of the
 * last step; *rebuilds = rebuilds done.  Capacity overflows are replayed from
 * the entry state internally.  Returns TB_ERR_UNSUPPORTED (state untouched)
 * when the system needs the general path (free axes, rows > 32 entries, > 2
 * species, tile kernel forced): call tb_md_step per step instead.  Replaces
 * the step loop of run_nve (system.py:427-460). */
int tb_md_run(tb_context *ctx, tb_nlist *nl, int64_t n, double *d_positions,
              double *d_velocities, double *d_forces, const double *d_mass,
              const int32_t *d_species, double dt, double accel, double r_cut, double skin,
              int rebuild_every, int precision, int scatter, int64_t steps, int record_every,
              double *d_series, double *d_result, int64_t *rebuilds);

/* ---- slab domain decomposition (north_star (4)) --------
 *
 * The reference has no decomposition; these entries replace no
 * reference symbol -- they split the evaluation / NVE run above over ranks
 * (one process per GPU) with results equal to the single-domain ones.  Each
 * rank owns a slab of whole x cell columns of the neighbour grid (>= 2 per
 * rank); ghosts are the atoms of the one column beyond each face (width >=
 * r_cut + skin), kept at unshifted coordinates so every displacement and pair
 * set equals the single-domain one; only owned atoms get list rows, so every
 * energy term is evaluated exactly once, and forces landing on ghosts are
 * returned to their owners (reverse halo).
 *
 * The caller owns the transport (NCCL / gloo P2P).  Message rows are float64,
 * laid out [to-left | to-right] in the SEND buffer; incoming rows go to
 * [from-left | from-right] of the RECV buffer (tb_dd_recv_buffer), or -- for
 * the forward position halo -- straight into the ghost rows of POS.
 *   rebuild:  tb_dd_migrate_pack -> send 9-double rows, exchange counts ->
 *             tb_dd_recv_buffer -> recv -> tb_dd_migrate_unpack;
 *             tb_dd_halo_pack -> send 2-double [id, species] rows ->
 *             tb_dd_recv_buffer -> recv -> tb_dd_halo_unpack;
 *             tb_dd_pack_positions -> positions halo -> tb_dd_build
 *   evaluate: tb_dd_pack_positions -> positions halo (SEND -> ghost rows of
 *             POS) -> tb_dd_compute -> ghost rows of FORCES to the
 *             neighbours, theirs into RECV -> tb_dd_reverse_add -> sum the
 *             [E, W6] result over ranks
 *   NVE step: tb_dd_kick_drift (max drift^2 over ranks decides the rebuild:
 *             skin/2 trigger, neighbor.py:220-229) -> [rebuild] -> evaluate
 *             -> tb_dd_kick (E_kin in result[7], summed over ranks). */
typedef struct tb_domain tb_domain;
#define TB_DD_POS 0     /* (n_owned + ghosts, 3) float64 */
#define TB_DD_VEL 1     /* (n_owned, 3) float64 */
#define TB_DD_FORCES 2  /* (n_owned + ghosts, 3) float64 */
#define TB_DD_MASS 3    /* (n_owned) float64 amu */
#define TB_DD_SPECIES 4 /* (n_owned + ghosts) int32 */
#define TB_DD_IDS 5     /* (n_owned + ghosts) int64 global atom ids */
#define TB_DD_SEND 6    /* message rows to the neighbours */
#define TB_DD_RECV 7    /* message rows from the neighbours */
/* rank of nranks; box / periodic as tb_build_neighbors (x must be periodic) */
int tb_dd_create(tb_context *ctx, int rank, int nranks, const double *box,
                 const int32_t *periodic, double r_cut, double skin, tb_domain **out);
void tb_dd_destroy(tb_domain *dd);
/* this rank's owned atoms (host or device arrays): positions, velocities,
 * per-atom masses, species, global ids */
int tb_dd_load(tb_domain *dd, int64_t n, const double *pos, const double *vel,
               const double *mass, const int32_t *species, const int64_t *ids);
/* out[10] = n_owned, ghosts from left, ghosts from right, send-left rows,
 * send-right rows, migrants to left, migrants to right, capacity, first and
 * last owned column */
int tb_dd_counts(const tb_domain *dd, int64_t *out);
/* device pointer of a domain buffer (valid until the next call that may grow
 * it: tb_dd_load, *_pack, *_unpack, tb_dd_recv_buffer) */
int tb_dd_buffer(tb_domain *dd, int which, void **ptr);
/* RECV buffer with room for rows x width doubles */
int tb_dd_recv_buffer(tb_domain *dd, int64_t rows, int width, void **ptr);
/* migration at a rebuild: owned atoms whose x column now belongs to the
 * left / right rank are packed (9 doubles) into SEND; synchronises.
 * TB_ERR_INPUT if an atom moved farther than one slab. */
int tb_dd_migrate_pack(tb_domain *dd, int64_t *n_to_left, int64_t *n_to_right);
/* kept atoms compacted in order, received rows [from-left | from-right]
 * appended; ghosts cleared */
int tb_dd_migrate_unpack(tb_domain *dd, int64_t n_from_left, int64_t n_from_right);
/* halo send lists (owned atoms in the first / last column) and their
 * [id, species] rows in SEND; synchronises */
int tb_dd_halo_pack(tb_domain *dd, int64_t *n_send_left, int64_t *n_send_right);
/* ghost ids / species from RECV; ghost rows follow the owned rows */
int tb_dd_halo_unpack(tb_domain *dd, int64_t n_ghost_left, int64_t n_ghost_right);
/* SEND <- positions of the send lists (3 doubles per row); asynchronous */
int tb_dd_pack_positions(tb_domain *dd);
/* owned-rows neighbour list over [owned | ghosts] (tb_build_neighbors_owned) */
int tb_dd_build(tb_domain *dd, tb_nlist *nl);
/* evaluation over the local atoms: FORCES on [owned | ghosts], d_result =
 * [E, W6] of the owned rows (device, 7+ doubles), d_stats may be NULL;
 * asynchronous */
int tb_dd_compute(tb_domain *dd, const tb_nlist *nl, int precision, int scatter,
                  double *d_result, uint64_t *d_stats);
/* FORCES[send lists] += RECV rows (forces the neighbours computed on their
 * ghosts); asynchronous, deterministic */
int tb_dd_reverse_add(tb_domain *dd);
/* v += dt/2 accel F/m, x += dt v, wrap (owned atoms); d_drift2 (device double)
 * = max min-image drift^2 against nl's build positions; asynchronous */
int tb_dd_kick_drift(tb_domain *dd, const tb_nlist *nl, double dt, double accel,
                     double *d_drift2);
/* v += dt/2 accel F/m (owned) and d_result[7] = this rank's kinetic energy */
int tb_dd_kick(tb_domain *dd, double dt, double accel, double *d_result);
/* owned atoms out (host or device pointers, each may be NULL) */
int tb_dd_export(tb_domain *dd, int64_t *ids, double *pos, double *vel, double *forces);

/* Diagnostic: measured FMA throughput of this GPU in TFLOP/s (2 flops per
 * FMA), precision TB_PREC_DOUBLE -> DFMA, TB_PREC_MIXED -> FFMA; the roofline
 * denominator for the CUDA-core pipes (MEASURED_PEAKS.json has no fp64/fp32
 * figure).  Best of several launches over all SMs. */
int tb_measure_peak(tb_context *ctx, int precision, double *tflops);

/* Library build tag (sm_100a, git describe) */
const char *tb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TERSOFF_B200_H */
