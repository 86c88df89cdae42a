/* kwb200 -- B200-native PIC cycle behind a plain C ABI.
 *
 * The drop-in boundary for the kernelweave.pic hot path
 * (reference: /root/reference/pkg/src/kernelweave/pic/sim.py:134-176,
 * Simulation.step).  Each entry point replaces one or more stage kernel
 * objects the reference launches through kw/kernel.py:232 `launch()`:
 *
 *   kwb_particles_advance  <- GatherKernel + PushKernel + MoveKernel +
 *                             DepositKernel (+ ATOMICS.add_dense)
 *                             pic/kernels.py:341-412, kw/atomics.py:147-163
 *   kwb_particles_shift    <- migrate_particles   pic/particles.py:316-345
 *   kwb_particles_advance_species / kwb_particles_shift_species
 *                          <- the per-species particle loop of Simulation.step
 *                             pic/sim.py:141-163 (all species, one shift)
 *   kwb_zero_step          <- J[:] = 0            pic/sim.py:138-140
 *   kwb_fields_faraday_half / kwb_fields_ampere also serve the host helpers
 *                             yee_update_b / yee_update_e  pic/fields.py:127-143
 *   kwb_fields_faraday_half<- FaradayHalfKernel   pic/kernels.py:415-431
 *   kwb_fields_ampere      <- AmpereKernel        pic/kernels.py:434-450
 *   kwb_fields_gather      <- gather_fields       pic/fields.py:95-118
 *   kwb_charge_density     <- Simulation.charge_density / _rho_tsc
 *                             pic/sim.py:183-189, pic/kernels.py:291-326
 *   kwb_continuity_residual<- the validate block  pic/sim.py:168-175
 *   kwb_particle_moments / kwb_field_stats
 *                          <- Simulation.diagnostics pic/sim.py:191-225
 *   kwb_init_khi           <- init_khi (on-device path)  pic/sim.py:239-302
 *   kwb_store_load / kwb_store_export (+ _counted / kwb_store_extract)
 *                          <- _bulk_fill / SuperCellStore.packed
 *                             pic/sim.py:305-328, pic/particles.py:174-186
 *
 * Conventions
 *  - All device memory is owned by the caller (PyTorch tensors); the library
 *    never allocates.  Pointers are device pointers.
 *  - Every call is asynchronous on `stream` and returns 0 on success or a
 *    negative KWB_E* code; kwb_last_error() gives the message (thread-local).
 *  - Field arrays: logical (nx, ny, nz), stored x fastest:
 *    index = (k * ny + j) * nx + i.  Periodic in x, y and z.
 *  - Particle stores ("cell-column frames"): one per species.  With
 *    V = scx*scy*scz cells per super cell (= the frame capacity) and K
 *    frames per super cell, slot (s, k, c) = (s * K + k) * V + c holds the
 *    k-th particle of local cell c = lx + scx * (ly + scy * lz) of super
 *    cell s.  Column (s, c) is filled in frames [0, front) and [K-back, K);
 *    the cell of a particle is implied by its column.  A frame therefore
 *    holds one particle of every cell, so a warp reading frame k of 32
 *    adjacent cells issues fully coalesced 128-byte loads, and the thread
 *    that owns cell c sees only particles of cell c (register-resident
 *    current deposit).
 *  - Super-cell index s = bx + gx * (by + gy * bz) (pic/sim.py:79-84).
 *  - dtype KWB_F32 / KWB_F64 selects the storage type F; arithmetic follows
 *    the reference's mixed-precision recipe with no
 *    FMA contraction, so particle results are bitwise equal to the reference.
 */
#ifndef KWB200_H
#define KWB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KWB_VERSION 1

#define KWB_F32 0
#define KWB_F64 1

#define KWB_OK 0
#define KWB_EINVAL (-1)
#define KWB_ECUDA (-2)

/* status words written by the device (int32 array of KWB_STATUS_WORDS) */
#define KWB_ST_MOVE_ERRORS 0   /* particles that moved >= 1 cell (ContractViolation) */
#define KWB_ST_EXCH_OVERFLOW 1 /* leavers that did not fit the exchange buffer */
#define KWB_ST_STORE_OVERFLOW 2/* arrivals that did not fit their super cell */
#define KWB_ST_LEAVERS 3       /* leavers summed over species this step */
#define KWB_ST_MAX_COUNT 4     /* max particles in one cell column after the shift */
#define KWB_ST_LOAD_ERRORS 5   /* kwb_store_load records that did not fit */
#define KWB_ST_GUARD_OVERFLOW 6/* kwb_store_extract records beyond the message capacity */
#define KWB_STATUS_WORDS 8

typedef struct CUstream_st *kwb_stream_t;

typedef struct kwb_grid {
    int32_t nx, ny, nz;    /* cells */
    int32_t scx, scy, scz; /* super cell (frame capacity = scx*scy*scz) */
    int32_t gx, gy, gz;    /* super-cell grid = cells / super cell */
    int32_t dtype;         /* KWB_F32 or KWB_F64 */
    double dx, dy, dz, dt;
} kwb_grid;

typedef struct kwb_species {
    double qm_half_dt; /* q dt / (2 m)             pic/sim.py:101-103 */
    double fac[3];     /* -q delta_a / (dt V)      pic/sim.py:104-110 */
    double dt_d[3];    /* dt / delta_a             pic/sim.py:100 */
    double q_inv_vol;  /* q / V                    pic/sim.py:188 */
    double charge, mass;
} kwb_species;

typedef struct kwb_store {
    void *ox, *oy, *oz;   /* F: in-cell offsets in [0, 1] */
    void *ux, *uy, *uz;   /* F: momentum gamma v (units of c) */
    void *w;              /* F: macro-particle weight */
    int32_t *front;       /* [n_sc * V] column fill from frame 0 upward */
    int32_t *back;        /* [n_sc * V] column fill from frame K-1 downward */
    int32_t frames_per_sc;/* K: frames per super cell */
} kwb_store;

typedef struct kwb_exchange {
    void *ox, *oy, *oz, *ux, *uy, *uz, *w; /* F[capacity] */
    int32_t *cx, *cy, *cz;                 /* global cell after the move */
    int32_t *dest;                         /* destination super cell */
    int32_t *count;                        /* [1] device counter, zeroed by advance */
    int32_t capacity;
} kwb_exchange;

typedef struct kwb_init {
    int32_t ppc, px, py, pz;       /* quiet-start sub-lattice, ppc = px*py*pz (pic/sim.py:36-52) */
    double stream_velocity;        /* KHI v0 (pic/params.py:48) */
    double perturbation;           /* KHI v_y amplitude (pic/params.py:49) */
    double thermal_u;              /* N(0, thermal_u^2) per momentum component */
    double weight;                 /* macro-particle weight of the species */
    uint64_t seed;                 /* Philox key (with the species index) */
    int32_t species_index;
    int32_t x_offset, y_offset, z_offset; /* global cell of local cell 0 (z-slabs) */
    int32_t global_nx, global_ny;  /* global extents for the KHI profile */
} kwb_init;

int kwb_version(void);
const char *kwb_last_error(void);

/* Fused gather -> Boris push -> move -> Esirkepov deposit for one species.
 * One CTA per super cell, one thread per cell.  Reads store `in`; writes
 * particles that stay in their cell to the front of the same column of
 * `out`, particles that change cell inside the super cell to the back of
 * their new column, and leavers of the super cell into `ex`.  Accumulates
 * current into J (which the caller zeroes once per step).
 * shape_order: 1 CIC, 2 TSC (reference), 3 PCS. */
int kwb_particles_advance(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                          const kwb_store *out, const kwb_exchange *ex,
                          void *const E[3], void *const B[3], void *const J[3],
                          int shape_order, int32_t *status, kwb_stream_t stream);

/* kwb_particles_advance for one z-slab of a decomposed domain, with the J
 * guard-plane halo sum fused into the deposit flush.  j_planes: DEVICE array
 * of 3 * g->nz pointers (component-major); j_planes[c * nz + z] is the base
 * of the nx*ny plane (x fastest) that local plane z of J[c] is added to.
 * Owned planes point into J[c]; guard planes point into the z-neighbour's
 * halo receive buffer (same-process memory, a peer pointer or a CUDA-IPC
 * mapping), so no separate J halo message is sent.  NULL: plain J.
 * Replaces the deposit + J-halo send of the reference's per-stage launch
 * (pic/sim.py:138-163 DepositKernel; kw/atomics.py:147-163 atomic_add_dense
 * for the wrapped tile rows). */
int kwb_particles_advance_zslab(const kwb_grid *g, const kwb_species *sp,
                                const kwb_store *in, const kwb_store *out,
                                const kwb_exchange *ex, void *const E[3], void *const B[3],
                                void *const J[3], void *const *j_planes, int shape_order,
                                int32_t *status, kwb_stream_t stream);

/* Super-cell shift: append the leavers in `ex` to the back of their new
 * columns in `out` (restores "every particle lives in its owning super cell"). */
int kwb_particles_shift(const kwb_grid *g, const kwb_store *out, const kwb_exchange *ex,
                        int32_t *status, kwb_stream_t stream);

/* Yee updates (in place). */
int kwb_fields_faraday_half(const kwb_grid *g, void *const E[3], void *const B[3],
                            double half_dt, kwb_stream_t stream);
int kwb_fields_ampere(const kwb_grid *g, void *const E[3], void *const B[3],
                      void *const J[3], double dt, kwb_stream_t stream);

/* The particle phase of a step for all species of a Simulation (the
 * reference launches its particle kernels per species, pic/sim.py:141-163):
 * kwb_particles_advance_species advances every species -- two species in
 * ONE fused launch (lane-level species fusion), otherwise one launch per
 * species, all appending their super-cell leavers to the one exchange buffer
 * (dest = super cell + species * n_super_cells) -- and
 * kwb_particles_shift_species then appends every leaver to its species'
 * store in one launch.  sp/in/out: n_species (<= 4) entries; status:
 * n_species x KWB_STATUS_WORDS; j_planes as kwb_particles_advance_zslab
 * (NULL: plain J). */
int kwb_particles_advance_species(const kwb_grid *g, int32_t n_species, const kwb_species *sp,
                                  const kwb_store *in, const kwb_store *out,
                                  const kwb_exchange *ex, void *const E[3], void *const B[3],
                                  void *const J[3], void *const *j_planes, int shape_order,
                                  int32_t *status, kwb_stream_t stream);
int kwb_particles_shift_species(const kwb_grid *g, int32_t n_species, const kwb_store *out,
                                const kwb_exchange *ex, int32_t *status, kwb_stream_t stream);
/* The same particle phase with each species' advance split in two kernels:
 * a dense gather/push/move pass writing new offsets, momenta and cell
 * carries into the workspace store ws[i] (same frames_per_sc as in[i]; its
 * front/back are ignored), then the deposit + in-super-cell shift pass that
 * reads them.  Identical results to kwb_particles_advance_species; PCS
 * (shape_order 3) or ws == NULL falls through to it. */
int kwb_particles_advance_split(const kwb_grid *g, int32_t n_species, const kwb_species *sp,
                                const kwb_store *in, const kwb_store *out, const kwb_store *ws,
                                const kwb_exchange *ex, void *const E[3], void *const B[3],
                                void *const J[3], void *const *j_planes, int shape_order,
                                int32_t *status, kwb_stream_t stream);

/* Multi-GPU plumbing for the fused z-slab halo (pic/decomp.py): enable
 * access from the CURRENT device to peer_device (already enabled = OK), and
 * an asynchronous copy on the caller's stream (unified addressing; used for
 * the E/B guard-plane pulls from the neighbour's lattices). */
int kwb_enable_peer_access(int32_t peer_device);
int kwb_copy_async(void *dst, const void *src, int64_t bytes, kwb_stream_t stream);

/* Debug builds (make checks: -DKWB_CHECKS): number of failed bounds checks
 * in the kernels since the last reset (synchronises the device); -1 in a
 * normal build. */
int64_t kwb_check_failures(int32_t reset);

/* Start of a step: J = 0 (J may be NULL to skip) and n_status status words
 * = 0, in one kernel (pic/sim.py:138-140). */
int kwb_zero_step(const kwb_grid *g, void *const J[3], int32_t *status, int32_t n_status,
                  kwb_stream_t stream);

/* E and B at n points (global cells[3n], in-cell offsets[3n] as double),
 * out[6n] in the storage type: Ex Ey Ez Bx By Bz per point.  The advance
 * kernel's gather recipe (pic/kernels.py:26-77).  Replaces the reference's
 * host helper gather_fields (pic/fields.py:95-118). */
int kwb_fields_gather(const kwb_grid *g, void *const E[3], void *const B[3], int64_t n,
                      const int32_t *cells, const double *offsets, void *out,
                      kwb_stream_t stream);

/* Validation charge density (float64, accumulated, caller zeroes rho). */
int kwb_charge_density(const kwb_grid *g, const kwb_species *sp, const kwb_store *st,
                       int shape_order, double *rho, kwb_stream_t stream);

/* out[0] = max |(rho_new - rho_prev)/dt + div J| (div J in storage type,
 * as numpy computes it, pic/fields.py:154-160); out[1] = max |G - G_prev|
 * with G = div E - rho_new (G_prev updated in place; pass NULL to skip). */
int kwb_continuity_residual(const kwb_grid *g, const double *rho_new, const double *rho_prev,
                            void *const J[3], void *const E[3], double *G_prev,
                            double *out, kwb_stream_t stream);

/* out[0] += census, out[1] += sum q w, out[2] += sum m (gamma-1) w (float64). */
int kwb_particle_moments(const kwb_grid *g, const kwb_species *sp, const kwb_store *st,
                         double *out, kwb_stream_t stream);

/* out[0] = sum over cells of E^2 + B^2 (float64), out[1] = max |div B|. */
int kwb_field_stats(const kwb_grid *g, void *const E[3], void *const B[3], double *out,
                    kwb_stream_t stream);

/* Append n particle records (global cells cx/cy/cz, 7 F arrays, any order)
 * to their columns; front/back must be valid (zero for an empty store). */
int kwb_store_load(const kwb_grid *g, const kwb_store *st, int64_t n,
                   const int32_t *cx, const int32_t *cy, const int32_t *cz,
                   void *const f7[7], int32_t *status, kwb_stream_t stream);

/* Export the particles of columns [col_begin, col_end) in canonical order
 * (super cell, then local cell, then frame); cell_start[i] = output offset of
 * column col_begin + i (exclusive scan of front + back).  Writes global
 * cells and the 7 F arrays.  clear != 0 empties the exported columns (the
 * z-slab decomposition extracts guard-layer leavers this way; a z-layer of
 * super cells is a contiguous column range). */
int kwb_store_export(const kwb_grid *g, const kwb_store *st, int64_t col_begin, int64_t col_end,
                     const int64_t *cell_start, int clear, int32_t *cx, int32_t *cy, int32_t *cz,
                     void *const f7[7], kwb_stream_t stream);

/* Bounded, host-synchronisation-free form of kwb_store_export with clear:
 * if the range holds at most `capacity` records (total read on the device
 * from cell_start[col_end - col_begin]) they are exported and the columns
 * emptied, and *count_out (device) = the total; otherwise nothing is
 * exported or cleared, *count_out = 0 and status[KWB_ST_GUARD_OVERFLOW]
 * counts the excess.  The z-slab decomposition ships guard-layer particles
 * in fixed-capacity messages this way. */
int kwb_store_extract(const kwb_grid *g, const kwb_store *st, int64_t col_begin,
                      int64_t col_end, const int64_t *cell_start, int64_t capacity,
                      int32_t *cx, int32_t *cy, int32_t *cz, void *const f7[7],
                      int64_t *count_out, int32_t *status, kwb_stream_t stream);

/* kwb_store_load with the record count on the device: appends
 * min(*n_dev, capacity) records. */
int kwb_store_load_counted(const kwb_grid *g, const kwb_store *st, const int64_t *n_dev,
                           int64_t capacity, const int32_t *cx, const int32_t *cy,
                           const int32_t *cz, void *const f7[7], int32_t *status,
                           kwb_stream_t stream);

/* On-device KHI/thermal start (pic/sim.py:239-302 semantics, Philox jitter):
 * fills every cell column with the ppc quiet-start particles of the species.
 * The store's front/back are set; frames_per_sc must be >= ppc. */
int kwb_init_khi(const kwb_grid *g, const kwb_init *ini, const kwb_store *st,
                 kwb_stream_t stream);

/* Copy every column into a store with a different frames_per_sc
 * (capacity growth). */
int kwb_store_repack(const kwb_grid *g, const kwb_store *src, const kwb_store *dst,
                     kwb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KWB200_H */
