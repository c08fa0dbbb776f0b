/*
 * adjamr_b200.h -- C ABI of the B200-native hot path of adjoint-guided
 * block-structured AMR (arxiv 1511.03645, reference package `adjamr`).
 *
 * Every entry point is stream-ordered, borrows caller-owned DEVICE pointers
 * (the Python host layer passes torch tensors' data_ptr()), and returns an
 * int status.  No torch or C++ types cross this boundary.
 *
 * The reference is pure Python/numpy and has no FFI of its own; each entry
 * point below names the reference function(s) it replaces (paths relative to
 * /root/reference/pkg/src/adjamr/).  INTEGRATION.md shows the ctypes binding
 * that the reference-side Python would add.
 *
 * Data layout in HBM (one "level store" per refinement level):
 *   q   : m component planes, component c of patch p, ghost-inclusive local
 *         cell (ii, jj) lives at q[c*comp_stride + p.offset + ii*p.pitch + jj].
 *         y (jj) is the contiguous axis, exactly like the reference's numpy
 *         `Patch.state` of shape (m, nx+2g, ny+2g) (geometry.py:109).
 *         In 1D the patch is a single column: ny = 1, pitch = 1.
 *   aux : naux material planes with the same per-patch offsets/pitch,
 *         plane stride aux_stride.  Acoustics: {c, z, rho, bulk};
 *         shallow water: {c, depth} (wet <=> depth > 0)  (equations.py:32-74).
 */
#ifndef ADJAMR_B200_H
#define ADJAMR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADJ_ABI_VERSION 8

/* status codes (mapped to the reference's exception classes by the host) */
#define ADJ_OK                 0
#define ADJ_ERR_CFL            1   /* solver.CflViolationError      solver.py:23  */
#define ADJ_ERR_NONFINITE      2   /* solver.NumericalBlowupError   solver.py:27  */
#define ADJ_ERR_SCHEDULING     3   /* solver.SchedulingError        solver.py:31  */
#define ADJ_ERR_OUT_OF_RANGE   4   /* geometry.OutOfRangeError      geometry.py:18 */
#define ADJ_ERR_BAD_ARG        5   /* ValueError                                   */
#define ADJ_ERR_CUDA          -1

/* equation systems (equations.py:423-493) */
#define ADJ_SYS_AC1D   0   /* Acoustics1D / AdjointAcoustics1D   */
#define ADJ_SYS_AC2D   1   /* Acoustics2D / AdjointAcoustics2D   */
#define ADJ_SYS_SWE2D  2   /* SweLinear2D / AdjointSweLinear2D   */

/* Riemann-solver form (EquationSet.form, equations.py:397, 464) */
#define ADJ_FORM_WAVE   0
#define ADJ_FORM_FWAVE  1

/* limiters (solver.py:20, 65-77) */
#define ADJ_LIM_NONE      0
#define ADJ_LIM_MINMOD    1
#define ADJ_LIM_MC        2
#define ADJ_LIM_SUPERBEE  3

/* step-kernel variants */
#define ADJ_VARIANT_EXACT 0   /* reference expression order, no FMA: bitwise parity */
#define ADJ_VARIANT_FAST  1   /* register-marching strip kernel, <=1e-12 norm-relative */

/* patch-edge bits of AdjPatch.edges (which sides meet the physical domain) */
#define ADJ_EDGE_XLO 1
#define ADJ_EDGE_XHI 2
#define ADJ_EDGE_YLO 4
#define ADJ_EDGE_YHI 8

/* boundary kinds per side (solver.BoundarySpec, solver.py:35-56) */
#define ADJ_BC_WALL    0
#define ADJ_BC_OUTFLOW 1
#define ADJ_BC_PERIODIC 2   /* extension (BASELINE C3): ghosts wrap to the opposite interior; both
                               sides of the axis periodic and every patch spanning the axis */

/* One patch of a level store (device-resident table). */
typedef struct AdjPatch {
    int64_t offset;      /* element offset of ghost-corner cell (0,0) in every plane */
    int64_t flag_word;   /* first uint32 word of this patch's flag bits (K3)          */
    int32_t nx, ny;      /* interior extents (ny = 1 in 1D)                            */
    int32_t pitch;       /* elements between consecutive x rows                        */
    int32_t lo_x, lo_y;  /* global index of the interior lower corner                  */
    int32_t edges;       /* ADJ_EDGE_* bits                                            */
    int32_t pad0, pad1;
} AdjPatch;

/* One unit of step work: an interior box [i0,i0+ni) x [j0,j0+nj) of a patch. */
typedef struct AdjTile {
    int32_t patch, i0, j0, ni, nj, pad;
} AdjTile;

/* Rectangle of ghost cells (K2 rect fills and plans; K4 overlaps). */
#define ADJ_RECT_COPY        0   /* dst cells <- src patch cells (same level)          */
#define ADJ_RECT_COARSE      1   /* dst cells <- bilinear/linear-in-time coarse interp */
typedef struct AdjRect {
    int32_t kind;
    int32_t dst_patch, src_patch;
    int32_t di0, dj0;     /* dst start, ghost-inclusive local coords           */
    int32_t ni, nj;       /* extent                                            */
    int32_t si0, sj0;     /* src start (COPY), ghost-inclusive local coords    */
    int32_t pad;
} AdjRect;

/* K2, planned form of a whole level fill (fill_level_ghosts, amr.py:479-491:
 * coarse interpolation, same-level copy, then physical boundaries) as ONE
 * gather launch.  The plan is built once per regrid on the device from the
 * level's disjoint COARSE + COPY rectangles (COARSE rects first) and its
 * boundary patches; every ghost cell the fill writes gets one entry.
 * Out-of-domain (physical) cells are resolved at build time to the entry
 * (or interior cell) their mirrored / extrapolated source ends up holding
 * (solver.py:84-146 applied after the in-domain phases), with the normal
 * component's sign flips as a bit mask, so the fill has no ordering
 * between entries.  Values are bitwise those of the three phases. */
typedef struct AdjGhostPlan {
    int32_t* dst;                /* [n] destination offset in the fine level plane               */
    int32_t* src;                /* [n] COPY: source offset (same plane); COARSE: coarse entry   */
    uint32_t* meta;              /* [n] bit 0: COARSE; bit 1+c: negate component c               */
    int32_t* c_base;             /* [nc] offset of (i0, j0) in the coarse level plane            */
    int32_t* c_step;             /* [nc] (i1-i0)*pitch | (j1-j0) << 30                          */
    double* c_wx;                /* [nc] x weight (geometry.py:248-260)                          */
    double* c_wy;                /* [nc] y weight (2D)                                           */
    int32_t n;                   /* entries                                                      */
    int32_t nc;                  /* COARSE rect cells = entries [0, nc), src == own index        */
} AdjGhostPlan;
typedef struct AdjGhostPlanBuildArgs {
    AdjGhostPlan plan;           /* arrays sized by the caller; n = rect cells + physical cells  */
    const AdjRect* rects;        /* COARSE rects first, then COPY rects (disjoint)               */
    const int32_t* rect_cell0;   /* [nrect+1] first entry of each rect (prefix of ni*nj)         */
    const AdjPatch* patches;     /* fine level table                                             */
    const AdjPatch* coarse_patches;
    const double* axis_w;        /* per-rect axis tables as in AdjGhostArgs                      */
    const int32_t* axis_i;
    const AdjPatch* edge_patches;/* fine patches touching the domain boundary (edges set)        */
    int32_t* owner;              /* [plane] scratch filled with -1 (entry writing each cell)     */
    int32_t* counter;            /* one int, zeroed: physical entries are appended after it      */
    int32_t nrect, rect_cells;   /* rect_cells = rect_cell0[nrect]: physical entries start here  */
    int32_t nedge, ndim, m;
    int32_t ghost, ghost_coarse, max_ghost_cells;
    int32_t bc[4];               /* x-lo, x-hi, y-lo, y-hi: ADJ_BC_*                             */
    int32_t normal_comp[2];
    void* stream;
} AdjGhostPlanBuildArgs;
int adj_ghost_plan_build(const AdjGhostPlanBuildArgs* a);
typedef struct AdjGhostPlanFillArgs {
    AdjGhostPlan plan;
    double* q;                   /* fine level state (COPY sources are read from it too)         */
    const double* q_coarse_old;  /* coarse state at t0 / t1 (may be NULL when nc == 0)           */
    const double* q_coarse_new;
    int64_t comp_stride, coarse_comp_stride;
    int32_t ndim, m, time_mode, pad;
    double w_time;
    const double* w_time_dev;    /* optional device weight (< 0: old only), as in AdjGhostArgs  */
    void* stream;
} AdjGhostPlanFillArgs;
int adj_fill_ghost_plan(const AdjGhostPlanFillArgs* a);

/* Restriction fused into the step of the finest level's last substep
 * (restrict_fine_to_coarse, amr.py:399-450): every r x r block of new fine
 * interior values is averaged into its covered coarse cell as the strip
 * march produces it.  cell[base[patch] + (x/r) * (ny/r) + y/r] is the coarse
 * cell's offset in the coarse plane (-1: not covered).  FAST 2D only, every
 * tile's i0, j0, ni, nj a multiple of r; sum order differs from numpy's (the
 * FAST tolerance). */
typedef struct AdjStepRestrict {
    double* q_coarse;            /* coarse level state written (cur)                              */
    const int32_t* cell;         /* per fine r x r block: coarse cell offset or -1                */
    const int32_t* base;         /* per fine patch: its first block in cell                       */
    int64_t coarse_comp_stride;
    int32_t ratio, pad;          /* ratio 2 or 4; 0: no fused restriction                          */
} AdjStepRestrict;

/* Level ghost fill fused into the step, per warp job (FAST 2D static-CFL
 * path): the level's planned fill (AdjGhostPlan entries, same values) is
 * regrouped by the step's warp jobs; before a job marches, its lanes fill the
 * ghost cells its strips read (entries [entry_off[job], entry_off[job+1]))
 * into q_in.  Entries of two jobs that overlap write identical values.  No
 * grid barrier: every source (same-level interiors, the coarse level) was
 * written by earlier launches.  COARSE entries carry their stencil inline.
 * cache_mode 1 also stores the entry's space-interpolated coarse values at
 * t0 and t1 (interpolate_patch on state_old / state, geometry.py:302-327) in
 * cache[c * n + e] (c < m: old, m + c: new); cache_mode 2 reads them instead
 * of the coarse level: the later substeps of one coarse interval reuse them,
 * which also keeps them off coarse cells a fused restriction rewrites. */
typedef struct AdjJobFill {
    const int32_t* entry_off;    /* [njob + 1] first entry of each warp job                      */
    const int32_t* dst;          /* [n] ghost cell offset in the level plane                      */
    const int32_t* src;          /* [n] COPY / physical: source offset in the level plane         */
    const uint32_t* meta;        /* [n] bit 0: COARSE; bit 1+c: negate component c                */
    const int32_t* c_base;       /* [n] COARSE: offset of (i0, j0) in the coarse level plane      */
    const int32_t* c_step;       /* [n] COARSE: (i1-i0)*pitch | (j1-j0) << 30                     */
    const double* c_wx;          /* [n] COARSE: x weight                                          */
    const double* c_wy;          /* [n] COARSE: y weight                                          */
    double* cache;               /* [2 m n] coarse values at t0 and t1, or NULL                   */
    const double* q_coarse_old;  /* coarse state at t0 / t1                                       */
    const double* q_coarse_new;
    int64_t coarse_comp_stride;
    int32_t n, cache_mode;       /* entries; 0: interpolate, 1: interpolate + store, 2: read cache */
    int32_t time_mode, pad;      /* 0: old only, 1: blend, 2: new only (as AdjGhostPlanFillArgs)  */
    double w_time;
    const double* w_time_dev;    /* optional device weight (< 0: old only)                        */
} AdjJobFill;

/* K1: wave-propagation step of every patch of a level.
 * Replaces step_patch / step_patch_1d / step_patch_2d (solver.py:415-522), the
 * Riemann and transverse solvers (equations.py:98-349), TimeReversed
 * (equations.py:496-534) and the limiter (solver.py:65-77, 317-348).
 * Reads q_in (ghosts filled), writes the interior of q_out (ping-pong buffers
 * replace Patch.save_old, geometry.py:123).  Outputs per patch: the maximum
 * |speed| over the reference's CFL interface ranges, x and y separately
 * (solver.py:425, 457-460), and a non-finite flag (solver.py:437, 510). */
typedef struct AdjStepArgs {
    const double* q_in;
    double* q_out;
    const double* aux;
    const AdjPatch* patches;   /* device */
    const AdjTile* tiles;      /* device */
    double* speed_max;         /* device, 2*npatch (x, y), zeroed by the call */
    int32_t* nonfinite;        /* device, npatch, zeroed by the call; 1: non-finite result,
                                  2: an EXACT tile larger than adj_step_tile_shape (not stepped) */
    int32_t* work_counter;     /* device, 2 ints (tile queue head, exit count), zeroed by the call
                                  unless ADJ_STEP_COUNTER_ZERO */
    const double* static_speed;/* optional device (x, y) per patch: material speed bound over the
                                  CFL ranges; when given, the FAST variant (no dry cells) copies it
                                  to speed_max instead of reducing per face (same values) */
    const int32_t* job_offsets;/* optional (FAST + static_speed): warp job j = tiles[job_offsets[j],
                                  job_offsets[j+1]); each tile of a job is a row strip placed at
                                  lanes [pad, pad + nj + 4) of the warp, all with the same ni */
    int32_t njob, pad2;
    int64_t comp_stride, aux_stride;
    int32_t npatch, ntile;
    int32_t ndim, ghost;
    int32_t system, form, reversed, limiter, variant, flags;   /* ADJ_STEP_* bits */
    double dt, dtdx, dtdy, gravity;
    void* stream;              /* cudaStream_t */
    AdjGhostPlanFillArgs prefill;  /* optional (prefill.plan.n > 0; FAST 2D with static_speed and
                                  ADJ_STEP_COUNTER_ZERO): the level's planned ghost fill of q_in runs
                                  inside this launch before the step (a grid barrier separates them);
                                  work_counter then holds 3 zeroed ints */
    AdjStepRestrict fine_restrict; /* optional (ratio > 0): restriction into the coarse level fused
                                  into this step (FAST 2D, static_speed, forward wave form) */
    AdjJobFill job_fill;       /* optional (job_fill.n > 0): the level's ghost fill per warp job
                                  (FAST 2D, static_speed, job_offsets, ADJ_STEP_COUNTER_ZERO, no prefill) */
    int32_t phys_bc[4];        /* ADJ_STEP_PHYS_IN: x-lo, x-hi, y-lo, y-hi ADJ_BC_* of the domain sides  */
    int32_t phys_normal[2];    /* component negated at an x / a y wall                                     */
    const int8_t* job_class;   /* optional with ADJ_STEP_WET_DRY (device, njob or ntile): 0 every cell of
                                  the job's strip windows wet (the all-wet march), 1 mixed (the wet/dry
                                  march), 2 every output cell dry (outputs copied: dq *= wet)              */
    double uniform_c, uniform_z;/* ADJ_STEP_UNIFORM_MAT: the aux planes' (c, z) of every cell, ghosts included */
    const double* job_uniform; /* optional with ADJ_STEP_UNIFORM_MAT (device, 2 per warp job or tile): the
                                  (c, z) every cell read by the job's strips holds (rows j0-2 .. j0+nj+1,
                                  columns i0-2 .. i0+ni+1 of each strip), or (0, 0) for a job that reads
                                  several materials (it marches per cell); replaces uniform_c / uniform_z */
} AdjStepArgs;
/* AdjStepArgs.flags */
#define ADJ_STEP_KEEP_NONFINITE 1   /* do not zero nonfinite: accumulate over launches */
#define ADJ_STEP_NO_SPEED_OUT   2   /* do not write speed_max (caller uses static_speed) */
#define ADJ_STEP_TWO_ROWS       4   /* FAST + static_speed: tiles are 64-row strips (<= 60 outputs),
                                       two rows per lane; no job_offsets */
#define ADJ_STEP_COUNTER_ZERO   8   /* FAST 2D: work_counter holds 2 ints that are zero on entry; the
                                       kernel leaves them zero (no memset node per launch) */
#define ADJ_STEP_PHYS_IN       16   /* FAST 2D static CFL, one patch spanning the level: the launch
                                       first performs fill_ghost_physical (solver.py:125-146) on q_in --
                                       each warp job writes the physical ghost cells its strip reads,
                                       sources from q_in's interior (side rules from phys_bc; corners x
                                       then y; nx, ny >= 2) -- so no separate fill launch precedes the
                                       step */
#define ADJ_STEP_WET_DRY       32   /* FAST, shallow water with dry cells (SweLinear2D forward wave
                                       form, or its adjoint as the time-reversed f-wave form), static
                                       CFL bound: wet <=> aux c > 0; a dry side of a face
                                       takes the wet side's state (normal momentum negated) and material,
                                       both-dry faces carry no waves, corrections only on wet-wet faces,
                                       transverse materials of dry cells at unit depth, dry cells keep
                                       their state (_swe_effective_states / _swe_transverse_material /
                                       dq *= wet, solver.py:357-387, 500-505); without this flag a FAST
                                       step assumes every cell wet */
#define ADJ_STEP_UNIFORM_MAT   64   /* hint, FAST 2D acoustics (forward wave form, static CFL bound): every
                                       cell of aux (ghosts included) holds c = uniform_c, z = uniform_z, so
                                       the material terms of the march (sample_patch_material's arrays,
                                       solver.py:180-205, as the Riemann and transverse solvers use them) are
                                       computed once per strip instead of per cell -- same operations on the
                                       same values; with job_uniform the material is given per warp job
                                       (piecewise-constant media: jobs away from the interfaces); other
                                       configurations ignore the flag and read aux */
int adj_step_level(const AdjStepArgs* a);

/* Tile shape (ni, nj) the given variant expects in AdjStepArgs.tiles. */
int adj_step_tile_shape(int variant, int ndim, int32_t* ni, int32_t* nj);

/* K2 (physical phase): wall / outflow ghost fill of every patch edge that
 * meets the domain boundary.  Replaces fill_ghost_physical (solver.py:125-146)
 * with its x-then-y, low-then-high slab order folded into one gather. */
typedef struct AdjPhysArgs {
    double* q;
    const AdjPatch* patches;   /* device */
    int64_t comp_stride;
    int32_t npatch, ndim, ghost, m;
    int32_t bc[4];             /* left, right, bottom, top: ADJ_BC_*          */
    int32_t normal_comp[2];    /* component negated at a wall, per axis      */
    int32_t max_ghost_cells;   /* max ghost cells of any patch (grid sizing) */
    int32_t pad;
    void* stream;
} AdjPhysArgs;
int adj_fill_physical(const AdjPhysArgs* a);

/* K2 (in-domain phase): same-level copies and coarse-to-fine space-time
 * interpolation over rectangles of ghost cells.  Replaces
 * fill_ghost_from_coarse + space_time_interp (solver.py:227-286),
 * interpolate_patch (geometry.py:302-327) and fill_ghost_same_level
 * (solver.py:208-224); rectangles are built on the host once per regrid.
 * Also used for regrid data movement (amr.py:504-551, kind 2/3). */
typedef struct AdjGhostArgs {
    double* q_dst;               /* destination level store                        */
    const double* q_src;         /* COPY source level store (may == q_dst)          */
    const double* q_coarse_old;  /* COARSE: coarse level state at t0                */
    const double* q_coarse_new;  /* COARSE: coarse level state at t1                */
    const AdjPatch* dst_patches; /* device */
    const AdjPatch* src_patches; /* device, COPY sources                            */
    const AdjPatch* coarse_patches; /* device, COARSE sources                       */
    const AdjRect* rects;        /* device; COPY and COARSE rects may be mixed when disjoint */
    int64_t dst_comp_stride, src_comp_stride, coarse_comp_stride;
    int32_t nrect, ndim, m, ghost_dst, ghost_src, ratio;
    double origin_x, origin_y;   /* hierarchy.origin                              */
    double dx_f, dy_f;           /* fine widths                                   */
    double dx_c, dy_c;           /* coarse widths                                 */
    double w_time;               /* clip((t-t0)/(t1-t0),0,1)                      */
    const double* w_time_dev;    /* optional: read w from device memory (graph replay) */
    const double* axis_w;        /* optional per-rect axis weights: COARSE rect r has its ni x-weights at
                                    axis_w[rect.pad], then its nj y-weights (geometry.py:248-260) */
    const int32_t* axis_i;       /* matching lower stencil indices (same layout)               */
    int32_t time_mode;           /* 0: old only, 1: blend old/new, 2: new only    */
    int32_t max_rect_cells;
    void* stream;
} AdjGhostArgs;
int adj_fill_ghost_rects(const AdjGhostArgs* a);


/* K4: conservative fine-to-coarse averaging.  Replaces
 * restrict_fine_to_coarse (amr.py:399-450); one AdjRect per (coarse patch,
 * fine patch) overlap, in COARSE interior-local coordinates (di0,dj0 coarse,
 * si0,sj0 the matching fine interior-local start). */
typedef struct AdjRestrictArgs {
    double* q_coarse;
    const double* q_fine;
    const double* aux_coarse;    /* swe: depth plane 1 -> wet mask            */
    const double* aux_fine;
    const AdjPatch* coarse_patches;
    const AdjPatch* fine_patches;
    const AdjRect* rects;
    int64_t coarse_comp_stride, fine_comp_stride;
    int64_t coarse_aux_stride, fine_aux_stride;
    int32_t nrect, ndim, m, ratio, swe, max_rect_cells;
    int32_t ghost_coarse, ghost_fine;
    /* optional planned form (built per regrid): one entry per covered coarse
       cell, used instead of rects when cell_dst != NULL */
    const int32_t* cell_dst;     /* coarse cell offset in the coarse plane                        */
    const int32_t* cell_src;     /* offset of its first fine child in the fine plane              */
    const int32_t* cell_meta;    /* bit 0: numpy flat order (overlap box one cell wide in y);
                                    bits 1..: fine patch pitch                                    */
    int32_t ncell, pad;
    void* stream;
} AdjRestrictArgs;
int adj_restrict(const AdjRestrictArgs* a);

/* K3: adjoint inner-product flagging.  Replaces inner_product_field /
 * inner_product_flags / AdjointFlagging.evaluate (adjoint.py:227-277),
 * interpolate_uniform (geometry.py:248-290) and _adjoint_dry_at
 * (adjoint.py:217-224).  The snapshot ring holds nsnap fields of shape
 * (m, nxa, nya) contiguous; snap_index lists the window's snapshots
 * (query_window_times, adjoint.py:192-214, evaluated on the host).
 * mode 0: reference windowed max over the listed snapshots.
 * mode 1: linear-in-time interpolation (AdjointSnapshotStore.interpolate_time,
 *         adjoint.py:98-110) at each entry of interp_times, blended from
 *         snapshots interp_k[n] and interp_k[n]+1 with weight interp_w[n]
 *         (interp_k < 0: use snapshot -interp_k-1 unblended). */
#define ADJ_FLAG_ROWS 1
#define ADJ_FLAG_PAIRS 2   /* with ADJ_FLAG_ROWS: every even-aligned column pair of every patch
                              shares its adjoint stencil column (ratio >= 4 on aligned grids) */
#define ADJ_FLAG_QUADS 4   /* with ADJ_FLAG_PAIRS: every even-aligned row pair shares its adjoint
                              stencil row too, and every patch has an even number of rows */
#define ADJ_FLAG_DIRECT 8  /* with ADJ_FLAG_ROWS: every interpolation weight is exactly 0 or 1
                              (forward cell centres on adjoint cell centres, e.g. equal grids):
                              the bilinear stencil reduces to one adjoint value per cell */
typedef struct AdjFlagArgs {
    const double* q;             /* forward level store                        */
    const double* aux;           /* forward aux (swe: depth plane 1)          */
    const AdjPatch* patches;     /* device */
    const double* ring;          /* device, nsnap*m*nxa*nya                    */
    const uint8_t* adj_wet;      /* device nxa*nya, or NULL                    */
    const int32_t* snap_index;   /* device, nidx (mode 0) / interp_k (mode 1) */
    const double* interp_w;      /* device, nidx (mode 1)                      */
    uint32_t* flag_bits;         /* device, bit-packed per patch (flag_word)   */
    unsigned long long* counts;  /* device, npatch raw flagged counts          */
    double* best;                /* device, per-interior-cell values or NULL  */
    const int64_t* best_offset;  /* device, per patch start into best, or NULL */
    int32_t* status;             /* device, 1 int: ADJ_ERR_OUT_OF_RANGE bits  */
    const double* axis_w;        /* optional per-patch row (x) then column (y) weights into the
                                    adjoint grid (interpolate_uniform arithmetic, host-precomputed);
                                    patch k's rows start at axis_off[2k], columns at axis_off[2k+1] */
    const int32_t* axis_i;       /* matching lower stencil indices                               */
    const int32_t* axis_dry;     /* matching _adjoint_dry_at cell indices (SWE), or NULL         */
    const int64_t* axis_off;     /* 2 per patch                                                  */
    int64_t comp_stride, aux_stride;
    int32_t npatch, ndim, m, ghost, swe, mode, nidx, nxa, nya, max_cells;
    int32_t layout;              /* ADJ_FLAG_ROWS: every patch row is a multiple of 128 cells and
                                    nxa, nya >= 2 (row-layout kernel for single-snapshot windows) */
    int32_t max_rows, max_cols;  /* ADJ_FLAG_ROWS: largest patch nx, ny                            */
    int32_t variant;             /* ADJ_VARIANT_EXACT: the reference's arithmetic (bitwise flags);
                                    ADJ_VARIANT_FAST: windows of >= 2 snapshots interpolate with
                                    per-cell corner weights and FMAs (inner products within ~1e-16
                                    relative; flags identical except within 1e-12 of the tolerance) */
    double origin_x, origin_y, dx, dy;             /* forward level geometry   */
    double a_origin_x, a_origin_y, a_dx, a_dy;     /* adjoint grid geometry    */
    double tolerance;
    double* envelope;            /* optional scratch of 6*nxa*nya doubles.  With best == NULL and
                                    tolerance > 1e-280 the call first writes the window's envelope
                                    max_k |snapshot_k| per adjoint node and component (planes 3..5)
                                    and its max over each bilinear stencil (planes 0..2); a cell
                                    whose bound sum_c |q_c| E_c (1 + 1e-12) is <= tolerance cannot
                                    be flagged (|qhat_c| <= E_c for the bilinear and time-linear
                                    weights) and skips its window.  Flags and counts are unchanged
                                    (quad-layout windows of >= 2 snapshots).                      */
    int32_t* work;               /* with envelope: scratch of 2 + 4 * (blocks of 2 rows x 64 columns)
                                    ints, the list of blocks that may exceed the tolerance          */
    void* stream;
} AdjFlagArgs;
int adj_flag_adjoint(const AdjFlagArgs* a);

/* Output path, on the device so only scalars / gauge values
 * cross to the host at output times.
 *
 * evaluate_J (adjoint.py:299-336) over one level: per interior cell not
 * covered by a finer patch (_uncovered_mask, adjoint.py:280-296) the signed
 * inner product sum_c qhat_c q_c with qhat = interpolate_uniform of the
 * store interpolated in time (interpolate_time, adjoint.py:98-110; the same
 * per-cell arithmetic as K3).  Per-block sums go to partial[patch *
 * blocks_x + block] (fixed order); the host multiplies each patch's sum by
 * the cell area and accumulates in patch order as the reference does. */
typedef struct AdjFunctionalArgs {
    const double* q;             /* forward level store                                          */
    const AdjPatch* patches;     /* device, the level's patches                                  */
    const double* ring;          /* snapshots (nsnap, m, nxa, nya)                               */
    const AdjPatch* finer;       /* optional: next finer level's patches (covered cells)         */
    uint8_t* covered;            /* scratch level_nx * level_ny bytes when finer != NULL          */
    double* partial;             /* [npatch * blocks_x]                                          */
    int32_t* status;             /* 1 int, zeroed: 1 = point outside the adjoint grid            */
    int64_t comp_stride;
    int32_t npatch, nfiner, ratio, ndim, m, ghost;
    int32_t nxa, nya, level_nx, level_ny, blocks_x, snap;   /* snap < 0: snapshot -snap-1;
                                                               else blend snap, snap+1 with w */
    double w;
    double origin_x, origin_y, dx, dy;          /* the level's geometry           */
    double a_origin_x, a_origin_y, a_dx, a_dy;  /* the adjoint grid's geometry    */
    void* stream;
} AdjFunctionalArgs;
int adj_functional(const AdjFunctionalArgs* a);

/* Gauges (record_gauge, runio.py:217-226): interpolate_patch with
 * interior_only (geometry.py:302-327) for ngauge points at once.  Per gauge
 * the host gives the patch's interior corner offset and pitch and the
 * stencil (i0, i1, j0, j1, wx, wy) from _axis_weights; out[g*m + c]. */
typedef struct AdjGauge {
    int64_t base;                /* offset of interior cell (0, 0) in the level plane */
    int32_t pitch, i0, i1, j0, j1, pad;
    double wx, wy;
} AdjGauge;
typedef struct AdjGaugeArgs {
    const double* q;
    const AdjGauge* gauges;      /* device */
    double* out;                 /* device, ngauge * m */
    int64_t comp_stride;
    int32_t ngauge, ndim, m, pad;
    void* stream;
} AdjGaugeArgs;
int adj_gauges(const AdjGaugeArgs* a);

/* K5: regrid flag post-processing on the device.  Replaces, for one parent
 * level, the per-patch region overrides of flag_cells (amr.py:137-154), the
 * box dilation of buffer_flags clipped to each patch (amr.py:157-179), the OR
 * into the level mask and the proper-nesting clip by the one-cell erosion of
 * the level's occupancy with edge padding (allowed_region_mask,
 * geometry.py:341-368; amr.py:580-581).  Input: K3's packed flags.  Output:
 * one byte per cell of the level index space (x-major, level_ny contiguous):
 * bit 0 = clipped flag, bit 1 = allowed; only this mask goes to the host
 * clusterer.  raw_count = flags after region overrides (amr.py:575). */
typedef struct AdjFlagMaskArgs {
    const uint32_t* flag_bits;   /* K3 flag words (AdjPatch.flag_word, row-major interior)          */
    const AdjPatch* patches;     /* parent level */
    const uint8_t* region_rows;  /* optional: bit k = row centre inside region k's x range          */
    const uint8_t* region_cols;  /*           bit k = column centre inside region k's y range       */
    const int32_t* region_row_off;  /* [npatch] first row entry of each patch                       */
    const int32_t* region_col_off;  /* [npatch] first column entry of each patch                    */
    uint8_t* mask;               /* level_nx * level_ny bytes, fully written                        */
    uint8_t* occupancy;          /* scratch, level_nx * level_ny bytes                               */
    unsigned long long* raw_count;  /* one counter, zeroed by the call                              */
    int32_t npatch, ndim, level_nx, level_ny, buffer, max_cells;
    uint32_t force_regions;      /* regions active at t with level+1 <= min_level (flags |= region) */
    uint32_t clear_regions;      /* regions active at t with level+1 >  max_level (flags &= ~region) */
    void* stream;
} AdjFlagMaskArgs;
int adj_flag_level_mask(const AdjFlagMaskArgs* a);

/* Host (no GPU): signature-bisection clustering of a flag mask, identical
 * to cluster() (amr.py:244-309).  mask: uint8 (nx, ny) row-major (ny = 1 in
 * 1D); max_edge <= 0: no cap.  boxes: 4 ints per box (lo_x, lo_y, hi_x,
 * hi_y) in emission order, effs: efficiency per box.  Returns
 * ADJ_ERR_BAD_ARG (nboxes = -1) when max_boxes is too small. */
int adj_cluster(const uint8_t* mask, int ndim, int nx, int ny, double efficiency, int max_edge,
                int32_t* boxes, double* effs, int max_boxes, int32_t* nboxes);

/* Last CUDA error string of the calling thread (diagnostics). */
const char* adj_last_error(void);
/* Host (no GPU): ghost-fill rectangles of one level, identical to
 * build_ghost_rects (the per-patch phases of fill_ghost_same_level /
 * fill_ghost_from_coarse, solver.py:208-263, as rectangles).  Boxes are
 * inclusive global (lo, hi), ndim ints each; coarse boxes in the coarse
 * index space (ratio to this level).  For every patch (or only patch `only`
 * >= 0) and ghost strip inside the domain: COPY rects from overlapping
 * same-level patches, then COARSE rects (of the strip, or with `disjoint` of
 * what the copies leave).  covered[k] = ghost cells of patch k the rects
 * fill.  ADJ_ERR_BAD_ARG with *nrects = the count needed when max_rects is
 * too small. */
int adj_ghost_rects(int ndim, int ghost, const int32_t* level_shape, int npatch, const int32_t* lo,
                    const int32_t* hi, int ncoarse, const int32_t* clo, const int32_t* chi, int ratio,
                    int only, int disjoint, AdjRect* rects, int max_rects, int32_t* nrects, int64_t* covered);

/* Host (no GPU): pairwise overlaps of dst boxes with src boxes (refined by
 * ratio) as rectangles in dst ghost-inclusive coordinates (kind COPY adds
 * src coordinates): the regrid fill of a new level from its parents and
 * the old level (amr.py:504-551).  Order: dst ascending, then src. */
int adj_box_overlaps(int ndim, int kind, int ndst, const int32_t* dlo, const int32_t* dhi, int gdst,
                     int nsrc, const int32_t* slo, const int32_t* shi, int gsrc, int ratio,
                     AdjRect* rects, int max_rects, int32_t* nrects);

/* Stream-ordered strided copy (cudaMemcpy2DAsync, cudaMemcpyDefault): height
 * rows of width bytes, row pitches in bytes.  step_patch_host moves a row slab
 * of every component plane with one call per direction (the planes sit
 * comp_stride apart on the device and nx*ny apart in the host state). */
int adj_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                     void* stream);

int adj_abi_version(void);

/* sizeof of an argument struct as this library was compiled, by name ("AdjStepArgs", ...); 0 for an
 * unknown name.  A binding checks its own layout against it before the first call. */
int adj_struct_size(const char* name);

#ifdef __cplusplus
}
#endif
#endif /* ADJAMR_B200_H */
