// extern "C" entry points of libadjamr_b200.so (declared in include/adjamr_b200.h).
#include "adj_common.cuh"
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

namespace adj {

static thread_local char g_err[512] = "";

int record_cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return ADJ_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return ADJ_ERR_CUDA;
}

int check_launch(const char* where) { return record_cuda(cudaGetLastError(), where); }

// ADJAMR_PDL=0 disables programmatic dependent launch (A/B measurements).
bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

int step_exact(const AdjStepArgs& a, cudaStream_t st);
int step_fast(const AdjStepArgs& a, cudaStream_t st);
void fast_tile_shape(int ndim, int32_t* ni, int32_t* nj);
int fill_physical(const AdjPhysArgs& a);
int fill_ghost_rects(const AdjGhostArgs& a);
int ghost_plan_build(const AdjGhostPlanBuildArgs& a, int rect_cells);
int fill_ghost_plan(const AdjGhostPlanFillArgs& a);
int restrict_level(const AdjRestrictArgs& a);
int flag_adjoint(const AdjFlagArgs& a);
int flag_level_mask(const AdjFlagMaskArgs& a);
int functional(const AdjFunctionalArgs& a);
int gauges(const AdjGaugeArgs& a);

static int bad(const char* msg) {
    snprintf(g_err, sizeof(g_err), "bad argument: %s", msg);
    return ADJ_ERR_BAD_ARG;
}

}  // namespace adj

extern "C" {

int adj_abi_version(void) { return ADJ_ABI_VERSION; }

int adj_struct_size(const char* name) {
    if (!name) return 0;
#define ADJ_SZ(T) if (!strcmp(name, #T)) return (int)sizeof(T);
    ADJ_SZ(AdjPatch) ADJ_SZ(AdjTile) ADJ_SZ(AdjRect) ADJ_SZ(AdjGhostPlan) ADJ_SZ(AdjGhostPlanBuildArgs)
    ADJ_SZ(AdjGhostPlanFillArgs) ADJ_SZ(AdjStepRestrict) ADJ_SZ(AdjJobFill) ADJ_SZ(AdjStepArgs) ADJ_SZ(AdjPhysArgs)
    ADJ_SZ(AdjGhostArgs) ADJ_SZ(AdjRestrictArgs) ADJ_SZ(AdjFlagArgs) ADJ_SZ(AdjFunctionalArgs) ADJ_SZ(AdjGauge)
    ADJ_SZ(AdjGaugeArgs) ADJ_SZ(AdjFlagMaskArgs)
#undef ADJ_SZ
    return 0;
}

const char* adj_last_error(void) { return adj::g_err; }

int adj_step_tile_shape(int variant, int ndim, int32_t* ni, int32_t* nj) {
    if (!ni || !nj) return adj::bad("null tile-shape outputs");
    if (variant == ADJ_VARIANT_EXACT) {
        if (ndim == 2) { *ni = 16; *nj = 16; } else { *ni = 256; *nj = 1; }
        return ADJ_OK;
    }
    if (variant == ADJ_VARIANT_FAST) { adj::fast_tile_shape(ndim, ni, nj); return ADJ_OK; }
    return adj::bad("unknown variant");
}

int adj_step_level(const AdjStepArgs* a) {
    if (!a) return adj::bad("null args");
    if (a->q_in == a->q_out) return adj::bad("q_in must not alias q_out");
    if (!a->q_in || !a->q_out || !a->aux || !a->patches || !a->tiles || !a->speed_max || !a->nonfinite ||
        !a->work_counter)
        return adj::bad("null pointer");
    if (a->ghost < 2) return adj::bad("ghost width must be >= 2");
    if (a->ndim == 1 && a->system != ADJ_SYS_AC1D) return adj::bad("1D requires acoustics-1d");
    if (a->ndim == 2 && a->system == ADJ_SYS_AC1D) return adj::bad("2D requires a 2D system");
    if (a->limiter < ADJ_LIM_NONE || a->limiter > ADJ_LIM_SUPERBEE) return adj::bad("limiter");
    if (!(a->dt > 0.0)) return adj::bad("dt must be positive");
    if (a->job_offsets && !(a->variant == ADJ_VARIANT_FAST && a->ndim == 2 && a->static_speed))
        return adj::bad("packed jobs (job_offsets) need the FAST 2D step with static_speed");
    if (a->prefill.plan.n > 0) {
        if (!(a->variant == ADJ_VARIANT_FAST && a->ndim == 2 && a->static_speed && (a->flags & ADJ_STEP_COUNTER_ZERO) &&
              !(a->flags & ADJ_STEP_TWO_ROWS)))
            return adj::bad("prefill needs the FAST 2D static-CFL path with ADJ_STEP_COUNTER_ZERO");
        if (a->prefill.q != a->q_in || a->prefill.ndim != 2 || a->prefill.m != 3)
            return adj::bad("prefill must fill q_in (2D, m = 3)");
        if (!(a->prefill.plan.dst && a->prefill.plan.src && a->prefill.plan.meta)) return adj::bad("null prefill plan");
        if (a->prefill.plan.nc > 0 && !(a->prefill.q_coarse_old && a->prefill.q_coarse_new && a->prefill.plan.c_base))
            return adj::bad("null prefill coarse state");
    }
    if (a->fine_restrict.ratio != 0) {
        const AdjStepRestrict& r = a->fine_restrict;
        if (!(a->variant == ADJ_VARIANT_FAST && a->ndim == 2 && a->static_speed && a->form == ADJ_FORM_WAVE &&
              !a->reversed && !(a->flags & ADJ_STEP_TWO_ROWS) && a->prefill.plan.n == 0))
            return adj::bad("fused restriction needs the FAST 2D static-CFL forward wave step without prefill");
        if (!(r.ratio == 2 || r.ratio == 4)) return adj::bad("fused restriction ratio must be 2 or 4");
        if (!(r.q_coarse && r.cell && r.base)) return adj::bad("null fused restriction tables");
    }
    if (a->flags & ADJ_STEP_PHYS_IN) {
        if (!(a->variant == ADJ_VARIANT_FAST && a->ndim == 2 && a->static_speed && a->npatch == 1 && a->ghost == 2 &&
              !(a->flags & ADJ_STEP_TWO_ROWS) && a->prefill.plan.n == 0 && a->job_fill.n == 0))
            return adj::bad("ADJ_STEP_PHYS_IN needs the FAST 2D static-CFL step of one patch, ghost width 2");
        for (int k = 0; k < 4; ++k)
            if (a->phys_bc[k] < ADJ_BC_WALL || a->phys_bc[k] > ADJ_BC_PERIODIC) return adj::bad("phys_bc");
        if ((a->phys_bc[0] == ADJ_BC_PERIODIC) != (a->phys_bc[1] == ADJ_BC_PERIODIC) ||
            (a->phys_bc[2] == ADJ_BC_PERIODIC) != (a->phys_bc[3] == ADJ_BC_PERIODIC))
            return adj::bad("periodic sides come in pairs");
    }
    if (a->job_fill.n > 0) {
        const AdjJobFill& f = a->job_fill;
        if (!(a->variant == ADJ_VARIANT_FAST && a->ndim == 2 && a->static_speed && a->job_offsets &&
              (a->flags & ADJ_STEP_COUNTER_ZERO) && !(a->flags & ADJ_STEP_TWO_ROWS) && a->prefill.plan.n == 0))
            return adj::bad("job fill needs the FAST 2D static-CFL step with job_offsets, "
                            "ADJ_STEP_COUNTER_ZERO and no prefill");
        if (!(f.entry_off && f.dst && f.src && f.meta)) return adj::bad("null job fill tables");
        if (f.cache_mode < 0 || f.cache_mode > 2 || (f.cache_mode && !f.cache))
            return adj::bad("job fill cache_mode needs a cache");
        if (f.cache_mode != 2 && f.c_base && !(f.q_coarse_old && f.q_coarse_new && f.c_step && f.c_wx && f.c_wy))
            return adj::bad("null job fill coarse state");
    }
    cudaStream_t st = (cudaStream_t)a->stream;
    int rc = ADJ_OK;
    const bool static_cfl = a->variant == ADJ_VARIANT_FAST && a->ndim == 2 && a->static_speed;
    if (static_cfl) {
        if (!(a->flags & ADJ_STEP_NO_SPEED_OUT))
            rc = adj::record_cuda(cudaMemcpyAsync(a->speed_max, a->static_speed, sizeof(double) * 2 * a->npatch,
                                                  cudaMemcpyDeviceToDevice, st), "copy static_speed");
    } else {
        rc = adj::record_cuda(cudaMemsetAsync(a->speed_max, 0, sizeof(double) * 2 * a->npatch, st), "memset speed_max");
    }
    if (rc) return rc;
    if (!(a->flags & ADJ_STEP_KEEP_NONFINITE)) {
        rc = adj::record_cuda(cudaMemsetAsync(a->nonfinite, 0, sizeof(int32_t) * a->npatch, st), "memset nonfinite");
        if (rc) return rc;
    }
    const bool counter_zero = (a->flags & ADJ_STEP_COUNTER_ZERO) && a->variant == ADJ_VARIANT_FAST && a->ndim == 2;
    if (!counter_zero) {
        rc = adj::record_cuda(cudaMemsetAsync(a->work_counter, 0, 2 * sizeof(int32_t), st), "memset work_counter");
        if (rc) return rc;
    }
    if (a->variant == ADJ_VARIANT_EXACT) return adj::step_exact(*a, st);
    if (a->variant == ADJ_VARIANT_FAST) return adj::step_fast(*a, st);
    return adj::bad("unknown variant");
}

int adj_fill_physical(const AdjPhysArgs* a) {
    if (!a || !a->q || !a->patches) return adj::bad("null pointer");
    if (a->ghost < 2) return adj::bad("ghost width must be >= 2");
    return adj::fill_physical(*a);
}

int adj_fill_ghost_rects(const AdjGhostArgs* a) {
    if (!a || !a->q_dst || !a->rects || !a->dst_patches || !(a->src_patches || a->coarse_patches))
        return adj::bad("null pointer");
    if (a->time_mode < 0 || a->time_mode > 2) return adj::bad("time_mode");
    return adj::fill_ghost_rects(*a);
}

int adj_ghost_plan_build(const AdjGhostPlanBuildArgs* a) {
    if (!a || !a->patches || !a->counter) return adj::bad("null pointer");
    if (!a->plan.dst || !a->plan.src || !a->plan.meta) return adj::bad("null plan arrays");
    if (a->nrect > 0 && !(a->rects && a->rect_cell0)) return adj::bad("rects need rect_cell0");
    if (a->plan.nc > 0 && !(a->coarse_patches && a->axis_w && a->axis_i && a->plan.c_base && a->plan.c_step &&
                            a->plan.c_wx && a->plan.c_wy))
        return adj::bad("COARSE entries need coarse patches, axis tables and coarse arrays");
    if (a->nedge > 0 && !a->edge_patches) return adj::bad("null edge patches");
    if (a->ghost < 2) return adj::bad("ghost width must be >= 2");
    if (a->m < 1 || a->m > 3) return adj::bad("m must be 1..3");
    cudaStream_t st = (cudaStream_t)a->stream;
    int rc = adj::record_cuda(cudaMemsetAsync(a->counter, 0, sizeof(int32_t), st), "memset counter");
    if (rc) return rc;
    return adj::ghost_plan_build(*a, a->rect_cells);
}

int adj_fill_ghost_plan(const AdjGhostPlanFillArgs* a) {
    if (!a || !a->q) return adj::bad("null pointer");
    if (a->plan.n > 0 && !(a->plan.dst && a->plan.src && a->plan.meta)) return adj::bad("null plan arrays");
    if (a->plan.nc > 0 && !(a->q_coarse_old && a->q_coarse_new && a->plan.c_base)) return adj::bad("null coarse state");
    if (a->m < 1 || a->m > 3) return adj::bad("m must be 1..3");
    if (a->time_mode < 0 || a->time_mode > 2) return adj::bad("time_mode");
    return adj::fill_ghost_plan(*a);
}

int adj_restrict(const AdjRestrictArgs* a) {
    if (!a || !a->q_coarse || !a->q_fine || !(a->rects || (a->cell_dst && a->cell_src && a->cell_meta)))
        return adj::bad("null pointer");
    if (a->ratio < 1) return adj::bad("ratio");
    if (a->swe && (!a->aux_coarse || !a->aux_fine)) return adj::bad("swe restriction needs aux");
    return adj::restrict_level(*a);
}

int adj_flag_adjoint(const AdjFlagArgs* a) {
    if (!a || !a->q || !a->patches || !a->ring || !a->snap_index || !a->flag_bits || !a->counts || !a->status)
        return adj::bad("null pointer");
    if (a->mode == 1 && !a->interp_w) return adj::bad("mode 1 needs interp_w");
    if (a->best && !a->best_offset) return adj::bad("best needs best_offset");
    cudaStream_t st = (cudaStream_t)a->stream;
    int rc = adj::record_cuda(cudaMemsetAsync(a->counts, 0, sizeof(unsigned long long) * a->npatch, st), "memset counts");
    if (rc) return rc;
    rc = adj::record_cuda(cudaMemsetAsync(a->status, 0, sizeof(int32_t), st), "memset status");
    if (rc) return rc;
    return adj::flag_adjoint(*a);
}

int adj_flag_level_mask(const AdjFlagMaskArgs* a) {
    if (!a || !a->mask || !a->occupancy || !a->raw_count) return adj::bad("null pointer");
    if (a->npatch > 0 && !(a->flag_bits && a->patches)) return adj::bad("null flags / patches");
    if (a->region_rows && (!a->region_row_off || (a->ndim == 2 && !(a->region_cols && a->region_col_off))))
        return adj::bad("region tables incomplete");
    if (a->level_nx < 1 || a->level_ny < 1 || a->buffer < 0) return adj::bad("level shape / buffer");
    return adj::flag_level_mask(*a);
}

int adj_functional(const AdjFunctionalArgs* a) {
    if (!a || !a->q || !a->patches || !a->ring || !a->partial || !a->status) return adj::bad("null pointer");
    if (a->finer && a->nfiner > 0 && (!a->covered || a->ratio < 1)) return adj::bad("covered mask needs scratch and ratio");
    if (a->blocks_x < 1 || a->npatch < 1) return adj::bad("empty launch");
    return adj::functional(*a);
}

int adj_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                     void* stream) {
    if (!dst || !src) return adj::bad("null pointer");
    if (width > dpitch || width > spitch) return adj::bad("width exceeds a pitch");
    if (width == 0 || height == 0) return ADJ_OK;
    const cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                            (cudaStream_t)stream);
    return adj::record_cuda(e, "cudaMemcpy2DAsync");
}

int adj_gauges(const AdjGaugeArgs* a) {
    if (!a || !a->q || (a->ngauge > 0 && (!a->gauges || !a->out))) return adj::bad("null pointer");
    return adj::gauges(*a);
}

}  // extern "C"
