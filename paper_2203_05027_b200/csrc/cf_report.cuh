// compute_report's final assembly (solver.py:219-242) and check_termination
// (solver.py:245-272) + the max_iters rule (:322-323), shared by the plan's
// k_finalize and the batched solver so both evaluate the same IEEE expressions.
#pragma once

#include <cmath>

#include "cf_common.h"

namespace cf {

// Partial fields in the order the reductions produce them.
struct ReportFields {
    double prim2, prim_inf, ax_inf, blam, nf_row;               // row part
    double dual2, dual_inf, stat2, stat_inf, atl_inf, pobj, cone_gap, nf_col;   // column part
};

__device__ __forceinline__ cf_report assemble_report(const ReportFields& f, int64_t k, bool extra_nonfinite) {
    cf_report r;
    r.iter = k;
    r.prim_res_inf = f.prim_inf;
    r.prim_res_2 = sqrt(f.prim2);
    r.dual_res_inf = f.dual_inf;
    r.dual_res_2 = sqrt(f.dual2);
    r.stat_res_inf = f.stat_inf;
    r.stat_res_2 = sqrt(f.stat2);
    r.ax_inf = f.ax_inf;
    r.atl_inf = f.atl_inf;
    r.cone_gap = f.cone_gap;
    r.pobj = f.pobj;
    r.dobj = -f.blam;
    r.gap = r.pobj + f.blam;
    r.nonfinite = (f.nf_row > 0.0 || f.nf_col > 0.0 || extra_nonfinite) ? 1 : 0;
    r.status = r.nonfinite ? CF_STATUS_DIVERGED : CF_STATUS_RUNNING;
    return r;
}

// check_termination + max_iters; r.status must be RUNNING or DIVERGED on entry
__device__ __forceinline__ int decide_status(const cf_report& r, const cf_config& c, int64_t k) {
    if (r.status != CF_STATUS_RUNNING) return r.status;
    bool ok;
    if (c.term_mode == CF_TERM_OSQP) {
        // Python max(a, b) returns a unless b > a
        const double mp = (c.b_inf > r.ax_inf) ? c.b_inf : r.ax_inf;
        const double md = (c.c_inf > r.atl_inf) ? c.c_inf : r.atl_inf;
        const double ep = c.eps_abs + c.eps_rel * mp;
        const double ed = c.eps_abs + c.eps_rel * md;
        ok = (r.prim_res_inf < ep) && (r.stat_res_inf < ed);
    } else if (c.term_mode == CF_TERM_SCS) {
        ok = (r.prim_res_2 <= c.scs_prim_bound) && (r.stat_res_2 <= c.scs_dual_bound) &&
             (fabs(r.gap) <= c.eps_gap * ((1.0 + fabs(r.pobj)) + fabs(r.dobj)));
    } else {
        ok = (r.prim_res_2 < c.target_prim_res) && (fabs(r.gap) < c.target_gap);
    }
    int status = ok ? CF_STATUS_SOLVED : CF_STATUS_RUNNING;
    if (status == CF_STATUS_RUNNING && k == c.max_iters) status = CF_STATUS_MAX_ITERS;
    return status;
}

}  // namespace cf
