/* TEST INFRASTRUCTURE — plain-C restatement of the reference hot path (the
 * "port" oracle). Produces exactly the result layout of the C ABI (include/xsp.h)
 * in malloc'd HOST memory, so product and oracle results diff column by column.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use it. */
#ifndef XSP_ORACLE_H
#define XSP_ORACLE_H

#include "xsp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* correlate() per trace (correlator.cpp:141-370) over HOST columns. */
int xspo_correlate(const xsp_span_cols* cols, const xsp_traces* traces, xsp_corr_out* out);
void xspo_corr_free(xsp_corr_out* out);

/* a8..a15 + a1 throughput + top-k (analysis.cpp:28-586) over a port correlation. */
int xspo_analyze(const xsp_span_cols* cols, const xsp_corr_out* corr, const xsp_groups* groups,
                 const xsp_system_spec* spec, const xsp_analysis_opts* opts, xsp_tables_out* out);
void xspo_tables_free(xsp_tables_out* out);

#ifdef __cplusplus
}
#endif

#endif
