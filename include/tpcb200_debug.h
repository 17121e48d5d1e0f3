/* Developer-only entry points of libtpcb200.so (tools/trace_*.py); not part
 * of the drop-in API in tpcb200.h.  The A/B switches of earlier builds are
 * environment variables read once at first use (TPCB_TRAIN_IMPL,
 * TPCB_GRID_CAP, TPCB_POLL_NS, TPCB_GEMM_BK, TPCB_GEMM_CLUSTER,
 * TPCB_GEMM_MODE — csrc/common.cuh Knobs). */
#ifndef TPCB200_DEBUG_H
#define TPCB200_DEBUG_H

#ifdef __cplusplus
extern "C" {
#endif

/* per-phase timestamps (clock64 pairs) of CTA 0 of the training and forward
 * kernels into d_trace[512]; NULL disables.  Process-global: tools only. */
int tpcb_debug_train_trace(long long* d_trace);

#ifdef __cplusplus
}
#endif
#endif /* TPCB200_DEBUG_H */
