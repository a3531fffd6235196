/*
 * fastid_b200_diag.h -- diagnostics of the experiments build only.
 *
 * _fastid_b200_diag.so is compiled from the same sources as the product
 * library with -DFASTID_EXPERIMENTS.  It adds the two process-global switches
 * below, which the timing tools in tools/ use.  Several experiment bits make
 * results wrong on purpose (e.g. skipping operand loads), so the product
 * library (_fastid_b200.so, include/fastid_b200.h) neither exports them nor
 * compiles the branches that read them.
 */
#ifndef FASTID_B200_DIAG_H
#define FASTID_B200_DIAG_H

#include "fastid_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Trace CTA 0 of subsequent tensor launches (kTrSlots clock64 stamps per tile
 * for the first `tiles` tiles; see TraceSlot in csrc/common.cuh); NULL = off. */
FASTID_API int fastid_debug_trace(long long* device_buf, int tiles);
/* Timing-experiment switches for subsequent launches (bits in csrc/common.cuh,
 * CompareArgs::debug_flags; 0 = normal).  Not thread-safe; results of some
 * bits are invalid by design. */
FASTID_API int fastid_debug_flags(int flags);

#ifdef __cplusplus
}
#endif

#endif /* FASTID_B200_DIAG_H */
