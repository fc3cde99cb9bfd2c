/*
 * stkde_diag.h -- development diagnostics of the tcgen05 engine, NOT part of the product
 * ABI (include/stkde.h): exported only by a -DSTKDE_TC_DIAG=1 build of the library
 * (scripts/build_variant.py prof -DSTKDE_TC_DIAG=1 -> libstkde_prof.so).
 */
#ifndef STKDE_DIAG_H_
#define STKDE_DIAG_H_
#include "../../include/stkde.h"
#ifdef __cplusplus
extern "C" {
#endif
/* With STKDE_TC_PROF=1 in the environment at plan creation, the tile kernel accumulates
 * clock64 phase totals of one thread per role (generator teams: [0..10], loader:
 * [16..23]; layout in stkde_tile_tc.cu); this copies the 32 u64 counters to out32 and
 * resets them.  Synchronises the device. */
int stkde_plan_tc_profile(stkde_plan_t plan, uint64_t *out32);
/* buf = device-accessible (e.g. pinned host) array of num_sms * 32 uint32; the tcgen05
 * kernel's warps publish their protocol state (tag << 24 | step) in it while running.
 * NULL disables. */
int stkde_plan_debug_progress(stkde_plan_t plan, void *buf);
#ifdef __cplusplus
}
#endif
#endif
