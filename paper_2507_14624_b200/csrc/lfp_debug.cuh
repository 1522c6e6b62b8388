// lfp_debug.cuh -- bounds / write-once instrumentation (debug builds).
//
// compute-sanitizer is not available on the GPU pool, so the library can be
// built with -DLFP_CHECK_BOUNDS=1 (liblfprobe_b200_check.so, built by
// __graft_entry__.build()): every probe-map, direction-table, payload,
// origin and ray-order read checks its index against the array extent, and
// every per-ray output record counts its writes in a caller-supplied
// counter array (lfp_debug_bounds). The tests then assert zero violations
// and that every ray's record was written exactly once -- the reference's
// guarantee that each prange iteration writes only its own rows
// (kernels.py:831-843). Release builds compile all of this away.
#pragma once

#ifndef LFP_CHECK_BOUNDS
#define LFP_CHECK_BOUNDS 0
#endif

namespace lfp {

struct DbgState {
    unsigned long long violations;   // failed checks
    int first_site;                  // site id of the first failure
    int pad;
    unsigned* wcount;                // per-output-record write counters
    long long n_out;                 // extent of wcount
};

#if LFP_CHECK_BOUNDS
__device__ DbgState g_dbg;

__device__ __forceinline__ bool dbg_check(bool ok, int site)
{
    if (!ok && atomicAdd(&g_dbg.violations, 1ull) == 0ull)
        g_dbg.first_site = site;
    return ok;
}
// index in [0, n)
#define LFP_BCHK(i, n, site) ::lfp::dbg_check((long long)(i) >= 0 && \
                                              (long long)(i) < (long long)(n), (site))
#define LFP_WCOUNT(oi)                                                     \
    do {                                                                   \
        if (::lfp::g_dbg.wcount &&                                         \
            LFP_BCHK((oi), ::lfp::g_dbg.n_out, 900))                       \
            atomicAdd(::lfp::g_dbg.wcount + (oi), 1u);                     \
    } while (0)
#else
#define LFP_BCHK(i, n, site) ((void)0)
#define LFP_WCOUNT(oi) ((void)0)
#endif

}  // namespace lfp
