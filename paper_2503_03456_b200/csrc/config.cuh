// config.cuh -- build-time switches of the solve path (no environment reads on the hot path).
//
// Every schedule choice below was A/B-measured on the B200 (DESIGN.md sections 8-9); the
// defaults are the measured winners.  Experiments rebuild with -DMSY_...=value
// (MSY_EXTRA_NVCC_FLAGS in build.py).  The only runtime environment variable the library
// reads is MSY_SCHUR_TIMING (diagnostic phase timing of sylv_schur, off by default).
#pragma once

#ifndef MSY_HESS_GMAX
#define MSY_HESS_GMAX -1       // cap on the cooperative Hessenberg panel grid (-1: the pair's nsm/2 rule)
#endif
#ifndef MSY_HESS_MODE
#define MSY_HESS_MODE 2        // Hessenberg panel: 2 = cooperative panel kernel, 0 = per-column kernels
#endif
#ifndef MSY_AZC
#define MSY_AZC 2              // Z application: 2 = cluster-split kernel near and far, 1 = near only, 0 = off
#endif
#ifndef MSY_MC_SERIAL
#define MSY_MC_SERIAL 0        // 1: multi-chain sweeps without the far-Z side stream
#endif
#ifndef MSY_SYNC_ENDGAME
#define MSY_SYNC_ENDGAME 0     // 1: endgame blocks on the sweep stream (no deferred column sides)
#endif
#ifndef MSY_CHAINS
#define MSY_CHAINS 8           // bulge chains per sweep (capped by KMAX and the shift block)
#endif
#ifndef MSY_NB_CHAIN
#define MSY_NB_CHAIN 0         // bulges per chain (0: MsCfg<S>::NB)
#endif
#ifndef MSY_SHIFT_TOL
#define MSY_SHIFT_TOL 1e-3     // deflation tolerance of the eigenvalue-only shift computation
#endif
#ifndef MSY_SMALL_SINGLE
#define MSY_SMALL_SINGLE 0     // 1: single-bulge one-CTA kernel for every small block
#endif
#ifndef MSY_MSS_AED
#define MSY_MSS_AED 0          // in-kernel AED window of the one-CTA multishift kernel (0: off, section 9)
#endif
#ifndef MSY_MSS_AEDG
#define MSY_MSS_AEDG 6
#endif
#ifndef MSY_NO_STREAM_PRIORITY
#define MSY_NO_STREAM_PRIORITY 0
#endif
#ifndef MSY_LANE_HESS_CAP
#define MSY_LANE_HESS_CAP 8    // cap on each batched lane's cooperative Hessenberg grid (0: none; m = 512: 16 -> 184, 8 -> 245, 4 -> 238 solves/s)
#endif
#ifndef MSY_FAR_MIN_TILES
#define MSY_FAR_MIN_TILES 64   // single-job Z applications of at least this many 32-wide tiles use the far kernel (-1: far kernel off)
#endif
