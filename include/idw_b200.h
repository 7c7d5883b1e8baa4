/*
 * idw_b200.h -- C ABI of libidw_b200.so, the sm_100a all-pairs IDW engine.
 *
 * The reference (`idwlayout`, pure Python + numba) has no FFI: its hot path is
 * an in-process call from the strategy layer into numba-compiled loops.  This
 * header is the seam that replaces those calls.  Every entry point names the
 * reference code it stands in for (paths relative to /root/reference/pkg/src).
 *
 *   idw_run / idw_run_device   replace the strategy bodies that drive
 *                              kernels.predict_block        (kernels.py:34-67,
 *                                 via strategies.run_naive   strategies.py:148-166
 *                                 and core.idw_predict_seq   core.py:119-148)
 *                              kernels.tile_accumulate +
 *                              kernels.finalize_block      (kernels.py:70-108,
 *                                 via strategies.run_tiled   strategies.py:169-199)
 *                              kernels.nested_improved_block +
 *                              kernels._tree_combine       (kernels.py:111-185,
 *                                 via strategies.run_nested_improved :234-261)
 *                              kernels.nested_original_block (kernels.py:188-248,
 *                                 via strategies.run_nested_original :202-231)
 *
 * Conventions
 *   - Plain C types only; no torch or CUDA types in signatures.
 *   - Every function returns 0 on success or a negative IDW_E* code; the
 *     message of the last failure on the calling thread is idw_last_error().
 *   - Validation that the reference performs in Python (core.py:93-116,
 *     layouts.py:80-82, strategies.py:125-134) stays in the Python host layer;
 *     the library re-checks structural arguments and fails loudly.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns IDW_E_CUDA.
 */
#ifndef IDW_B200_H
#define IDW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IDW_ABI_VERSION 2

/* Most query shards (device-list entries) one host-buffer call can drive. */
#define IDW_MAX_DEVICES 16

/* Layout kind codes == layouts._KIND_CODES (enum order, layouts.py:43-65). */
enum idw_kind { IDW_SOA = 0, IDW_AOS = 1, IDW_AOAS = 2, IDW_SOAOS = 3, IDW_HYBRID = 4 };

/* Precision codes == layouts._PRECISION_CODES (layouts.py:66). */
enum idw_precision { IDW_SINGLE = 0, IDW_DOUBLE = 1 };

/* Strategy codes, in strategies.STRATEGIES order (strategies.py:264-269). */
enum idw_variant {
  IDW_NAIVE = 0,            /* K1: one query per thread, global broadcast loads   */
  IDW_TILED = 1,            /* K2: smem tiles staged by cp.async.bulk + mbarriers */
  IDW_NESTED_ORIGINAL = 2,  /* K4: per-group tree + serial merge (paper "original CDP") */
  IDW_NESTED_IMPROVED = 3   /* K3: G strided lanes + xor-shuffle adjacent-pair tree */
};

/* Arithmetic mode.
 *   EXACT: IEEE round-to-nearest ops in the reference's order; p = 2 results are
 *          bit-identical to the numba reference (no FMA contraction, correctly
 *          rounded 1/d2).  General p uses CUDA pow (few-ulp from glibc pow).
 *   FAST:  MUFU rcp.approx (p = 2) / ex2(lg2 * wexp) (general p), FMA contraction,
 *          packed f32x2 arithmetic, per-tile (tiled) or per-chunk (nested)
 *          partial sums folded with compensated addition.  Coincident queries
 *          are detected and recomputed exactly by a fix-up pass.           */
enum idw_mode { IDW_EXACT = 0, IDW_FAST = 1 };

enum idw_err {
  IDW_OK = 0,
  IDW_E_ARG = -1,         /* malformed argument (kind/precision/buffers/sizes)  */
  IDW_E_UNSUPPORTED = -2, /* illegal layout/precision pair or variant         */
  IDW_E_CUDA = -3,        /* CUDA runtime failure or no device                */
  IDW_E_NOMEM = -4,       /* device allocation failure                        */
  IDW_E_NONFINITE = -5    /* a query coordinate is NaN/inf (core.ensure_finite) */
};

/* A point store == layouts.LayoutStore (layouts.py:143-170): kind, precision,
 * count and its raw byte buffers in buffer_shapes() order (layouts.py:85-104).
 * Buffers hold the exact bytes the reference packs (strides 4/8, 12/24,
 * 16/32, 16+16, 16+8); pads are never read as data.                        */
typedef struct idw_store {
  int32_t kind;            /* enum idw_kind                                   */
  int32_t precision;       /* enum idw_precision                              */
  int64_t count;           /* n >= 1                                          */
  int32_t nbuf;            /* number of buffers for `kind` (3, 1, 1, 2, 2)     */
  int32_t reserved;
  const void *buf[3];      /* buffer base pointers (host or device, see call) */
  int64_t nbytes[3];       /* == BufferSpec.nbytes                            */
} idw_store;

/* Params (core.py:31-47) + ExecConfig (strategies.py:41-66) + GPU knobs. */
typedef struct idw_params {
  double p;                /* power, > 0; p == 2 takes the reciprocal path    */
  double zero_eps;         /* coincidence threshold on d2, >= 0               */
  int32_t variant;         /* enum idw_variant                                */
  int32_t mode;            /* enum idw_mode                                   */
  int64_t group_size;      /* G (nested lanes per query; tiled query group)   */
  int64_t tile_size;       /* T (reference staging tile; informational)       */
  int32_t splits;          /* FAST tiled: summation chunks (0 = auto, from n) */
  int32_t device;          /* CUDA device ordinal when ndevices == 0          */
  /* Device list (ABI 2; idw_run / idw_run_xy / idw_run_device).  Entry
   * k evaluates query shard k: contiguous, whole 256-query units, sizes
   * within one unit (partition.shard_bounds).  The store goes host->device
   * once, to devices[0], and reaches the others by a cudaMemcpyPeerAsync
   * broadcast tree; each entry runs on its own stream and copies its
   * predictions straight into its slice of `out`.  Repeats are allowed (two
   * streams on one GPU).  Results are bit-identical for every list: no
   * query's arithmetic depends on its shard.  ndevices == 0 -> `device`.    */
  int32_t ndevices;
  int32_t devices[IDW_MAX_DEVICES];
} idw_params;

/* Optional per-call instrumentation (RunStats, strategies.py:104-115). */
typedef struct idw_stats {
  int64_t merge_events;    /* nested_original: m * ceil(n/G); others 0        */
  int64_t kernel_launches; /* kernels this call launched                      */
  double kernel_ms;        /* device time of the compute kernels (events)     */
  int64_t fixup_queries;   /* FAST: queries recomputed exactly (coincidence)  */
} idw_stats;

/* ABI version (IDW_ABI_VERSION) -- lets the ctypes loader refuse stale builds. */
int idw_abi_version(void);

/* Number of visible CUDA devices (0 if none); never fails. */
int idw_device_count(void);

/* Message of the last error on this thread ("" if none). */
const char *idw_last_error(void);

/* Blocking run over HOST memory: copies the store buffers and the query
 * coordinates (qx, qy: m values of the run dtype each, already cast RN as in
 * strategies._prepare, strategies.py:125-134) to the device(s), runs the
 * variant, and writes m run-dtype predictions into `out`.  `stats` may be
 * NULL (kernel_ms: the slowest device's kernels).  One host thread drives
 * every device of prm->devices (the reference's worker pool over query
 * blocks, strategies.py:41-66,137-145).  Replaces one whole
 * strategies.run_* call body.                                              */
int idw_run(const idw_store *store, const void *qx, const void *qy, int64_t m,
            const idw_params *prm, void *out, idw_stats *stats);

/* Blocking run over HOST memory that takes the reference's own query array:
 * `queries` holds m (x, y) float64 pairs, row-major -- what
 * core.as_query_array (core.py:93-101) returns.  The rest of
 * strategies._prepare (strategies.py:125-134) runs on the device: the
 * finiteness test of core.ensure_finite (core.py:113-116) and the
 * round-to-nearest cast to the run dtype.  A non-finite coordinate returns
 * IDW_E_NONFINITE ("invalid coordinate"; `out` is then unspecified).
 * Otherwise identical to idw_run.                                          */
int idw_run_xy(const idw_store *store, const double *queries, int64_t m,
               const idw_params *prm, void *out, idw_stats *stats);

/* Asynchronous run over DEVICE memory on `stream` (a cudaStream_t, NULL =
 * legacy default stream), on prm->device (or prm->devices[0]).  With
 * prm->ndevices > 1 every pointer lives on devices[0] and the call spreads
 * itself over the list: the store reaches the other entries by a
 * cudaMemcpyPeerAsync broadcast tree, entry k's query shard by a peer copy,
 * and its predictions come back into its slice of `out` by a peer copy (the
 * gather); `stream` waits for all entries.  Store buffers must stay readable up to
 * nbytes rounded up to 16 bytes (bulk copies move 16-byte granules) and start
 * on a 16-byte boundary (AoS: 4 / 8 bytes suffice for naive, nested_original
 * and EXACT nested_improved; tiled and FAST nested_improved stage tiles by
 * bulk copy) -- IDW_E_ARG otherwise.  Scratch
 * is stream-ordered (cudaMallocAsync).  stats->kernel_ms is not filled here. */
int idw_run_device(const idw_store *store, const void *qx, const void *qy, int64_t m,
                   const idw_params *prm, void *out, void *stream, idw_stats *stats);

/* Plans (one device: ndevices <= 1): one idw_run_device call captured into a CUDA graph (the bounding-box
 * pre-pass, the variant kernels, the fix-up pass and their stream-ordered
 * scratch), replayed by idw_plan_launch for ~3 us of host time instead of
 * one runtime call per kernel.  The plan keeps the store, query and output
 * DEVICE pointers it was created with: refill qx/qy (or the store) in place
 * between launches.  Launches of one plan must not overlap each other.    */
typedef struct idw_plan idw_plan;
int idw_plan_create(const idw_store *store, const void *qx, const void *qy, int64_t m,
                    const idw_params *prm, void *out, idw_plan **plan);
int idw_plan_launch(idw_plan *plan, void *stream);
/* Kernels one launch of the plan runs. */
int64_t idw_plan_launches(const idw_plan *plan);
/* Device time of the variant kernels and the fix-up pass of the plan's most
 * recent launch (timing event nodes inside the graph); blocks until done.  */
int idw_plan_kernel_ms(idw_plan *plan, double *variant_ms, double *fixup_ms);
void idw_plan_destroy(idw_plan *plan);

/* Device-side layout packer: fp64 component arrays x, y, z (n device values
 * each) cast round-to-nearest to the store's precision and written into the
 * preallocated device buffers of `dst` in its layout, pads zeroed -- the
 * bytes LayoutStore.from_arrays (layouts.py:172-186) produces.  Async on
 * `stream`.                                                                */
int idw_pack_device(const double *x, const double *y, const double *z, int64_t n,
                    const idw_store *dst, int device, void *stream);

/* Device-side layout converter: value copy from `src` to the preallocated
 * `dst` (same precision and count, any legal kinds), byte-identical to
 * LayoutStore.convert (layouts.py:251-255).  Async on `stream`.           */
int idw_convert_device(const idw_store *src, const idw_store *dst, int device, void *stream);

/* Device time of the last successful idw_run_device call on this thread:
 * the variant kernels (e.g. k_bbox + k_tiled_chunks) and the FAST fix-up pass,
 * from events recorded on the call's stream.  Blocks until they complete.   */
int idw_last_kernel_ms(double *variant_ms, double *fixup_ms);

/* Measured MUFU reciprocal rate of `device`: a register-resident loop of
 * independent rcp.approx.f32 over all SMs, timed with events.  Writes
 * rcp results per second (== the p = 2 fp32 pair roofline) and the mean SM
 * clock implied by the kernel's clock64() cycle count.                   */
int idw_mufu_peak(int device, double *rcp_per_s, double *sm_hz);

#ifdef __cplusplus
}
#endif
#endif /* IDW_B200_H */
