/*
 * wagma_b200.h -- C ABI of the B200-native WAGMA group-model-averaging hot path.
 *
 * The reference (`wagma` 0.1.0, /root/reference/pkg/src/wagma) is a pure
 * Python package with no FFI; its drop-in boundary for this path is the
 * Python API listed next to each entry point. The package
 * `paper_2005_00124_b200` binds exactly these symbols with ctypes and
 * exposes that Python API on top (topology.py, collective.py, optim.py).
 * No torch types cross this boundary: plain pointers (device pointers for
 * model vectors), sizes and int status codes.
 *
 * Status codes map 1:1 onto the reference exceptions:
 *   WG_EINVAL    -> topology.InvalidParamsError / optim.ConfigError (ValueError)
 *   WG_EVERSION  -> collective.VersionRegressionError
 *   WG_ESTALE    -> collective.ProtocolFault (staleness bound, collective.py:290-294)
 *   WG_EPROTO    -> collective.ProtocolFault (torn read, recycled descriptor, ...)
 *   WG_ETIMEOUT  -> collective.ProtocolFault (device watchdog: a peer never published)
 *   WG_ECUDA     -> RuntimeError (CUDA runtime failure)
 *   WG_EDIVERGE  -> optim.DivergenceError (non-finite gradient, optim.py:174-175)
 */
#ifndef WAGMA_B200_H
#define WAGMA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WG_OK 0
#define WG_EINVAL 1
#define WG_EVERSION 2
#define WG_ESTALE 3
#define WG_EPROTO 4
#define WG_ETIMEOUT 5
#define WG_ECUDA 6
#define WG_ENOMEM 7
#define WG_EDIVERGE 8 /* non-finite W' produced (gradient or replica); optim.DivergenceError */
#define WG_ESYNC 9    /* mismatched sync points: a rank joined iteration t as a global sync while another
                         joined it as a group round (collective.py:381-386); collective.ProtocolFault */

#define WG_RULE_EXAMPLE 0 /* topology.MASK_RULE_EXAMPLE ("example") */
#define WG_RULE_LITERAL 1 /* topology.MASK_RULE_LITERAL ("literal") */

#define WG_F32 0
#define WG_F64 1

/* ------------------------------------------------------------------------
 * Schedule generator (host, C++). Bit-exact with the reference.
 * ---------------------------------------------------------------------- */

/* GroupingParams(P, S, t).__post_init__ validation (topology.py:64-72). */
int wg_check_params(int P, int S, int64_t t);

/* phase_masks(GroupingParams(P, S, t), rule).masks (topology.py:118-142).
 * masks must hold >= log2(S) ints; *n_masks receives log2(S). */
int wg_phase_masks(int P, int S, int64_t t, int rule, int* masks, int* n_masks);

/* compute_groups(GroupingParams(P, S, t), rule) (topology.py:162-181):
 * groups sorted by smallest member, members ascending, flattened into
 * `members` (capacity P); group g occupies members[offsets[g] .. offsets[g+1]).
 * offsets must hold P+1 ints; *n_groups receives the group count. */
int wg_compute_groups(int P, int S, int64_t t, int rule, int* members, int* offsets, int* n_groups);

/* GroupPartition.group_of(rank) (topology.py:114-115): the sorted group of
 * `rank`; out capacity P; *n receives the group size. */
int wg_group_of(int P, int S, int64_t t, int rule, int rank, int* out, int* n);

/* peer(rank, mask, P) (topology.py:145-151). */
int wg_peer(int rank, int mask, int P, int* out);

/* mixing_reachable(GroupingParams(P, S, .), start_t, k, rule) (topology.py:184-208). */
int wg_mixing_reachable(int P, int S, int64_t start_t, int k, int rule, int* out);

/* Leaf order of the butterfly tree that the reference's recursive doubling
 * (collective.py:310-329) builds at `rank` for version t: leaf i is
 * rank ^ XOR{masks[r] : bit r of i}; out capacity 2^log2(S). This is the
 * fixed summation order of the device kernel. */
int wg_tree_leaves(int P, int S, int64_t t, int rule, int rank, int* out, int* n);

/* ------------------------------------------------------------------------
 * Device context: replaces the reference's `Simulator` + per-rank
 * `SendBuffer`/`GroupAllreduce`/`SyncAllreduce` endpoint state
 * (netsim.py:120-204, collective.py:84-447). One context per process/GPU;
 * it hosts ranks [gpu_index*R, (gpu_index+1)*R), R = P / n_gpus.
 * ---------------------------------------------------------------------- */

typedef struct wg_ctx wg_ctx;

typedef struct {
    int32_t P;                  /* total ranks (power of two, <= 64)          */
    int32_t S;                  /* group size (power of two, <= P)            */
    int32_t n_gpus;             /* processes / GPUs in the job (divides P)    */
    int32_t gpu_index;          /* this process's index in [0, n_gpus)        */
    int32_t device;             /* CUDA device ordinal                        */
    int32_t dtype;              /* WG_F32 / WG_F64                            */
    int32_t mask_rule;          /* WG_RULE_*                                  */
    int32_t activation_enabled; /* alpha: wait-avoiding activation (1) or
                                   blocking group allreduce (0, beta)         */
    int64_t n;                  /* elements per model replica                 */
    int64_t tau;                /* global sync period; 0 = None               */
    int64_t staleness_bound;    /* collective.py:290; <= 0 = None             */
    int32_t ring_depth;         /* send-ring slots per rank; 0 = auto (2*tau) */
    int32_t version_ring;       /* activation descriptors; 0 = auto           */
    int64_t grace_ns;           /* activator lock-in grace window             */
    int64_t timeout_ns;         /* device watchdog for every spin-wait        */
} wg_config;

int wg_ctx_create(const wg_config* cfg, wg_ctx** out);
int wg_ctx_destroy(wg_ctx* ctx);

/* Cross-process peer mapping over NVLink / NVSwitch (CUDA IPC). export writes
 * an opaque blob (<= 256 bytes); every process imports every other's blob. */
int wg_ctx_export(wg_ctx* ctx, void* blob, size_t cap, size_t* len);
int wg_ctx_import_peer(wg_ctx* ctx, int gpu_index, const void* blob, size_t len);

/* SendBuffer(initial_model) with stamp -1 (collective.py:93,169): copies the
 * device vector w0 (n elements of dtype) into rank's ring slot of stamp -1. */
int wg_ctx_set_initial_model(wg_ctx* ctx, int rank, const void* w0, void* stream);

/* SendBuffer.install(vec, iteration) (collective.py:95-101) outside a fused
 * launch (e.g. GroupAllreduce.install_fresh before a global sync): copies the
 * device vector into rank's ring slot for `stamp`, publishes every tile and
 * announces `stamp`, all ordered on `stream`. */
int wg_install(wg_ctx* ctx, int rank, int64_t stamp, const void* vec, void* stream);

/* Device pointer of `rank`'s send-buffer slot holding `stamp` (any rank; a
 * peer pointer for remote ranks), and the stamp it currently holds. */
int wg_ctx_slot(wg_ctx* ctx, int rank, int64_t stamp, void** ptr, int64_t* held_stamp);

/* Job kinds of one launch. */
#define WG_JOB_STEP 0        /* fused: local step + group average (Alg. 2 l.3-15)   */
#define WG_JOB_SYNC_STEP 1   /* fused: local step + global average (Alg. 2 l.16)     */
#define WG_JOB_LOCAL_STEP 2  /* fused: local step only (alpha = beta = 0)            */
#define WG_JOB_GROUP_SUM 3   /* GroupAllreduce.join_or_check(version, fresh) -> acc  */
#define WG_JOB_SYNC_SUM 4    /* SyncAllreduce.join(iteration, vec) -> total          */

#define WG_UPDATE_SGD 0
#define WG_UPDATE_MOMENTUM 1

typedef struct {
    int32_t rank;        /* global rank, must be hosted by this context      */
    int32_t kind;        /* WG_JOB_*                                          */
    int64_t version;     /* iteration t                                       */
    int32_t update_rule; /* WG_UPDATE_*                                       */
    int32_t pad;
    double eta;          /* EtaSchedule.rate(t, P, T)                         */
    double beta;         /* momentum coefficient                              */
    void* W;             /* STEP kinds: W_t in, W_{t+1} out (n elems)         */
    void* m;             /* momentum buffer in/out (MOMENTUM only)            */
    const void* g;       /* gradient (STEP kinds)                             */
    const void* fresh;   /* *_SUM kinds: W' to install and contribute         */
    void* acc_out;       /* *_SUM kinds: accumulator out                      */
} wg_job;

typedef struct {
    int64_t version;
    int64_t contrib_stamp; /* stamp this rank contributed (collective.py:289)  */
    int32_t timely;        /* stamp == version (collective.py:301)             */
    int32_t activator;     /* this rank raised the activation flag (is root)    */
    int32_t error;         /* WG_* device-side error latched for this job      */
    int32_t root;          /* rank that raised the version's activation flag,
                              -1 if none (sync, blocking or replayed versions);
                              the root of the reference's binomial ACT tree
                              (collective.py:263-274)                          */
} wg_job_status;

/* One launch = at most one job per local rank. forced_stamps (may be NULL)
 * is an [n_versions][P] table of contribution stamps for group versions in
 * `forced_versions` (replay of a recorded contribution log); other group
 * versions use the live activation protocol (or blocking mode). The launch
 * is asynchronous on `stream` (a cudaStream_t); statuses are readable with
 * wg_launch_status after the stream is synchronised. */
int wg_launch(wg_ctx* ctx, const wg_job* jobs, int n_jobs, const int64_t* forced_versions,
              const int64_t* forced_stamps, int n_forced, void* stream);

/* Status of job i of the most recent launch (after stream synchronisation). */
int wg_launch_status(wg_ctx* ctx, int i, wg_job_status* out);

/* Contribution stamps of all P ranks for group version `version` as locked by
 * the activation protocol (the device's contribution log,
 * collective.py:295-296). *locked = 0 if the version was not activated. */
int wg_query_version(wg_ctx* ctx, int64_t version, int64_t* stamps, int* locked);

/* Latched device error word (0 = none) and a one-line description. */
int wg_ctx_error(wg_ctx* ctx, int* code, int64_t* info);

/* Same error word, read from its host-mapped mirror without synchronising
 * any stream (errors latched by kernels that are still running may not be
 * visible yet). Lets a host loop raise DivergenceError one step later
 * instead of forcing a device round trip every iteration. */
int wg_ctx_error_async(wg_ctx* ctx, int* code, int64_t* info);
int wg_ctx_clear_error(wg_ctx* ctx);

/* Straggler injection (StragglerPolicy + compute_delay, netsim.py:64-117):
 * a device-side spin of `ns` nanoseconds on `stream`. */
int wg_delay(wg_ctx* ctx, int64_t ns, void* stream);

/* Replica diagnostics (compute_diagnostics, optim.py:199-210). wg_replicas_sum
 * adds sum_r W_r (fp64) of R device replicas (n elements) into `sum`;
 * wg_replicas_spread adds sum_r ||W_r - mu||^2 into out[0] and writes
 * max |W_r - W_0| into out[1] (fp64 device scalars, zero them first). With
 * the global mean mu (sum over every rank / P, all-reduced across
 * processes) and the all-reduced out[0], this is the spread potential
 * Gamma_t; out[1] == 0 is the bit-identity check after a global sync. */
int wg_replicas_sum(wg_ctx* ctx, const void* const* W, int R, double* sum, void* stream);
int wg_replicas_spread(wg_ctx* ctx, const void* const* W, int R, const double* mu, double* out, void* stream);

/* Instrumentation: per-CTA phase cycle counters (long long [grid][8]:
 * produce, publish, resolve, poll, consume, tiles) written by every
 * multi-GPU launch while dev_buf is non-NULL. */
int wg_ctx_set_profile(wg_ctx* ctx, void* dev_buf);

/* Number of element tiles and the tile size used by the kernels. */
int wg_ctx_geometry(wg_ctx* ctx, int64_t* tile_elems, int64_t* n_tiles, int* grid, int* ring_depth);

const char* wg_strerror(int code);
const char* wg_last_error_message(void);

#ifdef __cplusplus
}
#endif

#endif /* WAGMA_B200_H */
