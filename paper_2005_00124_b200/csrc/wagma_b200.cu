// B200-native WAGMA group-model-averaging hot path (sm_100a).
//
// One persistent kernel per launch fuses, tile by tile:
//   produce  local SGD / momentum step of every job in the launch
//            (optim.py:176-183), written once into the rank's send-ring slot
//            (SendBuffer.install, collective.py:95-101) and into shared memory;
//   publish  per-tile readiness flags (system-scope release) so peers on other
//            GPUs can pull the tile over NVLink as soon as it exists;
//   consume  the group sum: S leaves pulled with 128-bit loads from peer
//            send-ring slots (NVLink / NVSwitch) or from shared memory, summed
//            in the butterfly tree order of the reference's recursive doubling
//            (collective.py:310-329), then divided by S (timely), S+1 (late,
//            optim.py:439-447) or P (global sync, optim.py:449-452).
//
// The wait-avoiding activation (collective.py:192-308) is one activation
// descriptor per version on GPU 0: the first rank to arrive CASes it
// (system scope), waits at most a grace window for the other ranks to
// announce, locks every rank's contribution stamp (its latest announced
// version: fresh W' if it joined, its last-published stale W' otherwise) and
// releases it. No host round trip, no global barrier; only the periodic
// global sync (S = P, blocking) waits for everyone.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/wagma_b200.h"
#include "wagma_internal.h"

#ifndef WG_MINB
#define WG_MINB 3  // CTAs per SM the single-GPU kernel is register-budgeted for
#endif
#ifndef WG_MINB_AHEAD
#define WG_MINB_AHEAD 3
#endif

namespace wg {

// ---------------------------------------------------------------------------
// error reporting
// ---------------------------------------------------------------------------

static thread_local std::string g_last_error;

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define WG_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(WG_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));           \
    } while (0)

// ---------------------------------------------------------------------------
// device-memory arena (one per GPU, exported to peers with CUDA IPC)
// ---------------------------------------------------------------------------

struct Desc {                 // activation descriptor of one group version
    int64_t state;            // 0 free; (v+1)*4+1 locking; (v+1)*4+2 locked
    int64_t root;             // rank that raised the activation flag
    int64_t pad[14];
    int64_t stamps[kMaxP];    // contribution stamp of every rank
};

struct Layout {
    int64_t hdr;       // int64 error code, int64 error info
    int64_t announce;  // int64 [R] (128-byte stride): latest announced version
    int64_t complete;  // int64 [R][D]: stamp whose tiles are all published
    int64_t counter;   // uint32 [R][D]: tiles published for the current stamp
    int64_t syncmark;  // int64 [R][D]: 2(v+1) + (v joined as a global sync) of the stamp v in the slot, 0 never
    int64_t desc;      // Desc [Dv]  (used on GPU 0 only)
    int64_t flags;     // int64 [R][n_tiles][warps]: latest stamp published per warp-tile
    int64_t ring;      // T [R][D][npad]: send ring
    int64_t red_flags; // int64 [R][n_tiles]: latest version whose reduced tile is published (multi-GPU)
    int64_t red_ring;  // T [R][D][npad]: reduced tiles owned by the rank (split sums)
    int64_t part_flags;  // int64 [R][n_tiles]: latest version whose subtree partial is published (hier sums)
    int64_t part_ring;   // T [R][D][npad]: GPU-local subtree partials keyed by their first leaf rank
    int64_t total;
};

constexpr int kAnnounceStride = 16;  // int64 words (128 B)
constexpr int kWarps = kThreads / 32;
constexpr int kSplitMaxP = 8;  // split sums (reduce-scatter + all-gather) up to this many ranks
// A split sum of S members spread over `span` GPUs (L = S/span per GPU) moves
// (L/S)(S-L) + (1 - L/S) leaf-tiles over NVLink per tile against S - L for
// the pull; split when that saves at least a third: 2S >= 3(L + 1).
__host__ __device__ constexpr bool split_pays(int S, int span) { return 2 * S >= 3 * (S / span + 1); }
constexpr int64_t kNever = INT64_MIN / 2;

enum VersionMode : int32_t { kLive = 0, kForced = 1, kBlocking = 2, kSync = 3 };

struct DevJob {
    int32_t rank, local, kind, update_rule;
    int64_t version;
    int32_t vidx, plan, produces, pad;
    double eta, beta;
    void* W;
    void* m;
    const void* g;
    const void* fresh;
    void* acc_out;
};

struct DevVersion {
    int64_t version;
    int32_t mode, forced_idx;
};

struct DevPlan {
    int32_t vidx, n_leaves, log_leaves, divisor, n_members, divisor_pow2;
    int16_t leaves[kMaxLeaves];
    int8_t members[kMaxJobs];
};

// Split-sum owners of a plan: its sorted distinct members (see split_owner_index).
struct DevOwners {
    int32_t n;
    int16_t rank[kMaxLeaves];
};

struct LaunchParams {
    char* base[kMaxGpus];
    Layout L;
    int32_t P, S, R, G, gpu_index, D, Dv, n_jobs, n_versions, n_plans, need_fence, pad;
    int64_t n, npad, n_tiles, tile_elems;
    int64_t grace_ns, timeout_ns, staleness_bound;
    int32_t adaptive_grace, pad_ag;  // skip the grace wait for ranks late at the previous version
    int32_t job_of_rank[kMaxP];
    DevJob jobs[kMaxJobs];
    DevVersion versions[kMaxVersions];
    DevPlan plans[kMaxPlans];
    int64_t forced[kMaxVersions][kMaxP];
    DevOwners owners[kMaxPlans];
    wg_job_status* status;
    long long* prof;  // optional per-CTA phase cycle counters [grid][8]
    int32_t fence_scope;  // 0 sys, 1 gpu (default), 2 none (timing experiments only)
    int32_t nvl_stages;   // leaf-ring stages of the multi-GPU TMA kernel
    int32_t nvl_rows;     // leaf rows per stage the host sized the pull kernel's ring for
    int32_t split_stages; // reduced-tile ring stages of the split kernel
    int32_t split_span;   // minimum GPUs a group must span to be summed split
    int32_t red_warps;    // split kernel: stream-A reducer warps (4 or 8 of the 12 shared with stream B)
    int32_t loc_stages;   // single-GPU TMA kernel: input-ring stages
    int64_t* err_host;    // host-mapped mirror of the error word (wg_ctx_error_async)
    int32_t mg_cap_a, mg_cap_b;  // wagma_mg_kernel: phase-1 / phase-2 row capacity (chunk rows)
    int32_t mg_split;            // wagma_mg_kernel: split (reduce-scatter) partial sums where they pay
    int32_t tma_prod;            // wagma_nvl_kernel: TMA-fed producers (else per-thread cp.async rings)
    // hierarchical sums (multi-GPU pull kernel): a plan whose lowest plan_hl
    // tree levels stay inside one GPU exchanges GPU-local subtree partials
    // instead of leaves when all its members are timely
    int8_t plan_hl[kMaxPlans];   // 0: leaf pull
    int32_t n_parts;             // local partials this launch produces
    int8_t job_order[kMaxJobs];  // producer job order: every partial's leaves consecutive, in leaf order
    int8_t job_part[kMaxJobs];   // partial of the k-th produced job (-1: none)
    int8_t job_ppos[kMaxJobs];   // its leaf position inside the partial
    int8_t job_plast[kMaxJobs];  // last leaf of the partial: store it
    int16_t part_key[kMaxJobs];  // first leaf rank of each local partial (its buffer and flags)
    int64_t part_version[kMaxJobs];
};

// ---------------------------------------------------------------------------
// device helpers: scoped memory operations (PTX memory model)
// ---------------------------------------------------------------------------

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int64_t ld_relaxed_sys(const int64_t* p) {
    int64_t v;
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(int64_t* p, int64_t v) {
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t atom_cas_sys(int64_t* p, int64_t cmp, int64_t val) {
    int64_t old;
    asm volatile("atom.acq_rel.sys.global.cas.b64 %0, [%1], %2, %3;"
                 : "=l"(old)
                 : "l"(p), "l"(cmp), "l"(val)
                 : "memory");
    return old;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// Control words (announce, descriptors, slot completion, sync marks) at the
// narrowest correct scope: system scope when peers on other GPUs take part,
// GPU scope for a single-GPU context (every reader runs on this GPU; the host
// reads them only after the stream synchronised; the host-mapped error mirror
// stays system scope). A system-scope fence costs ~5 us.
__device__ __forceinline__ int64_t ld_acquire_sc(bool sys, const int64_t* p) {
    if (sys) return ld_acquire_sys(p);
    int64_t v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sc(bool sys, int64_t* p, int64_t v) {
    if (sys)
        st_release_sys(p, v);
    else
        asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sc(bool sys, int64_t* p, int64_t v) {
    if (sys)
        st_relaxed_sys(p, v);
    else
        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t atom_cas_sc(bool sys, int64_t* p, int64_t cmp, int64_t val) {
    if (sys) return atom_cas_sys(p, cmp, val);
    int64_t old;
    asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;"
                 : "=l"(old)
                 : "l"(p), "l"(cmp), "l"(val)
                 : "memory");
    return old;
}
__device__ __forceinline__ void fence_sc(bool sys) {
    if (sys)
        fence_sys();
    else
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// element traits: 16-byte vectors, IEEE round-to-nearest ops (no contraction)
// ---------------------------------------------------------------------------

template <typename T>
struct Tr;
template <>
struct Tr<float> {
    using V = float4;
    static constexpr int EPV = 4;
};
template <>
struct Tr<double> {
    using V = double2;
    static constexpr int EPV = 2;
};

__device__ __forceinline__ float4 vadd(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 vsub(float4 a, float4 b) {
    return make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z), __fsub_rn(a.w, b.w));
}
__device__ __forceinline__ float4 vscale(float s, float4 a) {
    return make_float4(__fmul_rn(s, a.x), __fmul_rn(s, a.y), __fmul_rn(s, a.z), __fmul_rn(s, a.w));
}
__device__ __forceinline__ float4 vdiv(float4 a, float d) {
    return make_float4(__fdiv_rn(a.x, d), __fdiv_rn(a.y, d), __fdiv_rn(a.z, d), __fdiv_rn(a.w, d));
}
__device__ __forceinline__ double2 vadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 vsub(double2 a, double2 b) {
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 vscale(double s, double2 a) {
    return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}
__device__ __forceinline__ double2 vdiv(double2 a, double d) {
    return make_double2(__ddiv_rn(a.x, d), __ddiv_rn(a.y, d));
}
// Non-finite component (NaN or +-Inf): the reference raises DivergenceError
// on a non-finite gradient (optim.py:174-175); a non-finite g, m or W makes
// W' non-finite, so the produced W' is what is checked.
__device__ __forceinline__ bool nonfinite(float4 v) {
    return !(fabsf(v.x) <= 3.402823466e38f && fabsf(v.y) <= 3.402823466e38f && fabsf(v.z) <= 3.402823466e38f &&
             fabsf(v.w) <= 3.402823466e38f);
}
__device__ __forceinline__ bool nonfinite(double2 v) {
    return !(fabs(v.x) <= 1.7976931348623157e308 && fabs(v.y) <= 1.7976931348623157e308);
}

// Caller-owned vectors (W, m, g, fresh, acc_out) have exactly n elements:
// full 16-byte vectors inside, element-wise handling of the ragged end
// (component by component: no address of a register vector is taken).
__device__ __forceinline__ float4 ld_tail(const float* b, int64_t idx, int64_t n) {
    return make_float4(idx < n ? b[idx] : 0.f, idx + 1 < n ? b[idx + 1] : 0.f, idx + 2 < n ? b[idx + 2] : 0.f,
                       idx + 3 < n ? b[idx + 3] : 0.f);
}
__device__ __forceinline__ double2 ld_tail(const double* b, int64_t idx, int64_t n) {
    return make_double2(idx < n ? b[idx] : 0.0, idx + 1 < n ? b[idx + 1] : 0.0);
}
__device__ __forceinline__ void st_tail(float* b, int64_t idx, int64_t n, float4 v) {
    if (idx < n) b[idx] = v.x;
    if (idx + 1 < n) b[idx + 1] = v.y;
    if (idx + 2 < n) b[idx + 2] = v.z;
    if (idx + 3 < n) b[idx + 3] = v.w;
}
__device__ __forceinline__ void st_tail(double* b, int64_t idx, int64_t n, double2 v) {
    if (idx < n) b[idx] = v.x;
    if (idx + 1 < n) b[idx + 1] = v.y;
}
template <typename T, bool FULL = false>
__device__ __forceinline__ typename Tr<T>::V ld_stream(const T* base, int64_t idx, int64_t n) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    if (FULL || idx + E <= n) return __ldcs(reinterpret_cast<const V*>(base + idx));
    return ld_tail(base, idx, n);
}
template <typename T, bool FULL = false>
__device__ __forceinline__ void st_stream(T* base, int64_t idx, int64_t n, typename Tr<T>::V v) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    if (FULL || idx + E <= n)
        __stcs(reinterpret_cast<V*>(base + idx), v);
    else
        st_tail(base, idx, n, v);
}

// ---------------------------------------------------------------------------
// arena addressing (rank r lives on GPU r / R at local index r % R)
// ---------------------------------------------------------------------------

__device__ __forceinline__ char* rank_base(const LaunchParams& p, int rank) { return p.base[rank / p.R]; }
__device__ __forceinline__ int64_t* announce_ptr(const LaunchParams& p, int rank) {
    return reinterpret_cast<int64_t*>(rank_base(p, rank) + p.L.announce) + (rank % p.R) * kAnnounceStride;
}
__device__ __forceinline__ int slot_of(const LaunchParams& p, int64_t stamp) {
    return int((stamp + 1) % p.D);
}
__device__ __forceinline__ int64_t* complete_ptr(const LaunchParams& p, int rank, int slot) {
    return reinterpret_cast<int64_t*>(rank_base(p, rank) + p.L.complete) + (rank % p.R) * p.D + slot;
}
__device__ __forceinline__ int64_t* syncmark_ptr(const LaunchParams& p, int rank, int slot) {
    return reinterpret_cast<int64_t*>(rank_base(p, rank) + p.L.syncmark) + (rank % p.R) * p.D + slot;
}
__device__ __forceinline__ unsigned* counter_ptr(const LaunchParams& p, int rank, int slot) {
    return reinterpret_cast<unsigned*>(rank_base(p, rank) + p.L.counter) + (rank % p.R) * p.D + slot;
}
// Readiness flag of one warp's part of a tile: the latest stamp whose W'
// is written there (monotone per rank; older stamps live in other slots).
__device__ __forceinline__ int64_t* flag_ptr(const LaunchParams& p, int rank, int64_t tile, int warp) {
    return reinterpret_cast<int64_t*>(rank_base(p, rank) + p.L.flags) +
           ((int64_t(rank % p.R) * p.n_tiles + tile) * kWarps + warp);
}
template <typename T>
__device__ __forceinline__ T* ring_ptr(const LaunchParams& p, int rank, int slot) {
    return reinterpret_cast<T*>(rank_base(p, rank) + p.L.ring) + (int64_t(rank % p.R) * p.D + slot) * p.npad;
}
__device__ __forceinline__ int64_t* red_flag_ptr(const LaunchParams& p, int rank, int64_t tile) {
    return reinterpret_cast<int64_t*>(rank_base(p, rank) + p.L.red_flags) + int64_t(rank % p.R) * p.n_tiles + tile;
}
template <typename T>
__device__ __forceinline__ T* red_ptr(const LaunchParams& p, int rank, int64_t version) {
    return reinterpret_cast<T*>(rank_base(p, rank) + p.L.red_ring) +
           (int64_t(rank % p.R) * p.D + version % p.D) * p.npad;
}
__device__ __forceinline__ int64_t* part_flag_ptr(const LaunchParams& p, int rank, int64_t tile) {
    return reinterpret_cast<int64_t*>(rank_base(p, rank) + p.L.part_flags) + int64_t(rank % p.R) * p.n_tiles + tile;
}
template <typename T>
__device__ __forceinline__ T* part_ptr(const LaunchParams& p, int rank, int64_t version) {
    return reinterpret_cast<T*>(rank_base(p, rank) + p.L.part_ring) +
           (int64_t(rank % p.R) * p.D + version % p.D) * p.npad;
}
__device__ __forceinline__ Desc* desc_ptr(const LaunchParams& p, int64_t version) {
    return reinterpret_cast<Desc*>(p.base[0] + p.L.desc) + (version % p.Dv);
}
__device__ __forceinline__ int64_t* err_ptr(const LaunchParams& p) {
    return reinterpret_cast<int64_t*>(p.base[p.gpu_index] + p.L.hdr);
}

__device__ __noinline__ void raise_error(const LaunchParams& p, int code, int64_t info) {
    int64_t* e = err_ptr(p);
    if (atomicCAS(reinterpret_cast<unsigned long long*>(e), 0ull, (unsigned long long)code) == 0ull) {
        e[1] = info;
        if (p.err_host) {  // host-mapped mirror: info first, then the code
            st_relaxed_sys(p.err_host + 1, info);
            st_release_sys(p.err_host, code);
        }
    }
    __threadfence_system();
}
__device__ __forceinline__ bool aborted(const LaunchParams& p) {
    return ld_relaxed_sys(err_ptr(p)) != 0;
}

// Spin until *addr == want. Returns 0 ok, WG_EPROTO if the word moved past
// `want` (slot reused / descriptor recycled), WG_ETIMEOUT on the watchdog.
__device__ int spin_eq(const LaunchParams& p, const int64_t* addr, int64_t want, uint64_t t0) {
    int64_t v = ld_acquire_sc(p.G > 1, addr);
    int it = 0;
    while (v != want) {
        if (v > want) return WG_EPROTO;
        if ((++it & 63) == 0) {
            if (globaltimer() - t0 > uint64_t(p.timeout_ns)) return WG_ETIMEOUT;
            if (aborted(p)) return WG_ETIMEOUT;
        }
        __nanosleep(64);
        v = ld_acquire_sc(p.G > 1, addr);
    }
    return 0;
}

// Spin until *addr >= want (monotone readiness flag). WG_EPROTO if it moved
// `ring` or more stamps past (the slot holding `want` was overwritten).
__device__ int spin_geq(const LaunchParams& p, const int64_t* addr, int64_t want, uint64_t t0) {
    int64_t v = ld_acquire_sys(addr);
    int it = 0;
    while (v < want) {
        if ((++it & 63) == 0) {
            if (globaltimer() - t0 > uint64_t(p.timeout_ns)) return WG_ETIMEOUT;
            if (aborted(p)) return WG_ETIMEOUT;
        }
        __nanosleep(32);
        v = ld_acquire_sys(addr);
    }
    return v >= want + p.D ? WG_EPROTO : 0;
}

// ---------------------------------------------------------------------------
// control phase (CTA 0, warp 0): announce, activation, lock-in
// ---------------------------------------------------------------------------

__device__ void control_phase(const LaunchParams& p, int* s_activator) {
    const int lane = threadIdx.x & 31;
    // Announce "rank r is producing W'_v in a running kernel" (the join,
    // collective.py:192-205). Activators lock contribution stamps from it.
    if (lane == 0) {
        for (int j = 0; j < p.n_jobs; ++j) {
            const DevJob& jb = p.jobs[j];
            if (!jb.produces) continue;
            // how this rank joins version v (global sync or group round): the
            // sync-point check of every consumer (check_sync_points)
            st_relaxed_sc(p.G > 1, syncmark_ptr(p, jb.rank, slot_of(p, jb.version)),
                           2 * (jb.version + 1) + (p.versions[jb.vidx].mode == kSync));
            st_release_sc(p.G > 1, announce_ptr(p, jb.rank), jb.version);
        }
        fence_sc(p.G > 1);
    }
    __syncwarp();
    for (int vi = 0; vi < p.n_versions; ++vi) {
        if (lane == 0) s_activator[vi] = 0;
        if (p.versions[vi].mode != kLive) continue;
        const int64_t v = p.versions[vi].version;
        Desc* d = desc_ptr(p, v);
        int act = 0;
        if (lane == 0) {
            // First arrival raises the activation flag (collective.py:214-218);
            // later arrivals find it raised (exactly-once, collective.py:236).
            int64_t st = ld_acquire_sc(p.G > 1, &d->state);
            for (;;) {
                const int64_t sv = st / 4 - 1;
                if (sv == v) break;
                if (sv > v) {  // descriptor recycled before this join
                    raise_error(p, WG_EPROTO, v);
                    break;
                }
                const int64_t old = atom_cas_sc(p.G > 1, &d->state, st, (v + 1) * 4 + 1);
                if (old == st) {
                    act = 1;
                    break;
                }
                st = old;
            }
        }
        act = __shfl_sync(0xffffffffu, act, 0);
        if (!act) continue;
        // the activation root: the lowest rank of this launch joining v
        int root = p.P;
        for (int j = 0; j < p.n_jobs; ++j)
            if (p.jobs[j].vidx == vi && p.jobs[j].rank < root) root = p.jobs[j].rank;
        if (lane == 0) {
            s_activator[vi] = 1;
            d->root = root;
        }
        // Bounded grace window: ranks on other GPUs that join within it are
        // timely. Ranks on this GPU announced at launch start (final).
        // Adaptive: a rank that has not even announced version v-1 is at
        // least a whole version behind (a straggler): it is not waited for,
        // so a persistent straggler does not cost every version the whole
        // window (it is still timely if it announces before the lock). A
        // rank slightly behind (it announced v-1) is waited for as usual.
        const uint64_t t0 = globaltimer();
        const int q0 = lane, q1 = lane + 32;
        bool skip0 = false, skip1 = false;
        if (p.adaptive_grace) {
            skip0 = q0 < p.P && ld_acquire_sc(p.G > 1, announce_ptr(p, q0)) < v - 1;
            skip1 = q1 < p.P && ld_acquire_sc(p.G > 1, announce_ptr(p, q1)) < v - 1;
        }
        int64_t a0 = kNever, a1 = kNever;
        for (;;) {
            bool in = true;
            if (q0 < p.P) {
                a0 = ld_acquire_sc(p.G > 1, announce_ptr(p, q0));
                if (a0 < v && q0 / p.R != p.gpu_index && !skip0) in = false;
            }
            if (q1 < p.P) {
                a1 = ld_acquire_sc(p.G > 1, announce_ptr(p, q1));
                if (a1 < v && q1 / p.R != p.gpu_index && !skip1) in = false;
            }
            if (__all_sync(0xffffffffu, in)) break;
            if (globaltimer() - t0 > uint64_t(p.grace_ns)) break;
            __nanosleep(200);
        }
        // Lock-in (collective.py:289-301): each rank contributes its latest
        // announced W' -- fresh if it joined v, its stale send buffer if not.
        if (q0 < p.P) {
            const int64_t s = a0 < v ? a0 : v;
            d->stamps[q0] = s;
            if (p.staleness_bound > 0 && s <= v - p.staleness_bound)
                raise_error(p, WG_ESTALE, v * 1024 + q0);  // collective.py:290-294
        }
        if (q1 < p.P) {
            const int64_t s = a1 < v ? a1 : v;
            d->stamps[q1] = s;
            if (p.staleness_bound > 0 && s <= v - p.staleness_bound) raise_error(p, WG_ESTALE, v * 1024 + q1);
        }
        __syncwarp();
        if (lane == 0) {
            fence_sc(p.G > 1);
            st_release_sc(p.G > 1, &d->state, (v + 1) * 4 + 2);
        }
        __syncwarp();
    }
}

// Rank whose arrival raised the activation flag of a job's live group
// version (read after the descriptor is locked), -1 for none.
__device__ __forceinline__ int32_t activation_root(const LaunchParams& p, const DevJob& jb, bool resolved) {
    if (!resolved || jb.vidx < 0 || p.versions[jb.vidx].mode != kLive) return -1;
    return int32_t(ld_relaxed_sys(&desc_ptr(p, p.versions[jb.vidx].version)->root));
}

// ---------------------------------------------------------------------------
// per-CTA shared state
// ---------------------------------------------------------------------------

enum LeafSrc : int8_t { kSrcPoll = -1, kSrcReady = -2 };

struct SmemCtl {
    int64_t stamps[kMaxVersions][kMaxP];     // contribution stamps per version
    int8_t leaf_src[kMaxPlans][kMaxLeaves];  // >=0: stage of job; -1 poll; -2 ready
    int16_t leaf_slot[kMaxPlans][kMaxLeaves];
    int32_t plan_polls[kMaxPlans];
    int32_t activator[kMaxVersions];
    int32_t abort;
};

#ifndef WG_NO_SYNC_CHECK
#define WG_NO_SYNC_CHECK 0
#endif
#ifndef WG_PUB_GATHER_P  // produced chunks published per fence at most (publisher of wagma_mg_kernel)
#define WG_PUB_GATHER_P 1
#endif
#ifndef WG_PUB_GATHER_R  // owned reduced chunks published per fence at most
#define WG_PUB_GATHER_R 1
#endif
// Sync-point agreement (collective.py:381-386: "mismatched sync points"), one
// warp of CTA 0 after the launch consumed its leaves. Every rank marks how it
// joins each version (control_phase: 2(v+1), +1 for a global sync):
//  - a global sync at v needs every rank to have joined v as a sync (its W'_v
//    was consumed, so its mark is on the way);
//  - a group round at v must not see a timely member that joined v as a sync.
// Either mismatch latches WG_ESYNC (info v * 1024 + rank), a ProtocolFault.
__device__ void check_sync_points(const LaunchParams& p, const SmemCtl& sm) {
    const int lane = threadIdx.x & 31;
    if (sm.abort || WG_NO_SYNC_CHECK) return;
    for (int vi = 0; vi < p.n_versions; ++vi) {
        const int64_t v = p.versions[vi].version;
        const bool sync = p.versions[vi].mode == kSync;
        const int slot = slot_of(p, v);
        for (int q = lane; q < p.P; q += 32) {
            const int64_t* mk = syncmark_ptr(p, q, slot);
            int64_t x = ld_acquire_sc(p.G > 1, mk);
            if (sync) {
                const uint64_t t0 = globaltimer();
                int it = 0;
                while (x < 2 * (v + 1)) {
                    if ((++it & 63) == 0 && (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p))) break;
                    __nanosleep(64);
                    x = ld_acquire_sc(p.G > 1, mk);
                }
                if (x == 2 * (v + 1)) raise_error(p, WG_ESYNC, v * 1024 + q);
            } else if (sm.stamps[vi][q] == v && x == 2 * (v + 1) + 1) {
                raise_error(p, WG_ESYNC, v * 1024 + q);
            }
        }
    }
}

// Resolve every plan's leaves to a source (after lock-in), executed by
// `nthr` threads starting at thread index `t0` (the whole CTA, or one warp)
// separated by `sync()`.
template <typename T, class Sync>
__device__ bool resolve_core(const LaunchParams& p, SmemCtl& sm, int tid, int nthr, Sync sync) {
    const uint64_t t0 = globaltimer();
    if (tid == 0) {
        for (int vi = 0; vi < p.n_versions && !sm.abort; ++vi) {
            if (p.versions[vi].mode != kLive) continue;
            const int64_t v = p.versions[vi].version;
            const int rc = spin_eq(p, &desc_ptr(p, v)->state, (v + 1) * 4 + 2, t0);
            if (rc) {
                raise_error(p, rc, v);
                sm.abort = 1;
            }
        }
    }
    sync();
    if (sm.abort) return false;
    for (int i = tid; i < p.n_versions * p.P; i += nthr) {
        const int vi = i / p.P, q = i % p.P;
        const DevVersion& dv = p.versions[vi];
        int64_t s;
        if (dv.mode == kLive)
            s = ld_relaxed_sys(&desc_ptr(p, dv.version)->stamps[q]);
        else if (dv.mode == kForced)
            s = p.forced[dv.forced_idx][q];
        else
            s = dv.version;
        sm.stamps[vi][q] = s;
    }
    sync();
    for (int i = tid; i < p.n_plans * kMaxLeaves; i += nthr) {
        const int pl = i / kMaxLeaves, li = i % kMaxLeaves;
        const DevPlan& P_ = p.plans[pl];
        if (li >= P_.n_leaves) continue;
        const int q = P_.leaves[li];
        const int64_t s = sm.stamps[P_.vidx][q];
        const int j = p.job_of_rank[q];
        int8_t src;
        if (s < -1) {
            raise_error(p, WG_EPROTO, q);
            sm.abort = 1;
            src = kSrcReady;
        } else if (j >= 0 && p.jobs[j].produces && p.jobs[j].version == s) {
            src = int8_t(j);  // produced by this launch: shared-memory stage
        } else {
            const int slot = slot_of(p, s);
            if (j >= 0 && p.jobs[j].produces && slot_of(p, p.jobs[j].version) == slot) {
                raise_error(p, WG_EPROTO, s);  // slot overwritten in this launch
                sm.abort = 1;
            }
            const int64_t c = ld_acquire_sc(p.G > 1, complete_ptr(p, q, slot));
            if (c > s) {
                raise_error(p, WG_EPROTO, s);  // send ring wrapped past the stamp
                sm.abort = 1;
            }
            src = (c == s) ? int8_t(kSrcReady) : int8_t(kSrcPoll);
            sm.leaf_slot[pl][li] = int16_t(slot);
        }
        sm.leaf_src[pl][li] = src;
    }
    sync();
    if (tid < p.n_plans) {
        int polls = 0;
        for (int li = 0; li < p.plans[tid].n_leaves; ++li) polls |= (sm.leaf_src[tid][li] == kSrcPoll);
        sm.plan_polls[tid] = polls;
    }
    sync();
    return !sm.abort;
}

template <typename T>
__device__ bool resolve_sources(const LaunchParams& p, SmemCtl& sm) {
    return resolve_core<T>(p, sm, threadIdx.x, blockDim.x, [] { __syncthreads(); });
}

// ---------------------------------------------------------------------------
// produce: local step, send-ring install, shared-memory stage
// ---------------------------------------------------------------------------

// Inputs are streamed through a per-thread shared-memory ring with cp.async
// (LDGSTS): each thread prefetches the W, g, m vectors of the next kDepth
// (tile, job) items it will compute, so memory-level parallelism does not
// depend on registers. A thread only ever reads the ring entries it filled
// itself, so no barrier is needed (cp.async.wait_group orders its own copies).
#ifndef WG_DEPTH
#define WG_DEPTH 3
#endif
constexpr int kDepth = WG_DEPTH;
// single-GPU loop A/B knobs: incremental issue cursor; per-job ring slot
// pointers from shared memory (else recomputed per item)
#ifndef WG_STEP_INCR
#define WG_STEP_INCR 0
#endif
#ifndef WG_STEP_SRING
#define WG_STEP_SRING 0
#endif

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Prefetch one item's inputs (zero-filled past n: the ragged end).
template <typename T>
__device__ __forceinline__ void issue_item(const LaunchParams& p, int64_t tile, int j, typename Tr<T>::V* slot) {
    constexpr int E = Tr<T>::EPV;
    const int tid = threadIdx.x;
    const int64_t idx = tile * p.tile_elems + int64_t(tid) * E;
    const int64_t rem = p.n - idx;
    const int bytes = rem >= E ? 16 : (rem > 0 ? int(rem * int64_t(sizeof(T))) : 0);
    const int64_t off = bytes ? idx : 0;
    const DevJob& jb = p.jobs[j];
    if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
        cp_async16(&slot[tid], static_cast<const T*>(jb.fresh) + off, bytes);
        return;
    }
    cp_async16(&slot[tid], static_cast<const T*>(jb.W) + off, bytes);
    cp_async16(&slot[kThreads + tid], static_cast<const T*>(jb.g) + off, bytes);
    if (jb.update_rule == WG_UPDATE_MOMENTUM)
        cp_async16(&slot[2 * kThreads + tid], static_cast<const T*>(jb.m) + off, bytes);
}

// Send-ring slot of every job of the launch (the W' it installs), computed
// once per CTA instead of a 64-bit modulo per item. Caller syncs after.
template <typename T>
__device__ __forceinline__ void init_ring_slots(const LaunchParams& p, T** ring_slot, int64_t** flag0 = nullptr) {
    if (threadIdx.x < p.n_jobs) {
        const DevJob& jb = p.jobs[threadIdx.x];
        ring_slot[threadIdx.x] = ring_ptr<T>(p, jb.rank, slot_of(p, jb.version));
        if (flag0) flag0[threadIdx.x] = flag_ptr(p, jb.rank, 0, 0);  // warp-tile flags of the job's rank
    }
}

// Local step of one item + send-ring install + stage (optim.py:176-183,
// collective.py:95-101). Returns true if the produced W' is non-finite.
template <typename T, bool STAGE = true>
__device__ __forceinline__ bool compute_item(const LaunchParams& p, int64_t tile, int j,
                                             const typename Tr<T>::V* slot, typename Tr<T>::V* stage,
                                             T* const* ring_slot, typename Tr<T>::V* wp_out = nullptr) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    const int tid = threadIdx.x;
    const int64_t idx = tile * p.tile_elems + int64_t(tid) * E;
    const DevJob& jb = p.jobs[j];
    V wp;
    bool bad = false;
    if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
        wp = slot[tid];
    } else {
        const V w = slot[tid];
        const V g = slot[kThreads + tid];
        const T eta = T(jb.eta);
        if (jb.update_rule == WG_UPDATE_MOMENTUM) {
            // m = beta*m + g ; W' = W - eta*m  (optim.py:179,183)
            const V mn = vadd(vscale(T(jb.beta), slot[2 * kThreads + tid]), g);
            st_stream<T>(static_cast<T*>(jb.m), idx, p.n, mn);
            wp = vsub(w, vscale(eta, mn));
        } else {
            wp = vsub(w, vscale(eta, g));  // W' = W - eta*g (optim.py:181-183)
        }
        bad = nonfinite(wp);  // zero-filled past n: the ragged end stays finite
        if (jb.kind == WG_JOB_LOCAL_STEP) {
            st_stream<T>(static_cast<T*>(jb.W), idx, p.n, wp);
            return bad;
        }
    }
    // SendBuffer.install: W' written once into the send ring, and staged
    T* const rs = ring_slot ? ring_slot[j] : ring_ptr<T>(p, jb.rank, slot_of(p, jb.version));
    __stcg(reinterpret_cast<V*>(rs + idx), wp);
    if (STAGE) stage[j * kThreads + tid] = wp;
    if (wp_out) *wp_out = wp;
    return bad;
}

// Latch DivergenceError (optim.py:174-175) for the jobs whose produced W'
// was non-finite in any thread of the warp: `bad` is a per-thread job mask.
__device__ __forceinline__ void report_divergence(const LaunchParams& p, unsigned bad) {
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) raise_error(p, WG_EDIVERGE, p.jobs[__ffs(bad) - 1].rank);
}

// Multi-GPU kernel: register-pipelined produce (the next job's loads in
// flight while the current one computes); keeps 3 CTAs/SM for NVLink latency.
// Loads of one job's inputs for this thread's vectors of a tile.
template <typename T>
__device__ __forceinline__ void load_job(const LaunchParams& p, const DevJob& jb, int64_t tbase,
                                         typename Tr<T>::V* a, typename Tr<T>::V* b, typename Tr<T>::V* c) {
    constexpr int E = Tr<T>::EPV;
    const int tid = threadIdx.x;
    if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
        const T* fr = static_cast<const T*>(jb.fresh);
#pragma unroll
        for (int k = 0; k < kVecPerThread; ++k) a[k] = ld_stream<T>(fr, tbase + int64_t(k * kThreads + tid) * E, p.n);
        return;
    }
    const T* W = static_cast<const T*>(jb.W);
    const T* g = static_cast<const T*>(jb.g);
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
        const int64_t idx = tbase + int64_t(k * kThreads + tid) * E;
        a[k] = ld_stream<T>(W, idx, p.n);
        b[k] = ld_stream<T>(g, idx, p.n);
    }
    if (jb.update_rule == WG_UPDATE_MOMENTUM) {
        const T* m = static_cast<const T*>(jb.m);
#pragma unroll
        for (int k = 0; k < kVecPerThread; ++k) c[k] = ld_stream<T>(m, tbase + int64_t(k * kThreads + tid) * E, p.n);
    }
}

template <typename T>
__device__ __forceinline__ void produce_tile_regs(const LaunchParams& p, int64_t tile, typename Tr<T>::V* stage,
                                                  T* const* ring_slot, unsigned& bad) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    constexpr int U = kVecPerThread;
    const int tid = threadIdx.x;
    const int64_t tbase = tile * p.tile_elems;
    // software pipeline: the next job's loads are in flight while this one
    // is computed and stored
    V cw[U], cg[U], cm[U];
    load_job<T>(p, p.jobs[0], tbase, cw, cg, cm);
    for (int j = 0; j < p.n_jobs; ++j) {
        const DevJob& jb = p.jobs[j];
        V nw[U], ng[U], nm[U];
        if (j + 1 < p.n_jobs) load_job<T>(p, p.jobs[j + 1], tbase, nw, ng, nm);
        V wp[U];
        if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
#pragma unroll
            for (int k = 0; k < U; ++k) wp[k] = cw[k];
        } else {
            const T eta = T(jb.eta);
            if (jb.update_rule == WG_UPDATE_MOMENTUM) {
                // m = beta*m + g ; W' = W - eta*m  (optim.py:179,183)
                T* m = static_cast<T*>(jb.m);
                const T beta = T(jb.beta);
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const V mn = vadd(vscale(beta, cm[k]), cg[k]);
                    st_stream<T>(m, tbase + int64_t(k * kThreads + tid) * E, p.n, mn);
                    wp[k] = vsub(cw[k], vscale(eta, mn));
                }
            } else {
                // W' = W - eta*g  (optim.py:181-183)
#pragma unroll
                for (int k = 0; k < U; ++k) wp[k] = vsub(cw[k], vscale(eta, cg[k]));
            }
#pragma unroll
            for (int k = 0; k < U; ++k) bad |= unsigned(nonfinite(wp[k])) << j;
            if (jb.kind == WG_JOB_LOCAL_STEP) {
                T* W = static_cast<T*>(jb.W);
#pragma unroll
                for (int k = 0; k < U; ++k) st_stream<T>(W, tbase + int64_t(k * kThreads + tid) * E, p.n, wp[k]);
            }
        }
        if (jb.produces) {
            // SendBuffer.install (collective.py:95-101): one write into the ring
            T* slot = ring_slot[j] + tbase;
#pragma unroll
            for (int k = 0; k < U; ++k) {
                __stcg(reinterpret_cast<V*>(slot + int64_t(k * kThreads + tid) * E), wp[k]);
                stage[(j * U + k) * kThreads + tid] = wp[k];  // thread-private stage
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            cw[k] = nw[k];
            cg[k] = ng[k];
            cm[k] = nm[k];
        }
    }
}

// Per-warp-tile readiness flags, only read by kernels on OTHER GPUs (ranks on
// this GPU either read this launch's shared-memory stage or a slot completed
// by an earlier launch). No CTA barrier: the warp's stores are ordered before
// lane 0's fence by __syncwarp, the fence before the flag store. Peer loads
// of this GPU's memory are served by this GPU's L2, so a GPU-scope fence
// orders data before flag for them (fence_scope 0 = strict system scope).
__device__ __forceinline__ void publish_tile(const LaunchParams& p, int64_t tile) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        const long long c0 = p.prof ? clock64() : 0;
        if (p.fence_scope == 0)
            fence_sys();
        else if (p.fence_scope == 1)
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * 8 + 6] += clock64() - c0;
        const int w = threadIdx.x >> 5;
        for (int j = 0; j < p.n_jobs; ++j) {
            const DevJob& jb = p.jobs[j];
            if (jb.produces) st_relaxed_sys(flag_ptr(p, jb.rank, tile, w), jb.version);
        }
    }
}

// After the tile loop: add this CTA's tile count to each produced slot's
// counter; the CTA completing the count publishes the whole slot (`complete`).
__device__ __forceinline__ void publish_slots(const LaunchParams& p, unsigned my_tiles) {
    __syncthreads();
    const int j = threadIdx.x;
    if (j < p.n_jobs && p.jobs[j].produces && my_tiles) {
        const DevJob& jb = p.jobs[j];
        const int slot = slot_of(p, jb.version);
        fence_sc(p.G > 1);
        unsigned* c = counter_ptr(p, jb.rank, slot);
        if (atomicAdd(c, my_tiles) + my_tiles == unsigned(p.n_tiles)) {
            *c = 0u;
            fence_sc(p.G > 1);
            st_release_sc(p.G > 1, complete_ptr(p, jb.rank, slot), jb.version);
        }
    }
}

// ---------------------------------------------------------------------------
// consume: butterfly-tree sum of the group's leaves, averaging rule
// ---------------------------------------------------------------------------

static_assert(kVecPerThread == 1, "the consume path is written for one 16-byte vector per thread");

// Butterfly tree over leaves [leaf0, leaf0 + 2^LOG): level r adds the
// subtrees that differ in bit r of the leaf index (collective.py:310-329).
// `fetch(leaf)` returns this thread's vector of a leaf.
template <typename T, int LOG>
struct TreeSum {
    template <class F>
    static __device__ __forceinline__ typename Tr<T>::V run(const F& fetch, int leaf0) {
        const auto a = TreeSum<T, LOG - 1>::run(fetch, leaf0);
        const auto b = TreeSum<T, LOG - 1>::run(fetch, leaf0 + (1 << (LOG - 1)));
        return vadd(a, b);
    }
};
template <typename T>
struct TreeSum<T, 0> {
    template <class F>
    static __device__ __forceinline__ typename Tr<T>::V run(const F& fetch, int leaf) {
        return fetch(leaf);
    }
};

// Trees of 16..64 leaves: 8-leaf subtrees combined through a 4-level
// register stack (static indices only), same pairing as the full tree.
template <typename T, class F>
__device__ __forceinline__ typename Tr<T>::V tree_sum_big(const F& fetch, int log_leaves) {
    using V = typename Tr<T>::V;
    V s0, s1, s2, s3;
    const int nchunks = 1 << (log_leaves - 3);
    for (int c = 0; c < nchunks; ++c) {
        V cur = TreeSum<T, 3>::run(fetch, c * 8);
        if (!(c & 1)) {
            s0 = cur;
            continue;
        }
        cur = vadd(s0, cur);
        if (!(c & 2)) {
            s1 = cur;
            continue;
        }
        cur = vadd(s1, cur);
        if (!(c & 4)) {
            s2 = cur;
            continue;
        }
        s3 = vadd(s2, cur);
    }
    return log_leaves == 4 ? s1 : (log_leaves == 5 ? s2 : s3);
}

template <typename T, class F>
__device__ __forceinline__ typename Tr<T>::V tree_sum(const F& fetch, int log_leaves) {
    switch (log_leaves) {
        case 0: return TreeSum<T, 0>::run(fetch, 0);
        case 1: return TreeSum<T, 1>::run(fetch, 0);
        case 2: return TreeSum<T, 2>::run(fetch, 0);
        case 3: return TreeSum<T, 3>::run(fetch, 0);
        default: return tree_sum_big<T>(fetch, log_leaves);
    }
}

// Averaging rule for every member of a plan (optim.py:439-452) given its sum.
// `own_wp(j)` returns this thread's W' of job j (only read for late members).
template <typename T, class OwnWp>
__device__ __forceinline__ void finish_members(const LaunchParams& p, const SmemCtl& sm, const DevPlan& P_,
                                               typename Tr<T>::V acc, int64_t idx, const OwnWp& own_wp) {
    using V = typename Tr<T>::V;
    // timely members share one result: acc/S or total/P (optim.py:442,452);
    // a power-of-two divisor is an exact reciprocal multiply (same IEEE result)
    const V avg = P_.divisor_pow2 ? vscale(T(1) / T(P_.divisor), acc) : vdiv(acc, T(P_.divisor));
    for (int mi = 0; mi < P_.n_members; ++mi) {
        const int j = P_.members[mi];
        const DevJob& jb = p.jobs[j];
        if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
            st_stream<T>(static_cast<T*>(jb.acc_out), idx, p.n, acc);
            continue;
        }
        const bool timely = jb.kind == WG_JOB_SYNC_STEP || sm.stamps[jb.vidx][jb.rank] == jb.version;
        // late member: (acc + W')/(S+1)  (optim.py:443-444), true IEEE division
        const V out = timely ? avg : vdiv(vadd(acc, own_wp(j)), T(P_.divisor + 1));
        st_stream<T>(static_cast<T*>(jb.W), idx, p.n, out);
    }
}

template <typename T>
__device__ bool consume_tile(const LaunchParams& p, SmemCtl& sm, int64_t tile, const typename Tr<T>::V* stage,
                             long long* poll_cycles = nullptr) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    constexpr int U = kVecPerThread;
    const int tid = threadIdx.x;
    const int64_t tbase = tile * p.tile_elems;
    for (int pl = 0; pl < p.n_plans; ++pl) {
        const DevPlan& P_ = p.plans[pl];
        if (sm.plan_polls[pl]) {
            const long long c0 = poll_cycles ? clock64() : 0;
            // wait until the peer warps that mirror this warp published
            // their part of the tile (per-warp flags, no CTA barrier)
            const int lane = tid & 31, w = tid >> 5;
            int rc = 0;
            for (int li = lane; li < P_.n_leaves; li += 32) {
                if (sm.leaf_src[pl][li] != kSrcPoll) continue;
                const int q = P_.leaves[li];
                const int64_t s = sm.stamps[P_.vidx][q];
                rc = spin_geq(p, flag_ptr(p, q, tile, w), s, globaltimer());
                if (rc) {
                    raise_error(p, rc, int64_t(q) << 32 | (tile & 0xffffffff));
                    sm.abort = 1;
                    break;
                }
            }
            __syncwarp();
            if (poll_cycles) *poll_cycles += clock64() - c0;
            if (__any_sync(0xffffffffu, rc != 0) || sm.abort) return false;
        }
        auto fetch = [&](int leaf) -> V {
            const int src = sm.leaf_src[pl][leaf];
            if (src >= 0) return stage[src * kThreads + tid];
            // 128-bit load of a peer's (NVLink) or an older local send slot;
            // .cg: L2 only, never a stale L1 line of a re-published slot.
            const T* base = ring_ptr<T>(p, P_.leaves[leaf], sm.leaf_slot[pl][leaf]) + tbase;
            return __ldcg(reinterpret_cast<const V*>(base + int64_t(tid) * E));
        };
        finish_members<T>(p, sm, P_, tree_sum<T>(fetch, P_.log_leaves), tbase + int64_t(tid) * E,
                          [&](int j) { return stage[j * kThreads + tid]; });
    }
    return true;
}

// ---------------------------------------------------------------------------
// the fused step kernel (persistent: grid <= co-resident CTAs)
// ---------------------------------------------------------------------------

template <typename T, bool AHEAD>
__global__ void __launch_bounds__(kThreads, AHEAD ? WG_MINB_AHEAD : WG_MINB) wagma_step_kernel(const __grid_constant__ LaunchParams p) {
    using V = typename Tr<T>::V;
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    V* stage = reinterpret_cast<V*>(dyn_smem);
    __shared__ SmemCtl sm;
    __shared__ T* s_ring[kMaxJobs];
    if (threadIdx.x == 0) sm.abort = 0;
    if (threadIdx.x < kMaxVersions) sm.activator[threadIdx.x] = 0;
    init_ring_slots<T>(p, s_ring);
    __syncthreads();
    if (blockIdx.x == 0) {
        if (threadIdx.x < 32) control_phase(p, sm.activator);
        __syncthreads();
    }
    bool resolved = false;
    unsigned my_tiles = 0;
    unsigned bad = 0;  // jobs whose W' was non-finite in this thread
    if constexpr (AHEAD) {
        V* stages[2] = {stage, stage + size_t(p.n_jobs) * kVecPerThread * kThreads};
        const bool prof = p.prof != nullptr && threadIdx.x == 0;
        long long cyc[6] = {0, 0, 0, 0, 0, 0};
        long long c0 = prof ? clock64() : 0;
        auto lap = [&](int i) {
            if (prof) {
                const long long c = clock64();
                cyc[i] += c - c0;
                c0 = c;
            }
        };
        int64_t tile = blockIdx.x;
        int buf = 0;
        if (tile < p.n_tiles) {
            produce_tile_regs<T>(p, tile, stages[0], s_ring, bad);
            lap(0);
            publish_tile(p, tile);
            lap(1);
            ++my_tiles;
        }
        while (tile < p.n_tiles) {
            const int64_t next = tile + gridDim.x;
            if (next < p.n_tiles) {
                produce_tile_regs<T>(p, next, stages[buf ^ 1], s_ring, bad);
                lap(0);
                publish_tile(p, next);
                lap(1);
                ++my_tiles;
            }
            if (!resolved) {
                if (!resolve_sources<T>(p, sm)) break;
                resolved = true;
                lap(2);
            }
            if (!consume_tile<T>(p, sm, tile, stages[buf], prof ? &cyc[3] : nullptr)) break;
            lap(4);
            tile = next;
            buf ^= 1;
        }
        if (prof) {
            cyc[4] -= cyc[3];
            for (int i = 0; i < 5; ++i) p.prof[blockIdx.x * 8 + i] = cyc[i];
            p.prof[blockIdx.x * 8 + 5] = my_tiles;
        }
    } else {
        // one GPU: nobody outside this CTA waits for its tiles
        const int J = p.n_jobs;
        V* ring = stage;  // [kDepth][3][kThreads], then the W' stage [J][kThreads]
        V* st = ring + kDepth * 3 * kThreads;
        const int64_t my_ntiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
#if WG_STEP_INCR
        // issue cursor (tile ik of this CTA, job ij) runs kDepth items ahead;
        // advanced incrementally (no 64-bit division per item)
        int64_t ik = 0;
        int ij = 0;
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
            if (ik < my_ntiles) issue_item<T>(p, int64_t(blockIdx.x) + ik * gridDim.x, ij, ring + d * 3 * kThreads);
            cp_async_commit();
            if (++ij == J) ij = 0, ++ik;
        }
        int rs = 0;
        for (int64_t kk = 0; kk < my_ntiles; ++kk) {
            const int64_t tile = int64_t(blockIdx.x) + kk * gridDim.x;
            for (int j = 0; j < J; ++j) {
                cp_async_wait<kDepth - 1>();
                V* slot = ring + rs * 3 * kThreads;
                bad |= unsigned(compute_item<T>(p, tile, j, slot, st, WG_STEP_SRING ? s_ring : nullptr)) << j;
                if (ik < my_ntiles) issue_item<T>(p, int64_t(blockIdx.x) + ik * gridDim.x, ij, slot);
                cp_async_commit();
                if (++ij == J) ij = 0, ++ik;
                if (++rs == kDepth) rs = 0;
            }
#else
        const int64_t n_items = my_ntiles * J;
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
            if (d < n_items)
                issue_item<T>(p, int64_t(blockIdx.x) + (d / J) * int64_t(gridDim.x), d % J, ring + d * 3 * kThreads);
            cp_async_commit();
        }
        int64_t i = 0;
        for (int64_t kk = 0; kk < my_ntiles; ++kk) {
            const int64_t tile = int64_t(blockIdx.x) + kk * gridDim.x;
            for (int j = 0; j < J; ++j, ++i) {
                cp_async_wait<kDepth - 1>();
                V* slot = ring + (i % kDepth) * 3 * kThreads;
                bad |= unsigned(compute_item<T>(p, tile, j, slot, st, WG_STEP_SRING ? s_ring : nullptr)) << j;
                const int64_t nx = i + kDepth;
                if (nx < n_items)
                    issue_item<T>(p, int64_t(blockIdx.x) + (nx / J) * int64_t(gridDim.x), int(nx % J), slot);
                cp_async_commit();
            }
#endif
            ++my_tiles;
            if (!resolved) {
                if (!resolve_sources<T>(p, sm)) break;
                resolved = true;
            }
            if (!consume_tile<T>(p, sm, tile, st)) break;
        }
        cp_async_wait<0>();
    }
    report_divergence(p, bad);
    publish_slots(p, sm.abort ? 0u : my_tiles);
    if (blockIdx.x == 0) {
        if (!resolved && !sm.abort) resolved = resolve_sources<T>(p, sm);
        __syncthreads();
        if (resolved && threadIdx.x < 32) check_sync_points(p, sm);
        __syncthreads();
        if (threadIdx.x < p.n_jobs) {
            const DevJob& jb = p.jobs[threadIdx.x];
            wg_job_status st;
            st.version = jb.version;
            st.contrib_stamp = (jb.kind == WG_JOB_LOCAL_STEP || !resolved) ? jb.version : sm.stamps[jb.vidx][jb.rank];
            st.timely = st.contrib_stamp == jb.version;
            st.root = activation_root(p, jb, resolved);
            st.activator = jb.vidx >= 0 && sm.activator[jb.vidx] && st.root == jb.rank;
            st.error = int32_t(ld_relaxed_sys(err_ptr(p)));
            p.status[threadIdx.x] = st;
        }
    }
}

// ---------------------------------------------------------------------------
// multi-GPU kernel: producer / puller / consumer warps
//
//  - 8 producer warps do the local step, install W' in the send ring and
//    publish a per-warp flag per tile; their inputs W, g, m come from an
//    issuer warp's TMA bulk copies into an mbarrier ring (>= 2 jobs per GPU,
//    tma_produce) or from per-thread cp.async rings (one job per GPU,
//    nvl_produce); they never wait on anything else, so they run ahead of the
//    pulls.
//  - 1 puller warp walks the same tiles: waits for every leaf's flag (peer
//    GPUs over NVLink, and this GPU's own producers), then fetches each
//    leaf-tile with one TMA bulk copy (cp.async.bulk global->shared; peer
//    memory is read over NVLink) into a deep shared-memory ring whose stages
//    are guarded by mbarriers (full: TMA bytes landed; empty: consumed).
//  - 8 consumer warps sum the leaves of each plan from shared memory in the
//    butterfly order and write W_{t+1}.
// One 576-thread CTA per SM (+ the issuer warp); stage count chosen from the
// shared-memory budget.
// ---------------------------------------------------------------------------

#ifndef WG_NVL_DEPTH
#define WG_NVL_DEPTH 5
#endif
#ifndef WG_NVL_TMA_LOCAL
#define WG_NVL_TMA_LOCAL 1
#endif
constexpr int kNvlDepth = WG_NVL_DEPTH;  // producer input ring (items): the TMA ring's stages
#ifndef WG_NVL_DEPTH_CPA
#define WG_NVL_DEPTH_CPA 3
#endif
constexpr int kNvlDepthCpa = WG_NVL_DEPTH_CPA < WG_NVL_DEPTH ? WG_NVL_DEPTH_CPA : WG_NVL_DEPTH;  // per-thread cp.async ring (one job per GPU)
#ifndef WG_SPLIT_DEPTH
#define WG_SPLIT_DEPTH 3
#endif
#ifndef WG_SPLIT_NSB
#define WG_SPLIT_NSB 16
#endif
constexpr int kSplitDepth = WG_SPLIT_DEPTH;  // producer ring depth in the split kernel
// split kernel: 1 = leaves on this GPU are TMA-copied into the stage like
// remote ones; 0 = reducers read them straight from L2 (they were produced
// by this CTA moments ago), and the shared memory goes to the producers
#ifndef WG_SPLIT_NSA_MIN  // stream-A stages reserved before stream B takes the rest
#define WG_SPLIT_NSA_MIN 4
#endif
#ifndef WG_SPLIT_ABATCH  // stream-A tiles per flag-poll batch (0: NSA - 1)
#define WG_SPLIT_ABATCH 0
#endif
#ifndef WG_SPLIT_TMA_LOCAL
#define WG_SPLIT_TMA_LOCAL 1
#endif
constexpr int kNvlMaxStages = 16;
// TMA-fed producers (an issuer warp streams the inputs by cp.async.bulk): in
// the pull kernel for launches of >= 2 jobs per GPU (measured 2 GPUs P=8 S=8
// 0.588 -> 0.552 ms with a 5-deep ring; one job per GPU stays on the cp.async
// rings, 0.235 vs 0.249 ms); not in the split kernel (4 GPUs S=8 0.450 vs 0.477)
#ifndef WG_TMA_PRODUCE
#define WG_TMA_PRODUCE 1
#endif
#ifndef WG_TMA_PRODUCE_SPLIT
#define WG_TMA_PRODUCE_SPLIT 0
#endif
constexpr int kNvlThreads = 2 * kThreads + 32 + (WG_TMA_PRODUCE ? 32 : 0);  // + TMA issuer warp
constexpr int kNvlMaxDyn = 200 * 1024;
constexpr int kPollPerLane = 8;
constexpr int kPullBatch = 8;  // tiles whose flags are polled and copies issued together
#ifndef WG_PUB_CHUNK
#define WG_PUB_CHUNK 8
#endif
constexpr int kPubChunk = WG_PUB_CHUNK;  // tiles published together (one fence per chunk)
constexpr int kPubRing = 16;   // per-chunk producer-completion counters (drift bound kPubRing/2 chunks)
constexpr int kRedRing = 32;   // per-tile reducer counters (reducers drift < kNvlMaxStages tiles)
constexpr int kMaxPoll = 32 * kPollPerLane;  // (leaf, warp) flags polled per tile

__device__ __forceinline__ unsigned smem_u32(const void* ptr) {
    return static_cast<unsigned>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Non-blocking test of an mbarrier phase (try_wait may suspend the thread
// for a while; a warp polling several barriers must not).
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred q;\n mbarrier.test_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Wait for an mbarrier phase with the watchdog; false on timeout / abort.
__device__ bool mbar_wait(const LaunchParams& p, uint64_t* bar, unsigned parity) {
    uint64_t t0 = 0;
    int it = 0;
    while (!mbar_try_wait(bar, parity)) {
        if ((++it & 255) == 0) {
            if (t0 == 0) {
                t0 = globaltimer();
            } else if (globaltimer() - t0 > uint64_t(p.timeout_ns)) {
                return false;
            }
            if (aborted(p)) return false;
        }
    }
    return true;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Same with an L2 cache policy (createpolicy), e.g. evict-first for inputs read once.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// ---------------------------------------------------------------------------
// single-GPU kernel: TMA producer warp, control warp, consumer warps
//
// All ranks of the launch live on this GPU, so nobody outside a CTA waits on
// its tiles and the step is a pure HBM stream: per chunk (kLocTiles tiles)
// and job, read W, g, m and write m, W' (send ring) and W_{t+1}.
//  - warp 0 (one elected lane) streams the inputs of every (chunk, job) item
//    with cp.async.bulk (TMA bulk copies, UBLKCP) into a ring of NS stages
//    guarded by mbarriers (full: bytes landed; empty: consumed), so the
//    bytes in flight per SM are set by the ring, not by registers;
//  - warp 1 runs the activation protocol (CTA 0) and resolves every plan's
//    leaves while the first items are being loaded and computed;
//  - the consumer warps compute the local step of each item from shared
//    memory, store m and the W' send-ring slot, keep W' in a thread-private
//    shared-memory stage, then sum each plan in the butterfly order and write
//    W_{t+1} (timely acc/S, late (acc + W')/(S+1), sync total/P).
// Every index is advanced incrementally (no 64-bit division per item).
// ---------------------------------------------------------------------------

#ifndef WG_LOC_TILES
#define WG_LOC_TILES 2
#endif
#ifndef WG_LOC_CONSUMER_WARPS
#define WG_LOC_CONSUMER_WARPS 16
#endif
#ifndef WG_LOC_EVICT_FIRST  // L2 evict-first policy on the TMA input loads (measured +1%)
#define WG_LOC_EVICT_FIRST 1
#endif
#ifndef WG_LOC_RING_CS  // send-ring stores evict-first (.cs) instead of .cg
#define WG_LOC_RING_CS 1
#endif
#ifndef WG_LOC_STACK  // 1: plans summed in registers in leaf order (no W' stage), shared memory all input ring
#define WG_LOC_STACK 0
#endif
constexpr int kLocTiles = WG_LOC_TILES;                    // tiles per chunk (per item)
constexpr int kLocConsumers = WG_LOC_CONSUMER_WARPS * 32;  // consumer threads
constexpr int kLocThreads = kLocConsumers + 64;            // + producer warp + control warp
constexpr int kLocChunkVecs = kLocTiles * kThreads;        // 16-byte vectors per row of a stage
constexpr int kLocVPT = kLocChunkVecs / kLocConsumers;     // vectors per consumer thread per item
constexpr int kLocMaxStages = 16;
constexpr int kMgMaxStagesA = 16, kMgMaxStagesB = 16;
static_assert(kLocChunkVecs % kLocConsumers == 0, "a chunk row must split evenly over the consumers");

// Per-job constants of the single-GPU kernel, staged in shared memory once
// (no per-item parameter-space loads or double -> float conversions).
template <typename T>
struct LocJob {
    T* W;
    T* m;
    const T* g;
    const T* fresh;
    T* ring;
    T eta, beta;
    int32_t kind, mom;
};

// Per-job constants staged in shared memory (thread j < n_jobs).
template <typename T>
__device__ __forceinline__ void init_loc_jobs(const LaunchParams& p, LocJob<T>* out) {
    const int j = threadIdx.x;
    if (j >= p.n_jobs) return;
    const DevJob& jb = p.jobs[j];
    LocJob<T> lj;
    lj.W = static_cast<T*>(jb.W);
    lj.m = static_cast<T*>(jb.m);
    lj.g = static_cast<const T*>(jb.g);
    lj.fresh = static_cast<const T*>(jb.fresh);
    lj.ring = jb.produces ? ring_ptr<T>(p, jb.rank, slot_of(p, jb.version)) : nullptr;
    lj.eta = T(jb.eta);
    lj.beta = T(jb.beta);
    lj.kind = jb.kind;
    lj.mom = jb.update_rule == WG_UPDATE_MOMENTUM;
    out[j] = lj;
}

// Consumer work for one item (job j of a chunk): local step, m and send-ring
// stores, W' into the thread-private stage. FULL: the chunk lies inside n.
template <typename T, bool FULL, int NT = kLocConsumers>
__device__ __forceinline__ unsigned loc_item(const LaunchParams& p, const LocJob<T>& jb, int j, int64_t e0,
                                             const typename Tr<T>::V* r, typename Tr<T>::V* wst, int ct,
                                             typename Tr<T>::V* out = nullptr) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    constexpr int VPT = kLocChunkVecs / NT;
    unsigned bad = 0;
    const bool sum = jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM;
#pragma unroll
    for (int kv = 0; kv < VPT; ++kv) {
        const int v = kv * NT + ct;
        const int64_t idx = e0 + int64_t(v) * E;
        const bool tail = !FULL && idx + E > p.n;  // ragged end: global loads, zero-filled
        V wp;
        if (sum) {
            wp = tail ? ld_tail(jb.fresh, idx, p.n) : r[v];
        } else {
            const V w = tail ? ld_tail(jb.W, idx, p.n) : r[v];
            const V g = tail ? ld_tail(jb.g, idx, p.n) : r[kLocChunkVecs + v];
            if (jb.mom) {
                // m = beta*m + g ; W' = W - eta*m  (optim.py:179,183)
                const V m0 = tail ? ld_tail(static_cast<const T*>(jb.m), idx, p.n) : r[2 * kLocChunkVecs + v];
                const V mn = vadd(vscale(jb.beta, m0), g);
                st_stream<T, FULL>(jb.m, idx, p.n, mn);
                wp = vsub(w, vscale(jb.eta, mn));
            } else {
                wp = vsub(w, vscale(jb.eta, g));  // W' = W - eta*g (optim.py:181-183)
            }
            bad |= unsigned(nonfinite(wp));
            if (jb.kind == WG_JOB_LOCAL_STEP) {
                st_stream<T, FULL>(jb.W, idx, p.n, wp);
                continue;
            }
        }
        // SendBuffer.install (collective.py:95-101): W' once into the ring
        if (FULL || idx < p.npad) {
            if (WG_LOC_RING_CS)
                __stcs(reinterpret_cast<V*>(jb.ring + idx), wp);
            else
                __stcg(reinterpret_cast<V*>(jb.ring + idx), wp);
        }
        if (wst) wst[j * kLocChunkVecs + v] = wp;
        if (out) out[kv] = wp;
    }
    return bad << j;
}

// Butterfly register stack: push leaf `pos` (its bits say which finished
// subtrees it closes); returns the combined value (the plan's sum at its
// last leaf). Same pairing as TreeSum (collective.py:310-329).
template <typename V, int U>
__device__ __forceinline__ void stack_push(V (&s)[5][U], V (&v)[U], int pos) {
#pragma unroll
    for (int k = 0; k < U; ++k) {
        if (pos & 1) {
            v[k] = vadd(s[0][k], v[k]);
            if (pos & 2) {
                v[k] = vadd(s[1][k], v[k]);
                if (pos & 4) {
                    v[k] = vadd(s[2][k], v[k]);
                    if (pos & 8) {
                        v[k] = vadd(s[3][k], v[k]);
                        s[4][k] = v[k];
                    } else {
                        s[3][k] = v[k];
                    }
                } else {
                    s[2][k] = v[k];
                }
            } else {
                s[1][k] = v[k];
            }
        } else {
            s[0][k] = v[k];
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kLocThreads, 1) wagma_local_kernel(const __grid_constant__ LaunchParams p) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    __shared__ SmemCtl sm;
    __shared__ LocJob<T> s_job[kMaxJobs];
    __shared__ __align__(8) uint64_t full[kLocMaxStages];
    __shared__ __align__(8) uint64_t empty[kLocMaxStages];
    __shared__ volatile int ready;
    // fast finish of a plan whose leaves are all this launch's W' and whose
    // members are all timely steps: W_{t+1} = avg for every member
    __shared__ int8_t s_fast[kMaxPlans];
    __shared__ int8_t s_leafjob[kMaxPlans][kMaxJobs];
    __shared__ int8_t s_nmem[kMaxPlans];
    __shared__ T* s_memW[kMaxPlans][kMaxJobs];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int J = p.n_jobs, NS = p.loc_stages;
    const int64_t chunk_elems = int64_t(kLocChunkVecs) * E;
    const int64_t n_chunks = (p.n_tiles + kLocTiles - 1) / kLocTiles;
    V* rows = reinterpret_cast<V*>(dyn_smem);               // [NS][3][kLocChunkVecs]: W, g, m of an item
    V* wst = WG_LOC_STACK ? nullptr : rows + size_t(NS) * 3 * kLocChunkVecs;  // [J][kLocChunkVecs]: W' of every job
    if (tid == 0) {
        sm.abort = 0;
        ready = 0;
        for (int st = 0; st < NS; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], kLocConsumers / 32);
        }
    }
    if (tid < kMaxVersions) sm.activator[tid] = 0;
    if (tid < J) {
        const DevJob& jb = p.jobs[tid];
        LocJob<T> lj;
        lj.W = static_cast<T*>(jb.W);
        lj.m = static_cast<T*>(jb.m);
        lj.g = static_cast<const T*>(jb.g);
        lj.fresh = static_cast<const T*>(jb.fresh);
        lj.ring = jb.produces ? ring_ptr<T>(p, jb.rank, slot_of(p, jb.version)) : nullptr;
        lj.eta = T(jb.eta);
        lj.beta = T(jb.beta);
        lj.kind = jb.kind;
        lj.mom = jb.update_rule == WG_UPDATE_MOMENTUM;
        s_job[tid] = lj;
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer: TMA bulk loads of every item ----------------
        if (lane == 0) {
            constexpr unsigned chunk_bytes = unsigned(kLocChunkVecs) * 16u;
            const uint64_t pol = WG_LOC_EVICT_FIRST ? policy_evict_first() : 0;
            auto load = [&](void* d, const T* src, unsigned nb, uint64_t* bar) {
                if (WG_LOC_EVICT_FIRST)
                    bulk_g2s_hint(d, src, nb, bar, pol);
                else
                    bulk_g2s(d, src, nb, bar);
            };
            int st = 0;
            unsigned ph = 0;
            int64_t k = 0;
            bool ok = true;
            for (int64_t c = blockIdx.x; c < n_chunks && ok; c += gridDim.x) {
                const int64_t e0 = c * chunk_elems;
                // caller vectors hold exactly n elements: whole 16-byte vectors by
                // TMA, the ragged end is read by the consumers from global memory
                const int64_t rem = (p.n - e0) * int64_t(sizeof(T));
                const unsigned bytes = rem >= chunk_bytes ? chunk_bytes : (rem > 0 ? unsigned(rem) & ~15u : 0u);
                for (int jj = 0; jj < J; ++jj, ++k) {
                    const int j = WG_LOC_STACK ? p.job_order[jj] : jj;
                    if (k >= NS && !mbar_wait(p, &empty[st], ph ^ 1u)) {
                        ok = false;
                        break;
                    }
                    const LocJob<T>& jb = s_job[j];
                    V* dst = rows + size_t(st) * 3 * kLocChunkVecs;
                    if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
                        mbar_arrive_expect_tx(&full[st], bytes);
                        if (bytes) load(dst, jb.fresh + e0, bytes, &full[st]);
                    } else {
                        mbar_arrive_expect_tx(&full[st], (jb.mom ? 3u : 2u) * bytes);
                        if (bytes) {
                            load(dst, jb.W + e0, bytes, &full[st]);
                            load(dst + kLocChunkVecs, jb.g + e0, bytes, &full[st]);
                            if (jb.mom) load(dst + 2 * kLocChunkVecs, jb.m + e0, bytes, &full[st]);
                        }
                    }
                    if (++st == NS) st = 0, ph ^= 1u;
                }
            }
            if (!ok) {
                raise_error(p, WG_ETIMEOUT, k);
                sm.abort = 1;
            }
        }
    } else if (warp == 1) {
        // ---------------- control: activation + leaf sources ----------------
        if (blockIdx.x == 0) control_phase(p, sm.activator);
        bool res = resolve_core<T>(p, sm, lane, 32, [] { __syncwarp(); });
        if (res && lane == 0) {
            // a leaf slot still being filled by an earlier launch (another
            // stream): wait until its launch completed the slot
            const uint64_t t0 = globaltimer();
            for (int pl = 0; pl < p.n_plans && res; ++pl)
                for (int li = 0; li < p.plans[pl].n_leaves && res; ++li) {
                    if (sm.leaf_src[pl][li] != kSrcPoll) continue;
                    const int q = p.plans[pl].leaves[li];
                    const int rc = spin_eq(p, complete_ptr(p, q, sm.leaf_slot[pl][li]),
                                           sm.stamps[p.plans[pl].vidx][q], t0);
                    if (rc) {
                        raise_error(p, rc, q);
                        sm.abort = 1;
                        res = false;
                    }
                    sm.leaf_src[pl][li] = kSrcReady;
                }
            // fast finish: every leaf staged here, every member a timely step
            for (int pl = 0; pl < p.n_plans; ++pl) {
                const DevPlan& P_ = p.plans[pl];
                bool fast = P_.n_leaves <= kMaxJobs;
                for (int li = 0; li < P_.n_leaves && fast; ++li) {
                    fast = sm.leaf_src[pl][li] >= 0;
                    if (fast) s_leafjob[pl][li] = sm.leaf_src[pl][li];
                }
                for (int mi = 0; mi < P_.n_members && fast; ++mi) {
                    const DevJob& jb = p.jobs[P_.members[mi]];
                    fast = (jb.kind == WG_JOB_STEP || jb.kind == WG_JOB_SYNC_STEP) &&
                           (jb.kind == WG_JOB_SYNC_STEP || sm.stamps[jb.vidx][jb.rank] == jb.version);
                    s_memW[pl][mi] = static_cast<T*>(jb.W);
                }
                s_nmem[pl] = int8_t(P_.n_members);
                s_fast[pl] = fast && P_.divisor_pow2 && (!WG_LOC_STACK || p.plan_hl[pl]);
            }
        }
        res = __shfl_sync(0xffffffffu, res, 0);
        if (lane == 0) {
            __threadfence_block();
            ready = res ? 1 : 2;
        }
    } else {
        // ---------------- consumers ----------------
        const int ct = tid - 64;
        unsigned bad = 0;
        int st = 0;
        unsigned ph = 0;
        bool ok = true, resolved = false;
        for (int64_t c = blockIdx.x; c < n_chunks && ok; c += gridDim.x) {
            const int64_t e0 = c * chunk_elems;
            const bool fullc = e0 + chunk_elems <= p.n;
#if WG_LOC_STACK
            // jobs in the host's leaf order: each plan's sum builds up in a
            // register stack and is finished at its last leaf
            V stk[5][kLocVPT];
            for (int jj = 0; jj < J; ++jj) {
                const int j = p.job_order[jj];
                if (!mbar_wait(p, &full[st], ph)) {
                    ok = false;
                    break;
                }
                const V* r = rows + size_t(st) * 3 * kLocChunkVecs;
                V wp[kLocVPT];
                if (fullc)
                    bad |= loc_item<T, true>(p, s_job[j], j, e0, r, nullptr, ct, wp);
                else
                    bad |= loc_item<T, false>(p, s_job[j], j, e0, r, nullptr, ct, wp);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == NS) st = 0, ph ^= 1u;
                const int pl = p.job_part[jj];
                if (pl < 0) continue;
                stack_push<V, kLocVPT>(stk, wp, p.job_ppos[jj]);
                if (!p.job_plast[jj]) continue;
                if (!resolved) {
                    while (ready == 0) __nanosleep(32);
                    __threadfence_block();
                    if (ready != 1) {
                        ok = false;
                        break;
                    }
                    resolved = true;
                }
                if (fullc && s_fast[pl]) {
                    // every member timely: one average, stored to each replica
                    const T inv = T(1) / T(p.plans[pl].divisor);
                    const int nm = s_nmem[pl];
#pragma unroll
                    for (int kv = 0; kv < kLocVPT; ++kv) {
                        const int64_t idx = e0 + int64_t(kv * kLocConsumers + ct) * E;
                        const V avg = vscale(inv, wp[kv]);
                        for (int mi = 0; mi < nm; ++mi) __stcs(reinterpret_cast<V*>(s_memW[pl][mi] + idx), avg);
                    }
                }
            }
            if (!ok) break;
            if (!resolved) {
                while (ready == 0) __nanosleep(32);
                __threadfence_block();
                if (ready != 1) break;
                resolved = true;
            }
            // plans not finished from the stack: the generic sum, W' read
            // back from the send slots this thread wrote
            for (int pl = 0; pl < p.n_plans; ++pl) {
                if (fullc && s_fast[pl]) continue;
                const DevPlan& P_ = p.plans[pl];
#pragma unroll
                for (int kv = 0; kv < kLocVPT; ++kv) {
                    const int v = kv * kLocConsumers + ct;
                    const int64_t idx = e0 + int64_t(v) * E;
                    if (idx >= p.npad) continue;
                    auto fetch = [&](int leaf) -> V {
                        const int src = sm.leaf_src[pl][leaf];
                        if (src >= 0) return __ldcg(reinterpret_cast<const V*>(s_job[src].ring + idx));
                        return __ldcg(reinterpret_cast<const V*>(
                            ring_ptr<T>(p, P_.leaves[leaf], sm.leaf_slot[pl][leaf]) + idx));
                    };
                    finish_members<T>(p, sm, P_, tree_sum<T>(fetch, P_.log_leaves), idx, [&](int j) {
                        return __ldcg(reinterpret_cast<const V*>(s_job[j].ring + idx));
                    });
                }
            }
            continue;
#endif
            for (int j = 0; j < J; ++j) {
                if (!mbar_wait(p, &full[st], ph)) {
                    ok = false;
                    break;
                }
                const V* r = rows + size_t(st) * 3 * kLocChunkVecs;
                if (fullc)
                    bad |= loc_item<T, true>(p, s_job[j], j, e0, r, wst, ct);
                else
                    bad |= loc_item<T, false>(p, s_job[j], j, e0, r, wst, ct);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == NS) st = 0, ph ^= 1u;
            }
            if (!ok) break;
            if (!resolved) {
                while (ready == 0) __nanosleep(32);
                __threadfence_block();
                if (ready != 1) break;
                resolved = true;
            }
            // group sums in the butterfly order + the averaging rule
            for (int pl = 0; pl < p.n_plans; ++pl) {
                const DevPlan& P_ = p.plans[pl];
                if (fullc && s_fast[pl]) {
                    // every member timely: one average, stored to each replica
                    const T inv = T(1) / T(P_.divisor);
                    const int nm = s_nmem[pl];
#pragma unroll
                    for (int kv = 0; kv < kLocVPT; ++kv) {
                        const int v = kv * kLocConsumers + ct;
                        const int64_t idx = e0 + int64_t(v) * E;
                        auto fetch = [&](int leaf) -> V { return wst[s_leafjob[pl][leaf] * kLocChunkVecs + v]; };
                        const V avg = vscale(inv, tree_sum<T>(fetch, P_.log_leaves));
                        for (int mi = 0; mi < nm; ++mi) __stcs(reinterpret_cast<V*>(s_memW[pl][mi] + idx), avg);
                    }
                    continue;
                }
#pragma unroll
                for (int kv = 0; kv < kLocVPT; ++kv) {
                    const int v = kv * kLocConsumers + ct;
                    const int64_t idx = e0 + int64_t(v) * E;
                    if (idx >= p.npad) continue;
                    auto fetch = [&](int leaf) -> V {
                        const int src = sm.leaf_src[pl][leaf];
                        if (src >= 0) return wst[src * kLocChunkVecs + v];
                        // an older send slot (stale member): L2 / HBM
                        return __ldcg(reinterpret_cast<const V*>(
                            ring_ptr<T>(p, P_.leaves[leaf], sm.leaf_slot[pl][leaf]) + idx));
                    };
                    finish_members<T>(p, sm, P_, tree_sum<T>(fetch, P_.log_leaves), idx,
                                      [&](int j) { return wst[j * kLocChunkVecs + v]; });
                }
            }
        }
        if (!ok) {
            if (lane == 0) raise_error(p, WG_ETIMEOUT, blockIdx.x);
            sm.abort = 1;
        }
        report_divergence(p, bad);
    }
    unsigned my_tiles = 0;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x)
        my_tiles += unsigned(p.n_tiles - c * kLocTiles < kLocTiles ? p.n_tiles - c * kLocTiles : kLocTiles);
    __syncthreads();
    if (ready != 1) sm.abort = 1;
    publish_slots(p, sm.abort ? 0u : my_tiles);
    if (blockIdx.x == 0) {
        __syncthreads();
        const bool res = ready == 1;
        if (res && threadIdx.x < 32) check_sync_points(p, sm);
        __syncthreads();
        if (tid < p.n_jobs) {
            const DevJob& jb = p.jobs[tid];
            wg_job_status stt;
            stt.version = jb.version;
            stt.contrib_stamp = (jb.kind == WG_JOB_LOCAL_STEP || !res) ? jb.version : sm.stamps[jb.vidx][jb.rank];
            stt.timely = stt.contrib_stamp == jb.version;
            stt.root = activation_root(p, jb, res);
            stt.activator = jb.vidx >= 0 && sm.activator[jb.vidx] && stt.root == jb.rank;
            stt.error = int32_t(ld_relaxed_sys(err_ptr(p)));
            p.status[tid] = stt;
        }
    }
}

// ---------------------------------------------------------------------------
// multi-GPU kernel with hierarchical sums on the TMA produce path
//
// The single-GPU kernel's produce side (TMA input ring, consumer warps
// computing W' from shared memory) plus the exchange, chunk by chunk:
//  - produce(c): W' of every job (m and send-ring stores), this GPU's
//    subtree partials (butterfly order) stored for the peers, then one fence
//    and the chunk's readiness flags (leaf flags of every produced rank,
//    partial flags);
//  - phase 1 (chunk c - kMgLag1): plans summed here -- leaf pull, partial
//    pull, or the chunks this GPU owns of a split (reduce-scatter) plan,
//    whose reduced chunk is stored and flagged for the other members;
//  - phase 2 (chunk c - kMgLag2): split plans owned elsewhere: the owner's
//    reduced chunk. Phase 1 never waits on another GPU's phase 1 or 2, so
//    no wait cycle exists.
// Warp 0 streams the inputs by TMA; warp 1 runs the activation protocol,
// resolves every plan's effective leaves (partials when all members are
// timely) and streams phase-1 rows (peers' partials/leaves over NVLink,
// this GPU's from L2); warp 2 streams phase-2 rows (owners' reduced
// chunks). The consumers never poll a flag.
// ---------------------------------------------------------------------------

#ifndef WG_MG_LAG1
#define WG_MG_LAG1 2
#endif
#ifndef WG_MG_LAG2
#define WG_MG_LAG2 4
#endif
#ifndef WG_MG_DIRECT_LOCAL  // 1: this GPU's partials read by the finishers from L2, else TMA rows
#define WG_MG_DIRECT_LOCAL 1
#endif
#ifndef WG_MG_SELF_PUB  // 1: the last producer warp of a chunk publishes it (the publisher warp only reduced chunks)
#define WG_MG_SELF_PUB 0
#endif
#ifndef WG_MG_IN_STAGES_MAX  // deepest input ring tried (the launch takes the deepest that fits)
#define WG_MG_IN_STAGES_MAX 5
#endif
#ifndef WG_MG_PUB_BATCH
#define WG_MG_PUB_BATCH 1
#endif
constexpr int kMgLag1 = WG_MG_LAG1, kMgLag2 = WG_MG_LAG2;
constexpr int kMgPubBatch = WG_MG_PUB_BATCH;  // chunks published per fence (< kMgPub)
#ifndef WG_MG_PROD_WARPS
#define WG_MG_PROD_WARPS 8
#endif
#ifndef WG_MG_FIN_WARPS
#define WG_MG_FIN_WARPS 8
#endif
constexpr int kMgProd = WG_MG_PROD_WARPS * 32;  // producer threads (W', partials)
constexpr int kMgFin = WG_MG_FIN_WARPS * 32;    // finisher threads (phase 1 and 2)
// role warps: input TMA, control/phase-1 puller, phase-2 puller, publisher
constexpr int kMgRoleWarps = 4;
constexpr int kMgThreads = kMgRoleWarps * 32 + kMgProd + kMgFin;
constexpr int kMgPub = 8;                         // chunks in flight between the consumers and the publisher
constexpr int kMgMaxEff = 16;                   // effective leaves per plan
enum MgMode : int8_t { kMgPull = 0, kMgHier = 1, kMgSplit = 2 };

template <typename T>
__global__ void __launch_bounds__(kMgThreads, 1) wagma_mg_kernel(const __grid_constant__ LaunchParams p) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    __shared__ SmemCtl sm;
    __shared__ LocJob<T> s_job[kMaxJobs];
    __shared__ __align__(8) uint64_t fin[kLocMaxStages], ein[kLocMaxStages];     // input ring
    __shared__ __align__(8) uint64_t fa[kMgMaxStagesA], ea[kMgMaxStagesA];       // phase-1 rows
    __shared__ __align__(8) uint64_t fb[kMgMaxStagesB], eb[kMgMaxStagesB];       // phase-2 rows
    __shared__ volatile int ready;
    // chunks of this CTA whose W' (every job) and partials the producers have
    // stored: the finishers read this launch's own W' (late members) and
    // this GPU's sources straight from L2 only below this count
    __shared__ volatile long long s_produced;
    __shared__ int s_nsa, s_nsb, s_rows_a, s_rows_b;
    // consumers -> publisher: chunk produced (pd) / owned chunk reduced (rd); acks (pk, rk)
    __shared__ __align__(8) uint64_t pd[kMgPub], pk[kMgPub], rd[kMgPub], rk[kMgPub];
    // WG_MG_SELF_PUB: per-chunk arrival counters of the producer warps (the
    // last warp to finish a chunk fences and raises its flags)
    __shared__ unsigned s_pubcnt[kPubRing];
    // local partials: buffers, flags and their leaf jobs in leaf order
    __shared__ T* s_part[kMaxJobs];
    __shared__ int64_t* s_pflag[kMaxJobs];
    __shared__ int8_t s_pjob[kMaxJobs][16];
    __shared__ int8_t s_plog[kMaxJobs];
    // per plan, after lock-in: mode, effective leaves (sources and flags)
    __shared__ int8_t s_mode[kMaxPlans], s_elog[kMaxPlans], s_ne[kMaxPlans];
    __shared__ const T* s_esrc[kMaxPlans][kMgMaxEff];       // effective leaf buffers (tile 0)
    __shared__ const int64_t* s_eflag[kMaxPlans][kMgMaxEff];  // their flags (tile 0)
    __shared__ int8_t s_estride[kMaxPlans][kMgMaxEff];      // flag words per tile (kWarps: leaf, 1: partial)
    __shared__ int64_t s_ewant[kMaxPlans][kMgMaxEff];
    __shared__ T* s_red[kMaxPlans][kMgMaxEff];              // split: reduced-chunk buffer of owner u
    __shared__ int64_t* s_redflag[kMaxPlans][kMgMaxEff];
    __shared__ int8_t s_ownlocal[kMaxPlans][kMgMaxEff];
    __shared__ int8_t s_erow[kMaxPlans][kMgMaxEff];        // row of the effective leaf in the chunk's rows, -1: read from L2
    __shared__ int8_t s_nrow[kMaxPlans];
    __shared__ int64_t s_ver[kMaxPlans];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int J = p.n_jobs, NSI = p.loc_stages, NP = p.n_plans;
    // optional per-CTA cycle counters (tools/phase_profile.py, WG_PROF_MG=1): 16 slots
    const long long kt0 = clock64();
    auto prof_add = [&](int slot, long long v) {
        if (p.prof) p.prof[blockIdx.x * 16 + slot] += v;
    };
    constexpr int C = kLocChunkVecs;
    const int64_t chunk_elems = int64_t(C) * E;
    const int64_t n_chunks = (p.n_tiles + kLocTiles - 1) / kLocTiles;
    const int64_t my_nchunks = blockIdx.x < n_chunks ? (n_chunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    V* rows_in = reinterpret_cast<V*>(dyn_smem);              // [NSI][3][C]
    V* wst = rows_in + size_t(NSI) * 3 * C;                   // [J][C]
    V* rows_a = wst + size_t(J) * C;                          // [mg_cap_a][C]
    V* rows_b = rows_a + size_t(p.mg_cap_a) * C;              // [mg_cap_b][C]
    if (tid == 0) {
        sm.abort = 0;
        ready = 0;
        s_produced = 0;
        for (int q = 0; q < kPubRing; ++q) s_pubcnt[q] = 0;
        for (int st = 0; st < NSI; ++st) {
            mbar_init(&fin[st], 1);
            mbar_init(&ein[st], kMgProd / 32);
        }
        for (int st = 0; st < kMgMaxStagesA; ++st) {
            mbar_init(&fa[st], 1);
            mbar_init(&ea[st], kMgFin / 32);
        }
        for (int st = 0; st < kMgMaxStagesB; ++st) {
            mbar_init(&fb[st], 1);
            mbar_init(&eb[st], kMgFin / 32);
        }
        for (int k = 0; k < kMgPub; ++k) {
            mbar_init(&pd[k], kMgProd / 32);
            mbar_init(&rd[k], kMgFin / 32);
            mbar_init(&pk[k], 1);
            mbar_init(&rk[k], 1);
        }
        for (int k = 0; k < J; ++k) {  // the producers' job order -> partial leaf lists
            const int pid = p.job_part[k];
            if (pid >= 0) {
                s_pjob[pid][p.job_ppos[k]] = p.job_order[k];
                if (p.job_plast[k]) s_plog[pid] = int8_t(31 - __clz(p.job_ppos[k] + 1));
            }
        }
    }
    if (tid < kMaxVersions) sm.activator[tid] = 0;
    if (tid < J) {
        const DevJob& jb = p.jobs[tid];
        LocJob<T> lj;
        lj.W = static_cast<T*>(jb.W);
        lj.m = static_cast<T*>(jb.m);
        lj.g = static_cast<const T*>(jb.g);
        lj.fresh = static_cast<const T*>(jb.fresh);
        lj.ring = jb.produces ? ring_ptr<T>(p, jb.rank, slot_of(p, jb.version)) : nullptr;
        lj.eta = T(jb.eta);
        lj.beta = T(jb.beta);
        lj.kind = jb.kind;
        lj.mom = jb.update_rule == WG_UPDATE_MOMENTUM;
        s_job[tid] = lj;
    }
    if (tid < p.n_parts) {
        s_part[tid] = part_ptr<T>(p, p.part_key[tid], p.part_version[tid]);
        s_pflag[tid] = part_flag_ptr(p, p.part_key[tid], 0);
    }
    __syncthreads();
    const unsigned chunk_bytes_full = unsigned(C) * 16u;
    // padded buffers (send ring, partials, reduced chunks): bytes of chunk kc
    auto pad_bytes = [&](int64_t c) -> unsigned {
        const int64_t t0 = c * kLocTiles;
        const int64_t nt = p.n_tiles - t0 < kLocTiles ? p.n_tiles - t0 : kLocTiles;
        return unsigned(nt * p.tile_elems * int64_t(sizeof(T)));
    };
    // owner (effective-leaf index) of chunk kc of a split plan
    auto owner = [&](int pl, int64_t kc) -> int { return int(kc % s_ne[pl]); };
    auto c_of = [&](int64_t kc) -> int64_t { return int64_t(blockIdx.x) + kc * gridDim.x; };
    // phase 1 of plan pl on CTA-local chunk kc (everything but split chunks owned elsewhere)
    auto ph1 = [&](int pl, int64_t kc) -> bool { return s_mode[pl] != kMgSplit || s_ownlocal[pl][owner(pl, kc)]; };
    // phase-1 TMA rows of chunk kc (-1: no phase 1), phase-2 rows (-1: none)
    auto rows_a_of = [&](int64_t kc) -> int {
        int ra = -1;
        for (int pl = 0; pl < NP; ++pl)
            if (ph1(pl, kc)) ra = (ra < 0 ? 0 : ra) + s_nrow[pl];
        return ra;
    };
    auto rows_b_of = [&](int64_t kc) -> int {
        int rb = 0;
        for (int pl = 0; pl < NP; ++pl) rb += !ph1(pl, kc);
        return rb ? rb : -1;
    };
    // phase-1 sources of chunk kc in a fixed order: visit(flag, stride, want, src, row or -1)
    auto srcs_a = [&](int64_t kc, auto&& visit) {
        int e = 0;
        for (int pl = 0; pl < NP; ++pl) {
            if (!ph1(pl, kc)) continue;
            for (int u = 0; u < s_ne[pl]; ++u)
                visit(s_eflag[pl][u], int(s_estride[pl][u]), s_ewant[pl][u], s_esrc[pl][u],
                      s_erow[pl][u] >= 0 ? e + s_erow[pl][u] : -1);
            e += s_nrow[pl];
        }
    };
    // phase-2 sources: the owners' reduced chunks
    auto srcs_b = [&](int64_t kc, auto&& visit) {
        int e = 0;
        for (int pl = 0; pl < NP; ++pl) {
            if (ph1(pl, kc)) continue;
            const int o = owner(pl, kc);
            visit(static_cast<const int64_t*>(s_redflag[pl][o]), 1, s_ver[pl], static_cast<const T*>(s_red[pl][o]), e++);
        }
    };
    // One non-blocking look at the flags >= want of one source over chunk c's
    // tiles (acquire loads): 1 ready, 0 not yet, -code on a protocol fault.
    auto probe = [&](const int64_t* f0, int stride, int64_t want, int64_t c) -> int {
        if (want == kNever) return 1;  // a completed older slot (checked at resolve)
        const int64_t t0 = c * kLocTiles;
        const int nt = int(p.n_tiles - t0 < kLocTiles ? p.n_tiles - t0 : kLocTiles);
        int ready = 1;
        for (int t = 0; t < nt; ++t)
            for (int w = 0; w < stride; ++w) {
                const int64_t* a = f0 + (t0 + t) * stride + w;
                int64_t x;
                if (p.fence_scope == 0)
                    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(x) : "l"(a) : "memory");
                else
                    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(x) : "l"(a) : "memory");
                if (x < want) ready = 0;
                else if (x >= want + p.D) return -WG_EPROTO;
            }
        return ready;
    };
    // Sliding-window puller (warps 1 and 2). Chunks in CTA order, up to W of
    // them in a window; the window's (chunk, source) pairs are dealt to the
    // lanes round-robin, so every lane probes about one flag set per sweep
    // (all in flight at once) and issues the TMA row copy of its pairs. A
    // chunk is delivered as soon as every pair of it and of every earlier
    // chunk was seen ready -- never held back by a later chunk's flags: on
    // another GPU a later chunk may wait, through its owner's reduce, on this
    // GPU consuming the earlier one (no wait cycle).
    auto puller = [&](int NS, V* rows, int rows_per_stage, uint64_t* full, uint64_t* empty, auto&& nrows,
                      auto&& srcs) -> bool {
        const int W = NS < kPullBatch ? NS : kPullBatch;
        int st = 0;
        unsigned ph = 0;
        int64_t k = 0, kc = 0;
        for (;;) {
            int64_t bk[kPullBatch];
            int nb = 0;
            while (kc < my_nchunks && nb < W) {
                if (nrows(kc) >= 0) bk[nb++] = kc;
                ++kc;
            }
            if (!nb) return true;
            int done = 0, spins = 0;
            unsigned seen = 0;  // this lane's pairs seen ready (bit = pair index / 32)
            const uint64_t t0 = globaltimer();
            while (done < nb) {
                int rc = 0, first = nb, qg = 0;
                for (int b = 0; b < nb; ++b) {
                    const int64_t c = c_of(bk[b]);
                    srcs(bk[b], [&](const int64_t* f, int stride, int64_t want, const T*, int) {
                        const int q = qg++;
                        if ((q & 31) != lane || b < done || (q < 1024 && ((seen >> (q >> 5)) & 1u))) return;
                        const int r = probe(f, stride, want, c);
                        if (r < 0)
                            rc = -r;
                        else if (r > 0)
                            seen |= q < 1024 ? 1u << (q >> 5) : 0u;
                        else if (b < first)
                            first = b;
                    });
                }
                if (rc) raise_error(p, rc, bk[done]);
                if (__any_sync(0xffffffffu, rc != 0)) return false;
                const int rdy = __reduce_min_sync(0xffffffffu, first);
                if (rdy == done) {
                    if ((++spins & 63) == 0 && (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p))) {
                        if (lane == 0) raise_error(p, WG_ETIMEOUT, bk[done]);
                        return false;
                    }
                    __nanosleep(32);
                    continue;
                }
                // the flags were read with acquire loads; order them before the
                // async-proxy (TMA) reads of the data they guard
                asm volatile("fence.proxy.async.global;" ::: "memory");
                qg = 0;
                for (int b = 0; b < rdy; ++b) {
                    if (b < done) {  // keep the pair numbering of the window
                        srcs(bk[b], [&](const int64_t*, int, int64_t, const T*, int) { ++qg; });
                        continue;
                    }
                    if (k >= NS && !mbar_wait(p, &empty[st], ph ^ 1u)) {
                        if (lane == 0) raise_error(p, WG_ETIMEOUT, bk[b]);
                        return false;
                    }
                    const int64_t c = c_of(bk[b]);
                    const unsigned cb = pad_bytes(c);
                    if (lane == 0) mbar_arrive_expect_tx(&full[st], unsigned(nrows(bk[b])) * cb);
                    __syncwarp();
                    srcs(bk[b], [&](const int64_t*, int, int64_t, const T* src, int row) {
                        if ((qg++ & 31) == lane && row >= 0)
                            bulk_g2s(rows + (size_t(st) * rows_per_stage + row) * C, src + c * chunk_elems, cb, &full[st]);
                    });
                    __syncwarp();
                    if (++st == NS) st = 0, ph ^= 1u;
                    ++k;
                }
                done = rdy;
            }
        }
    };
    auto fence_pub = [&]() {
        if (p.fence_scope == 0)
            fence_sys();
        else if (p.fence_scope == 1)
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
    };

    if (warp == 0) {
        // ---------------- input producer (TMA) ----------------
        if (lane == 0) {
            const uint64_t pol = WG_LOC_EVICT_FIRST ? policy_evict_first() : 0;
            auto load = [&](void* d, const T* src, unsigned nb, uint64_t* bar) {
                if (WG_LOC_EVICT_FIRST)
                    bulk_g2s_hint(d, src, nb, bar, pol);
                else
                    bulk_g2s(d, src, nb, bar);
            };
            int st = 0;
            unsigned ph = 0;
            int64_t k = 0;
            bool ok = true;
            for (int64_t c = blockIdx.x; c < n_chunks && ok; c += gridDim.x) {
                const int64_t e0 = c * chunk_elems;
                const int64_t rem = (p.n - e0) * int64_t(sizeof(T));
                const unsigned bytes = rem >= chunk_bytes_full ? chunk_bytes_full : (rem > 0 ? unsigned(rem) & ~15u : 0u);
                for (int jj = 0; jj < J; ++jj, ++k) {
                    const int j = p.job_order[jj];
                    const long long w0 = p.prof ? clock64() : 0;
                    if (k >= NSI && !mbar_wait(p, &ein[st], ph ^ 1u)) {
                        ok = false;
                        break;
                    }
                    if (p.prof) prof_add(12, clock64() - w0);
                    const LocJob<T>& jb = s_job[j];
                    V* dst = rows_in + size_t(st) * 3 * C;
                    if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
                        mbar_arrive_expect_tx(&fin[st], bytes);
                        if (bytes) load(dst, jb.fresh + e0, bytes, &fin[st]);
                    } else {
                        mbar_arrive_expect_tx(&fin[st], (jb.mom ? 3u : 2u) * bytes);
                        if (bytes) {
                            load(dst, jb.W + e0, bytes, &fin[st]);
                            load(dst + C, jb.g + e0, bytes, &fin[st]);
                            if (jb.mom) load(dst + 2 * C, jb.m + e0, bytes, &fin[st]);
                        }
                    }
                    if (++st == NSI) st = 0, ph ^= 1u;
                }
            }
            if (!ok) {
                raise_error(p, WG_ETIMEOUT, k);
                sm.abort = 1;
            }
            prof_add(13, clock64() - kt0);
        }
    } else if (warp == 1) {
        // ---------------- control + phase-1 puller ----------------
        if (blockIdx.x == 0) control_phase(p, sm.activator);
        bool res = resolve_core<T>(p, sm, lane, 32, [] { __syncwarp(); });
        if (res && lane == 0) {
            int ra_max = 0, rb_max = 0;
            for (int pl = 0; pl < NP; ++pl) {
                const DevPlan& P_ = p.plans[pl];
                const int64_t v = p.versions[P_.vidx].version;
                s_ver[pl] = v;
                bool hier = p.plan_hl[pl] > 0;
                for (int li = 0; li < P_.n_leaves && hier; ++li) hier = sm.stamps[P_.vidx][P_.leaves[li]] == v;
                int nr = 0;
                if (hier) {
                    const int hl = p.plan_hl[pl];
                    const int ne = P_.n_leaves >> hl;
                    unsigned gpus = 0;
                    for (int u = 0; u < ne; ++u) {
                        const int key = P_.leaves[u << hl];
                        gpus |= 1u << (key / p.R);
                        s_esrc[pl][u] = part_ptr<T>(p, key, v);
                        s_eflag[pl][u] = part_flag_ptr(p, key, 0);
                        s_estride[pl][u] = 1;
                        s_ewant[pl][u] = v;
                        s_red[pl][u] = red_ptr<T>(p, key, v);
                        s_redflag[pl][u] = red_flag_ptr(p, key, 0);
                        s_ownlocal[pl][u] = int8_t(key / p.R == p.gpu_index);
                        // this GPU's partials: read by the finishers from L2 (stored
                        // moments ago); only the peers' partials take TMA rows
                        s_erow[pl][u] = (WG_MG_DIRECT_LOCAL && s_ownlocal[pl][u]) ? int8_t(-1) : int8_t(nr++);
                    }
                    s_ne[pl] = int8_t(ne);
                    s_elog[pl] = int8_t(P_.log_leaves - hl);
                    s_mode[pl] = (p.mg_split && split_pays(ne, __popc(gpus))) ? kMgSplit : kMgHier;
                } else {
                    // leaf pull (a member is stale): every leaf's send slot; this
                    // GPU's leaves are read from L2 / HBM, the peers' by TMA
                    for (int li = 0; li < P_.n_leaves; ++li) {
                        const int q = P_.leaves[li];
                        const int64_t st = sm.stamps[P_.vidx][q];
                        s_esrc[pl][li] = ring_ptr<T>(p, q, slot_of(p, st));
                        s_eflag[pl][li] = flag_ptr(p, q, 0, 0);
                        s_estride[pl][li] = kWarps;
                        s_ewant[pl][li] = sm.leaf_src[pl][li] == kSrcReady ? kNever : st;
                        s_ownlocal[pl][li] = 1;
                        s_erow[pl][li] = q / p.R == p.gpu_index ? int8_t(-1) : int8_t(nr++);
                    }
                    s_ne[pl] = int8_t(P_.n_leaves);
                    s_elog[pl] = int8_t(P_.log_leaves);
                    s_mode[pl] = kMgPull;
                }
                s_nrow[pl] = int8_t(nr);
                ra_max += s_nrow[pl];
                rb_max += s_mode[pl] == kMgSplit;
            }
            s_rows_a = ra_max > 0 ? ra_max : 1;
            s_rows_b = rb_max;
            s_nsa = ra_max ? (p.mg_cap_a / ra_max < kMgMaxStagesA ? p.mg_cap_a / ra_max : kMgMaxStagesA) : kMgMaxStagesA;
            s_nsb = rb_max ? (p.mg_cap_b / rb_max < kMgMaxStagesB ? p.mg_cap_b / rb_max : kMgMaxStagesB) : kMgMaxStagesB;
            if (s_nsa < 1 || s_nsb < 1) {
                raise_error(p, WG_EINVAL, ra_max);
                res = false;
            }
        }
        res = __shfl_sync(0xffffffffu, res, 0);
        if (lane == 0) {
            __threadfence_block();
            ready = res ? 1 : 2;
            prof_add(11, clock64() - kt0);
        }
        __syncwarp();
        if (res) puller(s_nsa, rows_a, s_rows_a, fa, ea, rows_a_of, srcs_a);
        if (lane == 0) prof_add(7, clock64() - kt0);
    } else if (warp == 2) {
        // ---------------- phase-2 puller: owners' reduced chunks ----------------
        while (ready == 0) __nanosleep(64);
        __threadfence_block();
        if (ready == 1 && s_rows_b) puller(s_nsb, rows_b, s_rows_b, fb, eb, rows_b_of, srcs_b);
    } else if (warp == 3) {
        // ---------------- publisher: fences and readiness flags ----------------
        // Two independent streams, polled (never a blocking wait on one while
        // the other is ready):
        //  - produced chunks: once every producer warp arrived, one fence
        //    (cumulative over their stores, acquired through the mbarrier),
        //    then the chunk's flags (leaf flags of every produced rank, partial
        //    flags). This depends on nothing but this CTA's producers, so
        //    production is published whatever the peers do;
        //  - owned reduced chunks (split plans): after the finishers' arrival,
        //    one fence, then the reduced-chunk flags.
        // No producer or finisher ever waits on a fence.
        int64_t i = 0, x1 = 0, nown = 0;
        int rmode = 0;  // reduce stream: 0 waiting for lock-in, 1 active, 2 done / none
        uint64_t t0 = globaltimer();
        int spins = 0;
        if (WG_MG_SELF_PUB) i = my_nchunks;  // the producers publish their own chunks
        while (i < my_nchunks || rmode < 2) {
            bool prog = false;
            // every produced chunk whose producers all arrived: one fence for the run
            int64_t i1 = i;
            if (lane == 0)
                while (i1 < my_nchunks && i1 - i < WG_PUB_GATHER_P &&
                       mbar_test_wait(&pd[int(i1 % kMgPub)], unsigned((i1 / kMgPub) & 1)))
                    ++i1;
            i1 = __shfl_sync(0xffffffffu, i1, 0);
            if (i1 > i) {
                prog = true;
                if (lane == 0) {  // the producers' stores (acquired through pd) before the count
                    __threadfence_block();
                    s_produced = i1;
                }
                const long long w1 = clock64();
                if (lane == 0) fence_pub();
                __syncwarp();
                if (lane == 0 && p.prof) prof_add(9, clock64() - w1);
                for (int64_t b = i; b < i1; ++b) {
                    const int64_t tb = c_of(b) * kLocTiles;
                    const int nt = int(p.n_tiles - tb < kLocTiles ? p.n_tiles - tb : kLocTiles);
                    for (int e = lane; e < J * nt * kWarps; e += 32) {
                        const int w = e % kWarps, tt = (e / kWarps) % nt, j = e / (kWarps * nt);
                        const DevJob& jb = p.jobs[j];
                        if (jb.produces) st_relaxed_sys(flag_ptr(p, jb.rank, tb + tt, w), jb.version);
                    }
                    for (int e = lane; e < p.n_parts * nt; e += 32)
                        st_relaxed_sys(s_pflag[e / nt] + tb + e % nt, p.part_version[e / nt]);
                }
                __syncwarp();
                if (lane == 0)
                    for (int64_t b = i; b < i1; ++b) mbar_arrive(&pk[int(b % kMgPub)]);
                i = i1;
            }
            if (rmode == 0 && ready != 0) {
                __threadfence_block();
                rmode = ready == 1 ? 1 : 2;
            }
            if (rmode == 1) {
                // owned reduced chunks the finishers handed over: one fence for the run
                auto owned = [&](int64_t x) {
                    bool o = false;
                    for (int pl = 0; pl < NP; ++pl) o = o || (s_mode[pl] == kMgSplit && ph1(pl, x));
                    return o;
                };
                while (x1 < my_nchunks && !owned(x1)) ++x1;
                int64_t n1 = nown, y = x1;
                if (lane == 0)
                    while (y < my_nchunks && n1 - nown < WG_PUB_GATHER_R &&
                           mbar_test_wait(&rd[int(n1 % kMgPub)], unsigned((n1 / kMgPub) & 1))) {
                        ++n1;
                        ++y;
                        while (y < my_nchunks && !owned(y)) ++y;
                    }
                n1 = __shfl_sync(0xffffffffu, n1, 0);
                if (n1 > nown) {
                    prog = true;
                    if (lane == 0) fence_pub();
                    __syncwarp();
                    for (int64_t k = nown; k < n1; ++k) {
                        const int64_t tb = c_of(x1) * kLocTiles;
                        const int nt = int(p.n_tiles - tb < kLocTiles ? p.n_tiles - tb : kLocTiles);
                        for (int pl = 0; pl < NP; ++pl)
                            if (s_mode[pl] == kMgSplit && ph1(pl, x1) && lane < nt)
                                st_relaxed_sys(s_redflag[pl][owner(pl, x1)] + tb + lane, s_ver[pl]);
                        ++x1;
                        while (x1 < my_nchunks && !owned(x1)) ++x1;
                    }
                    __syncwarp();
                    if (lane == 0)
                        for (int64_t k = nown; k < n1; ++k) mbar_arrive(&rk[int(k % kMgPub)]);
                    nown = n1;
                }
                if (x1 >= my_nchunks) rmode = 2;
            }
            if (prog) {
                spins = 0;
                t0 = globaltimer();
            } else {
                __nanosleep(32);
                if ((++spins & 255) == 0 && (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p)))
                    break;  // the waiting side reports the timeout
            }
        }
        if (lane == 0) prof_add(10, clock64() - kt0);
    } else if (warp < kMgRoleWarps + kMgProd / 32) {
        // ---------------- producers: W', partials ----------------
        // Free-running: they never wait on another GPU, only on the input
        // ring and (kMgPub chunks back) on the produce publisher.
        constexpr int VP = C / kMgProd;
        const int ct = tid - kMgRoleWarps * 32;
        unsigned bad = 0;
        int sti = 0;
        unsigned phi = 0;
        bool ok = true;
        for (int64_t i = 0; ok && i < my_nchunks; ++i) {
            const int64_t e0 = c_of(i) * chunk_elems;
            const bool fullc = e0 + chunk_elems <= p.n;
            for (int jj = 0; jj < J; ++jj) {
                const int j = p.job_order[jj];
                const long long w0 = (p.prof && ct == 0) ? clock64() : 0;
                if (!mbar_wait(p, &fin[sti], phi)) {
                    ok = false;
                    break;
                }
                if (p.prof && ct == 0) prof_add(1, clock64() - w0);
                const V* r = rows_in + size_t(sti) * 3 * C;
                if (fullc)
                    bad |= loc_item<T, true, kMgProd>(p, s_job[j], j, e0, r, wst, ct);
                else
                    bad |= loc_item<T, false, kMgProd>(p, s_job[j], j, e0, r, wst, ct);
                __syncwarp();
                if (lane == 0) mbar_arrive(&ein[sti]);
                if (++sti == NSI) sti = 0, phi ^= 1u;
            }
            if (!ok) break;
            // this GPU's subtree partials (butterfly order inside the subtree)
            for (int pid = 0; pid < p.n_parts; ++pid) {
#pragma unroll
                for (int kv = 0; kv < VP; ++kv) {
                    const int v = kv * kMgProd + ct;
                    const int64_t idx = e0 + int64_t(v) * E;
                    if (idx >= p.npad) continue;
                    auto fetch = [&](int leaf) -> V { return wst[s_pjob[pid][leaf] * C + v]; };
                    __stcg(reinterpret_cast<V*>(s_part[pid] + idx), tree_sum<T>(fetch, s_plog[pid]));
                }
            }
            if (WG_MG_SELF_PUB) {
                // the last producer warp to finish chunk i issues one fence
                // (cumulative over the other warps' stores, acquired through the
                // shared-memory counter) and raises the chunk's flags; warps
                // drift by at most the input ring, far less than kPubRing chunks
                __syncwarp();
                unsigned old = 0;
                if (lane == 0) {
                    unsigned* cnt = &s_pubcnt[i & (kPubRing - 1)];
                    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                                 : "=r"(old)
                                 : "r"(smem_u32(cnt))
                                 : "memory");
                    if (old == kMgProd / 32 - 1) *cnt = 0;
                }
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old == kMgProd / 32 - 1) {
                    const long long w1 = clock64();
                    if (lane == 0) fence_pub();
                    __syncwarp();
                    if (lane == 0 && p.prof) prof_add(9, clock64() - w1);
                    const int64_t tb = c_of(i) * kLocTiles;
                    const int nt = int(p.n_tiles - tb < kLocTiles ? p.n_tiles - tb : kLocTiles);
                    for (int e = lane; e < J * nt * kWarps; e += 32) {
                        const int w = e % kWarps, tt = (e / kWarps) % nt, j = e / (kWarps * nt);
                        const DevJob& jb = p.jobs[j];
                        if (jb.produces) st_relaxed_sys(flag_ptr(p, jb.rank, tb + tt, w), jb.version);
                    }
                    for (int e = lane; e < p.n_parts * nt; e += 32)
                        st_relaxed_sys(s_pflag[e / nt] + tb + e % nt, p.part_version[e / nt]);
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        if (s_produced < i + 1) s_produced = i + 1;
                    }
                }
            } else {
                // hand the chunk to the publisher (fence + flags off this path)
                const int slot = int(i % kMgPub);
                const long long w0 = (p.prof && ct == 0) ? clock64() : 0;
                if (i >= kMgPub && !mbar_wait(p, &pk[slot], unsigned(((i / kMgPub) - 1) & 1))) {
                    ok = false;
                    break;
                }
                if (p.prof && ct == 0) prof_add(3, clock64() - w0);
                __syncwarp();
                if (lane == 0) mbar_arrive(&pd[slot]);
            }
        }
        if (!ok) {
            if (lane == 0) raise_error(p, WG_ETIMEOUT, blockIdx.x);
            sm.abort = 1;
        }
        report_divergence(p, bad);
        if (ct == 0) prof_add(0, clock64() - kt0);
    } else {
        // ---------------- finishers: phase 1 and phase 2 ----------------
        constexpr int VF = C / kMgFin;
        const int ct = tid - kMgRoleWarps * 32 - kMgProd;
        int sta = 0, stb = 0;
        unsigned pha = 0, phb = 0;
        int64_t nown = 0;  // owned reduced chunks handed to the publisher
        bool ok = true;
        {
            const long long w0 = clock64();
            while (ready == 0) __nanosleep(64);
            __threadfence_block();
            if (p.prof && ct == 0) prof_add(4, clock64() - w0);
        }
        constexpr int kLagB = kMgLag2 - kMgLag1;  // phase 2 trails phase 1 by this many chunks
        for (int64_t i = 0; ready == 1 && ok && i < my_nchunks + kLagB; ++i) {
            const int64_t x1 = i;
            if (x1 < my_nchunks && rows_a_of(x1) >= 0) {
                // ---- phase 1 of chunk x1 ----
                const int64_t e0 = c_of(x1) * chunk_elems;
                const long long w0 = (p.prof && ct == 0) ? clock64() : 0;
                // this CTA's producers are done with chunk x1 (a stale group's leaves
                // may all be complete older slots: then no flag orders this launch's
                // own W' -- read by late members -- before its use)
                if (s_produced <= x1) {
                    const uint64_t tw = globaltimer();
                    int it = 0;
                    while (s_produced <= x1) {
                        if ((++it & 255) == 0 && (globaltimer() - tw > uint64_t(p.timeout_ns) || aborted(p))) {
                            ok = false;
                            break;
                        }
                        __nanosleep(32);
                    }
                    if (!ok) break;
                }
                __threadfence_block();
                if (!mbar_wait(p, &fa[sta], pha)) {
                    ok = false;
                    break;
                }
                if (p.prof && ct == 0) prof_add(2, clock64() - w0);
                const V* lb = rows_a + size_t(sta) * s_rows_a * C;
                bool owned = false;
                int e = 0;
                for (int pl = 0; pl < NP; ++pl) {
                    if (!ph1(pl, x1)) continue;
                    const DevPlan& P_ = p.plans[pl];
#pragma unroll
                    for (int kv = 0; kv < VF; ++kv) {
                        const int v = kv * kMgFin + ct;
                        const int64_t idx = e0 + int64_t(v) * E;
                        if (idx >= p.npad) continue;
                        auto fetch = [&](int leaf) -> V {
                            const int row = s_erow[pl][leaf];
                            if (row >= 0) return lb[(e + row) * C + v];
                            return __ldcg(reinterpret_cast<const V*>(s_esrc[pl][leaf] + idx));
                        };
                        const V acc = tree_sum<T>(fetch, s_elog[pl]);
                        if (s_mode[pl] == kMgSplit)  // the owner's reduced chunk, for the other members
                            __stcg(reinterpret_cast<V*>(s_red[pl][owner(pl, x1)] + idx), acc);
                        finish_members<T>(p, sm, P_, acc, idx, [&](int j) {
                            return __ldcg(reinterpret_cast<const V*>(s_job[j].ring + idx));
                        });
                    }
                    owned = owned || s_mode[pl] == kMgSplit;
                    e += s_nrow[pl];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&ea[sta]);
                if (++sta == s_nsa) sta = 0, pha ^= 1u;
                if (owned) {  // the reduced chunk to the reduce publisher
                    const int slot = int(nown % kMgPub);
                    if (nown >= kMgPub && !mbar_wait(p, &rk[slot], unsigned(((nown / kMgPub) - 1) & 1))) {
                        ok = false;
                        break;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&rd[slot]);
                    ++nown;
                }
            }
            const int64_t x2 = i - kLagB;
            if (x2 >= 0 && x2 < my_nchunks && rows_b_of(x2) >= 0) {
                // ---- phase 2 of chunk x2: reduced chunks owned elsewhere ----
                const int64_t e0 = c_of(x2) * chunk_elems;
                if (!mbar_wait(p, &fb[stb], phb)) {
                    ok = false;
                    break;
                }
                const V* lb = rows_b + size_t(stb) * s_rows_b * C;
                int e = 0;
                for (int pl = 0; pl < NP; ++pl) {
                    if (ph1(pl, x2)) continue;
                    const DevPlan& P_ = p.plans[pl];
#pragma unroll
                    for (int kv = 0; kv < VF; ++kv) {
                        const int v = kv * kMgFin + ct;
                        const int64_t idx = e0 + int64_t(v) * E;
                        if (idx >= p.npad) continue;
                        finish_members<T>(p, sm, P_, lb[e * C + v], idx, [&](int j) {
                            return __ldcg(reinterpret_cast<const V*>(s_job[j].ring + idx));
                        });
                    }
                    ++e;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&eb[stb]);
                if (++stb == s_nsb) stb = 0, phb ^= 1u;
            }
        }
        if (!ok) {
            if (lane == 0) raise_error(p, WG_ETIMEOUT, blockIdx.x);
            sm.abort = 1;
        }
        if (ct == 0) prof_add(14, clock64() - kt0);
    }
    unsigned my_tiles = 0;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x)
        my_tiles += unsigned(p.n_tiles - c * kLocTiles < kLocTiles ? p.n_tiles - c * kLocTiles : kLocTiles);
    __syncthreads();
    if (ready != 1 || aborted(p)) sm.abort = 1;
    publish_slots(p, sm.abort ? 0u : my_tiles);
    if (blockIdx.x == 0) {
        __syncthreads();
        const bool res = ready == 1;
        if (res && threadIdx.x < 32) check_sync_points(p, sm);
        __syncthreads();
        if (tid < p.n_jobs) {
            const DevJob& jb = p.jobs[tid];
            wg_job_status stt;
            stt.version = jb.version;
            stt.contrib_stamp = (jb.kind == WG_JOB_LOCAL_STEP || !res) ? jb.version : sm.stamps[jb.vidx][jb.rank];
            stt.timely = stt.contrib_stamp == jb.version;
            stt.root = activation_root(p, jb, res);
            stt.activator = jb.vidx >= 0 && sm.activator[jb.vidx] && stt.root == jb.rank;
            stt.error = int32_t(ld_relaxed_sys(err_ptr(p)));
            p.status[tid] = stt;
        }
    }
}

// Producer warps of the multi-GPU kernels (warps 0..7): local step of every
// job for every tile of this CTA, send-ring install, and the tiles'
// readiness flags published in chunks of kPubChunk by the last warp to
// finish a chunk (one GPU-scope fence, cumulative over the other warps'
// stores acquired through the shared-memory counter). Never waits on a peer.
// ---------------------------------------------------------------------------
// TMA-fed producers of the multi-GPU kernels (WG_TMA_PRODUCE=1, defined above)
//
// The issuer warp's lane 0 streams W, g, m of every (tile, job) item with
// cp.async.bulk (L2 evict-first) into a ring of NSI stages [3][kThreads]
// guarded by mbarriers (fin: bytes landed; ein: the 8 producer warps are
// done); the producer warps only compute: m' and W' from shared memory, m and
// the send-ring slot stored, this GPU's subtree partials summed, the tiles'
// flags published in chunks of kPubChunk by the last warp to finish a chunk.
// Same per-item arithmetic and publication protocol as nvl_produce, with no
// per-thread load issue or address arithmetic on the producers' path.
// ---------------------------------------------------------------------------
constexpr int kTmaMaxStages = 16;

template <typename T, bool HIER>
__device__ void tma_issue(const LaunchParams& p, typename Tr<T>::V* ring, int NSI, uint64_t* fin, uint64_t* ein,
                          int64_t my_ntiles, const LocJob<T>* jobs) {
    using V = typename Tr<T>::V;
    if ((threadIdx.x & 31) != 0) return;
    const uint64_t pol = policy_evict_first();
    const unsigned tbytes = unsigned(kThreads) * 16u;
    const int J = p.n_jobs;
    int st = 0;
    unsigned ph = 0;
    int64_t k = 0;
    for (int64_t kk = 0; kk < my_ntiles; ++kk) {
        const int64_t e0 = (int64_t(blockIdx.x) + kk * gridDim.x) * p.tile_elems;
        const int64_t rem = (p.n - e0) * int64_t(sizeof(T));
        // caller vectors hold exactly n elements: whole 16-byte vectors by TMA,
        // the ragged end is read by the producers from global memory
        const unsigned bytes = rem >= tbytes ? tbytes : (rem > 0 ? unsigned(rem) & ~15u : 0u);
        for (int jj = 0; jj < J; ++jj, ++k) {
            const int j = HIER ? int(p.job_order[jj]) : jj;
            if (k >= NSI && !mbar_wait(p, &ein[st], ph ^ 1u)) {
                raise_error(p, WG_ETIMEOUT, k);
                return;
            }
            const LocJob<T>& jb = jobs[j];
            V* dst = ring + size_t(st) * 3 * kThreads;
            if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
                mbar_arrive_expect_tx(&fin[st], bytes);
                if (bytes) bulk_g2s_hint(dst, jb.fresh + e0, bytes, &fin[st], pol);
            } else {
                mbar_arrive_expect_tx(&fin[st], (jb.mom ? 3u : 2u) * bytes);
                if (bytes) {
                    bulk_g2s_hint(dst, jb.W + e0, bytes, &fin[st], pol);
                    bulk_g2s_hint(dst + kThreads, jb.g + e0, bytes, &fin[st], pol);
                    if (jb.mom) bulk_g2s_hint(dst + 2 * kThreads, jb.m + e0, bytes, &fin[st], pol);
                }
            }
            if (++st == NSI) st = 0, ph ^= 1u;
        }
    }
}

template <typename T, bool HIER>
__device__ unsigned tma_produce(const LaunchParams& p, typename Tr<T>::V* ring, int NSI, uint64_t* fin,
                                uint64_t* ein, int64_t my_ntiles, unsigned* pub_count, T* const* ring_slot,
                                int64_t* const* flag_base, unsigned& bad, const LocJob<T>* jobs,
                                T* const* part_base, int64_t* const* pflag_base, volatile long long* produced) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    const int tid = threadIdx.x, lane = tid & 31;
    const int J = p.n_jobs;
    const int NPa = HIER ? p.n_parts : 0;
    unsigned my_tiles = 0;
    int st = 0;
    unsigned ph = 0;
    for (int64_t kk = 0; kk < my_ntiles; ++kk) {
        const int64_t tile = int64_t(blockIdx.x) + kk * gridDim.x;
        const int64_t idx = tile * p.tile_elems + int64_t(tid) * E;
        const bool full = idx + E <= p.n;
        V s0, s1, s2, s3;  // butterfly stack of the partial being summed (<= 16 leaves)
        bool ok = true;
        for (int jj = 0; jj < J; ++jj) {
            const int j = HIER ? int(p.job_order[jj]) : jj;
            if (!mbar_wait(p, &fin[st], ph)) {
                ok = false;
                break;
            }
            const V* r = ring + size_t(st) * 3 * kThreads;
            const LocJob<T>& jb = jobs[j];
            V wp;
            if (jb.kind == WG_JOB_GROUP_SUM || jb.kind == WG_JOB_SYNC_SUM) {
                wp = full ? r[tid] : ld_tail(jb.fresh, idx, p.n);
            } else {
                const V w = full ? r[tid] : ld_tail(static_cast<const T*>(jb.W), idx, p.n);
                const V g = full ? r[kThreads + tid] : ld_tail(jb.g, idx, p.n);
                if (jb.mom) {
                    // m = beta*m + g ; W' = W - eta*m  (optim.py:179,183)
                    const V m0 = full ? r[2 * kThreads + tid] : ld_tail(static_cast<const T*>(jb.m), idx, p.n);
                    const V mn = vadd(vscale(jb.beta, m0), g);
                    st_stream<T>(jb.m, idx, p.n, mn);
                    wp = vsub(w, vscale(jb.eta, mn));
                } else {
                    wp = vsub(w, vscale(jb.eta, g));  // W' = W - eta*g (optim.py:181-183)
                }
                bad |= unsigned(nonfinite(wp)) << j;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ein[st]);
            if (++st == NSI) st = 0, ph ^= 1u;
            if (jb.kind == WG_JOB_LOCAL_STEP) {
                st_stream<T>(jb.W, idx, p.n, wp);
                continue;
            }
            // SendBuffer.install: W' written once into the send ring
            __stcg(reinterpret_cast<V*>(ring_slot[j] + idx), wp);
            if (NPa && p.job_part[jj] >= 0) {
                // partial = the subtree's butterfly sum (collective.py:321-329)
                const int pos = p.job_ppos[jj];
                V v = wp;
                if (pos & 1) {
                    v = vadd(s0, v);
                    if (pos & 2) {
                        v = vadd(s1, v);
                        if (pos & 4) {
                            v = vadd(s2, v);
                            if (pos & 8) v = vadd(s3, v); else s3 = v;
                        } else {
                            s2 = v;
                        }
                    } else {
                        s1 = v;
                    }
                } else {
                    s0 = v;
                }
                if (p.job_plast[jj])
                    __stcg(reinterpret_cast<V*>(part_base[p.job_part[jj]] + tile * p.tile_elems +
                                                int64_t(tid) * E),
                           v);
            }
        }
        if (!ok) {
            if (lane == 0) raise_error(p, WG_ETIMEOUT, kk);
            break;
        }
        // chunk publication: the last producer warp to finish a chunk fences
        // once (cumulative over the other warps' stores, acquired through the
        // shared-memory counter) and raises the chunk's flags
        const bool chunk_end = ((kk + 1) % kPubChunk == 0) || (kk + 1 == my_ntiles);
        if (chunk_end) {
            __syncwarp();
            unsigned old = 0;
            if (lane == 0) {
                unsigned* cnt = &pub_count[(kk / kPubChunk) & (kPubRing - 1)];
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(old)
                             : "r"(smem_u32(cnt))
                             : "memory");
                if (old == kWarps - 1) *cnt = 0;
            }
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == kWarps - 1) {
                if (p.fence_scope == 0)
                    fence_sys();
                else if (p.fence_scope == 1)
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                const int64_t k0 = kk - (kk % kPubChunk);
                const int nk = int(kk - k0 + 1);
                for (int e = lane; e < nk * J * kWarps; e += 32) {
                    const int w = e % kWarps, j = (e / kWarps) % J, b = e / (kWarps * J);
                    const DevJob& djb = p.jobs[j];
                    if (djb.produces)
                        st_relaxed_sys(flag_base[j] + (int64_t(blockIdx.x) + (k0 + b) * gridDim.x) * kWarps + w,
                                       djb.version);
                }
                if constexpr (HIER) {
                    for (int e = lane; e < nk * NPa; e += 32) {
                        const int pid = e % NPa, b = e / NPa;
                        st_relaxed_sys(pflag_base[pid] + int64_t(blockIdx.x) + (k0 + b) * gridDim.x,
                                       p.part_version[pid]);
                    }
                }
                __syncwarp();
                if (lane == 0 && produced) {
                    __threadfence_block();
                    if (*produced < kk + 1) *produced = kk + 1;
                }
            }
        }
        ++my_tiles;
        // warps cannot drift more than the input ring apart (every stage waits
        // for all 8 producer warps), far less than the counter ring
    }
    return my_tiles;
}

// A late member's own W' of this launch is read back from its send slot by
// the consumer warps (finish_members' own_wp). When every leaf of its group
// is a complete older slot or lives on another GPU, no polled flag orders
// this CTA's producers' store of that tile before the read: wait until the
// producers published the tile (CTA-local tile index kc).
__device__ __forceinline__ void wait_produced(const LaunchParams& p, const volatile long long* produced, int64_t kc) {
    if (*produced <= kc) {
        const uint64_t t0 = globaltimer();
        int it = 0;
        while (*produced <= kc) {
            if ((++it & 255) == 0) {
                if (aborted(p)) break;  // the producers latched an error: results are void
                if (globaltimer() - t0 > uint64_t(p.timeout_ns)) {
                    raise_error(p, WG_ETIMEOUT, kc);
                    break;
                }
            }
            __nanosleep(32);
        }
    }
    __threadfence_block();
}

template <typename T, int kNvlDepth, bool HIER = false>
__device__ __forceinline__ unsigned nvl_produce(const LaunchParams& p, typename Tr<T>::V* ring, int64_t my_ntiles,
                                                unsigned* pub_count, T* const* ring_slot,
                                                int64_t* const* flag_base, unsigned& bad,
                                                T* const* part_base = nullptr, int64_t* const* pflag_base = nullptr,
                                                volatile long long* produced = nullptr) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    const int lane = threadIdx.x & 31;
    const int J = p.n_jobs;
    const int NPa = HIER ? p.n_parts : 0;  // subtree partials produced here (hierarchical sums)
    auto order = [&](int k) { return HIER ? int(p.job_order[k]) : k; };
    unsigned my_tiles = 0;
    // issue cursor kNvlDepth items ahead, advanced incrementally; jobs in
    // p.job_order (each partial's leaves consecutive and in leaf order)
    int64_t ik = 0;
    int ij = 0;
#pragma unroll
    for (int d = 0; d < kNvlDepth; ++d) {
        if (ik < my_ntiles) issue_item<T>(p, int64_t(blockIdx.x) + ik * gridDim.x, order(ij), ring + d * 3 * kThreads);
        cp_async_commit();
        if (++ij == J) ij = 0, ++ik;
    }
    int rs = 0;
    for (int64_t kk = 0; kk < my_ntiles; ++kk) {
        const int64_t tile = int64_t(blockIdx.x) + kk * gridDim.x;
        V s0, s1, s2, s3;  // butterfly stack of the partial being summed (<= 16 leaves)
        for (int jj = 0; jj < J; ++jj) {
            const int j = order(jj);
            cp_async_wait<kNvlDepth - 1>();
            V* slot = ring + rs * 3 * kThreads;
            V wp;
            bad |= unsigned(compute_item<T, false>(p, tile, j, slot, nullptr, ring_slot, &wp)) << j;
            if (NPa && p.job_part[jj] >= 0) {
                // partial = the subtree's butterfly sum (collective.py:321-329):
                // leaf `pos` combines with the stack levels of its set bits
                const int pos = p.job_ppos[jj];
                V v = wp;
                if (pos & 1) {
                    v = vadd(s0, v);
                    if (pos & 2) {
                        v = vadd(s1, v);
                        if (pos & 4) {
                            v = vadd(s2, v);
                            if (pos & 8) v = vadd(s3, v); else s3 = v;
                        } else {
                            s2 = v;
                        }
                    } else {
                        s1 = v;
                    }
                } else {
                    s0 = v;
                }
                if (p.job_plast[jj])
                    __stcg(reinterpret_cast<V*>(part_base[p.job_part[jj]] + tile * p.tile_elems +
                                                int64_t(threadIdx.x) * E),
                           v);
            }
            if (ik < my_ntiles) issue_item<T>(p, int64_t(blockIdx.x) + ik * gridDim.x, order(ij), slot);
            cp_async_commit();
            if (++ij == J) ij = 0, ++ik;
            if (++rs == kNvlDepth) rs = 0;
        }
        // Tiles are published in chunks of kPubChunk: the last producer
        // warp to finish a chunk issues one GPU-scope fence (cumulative
        // over the other warps' stores, acquired through the shared-memory
        // counter) and writes the chunk's per-warp flags with all lanes.
        // No other warp ever waits on a fence.
        const bool chunk_end = ((kk + 1) % kPubChunk == 0) || (kk + 1 == my_ntiles);
        if (chunk_end) {
            __syncwarp();
            unsigned old = 0;
            if (lane == 0) {
                unsigned* cnt = &pub_count[(kk / kPubChunk) & (kPubRing - 1)];
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(old)
                             : "r"(smem_u32(cnt))
                             : "memory");
                if (old == kWarps - 1) *cnt = 0;
            }
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == kWarps - 1) {
                if (p.fence_scope == 0)
                    fence_sys();
                else if (p.fence_scope == 1)
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                const int64_t k0 = kk - (kk % kPubChunk);
                const int nk = int(kk - k0 + 1);
                for (int e = lane; e < nk * J * kWarps; e += 32) {
                    const int w = e % kWarps, j = (e / kWarps) % J, b = e / (kWarps * J);
                    const DevJob& jb = p.jobs[j];
                    if (jb.produces)
                        st_relaxed_sys(flag_base[j] + (int64_t(blockIdx.x) + (k0 + b) * gridDim.x) * kWarps + w,
                                       jb.version);
                }
                if constexpr (HIER) {
                    for (int e = lane; e < nk * NPa; e += 32) {  // the chunk's subtree partials
                        const int pid = e % NPa, b = e / NPa;
                        st_relaxed_sys(pflag_base[pid] + int64_t(blockIdx.x) + (k0 + b) * gridDim.x,
                                       p.part_version[pid]);
                    }
                }
                __syncwarp();
                if (lane == 0 && produced) {  // tiles [0, kk] of this CTA are stored
                    __threadfence_block();
                    if (*produced < kk + 1) *produced = kk + 1;
                }
            }
        }
        ++my_tiles;
        // bound the drift between producer warps (the counter ring)
        if ((kk + 1) % (kPubChunk * kPubRing / 2) == 0) {
            // named barrier over the 8 producer warps, OR-reducing the abort
            // flag so that all of them leave together
            int stop;
            asm volatile(
                "{\n .reg .pred a, b;\n setp.ne.s32 a, %1, 0;\n bar.red.or.pred b, 1, %2, a;\n"
                " selp.s32 %0, 1, 0, b;\n}\n"
                : "=r"(stop)
                : "r"(int(aborted(p))), "n"(kThreads)
                : "memory");
            if (stop) break;
        }
    }
    cp_async_wait<0>();
    return my_tiles;
}

template <typename T>
__global__ void __launch_bounds__(kNvlThreads, 1) wagma_nvl_kernel(const __grid_constant__ LaunchParams p) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    __shared__ SmemCtl sm;
    __shared__ T* s_ring[kMaxJobs];
    __shared__ int64_t* s_flag0[kMaxJobs];
    __shared__ T* s_part[kMaxJobs];           // local subtree partial buffers (this launch's version)
    __shared__ int64_t* s_pflag0[kMaxJobs];   // and their per-tile flags
    __shared__ __align__(8) uint64_t full[kNvlMaxStages];
    __shared__ __align__(8) uint64_t empty[kNvlMaxStages];
    __shared__ volatile int ready;
    __shared__ volatile long long s_produced;  // tiles of this CTA the producers published
    __shared__ __align__(8) uint64_t s_fin[kTmaMaxStages], s_ein[kTmaMaxStages];  // TMA input ring
    __shared__ LocJob<T> s_pj[kMaxJobs];
    // effective leaves of every plan, set after lock-in: the plan's leaves
    // (leaf pull) or its GPU-local subtree partials (hierarchical sum)
    __shared__ int eff_base[kMaxPlans + 1];
    __shared__ int8_t eff_log[kMaxPlans];
    __shared__ int8_t eff_row[kMaxPoll / kWarps];        // flat effective leaf -> TMA row (-1: read from global)
    __shared__ const T* s_leaf_src[kMaxPoll / kWarps];   // flat effective leaf -> its buffer (tile 0)
    __shared__ const int64_t* s_poll_ptr[kMaxPoll];      // flags to wait for (tile 0)
    __shared__ int64_t poll_s[kMaxPoll];
    __shared__ int8_t poll_stride[kMaxPoll];             // kWarps: per-warp leaf flags; 1: per-tile partial flags
    __shared__ int n_poll_sh, n_rows_sh, n_eff_sh, ns_sh;
    __shared__ unsigned pub_count[kPubRing];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        sm.abort = 0;
        ready = 0;
        s_produced = 0;
        for (int st = 0; st < kNvlDepth; ++st) {
            mbar_init(&s_fin[st], 1);
            mbar_init(&s_ein[st], kWarps);
        }
        for (int st = 0; st < kNvlMaxStages; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], kWarps);
        }
    }
    if (tid < kMaxVersions) sm.activator[tid] = 0;
    init_ring_slots<T>(p, s_ring, s_flag0);
    init_loc_jobs<T>(p, s_pj);
    if (tid < p.n_parts) {
        s_part[tid] = part_ptr<T>(p, p.part_key[tid], p.part_version[tid]);
        s_pflag0[tid] = part_flag_ptr(p, p.part_key[tid], 0);
    }
    if (tid < kPubRing) pub_count[tid] = 0;
    __syncthreads();
    // leaf-ring capacity (host-sized for leaf pulls of every plan): rows x stages
    const int cap_rows = p.nvl_stages * p.nvl_rows;
    V* leafbuf = reinterpret_cast<V*>(dyn_smem);                      // [NS][NR][kThreads]
    V* ring = leafbuf + size_t(cap_rows) * kThreads;                    // [kNvlDepth][3][kThreads]
    const int64_t my_ntiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const unsigned tile_bytes = unsigned(p.tile_elems * int64_t(sizeof(T)));
    unsigned my_tiles = 0;

    if (warp < kWarps) {
        // ---------------- producers ----------------
        const long long pc0 = clock64();
        unsigned bad = 0;
        if (WG_TMA_PRODUCE && p.tma_prod)
            my_tiles = p.n_parts ? tma_produce<T, true>(p, ring, kNvlDepth, s_fin, s_ein, my_ntiles, pub_count, s_ring,
                                                        s_flag0, bad, s_pj, s_part, s_pflag0, &s_produced)
                                 : tma_produce<T, false>(p, ring, kNvlDepth, s_fin, s_ein, my_ntiles, pub_count, s_ring,
                                                         s_flag0, bad, s_pj, nullptr, nullptr, &s_produced);
        else
            my_tiles = p.n_parts ? nvl_produce<T, kNvlDepthCpa, true>(p, ring, my_ntiles, pub_count, s_ring, s_flag0, bad,
                                                                   s_part, s_pflag0, &s_produced)
                                 : nvl_produce<T, kNvlDepthCpa, false>(p, ring, my_ntiles, pub_count, s_ring, s_flag0,
                                                                    bad, nullptr, nullptr, &s_produced);
        report_divergence(p, bad);
        if (p.prof && tid == 0) p.prof[blockIdx.x * 8 + 0] = clock64() - pc0;
    } else if (WG_TMA_PRODUCE && warp == 2 * kWarps + 1) {
        // ---------------- TMA input issuer ----------------
        if (!p.tma_prod)
            ;
        else if (p.n_parts)
            tma_issue<T, true>(p, ring, kNvlDepth, s_fin, s_ein, my_ntiles, s_pj);
        else
            tma_issue<T, false>(p, ring, kNvlDepth, s_fin, s_ein, my_ntiles, s_pj);
        my_tiles = 0;
    } else if (warp == 2 * kWarps) {
        // ---------------- puller ----------------
        if (blockIdx.x == 0) control_phase(p, sm.activator);
        bool resolved = resolve_core<T>(p, sm, lane, 32, [] { __syncwarp(); });
        __syncwarp();
        // every effective leaf goes through the ring; flags to wait for:
        // peers' in-progress tiles and this GPU's own producers (this launch)
        if (resolved && lane == 0) {
            int n_poll = 0, f = 0, nr = 0;
            for (int pl = 0; pl < p.n_plans; ++pl) {
                const DevPlan& P_ = p.plans[pl];
                const int64_t v = p.versions[P_.vidx].version;
                // hierarchical sum iff every member contributed fresh W'_v:
                // then every GPU of the group produced its subtree partials
                // of v (every GPU sees the same locked stamps)
                bool hier = p.plan_hl[pl] > 0;
                for (int li = 0; li < P_.n_leaves && hier; ++li) hier = sm.stamps[P_.vidx][P_.leaves[li]] == v;
                eff_base[pl] = f;
                if (hier) {
                    const int hl = p.plan_hl[pl];
                    eff_log[pl] = int8_t(P_.log_leaves - hl);
                    for (int u = 0; u < (P_.n_leaves >> hl); ++u, ++f) {
                        const int key = P_.leaves[u << hl];
                        s_leaf_src[f] = part_ptr<T>(p, key, v);
                        eff_row[f] = int8_t(nr++);
                        s_poll_ptr[n_poll] = part_flag_ptr(p, key, 0);
                        poll_s[n_poll] = v;
                        poll_stride[n_poll] = 1;
                        ++n_poll;
                    }
                } else {
                    eff_log[pl] = int8_t(P_.log_leaves);
                    for (int li = 0; li < P_.n_leaves; ++li, ++f) {
                        const int q = P_.leaves[li];
                        if (sm.leaf_src[pl][li] >= 0) sm.leaf_slot[pl][li] = int16_t(slot_of(p, sm.stamps[P_.vidx][q]));
                        s_leaf_src[f] = ring_ptr<T>(p, q, sm.leaf_slot[pl][li]);
                        eff_row[f] = (WG_NVL_TMA_LOCAL || q / p.R != p.gpu_index) ? int8_t(nr++) : int8_t(-1);
                        if (sm.leaf_src[pl][li] == kSrcReady) continue;
                        for (int w = 0; w < kWarps; ++w) {
                            if (n_poll == kMaxPoll) {
                                raise_error(p, WG_EINVAL, n_poll);
                                break;
                            }
                            s_poll_ptr[n_poll] = flag_ptr(p, q, 0, w);
                            poll_s[n_poll] = sm.stamps[P_.vidx][q];
                            poll_stride[n_poll] = kWarps;
                            ++n_poll;
                        }
                    }
                }
            }
            eff_base[p.n_plans] = f;
            n_poll_sh = n_poll;
            n_rows_sh = nr;
            n_eff_sh = f;
            // stages of the effective rows in the same shared memory
            ns_sh = nr == 0 ? kNvlMaxStages : (cap_rows / nr < kNvlMaxStages ? cap_rows / nr : kNvlMaxStages);
            __threadfence_block();
            ready = aborted(p) ? 2 : 1;
        } else if (!resolved && lane == 0) {
            ready = 2;
        }
        __syncwarp();
        resolved = resolved && ready == 1;
        const int n_poll = n_poll_sh, NR = n_rows_sh, NL = n_eff_sh, NS = ns_sh;
        // Batches of up to kPullBatch tiles: one round of flag loads (all
        // lanes, all tiles of the batch in flight), one acquire fence, then
        // the TMA copies of the whole batch.
        const int batch = NS - 1 < kPullBatch ? (NS > 1 ? NS - 1 : 1) : kPullBatch;
        long long cy_empty = 0, cy_poll = 0, cy_issue = 0;
        int st0 = 0, ph0 = 0;  // stage and phase of tile kc (no division per tile)
        for (int64_t kc = 0; resolved && kc < my_ntiles; kc += batch) {
            const int nb = int(my_ntiles - kc < batch ? my_ntiles - kc : batch);
            bool ok = true;
            long long c0 = clock64();
            for (int b = 0, st = st0, ph = ph0; b < nb && ok; ++b) {
                if (kc + b >= NS && !mbar_wait(p, &empty[st], unsigned(ph ^ 1))) ok = false;
                if (++st == NS) st = 0, ph ^= 1;
            }
            long long c1 = clock64();
            cy_empty += c1 - c0;
            if (!ok) {
                if (lane == 0) raise_error(p, WG_ETIMEOUT, kc);
                break;
            }
            int rc = 0;
            const int total = nb * n_poll;
            for (int base = 0; base < total && !rc; base += 32 * kPollPerLane) {
                int64_t v[kPollPerLane];
#pragma unroll
                for (int r = 0; r < kPollPerLane; ++r) {  // issue the loads together
                    const int e = base + lane + 32 * r;
                    if (e < total) {
                        const int idx = e % n_poll;
                        const int64_t tile = int64_t(blockIdx.x) + (kc + e / n_poll) * gridDim.x;
                        v[r] = ld_relaxed_sys(s_poll_ptr[idx] + tile * poll_stride[idx]);
                    }
                }
#pragma unroll
                for (int r = 0; r < kPollPerLane; ++r) {
                    const int e = base + lane + 32 * r;
                    if (e >= total || rc) continue;
                    const int idx = e % n_poll;
                    const int64_t tile = int64_t(blockIdx.x) + (kc + e / n_poll) * gridDim.x;
                    const uint64_t t0 = globaltimer();
                    int it = 0;
                    while (v[r] < poll_s[idx]) {
                        if ((++it & 63) == 0 && (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p))) {
                            rc = WG_ETIMEOUT;
                            break;
                        }
                        __nanosleep(32);
                        v[r] = ld_relaxed_sys(s_poll_ptr[idx] + tile * poll_stride[idx]);
                    }
                    if (!rc && v[r] >= poll_s[idx] + p.D) rc = WG_EPROTO;
                    if (rc) raise_error(p, rc, int64_t(idx) << 32 | (tile & 0xffffffff));
                }
            }
            if (__any_sync(0xffffffffu, rc != 0)) break;
            __syncwarp();
            long long c2 = clock64();
            cy_poll += c2 - c1;
            // flags were read relaxed: acquire fence (GPU scope suffices: tile
            // and flag are both read where they live, see publish_tile), then
            // order it before the async-proxy (TMA) reads; every lane fences,
            // then lane r issues the copies of TMA row r
            if (p.fence_scope == 0)
                fence_sys();
            else
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (int b = 0, st = st0; b < nb; ++b) {
                if (lane == 0) mbar_arrive_expect_tx(&full[st], unsigned(NR) * tile_bytes);
                if (++st == NS) st = 0;
            }
            __syncwarp();
            for (int e = lane; e < nb * NL; e += 32) {
                const int b = e / NL, f = e % NL;
                const int row = eff_row[f];
                if (row < 0) continue;
                const int st = st0 + b < NS ? st0 + b : st0 + b - NS;
                const int64_t tile = int64_t(blockIdx.x) + (kc + b) * gridDim.x;
                const T* src = s_leaf_src[f] + tile * p.tile_elems;
                bulk_g2s(leafbuf + (size_t(st) * NR + row) * kThreads, src, tile_bytes, &full[st]);
            }
            __syncwarp();
            st0 += nb;
            if (st0 >= NS) st0 -= NS, ph0 ^= 1;
            cy_issue += clock64() - c2;
        }
        if (p.prof && lane == 0) {
            p.prof[blockIdx.x * 8 + 1] = cy_empty;
            p.prof[blockIdx.x * 8 + 2] = cy_poll;
            p.prof[blockIdx.x * 8 + 3] = cy_issue;
        }
    } else {
        // ---------------- consumers ----------------
        const int ctid = tid - kThreads;  // vector index within the tile
        const long long cc0 = clock64();
        while (ready == 0) __nanosleep(64);
        __threadfence_block();
        const long long cc1 = clock64();
        long long cy_full = 0;
        if (ready == 1) {
            const int NR = n_rows_sh, NS = ns_sh;
            for (int64_t kc = 0, st = 0, ph = 0; kc < my_ntiles; ++kc) {
                const long long w0 = clock64();
                if (!mbar_wait(p, &full[st], unsigned(ph))) {
                    if (lane == 0) raise_error(p, WG_ETIMEOUT, kc);
                    break;
                }
                cy_full += clock64() - w0;
                const int64_t tile = int64_t(blockIdx.x) + kc * gridDim.x;
                const int64_t idx = tile * p.tile_elems + int64_t(ctid) * E;
                const V* lb = leafbuf + size_t(st) * NR * kThreads;
                for (int pl = 0; pl < p.n_plans; ++pl) {
                    const DevPlan& P_ = p.plans[pl];
                    const int base = eff_base[pl];
                    auto fetch = [&](int leaf) -> V {
                        const int row = eff_row[base + leaf];
                        if (row >= 0) return lb[row * kThreads + ctid];
                        // this GPU's leaf: the slot tile (published, usually in L2)
                        return __ldcg(reinterpret_cast<const V*>(
                            ring_ptr<T>(p, P_.leaves[leaf], sm.leaf_slot[pl][leaf]) + idx));
                    };
                    auto own_wp = [&](int j) -> V {
                        const DevJob& jb = p.jobs[j];
                        wait_produced(p, &s_produced, kc);
                        return __ldcg(reinterpret_cast<const V*>(ring_ptr<T>(p, jb.rank, slot_of(p, jb.version)) + idx));
                    };
                    // the tree over the effective leaves: levels above the
                    // partials pair them exactly as the full tree would
                    finish_members<T>(p, sm, P_, tree_sum<T>(fetch, eff_log[pl]), idx, own_wp);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == NS) st = 0, ph ^= 1;
            }
        }
        if (p.prof && ctid == 0) {
            p.prof[blockIdx.x * 8 + 4] = cy_full;
            p.prof[blockIdx.x * 8 + 6] = clock64() - cc0;
            p.prof[blockIdx.x * 8 + 7] = cc1 - cc0;
        }
    }
    if (aborted(p)) sm.abort = 1;
    publish_slots(p, sm.abort ? 0u : my_tiles);
    if (blockIdx.x == 0) {
        __syncthreads();
        const bool res = ready == 1;
        if (res && threadIdx.x < 32) check_sync_points(p, sm);
        __syncthreads();
        if (tid < p.n_jobs) {
            const DevJob& jb = p.jobs[tid];
            wg_job_status stt;
            stt.version = jb.version;
            stt.contrib_stamp = (jb.kind == WG_JOB_LOCAL_STEP || !res) ? jb.version : sm.stamps[jb.vidx][jb.rank];
            stt.timely = stt.contrib_stamp == jb.version;
            stt.root = activation_root(p, jb, res);
            stt.activator = jb.vidx >= 0 && sm.activator[jb.vidx] && stt.root == jb.rank;
            stt.error = int32_t(ld_relaxed_sys(err_ptr(p)));
            p.status[tid] = stt;
        }
    }
}

// ---------------------------------------------------------------------------
// multi-GPU kernel with split sums (reduce-scatter + all-gather)
//
// A group whose members all contributed fresh W' (every stamp == version)
// and that spans GPUs is summed split: tile t is reduced only by
// its owner (split_owner_index; same butterfly order, so the bits are unchanged),
// which publishes the reduced tile; every other member copies that one tile
// instead of all S leaves. NVLink ingress per GPU drops from (S-1)·N to
// about 2(S-1)/S·N. Groups with a stale member are summed by the pull.
//
// Warps (R = red_warps, 4 or 8 per launch): 0-7 producers (as in
// wagma_nvl_kernel); stream A (tiles this GPU reduces itself, and every tile
// of pulled groups): warp 8 puller, warps 9..8+R reducers (sum, store owned
// reduced tiles, write W_{t+1}); stream B (tiles reduced by an owner on
// another GPU): warp 9+R puller (waits for the owner's reduced-tile flag, one
// TMA copy per tile), warps 10+R..21 finishers; warp 22 publisher (fence +
// flags for runs of owned reduced tiles). Stream A never waits on stream B,
// so no cross-GPU wait cycle exists.
// ---------------------------------------------------------------------------

constexpr int kSplitPubWarp = 22;  // publisher warp (reduced-tile fences and flags)
constexpr int kSplitThreads = (23 + (WG_TMA_PRODUCE_SPLIT ? 1 : 0)) * 32;  // + TMA issuer warp (warp 23)
// puller wait counters for tools/phase_profile.py (off: they cost registers)
#ifdef WG_PROF_COUNTERS
#define WG_PCNT(...) __VA_ARGS__
#else
#define WG_PCNT(...)
#endif
// Stream A reducers and stream B finishers share 12 warps, split per launch
// (LaunchParams.red_warps, 4 or 8): B carries (n-1)/n of the tiles of a sum
// split over n GPUs, A the owned 1/n plus every tile of pulled groups.
// 0 = by the span (4 reducers when a split group spans >= 4 GPUs).
#ifndef WG_RED_WARPS
#define WG_RED_WARPS 0
#endif
constexpr int kRoleWarps = 12;

// Owner of a tile of a split sum: rotates along each CTA's tile sequence so
// every CTA reduces 1/n_owners of its tiles. kc is the CTA-local index of
// the tile (tile = blockIdx.x + kc * grid; the grid is identical on every
// GPU), so no division by the grid is needed.
__device__ __forceinline__ int split_owner_index(const LaunchParams& p, int pl, int kc) {
    return kc % p.owners[pl].n;
}

template <typename T>
__global__ void __launch_bounds__(kSplitThreads, 1) wagma_split_kernel(const __grid_constant__ LaunchParams p) {
    using V = typename Tr<T>::V;
    constexpr int E = Tr<T>::EPV;
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    __shared__ SmemCtl sm;
    __shared__ T* s_ring[kMaxJobs];
    __shared__ int64_t* s_flag0[kMaxJobs];
    __shared__ __align__(8) uint64_t fullA[kNvlMaxStages], emptyA[kNvlMaxStages];
    __shared__ __align__(8) uint64_t fullB[kNvlMaxStages], emptyB[kNvlMaxStages];
    __shared__ int64_t metaA_tile[kNvlMaxStages], metaB_tile[kNvlMaxStages];
    __shared__ int metaA_kc[kNvlMaxStages], metaB_kc[kNvlMaxStages];  // CTA-local tile index
    // per (plan, owner index): reduced-tile ring and flags of that owner, and
    // whether it lives on another GPU (no 64-bit division per tile)
    __shared__ T* s_red_base[kMaxPlans][kSplitMaxP];
    __shared__ int64_t* s_red_flag[kMaxPlans][kSplitMaxP];
    __shared__ int8_t s_owner_remote[kMaxPlans][kSplitMaxP];
    __shared__ const T* s_leaf_src[kMaxPoll / kWarps];  // flat leaf -> its send-ring slot
    __shared__ const int64_t* s_poll_ptr[kMaxPoll];     // (leaf, warp) flag of tile 0
    __shared__ unsigned metaA_mask[kNvlMaxStages], metaB_mask[kNvlMaxStages];
    __shared__ int leaf_base[kMaxPlans + 1];
    __shared__ int8_t row_of[kMaxPlans][kMaxLeaves];  // stage row of a leaf, -1: read from L2
    __shared__ int plan_rows[kMaxPlans + 1];
    __shared__ volatile int ready;
    __shared__ volatile long long s_produced;  // tiles of this CTA the producers published
    // hierarchical plans (GPU-local subtree partials as the effective leaves):
    // owners per plan, effective leaves, tree levels above them, flag stride
    __shared__ int8_t s_nown[kMaxPlans], s_neff[kMaxPlans], s_elog[kMaxPlans];
    __shared__ int8_t poll_stride[kMaxPoll];
    __shared__ T* s_part[kMaxJobs];
    __shared__ int64_t* s_pflag0[kMaxJobs];
    __shared__ __align__(8) uint64_t s_fin[kTmaMaxStages], s_ein[kTmaMaxStages];  // TMA input ring
    __shared__ LocJob<T> s_pj[kMaxJobs];
    __shared__ int64_t poll_s[kMaxPoll];
    __shared__ int plan_poll_base[kMaxPlans], plan_poll_cnt[kMaxPlans];
    __shared__ unsigned pub_count[kPubRing];
    __shared__ unsigned red_count[kRedRing];
    // owned reduced tiles handed from the reducers to the publisher warp
    __shared__ int64_t pubq_tile[kRedRing];
    __shared__ int pubq_kc[kRedRing];
    __shared__ unsigned pubq_mask[kRedRing];
    __shared__ int64_t pubq_seq[kRedRing];
    __shared__ volatile int64_t pub_done, pub_end;
    __shared__ int64_t bt_tile[kPullBatch];
    __shared__ int bt_kc[kPullBatch];
    __shared__ unsigned bt_mask[kPullBatch];
    __shared__ int bt_n;
    __shared__ int cell_pref[kPullBatch * kMaxPlans + 1];
    __shared__ int plan_split[kMaxPlans];
    __shared__ int64_t btB_tile[kPullBatch];
    __shared__ int btB_kc[kPullBatch];
    __shared__ unsigned btB_mask[kPullBatch];
    __shared__ int btB_n;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int NSA = p.nvl_stages, NSB = p.split_stages, NP = p.n_plans;
    if (tid == 0) {
        sm.abort = 0;
        ready = 0;
        s_produced = 0;
        for (int st = 0; st < kSplitDepth; ++st) {
            mbar_init(&s_fin[st], 1);
            mbar_init(&s_ein[st], kWarps);
        }
        for (int st = 0; st < NSA; ++st) {
            mbar_init(&fullA[st], 1);
            mbar_init(&emptyA[st], p.red_warps);
        }
        for (int st = 0; st < NSB; ++st) {
            mbar_init(&fullB[st], 1);
            mbar_init(&emptyB[st], kRoleWarps - p.red_warps);
        }
        int acc = 0, rows = 0;
        for (int pl = 0; pl < NP; ++pl) {
            leaf_base[pl] = acc;
            acc += p.plans[pl].n_leaves;
            int pr = 0;
            for (int li = 0; li < p.plans[pl].n_leaves; ++li) {
                const bool tma = WG_SPLIT_TMA_LOCAL || p.plans[pl].leaves[li] / p.R != p.gpu_index;
                row_of[pl][li] = int8_t(tma ? rows++ : -1);
                pr += tma;
            }
            plan_rows[pl] = pr;
        }
        leaf_base[NP] = acc;
        plan_rows[NP] = rows;
        for (int pl = 0; pl < NP; ++pl) {
            s_nown[pl] = int8_t(p.owners[pl].n);
            s_neff[pl] = int8_t(p.plans[pl].n_leaves);
            s_elog[pl] = int8_t(p.plans[pl].log_leaves);
        }
    }
    if (tid < p.n_parts) {
        s_part[tid] = part_ptr<T>(p, p.part_key[tid], p.part_version[tid]);
        s_pflag0[tid] = part_flag_ptr(p, p.part_key[tid], 0);
    }
    if (tid < kMaxVersions) sm.activator[tid] = 0;
    init_ring_slots<T>(p, s_ring, s_flag0);
    init_loc_jobs<T>(p, s_pj);
    if (tid < kPubRing) pub_count[tid] = 0;
    if (tid < kRedRing) {
        red_count[tid] = 0;
        pubq_seq[tid] = -1;
    }
    if (tid == 0) {
        pub_done = 0;
        pub_end = -1;
    }
    if (tid < NP * kSplitMaxP) {
        const int pl = tid / kSplitMaxP, oi = tid % kSplitMaxP;
        if (oi < p.owners[pl].n) {
            const int owner = p.owners[pl].rank[oi];
            s_red_base[pl][oi] = red_ptr<T>(p, owner, p.versions[p.plans[pl].vidx].version);
            s_red_flag[pl][oi] = red_flag_ptr(p, owner, 0);
            s_owner_remote[pl][oi] = int8_t(owner / p.R != p.gpu_index);
        }
    }
    __syncthreads();
    const int NL = leaf_base[NP];
    const int NR = plan_rows[NP];  // stage rows: leaves copied by TMA
    V* ringA = reinterpret_cast<V*>(dyn_smem);              // [NSA][NR][kThreads]
    V* ringB = ringA + size_t(NSA) * NR * kThreads;           // [NSB][NP][kThreads]
    V* ring = ringB + size_t(NSB) * NP * kThreads;            // [kSplitDepth][3][kThreads]
    const int64_t my_ntiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const unsigned tile_bytes = unsigned(p.tile_elems * int64_t(sizeof(T)));
    unsigned my_tiles = 0;
    // plans of a tile handled by stream A (mask A) or stream B (mask B)
    auto masks = [&](int kc, unsigned& ma, unsigned& mb) {
        ma = mb = 0;
        for (int pl = 0; pl < NP; ++pl) {
            const bool remote_owner = plan_split[pl] && s_owner_remote[pl][kc % s_nown[pl]];
            (remote_owner ? mb : ma) |= 1u << pl;
        }
    };
    auto acquire_for_tma = [&]() {
        if (p.fence_scope == 0)
            fence_sys();
        else
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
    };

    const long long t_start = clock64();
    auto prof_set = [&](int slot, long long v) {
        if (p.prof) p.prof[blockIdx.x * 16 + slot] = v;
    };
    if (warp < kWarps) {
        unsigned bad = 0;
        if (WG_TMA_PRODUCE_SPLIT)
            my_tiles = p.n_parts ? tma_produce<T, true>(p, ring, kSplitDepth, s_fin, s_ein, my_ntiles, pub_count,
                                                        s_ring, s_flag0, bad, s_pj, s_part, s_pflag0, &s_produced)
                                 : tma_produce<T, false>(p, ring, kSplitDepth, s_fin, s_ein, my_ntiles, pub_count,
                                                         s_ring, s_flag0, bad, s_pj, nullptr, nullptr, &s_produced);
        else
            my_tiles = p.n_parts ? nvl_produce<T, kSplitDepth, true>(p, ring, my_ntiles, pub_count, s_ring, s_flag0,
                                                                     bad, s_part, s_pflag0, &s_produced)
                                 : nvl_produce<T, kSplitDepth, false>(p, ring, my_ntiles, pub_count, s_ring, s_flag0,
                                                                      bad, nullptr, nullptr, &s_produced);
        report_divergence(p, bad);
        if (tid == 0) prof_set(0, clock64() - t_start);
    } else if (WG_TMA_PRODUCE_SPLIT && warp == kSplitPubWarp + 1) {
        // ---------------- TMA input issuer ----------------
        if (p.n_parts)
            tma_issue<T, true>(p, ring, kSplitDepth, s_fin, s_ein, my_ntiles, s_pj);
        else
            tma_issue<T, false>(p, ring, kSplitDepth, s_fin, s_ein, my_ntiles, s_pj);
    } else if (warp == kWarps) {
        // ---------------- stream A puller ----------------
        if (blockIdx.x == 0) control_phase(p, sm.activator);
        bool resolved = resolve_core<T>(p, sm, lane, 32, [] { __syncwarp(); });
        __syncwarp();
        if (resolved && lane == 0) {
            int n_poll = 0;
            for (int pl = 0; pl < NP; ++pl) {
                const DevPlan& P_ = p.plans[pl];
                const int64_t v = p.versions[P_.vidx].version;
                plan_poll_base[pl] = n_poll;
                // split when every member is timely, the group spans several GPUs
                // and the split saves NVLink bytes (split_pays)
                bool all_timely = true;
                for (int li = 0; li < P_.n_leaves; ++li) all_timely = all_timely && sm.stamps[P_.vidx][P_.leaves[li]] == v;
                if (p.plan_hl[pl] && all_timely) {
                    // hierarchical: the effective leaves are the GPUs' subtree
                    // partials (the producers' butterfly sums of 2^hl leaves),
                    // reduce-scattered over their keys when that saves bytes
                    const int hl = p.plan_hl[pl];
                    const int ne = P_.n_leaves >> hl;
                    unsigned gpus = 0;
                    for (int u = 0; u < ne; ++u) {
                        const int key = P_.leaves[u << hl];
                        gpus |= 1u << (key / p.R);
                        if (n_poll == kMaxPoll) {
                            raise_error(p, WG_EINVAL, n_poll);
                            break;
                        }
                        s_poll_ptr[n_poll] = part_flag_ptr(p, key, 0);
                        poll_stride[n_poll] = 1;
                        poll_s[n_poll] = v;
                        ++n_poll;
                        s_leaf_src[leaf_base[pl] + u] = part_ptr<T>(p, key, v);
                    }
                    const bool hsplit = __popc(gpus) >= p.split_span && split_pays(ne, __popc(gpus));
                    if (hsplit) {
                        for (int u = 0; u < ne; ++u) {
                            const int key = P_.leaves[u << hl];
                            s_red_base[pl][u] = red_ptr<T>(p, key, v);
                            s_red_flag[pl][u] = red_flag_ptr(p, key, 0);
                            s_owner_remote[pl][u] = int8_t(key / p.R != p.gpu_index);
                        }
                        s_nown[pl] = int8_t(ne);
                    }
                    s_neff[pl] = int8_t(ne);
                    s_elog[pl] = int8_t(P_.log_leaves - hl);
                    plan_poll_cnt[pl] = n_poll - plan_poll_base[pl];
                    plan_split[pl] = hsplit;
                    continue;
                }
                bool split = p.owners[pl].n == P_.n_leaves && p.owners[pl].n >= 2;
                bool remote = false;
                unsigned gpus = 0;
                for (int li = 0; li < P_.n_leaves; ++li) {
                    const int q = P_.leaves[li];
                    split = split && sm.stamps[P_.vidx][q] == v;
                    remote = remote || q / p.R != p.gpu_index;
                    gpus |= 1u << (q / p.R);
                }
                split = split && __popc(gpus) >= p.split_span && split_pays(p.owners[pl].n, __popc(gpus));
                for (int li = 0; li < P_.n_leaves; ++li) {
                    const int q = P_.leaves[li];
                    if (sm.leaf_src[pl][li] == kSrcReady) continue;
                    if (sm.leaf_src[pl][li] >= 0) sm.leaf_slot[pl][li] = int16_t(slot_of(p, sm.stamps[P_.vidx][q]));
                    for (int w = 0; w < kWarps; ++w) {
                        if (n_poll == kMaxPoll) {
                            raise_error(p, WG_EINVAL, n_poll);
                            break;
                        }
                        s_poll_ptr[n_poll] = flag_ptr(p, q, 0, w);
                        poll_stride[n_poll] = int8_t(kWarps);
                        poll_s[n_poll] = sm.stamps[P_.vidx][q];
                        ++n_poll;
                    }
                }
                plan_poll_cnt[pl] = n_poll - plan_poll_base[pl];
                plan_split[pl] = split && remote;
                for (int li = 0; li < P_.n_leaves; ++li)
                    s_leaf_src[leaf_base[pl] + li] = ring_ptr<T>(p, P_.leaves[li], sm.leaf_slot[pl][li]);
            }
            __threadfence_block();
#ifdef WG_PROF_NOCONSUME  // profiling only: producers alone (results are garbage)
            ready = 2;
#else
            ready = aborted(p) ? 2 : 1;
#endif
        } else if (!resolved && lane == 0) {
            ready = 2;
        }
        __syncwarp();
        resolved = resolved && ready == 1;
        int batch = NSA - 1 < kPullBatch ? (NSA > 1 ? NSA - 1 : 1) : kPullBatch;
        if (WG_SPLIT_ABATCH > 0 && WG_SPLIT_ABATCH < batch) batch = WG_SPLIT_ABATCH;
        int64_t kA = 0;
        int kc = 0, stA = 0, phA = 0;  // stage and phase of tile kA (no division per tile)
        bool ok = resolved;
        WG_PCNT(long long a_empty = 0, a_poll = 0, a_batches = 0;)
        while (ok) {
            // next batch of tiles with stream-A work
            if (lane == 0) {
                int n = 0;
                while (kc < my_ntiles && n < batch) {
                    unsigned ma, mb;
                    masks(kc, ma, mb);
                    if (ma) {
                        bt_tile[n] = int64_t(blockIdx.x) + int64_t(kc) * gridDim.x;
                        bt_kc[n] = kc;
                        bt_mask[n] = ma;
                        ++n;
                    }
                    ++kc;
                }
                bt_n = n;
            }
            __syncwarp();
            kc = __shfl_sync(0xffffffffu, kc, 0);
            const int nb = bt_n;
            if (nb == 0) break;
            WG_PCNT(long long c0 = clock64();)
            for (int b = 0, st = stA, ph = phA; b < nb && ok; ++b) {
                if (kA + b >= NSA && !mbar_wait(p, &emptyA[st], unsigned(ph ^ 1))) ok = false;
                if (++st == NSA) st = 0, ph ^= 1;
            }
            WG_PCNT(a_empty += clock64() - c0; c0 = clock64(); ++a_batches;)
            if (!ok) {
                if (lane == 0) raise_error(p, WG_ETIMEOUT, kA);
                break;
            }
            // producer flags of every leaf of the batch's active plans, all
            // loads in flight together (producers never wait, so waiting for
            // the whole batch cannot deadlock)
            if (lane == 0) {
                int acc = 0;
                for (int c = 0; c < nb * NP; ++c) {
                    cell_pref[c] = acc;
                    if (bt_mask[c / NP] >> (c % NP) & 1) acc += plan_poll_cnt[c % NP];
                }
                cell_pref[nb * NP] = acc;
            }
            __syncwarp();
            const int total = cell_pref[nb * NP];
            int rc = 0;
            for (int base = 0; base < total && !rc; base += 32 * kPollPerLane) {
                const int64_t* fp[kPollPerLane];
                int64_t want[kPollPerLane], v[kPollPerLane];
#pragma unroll
                for (int r = 0; r < kPollPerLane; ++r) {
                    const int e = base + lane + 32 * r;
                    fp[r] = nullptr;
                    if (e >= total) continue;
                    int c = 0;
                    while (cell_pref[c + 1] <= e) ++c;
                    const int idx = plan_poll_base[c % NP] + (e - cell_pref[c]);
                    fp[r] = s_poll_ptr[idx] + bt_tile[c / NP] * poll_stride[idx];
                    want[r] = poll_s[idx];
                    v[r] = ld_relaxed_sys(fp[r]);
                }
#pragma unroll
                for (int r = 0; r < kPollPerLane; ++r) {
                    if (!fp[r] || rc) continue;
                    const uint64_t t0 = globaltimer();
                    int it = 0;
                    while (v[r] < want[r]) {
                        if ((++it & 63) == 0 && (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p))) {
                            rc = WG_ETIMEOUT;
                            break;
                        }
                        __nanosleep(32);
                        v[r] = ld_relaxed_sys(fp[r]);
                    }
                    if (!rc && v[r] >= want[r] + p.D) rc = WG_EPROTO;
                    if (rc) raise_error(p, rc, want[r]);
                }
            }
            if (__any_sync(0xffffffffu, rc != 0)) break;
            WG_PCNT(a_poll += clock64() - c0;)
            acquire_for_tma();
            if (lane == 0) {
                for (int b = 0, st = stA; b < nb; ++b) {
                    unsigned rows = 0;
                    for (int pl = 0; pl < NP; ++pl)
                        if (bt_mask[b] >> pl & 1) rows += s_neff[pl] < p.plans[pl].n_leaves ? s_neff[pl] : plan_rows[pl];
                    metaA_tile[st] = bt_tile[b];
                    metaA_kc[st] = bt_kc[b];
                    metaA_mask[st] = bt_mask[b];
                    mbar_arrive_expect_tx(&fullA[st], rows * tile_bytes);
                    if (++st == NSA) st = 0;
                }
            }
            __syncwarp();
            for (int e = lane; e < nb * NL; e += 32) {
                const int b = e / NL, f = e % NL;
                int pl = 0;
                while (leaf_base[pl + 1] <= f) ++pl;
                if (!(bt_mask[b] >> pl & 1)) continue;
                const int li = f - leaf_base[pl];
                if (li >= s_neff[pl]) continue;  // hierarchical: the partials only
                const int r = row_of[pl][li];
                if (r < 0) continue;
                const int st = stA + b < NSA ? stA + b : stA + b - NSA;
                const T* src = s_leaf_src[f] + bt_tile[b] * p.tile_elems;
                bulk_g2s(ringA + (size_t(st) * NR + r) * kThreads, src, tile_bytes, &fullA[st]);
            }
            __syncwarp();
            kA += nb;
            stA += nb;
            if (stA >= NSA) stA -= NSA, phA ^= 1;
        }
        // end of stream A
        if (kA >= NSA && !mbar_wait(p, &emptyA[stA], unsigned(phA ^ 1))) ok = false;
        if (lane == 0) {
            metaA_tile[stA] = -1;
            mbar_arrive(&fullA[stA]);
            prof_set(1, clock64() - t_start);
            WG_PCNT(prof_set(8, a_empty); prof_set(9, a_poll); prof_set(10, a_batches);)
        }
    } else if (warp <= kWarps + p.red_warps) {
        // ---------------- stream A reducers ----------------
        const int rtid = tid - (kWarps + 1) * 32;
        const int ctid = rtid;  // first vector of this thread
        const int red_threads = p.red_warps * 32;
        while (ready == 0) __nanosleep(64);
        long long wait_a = 0;
        int64_t oq = 0;  // owned tiles so far (same count in every reducer warp)
        for (int64_t kA = 0, st = 0, ph = 0; ready == 1; ++kA) {
            const long long w0 = clock64();
            if (!mbar_wait(p, &fullA[st], unsigned(ph))) {
                if (lane == 0) raise_error(p, WG_ETIMEOUT, kA);
                break;
            }
            wait_a += clock64() - w0;
            const int64_t tile = metaA_tile[st];
            if (tile < 0) break;
            const unsigned mask = metaA_mask[st];
            const int kc = metaA_kc[st];
            const V* lb = ringA + size_t(st) * NR * kThreads;
            bool owned = false;
#pragma unroll 1
            for (int h = 0; h < kThreads / red_threads; ++h) {
            const int vec = rtid + h * red_threads;
            const int64_t idx = tile * p.tile_elems + int64_t(vec) * E;
            for (int pl = 0; pl < NP; ++pl) {
                if (!(mask >> pl & 1)) continue;
                const DevPlan& P_ = p.plans[pl];
                // local leaves from L2 (.cg: never a stale L1 line of a reused slot)
                const int base = leaf_base[pl];
                auto fetch = [&](int leaf) -> V {
                    if (WG_SPLIT_TMA_LOCAL) return lb[(base + leaf) * kThreads + vec];  // row == leaf index
                    const int r = row_of[pl][leaf];
                    if (r >= 0) return lb[r * kThreads + vec];
                    return __ldcg(reinterpret_cast<const V*>(
                        ring_ptr<T>(p, P_.leaves[leaf], sm.leaf_slot[pl][leaf]) + idx));
                };
                const V acc = tree_sum<T>(fetch, s_elog[pl]);
                if (plan_split[pl]) {  // this GPU owns the tile: publish the reduced tile
                    __stcg(reinterpret_cast<V*>(s_red_base[pl][kc % s_nown[pl]] + idx), acc);
                    owned = true;
                }
                auto own_wp = [&](int j) -> V {
                    const DevJob& jb = p.jobs[j];
                    wait_produced(p, &s_produced, kc);
                    return __ldcg(reinterpret_cast<const V*>(ring_ptr<T>(p, jb.rank, slot_of(p, jb.version)) + idx));
                };
                finish_members<T>(p, sm, P_, acc, idx, own_wp);
            }
            }
            // the stage is free once every lane has read it: release it before
            // the (slow) fence below so the puller refills it meanwhile
            __syncwarp();
            if (lane == 0) mbar_arrive(&emptyA[st]);
            if (owned) {
                // the last reducer warp of the tile hands it to the publisher
                // (which fences and raises the flags, off the reducers' path)
                if (lane == 0) {
                    unsigned* cnt = &red_count[kA & (kRedRing - 1)];
                    unsigned old;
                    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                                 : "=r"(old)
                                 : "r"(smem_u32(cnt))
                                 : "memory");
                    if (old == unsigned(p.red_warps - 1)) {
                        *cnt = 0;
                        const uint64_t t0 = globaltimer();
                        while (pub_done <= oq - kRedRing) {  // queue full: publisher lags
                            if (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p)) break;
                            __nanosleep(64);
                        }
                        const int slot = int(oq & (kRedRing - 1));
                        unsigned ms = 0;
                        for (int pl = 0; pl < NP; ++pl) ms |= (mask >> pl & 1) && plan_split[pl] ? 1u << pl : 0u;
                        pubq_tile[slot] = tile;
                        pubq_kc[slot] = kc;
                        pubq_mask[slot] = ms;
                        asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&pubq_seq[slot])),
                                     "l"(oq)
                                     : "memory");
                    }
                }
                ++oq;
            }
            if (++st == NSA) st = 0, ph ^= 1;
        }
        if (ctid == 0) {
            pub_end = oq;  // every owned tile has been handed over (or the stream stopped)
            prof_set(3, wait_a);
            prof_set(4, clock64() - t_start);
        }
    } else if (warp == kWarps + p.red_warps + 1) {
        // ---------------- stream B puller ----------------
        // Batches of up to kPullBatch tiles reduced on other GPUs: all the
        // owners' reduced-tile flags loaded at once, then tile by tile (in
        // order) wait, copy the reduced tiles.
        while (ready == 0) __nanosleep(64);
        int64_t kB = 0;
        int kc = 0, stB = 0, phB = 0;
        bool ok = ready == 1;
        WG_PCNT(long long b_empty = 0, b_poll = 0, b_notready = 0;)
        int batch = NSB - 1 < kPullBatch ? (NSB > 1 ? NSB - 1 : 1) : kPullBatch;
        batch = batch * NP > 32 ? (32 / NP > 0 ? 32 / NP : 1) : batch;  // one flag per lane
        while (ok) {
            if (lane == 0) {
                int n = 0;
                while (kc < my_ntiles && n < batch) {
                    unsigned ma, mb;
                    masks(kc, ma, mb);
                    if (mb) {
                        btB_tile[n] = int64_t(blockIdx.x) + int64_t(kc) * gridDim.x;
                        btB_kc[n] = kc;
                        btB_mask[n] = mb;
                        ++n;
                    }
                    ++kc;
                }
                btB_n = n;
            }
            __syncwarp();
            kc = __shfl_sync(0xffffffffu, kc, 0);
            const int nb = btB_n;
            if (nb == 0) break;
            // lane e -> (tile b = e / NP, plan e % NP)
            int64_t x = 0, want = 0;
            const int64_t* fp = nullptr;
            const int e = lane;
            if (e < nb * NP && (btB_mask[e / NP] >> (e % NP) & 1)) {
                const int pl = e % NP;
                want = p.versions[p.plans[pl].vidx].version;
                fp = s_red_flag[pl][btB_kc[e / NP] % s_nown[pl]] + btB_tile[e / NP];
                x = ld_relaxed_sys(fp);
            }
            int rc = 0;
            // usual case: every owner already published -> one fence for the batch
            const bool all_ready = __all_sync(0xffffffffu, !fp || x >= want);
            WG_PCNT(b_notready += !all_ready;)
            if (all_ready) acquire_for_tma();
            for (int bb = 0; bb < nb && ok; ++bb) {
                const int64_t k = kB + bb;
                const int st = stB;
                WG_PCNT(long long c0 = clock64();)
                if (k >= NSB && !mbar_wait(p, &emptyB[st], unsigned(phB ^ 1))) {
                    ok = false;
                    break;
                }
                if (++stB == NSB) stB = 0, phB ^= 1;
                WG_PCNT(b_empty += clock64() - c0; c0 = clock64();)
                if (!all_ready && fp && e / NP == bb) {
                    const uint64_t t0 = globaltimer();
                    int it = 0;
                    while (x < want) {
                        if ((++it & 63) == 0 && (globaltimer() - t0 > uint64_t(p.timeout_ns) || aborted(p))) {
                            rc = WG_ETIMEOUT;
                            break;
                        }
                        __nanosleep(32);
                        x = ld_relaxed_sys(fp);
                    }
                    if (!rc && x >= want + p.D) rc = WG_EPROTO;
                    if (rc) raise_error(p, rc, want);
                }
                if (__any_sync(0xffffffffu, rc != 0)) {
                    ok = false;
                    break;
                }
                WG_PCNT(b_poll += clock64() - c0;)
                if (!all_ready) acquire_for_tma();
                const int64_t tile = btB_tile[bb];
                const unsigned mb = btB_mask[bb];
                if (lane == 0) {
                    metaB_tile[st] = tile;
                    metaB_mask[st] = mb;
                    mbar_arrive_expect_tx(&fullB[st], unsigned(__popc(mb)) * tile_bytes);
                }
                __syncwarp();
                if (lane < NP && (mb >> lane & 1)) {
                    const T* src = s_red_base[lane][btB_kc[bb] % s_nown[lane]] + tile * p.tile_elems;
                    bulk_g2s(ringB + (size_t(st) * NP + lane) * kThreads, src, tile_bytes, &fullB[st]);
                }
                __syncwarp();
            }
            if (!ok) {
                if (lane == 0) raise_error(p, WG_ETIMEOUT, kB);
                break;
            }
            kB += nb;
        }
        if (kB >= NSB && !mbar_wait(p, &emptyB[stB], unsigned(phB ^ 1))) ok = false;
        if (lane == 0) {
            metaB_tile[stB] = -1;
            mbar_arrive(&fullB[stB]);
            prof_set(5, clock64() - t_start);
            WG_PCNT(prof_set(11, b_empty); prof_set(12, b_poll); prof_set(13, b_notready);)
        }
    } else if (warp == kSplitPubWarp) {
        // ---------------- publisher ----------------
        // Owned reduced tiles, in order: every run of consecutive ready tiles
        // gets one fence (cumulative over the reducers' stores, acquired
        // through the queue) and then its flags.
        while (ready == 0) __nanosleep(64);
        int64_t next = 0;
        const uint64_t t0 = globaltimer();
        while (ready == 1) {
            int n = 0;
            if (lane == 0) {
                for (;;) {
                    int64_t v;
                    asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];"
                                 : "=l"(v)
                                 : "r"(smem_u32(&pubq_seq[next & (kRedRing - 1)]))
                                 : "memory");
                    if (v == next) break;
                    const int64_t e = pub_end;
                    if ((e >= 0 && next >= e) || aborted(p)) {
                        n = -1;
                        break;
                    }
                    if (globaltimer() - t0 > uint64_t(p.timeout_ns)) {
                        raise_error(p, WG_ETIMEOUT, next);
                        n = -1;
                        break;
                    }
                    __nanosleep(32);
                }
                if (n == 0) {
                    n = 1;
                    while (n < kRedRing / 2) {
                        int64_t v;
                        asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];"
                                     : "=l"(v)
                                     : "r"(smem_u32(&pubq_seq[(next + n) & (kRedRing - 1)]))
                                     : "memory");
                        if (v != next + n) break;
                        ++n;
                    }
                }
            }
            n = __shfl_sync(0xffffffffu, n, 0);
            if (n < 0) break;
            __syncwarp();
            if (p.fence_scope == 0)
                fence_sys();
            else
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int e = lane; e < n * NP; e += 32) {
                const int slot = int((next + e / NP) & (kRedRing - 1)), pl = e % NP;
                if (pubq_mask[slot] >> pl & 1)
                    st_relaxed_sys(s_red_flag[pl][pubq_kc[slot] % s_nown[pl]] + pubq_tile[slot],
                                   p.versions[p.plans[pl].vidx].version);
            }
            __syncwarp();
            next += n;
            if (lane == 0) pub_done = next;
        }
    } else {
        // ---------------- stream B finishers (2 vectors per thread) ----------------
        const int ftid = tid - (kWarps + p.red_warps + 2) * 32;
        const int fin_threads = (kRoleWarps - p.red_warps) * 32;
        while (ready == 0) __nanosleep(64);
        long long wait_b = 0;
        WG_PCNT(long long fin_work = 0; const long long ready_at = clock64() - t_start;)
        for (int64_t kB = 0, st = 0, ph = 0; ready == 1; ++kB) {
            const long long w0 = clock64();
            if (!mbar_wait(p, &fullB[st], unsigned(ph))) {
                if (lane == 0) raise_error(p, WG_ETIMEOUT, kB);
                break;
            }
            wait_b += clock64() - w0;
            const int64_t tile = metaB_tile[st];
            if (tile < 0) break;
            const unsigned mask = metaB_mask[st];
            const V* lb = ringB + size_t(st) * NP * kThreads;
            WG_PCNT(const long long f0 = clock64();)
            for (int h = 0; h < kThreads / fin_threads; ++h) {
                const int vec = ftid + h * fin_threads;
                const int64_t idx = tile * p.tile_elems + int64_t(vec) * E;
                for (int pl = 0; pl < NP; ++pl) {
                    if (!(mask >> pl & 1)) continue;
                    auto own_wp = [&](int j) -> V {
                        const DevJob& jb = p.jobs[j];
                        return __ldcg(
                            reinterpret_cast<const V*>(ring_ptr<T>(p, jb.rank, slot_of(p, jb.version)) + idx));
                    };
                    finish_members<T>(p, sm, p.plans[pl], lb[pl * kThreads + vec], idx, own_wp);
                }
            }
            __syncwarp();
            WG_PCNT(fin_work += clock64() - f0;)
            if (lane == 0) mbar_arrive(&emptyB[st]);
            if (++st == NSB) st = 0, ph ^= 1;
        }
        if (ftid == 0) {
            prof_set(6, wait_b);
            prof_set(7, clock64() - t_start);
            WG_PCNT(prof_set(14, ready_at); prof_set(15, fin_work);)
        }
    }
    if (aborted(p)) sm.abort = 1;
    publish_slots(p, sm.abort ? 0u : my_tiles);
    if (blockIdx.x == 0) {
        __syncthreads();
        const bool res = ready == 1;
        if (res && threadIdx.x < 32) check_sync_points(p, sm);
        __syncthreads();
        if (tid < p.n_jobs) {
            const DevJob& jb = p.jobs[tid];
            wg_job_status stt;
            stt.version = jb.version;
            stt.contrib_stamp = (jb.kind == WG_JOB_LOCAL_STEP || !res) ? jb.version : sm.stamps[jb.vidx][jb.rank];
            stt.timely = stt.contrib_stamp == jb.version;
            stt.root = activation_root(p, jb, res);
            stt.activator = jb.vidx >= 0 && sm.activator[jb.vidx] && stt.root == jb.rank;
            stt.error = int32_t(ld_relaxed_sys(err_ptr(p)));
            p.status[tid] = stt;
        }
    }
}

// ---------------------------------------------------------------------------
// replica diagnostics (optim.py:199-210): sum of replicas, spread potential
// ---------------------------------------------------------------------------

struct ReplicaPtrs {
    const void* w[kMaxJobs];
};

// sum[e] += sum_r W_r[e] (fp64)
template <typename T>
__global__ void replicas_sum_kernel(ReplicaPtrs ptrs, int R, int64_t n, double* sum) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        T v[kMaxJobs];  // every replica's load in flight before the adds
#pragma unroll
        for (int r = 0; r < kMaxJobs; ++r)
            if (r < R) v[r] = __ldcs(static_cast<const T*>(ptrs.w[r]) + e);
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < kMaxJobs; ++r)
            if (r < R) acc += double(v[r]);
        sum[e] += acc;
    }
}

// out[0] += sum_r sum_e (W_r[e] - mu[e])^2 ; out[1] = max over r, e of |W_r[e] - W_0[e]|
template <typename T>
__global__ void replicas_spread_kernel(ReplicaPtrs ptrs, int R, int64_t n, const double* mu, double* out) {
    double g = 0.0, dmax = 0.0;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        T v[kMaxJobs];  // every replica's load in flight before the arithmetic
#pragma unroll
        for (int r = 0; r < kMaxJobs; ++r)
            if (r < R) v[r] = __ldcs(static_cast<const T*>(ptrs.w[r]) + e);
        const double m = mu[e];
        const double w0 = double(v[0]);
#pragma unroll
        for (int r = 0; r < kMaxJobs; ++r) {
            if (r >= R) break;
            const double w = double(v[r]);
            g += (w - m) * (w - m);
            dmax = fmax(dmax, fabs(w - w0));
        }
    }
    for (int o = 16; o; o >>= 1) {
        g += __shfl_xor_sync(0xffffffffu, g, o);
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], g);
        atomicMax(reinterpret_cast<unsigned long long*>(&out[1]), __double_as_longlong(dmax));  // dmax >= 0
    }
}

__global__ void fill_i64_kernel(int64_t* p, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) p[i] = v;
}

__global__ void delay_kernel(int64_t ns) {
    const uint64_t t0 = globaltimer();
    while (globaltimer() - t0 < uint64_t(ns)) __nanosleep(1000);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static size_t dyn_smem_bytes(int n_stage, bool ahead) {
    return size_t((ahead ? 0 : kDepth * 3) + n_stage) * kThreads * 16;
}
static bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
static int ilog2(int64_t n) {
    int r = 0;
    while ((int64_t(1) << (r + 1)) <= n) ++r;
    return r;
}

struct Blob {
    uint64_t magic;
    int32_t gpu_index, P, R, D, Dv, dtype;
    int64_t n, arena_bytes;
    // process-wide kernel choices that every GPU of a job must share: which
    // multi-GPU kernel runs (only the split kernel publishes reduced tiles),
    // its tile ownership (grid = SMs x occupancy) and the flag fence scope
    int32_t use_nvl, use_split, split_span, fence_scope, sms, occ_split, occ_nvl, use_hier;
    int32_t use_mg, pad_b;
    int64_t split_min_bytes, hier_split_max_bytes;
    cudaIpcMemHandle_t handle;
};
constexpr uint64_t kBlobMagic = 0x57474d4142323030ull;  // "WGMAB200"

}  // namespace wg

using namespace wg;

struct wg_ctx {
    wg_config cfg;
    int R, D, Dv;
    size_t esize;
    int64_t tile_elems, n_tiles, npad;
    Layout L;
    char* base[kMaxGpus];
    bool opened[kMaxGpus];
    char* arena;
    wg_job_status* status_host;
    wg_job_status* status_dev;
    int last_n_jobs;
    int sms;
    int occ[2 * kMaxJobs + 1];
    long long* prof;
    int fence_scope;
    int use_nvl;
    int use_split;
    int split_span;
    int64_t split_min_bytes;  // split sums only for replicas at least this large
    int occ_nvl[2];
    int occ_split[2];
    int use_loc;              // single-GPU launches: TMA kernel (else the cp.async kernel)
    int use_hier;             // multi-GPU: exchange GPU-local subtree partials where the tree allows
    int use_mg;               // hierarchical launches: the TMA-produce multi-GPU kernel (else the pull kernel)
    int mg_nsi_max;           // wagma_mg_kernel: deepest input ring tried (WG_MG_NSI_MAX)
    int64_t hier_split_max_bytes;  // reduce-scattered partials only up to this replica size
    int mg_dyn_max[2];        // dynamic shared memory available to wagma_mg_kernel<T>
    int adaptive_grace;       // activator skips the grace wait for ranks late at the previous version
    int loc_dyn_max[2];       // dynamic shared memory available to wagma_local_kernel<T>
    int64_t* err_host;        // host-mapped mirror of the error word
    int64_t* err_host_dev;
};

extern "C" {

const char* wg_strerror(int code) {
    switch (code) {
        case WG_OK: return "ok";
        case WG_EINVAL: return "invalid parameters";
        case WG_EVERSION: return "version regression";
        case WG_ESTALE: return "stale contribution violates staleness bound";
        case WG_EPROTO: return "protocol fault";
        case WG_ETIMEOUT: return "device watchdog timeout (peer never published)";
        case WG_ECUDA: return "CUDA runtime error";
        case WG_ENOMEM: return "out of memory";
        case WG_EDIVERGE: return "non-finite gradient or replica (divergence)";
        case WG_ESYNC: return "mismatched sync points";
        default: return "unknown error";
    }
}

const char* wg_last_error_message(void) { return g_last_error.c_str(); }

int wg_ctx_create(const wg_config* cfg, wg_ctx** out) {
    if (!cfg || !out) return fail(WG_EINVAL, "null argument");
    const wg_config& c = *cfg;
    if (!is_pow2(c.P) || c.P > kMaxP) return fail(WG_EINVAL, "P=%d must be a power of two <= %d", c.P, kMaxP);
    if (!is_pow2(c.S) || c.S > c.P) return fail(WG_EINVAL, "S=%d must be a power of two <= P", c.S);
    if (c.n_gpus < 1 || c.n_gpus > kMaxGpus || c.P % c.n_gpus)
        return fail(WG_EINVAL, "n_gpus=%d must divide P and be <= %d", c.n_gpus, kMaxGpus);
    if (c.gpu_index < 0 || c.gpu_index >= c.n_gpus) return fail(WG_EINVAL, "gpu_index out of range");
    if (c.P / c.n_gpus > kMaxJobs) return fail(WG_EINVAL, "at most %d ranks per GPU", kMaxJobs);
    if (c.dtype != WG_F32 && c.dtype != WG_F64) return fail(WG_EINVAL, "dtype");
    if (c.mask_rule != WG_RULE_EXAMPLE && c.mask_rule != WG_RULE_LITERAL) return fail(WG_EINVAL, "mask rule");
    if (c.n < 0 || c.tau < 0) return fail(WG_EINVAL, "n and tau must be >= 0");
    wg_ctx* ctx = new wg_ctx();
    std::memset(ctx, 0, sizeof(*ctx));
    ctx->cfg = c;
    if (ctx->cfg.grace_ns <= 0) ctx->cfg.grace_ns = 100000;
    if (ctx->cfg.timeout_ns <= 0) ctx->cfg.timeout_ns = 20000000000ll;
    ctx->R = c.P / c.n_gpus;
    // process-wide knobs (environment; identical on every process of a job)
    ctx->use_nvl = 1;
    if (const char* nv = getenv("WG_NVL")) ctx->use_nvl = atoi(nv);
    ctx->use_split = 1;
    if (const char* sp = getenv("WG_SPLIT")) ctx->use_split = atoi(sp);
    ctx->split_span = 2;  // the same on every process of a job (environment knob for experiments)
    if (const char* ss = getenv("WG_SPLIT_SPAN")) ctx->split_span = std::max(2, atoi(ss));
    // below ~8 MiB per replica the extra owner -> member hop of a split sum
    // costs more than the NVLink bytes it saves (measured: 4 GPUs S=4, 1 MiB
    // pull 0.047 vs split 0.059 ms, 4 MiB 0.069 vs 0.080, 16 MiB 0.130 vs 0.125)
    ctx->split_min_bytes = int64_t(8) << 20;
    if (const char* sm = getenv("WG_SPLIT_MIN_BYTES")) ctx->split_min_bytes = std::max<long long>(0, atoll(sm));
    ctx->use_loc = 1;
    if (const char* lc = getenv("WG_LOC")) ctx->use_loc = atoi(lc);
    // Hierarchical (GPU-local subtree) sums where the schedule allows, in the
    // split / pull kernels (partials reduce-scattered where that pays): measured
    // at P=8, n = 25.6M (profiles/r02_multigpu_ab.txt) 5-7% faster than the
    // leaf-level split / pull at 2 and 4 GPUs. The TMA-produce mg kernel is
    // opt-in (WG_MG=1; slower: its finishers trail its producers).
    ctx->use_hier = 1;
    if (const char* hh = getenv("WG_HIER")) ctx->use_hier = atoi(hh);
    ctx->use_mg = 0;
    if (const char* mg = getenv("WG_MG")) ctx->use_mg = atoi(mg);
    ctx->hier_split_max_bytes = int64_t(160) << 20;
    if (const char* hm = getenv("WG_HIER_SPLIT_MAX_BYTES")) ctx->hier_split_max_bytes = std::max<long long>(0, atoll(hm));
    ctx->mg_nsi_max = WG_MG_IN_STAGES_MAX;
    if (const char* ns = getenv("WG_MG_NSI_MAX")) ctx->mg_nsi_max = std::max(2, atoi(ns));
    ctx->adaptive_grace = 1;
    if (const char* ag = getenv("WG_ADAPTIVE_GRACE")) ctx->adaptive_grace = atoi(ag);
    ctx->fence_scope = 1;  // GPU scope for per-tile flags (see publish_tile)
    if (const char* fs = getenv("WG_FENCE_SCOPE")) {
        if (!strcmp(fs, "sys")) ctx->fence_scope = 0;
        if (!strcmp(fs, "none")) ctx->fence_scope = 2;  // timing experiments only: unsafe
    }
    ctx->D = c.ring_depth > 0 ? c.ring_depth : (c.tau > 0 ? int(std::max<int64_t>(2 * c.tau, 4)) : 16);
    ctx->Dv = c.version_ring > 0 ? c.version_ring : (c.tau > 0 ? int(std::max<int64_t>(2 * c.tau, 8)) : 64);
    if (ctx->D < 2 || ctx->D > 32767) {
        delete ctx;
        return fail(WG_EINVAL, "ring depth");
    }
    ctx->esize = c.dtype == WG_F32 ? 4 : 8;
    ctx->tile_elems = int64_t(kThreads) * kVecPerThread * (16 / int64_t(ctx->esize));
    ctx->n_tiles = std::max<int64_t>(1, (c.n + ctx->tile_elems - 1) / ctx->tile_elems);
    ctx->npad = ctx->n_tiles * ctx->tile_elems;
    Layout& L = ctx->L;
    int64_t off = 0;
    L.hdr = off;
    off = align_up(off + 256, 256);
    L.announce = off;
    off = align_up(off + int64_t(ctx->R) * kAnnounceStride * 8, 256);
    L.complete = off;
    off = align_up(off + int64_t(ctx->R) * ctx->D * 8, 256);
    L.counter = off;
    off = align_up(off + int64_t(ctx->R) * ctx->D * 4, 256);
    L.syncmark = off;
    off = align_up(off + int64_t(ctx->R) * ctx->D * 8, 256);
    L.desc = off;
    off = align_up(off + int64_t(ctx->Dv) * int64_t(sizeof(Desc)), 256);
    L.flags = off;
    off = align_up(off + int64_t(ctx->R) * ctx->n_tiles * kWarps * 8, 4096);
    L.ring = off;
    off = align_up(off + int64_t(ctx->R) * ctx->D * ctx->npad * int64_t(ctx->esize), 4096);
    const int64_t red = ((ctx->use_split && c.n_gpus >= ctx->split_span && c.P <= kSplitMaxP) ||
                         (ctx->use_hier && ctx->use_split && c.n_gpus >= 2)) ? 1 : 0;
    L.red_flags = off;
    off = align_up(off + red * int64_t(ctx->R) * ctx->n_tiles * 8, 4096);
    L.red_ring = off;
    off = align_up(off + red * int64_t(ctx->R) * ctx->D * ctx->npad * int64_t(ctx->esize), 4096);
    const int64_t hier = (ctx->use_hier && c.n_gpus >= 2) ? 1 : 0;
    L.part_flags = off;
    off = align_up(off + hier * int64_t(ctx->R) * ctx->n_tiles * 8, 4096);
    L.part_ring = off;
    off = align_up(off + hier * int64_t(ctx->R) * ctx->D * ctx->npad * int64_t(ctx->esize), 4096);
    L.total = off;

    int rc = WG_OK;
    do {
        cudaError_t e = cudaSetDevice(c.device);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaSetDevice(%d): %s", c.device, cudaGetErrorString(e)); break; }
        e = cudaMalloc(&ctx->arena, size_t(L.total));
        if (e != cudaSuccess) { rc = fail(WG_ENOMEM, "cudaMalloc(%lld): %s", (long long)L.total, cudaGetErrorString(e)); break; }
        e = cudaMemset(ctx->arena, 0, size_t(L.ring));
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaMemset: %s", cudaGetErrorString(e)); break; }
        auto fill = [&](int64_t byte_off, int64_t count, int64_t v) {
            if (count <= 0) return;
            fill_i64_kernel<<<256, 256>>>(reinterpret_cast<int64_t*>(ctx->arena + byte_off), count, v);
        };
        fill(L.announce, int64_t(ctx->R) * kAnnounceStride, -1);
        fill(L.complete, int64_t(ctx->R) * ctx->D, kNever);
        fill(L.flags, int64_t(ctx->R) * ctx->n_tiles * kWarps, kNever);
        if (L.red_ring > L.red_flags) fill(L.red_flags, int64_t(ctx->R) * ctx->n_tiles, kNever);
        if (L.part_ring > L.part_flags) fill(L.part_flags, int64_t(ctx->R) * ctx->n_tiles, kNever);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "arena init: %s", cudaGetErrorString(e)); break; }
        e = cudaHostAlloc(&ctx->status_host, sizeof(wg_job_status) * kMaxJobs, cudaHostAllocMapped);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaHostAlloc: %s", cudaGetErrorString(e)); break; }
        std::memset(ctx->status_host, 0, sizeof(wg_job_status) * kMaxJobs);
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->status_dev), ctx->status_host, 0);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e)); break; }
        const int max_smem = int(dyn_smem_bytes(2 * kMaxJobs, false));
        e = cudaFuncSetAttribute(wagma_step_kernel<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_step_kernel<double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_step_kernel<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_step_kernel<double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_nvl_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNvlMaxDyn);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_nvl_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNvlMaxDyn);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_split_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNvlMaxDyn);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wagma_split_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNvlMaxDyn);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e)); break; }
        {
            int optin = 0;
            e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
            cudaFuncAttributes fa[2];
            if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa[0], wagma_local_kernel<float>);
            if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa[1], wagma_local_kernel<double>);
            cudaFuncAttributes fm[2];
            if (e == cudaSuccess) e = cudaFuncGetAttributes(&fm[0], wagma_mg_kernel<float>);
            if (e == cudaSuccess) e = cudaFuncGetAttributes(&fm[1], wagma_mg_kernel<double>);
            for (int di = 0; di < 2 && e == cudaSuccess; ++di) {
                ctx->mg_dyn_max[di] = optin - int(fm[di].sharedSizeBytes) - 1024;
                e = cudaFuncSetAttribute(di == 0 ? (const void*)wagma_mg_kernel<float> : (const void*)wagma_mg_kernel<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->mg_dyn_max[di]);
            }
            for (int di = 0; di < 2 && e == cudaSuccess; ++di) {
                ctx->loc_dyn_max[di] = optin - int(fa[di].sharedSizeBytes) - 1024;
                e = cudaFuncSetAttribute(di == 0 ? (const void*)wagma_local_kernel<float> : (const void*)wagma_local_kernel<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->loc_dyn_max[di]);
            }
            if (e != cudaSuccess) { rc = fail(WG_ECUDA, "local kernel attributes: %s", cudaGetErrorString(e)); break; }
        }
        e = cudaHostAlloc(&ctx->err_host, 2 * sizeof(int64_t), cudaHostAllocMapped);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaHostAlloc: %s", cudaGetErrorString(e)); break; }
        ctx->err_host[0] = ctx->err_host[1] = 0;
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->err_host_dev), ctx->err_host, 0);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e)); break; }
        e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, c.device);
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "device attribute: %s", cudaGetErrorString(e)); break; }
        // multi-GPU grids (tile ownership) are fixed here, so peers can compare them at import
        for (int di = 0; di < 2 && e == cudaSuccess; ++di) {
            int o = 0;
            e = di == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_split_kernel<float>, kSplitThreads, kNvlMaxDyn)
                        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_split_kernel<double>, kSplitThreads, kNvlMaxDyn);
            ctx->occ_split[di] = o > 0 ? o : 1;
            if (e != cudaSuccess) break;
            e = di == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_nvl_kernel<float>, kNvlThreads, kNvlMaxDyn)
                        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_nvl_kernel<double>, kNvlThreads, kNvlMaxDyn);
            ctx->occ_nvl[di] = o > 0 ? o : 1;
        }
        if (e != cudaSuccess) { rc = fail(WG_ECUDA, "occupancy: %s", cudaGetErrorString(e)); break; }
    } while (0);
    if (rc != WG_OK) {
        if (ctx->arena) cudaFree(ctx->arena);
        if (ctx->status_host) cudaFreeHost(ctx->status_host);
        if (ctx->err_host) cudaFreeHost(ctx->err_host);
        delete ctx;
        return rc;
    }
    ctx->base[c.gpu_index] = ctx->arena;
    ctx->opened[c.gpu_index] = false;
    *out = ctx;
    return WG_OK;
}

int wg_ctx_destroy(wg_ctx* ctx) {
    if (!ctx) return WG_OK;
    cudaSetDevice(ctx->cfg.device);
    cudaDeviceSynchronize();
    for (int g = 0; g < kMaxGpus; ++g)
        if (ctx->opened[g] && ctx->base[g]) cudaIpcCloseMemHandle(ctx->base[g]);
    if (ctx->arena) cudaFree(ctx->arena);
    if (ctx->status_host) cudaFreeHost(ctx->status_host);
    if (ctx->err_host) cudaFreeHost(ctx->err_host);
    delete ctx;
    return WG_OK;
}

int wg_ctx_export(wg_ctx* ctx, void* blob, size_t cap, size_t* len) {
    if (!ctx || !blob || !len) return fail(WG_EINVAL, "null argument");
    if (cap < sizeof(Blob)) return fail(WG_EINVAL, "blob capacity %zu < %zu", cap, sizeof(Blob));
    Blob b;
    std::memset(&b, 0, sizeof(b));
    b.magic = kBlobMagic;
    b.gpu_index = ctx->cfg.gpu_index;
    b.P = ctx->cfg.P;
    b.R = ctx->R;
    b.D = ctx->D;
    b.Dv = ctx->Dv;
    b.dtype = ctx->cfg.dtype;
    b.n = ctx->cfg.n;
    b.arena_bytes = ctx->L.total;
    b.use_nvl = ctx->use_nvl;
    b.use_split = ctx->use_split;
    b.split_span = ctx->split_span;
    b.fence_scope = ctx->fence_scope;
    b.sms = ctx->sms;
    b.occ_split = ctx->occ_split[ctx->cfg.dtype == WG_F32 ? 0 : 1];
    b.occ_nvl = ctx->occ_nvl[ctx->cfg.dtype == WG_F32 ? 0 : 1];
    b.split_min_bytes = ctx->split_min_bytes;
    b.hier_split_max_bytes = ctx->hier_split_max_bytes;
    b.use_hier = ctx->use_hier;
    b.use_mg = ctx->use_mg;
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    WG_CUDA(cudaIpcGetMemHandle(&b.handle, ctx->arena));
    std::memcpy(blob, &b, sizeof(b));
    *len = sizeof(b);
    return WG_OK;
}

int wg_ctx_import_peer(wg_ctx* ctx, int gpu_index, const void* blob, size_t len) {
    if (!ctx || !blob) return fail(WG_EINVAL, "null argument");
    if (len != sizeof(Blob)) return fail(WG_EINVAL, "blob length %zu != %zu", len, sizeof(Blob));
    Blob b;
    std::memcpy(&b, blob, sizeof(b));
    if (b.magic != kBlobMagic) return fail(WG_EINVAL, "bad blob magic");
    if (b.gpu_index != gpu_index || gpu_index < 0 || gpu_index >= ctx->cfg.n_gpus)
        return fail(WG_EINVAL, "blob is for gpu %d, expected %d", b.gpu_index, gpu_index);
    if (b.P != ctx->cfg.P || b.R != ctx->R || b.D != ctx->D || b.Dv != ctx->Dv || b.dtype != ctx->cfg.dtype ||
        b.n != ctx->cfg.n || b.arena_bytes != ctx->L.total)
        return fail(WG_EINVAL, "peer %d context geometry differs", gpu_index);
    const int di = ctx->cfg.dtype == WG_F32 ? 0 : 1;
    if (b.use_nvl != ctx->use_nvl || b.use_split != ctx->use_split || b.split_span != ctx->split_span ||
        b.fence_scope != ctx->fence_scope || b.sms != ctx->sms || b.occ_split != ctx->occ_split[di] ||
        b.occ_nvl != ctx->occ_nvl[di] || b.split_min_bytes != ctx->split_min_bytes || b.use_hier != ctx->use_hier ||
        b.hier_split_max_bytes != ctx->hier_split_max_bytes ||
        b.use_mg != ctx->use_mg)
        return fail(WG_EINVAL,
                    "peer %d runs different kernel settings (WG_NVL/WG_SPLIT/WG_SPLIT_SPAN/WG_SPLIT_MIN_BYTES/"
                    "WG_FENCE_SCOPE/WG_HIER/WG_MG or SM count / occupancy differ)", gpu_index);
    if (gpu_index == ctx->cfg.gpu_index) return WG_OK;
    if (ctx->opened[gpu_index]) return WG_OK;
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    void* ptr = nullptr;
    WG_CUDA(cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess));
    ctx->base[gpu_index] = static_cast<char*>(ptr);
    ctx->opened[gpu_index] = true;
    return WG_OK;
}

static int local_index(wg_ctx* ctx, int rank) {
    if (rank < 0 || rank >= ctx->cfg.P || rank / ctx->R != ctx->cfg.gpu_index) return -1;
    return rank % ctx->R;
}

int wg_ctx_set_initial_model(wg_ctx* ctx, int rank, const void* w0, void* stream) {
    if (!ctx) return fail(WG_EINVAL, "null ctx");
    const int l = local_index(ctx, rank);
    if (l < 0) return fail(WG_EINVAL, "rank %d is not hosted by gpu %d", rank, ctx->cfg.gpu_index);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    char* slot0 = ctx->arena + ctx->L.ring + (int64_t(l) * ctx->D + 0) * ctx->npad * int64_t(ctx->esize);
    WG_CUDA(cudaMemsetAsync(slot0, 0, size_t(ctx->npad) * ctx->esize, s));
    if (ctx->cfg.n > 0) WG_CUDA(cudaMemcpyAsync(slot0, w0, size_t(ctx->cfg.n) * ctx->esize, cudaMemcpyDeviceToDevice, s));
    int64_t* flags0 = reinterpret_cast<int64_t*>(ctx->arena + ctx->L.flags) + int64_t(l) * ctx->n_tiles * kWarps;
    fill_i64_kernel<<<64, 256, 0, s>>>(flags0, ctx->n_tiles * kWarps, -1);
    int64_t* comp = reinterpret_cast<int64_t*>(ctx->arena + ctx->L.complete) + int64_t(l) * ctx->D + 0;
    fill_i64_kernel<<<1, 32, 0, s>>>(comp, 1, -1);
    WG_CUDA(cudaGetLastError());
    return WG_OK;
}

int wg_install(wg_ctx* ctx, int rank, int64_t stamp, const void* vec, void* stream) {
    if (!ctx || (!vec && ctx->cfg.n)) return fail(WG_EINVAL, "null argument");
    const int l = local_index(ctx, rank);
    if (l < 0) return fail(WG_EINVAL, "rank %d is not hosted by gpu %d", rank, ctx->cfg.gpu_index);
    if (stamp < 0) return fail(WG_EINVAL, "install stamp must be >= 0");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    const int slot = int((stamp + 1) % ctx->D);
    char* dst = ctx->arena + ctx->L.ring + (int64_t(l) * ctx->D + slot) * ctx->npad * int64_t(ctx->esize);
    if (ctx->cfg.n > 0) WG_CUDA(cudaMemcpyAsync(dst, vec, size_t(ctx->cfg.n) * ctx->esize, cudaMemcpyDeviceToDevice, s));
    int64_t* flags = reinterpret_cast<int64_t*>(ctx->arena + ctx->L.flags) + int64_t(l) * ctx->n_tiles * kWarps;
    fill_i64_kernel<<<64, 256, 0, s>>>(flags, ctx->n_tiles * kWarps, stamp);
    int64_t* comp = reinterpret_cast<int64_t*>(ctx->arena + ctx->L.complete) + int64_t(l) * ctx->D + slot;
    fill_i64_kernel<<<1, 32, 0, s>>>(comp, 1, stamp);
    int64_t* mark = reinterpret_cast<int64_t*>(ctx->arena + ctx->L.syncmark) + int64_t(l) * ctx->D + slot;
    fill_i64_kernel<<<1, 32, 0, s>>>(mark, 1, 2 * (stamp + 1));
    int64_t* ann = reinterpret_cast<int64_t*>(ctx->arena + ctx->L.announce) + int64_t(l) * kAnnounceStride;
    fill_i64_kernel<<<1, 32, 0, s>>>(ann, 1, stamp);
    WG_CUDA(cudaGetLastError());
    return WG_OK;
}

int wg_ctx_slot(wg_ctx* ctx, int rank, int64_t stamp, void** ptr, int64_t* held_stamp) {
    if (!ctx || !ptr) return fail(WG_EINVAL, "null argument");
    if (rank < 0 || rank >= ctx->cfg.P || stamp < -1) return fail(WG_EINVAL, "rank/stamp out of range");
    char* b = ctx->base[rank / ctx->R];
    if (!b) return fail(WG_EINVAL, "gpu %d not imported", rank / ctx->R);
    const int l = rank % ctx->R;
    const int slot = int((stamp + 1) % ctx->D);
    *ptr = b + ctx->L.ring + (int64_t(l) * ctx->D + slot) * ctx->npad * int64_t(ctx->esize);
    if (held_stamp) {
        WG_CUDA(cudaSetDevice(ctx->cfg.device));
        WG_CUDA(cudaMemcpy(held_stamp, b + ctx->L.complete + (int64_t(l) * ctx->D + slot) * 8, 8,
                           cudaMemcpyDeviceToHost));
    }
    return WG_OK;
}

static int occupancy(wg_ctx* ctx, int n_stage) {
    if (ctx->occ[n_stage] > 0) return ctx->occ[n_stage];
    int occ = 0;
    const size_t smem = dyn_smem_bytes(n_stage, ctx->cfg.n_gpus > 1);
    const bool ahead = ctx->cfg.n_gpus > 1;
    cudaError_t e;
    if (ctx->cfg.dtype == WG_F32)
        e = ahead ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wagma_step_kernel<float, true>, kThreads, smem)
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wagma_step_kernel<float, false>, kThreads, smem);
    else
        e = ahead ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wagma_step_kernel<double, true>, kThreads, smem)
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wagma_step_kernel<double, false>, kThreads, smem);
    if (e != cudaSuccess || occ < 1) occ = 1;
    ctx->occ[n_stage] = occ;
    return occ;
}

// Input-ring stages of wagma_local_kernel for a launch of n_jobs jobs (the W'
// stage takes one chunk row per job); < 2 means the launch does not fit.
static bool L_has_parts(const wg_ctx* ctx) { return ctx->L.part_ring > ctx->L.part_flags; }
static bool L_has_red(const wg_ctx* ctx) { return ctx->L.red_ring > ctx->L.red_flags; }

static int local_stages(wg_ctx* ctx, int n_jobs) {
    const int64_t row = int64_t(kLocChunkVecs) * 16;
    const int64_t avail = int64_t(ctx->loc_dyn_max[ctx->cfg.dtype == WG_F32 ? 0 : 1]) - (WG_LOC_STACK ? 0 : int64_t(n_jobs) * row);
    if (avail < 2 * 3 * row) return 0;
    return int(std::min<int64_t>(kLocMaxStages, avail / (3 * row)));
}

int wg_launch(wg_ctx* ctx, const wg_job* jobs, int n_jobs, const int64_t* forced_versions,
              const int64_t* forced_stamps, int n_forced, void* stream) {
    if (!ctx || (!jobs && n_jobs)) return fail(WG_EINVAL, "null argument");
    const wg_config& c = ctx->cfg;
    if (n_jobs < 1 || n_jobs > ctx->R) return fail(WG_EINVAL, "n_jobs=%d must be in [1, %d]", n_jobs, ctx->R);
    if (n_forced < 0 || n_forced > kMaxVersions || (n_forced && (!forced_versions || !forced_stamps)))
        return fail(WG_EINVAL, "forced stamp table");
    for (int g = 0; g < c.n_gpus; ++g)
        if (!ctx->base[g]) return fail(WG_EINVAL, "peer gpu %d not imported", g);

    static thread_local LaunchParams p;
    std::memset(&p, 0, sizeof(p));
    for (int g = 0; g < kMaxGpus; ++g) p.base[g] = ctx->base[g];
    p.L = ctx->L;
    p.P = c.P;
    p.S = c.S;
    p.R = ctx->R;
    p.G = c.n_gpus;
    p.gpu_index = c.gpu_index;
    p.D = ctx->D;
    p.Dv = ctx->Dv;
    p.need_fence = c.n_gpus > 1;
    p.n = c.n;
    p.npad = ctx->npad;
    p.n_tiles = ctx->n_tiles;
    p.tile_elems = ctx->tile_elems;
    p.grace_ns = c.grace_ns;
    p.adaptive_grace = ctx->adaptive_grace;
    p.timeout_ns = c.timeout_ns;
    p.staleness_bound = c.staleness_bound;
    p.status = ctx->status_dev;
    p.prof = ctx->prof;
    p.fence_scope = ctx->fence_scope;
    p.split_span = ctx->split_span;
    p.err_host = ctx->err_host_dev;
    for (int q = 0; q < kMaxP; ++q) p.job_of_rank[q] = -1;

    const size_t align_mask = 15;
    auto misaligned = [&](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & align_mask) != 0; };
    // jobs and their versions
    for (int j = 0; j < n_jobs; ++j) {
        const wg_job& in = jobs[j];
        const int l = local_index(ctx, in.rank);
        if (l < 0) return fail(WG_EINVAL, "job %d: rank %d not hosted here", j, in.rank);
        if (p.job_of_rank[in.rank] >= 0) return fail(WG_EINVAL, "rank %d has two jobs in one launch", in.rank);
        if (in.kind < WG_JOB_STEP || in.kind > WG_JOB_SYNC_SUM) return fail(WG_EINVAL, "job %d: kind", j);
        if (in.version < 0) return fail(WG_EINVAL, "job %d: negative version", j);
        const bool fused = in.kind <= WG_JOB_LOCAL_STEP;
        if (fused) {
            if (c.n && (!in.W || !in.g || misaligned(in.W) || misaligned(in.g)))
                return fail(WG_EINVAL, "job %d: W/g must be 16-byte aligned device pointers", j);
            if (in.update_rule == WG_UPDATE_MOMENTUM && c.n && (!in.m || misaligned(in.m)))
                return fail(WG_EINVAL, "job %d: momentum buffer", j);
            if (in.update_rule != WG_UPDATE_SGD && in.update_rule != WG_UPDATE_MOMENTUM)
                return fail(WG_EINVAL, "job %d: update rule", j);
        } else if (c.n && (!in.fresh || !in.acc_out || misaligned(in.fresh) || misaligned(in.acc_out))) {
            return fail(WG_EINVAL, "job %d: fresh/acc_out must be 16-byte aligned device pointers", j);
        }
        DevJob& d = p.jobs[j];
        d.rank = in.rank;
        d.local = l;
        d.kind = in.kind;
        d.update_rule = in.update_rule;
        d.version = in.version;
        d.eta = in.eta;
        d.beta = in.beta;
        d.W = in.W;
        d.m = in.m;
        d.g = in.g;
        d.fresh = in.fresh;
        d.acc_out = in.acc_out;
        d.produces = in.kind != WG_JOB_LOCAL_STEP;
        d.plan = -1;
        d.vidx = -1;
        p.job_of_rank[in.rank] = j;
        if (in.kind == WG_JOB_LOCAL_STEP) continue;
        const bool sync = in.kind == WG_JOB_SYNC_STEP || in.kind == WG_JOB_SYNC_SUM;
        int vi = -1;
        for (int k = 0; k < p.n_versions; ++k)
            if (p.versions[k].version == in.version) vi = k;
        if (vi < 0) {
            if (p.n_versions == kMaxVersions) return fail(WG_EINVAL, "too many versions in one launch");
            vi = p.n_versions++;
            DevVersion& dv = p.versions[vi];
            dv.version = in.version;
            dv.forced_idx = -1;
            if (sync) {
                dv.mode = kSync;
            } else {
                for (int f = 0; f < n_forced; ++f)
                    if (forced_versions[f] == in.version) dv.forced_idx = f;
                dv.mode = dv.forced_idx >= 0 ? kForced : (c.activation_enabled ? kLive : kBlocking);
            }
        } else if ((p.versions[vi].mode == kSync) != sync) {
            // collective.py:381-386: one rank syncs at t while another joins t as a group round
            return fail(WG_ESYNC, "version %lld mixes sync and group jobs (mismatched sync points)",
                        (long long)in.version);
        }
        d.vidx = vi;
    }
    for (int f = 0; f < n_forced; ++f)
        for (int q = 0; q < c.P; ++q) p.forced[f][q] = forced_stamps[int64_t(f) * c.P + q];
    p.n_jobs = n_jobs;

    // summation plans: one per distinct (version, group)
    int leaves[kMaxLeaves];
    for (int j = 0; j < n_jobs; ++j) {
        DevJob& d = p.jobs[j];
        if (d.kind == WG_JOB_LOCAL_STEP) continue;
        const bool sync = d.kind == WG_JOB_SYNC_STEP || d.kind == WG_JOB_SYNC_SUM;
        int nl = 0;
        if (sync) {
            nl = c.P;  // masks 1,2,..,P/2 (collective.py:368): leaf i = rank i
            for (int i = 0; i < nl; ++i) leaves[i] = i;
        } else {
            int grp[kMaxP], ng = 0;
            int rc = group_of(c.P, c.S, d.version, c.mask_rule, d.rank, grp, &ng);
            if (rc) return fail(rc, "group_of failed");
            rc = tree_leaves(c.P, c.S, d.version, c.mask_rule, grp[0], leaves, &nl);
            if (rc) return fail(rc, "tree_leaves failed");
            if (p.versions[d.vidx].mode == kBlocking || p.versions[d.vidx].mode == kSync) {
                // blocking: every local member must join in this launch
                for (int i = 0; i < ng; ++i) {
                    const int q = grp[i];
                    if (q / ctx->R != c.gpu_index) continue;
                    const int jq = p.job_of_rank[q];
                    if (jq < 0 || jobs[jq].version != d.version)
                        return fail(WG_EINVAL, "blocking version %lld: local member %d not in launch",
                                    (long long)d.version, q);
                }
            }
        }
        int pl = -1;
        for (int k = 0; k < p.n_plans && pl < 0; ++k) {
            const DevPlan& P_ = p.plans[k];
            if (P_.vidx != d.vidx || P_.n_leaves != nl) continue;
            bool same = true;
            for (int i = 0; i < nl && same; ++i) same = P_.leaves[i] == leaves[i];
            const bool same_kind = (p.jobs[P_.members[0]].kind == WG_JOB_SYNC_STEP ||
                                    p.jobs[P_.members[0]].kind == WG_JOB_SYNC_SUM) == sync;
            if (same && same_kind) pl = k;
        }
        if (pl < 0) {
            if (p.n_plans == kMaxPlans) return fail(WG_EINVAL, "too many plans");
            pl = p.n_plans++;
            DevPlan& P_ = p.plans[pl];
            P_.vidx = d.vidx;
            P_.n_leaves = nl;
            P_.log_leaves = ilog2(nl);
            P_.divisor = sync ? c.P : c.S;
            P_.divisor_pow2 = is_pow2(P_.divisor);
            int own[kMaxLeaves], no = 0;
            for (int i = 0; i < nl; ++i) own[no++] = leaves[i];
            std::sort(own, own + no);
            no = int(std::unique(own, own + no) - own);
            p.owners[pl].n = no;
            for (int i = 0; i < no; ++i) p.owners[pl].rank[i] = int16_t(own[i]);
            P_.n_members = 0;
            for (int i = 0; i < nl; ++i) P_.leaves[i] = int16_t(leaves[i]);
        }
        DevPlan& P_ = p.plans[pl];
        P_.members[P_.n_members++] = int8_t(j);
        d.plan = pl;
    }
    {
        // sync versions: all local ranks must join in the same launch
        for (int vi = 0; vi < p.n_versions; ++vi) {
            if (p.versions[vi].mode != kSync) continue;
            for (int l = 0; l < ctx->R; ++l) {
                const int q = c.gpu_index * ctx->R + l;
                const int jq = p.job_of_rank[q];
                if (jq < 0 || jobs[jq].version != p.versions[vi].version)
                    return fail(WG_EINVAL, "sync version %lld: local rank %d not in launch",
                                (long long)p.versions[vi].version, q);
            }
        }
    }

    // producer job order (identity unless subtree partials are produced)
    for (int j = 0; j < n_jobs; ++j) {
        p.job_order[j] = int8_t(j);
        p.job_part[j] = -1;
    }
    // Single GPU (register-stack kernel): jobs in each plan's leaf order when
    // every leaf is a distinct job of this launch at the plan's version
    // (plan_hl = 1 marks such a plan; the device confirms with the stamps)
    if (!p.need_fence && WG_LOC_STACK) {
        int nord = 0;
        bool placed[kMaxJobs] = {};
        for (int k = 0; k < p.n_plans; ++k) {
            const DevPlan& P_ = p.plans[k];
            bool ok = P_.n_leaves <= 16 && p.owners[k].n == P_.n_leaves;
            for (int li = 0; li < P_.n_leaves && ok; ++li) {
                const int jq = p.job_of_rank[P_.leaves[li]];
                ok = jq >= 0 && p.jobs[jq].produces && p.jobs[jq].vidx == P_.vidx && !placed[jq];
            }
            p.plan_hl[k] = int8_t(ok);
            if (!ok) continue;
            for (int li = 0; li < P_.n_leaves; ++li) {
                const int jq = p.job_of_rank[P_.leaves[li]];
                placed[jq] = true;
                p.job_order[nord] = int8_t(jq);
                p.job_part[nord] = int8_t(k);
                p.job_ppos[nord] = int8_t(li);
                p.job_plast[nord] = int8_t(li == P_.n_leaves - 1);
                ++nord;
            }
        }
        for (int j = 0; j < n_jobs; ++j)
            if (!placed[j]) {
                p.job_order[nord] = int8_t(j);
                p.job_part[nord] = -1;
                ++nord;
            }
    }
    // Hierarchical sums: a plan spanning GPUs whose lowest hl tree levels
    // stay inside one GPU (masks < R under the block rank mapping,
    // topology.py:127-128) is summed from GPU-local subtree partials of
    // 2^hl leaves when all members are timely; the producers compute this
    // GPU's partials in the butterfly order (bits unchanged). The choice
    // depends only on the schedule and this launch's jobs, identical on
    // every GPU that runs all its ranks at one version.
    bool any_hier = false;
    if (p.need_fence && ctx->use_hier && L_has_parts(ctx)) {
        int nord = 0, np = 0;
        bool placed[kMaxJobs] = {};
        for (int k = 0; k < p.n_plans; ++k) {
            DevPlan& P_ = p.plans[k];
            int hl = 0;
            unsigned gpus = 0;
            for (int li = 0; li < P_.n_leaves; ++li) gpus |= 1u << (P_.leaves[li] / ctx->R);
            if (__builtin_popcount(gpus) >= 2 && p.owners[k].n == P_.n_leaves) {
                for (int h = P_.log_leaves - 1; h >= 1 && !hl; --h) {
                    bool ok = true;
                    for (int li = 0; li < P_.n_leaves && ok; ++li)
                        ok = P_.leaves[li] / ctx->R == P_.leaves[li & ~((1 << h) - 1)] / ctx->R;
                    if (ok) hl = h;
                }
            }
            // this GPU produces its partials: every local leaf is a job of this launch at the plan's version
            for (int li = 0; li < P_.n_leaves && hl; ++li) {
                const int q = P_.leaves[li];
                if (q / ctx->R != c.gpu_index) continue;
                const int jq = p.job_of_rank[q];
                if (jq < 0 || !p.jobs[jq].produces || p.jobs[jq].vidx != P_.vidx || placed[jq]) hl = 0;
            }
            p.plan_hl[k] = int8_t(hl);
            if (!hl) continue;
            any_hier = true;
            for (int u = 0; u < (P_.n_leaves >> hl); ++u) {
                const int key = P_.leaves[u << hl];
                if (key / ctx->R != c.gpu_index) continue;
                if (np == kMaxJobs) return fail(WG_EINVAL, "too many subtree partials");
                p.part_key[np] = int16_t(key);
                p.part_version[np] = p.versions[P_.vidx].version;
                for (int i = 0; i < (1 << hl); ++i) {
                    const int jq = p.job_of_rank[P_.leaves[(u << hl) + i]];
                    placed[jq] = true;
                    p.job_order[nord] = int8_t(jq);
                    p.job_part[nord] = int8_t(np);
                    p.job_ppos[nord] = int8_t(i);
                    p.job_plast[nord] = int8_t(i == (1 << hl) - 1);
                    ++nord;
                }
                ++np;
            }
        }
        for (int j = 0; j < n_jobs; ++j)
            if (!placed[j]) {
                p.job_order[nord] = int8_t(j);
                p.job_part[nord] = -1;
                ++nord;
            }
        p.n_parts = np;
    }

    // dynamic shared memory: the cp.async input ring + one 16-byte stage
    // vector per thread per job (x2 when tiles are produced one ahead for
    // peers on other GPUs)
    const int n_stage = n_jobs * (p.need_fence ? 2 : 1);
    const size_t smem = dyn_smem_bytes(n_stage, p.need_fence);
    const int occ = occupancy(ctx, n_stage);
    const int64_t grid = std::min<int64_t>(ctx->n_tiles, int64_t(occ) * ctx->sms);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    WG_CUDA(cudaSetDevice(c.device));
    // multi-GPU: the TMA-puller kernel when its shared-memory rings fit
    int n_leaves_total = 0, n_rows = 0;
    for (int k = 0; k < p.n_plans; ++k) {
        n_leaves_total += p.plans[k].n_leaves;
        for (int li = 0; li < p.plans[k].n_leaves; ++li)
            n_rows += WG_NVL_TMA_LOCAL || p.plans[k].leaves[li] / ctx->R != c.gpu_index;
    }
    const size_t row = size_t(kThreads) * 16;
    const size_t nvl_fixed = size_t(kNvlDepth * 3) * row;
    const int nvl_stages =
        n_rows == 0 ? kNvlMaxStages
                    : int(std::min<size_t>(kNvlMaxStages, (size_t(kNvlMaxDyn) - nvl_fixed) / (size_t(n_rows) * row)));
    bool wide = false;  // some group of this launch spans >= 4 GPUs (same answer on every GPU)
    for (int k = 0; k < p.n_plans; ++k) {
        unsigned gpus = 0;
        for (int li = 0; li < p.plans[k].n_leaves; ++li) gpus |= 1u << (p.plans[k].leaves[li] / ctx->R);
        wide = wide || (__builtin_popcount(gpus) >= ctx->split_span && p.owners[k].n == p.plans[k].n_leaves &&
                        split_pays(p.owners[k].n, __builtin_popcount(gpus)));
    }
    // hierarchical plans whose subtree partials are worth reduce-scattering
    // (the split kernel then sums partials; same answer on every GPU)
    bool wide_h = false;
    for (int k = 0; k < p.n_plans && any_hier; ++k) {
        if (!p.plan_hl[k]) continue;
        unsigned gpus = 0;
        for (int li = 0; li < p.plans[k].n_leaves; ++li) gpus |= 1u << (p.plans[k].leaves[li] / ctx->R);
        const int np = p.plans[k].n_leaves >> p.plan_hl[k];
        wide_h = wide_h || (WG_SPLIT_TMA_LOCAL && __builtin_popcount(gpus) >= ctx->split_span &&
                            split_pays(np, __builtin_popcount(gpus)));
    }
    // Large replicas: reduce-scattering the partials (4+ GPUs) measured slower
    // than the leaf-level split (4 GPUs, S=8: 268 MB 1.104 vs 1.065 ms, 852 MB
    // 3.39 vs 3.09 ms; 102 MB 0.453 vs 0.483 ms): above hier_split_max_bytes such
    // a launch sums leaves (same decision on every GPU: it depends on the schedule)
    if (any_hier && wide_h && !ctx->use_mg && c.n * int64_t(ctx->esize) > ctx->hier_split_max_bytes) {
        any_hier = false;
        wide_h = false;
        for (int j = 0; j < n_jobs; ++j) {
            p.job_order[j] = int8_t(j);
            p.job_part[j] = -1;
        }
        for (int k = 0; k < p.n_plans; ++k) p.plan_hl[k] = 0;
        p.n_parts = 0;
    }
    int mg_rows_in = 0, mg_cap_a = 0, mg_cap_b = 0, mg_nsi = 0;
    if (any_hier && ctx->use_mg) {
        // wagma_mg_kernel shared memory, in chunk rows: input ring (3 rows per
        // stage) + W' stage (one row per job) + phase-1 rows + phase-2 rows.
        // Phase 1 must fit two chunks of the pull fallback (every remote leaf
        // of every plan: a member may turn out stale at lock-in) and two of
        // the hierarchical rows; phase 2 two chunks of reduced rows. The
        // deepest input ring that leaves that much wins (bytes in flight per
        // SM are what the produce stream is bound by).
        const int64_t row = int64_t(kLocChunkVecs) * 16;
        const int total_rows = int(ctx->mg_dyn_max[c.dtype == WG_F32 ? 0 : 1] / row);
        int n_split = 0, n_remote = 0, hier_rows = 0;
        for (int k = 0; k < p.n_plans; ++k) {
            for (int li = 0; li < p.plans[k].n_leaves; ++li) n_remote += p.plans[k].leaves[li] / ctx->R != c.gpu_index;
            if (!p.plan_hl[k]) continue;
            const int np = p.plans[k].n_leaves >> p.plan_hl[k];
            unsigned gpus = 0;
            for (int li = 0; li < p.plans[k].n_leaves; ++li) gpus |= 1u << (p.plans[k].leaves[li] / ctx->R);
            n_split += ctx->use_split && L_has_red(ctx) && split_pays(np, __builtin_popcount(gpus));
            hier_rows += np - WG_MG_DIRECT_LOCAL;  // the other GPUs' partials (this GPU's from L2)
        }
        for (int nsi = std::min(ctx->mg_nsi_max, kLocMaxStages); nsi >= 2 && !mg_nsi; --nsi) {
            const int rows_in = nsi * 3 + n_jobs;
            const int rest = total_rows - rows_in;
            const int cap_b = n_split ? std::min(8 * n_split, rest / 3) : 0;
            const int cap_a = rest - cap_b;
            if (cap_a >= std::max(n_remote, 2 * hier_rows) && cap_b >= 2 * n_split) {
                mg_nsi = nsi;
                mg_rows_in = rows_in;
                mg_cap_a = cap_a;
                mg_cap_b = cap_b;
            }
        }
    }
    if (mg_cap_a > 0) {
        p.loc_stages = mg_nsi;
        p.mg_cap_a = mg_cap_a;
        p.mg_cap_b = mg_cap_b;
        p.mg_split = ctx->use_split && L_has_red(ctx) && c.n * int64_t(ctx->esize) >= ctx->split_min_bytes;
        const size_t smem_mg = size_t(mg_rows_in + mg_cap_a + mg_cap_b) * size_t(kLocChunkVecs) * 16;
        const int64_t n_chunks = (ctx->n_tiles + kLocTiles - 1) / kLocTiles;
        const int64_t g = std::min<int64_t>(n_chunks, ctx->sms);
        if (c.dtype == WG_F32)
            wagma_mg_kernel<float><<<unsigned(g), kMgThreads, smem_mg, s>>>(p);
        else
            wagma_mg_kernel<double><<<unsigned(g), kMgThreads, smem_mg, s>>>(p);
    } else if (p.need_fence && ctx->use_split && c.P <= kSplitMaxP && c.n_gpus >= ctx->split_span &&
               (any_hier ? wide_h : wide) && c.n * int64_t(ctx->esize) >= ctx->split_min_bytes) {
        // split sums: every GPU of a job makes this same choice (it depends on
        // P and the process-wide knob only), so owners always publish the
        // reduced tiles their peers wait for
        // stream B (1 row per plan) gets what stream A (all leaves) leaves
        // after 4 stages, between 2 and 16 stages each
        int n_rows_split = 0;
        for (int k = 0; k < p.n_plans; ++k)
            for (int li = 0; li < p.plans[k].n_leaves; ++li)
                n_rows_split += WG_SPLIT_TMA_LOCAL || p.plans[k].leaves[li] / ctx->R != c.gpu_index;
        const size_t rowsA = size_t(std::max(n_rows_split, 1)) * row, rowsB = size_t(p.n_plans) * row;
        const size_t split_fixed = size_t(kSplitDepth * 3) * row;
        const size_t avail = size_t(kNvlMaxDyn) > split_fixed ? size_t(kNvlMaxDyn) - split_fixed : 0;
        const int nsb = int(std::max<size_t>(
            2, std::min<size_t>(WG_SPLIT_NSB, avail > WG_SPLIT_NSA_MIN * rowsA
                                                  ? (avail - WG_SPLIT_NSA_MIN * rowsA) / rowsB
                                                  : 0)));
        const size_t fixed = split_fixed + size_t(nsb) * rowsB;
        const int nsa = fixed >= size_t(kNvlMaxDyn)
                            ? 0
                            : int(std::min<size_t>(kNvlMaxStages, (size_t(kNvlMaxDyn) - fixed) / rowsA));
        if (nsa < 2 || n_leaves_total * kWarps > kMaxPoll)
            return fail(WG_EINVAL, "split launch does not fit shared memory (%d leaves)", n_leaves_total);
        p.nvl_stages = nsa;
        p.split_stages = nsb;
        int span_max = 0;
        for (int k = 0; k < p.n_plans; ++k) {
            unsigned gpus = 0;
            for (int li = 0; li < p.plans[k].n_leaves; ++li) gpus |= 1u << (p.plans[k].leaves[li] / ctx->R);
            span_max = std::max(span_max, __builtin_popcount(gpus));
        }
        p.red_warps = WG_RED_WARPS ? WG_RED_WARPS : (span_max >= 4 ? 4 : 8);
        const size_t smem_split = fixed + size_t(nsa) * n_rows_split * row;
        const int di = c.dtype == WG_F32 ? 0 : 1;
        if (ctx->occ_split[di] <= 0) {
            int o = 0;
            cudaError_t e2 = c.dtype == WG_F32
                                 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_split_kernel<float>,
                                                                                 kSplitThreads, kNvlMaxDyn)
                                 : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_split_kernel<double>,
                                                                                 kSplitThreads, kNvlMaxDyn);
            ctx->occ_split[di] = (e2 == cudaSuccess && o > 0) ? o : 1;
        }
        const int64_t g = std::min<int64_t>(ctx->n_tiles, int64_t(ctx->occ_split[di]) * ctx->sms);
        if (c.dtype == WG_F32)
            wagma_split_kernel<float><<<unsigned(g), kSplitThreads, smem_split, s>>>(p);
        else
            wagma_split_kernel<double><<<unsigned(g), kSplitThreads, smem_split, s>>>(p);
    } else if (p.need_fence && ctx->use_nvl && nvl_stages >= 2 && n_leaves_total * kWarps <= kMaxPoll &&
        n_leaves_total <= kMaxPlans * kMaxLeaves) {
        p.nvl_stages = nvl_stages;
        p.nvl_rows = n_rows;
        p.tma_prod = n_jobs >= 2;
        const size_t nvl_smem = nvl_fixed + size_t(nvl_stages) * n_rows * row;
        const int di = c.dtype == WG_F32 ? 0 : 1;
        if (ctx->occ_nvl[di] <= 0) {
            int o = 0;
            cudaError_t e2 = c.dtype == WG_F32
                                 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_nvl_kernel<float>,
                                                                                 kNvlThreads, kNvlMaxDyn)
                                 : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wagma_nvl_kernel<double>,
                                                                                 kNvlThreads, kNvlMaxDyn);
            ctx->occ_nvl[di] = (e2 == cudaSuccess && o > 0) ? o : 1;
        }
        const int64_t g = std::min<int64_t>(ctx->n_tiles, int64_t(ctx->occ_nvl[di]) * ctx->sms);
        if (c.dtype == WG_F32)
            wagma_nvl_kernel<float><<<unsigned(g), kNvlThreads, nvl_smem, s>>>(p);
        else
            wagma_nvl_kernel<double><<<unsigned(g), kNvlThreads, nvl_smem, s>>>(p);
    } else if (!p.need_fence && ctx->use_loc &&
               (p.loc_stages = local_stages(ctx, n_jobs)) >= 2) {
        const size_t row = size_t(kLocChunkVecs) * 16;
        const size_t loc_smem = (size_t(p.loc_stages) * 3 + (WG_LOC_STACK ? 0 : size_t(n_jobs))) * row;
        const int64_t n_chunks = (ctx->n_tiles + kLocTiles - 1) / kLocTiles;
        const int64_t g = std::min<int64_t>(n_chunks, ctx->sms);
        if (c.dtype == WG_F32)
            wagma_local_kernel<float><<<unsigned(g), kLocThreads, loc_smem, s>>>(p);
        else
            wagma_local_kernel<double><<<unsigned(g), kLocThreads, loc_smem, s>>>(p);
    } else if (c.dtype == WG_F32) {
        if (p.need_fence)
            wagma_step_kernel<float, true><<<unsigned(grid), kThreads, smem, s>>>(p);
        else
            wagma_step_kernel<float, false><<<unsigned(grid), kThreads, smem, s>>>(p);
    } else {
        if (p.need_fence)
            wagma_step_kernel<double, true><<<unsigned(grid), kThreads, smem, s>>>(p);
        else
            wagma_step_kernel<double, false><<<unsigned(grid), kThreads, smem, s>>>(p);
    }
    WG_CUDA(cudaGetLastError());
    ctx->last_n_jobs = n_jobs;
    return WG_OK;
}

int wg_launch_status(wg_ctx* ctx, int i, wg_job_status* out) {
    if (!ctx || !out) return fail(WG_EINVAL, "null argument");
    if (i < 0 || i >= ctx->last_n_jobs) return fail(WG_EINVAL, "job index %d out of range", i);
    std::memcpy(out, const_cast<const wg_job_status*>(ctx->status_host) + i, sizeof(*out));
    return WG_OK;
}

int wg_query_version(wg_ctx* ctx, int64_t version, int64_t* stamps, int* locked) {
    if (!ctx || !stamps || !locked || version < 0) return fail(WG_EINVAL, "bad argument");
    if (!ctx->base[0]) return fail(WG_EINVAL, "gpu 0 not imported");
    Desc d;
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    WG_CUDA(cudaMemcpy(&d, ctx->base[0] + ctx->L.desc + (version % ctx->Dv) * int64_t(sizeof(Desc)), sizeof(Desc),
                       cudaMemcpyDeviceToHost));
    *locked = d.state == (version + 1) * 4 + 2;
    for (int q = 0; q < ctx->cfg.P; ++q) stamps[q] = d.stamps[q];
    return WG_OK;
}

int wg_ctx_error(wg_ctx* ctx, int* code, int64_t* info) {
    if (!ctx || !code) return fail(WG_EINVAL, "null argument");
    int64_t h[2];
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    WG_CUDA(cudaMemcpy(h, ctx->arena + ctx->L.hdr, sizeof(h), cudaMemcpyDeviceToHost));
    *code = int(h[0]);
    if (info) *info = h[1];
    return WG_OK;
}

int wg_ctx_error_async(wg_ctx* ctx, int* code, int64_t* info) {
    if (!ctx || !code) return fail(WG_EINVAL, "null argument");
    const volatile int64_t* h = ctx->err_host;
    *code = int(h[0]);
    if (info) *info = h[1];
    return WG_OK;
}

int wg_ctx_clear_error(wg_ctx* ctx) {
    if (!ctx) return fail(WG_EINVAL, "null ctx");
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    WG_CUDA(cudaMemset(ctx->arena + ctx->L.hdr, 0, 16));
    ctx->err_host[0] = ctx->err_host[1] = 0;
    return WG_OK;
}

int wg_delay(wg_ctx* ctx, int64_t ns, void* stream) {
    if (!ctx) return fail(WG_EINVAL, "null ctx");
    if (ns <= 0) return WG_OK;
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    delay_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ns);
    WG_CUDA(cudaGetLastError());
    return WG_OK;
}

int wg_replicas_sum(wg_ctx* ctx, const void* const* W, int R, double* sum, void* stream) {
    if (!ctx || !W || !sum || R < 1 || R > kMaxJobs) return fail(WG_EINVAL, "bad replica list");
    ReplicaPtrs rp;
    for (int r = 0; r < R; ++r) rp.w[r] = W[r];
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ctx->cfg.dtype == WG_F32)
        replicas_sum_kernel<float><<<ctx->sms * 4, 256, 0, s>>>(rp, R, ctx->cfg.n, sum);
    else
        replicas_sum_kernel<double><<<ctx->sms * 4, 256, 0, s>>>(rp, R, ctx->cfg.n, sum);
    WG_CUDA(cudaGetLastError());
    return WG_OK;
}

int wg_replicas_spread(wg_ctx* ctx, const void* const* W, int R, const double* mu, double* out, void* stream) {
    if (!ctx || !W || !mu || !out || R < 1 || R > kMaxJobs) return fail(WG_EINVAL, "bad replica list");
    ReplicaPtrs rp;
    for (int r = 0; r < R; ++r) rp.w[r] = W[r];
    WG_CUDA(cudaSetDevice(ctx->cfg.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ctx->cfg.dtype == WG_F32)
        replicas_spread_kernel<float><<<ctx->sms * 4, 256, 0, s>>>(rp, R, ctx->cfg.n, mu, out);
    else
        replicas_spread_kernel<double><<<ctx->sms * 4, 256, 0, s>>>(rp, R, ctx->cfg.n, mu, out);
    WG_CUDA(cudaGetLastError());
    return WG_OK;
}

int wg_ctx_set_profile(wg_ctx* ctx, void* dev_buf) {
    if (!ctx) return fail(WG_EINVAL, "null ctx");
    ctx->prof = static_cast<long long*>(dev_buf);
    return WG_OK;
}

int wg_ctx_geometry(wg_ctx* ctx, int64_t* tile_elems, int64_t* n_tiles, int* grid, int* ring_depth) {
    if (!ctx) return fail(WG_EINVAL, "null ctx");
    if (tile_elems) *tile_elems = ctx->tile_elems;
    if (n_tiles) *n_tiles = ctx->n_tiles;
    if (grid) *grid = int(std::min<int64_t>(ctx->n_tiles, int64_t(occupancy(ctx, ctx->R * (ctx->cfg.n_gpus > 1 ? 2 : 1))) * ctx->sms));
    if (ring_depth) *ring_depth = ctx->D;
    return WG_OK;
}

}  // extern "C"
