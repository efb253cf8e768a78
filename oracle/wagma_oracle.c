/*
 * Oracle (TEST INFRASTRUCTURE): C restatement of one WAGMA iteration over P ranks.
 *
 * Restates the reference arithmetic of /root/reference/pkg/src/wagma
 * (see oracle/__init__.py for the usage rule -- only tests/, smoke() and
 * bench.py's CPU-baseline leg may load this library):
 *
 *   local step        m = beta*m + g ; W' = W - eta*m          optim.py:176-183
 *                     (SGD: W' = W - eta*g)                     optim.py:181-183
 *   send buffer       W' installed for peers                    collective.py:95-101
 *   group sum         per phase r: acc[p] = acc[p^mask_r] + acc[p]
 *                     (recursive doubling, incoming + acc)      collective.py:310-329
 *   averaging         timely acc/S ; late (acc + W')/(S+1)      optim.py:439-447
 *   global sync       masks 1,2,..,P/2 ; total/P                collective.py:368,428-436;
 *                                                               optim.py:449-452
 *
 * Every floating-point operation is a separate IEEE rounding in the
 * reference's operand order (compile with -ffp-contract=off). The element
 * range is processed in cache-sized blocks spread over OpenMP threads; each
 * block runs the whole iteration (all ranks, all phases), which is the
 * fastest faithful CPU schedule of the reference's per-rank message passing.
 * It is the `cpu_baseline` / `--impl reference` arm of bench.py and is
 * checked bit-exact against oracle/wagma_oracle.py by tests/test_oracle.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_BLOCK 2048
#define ORACLE_MAX_P 1024

#define DEFINE_ITERATION(T, SUFFIX)                                                              \
int oracle_wagma_iteration_##SUFFIX(int P, int S_div, const int* masks, int n_masks,             \
    long long n, T eta, T beta, int momentum,                                                    \
    T* const* W, T* const* m, const T* const* g, T* const* wprime,                               \
    const T* const* contrib, const int* timely, int nthreads)                                    \
{                                                                                                \
    if (P < 1 || P > ORACLE_MAX_P || n < 0 || n_masks < 0 || S_div < 1) return 1;               \
    for (int i = 0; i < n_masks; ++i) if (masks[i] <= 0 || masks[i] >= P) return 1;              \
    long long nblocks = (n + ORACLE_BLOCK - 1) / ORACLE_BLOCK;                                   \
    int bad = 0;                                                                                 \
    if (nthreads <= 0) nthreads = 1;                                                             \
    _Pragma("omp parallel num_threads(nthreads) reduction(|:bad)")                               \
    {                                                                                            \
        T* a = (T*)malloc(sizeof(T) * (size_t)P * ORACLE_BLOCK);                                  \
        T* b = (T*)malloc(sizeof(T) * (size_t)P * ORACLE_BLOCK);                                  \
        if (!a || !b) bad = 1;                                                                   \
        _Pragma("omp for schedule(static)")                                                      \
        for (long long blk = 0; blk < nblocks; ++blk) {                                          \
            if (!a || !b) continue;                                                              \
            long long lo = blk * ORACLE_BLOCK;                                                   \
            long long hi = lo + ORACLE_BLOCK < n ? lo + ORACLE_BLOCK : n;                        \
            int len = (int)(hi - lo);                                                            \
            /* local step per rank (optim.py:176-183) */                                         \
            for (int r = 0; r < P; ++r) {                                                        \
                T* w = W[r] + lo; const T* gr = g[r] + lo; T* wp = wprime[r] + lo;               \
                if (momentum) {                                                                  \
                    T* mr = m[r] + lo;                                                           \
                    for (int i = 0; i < len; ++i) {                                              \
                        T bm = beta * mr[i];                                                     \
                        T mn = bm + gr[i];                                                       \
                        mr[i] = mn;                                                              \
                        T step = eta * mn;                                                       \
                        wp[i] = w[i] - step;                                                     \
                    }                                                                            \
                } else {                                                                         \
                    for (int i = 0; i < len; ++i) { T step = eta * gr[i]; wp[i] = w[i] - step; }  \
                }                                                                                \
            }                                                                                    \
            /* snapshot contributions (collective.py:300) */                                     \
            for (int r = 0; r < P; ++r) {                                                        \
                const T* src = (contrib && contrib[r]) ? contrib[r] + lo : wprime[r] + lo;       \
                memcpy(a + (size_t)r * ORACLE_BLOCK, src, sizeof(T) * (size_t)len);               \
            }                                                                                    \
            /* recursive doubling: acc = incoming + acc (collective.py:325) */                   \
            T* cur = a; T* nxt = b;                                                              \
            for (int ph = 0; ph < n_masks; ++ph) {                                               \
                int mk = masks[ph];                                                              \
                for (int p = 0; p < P; ++p) {                                                    \
                    const T* inc = cur + (size_t)(p ^ mk) * ORACLE_BLOCK;                        \
                    const T* own = cur + (size_t)p * ORACLE_BLOCK;                               \
                    T* dst = nxt + (size_t)p * ORACLE_BLOCK;                                     \
                    for (int i = 0; i < len; ++i) dst[i] = inc[i] + own[i];                      \
                }                                                                                \
                T* tmp = cur; cur = nxt; nxt = tmp;                                              \
            }                                                                                    \
            /* averaging rule (optim.py:439-447; sync: optim.py:452) */                          \
            for (int r = 0; r < P; ++r) {                                                        \
                const T* acc = cur + (size_t)r * ORACLE_BLOCK;                                   \
                T* w = W[r] + lo; const T* wp = wprime[r] + lo;                                  \
                if (!timely || timely[r]) {                                                      \
                    T d = (T)S_div;                                                              \
                    for (int i = 0; i < len; ++i) w[i] = acc[i] / d;                             \
                } else {                                                                         \
                    T d = (T)(S_div + 1);                                                        \
                    for (int i = 0; i < len; ++i) { T s = acc[i] + wp[i]; w[i] = s / d; }        \
                }                                                                                \
            }                                                                                    \
        }                                                                                        \
        free(a); free(b);                                                                        \
    }                                                                                            \
    return bad ? 2 : 0;                                                                          \
}

DEFINE_ITERATION(float, f32)
DEFINE_ITERATION(double, f64)

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
