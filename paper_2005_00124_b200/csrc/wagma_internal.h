// Internal constants and host helpers shared by topology.cpp and wagma_b200.cu.
#pragma once
#include <cstdint>

namespace wg {

constexpr int kMaxTopoP = 1 << 30;  // schedule generator (host)
constexpr int kMaxP = 64;           // device path: ranks per job
constexpr int kMaxGpus = 8;         // one NVSwitch box
constexpr int kMaxJobs = 16;        // jobs (= local ranks) per launch
constexpr int kMaxVersions = 16;    // distinct versions per launch
constexpr int kMaxPlans = 16;       // distinct (version, group) sums per launch
constexpr int kMaxLeaves = 64;      // leaves of one summation tree (sync at P = 64)
constexpr int kThreads = 256;       // threads per CTA
constexpr int kVecPerThread = 1;    // 16-byte vectors per thread per tile

int check_params(int P, int S, int64_t t);
int phase_masks(int P, int S, int64_t t, int rule, int* masks, int* n_masks);
int compute_groups(int P, int S, int64_t t, int rule, int* members, int* offsets, int* n_groups);
int group_of(int P, int S, int64_t t, int rule, int rank, int* out, int* n);
int tree_leaves(int P, int S, int64_t t, int rule, int rank, int* out, int* n);
int peer(int rank, int mask, int P, int* out);
int mixing_reachable(int P, int S, int64_t start_t, int k, int rule, int* out);

}  // namespace wg
