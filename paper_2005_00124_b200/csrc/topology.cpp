// Butterfly / XOR-rotating group schedule generator (host C++).
//
// Bit-exact restatement of the reference schedule
// (/root/reference/pkg/src/wagma/topology.py): masks per iteration for the
// "example" and "literal" rules, the XOR-coset group partition sorted like
// compute_groups, peer(), mixing_reachable(), and the leaf order of the
// butterfly summation tree that the device kernel follows.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/wagma_b200.h"
#include "wagma_internal.h"

namespace wg {

static bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
static int ilog2(int64_t n) {
    int r = 0;
    while ((int64_t(1) << (r + 1)) <= n) ++r;
    return r;
}

// GroupingParams.__post_init__ (topology.py:64-72). The device path caps
// P at kMaxTopoP for the bitset-based helpers.
int check_params(int P, int S, int64_t t) {
    if (!is_pow2(P) || !is_pow2(S) || S > P || t < 0 || P > kMaxTopoP) return WG_EINVAL;
    return WG_OK;
}

// phase_masks (topology.py:118-142).
int phase_masks(int P, int S, int64_t t, int rule, int* masks, int* n_masks) {
    int rc = check_params(P, S, t);
    if (rc) return rc;
    const int gp = ilog2(S);   // group_phases (topology.py:79-80)
    const int GP = ilog2(P);   // global_phases (topology.py:75-76)
    if (rule == WG_RULE_EXAMPLE) {
        // masks[r] = 1 << ((t*gp + r) % GP)  (topology.py:127-128)
        if (GP == 0) {
            *n_masks = 0;
            return WG_OK;
        }
        const int64_t base = (t % GP) * gp % GP;  // (t*gp) mod GP without overflow
        for (int r = 0; r < gp; ++r) masks[r] = 1 << int((base + r) % GP);
        *n_masks = gp;
        return WG_OK;
    }
    if (rule == WG_RULE_LITERAL) {
        // mask = (mask << shift) % P ; 0 -> 1 ; shift = (shift+1) % GP
        // (topology.py:129-139), shift0 = (t*gp) % GP (topology.py:83-87)
        int64_t mask = 1;
        int shift = GP ? int((t % GP) * gp % GP) : 0;
        for (int r = 0; r < gp; ++r) {
            mask = (mask << shift) % P;
            if (mask == 0) mask = 1;
            masks[r] = int(mask);
            shift = GP ? (shift + 1) % GP : 0;
        }
        *n_masks = gp;
        return WG_OK;
    }
    return WG_EINVAL;
}

// _xor_span (topology.py:154-159): all XOR combinations, ascending.
static std::vector<int> xor_span(const int* masks, int n) {
    std::vector<int> span{0};
    for (int i = 0; i < n; ++i) {
        std::vector<int> add;
        for (int s : span) add.push_back(s ^ masks[i]);
        for (int a : add)
            if (std::find(span.begin(), span.end(), a) == span.end()) span.push_back(a);
    }
    std::sort(span.begin(), span.end());
    return span;
}

// compute_groups (topology.py:162-181).
int compute_groups(int P, int S, int64_t t, int rule, int* members, int* offsets, int* n_groups) {
    int masks[32];
    int nm = 0;
    int rc = phase_masks(P, S, t, rule, masks, &nm);
    if (rc) return rc;
    std::vector<int> span = xor_span(masks, nm);
    std::vector<char> seen(P, 0);
    int ng = 0, w = 0;
    offsets[0] = 0;
    std::vector<int> grp;
    for (int p = 0; p < P; ++p) {
        if (seen[p]) continue;
        grp.clear();
        for (int s : span) grp.push_back(p ^ s);
        std::sort(grp.begin(), grp.end());
        for (int q : grp) {
            seen[q] = 1;
            members[w++] = q;
        }
        offsets[++ng] = w;
    }
    *n_groups = ng;
    return WG_OK;
}

int group_of(int P, int S, int64_t t, int rule, int rank, int* out, int* n) {
    if (rank < 0 || rank >= P) return WG_EINVAL;
    int masks[32];
    int nm = 0;
    int rc = phase_masks(P, S, t, rule, masks, &nm);
    if (rc) return rc;
    std::vector<int> span = xor_span(masks, nm);
    std::vector<int> grp;
    for (int s : span) grp.push_back(rank ^ s);
    std::sort(grp.begin(), grp.end());
    for (size_t i = 0; i < grp.size(); ++i) out[i] = grp[i];
    *n = int(grp.size());
    return WG_OK;
}

// Leaf i of the recursive-doubling tree at `rank` (collective.py:310-329):
// rank ^ XOR{masks[r] : bit r of i}.
int tree_leaves(int P, int S, int64_t t, int rule, int rank, int* out, int* n) {
    if (rank < 0 || rank >= P) return WG_EINVAL;
    int masks[32];
    int nm = 0;
    int rc = phase_masks(P, S, t, rule, masks, &nm);
    if (rc) return rc;
    const int L = 1 << nm;
    for (int i = 0; i < L; ++i) {
        int q = rank;
        for (int r = 0; r < nm; ++r)
            if ((i >> r) & 1) q ^= masks[r];
        out[i] = q;
    }
    *n = L;
    return WG_OK;
}

// peer (topology.py:145-151).
int peer(int rank, int mask, int P, int* out) {
    if (rank < 0 || rank >= P) return WG_EINVAL;
    if (!(is_pow2(mask) && mask < P)) return WG_EINVAL;
    *out = rank ^ mask;
    return WG_OK;
}

// mixing_reachable (topology.py:184-208), with P-bit reach sets.
int mixing_reachable(int P, int S, int64_t start_t, int k, int rule, int* out) {
    if (k < 1 || start_t < 0) return WG_EINVAL;
    int rc = check_params(P, S, 0);
    if (rc) return rc;
    const int words = (P + 63) / 64;
    std::vector<uint64_t> reach(size_t(P) * words, 0), nxt;
    for (int p = 0; p < P; ++p) reach[size_t(p) * words + p / 64] |= uint64_t(1) << (p % 64);
    std::vector<int> members(P), offsets(P + 1);
    for (int64_t t = start_t; t < start_t + k; ++t) {
        int ng = 0;
        rc = compute_groups(P, S, t, rule, members.data(), offsets.data(), &ng);
        if (rc) return rc;
        nxt = reach;
        std::vector<uint64_t> merged(words);
        for (int g = 0; g < ng; ++g) {
            std::fill(merged.begin(), merged.end(), 0);
            for (int i = offsets[g]; i < offsets[g + 1]; ++i)
                for (int w = 0; w < words; ++w) merged[w] |= reach[size_t(members[i]) * words + w];
            for (int i = offsets[g]; i < offsets[g + 1]; ++i)
                for (int w = 0; w < words; ++w) nxt[size_t(members[i]) * words + w] = merged[w];
        }
        reach.swap(nxt);
    }
    int all = 1;
    for (int p = 0; p < P && all; ++p)
        for (int w = 0; w < words; ++w) {
            const int bits = std::min(64, P - w * 64);
            const uint64_t full = bits == 64 ? ~uint64_t(0) : ((uint64_t(1) << bits) - 1);
            if (reach[size_t(p) * words + w] != full) {
                all = 0;
                break;
            }
        }
    *out = all;
    return WG_OK;
}

}  // namespace wg

extern "C" {

int wg_check_params(int P, int S, int64_t t) { return wg::check_params(P, S, t); }
int wg_phase_masks(int P, int S, int64_t t, int rule, int* masks, int* n_masks) {
    return wg::phase_masks(P, S, t, rule, masks, n_masks);
}
int wg_compute_groups(int P, int S, int64_t t, int rule, int* members, int* offsets, int* n_groups) {
    return wg::compute_groups(P, S, t, rule, members, offsets, n_groups);
}
int wg_group_of(int P, int S, int64_t t, int rule, int rank, int* out, int* n) {
    return wg::group_of(P, S, t, rule, rank, out, n);
}
int wg_peer(int rank, int mask, int P, int* out) { return wg::peer(rank, mask, P, out); }
int wg_mixing_reachable(int P, int S, int64_t start_t, int k, int rule, int* out) {
    return wg::mixing_reachable(P, S, start_t, k, rule, out);
}
int wg_tree_leaves(int P, int S, int64_t t, int rule, int rank, int* out, int* n) {
    return wg::tree_leaves(P, S, t, rule, rank, out, n);
}

}  // extern "C"
