// levels.cu -- host planner of the level schedule (levels.h). Host code only.
#include <algorithm>
#include <queue>
#include <tuple>
#include <unordered_map>

#include "levels.h"

#include <cstdlib>

namespace mcinv {

namespace {

// stable counting sort of items by key in [0, nkeys): returns the permutation
// and fills ptr[nkeys + 1]
std::vector<int> bucket(const std::vector<int> &key, int nkeys, std::vector<int> &ptr) {
    ptr.assign(nkeys + 1, 0);
    for (int k : key) ptr[k + 1]++;
    for (int k = 0; k < nkeys; ++k) ptr[k + 1] += ptr[k];
    std::vector<int> fill(ptr.begin(), ptr.end() - 1), perm(key.size());
    for (size_t t = 0; t < key.size(); ++t) perm[fill[key[t]]++] = (int)t;
    return perm;
}

}  // namespace

std::string build_levels(const LevelInput &in, LevelPlan &P) {
    const int64_t n = in.n;
    const auto &up = *in.u_ptr;
    const auto &uc = *in.u_col;
    if ((int64_t)up.size() != n + 1) return "union lists missing";

    // lev(i) = 1 + max lev(j) over lower neighbours j < i (rows ascend, so
    // every lower neighbour is already levelled)
    P.level.assign(n, 0);
    int D = 0;
    for (int64_t i = 0; i < n; ++i) {
        int l = 0;
        for (int e = up[i]; e < up[i + 1]; ++e) {
            const int j = uc[e];
            if (j < i) l = std::max(l, P.level[j] + 1);
        }
        P.level[i] = l;
        D = std::max(D, l + 1);
    }
    P.D = D;
    const int nph = D + 1;

    // rows in level order; within a level (mutually independent rows, any order
    // is exact) by decreasing entry count, so the rows sharing a warp have
    // similar loop trip counts (less SIMT divergence); ties by ascending i
    std::vector<int> key(P.level.begin(), P.level.end());
    P.ord_row = bucket(key, nph, P.ph_row);
    P.ph_row.push_back(P.ph_row.back());  // [D+2]; phase D holds no rows
    for (int l = 0; l < D; ++l)
        std::stable_sort(P.ord_row.begin() + P.ph_row[l], P.ord_row.begin() + P.ph_row[l + 1],
                         [&](int x, int y) { return up[x + 1] - up[x] > up[y + 1] - up[y]; });

    // pattern slots: fused at the update of max(i, j) when min(i, j) is a lower
    // neighbour (or i == j); the first occurrence of a pair is fused, the rest
    // (duplicates, non-neighbour pairs) are deferred
    // (the pattern pairs sorted by row, then column, then index: a pair (a, b) is found by a
    // binary search in row a's columns; of duplicates only the first index is ever fused)
    std::vector<char> used;
    std::vector<int> pr_ptr, pr_idx;
    const int64_t pc = in.want_pattern ? (int64_t)in.p_row->size() : 0;
    if (pc > 0) {
        used.assign(pc, 0);
        const auto &pr = *in.p_row, &pcl = *in.p_col;
        std::vector<int> rk(pr.begin(), pr.end());
        pr_idx = bucket(rk, (int)n, pr_ptr);  // stable: index order within a row
        for (int64_t a = 0; a < n; ++a)
            std::stable_sort(pr_idx.begin() + pr_ptr[a], pr_idx.begin() + pr_ptr[a + 1],
                             [&](int x, int y) { return pcl[x] < pcl[y]; });
    }
    const auto take = [&](int64_t a, int64_t b) -> int {
        if (pc == 0) return -1;
        const auto &pcl = *in.p_col;
        const auto lo = std::lower_bound(pr_idx.begin() + pr_ptr[a], pr_idx.begin() + pr_ptr[a + 1], (int)b,
                                         [&](int x, int v) { return pcl[x] < v; });
        if (lo == pr_idx.begin() + pr_ptr[a + 1] || pcl[*lo] != b || used[*lo]) return -1;
        used[*lo] = 1;
        return *lo;
    };

    P.ord_eptr.assign(n + 1, 0);
    P.ord_dl.resize(n);
    P.ord_sg.resize(n);
    P.ord_pself.assign(n, -1);
    P.ent_col.clear();
    P.ent_a.clear();
    P.ent_b.clear();
    P.ent_pz.clear();
    P.ent_col.reserve(uc.size());
    P.fused_pairs = 0;
    for (int64_t o = 0; o < n; ++o) {
        const int i = P.ord_row[o];
        for (int e = up[i]; e < up[i + 1]; ++e) {
            const int j = uc[e];
            P.ent_col.push_back(j);
            P.ent_a.push_back((*in.u_a)[e]);
            P.ent_b.push_back((*in.u_b)[e]);
            if (in.want_pattern) {
                const int zx = j < i ? take(i, j) : -1;  // z_i conj(w_j)
                const int zy = j < i ? take(j, i) : -1;  // z_j conj(w_i)
                P.fused_pairs += (zx >= 0) + (zy >= 0);
                P.ent_pz.push_back(zx);
                P.ent_pz.push_back(zy);
            }
        }
        P.ord_eptr[o + 1] = (int)P.ent_col.size();
        P.ord_dl[o] = (*in.delta)[i];
        P.ord_sg[o] = (*in.sigma)[i];
        if (in.want_pattern) {
            P.ord_pself[o] = take(i, i);
            P.fused_pairs += P.ord_pself[o] >= 0;
        }
    }

    // deferred pattern pairs
    P.pp_i.clear();
    P.pp_j.clear();
    P.pp_slot.clear();
    {
        std::vector<int> pkey, pidx;
        for (int64_t p = 0; p < pc; ++p) {
            if (used[p]) continue;
            const int a = (*in.p_row)[p], b = (*in.p_col)[p];
            pkey.push_back(std::max(P.level[a], P.level[b]) + 1);
            pidx.push_back((int)p);
        }
        const std::vector<int> perm = bucket(pkey, nph, P.ph_pp);
        P.ph_pp.push_back(P.ph_pp.back());
        for (int t : perm) {
            const int p = pidx[t];
            P.pp_i.push_back((*in.p_row)[p]);
            P.pp_j.push_back((*in.p_col)[p]);
            P.pp_slot.push_back(p);
        }
        P.deferred_pairs = (int64_t)pidx.size();
    }

    // deferred trace items: Q row i -> conj(w_i) sum_j Q_ij z_j
    P.tq_row.clear();
    P.tq_eptr.assign(1, 0);
    P.tq_col.clear();
    P.tq_val.clear();
    {
        std::vector<int> tkey, trow;
        if (in.want_trace) {
            const auto &qp = *in.q_ptr;
            const auto &qc = *in.q_col;
            for (int64_t i = 0; i < n; ++i) {
                if (qp[i + 1] == qp[i]) continue;
                int l = P.level[i];
                for (int64_t e = qp[i]; e < qp[i + 1]; ++e) l = std::max(l, P.level[qc[e]]);
                tkey.push_back(l + 1);
                trow.push_back((int)i);
            }
        }
        const std::vector<int> perm = bucket(tkey, nph, P.ph_tq);
        P.ph_tq.push_back(P.ph_tq.back());
        for (int t : perm) {
            const int i = trow[t];
            P.tq_row.push_back(i);
            for (int64_t e = (*in.q_ptr)[i]; e < (*in.q_ptr)[i + 1]; ++e) {
                P.tq_col.push_back((*in.q_col)[e]);
                P.tq_val.push_back((*in.q_val)[e]);
            }
            P.tq_eptr.push_back((int)P.tq_col.size());
        }
    }

    P.max_rows = 0;
    for (int p = 0; p < nph; ++p) {
        const int w = (P.ph_row[p + 1] - P.ph_row[p]) + (P.ph_tq[p + 1] - P.ph_tq[p]) + (P.ph_pp[p + 1] - P.ph_pp[p]);
        P.max_rows = std::max(P.max_rows, w);
    }
    return "";
}

#ifndef MCINV_WINDOW_PER_GROUP
#define MCINV_WINDOW_PER_GROUP 1
#endif
constexpr bool kWindowPerGroup = MCINV_WINDOW_PER_GROUP;

std::vector<int> schedule_slots(int64_t n, const std::vector<int4> &rec, const std::vector<int> &ent_col, int R,
                                int L, int ecap, int similar) {
    // row i -> level-order index o; lower neighbours (the first nlow entries) and the
    // reverse edges (upper neighbours)
    // (records with x < 0 are not rows -- the trace items of v5 -- and nothing waits on them)
    std::vector<int> ord_of(n);
    for (int64_t o = 0; o < n; ++o)
        if (rec[o].x >= 0) ord_of[rec[o].x] = (int)o;
    std::vector<int> up_cnt(n + 1, 0);
    for (int64_t o = 0; o < n; ++o)
        for (int e = 0; e < (int)((unsigned)rec[o].z >> 16); ++e) up_cnt[ord_of[ent_col[rec[o].y + e]] + 1]++;
    for (int64_t o = 0; o < n; ++o) up_cnt[o + 1] += up_cnt[o];
    std::vector<int> up(up_cnt[n]), fill(up_cnt.begin(), up_cnt.end() - 1);
    for (int64_t o = 0; o < n; ++o)
        for (int e = 0; e < (int)((unsigned)rec[o].z >> 16); ++e) up[fill[ord_of[ent_col[rec[o].y + e]]]++] = (int)o;
    // height = longest path to a sink (level order is topological: reverse sweep)
    std::vector<int> height(n, 0);
    for (int64_t o = n - 1; o >= 0; --o)
        for (int q = up_cnt[o]; q < up_cnt[o + 1]; ++q) height[o] = std::max(height[o], height[up[q]] + 1);
    // list scheduling
    std::vector<int> pending(n), ready_at(n, 0), group_of(n, -1);
    for (int64_t o = 0; o < n; ++o) pending[o] = (int)((unsigned)rec[o].z >> 16);
    // candidates keyed by (ready group, -height): rows whose lower neighbours are all placed
    using Key = std::tuple<int, int, int>;  // (ready group, -height, o)
    std::priority_queue<Key, std::vector<Key>, std::greater<Key>> waiting;  // by ready group
    std::priority_queue<std::pair<int, int>> ready;                          // (height, -o) among ready
    for (int64_t o = 0; o < n; ++o)
        if (pending[o] == 0) waiting.push(Key(0, -height[o], (int)o));
    std::vector<int> slots;
    slots.reserve(n + n / 4);
    int64_t placed = 0;
    for (int G = 0; placed < n; ++G) {
        while (!waiting.empty() && std::get<0>(waiting.top()) <= G) {
            ready.push({-std::get<1>(waiting.top()), -std::get<2>(waiting.top())});
            waiting.pop();
        }
        int taken = 0, ents = 0;
        std::vector<int> now;
        // the similarity window is drawn once per group (the `similar` highest ready rows after
        // the group's first row) and the group's other rows are taken from it, each the first
        // of the least distance to the first row: the same choice rule as one window per row,
        // ~R times fewer heap operations (host planning is inside the e2e step)
        std::vector<std::pair<int, int>> win;
        bool win_drawn = false;
        while (taken < R) {
            int o;
            if (similar > 0 && taken > 0 && kWindowPerGroup) {
                if (!win_drawn) {
                    while (!ready.empty() && (int)win.size() < similar) {
                        win.push_back(ready.top());
                        ready.pop();
                    }
                    win_drawn = true;
                }
                if (win.empty()) break;
                const int o0 = now[0];
                auto dist = [&](int x) {
                    return std::abs((rec[x].z & 0xffff) - (rec[o0].z & 0xffff)) +
                           std::abs((int)((unsigned)rec[x].z >> 16) - (int)((unsigned)rec[o0].z >> 16));
                };
                int best = 0, bestd = 1 << 30;
                for (int q = 0; q < (int)win.size(); ++q) {
                    const int d = dist(-win[q].second);
                    if (d < bestd) {
                        bestd = d;
                        best = q;
                        if (d == 0) break;
                    }
                }
                o = -win[best].second;
                if (ecap > 0 && ents + (rec[o].z & 0xffff) > ecap) break;
                win.erase(win.begin() + best);
            } else if (!ready.empty() && similar > 0 && taken > 0) {
                // among the next `similar` ready rows (by height) take the one whose entry and
                // lower-neighbour counts are closest to the group's first row: the R rows of a
                // warp item then run their waits and gather loops with less divergence
                // (config 2 2.36 -> 2.43e10 with a window of 32; config 3 unchanged)
                const int o0 = now[0];
                auto dist = [&](int x) {
                    return std::abs((rec[x].z & 0xffff) - (rec[o0].z & 0xffff)) +
                           std::abs((int)((unsigned)rec[x].z >> 16) - (int)((unsigned)rec[o0].z >> 16));
                };
                // candidates in height order; stop at the first exact match (the same choice as
                // scanning the whole window: the first of the minimal distance)
                std::vector<std::pair<int, int>> cand;
                int best = 0, bestd = 1 << 30;
                while (!ready.empty() && (int)cand.size() < similar) {
                    cand.push_back(ready.top());
                    ready.pop();
                    const int d = dist(-cand.back().second);
                    if (d < bestd) {
                        bestd = d;
                        best = (int)cand.size() - 1;
                        if (d == 0) break;
                    }
                }
                o = -cand[best].second;
                for (int q = 0; q < (int)cand.size(); ++q)
                    if (q != best) ready.push(cand[q]);
                if (ecap > 0 && ents + (rec[o].z & 0xffff) > ecap) {
                    ready.push(cand[best]);
                    break;
                }
            } else if (!ready.empty()) {
                o = -ready.top().second;
                if (ecap > 0 && taken > 0 && ents + (rec[o].z & 0xffff) > ecap) break;  // block size cap
                ready.pop();
            } else if (!waiting.empty() && taken == 0) {
                o = std::get<2>(waiting.top());  // nothing ready: earliest-ready row (it will wait)
                waiting.pop();
            } else {
                break;
            }
            now.push_back(o);
            ents += rec[o].z & 0xffff;
            ++taken;
        }
        for (const auto &x : win) ready.push(x);
        for (int o : now) {
            group_of[o] = G;
            slots.push_back(o);
            ++placed;
        }
        while ((int)slots.size() % R) slots.push_back(-1);
        // rows of this group release their upper neighbours (not into this group: they
        // become candidates from group G + L, or G + 1 at the least)
        for (int o : now)
            for (int q = up_cnt[o]; q < up_cnt[o + 1]; ++q) {
                const int u = up[q];
                ready_at[u] = std::max(ready_at[u], G + std::max(L, 1));
                if (--pending[u] == 0) waiting.push(Key(ready_at[u], -height[u], u));
            }
    }
    return slots;
}

}  // namespace mcinv
