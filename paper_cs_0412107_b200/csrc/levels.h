// levels.h -- host planner of the level-scheduled sweep kernel (sweep3.cu).
//
// The sweep of Eq. (4)/(5) visits rows in ascending order:
// row i reads the NEW values of its lower neighbours (j < i, coupled to i by
// c_ij or c_ji) and the OLD values of its upper neighbours (j > i). These are
// the only ordering constraints, so any order in which every row runs after
// its lower neighbours and before its upper neighbours reads exactly the
// operands of the sequential sweep and gives bit-identical z and w. The
// planner groups rows into LEVELS: lev(i) = 1 + max{lev(j) : j < i, j a
// neighbour of i} (0 if none). Rows of one level are mutually independent, so
// a CTA updates all rows of a level for its chains at once and synchronises
// only between levels.
//
// Accumulation (Eq. 1/C and Eq. tr) in sampling sweeps:
//  - diag z_i conj(w_i) and the pattern pairs of row i with a LOWER neighbour
//    j (both values final) are fused into row i's update;
//  - every other requested pair (custom pattern elements, all trace terms
//    w_i^* Q_ij z_j) is a DEFERRED item of phase max(lev(i), lev(j)) + 1: both
//    values are final for the sweep and not yet overwritten by the next one.
//    Phase D (one past the last level) holds only deferred items.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>

namespace mcinv {

struct LevelInput {
    int64_t n = 0;
    // union lists (H1): entry (j, a = c_ij, b = conj(c_ji)), j ascending, j != i
    const std::vector<int> *u_ptr = nullptr, *u_col = nullptr;
    const std::vector<std::complex<double>> *u_a = nullptr, *u_b = nullptr;
    const std::vector<std::complex<double>> *delta = nullptr, *sigma = nullptr;
    bool want_pattern = false, want_trace = false;
    const std::vector<int> *p_row = nullptr, *p_col = nullptr;  // pattern element p = (p_row[p], p_col[p])
    const std::vector<int64_t> *q_ptr = nullptr;                // Q (canonical CSR)
    const std::vector<int> *q_col = nullptr;
    const std::vector<std::complex<double>> *q_val = nullptr;
};

struct LevelPlan {
    int D = 0;                       // update levels; phases 0..D
    std::vector<int> level;          // lev(i), for tests
    std::vector<int> ph_row;         // [D+2] level-order row range of phase p (phase D: empty)
    std::vector<int> ord_row;        // [n] rows in level order (decreasing entry count within a level)
    std::vector<int> ord_eptr;       // [n+1] entry range of level-order row o
    std::vector<int> ent_col;        // [nnz_u] union entries in level order
    std::vector<std::complex<double>> ent_a, ent_b;
    std::vector<int> ent_pz;         // [2 nnz_u] pattern slots {z_i w_j^*, z_j w_i^*} for j < i, else -1
    std::vector<std::complex<double>> ord_dl, ord_sg;  // [n] delta_i, sigma_i in level order
    std::vector<int> ord_pself;      // [n] pattern slot of (i, i) or -1
    // deferred trace items: one per Q row i, phase max(lev(i), lev(j in row)) + 1
    std::vector<int> ph_tq;          // [D+2]
    std::vector<int> tq_row, tq_eptr, tq_col;  // tq_eptr [items+1]
    std::vector<std::complex<double>> tq_val;
    // deferred pattern pairs (i, j, slot), phase max(lev(i), lev(j)) + 1
    std::vector<int> ph_pp;          // [D+2]
    std::vector<int> pp_i, pp_j, pp_slot;
    int max_rows = 0;                // max rows + deferred items of one phase
    int64_t fused_pairs = 0, deferred_pairs = 0;
};

// Build the plan; returns "" on success or an error message.
std::string build_levels(const LevelInput &in, LevelPlan &out);

// v4 slot schedule: a topological order of the
// lower-neighbour DAG cut into warp groups of R rows, where every row is placed
// at least L groups after the groups of all its lower neighbours when possible
// (L ~ the groups a CTA has in flight, so the counters it waits for are
// usually published already), longest remaining path first; a group that
// cannot be filled with such rows is completed with the rows that become ready
// earliest, and padded (-1) only when no row is left. Input: the level-order
// records (i, entry begin, count | lower << 16) and entry columns of the plan.
// Output: slot -> level-order index (or -1 for padding); size a multiple of R.
// n counts the records; records with x < 0 are items that wait on their entries like
// rows but that nothing waits on (v5's trace items).
// ecap > 0: a group takes no further row once its entries would exceed ecap (a
// single row may exceed it alone): bounds the group blocks staged by v5.
// similar > 0: a group's rows after the first are chosen among the next `similar`
// ready rows (by height) as the first whose entry and lower-neighbour counts are
// closest to the first row's (less divergence among a warp's rows).
std::vector<int> schedule_slots(int64_t n, const std::vector<int4> &rec, const std::vector<int> &ent_col, int R,
                                int L, int ecap = 0, int similar = 0);

}  // namespace mcinv
