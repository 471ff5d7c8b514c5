// plan.cu -- host planner for the step-scheduled sweep kernel; see plan.h.
#include <algorithm>
#include <cstring>
#include <queue>

#include "plan.h"

namespace mcinv {

namespace {

struct Ent {
    int j;
    std::complex<double> a, b;
};

// accumulation record of one partner row j (lower than the row i)
struct Part {
    int j;
    int pzi = -1, pzo = -1;
    std::complex<double> qr = 0.0, qc = 0.0;
    bool has_qr = false, has_qc = false;
};

struct RowAcc {
    int dslot = -1, pslot = -1;
    std::complex<double> qself = 0.0;
    std::vector<Part> parts;
};

struct Seg {
    int row;
    int first_entry, count;  // entries [first_entry, first_entry + count) of the row list
    bool first, last;
};

void put_scalar(unsigned char *p, std::complex<double> v, bool cplx) {
    double re = v.real(), im = v.imag();
    std::memcpy(p, &re, 8);
    if (cplx) std::memcpy(p + 8, &im, 8);
}

Part &part_for(RowAcc &ra, int j, int role) {
    // role 0 pzi, 1 pzo, 2 qr, 3 qc: first record of j with that role free
    for (Part &p : ra.parts) {
        if (p.j != j) continue;
        if ((role == 0 && p.pzi < 0) || (role == 1 && p.pzo < 0) || (role == 2 && !p.has_qr) ||
            (role == 3 && !p.has_qc))
            return p;
    }
    ra.parts.push_back(Part{j});
    return ra.parts.back();
}

}  // namespace

std::string build_plan(const PlanInput &in, int R, int C, HostPlan &out) {
    const int64_t n = in.n;
    const bool cplx = in.cplx;
    const int esz = cplx ? 16 : 8;
    const int zwsz = 2 * esz;
    const int BLK = 32 * zwsz;
    const int NGBUF = ngbuf(esz), NRING = nring(esz);
    const int GB_OFF = NRING * BLK;
    const int ZERO_OFF = GB_OFF + NGBUF * KCAP * BLK;
    if (R * C != 32) return "R * C must be 32";

    // ---- accumulation requests per row, keyed by r = max(i, j) (Eq. 1/C, Eq. tr)
    std::vector<RowAcc> acc(n);
    if (in.want_diag)
        for (int64_t i = 0; i < n; ++i) acc[i].dslot = (int)i;
    if (in.want_pattern) {
        const auto &pr = *in.p_row, &pc = *in.p_col;
        for (size_t p = 0; p < pr.size(); ++p) {
            const int r = pr[p], c = pc[p];
            if (r == c) {
                if (acc[r].pslot >= 0) return "duplicate diagonal pattern element";
                acc[r].pslot = (int)p;
            } else if (r > c) {
                part_for(acc[r], c, 0).pzi = (int)p;   // z_r conj(w_c) at row r
            } else {
                part_for(acc[c], r, 1).pzo = (int)p;   // z_r conj(w_c) at row c
            }
        }
    }
    if (in.want_trace) {
        const auto &qp = *in.q_ptr;
        const auto &qc = *in.q_col;
        const auto &qv = *in.q_val;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t e = qp[i]; e < qp[i + 1]; ++e) {
                const int j = qc[e];
                if (j == i) {
                    acc[i].qself += qv[e];
                } else if (j < i) {
                    Part &p = part_for(acc[i], j, 2);  // conj(w_i) Q_ij z_j at row i
                    p.qr = qv[e];
                    p.has_qr = true;
                } else {
                    Part &p = part_for(acc[j], (int)i, 3);  // conj(w_i) Q_ij z_j at row j
                    p.qc = qv[e];
                    p.has_qc = true;
                }
            }
    }

    // ---- entry lists (union of row i and column i of C, H1); partners must be
    // operands of the last two segments: append zero-coefficient duplicates
    std::vector<std::vector<Ent>> ent(n);
    int64_t dups = 0;
    for (int64_t i = 0; i < n; ++i) {
        auto &L = ent[i];
        const auto &up = *in.u_ptr;
        for (int e = up[i]; e < up[i + 1]; ++e) L.push_back(Ent{(*in.u_col)[e], (*in.u_a)[e], (*in.u_b)[e]});
        std::vector<int> partners;
        for (const Part &p : acc[i].parts) partners.push_back(p.j);
        std::sort(partners.begin(), partners.end());
        partners.erase(std::unique(partners.begin(), partners.end()), partners.end());
        if ((int)partners.size() > MAXPART)
            return "row " + std::to_string(i) + " has more than " + std::to_string(MAXPART) + " accumulation partners";
        for (int iter = 0;; ++iter) {
            if (iter > 4 * MAXPART) return "internal: partner placement did not converge";
            const int len = (int)L.size();
            const int nseg = len == 0 ? 1 : (len + KCAP - 1) / KCAP;
            const int W = nseg >= 2 ? (nseg - 2) * KCAP : 0;
            int missing = -1;
            for (int pj : partners) {
                bool ok = false;
                for (int k = W; k < len && !ok; ++k) ok = L[k].j == pj;
                if (!ok) {
                    missing = pj;
                    break;
                }
            }
            if (missing < 0) break;
            L.push_back(Ent{missing, 0.0, 0.0});
            ++dups;
        }
    }

    // ---- dependency graph: every operand relation i~j orients min -> max
    std::vector<std::vector<int>> succ(n);
    std::vector<int> npred(n, 0);
    {
        std::vector<std::pair<int, int>> edges;
        for (int64_t i = 0; i < n; ++i)
            for (const Ent &e : ent[i])
                if (e.j != i) edges.emplace_back(std::min<int>(i, e.j), std::max<int>(i, e.j));
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
        for (auto &e : edges) {
            succ[e.first].push_back(e.second);
            npred[e.second]++;
        }
    }

    // ---- list scheduling: steps of R slots, segments of a row consecutive in one slot
    std::vector<std::vector<Seg>> steps;  // steps[t][r]
    std::vector<int> fin_step(n, -1), fin_slot(n, -1);
    {
        std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
        for (int64_t i = 0; i < n; ++i)
            if (npred[i] == 0) ready.push((int)i);
        struct Active {
            int row = -1, next_seg = 0, nseg = 0;
        };
        std::vector<Active> act(R);
        int64_t done = 0;
        std::vector<int> newly;
        while (done < n) {
            std::vector<Seg> st(R, Seg{-1, 0, 0, false, false});
            for (int r = 0; r < R; ++r) {
                if (act[r].row < 0 && !ready.empty()) {
                    const int i = ready.top();
                    ready.pop();
                    const int len = (int)ent[i].size();
                    act[r].row = i;
                    act[r].next_seg = 0;
                    act[r].nseg = len == 0 ? 1 : (len + KCAP - 1) / KCAP;
                }
                if (act[r].row >= 0) {
                    const int i = act[r].row;
                    const int s = act[r].next_seg;
                    const int len = (int)ent[i].size();
                    Seg sg;
                    sg.row = i;
                    sg.first_entry = s * KCAP;
                    sg.count = std::max(0, std::min(KCAP, len - s * KCAP));
                    sg.first = s == 0;
                    sg.last = s == act[r].nseg - 1;
                    st[r] = sg;
                }
            }
            const int t = (int)steps.size();
            newly.clear();
            bool any = false;
            for (int r = 0; r < R; ++r) {
                if (act[r].row < 0) continue;
                any = true;
                if (st[r].last) {
                    const int i = act[r].row;
                    fin_step[i] = t;
                    fin_slot[i] = r;
                    ++done;
                    for (int s : succ[i])
                        if (--npred[s] == 0) newly.push_back(s);
                    act[r].row = -1;
                } else {
                    act[r].next_seg++;
                }
            }
            if (!any) return "scheduler stalled (cyclic dependency?)";
            steps.push_back(st);
            for (int s : newly) ready.push(s);
        }
    }
    while (steps.size() % NRING) steps.push_back(std::vector<Seg>(R, Seg{-1, 0, 0, false, false}));
    const int S = (int)steps.size();

    // smem value offset of operand k of the segment in slot r at step t
    auto value_off = [&](int t, int r, int k, int *col, bool *is_near) -> int {
        const Seg &sg = steps[t][r];
        const int i = sg.row;
        const int j = ent[i][sg.first_entry + k].j;
        const int tj = fin_step[j];
        const int d = (j < i) ? t - tj : S + t - tj;
        if (d < 1 || d > S) return -1;
        if (d <= PDIST) {
            *col = -1;
            *is_near = true;
            return ((((t - d) % NRING) + NRING) % NRING) * BLK + fin_slot[j] * C * zwsz;
        }
        *col = j;
        *is_near = false;
        return GB_OFF + ((t % NGBUF) * KCAP + k) * BLK + r * C * zwsz;
    };

    // ---- tiles
    out = HostPlan();
    out.R = R;
    out.C = C;
    out.steps = S;
    out.tile_off.assign(S + 1, 0);
    out.dup_entries = dups;
    std::vector<TileLayout> lay(S);
    for (int t = 0; t < S; ++t) {
        int K = 0, P = 0;
        for (int r = 0; r < R; ++r) {
            const Seg &sg = steps[t][r];
            if (sg.row < 0) continue;
            K = std::max(K, sg.count);
            if (sg.last) P = std::max(P, (int)acc[sg.row].parts.size());
        }
        lay[t] = TileLayout{K, P, R, esz};
        out.tile_off[t + 1] = out.tile_off[t] + lay[t].total();
        out.tile_slot_bytes = std::max(out.tile_slot_bytes, lay[t].total());
        out.max_parts = std::max(out.max_parts, P);
    }
    out.tiles.assign(out.tile_off[S], 0);
    for (int t = 0; t < S; ++t) {
        const TileLayout &L = lay[t];
        unsigned char *T = out.tiles.data() + out.tile_off[t];
        const int nt = (t + 8) % S;  // the producer issues tile t+8 while gathering step t
        int hdr[4] = {L.K, L.P, (int)(out.tile_off[nt + 1] - out.tile_off[nt]), in.want_trace ? 1 : 0};
        int64_t noff = out.tile_off[nt];
        std::memcpy(T, hdr, 16);
        std::memcpy(T + 16, &noff, 8);
        int *rows = (int *)(T + L.rows());
        for (int r = 0; r < R; ++r) {
            const Seg &sg = steps[t][r];
            rows[r] = sg.row;
            rows[R + r] = sg.row < 0 ? 0 : (4 | (sg.first ? 1 : 0) | (sg.last ? 2 : 0));
            rows[2 * R + r] = (sg.row >= 0 && sg.last) ? acc[sg.row].dslot : -1;
            rows[3 * R + r] = (sg.row >= 0 && sg.last) ? acc[sg.row].pslot : -1;
            if (sg.row >= 0 && sg.last) {
                put_scalar(T + L.dsq() + r * esz, (*in.delta)[sg.row], cplx);
                put_scalar(T + L.dsq() + (R + r) * esz, (*in.sigma)[sg.row], cplx);
                put_scalar(T + L.dsq() + (2 * R + r) * esz, acc[sg.row].qself, cplx);
            }
        }
        for (int k = 0; k < L.K; ++k)
            for (int r = 0; r < R; ++r) {
                int *meta = (int *)(T + L.meta() + 8 * (k * R + r));
                unsigned char *cf = T + L.coef() + 2 * esz * (k * R + r);
                const Seg &sg = steps[t][r];
                if (sg.row < 0 || k >= sg.count) {
                    meta[0] = ZERO_OFF;
                    meta[1] = -1;
                    continue;
                }
                int col = -1;
                bool nr = false;
                const int off = value_off(t, r, k, &col, &nr);
                if (off < 0) return "internal: bad operand distance";
                meta[0] = off;
                meta[1] = col;
                out.entries++;
                out.near_entries += nr;
                const Ent &e = ent[sg.row][sg.first_entry + k];
                put_scalar(cf, e.a, cplx);
                put_scalar(cf + esz, e.b, cplx);
            }
        for (int r = 0; r < R; ++r)
            if (steps[t][r].row >= 0) out.segments++;
        for (int q = 0; q < L.P; ++q)
            for (int r = 0; r < R; ++r) {
                unsigned char *pr = T + L.part() + L.part_bytes() * (q * R + r);
                int w4[4] = {ZERO_OFF, -1, -1, 0};
                std::complex<double> qr = 0.0, qc = 0.0;
                const Seg &sg = steps[t][r];
                if (sg.row >= 0 && sg.last && q < (int)acc[sg.row].parts.size()) {
                    const int i = sg.row;
                    const Part &pt = acc[i].parts[q];
                    // operand of the final segment (step t) or of the previous one (t-1)
                    int voff = -1;
                    for (int k = 0; k < sg.count && voff < 0; ++k)
                        if (ent[i][sg.first_entry + k].j == pt.j) {
                            int col;
                            bool nr;
                            voff = value_off(t, r, k, &col, &nr);
                        }
                    if (voff < 0 && !sg.first) {
                        const Seg &pv = steps[t - 1][r];
                        if (pv.row != i) return "internal: previous segment not in t-1";
                        for (int k = 0; k < pv.count && voff < 0; ++k)
                            if (ent[i][pv.first_entry + k].j == pt.j) {
                                int col;
                                bool nr;
                                voff = value_off(t - 1, r, k, &col, &nr);
                            }
                    }
                    if (voff < 0) return "internal: partner operand not found";
                    w4[0] = voff;
                    w4[1] = pt.pzi;
                    w4[2] = pt.pzo;
                    qr = pt.qr;
                    qc = pt.qc;
                    out.parts++;
                }
                std::memcpy(pr, w4, 16);
                put_scalar(pr + 16, qr, cplx);
                put_scalar(pr + 16 + esz, qc, cplx);
            }
    }
    return "";
}

}  // namespace mcinv
