// plan.h -- host planner for the step-scheduled sweep kernel (sweep2.cu).
//
// The sweep of Eq. (4)/(5) visits rows in ascending order;
// row i reads new values of its lower neighbours (j < i) and old values of
// its upper neighbours (j > i). Those are the ONLY ordering constraints: any
// execution order in which every row runs after its lower neighbours and
// before its upper neighbours reads exactly the same operands and produces
// bit-identical z, w. The planner builds such an order as a sequence of
// STEPS of up to R rows with no edges among them (list scheduling, lowest row
// first), so one warp can update R rows of C chains at once (lanes = C x R).
// DESIGN.md "Step schedule" has the argument; parity tests check it.
//
// Rows longer than KCAP entries are split into segments in consecutive steps
// of the same row slot. Each entry is classified by the distance d (in steps)
// from the step that produced its value: d <= PDIST: read from the in-smem
// ring of recent results; d > PDIST: gathered from HBM 8 steps ahead with
// cp.async. Accumulation partners of a row (Eq. 1/C pattern elements, Eq. tr
// Q terms) are operands of its last two segments (zero-coefficient duplicates
// are appended when needed), so the accumulator warp finds them in smem.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace mcinv {

constexpr int KCAP = 8;     // entries per row segment
constexpr int PDIST = 7;    // near/far threshold (steps): far operands are >= 8 steps old
constexpr int NTILE = 16;   // record tile slots
constexpr int MAXPART = 2 * KCAP;  // accumulation partners per row
// Gather-buffer step slots (16 real, 8 complex: shared-memory budget) and
// result-ring step slots (2 x gather slots; steps per sweep are padded to a
// multiple). Deeper buffers let the accumulation warps lag the update warp.
__host__ __device__ constexpr int ngbuf(int esz) { return esz == 8 ? 16 : 8; }
__host__ __device__ constexpr int nring(int esz) { return 2 * ngbuf(esz); }

struct PlanInput {
    int64_t n = 0;
    bool cplx = false;
    // union lists (H1): entry (j, a = c_ij, b = conj(c_ji)), j ascending, j != i
    const std::vector<int> *u_ptr = nullptr, *u_col = nullptr;
    const std::vector<std::complex<double>> *u_a = nullptr, *u_b = nullptr;
    const std::vector<std::complex<double>> *delta = nullptr, *sigma = nullptr;
    // pattern (p -> (row, col)); Q CSR rows (canonical)
    bool want_diag = false, want_pattern = false, want_trace = false;
    const std::vector<int> *p_row = nullptr, *p_col = nullptr;
    const std::vector<int64_t> *q_ptr = nullptr;
    const std::vector<int> *q_col = nullptr;
    const std::vector<std::complex<double>> *q_val = nullptr;
};

struct HostPlan {
    int R = 1, C = 32;
    int steps = 0;              // steps per sweep (padded to a multiple of nring)
    int tile_slot_bytes = 0;    // max tile bytes (16-aligned)
    int max_parts = 0;          // max partner records per row slot in a step
    std::vector<unsigned char> tiles;   // concatenated tiles
    std::vector<int64_t> tile_off;      // steps + 1
    // statistics
    int64_t segments = 0, entries = 0, near_entries = 0, parts = 0, dup_entries = 0;
};

// Build the plan; returns "" on success or an error message.
std::string build_plan(const PlanInput &in, int R, int C, HostPlan &out);

// Tile layout, shared with the kernel; every section offset is 16-aligned.
//   hdr   32 B : int K, int P, int next_bytes, int has_q; int64 next_off; pad
//   rows  16R  : int row[R], int flags[R] (1 first seg, 2 last seg, 4 busy),
//                int dslot[R] (diag slot or -1), int pslot[R] (pattern (i,i) slot or -1)
//   dsq   3R S : delta[R], sigma[R], qself[R] (Q_ii)
//   meta  K R  : int2 {smem value offset, gather column or -1}
//   coef  K R  : S a (Eq. 4 coefficient), S b (Eq. 5 coefficient)
//   part  P R  : {int voff, int pzi, int pzo, int pad, S qr, S qc}
//                pzi: pattern slot of z_i conj(w_j); pzo: slot of z_j conj(w_i)
//                qr = Q_ij (j < i), qc = Q_ji (j < i) for the trace w^dagger Q z
struct TileLayout {
    int K, P, R, esz;
    __host__ __device__ int rows() const { return 32; }
    __host__ __device__ int dsq() const { return 32 + r16(16 * R); }
    __host__ __device__ int meta() const { return dsq() + r16(3 * R * esz); }
    __host__ __device__ int coef() const { return meta() + r16(8 * K * R); }
    __host__ __device__ int part() const { return coef() + r16(2 * esz * K * R); }
    __host__ __device__ int part_bytes() const { return 16 + 2 * esz; }
    __host__ __device__ int total() const { return part() + r16(part_bytes() * P * R); }
    __host__ __device__ static int r16(int x) { return (x + 15) & ~15; }
};

// Shared-memory value area of the kernel (bytes): ring | gather buffer | zero block.
template <int ESZ> struct ValueArea {
    static constexpr int BLK = 32 * 2 * ESZ;  // one step slot: R rows x C chains x (z, w)
    static constexpr int NGB = ngbuf(ESZ), NRG = nring(ESZ);
    static constexpr int RING = 0;
    static constexpr int GBUF = NRG * BLK;
    static constexpr int ZERO = GBUF + NGB * KCAP * BLK;
    static constexpr int BYTES = ZERO + BLK;
};

}  // namespace mcinv
