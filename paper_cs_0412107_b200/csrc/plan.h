// plan.h -- host planner for the v2 sweep kernel (sweep2.cu).
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
// from the step that produced its value: d <= P: read from the in-smem ring of
// recent results; d > P: gathered from HBM P steps ahead with cp.async.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace mcinv {

constexpr int KCAP = 8;     // entries per row segment
constexpr int PDIST = 7;    // gather prefetch distance (steps)
constexpr int NRING = 8;    // ring / gbuf slots (PDIST + 1)
constexpr int NTILE = 16;   // record tile slots (tile for step T+15 issued at step T)

// item opcodes (accumulation at the final segment of a row; Eq. 1/C, Eq. tr)
enum ItemOp : int {
    IT_NOP = 0,
    IT_DIAG = 1,       // diag slot  += z_i conj(w_i)
    IT_PAT_ZI = 2,     // pat slot   += z_i conj(w_k)    (partner = entry k)
    IT_PAT_ZO = 3,     // pat slot   += z_k conj(w_i)
    IT_PAT_SELF = 4,   // pat slot   += z_i conj(w_i)
    IT_QROW = 5,       // qz += q z_k
    IT_QROW_SELF = 6,  // qz += q z_i
    IT_QCOL = 7        // qw += q conj(w_k)
};

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
    int steps = 0;              // steps per sweep (padded to a multiple of NRING)
    int tile_slot_bytes = 0;    // max tile bytes (16-aligned)
    int max_items = 0;
    std::vector<unsigned char> tiles;   // concatenated tiles
    std::vector<int64_t> tile_off;      // steps + 1
    // statistics
    int64_t segments = 0, entries = 0, near_entries = 0, items = 0, dup_entries = 0;
};

// Build the plan; returns "" on success or an error message.
std::string build_plan(const PlanInput &in, int R, int C, HostPlan &out);

// Tile layout, shared with the kernel. All section offsets are 16-aligned.
struct TileLayout {
    int K, I, R, esz;  // esz = sizeof(scalar) (8 or 16)
    __host__ __device__ int hdr() const { return 0; }                       // 32 B
    __host__ __device__ int rows() const { return 32; }                     // int rows[R], int flags[R]
    __host__ __device__ int dsig() const { return 32 + r16(8 * R); }        // S delta[R], S sigma[R]
    __host__ __device__ int meta() const { return dsig() + r16(2 * R * esz); }  // int2 meta[K][R]
    __host__ __device__ int coef() const { return meta() + r16(8 * K * R); }    // S a,b [K][R]
    __host__ __device__ int items() const { return coef() + r16(2 * esz * K * R); }  // item [I][R]
    // item: {int code (op | 8 * has_voff), int slot, int partner_row, int voff, S q, pad}
    __host__ __device__ int item_bytes() const { return 32; }
    __host__ __device__ int total() const { return items() + r16(item_bytes() * I * R); }
    __host__ __device__ static int r16(int x) { return (x + 15) & ~15; }
};

}  // namespace mcinv
