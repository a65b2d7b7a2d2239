// Host-side setup of the B200 Biot solver: stabilised P1-P1 assembly into the
// node-block layouts the sweep kernels read.  Internal header (not ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/biot_pit.h"

namespace biot {

constexpr int kMaxSlots = 32;

enum Path : int { PATH_BDIA = 1, PATH_ELL = 2 };

// Per-node neighbour blocks.  For node i and slot s (column node j):
//   blk[((i*S)+s)*W + c*NC + cc]  = AA[(i,c),(j,cc)]          (c, cc < NC)
//   blk[((i*S)+s)*W + NC*NC]      = A'[(i,p),(j,p)] = -H_ij    (pressure of A')
// where W = NC*NC + 1 rounded up to even (16-B aligned blocks); A'[(i,p),(j,u_e)] equals AA[(i,p),(j,u_e)] (both B^T) and is
// read from the AA block.  BDIA: j = i + offsets[s]; ELL: j = cols[i*S+s].
struct HostOperator {
    int d = 0, nc = 0;
    int64_t n_nodes = 0;
    int n_slots = 0;
    int path = 0;
    int64_t max_abs_offset = 0;
    std::vector<int64_t> offsets;   // BDIA, offsets[0] == 0 (self)
    std::vector<int32_t> cols;      // ELL, self in slot 0, padding repeats self with zero blocks
    std::vector<double> blk;        // n_nodes * S * block_width(nc)
    std::vector<double> load;       // f, n_nodes * nc
    std::vector<double> dinv;       // n_nodes * nc; 1/diag(A), 1/diag(S~p) on free DoFs, else 0
    std::vector<uint8_t> fixed;     // n_nodes * nc
    // further load terms (R24): sources (kind 0, coefficient row `src` of bc.source_coef) and
    // the Dirichlet lifting (kind 1: -AA_{free,D} x_D with c_n; kind 2: A'_{free,D} x_D with
    // c_{n-1}); free rows only, all-zero terms dropped
    struct LoadTerm {
        std::vector<double> f;      // n_nodes * nc
        int kind = 0, src = 0;
    };
    std::vector<LoadTerm> extra;
    double beta = 0.0;
    int64_t nnz_AA = 0, nnz_AP = 0; // nonzeros (free rows/cols, explicit zeros dropped)
};

// Returns "" on success, else an error message.  BDIA is used when the mesh has at
// most 7 (2D) / 15 (3D) distinct column-row offsets, otherwise ELL.
std::string assemble(const biot_mesh &mesh, const biot_material &mat, const biot_bc &bc,
                     double dt, HostOperator &op);

int block_width(int nc);

}  // namespace biot
