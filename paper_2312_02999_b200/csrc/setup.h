// Host-side one-time setup (untimed): validation, element matrices,
// the scalar PD matrix L (H = L (x) I3, Eq. 2), Dirichlet elimination,
// geometric nested-dissection ordering, supernodal symbolic + numeric Cholesky of L_FF,
// transpose incidence, surface edges and W.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pdipc {

struct HostMesh {
    int n = 0, T = 0, nf = 0;
    std::vector<int32_t> tets;          // [T][4]
    std::vector<double> rest;           // [n][3]
    std::vector<double> B;              // [T][9] D_m^{-1} row-major
    std::vector<double> w;              // [T]
    std::vector<uint8_t> is_fixed;      // [n]
    // factor ordering: q = factor position of a free vertex
    std::vector<int32_t> q2v;           // [nf]
    std::vector<int32_t> v2q;           // [n], -1 for fixed
    // transpose incidence in factor order: for q, (tet << 2 | corner) list
    std::vector<int32_t> inc_ptr;       // [nf+1]
    std::vector<int32_t> inc;           // [4T restricted to free]
    // surface
    int Ns = 0, Nt = 0, Ne = 0;
    std::vector<int32_t> tris;          // [Nt][3]
    std::vector<int32_t> edges;         // [Ne][2], sorted unique
    std::vector<int32_t> W_ptr, W_col;  // CSR of W (rows = surface verts), exact zeros dropped
    std::vector<double> W_val;
    std::vector<int32_t> WT_ptr, WT_row;  // CSR of W^T over factor positions q (free only)
    std::vector<double> WT_val;
    double mean_edge = 0.0;             // rest mean surface edge length
};

struct HostFactor {
    int nf = 0, nsn = 0;
    std::vector<int32_t> sn_c0;        // [nsn+1] first column of each supernode
    std::vector<int32_t> sn_rowptr;    // [nsn+1] into sn_rows
    std::vector<int32_t> sn_rows;      // row indices (factor positions); first w_s are c0..c1-1
    std::vector<int64_t> sn_valptr;    // [nsn+1] into vals (column-major, ld = nrows)
    std::vector<double> vals;
    std::vector<int32_t> sn_parent;    // [nsn], -1 root
    std::vector<int32_t> sn_fd;        // [nsn] first column of the subtree (postorder)
    std::vector<int32_t> col2sn;       // [nf]
    // forward-solve update segments: for target s, list of (d, klo, khi): rows R_d[klo..khi)
    // lie in s's columns
    std::vector<int32_t> seg_ptr, seg_d, seg_klo, seg_khi;
    std::vector<int32_t> sn_nchild;    // [nsn]
    // right-looking update rows: supernode d writes U rows uoff[d] .. uoff[d+1)-1, one per
    // off-diagonal row of d; factor row r gathers the U rows listed in rc_idx[rc_ptr[r]..]
    std::vector<int32_t> uoff;         // [nsn+1]
    std::vector<int32_t> urow_sn;      // [uoff[nsn]] owner supernode of each U row
    std::vector<int32_t> rc_ptr, rc_idx;
    std::vector<int32_t> urel;         // [nU] position of a U row's matrix row in the parent's R
    std::vector<int32_t> ch_ptr, ch;   // children of each supernode (increasing order)
    // inverse of each diagonal block (lower triangular, row-major w x w)
    std::vector<int64_t> dinv_ptr;     // [nsn+1]
    std::vector<double> dinv;
    // per supernode [L_ss^{-1}; L_off L_ss^{-1}], column-major ld nr, offsets sn_valptr (as vals)
    std::vector<double> Q;
    int max_width = 0, max_rows = 0, depth = 0;
    int64_t nnzL = 0;
};

// Returns 0 or a negative PD_IPC_E_* code with `err` filled.
int build_host_mesh(int n, int T, const int32_t *tets, int nfix, const int32_t *fixed,
                    const double *rest, int Ns, int Nt, const int32_t *tris,
                    const int32_t *embed_tet, const double *embed_w, HostMesh &m,
                    std::string &err);
int factorize(HostMesh &m, HostFactor &f, std::string &err);

// Number of (surface edge, surface triangle) pairs sharing no vertex whose closed segment
// strictly crosses the triangle at positions x [n][3] (surface s = W x).
// E_INTERSECTING / 8(c) O0 "no surface edge crosses a surface triangle"; a touching (zero
// distance) configuration is left to the distance check.  Uniform grid over the triangles.
long long surface_edge_triangle_crossings(const HostMesh &m, const double *x);

// W rows of points embedded in the rest mesh (lowest-index containing tet, barycentric weights
// clamped at -tol..0 and renormalised); 0 or PD_IPC_E_* with err filled.
int build_embedding(int n, int T, const int32_t *tets, const double *X, int np, const double *pts, double tol,
                    int32_t *etet, double *ew, std::string &err);

}  // namespace pdipc
