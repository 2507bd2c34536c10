// Host-side one-time setup of the PD+IPC solver (untimed).
//
// PAPER.md:72-85 (section 2.1, Eq. 1-2): per tet D_m = [X1-X0, X2-X0, X3-X0], w = det/6,
// B = D_m^{-1}; corner gradients g_c = row c-1 of B, g_0 = -(g_1+g_2+g_3); F = sum_c x_c g_c^T;
// H = sum_i w_i G_i^T G_i = L (x) I3 with the scalar L_uv = sum_i w_i g_{i,u}.g_{i,v}
// (SURVEY.md Z21, App. A.2).  "Its Cholesky factorization could be pre-computed"
// (PAPER.md:85): L_FF (Dirichlet vertices eliminated) is ordered by geometric
// nested dissection and factorised once by a left-looking supernodal Cholesky.
#include "setup.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "../../include/pd_ipc.h"

namespace pdipc {

static double det3(const double *M) {  // row-major
    return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
           M[2] * (M[3] * M[7] - M[4] * M[6]);
}

static void inv3(const double *M, double *I) {
    double d = det3(M);
    I[0] = (M[4] * M[8] - M[5] * M[7]) / d;
    I[1] = (M[2] * M[7] - M[1] * M[8]) / d;
    I[2] = (M[1] * M[5] - M[2] * M[4]) / d;
    I[3] = (M[5] * M[6] - M[3] * M[8]) / d;
    I[4] = (M[0] * M[8] - M[2] * M[6]) / d;
    I[5] = (M[2] * M[3] - M[0] * M[5]) / d;
    I[6] = (M[3] * M[7] - M[4] * M[6]) / d;
    I[7] = (M[1] * M[6] - M[0] * M[7]) / d;
    I[8] = (M[0] * M[4] - M[1] * M[3]) / d;
}

int build_host_mesh(int n, int T, const int32_t *tets, int nfix, const int32_t *fixed,
                    const double *rest, int Ns, int Nt, const int32_t *tris,
                    const int32_t *embed_tet, const double *embed_w, HostMesh &m,
                    std::string &err) {
    if (n <= 0 || T <= 0 || !tets || !rest) { err = "empty mesh"; return PD_IPC_E_ARG; }
    m.n = n;
    m.T = T;
    m.tets.assign(tets, tets + 4 * (size_t)T);
    m.rest.assign(rest, rest + 3 * (size_t)n);
    for (size_t i = 0; i < 3 * (size_t)n; ++i)
        if (!std::isfinite(rest[i])) { err = "non-finite rest position"; return PD_IPC_E_MESH; }
    m.B.resize(9 * (size_t)T);
    m.w.resize(T);
    for (int t = 0; t < T; ++t) {
        const int32_t *v = &tets[4 * t];
        for (int c = 0; c < 4; ++c)
            if (v[c] < 0 || v[c] >= n) { err = "tet index out of range"; return PD_IPC_E_MESH; }
        double Dm[9];
        for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a)
                Dm[a * 3 + c] = rest[3 * v[c + 1] + a] - rest[3 * v[0] + a];
        double d = det3(Dm);
        if (!(d > 0)) { err = "inverted or degenerate rest tet " + std::to_string(t); return PD_IPC_E_MESH; }
        m.w[t] = d / 6.0;
        inv3(Dm, &m.B[9 * (size_t)t]);
    }
    if (nfix <= 0 || !fixed) { err = "no Dirichlet vertices: H is singular"; return PD_IPC_E_NOT_SPD; }
    m.is_fixed.assign(n, 0);
    for (int i = 0; i < nfix; ++i) {
        if (fixed[i] < 0 || fixed[i] >= n) { err = "fixed index out of range"; return PD_IPC_E_MESH; }
        m.is_fixed[fixed[i]] = 1;
    }
    // ---- surface (s = W x)
    m.Ns = Ns;
    m.Nt = Nt;
    if (Nt > 0) {
        if (!tris || !embed_tet || !embed_w || Ns <= 0) { err = "surface arrays missing"; return PD_IPC_E_ARG; }
        m.tris.assign(tris, tris + 3 * (size_t)Nt);
        for (size_t i = 0; i < 3 * (size_t)Nt; ++i)
            if (tris[i] < 0 || tris[i] >= Ns) { err = "surface tri index out of range"; return PD_IPC_E_MESH; }
        m.W_ptr.assign(Ns + 1, 0);
        for (int j = 0; j < Ns; ++j) {
            int et = embed_tet[j];
            if (et < 0 || et >= T) { err = "embed_tet out of range"; return PD_IPC_E_MESH; }
            double sum = 0;
            for (int c = 0; c < 4; ++c) {
                double wv = embed_w[4 * j + c];
                if (!(wv >= 0.0 && wv <= 1.0)) { err = "W weight outside [0,1]"; return PD_IPC_E_MESH; }
                sum += wv;
                if (wv != 0.0) {
                    m.W_col.push_back(tets[4 * et + c]);
                    m.W_val.push_back(wv);
                }
            }
            if (std::fabs(sum - 1.0) > 1e-12) { err = "W row does not sum to 1"; return PD_IPC_E_MESH; }
            m.W_ptr[j + 1] = (int32_t)m.W_col.size();
        }
        // rest surface, degenerate triangles, mean edge length
        std::vector<double> s(3 * (size_t)Ns, 0.0);
        for (int j = 0; j < Ns; ++j)
            for (int k = m.W_ptr[j]; k < m.W_ptr[j + 1]; ++k)
                for (int a = 0; a < 3; ++a) s[3 * j + a] += m.W_val[k] * rest[3 * m.W_col[k] + a];
        std::vector<std::pair<int, int>> e;
        e.reserve(3 * (size_t)Nt);
        for (int f = 0; f < Nt; ++f) {
            const int32_t *t = &tris[3 * f];
            double u[3], v[3], c[3];
            for (int a = 0; a < 3; ++a) { u[a] = s[3 * t[1] + a] - s[3 * t[0] + a]; v[a] = s[3 * t[2] + a] - s[3 * t[0] + a]; }
            c[0] = u[1] * v[2] - u[2] * v[1];
            c[1] = u[2] * v[0] - u[0] * v[2];
            c[2] = u[0] * v[1] - u[1] * v[0];
            if (!(c[0] * c[0] + c[1] * c[1] + c[2] * c[2] > 0)) { err = "degenerate surface triangle"; return PD_IPC_E_MESH; }
            for (int k = 0; k < 3; ++k) {
                int a = t[k], b = t[(k + 1) % 3];
                e.push_back({std::min(a, b), std::max(a, b)});
            }
        }
        std::sort(e.begin(), e.end());
        e.erase(std::unique(e.begin(), e.end()), e.end());
        m.Ne = (int)e.size();
        m.edges.resize(2 * e.size());
        double sum_len = 0;
        for (size_t i = 0; i < e.size(); ++i) {
            m.edges[2 * i] = e[i].first;
            m.edges[2 * i + 1] = e[i].second;
            double l2 = 0;
            for (int a = 0; a < 3; ++a) {
                double d = s[3 * e[i].second + a] - s[3 * e[i].first + a];
                l2 += d * d;
            }
            sum_len += std::sqrt(l2);
        }
        m.mean_edge = e.empty() ? 0.0 : sum_len / e.size();
    } else {
        m.Ns = 0;
        m.Ne = 0;
        m.W_ptr.assign(1, 0);
    }
    return PD_IPC_OK;
}

// ------------------------------------------------------------------------------------------
// geometric nested dissection on the free-vertex graph
// ------------------------------------------------------------------------------------------
namespace {
struct NDCtx {
    const std::vector<int> *ptr, *adj;
    const double *xyz;              // [nf][3]
    std::vector<int> part;
    int tag = 0;
    std::vector<int> out;
};

void nd_rec(NDCtx &C, std::vector<int> verts) {
    if (verts.size() <= 48) {
        C.out.insert(C.out.end(), verts.begin(), verts.end());
        return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int v : verts)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], C.xyz[3 * v + a]);
            hi[a] = std::max(hi[a], C.xyz[3 * v + a]);
        }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
        if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
    size_t mid = verts.size() / 2;
    std::nth_element(verts.begin(), verts.begin() + mid, verts.end(), [&](int a, int b) {
        double ca = C.xyz[3 * a + ax], cb = C.xyz[3 * b + ax];
        return ca < cb || (ca == cb && a < b);
    });
    std::vector<int> A(verts.begin(), verts.begin() + mid), Bv(verts.begin() + mid, verts.end());
    int tB = ++C.tag;
    for (int v : Bv) C.part[v] = tB;
    std::vector<int> sep, Ap;
    for (int v : A) {
        bool touch = false;
        for (int k = (*C.ptr)[v]; k < (*C.ptr)[v + 1]; ++k)
            if (C.part[(*C.adj)[k]] == tB) { touch = true; break; }
        (touch ? sep : Ap).push_back(v);
    }
    std::sort(Ap.begin(), Ap.end());
    std::sort(Bv.begin(), Bv.end());
    std::sort(sep.begin(), sep.end());
    nd_rec(C, Ap);
    nd_rec(C, Bv);
    C.out.insert(C.out.end(), sep.begin(), sep.end());
}
}  // namespace

int factorize(HostMesh &m, HostFactor &f, std::string &err) {
    const int n = m.n, T = m.T;
    // free numbering (natural)
    std::vector<int> v2f(n, -1), f2v;
    for (int v = 0; v < n; ++v)
        if (!m.is_fixed[v]) { v2f[v] = (int)f2v.size(); f2v.push_back(v); }
    const int nf = (int)f2v.size();
    if (nf == 0) { err = "no free vertices"; return PD_IPC_E_MESH; }
    m.nf = nf;
    // ---- assemble L_FF (scalar) as sorted triplets -> CSR (free numbering)
    struct Trip { int r, c; double v; };
    std::vector<Trip> tr;
    tr.reserve(16 * (size_t)T);
    for (int t = 0; t < T; ++t) {
        const double *Bt = &m.B[9 * (size_t)t];
        double g[4][3];
        for (int a = 0; a < 3; ++a) {
            g[1][a] = Bt[0 * 3 + a];
            g[2][a] = Bt[1 * 3 + a];
            g[3][a] = Bt[2 * 3 + a];
            g[0][a] = -(g[1][a] + g[2][a] + g[3][a]);
        }
        for (int u = 0; u < 4; ++u) {
            int fu = v2f[m.tets[4 * t + u]];
            if (fu < 0) continue;
            for (int v = 0; v < 4; ++v) {
                int fv = v2f[m.tets[4 * t + v]];
                if (fv < 0) continue;
                double val = m.w[t] * (g[u][0] * g[v][0] + g[u][1] * g[v][1] + g[u][2] * g[v][2]);
                tr.push_back({fu, fv, val});
            }
        }
    }
    std::sort(tr.begin(), tr.end(), [](const Trip &a, const Trip &b) {
        return a.r < b.r || (a.r == b.r && a.c < b.c);
    });
    std::vector<int> Ap(nf + 1, 0), Ai;
    std::vector<double> Ax;
    for (size_t k = 0; k < tr.size();) {
        size_t e = k;
        double s = 0;
        while (e < tr.size() && tr[e].r == tr[k].r && tr[e].c == tr[k].c) s += tr[e++].v;
        Ai.push_back(tr[k].c);
        Ax.push_back(s);
        Ap[tr[k].r + 1]++;
        k = e;
    }
    tr.clear();
    tr.shrink_to_fit();
    for (int i = 0; i < nf; ++i) Ap[i + 1] += Ap[i];
    // ---- nested dissection on the off-diagonal graph
    std::vector<int> gptr(nf + 1, 0), gadj;
    for (int i = 0; i < nf; ++i) {
        for (int k = Ap[i]; k < Ap[i + 1]; ++k)
            if (Ai[k] != i) gadj.push_back(Ai[k]);
        gptr[i + 1] = (int)gadj.size();
    }
    std::vector<double> xyz(3 * (size_t)nf);
    for (int i = 0; i < nf; ++i)
        for (int a = 0; a < 3; ++a) xyz[3 * i + a] = m.rest[3 * f2v[i] + a];
    NDCtx C;
    C.ptr = &gptr;
    C.adj = &gadj;
    C.xyz = xyz.data();
    C.part.assign(nf, 0);
    std::vector<int> all(nf);
    std::iota(all.begin(), all.end(), 0);
    nd_rec(C, all);
    std::vector<int> ord = C.out;               // position -> free index
    // ---- etree of the permuted matrix (Liu), then postorder
    auto etree_of = [&](const std::vector<int> &o, std::vector<int> &parent) {
        std::vector<int> pos(nf);
        for (int k = 0; k < nf; ++k) pos[o[k]] = k;
        parent.assign(nf, -1);
        std::vector<int> anc(nf, -1);
        for (int k = 0; k < nf; ++k) {
            int fi = o[k];
            for (int e = Ap[fi]; e < Ap[fi + 1]; ++e) {
                int i = pos[Ai[e]];
                if (i >= k) continue;
                while (i != -1 && i < k) {
                    int nxt = anc[i];
                    anc[i] = k;
                    if (nxt == -1) { parent[i] = k; break; }
                    i = nxt;
                }
            }
        }
    };
    std::vector<int> parent;
    etree_of(ord, parent);
    {
        std::vector<int> head(nf, -1), next(nf, -1), post;
        post.reserve(nf);
        for (int j = nf - 1; j >= 0; --j)
            if (parent[j] != -1) { next[j] = head[parent[j]]; head[parent[j]] = j; }
        std::vector<int> stack;
        for (int r = 0; r < nf; ++r) {
            if (parent[r] != -1) continue;
            stack.push_back(r);
            while (!stack.empty()) {
                int p = stack.back();
                int c = head[p];
                if (c == -1) { stack.pop_back(); post.push_back(p); }
                else { head[p] = next[c]; stack.push_back(c); }
            }
        }
        std::vector<int> o2(nf);
        for (int k = 0; k < nf; ++k) o2[k] = ord[post[k]];
        ord.swap(o2);
        etree_of(ord, parent);
    }
    std::vector<int> pos(nf);
    for (int k = 0; k < nf; ++k) pos[ord[k]] = k;
    m.q2v.resize(nf);
    m.v2q.assign(n, -1);
    for (int k = 0; k < nf; ++k) {
        m.q2v[k] = f2v[ord[k]];
        m.v2q[f2v[ord[k]]] = k;
    }
    // ---- permuted lower pattern by column: rows i > j
    std::vector<int> Lp(nf + 1, 0), Li;
    std::vector<double> Lx;
    {
        std::vector<std::vector<std::pair<int, double>>> cols(nf);
        for (int fi = 0; fi < nf; ++fi) {
            int j = pos[fi];
            for (int e = Ap[fi]; e < Ap[fi + 1]; ++e) {
                int i = pos[Ai[e]];
                if (i >= j) cols[j].push_back({i, Ax[e]});
            }
        }
        for (int j = 0; j < nf; ++j) {
            std::sort(cols[j].begin(), cols[j].end());
            for (auto &pr : cols[j]) { Li.push_back(pr.first); Lx.push_back(pr.second); }
            Lp[j + 1] = (int)Li.size();
        }
    }
    // ---- column structures struct(j) = A_lower(:,j) U children structs \ {child}
    std::vector<int> nchild(nf, 0);
    std::vector<std::vector<int>> kids(nf);
    for (int j = 0; j < nf; ++j)
        if (parent[j] >= 0) { nchild[parent[j]]++; kids[parent[j]].push_back(j); }
    std::vector<std::vector<int>> cs(nf);
    std::vector<int> mark(nf, -1);
    for (int j = 0; j < nf; ++j) {
        std::vector<int> &S = cs[j];
        mark[j] = j;
        S.push_back(j);
        for (int e = Lp[j]; e < Lp[j + 1]; ++e)
            if (mark[Li[e]] != j) { mark[Li[e]] = j; S.push_back(Li[e]); }
        for (int c : kids[j]) {
            for (int r : cs[c])
                if (r > j && mark[r] != j) { mark[r] = j; S.push_back(r); }
        }
        std::sort(S.begin(), S.end());
        // children structures are no longer needed once the parent has absorbed them, except
        // the last column of each supernode; keep all (memory ~ nnz(L) ints)
    }
    // ---- supernodes: fundamental + small relaxed chains, capped width
    // Relaxed amalgamation: every etree chain (column j-1's parent is j) is merged up to CAP
    // columns, accepting explicit zeros.  The triangular solves are latency-bound (one work
    // item per supernode on the critical path), so fewer, wider supernodes win over the extra
    // flops; fundamental supernodes are merged regardless.
    const int CAP = 128, RELAX = 128;
    std::vector<int> sn_start;
    int width = 0;
    for (int j = 0; j < nf; ++j) {
        bool merge = false;
        if (j > 0 && parent[j - 1] == j && width < CAP) {
            bool fund = nchild[j] == 1 && cs[j - 1].size() == cs[j].size() + 1;
            merge = fund || width < RELAX;
        }
        if (!merge) { sn_start.push_back(j); width = 1; }
        else ++width;
    }
    sn_start.push_back(nf);
    const int nsn = (int)sn_start.size() - 1;
    f.nf = nf;
    f.nsn = nsn;
    f.sn_c0.assign(sn_start.begin(), sn_start.end());
    f.col2sn.resize(nf);
    for (int s = 0; s < nsn; ++s)
        for (int j = sn_start[s]; j < sn_start[s + 1]; ++j) f.col2sn[j] = s;
    f.sn_rowptr.assign(nsn + 1, 0);
    f.sn_valptr.assign(nsn + 1, 0);
    f.sn_parent.assign(nsn, -1);
    f.sn_rows.clear();
    for (int s = 0; s < nsn; ++s) {
        int c0 = sn_start[s], c1 = sn_start[s + 1];
        for (int j = c0; j < c1; ++j) f.sn_rows.push_back(j);
        for (int r : cs[c1 - 1])
            if (r >= c1) f.sn_rows.push_back(r);
        f.sn_rowptr[s + 1] = (int32_t)f.sn_rows.size();
        int nr = f.sn_rowptr[s + 1] - f.sn_rowptr[s];
        f.sn_valptr[s + 1] = f.sn_valptr[s] + (int64_t)nr * (c1 - c0);
        int pc = parent[c1 - 1];
        f.sn_parent[s] = pc < 0 ? -1 : f.col2sn[pc];
        f.max_width = std::max(f.max_width, c1 - c0);
        f.max_rows = std::max(f.max_rows, nr);
    }
    cs.clear();
    cs.shrink_to_fit();
    f.nnzL = f.sn_valptr[nsn];
    f.sn_nchild.assign(nsn, 0);
    f.sn_fd.resize(nsn);
    for (int s = 0; s < nsn; ++s) f.sn_fd[s] = sn_start[s];
    for (int s = 0; s < nsn; ++s) {
        int p = f.sn_parent[s];
        if (p >= 0) {
            f.sn_nchild[p]++;
            f.sn_fd[p] = std::min(f.sn_fd[p], f.sn_fd[s]);
        }
    }
    {
        std::vector<int> dep(nsn, 1);
        for (int s = nsn - 1; s >= 0; --s)
            if (f.sn_parent[s] >= 0) dep[s] = dep[f.sn_parent[s]] + 1;
        f.depth = *std::max_element(dep.begin(), dep.end());
    }
    // ---- update segments: for d, off-diagonal rows grouped by target supernode
    std::vector<std::vector<int>> segs(nsn);   // flattened triples (d, klo, khi)
    for (int d = 0; d < nsn; ++d) {
        int r0 = f.sn_rowptr[d], r1 = f.sn_rowptr[d + 1];
        int w = sn_start[d + 1] - sn_start[d];
        int k = w;
        while (k < r1 - r0) {
            int t = f.col2sn[f.sn_rows[r0 + k]];
            int k2 = k;
            while (k2 < r1 - r0 && f.col2sn[f.sn_rows[r0 + k2]] == t) ++k2;
            segs[t].push_back(d);
            segs[t].push_back(k);
            segs[t].push_back(k2);
            k = k2;
        }
    }
    f.seg_ptr.assign(nsn + 1, 0);
    for (int s = 0; s < nsn; ++s) {
        for (size_t i = 0; i < segs[s].size(); i += 3) {
            f.seg_d.push_back(segs[s][i]);
            f.seg_klo.push_back(segs[s][i + 1]);
            f.seg_khi.push_back(segs[s][i + 2]);
        }
        f.seg_ptr[s + 1] = (int32_t)f.seg_d.size();
    }
    // ---- numeric left-looking supernodal Cholesky
    f.vals.assign((size_t)f.nnzL, 0.0);
    std::vector<int> rowmap(nf, -1);
    std::vector<double> tmp;
    for (int s = 0; s < nsn; ++s) {
        const int c0 = sn_start[s], c1 = sn_start[s + 1], w = c1 - c0;
        const int r0 = f.sn_rowptr[s], nr = f.sn_rowptr[s + 1] - r0;
        double *Ls = &f.vals[(size_t)f.sn_valptr[s]];
        for (int k = 0; k < nr; ++k) rowmap[f.sn_rows[r0 + k]] = k;
        for (int j = c0; j < c1; ++j)
            for (int e = Lp[j]; e < Lp[j + 1]; ++e) Ls[rowmap[Li[e]] + (size_t)(j - c0) * nr] = Lx[e];
        for (int sg = f.seg_ptr[s]; sg < f.seg_ptr[s + 1]; ++sg) {
            const int d = f.seg_d[sg], klo = f.seg_klo[sg], khi = f.seg_khi[sg];
            const int dr0 = f.sn_rowptr[d], dnr = f.sn_rowptr[d + 1] - dr0;
            const int dw = sn_start[d + 1] - sn_start[d];
            const double *Ld = &f.vals[(size_t)f.sn_valptr[d]];
            const int m_rows = dnr - klo;
            tmp.assign((size_t)m_rows * dw, 0.0);         // row-major copy of rows klo..dnr-1
            for (int c = 0; c < dw; ++c)
                for (int i = 0; i < m_rows; ++i) tmp[(size_t)i * dw + c] = Ld[klo + i + (size_t)c * dnr];
            for (int jj = 0; jj < khi - klo; ++jj) {
                const int tc = f.sn_rows[dr0 + klo + jj] - c0;
                const double *rj = &tmp[(size_t)jj * dw];
                for (int ii = jj; ii < m_rows; ++ii) {
                    const double *ri = &tmp[(size_t)ii * dw];
                    double acc = 0;
                    for (int c = 0; c < dw; ++c) acc += ri[c] * rj[c];
                    Ls[rowmap[f.sn_rows[dr0 + klo + ii]] + (size_t)tc * nr] -= acc;
                }
            }
        }
        for (int k = 0; k < w; ++k) {
            double *ck = Ls + (size_t)k * nr;
            double piv = ck[k];
            if (!(piv > 0) || !std::isfinite(piv)) { err = "Cholesky pivot <= 0"; return PD_IPC_E_NOT_SPD; }
            double dk = std::sqrt(piv);
            ck[k] = dk;
            for (int i = k + 1; i < nr; ++i) ck[i] /= dk;
            for (int j = k + 1; j < w; ++j) {
                double *cj = Ls + (size_t)j * nr;
                double ljk = ck[j];
                for (int i = j; i < nr; ++i) cj[i] -= ck[i] * ljk;
            }
        }
        for (int k = 0; k < w; ++k)                      // keep the diagonal block lower
            for (int i = 0; i < k; ++i) Ls[i + (size_t)k * nr] = 0.0;
    }
    // ---- right-looking update rows (U) and their per-row gather lists, diagonal inverses
    {
        f.uoff.assign(nsn + 1, 0);
        for (int d = 0; d < nsn; ++d) {
            int w = sn_start[d + 1] - sn_start[d];
            int nr = f.sn_rowptr[d + 1] - f.sn_rowptr[d];
            f.uoff[d + 1] = f.uoff[d] + (nr - w);
        }
        f.urow_sn.resize(f.uoff[nsn]);
        std::vector<int> cnt(nf + 1, 0);
        for (int d = 0; d < nsn; ++d) {
            int w = sn_start[d + 1] - sn_start[d];
            for (int k = w; k < f.sn_rowptr[d + 1] - f.sn_rowptr[d]; ++k) {
                cnt[f.sn_rows[f.sn_rowptr[d] + k] + 1]++;
                f.urow_sn[f.uoff[d] + k - w] = d;
            }
        }
        // Multifrontal extend-add lists: the update block of supernode c (one U row per
        // off-diagonal row of c, already including c's own children) is consumed by its
        // parent s: rows that are columns of s are subtracted from s's right-hand side, the
        // others are added into s's own update block.  rc lists are indexed by the supernode
        // row slot sn_rowptr[s] + p (p = position of the row in R_s); sources are the child
        // U rows landing on that row, in increasing child order (deterministic).
        (void)cnt;
        const int nslots = f.sn_rowptr[nsn];
        std::vector<int> scount(nslots + 1, 0);
        std::vector<std::vector<std::pair<int, int>>> src(nsn);   // per parent: (slot, u)
        for (int c = 0; c < nsn; ++c) {
            const int s = f.sn_parent[c];
            if (s < 0) continue;
            const int wc = sn_start[c + 1] - sn_start[c];
            const int *Rs = &f.sn_rows[f.sn_rowptr[s]];
            const int nrs = f.sn_rowptr[s + 1] - f.sn_rowptr[s];
            for (int k = wc; k < f.sn_rowptr[c + 1] - f.sn_rowptr[c]; ++k) {
                const int r = f.sn_rows[f.sn_rowptr[c] + k];
                const int p = (int)(std::lower_bound(Rs, Rs + nrs, r) - Rs);
                if (p >= nrs || Rs[p] != r) { err = "supernode row containment violated"; return PD_IPC_E_NOT_SPD; }
                src[s].push_back({f.sn_rowptr[s] + p, f.uoff[c] + k - wc});
            }
        }
        f.urel.assign(f.uoff[nsn], -1);
        for (int s = 0; s < nsn; ++s)
            for (auto &pr : src[s]) f.urel[pr.second] = pr.first - f.sn_rowptr[s];
        f.ch_ptr.assign(nsn + 1, 0);
        for (int c = 0; c < nsn; ++c)
            if (f.sn_parent[c] >= 0) f.ch_ptr[f.sn_parent[c] + 1]++;
        for (int s = 0; s < nsn; ++s) f.ch_ptr[s + 1] += f.ch_ptr[s];
        f.ch.assign(f.ch_ptr[nsn], 0);
        {
            std::vector<int> cf(f.ch_ptr.begin(), f.ch_ptr.end() - 1);
            for (int c = 0; c < nsn; ++c)
                if (f.sn_parent[c] >= 0) f.ch[cf[f.sn_parent[c]]++] = c;
        }
        for (int s = 0; s < nsn; ++s)
            for (auto &pr : src[s]) scount[pr.first + 1]++;
        f.rc_ptr.assign(nslots + 1, 0);
        for (int i = 0; i < nslots; ++i) f.rc_ptr[i + 1] = f.rc_ptr[i] + scount[i + 1];
        f.rc_idx.assign(f.rc_ptr[nslots], 0);
        std::vector<int> fill(f.rc_ptr.begin(), f.rc_ptr.end() - 1);
        for (int s = 0; s < nsn; ++s)          // children in increasing order
            for (auto &pr : src[s]) f.rc_idx[fill[pr.first]++] = pr.second;
        f.dinv_ptr.assign(nsn + 1, 0);
        for (int s = 0; s < nsn; ++s) {
            int w = sn_start[s + 1] - sn_start[s];
            f.dinv_ptr[s + 1] = f.dinv_ptr[s] + (int64_t)w * w;
        }
        f.dinv.assign((size_t)f.dinv_ptr[nsn], 0.0);
        for (int s = 0; s < nsn; ++s) {
            const int w = sn_start[s + 1] - sn_start[s], nr = f.sn_rowptr[s + 1] - f.sn_rowptr[s];
            const double *Ls = &f.vals[(size_t)f.sn_valptr[s]];
            double *D = &f.dinv[(size_t)f.dinv_ptr[s]];
            for (int c = 0; c < w; ++c)            // column c of L_ss^{-1} by forward substitution
                for (int i = c; i < w; ++i) {
                    double acc = (i == c) ? 1.0 : 0.0;
                    for (int k = c; k < i; ++k) acc -= Ls[i + (size_t)k * nr] * D[(size_t)k * w + c];
                    D[(size_t)i * w + c] = acc / Ls[i + (size_t)i * nr];
                }
        }
        // Q_s = [L_ss^{-1}; L_off L_ss^{-1}] (column-major, ld nr, the layout of L): the forward
        // solve's item block b computes rows of Q_s x_s, the backward solve Q_s^T [z_s; -x_R].
        f.Q.assign(f.vals.size(), 0.0);
        for (int s = 0; s < nsn; ++s) {
            const int w = sn_start[s + 1] - sn_start[s], nr = f.sn_rowptr[s + 1] - f.sn_rowptr[s];
            const double *Ls = &f.vals[(size_t)f.sn_valptr[s]];
            const double *D = &f.dinv[(size_t)f.dinv_ptr[s]];
            double *Qs = &f.Q[(size_t)f.sn_valptr[s]];
            for (int k = 0; k < w; ++k)
                for (int i = k; i < w; ++i) Qs[i + (size_t)k * nr] = D[(size_t)i * w + k];
            for (int k = 0; k < w; ++k)
                for (int r = w; r < nr; ++r) {
                    double acc = 0.0;
                    for (int j = k; j < w; ++j) acc += Ls[r + (size_t)j * nr] * D[(size_t)j * w + k];
                    Qs[r + (size_t)k * nr] = acc;
                }
        }
    }
    // ---- transpose incidence in factor order and W^T over factor positions
    {
        std::vector<std::vector<int>> incl(nf);
        for (int t = 0; t < T; ++t)
            for (int c = 0; c < 4; ++c) {
                int q = m.v2q[m.tets[4 * t + c]];
                if (q >= 0) incl[q].push_back((t << 2) | c);
            }
        m.inc_ptr.assign(nf + 1, 0);
        m.inc.clear();
        for (int q = 0; q < nf; ++q) {
            m.inc.insert(m.inc.end(), incl[q].begin(), incl[q].end());
            m.inc_ptr[q + 1] = (int32_t)m.inc.size();
        }
        std::vector<std::vector<std::pair<int, double>>> wt(nf);
        for (int j = 0; j < m.Ns; ++j)
            for (int k = m.W_ptr[j]; k < m.W_ptr[j + 1]; ++k) {
                int q = m.v2q[m.W_col[k]];
                if (q >= 0) wt[q].push_back({j, m.W_val[k]});
            }
        m.WT_ptr.assign(nf + 1, 0);
        for (int q = 0; q < nf; ++q) {
            for (auto &pr : wt[q]) { m.WT_row.push_back(pr.first); m.WT_val.push_back(pr.second); }
            m.WT_ptr[q + 1] = (int32_t)m.WT_row.size();
        }
    }
    return PD_IPC_OK;
}


// ------------------------------------------------------------------ intersection check ------
// Segment pq strictly crosses triangle abc iff p and q lie strictly on opposite sides of the
// triangle's plane and the line pq passes strictly inside the three edges (signed volumes of
// the same sign).  Zero volumes (touching, coplanar) are not counted: a touching pair has a
// zero distance, which the distance check reports.
static inline double orient3(const double *a, const double *b, const double *c, const double *d) {
    const double ux = b[0] - a[0], uy = b[1] - a[1], uz = b[2] - a[2];
    const double vx = c[0] - a[0], vy = c[1] - a[1], vz = c[2] - a[2];
    const double wx = d[0] - a[0], wy = d[1] - a[1], wz = d[2] - a[2];
    return ux * (vy * wz - vz * wy) - uy * (vx * wz - vz * wx) + uz * (vx * wy - vy * wx);
}

long long surface_edge_triangle_crossings(const HostMesh &m, const double *x) {
    if (m.Nt == 0 || m.Ne == 0) return 0;
    std::vector<double> s(3 * (size_t)m.Ns, 0.0);
    for (int j = 0; j < m.Ns; ++j)
        for (int k = m.W_ptr[j]; k < m.W_ptr[j + 1]; ++k)
            for (int a = 0; a < 3; ++a) s[3 * (size_t)j + a] += m.W_val[k] * x[3 * (size_t)m.W_col[k] + a];
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int j = 0; j < m.Ns; ++j)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], s[3 * (size_t)j + a]);
            hi[a] = std::max(hi[a], s[3 * (size_t)j + a]);
        }
    // cell = max(mean edge, box extent / 256) so the grid stays bounded
    double cell = std::max(m.mean_edge, 1e-300);
    for (int a = 0; a < 3; ++a) cell = std::max(cell, (hi[a] - lo[a]) / 256.0);
    int dim[3];
    for (int a = 0; a < 3; ++a) dim[a] = std::max(1, (int)std::floor((hi[a] - lo[a]) / cell) + 1);
    auto cidx = [&](double v, int a) { return std::min(dim[a] - 1, std::max(0, (int)std::floor((v - lo[a]) / cell))); };
    // bin triangles by their boxes
    std::vector<std::pair<long long, int>> ent;
    for (int t = 0; t < m.Nt; ++t) {
        int c0[3], c1[3];
        for (int a = 0; a < 3; ++a) {
            double l = 1e300, h = -1e300;
            for (int k = 0; k < 3; ++k) {
                const double v = s[3 * (size_t)m.tris[3 * t + k] + a];
                l = std::min(l, v);
                h = std::max(h, v);
            }
            c0[a] = cidx(l, a);
            c1[a] = cidx(h, a);
        }
        for (int i = c0[0]; i <= c1[0]; ++i)
            for (int j = c0[1]; j <= c1[1]; ++j)
                for (int k = c0[2]; k <= c1[2]; ++k)
                    ent.push_back({((long long)i * dim[1] + j) * dim[2] + k, t});
    }
    std::sort(ent.begin(), ent.end());
    long long count = 0;
    std::vector<int> seen;
    for (int e = 0; e < m.Ne; ++e) {
        const int p = m.edges[2 * e], q = m.edges[2 * e + 1];
        const double *P = &s[3 * (size_t)p], *Q = &s[3 * (size_t)q];
        int c0[3], c1[3];
        for (int a = 0; a < 3; ++a) {
            c0[a] = cidx(std::min(P[a], Q[a]), a);
            c1[a] = cidx(std::max(P[a], Q[a]), a);
        }
        seen.clear();
        for (int i = c0[0]; i <= c1[0]; ++i)
            for (int j = c0[1]; j <= c1[1]; ++j)
                for (int k = c0[2]; k <= c1[2]; ++k) {
                    const long long key = ((long long)i * dim[1] + j) * dim[2] + k;
                    auto it = std::lower_bound(ent.begin(), ent.end(), std::make_pair(key, -1));
                    for (; it != ent.end() && it->first == key; ++it) seen.push_back(it->second);
                }
        std::sort(seen.begin(), seen.end());
        seen.erase(std::unique(seen.begin(), seen.end()), seen.end());
        for (int t : seen) {
            const int a = m.tris[3 * t], b = m.tris[3 * t + 1], c = m.tris[3 * t + 2];
            if (a == p || a == q || b == p || b == q || c == p || c == q) continue;
            const double *A = &s[3 * (size_t)a], *B = &s[3 * (size_t)b], *Cc = &s[3 * (size_t)c];
            // signed volumes below tol = 1e-12 L^3 (L the longest of the four edges) are rounding
            // noise of (near-)coplanar configurations -- e.g. the flat pieces of a subdivided
            // surface -- and count as zero
            auto d2 = [](const double *x, const double *y) {
                return (x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]) + (x[2] - y[2]) * (x[2] - y[2]);
            };
            const double L2 = std::max(std::max(d2(P, Q), d2(A, B)), std::max(d2(B, Cc), d2(Cc, A)));
            const double tol = 1e-12 * L2 * std::sqrt(L2);
            const double op = orient3(A, B, Cc, P), oq = orient3(A, B, Cc, Q);
            if (!((op > tol && oq < -tol) || (op < -tol && oq > tol))) continue;
            const double u = orient3(P, Q, A, B), v = orient3(P, Q, B, Cc), w = orient3(P, Q, Cc, A);
            if ((u > tol && v > tol && w > tol) || (u < -tol && v < -tol && w < -tol)) ++count;
        }
    }
    return count;
}

}  // namespace pdipc

namespace pdipc {

// ------------------------------------------------------------------ embedding --
// W rows for points embedded in the rest tet mesh ("embedded surface"; SPEC.md:53-61
// build_embedding, :81 tie rule): the lowest-index tet whose barycentric coordinates of the point
// are all >= -tol; weights = those coordinates with negatives (|.| <= tol) clamped to 0 and the
// row renormalised to sum 1.  Uniform grid over the tets' rest boxes.
int build_embedding(int n, int T, const int32_t *tets, const double *X, int np, const double *pts, double tol,
                    int32_t *etet, double *ew, std::string &err) {
    if (n <= 0 || T <= 0 || np < 0 || !tets || !X || (np > 0 && (!pts || !etet || !ew))) {
        err = "build_embedding: bad arguments";
        return PD_IPC_E_ARG;
    }
    for (int t = 0; t < 4 * T; ++t)
        if (tets[t] < 0 || tets[t] >= n) {
            err = "build_embedding: tet vertex index out of range";
            return PD_IPC_E_MESH;
        }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300}, el = 0.0;
    for (int v = 0; v < n; ++v)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], X[3 * (size_t)v + a]);
            hi[a] = std::max(hi[a], X[3 * (size_t)v + a]);
        }
    for (int t = 0; t < T; ++t) {
        const double *p0 = X + 3 * (size_t)tets[4 * t], *p1 = X + 3 * (size_t)tets[4 * t + 1];
        el += std::sqrt((p1[0] - p0[0]) * (p1[0] - p0[0]) + (p1[1] - p0[1]) * (p1[1] - p0[1]) +
                        (p1[2] - p0[2]) * (p1[2] - p0[2]));
    }
    const double cell = std::max(el / T, 1e-300);
    int dim[3];
    for (int a = 0; a < 3; ++a) dim[a] = std::max(1, std::min(1024, (int)std::floor((hi[a] - lo[a]) / cell) + 1));
    auto cid = [&](double v, int a) {
        const double c = (hi[a] > lo[a]) ? (v - lo[a]) / (hi[a] - lo[a]) * dim[a] : 0.0;
        return std::min(dim[a] - 1, std::max(0, (int)std::floor(c)));
    };
    std::vector<std::pair<long long, int>> ent;
    for (int t = 0; t < T; ++t) {
        int c0[3], c1[3];
        for (int a = 0; a < 3; ++a) {
            double l = 1e300, h = -1e300;
            for (int k = 0; k < 4; ++k) {
                const double v = X[3 * (size_t)tets[4 * t + k] + a];
                l = std::min(l, v);
                h = std::max(h, v);
            }
            const double pad = 1e-9 * cell;   // points within tolerance just outside the box
            c0[a] = cid(l - pad, a);
            c1[a] = cid(h + pad, a);
        }
        for (int i = c0[0]; i <= c1[0]; ++i)
            for (int j = c0[1]; j <= c1[1]; ++j)
                for (int k = c0[2]; k <= c1[2]; ++k) ent.push_back({((long long)i * dim[1] + j) * dim[2] + k, t});
    }
    std::sort(ent.begin(), ent.end());   // within a cell: increasing tet index
    for (int q = 0; q < np; ++q) {
        const double *p = pts + 3 * (size_t)q;
        const long long key = ((long long)cid(p[0], 0) * dim[1] + cid(p[1], 1)) * dim[2] + cid(p[2], 2);
        auto it = std::lower_bound(ent.begin(), ent.end(), std::make_pair(key, -1));
        int found = -1;
        double lam[4] = {0, 0, 0, 0};
        for (; it != ent.end() && it->first == key; ++it) {
            const int t = it->second;
            const double *x0 = X + 3 * (size_t)tets[4 * t];
            double D[3][3], r[3];
            for (int a = 0; a < 3; ++a) {
                for (int c = 0; c < 3; ++c) D[a][c] = X[3 * (size_t)tets[4 * t + c + 1] + a] - x0[a];
                r[a] = p[a] - x0[a];
            }
            const double det = D[0][0] * (D[1][1] * D[2][2] - D[1][2] * D[2][1]) -
                               D[0][1] * (D[1][0] * D[2][2] - D[1][2] * D[2][0]) +
                               D[0][2] * (D[1][0] * D[2][1] - D[1][1] * D[2][0]);
            if (!(std::fabs(det) > 0)) continue;
            double l[3];   // Cramer's rule: D l = r
            for (int c = 0; c < 3; ++c) {
                double M[3][3];
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) M[a][b] = b == c ? r[a] : D[a][b];
                l[c] = (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                        M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                        M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0])) / det;
            }
            const double l0 = 1.0 - l[0] - l[1] - l[2];
            if (l0 >= -tol && l[0] >= -tol && l[1] >= -tol && l[2] >= -tol) {
                if (found < 0 || t < found) {
                    found = t;
                    lam[0] = l0;
                    lam[1] = l[0];
                    lam[2] = l[1];
                    lam[3] = l[2];
                }
            }
        }
        if (found < 0) {
            err = "build_embedding: point " + std::to_string(q) + " lies outside every tet";
            return PD_IPC_E_MESH;
        }
        double sum = 0.0;
        for (int k = 0; k < 4; ++k) {
            lam[k] = std::max(0.0, lam[k]);
            sum += lam[k];
        }
        etet[q] = found;
        for (int k = 0; k < 4; ++k) ew[4 * (size_t)q + k] = lam[k] / sum;
    }
    return 0;
}

}  // namespace pdipc
