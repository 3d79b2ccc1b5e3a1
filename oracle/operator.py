"""The d x d block coefficient matrix, assembled element by element by Gauss quadrature.

Oracle (test infrastructure only).

The product path evaluates the operator matrix-free as sums of Kronecker products;
this oracle never uses that structure.  It assembles the sparse matrix entry by entry
from the bilinear form, evaluating the integrand with explicit vector calculus on the
tensor-product B-spline basis functions psi = N_{i_1}(x_1)..N_{i_d}(x_d) e_j
(PAPER.md:409-437 (2D space V_h), 494-513 (3D)).

Two bilinear forms:
  * kind="alfven"  (the north-star operator; reading R1 in DESIGN.md): the weak form of
        L_A u = nu u - beta lambda grad(div u) - lambda b0 x (curl curl (b0 x u))
     with homogeneous Dirichlet conditions:
        a(u,v) = nu (u,v) + beta lambda (div u, div v) + lambda (curl(b0 x u), curl(b0 x v)).
    In 2D, u = (u1,u2,0), b0 = (b1,b2,0), no x3-dependence.
  * kind="curldiv" (the paper's model operator, eq:curl-div):
        a(u,v) = alpha (curl u, curl v) + beta (div u, div v),
    2D curl u = d1 u2 - d2 u1.
Unknown ordering: component-major, then lexicographic with direction 1 slowest
("u^1 := [u^1_{2,2}, ..., u^1_{n1+p-1,n2+p-1}]").
"""
import itertools

import numpy as np
import scipy.sparse as sp

from .bspline import element_tables


def form_alfven(nu, beta, lam, b0):
    return dict(kind="alfven", nu=float(nu), beta=float(beta), lam=float(lam), b0=tuple(float(v) for v in b0))


def form_curldiv(alpha, beta):
    return dict(kind="curldiv", alpha=float(alpha), beta=float(beta))


def _features(form, d, Nv, G):
    """Integrand terms for every vector basis function psi = N e_j at every quad point.

    Nv[E,Q,L] scalar values, G[E,Q,L,d] scalar gradients.  Returns a list of
    (coef, F) with F[E,Q,j,L,c]: the c-th entry of the term's vector for psi = N_L e_j;
    a(psi_a, psi_b) = sum_terms coef * sum_Q w * F_a . F_b.
    """
    E, Q, L = Nv.shape
    G3 = np.zeros((E, Q, L, 3))
    G3[..., :d] = G
    terms = []
    if form["kind"] == "alfven":
        # value: psi itself
        val = np.zeros((E, Q, d, L, d))
        for j in range(d):
            val[:, :, j, :, j] = Nv
        terms.append((form["nu"], val))
        # div psi = d_j N
        div = np.zeros((E, Q, d, L, 1))
        for j in range(d):
            div[:, :, j, :, 0] = G[..., j]
        terms.append((form["beta"] * form["lam"], div))
        # curl(b0 x psi) = curl(N c) with c = b0 x e_j constant: = grad N x c
        b0 = np.zeros(3)
        b0[: len(form["b0"])] = form["b0"]
        cb = np.zeros((E, Q, d, L, 3))
        for j in range(d):
            ej = np.zeros(3)
            ej[j] = 1.0
            c = np.cross(b0, ej)
            cb[:, :, j, :, :] = np.cross(G3, c[None, None, None, :])
        terms.append((form["lam"], cb))
    elif form["kind"] == "curldiv":
        if d == 2:
            curl = np.zeros((E, Q, d, L, 1))
            curl[:, :, 0, :, 0] = -G[..., 1]      # curl(N e_1) = -d2 N
            curl[:, :, 1, :, 0] = G[..., 0]       # curl(N e_2) =  d1 N
        else:
            curl = np.zeros((E, Q, d, L, 3))
            for j in range(d):
                ej = np.zeros(3)
                ej[j] = 1.0
                curl[:, :, j, :, :] = np.cross(G3, ej[None, None, None, :])  # curl(N e_j) = grad N x e_j
        terms.append((form["alpha"], curl))
        div = np.zeros((E, Q, d, L, 1))
        for j in range(d):
            div[:, :, j, :, 0] = G[..., j]
        terms.append((form["beta"], div))
    else:
        raise ValueError(form["kind"])
    return terms


class Discretization:
    """Tensor-product B-spline space of degree p on n^d uniform elements, Dirichlet."""

    def __init__(self, d: int, p: int, n: int):
        self.d, self.p, self.n = d, p, n
        self.m = n + p - 2
        self.nscal = self.m ** d
        self.ndof = d * self.nscal
        self.q = p + 1
        self._cache = {}      # 1D element tables, computed on demand (large n: few elements used)

    def _tables(self, els):
        """(wq, B, D) rows for the listed 1D elements (see bspline.element_tables)."""
        miss = sorted(set(int(e) for e in els) - self._cache.keys())
        if miss:
            _, wq, B, D = element_tables(self.p, self.n, self.q, miss)
            for k, e in enumerate(miss):
                self._cache[e] = (wq[k], B[k], D[k])
        wq = np.array([self._cache[int(e)][0] for e in els])
        B = np.array([self._cache[int(e)][1] for e in els])
        D = np.array([self._cache[int(e)][2] for e in els])
        return wq, B, D

    def _element_data(self, elems):
        """Scalar basis values/gradients on a batch of elements (rows of multi-indices)."""
        d, p, q = self.d, self.p, self.q
        E = len(elems)
        # quadrature points / local functions as tensor products over directions
        qidx = np.array(list(itertools.product(range(q), repeat=d)))          # (Q,d)
        lidx = np.array(list(itertools.product(range(p + 1), repeat=d)))      # (L,d)
        Q, L = len(qidx), len(lidx)
        Nv = np.ones((E, Q, L))
        G = np.ones((E, Q, L, d))
        W = np.ones((E, Q))
        for l in range(d):
            wq, B, D = self._tables(elems[:, l])
            b = B[:, qidx[:, l], :][:, :, lidx[:, l]]     # (E,Q,L)
            db = D[:, qidx[:, l], :][:, :, lidx[:, l]]
            W *= wq[:, qidx[:, l]]
            Nv = Nv * b
            for c in range(d):
                G[..., c] *= db if c == l else b
        # global scalar interior index of each local function (-1 if a removed boundary spline)
        gidx = np.zeros((E, L), dtype=np.int64)
        valid = np.ones((E, L), dtype=bool)
        for l in range(d):
            i1 = elems[:, l][:, None] + lidx[None, :, l] + 1       # 1-based spline index
            k = i1 - 2
            valid &= (k >= 0) & (k < self.m)
            gidx = gidx * self.m + np.clip(k, 0, self.m - 1)
        return W, Nv, G, gidx, valid

    def local_matrices(self, form, elems):
        W, Nv, G, gidx, valid = self._element_data(elems)
        terms = _features(form, self.d, Nv, G)
        E, Q, L = Nv.shape
        d = self.d
        K = np.zeros((E, d * L, d * L))
        for coef, F in terms:
            if coef == 0.0:
                continue
            # K[e,a,b] += coef * sum_{q,c} W[e,q] F[e,q,a,c] F[e,q,b,c]: one matrix product per
            # element (library primitive numpy.matmul) over the flattened (q, c) index
            C = F.shape[-1]
            Fr = F.reshape(E, Q, d * L, C)
            X = Fr.transpose(0, 2, 1, 3).reshape(E, d * L, Q * C)
            Xw = (Fr * W[:, :, None, None]).transpose(0, 2, 1, 3).reshape(E, d * L, Q * C)
            K += coef * np.matmul(Xw, X.transpose(0, 2, 1))
        # global vector dof index: component j, scalar index
        gv = (np.arange(d)[None, :, None] * self.nscal + gidx[:, None, :]).reshape(E, d * L)
        vv = np.broadcast_to(valid[:, None, :], (E, d, L)).reshape(E, d * L)
        return K, gv, vv

    def assemble(self, form, chunk=None) -> sp.csr_matrix:
        """The full sparse matrix (test sizes only)."""
        elems = np.array(list(itertools.product(range(self.n), repeat=self.d)))
        if chunk is None:   # elements per batch: ~150 MB of feature arrays
            L = (self.p + 1) ** self.d
            chunk = max(1, int(1.5e8 // (8 * L * L * self.d * self.d)))
        rows, cols, vals = [], [], []
        A = sp.csr_matrix((self.ndof, self.ndof))
        for s in range(0, len(elems), chunk):
            K, gv, vv = self.local_matrices(form, elems[s: s + chunk])
            msk = vv[:, :, None] & vv[:, None, :]
            r = np.broadcast_to(gv[:, :, None], K.shape)[msk]
            c = np.broadcast_to(gv[:, None, :], K.shape)[msk]
            A = A + sp.coo_matrix((K[msk], (r, c)), shape=(self.ndof, self.ndof)).tocsr()
        A.sum_duplicates()
        return A

    def support_elements(self, dof):
        """Elements on which the basis function of vector dof ``dof`` is nonzero."""
        flat = dof % self.nscal
        ks = []
        for l in range(self.d):
            ks.append(flat // self.m ** (self.d - 1 - l) % self.m)
        rng = []
        for k in ks:
            i = k + 2                      # 1-based spline index
            rng.append(range(max(0, i - self.p - 1), min(self.n, i)))
        return np.array(list(itertools.product(*rng)), dtype=np.int64)

    def sampled_apply(self, form, x, dofs):
        """(A x)[dofs] computed row by row from the element integrals (any problem size).

        Per sampled dof only the local-matrix row of that basis function is formed:
        row_e = sum_terms coef sum_q w F_row(q) . F(q) over the elements of its support.
        """
        out = np.zeros(len(dofs))
        d = self.d
        for t, I in enumerate(dofs):
            I = int(I)
            elems = self.support_elements(I)
            W, Nv, G, gidx, valid = self._element_data(elems)
            terms = _features(form, d, Nv, G)
            E, Q, L = Nv.shape
            gv = (np.arange(d)[None, :, None] * self.nscal + gidx[:, None, :]).reshape(E, d * L)
            vv = np.broadcast_to(valid[:, None, :], (E, d, L)).reshape(E, d * L)
            s = 0.0
            for e in range(E):
                rows = np.nonzero((gv[e] == I) & vv[e])[0]
                if len(rows) == 0:
                    continue
                r = rows[0]
                krow = np.zeros(d * L)
                for coef, F in terms:
                    if coef == 0.0:
                        continue
                    Fr = F[e].reshape(Q, d * L, F.shape[-1])
                    krow += coef * np.einsum("q,qc,qbc->b", W[e], Fr[:, r, :], Fr)
                cm = vv[e]
                s += float(np.dot(krow[cm], x[gv[e, cm]]))
            out[t] = s
        return out
