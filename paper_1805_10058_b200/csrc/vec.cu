// R7: vector kernels of PCG / the V-cycle, with fused updates and deterministic reductions.
// Dot products: each CTA of a fixed-size grid reduces its grid-stride share (warp shuffle,
// then shared memory) into partial[blockIdx.x]; a one-CTA finalize sums the partials in a
// fixed order.  Scalars (alpha, beta numerators/denominators) stay on the device.
#include <algorithm>

#include "internal.cuh"

namespace igacd {

constexpr int VBS = 256;

int vec_ctas(size_t n) {
  long long b = (long long)((n + VBS * 4 - 1) / (VBS * 4));
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (int)b;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, size_t n, double* partial) {
  __shared__ double red[VBS / 32];
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS)
    s = fma(a[i], b[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_finalize(const double* partial, int np, double* dst) {
  __shared__ double red[VBS / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += VBS) s += partial[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *dst = s;
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) b[i] = a[i];
}

__global__ void k_zero(double* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) a[i] = 0.0;
}

// a *= sqrt(1/ *den)  (normalise by a device-side squared norm)
__global__ void k_normalize(double* a, const double* sq, size_t n) {
  const double f = 1.0 / sqrt(*sq);
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) a[i] *= f;
}

// D_i(point) from the bands: diagonal of sum_P C_P (x) F_P (A has a zero diagonal)
template <int DIM>
__device__ __forceinline__ double diag_at(const OpParams& op, int p, size_t gidx) {
  const int m = op.m;
  const int W = 2 * p + 1;
  const size_t ns = DIM == 2 ? (size_t)m * m : (size_t)m * m * m;
  const int i = (int)(gidx / ns);   // component (0 for the scalar system)
  size_t f = gidx % ns;
  int k[3] = {0, 0, 0};
#pragma unroll
  for (int l = DIM - 1; l >= 0; --l) { k[l] = (int)(f % m); f /= m; }
  double Mv[3], Sv[3];
#pragma unroll
  for (int l = 0; l < DIM; ++l) {
    Mv[l] = __ldg(op.bM + (size_t)k[l] * W + p);
    Sv[l] = __ldg(op.bS + (size_t)k[l] * W + p);
  }
  if (DIM == 2)
    return op.c.mass[i][i] * Mv[0] * Mv[1] + op.c.S[0][i][i] * Sv[0] * Mv[1] + op.c.S[1][i][i] * Mv[0] * Sv[1];
  return op.c.mass[i][i] * Mv[0] * Mv[1] * Mv[2] + op.c.S[0][i][i] * Sv[0] * Mv[1] * Mv[2] +
         op.c.S[1][i][i] * Mv[0] * Sv[1] * Mv[2] + op.c.S[2][i][i] * Mv[0] * Mv[1] * Sv[2];
}

template <int DIM>
__global__ void k_scale_dinv(OpParams op, int p, const double* __restrict__ b, double* __restrict__ x, double omega,
                             size_t n) {
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS)
    x[i] = omega * b[i] / diag_at<DIM>(op, p, i);
}

template <int DIM>
__global__ void k_dvdot(OpParams op, int p, const double* __restrict__ v, size_t n, double* partial) {
  __shared__ double red[VBS / 32];
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS)
    s = fma(diag_at<DIM>(op, p, i) * v[i], v[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// counter-based start vector of the power iteration (reading R4; inputs/generators.py):
// v[k] = (((k+1) * 0x9E3779B97F4A7C15 mod 2^64) >> 11) * 2^-53 - 0.5
__global__ void k_hash_vector(double* v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) {
    const unsigned long long h = (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ULL;
    v[i] = (double)(h >> 11) * 0x1.0p-53 - 0.5;
  }
}

// alpha = rz/pq;  x += alpha p;  r -= alpha q;  partial ||r||^2
__global__ void k_pcg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ q, size_t n, const double* rz, const double* pq,
                         double* partial) {
  __shared__ double red[VBS / 32];
  const double alpha = *rz / *pq;
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_axpy1(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) b[i] += a[i];
}

// beta = rz_new/rz_old;  p = z + beta p
__global__ void k_pcg_p(double* __restrict__ p, const double* __restrict__ z, size_t n, const double* rzn,
                        const double* rzo) {
  const double beta = *rzn / *rzo;
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS)
    p[i] = fma(beta, p[i], z[i]);
}

#define LAUNCH_TAIL() \
  IGACD_LAUNCH_CHECK(); \
  count_launch(h)

void launch_dot(Handle& h, const double* a, const double* b, size_t n, double* partial, cudaStream_t s) {
  k_dot<<<vec_ctas(n), VBS, 0, s>>>(a, b, n, partial);
  LAUNCH_TAIL();
}
void launch_finalize(Handle& h, const double* partial, int np, double* dst, cudaStream_t s) {
  k_finalize<<<1, VBS, 0, s>>>(partial, np, dst);
  LAUNCH_TAIL();
}
void launch_copy(Handle& h, const double* a, double* b, size_t n, cudaStream_t s) {
  k_copy<<<vec_ctas(n), VBS, 0, s>>>(a, b, n);
  LAUNCH_TAIL();
}
void launch_axpy_inplace(Handle& h, const double* a, double* b, size_t n, cudaStream_t s) {
  k_axpy1<<<vec_ctas(n), VBS, 0, s>>>(a, b, n);
  LAUNCH_TAIL();
}
void launch_zero(Handle& h, double* a, size_t n, cudaStream_t s) {
  k_zero<<<vec_ctas(n), VBS, 0, s>>>(a, n);
  LAUNCH_TAIL();
}
void launch_scale(Handle& h, double* a, const double* sq, const double*, size_t n, cudaStream_t s) {
  k_normalize<<<vec_ctas(n), VBS, 0, s>>>(a, sq, n);
  LAUNCH_TAIL();
}
void launch_scale_dinv(Handle& h, int sy, int level, const double* b, double* x, double omega, cudaStream_t s) {
  const SysLevel& L = h.sys[sy].lv[level];
  if (h.dim == 2) k_scale_dinv<2><<<vec_ctas(L.ndof), VBS, 0, s>>>(L.op, h.p, b, x, omega, L.ndof);
  else k_scale_dinv<3><<<vec_ctas(L.ndof), VBS, 0, s>>>(L.op, h.p, b, x, omega, L.ndof);
  LAUNCH_TAIL();
}
void launch_dvdot(Handle& h, int sy, int level, const double* v, double* partial, cudaStream_t s) {
  const SysLevel& L = h.sys[sy].lv[level];
  if (h.dim == 2) k_dvdot<2><<<vec_ctas(L.ndof), VBS, 0, s>>>(L.op, h.p, v, L.ndof, partial);
  else k_dvdot<3><<<vec_ctas(L.ndof), VBS, 0, s>>>(L.op, h.p, v, L.ndof, partial);
  LAUNCH_TAIL();
}
void launch_hash_vector(Handle& h, double* v, size_t n, cudaStream_t s) {
  k_hash_vector<<<vec_ctas(n), VBS, 0, s>>>(v, n);
  LAUNCH_TAIL();
}
void launch_pcg_update_xr(Handle& h, double* x, double* r, const double* p, const double* q, size_t n,
                          const double* rz, const double* pq, double* partial, cudaStream_t s) {
  k_pcg_xr<<<vec_ctas(n), VBS, 0, s>>>(x, r, p, q, n, rz, pq, partial);
  LAUNCH_TAIL();
}
void launch_pcg_update_p(Handle& h, double* p, const double* z, size_t n, const double* rzn, const double* rzo,
                         cudaStream_t s) {
  k_pcg_p<<<vec_ctas(n), VBS, 0, s>>>(p, z, n, rzn, rzo);
  LAUNCH_TAIL();
}


// ---- GMRES (Arnoldi) kernels: up to MDOT vectors per launch -----------------------------------
struct VecSet {
  const double* v[MDOT];
};

// partial[j * np + cta] = sum_i w_i v_j,i  (j < nv), fixed-order block reductions
__global__ void k_mdot(const double* __restrict__ w, VecSet V, int nv, size_t n, double* partial, int np) {
  __shared__ double red[VBS / 32];
  double s[MDOT];
#pragma unroll
  for (int j = 0; j < MDOT; ++j) s[j] = 0.0;
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) {
    const double wi = w[i];
#pragma unroll
    for (int j = 0; j < MDOT; ++j)
      if (j < nv) s[j] = fma(wi, V.v[j][i], s[j]);
  }
#pragma unroll
  for (int j = 0; j < MDOT; ++j) {
    if (j >= nv) break;
    const double t = block_sum(s[j], red);
    if (threadIdx.x == 0) partial[j * np + blockIdx.x] = t;
    __syncthreads();
  }
}

// dst[j] = sum_c partial[j * np + c], one block per j
__global__ void k_finalize_multi(const double* partial, int np, double* dst) {
  __shared__ double red[VBS / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += VBS) s += partial[blockIdx.x * np + i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) dst[blockIdx.x] = s;
}

// w += sign * sum_j c_j v_j  (c on the device)
__global__ void k_maxpy(double* __restrict__ w, VecSet V, int nv, const double* __restrict__ c, double sign,
                        size_t n) {
  double cj[MDOT];
#pragma unroll
  for (int j = 0; j < MDOT; ++j) cj[j] = j < nv ? sign * c[j] : 0.0;
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) {
    double a = w[i];
#pragma unroll
    for (int j = 0; j < MDOT; ++j)
      if (j < nv) a = fma(cj[j], V.v[j][i], a);
    w[i] = a;
  }
}

__global__ void k_scal(double* a, double f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)VBS + threadIdx.x; i < n; i += (size_t)gridDim.x * VBS) a[i] *= f;
}

void launch_mdot(Handle& h, const double* w, const double* const* V, int nv, size_t n, double* partial, double* dst,
                 cudaStream_t s) {
  const int np = vec_ctas(n);
  for (int g = 0; g < nv; g += MDOT) {
    VecSet vs{};
    const int k = std::min(MDOT, nv - g);
    for (int j = 0; j < k; ++j) vs.v[j] = V[g + j];
    k_mdot<<<np, VBS, 0, s>>>(w, vs, k, n, partial, np);
    LAUNCH_TAIL();
    k_finalize_multi<<<k, VBS, 0, s>>>(partial, np, dst + g);
    LAUNCH_TAIL();
  }
}

void launch_maxpy(Handle& h, double* w, const double* const* V, int nv, const double* c, double sign, size_t n,
                  cudaStream_t s) {
  for (int g = 0; g < nv; g += MDOT) {
    VecSet vs{};
    const int k = std::min(MDOT, nv - g);
    for (int j = 0; j < k; ++j) vs.v[j] = V[g + j];
    k_maxpy<<<vec_ctas(n), VBS, 0, s>>>(w, vs, k, c + g, sign, n);
    LAUNCH_TAIL();
  }
}

void launch_scal(Handle& h, double* a, double f, size_t n, cudaStream_t s) {
  k_scal<<<vec_ctas(n), VBS, 0, s>>>(a, f, n);
  LAUNCH_TAIL();
}

}  // namespace igacd
