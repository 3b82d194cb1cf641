// Problem setup and the shifted-Laplacian Galerkin multigrid hierarchy.
//
// Setup arithmetic that the reference does on the host (mass, shifted
// centre, Jacobi diagonal inverse, banded LU of the coarsest operator) is
// restated here with std::complex<double> in the reference's evaluation
// order, so these arrays are bitwise equal to the reference's; the Galerkin
// planes are formed on the GPU in the reference's summation order (exact
// power-of-two weights), so they are bitwise equal too (tests pin this).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include <cstdlib>
#include <type_traits>

#include "solver.hpp"
#include "profile.hpp"

namespace hz {

// ------------------------------------------------------------------ Problem
// Compact 27-point weights (scripts/design_27pt.py: least-squares fit of the
// plane-wave phase velocity over directions and 4-12 points per wavelength,
// all weights nonnegative; max phase-velocity error 1.1e-3 at 10 ppw against
// 1.6e-2 for the 7-point stencil). Laplacian: a1 faces / a2 edges / a3
// corners; mass: c0 centre, c1 faces, c2 edges, c3 corners.
namespace {
constexpr double k27_a1 = 0.30896924112207297, k27_a2 = 0.5974547869846899;
constexpr double k27_c1 = 0.49495786061914238, k27_c2 = 0.023557529253244218, k27_c3 = 2.4579791982563098e-08;
}  // namespace
void weights27(double h, double* lap, double* mu) {
  const double a3 = 1.0 - k27_a1 - k27_a2, c0 = 1.0 - k27_c1 - k27_c2 - k27_c3, ih2 = 1.0 / (h * h);
  lap[1] = k27_a1 * ih2;
  lap[2] = k27_a2 * ih2 / 4.0;
  lap[3] = a3 * ih2 / 4.0;
  lap[0] = -(6.0 * lap[1] + 12.0 * lap[2] + 8.0 * lap[3]);
  mu[0] = c0;
  mu[1] = k27_c1 / 6.0;
  mu[2] = k27_c2 / 12.0;
  mu[3] = k27_c3 / 8.0;
}

void Problem::weights27(double* w8) const { ::hz::weights27(h[0], w8, w8 + 4); }

void Problem::build_coef27(double shift, double2* planes, cudaStream_t s) const {
  double lap[4], mu[4];
  ::hz::weights27(h[0], lap, mu);
  launch_build27(LevelGeom(n[0], n[1], n[2], 1), lap, mu, d_mass.get(), d_m.get(), shift * omega * omega, planes, s);
}

Problem::Problem(int ndim_, const int64_t* n_, const double* h_, const double* m_, double omega_,
                 double gamma_base_, const double* ramp_, bool allow_coarse, int device_, int stencil_)
    : ndim(ndim_), omega(omega_), gamma_base(gamma_base_), device(device_), stencil(stencil_) {
  if (stencil != 7 && stencil != 27) throw HzError(kValidation, "helmholtz: stencil must be 7 or 27");
  if (stencil == 27) {
    if (ndim_ != 3) throw HzError(kValidation, "helmholtz: the compact 27-point stencil is 3D only");
    if (!(h_[0] == h_[1] && h_[1] == h_[2]))
      throw HzError(kValidation, "helmholtz: the compact 27-point stencil needs uniform spacing");
  }
  // RegularGrid ctor (src/grid.cpp:10-27)
  if (ndim != 2 && ndim != 3) throw HzError(kValidation, "grid: ndim must be 2 or 3");
  for (int a = 0; a < 3; ++a) {
    n[a] = n_[a];
    h[a] = h_[a];
  }
  if (ndim == 2) {
    n[2] = 1;
    h[2] = 1.0;
  }
  for (int a = 0; a < ndim; ++a) {
    if (n[a] < 3) throw HzError(kValidation, "grid: axis " + std::to_string(a) + " needs at least 3 nodes");
    if (!(h[a] > 0.0))
      throw HzError(kValidation, "grid: spacing on axis " + std::to_string(a) + " must be positive");
  }
  const int64_t nn = num_nodes();
  // element indices of a block are 32-bit (n*k checked per solve)
  if (nn >= (int64_t(1) << 31)) throw HzError(kValidation, "grid: node count overflows the index type");
  if (!m_ || !ramp_) throw HzError(kValidation, "helmholtz: null model or attenuation");
  m.assign(m_, m_ + nn);
  ramp.assign(ramp_, ramp_ + nn);
  for (double x : m)  // SlownessSquaredModel (src/model.cpp:13-19)
    if (!(x > 0.0)) throw HzError(kValidation, "model: slowness-squared values must be positive");
  // HelmholtzProblem ctor (src/helmholtz.cpp:16-38)
  if (!(omega > 0.0)) throw HzError(kValidation, "helmholtz: omega must be positive");
  const double ppw = points_per_wavelength();
  if (ppw < 10.0 - 1e-12 && !allow_coarse)
    throw HzError(kValidation, "helmholtz: " + std::to_string(ppw) +
                                   " grid points per wavelength (need >= 10); pass allow_coarse to override");
  center_lap = 0.0;
  for (int k = 0; k < 3; ++k) {
    inv_h2[k] = (n[k] > 1) ? 1.0 / (h[k] * h[k]) : 0.0;
    center_lap -= 2.0 * inv_h2[k];
  }
  mass.resize(nn);
  gamma_factor.resize(nn);
  std::vector<cplx> center(nn);
  for (int64_t i = 0; i < nn; ++i) {
    const double gam = gamma_base + omega * ramp[i];  // AttenuationField::gamma_at
    gamma_factor[i] = cplx(1.0, -gam / omega);
    mass[i] = omega * omega * gamma_factor[i] * m[i];
    center[i] = center_lap + mass[i];  // apply_block centre (src/helmholtz.cpp:84)
  }
  DeviceGuard dg(device);
  d_center.alloc(nn);
  d_gf.alloc(nn);
  HZ_CUDA(cudaMemcpy(d_center.get(), center.data(), nn * sizeof(double2), cudaMemcpyHostToDevice));
  HZ_CUDA(cudaMemcpy(d_gf.get(), gamma_factor.data(), nn * sizeof(double2), cudaMemcpyHostToDevice));
  if (stencil == 27) {
    d_mass.alloc(nn);
    d_m.alloc(nn);
    HZ_CUDA(cudaMemcpy(d_mass.get(), mass.data(), nn * sizeof(double2), cudaMemcpyHostToDevice));
    HZ_CUDA(cudaMemcpy(d_m.get(), m.data(), nn * sizeof(double), cudaMemcpyHostToDevice));
    HZ_CUDA(cudaDeviceSynchronize());
  }
}

double Problem::min_h() const {
  double mh = h[0];
  for (int a = 1; a < ndim; ++a) mh = std::min(mh, h[a]);
  return mh;
}

double Problem::points_per_wavelength() const {
  const double smax = std::sqrt(*std::max_element(m.begin(), m.end()));
  return 2.0 * M_PI / (omega * smax * min_h());
}

std::vector<cplx> Problem::shifted_center(double shift) const {
  const int64_t nn = num_nodes();
  std::vector<cplx> c(nn);
  const cplx shift_term(0.0, -shift * omega * omega);
  for (int64_t i = 0; i < nn; ++i) c[i] = center_lap + mass[i] + shift_term * m[i];
  return c;
}

LevelOp<double> Problem::fine_op(int k) const {
  LevelOp<double> op;
  op.kind = stencil == 27 ? kFine27 : kFine;
  op.ndim = ndim;
  op.g = LevelGeom(n[0], n[1], n[2], k);
  op.center = stencil == 27 ? d_mass.get() : d_center.get();
  if (stencil == 27) weights27(op.w27);
  for (int a = 0; a < 3; ++a) op.w[a] = inv_h2[a];
  return op;
}

// ------------------------------------------------------------------ helpers
namespace {

// coarsen_dims (src/multigrid.cpp:11-25)
std::array<int64_t, 3> coarsen(const std::array<int64_t, 3>& d) {
  std::array<int64_t, 3> out = d;
  for (int k = 0; k < 3; ++k) {
    if (d[k] <= 1) continue;
    if (d[k] % 2 == 0)
      throw HzError(kValidation, "multigrid: axis " + std::to_string(k) + " has even node count " +
                                     std::to_string(d[k]) + "; not coarsenable");
    const int64_t nc = (d[k] - 1) / 2 + 1;
    if (nc < 3)
      throw HzError(kValidation, "multigrid: axis " + std::to_string(k) +
                                     " too small to coarsen (coarse count " + std::to_string(nc) + ")");
    out[k] = nc;
  }
  return out;
}

std::vector<cplx> invert_diag(const std::vector<cplx>& d) {
  std::vector<cplx> inv(d.size());
  for (size_t i = 0; i < d.size(); ++i) {
    if (d[i] == cplx{}) throw HzError(kFactorization, "multigrid: zero diagonal entry");
    inv[i] = cplx{1} / d[i];
  }
  return inv;
}

// BandedLU::factor / factor_inplace restated (inc/dense.hpp:179-216,
// src/dense.cpp:9-37): gbtrf-style row pivoting within kl subdiagonals.
struct BandedFactor {
  int64_t n = 0, kl = 0, ku = 0, ld = 0;
  std::vector<cplx> ab;
  std::vector<int64_t> piv;
  cplx& at(int64_t i, int64_t j) { return ab[(kl + ku + i - j) + j * ld]; }
  void factor() {
    for (int64_t k = 0; k < n; ++k) {
      const int64_t imax = std::min(n - 1, k + kl);
      int64_t p = k;
      double best = std::norm(at(k, k));
      for (int64_t i = k + 1; i <= imax; ++i) {
        const double v = std::norm(at(i, k));
        if (v > best) {
          best = v;
          p = i;
        }
      }
      if (!(best > 0.0)) throw HzError(kFactorization, "banded LU: singular pivot at " + std::to_string(k));
      piv[k] = p;
      const int64_t jmax = std::min(n - 1, k + kl + ku);
      if (p != k)
        for (int64_t j = k; j <= jmax; ++j) std::swap(at(k, j), at(p, j));
      const cplx inv = cplx{1} / at(k, k);
      for (int64_t i = k + 1; i <= imax; ++i) {
        const cplx l = at(i, k) * inv;
        at(i, k) = l;
        if (l != cplx{})
          for (int64_t j = k + 1; j <= jmax; ++j) at(i, j) -= l * at(k, j);
      }
    }
  }
};

}  // namespace

// ------------------------------------------------------------------ build
template <>
std::unique_ptr<Hierarchy<double>> Hierarchy<double>::build(const Problem& p, int nlevels,
                                                            double shift, cudaStream_t s) {
  if (nlevels < 2) throw HzError(kValidation, "multigrid: need at least 2 levels");
  auto H = std::make_unique<Hierarchy<double>>();
  H->ndim_ = p.ndim;
  std::vector<std::array<int64_t, 3>> dims(nlevels);
  dims[0] = p.n;
  for (int l = 0; l + 1 < nlevels; ++l) dims[l + 1] = coarsen(dims[l]);
  H->levels_.resize(nlevels);
  // level 0: shifted fine operator (to_csr(shift), src/helmholtz.cpp:102-122)
  if (p.stencil == 27) {  // compact 27-point fine operator with gamma + shift * omega
    auto& L0 = H->levels_[0];
    L0.dims = dims[0];
    L0.kind = kFine27;
    const int64_t nn = p.num_nodes();
    p.weights27(L0.w27);
    L0.center.alloc(nn);
    L0.inv_diag.alloc(nn);
    launch_shift_mass(nn, p.d_mass.get(), p.d_m.get(), shift * p.omega * p.omega, L0.center.get(), s);
    launch_inv_centre27(nn, L0.w27[0], L0.w27[4], L0.center.get(), L0.inv_diag.get(), s);
    HZ_CUDA(cudaStreamSynchronize(s));
  } else {
    auto& L0 = H->levels_[0];
    L0.dims = dims[0];
    L0.kind = kFine;
    for (int a = 0; a < 3; ++a) L0.w[a] = p.inv_h2[a];
    const auto c = p.shifted_center(shift);
    const auto inv = invert_diag(c);
    L0.center.alloc(c.size());
    L0.inv_diag.alloc(c.size());
    L0.center.upload(c.data(), c.size(), s);
    L0.inv_diag.upload(inv.data(), inv.size(), s);
    HZ_CUDA(cudaStreamSynchronize(s));
  }
  const int S = p.ndim == 3 ? 27 : 9;
  const int sc = p.ndim == 3 ? 13 : 4;  // centre plane
  for (int l = 1; l < nlevels; ++l) {
    auto& L = H->levels_[l];
    L.dims = dims[l];
    L.kind = kStencil;
    const int64_t nc = L.nodes();
    L.coef.alloc(size_t(S) * nc);
    LevelGeom gc(dims[l][0], dims[l][1], dims[l][2], 1);
    if (l == 1 && p.stencil == 27) {
      // the Galerkin product reads coefficient planes: materialise the
      // shifted 27-point operator's (identical couplings) for this step only
      DevBuf<double2> planes(size_t(27) * p.num_nodes());
      p.build_coef27(shift, planes.get(), s);
      LevelOp<double> f = H->op(0, 1);
      f.kind = kStencil;
      f.coef = planes.get();
      launch_galerkin(f, gc, L.coef.get(), s);
      HZ_CUDA(cudaStreamSynchronize(s));
    } else {
      launch_galerkin(H->op(l - 1, 1), gc, L.coef.get(), s);
    }
    std::vector<cplx> diag(nc);
    HZ_CUDA(cudaMemcpyAsync(diag.data(), L.coef.get() + size_t(sc) * nc, nc * sizeof(double2),
                            cudaMemcpyDeviceToHost, s));
    HZ_CUDA(cudaStreamSynchronize(s));
    const auto inv = invert_diag(diag);
    L.inv_diag.alloc(nc);
    L.inv_diag.upload(inv.data(), nc, s);
  }
  // coarsest, large 3D: block-tridiagonal plane factorisation on the device
  // (HZ_COARSE=dense|bt overrides the size rule)
  {
    const auto& Lc = H->levels_.back();
    const int64_t nc = Lc.nodes();
    const char* mode = std::getenv("HZ_COARSE");
    bool bt = p.ndim == 3 && nc > 6000;
    if (mode && std::string(mode) == "bt") bt = p.ndim == 3;
    if (mode && std::string(mode) == "dense") bt = false;
    if (bt) {
      const LevelGeom gc(Lc.dims[0], Lc.dims[1], Lc.dims[2], 1);
      // Moderate coarse grids (config 3: 33x33x17): the explicit inverse,
      // formed once from the plane factors (A X = I in 64-column chunks), makes
      // every coarse solve one streaming product instead of 2 n2 - 1 dependent
      // plane steps (HZ_BT_INVERSE_MAX nodes; 0 keeps the plane solve)
      const char* inv_env = std::getenv("HZ_BT_INVERSE_MAX");
      const int64_t inv_max = inv_env ? int64_t(std::atoll(inv_env)) : int64_t(0);
      // the plane solve sweeps along the longest axis (coarse_bt.cu)
      if (nc > inv_max) bt_sweep_perm(Lc.dims.data(), H->bt_perm_);
      H->bt_ = true;
      if (H->bt_permuted()) {
        const LevelGeom gT = bt_permuted_geom(gc, H->bt_perm_);
        const int64_t m = int64_t(gT.n0) * gT.n1;
        const size_t sz = size_t(gT.n2) * m * inv_ld(m);
        H->bt_coef_.alloc(size_t(27) * nc);
        bt_permute_coef(gc, H->bt_perm_, Lc.coef.get(), H->bt_coef_.get(), s);
        H->bt_ET_.alloc(sz);
        H->bt_FT_.alloc(sz);
        bt_factor(gT, H->bt_coef_.get(), H->bt_ET_.get(), H->bt_FT_.get(), s);
        return H;
      }
      const int64_t m = Lc.dims[0] * Lc.dims[1];
      const size_t sz = size_t(Lc.dims[2]) * m * inv_ld(m);
      H->bt_ET_.alloc(sz);
      H->bt_FT_.alloc(sz);
      bt_factor(gc, Lc.coef.get(), H->bt_ET_.get(), H->bt_FT_.get(), s);
      if (nc <= inv_max) {
        H->ainvT_ = bt_explicit_inverse(gc, Lc.coef.get(), H->bt_ET_.get(), H->bt_FT_.get(), s);
        H->bt_ = false;
        H->bt_ET_ = DevBuf<double2>();
        H->bt_FT_ = DevBuf<double2>();
      }
      return H;
    }
  }
  // coarsest: banded LU over the stencil profile, then explicit inverse
  {
    const auto& Lc = H->levels_.back();
    const int64_t nc = Lc.nodes();
    const int64_t n0 = Lc.dims[0], n1 = Lc.dims[1];
    const int64_t band = p.ndim == 3 ? n0 * n1 + n0 + 1 : n0 + 1;
    H->band_ = band;
    std::vector<cplx> coef(size_t(S) * nc);
    HZ_CUDA(cudaMemcpyAsync(coef.data(), Lc.coef.get(), coef.size() * sizeof(double2),
                            cudaMemcpyDeviceToHost, s));
    HZ_CUDA(cudaStreamSynchronize(s));
    BandedFactor f;
    f.n = nc;
    f.kl = f.ku = band;
    f.ld = 2 * f.kl + f.ku + 1;
    f.ab.assign(size_t(f.ld) * nc, cplx{});
    f.piv.assign(nc, 0);
    const int64_t n2 = Lc.dims[2];
    for (int64_t kz = 0; kz < n2; ++kz)
      for (int64_t j = 0; j < n1; ++j)
        for (int64_t i = 0; i < n0; ++i) {
          const int64_t r = i + n0 * (j + n1 * kz);
          for (int dz = (p.ndim == 3 ? -1 : 0); dz <= (p.ndim == 3 ? 1 : 0); ++dz)
            for (int dy = -1; dy <= 1; ++dy)
              for (int dx = -1; dx <= 1; ++dx) {
                const int64_t ii = i + dx, jj = j + dy, kk = kz + dz;
                if (ii < 0 || ii >= n0 || jj < 0 || jj >= n1 || kk < 0 || kk >= n2) continue;
                const int sidx = (p.ndim == 3 ? (dz + 1) * 9 : 0) + (dy + 1) * 3 + (dx + 1);
                f.at(r, ii + n0 * (jj + n1 * kk)) += coef[size_t(sidx) * nc + r];
              }
        }
    f.factor();
    DevBuf<double2> dab(f.ab.size());
    DevBuf<int64_t> dpiv(nc);
    dab.upload(f.ab.data(), f.ab.size(), s);
    dpiv.upload(f.piv.data(), nc, s);
    H->ainvT_.alloc(size_t(nc) * inv_ld(nc));
    launch_banded_inverse(nc, f.kl, f.ku, f.ld, dab.get(), dpiv.get(), H->ainvT_.get(), s);
    HZ_CUDA(cudaStreamSynchronize(s));
  }
  return H;
}

// DenseLuSmall (src/helmholtz_solver.cpp:11-17): the reference factors the
// dense unshifted operator with partial pivoting. Rows below the band are
// zero in every pivot column, so the banded pivoted LU takes the same pivots
// and produces the same factors; the solve is the explicit inverse.
DevBuf<double2> dense_inverse(const Problem& p, cudaStream_t s) {
  const int64_t nn = p.num_nodes();
  const int64_t n0 = p.n[0], n1 = p.n[1], n2 = p.n[2];
  const int64_t band = p.ndim == 3 ? n0 * n1 : n0;
  BandedFactor f;
  f.n = nn;
  f.kl = f.ku = band;
  f.ld = 2 * f.kl + f.ku + 1;
  f.ab.assign(size_t(f.ld) * nn, cplx{});
  f.piv.assign(nn, 0);
  for (int64_t kz = 0; kz < n2; ++kz)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t i = 0; i < n0; ++i) {
        const int64_t r = i + n0 * (j + n1 * kz);
        f.at(r, r) += p.center_lap + p.mass[r];
        if (i > 0) f.at(r, r - 1) += p.inv_h2[0];
        if (i + 1 < n0) f.at(r, r + 1) += p.inv_h2[0];
        if (j > 0) f.at(r, r - n0) += p.inv_h2[1];
        if (j + 1 < n1) f.at(r, r + n0) += p.inv_h2[1];
        if (kz > 0) f.at(r, r - n0 * n1) += p.inv_h2[2];
        if (kz + 1 < n2) f.at(r, r + n0 * n1) += p.inv_h2[2];
      }
  f.factor();
  DevBuf<double2> dab(f.ab.size());
  DevBuf<int64_t> dpiv(nn);
  dab.upload(f.ab.data(), f.ab.size(), s);
  dpiv.upload(f.piv.data(), nn, s);
  DevBuf<double2> out(size_t(nn) * inv_ld(nn));
  launch_banded_inverse(nn, f.kl, f.ku, f.ld, dab.get(), dpiv.get(), out.get(), s);
  HZ_CUDA(cudaStreamSynchronize(s));
  return out;
}

template <>
std::unique_ptr<Hierarchy<float>> Hierarchy<float>::rounded(const Hierarchy<double>& h64,
                                                            cudaStream_t s) {
  auto H = std::make_unique<Hierarchy<float>>();
  H->ndim_ = h64.ndim_;
  H->band_ = h64.band_;
  H->levels_.resize(h64.levels_.size());
  for (size_t l = 0; l < h64.levels_.size(); ++l) {
    const auto& a = h64.levels_[l];
    auto& b = H->levels_[l];
    b.dims = a.dims;
    b.kind = a.kind;
    for (int q = 0; q < 3; ++q) b.w[q] = float(a.w[q]);
    for (int q = 0; q < 8; ++q) b.w27[q] = float(a.w27[q]);
    auto cast = [&](const DevBuf<double2>& src, DevBuf<float2>& dst) {
      if (!src.size()) return;
      dst.alloc(src.size());
      launch_cast<float2, double2>(int64_t(src.size()), src.get(), dst.get(), s);
    };
    cast(a.center, b.center);
    cast(a.coef, b.coef);
    cast(a.inv_diag, b.inv_diag);
    if (b.kind == kStencil && h64.ndim_ == 2 && b.coef.size()) {
      // 2D Galerkin level: (9 coefficients, D^{-1}) per node in one 80-byte
      // record, so a grid row is one 16-byte-aligned bulk copy (stencil9_k8)
      const size_t nn = b.inv_diag.size();
      b.cd.alloc(10 * nn);
      for (int q = 0; q < 10; ++q) {
        const float2* src = q < 9 ? b.coef.get() + size_t(q) * nn : b.inv_diag.get();
        HZ_CUDA(cudaMemcpy2DAsync(b.cd.get() + q, 10 * sizeof(float2), src, sizeof(float2), sizeof(float2), nn,
                                  cudaMemcpyDeviceToDevice, s));
      }
    }
    if (b.kind == kStencil && h64.ndim_ == 3 && b.coef.size() && b.nodes() >= galerkin3d_min_nodes()) {
      // large 3D Galerkin level: the 27 coefficients (and D^{-1}) per node as
      // three 80-byte record groups for the plane-streaming kernel (galerkin3d.cu)
      b.cd.alloc(size_t(30) * b.nodes());
      launch_galerkin3d_records(b.nodes(), b.coef.get(), b.inv_diag.get(), b.cd.get(), s);
    }
    if ((b.kind == kFine || b.kind == kFine27) && b.center.size()) {
      // (centre, D^{-1}) per node in one 16-byte record: a row of the fine
      // grid is then one 16-byte-aligned bulk copy whatever n0's parity
      const size_t nn = b.center.size();
      b.cd.alloc(2 * nn);
      HZ_CUDA(cudaMemcpy2DAsync(b.cd.get(), 2 * sizeof(float2), b.center.get(), sizeof(float2), sizeof(float2), nn,
                                cudaMemcpyDeviceToDevice, s));
      HZ_CUDA(cudaMemcpy2DAsync(b.cd.get() + 1, 2 * sizeof(float2), b.inv_diag.get(), sizeof(float2),
                                sizeof(float2), nn, cudaMemcpyDeviceToDevice, s));
    }
  }
  auto cast_all = [&](const DevBuf<double2>& src, DevBuf<float2>& dst) {
    if (!src.size()) return;
    dst.alloc(src.size());
    launch_cast<float2, double2>(int64_t(src.size()), src.get(), dst.get(), s);
  };
  cast_all(h64.ainvT_, H->ainvT_);
  H->bt_ = h64.bt_;
  for (int a = 0; a < 3; ++a) H->bt_perm_[a] = h64.bt_perm_[a];
  cast_all(h64.bt_coef_, H->bt_coef_);
  cast_all(h64.bt_ET_, H->bt_ET_);
  cast_all(h64.bt_FT_, H->bt_FT_);
  HZ_CUDA(cudaStreamSynchronize(s));
  return H;
}

template <class T>
LevelOp<T> Hierarchy<T>::op(int l, int k) const {
  const auto& L = levels_[l];
  LevelOp<T> o;
  o.kind = L.kind;
  o.ndim = ndim_;
  o.g = LevelGeom(L.dims[0], L.dims[1], L.dims[2], k);
  o.center = L.center.get();
  o.coef = L.coef.get();
  o.inv_diag = L.inv_diag.get();
  o.cd = L.cd.get();
  for (int a = 0; a < 3; ++a) o.w[a] = L.w[a];
  for (int a = 0; a < 8; ++a) o.w27[a] = L.w27[a];
  o.level = l;
  return o;
}

template <class T>
void Hierarchy<T>::download_level(int l, std::vector<cplx>& out) const {
  const auto& L = levels_[l];
  const DevBuf<V>& src = L.kind == kStencil ? L.coef : L.center;
  std::vector<V> tmp(src.size());
  HZ_CUDA(cudaMemcpy(tmp.data(), src.get(), src.bytes(), cudaMemcpyDeviceToHost));
  out.resize(tmp.size());
  for (size_t i = 0; i < tmp.size(); ++i) out[i] = cplx(tmp[i].x, tmp[i].y);
}

template <class T>
std::unique_ptr<Hierarchy<T>> Hierarchy<T>::replica(int device, cudaStream_t s) const {
  DeviceGuard g(device);
  auto H = std::make_unique<Hierarchy<T>>();
  H->ndim_ = ndim_;
  H->band_ = band_;
  H->levels_.resize(levels_.size());
  auto copy = [&](const DevBuf<V>& src, DevBuf<V>& dst) {
    if (!src.size()) return;
    dst.alloc(src.size());
    int sdev = 0;
    cudaPointerAttributes a{};
    HZ_CUDA(cudaPointerGetAttributes(&a, src.get()));
    sdev = a.device;
    HZ_CUDA(cudaMemcpyPeerAsync(dst.get(), device, src.get(), sdev, src.bytes(), s));
  };
  for (size_t l = 0; l < levels_.size(); ++l) {
    const auto& A = levels_[l];
    auto& B = H->levels_[l];
    B.dims = A.dims;
    B.kind = A.kind;
    for (int a = 0; a < 3; ++a) B.w[a] = A.w[a];
    copy(A.center, B.center);
    copy(A.coef, B.coef);
    copy(A.inv_diag, B.inv_diag);
  }
  HZ_CUDA(cudaStreamSynchronize(s));
  return H;
}

// A view of the same operators with its own cycle workspace: the hierarchy is
// immutable after build and only the workspaces are written by a cycle
// (inc/multigrid.hpp:37-39: distinct blocks may cycle concurrently), so
// views on different streams run concurrently. The view must not outlive
// this hierarchy.
template <class T>
std::unique_ptr<Hierarchy<T>> Hierarchy<T>::share() const {
  if (sl_) throw HzError(kState, "hierarchy views of a slab-decomposed hierarchy are not supported");
  auto H = std::make_unique<Hierarchy<T>>();
  H->ndim_ = ndim_;
  H->band_ = band_;
  H->bt_ = bt_;
  auto alias = [](const auto& src, auto& dst) {
    if (src.size()) dst.adopt(std::shared_ptr<void>(static_cast<void*>(src.get()), [](void*) {}), src.size());
  };
  H->levels_.resize(levels_.size());
  for (size_t l = 0; l < levels_.size(); ++l) {
    const auto& A = levels_[l];
    auto& B = H->levels_[l];
    B.dims = A.dims;
    B.kind = A.kind;
    for (int a = 0; a < 3; ++a) B.w[a] = A.w[a];
    for (int a = 0; a < 8; ++a) B.w27[a] = A.w27[a];
    alias(A.center, B.center);
    alias(A.coef, B.coef);
    alias(A.inv_diag, B.inv_diag);
    alias(A.cd, B.cd);
  }
  alias(ainvT_, H->ainvT_);
  for (int a = 0; a < 3; ++a) H->bt_perm_[a] = bt_perm_[a];
  alias(bt_coef_, H->bt_coef_);
  alias(bt_ET_, H->bt_ET_);
  alias(bt_FT_, H->bt_FT_);
  return H;
}

template <class T>
void Hierarchy<T>::attach_slabs(const Slabs* sl, std::vector<const Hierarchy<T>*> reps) {
  if (sl && sl->levels() != num_levels()) throw HzError(kValidation, "slabs: level count mismatch");
  if (sl && int(reps.size()) != sl->parts()) throw HzError(kValidation, "slabs: one hierarchy per part");
  sl_ = sl;
  reps_ = std::move(reps);
  for (auto& r : reps_)
    if (!r) r = this;
  ws_k_ = 0;  // workspaces are re-laid out over the slabs
}

template <class T>
template <class F>
void Hierarchy<T>::on_level(int l, int k, cudaStream_t s, F&& f) {
  if (!slab_level(l)) {
    f(op(l, k), s, int64_t(0), levels_[l].nodes());
    return;
  }
  sl_->each(l, [&](int p, int64_t r0, int64_t nr, cudaStream_t st) {
    LevelOp<T> o = reps_[p]->op(l, k);
    o.g = o.g.slab(sl_->z0(l, p), sl_->z1(l, p));
    f(o, st, r0, nr);
  });
}

// ------------------------------------------------------------------ cycle
// the fused finest-level visit (fused.cu) covers V/W/K cycles with 2 pre- and
// 2 post-sweeps on a single-domain 2D fine grid
template <class T>
bool Hierarchy<T>::fused_level0(const CycleSpec& spec, int k) const {
  return num_levels() > 1 && !sl_ && spec.pre == 2 && spec.post == 2 && fused_fine_vcycle_ok(op(0, k));
}

template <class T>
void Hierarchy<T>::ensure_ws(int k) {
  if (ws_k_ == k) return;
  clear_graphs();  // captured cycles reference the old workspaces
  const int L = num_levels();
  wx_.resize(L);
  wt_.resize(L);
  wb_.resize(L);
  wr_.resize(L);
  for (int l = 0; l < L; ++l) {
    const size_t e = size_t(levels_[l].nodes()) * k;
    // slab levels (and the first agglomerated level, written by every
    // part's restriction) follow the slab layout
    const bool span = sl_ && l <= sl_->agg_level();
    auto get = [&](DevBuf<V>& b) {
      if (span)
        alloc_span(b, *sl_, l, k);
      else
        b.alloc(e);
    };
    if (l > 0 || std::is_same<T, float>::value) {  // level 0: cycle_cast's b32 / x
      get(wx_[l]);
      get(wb_[l]);
    }
    if (l + 1 < L) {
      get(wt_[l]);
      get(wr_[l]);
    }
  }
  const int64_t nc = coarse_n();
  if (bt_) {
    const auto& Lc = levels_.back();
    const LevelGeom gT = bt_permuted_geom(LevelGeom(Lc.dims[0], Lc.dims[1], Lc.dims[2], k), bt_perm_);
    const int64_t m = int64_t(gT.n0) * gT.n1;
    cpart_.alloc(size_t(2) * std::max(coarse_split(m, k), 1) * m * k);
    bt_r_.alloc(size_t(2) * m * k);
    bt_aux_.ensure();
    if (bt_permuted()) {
      bt_b_.alloc(size_t(nc) * k);
      bt_x_.alloc(size_t(nc) * k);
    }
  } else {
    cpart_.alloc(size_t(std::max(coarse_split(nc, k), 1)) * nc * k);
  }
  ws_k_ = k;
}

// HZ_BT_GRAPH (default 1): outside a captured cycle the plane solver's chain
// runs from its own CUDA graph (first use direct, captured on the second);
// the same kernels in the same order, so the results are bitwise those of
// the direct launches.
template <class T>
void Hierarchy<T>::coarse_solve(int k, const V* b, V* x, cudaStream_t s) {
  ensure_ws(k);
  if (!bt_) {
    launch_coarse_solve<T>(coarse_n(), k, ainvT_.get(), b, x, cpart_.get(), s);
    return;
  }
  const auto& Lc = levels_.back();
  const LevelGeom gT = bt_permuted_geom(LevelGeom(Lc.dims[0], Lc.dims[1], Lc.dims[2], k), bt_perm_);
  const double m = double(gT.n0) * gT.n1, np = double(gT.n2);
  ProfScope prof(sizeof(T) == 8 ? "coarse_bt_c128" : "coarse_bt_c64", (2.0 * np - 1.0) * m * m * sizeof(V), s,
                 8.0 * (2.0 * np - 1.0) * m * m * k);
  const char* ge = std::getenv("HZ_BT_GRAPH");
  // a stream some caller is capturing takes the launches directly (they join the caller's graph)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  HZ_CUDA(cudaStreamIsCapturing(s, &cap));
  if (sl_ || is_capturing() || cap != cudaStreamCaptureStatusNone || (ge && ge[0] == '0')) {
    coarse_solve_bt(k, b, x, s);
    return;
  }
  if (bt_graphs_.size() > 32) {  // caller-owned blocks at ever new addresses
    for (auto& kv : bt_graphs_)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    bt_graphs_.clear();
  }
  const auto key = std::make_tuple(static_cast<const void*>(b), static_cast<const void*>(x), k);
  auto it = bt_graphs_.find(key);
  if (it == bt_graphs_.end()) {  // first use: direct (function attributes, lazy state)
    coarse_solve_bt(k, b, x, s);
    bt_graphs_.emplace(key, GraphRec{});
    return;
  }
  GraphRec& g = it->second;
  if (!g.exec) {
    cudaGraph_t graph = nullptr;
    HZ_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    set_capturing(true);
    try {
      coarse_solve_bt(k, b, x, s);
    } catch (...) {
      set_capturing(false);
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    set_capturing(false);
    HZ_CUDA(cudaStreamEndCapture(s, &graph));
    size_t nn = 0;
    HZ_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    HZ_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
    g.kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      HZ_CUDA(cudaGraphNodeGetType(nd, &ty));
      if (ty == cudaGraphNodeTypeKernel) ++g.kernels;
    }
    const cudaError_t st = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    HZ_CUDA(st);
  }
  HZ_CUDA(cudaGraphLaunch(g.exec, s));
  add_launches(g.kernels);
}

template <class T>
void Hierarchy<T>::coarse_solve_bt(int k, const V* b, V* x, cudaStream_t s) {
  if (bt_) {
    const auto& Lc = levels_.back();
    const LevelGeom gc(Lc.dims[0], Lc.dims[1], Lc.dims[2], k);
    if (bt_permuted()) {
      const LevelGeom gT = bt_permuted_geom(gc, bt_perm_);
      bt_permute_vec<T>(gc, bt_perm_, k, false, b, bt_b_.get(), s);
      bt_solve<T>(gT, bt_coef_.get(), bt_ET_.get(), bt_FT_.get(), k, bt_b_.get(), bt_x_.get(), bt_r_.get(),
                  cpart_.get(), bt_aux_, s);
      bt_permute_vec<T>(gc, bt_perm_, k, true, bt_x_.get(), x, s);
      return;
    }
    bt_solve<T>(gc, Lc.coef.get(), bt_ET_.get(), bt_FT_.get(), k, b, x, bt_r_.get(), cpart_.get(), bt_aux_, s);
    return;
  }
  launch_coarse_solve<T>(coarse_n(), k, ainvT_.get(), b, x, cpart_.get(), s);
}

template <class T>
void Hierarchy<T>::cycle(const CycleSpec& spec, int k, const V* b, V* x, bool x_zero,
                         cudaStream_t s) {
  ensure_ws(k);
  cycle_rec(0, spec, k, b, x, x_zero, s);
}

// relax (src/multigrid.cpp:119-136): every sweep writes the other buffer and
// swaps, so an even number of sweeps per visit ends in the caller's x.
template <class T>
void Hierarchy<T>::relax(int l, const CycleSpec& spec, int sweeps, int k, const V* b, V*& cur,
                         V*& other, bool& cur_zero, cudaStream_t s) {
  const T wj = T(spec.jacobi_weight);
  const bool sl = slab_level(l);
  if constexpr (std::is_same<T, float>::value) {
    // both sweeps of a V(2,2) visit of a large 2D Galerkin level in one launch
    // (fused.cu); the result lands in `other`, which becomes the iterate
    if (sweeps == 2 && !sl && l > 0 &&
        launch_stencil9_pair_k8(op(l, k), wj, cur_zero ? nullptr : cur, b, other, s)) {
      std::swap(cur, other);
      cur_zero = false;
      return;
    }
  }
  for (int sw = 0; sw < sweeps; ++sw) {
    // one exchange step per sweep: a part's sweep reads its neighbours'
    // faces of cur (and must not overwrite `other` while they still read it)
    if (sl) sl_->neighbours();
    const V* c = cur;
    V* o = other;
    const bool z = cur_zero;
    on_level(l, k, s, [&](const LevelOp<T>& op_, cudaStream_t st, int64_t, int64_t) {
      if (z)
        launch_jacobi_zero<T, V>(op_, wj, b, o, st);
      else
        launch_jacobi<T>(op_, wj, c, b, o, st);
    });
    std::swap(cur, other);
    cur_zero = false;
  }
}

// cycle_rec (src/multigrid.cpp:162-199)
template <class T>
void Hierarchy<T>::cycle_rec(int l, const CycleSpec& spec, int k, const V* b, V* x, bool x_zero,
                             cudaStream_t s) {
  const int L = num_levels();
  if (l == L - 1) {
    coarse_solve(k, b, x, s);
    return;
  }
  if (l == 0 && x_zero && fused_level0(spec, k)) {
    // fused finest-level visit: pre-smoothing + residual + restriction,
    // coarse visit(s), prolongation + post-smoothing (fused.cu)
    const LevelGeom gc(levels_[1].dims[0], levels_[1].dims[1], levels_[1].dims[2], k);
    const T wj = T(spec.jacobi_weight);
    V* x2 = wt_[0].get();
    launch_fused_pre<T, V>(op(0, k), gc, wj, b, x2, wb_[1].get(), s);
    coarse_visit(0, spec, k, s);
    launch_fused_post<T, V, V>(op(0, k), gc, wj, x2, wx_[1].get(), b, x, s);
    return;
  }
  V* cur = x;
  V* other = wt_[l].get();
  bool cur_zero = x_zero;
  if constexpr (std::is_same<T, float>::value) {
    // large 2D Galerkin level visited from x = 0: both pre-sweeps, the
    // residual and its restriction in one launch (fused.cu); the iterate
    // lands in `other`, the correction and the post-sweeps follow as usual
    if (l > 0 && x_zero && !sl_ && spec.pre == 2) {
      const LevelGeom gcl(levels_[l + 1].dims[0], levels_[l + 1].dims[1], levels_[l + 1].dims[2], k);
      if (launch_stencil9_pre_k8(op(l, k), gcl, T(spec.jacobi_weight), b, other, wb_[l + 1].get(), s)) {
        std::swap(cur, other);
        coarse_visit(l, spec, k, s);
        launch_prolong_correct<T>(op(l, k).g, gcl, ndim_, wx_[l + 1].get(), cur, s);
        cur_zero = false;
        relax(l, spec, spec.post, k, b, cur, other, cur_zero, s);
        if (cur != x)
          HZ_CUDA(cudaMemcpyAsync(x, cur, size_t(levels_[l].nodes()) * k * sizeof(V), cudaMemcpyDeviceToDevice, s));
        return;
      }
    }
  }
  relax(l, spec, spec.pre, k, b, cur, other, cur_zero, s);
  const size_t rowb = size_t(k) * sizeof(V);
  coarse_correction(l, spec, k, b, cur, cur_zero, s);
  cur_zero = false;
  relax(l, spec, spec.post, k, b, cur, other, cur_zero, s);
  if (cur != x)
    on_level(l, k, s, [&](const LevelOp<T>&, cudaStream_t st, int64_t r0, int64_t nr) {
      HZ_CUDA(cudaMemcpyAsync(x + r0 * k, cur + r0 * k, size_t(nr) * rowb, cudaMemcpyDeviceToDevice, st));
    });
}

// the middle of cycle_rec: residual, restriction, coarse visit(s) and the
// prolongated correction of cur (zeroed first when cur_zero)
template <class T>
void Hierarchy<T>::coarse_correction(int l, const CycleSpec& spec, int k, const V* b, V* cur, bool cur_zero,
                                     cudaStream_t s) {
  const bool sl = slab_level(l);
  const size_t rowb = size_t(k) * sizeof(V);
  if (cur_zero)
    on_level(l, k, s, [&](const LevelOp<T>&, cudaStream_t st, int64_t r0, int64_t nr) {
      HZ_CUDA(cudaMemsetAsync(cur + r0 * k, 0, size_t(nr) * rowb, st));
    });
  const LevelGeom gc(levels_[l + 1].dims[0], levels_[l + 1].dims[1], levels_[l + 1].dims[2], k);
  if (sl) sl_->neighbours();
  on_level(l, k, s, [&](const LevelOp<T>& o, cudaStream_t st, int64_t, int64_t) {
    launch_residual<T>(o, cur, b, wr_[l].get(), st);
  });
  if (sl) {
    // every part restricts onto its planes of level l+1 (also when l+1 is
    // agglomerated: the restriction reads level-l faces of the neighbours)
    sl_->neighbours();
    sl_->each(l, [&](int p, int64_t, int64_t, cudaStream_t st) {
      const LevelGeom gf = reps_[p]->op(l, k).g;
      launch_restrict<T>(gf, gc.slab(sl_->z0(l + 1, p), sl_->z1(l + 1, p)), ndim_, wr_[l].get(),
                         wb_[l + 1].get(), st);
    });
  } else {
    launch_restrict<T>(op(l, k).g, gc, ndim_, wr_[l].get(), wb_[l + 1].get(), s);
  }
  V* ec = wx_[l + 1].get();
  // the first agglomerated level runs on part 0 alone
  const bool agg = sl && !slab_level(l + 1);
  if (agg) sl_->join();
  coarse_visit(l, spec, k, s);
  if (agg) sl_->fork();
  if (sl) sl_->neighbours();
  on_level(l, k, s, [&](const LevelOp<T>& o, cudaStream_t st, int64_t, int64_t) {
    launch_prolong_correct<T>(o.g, gc, ndim_, ec, cur, st);
  });
}

// The coarse part of the cycle (levels > l0, HZ_PRIO_FROM, default 0) runs on
// a high-priority stream forked from / joined to the caller's: its many small,
// latency-bound kernels then take SMs ahead of the large fine-level and
// Krylov kernels that concurrent solves (RHS groups, frequencies) keep queued,
// instead of waiting behind them. Same kernels, same order: bitwise equal.
// Off by default (HZ_PRIO=1 enables): no gain measured at the bench blocking
// (1.309 vs 1.323 ms per cycle, profiles/r01_prio_variants.txt).
namespace {
bool prio_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HZ_PRIO");
    return e && e[0] == '1';
  }();
  return on;
}
int prio_from() {
  static const int l0 = [] {
    const char* e = std::getenv("HZ_PRIO_FROM");
    return e ? std::atoi(e) : 0;
  }();
  return l0;
}
}  // namespace

template <class T>
void Hierarchy<T>::clear_graphs() {
  for (auto& kv : graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  graphs_.clear();
  for (auto& kv : bt_graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  bt_graphs_.clear();
}

template <class T>
template <class XO>
void Hierarchy<T>::cycle_cast_graph(const CycleSpec& spec, int k, const double2* b64, XO* x64, cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("HZ_CYCLE_GRAPHS");
    return !(e && e[0] == '0');
  }();
  if (!on || sl_ || spec.kind == CycleKind::K || profiling_enabled()) {
    cycle_cast(spec, k, b64, x64, s);
    return;
  }
  const GraphKey key{b64, x64, k, int(spec.kind), spec.pre, spec.post, spec.jacobi_weight};
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {  // first use: run directly (workspaces, smem limits)
    cycle_cast(spec, k, b64, x64, s);
    graphs_.emplace(key, GraphRec{});
    return;
  }
  GraphRec& g = it->second;
  if (!g.exec) {
    cudaGraph_t graph = nullptr;
    HZ_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    set_capturing(true);
    try {
      cycle_cast(spec, k, b64, x64, s);
    } catch (...) {
      set_capturing(false);
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    set_capturing(false);
    HZ_CUDA(cudaStreamEndCapture(s, &graph));
    size_t nn = 0;
    HZ_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    HZ_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
    g.kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      HZ_CUDA(cudaGraphNodeGetType(nd, &ty));
      if (ty == cudaGraphNodeTypeKernel) ++g.kernels;
    }
    const cudaError_t st = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    HZ_CUDA(st);
  }
  HZ_CUDA(cudaGraphLaunch(g.exec, s));
  add_launches(g.kernels);
}

template <class T>
Hierarchy<T>::~Hierarchy() {
  clear_graphs();
  if (hp_fork_) cudaEventDestroy(hp_fork_);
  if (hp_join_) cudaEventDestroy(hp_join_);
  if (hp_) cudaStreamDestroy(hp_);
}

template <class T>
void Hierarchy<T>::coarse_visit(int l, const CycleSpec& spec, int k, cudaStream_t s) {
  if (l == prio_from() && !sl_ && prio_enabled()) {
    if (!hp_) {
      int lo = 0, hi = 0;
      HZ_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      HZ_CUDA(cudaStreamCreateWithPriority(&hp_, cudaStreamNonBlocking, hi));
      HZ_CUDA(cudaEventCreateWithFlags(&hp_fork_, cudaEventDisableTiming));
      HZ_CUDA(cudaEventCreateWithFlags(&hp_join_, cudaEventDisableTiming));
    }
    HZ_CUDA(cudaEventRecord(hp_fork_, s));
    HZ_CUDA(cudaStreamWaitEvent(hp_, hp_fork_, 0));
    coarse_visit_on(l, spec, k, hp_);
    HZ_CUDA(cudaEventRecord(hp_join_, hp_));
    HZ_CUDA(cudaStreamWaitEvent(s, hp_join_, 0));
    return;
  }
  coarse_visit_on(l, spec, k, s);
}

template <class T>
void Hierarchy<T>::coarse_visit_on(int l, const CycleSpec& spec, int k, cudaStream_t s) {
  const int L = num_levels();
  const bool sl = slab_level(l);
  V* ec = wx_[l + 1].get();
  const V* rc = wb_[l + 1].get();
  switch (spec.kind) {
    case CycleKind::V:
      cycle_rec(l + 1, spec, k, rc, ec, true, s);
      break;
    case CycleKind::W:
      cycle_rec(l + 1, spec, k, rc, ec, true, s);
      if (l + 1 < L - 1) cycle_rec(l + 1, spec, k, rc, ec, false, s);
      break;
    case CycleKind::K:
      if (l + 1 == L - 1)
        cycle_rec(l + 1, spec, k, rc, ec, true, s);
      else if (sl && slab_level(l + 1))
        throw HzError(kValidation, "slabs: K-cycle inner Krylov levels must be agglomerated");
      else
        kcycle_coarse(l + 1, spec, k, rc, ec, s);
      break;
  }
}

// One cycle of the complex64 hierarchy applied to a complex128 block (the
// mixed-precision preconditioner): b64 -> x64 with the casts fused into the
// first two and the last fine-level sweeps when the fine level allows it;
// otherwise cast, cycle, cast.
// XO = float2: the cycle's complex64 result without the up-cast (exact: the
// c128 value would be its widening), for FGMRES's complex64 Z blocks.
template <class T>
template <class XO>
void Hierarchy<T>::cycle_cast(const CycleSpec& spec, int k, const double2* b64, XO* x64, cudaStream_t s) {
  if constexpr (!std::is_same<T, float>::value) {
    throw HzError(kState, "cycle_cast: complex64 hierarchies only");
  } else {
    ensure_ws(k);
    const int L = num_levels();
    V* b32 = wb_[0].get();
    V* x = wx_[0].get();
    static const bool allow = [] {  // HZ_FUSED_CAST=0: unfused reference path
      const char* e = std::getenv("HZ_FUSED_CAST");
      return !(e && e[0] == '0');
    }();
    const bool fused = allow && L > 1 && fused_fine_ok(op(0, k)) && cast_zero_ok(op(0, k)) && spec.pre >= 1 &&
                       spec.post >= 1;
    if (!fused) {
      on_level(0, k, s, [&](const LevelOp<T>&, cudaStream_t st, int64_t r0, int64_t nr) {
        launch_cast<float2, double2>(nr * k, b64 + r0 * k, b32 + r0 * k, st);
      });
      cycle_rec(0, spec, k, b32, x, true, s);
      on_level(0, k, s, [&](const LevelOp<T>&, cudaStream_t st, int64_t r0, int64_t nr) {
        if constexpr (std::is_same<XO, double2>::value)
          launch_cast<double2, float2>(nr * k, x + r0 * k, x64 + r0 * k, st);
        else
          HZ_CUDA(cudaMemcpyAsync(x64 + r0 * k, x + r0 * k, size_t(nr) * k * sizeof(float2),
                                  cudaMemcpyDeviceToDevice, st));
      });
      return;
    }
    const T wj = T(spec.jacobi_weight);
    if (fused_level0(spec, k)) {
      const LevelGeom gc(levels_[1].dims[0], levels_[1].dims[1], levels_[1].dims[2], k);
      launch_fused_pre<T, double2>(op(0, k), gc, wj, b64, x, wb_[1].get(), s);
      coarse_visit(0, spec, k, s);
      launch_fused_post<T, double2, XO>(op(0, k), gc, wj, x, wx_[1].get(), b64, x64, s);
      return;
    }
    const bool sl = slab_level(0);
    if (sl) sl_->neighbours();
    on_level(0, k, s, [&](const LevelOp<T>& o, cudaStream_t st, int64_t, int64_t) {
      launch_jacobi_zero_cast(o, wj, b64, b32, x, st);
    });
    V* cur = x;
    V* other = wt_[0].get();
    bool cur_zero = false;
    relax(0, spec, spec.pre - 1, k, b32, cur, other, cur_zero, s);
    coarse_correction(0, spec, k, b32, cur, false, s);
    relax(0, spec, spec.post - 1, k, b32, cur, other, cur_zero, s);
    if (sl) sl_->neighbours();
    on_level(0, k, s, [&](const LevelOp<T>& o, cudaStream_t st, int64_t, int64_t) {
      if constexpr (std::is_same<XO, double2>::value)
        launch_jacobi_out64(o, wj, cur, b32, x64, st);
      else
        launch_jacobi<T>(o, wj, cur, b32, x64, st);
    });
  }
}

// kcycle_coarse (src/multigrid.cpp:138-160): k_inner block FGMRES iterations
// on level l, tol 0, preconditioned by cycle_rec(l).
template <class T>
void Hierarchy<T>::kcycle_coarse(int l, const CycleSpec& spec, int k, const V* b, V* x,
                                 cudaStream_t s) {
  if (int(kfgm_.size()) < num_levels()) kfgm_.resize(num_levels());
  if (!kfgm_[l]) kfgm_[l] = std::make_unique<Fgmres<T>>();
  DevOp<T> dop;
  dop.n = levels_[l].nodes();
  dop.apply = [this, l](const V* in, V* out, int kk, cudaStream_t st) {
    launch_apply<T>(op(l, kk), in, out, st);
  };
  const size_t bytes = size_t(levels_[l].nodes()) * k * sizeof(V);
  dop.prec = [this, l, spec, bytes](const V* in, V* out, int kk, cudaStream_t st) {
    cycle_rec(l, spec, kk, in, out, true, st);
  };
  (void)bytes;
  kfgm_[l]->solve(dop, k, b, x, spec.k_inner, 0.0, spec.k_inner, s);
}

template class Hierarchy<double>;
template class Hierarchy<float>;
template void Hierarchy<float>::cycle_cast<double2>(const CycleSpec&, int, const double2*, double2*, cudaStream_t);
template void Hierarchy<float>::cycle_cast<float2>(const CycleSpec&, int, const double2*, float2*, cudaStream_t);
template void Hierarchy<float>::cycle_cast_graph<double2>(const CycleSpec&, int, const double2*, double2*,
                                                          cudaStream_t);
template void Hierarchy<float>::cycle_cast_graph<float2>(const CycleSpec&, int, const double2*, float2*,
                                                         cudaStream_t);

}  // namespace hz
