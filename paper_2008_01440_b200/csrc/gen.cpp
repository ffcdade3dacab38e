// SPDX-License-Identifier: Apache-2.0
//
// Builder-defined input generators for BASELINE.json configs 3 and 4 (the
// reference has no such generators). They produce the int32 CSR
// both the device operator and the CPU oracle consume, so the two sides see
// bit-identical matrices. Values are assembled element by element in a fixed
// (cell-index) order from a symmetric element matrix, so a_ij == a_ji bitwise,
// which CsrMatrix(..., sym_tol = 0) requires (proj/src/linop.cpp:137-157).
//
// Mesh: (nx+1)^3 unit hexahedral cells, (nx+2)^3 nodes, the nx^3 interior nodes
// are unknowns (homogeneous Dirichlet boundary eliminated), lexicographic
// i-fastest numbering like StencilOperator (proj/src/linop.cpp:241-244).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "pcgx.h"

namespace {

uint64_t splitmix_at(uint64_t seed, uint64_t i) {  // i-th draw, as eigenest.cpp:13-18
  uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
double unit_open(uint64_t bits) {  // (0, 1]
  return (static_cast<double>(bits >> 11) + 1.0) * 0x1.0p-53;
}

// Q1 Laplace stiffness on the unit cube: K[a][b] for local nodes a, b in
// {0..7} (bit 0 = x, bit 1 = y, bit 2 = z) = sum_d S_d (x) M_e (x) M_f over
// the 1D stiffness S = [[1,-1],[-1,1]] and mass M = [[1/3,1/6],[1/6,1/3]],
// with edge lengths h = (1, 1.25, 1.5) so every one of the 27 couplings is
// nonzero (the isotropic cube has exactly-zero axis couplings).
void q1_diffusion(double K[8][8]) {
  const double h[3] = {1.0, 1.25, 1.5};
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      double v = 0.0;
      for (int d = 0; d < 3; ++d) {
        double t = 1.0;
        for (int e = 0; e < 3; ++e) {
          const bool same = ((a >> e) & 1) == ((b >> e) & 1);
          if (e == d) t *= (same ? 1.0 : -1.0) / h[e];
          else t *= h[e] * (same ? (1.0 / 3.0) : (1.0 / 6.0));
        }
        v += t;
      }
      K[a][b] = v;
    }
  for (int a = 0; a < 8; ++a)
    for (int b = a + 1; b < 8; ++b) K[b][a] = K[a][b];
}

// Q1 isotropic linear-elasticity stiffness on the unit cube, 2x2x2 Gauss
// (exact for a box), Voigt order (xx, yy, zz, xy, yz, xz); dof index 3*a + c.
void q1_elasticity(double lambda, double mu, double K[24][24]) {
  std::memset(K, 0, sizeof(double) * 24 * 24);
  const double g[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  double D[6][6] = {};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) D[i][j] = lambda + (i == j ? 2.0 * mu : 0.0);
  for (int i = 3; i < 6; ++i) D[i][i] = mu;
  for (int qz = 0; qz < 2; ++qz)
    for (int qy = 0; qy < 2; ++qy)
      for (int qx = 0; qx < 2; ++qx) {
        const double xi[3] = {g[qx], g[qy], g[qz]};
        double dN[8][3];
        for (int a = 0; a < 8; ++a)
          for (int d = 0; d < 3; ++d) {
            double t = ((a >> d) & 1) ? 1.0 : -1.0;
            for (int e = 0; e < 3; ++e)
              if (e != d) t *= ((a >> e) & 1) ? xi[e] : (1.0 - xi[e]);
            dN[a][d] = t;
          }
        double B[6][24] = {};
        for (int a = 0; a < 8; ++a) {
          const double nx = dN[a][0], ny = dN[a][1], nz = dN[a][2];
          B[0][3 * a + 0] = nx;
          B[1][3 * a + 1] = ny;
          B[2][3 * a + 2] = nz;
          B[3][3 * a + 0] = ny;
          B[3][3 * a + 1] = nx;
          B[4][3 * a + 1] = nz;
          B[4][3 * a + 2] = ny;
          B[5][3 * a + 0] = nz;
          B[5][3 * a + 2] = nx;
        }
        const double w = 0.125;
        for (int i = 0; i < 24; ++i)
          for (int j = i; j < 24; ++j) {
            double v = 0.0;
            for (int k = 0; k < 6; ++k)
              for (int l = 0; l < 6; ++l) v += B[k][i] * D[k][l] * B[l][j];
            K[i][j] += w * v;
          }
      }
  for (int i = 0; i < 24; ++i)
    for (int j = i + 1; j < 24; ++j) K[j][i] = K[i][j];
}

struct Mesh {
  int64_t nx;
  int64_t n_nodes() const { return nx * nx * nx; }
  int64_t ncell() const { return nx + 1; }
  // neighbour count of interior node coordinate c in one direction
  int cnt(int64_t c) const { return (c > 0 ? 1 : 0) + 1 + (c < nx - 1 ? 1 : 0); }
  int64_t row_neighbours(int64_t i, int64_t j, int64_t k) const {
    return (int64_t)cnt(i) * cnt(j) * cnt(k);
  }
};

// Fills the node-level pattern and calls emit(row_node, col_node, a, b, cell)
// for every shared cell (a, b = local corner ids of the two nodes in that cell),
// in ascending neighbour order and, per neighbour, ascending cell order.
template <class CellWeight, class Emit>
void assemble_rows(const Mesh& m, int64_t node, CellWeight&&, Emit&& emit_neighbour) {
  const int64_t nx = m.nx;
  const int64_t i = node % nx, j = (node / nx) % nx, k = node / (nx * nx);
  for (int dz = -1; dz <= 1; ++dz) {
    if (k + dz < 0 || k + dz >= nx) continue;
    for (int dy = -1; dy <= 1; ++dy) {
      if (j + dy < 0 || j + dy >= nx) continue;
      for (int dx = -1; dx <= 1; ++dx) {
        if (i + dx < 0 || i + dx >= nx) continue;
        emit_neighbour(dx, dy, dz, i, j, k);
      }
    }
  }
}

// Interior node (i, j, k) (0-based unknown coords) is mesh node (i+1, j+1, k+1);
// cell (ci, cj, ck) spans mesh nodes ci..ci+1 etc. For the node pair (p, p+o)
// the shared cells in direction d are: o_d = 0 -> cells {p_d - 1, p_d} (mesh
// coords), o_d = +1 -> {p_d}, o_d = -1 -> {p_d - 1}; local corner bit of the
// node in cell c is (mesh_coord - c).
template <class F>
void for_shared_cells(int64_t i, int64_t j, int64_t k, int dx, int dy, int dz, F&& f) {
  const int64_t p[3] = {i + 1, j + 1, k + 1};
  const int o[3] = {dx, dy, dz};
  int64_t lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    if (o[d] == 0) {
      lo[d] = p[d] - 1;
      hi[d] = p[d];
    } else if (o[d] > 0) {
      lo[d] = hi[d] = p[d];
    } else {
      lo[d] = hi[d] = p[d] - 1;
    }
  }
  for (int64_t cz = lo[2]; cz <= hi[2]; ++cz)
    for (int64_t cy = lo[1]; cy <= hi[1]; ++cy)
      for (int64_t cx = lo[0]; cx <= hi[0]; ++cx) {
        const int a = (int)((p[0] - cx) | ((p[1] - cy) << 1) | ((p[2] - cz) << 2));
        const int b = (int)((p[0] + o[0] - cx) | ((p[1] + o[1] - cy) << 1) | ((p[2] + o[2] - cz) << 2));
        f(cx, cy, cz, a, b);
      }
}

thread_local std::string g_gen_err;

}  // namespace

extern "C" {

pcgx_status pcgx_gen_fe27_size(int64_t nx, int64_t* n, int64_t* nnz) {
  if (nx < 1) return PCGX_ERR_INVALID;
  *n = nx * nx * nx;
  const int64_t t = 3 * nx - 2;
  *nnz = t * t * t;
  return (*nnz >= (1LL << 31)) ? PCGX_ERR_OVERFLOW : PCGX_OK;
}

pcgx_status pcgx_gen_fe27_fill(int64_t nx, double sigma, uint64_t seed, int32_t* row_ptr,
                               int32_t* col_idx, double* values) {
  int64_t n, nnz;
  const pcgx_status st = pcgx_gen_fe27_size(nx, &n, &nnz);
  if (st != PCGX_OK) return st;
  const Mesh m{nx};
  const int64_t nc = nx + 1;
  // cell coefficients kappa_c = exp(sigma * N(0,1)), Box-Muller on draws 2c, 2c+1
  std::vector<double> kappa((size_t)(nc * nc * nc));
  const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nc * nc * nc; ++c) {
    const double u1 = unit_open(splitmix_at(seed, 2 * (uint64_t)c));
    const double u2 = unit_open(splitmix_at(seed, 2 * (uint64_t)c + 1));
    const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
    kappa[(size_t)c] = std::exp(sigma * g);
  }
  double K[8][8];
  q1_diffusion(K);
  row_ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = r % nx, j = (r / nx) % nx, k = r / (nx * nx);
    row_ptr[r + 1] = (int32_t)(row_ptr[r] + m.row_neighbours(i, j, k));
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    int64_t pos = row_ptr[r];
    assemble_rows(m, r, 0, [&](int dx, int dy, int dz, int64_t i, int64_t j, int64_t k) {
      double v = 0.0;
      for_shared_cells(i, j, k, dx, dy, dz, [&](int64_t cx, int64_t cy, int64_t cz, int a, int b) {
        v += kappa[(size_t)((cz * nc + cy) * nc + cx)] * K[a][b];
      });
      col_idx[pos] = (int32_t)(((k + dz) * nx + (j + dy)) * nx + (i + dx));
      values[pos] = v;
      ++pos;
    });
  }
  return PCGX_OK;
}

pcgx_status pcgx_gen_elast27_size(int64_t nx, int64_t* n, int64_t* nnz) {
  if (nx < 1) return PCGX_ERR_INVALID;
  *n = 3 * nx * nx * nx;
  const int64_t t = 3 * nx - 2;
  *nnz = 9 * t * t * t;
  return (*nnz >= (1LL << 31)) ? PCGX_ERR_OVERFLOW : PCGX_OK;
}

pcgx_status pcgx_gen_elast27_fill(int64_t nx, double lambda, double mu, double eps,
                                  uint64_t seed, int32_t* row_ptr, int32_t* col_idx,
                                  double* values) {
  int64_t n, nnz;
  const pcgx_status st = pcgx_gen_elast27_size(nx, &n, &nnz);
  if (st != PCGX_OK) return st;
  if (!(eps >= 0.0) || !(mu > 0.0) || !(lambda >= 0.0)) return PCGX_ERR_INVALID;
  const Mesh m{nx};
  const int64_t nc = nx + 1;
  std::vector<double> scale((size_t)(nc * nc * nc));
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nc * nc * nc; ++c) {
    const double u = static_cast<double>(splitmix_at(seed, (uint64_t)c) >> 11) * 0x1.0p-53;
    scale[(size_t)c] = 1.0 + eps * u;
  }
  static double K[24][24];
  q1_elasticity(lambda, mu, K);
  const int64_t nn = m.n_nodes();
  row_ptr[0] = 0;
  for (int64_t node = 0; node < nn; ++node) {
    const int64_t i = node % nx, j = (node / nx) % nx, k = node / (nx * nx);
    const int64_t per_row = 3 * m.row_neighbours(i, j, k);
    for (int c = 0; c < 3; ++c) {
      const int64_t r = 3 * node + c;
      row_ptr[r + 1] = (int32_t)(row_ptr[r] + per_row);
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t node = 0; node < nn; ++node) {
    for (int comp = 0; comp < 3; ++comp) {
      const int64_t r = 3 * node + comp;
      int64_t pos = row_ptr[r];
      assemble_rows(m, node, 0, [&](int dx, int dy, int dz, int64_t i, int64_t j, int64_t k) {
        const int64_t col_node = ((k + dz) * nx + (j + dy)) * nx + (i + dx);
        for (int c2 = 0; c2 < 3; ++c2) {
          double v = 0.0;
          for_shared_cells(i, j, k, dx, dy, dz,
                           [&](int64_t cx, int64_t cy, int64_t cz, int a, int b) {
                             v += scale[(size_t)((cz * nc + cy) * nc + cx)] *
                                  K[3 * a + comp][3 * b + c2];
                           });
          col_idx[pos] = (int32_t)(3 * col_node + c2);
          values[pos] = v;
          ++pos;
        }
      });
    }
  }
  return PCGX_OK;
}

}  // extern "C"
