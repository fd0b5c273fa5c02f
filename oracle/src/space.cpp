// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates mesh.cpp, dof_space.cpp and block_vector.hpp.
#include "oracle/oracle.hpp"

#include <cmath>

namespace oracle
{

// ---------------------------------------------------------------- mesh.cpp
Mesh
Mesh::build_cartesian(const Box &domain, int base_nx, int base_ny, int levels)
{
  if (base_nx < 1 || base_ny < 1)
    throw std::invalid_argument("Mesh: base cell counts must be >= 1");
  if (levels < 1)
    throw std::invalid_argument("Mesh: need at least one level");
  if (!(domain.width() > 0.0) || !(domain.height() > 0.0))
    throw std::invalid_argument("Mesh: domain box has non-positive extent");
  return Mesh(domain, base_nx, base_ny, levels);
}

void
Mesh::check_level(int l) const
{
  if (l < 0 || l >= levels_)
    throw std::out_of_range("Mesh: level out of range");
}

Box
Mesh::cell_box(int l, int cell) const
{
  check_level(l);
  const auto [ix, iy] = cell_coords(l, cell);
  const double dx = hx(l), dy = hy(l);
  return Box{domain_.x0 + ix * dx, domain_.y0 + iy * dy, domain_.x0 + (ix + 1) * dx, domain_.y0 + (iy + 1) * dy};
}

std::array<int, 4>
Mesh::children(int l, int cell) const
{
  check_level(l + 1);
  const auto [ix, iy] = cell_coords(l, cell);
  const int f = l + 1;
  return {cell_index(f, 2 * ix, 2 * iy), cell_index(f, 2 * ix + 1, 2 * iy), cell_index(f, 2 * ix, 2 * iy + 1),
          cell_index(f, 2 * ix + 1, 2 * iy + 1)};
}

int
Mesh::parent(int l, int cell) const
{
  check_level(l);
  if (l == 0)
    throw std::out_of_range("Mesh: level 0 cells have no parent");
  const auto [ix, iy] = cell_coords(l, cell);
  return cell_index(l - 1, ix / 2, iy / 2);
}

std::vector<int>
Mesh::cells_of_vertex(int l, int v) const
{
  check_level(l);
  if (v < 0 || v >= n_vertices(l))
    throw std::out_of_range("Mesh: unknown vertex id");
  const auto [vx, vy] = vertex_coords(l, v);
  const int nx = cells_x(l), ny = cells_y(l);
  std::vector<int> cells;
  for (int cy = vy - 1; cy <= vy; ++cy)
    for (int cx = vx - 1; cx <= vx; ++cx)
      if (cx >= 0 && cx < nx && cy >= 0 && cy < ny)
        cells.push_back(cell_index(l, cx, cy));
  std::sort(cells.begin(), cells.end());
  return cells;
}

std::vector<int>
Mesh::vertex_neighbors(int l, int cell) const
{
  check_level(l);
  const auto [ix, iy] = cell_coords(l, cell);
  const int nx = cells_x(l), ny = cells_y(l);
  std::vector<int> cells;
  for (int cy = iy - 1; cy <= iy + 1; ++cy)
    for (int cx = ix - 1; cx <= ix + 1; ++cx)
      if (cx >= 0 && cx < nx && cy >= 0 && cy < ny)
        cells.push_back(cell_index(l, cx, cy));
  return cells;
}

// ---------------------------------------------------------------- dof_space.cpp
VelocitySpace::VelocitySpace(const Mesh &mesh, int level, int r)
  : mesh_(&mesh), level_(level), r_(r), basis_(gauss_lobatto_points(r + 2))
{
  if (r < 1)
    throw std::invalid_argument("VelocitySpace: r must be >= 1");
  const int nx = mesh.cells_x(level), ny = mesh.cells_y(level);
  const int p = r + 1;
  grid_x_ = nx * p + 1;
  grid_y_ = ny * p + 1;
  n_scalar_ = grid_x_ * grid_y_;
  const int n1 = p + 1;
  cell_dofs_.resize(mesh.n_cells(level));
  for (int cell = 0; cell < mesh.n_cells(level); ++cell)
    {
      const auto [cx, cy] = mesh.cell_coords(level, cell);
      auto &dofs = cell_dofs_[cell];
      dofs.resize(n1 * n1);
      for (int iy = 0; iy < n1; ++iy)
        for (int ix = 0; ix < n1; ++ix)
          dofs[iy * n1 + ix] = (cy * p + iy) * grid_x_ + (cx * p + ix);
    }
  const Box dom = mesh.domain();
  const double dx = mesh.hx(level), dy = mesh.hy(level);
  coord_x_.resize(grid_x_);
  coord_y_.resize(grid_y_);
  const Vec &nodes = basis_.nodes();
  for (int cx = 0; cx < nx; ++cx)
    for (int a = 0; a < n1; ++a)
      coord_x_[cx * p + a] = dom.x0 + dx * (cx + 0.5 * (nodes[a] + 1.0));
  for (int cy = 0; cy < ny; ++cy)
    for (int a = 0; a < n1; ++a)
      coord_y_[cy * p + a] = dom.y0 + dy * (cy + 0.5 * (nodes[a] + 1.0));
  coord_x_.back() = dom.x1;
  coord_y_.back() = dom.y1;
  boundary_.assign(n_scalar_, 0);
  for (int j = 0; j < grid_y_; ++j)
    for (int i = 0; i < grid_x_; ++i)
      if (i == 0 || i == grid_x_ - 1 || j == 0 || j == grid_y_ - 1)
        {
          boundary_[j * grid_x_ + i] = 1;
          boundary_list_.push_back(j * grid_x_ + i);
        }
}

void
VelocitySpace::zero_constrained(double *v) const
{
  for (int comp = 0; comp < 2; ++comp)
    for (const int s : boundary_list_)
      v[static_cast<Index>(comp) * n_scalar_ + s] = 0.0;
}

void
VelocitySpace::set_boundary_values(double *v, const std::function<double(double, double, double, int)> &g,
                                   double t) const
{
  for (const int s : boundary_list_)
    {
      const double x = node_x(s), y = node_y(s);
      for (int comp = 0; comp < 2; ++comp)
        v[static_cast<Index>(comp) * n_scalar_ + s] = g(x, y, t, comp);
    }
}

PressureSpace::PressureSpace(const Mesh &mesh, int level, int r)
  : mesh_(&mesh), level_(level), r_(r), basis_(r, 2)
{
  if (r < 1)
    throw std::invalid_argument("PressureSpace: r must be >= 1");
  const int n_cells = mesh.n_cells(level);
  const int np = basis_.size();
  n_dofs_ = static_cast<Index>(n_cells) * np;
  const double jdet = 0.25 * mesh.hx(level) * mesh.hy(level);
  mass_diag_.resize(n_dofs_);
  one_.assign(n_dofs_, 0.0);
  mean_.assign(n_dofs_, 0.0);
  for (int cell = 0; cell < n_cells; ++cell)
    {
      for (int l = 0; l < np; ++l)
        mass_diag_[static_cast<size_t>(cell) * np + l] = jdet * basis_.gram_diagonal(l);
      one_[static_cast<size_t>(cell) * np] = 1.0;
      mean_[static_cast<size_t>(cell) * np] = jdet * basis_.gram_diagonal(0);
    }
  volume_ = mesh.domain().volume();
}

double
PressureSpace::mean_integral(const double *p) const
{
  double s = 0.0;
  for (Index i = 0; i < n_dofs_; ++i)
    s += mean_[i] * p[i];
  return s;
}

void
PressureSpace::project_mean_zero(double *p) const
{
  const double mean = mean_integral(p) / volume_;
  const int np = basis_.size();
  for (int cell = 0; cell < mesh_->n_cells(level_); ++cell)
    p[static_cast<Index>(cell) * np] -= mean;
}

// ---------------------------------------------------------------- block_vector.hpp
double
BlockVector::norm() const
{
  double s = 0.0;
  for (const double v : data)
    s += v * v;
  return std::sqrt(s);
}

double
BlockVector::dot(const BlockVector &o) const
{
  double s = 0.0;
  for (size_t i = 0; i < data.size(); ++i)
    s += data[i] * o.data[i];
  return s;
}

BlockVector &
BlockVector::operator+=(const BlockVector &o)
{
  for (size_t i = 0; i < data.size(); ++i)
    data[i] += o.data[i];
  return *this;
}

BlockVector &
BlockVector::operator-=(const BlockVector &o)
{
  for (size_t i = 0; i < data.size(); ++i)
    data[i] -= o.data[i];
  return *this;
}

BlockVector &
BlockVector::operator*=(double s)
{
  for (double &v : data)
    v *= s;
  return *this;
}

void
require_same_shape(const BlockVector &a, const BlockVector &b, const char *where)
{
  if (!a.same_shape(b))
    throw std::invalid_argument(std::string(where) + ": block vector shape mismatch");
}

} // namespace oracle
