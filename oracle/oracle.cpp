// oracle.cpp -- plain fp64 CPU oracle of the MIS-SLAM registration hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  Written from PAPER.md and the
// readings in DESIGN.md §3 in the paper's order and notation; no blocking,
// fusion or reordering beyond what the definitions state.  Shares no code with
// the CUDA path.
//
// Citations: P:n = PAPER.md line n (section / equation / algorithm named
// beside it); S:n = SPEC.md line n; R-An = DESIGN.md reading An.
#include "oracle.h"

#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <utility>
#include <vector>
#include <algorithm>

#include <omp.h>

namespace {

// Host threads of the oracle (or_set_threads; default 1).  Only the loops over independent items
// (points, pixels, queries) are split; the per-thread partial normal equations are merged in
// thread order, so a fixed thread count gives a fixed summation order.  Used by bench.py's
// all-cores timing column; the pins and parity tests run single-threaded.
int g_threads = 1;

typedef std::array<double, 3> V3;
typedef std::array<double, 9> M3;     // row-major
typedef std::array<double, 36> B6;    // 6x6 row-major

const double kInf = std::numeric_limits<double>::infinity();

V3 v3(double a, double b, double c) { V3 r = {a, b, c}; return r; }
V3 load3(const float* p) { return v3((double)p[0], (double)p[1], (double)p[2]); }
V3 add(const V3& a, const V3& b) { return v3(a[0] + b[0], a[1] + b[1], a[2] + b[2]); }
V3 sub(const V3& a, const V3& b) { return v3(a[0] - b[0], a[1] - b[1], a[2] - b[2]); }
V3 scale(const V3& a, double s) { return v3(a[0] * s, a[1] * s, a[2] * s); }
double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
double norm(const V3& a) { return std::sqrt(dot(a, a)); }
V3 cross(const V3& a, const V3& b) {
  return v3(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
}
V3 mul(const M3& R, const V3& x) {
  return v3(R[0] * x[0] + R[1] * x[1] + R[2] * x[2],
            R[3] * x[0] + R[4] * x[1] + R[5] * x[2],
            R[6] * x[0] + R[7] * x[1] + R[8] * x[2]);
}
V3 mulT(const M3& R, const V3& x) {   // R^T x
  return v3(R[0] * x[0] + R[3] * x[1] + R[6] * x[2],
            R[1] * x[0] + R[4] * x[1] + R[7] * x[2],
            R[2] * x[0] + R[5] * x[1] + R[8] * x[2]);
}
M3 matmul(const M3& A, const M3& B) {
  M3 C;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int l = 0; l < 3; ++l) s += A[3 * i + l] * B[3 * l + j];
      C[3 * i + j] = s;
    }
  return C;
}
M3 node_R(const double* Rt, int j) { M3 R; for (int a = 0; a < 9; ++a) R[a] = Rt[12 * j + a]; return R; }
V3 node_t(const double* Rt, int j) { return v3(Rt[12 * j + 9], Rt[12 * j + 10], Rt[12 * j + 11]); }
M3 pose_R(const double* pose) { M3 R; for (int a = 0; a < 9; ++a) R[a] = pose[a]; return R; }
V3 pose_T(const double* pose) { return v3(pose[9], pose[10], pose[11]); }

bool depth_ok(float d) { return std::isfinite(d) && d > 0.0f; }

// ---- O0: back-projection Pi(u, D) ("back-projection function")
V3 back_project(const or_frame* f, int x, int y, double D) {
  return v3(((double)x - f->cx) * D / f->fx, ((double)y - f->cy) * D / f->fy, D);
}

// Central-difference normal, R-A11 (paper silent on the estimator):
// N = normalize((q(x+1,y)-q(x-1,y)) x (q(x,y+1)-q(x,y-1))), flipped so N.q < 0.
bool pixel_normal(const or_frame* f, int x, int y, V3* N) {
  const int W = f->W, H = f->H;
  if (x <= 0 || y <= 0 || x >= W - 1 || y >= H - 1) return false;
  const float* D = f->depth;
  float c = D[y * W + x], l = D[y * W + x - 1], r = D[y * W + x + 1];
  float u = D[(y - 1) * W + x], d = D[(y + 1) * W + x];
  if (!depth_ok(c) || !depth_ok(l) || !depth_ok(r) || !depth_ok(u) || !depth_ok(d)) return false;
  V3 dx = sub(back_project(f, x + 1, y, r), back_project(f, x - 1, y, l));
  V3 dy = sub(back_project(f, x, y + 1, d), back_project(f, x, y - 1, u));
  V3 n = cross(dx, dy);
  double len = norm(n);
  if (len < 1e-12) return false;
  n = scale(n, 1.0 / len);
  if (dot(n, back_project(f, x, y, c)) > 0) n = scale(n, -1.0);
  *N = n;
  return true;
}

// ---- Eq. 2 skinning, normalised (R-A6); ties -> lower id
void skin_one(const V3& v, int m, const float* g, int k, int32_t* idx, double* w, double* margin) {
  // the k+1 smallest (distance, id) pairs in lexicographic order, by insertion
  std::vector<std::pair<double, int> > d;
  for (int j = 0; j < m; ++j) {
    std::pair<double, int> c = std::make_pair(norm(sub(v, load3(g + 3 * j))), j);
    if ((int)d.size() == k + 1 && !(c < d.back())) continue;
    if ((int)d.size() == k + 1) d.pop_back();
    d.insert(std::upper_bound(d.begin(), d.end(), c), c);   // equal distances -> lower id first
  }
  double dmax = d[k].first;        // distance to the (k+1)-th nearest node
  double sum = 0;
  for (int s = 0; s < k; ++s) {
    idx[s] = d[s].second;
    w[s] = (dmax > 0) ? 1.0 - d[s].first / dmax : 1.0 / k;   // d_max = 0 -> 1/k
    sum += w[s];
  }
  for (int s = 0; s < k; ++s) w[s] = (sum > 0) ? w[s] / sum : 1.0 / k;
  if (margin) *margin = (d[k].first > 0) ? (d[k].first - d[k - 1].first) / d[k].first : 0.0;
}

// ---- O3a: Eq. 1 warp with A_j = R_j (R-A1) and normalised weights (R-A6)
// x_hat = sum_j w_j (R_j (v - g_j) + g_j + t_j);  v~ = R x_hat + T;
// m_hat = sum_j w_j R_j n;  n~ = R m_hat / |m_hat|.
struct Warped {
  bool ok;
  double wn[8];      // normalised weights
  V3 a[8];           // a_j = R_j (v - g_j)
  V3 x_hat, m_hat, vt, nt;
};

Warped warp_point(const V3& v, const V3& n, int k, const int32_t* idx, const double* wraw,
                  const float* g, const double* Rt, const double* pose) {
  Warped o;
  o.ok = false;
  double W = 0;
  for (int s = 0; s < k; ++s) W += wraw[s];
  if (!(W > 0)) return o;
  o.x_hat = v3(0, 0, 0);
  o.m_hat = v3(0, 0, 0);
  for (int s = 0; s < k; ++s) {
    int j = idx[s];
    o.wn[s] = wraw[s] / W;
    M3 Rj = node_R(Rt, j);
    V3 gj = load3(g + 3 * j);
    o.a[s] = mul(Rj, sub(v, gj));
    o.x_hat = add(o.x_hat, scale(add(add(o.a[s], gj), node_t(Rt, j)), o.wn[s]));
    o.m_hat = add(o.m_hat, scale(mul(Rj, n), o.wn[s]));
  }
  M3 R = pose_R(pose);
  o.vt = add(mul(R, o.x_hat), pose_T(pose));
  double ml = norm(o.m_hat);
  if (ml < 1e-12) return o;
  o.nt = mul(R, scale(o.m_hat, 1.0 / ml));
  o.ok = true;
  return o;
}

// ---- Projection P and pixel rounding floor(u + 0.5) (R-A10)
struct Proj { bool z_ok, in_frame; int px, py; double margin; };
Proj project(const or_frame* f, const V3& p) {
  Proj r;
  r.z_ok = p[2] > 0;
  r.in_frame = false;
  r.px = r.py = -1;
  r.margin = std::fabs(p[2]);
  if (!r.z_ok) return r;
  double u = f->fx * p[0] / p[2] + f->cx;
  double v = f->fy * p[1] / p[2] + f->cy;
  double fu = std::floor(u + 0.5), fv = std::floor(v + 0.5);
  double mu = std::min(u + 0.5 - fu, fu + 1.0 - (u + 0.5));   // distance of u+0.5 to an integer
  double mv = std::min(v + 0.5 - fv, fv + 1.0 - (v + 0.5));
  r.margin = std::min(r.margin, std::min(mu, mv));
  if (fu < 0 || fv < 0 || fu >= f->W || fv >= f->H) return r;
  r.px = (int)fu;
  r.py = (int)fv;
  r.in_frame = true;
  return r;
}

// ---- O3b: Eq. 7 gates with the warped point (R-A7), angle < eps_n (R-A8)
struct Assoc { int32_t pix; uint8_t why; double margin; V3 q, N; };
Assoc associate_point(const or_params* prm, const or_frame* f, const Warped& w) {
  Assoc a;
  a.pix = -1;
  a.why = 0;
  a.margin = kInf;
  if (!w.ok) return a;
  Proj pr = project(f, w.vt);
  a.margin = pr.margin;
  if (!pr.z_ok) return a;
  a.why |= OR_Z;
  if (!pr.in_frame) return a;
  a.why |= OR_FRAME;
  float D = f->depth[pr.py * f->W + pr.px];
  if (!depth_ok(D)) return a;
  a.why |= OR_DEPTH;
  if (!pixel_normal(f, pr.px, pr.py, &a.N)) return a;
  a.why |= OR_NORMAL;
  a.q = back_project(f, pr.px, pr.py, (double)D);
  double d = norm(sub(w.vt, a.q));
  a.margin = std::min(a.margin, std::fabs(d - prm->eps_d) / prm->eps_d);
  if (!(d < prm->eps_d)) return a;
  a.why |= OR_DIST;
  double c = dot(w.nt, a.N), ce = std::cos(prm->eps_n_deg * M_PI / 180.0);
  a.margin = std::min(a.margin, std::fabs(c - ce));
  if (!(c > ce)) return a;
  a.why |= OR_ANGLE;
  a.pix = pr.py * f->W + pr.px;
  return a;
}

// ---- block-sparse normal equations: upper blocks (j <= l), full 6x6 each
struct System {
  int m;
  std::map<std::pair<int, int>, B6> blk;
  std::vector<double> rhs;
  double E[6];       // E_data, E_pt, E_reg, E_corr, E_r, E_p (the last two: NEXT-2 only)
  int64_t n_assoc;
  explicit System(int m_) : m(m_), rhs(6 * m_, 0.0), n_assoc(0) { for (int a = 0; a < 6; ++a) E[a] = 0; }
  // H += w * Ja^T Jb for rows r (Ja: rows x 6 for node a, Jb for node b)
  void add_pair(int a, const double* Ja, int b, const double* Jb, int rows, double w) {
    if (a <= b) {
      B6& B = blk[std::make_pair(a, b)];
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          double s = 0;
          for (int r = 0; r < rows; ++r) s += Ja[6 * r + i] * Jb[6 * r + j];
          B[6 * i + j] += w * s;
        }
    } else {
      B6& B = blk[std::make_pair(b, a)];
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          double s = 0;
          for (int r = 0; r < rows; ++r) s += Jb[6 * r + i] * Ja[6 * r + j];
          B[6 * i + j] += w * s;
        }
    }
  }
  // rhs_a -= w * Ja^T r
  void add_rhs(int a, const double* Ja, const double* r, int rows, double w) {
    for (int i = 0; i < 6; ++i) {
      double s = 0;
      for (int q = 0; q < rows; ++q) s += Ja[6 * q + i] * r[q];
      rhs[6 * a + i] -= w * s;
    }
  }
};

// J_pt,j = w_j R [-[a_j]x, I]  (3x6), from dv~/d(dtheta_j) = -w_j R [a_j]x (left update, R-A18)
void jac_point(const M3& R, double wj, const V3& a, double* J) {
  // -[a]x = [[0, a2, -a1], [-a2, 0, a0], [a1, -a0, 0]]
  double S[9] = {0, a[2], -a[1], -a[2], 0, a[0], a[1], -a[0], 0};
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      double s = 0, t = 0;
      for (int l = 0; l < 3; ++l) { s += R[3 * r + l] * S[3 * l + c]; }
      t = R[3 * r + c];
      J[6 * r + c] = wj * s;
      J[6 * r + 3 + c] = wj * t;
    }
  }
}

// Point term rows for one associated point: plane (1 row) and point (3 rows)
void point_rows(const M3& R, const Warped& w, const Assoc& as, int k,
                double* Jpl /*k x 6*/, double* Jpt /*k x 18*/, double* rpl, double* rpt) {
  // Eq. 8: r_pl = N^T (v~ - q); north_star point-to-point: r_pt = v~ - q
  V3 d = sub(w.vt, as.q);
  *rpl = dot(as.N, d);
  rpt[0] = d[0]; rpt[1] = d[1]; rpt[2] = d[2];
  V3 np = mulT(R, as.N);   // n' = R^T N
  for (int s = 0; s < k; ++s) {
    V3 c = cross(w.a[s], np);   // d r_pl / d dtheta_j = w_j (a_j x n')^T
    for (int i = 0; i < 3; ++i) {
      Jpl[6 * s + i] = w.wn[s] * c[i];
      Jpl[6 * s + 3 + i] = w.wn[s] * np[i];
    }
    jac_point(R, w.wn[s], w.a[s], Jpt + 18 * s);
  }
}

// Eq. 6, alpha = 1, directed edges (R-A14):
// e = R_j (g_l - g_j) + g_j + t_j - g_l - t_l; J_j = [-[b]x, I], J_l = [0, -I], b = R_j (g_l - g_j)
void reg_edge(const or_problem* p, const double* Rt, int j, int l, double* e, double* Jj, double* Jl) {
  V3 gj = load3(p->g + 3 * j), gl = load3(p->g + 3 * l);
  V3 b = mul(node_R(Rt, j), sub(gl, gj));
  V3 ev = sub(add(add(b, gj), node_t(Rt, j)), add(gl, node_t(Rt, l)));
  e[0] = ev[0]; e[1] = ev[1]; e[2] = ev[2];
  double S[9] = {0, b[2], -b[1], -b[2], 0, b[0], b[1], -b[0], 0};   // -[b]x
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      Jj[6 * r + c] = S[3 * r + c];
      Jj[6 * r + 3 + c] = (r == c) ? 1.0 : 0.0;
      Jl[6 * r + c] = 0.0;
      Jl[6 * r + 3 + c] = (r == c) ? -1.0 : 0.0;
    }
}

// Eq. 9, squared 3-vector residual (R-A12): e_f = warp(V_f) - V'_f
bool feature_rows(const or_problem* p, int k, const double* Rt, const double* pose, int f,
                  const int32_t* fidx, const double* fw, Warped* w, double* e, double* J) {
  V3 v = load3(p->fsrc + 3 * f);
  *w = warp_point(v, v3(0, 0, 1), k, fidx + k * f, fw + k * f, p->g, Rt, pose);
  double W = 0;
  for (int s = 0; s < k; ++s) W += fw[k * f + s];
  if (!(W > 0)) return false;
  V3 d = sub(w->vt, load3(p->fdst + 3 * f));
  e[0] = d[0]; e[1] = d[1]; e[2] = d[2];
  M3 R = pose_R(pose);
  for (int s = 0; s < k; ++s) jac_point(R, w->wn[s], w->a[s], J + 18 * s);
  return true;
}

void wraw_of(const or_problem* p, int k, int64_t i, double* wr) {
  for (int s = 0; s < k; ++s) wr[s] = (double)p->w[k * i + s];
}

// O3a-d, O3g for the points [i0, i1): data (Eq. 8) and dense point-to-point terms
// ---- NEXT-2 (Eq. 10): pose priors.  Scope orientation O = R^T (R world->camera)
// as ZYX Euler angles O = Rz(psi) Ry(theta) Rx(phi) ("ZYX", A38); scope position
// c = -R^T T, the camera centre in the world frame (A39).
V3 euler_zyx(const M3& O) {
  double s = -O[6];
  s = s > 1.0 ? 1.0 : (s < -1.0 ? -1.0 : s);
  return v3(std::atan2(O[3], O[0]), std::asin(s), std::atan2(O[7], O[8]));
}
double wrap_pi(double a) {   // to (-pi, pi]
  while (a > M_PI) a -= 2.0 * M_PI;
  while (a <= -M_PI) a += 2.0 * M_PI;
  return a;
}
M3 transpose(const M3& A) {
  M3 T;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * i + j] = A[3 * j + i];
  return T;
}
// r = [wrap(e(O) - e(O0)); c - c0], J = d r / d[dphi, dtau] (6x6 row-major) under A37's increment:
//  O' = Exp(dphi)^T O = Exp(-dphi) O, a left (spatial) rotation by -dphi, and d e = E_s^-1 omega
//  with E_s = [e_z, Rz(psi) e_y, Rz(psi) Ry(theta) e_x] (the Euler rates -> angular velocity map);
//  c' = -Exp(-dphi)(R^T T + dtau) = c - dtau + [c]x dphi to first order.
// Returns 1 (E_r rows zeroed) at gimbal lock |cos theta| < 1e-6.
int pose_prior(const double* prior, const double* cur, double* r, double* J) {
  const M3 O = transpose(pose_R(cur)), O0 = transpose(pose_R(prior));
  const V3 e = euler_zyx(O), e0 = euler_zyx(O0);
  const V3 c = scale(mulT(pose_R(cur), pose_T(cur)), -1.0), c0 = scale(mulT(pose_R(prior), pose_T(prior)), -1.0);
  for (int a = 0; a < 36; ++a) J[a] = 0.0;
  for (int a = 0; a < 3; ++a) { r[a] = wrap_pi(e[a] - e0[a]); r[3 + a] = c[a] - c0[a]; }
  // E_p rows: [ [c]x , -I ]
  const double C[9] = {0, -c[2], c[1], c[2], 0, -c[0], -c[1], c[0], 0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      J[6 * (3 + i) + j] = C[3 * i + j];
      J[6 * (3 + i) + 3 + j] = (i == j) ? -1.0 : 0.0;
    }
  const double cps = std::cos(e[0]), sps = std::sin(e[0]), cth = std::cos(e[1]), sth = std::sin(e[1]);
  if (std::fabs(cth) < 1e-6) { r[0] = r[1] = r[2] = 0.0; return 1; }
  // E_s (columns e_z, Rz e_y, Rz Ry e_x), inverted by the 3x3 adjugate
  const double Es[9] = {0.0, -sps, cps * cth,
                        0.0, cps, sps * cth,
                        1.0, 0.0, -sth};
  double inv[9];
  const double det = Es[0] * (Es[4] * Es[8] - Es[5] * Es[7]) - Es[1] * (Es[3] * Es[8] - Es[5] * Es[6]) +
                     Es[2] * (Es[3] * Es[7] - Es[4] * Es[6]);
  inv[0] = (Es[4] * Es[8] - Es[5] * Es[7]) / det; inv[1] = (Es[2] * Es[7] - Es[1] * Es[8]) / det;
  inv[2] = (Es[1] * Es[5] - Es[2] * Es[4]) / det; inv[3] = (Es[5] * Es[6] - Es[3] * Es[8]) / det;
  inv[4] = (Es[0] * Es[8] - Es[2] * Es[6]) / det; inv[5] = (Es[2] * Es[3] - Es[0] * Es[5]) / det;
  inv[6] = (Es[3] * Es[7] - Es[4] * Es[6]) / det; inv[7] = (Es[1] * Es[6] - Es[0] * Es[7]) / det;
  inv[8] = (Es[0] * Es[4] - Es[1] * Es[3]) / det;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[6 * i + j] = -inv[3 * i + j];   // omega = -dphi
  return 0;
}

// NEXT-2 (A37): with the pose unknown, v~ = R (Exp(dphi) x_hat + dtau) + T, so
// dv~/d[dphi, dtau] = R [-[x_hat]x, I]: the pose enters every point / feature row like a node
// of weight 1 with a = x_hat; its rows are appended as slot k with unknown id m.
void pose_slot_rows(const M3& R, const Warped& w, const Assoc* as, double* Jpl, double* Jpt) {
  if (as) {
    V3 np = mulT(R, as->N);
    V3 c = cross(w.x_hat, np);
    for (int i = 0; i < 3; ++i) { Jpl[i] = c[i]; Jpl[3 + i] = np[i]; }
  }
  jac_point(R, 1.0, w.x_hat, Jpt);
}

void assemble_points(const or_params* prm, const or_problem* p, const or_frame* f, const double* pose,
                     const double* Rt, int64_t i0, int64_t i1, System* S) {
  const int k = prm->k;
  const int ks = k + (prm->joint_pose ? 1 : 0);   // slots incl. the pose (unknown m)
  M3 R = pose_R(pose);
  double Jpl[9 * 6], Jpt[9 * 18], rpl, rpt[3];
  int32_t ids[9];
  for (int64_t i = i0; i < i1; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    Warped w = warp_point(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, Rt, pose);
    Assoc as = associate_point(prm, f, w);
    if (as.pix < 0) continue;
    S->n_assoc++;
    point_rows(R, w, as, k, Jpl, Jpt, &rpl, rpt);
    for (int a = 0; a < k; ++a) ids[a] = p->idx[k * i + a];
    if (ks > k) { pose_slot_rows(R, w, &as, Jpl + 6 * k, Jpt + 18 * k); ids[k] = p->m; }
    S->E[0] += rpl * rpl;
    S->E[1] += rpt[0] * rpt[0] + rpt[1] * rpt[1] + rpt[2] * rpt[2];
    for (int a = 0; a < ks; ++a) {
      int ja = ids[a];
      for (int b = 0; b < ks; ++b) {
        int jb = ids[b];
        if (ja > jb || (ja == jb && a > b)) continue;   // each unordered slot pair once
        S->add_pair(ja, Jpl + 6 * a, jb, Jpl + 6 * b, 1, prm->w_data);
        S->add_pair(ja, Jpt + 18 * a, jb, Jpt + 18 * b, 3, prm->w_pt);
        if (ja == jb && a != b) {   // same node in two slots: add the mirrored product too
          S->add_pair(jb, Jpl + 6 * b, ja, Jpl + 6 * a, 1, prm->w_data);
          S->add_pair(jb, Jpt + 18 * b, ja, Jpt + 18 * a, 3, prm->w_pt);
        }
      }
      S->add_rhs(ja, Jpl + 6 * a, &rpl, 1, prm->w_data);
      S->add_rhs(ja, Jpt + 18 * a, rpt, 3, prm->w_pt);
    }
  }
}

void assemble(const or_params* prm, const or_problem* p, const or_frame* f, const double* pose, const double* Rt,
              const int32_t* fidx, const double* fw, System* S) {
  const int k = prm->k;
  if (g_threads <= 1) {
    assemble_points(prm, p, f, pose, Rt, 0, p->n, S);
  } else {   // T contiguous point ranges, merged in range order
    const int T = g_threads;
    std::vector<System> part(T, System(S->m));
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) assemble_points(prm, p, f, pose, Rt, p->n * t / T, p->n * (t + 1) / T, &part[t]);
    for (int t = 0; t < T; ++t) {
      for (const auto& kv : part[t].blk) {
        B6& B = S->blk[kv.first];
        for (int a = 0; a < 36; ++a) B[a] += kv.second[a];
      }
      for (int i = 0; i < 6 * S->m; ++i) S->rhs[i] += part[t].rhs[i];
      for (int a = 0; a < 4; ++a) S->E[a] += part[t].E[a];
      S->n_assoc += part[t].n_assoc;
    }
  }
  // O3e: regulariser
  double e[3], Jj[18], Jl[18];
  for (int j = 0; j < p->m; ++j)
    for (int s = 0; s < prm->n_nbr; ++s) {
      int l = p->nbr[prm->n_nbr * j + s];
      if (l < 0) continue;
      reg_edge(p, Rt, j, l, e, Jj, Jl);
      S->E[2] += e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
      S->add_pair(j, Jj, j, Jj, 3, prm->w_reg);
      S->add_pair(l, Jl, l, Jl, 3, prm->w_reg);
      S->add_pair(j, Jj, l, Jl, 3, prm->w_reg);
      S->add_rhs(j, Jj, e, 3, prm->w_reg);
      S->add_rhs(l, Jl, e, 3, prm->w_reg);
    }
  // O3f: features (NEXT-2: plus the pose slot, A37)
  const int ks = k + (prm->joint_pose ? 1 : 0);
  double Jf[9 * 18];
  int32_t ids[9];
  for (int q = 0; q < p->nf; ++q) {
    Warped w;
    if (!feature_rows(p, k, Rt, pose, q, fidx, fw, &w, e, Jf)) continue;
    for (int a = 0; a < k; ++a) ids[a] = fidx[k * q + a];
    if (ks > k) { pose_slot_rows(pose_R(pose), w, nullptr, nullptr, Jf + 18 * k); ids[k] = p->m; }
    S->E[3] += e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
    for (int a = 0; a < ks; ++a) {
      int ja = ids[a];
      for (int b = 0; b < ks; ++b) {
        int jb = ids[b];
        if (ja > jb || (ja == jb && a > b)) continue;
        S->add_pair(ja, Jf + 18 * a, jb, Jf + 18 * b, 3, prm->w_corr);
        if (ja == jb && a != b) S->add_pair(jb, Jf + 18 * b, ja, Jf + 18 * a, 3, prm->w_corr);
      }
      S->add_rhs(ja, Jf + 18 * a, e, 3, prm->w_corr);
    }
  }
  // NEXT-2: the pose priors of Eq. 10 on unknown m (A38-A39)
  if (prm->joint_pose) {
    double r[6], J[36];
    pose_prior(f->pose, pose, r, J);
    S->E[4] = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    S->E[5] = r[3] * r[3] + r[4] * r[4] + r[5] * r[5];
    S->add_pair(p->m, J, p->m, J, 3, prm->w_r);
    S->add_pair(p->m, J + 18, p->m, J + 18, 3, prm->w_p);
    S->add_rhs(p->m, J, r, 3, prm->w_r);
    S->add_rhs(p->m, J + 18, r + 3, 3, prm->w_p);
  }
}

double total_energy(const or_params* prm, const double* E) {
  double s = prm->w_data * E[0] + prm->w_pt * E[1] + prm->w_reg * E[2] + prm->w_corr * E[3];
  if (prm->joint_pose) s += prm->w_r * E[4] + prm->w_p * E[5];
  return s;
}

// ---- linear algebra for O3h
// y = (H + lambda I) x with H given by its upper blocks
void spmv(const System& S, double lambda, const std::vector<double>& x, std::vector<double>& y) {
  std::fill(y.begin(), y.end(), 0.0);
  for (std::map<std::pair<int, int>, B6>::const_iterator it = S.blk.begin(); it != S.blk.end(); ++it) {
    int j = it->first.first, l = it->first.second;
    const B6& B = it->second;
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        y[6 * j + a] += B[6 * a + b] * x[6 * l + b];
        if (j != l) y[6 * l + b] += B[6 * a + b] * x[6 * j + a];
      }
  }
  for (size_t i = 0; i < y.size(); ++i) y[i] += lambda * x[i];
}

// in-place Cholesky A = L L^T (n x n, row-major); false if not positive definite
bool cholesky(std::vector<double>& A, int n) {
  for (int j = 0; j < n; ++j) {
    double s = A[j * n + j];
    for (int l = 0; l < j; ++l) s -= A[j * n + l] * A[j * n + l];
    if (!(s > 0)) return false;
    double d = std::sqrt(s);
    A[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A[i * n + j];
      for (int l = 0; l < j; ++l) t -= A[i * n + l] * A[j * n + l];
      A[i * n + j] = t / d;
    }
  }
  return true;
}
void chol_solve(const std::vector<double>& L, int n, const double* b, double* x) {
  std::vector<double> y(n);
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int l = 0; l < i; ++l) s -= L[i * n + l] * y[l];
    y[i] = s / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int l = i + 1; l < n; ++l) s -= L[l * n + i] * x[l];
    x[i] = s / L[i * n + i];
  }
}

// Block-Jacobi preconditioner M_j = (H_jj + lambda I + mu_j I)^-1, mu_j = 1e-9 tr(H_jj)/6 (R-A17)
void block_jacobi(const System& S, double lambda, std::vector<double>& Minv) {
  Minv.assign(36 * S.m, 0.0);
  for (int j = 0; j < S.m; ++j) {
    std::vector<double> A(36, 0.0);
    std::map<std::pair<int, int>, B6>::const_iterator it = S.blk.find(std::make_pair(j, j));
    if (it != S.blk.end()) for (int a = 0; a < 36; ++a) A[a] = it->second[a];
    double tr = A[0] + A[7] + A[14] + A[21] + A[28] + A[35];
    double mu = 1e-9 * tr / 6.0;
    for (int a = 0; a < 6; ++a) A[7 * a] += lambda + mu;
    std::vector<double> L = A;
    if (!cholesky(L, 6)) continue;   // leaves M_j = 0 (never happens with lambda > 0)
    for (int c = 0; c < 6; ++c) {
      double e[6] = {0, 0, 0, 0, 0, 0}, col[6];
      e[c] = 1.0;
      chol_solve(L, 6, e, col);
      for (int r = 0; r < 6; ++r) Minv[36 * j + 6 * r + c] = col[r];
    }
  }
}

void apply_M(const std::vector<double>& Minv, int m, const std::vector<double>& r, std::vector<double>& z) {
  for (int j = 0; j < m; ++j)
    for (int a = 0; a < 6; ++a) {
      double s = 0;
      for (int b = 0; b < 6; ++b) s += Minv[36 * j + 6 * a + b] * r[6 * j + b];
      z[6 * j + a] = s;
    }
}
double vdot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// PCG from x0 = 0: fixed P iterations (MIRROR) or to a
// relative residual of 1e-12 (EXACT for large systems).  Early stop if
// r.z == 0 or p.Ap <= 0.
int pcg(const System& S, double lambda, const std::vector<double>& b, int max_it, double rel_tol,
        std::vector<double>& x) {
  const int n = 6 * S.m;
  std::vector<double> Minv, r(b), z(n), p(n), Ap(n);
  block_jacobi(S, lambda, Minv);
  x.assign(n, 0.0);
  apply_M(Minv, S.m, r, z);
  p = z;
  double rz = vdot(r, z), b2 = vdot(b, b);
  int it = 0;
  for (; it < max_it; ++it) {
    if (rel_tol > 0 && vdot(r, r) <= rel_tol * rel_tol * b2) break;
    if (rz == 0) break;
    spmv(S, lambda, p, Ap);
    double pAp = vdot(p, Ap);
    if (!(pAp > 0)) break;
    double alpha = rz / pAp;
    for (int i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; }
    apply_M(Minv, S.m, r, z);
    double rz_new = vdot(r, z);
    double beta = rz_new / rz;
    rz = rz_new;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  return it;
}

int solve_system(const System& S, double lambda, int mode, int pcg_iters, std::vector<double>& x) {
  const int n = 6 * S.m;
  if (mode == 1) return pcg(S, lambda, S.rhs, pcg_iters, 0.0, x);
  if (n <= 600) {   // EXACT, small: dense Cholesky of H + lambda I
    std::vector<double> A((size_t)n * n, 0.0);
    for (std::map<std::pair<int, int>, B6>::const_iterator it = S.blk.begin(); it != S.blk.end(); ++it) {
      int j = it->first.first, l = it->first.second;
      for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) {
          A[(size_t)(6 * j + a) * n + 6 * l + b] += it->second[6 * a + b];
          if (j != l) A[(size_t)(6 * l + b) * n + 6 * j + a] += it->second[6 * a + b];
        }
    }
    for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += lambda;
    x.assign(n, 0.0);
    if (!cholesky(A, n)) return -1;
    chol_solve(A, n, S.rhs.data(), x.data());
    return 0;
  }
  return pcg(S, lambda, S.rhs, 20 * n, 1e-12, x);
}

// O3i: R_j <- Exp(dtheta_j) R_j, t_j += dt_j (R-A18)
void update_nodes(int m, const std::vector<double>& x, double* Rt) {
  for (int j = 0; j < m; ++j) {
    double w[3] = {x[6 * j], x[6 * j + 1], x[6 * j + 2]}, E[9];
    or_exp(w, E);
    M3 Em, Rj = node_R(Rt, j);
    for (int a = 0; a < 9; ++a) Em[a] = E[a];
    M3 Rn = matmul(Em, Rj);
    for (int a = 0; a < 9; ++a) Rt[12 * j + a] = Rn[a];
    for (int a = 0; a < 3; ++a) Rt[12 * j + 9 + a] += x[6 * j + 3 + a];
  }
}

// NEXT-2, A37: R <- R Exp(dphi), T <- T + R dtau (x[0..6) = [dphi, dtau])
void update_pose(const double* x, double* pose) {
  double w[3] = {x[0], x[1], x[2]}, E[9];
  or_exp(w, E);
  M3 Em, R = pose_R(pose);
  for (int a = 0; a < 9; ++a) Em[a] = E[a];
  const V3 dT = mul(R, v3(x[3], x[4], x[5]));
  M3 Rn = matmul(R, Em);
  for (int a = 0; a < 9; ++a) pose[a] = Rn[a];
  for (int a = 0; a < 3; ++a) pose[9 + a] += dT[a];
}

int n_unknown_blocks(const or_params* prm, const or_problem* p) { return p->m + (prm->joint_pose ? 1 : 0); }

int64_t system_impl(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                    const double* pose, const int32_t* fidx, const double* fw, int64_t cap, int32_t* brow,
                    int32_t* bcol, double* bval, double* rhs, double* energy, int64_t* n_assoc);
int64_t residuals_impl(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                       const double* pose, const int32_t* pix_frozen, const int32_t* fidx, const double* fw,
                       int64_t cap_rows, double* r, double* J);
void register_impl(const or_params* prm, const or_problem* p, const or_frame* f, double* Rt, double* pose,
                   double* energy, int64_t* n_assoc, int32_t* accepted);

void feature_skin(const or_problem* p, int k, std::vector<int32_t>& fidx, std::vector<double>& fw) {
  fidx.assign((size_t)k * p->nf, 0);
  fw.assign((size_t)k * p->nf, 0.0);
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int q = 0; q < p->nf; ++q)
    skin_one(load3(p->fsrc + 3 * q), p->m, p->g, k, &fidx[k * q], &fw[k * q], nullptr);
}

}  // namespace

extern "C" {

void or_frame_prep(const or_frame* f, double* q, double* N, uint8_t* dvalid, uint8_t* nvalid) {
  for (int y = 0; y < f->H; ++y)
    for (int x = 0; x < f->W; ++x) {
      int i = y * f->W + x;
      float D = f->depth[i];
      dvalid[i] = depth_ok(D) ? 1 : 0;
      V3 qq = dvalid[i] ? back_project(f, x, y, (double)D) : v3(0, 0, 0);
      V3 nn = v3(0, 0, 0);
      nvalid[i] = pixel_normal(f, x, y, &nn) ? 1 : 0;
      for (int a = 0; a < 3; ++a) { q[3 * i + a] = qq[a]; N[3 * i + a] = nn[a]; }
    }
}

void or_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }

void or_skin(int64_t nq, const float* p, int32_t m, const float* g, int32_t k,
             int32_t* idx, double* w, double* margin) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int64_t i = 0; i < nq; ++i)
    skin_one(load3(p + 3 * i), m, g, k, idx + k * i, w + k * i, margin ? margin + i : nullptr);
}

void or_exp(const double w[3], double R[9]) {
  double th = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};   // [w]x
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int l = 0; l < 3; ++l) s += K[3 * i + l] * K[3 * l + j];
      K2[3 * i + j] = s;
    }
  double A, B;
  if (th < 1e-12) { A = 1.0; B = 0.0; }                 // first order
  else { A = std::sin(th) / th; B = (1.0 - std::cos(th)) / (th * th); }
  for (int i = 0; i < 9; ++i) R[i] = ((i % 4) == 0 ? 1.0 : 0.0) + A * K[i] + B * K2[i];
}

void or_warp(const or_problem* p, int32_t k, const double* Rt, const double pose[12],
             double* x_hat, double* n_hat, double* vt, double* nt, uint8_t* ok) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int64_t i = 0; i < p->n; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    Warped w = warp_point(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, Rt, pose);
    ok[i] = w.ok ? 1 : 0;
    for (int a = 0; a < 3; ++a) {
      x_hat[3 * i + a] = w.ok ? w.x_hat[a] : 0.0;
      n_hat[3 * i + a] = w.ok ? w.m_hat[a] / norm(w.m_hat) : 0.0;
      vt[3 * i + a] = w.ok ? w.vt[a] : 0.0;
      nt[3 * i + a] = w.ok ? w.nt[a] : 0.0;
    }
  }
}

void or_associate(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                  int32_t* pix, uint8_t* why, double* margin) {
  const int k = prm->k;
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int64_t i = 0; i < p->n; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    Warped w = warp_point(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, Rt, f->pose);
    Assoc a = associate_point(prm, f, w);
    pix[i] = a.pix;
    why[i] = a.why;
    margin[i] = a.margin;
  }
}

int64_t or_system(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                  const int32_t* fidx, const double* fw, int64_t cap,
                  int32_t* brow, int32_t* bcol, double* bval, double* rhs, double energy[5],
                  int64_t* n_assoc) {
  or_params q = *prm;
  q.joint_pose = 0;
  double E7[7];
  const int64_t nb = system_impl(&q, p, f, Rt, f->pose, fidx, fw, cap, brow, bcol, bval, rhs, E7, n_assoc);
  for (int a = 0; a < 4; ++a) energy[a] = E7[a];
  energy[4] = E7[6];
  return nb;
}

int64_t or_system_pose(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                       const double pose_cur[12], const int32_t* fidx, const double* fw, int64_t cap,
                       int32_t* brow, int32_t* bcol, double* bval, double* rhs, double energy[7],
                       int64_t* n_assoc) {
  or_params q = *prm;
  q.joint_pose = 1;
  return system_impl(&q, p, f, Rt, pose_cur, fidx, fw, cap, brow, bcol, bval, rhs, energy, n_assoc);
}

}  // extern "C"

namespace {
int64_t system_impl(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                    const double* pose, const int32_t* fidx, const double* fw, int64_t cap, int32_t* brow,
                    int32_t* bcol, double* bval, double* rhs, double* energy, int64_t* n_assoc) {
  System S(n_unknown_blocks(prm, p));
  assemble(prm, p, f, pose, Rt, fidx, fw, &S);
  int64_t nb = 0;
  for (std::map<std::pair<int, int>, B6>::const_iterator it = S.blk.begin(); it != S.blk.end(); ++it, ++nb) {
    if (nb >= cap) continue;
    brow[nb] = it->first.first;
    bcol[nb] = it->first.second;
    for (int a = 0; a < 36; ++a) bval[36 * nb + a] = it->second[a];
  }
  for (int i = 0; i < 6 * S.m; ++i) rhs[i] = S.rhs[i];
  for (int a = 0; a < 6; ++a) energy[a] = S.E[a];
  energy[6] = total_energy(prm, S.E);
  *n_assoc = S.n_assoc;
  return nb;
}
}  // namespace

extern "C" {
int64_t or_residuals(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                     const int32_t* pix_frozen, const int32_t* fidx, const double* fw,
                     int64_t cap_rows, double* r, double* J) {
  or_params q = *prm;
  q.joint_pose = 0;
  return residuals_impl(&q, p, f, Rt, f->pose, pix_frozen, fidx, fw, cap_rows, r, J);
}

int64_t or_residuals_pose(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                          const double pose_cur[12], const int32_t* pix_frozen, const int32_t* fidx,
                          const double* fw, int64_t cap_rows, double* r, double* J) {
  or_params q = *prm;
  q.joint_pose = 1;
  return residuals_impl(&q, p, f, Rt, pose_cur, pix_frozen, fidx, fw, cap_rows, r, J);
}
}  // extern "C"

namespace {
int64_t residuals_impl(const or_params* prm, const or_problem* p, const or_frame* f, const double* Rt,
                       const double* pose, const int32_t* pix_frozen, const int32_t* fidx, const double* fw,
                       int64_t cap_rows, double* r, double* J) {
  const int k = prm->k, ncol = 6 * n_unknown_blocks(prm, p);
  const bool joint = prm->joint_pose != 0;
  M3 R = pose_R(pose);
  int64_t row = 0;
  double Jpl[8 * 6], Jpt[8 * 18], rpl, rpt[3];
  const double sd = std::sqrt(prm->w_data), sp = std::sqrt(prm->w_pt);
  const double sr = std::sqrt(prm->w_reg), sc = std::sqrt(prm->w_corr);
  for (int64_t i = 0; i < p->n; ++i) {
    if (pix_frozen[i] < 0) continue;
    double wr[8];
    wraw_of(p, k, i, wr);
    Warped w = warp_point(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, Rt, pose);
    if (!w.ok) continue;
    Assoc as;
    int px = pix_frozen[i] % f->W, py = pix_frozen[i] / f->W;
    as.q = back_project(f, px, py, (double)f->depth[pix_frozen[i]]);
    if (!pixel_normal(f, px, py, &as.N)) continue;
    point_rows(R, w, as, k, Jpl, Jpt, &rpl, rpt);
    if (row + 4 > cap_rows) return -1;
    double* J0 = J + (size_t)row * ncol;
    std::memset(J0, 0, sizeof(double) * 4 * ncol);
    r[row] = sd * rpl;
    for (int c = 0; c < 3; ++c) r[row + 1 + c] = sp * rpt[c];
    for (int s = 0; s < k; ++s) {
      int j = p->idx[k * i + s];
      for (int c = 0; c < 6; ++c) {
        J0[6 * j + c] += sd * Jpl[6 * s + c];
        for (int q = 0; q < 3; ++q) J0[(size_t)(1 + q) * ncol + 6 * j + c] += sp * Jpt[18 * s + 6 * q + c];
      }
    }
    if (joint) {   // pose columns (A37)
      double Jplp[6], Jptp[18];
      pose_slot_rows(R, w, &as, Jplp, Jptp);
      const int j = p->m;
      for (int c = 0; c < 6; ++c) {
        J0[6 * j + c] += sd * Jplp[c];
        for (int q = 0; q < 3; ++q) J0[(size_t)(1 + q) * ncol + 6 * j + c] += sp * Jptp[6 * q + c];
      }
    }
    row += 4;
  }
  double e[3], Jj[18], Jl[18];
  for (int j = 0; j < p->m; ++j)
    for (int s = 0; s < prm->n_nbr; ++s) {
      int l = p->nbr[prm->n_nbr * j + s];
      if (l < 0) continue;
      reg_edge(p, Rt, j, l, e, Jj, Jl);
      if (row + 3 > cap_rows) return -1;
      double* J0 = J + (size_t)row * ncol;
      std::memset(J0, 0, sizeof(double) * 3 * ncol);
      for (int q = 0; q < 3; ++q) {
        r[row + q] = sr * e[q];
        for (int c = 0; c < 6; ++c) {
          J0[(size_t)q * ncol + 6 * j + c] += sr * Jj[6 * q + c];
          J0[(size_t)q * ncol + 6 * l + c] += sr * Jl[6 * q + c];
        }
      }
      row += 3;
    }
  double Jf[8 * 18];
  for (int q = 0; q < p->nf; ++q) {
    Warped w;
    if (!feature_rows(p, k, Rt, pose, q, fidx, fw, &w, e, Jf)) continue;
    if (row + 3 > cap_rows) return -1;
    double* J0 = J + (size_t)row * ncol;
    std::memset(J0, 0, sizeof(double) * 3 * ncol);
    double Jfp[18];
    if (joint) pose_slot_rows(R, w, nullptr, nullptr, Jfp);
    for (int a = 0; a < 3; ++a) {
      r[row + a] = sc * e[a];
      for (int s = 0; s < k; ++s) {
        int j = fidx[k * q + s];
        for (int c = 0; c < 6; ++c) J0[(size_t)a * ncol + 6 * j + c] += sc * Jf[18 * s + 6 * a + c];
      }
      if (joint)
        for (int c = 0; c < 6; ++c) J0[(size_t)a * ncol + 6 * p->m + c] += sc * Jfp[6 * a + c];
    }
    row += 3;
  }
  if (joint) {   // Eq. 10 prior rows (A38-A39), last
    double rr[6], Jp[36];
    pose_prior(f->pose, pose, rr, Jp);
    if (row + 6 > cap_rows) return -1;
    double* J0 = J + (size_t)row * ncol;
    std::memset(J0, 0, sizeof(double) * 6 * ncol);
    for (int a = 0; a < 6; ++a) {
      const double sw = std::sqrt(a < 3 ? prm->w_r : prm->w_p);
      r[row + a] = sw * rr[a];
      for (int c = 0; c < 6; ++c) J0[(size_t)a * ncol + 6 * p->m + c] = sw * Jp[6 * a + c];
    }
    row += 6;
  }
  return row;
}
}  // namespace

extern "C" {

int32_t or_solve(int32_t m, int64_t nblk, const int32_t* brow, const int32_t* bcol, const double* bval,
                 const double* rhs, double lambda, int32_t mode, int32_t pcg_iters, double* x) {
  System S(m);
  for (int64_t b = 0; b < nblk; ++b) {
    B6& B = S.blk[std::make_pair(brow[b], bcol[b])];
    for (int a = 0; a < 36; ++a) B[a] = bval[36 * b + a];
  }
  for (int i = 0; i < 6 * m; ++i) S.rhs[i] = rhs[i];
  std::vector<double> xs;
  int32_t it = solve_system(S, lambda, mode, pcg_iters, xs);
  for (int i = 0; i < 6 * m; ++i) x[i] = xs[i];
  return it;
}

void or_register(const or_params* prm, const or_problem* p, const or_frame* f, double* Rt,
                 double* energy, int64_t* n_assoc, int32_t* accepted) {
  or_params q = *prm;
  q.joint_pose = 0;
  double pose[12];
  for (int a = 0; a < 12; ++a) pose[a] = f->pose[a];
  std::vector<double> E7(7 * (size_t)(prm->gn_iters + 1));
  register_impl(&q, p, f, Rt, pose, E7.data(), n_assoc, accepted);
  for (int it = 0; it <= prm->gn_iters; ++it) {
    for (int a = 0; a < 4; ++a) energy[5 * it + a] = E7[7 * it + a];
    energy[5 * it + 4] = E7[7 * it + 6];
  }
}

void or_register_pose(const or_params* prm, const or_problem* p, const or_frame* f, double* Rt, double* pose_io,
                      double* energy, int64_t* n_assoc, int32_t* accepted) {
  or_params q = *prm;
  q.joint_pose = 1;
  register_impl(&q, p, f, Rt, pose_io, energy, n_assoc, accepted);
}

void or_euler_zyx(const double O[9], double e[3]) {
  M3 M;
  for (int a = 0; a < 9; ++a) M[a] = O[a];
  V3 v = euler_zyx(M);
  for (int a = 0; a < 3; ++a) e[a] = v[a];
}

int32_t or_pose_prior(const double prior[12], const double cur[12], double r[6], double J[36]) {
  return pose_prior(prior, cur, r, J);
}
}  // extern "C"

namespace {
// O3 (+ NEXT-2 when prm->joint_pose): fixed-G Gauss-Newton or LM over the nodes and, jointly,
// the pose (unknown m); energy rows of 7 (E_data, E_pt, E_reg, E_corr, E_r, E_p, total).
void register_impl(const or_params* prm, const or_problem* p, const or_frame* f, double* Rt, double* pose,
                   double* energy, int64_t* n_assoc, int32_t* accepted) {
  std::vector<int32_t> fidx;
  std::vector<double> fw;
  feature_skin(p, prm->k, fidx, fw);   // O1 on the (fixed) node positions
  const int nu = n_unknown_blocks(prm, p);
  auto step = [&](const std::vector<double>& x) {
    update_nodes(p->m, x, Rt);
    if (prm->joint_pose) update_pose(x.data() + 6 * p->m, pose);
  };
  auto record = [&](int it, const System& S) {
    for (int a = 0; a < 6; ++a) energy[7 * it + a] = S.E[a];
    energy[7 * it + 6] = total_energy(prm, S.E);
    n_assoc[it] = S.n_assoc;
  };
  if (!prm->lm) {
    for (int it = 0; it <= prm->gn_iters; ++it) {
      System S(nu);
      assemble(prm, p, f, pose, Rt, fidx.data(), fw.data(), &S);
      record(it, S);
      if (accepted) accepted[it] = 1;
      if (it == prm->gn_iters) break;   // final energy only
      std::vector<double> x;
      solve_system(S, prm->lambda, prm->solve_mode, prm->pcg_iters, x);
      step(x);
    }
    return;
  }
  // Levenberg-Marquardt, Marquardt damping H + mu diag(H) (R-A29)
  const size_t ns = 12 * (size_t)p->m;
  std::vector<double> base(Rt, Rt + ns);   // last accepted state
  std::vector<double> base_pose(pose, pose + 12);
  System acc(nu);                          // its normal equations
  double E_acc = 0.0, mu = prm->lm_mu0;
  for (int it = 0; it <= prm->gn_iters; ++it) {
    System S(nu);
    assemble(prm, p, f, pose, Rt, fidx.data(), fw.data(), &S);   // at the trial state
    record(it, S);
    const double E = total_energy(prm, S.E);
    const bool ok = it == 0 || E < E_acc;
    if (accepted) accepted[it] = ok ? 1 : 0;
    if (ok) {
      std::copy(Rt, Rt + ns, base.begin());
      std::copy(pose, pose + 12, base_pose.begin());
      acc = S;
      E_acc = E;
      if (it > 0) mu *= 0.5;
    } else {
      std::copy(base.begin(), base.end(), Rt);
      std::copy(base_pose.begin(), base_pose.end(), pose);
      mu *= 10.0;
    }
    if (it == prm->gn_iters) break;   // the final trial is only evaluated
    System D = acc;                   // damped copy: diagonal entries of H times (1 + mu)
    for (int j = 0; j < nu; ++j) {
      std::map<std::pair<int, int>, B6>::iterator d = D.blk.find(std::make_pair(j, j));
      if (d != D.blk.end())
        for (int a = 0; a < 6; ++a) d->second[7 * a] *= 1.0 + mu;
    }
    std::vector<double> x;
    solve_system(D, prm->lambda, prm->solve_mode, prm->pcg_iters, x);
    step(x);   // Rt == base here: the step starts from the accepted state
  }
}
}  // namespace

extern "C" {
void or_warp_model(const or_problem* p, int32_t k, const double* Rt, double* xyz_out, double* nrm_out,
                   double* g_out) {
  double pose[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int64_t i = 0; i < p->n; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    Warped w = warp_point(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, Rt, pose);
    for (int a = 0; a < 3; ++a) {
      xyz_out[3 * i + a] = w.ok ? w.x_hat[a] : (double)p->xyz[3 * i + a];
      nrm_out[3 * i + a] = w.ok ? w.nt[a] : (double)p->nrm[3 * i + a];
    }
  }
  for (int j = 0; j < p->m; ++j)   // A26: g_j <- g_j + t_j (then R_j = I, t_j = 0)
    for (int a = 0; a < 3; ++a) g_out[3 * j + a] = (double)p->g[3 * j + a] + Rt[12 * j + 9 + a];
}

int64_t or_fuse(const or_params* prm, const or_model* mdl, const or_frame* f, const float* rgb_obs,
                int32_t frame_index, int32_t m, const float* g,
                double* xyz_out, double* nrm_out, double* rgb_out, double* weight_out, int32_t* stamp_out,
                int32_t* lift_idx, double* lift_w, double* lift_margin,
                int64_t* owner, double* key_margin, uint8_t* why, double* gate_margin) {
  const int W = f->W, H = f->H, k = prm->k;
  const M3 R = pose_R(f->pose);
  const V3 T = pose_T(f->pose);
  const double cd = std::cos(prm->delta_deg * M_PI / 180.0);
  std::vector<double> best(W * H, kInf), second(W * H, kInf);
  for (int i = 0; i < W * H; ++i) owner[i] = -1;
  std::vector<int32_t> pix(mdl->n, -1);
  std::vector<double> dz(mdl->n, 0.0);
  // O5 / Alg. 1: v~ = R v + T, gates, exclusive per pixel with key (|dz|, i)
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int64_t i = 0; i < mdl->n; ++i) {
    V3 vt = add(mul(R, load3(mdl->xyz + 3 * i)), T);
    V3 nt = mul(R, load3(mdl->nrm + 3 * i));
    Proj pr = project(f, vt);
    uint8_t wb = 0;
    double mg = pr.margin;
    if (pr.z_ok) {
      wb |= OR_Z;
      if (pr.in_frame) {
        wb |= OR_FRAME;
        int q = pr.py * W + pr.px;
        float D = f->depth[q];
        V3 N;
        if (depth_ok(D)) {
          wb |= OR_DEPTH;
          if (pixel_normal(f, pr.px, pr.py, &N)) {
            wb |= OR_NORMAL;
            double d = std::fabs(vt[2] - (double)D);
            double tz = std::min(prm->tau_z, prm->trunc);   // Alg. 1 gate and Eq. 11 truncation (R-A20)
            mg = std::min(mg, std::fabs(d - tz) / tz);
            if (d < tz) {
              wb |= OR_DIST;
              double c = dot(nt, N);
              mg = std::min(mg, std::fabs(c - cd));
              if (c > cd) {
                wb |= OR_ANGLE;
                pix[i] = q;
                dz[i] = d;
              }
            }
          }
        }
      }
    }
    why[i] = wb;
    gate_margin[i] = mg;
  }
  for (int64_t i = 0; i < mdl->n; ++i) {   // lexicographic (|dz|, i) minimum per pixel (R-A19)
    if (pix[i] < 0) continue;
    int q = pix[i];
    if (dz[i] < best[q]) { second[q] = best[q]; best[q] = dz[i]; owner[q] = i; }
    else if (dz[i] < second[q]) second[q] = dz[i];
    else if (dz[i] == best[q]) second[q] = dz[i];
  }
  for (int q = 0; q < W * H; ++q) key_margin[q] = second[q] - best[q];
  // copy, then Eq. 12-15 on each pixel's winner (R-A21: 3-D weighted average)
  for (int64_t i = 0; i < mdl->n; ++i) {
    for (int a = 0; a < 3; ++a) {
      xyz_out[3 * i + a] = mdl->xyz[3 * i + a];
      nrm_out[3 * i + a] = mdl->nrm[3 * i + a];
      rgb_out[3 * i + a] = mdl->rgb[3 * i + a];
    }
    weight_out[i] = mdl->weight[i];
    stamp_out[i] = mdl->stamp[i];
  }
  for (int q = 0; q < W * H; ++q) {
    int64_t i = owner[q];
    if (i < 0) continue;
    int px = q % W, py = q / W;
    V3 Q = back_project(f, px, py, (double)f->depth[q]);
    V3 N;
    pixel_normal(f, px, py, &N);
    double om = mdl->weight[i];
    V3 vt = add(mul(R, load3(mdl->xyz + 3 * i)), T);
    V3 nt = mul(R, load3(mdl->nrm + 3 * i));
    V3 pf = scale(add(scale(vt, om), Q), 1.0 / (om + 1.0));                  // Eq. 12 (3-D)
    V3 nf = scale(add(scale(nt, om), N), 1.0 / (om + 1.0));                  // Eq. 14
    nf = scale(nf, 1.0 / norm(nf));
    V3 vw = mulT(R, sub(pf, T)), nw = mulT(R, nf);
    for (int a = 0; a < 3; ++a) {
      xyz_out[3 * i + a] = vw[a];
      nrm_out[3 * i + a] = nw[a];
      if (rgb_obs) rgb_out[3 * i + a] = (om * mdl->rgb[3 * i + a] + (double)rgb_obs[3 * q + a]) / (om + 1.0);  // Eq. 13
    }
    weight_out[i] = std::min(om + 1.0, prm->omega_max);                       // Eq. 15
    stamp_out[i] = frame_index;
  }
  // O6: Alg. 2 Step 3 "else" branch: lift valid, unregistered pixels, row-major
  int64_t nl = 0;
  for (int q = 0; q < W * H; ++q) {
    if (owner[q] >= 0) continue;
    int px = q % W, py = q / W;
    if (!depth_ok(f->depth[q])) continue;
    V3 N;
    if (!pixel_normal(f, px, py, &N)) continue;
    V3 Q = back_project(f, px, py, (double)f->depth[q]);
    V3 vw = mulT(R, sub(Q, T)), nw = mulT(R, N);
    int64_t o = mdl->n + nl;
    for (int a = 0; a < 3; ++a) {
      xyz_out[3 * o + a] = vw[a];
      nrm_out[3 * o + a] = nw[a];
      rgb_out[3 * o + a] = rgb_obs ? (double)rgb_obs[3 * q + a] : 0.0;
    }
    weight_out[o] = 1.0;
    stamp_out[o] = frame_index;
    ++nl;
  }
  // Eq. 2 skinning of the lifted points on the current g (each independent)
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int64_t l = 0; l < nl; ++l) {
    const int64_t o = mdl->n + l;
    float pf[3] = {(float)xyz_out[3 * o], (float)xyz_out[3 * o + 1], (float)xyz_out[3 * o + 2]};   // as the GPU stores it
    skin_one(load3(pf), m, g, k, lift_idx + k * l, lift_w + k * l, lift_margin + l);
  }
  return nl;
}

// O7 (NEXT-1): Alg. 3, "Down sample point cloud according to grid size" read as
// P:597 "setting a fixed box to average points fill inside each 3D box" with the averages of
// S:369 (readings A30-A34), then the deletion test of Alg. 3 line 3 in the form of S:369.
int64_t or_filter(int64_t n, const float* xyz, const float* nrm, const float* rgb, const float* weight,
                  const int32_t* stamp, const int64_t* ids, float grid, int32_t frame_index, int32_t tau_time,
                  float tau_weight, float omega_max, double* xyz_out, double* nrm_out, double* rgb_out,
                  double* weight_out, int32_t* stamp_out, int64_t* ids_out, uint8_t* stable_out,
                  int64_t* cells_out) {
  // the fixed boxes: members of every cell in ascending input index (A30, A31)
  std::map<std::array<int64_t, 3>, std::vector<int64_t>> cells;
  for (int64_t i = 0; i < n; ++i) {
    std::array<int64_t, 3> key;
    for (int a = 0; a < 3; ++a) {
      float q = xyz[3 * i + a] / grid;   // fp32 division and floor: the decision's precision (A30)
      key[a] = (int64_t)floorf(q);
    }
    cells[key].push_back(i);
  }
  if (cells_out) *cells_out = (int64_t)cells.size();
  int64_t o = 0;
  for (const auto& cell : cells) {   // std::map: ascending (kx, ky, kz) (A33)
    const std::vector<int64_t>& mem = cell.second;
    double wsum = 0.0;
    for (int64_t i : mem) wsum += (double)weight[i];
    const bool weighted = wsum > 0.0;
    V3 v = v3(0, 0, 0), nn = v3(0, 0, 0), c = v3(0, 0, 0);
    double den = 0.0;
    int32_t t = std::numeric_limits<int32_t>::min();
    for (int64_t i : mem) {
      const double wi = weighted ? (double)weight[i] : 1.0;
      for (int a = 0; a < 3; ++a) {
        v[a] += wi * (double)xyz[3 * i + a];
        nn[a] += wi * (double)nrm[3 * i + a];
        c[a] += wi * (double)rgb[3 * i + a];
      }
      den += wi;
      t = std::max(t, stamp[i]);
    }
    const double len = std::sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
    const double om = std::min(wsum, (double)omega_max);            // Eq. 15 cap
    // Alg. 3 line 3 as S:369: t_k < frame - tau_time and omega_k < tau_weight -> delete
    if ((int64_t)t < (int64_t)frame_index - (int64_t)tau_time && om < (double)tau_weight) continue;
    for (int a = 0; a < 3; ++a) {
      xyz_out[3 * o + a] = v[a] / den;
      nrm_out[3 * o + a] = len > 0.0 ? nn[a] / len : (double)nrm[3 * mem[0] + a];
      rgb_out[3 * o + a] = c[a] / den;
    }
    weight_out[o] = om;
    stamp_out[o] = t;                                                  // Alg. 3 keeps the max stamp
    ids_out[o] = ids ? ids[mem[0]] : mem[0];
    stable_out[o] = om >= (double)tau_weight ? 1 : 0;                  // S_i (A32)
    ++o;
  }
  return o;
}

// O8 (NEXT-1, Alg. 2 Step 5 "Regenerate node and corresponding rotation and translation"),
// in the form of S:102-104 (reading A36): nodes = the centroids (plain fp64 mean) of the occupied
// axis-aligned cells of size `grid` -- (floor(x/grid), floor(y/grid), floor(z/grid)), each quotient
// an IEEE fp32 division and floor (as A30) -- in ascending (kx, ky, kz) order; R_j = I, t_j = 0;
// N(j) = the n_nbr nearest other nodes by Euclidean distance, ties to the lower index, -1 padded.
// nbr_margin[j]: relative gap between the n_nbr-th and the next distance (1 if none).
int64_t or_regenerate_nodes(int64_t n, const float* xyz, float grid, int32_t n_nbr, double* g_out,
                            int32_t* nbr_out, double* nbr_margin) {
  std::map<std::array<int64_t, 3>, std::vector<int64_t>> cells;
  for (int64_t i = 0; i < n; ++i) {
    std::array<int64_t, 3> key;
    for (int a = 0; a < 3; ++a) key[a] = (int64_t)floorf(xyz[3 * i + a] / grid);
    cells[key].push_back(i);
  }
  int64_t m = 0;
  for (const auto& cell : cells) {   // ascending (kx, ky, kz)
    V3 c = v3(0, 0, 0);
    for (int64_t i : cell.second) c = add(c, load3(xyz + 3 * i));
    c = scale(c, 1.0 / (double)cell.second.size());
    for (int a = 0; a < 3; ++a) g_out[3 * m + a] = c[a];
    ++m;
  }
  for (int64_t j = 0; j < m; ++j) {
    std::vector<std::pair<double, int64_t> > d;   // (distance, id) of every other node, sorted
    const V3 gj = v3(g_out[3 * j], g_out[3 * j + 1], g_out[3 * j + 2]);
    for (int64_t l = 0; l < m; ++l)
      if (l != j) d.push_back(std::make_pair(norm(sub(v3(g_out[3 * l], g_out[3 * l + 1], g_out[3 * l + 2]), gj)), l));
    std::sort(d.begin(), d.end());
    for (int s = 0; s < n_nbr; ++s) nbr_out[(int64_t)n_nbr * j + s] = s < (int)d.size() ? (int32_t)d[s].second : -1;
    nbr_margin[j] = ((int)d.size() > n_nbr && n_nbr > 0 && d[n_nbr].first > 0)
                        ? (d[n_nbr].first - d[n_nbr - 1].first) / d[n_nbr].first : 1.0;
  }
  return m;
}

}  // extern "C"

// =====================================================================================
// O9 (NEXT-4): affine nodes A_j + E_rot ("affine matrix A_j", Eq. 1 with A_j, Eq. 4-5
// E_rot, Eq. 6 with A_j; readings A41-A45).  Node state At (m x 12): A_j row-major (9), t_j (3);
// 12 unknowns per node [dA_j row-major, dt_j] with the additive update A_j += dA_j, t_j += dt_j
// (A41).  Normals warp by the inverse transpose, n~ = normalize(R sum_j w_j A_j^-T n), A_j itself
// if |det A_j| < 1e-9 (A43).  Written out separately from the SE(3) path above (12 x 12
// blocks); the same Gauss-Newton loop (fixed G, P), the same solve modes.
// =====================================================================================
namespace {

typedef std::array<double, 144> B12;

M3 aff_A(const double* At, int j) { M3 A; for (int a = 0; a < 9; ++a) A[a] = At[12 * j + a]; return A; }
V3 aff_t(const double* At, int j) { return v3(At[12 * j + 9], At[12 * j + 10], At[12 * j + 11]); }

// inverse transpose of A (cofactor matrix / det); A itself when |det| < 1e-9 (A43)
M3 inv_transpose(const M3& A) {
  M3 C;   // cofactors C[i][j] = (-1)^(i+j) minor(i, j)
  C[0] = A[4] * A[8] - A[5] * A[7]; C[1] = A[5] * A[6] - A[3] * A[8]; C[2] = A[3] * A[7] - A[4] * A[6];
  C[3] = A[2] * A[7] - A[1] * A[8]; C[4] = A[0] * A[8] - A[2] * A[6]; C[5] = A[1] * A[6] - A[0] * A[7];
  C[6] = A[1] * A[5] - A[2] * A[4]; C[7] = A[2] * A[3] - A[0] * A[5]; C[8] = A[0] * A[4] - A[1] * A[3];
  const double det = A[0] * C[0] + A[1] * C[1] + A[2] * C[2];
  if (std::fabs(det) < 1e-9) return A;
  for (int a = 0; a < 9; ++a) C[a] /= det;   // (A^-1)^T = cof(A) / det
  return C;
}

struct WarpedA {
  bool ok;
  double wn[8];
  V3 d[8];          // d_j = v - g_j
  V3 x_hat, m_hat, vt, nt;
};

// Eq. 1 with affine A_j, weights normalised (R-A6); normal by A_j^-T (A43)
WarpedA warp_point_aff(const V3& v, const V3& n, int k, const int32_t* idx, const double* wraw, const float* g,
                       const double* At, const double* pose) {
  WarpedA o;
  o.ok = false;
  double W = 0;
  for (int s = 0; s < k; ++s) W += wraw[s];
  if (!(W > 0)) return o;
  o.x_hat = v3(0, 0, 0);
  o.m_hat = v3(0, 0, 0);
  for (int s = 0; s < k; ++s) {
    const int j = idx[s];
    o.wn[s] = wraw[s] / W;
    const V3 gj = load3(g + 3 * j);
    o.d[s] = sub(v, gj);
    o.x_hat = add(o.x_hat, scale(add(add(mul(aff_A(At, j), o.d[s]), gj), aff_t(At, j)), o.wn[s]));
    o.m_hat = add(o.m_hat, scale(mul(inv_transpose(aff_A(At, j)), n), o.wn[s]));
  }
  const M3 R = pose_R(pose);
  o.vt = add(mul(R, o.x_hat), pose_T(pose));
  const double ml = norm(o.m_hat);
  if (ml < 1e-12) return o;
  o.nt = mul(R, scale(o.m_hat, 1.0 / ml));
  o.ok = true;
  return o;
}

// the Eq. 7 gates on an affine-warped point (same gates as associate_point)
Assoc associate_aff(const or_params* prm, const or_frame* f, const WarpedA& w) {
  Warped s;
  s.ok = w.ok;
  s.vt = w.vt;
  s.nt = w.nt;
  return associate_point(prm, f, s);
}

// Jacobian of the warped camera-frame point w.r.t. node slot s (3 x 12): columns (r, c) of dA
// (row-major) = w_j d_c R e_r; columns of dt = w_j R
void jac_point_aff(const M3& R, double wj, const V3& d, double* J /*3 x 12*/) {
  for (int q = 0; q < 3; ++q) {
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) J[12 * q + 3 * r + c] = wj * d[c] * R[3 * q + r];
    for (int c = 0; c < 3; ++c) J[12 * q + 9 + c] = wj * R[3 * q + c];
  }
}

// Eq. 5: r = [c1.c2, c1.c3, c2.c3, c1.c1 - 1, c2.c2 - 1, c3.c3 - 1] of the columns
// c_i of A; J (6 x 9) w.r.t. A row-major (A[r][c] is entry r of column c)
void rot_rows(const M3& A, double* r, double* J) {
  V3 c[3];
  for (int i = 0; i < 3; ++i) c[i] = v3(A[i], A[3 + i], A[6 + i]);
  const int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {1, 2, 2, 0, 1, 2};
  for (int q = 0; q < 6; ++q) {
    const int a = pa[q], b = pb[q];
    r[q] = dot(c[a], c[b]) - (a == b ? 1.0 : 0.0);
    for (int e = 0; e < 9; ++e) J[9 * q + e] = 0.0;
    for (int row = 0; row < 3; ++row) {   // d(c_a . c_b) / dA[row][a] = c_b[row], / dA[row][b] = c_a[row]
      J[9 * q + 3 * row + a] += c[b][row];
      J[9 * q + 3 * row + b] += c[a][row];
    }
  }
}

struct SystemA {
  int m;
  std::map<std::pair<int, int>, B12> blk;   // upper blocks (j <= l)
  std::vector<double> rhs;
  double E[5];   // E_data, E_pt, E_reg, E_corr, E_rot
  int64_t n_assoc;
  explicit SystemA(int m_) : m(m_), rhs(12 * m_, 0.0), n_assoc(0) { for (int a = 0; a < 5; ++a) E[a] = 0; }
  // H(a, b) += w Ja^T Jb over `rows` rows (Ja, Jb: rows x 12)
  void add_pair(int a, const double* Ja, int b, const double* Jb, int rows, double w) {
    const bool sw = a > b;
    B12& B = blk[sw ? std::make_pair(b, a) : std::make_pair(a, b)];
    const double* X = sw ? Jb : Ja;
    const double* Y = sw ? Ja : Jb;
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 12; ++j) {
        double s = 0;
        for (int q = 0; q < rows; ++q) s += X[12 * q + i] * Y[12 * q + j];
        B[12 * i + j] += w * s;
      }
  }
  void add_rhs(int a, const double* Ja, const double* r, int rows, double w) {
    for (int i = 0; i < 12; ++i) {
      double s = 0;
      for (int q = 0; q < rows; ++q) s += Ja[12 * q + i] * r[q];
      rhs[12 * a + i] -= w * s;
    }
  }
  // every slot pair of one residual group (ids may repeat: both orders then)
  void add_group(const int32_t* ids, const double* J, int ks, int rows, const double* r, double w) {
    for (int a = 0; a < ks; ++a) {
      for (int b = 0; b < ks; ++b) {
        if (ids[a] > ids[b] || (ids[a] == ids[b] && a > b)) continue;
        add_pair(ids[a], J + 12 * rows * a, ids[b], J + 12 * rows * b, rows, w);
        if (ids[a] == ids[b] && a != b) add_pair(ids[b], J + 12 * rows * b, ids[a], J + 12 * rows * a, rows, w);
      }
      add_rhs(ids[a], J + 12 * rows * a, r, rows, w);
    }
  }
};

double total_energy_aff(const or_params* prm, const double* E) {
  return prm->w_data * E[0] + prm->w_pt * E[1] + prm->w_reg * E[2] + prm->w_corr * E[3] + prm->w_rot * E[4];
}

void assemble_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At, const int32_t* fidx,
                  const double* fw, SystemA* S) {
  const int k = prm->k;
  const M3 R = pose_R(f->pose);
  double Jpl[8 * 12], Jpt[8 * 36];
  for (int64_t i = 0; i < p->n; ++i) {   // O9a: data (Eq. 8) and point-to-point terms
    double wr[8];
    wraw_of(p, k, i, wr);
    WarpedA w = warp_point_aff(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, At, f->pose);
    Assoc as = associate_aff(prm, f, w);
    if (as.pix < 0) continue;
    S->n_assoc++;
    const V3 dd = sub(w.vt, as.q);
    const double rpl = dot(as.N, dd), rpt[3] = {dd[0], dd[1], dd[2]};
    for (int s = 0; s < k; ++s) {
      jac_point_aff(R, w.wn[s], w.d[s], Jpt + 36 * s);
      for (int c = 0; c < 12; ++c)   // plane row = N^T (point rows)
        Jpl[12 * s + c] = as.N[0] * Jpt[36 * s + c] + as.N[1] * Jpt[36 * s + 12 + c] + as.N[2] * Jpt[36 * s + 24 + c];
    }
    S->E[0] += rpl * rpl;
    S->E[1] += rpt[0] * rpt[0] + rpt[1] * rpt[1] + rpt[2] * rpt[2];
    S->add_group(p->idx + k * i, Jpl, k, 1, &rpl, prm->w_data);
    S->add_group(p->idx + k * i, Jpt, k, 3, rpt, prm->w_pt);
  }
  // O9b: Eq. 6 with A_j: e = A_j (g_l - g_j) + g_j + t_j - g_l - t_l
  for (int j = 0; j < p->m; ++j)
    for (int s = 0; s < prm->n_nbr; ++s) {
      const int l = p->nbr[prm->n_nbr * j + s];
      if (l < 0) continue;
      const V3 gj = load3(p->g + 3 * j), gl = load3(p->g + 3 * l), d = sub(gl, gj);
      const V3 e = sub(add(add(mul(aff_A(At, j), d), gj), aff_t(At, j)), add(gl, aff_t(At, l)));
      double Jj[36], Jl[36];
      for (int a = 0; a < 36; ++a) Jj[a] = Jl[a] = 0.0;
      for (int q = 0; q < 3; ++q) {
        for (int c = 0; c < 3; ++c) Jj[12 * q + 3 * q + c] = d[c];   // de_q / dA_j[q][c]
        Jj[12 * q + 9 + q] = 1.0;
        Jl[12 * q + 9 + q] = -1.0;
      }
      const double ev[3] = {e[0], e[1], e[2]};
      S->E[2] += dot(e, e);
      S->add_pair(j, Jj, j, Jj, 3, prm->w_reg);
      S->add_pair(l, Jl, l, Jl, 3, prm->w_reg);
      S->add_pair(j, Jj, l, Jl, 3, prm->w_reg);
      S->add_rhs(j, Jj, ev, 3, prm->w_reg);
      S->add_rhs(l, Jl, ev, 3, prm->w_reg);
    }
  // O9c: Eq. 9 features
  for (int q = 0; q < p->nf; ++q) {
    double W = 0;
    for (int s = 0; s < k; ++s) W += fw[k * q + s];
    if (!(W > 0)) continue;
    WarpedA w = warp_point_aff(load3(p->fsrc + 3 * q), v3(0, 0, 1), k, fidx + k * q, fw + k * q, p->g, At, f->pose);
    const V3 e = sub(w.vt, load3(p->fdst + 3 * q));
    const double ev[3] = {e[0], e[1], e[2]};
    double Jf[8 * 36];
    for (int s = 0; s < k; ++s) jac_point_aff(R, w.wn[s], w.d[s], Jf + 36 * s);
    S->E[3] += dot(e, e);
    S->add_group(fidx + k * q, Jf, k, 3, ev, prm->w_corr);
  }
  // O9d: Eq. 4-5 E_rot on every node (A42)
  for (int j = 0; j < p->m; ++j) {
    double r[6], J9[54], J[72];
    rot_rows(aff_A(At, j), r, J9);
    for (int q = 0; q < 6; ++q) {
      for (int c = 0; c < 12; ++c) J[12 * q + c] = c < 9 ? J9[9 * q + c] : 0.0;
      S->E[4] += r[q] * r[q];
    }
    S->add_pair(j, J, j, J, 6, prm->w_rot);
    S->add_rhs(j, J, r, 6, prm->w_rot);
  }
}

// O9e: solve (H + lambda I) x = rhs: EXACT (dense Cholesky, or PCG to 1e-12) or MIRROR (block-Jacobi
// PCG with the GPU's P; M_j = (H_jj + lambda I + mu_j I)^-1, mu_j = 1e-9 tr(H_jj)/12, A17)
void spmv_aff(const SystemA& S, double lambda, const std::vector<double>& x, std::vector<double>& y) {
  std::fill(y.begin(), y.end(), 0.0);
  for (const auto& kv : S.blk) {
    const int j = kv.first.first, l = kv.first.second;
    const B12& B = kv.second;
    for (int a = 0; a < 12; ++a)
      for (int b = 0; b < 12; ++b) {
        y[12 * j + a] += B[12 * a + b] * x[12 * l + b];
        if (j != l) y[12 * l + b] += B[12 * a + b] * x[12 * j + a];
      }
  }
  for (size_t i = 0; i < y.size(); ++i) y[i] += lambda * x[i];
}

int solve_aff(const SystemA& S, double lambda, int mode, int pcg_iters, std::vector<double>& x) {
  const int n = 12 * S.m;
  if (mode == 0 && n <= 1200) {
    std::vector<double> A((size_t)n * n, 0.0);
    for (const auto& kv : S.blk) {
      const int j = kv.first.first, l = kv.first.second;
      for (int a = 0; a < 12; ++a)
        for (int b = 0; b < 12; ++b) {
          A[(size_t)(12 * j + a) * n + 12 * l + b] += kv.second[12 * a + b];
          if (j != l) A[(size_t)(12 * l + b) * n + 12 * j + a] += kv.second[12 * a + b];
        }
    }
    for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += lambda;
    x.assign(n, 0.0);
    if (!cholesky(A, n)) return -1;
    chol_solve(A, n, S.rhs.data(), x.data());
    return 0;
  }
  std::vector<double> Minv(144 * (size_t)S.m, 0.0);
  for (int j = 0; j < S.m; ++j) {
    std::vector<double> A(144, 0.0);
    auto it = S.blk.find(std::make_pair(j, j));
    if (it != S.blk.end()) for (int a = 0; a < 144; ++a) A[a] = it->second[a];
    double tr = 0;
    for (int a = 0; a < 12; ++a) tr += A[13 * a];
    for (int a = 0; a < 12; ++a) A[13 * a] += lambda + 1e-9 * tr / 12.0;
    if (!cholesky(A, 12)) continue;
    for (int c = 0; c < 12; ++c) {
      double e[12] = {0}, col[12];
      e[c] = 1.0;
      chol_solve(A, 12, e, col);
      for (int r = 0; r < 12; ++r) Minv[144 * j + 12 * r + c] = col[r];
    }
  }
  auto applyM = [&](const std::vector<double>& r, std::vector<double>& z) {
    for (int j = 0; j < S.m; ++j)
      for (int a = 0; a < 12; ++a) {
        double s = 0;
        for (int b = 0; b < 12; ++b) s += Minv[144 * j + 12 * a + b] * r[12 * j + b];
        z[12 * j + a] = s;
      }
  };
  const int max_it = mode == 1 ? pcg_iters : 20 * n;
  const double rel_tol = mode == 1 ? 0.0 : 1e-12;
  std::vector<double> r(S.rhs), z(n), p(n), Ap(n);
  x.assign(n, 0.0);
  applyM(r, z);
  p = z;
  double rz = vdot(r, z), b2 = vdot(S.rhs, S.rhs);
  int it = 0;
  for (; it < max_it; ++it) {
    if (rel_tol > 0 && vdot(r, r) <= rel_tol * rel_tol * b2) break;
    if (rz == 0) break;
    spmv_aff(S, lambda, p, Ap);
    const double pAp = vdot(p, Ap);
    if (!(pAp > 0)) break;
    const double alpha = rz / pAp;
    for (int i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; }
    applyM(r, z);
    const double rz_new = vdot(r, z), beta = rz_new / rz;
    rz = rz_new;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  return it;
}

}  // namespace

extern "C" {

void or_warp_aff(const or_problem* p, int32_t k, const double* At, const double pose[12], double* x_hat,
                 double* n_hat, double* vt, double* nt, uint8_t* ok) {
  for (int64_t i = 0; i < p->n; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    WarpedA w = warp_point_aff(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, At, pose);
    ok[i] = w.ok ? 1 : 0;
    for (int a = 0; a < 3; ++a) {
      x_hat[3 * i + a] = w.ok ? w.x_hat[a] : 0.0;
      n_hat[3 * i + a] = w.ok ? w.m_hat[a] / norm(w.m_hat) : 0.0;
      vt[3 * i + a] = w.ok ? w.vt[a] : 0.0;
      nt[3 * i + a] = w.ok ? w.nt[a] : 0.0;
    }
  }
}

void or_associate_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At, int32_t* pix,
                      uint8_t* why, double* margin) {
  const int k = prm->k;
  for (int64_t i = 0; i < p->n; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    WarpedA w = warp_point_aff(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, At, f->pose);
    Assoc a = associate_aff(prm, f, w);
    pix[i] = a.pix;
    why[i] = a.why;
    margin[i] = a.margin;
  }
}

void or_rot(const double A[9], double r[6], double J[54]) {
  M3 M;
  for (int a = 0; a < 9; ++a) M[a] = A[a];
  rot_rows(M, r, J);
}

int64_t or_system_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At,
                      const int32_t* fidx, const double* fw, int64_t cap, int32_t* brow, int32_t* bcol, double* bval,
                      double* rhs, double energy[6], int64_t* n_assoc) {
  SystemA S(p->m);
  assemble_aff(prm, p, f, At, fidx, fw, &S);
  int64_t nb = 0;
  for (auto it = S.blk.begin(); it != S.blk.end(); ++it, ++nb) {
    if (nb >= cap) continue;
    brow[nb] = it->first.first;
    bcol[nb] = it->first.second;
    for (int a = 0; a < 144; ++a) bval[144 * nb + a] = it->second[a];
  }
  for (int i = 0; i < 12 * p->m; ++i) rhs[i] = S.rhs[i];
  for (int a = 0; a < 5; ++a) energy[a] = S.E[a];
  energy[5] = total_energy_aff(prm, S.E);
  *n_assoc = S.n_assoc;
  return nb;
}

int64_t or_residuals_aff(const or_params* prm, const or_problem* p, const or_frame* f, const double* At,
                         const int32_t* pix_frozen, const int32_t* fidx, const double* fw, int64_t cap_rows, double* r,
                         double* J) {
  const int k = prm->k, ncol = 12 * p->m;
  const M3 R = pose_R(f->pose);
  const double sd = std::sqrt(prm->w_data), sp = std::sqrt(prm->w_pt), sr = std::sqrt(prm->w_reg),
               sc = std::sqrt(prm->w_corr), so = std::sqrt(prm->w_rot);
  int64_t row = 0;
  double Jp[36];
  for (int64_t i = 0; i < p->n; ++i) {
    if (pix_frozen[i] < 0) continue;
    double wr[8];
    wraw_of(p, k, i, wr);
    WarpedA w = warp_point_aff(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, At, f->pose);
    if (!w.ok) continue;
    const int px = pix_frozen[i] % f->W, py = pix_frozen[i] / f->W;
    V3 N;
    if (!pixel_normal(f, px, py, &N)) continue;
    const V3 q = back_project(f, px, py, (double)f->depth[pix_frozen[i]]);
    if (row + 4 > cap_rows) return -1;
    double* J0 = J + (size_t)row * ncol;
    std::memset(J0, 0, sizeof(double) * 4 * ncol);
    const V3 dd = sub(w.vt, q);
    r[row] = sd * dot(N, dd);
    for (int c = 0; c < 3; ++c) r[row + 1 + c] = sp * dd[c];
    for (int s = 0; s < k; ++s) {
      const int j = p->idx[k * i + s];
      jac_point_aff(R, w.wn[s], w.d[s], Jp);
      for (int c = 0; c < 12; ++c) {
        J0[12 * j + c] += sd * (N[0] * Jp[c] + N[1] * Jp[12 + c] + N[2] * Jp[24 + c]);
        for (int qq = 0; qq < 3; ++qq) J0[(size_t)(1 + qq) * ncol + 12 * j + c] += sp * Jp[12 * qq + c];
      }
    }
    row += 4;
  }
  for (int j = 0; j < p->m; ++j)
    for (int s = 0; s < prm->n_nbr; ++s) {
      const int l = p->nbr[prm->n_nbr * j + s];
      if (l < 0) continue;
      const V3 gj = load3(p->g + 3 * j), gl = load3(p->g + 3 * l), d = sub(gl, gj);
      const V3 e = sub(add(add(mul(aff_A(At, j), d), gj), aff_t(At, j)), add(gl, aff_t(At, l)));
      if (row + 3 > cap_rows) return -1;
      double* J0 = J + (size_t)row * ncol;
      std::memset(J0, 0, sizeof(double) * 3 * ncol);
      for (int qq = 0; qq < 3; ++qq) {
        r[row + qq] = sr * e[qq];
        for (int c = 0; c < 3; ++c) J0[(size_t)qq * ncol + 12 * j + 3 * qq + c] += sr * d[c];
        J0[(size_t)qq * ncol + 12 * j + 9 + qq] += sr;
        J0[(size_t)qq * ncol + 12 * l + 9 + qq] -= sr;
      }
      row += 3;
    }
  for (int q = 0; q < p->nf; ++q) {
    double W = 0;
    for (int s = 0; s < k; ++s) W += fw[k * q + s];
    if (!(W > 0)) continue;
    WarpedA w = warp_point_aff(load3(p->fsrc + 3 * q), v3(0, 0, 1), k, fidx + k * q, fw + k * q, p->g, At, f->pose);
    const V3 e = sub(w.vt, load3(p->fdst + 3 * q));
    if (row + 3 > cap_rows) return -1;
    double* J0 = J + (size_t)row * ncol;
    std::memset(J0, 0, sizeof(double) * 3 * ncol);
    for (int a = 0; a < 3; ++a) r[row + a] = sc * e[a];
    for (int s = 0; s < k; ++s) {
      const int j = fidx[k * q + s];
      jac_point_aff(R, w.wn[s], w.d[s], Jp);
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 12; ++c) J0[(size_t)a * ncol + 12 * j + c] += sc * Jp[12 * a + c];
    }
    row += 3;
  }
  for (int j = 0; j < p->m; ++j) {
    double rr[6], J9[54];
    rot_rows(aff_A(At, j), rr, J9);
    if (row + 6 > cap_rows) return -1;
    double* J0 = J + (size_t)row * ncol;
    std::memset(J0, 0, sizeof(double) * 6 * ncol);
    for (int q = 0; q < 6; ++q) {
      r[row + q] = so * rr[q];
      for (int c = 0; c < 9; ++c) J0[(size_t)q * ncol + 12 * j + c] = so * J9[9 * q + c];
    }
    row += 6;
  }
  return row;
}

int32_t or_solve_aff(int32_t m, int64_t nblk, const int32_t* brow, const int32_t* bcol, const double* bval,
                     const double* rhs, double lambda, int32_t mode, int32_t pcg_iters, double* x) {
  SystemA S(m);
  for (int64_t b = 0; b < nblk; ++b) {
    B12& B = S.blk[std::make_pair(brow[b], bcol[b])];
    for (int a = 0; a < 144; ++a) B[a] = bval[144 * b + a];
  }
  for (int i = 0; i < 12 * m; ++i) S.rhs[i] = rhs[i];
  std::vector<double> xs;
  const int32_t it = solve_aff(S, lambda, mode, pcg_iters, xs);
  for (int i = 0; i < 12 * m; ++i) x[i] = xs[i];
  return it;
}

// O9f: fixed-G Gauss-Newton over the affine nodes; energy (G+1) x 6 (E_data, E_pt, E_reg, E_corr,
// E_rot, weighted total); At (m x 12) initial state on entry, result on exit
void or_register_aff(const or_params* prm, const or_problem* p, const or_frame* f, double* At, double* energy,
                     int64_t* n_assoc, int32_t* accepted) {
  std::vector<int32_t> fidx;
  std::vector<double> fw;
  feature_skin(p, prm->k, fidx, fw);
  auto record = [&](int it, const SystemA& S) {
    for (int a = 0; a < 5; ++a) energy[6 * it + a] = S.E[a];
    energy[6 * it + 5] = total_energy_aff(prm, S.E);
    n_assoc[it] = S.n_assoc;
  };
  auto step = [&](const std::vector<double>& x) {
    for (int j = 0; j < p->m; ++j)   // A41: additive update
      for (int a = 0; a < 12; ++a) At[12 * j + a] += x[12 * j + a];
  };
  if (!prm->lm) {
    for (int it = 0; it <= prm->gn_iters; ++it) {
      SystemA S(p->m);
      assemble_aff(prm, p, f, At, fidx.data(), fw.data(), &S);
      record(it, S);
      if (accepted) accepted[it] = 1;
      if (it == prm->gn_iters) break;
      std::vector<double> x;
      solve_aff(S, prm->lambda, prm->solve_mode, prm->pcg_iters, x);
      step(x);
    }
    return;
  }
  // Levenberg-Marquardt with the schedule of R-A29, as register_impl
  const size_t ns = 12 * (size_t)p->m;
  std::vector<double> base(At, At + ns);
  SystemA acc(p->m);
  double E_acc = 0.0, mu = prm->lm_mu0;
  for (int it = 0; it <= prm->gn_iters; ++it) {
    SystemA S(p->m);
    assemble_aff(prm, p, f, At, fidx.data(), fw.data(), &S);
    record(it, S);
    const double E = total_energy_aff(prm, S.E);
    const bool ok = it == 0 || E < E_acc;
    if (accepted) accepted[it] = ok ? 1 : 0;
    if (ok) {
      std::copy(At, At + ns, base.begin());
      acc = S;
      E_acc = E;
      if (it > 0) mu *= 0.5;
    } else {
      std::copy(base.begin(), base.end(), At);
      mu *= 10.0;
    }
    if (it == prm->gn_iters) break;
    SystemA D = acc;   // damped copy: diagonal entries of H times (1 + mu)
    for (int j = 0; j < p->m; ++j) {
      auto d = D.blk.find(std::make_pair(j, j));
      if (d != D.blk.end())
        for (int a = 0; a < 12; ++a) d->second[13 * a] *= 1.0 + mu;
    }
    std::vector<double> x;
    solve_aff(D, prm->lambda, prm->solve_mode, prm->pcg_iters, x);
    step(x);
  }
}

// O9g: the converged affine field applied (live world state), normals by A^-T, nodes g + t (A45)
void or_warp_model_aff(const or_problem* p, int32_t k, const double* At, double* xyz_out, double* nrm_out,
                       double* g_out) {
  const double pose[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
  for (int64_t i = 0; i < p->n; ++i) {
    double wr[8];
    wraw_of(p, k, i, wr);
    WarpedA w = warp_point_aff(load3(p->xyz + 3 * i), load3(p->nrm + 3 * i), k, p->idx + k * i, wr, p->g, At, pose);
    for (int a = 0; a < 3; ++a) {
      xyz_out[3 * i + a] = w.ok ? w.x_hat[a] : (double)p->xyz[3 * i + a];
      nrm_out[3 * i + a] = w.ok ? w.nt[a] : (double)p->nrm[3 * i + a];
    }
  }
  for (int j = 0; j < p->m; ++j)
    for (int a = 0; a < 3; ++a) g_out[3 * j + a] = (double)p->g[3 * j + a] + At[12 * j + 9 + a];
}

}  // extern "C"
