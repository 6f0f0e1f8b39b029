// picard.cu -- host-side Picard driver of libgmaf (Sec. 2.3, Eqs. 2.10-2.22, PAPER.md:93-157;
// SURVEY 8(f) NEXT-1).  Every pressure solve and force integral runs on the device through the
// public ABI (gmaf_thickness -> gmaf_assemble -> gmaf_solve -> gmaf_integrate on the 9 joint
// working conditions); what remains here is 4-vector / 4x4 host arithmetic.
//
// The paper defines the iteration but not the loads; the generalized forces and the load
// models are DESIGN.md readings:
//   R-A28  F1..F4 are conjugate to e1..e4 by rigid-body virtual work.  Eq. 2.3 places the
//          piston axis at x_c(y) = e1 + (e3 - e1) y / L_F, y_c(y) = e2 + (e4 - e2) y / L_F, so
//          a wrench (F_X, F_Y, M_X, M_Y about the bottom centre) gives
//          F1 = F_X - M_Y/L_F, F2 = F_Y + M_X/L_F, F3 = M_Y/L_F, F4 = -M_X/L_F.
//   R-A29  external load = lateral part of the swashplate reaction to the pressure thrust
//          p_in pi R_k^2 on the piston bottom, T = p_in pi R_k^2 tan(beta), along
//          (-cos phi, sin phi) in the piston frame (X radial, Y tangential), at y = L_F.
//   R-A30  inertial load = centrifugal (m_k + m_G) omega_s^2 R_b along +X; m_k at y = L_F/2,
//          m_G at y = L_F (the stroke acceleration is axial and has no lateral part).
//   R-A31  update: SIMPLIFIED Eqs. 2.21-2.22; GENERAL = Eq. 2.12 with the same backward
//          difference e^(k+1) - e^(k) = dt (edot^(k+1) - edot^(k)), i.e.
//          (dt J_e + J_edot) d = -F.  A time step starts at e = e_l + dt edot_l, edot = edot_l
//          and stops when ||F|| <= eps_dyn max(||F_E||, 1 N).
#include <cmath>
#include <cstring>

#include "../../include/gmaf.h"
#include "gmaf_internal.cuh"

namespace gmaf {
gmaf_status ctx_fail(gmaf_ctx* c, gmaf_status code, const char* msg);
}

namespace {

constexpr double kPi = 3.14159265358979323846;

// Solve the 4x4 system M x = b by Gaussian elimination with partial pivoting.
bool solve4(const double* Min, const double* b, double* x) {
  double M[4][5];
  double scale = 0.0;
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 4; ++j) {
      M[i][j] = Min[4 * i + j];
      scale = std::fmax(scale, std::fabs(M[i][j]));
    }
    M[i][4] = b[i];
  }
  if (!(scale > 0.0) || !std::isfinite(scale)) return false;
  for (int c = 0; c < 4; ++c) {
    int p = c;
    for (int r = c + 1; r < 4; ++r)
      if (std::fabs(M[r][c]) > std::fabs(M[p][c])) p = r;
    if (std::fabs(M[p][c]) <= 1e-30 * scale) return false;
    if (p != c)
      for (int j = 0; j < 5; ++j) std::swap(M[p][j], M[c][j]);
    for (int r = c + 1; r < 4; ++r) {
      const double f = M[r][c] / M[c][c];
      for (int j = c; j < 5; ++j) M[r][j] -= f * M[c][j];
    }
  }
  for (int i = 3; i >= 0; --i) {
    double s = M[i][4];
    for (int j = i + 1; j < 4; ++j) s -= M[i][j] * x[j];
    x[i] = s / M[i][i];
  }
  return true;
}

double norm4(const double* v) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]); }

// R-A28: generalized force of a wrench (pressure + shear parts)
void oil_general_force(const double* w, double LF, double* F) {
  const double FX = w[0] + w[6], FY = w[1] + w[7];
  const double MX = w[3] + w[9], MY = w[4] + w[10];
  F[0] = FX - MY / LF;
  F[1] = FY + MX / LF;
  F[2] = MY / LF;
  F[3] = -MX / LF;
}

}  // namespace

extern "C" {

gmaf_status gmaf_general_forces(const gmaf_pump* pump, const gmaf_condition* cond, double phi,
                                const double* wrench12, double* F_oil4, double* F_ext4, double* F_in4) {
  if (!pump || !cond || !(cond->L_F > 0.0)) return GMAF_E_INVALID_ARG;
  if (F_oil4) {
    if (!wrench12) return GMAF_E_INVALID_ARG;
    oil_general_force(wrench12, cond->L_F, F_oil4);
  }
  if (F_ext4) {   // R-A29
    const double T = cond->p_in * (kPi * pump->R_k * pump->R_k) * std::tan(pump->beta);
    F_ext4[0] = 0.0;
    F_ext4[1] = 0.0;
    F_ext4[2] = -T * std::cos(phi);
    F_ext4[3] = T * std::sin(phi);
  }
  if (F_in4) {    // R-A30
    const double w2R = pump->omega_s * pump->omega_s * pump->R_b;
    F_in4[0] = 0.5 * pump->m_k * w2R;
    F_in4[1] = 0.0;
    F_in4[2] = 0.5 * pump->m_k * w2R + pump->m_G * w2R;
    F_in4[3] = 0.0;
  }
  return GMAF_OK;
}

gmaf_status gmaf_picard_iteration(gmaf_ctx* ctx, const gmaf_pump* pump, const gmaf_condition* state,
                                  double phi, double dt, int32_t scheme, double de, double dedot,
                                  double tol, double omega, int32_t max_iter, int32_t warm_start,
                                  gmaf_picard_iterate* out) {
  if (!ctx || !pump || !state || !out) return GMAF_E_INVALID_ARG;
  if (gmaf::ctx_conditions(ctx) != 9 || gmaf::ctx_world(ctx) != 1)
    return gmaf::ctx_fail(ctx, GMAF_E_INVALID_ARG, "picard: needs a single-rank context with K = 9");
  if (!(dt > 0.0) || !(de > 0.0) || !(dedot > 0.0) ||
      (scheme != GMAF_PICARD_SIMPLIFIED && scheme != GMAF_PICARD_GENERAL))
    return gmaf::ctx_fail(ctx, GMAF_E_INVALID_ARG, "picard: dt, de, dedot must be > 0 and scheme known");
  // the 9 working conditions (Eqs. 2.17-2.19): base, e_j + de, edot_j + dedot
  gmaf_condition conds[9];
  for (int k = 0; k < 9; ++k) conds[k] = *state;
  for (int j = 0; j < 4; ++j) {
    conds[1 + j].e[j] += de;
    conds[5 + j].edot[j] += dedot;
  }
  gmaf_status s = gmaf_thickness(ctx, conds);
  if (s != GMAF_OK) return s;
  if ((s = gmaf_assemble(ctx)) != GMAF_OK) return s;
  gmaf_solve_stats st;
  std::memset(&st, 0, sizeof(st));
  if ((s = gmaf_solve(ctx, tol, omega, GMAF_PRECOND_ASSOR2, GMAF_COUPLED, max_iter, warm_start, &st, nullptr)) !=
      GMAF_OK)
    return s;
  double W[9 * 12];
  if ((s = gmaf_integrate(ctx, W)) != GMAF_OK) return s;
  // general forces of the 9 conditions (the loads do not depend on e or edot)
  double Fo[9][4];
  for (int k = 0; k < 9; ++k) oil_general_force(W + 12 * k, state->L_F, Fo[k]);
  gmaf_general_forces(pump, state, phi, nullptr, nullptr, out->F_ext, out->F_inertial);
  for (int i = 0; i < 4; ++i) {
    out->F_oil[i] = Fo[0][i];
    out->F[i] = out->F_ext[i] + out->F_inertial[i] + Fo[0][i];   // Eq. 2.10
  }
  std::memcpy(out->wrench, W, sizeof(out->wrench));
  // finite-difference Jacobians (Eqs. 2.13-2.14), column j from condition 1+j / 5+j
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      out->J_e[4 * i + j] = (Fo[1 + j][i] - Fo[0][i]) / de;
      out->J_edot[4 * i + j] = (Fo[5 + j][i] - Fo[0][i]) / dedot;
    }
  // update (R-A31)
  double M[16], rhs[4], d[4];
  for (int q = 0; q < 16; ++q)
    M[q] = scheme == GMAF_PICARD_GENERAL ? dt * out->J_e[q] + out->J_edot[q] : out->J_edot[q];
  for (int i = 0; i < 4; ++i) rhs[i] = -out->F[i];
  if (!solve4(M, rhs, d)) return gmaf::ctx_fail(ctx, GMAF_E_SINGULAR, "picard: singular update matrix");
  for (int i = 0; i < 4; ++i) {
    out->edot_next[i] = state->edot[i] + d[i];
    out->e_next[i] = state->e[i] + dt * d[i];
  }
  out->pcg_iterations = st.iterations;
  out->pad = 0;
  return GMAF_OK;
}

gmaf_status gmaf_picard_step(gmaf_ctx* ctx, const gmaf_pump* pump, gmaf_condition* state, double phi,
                             double dt, int32_t scheme, double de, double dedot, double eps_dyn,
                             int32_t max_picard, double tol, double omega, int32_t max_iter,
                             int32_t* n_picard, double* residual, int32_t* pcg_iterations) {
  if (!ctx || !pump || !state || !(eps_dyn > 0.0) || max_picard < 1)
    return gmaf::ctx_fail(ctx, GMAF_E_INVALID_ARG, "picard step: bad arguments");
  gmaf_condition cur = *state;
  for (int j = 0; j < 4; ++j) cur.e[j] = state->e[j] + dt * state->edot[j];   // e = e_l + dt edot_l
  double Fe[4];
  gmaf_general_forces(pump, &cur, phi, nullptr, nullptr, Fe, nullptr);
  const double scale = std::fmax(norm4(Fe), 1.0);
  int32_t pcg = 0;
  double res = 0.0;
  gmaf_picard_iterate it;
  gmaf_status result = GMAF_E_NO_CONVERGENCE;
  int k = 0;
  for (; k < max_picard; ++k) {
    const gmaf_status s = gmaf_picard_iteration(ctx, pump, &cur, phi, dt, scheme, de, dedot, tol, omega,
                                                max_iter, 1 /* warm: the previous p */, &it);
    if (s != GMAF_OK) return s;
    pcg += it.pcg_iterations;
    res = norm4(it.F) / scale;
    if (res <= eps_dyn) { result = GMAF_OK; ++k; break; }
    for (int j = 0; j < 4; ++j) { cur.e[j] = it.e_next[j]; cur.edot[j] = it.edot_next[j]; }
  }
  *state = cur;
  if (n_picard) *n_picard = k;
  if (residual) *residual = res;
  if (pcg_iterations) *pcg_iterations = pcg;
  if (result != GMAF_OK) return gmaf::ctx_fail(ctx, GMAF_E_NO_CONVERGENCE, "picard step: max_picard reached");
  return GMAF_OK;
}

}  // extern "C"
