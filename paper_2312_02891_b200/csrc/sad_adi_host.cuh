// sad_adi_host.cuh -- the device-resident ADI outer loop in C++ (included at
// the end of sad_capi.cu).  Same loop as DeviceAdi.run (paper_2312_02891_b200/
// adi.py), i.e. the reference's run_with_state (adi.py:553-607) with adi_step
// (adi.py:510-537): per step the paper's tolerance budget and the admissible
// (delta_A, delta_B) (adi.py:347-408, host scalars), the two inner solves (the
// persistent GMRES kernel, concurrently on two streams or back to back), M z /
// C^T y, the fused epilogue and the r x r Gram algebra for ||res||, u, v and
// ||w t^*||.  The only difference from the Python loop is where the host logic
// runs: in C++, so a small config's outer step costs the solves plus a few
// microseconds of host work instead of ~0.2 ms of interpreter time.
#pragma once

#include <complex>

namespace {

using cplx = std::complex<double>;

constexpr double kCBound = 3.414213562373095;   // C_BOUND = 2 + sqrt(2) (adi.py:27)

// Hermitian eigenvalues (ascending) and optionally eigenvectors (columns of V)
// of the n x n row-major matrix A (n <= 8) by cyclic complex Jacobi rotations.
void herm_eig(int n, const cplx* Ain, double* w, cplx* V) {
  cplx A[64];
  for (int i = 0; i < n * n; ++i) A[i] = Ain[i];
  for (int i = 0; i < n; ++i) {        // Hermitian part
    A[i * n + i] = cplx(A[i * n + i].real(), 0.0);
    for (int j = i + 1; j < n; ++j) {
      const cplx h = 0.5 * (A[i * n + j] + std::conj(A[j * n + i]));
      A[i * n + j] = h;
      A[j * n + i] = std::conj(h);
    }
  }
  if (V)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) V[i * n + j] = cplx(i == j ? 1.0 : 0.0, 0.0);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += std::norm(A[i * n + i]);
      for (int j = i + 1; j < n; ++j) off += std::norm(A[i * n + j]);
    }
    if (off <= 1e-32 * diag || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const cplx apq = A[p * n + q];
        const double g = std::abs(apq);
        if (g == 0.0) continue;
        const cplx ph = apq / g;                       // e^{i phi}
        const double app = A[p * n + p].real(), aqq = A[q * n + q].real();
        const double theta = (aqq - app) / (2.0 * g);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        // J = P R with P = diag(1, conj(ph)) on (p, q): columns p, q of J
        const cplx jpp = c, jqp = -s * std::conj(ph), jpq = s, jqq = c * std::conj(ph);
        // A <- A J (columns p, q)
        for (int i = 0; i < n; ++i) {
          const cplx aip = A[i * n + p], aiq = A[i * n + q];
          A[i * n + p] = aip * jpp + aiq * jqp;
          A[i * n + q] = aip * jpq + aiq * jqq;
        }
        // A <- J^H A (rows p, q)
        for (int j = 0; j < n; ++j) {
          const cplx apj = A[p * n + j], aqj = A[q * n + j];
          A[p * n + j] = std::conj(jpp) * apj + std::conj(jqp) * aqj;
          A[q * n + j] = std::conj(jpq) * apj + std::conj(jqq) * aqj;
        }
        A[p * n + q] = A[q * n + p] = 0.0;
        A[p * n + p] = cplx(A[p * n + p].real(), 0.0);
        A[q * n + q] = cplx(A[q * n + q].real(), 0.0);
        if (V)
          for (int i = 0; i < n; ++i) {
            const cplx vip = V[i * n + p], viq = V[i * n + q];
            V[i * n + p] = vip * jpp + viq * jqp;
            V[i * n + q] = vip * jpq + viq * jqq;
          }
      }
  }
  // ascending order (with vectors)
  int idx[8];
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx, idx + n, [&](int a, int b) { return A[a * n + a].real() < A[b * n + b].real(); });
  cplx Vs[64];
  for (int k = 0; k < n; ++k) {
    w[k] = A[idx[k] * n + idx[k]].real();
    if (V)
      for (int i = 0; i < n; ++i) Vs[i * n + k] = V[i * n + idx[k]];
  }
  if (V)
    for (int i = 0; i < n * n; ++i) V[i] = Vs[i];
}

double lmax_herm2(double a, cplx b, double d) {
  const double h = 0.5 * (a - d);
  return 0.5 * (a + d) + std::sqrt(h * h + std::norm(b));
}

// sigma_max(X) from G = X^H X (device.py sigma_max_from_gram)
double sigma_max_gram(const cplx* G, int r) {
  if (r == 1) return std::sqrt(std::max(G[0].real(), 0.0));
  if (r == 2) {
    const cplx b = 0.5 * (G[1] + std::conj(G[2]));
    return std::sqrt(std::max(lmax_herm2(G[0].real(), b, G[3].real()), 0.0));
  }
  double w[8];
  herm_eig(r, G, w, nullptr);
  return std::sqrt(std::max(w[r - 1], 0.0));
}

// ||w t^*||_2 from Gw, Gt (device.py product_norm_from_grams)
double product_norm(const cplx* Gw, const cplx* Gt, int r) {
  if (r == 1) return std::sqrt(std::max(Gw[0].real() * Gt[0].real(), 0.0));
  if (r == 2) {
    const cplx bw = 0.5 * (Gw[1] + std::conj(Gw[2])), bt = 0.5 * (Gt[1] + std::conj(Gt[2]));
    const double aw = Gw[0].real(), dw = Gw[3].real(), at = Gt[0].real(), dt = Gt[3].real();
    const double tr = aw * at + dw * dt + 2.0 * (bw * std::conj(bt)).real();
    const double det = std::max(aw * dw - std::norm(bw), 0.0) * std::max(at * dt - std::norm(bt), 0.0);
    const double lam = 0.5 * tr + std::sqrt(std::max(0.25 * tr * tr - det, 0.0));
    return std::sqrt(std::max(lam, 0.0));
  }
  double lw[8], lk[8];
  cplx Q[64], half[64], K[64], T[64];
  herm_eig(r, Gw, lw, Q);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      cplx acc = 0.0;
      for (int k = 0; k < r; ++k) acc += Q[i * r + k] * std::sqrt(std::max(lw[k], 0.0)) * std::conj(Q[j * r + k]);
      half[i * r + j] = acc;
    }
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      cplx acc = 0.0;
      for (int k = 0; k < r; ++k) acc += half[i * r + k] * Gt[k * r + j];
      T[i * r + j] = acc;
    }
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      cplx acc = 0.0;
      for (int k = 0; k < r; ++k) acc += T[i * r + k] * half[k * r + j];
      K[i * r + j] = acc;
    }
  herm_eig(r, K, lk, nullptr);
  return std::sqrt(std::max(lk[r - 1], 0.0));
}

}  // namespace

// tolerance_budget (adi.py:347-361)
static double adi_budget(const sad_adi_config& c, int k, double u, double v, double eps) {
  const bool bl = c.strategy == SAD_STRAT_DYNAMIC_MID_BL || c.strategy == SAD_STRAT_DYNAMIC_B_BL;
  if (bl) {
    const double allowance = c.xi * k * eps / (2.0 * kCBound * c.kmax);
    return std::fabs(allowance - u - v) / kCBound;
  }
  return c.xi * eps / (2.0 * kCBound * kCBound * c.kmax);
}

// choose_tolerances (adi.py:372-408) for the iterative strategies
static void adi_choose(const sad_adi_config& c, double nw, double nt, double eps, double& dA,
                       double& dB, int& clA, int& clB) {
  const double tiny = 1e-300;
  clA = clB = 0;
  if (c.strategy == SAD_STRAT_FIXED) {
    dA = dB = c.fixed_delta;
    return;
  }
  if (c.strategy == SAD_STRAT_DYNAMIC_MID || c.strategy == SAD_STRAT_DYNAMIC_MID_BL) {
    const double mid = 0.5 * (std::min(c.delta_max_A, eps / std::max(nt, tiny)) - c.delta_min_A);
    dA = std::max(mid, c.delta_min_A);
    const double rawB = (eps - dA * nt) / (2.0 * dA + nw);
    dB = std::max(std::min(rawB, c.delta_max_B), c.delta_min_B);
    clA = mid < c.delta_min_A;
    clB = rawB < c.delta_min_B;
    return;
  }
  dB = c.delta_min_B;   // DYNAMIC_B(_BL)
  const double rawA = (eps - dB * nw) / (nt + 2.0 * dB);
  dA = std::max(std::min(rawA, c.delta_max_A), c.delta_min_A);
  clA = rawA < c.delta_min_A;
}

extern "C" int sad_adi_run(sad_ctx* ctx, const sad_adi_config* cfg, int r, int dtype, int64_t nA,
                           int64_t nB, sad_gmres* wsA, sad_gmres* wsB, sad_op* const* opsA,
                           sad_op* const* opsB, const double* gammas, sad_csr* M, sad_csr* C,
                           void* w, void* t, void* z_base, void* y_base, void* resA, void* resB,
                           void* mz_buf, void* cty_buf, int concurrent, void* stream_main,
                           void* streamA, void* streamB, double* records, int* steps_out,
                           double* summary) {
  if (!ctx || !cfg || !wsA || !wsB || !opsA || !opsB || !gammas || !w || !t || !z_base ||
      !y_base || !resA || !resB || !records || !steps_out || !summary)
    return SAD_EINVAL;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (cfg->strategy < SAD_STRAT_FIXED || cfg->strategy > SAD_STRAT_DYNAMIC_B_BL)
    return set_err(ctx, SAD_EINVAL, "strategy %d is not an iterative strategy", cfg->strategy);
  if ((M && !mz_buf) || (C && !cty_buf)) return set_err(ctx, SAD_EINVAL, "mass product buffers missing");
  const size_t esz = dtype == SAD_F64 ? 8 : 16;
  cudaStream_t sm = S_(stream_main), sa = S_(streamA), sb = S_(streamB);
  std::vector<cplx> G(6 * r * r), Gw(r * r), Gt(r * r);
  rc = sad_gram(ctx, nA, r, dtype, w, w, reinterpret_cast<double*>(Gw.data()), stream_main);
  if (rc) return rc;
  rc = sad_gram(ctx, nB, r, dtype, t, t, reinterpret_cast<double*>(Gt.data()), stream_main);
  if (rc) return rc;
  const double res0 = product_norm(Gw.data(), Gt.data(), r);
  summary[0] = res0;
  *steps_out = 0;
  if (res0 == 0.0) {
    summary[1] = 1.0;   // converged
    summary[2] = 0.0;
    return SAD_OK;
  }
  const double gap = cfg->has_gap_budget ? cfg->gap_budget : cfg->outer_tolerance * res0;
  double u = 0.0, v = 0.0, res = res0;
  int64_t itA[8], itB[8];
  double nrA[8], nrB[8];
  uint8_t cvA[8], cvB[8];
  cudaEvent_t ev = nullptr;
  CK(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  int k_done = 0;
  for (int k = 1; k <= cfg->kmax; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    const double eps_hat = adi_budget(*cfg, k, u, v, gap);
    double dA, dB;
    int clA, clB;
    adi_choose(*cfg, sigma_max_gram(Gw.data(), r), sigma_max_gram(Gt.data(), r), eps_hat, dA, dB,
               clA, clB);
    const double tolA = (dA > 0.0 ? dA : 1.0) / r, tolB = (dB > 0.0 ? dB : 1.0) / r;
    void* z = static_cast<char*>(z_base) + (size_t)(k - 1) * nA * r * esz;
    void* y = static_cast<char*>(y_base) + (size_t)(k - 1) * nB * r * esz;
    sad_op* oa = opsA[k - 1];
    sad_op* ob = opsB[k - 1];
    if (concurrent) {
      CK(ctx, cudaEventRecord(ev, sm));
      CK(ctx, cudaStreamWaitEvent(sa, ev, 0));
      CK(ctx, cudaStreamWaitEvent(sb, ev, 0));
      if ((rc = sad_gmres_launch(wsA, oa, w, z, tolA, cfg->max_inner_iterations, streamA))) break;
      if ((rc = sad_gmres_launch(wsB, ob, t, y, tolB, cfg->max_inner_iterations, streamB))) break;
      if ((rc = sad_gmres_finish(wsA, resA, streamA, itA, nrA, cvA))) break;
      if ((rc = sad_gmres_finish(wsB, resB, streamB, itB, nrB, cvB))) break;
    } else {
      if ((rc = sad_gmres_launch(wsA, oa, w, z, tolA, cfg->max_inner_iterations, stream_main))) break;
      if ((rc = sad_gmres_finish(wsA, resA, stream_main, itA, nrA, cvA))) break;
      if ((rc = sad_gmres_launch(wsB, ob, t, y, tolB, cfg->max_inner_iterations, stream_main))) break;
      if ((rc = sad_gmres_finish(wsB, resB, stream_main, itB, nrB, cvB))) break;
    }
    const double gre = gammas[2 * (k - 1)], gim = gammas[2 * (k - 1) + 1];
    const void* mz = z;
    const void* cty = y;
    if (M) {
      if ((rc = sad_csr_apply(M, 0, r, dtype, z, mz_buf, stream_main))) break;
      mz = mz_buf;
    }
    if (C) {
      if ((rc = sad_csr_apply(C, 1, r, dtype, y, cty_buf, stream_main))) break;
      cty = cty_buf;
    }
    rc = sad_adi_epilogue(ctx, nA, nB, r, dtype, gre, gim, mz, resA, w, cty, resB, t,
                          reinterpret_cast<double*>(G.data()), stream_main);
    if (rc) break;
    const cplx* Gp = G.data();
    const double rA = sigma_max_gram(Gp + 0 * r * r, r), rB = sigma_max_gram(Gp + 1 * r * r, r);
    const double ag = std::abs(cplx(gre, gim));
    u += ag * sigma_max_gram(Gp + 2 * r * r, r) * rB;
    v += ag * sigma_max_gram(Gp + 3 * r * r, r) * rA;
    for (int i = 0; i < r * r; ++i) {
      Gw[i] = Gp[4 * r * r + i];
      Gt[i] = Gp[5 * r * r + i];
    }
    res = product_norm(Gw.data(), Gt.data(), r);
    long long sa_it = 0, sb_it = 0;
    int ca = 1, cb = 1;
    for (int c = 0; c < r; ++c) {
      sa_it += itA[c];
      sb_it += itB[c];
      ca &= cvA[c] ? 1 : 0;
      cb &= cvB[c] ? 1 : 0;
    }
    double* rec = records + (size_t)(k - 1) * SAD_ADI_REC;
    rec[0] = res / res0;
    rec[1] = dA;
    rec[2] = dB;
    rec[3] = rA;
    rec[4] = rB;
    rec[5] = (double)sa_it;
    rec[6] = (double)sb_it;
    rec[7] = u;
    rec[8] = v;
    rec[9] = ca;
    rec[10] = cb;
    rec[11] = clA;
    rec[12] = clB;
    rec[13] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    k_done = k;
    if (res < cfg->outer_tolerance * res0) break;
  }
  cudaEventDestroy(ev);
  *steps_out = k_done;
  summary[1] = res < cfg->outer_tolerance * res0 ? 1.0 : 0.0;
  summary[2] = res / res0;
  summary[3] = u;
  summary[4] = v;
  return rc;
}
