"""Mutation check of the oracle's pins (test infrastructure).

For each plausible mistake in oracle/sipref.c (a dropped term, a wrong index,
a wrong schedule, ...) build a mutated copy of the oracle in a temporary
directory and run the CPU pin suite (tests/test_oracle_pins.py) against it.
A mutation must make at least one pin fail ("killed"); a surviving mutation
means a part of the oracle is unpinned.  DESIGN.md section 7 lists the
result.

usage: python tools/oracle_mutations.py [-k NAME]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, original text, mutated text) -- each original must occur exactly once
MUTATIONS = [
    ("vhat_new_y", "vh[i][j] = v[i][j] + rho[i] * (y[i][j] - s[i][j]);",
     "vh[i][j] = v[i][j] + rho[i] * (yn[j] - s[i][j]);"),
    ("vhat_new_v", "for (int64_t j = 0; j < M[i]; ++j) {\n        v[i][j] = rho[i] * (yn[j] - w[j]);\n        y[i][j] = yn[j];\n      }\n    }",
     "for (int64_t j = 0; j < M[i]; ++j) {\n        v[i][j] = rho[i] * (yn[j] - w[j]);\n        y[i][j] = yn[j];\n      }\n      if (adapt) for (int64_t j = 0; j < M[i]; ++j) vh[i][j] = v[i][j] + rho[i] * (y[i][j] - s[i][j]);\n    }"),
    ("adapt_even_k", "(k % o->adapt_every == 1)", "(k % o->adapt_every == 0)"),
    ("first_call_skips_snapshot", "      first_adapt = 0;\n", "      if (first_adapt) { first_adapt = 0; continue; }\n"),
    ("first_call_adapts", "      if (!first_adapt) {", "      if (1) {"),
    ("no_gamma_clamp", "if (gn > o->gamma_max) gn = o->gamma_max;", "(void)0;"),
    ("no_rho_ratio_clamp", "if (rho[i] < lo) rho[i] = lo;", "(void)lo;"),
    ("rho_clamp_before_new_rho_p1", "double lo = rho[p] / o->rho_ratio_cap, hi = rho[p] * o->rho_ratio_cap;",
     "double lo = o->rho0 / o->rho_ratio_cap, hi = o->rho0 * o->rho_ratio_cap;"),
    ("dg_sign", "double dg = -(y[i] - y0[i]);", "double dg = (y[i] - y0[i]);"),
    ("dh_against_current", "double dh = s[i] - s0[i];", "double dh = s[i];"),
    ("hist_window_4", "for (int j = 0; j < hist_count; ++j) {", "for (int j = 0; j < hist_count - 1; ++j) {"),
    ("hist_no_push", "    hist_head = (hist_head + 1) % S;\n    memcpy(hist[hist_head], x, (size_t)N * sizeof(double));",
     "    (void)0;"),
    ("check_every_off_by_one", "if (o->check_every > 0 && k % o->check_every == 0) {", "if (o->check_every > 0 && k % o->check_every == 1) {"),
    ("dist_prox_rho_i", "y[i] = (m[i] + rho * w[i]) / (1.0 + rho);", "y[i] = (m[i] + rho * w[i]) / (2.0 + rho);"),
    ("dual_sign", "v[i][j] = rho[i] * (yn[j] - w[j]);", "v[i][j] = rho[i] * (w[j] - yn[j]);"),
    ("relax_swapped", "xbar[j] = gam[i] * s[i][j] + (1.0 - gam[i]) * y[i][j];", "xbar[j] = gam[i] * y[i][j] + (1.0 - gam[i]) * s[i][j];"),
    ("w_no_dual", "w[j] = xbar[j] - v[i][j] / rho[i];", "w[j] = xbar[j];"),
    ("rhs_no_v", "u[j] = rho[i] * y[i][j] + v[i][j];", "u[j] = rho[i] * y[i][j];"),
    ("cg_no_eq25", "if (eq25 && sqrt(rr) / bn < tol) break;", "(void)tol;"),
    ("eq25_factor", "double tol = 0.1 * sqrt(rr) / bn;", "double tol = 0.5 * sqrt(rr) / bn;"),
    ("l1_theta_index", "double t = (cs - sigma) / (double)(j + 1);", "double t = (cs - sigma) / (double)(j + 2);"),
    ("card_ties_high_index", "static int cmp_keyidx(const void *pa, const void *pb) {\n  const keyidx *a = (const keyidx *)pa, *b = (const keyidx *)pb;\n  if (a->a > b->a) return -1;\n  if (a->a < b->a) return 1;\n  return (a->i > b->i) - (a->i < b->i);",
     "static int cmp_keyidx(const void *pa, const void *pb) {\n  const keyidx *a = (const keyidx *)pa, *b = (const keyidx *)pb;\n  if (a->a > b->a) return -1;\n  if (a->a < b->a) return 1;\n  return (a->i < b->i) - (a->i > b->i);"),
    ("rank_ties_high_index", "static int cmp_sv(const void *pa, const void *pb) {\n  const keyidx *a = (const keyidx *)pa, *b = (const keyidx *)pb;\n  if (a->a > b->a) return -1;\n  if (a->a < b->a) return 1;\n  return (a->i > b->i) - (a->i < b->i);",
     "static int cmp_sv(const void *pa, const void *pb) {\n  const keyidx *a = (const keyidx *)pa, *b = (const keyidx *)pb;\n  if (a->a > b->a) return -1;\n  if (a->a < b->a) return 1;\n  return (a->i < b->i) - (a->i > b->i);"),
    ("dz_adj_sign", "if (iz >= 1) a += y[((iz - 1) * g->n[1] + iy) * g->n[2] + ix];",
     "if (iz >= 1) a -= y[((iz - 1) * g->n[1] + iy) * g->n[2] + ix];"),
    ("dx_fwd_h", "(x[IDX(g, iz, iy, ix + 1)] - x[IDX(g, iz, iy, ix)]) / g->h[2];",
     "(x[IDX(g, iz, iy, ix + 1)] - x[IDX(g, iz, iy, ix)]) / g->h[0];"),
    ("annulus_zero_e1", "if (s->sigma_lo > 0.0 && M > 0) y[0] = s->sigma_lo;", "(void)0;"),
    ("feas_den", "double den = nrm2(M, sv);", "double den = 1.0 + 0.0 * nrm2(M, sv);"),
    ("restrict_mean", "double inv = 1.0 / (double)(2 * by * 2);", "double inv = 1.0 / (double)(2 * by * 2 + 1);"),
    ("prolong_dz_shape", "case SIPREF_OP_DZ: sipref_interp(cz - 1, cy, cx, c, fz - 1, fy, fx, f); break;",
     "case SIPREF_OP_DZ: sipref_interp(cz - 1, cy, cx, c, fz - 1, fy, fx, f); f[0] = c[0] + 1.0; break;"),
    ("prolong_tv_offset", "c += (cz - 1) * cy * cx; f += (fz - 1) * fy * fx;", "c += (cz - 1) * cy * cx; f += (fz - 2) * fy * fx;"),
    ("relative_l1_uses_l2", "if (in->type == SIPREF_L1) out->sigma = in->sigma * n1;", "if (in->type == SIPREF_L1) out->sigma = in->sigma * n2;"),
    ("relative_k_ceil", "out->k = (int64_t)floor(in->k_frac", "out->k = (int64_t)ceil(in->k_frac"),
    ("ml_rho_reset", "memcpy(rho, rbuf, (size_t)P * sizeof(double));", "(void)rbuf;"),
    ("svd_rotation_sign", "          xi[r] = cs * u - sn * v;", "          xi[r] = cs * u + sn * v;"),
    ("svd_loose_convergence", "if (c == 0.0 || fabs(c) <= 1e-15 * sqrt(a * b)) continue;",
     "if (c == 0.0 || fabs(c) <= 1e-3 * sqrt(a * b)) continue;"),
    ("rank_keeps_r_plus_1", "f[t[q].i] = (q < s->k) ? lam[t[q].i] : 0.0;", "f[t[q].i] = (q <= s->k) ? lam[t[q].i] : 0.0;"),
    ("nuclear_radius_halved", "proj_l1(n, lam, s->sigma, f);", "proj_l1(n, lam, 0.5 * s->sigma, f);"),
    ("matrix_view_3d_rows", "else { *rows = fy; *cols = fx; }", "else { *rows = fz; *cols = fx; }"),
    ("nuclear_relative_l1", "out->sigma = in->sigma * nuc;", "out->sigma = in->sigma * nuc * 1.0001;"),
    ("dct_dc_unscaled", "double s = kk == 0 ? sqrt(1.0 / (double)L) : sqrt(2.0 / (double)L);",
     "double s = sqrt(2.0 / (double)L);"),
    ("dct_inverse_is_forward", "int64_t kk = inverse ? n : k, nn = inverse ? k : n;", "int64_t kk = k, nn = n;"),
    ("dct_relative_untransformed", "    sipref_dct(g, 0, am, cm);\n    for (int64_t j = 0; j < M; ++j) n1d",
     "    memcpy(cm, am, (size_t)M * sizeof(double));\n    for (int64_t j = 0; j < M; ++j) n1d"),
    ("haar_unnormalised", "const double r2 = sqrt(0.5);", "const double r2 = 0.5;"),
    ("haar_one_level", "for (int64_t n = L; n > 1; n /= 2) {", "for (int64_t n = L; n > L / 2 && n > 1; n /= 2) {"),
    ("haar_inverse_swapped", "t[2 * i + 1] = (u[i] - u[n / 2 + i]) * r2;", "t[2 * i + 1] = (u[n / 2 + i] - u[i]) * r2;"),
    ("haar_z_axis_skipped", "  haar_axis(nz, 1, ny * nx, 0, ny * nx, inverse, y);\n", ""),
    ("dykstra_weight", "const double w = 1.0 / (double)p;", "const double w = 1.0 / (double)(p + 1);"),
    ("dykstra_v_sign", "v[i][j] = x[j] + v[i][j] - y[i][j];", "v[i][j] = x[j] - v[i][j] + y[i][j];"),
    ("dykstra_l1_count_all", "if (sets[i].type == SIPREF_L1) l1p += it;", "l1p += it;"),
]


def run(name, orig, mut, tmp):
    src = open(os.path.join(ROOT, "oracle", "sipref.c")).read()
    if src.count(orig) != 1:
        return name, "BAD-PATTERN"
    d = os.path.join(tmp, name)
    shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(d, "oracle"),
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    for sub in ("sip_inputs", "tests"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub), ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
    with open(os.path.join(d, "oracle", "sipref.c"), "w") as f:
        f.write(src.replace(orig, mut))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_oracle_pins.py"], cwd=d, capture_output=True, text=True, timeout=1200)
    killed = r.returncode != 0
    first = ""
    for line in r.stdout.splitlines():
        if line.startswith("FAILED"):
            first = line.split(" ")[1].split("::")[-1]
            break
    return name, ("killed by " + first) if killed else "SURVIVED"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    a = ap.parse_args()
    with tempfile.TemporaryDirectory() as tmp:
        for name, orig, mut in MUTATIONS:
            if a.k and a.k not in name:
                continue
            n, res = run(name, orig, mut, tmp)
            print(f"{n:32s} {res}", flush=True)


if __name__ == "__main__":
    main()
