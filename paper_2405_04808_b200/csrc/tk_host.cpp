// Host-side setup routines of libtempokkt_b200.so (CPU, no CUDA calls):
//  * theta-method forward marches with per-step Newton (timedisc.py:152-191)
//    for van der Pol (problems.py:42-97) and P1 Burgers (problems.py:149-197),
//    exploiting the 2x2 / tridiagonal Jacobian instead of a dense LU;
//  * scalar cyclic-reduction coefficients for the constant control weight.
// These run once per hierarchy build, outside the timed hot path.
#include <math.h>
#include <string.h>

#include <vector>

#include "tempokkt_b200.h"

namespace {

constexpr int kNewtonMax = 25;  // timedisc.py:32

double norm2(const double* x, int n) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += x[k] * x[k];
    return sqrt(s);
}

// ---------------- van der Pol --------------------------------------------
void vdp_f(double mu, int nc, const double* u, const double* z, double* f) {
    const double z0 = nc == 2 ? z[0] : 0.0;
    const double z1 = nc == 2 ? z[1] : z[0];
    f[0] = u[1] + z0;
    f[1] = mu * (1.0 - u[0] * u[0]) * u[1] - u[0] + z1;
}

void vdp_residual(double dt, double th, double mu, int nc, const double* v, const double* u,
                  const double* z, double* r) {
    r[0] = v[0] - u[0];
    r[1] = v[1] - u[1];
    double f[2];
    if (th != 0.0) {
        vdp_f(mu, nc, u, z, f);
        r[0] = r[0] + dt * th * f[0];
        r[1] = r[1] + dt * th * f[1];
    }
    if (th != 1.0) {
        vdp_f(mu, nc, v, z, f);
        r[0] = r[0] + dt * (1.0 - th) * f[0];
        r[1] = r[1] + dt * (1.0 - th) * f[1];
    }
}

// ---------------- Burgers -------------------------------------------------
struct Burgers {
    int n;
    double h, nu, hs, hd;
    Burgers(int n_, double nu_) : n(n_), h(1.0 / (n_ + 1)), nu(nu_) {
        hs = h / 6.0;
        hd = 4.0 * h / 6.0;
    }
    // y = M x
    void mass(const double* x, double* y) const {
        for (int j = 0; j < n; ++j) {
            double s = hd * x[j];
            if (j > 0) s += hs * x[j - 1];
            if (j < n - 1) s += hs * x[j + 1];
            y[j] = s;
        }
    }
    // F(u, z) = -nu*A u - N(u) + M z
    void f(const double* u, const double* z, double* out, double* tmp) const {
        mass(z, tmp);
        for (int j = 0; j < n; ++j) {
            const double um = j > 0 ? u[j - 1] : 0.0;
            const double up = j < n - 1 ? u[j + 1] : 0.0;
            double au = (2.0 / h) * u[j];
            if (j > 0) au += (-1.0 / h) * um;
            if (j < n - 1) au += (-1.0 / h) * up;
            const double conv = (up * up + u[j] * up - u[j] * um - um * um) / 6.0;
            out[j] = -nu * au - conv + tmp[j];
        }
    }
    // tridiagonal F_u(u) as sub/diag/sup
    void fu(const double* u, double* sub, double* dia, double* sup) const {
        for (int j = 0; j < n; ++j) {
            const double um = j > 0 ? u[j - 1] : 0.0;
            const double up = j < n - 1 ? u[j + 1] : 0.0;
            dia[j] = (-nu) * (2.0 / h) - (up - um) / 6.0;
            sub[j] = j > 0 ? (-nu) * (-1.0 / h) - (-u[j] - 2.0 * um) / 6.0 : 0.0;
            sup[j] = j < n - 1 ? (-nu) * (-1.0 / h) - (2.0 * up + u[j]) / 6.0 : 0.0;
        }
    }
};

// Tridiagonal solve with partial pivoting (LAPACK dgtsv algorithm); a, b, c
// (sub, diag, sup) and rhs are overwritten.  Returns false if singular.
bool gtsv(int n, double* dl, double* d, double* du, double* rhs) {
    std::vector<double> du2(n > 2 ? n - 2 : 1, 0.0);
    for (int i = 0; i < n - 1; ++i) {
        if (fabs(d[i]) >= fabs(dl[i + 1])) {
            if (d[i] == 0.0) return false;
            const double fact = dl[i + 1] / d[i];
            d[i + 1] -= fact * du[i];
            rhs[i + 1] -= fact * rhs[i];
            if (i < n - 2) du2[i] = 0.0;
        } else {
            const double fact = d[i] / dl[i + 1];
            d[i] = dl[i + 1];
            double t = d[i + 1];
            d[i + 1] = du[i] - fact * t;
            if (i < n - 2) {
                du2[i] = du[i + 1];
                du[i + 1] = -fact * du2[i];
            }
            du[i] = t;
            t = rhs[i];
            rhs[i] = rhs[i + 1];
            rhs[i + 1] = t - fact * rhs[i + 1];
        }
    }
    if (d[n - 1] == 0.0) return false;
    rhs[n - 1] /= d[n - 1];
    if (n > 1) rhs[n - 2] = (rhs[n - 2] - du[n - 2] * rhs[n - 1]) / d[n - 2];
    for (int i = n - 3; i >= 0; --i)
        rhs[i] = (rhs[i] - du[i] * rhs[i + 1] - du2[i] * rhs[i + 2]) / d[i];
    return true;
}

}  // namespace

extern "C" {

int tk_forward_vanderpol_host(int32_t n_steps, double dt, double theta, double mu,
                              int32_t n_controls, const double* u0, const double* z,
                              double newton_tol, double* states) {
    if (n_steps < 1 || !u0 || !z || !states || (n_controls != 1 && n_controls != 2))
        return TK_ERR_ARG;
    double up[2] = {u0[0], u0[1]};
    for (int i = 0; i < n_steps; ++i) {
        const double* zi = z + (size_t)i * n_controls;
        double u[2] = {up[0], up[1]};
        const double tol = newton_tol * norm2(up, 2) + newton_tol;
        bool ok = false;
        double r[2];
        for (int it = 0; it < kNewtonMax; ++it) {
            vdp_residual(dt, theta, mu, n_controls, up, u, zi, r);
            if (norm2(r, 2) <= tol) { ok = true; break; }
            // K = -I + dt*theta*F_u(u)
            const double c = dt * theta;
            const double a00 = -1.0, a01 = c;
            const double a10 = c * (-2.0 * mu * u[0] * u[1] - 1.0);
            const double a11 = -1.0 + c * (mu * (1.0 - u[0] * u[0]));
            // 2x2 LU with partial pivoting
            double du0, du1;
            if (fabs(a00) >= fabs(a10)) {
                const double l = a10 / a00;
                const double u11 = a11 - l * a01;
                const double y1 = r[1] - l * r[0];
                du1 = y1 / u11;
                du0 = (r[0] - a01 * du1) / a00;
            } else {
                const double l = a00 / a10;
                const double u11 = a01 - l * a11;
                const double y1 = r[0] - l * r[1];
                du1 = y1 / u11;
                du0 = (r[1] - a11 * du1) / a10;
            }
            u[0] -= du0;
            u[1] -= du1;
        }
        if (!ok) {
            vdp_residual(dt, theta, mu, n_controls, up, u, zi, r);
            if (norm2(r, 2) > tol) return TK_ERR_NEWTON;
        }
        states[2 * i] = u[0];
        states[2 * i + 1] = u[1];
        up[0] = u[0];
        up[1] = u[1];
    }
    return TK_OK;
}

int tk_forward_burgers_host(int32_t n_steps, int32_t n_u, double dt, double theta, double nu,
                            const double* u0, const double* z, double newton_tol,
                            double* states) {
    if (n_steps < 1 || n_u < 2 || !u0 || !z || !states) return TK_ERR_ARG;
    const int n = n_u;
    Burgers P(n, nu);
    std::vector<double> up(u0, u0 + n), u(n), r(n), f(n), tmp(n), mu_(n), sub(n), dia(n), sup(n);
    for (int i = 0; i < n_steps; ++i) {
        const double* zi = z + (size_t)i * n;
        u = up;
        P.mass(up.data(), mu_.data());
        const double tol = newton_tol * norm2(mu_.data(), n) + newton_tol;
        bool ok = false;
        auto residual = [&]() {
            for (int j = 0; j < n; ++j) tmp[j] = up[j] - u[j];
            P.mass(tmp.data(), r.data());
            if (theta != 0.0) {
                P.f(u.data(), zi, f.data(), tmp.data());
                for (int j = 0; j < n; ++j) r[j] = r[j] + dt * theta * f[j];
            }
            if (theta != 1.0) {
                P.f(up.data(), zi, f.data(), tmp.data());
                for (int j = 0; j < n; ++j) r[j] = r[j] + dt * (1.0 - theta) * f[j];
            }
        };
        for (int it = 0; it < kNewtonMax; ++it) {
            residual();
            if (norm2(r.data(), n) <= tol) { ok = true; break; }
            P.fu(u.data(), sub.data(), dia.data(), sup.data());
            const double c = dt * theta;
            for (int j = 0; j < n; ++j) {
                sub[j] = -P.hs + c * sub[j];
                dia[j] = -P.hd + c * dia[j];
                sup[j] = -P.hs + c * sup[j];
            }
            // gtsv expects dl[i+1] = A(i+1, i), du[i] = A(i, i+1)
            if (!gtsv(n, sub.data(), dia.data(), sup.data(), r.data())) return TK_ERR_NEWTON;
            for (int j = 0; j < n; ++j) u[j] -= r[j];
        }
        if (!ok) {
            residual();
            if (norm2(r.data(), n) > tol) return TK_ERR_NEWTON;
        }
        memcpy(states + (size_t)i * n, u.data(), sizeof(double) * n);
        up = u;
    }
    return TK_OK;
}

int tk_cr_scalar_factor(int32_t n, const double* tri, double* out) {
    if (n < 1 || !tri || !out) return TK_ERR_ARG;
    std::vector<double> d(tri + n, tri + 2 * n), e(tri + 2 * n, tri + 3 * n);
    double* cinv = out;
    double* cup = out + n;
    double* clo = out + 2 * n;
    for (int j = 0; j < n; ++j) { cinv[j] = 0.0; cup[j] = 0.0; clo[j] = 0.0; }
    if (n >= 1) e[n - 1] = 0.0;
    int top = 0;
    while ((2 << top) <= n) ++top;  // floor(log2 n)
    for (int lev = 0; lev < top; ++lev) {
        const int s = 1 << lev;
        for (int p = s - 1; p < n; p += 2 * s) {
            cinv[p] = 1.0 / d[p];
            cup[p] = (p + s < n) ? e[p] : 0.0;
            clo[p] = (p - s >= 0) ? e[p - s] : 0.0;
        }
        for (int j = 2 * s - 1; j < n; j += 2 * s) {
            const int p = j - s, q = j + s;
            double dj = d[j] - e[p] * cinv[p] * e[p];
            double ej = 0.0;
            if (q < n) {
                dj -= e[j] * cinv[q] * e[j];
                if (q + s < n) ej = -e[j] * cinv[q] * e[q];
            }
            d[j] = dj;
            e[j] = ej;
        }
    }
    const int r = (1 << top) - 1;
    cinv[r] = 1.0 / d[r];
    return TK_OK;
}

int tk_cr_scalar_solve_host(int32_t n, const double* coef, const double* f, double* x) {
    if (n < 1 || !coef || !f || !x) return TK_ERR_ARG;
    const double* cinv = coef;
    const double* cup = coef + n;
    const double* clo = coef + 2 * n;
    std::vector<double> w(f, f + n);
    int top = 0;
    while ((2 << top) <= n) ++top;
    for (int lev = 0; lev < top; ++lev) {
        const int s = 1 << lev;
        for (int j = 2 * s - 1; j < n; j += 2 * s) {
            const int p = j - s, q = j + s;
            double v = w[j] - cup[p] * cinv[p] * w[p];
            if (q < n) v -= clo[q] * cinv[q] * w[q];
            w[j] = v;
        }
    }
    const int r = (1 << top) - 1;
    w[r] = cinv[r] * w[r];
    for (int lev = top - 1; lev >= 0; --lev) {
        const int s = 1 << lev;
        for (int p = s - 1; p < n; p += 2 * s) {
            double v = w[p];
            if (p - s >= 0) v -= clo[p] * w[p - s];
            if (p + s < n) v -= cup[p] * w[p + s];
            w[p] = cinv[p] * v;
        }
    }
    memcpy(x, w.data(), sizeof(double) * n);
    return TK_OK;
}

}  // extern "C"
