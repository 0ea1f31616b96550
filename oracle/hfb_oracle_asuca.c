/* hfb_oracle_asuca.c — TEST INFRASTRUCTURE ONLY: the CPU restatement of
 * apps/dycore/asuca.h90 (the ASUCA time scheme: RK3 long step, RK2 HE-VI acoustic
 * short steps with lateral/upper damping, limited advection of rho, theta and momentum),
 * region for region in the order the reference interpreter executes it under
 * run_reference (/root/reference/proj/src/interp.cpp:1271-1336: last domain outermost,
 * K innermost), binary64 with one rounding per operation and the reference parser's
 * left-associative trees (/root/reference/proj/src/parser.cpp:174-211). Compile with
 * -ffp-contract=off. Pinned by tests/test_oracle_golden.py against the asuca_* fixtures
 * the reference interpreter produced (tests/golden/make_golden.py).
 *
 * Routine-local arrays of asuca_step (fluxes, tendencies, the step's base state) are
 * materialised in scratch with the dialect's declared bounds. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "hfb_oracle.h"

#define AT(v, k, i, j) ((v).p[(v).off + (int64_t)(k) * (v).sk + (int64_t)(i) * (v).si + (int64_t)(j) * (v).sj])

typedef struct {
  double* p;
  int64_t k0, i0, j0, ni, nj;
} arr3;

#define A3(a, k, i, j) ((a).p[(((int64_t)(k) - (a).k0) * (a).ni + ((int64_t)(i) - (a).i0)) * (a).nj + ((int64_t)(j) - (a).j0)])

enum {
  RHOB, THB, UB, VB, WBB, PB, FRHO, FTH, FU, FV, FW,
  FXT, FYT, FZT, FXR, FYR, FZR,
  GXU, GYU, GZU, CXU, CYU, CZU,
  GXV, GYV, GZV, CXV, CYV, CZV,
  GXW, GYW, GZW, CXW, CYW, CZW,
  UN, VN, PS, PA, WN, PN, NSCR
};

static double* g_buf[NSCR];
static size_t g_cap[NSCR];

static int mk(int id, arr3* a, int64_t k0, int64_t k1, int64_t i0, int64_t i1, int64_t j0,
              int64_t j1) {
  a->k0 = k0;
  a->i0 = i0;
  a->j0 = j0;
  a->ni = i1 - i0 + 1;
  a->nj = j1 - j0 + 1;
  size_t n = (size_t)((k1 - k0 + 1) * a->ni * a->nj);
  if (g_cap[id] < n) {
    free(g_buf[id]);
    g_buf[id] = (double*)calloc(n, sizeof(double));
    g_cap[id] = g_buf[id] ? n : 0;
  }
  a->p = g_buf[id];
  return a->p != NULL;
}

/* asuca.h90 asu_minmod / asu_flux */
static inline double asu_minmod(double a, double b) {
  if (a * b <= 0.0) return 0.0;
  if (fabs(a) < fabs(b)) return a;
  return b;
}

static inline double asu_flux(double vel, double qm1, double q0, double qp1, double qp2, int lo,
                              int hi) {
  if (vel >= 0.0) {
    double s = lo ? 0.0 : asu_minmod(q0 - qm1, qp1 - q0);
    return vel * (q0 + 0.5 * s);
  }
  double s = hi ? 0.0 : asu_minmod(qp1 - q0, qp2 - qp1);
  return vel * (qp1 - 0.5 * s);
}

static inline int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
/* interp.cpp:629-645 max: the first argument unless a later one is strictly greater */
static inline double dmax(double a, double b) { return b > a ? b : a; }

#define FOR_JIK(ilo, ihi, jlo, jhi, klo, khi)                 \
  _Pragma("omp parallel for schedule(static)")                \
  for (int64_t j = (jlo); j <= (jhi); ++j)                    \
    for (int64_t i = (ilo); i <= (ihi); ++i)                  \
      for (int64_t k = (klo); k <= (khi); ++k)

/* the HE-VI column solve of step h from (w, ps): writes the solved w into wout (whole
 * column, wout(nz) = 0) and the updated pressure into pout */
static void hevi(const ora_asuca_params* q, double h, ora_view rho, ora_view th, ora_view w,
                 arr3 fw, arr3 ps, arr3* wout, arr3 pout) {
  const int64_t nx = q->nx, ny = q->ny, nz = q->nz;
  const double cs2 = q->cs2, rdz = q->rdz, grav = q->grav, th0 = q->th0;
#pragma omp parallel
  {
    double* cp = (double*)malloc(sizeof(double) * (size_t)(nz + 1));
    double* dp = (double*)malloc(sizeof(double) * (size_t)(nz + 1));
    double* wc = (double*)malloc(sizeof(double) * (size_t)(nz + 1));
#pragma omp for schedule(static)
    for (int64_t j = 1; j <= ny; ++j)
      for (int64_t i = 1; i <= nx; ++i) {
        for (int64_t k = 1; k <= nz - 1; ++k) {
          double rf = 0.5 * (AT(rho, k, i, j) + AT(rho, k + 1, i, j));
          double beta = h * h * cs2 * rdz * rdz / rf;
          double dd = AT(w, k, i, j) - h * rdz * (A3(ps, k + 1, i, j) - A3(ps, k, i, j)) / rf;
          dd = dd + h * grav * (0.5 * (AT(th, k, i, j) + AT(th, k + 1, i, j)) - th0) / th0;
          dd = dd + h * A3(fw, k, i, j);
          double bb = 1.0 + 2.0 * beta;
          if (k == 1) {
            cp[k] = -beta / bb;
            dp[k] = dd / bb;
          } else {
            double m = bb + beta * cp[k - 1];
            cp[k] = -beta / m;
            dp[k] = (dd + beta * dp[k - 1]) / m;
          }
        }
        wc[nz] = 0.0;
        wc[nz - 1] = dp[nz - 1];
        for (int64_t kk = 2; kk <= nz - 1; ++kk) {
          int64_t k = nz - kk;
          wc[k] = dp[k] - cp[k] * wc[k + 1];
        }
        for (int64_t k = 1; k <= nz; ++k) {
          if (wout) A3(*wout, k, i, j) = wc[k];
          if (k == 1)
            A3(pout, k, i, j) = A3(ps, k, i, j) - h * cs2 * rdz * wc[k];
          else
            A3(pout, k, i, j) = A3(ps, k, i, j) - h * cs2 * rdz * (wc[k] - wc[k - 1]);
        }
      }
    free(cp);
    free(dp);
    free(wc);
  }
}

/* PGF (h) from u, v at pressure pp plus h * slow tendency, then the pressure after the
 * horizontal divergence */
static void pgf_div(const ora_asuca_params* q, double h, ora_view u, ora_view v, ora_view p,
                    const double* pp_base, arr3 pp, int use_arr, arr3 fu, arr3 fv, arr3 un,
                    arr3 vn, arr3 ps) {
  const int64_t nx = q->nx, ny = q->ny, nz = q->nz;
  const double rdx = q->rdx, rdy = q->rdy, cs2 = q->cs2;
  (void)pp_base;
#define PP(k, i, j) (use_arr ? A3(pp, k, i, j) : AT(p, k, i, j))
  FOR_JIK(1, nx, 1, ny, 1, nz) {
    A3(un, k, i, j) = (i == nx) ? 0.0
                                : AT(u, k, i, j) - h * rdx * (PP(k, i + 1, j) - PP(k, i, j)) +
                                      h * A3(fu, k, i, j);
    A3(vn, k, i, j) = (j == ny) ? 0.0
                                : AT(v, k, i, j) - h * rdy * (PP(k, i, j + 1) - PP(k, i, j)) +
                                      h * A3(fv, k, i, j);
  }
#undef PP
  FOR_JIK(1, nx, 1, ny, 1, nz) {
    double uw = (i == 1) ? 0.0 : A3(un, k, i - 1, j);
    double vs = (j == 1) ? 0.0 : A3(vn, k, i, j - 1);
    A3(ps, k, i, j) = AT(p, k, i, j) - h * cs2 * (rdx * (A3(un, k, i, j) - uw) +
                                                  rdy * (A3(vn, k, i, j) - vs));
  }
}

int ora_asuca_step(const ora_asuca_params* q, ora_view rho, ora_view th, ora_view u,
                   ora_view v, ora_view w, ora_view p) {
  const int64_t nx = q->nx, ny = q->ny, nz = q->nz;
  const double rdx = q->rdx, rdy = q->rdy, rdz = q->rdz, dt = q->dt;
  if (nz < 2 || q->nsound < 3) return -1;
  arr3 a[NSCR];
  int ok = 1;
  for (int id = RHOB; id <= FW; ++id) ok &= mk(id, &a[id], 1, nz, 1, nx, 1, ny);
  ok &= mk(FXT, &a[FXT], 1, nz, 0, nx, 1, ny) & mk(FYT, &a[FYT], 1, nz, 1, nx, 0, ny) &
        mk(FZT, &a[FZT], 0, nz, 1, nx, 1, ny) & mk(FXR, &a[FXR], 1, nz, 0, nx, 1, ny) &
        mk(FYR, &a[FYR], 1, nz, 1, nx, 0, ny) & mk(FZR, &a[FZR], 0, nz, 1, nx, 1, ny);
  ok &= mk(GXU, &a[GXU], 1, nz, 1, nx, 1, ny) & mk(GYU, &a[GYU], 1, nz, 1, nx, 0, ny) &
        mk(GZU, &a[GZU], 0, nz, 1, nx, 1, ny) & mk(CXU, &a[CXU], 1, nz, 1, nx, 1, ny) &
        mk(CYU, &a[CYU], 1, nz, 1, nx, 0, ny) & mk(CZU, &a[CZU], 0, nz, 1, nx, 1, ny);
  ok &= mk(GXV, &a[GXV], 1, nz, 0, nx, 1, ny) & mk(GYV, &a[GYV], 1, nz, 1, nx, 1, ny) &
        mk(GZV, &a[GZV], 0, nz, 1, nx, 1, ny) & mk(CXV, &a[CXV], 1, nz, 0, nx, 1, ny) &
        mk(CYV, &a[CYV], 1, nz, 1, nx, 1, ny) & mk(CZV, &a[CZV], 0, nz, 1, nx, 1, ny);
  ok &= mk(GXW, &a[GXW], 1, nz, 0, nx, 1, ny) & mk(GYW, &a[GYW], 1, nz, 1, nx, 0, ny) &
        mk(GZW, &a[GZW], 1, nz, 1, nx, 1, ny) & mk(CXW, &a[CXW], 1, nz, 0, nx, 1, ny) &
        mk(CYW, &a[CYW], 1, nz, 1, nx, 0, ny) & mk(CZW, &a[CZW], 1, nz, 1, nx, 1, ny);
  for (int id = UN; id <= PN; ++id) ok &= mk(id, &a[id], 1, nz, 1, nx, 1, ny);
  if (!ok) return -2;

  const double dtau = dt / (double)q->nsound;
  FOR_JIK(1, nx, 1, ny, 1, nz) {
    A3(a[RHOB], k, i, j) = AT(rho, k, i, j);
    A3(a[THB], k, i, j) = AT(th, k, i, j);
    A3(a[UB], k, i, j) = AT(u, k, i, j);
    A3(a[VB], k, i, j) = AT(v, k, i, j);
    A3(a[WBB], k, i, j) = AT(w, k, i, j);
    A3(a[PB], k, i, j) = AT(p, k, i, j);
  }
  for (int stg = 1; stg <= 3; ++stg) {
    double dtf;
    int64_t nsm;
    if (stg == 1) {
      dtf = dt / 3.0;
      nsm = q->nsound / 3;
    } else if (stg == 2) {
      dtf = dt / 2.0;
      nsm = q->nsound / 2;
    } else {
      dtf = dt;
      nsm = q->nsound;
    }
    /* theta / rho face fluxes */
    FOR_JIK(0, nx, 1, ny, 1, nz) {
      if (i == 0 || i == nx) {
        A3(a[FXT], k, i, j) = 0.0;
        A3(a[FXR], k, i, j) = 0.0;
      } else {
        A3(a[FXT], k, i, j) = asu_flux(AT(u, k, i, j), AT(th, k, imax(i - 1, 1), j), AT(th, k, i, j),
                                       AT(th, k, i + 1, j), AT(th, k, imin(i + 2, nx), j), i == 1,
                                       i + 1 == nx);
        A3(a[FXR], k, i, j) = asu_flux(AT(u, k, i, j), AT(rho, k, imax(i - 1, 1), j),
                                       AT(rho, k, i, j), AT(rho, k, i + 1, j),
                                       AT(rho, k, imin(i + 2, nx), j), i == 1, i + 1 == nx);
      }
    }
    FOR_JIK(1, nx, 0, ny, 1, nz) {
      if (j == 0 || j == ny) {
        A3(a[FYT], k, i, j) = 0.0;
        A3(a[FYR], k, i, j) = 0.0;
      } else {
        A3(a[FYT], k, i, j) = asu_flux(AT(v, k, i, j), AT(th, k, i, imax(j - 1, 1)), AT(th, k, i, j),
                                       AT(th, k, i, j + 1), AT(th, k, i, imin(j + 2, ny)), j == 1,
                                       j + 1 == ny);
        A3(a[FYR], k, i, j) = asu_flux(AT(v, k, i, j), AT(rho, k, i, imax(j - 1, 1)),
                                       AT(rho, k, i, j), AT(rho, k, i, j + 1),
                                       AT(rho, k, i, imin(j + 2, ny)), j == 1, j + 1 == ny);
      }
    }
    FOR_JIK(1, nx, 1, ny, 0, nz) {
      if (k == 0 || k == nz) {
        A3(a[FZT], k, i, j) = 0.0;
        A3(a[FZR], k, i, j) = 0.0;
      } else {
        A3(a[FZT], k, i, j) = asu_flux(AT(w, k, i, j), AT(th, imax(k - 1, 1), i, j), AT(th, k, i, j),
                                       AT(th, k + 1, i, j), AT(th, imin(k + 2, nz), i, j), k == 1,
                                       k + 1 == nz);
        A3(a[FZR], k, i, j) = asu_flux(AT(w, k, i, j), AT(rho, imax(k - 1, 1), i, j),
                                       AT(rho, k, i, j), AT(rho, k + 1, i, j),
                                       AT(rho, imin(k + 2, nz), i, j), k == 1, k + 1 == nz);
      }
    }
    /* u: x through the cell centres */
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      double qb = (i == 1) ? 0.0 : AT(u, k, i - 1, j);
      double qc = (i == nx) ? 0.0 : AT(u, k, i, j);
      double qa = (i <= 2) ? 0.0 : AT(u, k, i - 2, j);
      double qd = (i + 1 >= nx) ? 0.0 : AT(u, k, i + 1, j);
      A3(a[CXU], k, i, j) = 0.5 * (qb + qc);
      A3(a[GXU], k, i, j) = asu_flux(A3(a[CXU], k, i, j), qa, qb, qc, qd, i == 1, i == nx);
    }
    FOR_JIK(1, nx, 0, ny, 1, nz) {
      if (j == 0 || j == ny || i == nx) {
        A3(a[CYU], k, i, j) = 0.0;
        A3(a[GYU], k, i, j) = 0.0;
      } else {
        A3(a[CYU], k, i, j) = 0.5 * (AT(v, k, i, j) + AT(v, k, i + 1, j));
        A3(a[GYU], k, i, j) = asu_flux(A3(a[CYU], k, i, j), AT(u, k, i, imax(j - 1, 1)), AT(u, k, i, j),
                                       AT(u, k, i, j + 1), AT(u, k, i, imin(j + 2, ny)), j == 1,
                                       j + 1 == ny);
      }
    }
    FOR_JIK(1, nx, 1, ny, 0, nz) {
      if (k == 0 || k == nz || i == nx) {
        A3(a[CZU], k, i, j) = 0.0;
        A3(a[GZU], k, i, j) = 0.0;
      } else {
        A3(a[CZU], k, i, j) = 0.5 * (AT(w, k, i, j) + AT(w, k, i + 1, j));
        A3(a[GZU], k, i, j) = asu_flux(A3(a[CZU], k, i, j), AT(u, imax(k - 1, 1), i, j), AT(u, k, i, j),
                                       AT(u, k + 1, i, j), AT(u, imin(k + 2, nz), i, j), k == 1,
                                       k + 1 == nz);
      }
    }
    /* v */
    FOR_JIK(0, nx, 1, ny, 1, nz) {
      if (i == 0 || i == nx || j == ny) {
        A3(a[CXV], k, i, j) = 0.0;
        A3(a[GXV], k, i, j) = 0.0;
      } else {
        A3(a[CXV], k, i, j) = 0.5 * (AT(u, k, i, j) + AT(u, k, i, j + 1));
        A3(a[GXV], k, i, j) = asu_flux(A3(a[CXV], k, i, j), AT(v, k, imax(i - 1, 1), j), AT(v, k, i, j),
                                       AT(v, k, i + 1, j), AT(v, k, imin(i + 2, nx), j), i == 1,
                                       i + 1 == nx);
      }
    }
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      double qb = (j == 1) ? 0.0 : AT(v, k, i, j - 1);
      double qc = (j == ny) ? 0.0 : AT(v, k, i, j);
      double qa = (j <= 2) ? 0.0 : AT(v, k, i, j - 2);
      double qd = (j + 1 >= ny) ? 0.0 : AT(v, k, i, j + 1);
      A3(a[CYV], k, i, j) = 0.5 * (qb + qc);
      A3(a[GYV], k, i, j) = asu_flux(A3(a[CYV], k, i, j), qa, qb, qc, qd, j == 1, j == ny);
    }
    FOR_JIK(1, nx, 1, ny, 0, nz) {
      if (k == 0 || k == nz || j == ny) {
        A3(a[CZV], k, i, j) = 0.0;
        A3(a[GZV], k, i, j) = 0.0;
      } else {
        A3(a[CZV], k, i, j) = 0.5 * (AT(w, k, i, j) + AT(w, k, i, j + 1));
        A3(a[GZV], k, i, j) = asu_flux(A3(a[CZV], k, i, j), AT(v, imax(k - 1, 1), i, j), AT(v, k, i, j),
                                       AT(v, k + 1, i, j), AT(v, imin(k + 2, nz), i, j), k == 1,
                                       k + 1 == nz);
      }
    }
    /* w */
    FOR_JIK(0, nx, 1, ny, 1, nz) {
      if (i == 0 || i == nx || k == nz) {
        A3(a[CXW], k, i, j) = 0.0;
        A3(a[GXW], k, i, j) = 0.0;
      } else {
        A3(a[CXW], k, i, j) = 0.5 * (AT(u, k, i, j) + AT(u, k + 1, i, j));
        A3(a[GXW], k, i, j) = asu_flux(A3(a[CXW], k, i, j), AT(w, k, imax(i - 1, 1), j), AT(w, k, i, j),
                                       AT(w, k, i + 1, j), AT(w, k, imin(i + 2, nx), j), i == 1,
                                       i + 1 == nx);
      }
    }
    FOR_JIK(1, nx, 0, ny, 1, nz) {
      if (j == 0 || j == ny || k == nz) {
        A3(a[CYW], k, i, j) = 0.0;
        A3(a[GYW], k, i, j) = 0.0;
      } else {
        A3(a[CYW], k, i, j) = 0.5 * (AT(v, k, i, j) + AT(v, k + 1, i, j));
        A3(a[GYW], k, i, j) = asu_flux(A3(a[CYW], k, i, j), AT(w, k, i, imax(j - 1, 1)), AT(w, k, i, j),
                                       AT(w, k, i, j + 1), AT(w, k, i, imin(j + 2, ny)), j == 1,
                                       j + 1 == ny);
      }
    }
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      double qb = (k == 1) ? 0.0 : AT(w, k - 1, i, j);
      double qc = (k == nz) ? 0.0 : AT(w, k, i, j);
      double qa = (k <= 2) ? 0.0 : AT(w, k - 2, i, j);
      double qd = (k + 1 >= nz) ? 0.0 : AT(w, k + 1, i, j);
      A3(a[CZW], k, i, j) = 0.5 * (qb + qc);
      A3(a[GZW], k, i, j) = asu_flux(A3(a[CZW], k, i, j), qa, qb, qc, qd, k == 1, k == nz);
    }
    /* theta (advective form) and rho (flux form) tendencies */
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      double ue = (i == nx) ? 0.0 : AT(u, k, i, j);
      double uw = (i == 1) ? 0.0 : AT(u, k, i - 1, j);
      double vnf = (j == ny) ? 0.0 : AT(v, k, i, j);
      double vs = (j == 1) ? 0.0 : AT(v, k, i, j - 1);
      double wt = (k == nz) ? 0.0 : AT(w, k, i, j);
      double wb = (k == 1) ? 0.0 : AT(w, k - 1, i, j);
      double div = rdx * (ue - uw) + rdy * (vnf - vs);
      div = div + rdz * (wt - wb);
      double flux = rdx * (A3(a[FXT], k, i, j) - A3(a[FXT], k, i - 1, j)) +
                    rdy * (A3(a[FYT], k, i, j) - A3(a[FYT], k, i, j - 1));
      flux = flux + rdz * (A3(a[FZT], k, i, j) - A3(a[FZT], k - 1, i, j));
      A3(a[FTH], k, i, j) = AT(th, k, i, j) * div - flux;
      flux = rdx * (A3(a[FXR], k, i, j) - A3(a[FXR], k, i - 1, j)) +
             rdy * (A3(a[FYR], k, i, j) - A3(a[FYR], k, i, j - 1));
      flux = flux + rdz * (A3(a[FZR], k, i, j) - A3(a[FZR], k - 1, i, j));
      A3(a[FRHO], k, i, j) = 0.0 - flux;
    }
    /* momentum tendencies */
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      double div, flux;
      if (i == nx) {
        A3(a[FU], k, i, j) = 0.0;
      } else {
        div = rdx * (A3(a[CXU], k, i + 1, j) - A3(a[CXU], k, i, j)) +
              rdy * (A3(a[CYU], k, i, j) - A3(a[CYU], k, i, j - 1));
        div = div + rdz * (A3(a[CZU], k, i, j) - A3(a[CZU], k - 1, i, j));
        flux = rdx * (A3(a[GXU], k, i + 1, j) - A3(a[GXU], k, i, j)) +
               rdy * (A3(a[GYU], k, i, j) - A3(a[GYU], k, i, j - 1));
        flux = flux + rdz * (A3(a[GZU], k, i, j) - A3(a[GZU], k - 1, i, j));
        A3(a[FU], k, i, j) = AT(u, k, i, j) * div - flux;
      }
      if (j == ny) {
        A3(a[FV], k, i, j) = 0.0;
      } else {
        div = rdx * (A3(a[CXV], k, i, j) - A3(a[CXV], k, i - 1, j)) +
              rdy * (A3(a[CYV], k, i, j + 1) - A3(a[CYV], k, i, j));
        div = div + rdz * (A3(a[CZV], k, i, j) - A3(a[CZV], k - 1, i, j));
        flux = rdx * (A3(a[GXV], k, i, j) - A3(a[GXV], k, i - 1, j)) +
               rdy * (A3(a[GYV], k, i, j + 1) - A3(a[GYV], k, i, j));
        flux = flux + rdz * (A3(a[GZV], k, i, j) - A3(a[GZV], k - 1, i, j));
        A3(a[FV], k, i, j) = AT(v, k, i, j) * div - flux;
      }
      if (k == nz) {
        A3(a[FW], k, i, j) = 0.0;
      } else {
        div = rdx * (A3(a[CXW], k, i, j) - A3(a[CXW], k, i - 1, j)) +
              rdy * (A3(a[CYW], k, i, j) - A3(a[CYW], k, i, j - 1));
        div = div + rdz * (A3(a[CZW], k + 1, i, j) - A3(a[CZW], k, i, j));
        flux = rdx * (A3(a[GXW], k, i, j) - A3(a[GXW], k, i - 1, j)) +
               rdy * (A3(a[GYW], k, i, j) - A3(a[GYW], k, i, j - 1));
        flux = flux + rdz * (A3(a[GZW], k + 1, i, j) - A3(a[GZW], k, i, j));
        A3(a[FW], k, i, j) = AT(w, k, i, j) * div - flux;
      }
    }
    /* acoustic short steps from the state at the start of the step */
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      AT(u, k, i, j) = A3(a[UB], k, i, j);
      AT(v, k, i, j) = A3(a[VB], k, i, j);
      AT(w, k, i, j) = A3(a[WBB], k, i, j);
      AT(p, k, i, j) = A3(a[PB], k, i, j);
    }
    for (int64_t ss = 1; ss <= nsm; ++ss) {
      const double h = 0.5 * dtau;
      pgf_div(q, h, u, v, p, NULL, a[PA], 0, a[FU], a[FV], a[UN], a[VN], a[PS]);
      hevi(q, h, rho, th, w, a[FW], a[PS], NULL, a[PA]);
      pgf_div(q, dtau, u, v, p, NULL, a[PA], 1, a[FU], a[FV], a[UN], a[VN], a[PS]);
      hevi(q, dtau, rho, th, w, a[FW], a[PS], &a[WN], a[PN]);
      /* damping + the short-step state */
#pragma omp parallel for schedule(static)
      for (int64_t j = 1; j <= ny; ++j)
        for (int64_t i = 1; i <= nx; ++i) {
          double ax = (double)imax(0, imax(q->nbnd + 1 - i, i - nx + q->nbnd)) * q->rnbnd;
          double ay = (double)imax(0, imax(q->nbnd + 1 - j, j - ny + q->nbnd)) * q->rnbnd;
          for (int64_t k = 1; k <= nz; ++k) {
            double az = (double)imax(0, k - q->kdmp) * q->rnzd;
            double tau = dtau * q->rdmp * dmax(dmax(ax, ay), az);
            AT(u, k, i, j) = A3(a[UN], k, i, j) - tau * A3(a[UN], k, i, j);
            AT(v, k, i, j) = A3(a[VN], k, i, j) - tau * A3(a[VN], k, i, j);
            AT(w, k, i, j) = A3(a[WN], k, i, j) - tau * A3(a[WN], k, i, j);
            AT(p, k, i, j) = A3(a[PN], k, i, j);
          }
        }
    }
    /* end of the stage */
    FOR_JIK(1, nx, 1, ny, 1, nz) {
      AT(th, k, i, j) = A3(a[THB], k, i, j) + dtf * A3(a[FTH], k, i, j);
      AT(rho, k, i, j) = A3(a[RHOB], k, i, j) + dtf * A3(a[FRHO], k, i, j);
    }
  }
  return 0;
}

int ora_asuca_run(int64_t nsteps, const ora_asuca_params* prm, ora_view rho, ora_view th,
                  ora_view u, ora_view v, ora_view w, ora_view p) {
  for (int64_t s = 0; s < nsteps; ++s) {
    int rc = ora_asuca_step(prm, rho, th, u, v, w, p);
    if (rc) return rc;
  }
  return 0;
}
