/* hfb_oracle.c — TEST INFRASTRUCTURE ONLY (see hfb_oracle.h for the contract).
 *
 * Plain-C restatement of the reference's hot-path kernels, each function citing
 * the Hybrid-Fortran source it follows. Build: oracle/Makefile
 * (-O3 -ffp-contract=off -fopenmp). Never linked into the product library.
 */
#include "hfb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AT(v, k, i, j) ((v).p[(v).off + (int64_t)(k) * (v).sk + (int64_t)(i) * (v).si + (int64_t)(j) * (v).sj])
#define AT4(v, k, i, j, l)                                                                     \
  ((v).p[(v).off + (int64_t)(k) * (v).sk + (int64_t)(i) * (v).si + (int64_t)(j) * (v).sj +     \
         (int64_t)(l) * (v).sl])

int ora_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ora_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* interp.cpp:22-28 */
uint64_t ora_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void ora_fill(double* dst, int64_t n, uint64_t seed, double offset, double scale) {
#pragma omp parallel for schedule(static)
  for (int64_t f = 0; f < n; ++f) {
    double u = (double)(ora_splitmix64((seed << 40) + (uint64_t)f) >> 11) * 0x1.0p-53;
    dst[f] = offset + scale * u;
  }
}

/* ------------------------------------------------------------------------- */
/* diffusion.h90:23-41 — region 1 (7-point stencil, Dirichlet copy on the global
 * boundary), region 2 (t_old = t_new). */
void ora_diffuse_step(int64_t nx, int64_t ny, int64_t nz, double coef, ora_view t_old,
                      ora_view t_new) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        double c = AT(t_old, k, i, j);
        if (i == 1 || i == nx || j == 1 || j == ny || k == 1 || k == nz) {
          AT(t_new, k, i, j) = c;
        } else {
          double s = AT(t_old, k - 1, i, j) + AT(t_old, k + 1, i, j);
          s = s + AT(t_old, k, i - 1, j);
          s = s + AT(t_old, k, i + 1, j);
          s = s + AT(t_old, k, i, j - 1);
          s = s + AT(t_old, k, i, j + 1);
          s = s - 6.0 * c;
          AT(t_new, k, i, j) = c + coef * s;
        }
      }
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) AT(t_old, k, i, j) = AT(t_new, k, i, j);
}

/* diffusion.h90:44-54 */
void ora_diffusion_run(int64_t nsteps, int64_t nx, int64_t ny, int64_t nz, double coef,
                       ora_view t_old, ora_view t_new) {
  for (int64_t s = 0; s < nsteps; ++s) ora_diffuse_step(nx, ny, nz, coef, t_old, t_new);
}

/* damping.h90:38-48: d = (m*(r + b1) + t*(r + b2)) - r */
void ora_damping(int64_t nx_mn, int64_t nx_mx, int64_t ny_mn, int64_t ny_mx, int64_t nz_mn,
                 int64_t nz_mx, double tratio_bnd, double mtratio_bnd, ora_view dens_ref_f,
                 ora_view dens_ptb_damp, ora_view dens_ptb_bnd) {
#pragma omp parallel for schedule(static)
  for (int64_t j = ny_mn; j <= ny_mx; ++j)
    for (int64_t i = nx_mn; i <= nx_mx; ++i)
      for (int64_t k = nz_mn; k <= nz_mx; ++k) {
        double r = AT(dens_ref_f, k, i, j);
        double b1 = AT4(dens_ptb_bnd, k, i, j, 1);
        double b2 = AT4(dens_ptb_bnd, k, i, j, 2);
        AT(dens_ptb_damp, k, i, j) = (mtratio_bnd * (r + b1) + tratio_bnd * (r + b2)) - r;
      }
}

/* bounded.h90:19-21 over i in [2, nx-1], j in [2, ny-1] */
void ora_bounded(int64_t nx, int64_t ny, ora_view a, ora_view b) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 2; j <= ny - 1; ++j)
    for (int64_t i = 2; i <= nx - 1; ++i)
      AT(b, 0, i, j) = 0.25 * (((AT(a, 0, i - 1, j) + AT(a, 0, i + 1, j)) + AT(a, 0, i, j - 1)) +
                               AT(a, 0, i, j + 1));
}

/* driver.h90:3-17 */
void ora_sf_setup(int64_t ntlm, int64_t nx, int64_t ny, ora_view cover_frac) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t lt = 1; lt <= ntlm; ++lt) AT(cover_frac, lt, i, j) = AT(cover_frac, lt, i, j) - 0.5;
}

/* surface_flux.h90:3-10 (sf_slab_flx_land_run) inlined into :32-48 per column;
 * `x ** 2` is (1.0*x)*x == x*x exactly (interp.cpp:740-743). */
void ora_sf_physics_run(int64_t nx, int64_t ny, int64_t tile_land, ora_view cover_frac,
                        ora_view wind_speed, ora_view flx_sum_x, ora_view flx_sum_y) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) {
      double cf = AT(cover_frac, tile_land, i, j);
      double taux, tauy, uf;
      if (cf > 0.0) {
        taux = 0.1 * cf;
        tauy = 0.2 * cf * cf;
        uf = sqrt(sqrt(taux * taux + tauy * tauy));
      } else {
        taux = 0.0;
        tauy = 0.0;
        uf = 0.0;
      }
      AT(flx_sum_x, 0, i, j) = taux;
      AT(flx_sum_y, 0, i, j) = tauy;
      AT(wind_speed, 0, i, j) = uf;
    }
}

/* reduction.h90:21-25 */
double ora_grid_total(int64_t nx, int64_t ny, int64_t nz, double total, ora_view y, int mode) {
  if (mode == 0) {
    for (int64_t j = 1; j <= ny; ++j)
      for (int64_t i = 1; i <= nx; ++i)
        for (int64_t k = 1; k <= nz; ++k) total = total + AT(y, k, i, j);
    return total;
  }
  /* interp.cpp:1117-1173: per-iteration partials from the identity, combined in
   * linear-id order (innermost parallel loop, i, fastest) from the initial value. */
  double acc = total;
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) {
      double part = 0.0;
      for (int64_t k = 1; k <= nz; ++k) part = part + AT(y, k, i, j);
      acc += part;
    }
  return acc;
}

/* ------------------------------------------------------------------------- */
/* apps/dycore/dycore.h90 */

static inline double minmod(double a, double b) {
  /* dycore.h90 subroutine minmod */
  if (a * b <= 0.0) return 0.0;
  if (fabs(a) < fabs(b)) return a;
  return b;
}

typedef struct {
  double* p;
  int64_t nk, ni, nj; /* extents incl. the 0 face where declared */
  int64_t k0, i0, j0; /* lower bounds */
} scratch3;

static double* s3(scratch3* s, int64_t k, int64_t i, int64_t j) {
  return &s->p[((k - s->k0) * s->ni + (i - s->i0)) * s->nj + (j - s->j0)];
}

/* Scratch arrays persist across calls (the dialect's routine-local arrays are
 * re-elaborated per call; reusing the memory keeps page faults out of the timed CPU
 * baseline). Slot `id` grows on demand; not re-entrant. */
static double* g_scratch[9];
static size_t g_scratch_n[9];

static int s3_alloc(int id, scratch3* s, int64_t k0, int64_t k1, int64_t i0, int64_t i1,
                    int64_t j0, int64_t j1) {
  s->k0 = k0;
  s->i0 = i0;
  s->j0 = j0;
  s->nk = k1 - k0 + 1;
  s->ni = i1 - i0 + 1;
  s->nj = j1 - j0 + 1;
  size_t n = (size_t)(s->nk * s->ni * s->nj);
  if (g_scratch_n[id] < n) {
    free(g_scratch[id]);
    g_scratch[id] = (double*)malloc(sizeof(double) * n);
    g_scratch_n[id] = g_scratch[id] ? n : 0;
    if (g_scratch[id]) {
#pragma omp parallel for schedule(static)
      for (int64_t q = 0; q < (int64_t)n; ++q) g_scratch[id][q] = 0.0; /* first touch */
    }
  }
  s->p = g_scratch[id];
  return s->p != NULL;
}

/* One evaluation of the dynamics at the current state (th, u, v, w, p) applied with
 * step `dt` to the base state (thb, ub, vb, wb, pb); the result replaces the current
 * state. dycore_step is the stage with base == current and dt = q->dt; rk3_step runs
 * three stages with dt/3, dt/2, dt from the state at the start of the step. */
static int dycore_stage(const ora_dyn_params* q, double dt, ora_view rho, ora_view th,
                        ora_view u, ora_view v, ora_view w, ora_view p, ora_view thb,
                        ora_view ub, ora_view vb, ora_view wb, ora_view pb) {
  const int64_t nx = q->nx, ny = q->ny, nz = q->nz;
  const double rdx = q->rdx, rdy = q->rdy, rdz = q->rdz, cs2 = q->cs2, grav = q->grav,
               th0 = q->th0;
  if (nz < 2) return -1;
  scratch3 fx, fy, fz, thn, un, vn, ps, wn, pn;
  int ok = s3_alloc(0, &fx, 1, nz, 0, nx, 1, ny) & s3_alloc(1, &fy, 1, nz, 1, nx, 0, ny) &
           s3_alloc(2, &fz, 0, nz, 1, nx, 1, ny) & s3_alloc(3, &thn, 1, nz, 1, nx, 1, ny) &
           s3_alloc(4, &un, 1, nz, 1, nx, 1, ny) & s3_alloc(5, &vn, 1, nz, 1, nx, 1, ny) &
           s3_alloc(6, &ps, 1, nz, 1, nx, 1, ny) & s3_alloc(7, &wn, 1, nz, 1, nx, 1, ny) &
           s3_alloc(8, &pn, 1, nz, 1, nx, 1, ny);
  if (!ok) return -2;

  /* region 1: x-face fluxes, i = 0..nx */
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 0; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        double f;
        if (i == 0 || i == nx) {
          f = 0.0;
        } else if (AT(u, k, i, j) >= 0.0) {
          double s = (i == 1) ? 0.0
                              : minmod(AT(th, k, i, j) - AT(th, k, i - 1, j),
                                       AT(th, k, i + 1, j) - AT(th, k, i, j));
          f = AT(u, k, i, j) * (AT(th, k, i, j) + 0.5 * s);
        } else {
          double s = (i + 1 == nx) ? 0.0
                                   : minmod(AT(th, k, i + 1, j) - AT(th, k, i, j),
                                            AT(th, k, i + 2, j) - AT(th, k, i + 1, j));
          f = AT(u, k, i, j) * (AT(th, k, i + 1, j) - 0.5 * s);
        }
        *s3(&fx, k, i, j) = f;
      }
  /* region 2: y-face fluxes, j = 0..ny */
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        double f;
        if (j == 0 || j == ny) {
          f = 0.0;
        } else if (AT(v, k, i, j) >= 0.0) {
          double s = (j == 1) ? 0.0
                              : minmod(AT(th, k, i, j) - AT(th, k, i, j - 1),
                                       AT(th, k, i, j + 1) - AT(th, k, i, j));
          f = AT(v, k, i, j) * (AT(th, k, i, j) + 0.5 * s);
        } else {
          double s = (j + 1 == ny) ? 0.0
                                   : minmod(AT(th, k, i, j + 1) - AT(th, k, i, j),
                                            AT(th, k, i, j + 2) - AT(th, k, i, j + 1));
          f = AT(v, k, i, j) * (AT(th, k, i, j + 1) - 0.5 * s);
        }
        *s3(&fy, k, i, j) = f;
      }
  /* region 3: z-face fluxes, k = 0..nz */
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 0; k <= nz; ++k) {
        double f;
        if (k == 0 || k == nz) {
          f = 0.0;
        } else if (AT(w, k, i, j) >= 0.0) {
          double s = (k == 1) ? 0.0
                              : minmod(AT(th, k, i, j) - AT(th, k - 1, i, j),
                                       AT(th, k + 1, i, j) - AT(th, k, i, j));
          f = AT(w, k, i, j) * (AT(th, k, i, j) + 0.5 * s);
        } else {
          double s = (k + 1 == nz) ? 0.0
                                   : minmod(AT(th, k + 1, i, j) - AT(th, k, i, j),
                                            AT(th, k + 2, i, j) - AT(th, k + 1, i, j));
          f = AT(w, k, i, j) * (AT(th, k + 1, i, j) - 0.5 * s);
        }
        *s3(&fz, k, i, j) = f;
      }
  /* region 4: flux divergence + velocity-divergence correction */
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        double ue = (i == nx) ? 0.0 : AT(u, k, i, j);
        double uw = (i == 1) ? 0.0 : AT(u, k, i - 1, j);
        double vnf = (j == ny) ? 0.0 : AT(v, k, i, j);
        double vs = (j == 1) ? 0.0 : AT(v, k, i, j - 1);
        double wt = (k == nz) ? 0.0 : AT(w, k, i, j);
        double wb = (k == 1) ? 0.0 : AT(w, k - 1, i, j);
        double t = AT(th, k, i, j);
        double flux = rdx * (*s3(&fx, k, i, j) - *s3(&fx, k, i - 1, j)) +
                      rdy * (*s3(&fy, k, i, j) - *s3(&fy, k, i, j - 1));
        flux = flux + rdz * (*s3(&fz, k, i, j) - *s3(&fz, k - 1, i, j));
        double div = rdx * (ue - uw) + rdy * (vnf - vs);
        div = div + rdz * (wt - wb);
        *s3(&thn, k, i, j) = AT(thb, k, i, j) - dt * (flux - t * div);
      }
  /* region 5: horizontal pressure gradient */
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        *s3(&un, k, i, j) =
            (i == nx) ? 0.0 : AT(ub, k, i, j) - dt * rdx * (AT(p, k, i + 1, j) - AT(p, k, i, j));
        *s3(&vn, k, i, j) =
            (j == ny) ? 0.0 : AT(vb, k, i, j) - dt * rdy * (AT(p, k, i, j + 1) - AT(p, k, i, j));
      }
  /* region 6: pressure after the horizontal divergence */
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        double uw = (i == 1) ? 0.0 : *s3(&un, k, i - 1, j);
        double vs = (j == 1) ? 0.0 : *s3(&vn, k, i, j - 1);
        *s3(&ps, k, i, j) = AT(pb, k, i, j) - dt * cs2 * (rdx * (*s3(&un, k, i, j) - uw) +
                                                          rdy * (*s3(&vn, k, i, j) - vs));
      }
  /* region 7: HE-VI Thomas sweep per column, then the pressure update */
#pragma omp parallel
  {
    double* cp = (double*)malloc(sizeof(double) * (size_t)(nz + 1));
    double* dp = (double*)malloc(sizeof(double) * (size_t)(nz + 1));
#pragma omp for schedule(static)
    for (int64_t j = 1; j <= ny; ++j)
      for (int64_t i = 1; i <= nx; ++i) {
        for (int64_t k = 1; k <= nz - 1; ++k) {
          double rf = 0.5 * (AT(rho, k, i, j) + AT(rho, k + 1, i, j));
          double beta = dt * dt * cs2 * rdz * rdz / rf;
          double dd = AT(wb, k, i, j) - dt * rdz * (*s3(&ps, k + 1, i, j) - *s3(&ps, k, i, j)) / rf;
          dd = dd + dt * grav * (0.5 * (AT(th, k, i, j) + AT(th, k + 1, i, j)) - th0) / th0;
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
        *s3(&wn, nz, i, j) = 0.0;
        *s3(&wn, nz - 1, i, j) = dp[nz - 1];
        for (int64_t kk = 2; kk <= nz - 1; ++kk) {
          int64_t k = nz - kk;
          *s3(&wn, k, i, j) = dp[k] - cp[k] * *s3(&wn, k + 1, i, j);
        }
        for (int64_t k = 1; k <= nz; ++k) {
          if (k == 1)
            *s3(&pn, k, i, j) = *s3(&ps, k, i, j) - dt * cs2 * rdz * *s3(&wn, k, i, j);
          else
            *s3(&pn, k, i, j) =
                *s3(&ps, k, i, j) - dt * cs2 * rdz * (*s3(&wn, k, i, j) - *s3(&wn, k - 1, i, j));
        }
      }
    free(cp);
    free(dp);
  }
  /* region 8: state update */
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k) {
        AT(th, k, i, j) = *s3(&thn, k, i, j);
        AT(u, k, i, j) = *s3(&un, k, i, j);
        AT(v, k, i, j) = *s3(&vn, k, i, j);
        AT(w, k, i, j) = *s3(&wn, k, i, j);
        AT(p, k, i, j) = *s3(&pn, k, i, j);
      }
  return 0;
}

int ora_dycore_step(const ora_dyn_params* q, ora_view rho, ora_view th, ora_view u, ora_view v,
                    ora_view w, ora_view p) {
  return dycore_stage(q, q->dt, rho, th, u, v, w, p, th, u, v, w, p);
}

/* dycore.h90 rk3_step: base copies (routine locals), three stages */
static double* g_base[5];
static size_t g_base_n;

int ora_rk3_step(const ora_dyn_params* q, ora_view rho, ora_view th, ora_view u, ora_view v,
                 ora_view w, ora_view p) {
  const int64_t nx = q->nx, ny = q->ny, nz = q->nz;
  const size_t n = (size_t)(nx * ny * nz);
  if (g_base_n < n) {
    for (int f = 0; f < 5; ++f) {
      free(g_base[f]);
      g_base[f] = (double*)malloc(sizeof(double) * n);
      if (!g_base[f]) return -2;
    }
    g_base_n = n;
  }
  /* base views: (k, i, j) dense, j fastest */
  ora_view bv[5];
  for (int f = 0; f < 5; ++f) {
    bv[f].p = g_base[f];
    bv[f].sk = nx * ny;
    bv[f].si = ny;
    bv[f].sj = 1;
    bv[f].sl = 0;
    bv[f].off = -(bv[f].sk + bv[f].si + bv[f].sj);
  }
  ora_view cur[5] = {th, u, v, w, p};
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i)
      for (int64_t k = 1; k <= nz; ++k)
        for (int f = 0; f < 5; ++f) AT(bv[f], k, i, j) = AT(cur[f], k, i, j);
  const double dts[3] = {q->dt / 3.0, q->dt / 2.0, q->dt};
  for (int s = 0; s < 3; ++s) {
    int rc = dycore_stage(q, dts[s], rho, th, u, v, w, p, bv[0], bv[1], bv[2], bv[3], bv[4]);
    if (rc) return rc;
  }
  return 0;
}

int ora_rk3_run(int64_t nsteps, const ora_dyn_params* prm, ora_view rho, ora_view th, ora_view u,
                ora_view v, ora_view w, ora_view p) {
  for (int64_t s = 0; s < nsteps; ++s) {
    int rc = ora_rk3_step(prm, rho, th, u, v, w, p);
    if (rc) return rc;
  }
  return 0;
}

int ora_dycore_run(int64_t nsteps, const ora_dyn_params* prm, ora_view rho, ora_view th,
                   ora_view u, ora_view v, ora_view w, ora_view p) {
  for (int64_t s = 0; s < nsteps; ++s) {
    int rc = ora_dycore_step(prm, rho, th, u, v, w, p);
    if (rc) return rc;
  }
  return 0;
}

/* apps/dycore/dycore.h90 column_physics: per column, one K pass */
void ora_column_physics(const ora_dyn_params* q, double ch, double rrelax, ora_view rho,
                        ora_view th, ora_view u, ora_view v, ora_view tsfc, ora_view colm) {
  const int64_t nx = q->nx, ny = q->ny, nz = q->nz;
  const double dt = q->dt, rdz = q->rdz;
#pragma omp parallel for schedule(static)
  for (int64_t j = 1; j <= ny; ++j)
    for (int64_t i = 1; i <= nx; ++i) {
      double cs = 0.0, cm = 0.0;
      for (int64_t k = 1; k <= nz; ++k) {
        AT(th, k, i, j) = AT(th, k, i, j) - dt * rrelax * (AT(th, k, i, j) - AT(colm, 0, i, j));
        if (k == 1) {
          double wspd = sqrt(AT(u, k, i, j) * AT(u, k, i, j) + AT(v, k, i, j) * AT(v, k, i, j));
          AT(th, k, i, j) = AT(th, k, i, j) + dt * ch * wspd * (AT(tsfc, 0, i, j) - AT(th, k, i, j)) *
                                                   rdz / AT(rho, k, i, j);
        }
        cs = cs + AT(rho, k, i, j) * AT(th, k, i, j);
        cm = cm + AT(rho, k, i, j);
      }
      AT(colm, 0, i, j) = cs / cm;
    }
}

int ora_full_run(int64_t nsteps, const ora_dyn_params* prm, double ch, double rrelax,
                 ora_view rho, ora_view th, ora_view u, ora_view v, ora_view w, ora_view p,
                 ora_view tsfc, ora_view colm) {
  for (int64_t s = 0; s < nsteps; ++s) {
    int rc = ora_dycore_step(prm, rho, th, u, v, w, p);
    if (rc) return rc;
    ora_column_physics(prm, ch, rrelax, rho, th, u, v, tsfc, colm);
  }
  return 0;
}
