/*
 * oracle/mpap_oracle.c -- plain, slow, sequential CPU oracle of the MPAP hot
 * path (Ichter et al., arXiv 1705.02408; /root/reference/PAPER.md = "P:n").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1705_02408_b200/csrc); both follow the numeric contract written in
 * DESIGN.md §3 ("Numeric contract"), each implemented independently.
 *
 * What it computes, in the paper's order and notation:
 *   orc_build   -- Alg. 2 BuildGraph + Alg. 1 line 2 heuristic
 *                  precompute (§4.1 heuristic P:323-328,
 *                  §5.2 learned heuristic P:476-477), under readings R6-R12.
 *   orc_search  -- Alg. 3 Explore literally: P, P_open, G, i,
 *                  RemoveDominated, PH, cutoff (A3.9),
 *                  termination (A3.5), argmin (A3.20-21)
 *                  under readings R3-R5, R13-R16, R24-R27.
 *   orc_mc_*    -- Alg. 1 step 4 Monte Carlo verification
 *                  with the §4.1 simulation model, readings
 *                  R31-R36 (NEXT-4).
 *
 * Pins: tests/test_oracle_*.py (closed forms, brute force, Dijkstra in the
 * exact regime, dense-sampling collision, SPEC worked examples; Monte Carlo:
 * double-integrated white-noise variance, exact fixes, Kalman consistency,
 * zero-noise tracking).  tests/test_oracle_pins.py pins mlp_out0 (exact
 * rational forward pass), the double-integrator branch of orc_collision
 * (dense sampling of the independently solved cubic's polyline, targeted
 * boxes), di_traj/di_pos/di_vel (independent linear solve) and the FOV cone
 * around the interpolated heading (atan2 angles, distinct headings).
 * Parity unpinned: orc_search at
 * lambda = 0.5 on the C1-C5 roadmaps beyond its invariants, and whole-edge
 * heuristic summaries on the generated environments (pinned only through
 * their primitives).
 *
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (no implicit FMA contraction, no fast-math: every + - * / sqrt is one
 * correctly rounded IEEE-754 binary64 / binary32 operation, and the explicit
 * fma() calls the contract writes are single correctly rounded fused
 * operations, N2/N5).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* parameters (the oracle's own struct; mirrors the fields of DESIGN.md §3)  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t pos_dim;       /* d in {2,3}                                      */
  int32_t dynamics;      /* 0 kinematic, 1 double integrator (R7)           */
  int32_t has_heading;   /* row carries (cos yaw, sin yaw) (R21, N1)        */
  int32_t heuristic;     /* 0 omni, 1 fov-velocity, 2 fov-heading, 3 +MLP   */
  double ws_lo[3], ws_hi[3];
  double control_weight; /* r_u in J = int (1 + r_u |u|^2) dt (R7)          */
  double nominal_speed;  /* kinematic edge duration = length / speed (R9)   */
  double dt;             /* heuristic step                          */
  double collision_dt;   /* polyline resolution of curved edges (R8)        */
  double n_f;            /* features needed to offset drift     */
  double fov_cos_half;   /* cos of FOV half angle                   */
  double max_range;      /* feature range                       */
  const double *mlp;     /* 122 weights, W1[8x3] b1[8] W2[8x8] b2[8] W3[2x8] b3[2] */
  double mlp_gain;       /* gamma (R12)                                     */
  double v_ref, w_ref;   /* MLP input scales (R12)                          */
} orc_params;

typedef struct {
  const double *samples; int32_t n; int32_t stride;
  const double *obstacles; int32_t n_obstacles;   /* [O][2d] lo[d] hi[d] */
  const double *features; int32_t n_features;     /* [F][d]              */
  double r;                                       /* r_n         */
  int32_t use_prefilter;  /* conservative DI neighbour prefilter (R7 step 7); only skips work */
} orc_env;

/* ------------------------------------------------------------------------ */
/* geometry                                                                  */
/* ------------------------------------------------------------------------ */

/* Closed segment [A,B] vs closed box [lo,hi]: slab clipping (
 * reading R8).  Exact operation order of DESIGN.md §3 "slab". */
int orc_seg_hits_box(const double *A, const double *B, const double *lo,
                     const double *hi, int d) {
  double t0 = 0.0, t1 = 1.0;
  for (int k = 0; k < d; ++k) {
    double dk = B[k] - A[k];
    if (dk == 0.0) {
      if (A[k] < lo[k] || A[k] > hi[k]) return 0;
    } else {
      double inv = 1.0 / dk;
      double ta = (lo[k] - A[k]) * inv;
      double tb = (hi[k] - A[k]) * inv;
      if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return 0;
    }
  }
  return 1;
}

static int seg_hits_any(const double *A, const double *B, const orc_env *E, int d) {
  for (int o = 0; o < E->n_obstacles; ++o) {
    const double *bx = E->obstacles + (size_t)o * 2 * d;
    if (orc_seg_hits_box(A, B, bx, bx + d, d)) return 1;
  }
  return 0;
}

static int outside_ws(const double *P, const orc_params *prm, int d) {
  for (int k = 0; k < d; ++k)
    if (P[k] < prm->ws_lo[k] || P[k] > prm->ws_hi[k]) return 1;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Cost -- reading R7                                                */
/* ------------------------------------------------------------------------ */

/* Kinematic: Euclidean length, squared differences summed x, y, z in order. */
double orc_cost_kinematic(const double *pu, const double *pv, int d) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double dk = pv[k] - pu[k];
    acc = acc + dk * dk;
  }
  return sqrt(acc);
}

typedef struct { double vv, av, aa, B, C, D, ru; } di_coef;

static void di_coefs(const double *su, const double *sv, int d, double ru, di_coef *k) {
  const double *p0 = su, *v0 = su + d, *p1 = sv, *v1 = sv + d;
  double vv = 0.0, av = 0.0, aa = 0.0;
  for (int j = 0; j < d; ++j) {
    double a = p1[j] - p0[j];
    vv = vv + ((v0[j] * v0[j] + v0[j] * v1[j]) + v1[j] * v1[j]);
    av = av + a * (v0[j] + v1[j]);
    aa = aa + a * a;
  }
  k->vv = vv; k->av = av; k->aa = aa; k->ru = ru;
  k->B = (4.0 * ru) * vv;
  k->C = (24.0 * ru) * av;
  k->D = (36.0 * ru) * aa;
}

/* q(tau) = tau^4 - B tau^2 + C tau - D: numerator of c'(tau) (R7 step 3). */
static double di_q(const di_coef *k, double t) { return ((t * t - k->B) * t + k->C) * t - k->D; }
/* q'(tau) = 4 tau^3 - 2 B tau + C */
static double di_qp(const di_coef *k, double t) { return ((4.0 * (t * t)) - (2.0 * k->B)) * t + k->C; }
/* c(tau) = tau + r_u (4 vv / tau - 12 av / tau^2 + 12 aa / tau^3) */
static double di_c(const di_coef *k, double t) {
  double t2 = t * t;
  double t3 = t2 * t;
  return t + k->ru * ((((4.0 * k->vv) / t) - ((12.0 * k->av) / t2)) + ((12.0 * k->aa) / t3));
}

/* Bisection on [lo,hi] of a sign change of f (which = 0: q, 1: q'), at most
 * 100 halvings or until the midpoint no longer moves; returns hi. */
static double di_bisect(const di_coef *k, int which, double lo, double hi) {
  int hi_pos = (which == 0 ? di_q(k, hi) : di_qp(k, hi)) > 0.0;
  for (int it = 0; it < 100; ++it) {
    double mid = lo + 0.5 * (hi - lo);
    if (!(mid > lo && mid < hi)) break;
    double fm = (which == 0) ? di_q(k, mid) : di_qp(k, mid);
    if ((fm > 0.0) == hi_pos) hi = mid; else lo = mid;
  }
  return hi;
}

/* Double-integrator optimal time+energy connection (R7 steps 1-5).
 * Returns 1 and (c*, tau*) if some local minimiser of c on (0, r] exists,
 * else 0.  Pairs with identical positions (D == 0) have no edge (R7). */
int orc_cost_di(const double *su, const double *sv, int d, double ru, double r,
                double *c_out, double *tau_out) {
  di_coef k;
  di_coefs(su, sv, d, ru, &k);
  if (k.D == 0.0) return 0;
  /* breakpoints: 0, roots of q' (each monotone piece of q'), r */
  double bp[6];
  int nb = 0;
  bp[nb++] = 0.0;
  double tc = (k.B > 0.0) ? sqrt(k.B / 6.0) : 0.0;   /* q'' = 12 t^2 - 2B = 0 */
  double pieces[3];
  int np = 0;
  pieces[np++] = 0.0;
  if (tc > 0.0 && tc < r) pieces[np++] = tc;
  pieces[np++] = r;
  for (int s = 0; s + 1 < np; ++s) {
    double a = pieces[s], b = pieces[s + 1];
    double fa = di_qp(&k, a), fb = di_qp(&k, b);
    if ((fa > 0.0 && fb < 0.0) || (fa < 0.0 && fb > 0.0))
      bp[nb++] = di_bisect(&k, 1, a, b);
  }
  bp[nb++] = r;
  /* sort breakpoints (insertion sort, at most 4 entries) */
  for (int i = 1; i < nb; ++i) {
    double x = bp[i];
    int j = i - 1;
    while (j >= 0 && bp[j] > x) { bp[j + 1] = bp[j]; --j; }
    bp[j + 1] = x;
  }
  int found = 0;
  double best_c = 0.0, best_t = 0.0;
  for (int s = 0; s + 1 < nb; ++s) {
    double a = bp[s], b = bp[s + 1];
    if (!(b > a)) continue;
    if (di_q(&k, a) <= 0.0 && di_q(&k, b) > 0.0) {
      double t = di_bisect(&k, 0, a, b);
      double c = di_c(&k, t);
      if (!found || c < best_c || (c == best_c && t < best_t)) {
        found = 1; best_c = c; best_t = t;
      }
    }
  }
  if (!found) return 0;
  *c_out = best_c;
  *tau_out = best_t;
  return 1;
}

/* Trajectory coefficients p(t) = p0 + v0 t + c2 t^2 + c3 t^3 (R7 step 6). */
static void di_traj(const double *su, const double *sv, int d, double tau, double *c2, double *c3) {
  const double *p0 = su, *v0 = su + d, *p1 = sv, *v1 = sv + d;
  double tau2 = tau * tau;
  double tau3 = tau2 * tau;
  for (int j = 0; j < d; ++j) {
    double dp = (p1[j] - p0[j]) - v0[j] * tau;
    double dl = v1[j] - v0[j];
    c2[j] = (3.0 * dp - dl * tau) / tau2;
    c3[j] = (dl * tau - 2.0 * dp) / tau3;
  }
}

static void di_pos(const double *su, const double *c2, const double *c3, int d, double t, double *x) {
  const double *p0 = su, *v0 = su + d;
  for (int j = 0; j < d; ++j) x[j] = fma(t, fma(t, fma(t, c3[j], c2[j]), v0[j]), p0[j]);
}

static void di_vel(const double *su, const double *c2, const double *c3, int d, double t, double *v) {
  const double *v0 = su + d;
  for (int j = 0; j < d; ++j) v[j] = fma(t, fma(t, 3.0 * c3[j], 2.0 * c2[j]), v0[j]);
}

/* Exported for the pins: position and velocity at time t of the edge's cubic
 * (di_traj + di_pos + di_vel, unchanged). */
void orc_di_state(const double *su, const double *sv, int d, double tau, double t, double *x, double *v) {
  double c2[3], c3[3];
  di_traj(su, sv, d, tau, c2, c3);
  di_pos(su, c2, c3, d, t, x);
  di_vel(su, c2, c3, d, t, v);
}

/* ------------------------------------------------------------------------ */
/* Collision(u, v) (A2.5 P:215) -- reading R8                         */
/* ------------------------------------------------------------------------ */
int orc_collision(const orc_env *E, const orc_params *prm, int u, int v, double tau) {
  int d = prm->pos_dim;
  const double *su = E->samples + (size_t)u * E->stride;
  const double *sv = E->samples + (size_t)v * E->stride;
  if (prm->dynamics == 0) {
    return seg_hits_any(su, sv, E, d);
  }
  double c2[3], c3[3], A[3], B[3];
  di_traj(su, sv, d, tau, c2, c3);
  double kc = ceil(tau / prm->collision_dt);
  int Kc = (kc < 1.0) ? 1 : (int)kc;
  di_pos(su, c2, c3, d, 0.0, A);
  if (outside_ws(A, prm, d)) return 1;
  for (int k = 1; k <= Kc; ++k) {
    double t = ((double)k * tau) / (double)Kc;
    di_pos(su, c2, c3, d, t, B);
    if (outside_ws(B, prm, d)) return 1;
    if (seg_hits_any(A, B, E, d)) return 1;
    for (int j = 0; j < d; ++j) A[j] = B[j];
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Perception heuristic along an edge (A1.2 P:178; §4.1; §5.2      */
/* P:476-477) -- readings R9 (discretisation), R10 (tropical summary),       */
/* R12 (learned-style MLP).                                                   */
/* ------------------------------------------------------------------------ */

/* number of features visible from position x with heading vector hv
 * ("in the field of view and unobstructed"). */
int orc_visible_count(const orc_env *E, const orc_params *prm, const double *x, const double *hv) {
  int d = prm->pos_dim;
  double R2 = prm->max_range * prm->max_range;
  double cos2 = prm->fov_cos_half * prm->fov_cos_half;
  int count = 0;
  for (int f = 0; f < E->n_features; ++f) {
    const double *F = E->features + (size_t)f * d;
    double dl[3];
    double dd = 0.0;
    for (int j = 0; j < d; ++j) { dl[j] = F[j] - x[j]; dd = fma(dl[j], dl[j], dd); }
    if (dd > R2) continue;                                   /* in range */
    if (prm->heuristic != 0) {                               /* in FOV cone */
      double hh = 0.0, dot = 0.0;
      for (int j = 0; j < d; ++j) hh = fma(hv[j], hv[j], hh);
      for (int j = 0; j < d; ++j) dot = fma(hv[j], dl[j], dot);
      if (!(hh > 0.0)) continue;
      if (dot < 0.0) continue;
      if (dot * dot < cos2 * (hh * dd)) continue;
    }
    if (seg_hits_any(x, F, E, d)) continue;                  /* unobstructed */
    ++count;
  }
  return count;
}

/* 3-8-8-2 ReLU net, sums in index order starting from the bias (R12). */
static double mlp_out0(const double *w, double z0, double z1, double z2) {
  const double *W1 = w, *b1 = w + 24, *W2 = w + 32, *b2 = w + 96, *W3 = w + 104, *b3 = w + 120;
  double h1[8], h2[8];
  for (int i = 0; i < 8; ++i) {
    double a = b1[i];
    a = fma(W1[i * 3 + 0], z0, a);
    a = fma(W1[i * 3 + 1], z1, a);
    a = fma(W1[i * 3 + 2], z2, a);
    h1[i] = (a > 0.0) ? a : 0.0;
  }
  for (int i = 0; i < 8; ++i) {
    double a = b2[i];
    for (int j = 0; j < 8; ++j) a = fma(W2[i * 8 + j], h1[j], a);
    h2[i] = (a > 0.0) ? a : 0.0;
  }
  double o = b3[0];
  for (int j = 0; j < 8; ++j) o = fma(W3[0 * 8 + j], h2[j], o);
  return o;
}

/* Exported for the pins (tests/test_oracle_build.py): the same function. */
double orc_mlp_out0(const double *w, double z0, double z1, double z2) { return mlp_out0(w, z0, z1, z2); }

/* Per-step increments inc_k (k = 0..K-1) of edge u->v; returns K, or the
 * required size if it exceeds cap (then inc is not written past cap). */
int orc_edge_increments(const orc_env *E, const orc_params *prm, int u, int v,
                        double c64, double tau, double *inc, int cap) {
  int d = prm->pos_dim;
  const double *su = E->samples + (size_t)u * E->stride;
  const double *sv = E->samples + (size_t)v * E->stride;
  double T = (prm->dynamics == 0) ? (c64 / prm->nominal_speed) : tau;
  double kk = ceil(T / prm->dt);
  int K = (kk < 1.0) ? 1 : (int)kk;
  double Dl = T / (double)K;
  double c2[3] = {0, 0, 0}, c3[3] = {0, 0, 0};
  if (prm->dynamics == 1) di_traj(su, sv, d, T, c2, c3);
  int hoff = (prm->dynamics == 1 ? 2 * d : d);
  double omega = 0.0;
  if (prm->has_heading) {
    double ex = sv[hoff] - su[hoff], ey = sv[hoff + 1] - su[hoff + 1];
    omega = sqrt(ex * ex + ey * ey) / T;
  }
  for (int k = 0; k < K; ++k) {
    double t = (double)k * Dl;
    double x[3], hv[3] = {0, 0, 0}, vel[3] = {0, 0, 0};
    if (prm->dynamics == 0) {
      double s = t / T;
      for (int j = 0; j < d; ++j) x[j] = fma(s, sv[j] - su[j], su[j]);
    } else {
      di_pos(su, c2, c3, d, t, x);
      di_vel(su, c2, c3, d, t, vel);
    }
    if (prm->heuristic == 1) {
      if (prm->dynamics == 1) { for (int j = 0; j < d; ++j) hv[j] = vel[j]; }
      else { for (int j = 0; j < d; ++j) hv[j] = sv[j] - su[j]; }
    } else if (prm->heuristic >= 2) {
      double s = t / T;
      hv[0] = fma(s, sv[hoff], (1.0 - s) * su[hoff]);
      hv[1] = fma(s, sv[hoff + 1], (1.0 - s) * su[hoff + 1]);
      if (d == 3) hv[2] = 0.0;
    }
    int kv = orc_visible_count(E, prm, x, hv);
    double in = Dl - (double)kv * (Dl / prm->n_f);
    if (prm->heuristic == 3) {
      double speed;
      if (prm->dynamics == 1) {
        double ss = 0.0;
        for (int j = 0; j < d; ++j) ss = fma(vel[j], vel[j], ss);
        speed = sqrt(ss);
      } else {
        speed = prm->nominal_speed;
      }
      double z0 = speed / prm->v_ref;
      double z1 = omega / prm->w_ref;
      double z2 = (double)kv / prm->n_f;
      double o = mlp_out0(prm->mlp, z0, z1, z2);
      in = in + Dl * (prm->mlp_gain * o);
    }
    if (k < cap) inc[k] = in;
  }
  return K;
}

/* Tropical summary of an edge (R10): h -> max(c, h + s) composes the per-step
 * clamp maps h -> max(0, h + inc_k) of P:324-328 in time order. */
void orc_fold_summary(const double *inc, int K, double *s_out, double *c_out) {
  double s = 0.0, c = 0.0;
  for (int k = 0; k < K; ++k) {
    double t = c + inc[k];
    c = (t > 0.0) ? t : 0.0;
    s = s + inc[k];
  }
  *s_out = s;
  *c_out = c;
}

/* Peak summary of an edge (NEXT-3; Eq. 2's "for all t"): the largest
 * value the per-step fold reaches along the edge, from h0, is
 * max(C, h0 + S) with S = max over prefixes of s and C = max over prefixes of
 * c (prefix 0 included: S, C >= 0).  Same fold as orc_fold_summary. */
void orc_fold_peak(const double *inc, int K, double *S_out, double *C_out) {
  double s = 0.0, c = 0.0, S = 0.0, C = 0.0;
  for (int k = 0; k < K; ++k) {
    double t = c + inc[k];
    c = (t > 0.0) ? t : 0.0;
    s = s + inc[k];
    S = (s > S) ? s : S;
    C = (c > C) ? c : C;
  }
  *S_out = S;
  *C_out = C;
}

/* Largest value of the stepwise fold from h0 over the steps (plain definition
 * for the pins of orc_fold_peak). */
double orc_fold_stepwise_peak(double h0, const double *inc, int K) {
  double h = h0, mx = h0;
  for (int k = 0; k < K; ++k) {
    double t = h + inc[k];
    h = (t > 0.0) ? t : 0.0;
    if (h > mx) mx = h;
  }
  return mx;
}

/* Stepwise clamp fold of P:324-328 from h0 (the plain definition; used by the
 * pins to check the summary). */
double orc_fold_stepwise(double h0, const double *inc, int K) {
  double h = h0;
  for (int k = 0; k < K; ++k) {
    double t = h + inc[k];
    h = (t > 0.0) ? t : 0.0;
  }
  return h;
}

/* One directed pair u -> v: cost decision, collision, heuristic summary.
 * Returns 1 iff v in Near(u) (Cost(u,v) < r); fills outputs then. */
int orc_edge(const orc_env *E, const orc_params *prm, int u, int v,
             double *c64, double *tau, int *coll, double *s64, double *h64) {
  int d = prm->pos_dim;
  const double *su = E->samples + (size_t)u * E->stride;
  const double *sv = E->samples + (size_t)v * E->stride;
  double c, t;
  if (prm->dynamics == 0) {
    c = orc_cost_kinematic(su, sv, d);
    t = c / prm->nominal_speed;
    if (!(c < E->r)) return 0;
  } else {
    if (E->use_prefilter) {
      /* R7 step 7: |p1-p0| < |v0| r + r^2/sqrt(3 r_u) and |v1-v0| < r/sqrt(r_u),
       * tested with 1e-9 relative slack; a necessary condition only. */
      double ru = prm->control_weight, r = E->r;
      double dp2 = 0.0, dv2 = 0.0, v02 = 0.0;
      for (int j = 0; j < d; ++j) {
        double a = sv[j] - su[j], b = sv[d + j] - su[d + j];
        dp2 += a * a; dv2 += b * b; v02 += su[d + j] * su[d + j];
      }
      double bp = sqrt(v02) * r + r * r / sqrt(3.0 * ru);
      double bv = r / sqrt(ru);
      bp *= (1.0 + 1e-9); bv *= (1.0 + 1e-9);
      if (dp2 > bp * bp || dv2 > bv * bv) return 0;
    }
    if (!orc_cost_di(su, sv, d, prm->control_weight, E->r, &c, &t)) return 0;
    if (!(c < E->r)) return 0;
  }
  *c64 = c;
  *tau = t;
  *coll = orc_collision(E, prm, u, v, t);
  *s64 = 0.0;
  *h64 = 0.0;
  if (!*coll) {
    int cap = 4096;
    double stackbuf[4096];
    double *inc = stackbuf;
    int K = orc_edge_increments(E, prm, u, v, c, t, inc, cap);
    if (K > cap) {
      inc = (double *)malloc(sizeof(double) * (size_t)K);
      orc_edge_increments(E, prm, u, v, c, t, inc, K);
    }
    orc_fold_summary(inc, K, s64, h64);
    if (inc != stackbuf) free(inc);
  }
  return 1;
}

/* Peak summary (S, C) of edge u -> v (0, 0 if colliding or not an edge). */
int orc_edge_peak(const orc_env *E, const orc_params *prm, int u, int v, double *S64, double *C64) {
  double c64, tau, s64, h64;
  int cl;
  *S64 = 0.0;
  *C64 = 0.0;
  if (!orc_edge(E, prm, u, v, &c64, &tau, &cl, &s64, &h64)) return 0;
  if (cl) return 1;
  int K = orc_edge_increments(E, prm, u, v, c64, tau, NULL, 0);
  double *inc = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
  orc_edge_increments(E, prm, u, v, c64, tau, inc, K);
  orc_fold_peak(inc, K, S64, C64);
  free(inc);
  return 1;
}

/* Peaks of every edge of a built CSR (rows of orc_build). */
void orc_build_peaks(const orc_env *E, const orc_params *prm, const int32_t *row_ptr, const int32_t *dst,
                     float *S, float *C) {
  for (int u = 0; u < E->n; ++u) {
    for (int32_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      double S64, C64;
      orc_edge_peak(E, prm, u, dst[e], &S64, &C64);
      S[e] = (float)S64;
      C[e] = (float)C64;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Alg. 2 BuildGraph + Alg. 1 line 2.                    */
/* Row u lists v != u with Cost(u,v) < r in ascending v (R6); each entry      */
/* carries w = (float)c64, coll, s = (float)s64, c = (float)c64h (N4).        */
/* Two passes: pass 0 counts (row_ptr), pass 1 fills.  Returns nnz, or -1.   */
/* ------------------------------------------------------------------------ */
int64_t orc_build(const orc_env *E, const orc_params *prm, int32_t *row_ptr,
                  int32_t *dst, uint8_t *coll, float *w, float *s, float *c,
                  double *tau_out, int64_t cap) {
  int64_t nnz = 0;
  row_ptr[0] = 0;
  for (int u = 0; u < E->n; ++u) {
    for (int v = 0; v < E->n; ++v) {
      if (v == u) continue;                              /* V \ {v}, A2.3 */
      double c64, tau, s64, h64;
      int cl;
      if (!orc_edge(E, prm, u, v, &c64, &tau, &cl, &s64, &h64)) continue;
      if (nnz < cap) {
        dst[nnz] = v;
        coll[nnz] = (uint8_t)cl;
        w[nnz] = (float)c64;
        s[nnz] = (float)s64;
        c[nnz] = (float)h64;
        if (tau_out) tau_out[nnz] = tau;
      }
      ++nnz;
    }
    row_ptr[u + 1] = (int32_t)nnz;
  }
  return nnz;
}

/* Same as orc_build for a subset of rows (sampled parity at full size). */
int64_t orc_build_row(const orc_env *E, const orc_params *prm, int u,
                      int32_t *dst, uint8_t *coll, float *w, float *s, float *c,
                      int64_t cap) {
  int64_t k = 0;
  for (int v = 0; v < E->n; ++v) {
    if (v == u) continue;
    double c64, tau, s64, h64;
    int cl;
    if (!orc_edge(E, prm, u, v, &c64, &tau, &cl, &s64, &h64)) continue;
    if (k < cap) {
      dst[k] = v; coll[k] = (uint8_t)cl; w[k] = (float)c64; s[k] = (float)s64; c[k] = (float)h64;
    }
    ++k;
  }
  return k;
}

/* ------------------------------------------------------------------------ */
/* Alg. 3 Explore, literal.                                      */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t status;     /* 0 OK, 3 NO_FEASIBLE_PLAN, 5 OOM                  */
  int32_t path_len;
  int32_t waves;      /* non-empty groups expanded (R24)                  */
  int32_t pad;
  float cost, h, h_peak, pad2;
  int64_t relaxations, labels_inserted;
} orc_result;

typedef struct {      /* per non-empty wave counters (§8(c) counters)    */
  int64_t i;          /* group index                                      */
  int64_t group;      /* |G_i|                                            */
  int64_t relax;      /* (p in G, free edge) pairs (R23)                  */
  int64_t beta_pass;  /* candidates with h <= beta (A3.9)                 */
  int64_t inserted;   /* candidates still in P after RemoveDominated      */
  int64_t killed;     /* pre-existing open plans removed (A3.15)          */
  int64_t touched;    /* nodes receiving >= 1 beta-passing candidate      */
  int64_t stair_sum;  /* sum over touched x of |ND(P(x))| before the wave */
  int64_t e_rows;     /* sum over DISTINCT heads x of G_i of deg_free(x):
                         the CSR entries the wave must read once (§8(d) E_rows) */
} orc_wave;

typedef struct { int32_t *a; int64_t n, cap; } ivec;
static int iv_push(ivec *v, int32_t x) {
  if (v->n == v->cap) {
    int64_t nc = v->cap ? 2 * v->cap : 8;
    int32_t *na = (int32_t *)realloc(v->a, sizeof(int32_t) * (size_t)nc);
    if (!na) return 0;
    v->a = na; v->cap = nc;
  }
  v->a[v->n++] = x;
  return 1;
}

typedef struct {
  int32_t *node, *parent;
  float *cost, *h;
  uint8_t *open, *inP;
  int64_t n, cap;
} labels_t;

static int lab_push(labels_t *L, int32_t node, int32_t parent, float cost, float h) {
  if (L->n == L->cap) {
    int64_t nc = L->cap ? 2 * L->cap : 1024;
    L->node = (int32_t *)realloc(L->node, sizeof(int32_t) * nc);
    L->parent = (int32_t *)realloc(L->parent, sizeof(int32_t) * nc);
    L->cost = (float *)realloc(L->cost, sizeof(float) * nc);
    L->h = (float *)realloc(L->h, sizeof(float) * nc);
    L->open = (uint8_t *)realloc(L->open, nc);
    L->inP = (uint8_t *)realloc(L->inP, nc);
    if (!L->node || !L->parent || !L->cost || !L->h || !L->open || !L->inP) return -1;
    L->cap = nc;
  }
  int64_t id = L->n++;
  L->node[id] = node; L->parent[id] = parent; L->cost[id] = cost; L->h[id] = h;
  L->open[id] = 1; L->inP[id] = 1;
  return (int)id;
}

/* p_dom dominates p  <=>  p.cost > p_dom.cost  and  p.h >= p_dom.h */
static int dominates(const labels_t *L, int32_t pd, int32_t p) {
  return (L->cost[p] > L->cost[pd]) && (L->h[p] >= L->h[pd]);
}

/* |ND(P(x))|: members of P(x) not dominated by any member of P(x). */
static int64_t nd_size(const labels_t *L, const ivec *Px) {
  int64_t k = 0;
  for (int64_t a = 0; a < Px->n; ++a) {
    int dom = 0;
    for (int64_t b = 0; b < Px->n && !dom; ++b)
      if (dominates(L, Px->a[b], Px->a[a])) dom = 1;
    if (!dom) ++k;
  }
  return k;
}

static int path_of(const labels_t *L, int32_t id, int32_t *buf, int cap) {
  int len = 0;
  for (int32_t x = id; x >= 0; x = L->parent[x]) ++len;
  if (len > cap) return len;
  int k = len - 1;
  for (int32_t x = id; x >= 0; x = L->parent[x]) buf[k--] = L->node[x];
  return len;
}

/* lexicographic order of node sequences; a proper prefix is smaller (R16) */
static int path_less(const int32_t *a, int la, const int32_t *b, int lb) {
  int m = la < lb ? la : lb;
  for (int k = 0; k < m; ++k) {
    if (a[k] != b[k]) return a[k] < b[k];
  }
  return la < lb;
}

/* forall_t != 0 (NEXT-3): the cutoff A3.9 is applied to every step along
 * the edge, peak = max(C_e, p.h + S_e) <= beta (f32, same max as PH), instead
 * of the node value only (reading R11).  Everything else is Alg. 3. */
int orc_search_ex(int32_t n, const int32_t *row_ptr, const int32_t *dst, const uint8_t *coll,
                  const float *w, const float *s, const float *c, const uint8_t *goal,
                  int32_t start, double beta, double lambda, double r,
                  int32_t *path, int32_t path_cap, orc_result *res,
                  orc_wave *waves, int32_t waves_cap, const float *S, const float *C, int32_t forall_t);

int orc_search(int32_t n, const int32_t *row_ptr, const int32_t *dst, const uint8_t *coll,
               const float *w, const float *s, const float *c, const uint8_t *goal,
               int32_t start, double beta, double lambda, double r,
               int32_t *path, int32_t path_cap, orc_result *res,
               orc_wave *waves, int32_t waves_cap) {
  return orc_search_ex(n, row_ptr, dst, coll, w, s, c, goal, start, beta, lambda, r, path, path_cap, res, waves,
                       waves_cap, NULL, NULL, 0);
}

int orc_search_ex(int32_t n, const int32_t *row_ptr, const int32_t *dst, const uint8_t *coll,
                  const float *w, const float *s, const float *c, const uint8_t *goal,
                  int32_t start, double beta, double lambda, double r,
                  int32_t *path, int32_t path_cap, orc_result *res,
                  orc_wave *waves, int32_t waves_cap, const float *S, const float *C, int32_t forall_t) {
  memset(res, 0, sizeof(*res));
  const double T = lambda * r;                    /* threshold step lambda r_n */
  labels_t L;
  memset(&L, 0, sizeof(L));
  ivec *P = (ivec *)calloc((size_t)n, sizeof(ivec));
  ivec open = {0}, G = {0}, nopen = {0};
  uint8_t *touched = (uint8_t *)calloc((size_t)n, 1);
  uint8_t *rowseen = (uint8_t *)calloc((size_t)n, 1);
  ivec touched_list = {0}, heads = {0};
  if (!P || !touched || !rowseen) { res->status = 5; return 5; }

  /* A3.1-A3.4 */
  int32_t root = lab_push(&L, start, -1, 0.0f, 0.0f);
  iv_push(&P[start], root);
  iv_push(&open, root);
  iv_push(&G, root);
  int64_t i = 0;
  int32_t nwaves = 0;
  int64_t relax_total = 0, inserted_total = 0;

  for (;;) {
    /* A3.5: while P_open != {} and no g in G with head in X_goal and h <= beta */
    if (open.n == 0) break;
    int stop = 0;
    for (int64_t k = 0; k < G.n; ++k) {
      int32_t g = G.a[k];
      if (goal[L.node[g]] && (double)L.h[g] <= beta) { stop = 1; break; }
    }
    if (stop) break;

    orc_wave wv;
    memset(&wv, 0, sizeof(wv));
    wv.i = i;
    wv.group = G.n;
    int nonempty = G.n > 0;
    const int64_t first_new = L.n;   /* labels created this wave: [first_new, L.n) */

    /* §8(d) E_rows: collision-free entries of the distinct heads of G_i */
    for (int64_t k = 0; k < G.n; ++k) {
      int32_t u = L.node[G.a[k]];
      if (rowseen[u]) continue;
      rowseen[u] = 1;
      iv_push(&heads, u);
      for (int32_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) wv.e_rows += !coll[e];
    }
    for (int64_t k = 0; k < heads.n; ++k) rowseen[heads.a[k]] = 0;
    heads.n = 0;

    /* A3.6-A3.14: for all p in G, for all x in N(p.head) */
    for (int64_t k = 0; k < G.n; ++k) {
      int32_t p = G.a[k];
      int32_t u = L.node[p];
      float pc = L.cost[p], ph = L.h[p];
      for (int32_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
        if (coll[e]) continue;                       /* N(v) excludes colliding (A2.5) */
        ++wv.relax;
        int32_t x = dst[e];
        float qc = pc + w[e];                        /* p.cost + Cost(p.head, x)   */
        float t = ph + s[e];                         /* PH(x, p) = max(c_e, h + s_e) (R10) */
        float qh = (t > c[e]) ? t : c[e];
        int ok = (double)qh <= beta;                 /* A3.9 cutoff                */
        if (forall_t && ok) {                        /* NEXT-3: every step of the edge */
          float t2 = ph + S[e];
          float pk = (t2 > C[e]) ? t2 : C[e];
          ok = (double)pk <= beta;
        }
        if (ok) {
          ++wv.beta_pass;
          if (!touched[x]) {
            touched[x] = 1;
            iv_push(&touched_list, x);
            wv.stair_sum += nd_size(&L, &P[x]);
          }
          int32_t q = lab_push(&L, x, p, qc, qh);
          if (q < 0) { res->status = 5; return 5; }
          iv_push(&P[x], q);                          /* A3.10 */
          iv_push(&open, q);                          /* A3.11 */
        }
      }
    }
    wv.touched = touched_list.n;

    /* A3.15 RemoveDominated(P, P_open): every open p dominated by some
     * same-head plan of P is removed from P_open and P (simultaneously). */
    int64_t nmark = 0;
    uint8_t *mark = (uint8_t *)calloc((size_t)(open.n ? open.n : 1), 1);
    for (int64_t k = 0; k < open.n; ++k) {
      int32_t a = open.a[k];
      ivec *Px = &P[L.node[a]];
      for (int64_t b = 0; b < Px->n; ++b)
        if (dominates(&L, Px->a[b], a)) { mark[k] = 1; ++nmark; break; }
    }
    nopen.n = 0;
    for (int64_t k = 0; k < open.n; ++k) {
      int32_t a = open.a[k];
      if (mark[k]) {
        L.open[a] = 0;
        L.inP[a] = 0;
        if (a < first_new) ++wv.killed;   /* else: a candidate of this wave */
      } else {
        iv_push(&nopen, a);
      }
    }
    free(mark);
    /* compact P lists of nodes that lost members */
    if (nmark) {
      for (int32_t x = 0; x < n; ++x) {
        ivec *Px = &P[x];
        int64_t m = 0;
        for (int64_t b = 0; b < Px->n; ++b)
          if (L.inP[Px->a[b]]) Px->a[m++] = Px->a[b];
        Px->n = m;
      }
    }
    { ivec tmp = open; open = nopen; nopen = tmp; }
    for (int64_t k = first_new; k < L.n; ++k)
      if (L.inP[k]) ++wv.inserted;

    /* A3.16 P_open <- P_open \ G */
    for (int64_t k = 0; k < G.n; ++k) L.open[G.a[k]] = 0;
    nopen.n = 0;
    for (int64_t k = 0; k < open.n; ++k)
      if (L.open[open.a[k]]) iv_push(&nopen, open.a[k]);
    { ivec tmp = open; open = nopen; nopen = tmp; }

    if (nonempty) {
      relax_total += wv.relax;
      inserted_total += wv.inserted;
      if (waves && nwaves < waves_cap) waves[nwaves] = wv;
      ++nwaves;
    }
    for (int64_t k = 0; k < touched_list.n; ++k) touched[touched_list.a[k]] = 0;
    touched_list.n = 0;

    /* A3.17-A3.18 */
    ++i;
    G.n = 0;
    for (int64_t k = 0; k < open.n; ++k) {
      int32_t p = open.a[k];
      if ((double)L.cost[p] <= (double)i * T) iv_push(&G, p);
    }
  }

  /* A3.20-A3.21: P_candidates = plans of P at goal nodes; argmin cost,
   * ties by h, then lexicographic node sequence (R16). */
  int32_t best = -1;
  int32_t *pa = (int32_t *)malloc(sizeof(int32_t) * 65536);
  int32_t *pb = (int32_t *)malloc(sizeof(int32_t) * 65536);
  for (int32_t x = 0; x < n; ++x) {
    if (!goal[x]) continue;
    for (int64_t b = 0; b < P[x].n; ++b) {
      int32_t q = P[x].a[b];
      if (best < 0) { best = q; continue; }
      if (L.cost[q] < L.cost[best]) { best = q; continue; }
      if (L.cost[q] > L.cost[best]) continue;
      if (L.h[q] < L.h[best]) { best = q; continue; }
      if (L.h[q] > L.h[best]) continue;
      int la = path_of(&L, q, pa, 65536), lb = path_of(&L, best, pb, 65536);
      if (path_less(pa, la, pb, lb)) best = q;
    }
  }
  res->waves = nwaves;
  res->relaxations = relax_total;
  res->labels_inserted = inserted_total;
  if (best < 0) {
    res->status = 3;
  } else {
    int len = path_of(&L, best, pa, 65536);
    res->path_len = len;
    res->cost = L.cost[best];
    res->h = L.h[best];
    float hp = 0.0f;
    for (int32_t x = best; x >= 0; x = L.parent[x]) if (L.h[x] > hp) hp = L.h[x];
    res->h_peak = hp;
    if (len <= path_cap) memcpy(path, pa, sizeof(int32_t) * (size_t)len);
    res->status = (len <= path_cap) ? 0 : 4;
  }
  free(pa); free(pb);
  for (int32_t x = 0; x < n; ++x) free(P[x].a);
  free(P); free(open.a); free(G.a); free(nopen.a); free(touched); free(touched_list.a);
  free(rowseen); free(heads.a);
  free(L.node); free(L.parent); free(L.cost); free(L.h); free(L.open); free(L.inP);
  return res->status;
}

/* Goal membership of every node: position in the closed box (R20). */
void orc_goal_mask(const double *samples, int32_t n, int32_t stride, int32_t d,
                   const double *lo, const double *hi, uint8_t *out) {
  for (int32_t x = 0; x < n; ++x) {
    const double *p = samples + (size_t)x * stride;
    int in = 1;
    for (int k = 0; k < d; ++k) if (p[k] < lo[k] || p[k] > hi[k]) in = 0;
    out[x] = (uint8_t)in;
  }
}

/* ------------------------------------------------------------------------ */
/* Monte Carlo verification (Alg. 1 step 4; §3; simulation */
/* model §4.1) -- NEXT-4, readings R31-R36 of DESIGN.md §4.       */
/* One trial = closed-loop simulation of the 6D double integrator tracking  */
/* the plan's nominal trajectory with an LQR-type feedback on the ESTIMATED */
/* state, an inertial estimate from a noisy accelerometer,  */
/* a translation-only 3D-to-3D position fix from the features in view from  */
/* the TRUE state, fused by a Kalman filter.  Output:   */
/* max_t |x_hat - x| and max_t |x_nom - x|; p_hat = P(max err >= delta)     */
/* (Eq. 1; "asymptotically exact probability").                 */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t trials;
  int32_t pad;
  uint64_t seed;
  double sigma_imu;   /* accelerometer white noise per axis (m/s^2) */
  double sigma_vis;   /* feature relative-position noise per axis (m) */
  double u_max;       /* per-axis control limit                              */
  double k_p, k_d;    /* tracking gains per axis (LQR)                */
  double p0_pos, p0_vel;  /* initial filter covariance diag                  */
  double delta;       /* localisation error bound delta_x_hat (Eq. 1)        */
} orc_mc;

typedef struct {     /* extra per-trial outputs used by the oracle's pins    */
  double err_final[3];     /* x_hat - x at the last step                     */
  double p11, p12, p22;    /* filter covariance at the last step             */
  int64_t steps;           /* simulation steps                               */
  int64_t draws;           /* normals consumed                               */
  int64_t fixes;           /* steps with >= 1 feature in view                */
} orc_mc_trace;

/* counter-based generator (R33): SplitMix64's finaliser over a Weyl sequence. */
static uint64_t mc_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* normal number `idx` of trial `trial`: Irwin-Hall sum of 12 uniform 32-bit
 * words (the two halves of 6 consecutive 64-bit draws) minus 6 (R33). */
double orc_mc_normal(uint64_t seed, uint64_t trial, uint64_t idx) {
  const uint64_t G = 0x9E3779B97F4A7C15ULL;
  uint64_t key = mc_mix(seed + G * (trial + 1ULL));
  uint64_t S = 0;
  for (int i = 0; i < 6; ++i) {
    uint64_t w = mc_mix(key + G * (idx * 6ULL + (uint64_t)i + 1ULL));
    S += (w & 0xffffffffULL) + (w >> 32);
  }
  return (double)S * (1.0 / 4294967296.0) - 6.0;
}

/* features in view from x with heading hv (same predicate as the heuristic,
 * P:319 "in the field of view and unobstructed"); writes their indices. */
static int visible_list(const orc_env *E, const orc_params *prm, const double *x, const double *hv, int32_t *out) {
  int d = prm->pos_dim;
  double R2 = prm->max_range * prm->max_range;
  double cos2 = prm->fov_cos_half * prm->fov_cos_half;
  int count = 0;
  for (int f = 0; f < E->n_features; ++f) {
    const double *F = E->features + (size_t)f * d;
    double dl[3];
    double dd = 0.0;
    for (int j = 0; j < d; ++j) { dl[j] = F[j] - x[j]; dd = fma(dl[j], dl[j], dd); }
    if (dd > R2) continue;
    if (prm->heuristic != 0) {
      double hh = 0.0, dot = 0.0;
      for (int j = 0; j < d; ++j) hh = fma(hv[j], hv[j], hh);
      for (int j = 0; j < d; ++j) dot = fma(hv[j], dl[j], dot);
      if (!(hh > 0.0)) continue;
      if (dot < 0.0) continue;
      if (dot * dot < cos2 * (hh * dd)) continue;
    }
    if (seg_hits_any(x, F, E, d)) continue;
    out[count++] = f;
  }
  return count;
}

/* One trial along plan path[0..L-1] (double-integrator roadmap only).
 * Returns 0, or -1 if a plan edge has no connection (not an r-disc edge). */
int orc_mc_trial(const orc_env *E, const orc_params *prm, const int32_t *path, int32_t L,
                 const orc_mc *mc, uint64_t trial, double *max_err, double *max_dev, orc_mc_trace *tr) {
  if (prm->dynamics != 1 || L < 1) return -1;
  int d = prm->pos_dim;
  int hoff = 2 * d;
  const double *s0 = E->samples + (size_t)path[0] * E->stride;
  double x[3] = {0, 0, 0}, v[3] = {0, 0, 0}, xh[3] = {0, 0, 0}, vh[3] = {0, 0, 0};
  for (int j = 0; j < d; ++j) { x[j] = s0[j]; v[j] = s0[d + j]; xh[j] = s0[j]; vh[j] = s0[d + j]; }
  double p11 = mc->p0_pos, p12 = 0.0, p22 = mc->p0_vel;
  const double q = mc->sigma_imu * mc->sigma_imu;
  const double rv = mc->sigma_vis * mc->sigma_vis;
  double me = 0.0, md = 0.0;
  uint64_t ctr = 0;
  int64_t steps = 0, fixes = 0;
  int32_t *vis = (int32_t *)malloc(sizeof(int32_t) * (size_t)(E->n_features > 0 ? E->n_features : 1));
  for (int32_t e = 0; e + 1 < L; ++e) {
    const double *su = E->samples + (size_t)path[e] * E->stride;
    const double *sv = E->samples + (size_t)path[e + 1] * E->stride;
    double c64, T;
    if (!orc_cost_di(su, sv, d, prm->control_weight, E->r, &c64, &T)) { free(vis); return -1; }
    double c2[3] = {0, 0, 0}, c3[3] = {0, 0, 0};
    di_traj(su, sv, d, T, c2, c3);
    double kk = ceil(T / prm->dt);
    int K = (kk < 1.0) ? 1 : (int)kk;
    double Dl = T / (double)K;
    double D2 = Dl * Dl;
    for (int k = 0; k < K; ++k) {
      double t = (double)k * Dl;
      double xn[3], vn[3], an[3] = {0, 0, 0};
      di_pos(su, c2, c3, d, t, xn);
      di_vel(su, c2, c3, d, t, vn);
      for (int j = 0; j < d; ++j) an[j] = fma(t, 6.0 * c3[j], 2.0 * c2[j]);   /* nominal acceleration */
      /* (1) control on the estimate, saturated (R32) */
      double u[3] = {0, 0, 0};
      for (int j = 0; j < d; ++j) {
        double uj = (an[j] + mc->k_p * (xn[j] - xh[j])) + mc->k_d * (vn[j] - vh[j]);
        if (uj > mc->u_max) uj = mc->u_max;
        if (uj < -mc->u_max) uj = -mc->u_max;
        u[j] = uj;
      }
      /* (2) true dynamics x'' = u, semi-implicit Euler */
      for (int j = 0; j < d; ++j) { v[j] = v[j] + u[j] * Dl; x[j] = x[j] + v[j] * Dl; }
      /* (3) accelerometer = true acceleration + noise; filter prediction */
      for (int j = 0; j < d; ++j) {
        double am = u[j] + mc->sigma_imu * orc_mc_normal(mc->seed, trial, ctr++);
        vh[j] = vh[j] + am * Dl;
        xh[j] = xh[j] + vh[j] * Dl;
      }
      {
        double a = Dl * p12;
        double n11 = (((p11 + a) + a) + D2 * p22) + q * (D2 * D2);
        double n12 = (p12 + Dl * p22) + q * (D2 * Dl);
        double n22 = p22 + q * D2;
        p11 = n11; p12 = n12; p22 = n22;
      }
      /* (4) features in view from the TRUE state at t + Dl (yaw tracked exactly) */
      double t1 = (double)(k + 1) * Dl;
      double hv[3] = {0, 0, 0};
      if (prm->heuristic == 1) {
        for (int j = 0; j < d; ++j) hv[j] = v[j];
      } else if (prm->heuristic >= 2) {
        double s = t1 / T;
        hv[0] = fma(s, sv[hoff], (1.0 - s) * su[hoff]);
        hv[1] = fma(s, sv[hoff + 1], (1.0 - s) * su[hoff + 1]);
      }
      int kv = visible_list(E, prm, x, hv, vis);
      /* (5) translation-only 3D-to-3D fix: mean over features of f - z_f, with
       * z_f = (f - x) + noise; Kalman update with R = sigma^2 / k */
      if (kv > 0) {
        double sum[3] = {0, 0, 0};
        for (int i = 0; i < kv; ++i) {
          const double *F = E->features + (size_t)vis[i] * d;
          for (int j = 0; j < d; ++j) {
            double z = (F[j] - x[j]) + mc->sigma_vis * orc_mc_normal(mc->seed, trial, ctr++);
            sum[j] = sum[j] + (F[j] - z);
          }
        }
        double Rm = rv / (double)kv;
        double S = p11 + Rm;
        double K1 = 0.0, K2 = 0.0;          /* S == 0: no uncertainty left, no gain (R34) */
        if (S > 0.0) { K1 = p11 / S; K2 = p12 / S; }
        for (int j = 0; j < d; ++j) {
          double fix = sum[j] / (double)kv;
          double y = fix - xh[j];
          xh[j] = xh[j] + K1 * y;
          vh[j] = vh[j] + K2 * y;
        }
        double n11 = p11 - K1 * p11;
        double n12 = p12 - K1 * p12;
        double n22 = p22 - K2 * p12;
        p11 = n11; p12 = n12; p22 = n22;
        ++fixes;
      }
      /* (6) localisation error and deviation from the nominal at t + Dl */
      double xn1[3];
      di_pos(su, c2, c3, d, t1, xn1);
      double ee = 0.0, dd = 0.0;
      for (int j = 0; j < d; ++j) {
        double a = xh[j] - x[j];
        double b = xn1[j] - x[j];
        ee = ee + a * a;
        dd = dd + b * b;
      }
      double err = sqrt(ee), dev = sqrt(dd);
      if (err > me) me = err;
      if (dev > md) md = dev;
      ++steps;
    }
  }
  free(vis);
  *max_err = me;
  *max_dev = md;
  if (tr) {
    for (int j = 0; j < 3; ++j) tr->err_final[j] = xh[j] - x[j];
    tr->p11 = p11; tr->p12 = p12; tr->p22 = p22;
    tr->steps = steps; tr->draws = (int64_t)ctr; tr->fixes = fixes;
  }
  return 0;
}

/* All trials; returns the number with max_err >= delta (p_hat = count/trials,
 * P:290), or -1 on an invalid plan edge. */
int64_t orc_mc_verify(const orc_env *E, const orc_params *prm, const int32_t *path, int32_t L,
                      const orc_mc *mc, uint64_t trial0, int32_t ntrials, double *max_err, double *max_dev) {
  int64_t exceed = 0;
  for (int32_t i = 0; i < ntrials; ++i) {
    if (orc_mc_trial(E, prm, path, L, mc, trial0 + (uint64_t)i, &max_err[i], &max_dev[i], NULL) != 0) return -1;
    if (max_err[i] >= mc->delta) ++exceed;
  }
  return exceed;
}
