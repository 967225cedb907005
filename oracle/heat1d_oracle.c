/*
 * heat1d_oracle.c -- the CPU ORACLE for the 1D periodic heat-equation stencil.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or execute this
 * file.  The product path (paper_2307_01117_b200/, libheat1d.so) never links,
 * imports or calls it, and it shares no code with the CUDA path.
 *
 * What it computes (arxiv 2307.01117, §2 "Model problem"):
 *   - grid x_i = i*h, i = 0..N-1
 *   - forward-Euler, 2nd-order central difference, Eq. 2
 *       u(t+dt, x_i) = u(t,x_i) + dt*alpha*(u_{i-1} - 2u_i + u_{i+1}) / D
 *     with D = h^2 (reading c1 in DESIGN.md: Eq. 2 prints "2h", which is
 *     dimensionally inconsistent with Eq. 1; the literal 2h is an option)
 *   - periodic boundary u(t,x) = u(t, L+x)
 *   - the segmented parallel algorithm with ghost zones
 *
 * Fixed arithmetic (readings c3/c4 in DESIGN.md): r = (k*dt)/(dx*dx) once,
 * then every cell update is the binary64 expression
 *       v = b + r*((a - 2.0*b) + c)      a=u[i-1], b=u[i], c=u[i+1]
 * evaluated left to right, round-to-nearest-even, no contraction, no
 * reassociation.  Build with -O2 -ffp-contract=off (never -ffast-math).
 * Double-buffered (Jacobi), reading c5.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): exact rational brute force on
 * rings of 3..8 cells and on the 1000-cell C1 ring, hand-evaluated values
 * (tests/golden/), the single-Fourier-mode closed form, conservation of
 * sum(u), the discrete max principle, convergence to the mean, and the
 * decomposition invariants (O2 == O1, O3 == O1, rotation, split runs).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* r = k*dt/dx^2 (BASELINE.json north_star formula; reading c4).
 * paper_2h != 0 selects the literal Eq. 2 denominator 2h. */
double oracle_r(double k, double dt, double dx, int paper_2h)
{
    if (paper_2h)
        return (k * dt) / (2.0 * dx);
    return (k * dt) / (dx * dx);
}

/* One application of Eq. 2 to the three time-t values (left, mid, right). */
static double eq2(double a, double b, double c, double r)
{
    return b + r * ((a - 2.0 * b) + c);
}

/* O1 -- the plain definition: nt Jacobi sweeps over the periodic ring
 * u[0..N), in place (u holds u(nt) on return).  PAPER.md:66-71.
 * Returns 0, or -1 if the scratch buffer cannot be allocated / bad args. */
int oracle_run(double *u, int64_t N, double r, int64_t nt)
{
    if (N < 1 || nt < 0)
        return -1;
    double *v = (double *)malloc((size_t)N * sizeof(double));
    if (!v)
        return -1;
    double *cur = u, *nxt = v;
    for (int64_t t = 0; t < nt; t++) {
        for (int64_t i = 0; i < N; i++) {
            int64_t il = (i == 0) ? N - 1 : i - 1;     /* periodic */
            int64_t ir = (i == N - 1) ? 0 : i + 1;
            nxt[i] = eq2(cur[il], cur[i], cur[ir], r);
        }
        double *tmp = cur; cur = nxt; nxt = tmp;
    }
    if (cur != u)
        memcpy(u, cur, (size_t)N * sizeof(double));
    free(v);
    return 0;
}

/* O2 -- the paper's segmented algorithm run sequentially:
 * np segments of nx cells, each stored with one ghost cell per side; every
 * step each segment first receives its ghosts from its periodic neighbours
 * (the queue exchange), then applies Eq. 2 to its own cells.
 * u has nx*np cells, segment p owns u[p*nx .. (p+1)*nx). */
int oracle_segmented(double *u, int64_t nx, int64_t np, double r, int64_t nt)
{
    if (nx < 1 || np < 1 || nt < 0)
        return -1;
    int64_t w = nx + 2;                          /* ghost | nx cells | ghost */
    double *seg = (double *)malloc((size_t)(w * np) * sizeof(double));
    double *nxt = (double *)malloc((size_t)(w * np) * sizeof(double));
    if (!seg || !nxt) {
        free(seg); free(nxt);
        return -1;
    }
    for (int64_t p = 0; p < np; p++)
        memcpy(seg + p * w + 1, u + p * nx, (size_t)nx * sizeof(double));
    for (int64_t t = 0; t < nt; t++) {
        /* exchange: left ghost <- last cell of left neighbour,
         *           right ghost <- first cell of right neighbour */
        for (int64_t p = 0; p < np; p++) {
            int64_t pl = (p == 0) ? np - 1 : p - 1;
            int64_t pr = (p == np - 1) ? 0 : p + 1;
            seg[p * w + 0] = seg[pl * w + nx];
            seg[p * w + nx + 1] = seg[pr * w + 1];
        }
        /* local sweeps */
        for (int64_t p = 0; p < np; p++) {
            const double *s = seg + p * w;
            double *d = nxt + p * w;
            for (int64_t j = 1; j <= nx; j++)
                d[j] = eq2(s[j - 1], s[j], s[j + 1], r);
        }
        double *tmp = seg; seg = nxt; nxt = tmp;
    }
    for (int64_t p = 0; p < np; p++)
        memcpy(u + p * nx, seg + p * w + 1, (size_t)nx * sizeof(double));
    free(seg); free(nxt);
    return 0;
}

/* O3 -- light-cone window.  w0 holds the initial values of cells
 * [a - t, b + t) (indices taken mod N by the caller), len = (b - a) + 2t.
 * Each step applies Eq. 2 to every cell whose three inputs lie in the
 * window, so the window shrinks by one cell per side per step; after t
 * steps out[0 .. b-a) = u(t) on [a, b).  Domain of dependence of Eq. 2. */
int oracle_window(const double *w0, int64_t len, int64_t t, double r, double *out)
{
    if (t < 0 || len < 2 * t + 1)
        return -1;
    double *cur = (double *)malloc((size_t)len * sizeof(double));
    double *nxt = (double *)malloc((size_t)len * sizeof(double));
    if (!cur || !nxt) {
        free(cur); free(nxt);
        return -1;
    }
    memcpy(cur, w0, (size_t)len * sizeof(double));
    int64_t n = len;
    for (int64_t s = 0; s < t; s++) {
        for (int64_t j = 0; j + 2 < n; j++)
            nxt[j] = eq2(cur[j], cur[j + 1], cur[j + 2], r);
        n -= 2;
        double *tmp = cur; cur = nxt; nxt = tmp;
    }
    memcpy(out, cur, (size_t)n * sizeof(double));
    free(cur); free(nxt);
    return 0;
}
