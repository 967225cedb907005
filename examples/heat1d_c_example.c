/* heat1d_c_example.c -- the C ABI (include/heat1d.h) used from plain C99, no Python, no torch.
 *
 *   cc -std=c99 -I include examples/heat1d_c_example.c -L paper_2307_01117_b200 -lheat1d \
 *      -Wl,-rpath,$PWD/paper_2307_01117_b200 -o heat1d_c_example
 *   ./heat1d_c_example [N] [nt]
 *
 * Solves the paper's model problem (§2): u(0, x_i) = x_i on a periodic ring of N
 * cells (dx = 1), r = k dt/dx^2 = 1/2, nt steps, once with heat1d_set_initial + heat1d_run +
 * heat1d_get and once with heat1d_solve_host, and prints the conserved total heat sum(u)
 * and a checksum.  Exit code 0 iff both paths agree bitwise and sum(u)
 * is conserved to 1e-9 relative. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "heat1d.h"

static int check(int rc, heat1d_t h, const char *what) {
    if (rc != HEAT1D_OK) {
        fprintf(stderr, "%s: %s (%s)\n", what, heat1d_strerror(rc), heat1d_last_error(h));
        exit(2);
    }
    return rc;
}

int main(int argc, char **argv) {
    const int64_t N = argc > 1 ? atoll(argv[1]) : 1000000;   /* the paper's 1e6 cells ...   */
    const int64_t nt = argc > 2 ? atoll(argv[2]) : 1000;     /* ... and 1000 steps */
    double *u0 = malloc((size_t)N * sizeof(double));
    double *a = malloc((size_t)N * sizeof(double));
    double *b = malloc((size_t)N * sizeof(double));
    if (!u0 || !a || !b) return 3;
    for (int64_t i = 0; i < N; ++i) u0[i] = (double)i; /* u(0, x_i) = x_i */

    heat1d_opts o;
    heat1d_opts_default(&o);
    o.resident = 0; /* exercise the temporal-blocked pass kernel and the streamed solve */
    heat1d_t h = NULL;
    check(heat1d_create(&h, N, 1, nt, 0.5, 1.0, 1.0, &o), NULL, "heat1d_create");
    check(heat1d_set_initial(h, u0, N), h, "heat1d_set_initial");
    check(heat1d_run(h, nt), h, "heat1d_run");
    check(heat1d_get(h, a, N), h, "heat1d_get");
    check(heat1d_solve_host(h, u0, N, nt, b), h, "heat1d_solve_host");

    heat1d_info_t info;
    memset(&info, 0, sizeof info);
    info.size = sizeof info;
    check(heat1d_info(h, &info), h, "heat1d_info");
    heat1d_destroy(h);

    long double s0 = 0, s1 = 0, sa = 0;
    uint64_t ck = 0;
    for (int64_t i = 0; i < N; ++i) {
        s0 += u0[i];
        s1 += a[i];
        sa += u0[i] < 0 ? -u0[i] : u0[i];
        uint64_t bits;
        memcpy(&bits, &a[i], sizeof bits);
        ck = ck * 1099511628211ull ^ bits;
    }
    const int same = memcmp(a, b, (size_t)N * sizeof(double)) == 0;
    const long double drift = (s1 - s0) < 0 ? s0 - s1 : s1 - s0;
    printf("N=%lld nt=%lld T=%d dp_ops=%d windows=%lld  sum(u0)=%.17Lg sum(u)=%.17Lg  checksum=%016llx  "
           "solve_host==run:%s\n",
           (long long)N, (long long)nt, info.T, info.dp_ops, (long long)info.stream_windows, s0, s1,
           (unsigned long long)ck, same ? "yes" : "NO");
    free(u0);
    free(a);
    free(b);
    return (same && drift <= 1e-9L * sa) ? 0 : 1;
}
