/*
 * dfft_oracle.c — plain, slow, obviously-correct CPU oracle for the distributed 3D FFT.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2601_12209_b200/, libdfft.so) never links, imports or calls it, and this file
 * shares no source with the CUDA library (no common headers, tables or helpers).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   - the 3D DFT of P:90-96 (§III-A):
 *       Â(kx,ky,kz) = Σ_i Σ_j Σ_l A(i,j,l) · exp(-2πi (kx·i/Nx + ky·j/Ny + kz·l/Nz))
 *     evaluated, as P:97 says, "as a sequence of three independent 1D transforms applied
 *     along the x, y, and z dimensions" (P:101-105 order: x, then y, then z);
 *   - the inverse "same sequence applied in reverse order" (§IV-A): z, y, x with the
 *     conjugate kernel, then ×1/(Nx·Ny·Nz) (reading R1: normalisation);
 *   - R2C (§V-A/B, "exploiting Hermitian symmetry"): the c2c DFT of (x + 0i),
 *     keeping kx ∈ [0, Nx/2] (reading R8); C2R: Hermitian extension along x
 *     (X[Nx-kx, -ky, -kz] = conj X[kx,ky,kz] for 1 ≤ kx < Nx/2), full c2c inverse, real part;
 *   - brute-force O(N²) DFTs (1D and 3D) used to pin the fast path above;
 *   - direct O(N) evaluation of single output bins of the definition, regenerating the input
 *     from the counter-based generator on the fly, for sampled parity at full size.
 * Everything is fp64 (twiddles from x87 long double cosl/sinl, never recurrences).
 *
 * Input generator: value of part p ∈ {0 re, 1 im} at global
 * linear index g = x + Nx·(y + Ny·z) is U(splitmix64((seed << 32) ^ (2g + p))),
 * U(u) = (u >> 11)·2^-52 − 1 ∈ [−1, 1), optionally rounded to float (fp32 plans).
 * The GPU side has its own independent implementation in inputs/; tests check the bits agree.
 *
 * Layout convention: a 3D complex array is interleaved (re, im) doubles, x fastest:
 *   a[2*(x + nx*(y + ny*z)) + {0,1}].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI_L 3.141592653589793238462643383279502884L

/* ------------------------------------------------------------------ generator */

static uint64_t or_splitmix64(uint64_t state) {
    uint64_t z = state + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double or_uniform(uint64_t seed, int64_t g, int part, int round_f32) {
    uint64_t state = (seed << 32) ^ (uint64_t)(2 * g + part);
    double v = (double)(or_splitmix64(state) >> 11) * 0x1p-52 - 1.0;
    if (round_f32) v = (double)(float)v;
    return v;
}

/* Fill a complex box [lo, lo+n) of the global (gnx,gny,gnz) grid, interleaved re/im. */
void or_gen_complex_box(uint64_t seed, int64_t gnx, int64_t gny, int64_t gnz,
                        const int64_t lo[3], const int64_t n[3], int round_f32, double* out) {
    (void)gnz;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < n[2]; ++z)
        for (int64_t y = 0; y < n[1]; ++y)
            for (int64_t x = 0; x < n[0]; ++x) {
                int64_t g = (lo[0] + x) + gnx * ((lo[1] + y) + gny * (lo[2] + z));
                int64_t l = x + n[0] * (y + n[1] * z);
                out[2 * l] = or_uniform(seed, g, 0, round_f32);
                out[2 * l + 1] = or_uniform(seed, g, 1, round_f32);
            }
}

/* Real box (R2C input): the re part of the same generator. */
void or_gen_real_box(uint64_t seed, int64_t gnx, int64_t gny, int64_t gnz,
                     const int64_t lo[3], const int64_t n[3], int round_f32, double* out) {
    (void)gnz;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < n[2]; ++z)
        for (int64_t y = 0; y < n[1]; ++y)
            for (int64_t x = 0; x < n[0]; ++x) {
                int64_t g = (lo[0] + x) + gnx * ((lo[1] + y) + gny * (lo[2] + z));
                out[x + n[0] * (y + n[1] * z)] = or_uniform(seed, g, 0, round_f32);
            }
}

/* ------------------------------------------------------------------ twiddles */

/* w[k] = exp(sign·2πi·k/n), k ∈ [0, n), from long double; sign = -1 forward. */
static void or_twiddles(int64_t n, int sign, double* w) {
    for (int64_t k = 0; k < n; ++k) {
        long double a = 2.0L * OR_PI_L * (long double)k / (long double)n;
        w[2 * k] = (double)cosl(a);
        w[2 * k + 1] = (double)(sign * sinl(a));
    }
}

/* ------------------------------------------------------------------ 1D brute force */

/* X[k] = Σ_t x[t]·exp(sign·2πi·k·t/n): the definition, O(n²). */
void or_dft1d_naive(const double* x, int64_t n, int sign, double* X) {
    double* w = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    or_twiddles(n, sign, w);
    for (int64_t k = 0; k < n; ++k) {
        long double sr = 0, si = 0;
        for (int64_t t = 0; t < n; ++t) {
            int64_t m = (k * t) % n;
            sr += (long double)x[2 * t] * w[2 * m] - (long double)x[2 * t + 1] * w[2 * m + 1];
            si += (long double)x[2 * t] * w[2 * m + 1] + (long double)x[2 * t + 1] * w[2 * m];
        }
        X[2 * k] = (double)sr;
        X[2 * k + 1] = (double)si;
    }
    free(w);
}

/* ------------------------------------------------------------------ 1D fast FFT */

static int64_t or_smallest_factor(int64_t n) {
    for (int64_t p = 2; p * p <= n; ++p)
        if (n % p == 0) return p;
    return n;
}

/*
 * Recursive mixed-radix Cooley-Tukey (decimation in time), out-of-place:
 *   n = p·m, p = smallest prime factor;
 *   X[k1 + m·k2] = Σ_{r<p} w_n^{r·k1}·w_p^{r·k2}·Y_r[k1],  Y_r = DFT_m(x[r], x[r+p], ...).
 * `x` is read with element stride `xs`. `w` is the length-N table exp(sign 2πi k/N) of the
 * top-level length N, and `ws` = N/n is the step that turns it into the table for n.
 */
static void or_fft_rec(const double* x, int64_t xs, int64_t n, double* X,
                       const double* w, int64_t ws, double* tmp) {
    if (n == 1) {
        X[0] = x[0];
        X[1] = x[1];
        return;
    }
    int64_t p = or_smallest_factor(n);
    int64_t m = n / p;
    if (m == 1) { /* prime length: plain DFT with the table */
        for (int64_t k = 0; k < n; ++k) {
            double sr = 0, si = 0;
            for (int64_t t = 0; t < n; ++t) {
                int64_t e = ((k * t) % n) * ws;
                double xr = x[2 * t * xs], xi = x[2 * t * xs + 1];
                sr += xr * w[2 * e] - xi * w[2 * e + 1];
                si += xr * w[2 * e + 1] + xi * w[2 * e];
            }
            X[2 * k] = sr;
            X[2 * k + 1] = si;
        }
        return;
    }
    /* sub-transforms Y_r (r < p) of the decimated sequences, stored in X[r·m ...] */
    for (int64_t r = 0; r < p; ++r)
        or_fft_rec(x + 2 * r * xs, xs * p, m, X + 2 * r * m, w, ws * p, tmp);
    /* combine: for each k1 gather Y_r[k1]·w_n^{r·k1}, then a p-point DFT over r */
    for (int64_t k1 = 0; k1 < m; ++k1) {
        for (int64_t r = 0; r < p; ++r) {
            int64_t e = (r * k1) * ws; /* w_n^{r k1} = w_N^{r k1 · N/n} */
            double yr = X[2 * (r * m + k1)], yi = X[2 * (r * m + k1) + 1];
            tmp[2 * r] = yr * w[2 * e] - yi * w[2 * e + 1];
            tmp[2 * r + 1] = yr * w[2 * e + 1] + yi * w[2 * e];
        }
        for (int64_t k2 = 0; k2 < p; ++k2) {
            double sr = 0, si = 0;
            for (int64_t r = 0; r < p; ++r) {
                int64_t e = ((r * k2) % p) * (n / p) * ws; /* w_p^{r k2} = w_N^{r k2 · N/p} */
                sr += tmp[2 * r] * w[2 * e] - tmp[2 * r + 1] * w[2 * e + 1];
                si += tmp[2 * r] * w[2 * e + 1] + tmp[2 * r + 1] * w[2 * e];
            }
            tmp[2 * (p + k2)] = sr;
            tmp[2 * (p + k2) + 1] = si;
        }
        for (int64_t k2 = 0; k2 < p; ++k2) {
            X[2 * (k1 + m * k2)] = tmp[2 * (p + k2)];
            X[2 * (k1 + m * k2) + 1] = tmp[2 * (p + k2) + 1];
        }
    }
}

/* Iterative radix-2 DIT for n = 2^m: bit-reversal permutation then m butterfly passes. */
static void or_fft_radix2(double* a, int64_t n, const double* w) {
    for (int64_t i = 1, j = 0; i < n; ++i) {
        int64_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double tr = a[2 * i], ti = a[2 * i + 1];
            a[2 * i] = a[2 * j];
            a[2 * i + 1] = a[2 * j + 1];
            a[2 * j] = tr;
            a[2 * j + 1] = ti;
        }
    }
    for (int64_t len = 2; len <= n; len <<= 1) {
        int64_t step = n / len;
        for (int64_t i = 0; i < n; i += len)
            for (int64_t k = 0; k < len / 2; ++k) {
                double wr = w[2 * k * step], wi = w[2 * k * step + 1];
                double* u = a + 2 * (i + k);
                double* v = a + 2 * (i + k + len / 2);
                double vr = v[0] * wr - v[1] * wi, vi = v[0] * wi + v[1] * wr;
                v[0] = u[0] - vr;
                v[1] = u[1] - vi;
                u[0] += vr;
                u[1] += vi;
            }
    }
}

/* In-place 1D FFT of a contiguous interleaved line; sign -1 forward, +1 inverse (no scale). */
typedef struct {
    int64_t n;
    int sign;
    double* w;   /* 2n */
    double* buf; /* 2n */
    double* tmp; /* 4n */
} or_line_plan;

static void or_line_init(or_line_plan* lp, int64_t n, int sign) {
    lp->n = n;
    lp->sign = sign;
    lp->w = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    lp->buf = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    lp->tmp = (double*)malloc(sizeof(double) * 4 * (size_t)n + 64);
    or_twiddles(n, sign, lp->w);
}

static void or_line_free(or_line_plan* lp) {
    free(lp->w);
    free(lp->buf);
    free(lp->tmp);
}

static void or_line_exec(or_line_plan* lp, double* a) {
    int64_t n = lp->n;
    if ((n & (n - 1)) == 0) {
        or_fft_radix2(a, n, lp->w);
    } else {
        or_fft_rec(a, 1, n, lp->buf, lp->w, 1, lp->tmp);
        memcpy(a, lp->buf, sizeof(double) * 2 * (size_t)n);
    }
}

void or_fft1d(double* a, int64_t n, int sign) {
    or_line_plan lp;
    or_line_init(&lp, n, sign);
    or_line_exec(&lp, a);
    or_line_free(&lp);
}

/* ------------------------------------------------------------------ 3D */

/*
 * 1D FFTs along one axis of the (nx,ny,nz) array: gather each line (strided for y, z),
 * transform, scatter back.  axis 0 = x, 1 = y, 2 = z.
 */
static void or_axis_pass(double* a, int64_t nx, int64_t ny, int64_t nz, int axis, int sign) {
    int64_t n = axis == 0 ? nx : axis == 1 ? ny : nz;
    int64_t stride = axis == 0 ? 1 : axis == 1 ? nx : nx * ny;
    int64_t nlines = nx * ny * nz / n;
#pragma omp parallel
    {
        or_line_plan lp;
        or_line_init(&lp, n, sign);
        double* line = (double*)malloc(sizeof(double) * 2 * (size_t)n);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < nlines; ++l) {
            int64_t base;
            if (axis == 0) base = l * nx;                            /* l = y + ny z */
            else if (axis == 1) base = (l % nx) + (l / nx) * nx * ny; /* l = x + nx z */
            else base = l;                                            /* l = x + nx y */
            for (int64_t t = 0; t < n; ++t) {
                line[2 * t] = a[2 * (base + t * stride)];
                line[2 * t + 1] = a[2 * (base + t * stride) + 1];
            }
            or_line_exec(&lp, line);
            for (int64_t t = 0; t < n; ++t) {
                a[2 * (base + t * stride)] = line[2 * t];
                a[2 * (base + t * stride) + 1] = line[2 * t + 1];
            }
        }
        free(line);
        or_line_free(&lp);
    }
}

/* Forward (sign -1): x, y, z.  Inverse (sign +1): z, y, x, ×1/N. */
void or_fft3d(double* a, int64_t nx, int64_t ny, int64_t nz, int sign) {
    if (sign < 0) {
        or_axis_pass(a, nx, ny, nz, 0, -1);
        or_axis_pass(a, nx, ny, nz, 1, -1);
        or_axis_pass(a, nx, ny, nz, 2, -1);
    } else {
        or_axis_pass(a, nx, ny, nz, 2, +1);
        or_axis_pass(a, nx, ny, nz, 1, +1);
        or_axis_pass(a, nx, ny, nz, 0, +1);
        double s = 1.0 / ((double)nx * (double)ny * (double)nz);
        int64_t N = nx * ny * nz;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < 2 * N; ++i) a[i] *= s;
    }
}

/* The 3D definition P:91-96 as a triple sum over the input for every output, O(N²). */
void or_dft3d_naive(const double* a, int64_t nx, int64_t ny, int64_t nz, int sign, double* out) {
    for (int64_t kz = 0; kz < nz; ++kz)
        for (int64_t ky = 0; ky < ny; ++ky)
            for (int64_t kx = 0; kx < nx; ++kx) {
                long double sr = 0, si = 0;
                for (int64_t z = 0; z < nz; ++z)
                    for (int64_t y = 0; y < ny; ++y)
                        for (int64_t x = 0; x < nx; ++x) {
                            long double ph = (long double)sign * 2.0L * OR_PI_L *
                                ((long double)((kx * x) % nx) / nx + (long double)((ky * y) % ny) / ny +
                                 (long double)((kz * z) % nz) / nz);
                            long double c = cosl(ph), s = sinl(ph);
                            const double* v = a + 2 * (x + nx * (y + ny * z));
                            sr += v[0] * c - v[1] * s;
                            si += v[0] * s + v[1] * c;
                        }
                out[2 * (kx + nx * (ky + ny * kz))] = (double)sr;
                out[2 * (kx + nx * (ky + ny * kz)) + 1] = (double)si;
            }
}

/* R2C: c2c of (x + 0i), keep kx ∈ [0, nx/2] -> out is (nx/2+1, ny, nz) complex. */
void or_rfft3d(const double* real, int64_t nx, int64_t ny, int64_t nz, double* out) {
    int64_t N = nx * ny * nz, nxc = nx / 2 + 1;
    double* a = (double*)malloc(sizeof(double) * 2 * (size_t)N);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        a[2 * i] = real[i];
        a[2 * i + 1] = 0.0;
    }
    or_fft3d(a, nx, ny, nz, -1);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nxc; ++x) {
                out[2 * (x + nxc * (y + ny * z))] = a[2 * (x + nx * (y + ny * z))];
                out[2 * (x + nxc * (y + ny * z)) + 1] = a[2 * (x + nx * (y + ny * z)) + 1];
            }
    free(a);
}

/*
 * C2R (reading R8): Hermitian-extend the (nx/2+1, ny, nz) half spectrum along x,
 * X[nx-kx, (ny-ky)%ny, (nz-kz)%nz] = conj X[kx, ky, kz] for 1 <= kx < nx/2, run the full
 * c2c inverse (×1/N) and keep the real part.  Bins kx = 0 and kx = nx/2 are used as given.
 */
void or_irfft3d(const double* half, int64_t nx, int64_t ny, int64_t nz, double* real_out) {
    int64_t N = nx * ny * nz, nxc = nx / 2 + 1;
    double* a = (double*)malloc(sizeof(double) * 2 * (size_t)N);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double re, im;
                if (x < nxc) {
                    re = half[2 * (x + nxc * (y + ny * z))];
                    im = half[2 * (x + nxc * (y + ny * z)) + 1];
                } else {
                    int64_t sx = nx - x, sy = (ny - y) % ny, sz = (nz - z) % nz;
                    re = half[2 * (sx + nxc * (sy + ny * sz))];
                    im = -half[2 * (sx + nxc * (sy + ny * sz)) + 1];
                }
                a[2 * (x + nx * (y + ny * z))] = re;
                a[2 * (x + nx * (y + ny * z)) + 1] = im;
            }
    or_fft3d(a, nx, ny, nz, +1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) real_out[i] = a[2 * i];
    free(a);
}

/* ------------------------------------------------------------------ real-to-real (DCT) */

/*
 * R2R transforms (P:403 lists C2C, R2C and R2R; the algorithm is unstated — reading R21):
 * the forward R2R is the DCT-II along every axis (FFTW REDFT10, the transform of a Bounded /
 * Neumann direction):  X_k = 2 Σ_{n<N} x_n cos(π k (2n+1) / (2N)),  k < N;
 * the inverse is the DCT-III along every axis divided by 2N (so inverse(forward(x)) = x):
 *   x_n = (X_0 + 2 Σ_{0<k<N} X_k cos(π k (2n+1) / (2N))) / (2N).
 * Written as the definitions (O(N) per output, cosines in long double), one axis at a time
 * (the 3D transform is separable exactly like the DFT).
 */
static void or_dct_line(const double* x, int64_t xs, int64_t n, int inverse, double* y, int64_t ys,
                        const double* c /* cos(π m / (2n)), m < 4n */) {
    for (int64_t a = 0; a < n; ++a) {
        long double acc = 0.0L;
        if (!inverse) {
            for (int64_t b = 0; b < n; ++b) acc += (long double)x[b * xs] * c[(a * (2 * b + 1)) % (4 * n)];
            y[a * ys] = (double)(2.0L * acc);
        } else {
            acc = (long double)x[0];
            for (int64_t b = 1; b < n; ++b) acc += 2.0L * (long double)x[b * xs] * c[(b * (2 * a + 1)) % (4 * n)];
            y[a * ys] = (double)(acc / (long double)(2 * n));
        }
    }
}

static void or_dct_axis(double* a, int64_t nx, int64_t ny, int64_t nz, int axis, int inverse) {
    int64_t n = axis == 0 ? nx : axis == 1 ? ny : nz;
    int64_t stride = axis == 0 ? 1 : axis == 1 ? nx : nx * ny;
    int64_t lines = nx * ny * nz / n;
    double* c = (double*)malloc(sizeof(double) * 4 * (size_t)n);
    for (int64_t m = 0; m < 4 * n; ++m)
        c[m] = (double)cosl(3.14159265358979323846264338327950288L * (long double)m / (long double)(2 * n));
#pragma omp parallel
    {
        double* in = (double*)malloc(sizeof(double) * (size_t)n);
        double* out = (double*)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < lines; ++l) {
            int64_t base;
            if (axis == 0) base = l * nx;
            else if (axis == 1) base = (l % nx) + (l / nx) * nx * ny;
            else base = l;
            for (int64_t t = 0; t < n; ++t) in[t] = a[base + t * stride];
            or_dct_line(in, 1, n, inverse, out, 1, c);
            for (int64_t t = 0; t < n; ++t) a[base + t * stride] = out[t];
        }
        free(in);
        free(out);
    }
    free(c);
}

/* 3D DCT-II (forward) / DCT-III / (2N) (inverse), in place on a real (nx, ny, nz) array. */
void or_dct3d(double* a, int64_t nx, int64_t ny, int64_t nz, int inverse) {
    for (int axis = 0; axis < 3; ++axis) or_dct_axis(a, nx, ny, nz, inverse ? 2 - axis : axis, inverse);
}

/* ------------------------------------------------------------------ periodic Poisson solve */

/*
 * Periodic Poisson solve ∇²φ = f on an nx×ny×nz grid with spacings (dx, dy, dz): the paper's
 * application (§VI-B: the Oceananigans pressure solver on a (Periodic, Periodic,
 * Periodic) box) with the operator the paper leaves unstated taken as the second-order
 * 7-point discrete Laplacian (reading R20).  Its eigenvalue on the Fourier mode k is
 *   λ(k) = -Σ_d (2 sin(π k_d / n_d) / Δ_d)²,
 * so, step by step: F = R2C(f); Φ(k) = F(k) / λ(k) for k ≠ 0, Φ(0) = 0 (zero-mean solution);
 * φ = C2R(Φ).  λ is evaluated in long double (sinl), rounded once.
 */
void or_poisson_eigen(int64_t n, double h, double* lam) {
    for (int64_t k = 0; k < n; ++k) {
        long double s = 2.0L * sinl(3.14159265358979323846264338327950288L * (long double)k / (long double)n) /
                        (long double)h;
        lam[k] = (double)(-(s * s));
    }
}

void or_poisson3d(const double* f, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
                  double* phi) {
    int64_t nxc = nx / 2 + 1;
    double* F = (double*)malloc(sizeof(double) * 2 * (size_t)(nxc * ny * nz));
    double* lx = (double*)malloc(sizeof(double) * (size_t)nx);
    double* ly = (double*)malloc(sizeof(double) * (size_t)ny);
    double* lz = (double*)malloc(sizeof(double) * (size_t)nz);
    or_poisson_eigen(nx, dx, lx);
    or_poisson_eigen(ny, dy, ly);
    or_poisson_eigen(nz, dz, lz);
    or_rfft3d(f, nx, ny, nz, F);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nxc; ++x) {
                double lam = lx[x] + ly[y] + lz[z];
                double* v = F + 2 * (x + nxc * (y + ny * z));
                if (x == 0 && y == 0 && z == 0) {
                    v[0] = 0.0;
                    v[1] = 0.0;
                } else {
                    v[0] /= lam;
                    v[1] /= lam;
                }
            }
    or_irfft3d(F, nx, ny, nz, phi);
    free(F);
    free(lx);
    free(ly);
    free(lz);
}

/* 7-point periodic discrete Laplacian (the operator R20 inverts), used only by the pins. */
void or_laplacian7(const double* phi, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
                   double* out) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
#define PHI(a, b, c) phi[(((a) + nx) % nx) + nx * ((((b) + ny) % ny) + ny * (((c) + nz) % nz))]
                double c0 = PHI(x, y, z);
                out[x + nx * (y + ny * z)] = (PHI(x + 1, y, z) - 2 * c0 + PHI(x - 1, y, z)) / (dx * dx) +
                                             (PHI(x, y + 1, z) - 2 * c0 + PHI(x, y - 1, z)) / (dy * dy) +
                                             (PHI(x, y, z + 1) - 2 * c0 + PHI(x, y, z - 1)) / (dz * dz);
#undef PHI
            }
}

/* ------------------------------------------------------------------ sampled bins */

/*
 * One output bin of the forward definition for the seeded generator input, with
 * the input regenerated on the fly (no N-sized memory):
 *   X(kx,ky,kz) = Σ_z w_nz^{kz z} Σ_y w_ny^{ky y} Σ_x w_nx^{kx x} A(x,y,z).
 * real_input != 0 takes the R2C input (re part, im = 0).  O(N) work per bin.
 */
void or_dft3d_bin_seeded(uint64_t seed, int64_t nx, int64_t ny, int64_t nz, int round_f32,
                         int real_input, int64_t kx, int64_t ky, int64_t kz, double out[2]) {
    double* wx = (double*)malloc(sizeof(double) * 2 * (size_t)nx);
    double* wy = (double*)malloc(sizeof(double) * 2 * (size_t)ny);
    double* wz = (double*)malloc(sizeof(double) * 2 * (size_t)nz);
    or_twiddles(nx, -1, wx);
    or_twiddles(ny, -1, wy);
    or_twiddles(nz, -1, wz);
    double tr = 0, ti = 0;
#pragma omp parallel for reduction(+ : tr, ti) schedule(static)
    for (int64_t z = 0; z < nz; ++z) {
        double zr = 0, zi = 0;
        for (int64_t y = 0; y < ny; ++y) {
            double yr = 0, yi = 0;
            for (int64_t x = 0; x < nx; ++x) {
                int64_t g = x + nx * (y + ny * z);
                double ar = or_uniform(seed, g, 0, round_f32);
                double ai = real_input ? 0.0 : or_uniform(seed, g, 1, round_f32);
                int64_t e = (kx * x) % nx;
                yr += ar * wx[2 * e] - ai * wx[2 * e + 1];
                yi += ar * wx[2 * e + 1] + ai * wx[2 * e];
            }
            int64_t e = (ky * y) % ny;
            zr += yr * wy[2 * e] - yi * wy[2 * e + 1];
            zi += yr * wy[2 * e + 1] + yi * wy[2 * e];
        }
        int64_t e = (kz * z) % nz;
        tr += zr * wz[2 * e] - zi * wz[2 * e + 1];
        ti += zr * wz[2 * e + 1] + zi * wz[2 * e];
    }
    out[0] = tr;
    out[1] = ti;
    free(wx);
    free(wy);
    free(wz);
}

/* ------------------------------------------------------------------ error metrics */

/* Σ|a-b|² and Σ|b|² over n doubles (complex arrays pass 2n), Kahan-compensated. */
void or_err_sums(const double* a, const double* b, int64_t n, double out[2]) {
    double se = 0, ce = 0, sr = 0, cr = 0;
    for (int64_t i = 0; i < n; ++i) {
        double d = a[i] - b[i];
        double y = d * d - ce;
        double t = se + y;
        ce = (t - se) - y;
        se = t;
        y = b[i] * b[i] - cr;
        t = sr + y;
        cr = (t - sr) - y;
        sr = t;
    }
    out[0] = se;
    out[1] = sr;
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count for the timing legs (torchrun sets OMP_NUM_THREADS=1 per rank). */
void or_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ per-axis transform kinds (f4) */

/*
 * Bounded directions ("C2C, R2C and R2R"; "DCT and DST"; P:620 the (Periodic,
 * Periodic, Bounded) topology): each axis carries its own 1D transform, kind
 *   0 = DFT   (Periodic):                     X_k = Σ_n x_n e^{∓2πi kn/N}
 *   1 = DCT-II (Bounded, Neumann; REDFT10):   X_k = 2 Σ_n x_n cos(π k (2n+1) / (2N))
 *   2 = DST-II (Bounded, Dirichlet; RODFT10): X_k = 2 Σ_n x_n sin(π (k+1) (2n+1) / (2N))
 * with inverses DFT⁺/N, DCT-III/(2N) and DST-III/(2N) (RODFT01):
 *   x_n = ((-1)^n X_{N-1} + 2 Σ_{k<N-1} X_k sin(π (k+1) (2n+1) / (2N))) / (2N)
 * (reading R22).  The 3D transform applies the axes in the paper's order (x, y, z
 * forward; z, y, x inverse).  A real-coefficient transform (DCT / DST) of
 * complex data transforms the real and imaginary parts alike (it is linear), which is how a
 * bounded direction follows an R2C (periodic) x axis.  Sums written out, sines in long double.
 */
static void or_dst_line(const double* x, int64_t n, int inverse, double* y, const double* s /* sin(π m/(2n)), m < 4n */) {
    for (int64_t a = 0; a < n; ++a) {
        long double acc = 0.0L;
        if (!inverse) {
            for (int64_t b = 0; b < n; ++b) acc += (long double)x[b] * s[((a + 1) * (2 * b + 1)) % (4 * n)];
            y[a] = (double)(2.0L * acc);
        } else {
            acc = (a % 2 ? -1.0L : 1.0L) * (long double)x[n - 1];
            for (int64_t b = 0; b + 1 < n; ++b) acc += 2.0L * (long double)x[b] * s[((b + 1) * (2 * a + 1)) % (4 * n)];
            y[a] = (double)(acc / (long double)(2 * n));
        }
    }
}

/* One axis of a complex (nx, ny, nz) array (interleaved re, im): kind 0 = the DFT (sign -1 forward;
 * inverse sign +1 and ×1/n), kinds 1 / 2 = DCT / DST of the real and the imaginary parts. */
void or_axis_transform(double* a, int64_t nx, int64_t ny, int64_t nz, int axis, int kind, int inverse) {
    const int64_t n = axis == 0 ? nx : axis == 1 ? ny : nz;
    const int64_t stride = axis == 0 ? 1 : axis == 1 ? nx : nx * ny;
    const int64_t lines = nx * ny * nz / n;
    double* tab = (double*)malloc(sizeof(double) * 4 * (size_t)n);
    for (int64_t m = 0; m < 4 * n; ++m) {
        const long double ang = OR_PI_L * (long double)m / (long double)(2 * n);
        tab[m] = (double)(kind == 2 ? sinl(ang) : cosl(ang));
    }
#pragma omp parallel
    {
        double* line = (double*)malloc(sizeof(double) * 2 * (size_t)n);
        double* in = (double*)malloc(sizeof(double) * (size_t)n);
        double* out = (double*)malloc(sizeof(double) * (size_t)n);
        or_line_plan lp;
        if (kind == 0) or_line_init(&lp, n, inverse ? +1 : -1);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < lines; ++l) {
            int64_t base;
            if (axis == 0) base = l * nx;
            else if (axis == 1) base = (l % nx) + (l / nx) * nx * ny;
            else base = l;
            if (kind == 0) {
                for (int64_t t = 0; t < n; ++t) {
                    line[2 * t] = a[2 * (base + t * stride)];
                    line[2 * t + 1] = a[2 * (base + t * stride) + 1];
                }
                or_line_exec(&lp, line);
                const double sc = inverse ? 1.0 / (double)n : 1.0;
                for (int64_t t = 0; t < n; ++t) {
                    a[2 * (base + t * stride)] = line[2 * t] * sc;
                    a[2 * (base + t * stride) + 1] = line[2 * t + 1] * sc;
                }
            } else {
                for (int part = 0; part < 2; ++part) {
                    for (int64_t t = 0; t < n; ++t) in[t] = a[2 * (base + t * stride) + part];
                    if (kind == 1) or_dct_line(in, 1, n, inverse, out, 1, tab);
                    else or_dst_line(in, n, inverse, out, tab);
                    for (int64_t t = 0; t < n; ++t) a[2 * (base + t * stride) + part] = out[t];
                }
            }
        }
        if (kind == 0) or_line_free(&lp);
        free(line);
        free(in);
        free(out);
    }
    free(tab);
}

/* R2C along x only: each real x-line → c2c DFT of (x + 0i), bins 0..nx/2 (reading R8, per line). */
void or_rfft_x(const double* real, int64_t nx, int64_t ny, int64_t nz, double* out) {
    const int64_t nxc = nx / 2 + 1;
#pragma omp parallel
    {
        double* line = (double*)malloc(sizeof(double) * 2 * (size_t)nx);
        or_line_plan lp;
        or_line_init(&lp, nx, -1);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < ny * nz; ++l) {
            for (int64_t t = 0; t < nx; ++t) {
                line[2 * t] = real[l * nx + t];
                line[2 * t + 1] = 0.0;
            }
            or_line_exec(&lp, line);
            memcpy(out + 2 * l * nxc, line, sizeof(double) * 2 * (size_t)nxc);
        }
        or_line_free(&lp);
        free(line);
    }
}

/* C2R along x only: Hermitian-extend each half line (X[nx-k] = conj X[k], 1 <= k < nx/2; the
 * imaginary parts of bins 0 and nx/2 dropped), inverse DFT ×1/nx, real part (reading R8). */
void or_irfft_x(const double* half, int64_t nx, int64_t ny, int64_t nz, double* real_out) {
    const int64_t nxc = nx / 2 + 1;
#pragma omp parallel
    {
        double* line = (double*)malloc(sizeof(double) * 2 * (size_t)nx);
        or_line_plan lp;
        or_line_init(&lp, nx, +1);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < ny * nz; ++l) {
            const double* h = half + 2 * l * nxc;
            for (int64_t t = 0; t < nx; ++t) {
                if (t < nxc) {
                    line[2 * t] = h[2 * t];
                    line[2 * t + 1] = (t == 0 || 2 * t == nx) ? 0.0 : h[2 * t + 1];
                } else {
                    line[2 * t] = h[2 * (nx - t)];
                    line[2 * t + 1] = -h[2 * (nx - t) + 1];
                }
            }
            or_line_exec(&lp, line);
            for (int64_t t = 0; t < nx; ++t) real_out[l * nx + t] = line[2 * t] / (double)nx;
        }
        or_line_free(&lp);
        free(line);
    }
}

/*
 * Eigenvalues of the second-order 3-point difference along one axis of n cells, spacing h, on
 * the basis of its transform kind (reading R22):
 *   DFT (periodic):                       λ_k = -(2 sin(π k / n) / h)²
 *   DCT-II (Neumann, cell-centred mirror): λ_k = -(2 sin(π k / (2n)) / h)²
 *   DST-II (Dirichlet, cell-centred antimirror): λ_k = -(2 sin(π (k+1) / (2n)) / h)²
 */
void or_poisson_eigen_kind(int64_t n, double h, int kind, double* lam) {
    for (int64_t k = 0; k < n; ++k) {
        const long double ang = kind == 0 ? OR_PI_L * (long double)k / (long double)n
                              : kind == 1 ? OR_PI_L * (long double)k / (long double)(2 * n)
                                          : OR_PI_L * (long double)(k + 1) / (long double)(2 * n);
        const long double s = 2.0L * sinl(ang) / (long double)h;
        lam[k] = (double)(-(s * s));
    }
}
