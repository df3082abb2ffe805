/*
 * lif_oracle.c -- the CPU ORACLE for the temporally fused LIF path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2408_00280_b200/) never imports, links or executes anything under oracle/,
 * and this file shares no code, header, constant or helper with csrc/.
 *
 * What it is: the plain definition of what the fused kernels compute, written as a
 * per-time-step loop over t with an inner loop over neurons, in fp64 on the exact
 * input values.  Temporal fusion only reorders memory traffic ("reordering
 * computations does not impact the end results"), so the oracle is the
 * step-wise definition itself: no blocking, no fusion, no reordering.
 *
 * Citations (PAPER.md line numbers; BJ = BASELINE.json; SURVEY = SURVEY.md section):
 *   initial state    v^(0) = V_rest
 *   charge  (Eq. 1)  v^t = k v^{t-1}(1-y^{t-1}) + V_rest y^{t-1} + x^t
 *   fire    (Eq. 2)  y^t = H(v^t - V_th), H(z) = 1 iff z >= 0
 *   backward(Eq. 3)  grad x^t = k grad v^{t+1}[1 - y^t - v^t d(v^t)] + grad y^t d(v^t)
 *                                                                  PAPER.md:184-189
 *   sigmoid surrogate d(x) = a e^{-ax}/(1+e^{-ax})^2, a = 4
 *   north-star charge H[t] = V[t-1] + (X[t] - (V[t-1] - V_reset))/tau, hard/soft reset
 *                                                                  BJ.north_star
 * Readings of silent / ambiguous points are SURVEY.md 8(c).3 R1-R22 and DESIGN.md
 * "Readings"; the ones this file depends on are cited inline (R2, R3, R4, R5, R6, R8,
 * R10, R11, R12).
 *
 * Variable names: H[t,n] is the pre-reset membrane potential (the paper's v^(t)),
 * S[t,n] the spike (the paper's y^(t)), V the post-reset potential carried to t+1.
 * Layout of every [T, N] array: row-major, time-major, element (t, n) at t*N + n
 * ("memory alignment post-concatenation").
 *
 * Parity pins: every function here is pinned by tests/test_oracle_pins.py
 * (closed forms, scipy.signal.lfilter special cases, hand traces under tests/golden/,
 * the paper's literal Eq. 1 / Eq. 3 at V_reset = 0, and finite differences of the
 * surrogate-smoothed model).  Parity unpinned: the arctan surrogate's and the soft
 * reset's scale conventions relative to any external library --
 * they are pinned only for internal consistency (closed form of d_atan(0), its
 * integral, and finite differences).
 *
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -o liblif_oracle.so lif_oracle.c -lm
 * (no fast-math; -ffp-contract=off keeps every a*b+c as two roundings, as written).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

typedef struct {
    double tau;          /* membrane time constant; k = 1 - 1/tau            */
    double v_th;         /* threshold V_th                                    */
    double v_reset;      /* reset / resting potential V_rest            */
    int    soft_reset;   /* 0: hard reset (Eq. 1 via (1-y), V_rest*y); 1: soft (BJ.north_star) */
    int    decay_input;  /* 1: H = V + (X - (V - Vr))/tau (BJ); 0: H = V - (V - Vr)/tau + X (Eq. 1) */
    int    detach_reset; /* 1: drop the gradient through the reset               */
    int    surrogate;    /* 0: sigmoid; 1: arctan            */
    double alpha;        /* surrogate sharpness (4.0)                          */
    int    smoothed;     /* 1: replace the Heaviside by the surrogate's primitive everywhere
                            (forward fire, reset, and the backward's (1 - S)); used ONLY for
                            finite-difference pins, SURVEY 8(c).2                            */
} lif_oracle_params;

static const double ORACLE_PI = 3.14159265358979323846;

/* Surrogate derivative delta(u), u = H - V_th (centred where the Heaviside
 * switches).  Sigmoid: PAPER.md:439, evaluated in the |u| form, which is
 * the same value because a e^{-au}/(1+e^{-au})^2 is even in u.  Arctan: SURVEY R11. */
double lif_oracle_surrogate(const lif_oracle_params* p, double u)
{
    if (p->surrogate == 0) {
        double e = exp(-p->alpha * fabs(u));
        return p->alpha * e / ((1.0 + e) * (1.0 + e));
    } else {
        double z = (ORACLE_PI / 2.0) * p->alpha * u;
        return (p->alpha / 2.0) / (1.0 + z * z);
    }
}

/* The surrogate's primitive (the smooth step whose derivative is delta).  Sigmoid:
 * sigma(a u) = 1/(1+e^{-a u}) ("delta = sigma'");  arctan:
 * 1/2 + arctan(pi/2 a u)/pi.  Used only when p->smoothed. */
double lif_oracle_smooth_step(const lif_oracle_params* p, double u)
{
    if (p->surrogate == 0) {
        return 1.0 / (1.0 + exp(-p->alpha * u));
    } else {
        return 0.5 + atan((ORACLE_PI / 2.0) * p->alpha * u) / ORACLE_PI;
    }
}

/* Spike of Eq. 2: 1 iff H - V_th >= 0, compared as H >= V_th
 * (SURVEY R3).  NaN H gives 0. */
static double fire(const lif_oracle_params* p, double H)
{
    if (p->smoothed) return lif_oracle_smooth_step(p, H - p->v_th);
    return (H >= p->v_th) ? 1.0 : 0.0;
}

/*
 * Forward over all T steps.
 *   x       [T, N]  input currents (fp32/bf16 values widened to double by the caller)
 *   v_init  [N] or NULL -> V_reset (no prior spike)
 *   S_out   [T, N]  spikes (0.0 / 1.0; the smooth step when p->smoothed)
 *   H_out   [T, N]  pre-reset potential (the paper's v^(t), which Eq. 3 consumes)
 *   V_out   [T, N] or NULL: post-reset potential after each step
 *   v_final [N] or NULL: V after step T-1 (segment carry-out)
 */
void lif_oracle_forward(const lif_oracle_params* p, int64_t T, int64_t N,
                        const double* x, const double* v_init,
                        double* S_out, double* H_out, double* V_out, double* v_final,
                        double* V_work /* [N] scratch owned by the caller */)
{
    double* V = V_work;
    const double k = 1.0 - 1.0 / p->tau;   /* k_tau = 1 - 1/tau */
    for (int64_t n = 0; n < N; ++n) V[n] = v_init ? v_init[n] : p->v_reset;

    for (int64_t t = 0; t < T; ++t) {
        for (int64_t n = 0; n < N; ++n) {
            double X = x[t * N + n];
            double Vp = V[n];
            double H;
            /* charge (Eq. 1 / BJ.north_star; SURVEY 0.1 shows they are one family) */
            if (p->decay_input)
                H = Vp + (X - (Vp - p->v_reset)) / p->tau;   /* BJ.north_star, verbatim */
            else   /* Eq. 1 as printed, k_tau v^(t-1) + x^(t), plus the
                      V_reset/tau offset of the family (0 at the paper's V_rest = 0) */
                H = k * Vp + p->v_reset / p->tau + X;
            /* fire (Eq. 2) */
            double S = fire(p, H);
            /* reset: hard = V_rest*y + (1-y)*(...) of Eq. 1; soft = BJ.north_star */
            double Vn;
            if (p->soft_reset)
                Vn = H - p->v_th * S;
            else if (p->smoothed)
                Vn = H * (1.0 - S) + p->v_reset * S;
            else
                Vn = (S != 0.0) ? p->v_reset : H;
            V[n] = Vn;
            S_out[t * N + n] = S;
            H_out[t * N + n] = H;
            if (V_out) V_out[t * N + n] = Vn;
        }
    }
    if (v_final)
        for (int64_t n = 0; n < N; ++n) v_final[n] = V[n];
}

/*
 * Backward (surrogate-gradient BPTT), walking t = T-1 .. 0.
 *   gS          [T, N]  dL/dS[t] from the next layer (the paper's grad y^t)
 *   H           [T, N]  pre-reset potentials from the forward; S is re-derived from H
 *                       by Eq. 2 (it is a function of H alone)
 *   grad_v_final[N] or NULL -> 0: dL/dV[T-1] from a later time segment
 *   gX          [T, N]  dL/dX[t]
 *   grad_v_init [N] or NULL: dL/dV[-1] (carry-out to an earlier segment)
 *   delta_out / dvdh_out [T, N] or NULL: the per-step delta and dV/dH (exposed so the
 *                       parity comparator can bound rounding error; no other use)
 *
 * Derivation: with k = 1 - 1/tau and s = dH/dX = (decay_input ? 1/tau : 1),
 *   dH[t+1]/dV[t] = k in both charge forms;
 *   hard reset V = H(1-S) + V_reset S  =>  dV/dH = (1 - S) + (V_reset - H) delta;
 *   soft reset V = H - V_th S          =>  dV/dH = 1 - V_th delta;
 *   (detach_reset drops the delta term of dV/dH)
 *   gH[t] = gS[t] delta[t] + gV[t] dV/dH[t];   gX[t] = s gH[t];   gV[t-1] = k gH[t].
 * In paper mode (V_reset = 0, hard, decay_input = 0) gX[t] = gH[t] and this is literally
 * Eq. 3: gX^t = k gX^{t+1} [1 - y^t - v^t delta(v^t)] + grad y^t delta(v^t).
 */
void lif_oracle_backward(const lif_oracle_params* p, int64_t T, int64_t N,
                         const double* gS, const double* H,
                         const double* grad_v_final,
                         double* gX, double* grad_v_init,
                         double* gV_work /* [N] scratch owned by the caller */,
                         double* delta_out /* [T, N] or NULL: delta[t, n] */,
                         double* dvdh_out  /* [T, N] or NULL: dV/dH[t, n] */)
{
    const double k = 1.0 - 1.0 / p->tau;
    const double s = p->decay_input ? 1.0 / p->tau : 1.0;
    double* gV = gV_work;
    for (int64_t n = 0; n < N; ++n) gV[n] = grad_v_final ? grad_v_final[n] : 0.0;

    for (int64_t t = T - 1; t >= 0; --t) {
        for (int64_t n = 0; n < N; ++n) {
            double h = H[t * N + n];
            double u = h - p->v_th;
            double delta = lif_oracle_surrogate(p, u);
            double S = fire(p, h);
            double dVdH;
            if (p->soft_reset)
                dVdH = 1.0 - (p->detach_reset ? 0.0 : p->v_th * delta);
            else
                dVdH = (1.0 - S) + (p->detach_reset ? 0.0 : (p->v_reset - h) * delta);
            double gH = gS[t * N + n] * delta + gV[n] * dVdH;
            if (delta_out) delta_out[t * N + n] = delta;
            if (dvdh_out) dvdh_out[t * N + n] = dVdH;
            gX[t * N + n] = s * gH;
            gV[n] = k * gH;
        }
    }
    if (grad_v_init)
        for (int64_t n = 0; n < N; ++n) grad_v_init[n] = gV[n];
}

/*
 * Per-channel affine prologue (a BatchNorm affine folded into the LIF
 * input).  Plain definition: the layer's input current is
 *     X'[t, n] = scale[c] * X[t, n] + shift[c],   c = (n / HW) % C,
 * and, by the chain rule through that line,
 *     dL/dX[t, n] = scale[c] * dL/dX'[t, n],
 *     dL/dscale[c] = sum_{t, n: c(n) = c} dL/dX'[t, n] * X[t, n],
 *     dL/dshift[c] = sum_{t, n: c(n) = c} dL/dX'[t, n].
 * Pinned by finite differences of the smoothed model (tests/test_oracle_pins.py).
 */
void lif_oracle_affine_input(int64_t T, int64_t N, const double* x, const double* scale,
                             const double* shift, int64_t C, int64_t HW, double* xout)
{
    for (int64_t t = 0; t < T; ++t)
        for (int64_t n = 0; n < N; ++n) {
            int64_t c = (n / HW) % C;
            xout[t * N + n] = scale[c] * x[t * N + n] + shift[c];
        }
}

void lif_oracle_affine_grads(int64_t T, int64_t N, const double* x, const double* gxp,
                             const double* scale, int64_t C, int64_t HW,
                             double* gx, double* gscale, double* gshift)
{
    for (int64_t c = 0; c < C; ++c) { gscale[c] = 0.0; gshift[c] = 0.0; }
    for (int64_t t = 0; t < T; ++t)
        for (int64_t n = 0; n < N; ++n) {
            int64_t c = (n / HW) % C;
            double g = gxp[t * N + n];
            gx[t * N + n] = scale[c] * g;
            gscale[c] += g * x[t * N + n];
            gshift[c] += g;
        }
}

/*
 * Residual add in the prologue ("fold the preceding BN affine / residual
 * add into the LIF prologue"; the spiking-ResNet block feeds its LIF neuron with
 * BN(conv(.)) + shortcut).  Plain definition: the layer's input current is
 *     X'[t, n] = scale[c] * X[t, n] + shift[c] + R[t, n],   c = (n / HW) % C,
 * with R the shortcut tensor, and by the chain rule
 *     dL/dR[t, n] = dL/dX'[t, n]
 * while dL/dX, dL/dscale and dL/dshift are lif_oracle_affine_grads' (R does not enter them).
 * Pinned by finite differences of the smoothed model with respect to R
 * (tests/test_oracle_pins.py).
 */
void lif_oracle_affine_residual_input(int64_t T, int64_t N, const double* x, const double* scale,
                                      const double* shift, const double* r, int64_t C, int64_t HW,
                                      double* xout)
{
    for (int64_t t = 0; t < T; ++t)
        for (int64_t n = 0; n < N; ++n) {
            int64_t c = (n / HW) % C;
            xout[t * N + n] = scale[c] * x[t * N + n] + shift[c] + r[t * N + n];
        }
}
