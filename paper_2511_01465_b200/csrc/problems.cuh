// problems.cuh — device functors for the ODE right-hand sides.
//
// The reference's plug-in is OdeProblem(f_into, jac_into) (problems.py:36-65),
// numba dispatchers the solver kernels specialise on (_kernels.py:7-9).  Here
// each problem is a functor type the fused kernels are templated on; the
// parameters arrive by value in the kernel arguments.  Expression trees keep
// the reference's association order (problems.py file:line per functor) so that
// the only differences from the CPU oracle are FMA contraction and the scan's
// association.  Jacobians are written densely, zeros included, exactly like
// the reference's jac_into: 0*inf = NaN must leak the same way.
#pragma once

#include "../../include/odescan_b200.h"

namespace odx {

struct ProbParams {
    double p[ODX_MAX_PARAMS];
};

// problems.py:85-99 (r, K)
struct Logistic {
    static constexpr int D = 1;
    double r, K;
    __device__ __forceinline__ explicit Logistic(const ProbParams& q) : r(q.p[0]), K(q.p[1]) {}
    __device__ __forceinline__ void f(const double* x, double* o) const {
        o[0] = r * x[0] * (1.0 - x[0] / K);
    }
    __device__ __forceinline__ void jac(const double* x, double* J) const {
        J[0] = r * (1.0 - 2.0 * x[0] / K);
    }
};

// problems.py:117-134 with mu as a parameter (BASELINE cfg 2: mu=10, cfg 5: mu=1)
struct VanDerPol {
    static constexpr int D = 2;
    double mu;
    __device__ __forceinline__ explicit VanDerPol(const ProbParams& q) : mu(q.p[0]) {}
    __device__ __forceinline__ void f(const double* x, double* o) const {
        o[0] = x[1];
        o[1] = mu * (1.0 - x[0] * x[0]) * x[1] - x[0];
    }
    __device__ __forceinline__ void jac(const double* x, double* J) const {
        J[0] = 0.0;
        J[1] = 1.0;
        J[2] = -2.0 * mu * x[0] * x[1] - 1.0;
        J[3] = mu * (1.0 - x[0] * x[0]);
    }
};

// problems.py:155-226 (g, l, m_c, m_p); SQ selects the centripetal variant
template <bool SQ>
struct CartPoleT {
    static constexpr int D = 4;
    double G, L, MC, MP;
    __device__ __forceinline__ explicit CartPoleT(const ProbParams& q)
        : G(q.p[0]), L(q.p[1]), MC(q.p[2]), MP(q.p[3]) {}
    __device__ __forceinline__ void f(const double* x, double* o) const {
        double s = sin(x[2]), c = cos(x[2]), w = x[3];
        double den = MC + MP * s * s;
        o[0] = x[1];
        if (SQ)
            o[1] = MP * s * (L * w * w + G * c) / den;
        else
            o[1] = MP * s * (L * w + G * c) / den;
        o[2] = w;
        o[3] = (-MP * L * w * w * c * s - (MC + MP) * G * s) / (L * den);
    }
    __device__ __forceinline__ void jac(const double* x, double* J) const {
        double s = sin(x[2]), c = cos(x[2]), w = x[3];
        double den = MC + MP * s * s;
        double dden = 2.0 * MP * s * c;
#pragma unroll
        for (int i = 0; i < 16; i++) J[i] = 0.0;
        J[1] = 1.0;
        J[11] = 1.0;
        double num1, dnum1;
        if (SQ) {
            num1 = MP * s * (L * w * w + G * c);
            dnum1 = MP * c * (L * w * w + G * c) + MP * s * (-G * s);
        } else {
            num1 = MP * s * (L * w + G * c);
            dnum1 = MP * c * (L * w + G * c) + MP * s * (-G * s);
        }
        J[6] = dnum1 / den - num1 * dden / (den * den);
        J[7] = SQ ? 2.0 * MP * s * L * w / den : MP * s * L / den;
        double num3 = -MP * L * w * w * c * s - (MC + MP) * G * s;
        double dnum3 = -MP * L * w * w * (c * c - s * s) - (MC + MP) * G * c;
        J[14] = dnum3 / (L * den) - num3 * dden / (L * den * den);
        J[15] = -2.0 * MP * L * w * c * s / (L * den);
    }
};
using CartPole = CartPoleT<false>;
using CartPoleSq = CartPoleT<true>;

// problems.py:245-254 (lambda)
struct Dahlquist {
    static constexpr int D = 1;
    double lam;
    __device__ __forceinline__ explicit Dahlquist(const ProbParams& q) : lam(q.p[0]) {}
    __device__ __forceinline__ void f(const double* x, double* o) const { o[0] = lam * x[0]; }
    __device__ __forceinline__ void jac(const double*, double* J) const { J[0] = lam; }
};

// problems.py:275-297 (k1, k2, k3)
struct Robertson {
    static constexpr int D = 3;
    double k1, k2, k3;
    __device__ __forceinline__ explicit Robertson(const ProbParams& q)
        : k1(q.p[0]), k2(q.p[1]), k3(q.p[2]) {}
    __device__ __forceinline__ void f(const double* x, double* o) const {
        o[0] = -k1 * x[0] + k3 * x[1] * x[2];
        o[1] = k1 * x[0] - k2 * x[1] * x[1] - k3 * x[1] * x[2];
        o[2] = k2 * x[1] * x[1];
    }
    __device__ __forceinline__ void jac(const double* x, double* J) const {
        J[0] = -k1;
        J[1] = k3 * x[2];
        J[2] = k3 * x[1];
        J[3] = k1;
        J[4] = -2.0 * k2 * x[1] - k3 * x[2];
        J[5] = -k3 * x[1];
        J[6] = 0.0;
        J[7] = 2.0 * k2 * x[1];
        J[8] = 0.0;
    }
};

// BASELINE cfg 1/3 (sigma, rho, beta); same tree as oracle/odescan_oracle.c
struct Lorenz63 {
    static constexpr int D = 3;
    double sigma, rho, beta;
    __device__ __forceinline__ explicit Lorenz63(const ProbParams& q)
        : sigma(q.p[0]), rho(q.p[1]), beta(q.p[2]) {}
    __device__ __forceinline__ void f(const double* x, double* o) const {
        o[0] = sigma * (x[1] - x[0]);
        o[1] = x[0] * (rho - x[2]) - x[1];
        o[2] = x[0] * x[1] - beta * x[2];
    }
    __device__ __forceinline__ void jac(const double* x, double* J) const {
        J[0] = -sigma; J[1] = sigma; J[2] = 0.0;
        J[3] = rho - x[2]; J[4] = -1.0; J[5] = -x[0];
        J[6] = x[1]; J[7] = x[0]; J[8] = -beta;
    }
};

// tests/test_newton_pint.py:28-46
struct ExpGrowth {
    static constexpr int D = 1;
    __device__ __forceinline__ explicit ExpGrowth(const ProbParams&) {}
    __device__ __forceinline__ void f(const double* x, double* o) const { o[0] = exp(x[0]); }
    __device__ __forceinline__ void jac(const double* x, double* J) const { J[0] = exp(x[0]); }
};

// tests/test_newton_pint.py:49-68
struct Square {
    static constexpr int D = 1;
    __device__ __forceinline__ explicit Square(const ProbParams&) {}
    __device__ __forceinline__ void f(const double* x, double* o) const { o[0] = x[0] * x[0]; }
    __device__ __forceinline__ void jac(const double* x, double* J) const { J[0] = 2.0 * x[0]; }
};

// dx/dt = A x, A row-major in params (affine-system checks, crit 8)
template <int DD>
struct Linear {
    static constexpr int D = DD;
    double A[DD * DD];
    __device__ __forceinline__ explicit Linear(const ProbParams& q) {
#pragma unroll
        for (int i = 0; i < DD * DD; i++) A[i] = q.p[i];
    }
    __device__ __forceinline__ void f(const double* x, double* o) const {
#pragma unroll
        for (int r = 0; r < DD; r++) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < DD; q++) acc += A[r * DD + q] * x[q];
            o[r] = acc;
        }
    }
    __device__ __forceinline__ void jac(const double*, double* J) const {
#pragma unroll
        for (int i = 0; i < DD * DD; i++) J[i] = A[i];
    }
};

}  // namespace odx
