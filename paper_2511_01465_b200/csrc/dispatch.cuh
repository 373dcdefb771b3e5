// dispatch.cuh — problem-id -> functor-type dispatch for the small-d paths.
#pragma once

#include "problems.cuh"

namespace odx {

// Every small-d problem with a compiled device path (d <= 4).
#define ODX_FOR_EACH_SMALL_PROBLEM(X) \
    X(Logistic)                       \
    X(VanDerPol)                      \
    X(CartPole)                       \
    X(CartPoleSq)                     \
    X(Dahlquist)                      \
    X(Robertson)                      \
    X(Lorenz63)                       \
    X(ExpGrowth)                      \
    X(Square)                         \
    X(Linear<1>)                      \
    X(Linear<2>)                      \
    X(Linear<3>)                      \
    X(Linear<4>)

// Calls fn.template operator()<P>() for the functor type selected by
// (problem_id, dim); returns ODX_EUNSUPPORTED when there is none.
template <class Fn>
int with_small_problem(int problem_id, int dim, Fn&& fn) {
    switch (problem_id) {
    case ODX_PROB_LOGISTIC: return dim == 1 ? fn.template operator()<Logistic>() : ODX_EINVAL;
    case ODX_PROB_VDP: return dim == 2 ? fn.template operator()<VanDerPol>() : ODX_EINVAL;
    case ODX_PROB_CARTPOLE: return dim == 4 ? fn.template operator()<CartPole>() : ODX_EINVAL;
    case ODX_PROB_CARTPOLE_SQ: return dim == 4 ? fn.template operator()<CartPoleSq>() : ODX_EINVAL;
    case ODX_PROB_DAHLQUIST: return dim == 1 ? fn.template operator()<Dahlquist>() : ODX_EINVAL;
    case ODX_PROB_ROBERTSON: return dim == 3 ? fn.template operator()<Robertson>() : ODX_EINVAL;
    case ODX_PROB_LORENZ63: return dim == 3 ? fn.template operator()<Lorenz63>() : ODX_EINVAL;
    case ODX_PROB_EXP_GROWTH: return dim == 1 ? fn.template operator()<ExpGrowth>() : ODX_EINVAL;
    case ODX_PROB_SQUARE: return dim == 1 ? fn.template operator()<Square>() : ODX_EINVAL;
    case ODX_PROB_LINEAR:
        switch (dim) {
        case 1: return fn.template operator()<Linear<1>>();
        case 2: return fn.template operator()<Linear<2>>();
        case 3: return fn.template operator()<Linear<3>>();
        case 4: return fn.template operator()<Linear<4>>();
        default: return ODX_EUNSUPPORTED;
        }
    default: return ODX_EUNSUPPORTED;
    }
}

}  // namespace odx
