// dispatch.cuh — runtime (shape, form, unit-weight, division mode) to
// compile-time kernel template arguments.
#pragma once
#include "common.cuh"

namespace sl {

struct KernelKey {
  int shape;  // sl::Shape (Q1 resolved)
  int form;   // 0 = R, 1 = D
  bool unit;  // all compact weights == -1
  int div;    // DivMode
};

template <int S, int F, bool U, typename Fn>
cudaError_t dispatch_div(int div, Fn &&fn) {
  if (div == DIV_POW2) return fn.template operator()<S, F, U, DIV_POW2>();
  if (div == DIV_RCP) return fn.template operator()<S, F, U, DIV_RCP>();
  return fn.template operator()<S, F, U, DIV_IEEE>();
}

template <int S, int F, typename Fn>
cudaError_t dispatch_unit(bool unit, int div, Fn &&fn) {
  return unit ? dispatch_div<S, F, true>(div, fn) : dispatch_div<S, F, false>(div, fn);
}

template <int S, typename Fn>
cudaError_t dispatch_form(int form, bool unit, int div, Fn &&fn) {
  return form == 1 ? dispatch_unit<S, 1>(unit, div, fn) : dispatch_unit<S, 0>(unit, div, fn);
}

// fn is a lambda template: []<int S, int F, bool U, int D>() -> cudaError_t
template <typename Fn>
cudaError_t dispatch(const KernelKey &k, Fn &&fn) {
  switch (k.shape) {
    case FD5: return dispatch_form<FD5>(k.form, k.unit, k.div, fn);
    case FE9: return dispatch_form<FE9>(k.form, k.unit, k.div, fn);
    case FD7: return dispatch_form<FD7>(k.form, k.unit, k.div, fn);
    case FE27: return dispatch_form<FE27>(k.form, k.unit, k.div, fn);
    case Q1: return dispatch_form<Q1>(k.form, k.unit, k.div, fn);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sl
