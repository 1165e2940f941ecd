// cko_dual.cuh — forward-mode dual numbers on the device.
//
// The device twin of the reference's Dual<W> (dual.hpp:15-186): a value and W
// tangent lanes, the same propagation rules and the same fixed subgradients at
// kinks (d|x|/dx = 0 at 0, the positive-part ramp has derivative 0 for
// x <= 0), and pow through the shared pow_value so every derivative strategy
// sees the same value arithmetic. With W = 8 one model evaluation yields eight
// Jacobian columns or eight parameter sensitivities
// (ModelBase::jacobian_forward_ad / param_vjp_forward_ad, ode_model.hpp:132-182).
#pragma once

#include "cko_models.cuh"

namespace cko {

// keep the double overloads visible next to the dual ones declared below
using ::cos;
using ::fabs;
using ::log;
using ::sin;
using ::tanh;

template <int W>
struct Dual {
  double v;
  double d[W];
  __device__ Dual() : v(0.0) {
#pragma unroll
    for (int l = 0; l < W; ++l) d[l] = 0.0;
  }
  __device__ Dual(double x) : v(x) {  // NOLINT: implicit like the reference
#pragma unroll
    for (int l = 0; l < W; ++l) d[l] = 0.0;
  }
  __device__ Dual& operator+=(const Dual& o) {
    v += o.v;
#pragma unroll
    for (int l = 0; l < W; ++l) d[l] += o.d[l];
    return *this;
  }
  __device__ Dual& operator-=(const Dual& o) {
    v -= o.v;
#pragma unroll
    for (int l = 0; l < W; ++l) d[l] -= o.d[l];
    return *this;
  }
};

template <int W>
__device__ inline Dual<W> operator+(Dual<W> a, const Dual<W>& b) { return a += b; }
template <int W>
__device__ inline Dual<W> operator-(Dual<W> a, const Dual<W>& b) { return a -= b; }
template <int W>
__device__ inline Dual<W> operator-(const Dual<W>& a) {
  Dual<W> r;
  r.v = -a.v;
#pragma unroll
  for (int l = 0; l < W; ++l) r.d[l] = -a.d[l];
  return r;
}
template <int W>
__device__ inline Dual<W> operator*(const Dual<W>& a, const Dual<W>& b) {
  Dual<W> r;
  r.v = xmul(a.v, b.v);
#pragma unroll
  for (int l = 0; l < W; ++l) r.d[l] = xadd(xmul(a.d[l], b.v), xmul(a.v, b.d[l]));
  return r;
}
template <int W>
__device__ inline Dual<W> operator/(const Dual<W>& a, const Dual<W>& b) {
  Dual<W> r;
  const double inv = 1.0 / b.v;
  r.v = xmul(a.v, inv);
#pragma unroll
  for (int l = 0; l < W; ++l) r.d[l] = xmul(xsub(a.d[l], xmul(r.v, b.d[l])), inv);
  return r;
}
template <int W>
__device__ inline Dual<W> operator+(Dual<W> a, double b) {
  a.v += b;
  return a;
}
template <int W>
__device__ inline Dual<W> operator+(double a, Dual<W> b) {
  b.v = a + b.v;
  return b;
}
template <int W>
__device__ inline Dual<W> operator-(Dual<W> a, double b) {
  a.v -= b;
  return a;
}
template <int W>
__device__ inline Dual<W> operator-(double a, const Dual<W>& b) { return -b + a; }
template <int W>
__device__ inline Dual<W> operator*(Dual<W> a, double b) {
  a.v = xmul(a.v, b);
#pragma unroll
  for (int l = 0; l < W; ++l) a.d[l] = xmul(a.d[l], b);
  return a;
}
template <int W>
__device__ inline Dual<W> operator*(double a, const Dual<W>& b) { return b * a; }
template <int W>
__device__ inline Dual<W> operator/(const Dual<W>& a, double b) { return a * (1.0 / b); }
template <int W>
__device__ inline Dual<W> operator/(double a, const Dual<W>& b) { return Dual<W>(a) / b; }
template <int W>
__device__ inline bool operator>(const Dual<W>& a, double b) { return a.v > b; }
template <int W>
__device__ inline bool operator<(const Dual<W>& a, double b) { return a.v < b; }

template <int W>
__device__ inline Dual<W> chain(double value, double dcoef, const Dual<W>& x) {
  Dual<W> r;
  r.v = value;
#pragma unroll
  for (int l = 0; l < W; ++l) r.d[l] = xmul(dcoef, x.d[l]);
  return r;
}
template <int W>
__device__ inline Dual<W> sin(const Dual<W>& x) { return chain(::sin(x.v), ::cos(x.v), x); }
template <int W>
__device__ inline Dual<W> cos(const Dual<W>& x) { return chain(::cos(x.v), -::sin(x.v), x); }
template <int W>
__device__ inline Dual<W> tanh(const Dual<W>& x) {
  const double t = ::tanh(x.v);
  return chain(t, 1.0 - t * t, x);
}
template <int W>
__device__ inline Dual<W> fabs(const Dual<W>& x) {
  const double s = x.v > 0.0 ? 1.0 : (x.v < 0.0 ? -1.0 : 0.0);
  return chain(::fabs(x.v), s, x);
}
template <int W>
__device__ inline Dual<W> positive_part(const Dual<W>& x) {
  return x.v > 0.0 ? x : Dual<W>(0.0);
}
__device__ inline double positive_part(double x) { return x > 0.0 ? x : 0.0; }
template <int W>
__device__ inline double sign_of(const Dual<W>& x) { return x.v > 0.0 ? 1.0 : (x.v < 0.0 ? -1.0 : 0.0); }
template <int W>
__device__ inline Dual<W> pow(const Dual<W>& b, const Dual<W>& e) {
  const double value = pow_value(b.v, e.v);
  const double db = (b.v != 0.0) ? e.v * pow_value(b.v, e.v - 1.0) : 0.0;
  const double de = (b.v > 0.0) ? value * ::log(b.v) : 0.0;
  Dual<W> r;
  r.v = value;
#pragma unroll
  for (int l = 0; l < W; ++l) r.d[l] = xadd(xmul(db, b.d[l]), xmul(de, e.d[l]));
  return r;
}
__device__ inline double pow(double b, double e) { return pow_value(b, e); }
__device__ inline double value_of(double x) { return x; }
template <int W>
__device__ inline double value_of(const Dual<W>& x) { return x.v; }

// A double whose every operation rounds separately (no FMA contraction): the
// plain-value instantiation of the templated evaluations, so the device's
// finite-difference Jacobian and the rate built from them follow the
// reference's (uncontracted) arithmetic.
struct Exact {
  double v;
  __device__ Exact() : v(0.0) {}
  __device__ Exact(double x) : v(x) {}  // NOLINT: implicit like a double
  __device__ Exact& operator+=(const Exact& o) { v = xadd(v, o.v); return *this; }
  __device__ Exact& operator-=(const Exact& o) { v = xsub(v, o.v); return *this; }
};
__device__ inline Exact operator+(Exact a, Exact b) { return Exact(xadd(a.v, b.v)); }
__device__ inline Exact operator-(Exact a, Exact b) { return Exact(xsub(a.v, b.v)); }
__device__ inline Exact operator-(Exact a) { return Exact(-a.v); }
__device__ inline Exact operator*(Exact a, Exact b) { return Exact(xmul(a.v, b.v)); }
__device__ inline Exact operator/(Exact a, Exact b) { return Exact(a.v / b.v); }
__device__ inline Exact operator+(Exact a, double b) { return Exact(xadd(a.v, b)); }
__device__ inline Exact operator+(double a, Exact b) { return Exact(xadd(a, b.v)); }
__device__ inline Exact operator-(Exact a, double b) { return Exact(xsub(a.v, b)); }
__device__ inline Exact operator-(double a, Exact b) { return Exact(xsub(a, b.v)); }
__device__ inline Exact operator*(Exact a, double b) { return Exact(xmul(a.v, b)); }
__device__ inline Exact operator*(double a, Exact b) { return Exact(xmul(a, b.v)); }
__device__ inline Exact operator/(Exact a, double b) { return Exact(a.v / b); }
__device__ inline Exact operator/(double a, Exact b) { return Exact(a / b.v); }
__device__ inline bool operator>(Exact a, double b) { return a.v > b; }
__device__ inline bool operator<(Exact a, double b) { return a.v < b; }
__device__ inline Exact sin(Exact x) { return Exact(::sin(x.v)); }
__device__ inline Exact cos(Exact x) { return Exact(::cos(x.v)); }
__device__ inline Exact tanh(Exact x) { return Exact(::tanh(x.v)); }
__device__ inline Exact fabs(Exact x) { return Exact(::fabs(x.v)); }
__device__ inline Exact positive_part(Exact x) { return x.v > 0.0 ? x : Exact(0.0); }
__device__ inline double sign_of(Exact x) { return x.v > 0.0 ? 1.0 : (x.v < 0.0 ? -1.0 : 0.0); }
__device__ inline Exact pow(Exact b, Exact e) { return Exact(pow_value(b.v, e.v)); }
__device__ inline double value_of(Exact x) { return x.v; }
struct ParamExact {
  const double* p;
  __device__ Exact operator()(int j) const { return Exact(p[j]); }
};

using Dual8 = Dual<8>;
constexpr int kFadMaxN = 32;  // state sizes the forward-mode device paths hold per thread

// Parameter views for the templated model evaluations: plain values, or values
// with unit tangents seeded on a window of parameters [j0, j0 + lanes).
struct ParamPlain {
  const double* p;
  __device__ double operator()(int j) const { return p[j]; }
};
template <int W>
struct ParamSeeded {
  const double* p;
  int j0, lanes;
  __device__ Dual<W> operator()(int j) const {
    Dual<W> r(p[j]);
    const int l = j - j0;
    if (l >= 0 && l < lanes) r.d[l] = 1.0;
    return r;
  }
};
template <int W>
struct ParamAsDual {
  const double* p;
  __device__ Dual<W> operator()(int j) const { return Dual<W>(p[j]); }
};

}  // namespace cko
