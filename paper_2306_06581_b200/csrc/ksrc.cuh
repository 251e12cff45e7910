// ksrc.cuh -- device views of the Gibbs kernel and its cost (dense or
// recomputed from coordinates exactly as pairwise_cost + the caller's
// normalisation + kernel_from_cost, proj/src/geometry.cpp:16-102).
#pragma once

#include "common.cuh"
#include "internal.h"

namespace spk {

__device__ __forceinline__ double coord_cost(const double* p, const double* q, int dim, int kind, double eta) {
  if (kind == SPK_COST_SQEUCLID) return cost_entry<0>(p, q, dim, eta);
  if (kind == SPK_COST_EUCLID) return cost_entry<1>(p, q, dim, eta);
  return cost_entry<2>(p, q, dim, eta);
}

struct KCoords {
  const double* x;
  const double* y;
  int64_t n;
  int dim, kind;
  double eta, scale, eps;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    const double c = coord_cost(x + i * dim, y + j * dim, dim, kind, eta) / scale;
    return isinf(c) ? 0.0 : exp_ref(-c / eps);
  }
};

struct KDense {
  const double* K;
  int64_t n;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const { return K[i * n + j]; }
};

struct CostSrc {
  const double* C;  // dense n*n or nullptr
  const double* x;
  const double* y;
  int64_t n;
  int dim, kind;
  double eta, scale;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    if (C) return C[i * n + j];
    return coord_cost(x + i * dim, y + j * dim, dim, kind, eta) / scale;
  }
};

inline KCoords kcoords_of(const DevKernel& dk) {
  return KCoords{dk.x.as<double>(), dk.y.as<double>(), dk.n, dk.dim, dk.kind, dk.eta, dk.scale, dk.eps};
}

inline CostSrc cost_src_of(const DevKernel* dk) {
  CostSrc c{};
  if (!dk) return c;
  c.C = dk->dense ? dk->C.as<double>() : nullptr;
  c.x = dk->x.as<double>();
  c.y = dk->y.as<double>();
  c.n = dk->n;
  c.dim = dk->dim;
  c.kind = dk->kind;
  c.eta = dk->eta;
  c.scale = dk->scale;
  return c;
}

}  // namespace spk
