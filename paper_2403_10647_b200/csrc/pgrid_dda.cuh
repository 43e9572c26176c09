// Grid consumer: Moller-Trumbore + 3-D DDA ray casting over a built
// grid, bit-exact against the reference's compiled lane (kernels/_ckernels.pyx:112-260).
//
// Exactness: the reference is Cython compiled by gcc for x86-64 (SSE2 doubles, no FMA, every
// product and sum rounded on its own, sums associated left to right). Every arithmetic step
// below is written with an explicit round-to-nearest intrinsic (__dmul_rn / __dadd_rn /
// __dsub_rn / __ddiv_rn) so nvcc cannot contract a multiply-add into an FMA, and the double ->
// int64 cast emulates x86 cvttsd2si (np_floor_i64). Comparison chains and their NaN behaviour
// follow the C source statement by statement.
#pragma once

#include <math_constants.h>

namespace pgrid {

constexpr double kBaryEps = 1e-9;  // pykernels.py:16 / _ckernels.pyx:16
constexpr double kDetEps = 1e-12;  // pykernels.py:17
constexpr double kTEps = 1e-9;     // pykernels.py:18

// Prepared triangle: v0, e1 = v1 - v0, e2 = v2 - v0 (exactly the reference's first six
// subtractions, done once per triangle instead of once per test), padded to 80 bytes so a
// test is five 16-byte loads of one contiguous record.
struct __align__(16) TriRec {
  double v0x, v0y, v0z, e1x, e1y, e1z, e2x, e2y, e2z, pad;
};

__global__ void __launch_bounds__(256)
k_dda_prepare(const double* __restrict__ V, long long nv, const int* __restrict__ T, long long n,
              TriRec* __restrict__ out, unsigned* __restrict__ err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = __ldg(T + 3 * i), b = __ldg(T + 3 * i + 1), c = __ldg(T + 3 * i + 2);
  TriRec r;
  if (a < 0 || b < 0 || c < 0 || a >= nv || b >= nv || c >= nv) {
    atomicOr(err, 2u);  // geometry.py:41-43 (TriangleMesh rejects out-of-range indices)
    r = TriRec{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  } else {
    const double* p0 = V + 3 * (long long)a;
    const double* p1 = V + 3 * (long long)b;
    const double* p2 = V + 3 * (long long)c;
    const double x0 = __ldg(p0), y0 = __ldg(p0 + 1), z0 = __ldg(p0 + 2);
    r.v0x = x0;
    r.v0y = y0;
    r.v0z = z0;
    r.e1x = __dsub_rn(__ldg(p1), x0);
    r.e1y = __dsub_rn(__ldg(p1 + 1), y0);
    r.e1z = __dsub_rn(__ldg(p1 + 2), z0);
    r.e2x = __dsub_rn(__ldg(p2), x0);
    r.e2y = __dsub_rn(__ldg(p2 + 1), y0);
    r.e2z = __dsub_rn(__ldg(p2 + 2), z0);
    r.pad = 0.0;
  }
  out[i] = r;
}

// _ckernels.pyx:112-143 (_ray_tri): returns t >= 0 or -1.0 on a miss.
__device__ __forceinline__ double ray_tri(double ox, double oy, double oz, double dx, double dy, double dz,
                                          const TriRec* __restrict__ tr) {
  const double2* q2 = reinterpret_cast<const double2*>(tr);
  const double2 a = __ldg(q2), b = __ldg(q2 + 1), c = __ldg(q2 + 2), d = __ldg(q2 + 3), e = __ldg(q2 + 4);
  const double v0x = a.x, v0y = a.y, v0z = b.x, e1x = b.y, e1y = c.x, e1z = c.y, e2x = d.x, e2y = d.y, e2z = e.x;
  const double px = __dsub_rn(__dmul_rn(dy, e2z), __dmul_rn(dz, e2y));
  const double py = __dsub_rn(__dmul_rn(dz, e2x), __dmul_rn(dx, e2z));
  const double pz = __dsub_rn(__dmul_rn(dx, e2y), __dmul_rn(dy, e2x));
  const double det = __dadd_rn(__dadd_rn(__dmul_rn(e1x, px), __dmul_rn(e1y, py)), __dmul_rn(e1z, pz));
  if (-kDetEps < det && det < kDetEps) return -1.0;
  const double inv = __ddiv_rn(1.0, det);
  const double tx = __dsub_rn(ox, v0x), ty = __dsub_rn(oy, v0y), tz = __dsub_rn(oz, v0z);
  const double u = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(tx, px), __dmul_rn(ty, py)), __dmul_rn(tz, pz)), inv);
  if (u < -kBaryEps || u > 1.0 + kBaryEps) return -1.0;
  const double qx = __dsub_rn(__dmul_rn(ty, e1z), __dmul_rn(tz, e1y));
  const double qy = __dsub_rn(__dmul_rn(tz, e1x), __dmul_rn(tx, e1z));
  const double qz = __dsub_rn(__dmul_rn(tx, e1y), __dmul_rn(ty, e1x));
  const double v = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, qx), __dmul_rn(dy, qy)), __dmul_rn(dz, qz)), inv);
  if (v < -kBaryEps || __dadd_rn(u, v) > 1.0 + kBaryEps) return -1.0;
  const double t = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz)), inv);
  if (t < -kTEps) return -1.0;
  return t > 0.0 ? t : 0.0;
}

#ifndef DDA_MIN_CTAS
#define DDA_MIN_CTAS 6  // 80 registers: 24 warps per SM (measured best of 4, 6, 8) to hide the dependent G -> O -> triangle loads
#endif

struct DdaGrid {
  double lo[3], hi[3], cs[3];
  long long nd[3];
  long long ntri;
};

// _ckernels.pyx:146-260, one thread per ray. The traversal of a ray whose loop never ends
// in the reference (zero / NaN direction with an unbounded segment) is cut after
// sum(dims) + 3 cells; every terminating ray visits fewer cells than that.
__global__ void __launch_bounds__(128, DDA_MIN_CTAS)
k_dda_cast(const unsigned* __restrict__ G, const unsigned* __restrict__ O, const TriRec* __restrict__ tris,
           DdaGrid gs, const double* __restrict__ orig, const double* __restrict__ dirv,
           const double* __restrict__ tmax, long long nrays, long long* __restrict__ ids, double* __restrict__ ts,
           unsigned* __restrict__ err) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrays) return;
  const double o[3] = {__ldg(orig + 3 * r), __ldg(orig + 3 * r + 1), __ldg(orig + 3 * r + 2)};
  const double d[3] = {__ldg(dirv + 3 * r), __ldg(dirv + 3 * r + 1), __ldg(dirv + 3 * r + 2)};
  const double tm = __ldg(tmax + r);
  long long best_id = -1;
  double best_t = CUDART_INF;
  double t0 = 0.0, t1 = tm;
  bool miss = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (d[k] != 0.0) {
      double ta = __ddiv_rn(__dsub_rn(gs.lo[k], o[k]), d[k]);
      double tb = __ddiv_rn(__dsub_rn(gs.hi[k], o[k]), d[k]);
      if (ta > tb) {
        const double x = ta;
        ta = tb;
        tb = x;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    } else if (o[k] < gs.lo[k] || o[k] > gs.hi[k]) {
      miss = true;
    }
  }
  if (!(miss || t0 > t1)) {
    long long cell[3];
    int step[3];
    double tnext[3], tdelta[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double p = __dadd_rn(o[k], __dmul_rn(d[k], t0));
      long long cc = np_floor_i64(__ddiv_rn(__dsub_rn(p, gs.lo[k]), gs.cs[k]));
      if (cc < 0) cc = 0;
      if (cc > gs.nd[k] - 1) cc = gs.nd[k] - 1;
      cell[k] = cc;
      if (d[k] > 0.0) {
        step[k] = 1;
        tnext[k] = __ddiv_rn(__dsub_rn(__dadd_rn(gs.lo[k], __dmul_rn((double)(cc + 1), gs.cs[k])), o[k]), d[k]);
        tdelta[k] = __ddiv_rn(gs.cs[k], d[k]);
      } else if (d[k] < 0.0) {
        step[k] = -1;
        tnext[k] = __ddiv_rn(__dsub_rn(__dadd_rn(gs.lo[k], __dmul_rn((double)cc, gs.cs[k])), o[k]), d[k]);
        tdelta[k] = __ddiv_rn(-gs.cs[k], d[k]);
      } else {
        step[k] = 0;
        tnext[k] = CUDART_INF;
        tdelta[k] = CUDART_INF;
      }
    }
    double t_entry = t0;
    const long long cap = gs.nd[0] + gs.nd[1] + gs.nd[2] + 3;
    const long long stride[3] = {1, gs.nd[0], gs.nd[0] * gs.nd[1]};
    long long cid = cell[0] + gs.nd[0] * (cell[1] + gs.nd[1] * cell[2]);
    unsigned s0 = __ldg(G + cid), s1 = __ldg(G + cid + 1);
    for (long long it = 0; it < cap; ++it) {
      double t_exit = tnext[0];
      if (tnext[1] < t_exit) t_exit = tnext[1];
      if (tnext[2] < t_exit) t_exit = tnext[2];
      // the step taken after this cell depends on tnext only: choose it now and fetch the
      // next cell's G range while this cell's candidates are tested
      int axis;
      if (tnext[0] <= tnext[1] && tnext[0] <= tnext[2])
        axis = 0;
      else if (tnext[1] <= tnext[2])
        axis = 1;
      else
        axis = 2;
      const int stp = axis == 0 ? step[0] : axis == 1 ? step[1] : step[2];
      const long long nc = (axis == 0 ? cell[0] : axis == 1 ? cell[1] : cell[2]) + stp;
      const long long lim = axis == 0 ? gs.nd[0] : axis == 1 ? gs.nd[1] : gs.nd[2];
      const bool inside = nc >= 0 && nc < lim;
      const long long ncid = cid + (long long)stp * (axis == 0 ? stride[0] : axis == 1 ? stride[1] : stride[2]);
      unsigned n0 = 0, n1 = 0;
      if (inside) {
        n0 = __ldg(G + ncid);
        n1 = __ldg(G + ncid + 1);
      }
      const double lo_t = __dsub_rn(t_entry, kTEps), hi_t = __dadd_rn(t_exit, kTEps);
      for (unsigned slot = s0; slot < s1; ++slot) {
        const unsigned tri = __ldg(O + slot);
        if ((long long)tri >= gs.ntri) {
          atomicOr(err, 4u);  // O does not belong to this mesh
          continue;
        }
        const double t = ray_tri(o[0], o[1], o[2], d[0], d[1], d[2], tris + tri);
        if (t < 0.0 || t > tm) continue;
        if (t < lo_t || t > hi_t) continue;
        if (t < __dsub_rn(best_t, kTEps) ||
            ((__dsub_rn(t, best_t) <= kTEps && __dsub_rn(best_t, t) <= kTEps) &&
             (best_id < 0 || (long long)(int)tri < best_id))) {
          best_t = t;
          best_id = (int)tri;
        }
      }
      if (best_id >= 0 && t_exit > __dadd_rn(best_t, kTEps)) break;
      if (!inside) break;
      if (axis == 0) cell[0] = nc; else if (axis == 1) cell[1] = nc; else cell[2] = nc;
      cid = ncid;
      t_entry = t_exit;
      if (axis == 0) tnext[0] = __dadd_rn(tnext[0], tdelta[0]);
      else if (axis == 1) tnext[1] = __dadd_rn(tnext[1], tdelta[1]);
      else tnext[2] = __dadd_rn(tnext[2], tdelta[2]);
      if (t_entry > __dadd_rn(t1, kTEps)) break;
      s0 = n0;
      s1 = n1;
    }
  }
  ids[r] = best_id;
  ts[r] = best_id >= 0 ? best_t : CUDART_INF;
}

}  // namespace pgrid
