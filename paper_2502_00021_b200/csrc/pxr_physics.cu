// Planar articulated-body dynamics, resets and forward kinematics on the
// device -- SURVEY.md 8(f) row 1 ("GPU physics + FK + reset"), so that the
// reference's Env.step() runs without a host round trip.
//
// f64, mirroring the reference's numba kernels operation by operation (all
// under /root/reference/pkg/src/pixelctrl/), as one thread per env (large
// batches) or 32 / 16 / 8 lanes per env (the latency-bound smaller batches;
// same arithmetic per element, bit-identical results):
//   _kinematics_pass  physics.py:144-163
//   _rnea             physics.py:166-238
//   _solve_spd        physics.py:241-269
//   _step_batch       physics.py:272-420 (contacts, limits, RNEA bias +
//                     mass matrix, Cholesky, semi-implicit Euler, guard)
//   compute_reward    physics.py:468-477
//   reset_state / Env._reset_rows  physics.py:487-510, env.py:142-153
// Every operation rounds as the reference's does (-fmad=false, same order)
// and the f64 sin / cos are glibc's, restated (pxr_glibc_sincos.cuh), so
// dynamics, rewards, FK and the reset qpos draws are bit-identical to the
// reference (tests/test_env_gpu.py, test_physics_api.py; the recorded
// reference rollouts reproduce in full, tests/test_recorder.py). The log of
// the reset qvel Box-Muller draw (prng.py:138-152) is numpy's AVX-512 SVML
// log, restated in pxr_numpy_log.cuh.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"
#include "pxr_glibc_sincos.cuh"
#include "pxr_numpy_log.cuh"
#include "pxr_math.cuh"

namespace pxr {

constexpr int kMaxL = 16;  // links (dof <= 18)
constexpr int kMaxD = kMaxL + 2;

constexpr double GRAVITY = 9.81;
constexpr double CONTACT_SPRING = 4000.0;
constexpr double CONTACT_DAMPING = 40.0;
constexpr double FRICTION_GAIN = 40.0;
constexpr double FRICTION_MU = 0.8;
constexpr double LIMIT_SPRING = 300.0;
constexpr double LIMIT_DAMPING = 2.0;
constexpr double JOINT_DAMPING = 0.1;
constexpr double VEL_CLAMP = 100.0;
constexpr double DIVERGED = 1e8;

struct Model {
  const int32_t *parent;
  const double *adist, *length, *mass, *inertia;
  const double *limit_lo, *limit_hi, *torque_max;
  int nl;
};

// physics.py:166-238 (with the kinematics pass of 144-163 folded in). The
// link angles depend on q only, so their cos / sin (ct, st) are computed once
// per substep by the caller -- the same values the reference recomputes in
// every pass.
__device__ void rnea(const Model &m, const double *q, const double *qd, const double *qdd,
                     const double *ct, const double *st, double grav, const double *fex,
                     const double *fez, const double *tex, bool use_ext, double *out) {
  double omega[kMaxL], alpha[kMaxL], ox[kMaxL], oz[kMaxL], vox[kMaxL],
      voz[kMaxL], aox[kMaxL], aoz[kMaxL], fx[kMaxL], fz[kMaxL], nq[kMaxL];
  const int nl = m.nl;
  omega[0] = qd[2]; alpha[0] = qdd[2];
  ox[0] = q[0]; oz[0] = q[1];
  vox[0] = qd[0]; voz[0] = qd[1];
  aox[0] = qdd[0]; aoz[0] = qdd[1];
  for (int i = 1; i < nl; i++) {
    const int p = m.parent[i];
    const double c = ct[p], s = st[p];
    const double a = m.adist[i];
    ox[i] = ox[p] + a * c;
    oz[i] = oz[p] + a * s;
    vox[i] = vox[p] + omega[p] * a * (-s);
    voz[i] = voz[p] + omega[p] * a * c;
    aox[i] = aox[p] + alpha[p] * a * (-s) - omega[p] * omega[p] * a * c;
    aoz[i] = aoz[p] + alpha[p] * a * c - omega[p] * omega[p] * a * s;
    omega[i] = omega[p] + qd[3 + i - 1];
    alpha[i] = alpha[p] + qdd[3 + i - 1];
  }
  for (int i = 0; i < nl; i++) fx[i] = fz[i] = nq[i] = 0.0;
  for (int i = nl - 1; i >= 0; i--) {
    const double h = 0.5 * m.length[i];
    const double c = ct[i], s = st[i];
    const double acx = aox[i] + alpha[i] * h * (-s) - omega[i] * omega[i] * h * c;
    const double acz = aoz[i] + alpha[i] * h * c - omega[i] * omega[i] * h * s;
    const double gfx = m.mass[i] * acx;
    const double gfz = m.mass[i] * (acz + grav);
    fx[i] += gfx;
    fz[i] += gfz;
    nq[i] += m.inertia[i] * alpha[i] + (h * c) * gfz - (h * s) * gfx;
    if (use_ext) {
      fx[i] -= fex[i];
      fz[i] -= fez[i];
      nq[i] -= tex[i];
    }
    const int p = m.parent[i];
    if (p >= 0) {
      const double cp = ct[p], sp = st[p];
      const double rx = m.adist[i] * cp, rz = m.adist[i] * sp;
      fx[p] += fx[i];
      fz[p] += fz[i];
      nq[p] += nq[i] + rx * fz[i] - rz * fx[i];
    }
  }
  out[0] = fx[0];
  out[1] = fz[0];
  out[2] = nq[0];
  for (int i = 1; i < nl; i++) out[2 + i] = nq[i];
}

// physics.py:241-269, M row-major nd x nd
__device__ void solve_spd(double *M, const double *rhs, double *x, int active0, int n, int ld) {
  for (int i = active0; i < n; i++) {
    for (int j = active0; j <= i; j++) {
      double acc = M[i * ld + j];
      for (int t = active0; t < j; t++) acc -= M[i * ld + t] * M[j * ld + t];
      if (i == j) {
        if (acc < 1e-12) acc = 1e-12;
        M[i * ld + i] = sqrt(acc);
      } else {
        M[i * ld + j] = acc / M[j * ld + j];
      }
    }
  }
  for (int i = 0; i < active0; i++) x[i] = 0.0;
  for (int i = active0; i < n; i++) {
    double acc = rhs[i];
    for (int t = active0; t < i; t++) acc -= M[i * ld + t] * x[t];
    x[i] = acc / M[i * ld + i];
  }
  for (int i = n - 1; i >= active0; i--) {
    double acc = x[i];
    for (int t = i + 1; t < n; t++) acc -= M[t * ld + i] * x[t];
    x[i] = acc / M[i * ld + i];
  }
}

struct StepArgs {
  Model m;
  double *qpos, *qvel;
  int64_t *step_count;
  uint8_t *done;
  const double *actions;
  double *reward;  // accumulated (+=) per control step
  int64_t batch;
  int substeps, fixed_root, has_min_h;
  double h, dt, min_h, forward_weight, ctrl_cost;
  int64_t ep_len;
};

// numpy's pairwise sum (the order np.sum uses for a contiguous row of < 8
// or up to 128 elements): 8 running partials, then a fixed tree.
__device__ double np_sum(const double *v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; i++) r += v[i];
    return r;
  }
  double r[8];
  for (int k = 0; k < 8; k++) r[k] = v[k];
  int i = 8;
  for (; i + 8 <= n; i += 8)
    for (int k = 0; k < 8; k++) r[k] += v[i + k];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += v[i];
  return res;
}

__global__ void physics_step_kernel(StepArgs a) {
  const Model &m = a.m;
  const int nl = m.nl, nd = nl + 2, nj = nd - 3;
  const int active0 = a.fixed_root ? 3 : 0;
  PXR_DCHECK(nl >= 1 && nl <= kMaxL && nd <= kMaxD && m.parent[0] < 0);
#ifdef PXR_CHECKED
  for (int i = 1; i < nl; i++) PXR_DCHECK(m.parent[i] >= 0 && m.parent[i] < i);
#endif
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < a.batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    double qb[kMaxD], qdb[kMaxD], q0[kMaxD], tau[kMaxD], bias[kMaxD], col[kMaxD], rhs[kMaxD],
        qdd[kMaxD], zeros[kMaxD], unit[kMaxD];
    double M[kMaxD * kMaxD];
    double fex[kMaxL], fez[kMaxL], tex[kMaxL];
    double *q = a.qpos + b * nd, *qd = a.qvel + b * nd;
    const double *act = a.actions + b * nj;
    for (int d = 0; d < nd; d++) {
      qb[d] = q[d];
      qdb[d] = qd[d];
      q0[d] = q[d];
      zeros[d] = 0.0;
      unit[d] = 0.0;
    }
    const double x_before = q[0];
    for (int sub = 0; sub < a.substeps; sub++) {
      // kinematics pass (physics.py:144-163)
      double theta[kMaxL], ct[kMaxL], st[kMaxL], omega[kMaxL], ox[kMaxL], oz[kMaxL],
          vox[kMaxL], voz[kMaxL];
      theta[0] = qb[2];
      for (int i = 1; i < nl; i++) theta[i] = theta[m.parent[i]] + qb[3 + i - 1];
      for (int i = 0; i < nl; i++) {
        ct[i] = glibc_cos(theta[i]);
        st[i] = glibc_sin(theta[i]);
      }
      omega[0] = qdb[2];
      ox[0] = qb[0]; oz[0] = qb[1];
      vox[0] = qdb[0]; voz[0] = qdb[1];
      for (int i = 1; i < nl; i++) {
        const int p = m.parent[i];
        const double c = ct[p], s = st[p];
        const double ad = m.adist[i];
        ox[i] = ox[p] + ad * c;
        oz[i] = oz[p] + ad * s;
        vox[i] = vox[p] + omega[p] * ad * (-s);
        voz[i] = voz[p] + omega[p] * ad * c;
        omega[i] = omega[p] + qdb[3 + i - 1];
      }
      // ground contact at both capsule ends (physics.py:321-353)
      for (int i = 0; i < nl; i++) fex[i] = fez[i] = tex[i] = 0.0;
      for (int i = 0; i < nl; i++) {
        const double c = ct[i], s = st[i];
        for (int end = 0; end < 2; end++) {
          double px, pz, vx, vz;
          if (end == 0) {
            px = ox[i]; pz = oz[i]; vx = vox[i]; vz = voz[i];
          } else {
            px = ox[i] + m.length[i] * c;
            pz = oz[i] + m.length[i] * s;
            vx = vox[i] + omega[i] * m.length[i] * (-s);
            vz = voz[i] + omega[i] * m.length[i] * c;
          }
          if (pz < 0.0) {
            double fn = -CONTACT_SPRING * pz - CONTACT_DAMPING * vz;
            if (fn < 0.0) fn = 0.0;
            double ft = -FRICTION_GAIN * vx;
            const double cap = FRICTION_MU * fn;
            if (ft > cap) ft = cap;
            else if (ft < -cap) ft = -cap;
            fex[i] += ft;
            fez[i] += fn;
            const double rxx = px - ox[i], rzz = pz - oz[i];
            tex[i] += rxx * fn - rzz * ft;
          }
        }
      }
      // actuation + joint-limit penalty (physics.py:355-370)
      for (int d = 0; d < nd; d++) tau[d] = 0.0;
      for (int j = 0; j < nj; j++) {
        double av = act[j];
        if (av > 1.0) av = 1.0;
        else if (av < -1.0) av = -1.0;
        double t = av * m.torque_max[j];
        const double qj = qb[3 + j];
        if (qj < m.limit_lo[j]) t += LIMIT_SPRING * (m.limit_lo[j] - qj) - LIMIT_DAMPING * qdb[3 + j];
        else if (qj > m.limit_hi[j]) t -= LIMIT_SPRING * (qj - m.limit_hi[j]) + LIMIT_DAMPING * qdb[3 + j];
        t -= JOINT_DAMPING * qdb[3 + j];
        tau[3 + j] = t;
      }
      rnea(m, qb, qdb, zeros, ct, st, GRAVITY, fex, fez, tex, true, bias);
      for (int j = 0; j < nd; j++) unit[j] = 0.0;
      for (int j = active0; j < nd; j++) {
        unit[j] = 1.0;
        rnea(m, qb, zeros, unit, ct, st, 0.0, fex, fez, tex, false, col);
        unit[j] = 0.0;
        for (int i = 0; i < nd; i++) M[i * kMaxD + j] = col[i];
      }
      for (int d = 0; d < nd; d++) rhs[d] = tau[d] - bias[d];
      solve_spd(M, rhs, qdd, active0, nd, kMaxD);
      for (int d = 0; d < nd; d++) {
        double v = qdb[d] + a.h * qdd[d];
        if (v > VEL_CLAMP) v = VEL_CLAMP;
        else if (v < -VEL_CLAMP) v = -VEL_CLAMP;
        qdb[d] = v;
        qb[d] += a.h * v;
      }
    }
    // non-finite guard (physics.py:401-412)
    bool finite = true;
    for (int d = 0; d < nd; d++) {
      if (!(isfinite(qb[d]) && isfinite(qdb[d]))) finite = false;
      else if (qb[d] > DIVERGED || qb[d] < -DIVERGED) finite = false;
    }
    if (!finite) {
      for (int d = 0; d < nd; d++) {
        qb[d] = q0[d];
        qdb[d] = 0.0;
      }
      a.done[b] = 1;
    }
    for (int d = 0; d < nd; d++) {
      q[d] = qb[d];
      qd[d] = qdb[d];
    }
    a.step_count[b] += 1;
    if (a.step_count[b] >= a.ep_len) a.done[b] = 1;
    if (a.has_min_h && q[1] < a.min_h) a.done[b] = 1;
    // compute_reward (physics.py:468-477) on this control step
    double sq[kMaxD];
    for (int j = 0; j < nj; j++) {
      double av = act[j];
      av = av > 1.0 ? 1.0 : (av < -1.0 ? -1.0 : av);
      sq[j] = av * av;
    }
    const double forward = (q[0] - x_before) / a.dt;
    a.reward[b] += a.forward_weight * forward - a.ctrl_cost * np_sum(sq, nj);
  }
}

// The same control step with one WARP per env (small and medium batches,
// where one thread per env leaves the GPU idle and the per-env chain is the
// latency): per substep the link trig, contacts, torques and integration
// run one link / dof per lane, the mass-matrix columns (one RNEA pass each)
// and the bias pass run on separate lanes, and the Cholesky factor is built
// column by column with its rows in parallel. Every element is computed by
// the same operations in the same order as physics_step_kernel, so the two
// kernels agree bit for bit (tests/test_physics_api.py).

struct WarpPhys {
  double qb[kMaxD], qdb[kMaxD], q0[kMaxD], tau[kMaxD], bias[kMaxD], rhs[kMaxD], qdd[kMaxD];
  double M[kMaxD * kMaxD];
  double theta[kMaxL], ct[kMaxL], st[kMaxL], omega[kMaxL], ox[kMaxL], oz[kMaxL], vox[kMaxL],
      voz[kMaxL], fex[kMaxL], fez[kMaxL], tex[kMaxL];
};

// kLanes lanes per env (32, 16 or 8: 1, 2 or 4 envs per warp); per-link /
// per-dof / per-column work is strided over the env's lanes. Fewer lanes per
// env: more envs in flight, longer per-env chain -- see the dispatch below.
template <int kLanes>
__global__ void __launch_bounds__(kLanes == 8 ? 64 : 128) physics_step_warp_kernel(StepArgs a) {
  constexpr int kPer = 32 / kLanes;                  // envs per warp
  constexpr int kWarpsPB = kLanes == 8 ? 2 : 4;      // warps per block
  __shared__ WarpPhys s_env[kWarpsPB * kPer];
  const Model &m = a.m;
  const int nl = m.nl, nd = nl + 2, nj = nd - 3;
  const int active0 = a.fixed_root ? 3 : 0;
  const int lane = threadIdx.x & (kLanes - 1);
  const int slot = threadIdx.x / kLanes;
  WarpPhys &S = s_env[slot];
  PXR_DCHECK(nl >= 1 && nl <= kMaxL && nd <= kMaxD && m.parent[0] < 0);
  // every lane of a block runs the same iterations (the warp syncs span the
  // envs sharing a warp); a slot past the batch recomputes env 0 unstored
  for (int64_t base = (int64_t)blockIdx.x * (kWarpsPB * kPer); base < a.batch;
       base += (int64_t)gridDim.x * (kWarpsPB * kPer)) {
    // (a warp with no env left skips -- warp-uniform; otherwise its lanes
    // stay in lockstep)
    if (base + (int64_t)(threadIdx.x >> 5) * kPer >= a.batch) continue;
    const bool valid = base + slot < a.batch;
    const int64_t b = valid ? base + slot : 0;
    double *q = a.qpos + b * nd, *qd = a.qvel + b * nd;
    const double *act = a.actions + b * nj;
    for (int d = lane; d < nd; d += kLanes) {
      S.qb[d] = q[d];
      S.qdb[d] = qd[d];
      S.q0[d] = q[d];
    }
    __syncwarp();
    const double x_before = S.qb[0];
    for (int sub = 0; sub < a.substeps; sub++) {
      // kinematics pass (physics.py:144-163): angle chain, per-link trig,
      // velocity chain
      if (lane == 0) {
        S.theta[0] = S.qb[2];
        for (int i = 1; i < nl; i++) S.theta[i] = S.theta[m.parent[i]] + S.qb[3 + i - 1];
      }
      __syncwarp();
      for (int i = lane; i < nl; i += kLanes) {
        S.ct[i] = glibc_cos(S.theta[i]);
        S.st[i] = glibc_sin(S.theta[i]);
      }
      __syncwarp();
      if (lane == 0) {
        S.omega[0] = S.qdb[2];
        S.ox[0] = S.qb[0]; S.oz[0] = S.qb[1];
        S.vox[0] = S.qdb[0]; S.voz[0] = S.qdb[1];
        for (int i = 1; i < nl; i++) {
          const int p = m.parent[i];
          const double c = S.ct[p], s = S.st[p];
          const double ad = m.adist[i];
          S.ox[i] = S.ox[p] + ad * c;
          S.oz[i] = S.oz[p] + ad * s;
          S.vox[i] = S.vox[p] + S.omega[p] * ad * (-s);
          S.voz[i] = S.voz[p] + S.omega[p] * ad * c;
          S.omega[i] = S.omega[p] + S.qdb[3 + i - 1];
        }
      }
      __syncwarp();
      // ground contact at both capsule ends (physics.py:321-353), one link per lane
      for (int i = lane; i < nl; i += kLanes) {
        const double c = S.ct[i], s = S.st[i];
        double fx = 0.0, fz = 0.0, tx = 0.0;
        for (int end = 0; end < 2; end++) {
          double px, pz, vx, vz;
          if (end == 0) {
            px = S.ox[i]; pz = S.oz[i]; vx = S.vox[i]; vz = S.voz[i];
          } else {
            px = S.ox[i] + m.length[i] * c;
            pz = S.oz[i] + m.length[i] * s;
            vx = S.vox[i] + S.omega[i] * m.length[i] * (-s);
            vz = S.voz[i] + S.omega[i] * m.length[i] * c;
          }
          if (pz < 0.0) {
            double fn = -CONTACT_SPRING * pz - CONTACT_DAMPING * vz;
            if (fn < 0.0) fn = 0.0;
            double ft = -FRICTION_GAIN * vx;
            const double cap = FRICTION_MU * fn;
            if (ft > cap) ft = cap;
            else if (ft < -cap) ft = -cap;
            fx += ft;
            fz += fn;
            const double rxx = px - S.ox[i], rzz = pz - S.oz[i];
            tx += rxx * fn - rzz * ft;
          }
        }
        S.fex[i] = fx;
        S.fez[i] = fz;
        S.tex[i] = tx;
      }
      // actuation + joint-limit penalty (physics.py:355-370), one dof per lane
      for (int d = lane; d < nd; d += kLanes) {
        double t = 0.0;
        if (d >= 3) {
          const int j = d - 3;
          double av = act[j];
          if (av > 1.0) av = 1.0;
          else if (av < -1.0) av = -1.0;
          t = av * m.torque_max[j];
          const double qj = S.qb[3 + j];
          if (qj < m.limit_lo[j]) t += LIMIT_SPRING * (m.limit_lo[j] - qj) - LIMIT_DAMPING * S.qdb[3 + j];
          else if (qj > m.limit_hi[j]) t -= LIMIT_SPRING * (qj - m.limit_hi[j]) + LIMIT_DAMPING * S.qdb[3 + j];
          t -= JOINT_DAMPING * S.qdb[3 + j];
        }
        S.tau[d] = t;
      }
      __syncwarp();
      // the mass-matrix columns (item j) and the RNEA bias (item nd)
      for (int it = lane; it <= nd; it += kLanes) {
        if (it < active0) continue;
        double zeros[kMaxD], vec[kMaxD], col[kMaxD];
        for (int d = 0; d < nd; d++) {
          zeros[d] = 0.0;
          vec[d] = d == it ? 1.0 : 0.0;
        }
        if (it == nd) {
          rnea(m, S.qb, S.qdb, zeros, S.ct, S.st, GRAVITY, S.fex, S.fez, S.tex, true, col);
          for (int d = 0; d < nd; d++) S.bias[d] = col[d];
        } else {
          rnea(m, S.qb, zeros, vec, S.ct, S.st, 0.0, S.fex, S.fez, S.tex, false, col);
          for (int i = 0; i < nd; i++) S.M[i * kMaxD + it] = col[i];
        }
      }
      __syncwarp();
      for (int d = lane; d < nd; d += kLanes) S.rhs[d] = S.tau[d] - S.bias[d];
      // Cholesky (physics.py:241-269 / solve_spd): column j, then its rows
      for (int j = active0; j < nd; j++) {
        if (lane == 0) {
          double acc = S.M[j * kMaxD + j];
          for (int t = active0; t < j; t++) acc -= S.M[j * kMaxD + t] * S.M[j * kMaxD + t];
          if (acc < 1e-12) acc = 1e-12;
          S.M[j * kMaxD + j] = sqrt(acc);
        }
        __syncwarp();
        for (int i = j + 1 + lane; i < nd; i += kLanes) {
          double acc = S.M[i * kMaxD + j];
          for (int t = active0; t < j; t++) acc -= S.M[i * kMaxD + t] * S.M[j * kMaxD + t];
          S.M[i * kMaxD + j] = acc / S.M[j * kMaxD + j];
        }
        __syncwarp();
      }
      if (lane == 0) {  // the two triangular solves
        double *x = S.qdd;
        for (int i = 0; i < active0; i++) x[i] = 0.0;
        for (int i = active0; i < nd; i++) {
          double acc = S.rhs[i];
          for (int t = active0; t < i; t++) acc -= S.M[i * kMaxD + t] * x[t];
          x[i] = acc / S.M[i * kMaxD + i];
        }
        for (int i = nd - 1; i >= active0; i--) {
          double acc = x[i];
          for (int t = i + 1; t < nd; t++) acc -= S.M[t * kMaxD + i] * x[t];
          x[i] = acc / S.M[i * kMaxD + i];
        }
      }
      __syncwarp();
      for (int d = lane; d < nd; d += kLanes) {  // semi-implicit Euler (physics.py:389-398)
        double v = S.qdb[d] + a.h * S.qdd[d];
        if (v > VEL_CLAMP) v = VEL_CLAMP;
        else if (v < -VEL_CLAMP) v = -VEL_CLAMP;
        S.qdb[d] = v;
        S.qb[d] += a.h * v;
      }
      __syncwarp();
    }
    if (lane == 0 && valid) {
      // non-finite guard (physics.py:401-412)
      bool finite = true;
      for (int d = 0; d < nd; d++) {
        if (!(isfinite(S.qb[d]) && isfinite(S.qdb[d]))) finite = false;
        else if (S.qb[d] > DIVERGED || S.qb[d] < -DIVERGED) finite = false;
      }
      if (!finite) {
        for (int d = 0; d < nd; d++) {
          S.qb[d] = S.q0[d];
          S.qdb[d] = 0.0;
        }
        a.done[b] = 1;
      }
      for (int d = 0; d < nd; d++) {
        q[d] = S.qb[d];
        qd[d] = S.qdb[d];
      }
      a.step_count[b] += 1;
      if (a.step_count[b] >= a.ep_len) a.done[b] = 1;
      if (a.has_min_h && q[1] < a.min_h) a.done[b] = 1;
      // compute_reward (physics.py:468-477) on this control step
      double sq[kMaxD];
      for (int j = 0; j < nj; j++) {
        double av = act[j];
        av = av > 1.0 ? 1.0 : (av < -1.0 ? -1.0 : av);
        sq[j] = av * av;
      }
      const double forward = (q[0] - x_before) / a.dt;
      a.reward[b] += a.forward_weight * forward - a.ctrl_cost * np_sum(sq, nj);
    }
    __syncwarp();
  }
}

// prng.py:124-135 uniform(key, n, lo, hi) draws for one key into out[0..n)
__device__ void uniform_draws(uint64_t khi, uint64_t klo, int n, double lo, double hi,
                              double *out) {
  const double cap = nextafter(hi, -INFINITY);
  for (int b = 0; 2 * b < n; b++) {
    uint64_t w0, w1;
    threefry2x64(khi, klo, (uint64_t)b, 0, w0, w1);
    const uint64_t w[2] = {w0, w1};
    for (int k = 0; k < 2 && 2 * b + k < n; k++) {
      const double u = (double)(w[k] >> 11) * 0x1p-53;
      const double v = lo + u * (hi - lo);
      out[2 * b + k] = v < cap ? v : cap;  // np.minimum
    }
  }
}

// prng.py:138-152 normal(key, n): Box-Muller over 2*ceil(n/2) words
__device__ void normal_draws(uint64_t khi, uint64_t klo, int n, double *out) {
  const int mm = (n + 1) / 2;
  uint64_t bits[kMaxD + 2];
  for (int b = 0; 2 * b < 2 * mm; b++) {
    uint64_t w0, w1;
    threefry2x64(khi, klo, (uint64_t)b, 0, w0, w1);
    bits[2 * b] = w0;
    bits[2 * b + 1] = w1;
  }
  for (int i = 0; i < mm; i++) {
    const double u1 = ((double)(bits[i] >> 11) + 1.0) * 0x1p-53;
    const double u2 = (double)(bits[mm + i] >> 11) * 0x1p-53;
    const double r = sqrt(-2.0 * numpy_log(u1));  // np.log: numpy's SVML log
    const double th = 2.0 * 3.141592653589793 * u2;
    if (i < n) out[i] = r * glibc_cos(th);
    if (mm + i < n) out[mm + i] = r * glibc_sin(th);
  }
}

// reset of env rows (physics.py:499-504 / env.py:150-152): k = the env's
// key; qpos = rest + U(fold_in(k, 0)); qvel = 0.05 * N(fold_in(k, 1)).
// mode 0 (reset_state, make_env): k = split(R, .)[g] = TF(R, (g, 1)) for all
//   envs; mode 1 (auto-reset in step): only envs with done != 0, with
//   k = fold_in(key_t, LB + g) = TF(key_t, (LB + g, 2)); their episode
//   totals move to info_* and the counters clear (env.py:219-238).
__global__ void reset_kernel(const double *rest, int nd, double *qpos, double *qvel,
                             int64_t *step_count, uint8_t *done, double *ep_return,
                             int64_t *ep_length, double *info_return, int64_t *info_length,
                             const double *reward, int64_t batch, uint64_t khi, uint64_t klo,
                             uint64_t env_offset, uint64_t logical_batch, int mode,
                             const uint64_t *dkey) {
  if (dkey != nullptr) {  // key_t written on the device this step (graph replay)
    khi = dkey[0];
    klo = dkey[1];
  }
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = env_offset + (uint64_t)b;
    uint64_t kh, kl;
    if (mode == 0) {
      threefry2x64(khi, klo, g, 1, kh, kl);
    } else {
      // episode bookkeeping for every env (env.py:219-224)
      const double ret = ep_return[b] + reward[b];
      const int64_t len = ep_length[b] + 1;
      const bool d = done[b] != 0;
      info_return[b] = d ? ret : 0.0;
      info_length[b] = d ? len : 0;
      ep_return[b] = d ? 0.0 : ret;
      ep_length[b] = d ? 0 : len;
      if (!d) continue;
      threefry2x64(khi, klo, logical_batch + g, 2, kh, kl);
    }
    uint64_t k0h, k0l, k1h, k1l;
    threefry2x64(kh, kl, 0, 2, k0h, k0l);  // fold_in(k, 0)
    threefry2x64(kh, kl, 1, 2, k1h, k1l);  // fold_in(k, 1)
    double u[kMaxD], nrm[kMaxD];
    uniform_draws(k0h, k0l, nd, -0.1, 0.1, u);
    normal_draws(k1h, k1l, nd, nrm);
    for (int d = 0; d < nd; d++) {
      qpos[b * nd + d] = rest[d] + u[d];
      qvel[b * nd + d] = nrm[d] * 0.05;
    }
    step_count[b] = 0;
    if (mode == 0) {
      done[b] = 0;
      ep_return[b] = 0.0;
      ep_length[b] = 0;
    } else {
      done[b] = 0;  // sys.done cleared (env.py:234); the step's done output is a copy
    }
  }
}

// physics.py:114-137 (same kernel as pxr_forward_kinematics, own copy here)
__global__ void fk_env_kernel(const double *qpos, const int32_t *parent, const double *adist,
                              int nl, int64_t batch, double *poses) {
  pdl_trigger();  // the render launch that follows may be scheduled now
  const int dof = 3 + nl - 1;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    const double *q = qpos + b * dof;
    double *out = poses + b * nl * 3;
    out[0] = q[0];
    out[1] = q[1];
    out[2] = q[2];
    for (int i = 1; i < nl; i++) {
      const int pp = parent[i];
      const double th = out[3 * pp + 2];
      out[3 * i + 0] = out[3 * pp + 0] + adist[i] * glibc_cos(th);
      out[3 * i + 1] = out[3 * pp + 1] + adist[i] * glibc_sin(th);
      out[3 * i + 2] = th + q[3 + i - 1];
    }
  }
}

// Lanes per env by batch (tools/phys_bench.py on a B200, Humanoid / HalfCheetah,
// round 2): half a warp per env with the smallest shared-memory carveout (the
// lanes' RNEA state stays in L1) up to two waves of 8-env blocks (B=1: 0.16 /
// 0.10 ms against 0.65 / 0.25 ms for one thread per env; B=1000: 0.17 /
// 0.10; B=2048: 0.34 / 0.19), then a quarter warp up to ~6k for models of
// 10+ dofs (B=4096: 0.58 against 0.79 ms), one thread per env above
// (B=16384: 1.04 against 1.77 ms for a quarter warp). One warp per env
// (same carveout) is as fast as half a warp up to ~600 envs and is kept for
// PXR_DEBUG_PHYS=warp.
constexpr int64_t kHalfEnvMax = 2368, kQuarterEnvMax = 6144;

static inline unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 65536) b = 65536;
  return (unsigned)b;
}

}  // namespace pxr

using namespace pxr;

extern "C" pxr_status pxr_physics_step(const pxr_model *model, double *qpos, double *qvel,
                                       int64_t *step_count, uint8_t *done,
                                       const double *actions, double *reward, int64_t batch,
                                       void *stream) {
  if (model == nullptr || qpos == nullptr || qvel == nullptr || step_count == nullptr ||
      done == nullptr || actions == nullptr || reward == nullptr)
    return set_invalid("pxr_physics_step: null argument");
  if (batch < 1) return set_invalid("batch must be >= 1");
  if (model->n_links < 1 || model->n_links > kMaxL)
    return set_unsupported("pxr_physics_step: 1..16 links");
  StepArgs a{};
  a.m = Model{model->parent, model->anchor_dist, model->length, model->mass, model->inertia,
              model->limit_lo, model->limit_hi, model->torque_max, model->n_links};
  a.qpos = qpos;
  a.qvel = qvel;
  a.step_count = step_count;
  a.done = done;
  a.actions = actions;
  a.reward = reward;
  a.batch = batch;
  a.substeps = model->substeps;
  a.fixed_root = model->fixed_root;
  a.has_min_h = model->has_min_root_height;
  a.dt = model->dt;
  a.h = model->dt / model->substeps;
  a.min_h = model->min_root_height;
  a.forward_weight = model->forward_weight;
  a.ctrl_cost = model->ctrl_cost;
  a.ep_len = model->episode_length;
  // sub-warp kernels in the latency-bound range, one thread per env above
  // (throughput); PXR_DEBUG_PHYS=warp|half|quarter|thread forces one
  const char *force = debug_knob(kDbgPhys);
  const int nd = model->n_links + 2;
  char kind = batch <= kHalfEnvMax                    ? 'h'
              : (nd >= 12 && batch <= kQuarterEnvMax) ? 'q'
                                                      : 't';
  if (force != nullptr) kind = force[0];
  cudaStream_t st = (cudaStream_t)stream;
  {
    // warp / half warp per env: the lanes' RNEA state lives in local memory
    // (L1), so ask for the smallest shared-memory carveout (set once per
    // device; at ~100 envs the default split left the warps' working set
    // spilling to L2: Humanoid B=100 0.32 -> 0.17 ms). The quarter-warp
    // kernel keeps the default (at its batches occupancy needs the shared
    // memory: B=4096 0.58 against 0.75 ms).
    static bool carveout_set[64] = {};
    const DeviceFacts &df = device_facts();
    if (!carveout_set[df.device & 63]) {
      cudaFuncSetAttribute((const void *)physics_step_warp_kernel<32>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaFuncSetAttribute((const void *)physics_step_warp_kernel<16>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      (void)cudaGetLastError();
      carveout_set[df.device & 63] = true;
    }
  }
  if (kind == 'w') {  // 4 envs per 128-thread block
    physics_step_warp_kernel<32><<<blocks_for((batch + 3) / 4, 1), 128, 0, st>>>(a);
    return check_launch("physics_step_warp_kernel");
  }
  if (kind == 'h') {  // 8 envs per 128-thread block
    physics_step_warp_kernel<16><<<blocks_for((batch + 7) / 8, 1), 128, 0, st>>>(a);
    return check_launch("physics_step_warp_kernel");
  }
  if (kind == 'q') {  // 8 envs per 64-thread block
    physics_step_warp_kernel<8><<<blocks_for((batch + 7) / 8, 1), 64, 0, st>>>(a);
    return check_launch("physics_step_warp_kernel");
  }
  physics_step_kernel<<<blocks_for(batch, 64), 64, 0, (cudaStream_t)stream>>>(a);
  return check_launch("physics_step_kernel");
}

extern "C" pxr_status pxr_reset_envs(const pxr_model *model, double *qpos, double *qvel,
                                     int64_t *step_count, uint8_t *done, double *ep_return,
                                     int64_t *ep_length, double *info_return,
                                     int64_t *info_length, const double *reward, int64_t batch,
                                     uint64_t key_hi, uint64_t key_lo, uint64_t env_offset,
                                     uint64_t logical_batch, int32_t mode,
                                     const uint64_t *device_key, void *stream) {
  if (model == nullptr || qpos == nullptr || qvel == nullptr || step_count == nullptr ||
      done == nullptr || ep_return == nullptr || ep_length == nullptr)
    return set_invalid("pxr_reset_envs: null argument");
  if (mode != 0 && (info_return == nullptr || info_length == nullptr || reward == nullptr))
    return set_invalid("pxr_reset_envs: auto-reset needs reward and info outputs");
  if (batch < 1) return set_invalid("batch must be >= 1");
  if (model->n_links < 1 || model->n_links > kMaxL)
    return set_unsupported("pxr_reset_envs: 1..16 links");
  reset_kernel<<<blocks_for(batch, 128), 128, 0, (cudaStream_t)stream>>>(
      model->rest_qpos, model->n_links + 2, qpos, qvel, step_count, done, ep_return, ep_length,
      info_return, info_length, reward, batch, key_hi, key_lo, env_offset, logical_batch, mode,
      device_key);
  return check_launch("reset_kernel");
}

extern "C" pxr_status pxr_env_poses(const pxr_model *model, const double *qpos, int64_t batch,
                                    double *poses, void *stream) {
  if (model == nullptr || qpos == nullptr || poses == nullptr) return set_invalid("null FK args");
  if (batch < 1 || model->n_links < 1 || model->n_links > 64) return set_invalid("bad FK sizes");
  fk_env_kernel<<<blocks_for(batch, 128), 128, 0, (cudaStream_t)stream>>>(
      qpos, model->parent, model->anchor_dist, model->n_links, batch, poses);
  return check_launch("fk_env_kernel");
}
