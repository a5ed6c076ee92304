// uuv_task.cuh — per-env reset (declarative samplers) and the task epilogue.
#pragma once

#include "uuv_device.cuh"

namespace uuv {

// Device view of one batch (uuv_state with typed pointers).
template <typename R> struct StateView {
  R* p; R* q; R* nu; R* act; R* cur;
  int32_t* steps; int32_t* episodes; uint8_t* diverged;
  const uint8_t* type_id;
  double* ov; uint16_t* ov_keys;
  int32_t slot[UUV_OV_COUNT];
  int32_t n_slots, a_max;
  int64_t n, ld, env_offset;
};

// Task constants in the batch precision.
template <typename R> struct TaskR {
  int32_t kind, episode_length, traj_kind, obs_dim;
  R bounds, nu_max, fail_penalty;
  R w_p, w_a, w_v, w_u, w_b, r_tol, speed_cap;
  R dock_bonus, w_dock_dist, w_impact, w_level;
  R target_p[3], target_q[4];
  R success_tol;
  R dock_centre[3], dock_radius;
  R traj_radius, traj_rate, traj_climb, traj_z0, traj_phase;
  R traj_amp[3], traj_rates[3];
};

// ------------------------------------------------------------------ reset one env
// engine.py:493-511 with the declarative sampler of tasks/core.py:282-289:
// episodes += 1; Philox(seed, env_offset + i, episode); overlay draws (sorted
// keys), current, start box.  Writes episodes, overlay record, key mask and
// current to memory; returns the new kinematic state in registers.
template <typename R>
UUV_D void reset_env(const StateView<R>& sv, int64_t i, const uuv_sampler& smp, uint64_t seed,
                     R& px, R& py, R& pz, Q4<R>& q, R* nu, V3<R>& cur) {
  const int32_t ep = sv.episodes[i] + 1;
  sv.episodes[i] = ep;
  EnvRng g;
  g.init(smp.rng_mode, seed, (uint64_t)(sv.env_offset + i), (uint64_t)(int64_t)ep);
  const int64_t ld = sv.ld;
  // identity record: ratios 1, cobm/payload/positions/jitter 0
  // (cold code, run for finished rows only: loops stay rolled to keep the task
  // kernels' instruction footprint small)
  if (sv.ov != nullptr) {
#pragma unroll 1
    for (int k = 0; k < UUV_OV_COUNT; ++k) {
      const int s0 = sv.slot[k];
      if (s0 < 0) continue;
      const int width = k == UUV_OV_PAYLOAD_POS ? 3 : (k == UUV_OV_JITTER ? 3 * UUV_MAX_ACT : 1);
      const double ident = k <= UUV_OV_THRUST_COEFF ? 1.0 : 0.0;
#pragma unroll 1
      for (int c = 0; c < width; ++c) sv.ov[(s0 + c) * ld + i] = ident;
    }
  }
  uint16_t keys = 0;
#pragma unroll 1
  for (int d = 0; d < smp.n_overlay; ++d) {
    const uuv_draw& dr = smp.overlay[d];
    double v[3] = {0.0, 0.0, 0.0};
#pragma unroll 1
    for (int c = 0; c < dr.n_draws; ++c) {
      const double x = draw(g, dr, smp.pw_table);
      v[0] = c == 0 ? x : v[0];
      v[1] = c == 1 ? x : v[1];
      v[2] = c == 2 ? x : v[2];
    }
    keys |= (uint16_t)(1u << dr.key);
    const int s0 = sv.slot[dr.key];
    if (sv.ov == nullptr || s0 < 0) continue;
    if (dr.key == UUV_OV_JITTER) {
      for (int j = 0; j < UUV_MAX_ACT; ++j)
        for (int c = 0; c < 3; ++c) sv.ov[(s0 + 3 * j + c) * ld + i] = v[c];
    } else {
      for (int c = 0; c < dr.n_draws; ++c) sv.ov[(s0 + c) * ld + i] = v[c];
    }
  }
  if (sv.ov_keys != nullptr) sv.ov_keys[i] = keys;
  // current (randomization.py:225-234)
  double cx = 0.0, cy = 0.0;
  if (smp.current_mode != UUV_CURRENT_NONE) {
    const double speed = draw(g, smp.current_speed, smp.pw_table);
    const double heading = smp.current_mode == UUV_CURRENT_RANDOM_HEADING
                               ? g.uniform(0.0, 6.283185307179586)
                               : draw(g, smp.current_heading, smp.pw_table);
    double sh, ch;
    sincos_<double>(heading, &sh, &ch);
    cx = speed * ch;
    cy = speed * sh;
  }
  cur = V3<R>{(R)cx, (R)cy, R(0)};
  if (sv.cur != nullptr) {
    sv.cur[0 * ld + i] = (R)cx;
    sv.cur[1 * ld + i] = (R)cy;
    sv.cur[2 * ld + i] = R(0);
  }
  // start pose / velocity
  if (smp.start_mode == UUV_START_BOX) {
    double pp[3], eu[3];
    // one rolled loop over the 12 draws in the reference's order: p (3), euler (3), nu (6)
    const double* lo[3] = {smp.p_lo, smp.eul_lo, smp.nu_lo};
    const double* hi[3] = {smp.p_hi, smp.eul_hi, smp.nu_hi};
    double dv[12];
#pragma unroll 1
    for (int c = 0; c < 12; ++c) {
      const int grp = c < 3 ? 0 : (c < 6 ? 1 : 2), k = c < 3 ? c : (c < 6 ? c - 3 : c - 6);
      dv[c] = g.uniform(lo[grp][k], hi[grp][k]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) pp[c] = __dadd_rn(smp.p_base[c], dv[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c) eu[c] = dv[3 + c];
#pragma unroll
    for (int c = 0; c < 6; ++c) nu[c] = (R)dv[6 + c];
    px = (R)pp[0]; py = (R)pp[1]; pz = (R)pp[2];
    const Q4<double> qd = euler_quat(eu[0], eu[1], eu[2]);
    q = Q4<R>{(R)qd.w, (R)qd.x, (R)qd.y, (R)qd.z};
  } else {
    px = py = pz = R(0);
    q = Q4<R>{R(1), R(0), R(0), R(0)};
    for (int c = 0; c < 6; ++c) nu[c] = R(0);
  }
}

// ------------------------------------------------------------------ reference trajectory
// trajectories.py:56-83
template <typename R>
UUV_D void ref_point(const TaskR<R>& t, R tt, V3<R>& p, V3<R>& v) {
  if (t.traj_kind == UUV_TRAJ_HELIX) {
    const R w = t.traj_rate, r = t.traj_radius, c = t.traj_climb;
    R s, co;
    sincos_<R>(w * tt, &s, &co);
    p = V3<R>{r * co, r * s, t.traj_z0 + c * tt};
    v = V3<R>{-r * w * s, r * w * co, c};
  } else {
    const R ax = t.traj_amp[0], ay = t.traj_amp[1], az = t.traj_amp[2];
    const R rx = t.traj_rates[0], ry = t.traj_rates[1], rz = t.traj_rates[2];
    R s0, c0, s1, c1, s2, c2;
    sincos_<R>(rx * tt, &s0, &c0);
    sincos_<R>(ry * tt + t.traj_phase, &s1, &c1);
    sincos_<R>(rz * tt, &s2, &c2);
    p = V3<R>{ax * s0, ay * s1, t.traj_z0 + az * s2};
    v = V3<R>{ax * rx * c0, ay * ry * c1, az * rz * c2};
  }
}

template <typename R>
UUV_D V3<R> task_target(const TaskR<R>& t, int32_t steps, R dt, V3<R>* vref) {
  if (t.kind == UUV_TASK_TRACKING) {
    V3<R> p, v;
    ref_point(t, (R)steps * dt, p, v);
    if (vref) *vref = v;
    return p;
  }
  if (t.kind == UUV_TASK_STATION) return V3<R>{t.target_p[0], t.target_p[1], t.target_p[2]};
  return V3<R>{t.dock_centre[0], t.dock_centre[1], t.dock_centre[2]};
}

// Observation row (tasks/core.py:316-321): [R^T(p_t - p), log(q* (x) q_t), nu, prev_u, extras].
// Returns |log(q* (x) q_t)| through att_err.
template <typename R>
UUV_D void observe_row(const TaskR<R>& t, int A, R px, R py, R pz, Q4<R> q, const R* nu,
                       const R* pu, int32_t steps, R dt, R* out, R* att_err) {
  V3<R> vref{R(0), R(0), R(0)};
  const V3<R> tp = task_target(t, steps, dt, &vref);
  const V3<R> ep = qrot_inv(q, tp - V3<R>{px, py, pz});
  const Q4<R> tq{t.target_q[0], t.target_q[1], t.target_q[2], t.target_q[3]};
  const V3<R> ea = rotvec(qmul(qconj(q), tq));
  out[0] = ep.x; out[1] = ep.y; out[2] = ep.z;
  out[3] = ea.x; out[4] = ea.y; out[5] = ea.z;
#pragma unroll
  for (int k = 0; k < 6; ++k) out[6 + k] = nu[k];
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j)
    if (j < A) out[12 + j] = pu[j];
  if (t.kind == UUV_TASK_TRACKING) {
    const V3<R> vb = qrot_inv(q, vref);
    out[12 + A] = vb.x; out[13 + A] = vb.y; out[14 + A] = vb.z;
  } else if (t.kind == UUV_TASK_DOCKING) {
    out[12 + A] = t.dock_centre[2] - pz;
  }
  if (att_err) *att_err = norm(ea);
}

// Reward / termination / info of one env after the physics step
// (tasks/core.py:170-214, 339-361, 409-414, 465-473, 509-523).
template <typename R> struct TaskOut {
  R reward, pos_err, att_err, metric, time, c_dist, c_speed, c_att;
  bool terminated, truncated, finished, failure, success, contact;
};

template <typename R>
UUV_D void task_eval(const TaskR<R>& t, int A, R px, R py, R pz, Q4<R> q, const R* nu,
                     const R* du, int32_t steps, bool diverged, R dt, R* dev_sum, TaskOut<R>& o) {
  const R nanv = nan_<R>();
  const V3<R> p{px, py, pz};
  V3<R> vref{R(0), R(0), R(0)};
  const V3<R> tp = task_target(t, steps, dt, &vref);
  const V3<R> ew = tp - p;
  const Q4<R> tq{t.target_q[0], t.target_q[1], t.target_q[2], t.target_q[3]};
  const V3<R> ea = rotvec(qmul(qconj(q), tq));
  R du2 = R(0);
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j)
    if (j < A) du2 += du[j] * du[j];
  const R e_u = sqrt_<R>(du2);
  R nu2 = R(0);
#pragma unroll
  for (int k = 0; k < 6; ++k) nu2 += nu[k] * nu[k];
  const R nu_n = sqrt_<R>(nu2);
  R reward;
  bool done = false;
  o.metric = nanv;
  o.c_dist = o.c_speed = o.c_att = nanv;
  o.contact = false;
  if (t.kind == UUV_TASK_STATION) {
    const R e_p = norm(qrot_inv(q, ew));
    const R e_a = norm(ea);
    const R e_v = minc_<R>(nu_n, t.speed_cap);
    reward = -t.w_p * e_p - t.w_a * e_a - t.w_v * e_v - t.w_u * e_u +
             t.w_b * (e_p < t.r_tol ? R(1) : R(0));
  } else if (t.kind == UUV_TASK_TRACKING) {
    const V3<R> vw = qrot(q, V3<R>{nu[0], nu[1], nu[2]});
    const R e_p = norm(p - tp);
    const R e_v = minc_<R>(norm(vw - vref), t.speed_cap);
    reward = -t.w_p * e_p - t.w_v * e_v - t.w_u * e_u;
    const R dev = *dev_sum + e_p;
    *dev_sum = dev;
    o.metric = dev * rcp_((R)(steps > 1 ? steps : 1));
  } else {
    const V3<R> vw = qrot(q, V3<R>{nu[0], nu[1], nu[2]});
    const V3<R> c{t.dock_centre[0], t.dock_centre[1], t.dock_centre[2]};
    const V3<R> delta = p - c;
    const R planar = sqrt_<R>(delta.x * delta.x + delta.y * delta.y);
    const bool contact = (pz >= c.z) && (planar <= t.dock_radius);
    const R speed = minc_<R>(norm(vw), t.speed_cap);
    const R att = norm(rotvec(q));
    const R terminal = t.dock_bonus - t.w_dock_dist * planar - t.w_impact * speed - t.w_level * att;
    reward = -t.w_p * norm(delta) + (contact ? terminal : R(0));
    reward = reward - t.w_u * e_u;
    o.contact = contact;
    done = contact;
    o.metric = planar;
    if (contact) { o.c_dist = planar; o.c_speed = speed; o.c_att = att; }
  }
  const bool fail = (abs_<R>(px) > t.bounds) || (abs_<R>(py) > t.bounds) ||
                    (abs_<R>(pz) > t.bounds) || (nu_n > t.nu_max) || diverged;
  o.reward = fail ? -t.fail_penalty : reward;
  o.terminated = done || fail;
  o.truncated = (steps >= t.episode_length) && !o.terminated;
  o.finished = o.terminated || o.truncated;
  o.failure = fail;
  o.pos_err = norm(ew);
  o.att_err = norm(ea);
  o.time = (R)steps * dt;
  if (t.kind == UUV_TASK_STATION) {
    o.metric = o.pos_err;
    o.success = o.finished && !fail && (o.pos_err < t.r_tol);
  } else if (t.kind == UUV_TASK_TRACKING) {
    o.success = o.truncated && (o.metric < t.success_tol);
  } else {
    o.success = o.contact;
  }
}

}  // namespace uuv
