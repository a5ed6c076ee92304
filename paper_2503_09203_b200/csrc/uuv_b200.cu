// uuv_b200.cu — sm_100a kernels and the C ABI declared in include/uuv_b200.h.
//
// Kernels (one env per thread, 128-thread CTAs, SoA state, K substeps fused):
//   k_step        step_batch            (engine.py:465-484)
//   k_task_step   VecTaskEnv.step       (tasks/core.py:328-370), fused physics +
//                 reward/termination + auto-reset + next observation + stats
//   k_reset       reset_envs            (engine.py:487-512), declarative samplers
//   k_task_reset  VecTaskEnv.reset / observe (tasks/core.py:294-321)
//   k_stats       deterministic reduction of the per-CTA rollout statistics
//   k_derive      BatchParams rows for inspection (engine.py:193-234)
//   k_terms       first-substep intermediates for parity tests
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <type_traits>
#include <string>
#include <vector>

#include "uuv_task.cuh"

using namespace uuv;

// Translation-unit split: the Makefile compiles this file once per UUV_TU so
// the kernel families build in parallel (1 = C ABI + reset/statistics/
// inspection kernels, 2 = physics step kernels, 3 = task step kernels,
// 4 = policy step kernels, 5 = step server).  UUV_TU 0 builds everything.
#ifndef UUV_TU
#define UUV_TU 0
#endif
// L2 prefetch of the command row before griddepcontrol.wait (k_step).  Measured
// (A/B on one box): cfg2 4096 envs 2.42 -> 2.31 us, 1M envs -7%; bluerov no-DR +2%.
#ifndef UUV_CMD_PREFETCH
#define UUV_CMD_PREFETCH 1
#endif
#define UUV_TU_MAIN (UUV_TU == 0 || UUV_TU == 1)
#define UUV_TU_STEP (UUV_TU == 0 || UUV_TU == 2)
#define UUV_TU_TASK (UUV_TU == 0 || UUV_TU == 3)
#define UUV_TU_POLICY (UUV_TU == 0 || UUV_TU == 4)
#define UUV_TU_SERVE (UUV_TU == 0 || UUV_TU == 5)

namespace uuv_tu {
extern thread_local std::string g_err;  // uuv_last_error's message (defined in TU 1)
// Every kernel instantiation the library can launch registers itself at load
// time (KernelReg below), so a step server can force them all resident first:
// under CUDA lazy loading, the first launch of an unloaded kernel waits for the
// device, which would stall behind a resident server until its idle timeout.
void register_kernel(const void* fn);
}
template <auto K> struct KernelReg {
  static const bool ok;
};
template <auto K> const bool KernelReg<K>::ok = (uuv_tu::register_kernel((const void*)K), true);
#define UUV_REGISTER(...) (void)KernelReg<__VA_ARGS__>::ok

namespace {

constexpr int kBlock = 128;
// Minimum resident CTAs per SM requested from ptxas (register cap = 65536 /
// (kBlock * minB)); tuned on B200 with scripts/sweep.py.
#ifndef UUV_MINB_F32
#define UUV_MINB_F32 4
#endif
#ifndef UUV_MINB_F64
#define UUV_MINB_F64 2
#endif
template <typename R> struct MinB;
template <> struct MinB<float> { static constexpr int value = UUV_MINB_F32; };
template <> struct MinB<double> { static constexpr int value = UUV_MINB_F64; };
constexpr int kObsMax = 12 + UUV_MAX_ACT + 3;
// High-occupancy DR step kernel: min CTAs/SM and the batch size from which it is
// used.  Measured (A/B, B200): cfg2 1M envs 54.9 -> 49.1 us, cfg5 physics 75.5 ->
// 68.9 us; at 4096 envs it is 2-4% slower (spill latency), hence the threshold.
constexpr int kMinBHi = 5;
#ifndef UUV_HI_OCC_MIN_ENVS
#define UUV_HI_OCC_MIN_ENVS 131072
#endif
// Min CTAs/SM of the float task-step kernel (A/B builds override it).
#ifndef UUV_MINB_TASK_F32
#define UUV_MINB_TASK_F32 UUV_MINB_F32
#endif
template <typename R> struct MinBTask { static constexpr int value = MinB<R>::value; };
template <> struct MinBTask<float> { static constexpr int value = UUV_MINB_TASK_F32; };

uuv_status fail(uuv_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
uuv_status fail(uuv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  uuv_tu::g_err = buf;
  return s;
}

uuv_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return UUV_OK;
}

// ------------------------------------------------------------------ host-side hull compilation
bool is_diag(const double* M) {
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c)
      if (r != c && M[6 * r + c] != 0.0) return false;
  return true;
}

template <typename R>
void build_hull(const uuv_hull& src, Hull<R>& dst) {
  memset(&dst, 0, sizeof dst);
  HullR<R>& h = dst.r;
  HullD& d = dst.d;
  h.n_act = src.n_act;
  h.flags = src.flags & ~kHullReaction;
  if (is_diag(src.M_A) && is_diag(src.D_lin) && is_diag(src.D_quad)) h.flags |= UUV_HULL_DIAGONAL;
  else h.flags &= ~UUV_HULL_DIAGONAL;
  h.mlp_layers = src.mlp_layers;
  h.mlp_relu = src.mlp_relu;
  for (int k = 0; k <= UUV_MLP_MAX_LAYERS; ++k) h.mlp_sizes[k] = src.mlp_sizes[k];
  for (int j = 0; j < UUV_MAX_ACT; ++j) {
    h.kind[j] = src.kind[j];
    h.model[j] = src.model[j];
    h.limit[j] = (R)src.limit[j];
    h.deadzone[j] = (R)src.deadzone[j];
    h.reaction[j] = (R)src.reaction[j];
    for (int c = 0; c < 3; ++c) {
      h.axis[j][c] = (R)src.axis[j][c];
      h.fin_xf[j][c] = (R)src.fin_xf[j][c];
      h.fin_yf[j][c] = (R)src.fin_yf[j][c];
      h.mount[j][c] = (R)src.mount[j][c];
      d.mount[j][c] = src.mount[j][c];
    }
    h.fin_area[j] = (R)src.fin_area[j];
    h.fin_cla[j] = (R)src.fin_cla[j];
    h.fin_cd0[j] = (R)src.fin_cd0[j];
    h.fin_kd[j] = (R)src.fin_kd[j];
    h.fin_stall[j] = (R)src.fin_stall[j];
    h.fin_rho[j] = (R)src.fin_rho[j];
    h.ct[j] = (R)src.thrust_coeff[j];
    h.tc[j] = (R)src.time_constant[j];
    const double* m = src.mount[j];
    const double* x = src.axis[j];
    h.mxa[j][0] = (R)(m[1] * x[2] - m[2] * x[1]);
    h.mxa[j][1] = (R)(m[2] * x[0] - m[0] * x[2]);
    h.mxa[j][2] = (R)(m[0] * x[1] - m[1] * x[0]);
    if (j < src.n_act && src.reaction[j] != 0.0) h.flags |= kHullReaction;
    d.ct[j] = src.thrust_coeff[j];
    d.tc[j] = src.time_constant[j] > 0 ? src.time_constant[j] : 1.0;
  }
  for (int k = 0; k < 36; ++k) {
    h.M_A[k] = (R)src.M_A[k];
    h.D_lin[k] = (R)src.D_lin[k];
    h.D_quad[k] = (R)src.D_quad[k];
  }
  for (int k = 0; k < UUV_MLP_MAX_PARAMS; ++k) h.mlp[k] = (R)src.mlp[k];
  d.mass = src.mass;
  d.volume = src.volume;
  d.rhog = src.rho * src.g;  // B = (rho * g) * V  (hydrodynamics.py:179)
  d.g = src.g;
  for (int c = 0; c < 3; ++c) { d.r_g[c] = src.r_g[c]; d.r_b[c] = src.r_b[c]; }
  for (int k = 0; k < 9; ++k) d.inertia[k] = src.inertia[k];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) d.M_A[tri(i, j)] = src.M_A[6 * i + j];
  // base derived parameters (overlay-free rows)
  EnvD e;
  e.mass = d.mass; e.volume = d.volume; e.W = d.mass * d.g; e.B = d.rhog * d.volume;
  e.a = 1.0; e.d = 1.0; e.rt = 1.0; e.rc = 1.0;
  for (int c = 0; c < 3; ++c) { e.r_g[c] = d.r_g[c]; e.r_b[c] = d.r_b[c]; }
  for (int k = 0; k < 9; ++k) e.I[k] = d.inertia[k];
  double M[21], L[15], Di[6];
  mass_matrix_d(d, e, M);
  ldl6_factor<double>(M, L, Di, Rcp<double>());
  for (int k = 0; k < 15; ++k) h.L[k] = (R)L[k];
  for (int k = 0; k < 6; ++k) h.dinv[k] = (R)Di[k];
  h.mass = (R)e.mass; h.W = (R)e.W; h.B = (R)e.B;
  for (int c = 0; c < 3; ++c) { h.r_g[c] = (R)e.r_g[c]; h.r_b[c] = (R)e.r_b[c]; }
  h.I[0] = (R)e.I[0]; h.I[1] = (R)e.I[4]; h.I[2] = (R)e.I[8];
  h.I[3] = (R)e.I[1]; h.I[4] = (R)e.I[2]; h.I[5] = (R)e.I[5];
}

template <typename R>
void build_task(const uuv_task& s, TaskR<R>& t) {
  t.kind = s.kind; t.episode_length = s.episode_length; t.traj_kind = s.traj_kind;
  t.obs_dim = s.obs_dim;
  t.bounds = (R)s.bounds; t.nu_max = (R)s.nu_max; t.fail_penalty = (R)s.fail_penalty;
  t.w_p = (R)s.w_p; t.w_a = (R)s.w_a; t.w_v = (R)s.w_v; t.w_u = (R)s.w_u; t.w_b = (R)s.w_b;
  t.r_tol = (R)s.r_tol; t.speed_cap = (R)s.speed_cap;
  t.dock_bonus = (R)s.dock_bonus; t.w_dock_dist = (R)s.w_dock_dist;
  t.w_impact = (R)s.w_impact; t.w_level = (R)s.w_level;
  for (int c = 0; c < 3; ++c) {
    t.target_p[c] = (R)s.target_p[c];
    t.dock_centre[c] = (R)s.dock_centre[c];
    t.traj_amp[c] = (R)s.traj_amp[c];
    t.traj_rates[c] = (R)s.traj_rates[c];
  }
  for (int c = 0; c < 4; ++c) t.target_q[c] = (R)s.target_q[c];
  t.success_tol = (R)s.success_tol; t.dock_radius = (R)s.dock_radius;
  t.traj_radius = (R)s.traj_radius; t.traj_rate = (R)s.traj_rate; t.traj_climb = (R)s.traj_climb;
  t.traj_z0 = (R)s.traj_z0; t.traj_phase = (R)s.traj_phase;
}

template <typename R>
StateView<R> make_view(const uuv_state& s) {
  StateView<R> v;
  v.p = (R*)s.p; v.q = (R*)s.q; v.nu = (R*)s.nu; v.act = (R*)s.act; v.cur = (R*)s.current_ned;
  v.steps = s.steps; v.episodes = s.episodes; v.diverged = s.diverged; v.type_id = s.type_id;
  v.ov = s.overlay; v.ov_keys = s.overlay_keys;
  for (int k = 0; k < UUV_OV_COUNT; ++k) v.slot[k] = s.overlay ? s.slot[k] : -1;
  v.n_slots = s.n_slots; v.a_max = s.a_max;
  v.n = s.n_envs; v.ld = s.ld; v.env_offset = s.env_offset;
  return v;
}

}  // namespace

struct uuv_ctx {
  std::vector<uuv_hull> hulls;
  std::vector<Hull<float>> hf;
  std::vector<Hull<double>> hd;
  // fork/join streams for per-run mixed-fleet steps (created on first use)
  mutable std::vector<cudaStream_t> fork;
  mutable std::vector<cudaEvent_t> done;
  mutable cudaEvent_t forked = nullptr;
  ~uuv_ctx() {
    // A context is often released by a garbage collector at an arbitrary point --
    // possibly while another stream of the process is being captured into a CUDA
    // graph, where (in the default global capture mode) destroying a stream or an
    // event is a prohibited call that invalidates that capture.  These handles were
    // never captured, so destroy them in relaxed mode.
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    for (cudaStream_t s : fork) cudaStreamDestroy(s);
    for (cudaEvent_t e : done) cudaEventDestroy(e);
    if (forked) cudaEventDestroy(forked);
    cudaThreadExchangeStreamCaptureMode(&mode);
  }
};

// ================================================================== kernels

// Device addresses of the caller's pinned result rows (uuv_host_out): the step
// kernel stores them over the host link next to its HBM stores.
struct HostOut {
  void* pose;          // (13, n) Real: p, q, nu; or null
  void* act;           // (n_act, n) Real; or null
  int32_t* steps;      // (n); or null
  uint8_t* div;        // (n); or null
  int32_t n_act;
  int32_t any;         // 0: no host rows at all
};

template <typename R, int NT> struct StepArgs {
  Hull<R> hull[NT];
  int8_t cls[NT];  // mixed fleets: per-type specialisation (see hull_class)
  StateView<R> sv;
  const R* cmd;
  int64_t cmd_ld;
  int32_t K;
  R dt;
  int32_t early_trigger;  // single-wave grid: let the next step's CTAs launch now
  HostOut out;            // optional host-mapped result rows (uuv_step_host)
  int32_t prefetch_ov;    // DR record beyond L2: prefetch it ahead of the dependent-launch wait
};

// Programmatic dependent launch (PDL).  Step kernels are launched with
// programmatic stream serialisation, so kernel k+1 of a rollout is scheduled
// while kernel k drains; griddepcontrol.wait then blocks until kernel k has
// completed and its writes are visible.  Nothing reads global memory before
// the wait.  A single-wave grid also triggers its dependents at entry.
UUV_D void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
UUV_D void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// UUV_PDL: 0 off, 1 trigger dependents at kernel entry, 2 after the stores, 3 once
// the loads are issued, 4 (default) = 3 for grids of at most 64 CTAs, else 2.
// Measured on B200, cfg2 @4096 envs: graph of 100 steps with fixed commands
// 2.57 / 3.29 / 2.34 us (modes 0/1/2); bench workload (per-step commands from a
// ring larger than L2) 3.18 / 3.29 / 3.16 / 2.39 us (modes 0/1/2/3).
static int pdl_mode() {
  static const int m = [] {
    const char* v = getenv("UUV_PDL");
    return v ? atoi(v) : 4;
  }();
  return m;
}
static bool pdl_enabled() { return pdl_mode() != 0; }

template <typename Kernel, typename Args>
cudaError_t launch_pdl(Kernel k, unsigned grid, cudaStream_t s, const Args& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, a);
}

// Largest grid that is resident in one wave (CTAs per SM from the occupancy API).
template <typename Kernel>
int64_t one_wave_ctas(Kernel k) {
  static thread_local std::map<std::pair<int, const void*>, int64_t> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(dev, (const void*)k);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBlock, 0);
  const int64_t v = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  cache[key] = v;
  return v;
}

// Load env i's kinematic state (SoA, coalesced).
template <typename R>
UUV_D void load_state(const StateView<R>& sv, int64_t i, int A, R& px, R& py, R& pz, Q4<R>& q,
                      R* nu, R* act) {
  const int64_t ld = sv.ld;
  px = sv.p[i]; py = sv.p[ld + i]; pz = sv.p[2 * ld + i];
  q = Q4<R>{sv.q[i], sv.q[ld + i], sv.q[2 * ld + i], sv.q[3 * ld + i]};
#pragma unroll
  for (int k = 0; k < 6; ++k) nu[k] = sv.nu[k * ld + i];
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j) act[j] = j < A ? sv.act[j * ld + i] : R(0);
}

template <typename R>
UUV_D void store_state(const StateView<R>& sv, int64_t i, int A, R px, R py, R pz, Q4<R> q,
                       const R* nu, const R* act) {
  const int64_t ld = sv.ld;
  sv.p[i] = px; sv.p[ld + i] = py; sv.p[2 * ld + i] = pz;
  sv.q[i] = q.w; sv.q[ld + i] = q.x; sv.q[2 * ld + i] = q.y; sv.q[3 * ld + i] = q.z;
#pragma unroll
  for (int k = 0; k < 6; ++k) sv.nu[k * ld + i] = nu[k];
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j)
    if (j < A) sv.act[j * ld + i] = act[j];
}

// Physics of one control step for env i; returns the post-step diverged flag.
// K substeps for one env.  The overlay record is read at (ov, ov_ld, ov_i) — global
// memory (a base pointer, leading dimension and row index); jitter always comes from
// the global record.
// LEAN 1 (a lean batch, see lean_batch: K = 1, no current / reaction / jitter): the
// branch-free substep<LEAN>, as every step-family kernel takes it for such batches.
// LEAN 2 / 3 (a lean task batch, see lean_task: any K, no reaction / jitter, without /
// with the current): the K substeps run to the end, an earlier failure holds the
// state (the same result as stopping at it), as every task-family kernel takes it.
template <typename R, bool DR, int AC, bool DM, bool PRE = false, int LEAN = 0>
UUV_D bool physics_at(const Hull<R>& H, const StateView<R>& sv, int64_t i, const double* ov,
                      int64_t ov_ld, int64_t ov_i, bool has_cur, V3<R> cur, int K, R dt,
                      const R* u, R& px, R& py, R& pz, Q4<R>& q, R* nu, R* act) {
  Sub<R> s;
  const double* jit = nullptr;
  if (DR) {
    EnvD e;
    derive_env(H.d, ov, ov_ld, ov_i, sv.slot, e);
    sub_from_env<R, DM, PRE, AC>(H.r, e, s);
    if (!LEAN && sv.slot[UUV_OV_JITTER] >= 0) jit = sv.ov + sv.slot[UUV_OV_JITTER] * sv.ld + i;
  }
  if constexpr (LEAN == 1)
    return !substep<R, DR, false, AC, DM, false, PRE, 1>(H.r, s, nullptr, sv.ld, px, py, pz, q, nu,
                                                        act, u, false, cur, dt, nullptr);
  if constexpr (LEAN >= 2) {
    bool failed = false;
    for (int k = 0; k < K; ++k)
      failed |= !substep<R, DR, false, AC, DM, false, PRE, LEAN>(H.r, s, nullptr, sv.ld, px, py, pz,
                                                                 q, nu, act, u, has_cur, cur, dt,
                                                                 nullptr, failed);
    return failed;
  }
  bool ok = true;
  // the jitter record is present for every env of a launch or for none: one
  // specialisation per case keeps its code out of the common loop
  auto run = [&](auto with_jit) {
    for (int k = 0; k < K; ++k) {
      if (!substep<R, DR, false, AC, DM, decltype(with_jit)::value, PRE>(
              H.r, s, jit, sv.ld, px, py, pz, q, nu, act, u, has_cur, cur, dt, nullptr)) {
        ok = false;
        break;
      }
    }
  };
  if (DR && jit != nullptr) run(std::true_type{});
  else run(std::false_type{});
  return !ok;
}

template <typename R, bool DR, int AC, bool DM, bool PRE = false, int LEAN = 0>
UUV_D bool physics(const Hull<R>& H, const StateView<R>& sv, int64_t i, int K, R dt, const R* u,
                   R& px, R& py, R& pz, Q4<R>& q, R* nu, R* act) {
  const bool has_cur = LEAN ? LEAN == 3 : sv.cur != nullptr;
  V3<R> cur{R(0), R(0), R(0)};
  if (has_cur) cur = V3<R>{sv.cur[i], sv.cur[sv.ld + i], sv.cur[2 * sv.ld + i]};
  return physics_at<R, DR, AC, DM, PRE, LEAN>(H, sv, i, sv.ov, sv.ld, i, has_cur, cur, K, dt, u, px,
                                              py, pz, q, nu, act);
}

// Inputs of one env's step, all loaded before any arithmetic (one memory round trip).
template <typename R> struct StepIn {
  R px, py, pz;
  Q4<R> q;
  R nu[6], act[UUV_MAX_ACT], u[UUV_MAX_ACT];
  int32_t steps;
  uint8_t div, ty;
};

template <typename R, int NT, int AC>
UUV_D void load_in(const StepArgs<R, NT>& a, int64_t i, StepIn<R>& in) {
  const StateView<R>& sv = a.sv;
  in.ty = NT > 1 ? sv.type_id[i] : 0;
  const int A = AC > 0 ? AC : a.hull[in.ty].r.n_act;
  constexpr int NA = AC > 0 ? AC : UUV_MAX_ACT;
  in.steps = sv.steps[i];
  in.div = sv.diverged[i];
  const R* crow = a.cmd + i * a.cmd_ld;
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j)
    in.u[j] = (j < NA && j < A) ? clip_<R>(crow[j], R(-1), R(1)) : R(0);
  load_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
}

// The step's result rows of env i into the caller's host buffers (every field
// step_batch mutates in place, engine.py:418, 444-449).  Called on every exit of
// step_env / serve_env, frozen rows included.
template <typename R>
UUV_D void put_host_out(const HostOut& o, int64_t i, int64_t n, const StepIn<R>& in,
                        int32_t steps, uint8_t div) {
  if (!o.any) return;
  if (o.pose != nullptr) {
    R* p = (R*)o.pose + i;
    p[0] = in.px; p[n] = in.py; p[2 * n] = in.pz;
    p[3 * n] = in.q.w; p[4 * n] = in.q.x; p[5 * n] = in.q.y; p[6 * n] = in.q.z;
#pragma unroll
    for (int k = 0; k < 6; ++k) p[(7 + k) * n] = in.nu[k];
  }
  if (o.act != nullptr) {
    R* p = (R*)o.act + i;
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j)
      if (j < o.n_act) p[j * n] = in.act[j];
  }
  if (o.steps != nullptr) o.steps[i] = steps;
  if (o.div != nullptr) o.div[i] = div;
}

template <typename R, int NT, bool DR, int AC, bool DM, bool BRANCHLESS = false, bool LEAN = false>
UUV_D void step_env(const StepArgs<R, NT>& a, int64_t i, StepIn<R>& in) {
  const StateView<R>& sv = a.sv;
  if (!BRANCHLESS) {
    if (in.div) {  // frozen rows stay frozen (engine.py:411, 441-449)
      sv.steps[i] = in.steps + 1;
      put_host_out(a.out, i, sv.n, in, in.steps + 1, 1);
      return;
    }
    const Hull<R>& H = a.hull[in.ty];
    const int A = AC > 0 ? AC : H.r.n_act;
    const bool div = physics<R, DR, AC, DM, true, LEAN>(H, sv, i, a.K, a.dt, in.u, in.px, in.py,
                                                        in.pz, in.q, in.nu, in.act);
    store_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
    sv.diverged[i] = div ? 1 : 0;
    sv.steps[i] = in.steps + 1;
    put_host_out(a.out, i, sv.n, in, in.steps + 1, div ? 1 : 0);
    return;
  }
  // BRANCHLESS (small-batch DR build): the physics runs for every row and frozen
  // rows (engine.py:411, 441-449) just do not store it.  With no branch on the
  // diverged flag ahead of the physics, the DR-record loads issue together with
  // the state loads instead of after them: one memory round trip instead of two
  // (cfg2 @4096 envs 2.20 -> 2.09 us).  The 96-register large-batch build keeps
  // the branch (register pressure; +40% otherwise).
  const Hull<R>& H = a.hull[in.ty];
  const int A = AC > 0 ? AC : H.r.n_act;
  const bool div = physics<R, DR, AC, DM, true, LEAN>(H, sv, i, a.K, a.dt, in.u, in.px, in.py, in.pz,
                                                      in.q, in.nu, in.act);
  if (!in.div) {
    store_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
    sv.diverged[i] = div ? 1 : 0;
  } else if (a.out.any) {  // frozen: its stored state is untouched; re-read it for the host rows
    load_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
  }
  sv.steps[i] = in.steps + 1;
  put_host_out(a.out, i, sv.n, in, in.steps + 1, (in.div || div) ? 1 : 0);
}

// Mixed fleets: every env takes its vehicle type's specialised path (types are
// contiguous env blocks, so the switch is warp-uniform except at block edges).
// The float64 (validation) fleet kernels take the two generic paths only: eight
// inlined specialisations left them at 255 registers with ~2 KB of spills.
UUV_D bool diag_class(int8_t c) { return c == 1 || c == 2 || c == 5 || c == 6; }

template <typename R, int NT, bool DR, int AC, bool DM, bool BRANCHLESS = false, bool LEAN = false>
UUV_D void step_any(const StepArgs<R, NT>& a, int64_t i, StepIn<R>& in) {
  if constexpr (NT > 1 && sizeof(R) == 8) {
    if (diag_class(a.cls[in.ty])) step_env<R, NT, DR, 0, true>(a, i, in);
    else step_env<R, NT, DR, 0, false>(a, i, in);
  } else if constexpr (NT > 1) {
    switch (a.cls[in.ty]) {
      case 1: step_env<R, NT, DR, 6, true>(a, i, in); return;
      case 2: step_env<R, NT, DR, 8, true>(a, i, in); return;
      case 3: step_env<R, NT, DR, 6, false>(a, i, in); return;
      case 4: step_env<R, NT, DR, 8, false>(a, i, in); return;
      case 5: step_env<R, NT, DR, 0, true>(a, i, in); return;
      case 6: step_env<R, NT, DR, kFinLayout, true>(a, i, in); return;
      case 7: step_env<R, NT, DR, kFinLayout, false>(a, i, in); return;
      default: step_env<R, NT, DR, 0, false>(a, i, in); return;
    }
  } else {
    // the small-batch DR build issues every load before the diverged-flag branch
    step_env<R, NT, DR, AC, DM, BRANCHLESS && DR, LEAN>(a, i, in);
  }
}

// L2 prefetch of the DR-record slots the per-launch derivation reads (keys up to
// and including payload_position); issued before the dependent-launch wait.
template <typename R>
UUV_D void prefetch_overlay_l2(const StateView<R>& sv, int64_t i) {
#pragma unroll
  for (int k = 0; k <= UUV_OV_PAYLOAD_POS; ++k) {
    const int s0 = sv.slot[k];
    if (s0 >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(sv.ov + s0 * sv.ld + i));
  }
}

// HI: the high-occupancy build of the float DR kernel (register cap 96 instead of
// 128, a few spills to L1), launched for large batches where more resident warps
// hide HBM latency; the default build serves the latency-bound small batches.
template <typename R, int NT, bool DR, int AC, bool DM, bool HI = false, bool LEAN = false>
__global__ void __launch_bounds__(kBlock, HI ? kMinBHi : ((NT > 1 && sizeof(R) == 4) ? 3 : MinB<R>::value))
    k_step(const __grid_constant__ StepArgs<R, NT> a) {
  if (a.early_trigger == 1) pdl_trigger();
#if UUV_CMD_PREFETCH
  {  // the command row and the DR record do not depend on the previous step: start
     // their DRAM fetches into L2 while that step drains (hints: L2 is the point
     // of coherence, the loads themselves follow the wait)
    const int64_t i0 = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i0 < a.sv.n) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.cmd + i0 * a.cmd_ld));
      // (DR record: only when the batch does not stay L2-resident -- otherwise
      // the slot lookups at kernel entry cost more than they hide; measured
      // 4096 envs +8%, 262k +8%, 1M -7.5%, 4M -6%)
      if (DR && HI && a.prefetch_ov) prefetch_overlay_l2(a.sv, i0);
    }
  }
#endif
  pdl_wait();
  struct ExitTrigger {
    bool on;
    __device__ ~ExitTrigger() {
      if (on) pdl_trigger();
    }
  } exit_trigger{a.early_trigger == 2};
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  if (i >= a.sv.n) return;
  StepIn<R> cur;
  load_in<R, NT, AC>(a, i, cur);
  // mode 3: release the next step once this step's loads are issued -- it is
  // already past its own wait here, so at most two grids are in flight, and the
  // next step's command prefetch overlaps this step's compute
  if (a.early_trigger == 3) pdl_trigger();
  step_any<R, NT, DR, AC, DM, !HI, LEAN>(a, i, cur);
}

// ------------------------------------------------------------------ multi-step rollout
// T control steps of every env in ONE launch, the state in registers from the
// first step to the last: step t applies commands slot (start + t) mod n_slots
// of a (n_slots, n, cmd_ld) ring -- exactly step_batch(state, ring[slot]) T
// times (engine.py:465-484), bit for bit (same substep code, same parameters):
// frozen rows stay frozen and count steps, a non-finite substep freezes the row
// at its last finite state.  Per launch instead of per step: the state loads,
// the DR derivation (derive_env + sub_from_env) and the state stores (the states
// between the first and the last step are dead stores, as the substeps' are in
// k_step); per step: the command row (loaded one step ahead) and the optional
// (T, trace_rows, trace_ld) trace: p, q, nu (13 rows), then act (A rows) when
// trace_rows = 13 + A.  Commands and trace may live in mapped pinned host memory:
// the command rows are then read over the host link one step ahead and the trace
// rows written back as they are produced, so a whole host-to-host rollout is one
// launch.  With `ready`
// set, step t first waits (acquire, GPU scope) until *ready > t: a producer on
// another stream fills the ring slot and then raises the counter -- the device-
// side command ring of a resident stepper.
// Host-side description of one rollout (shared by the translation units).
struct RolloutSpec {
  const void* cmd;
  int64_t cmd_ld, slot_stride;
  int32_t n_slots, start, steps;
  void* trace;
  int64_t trace_ld;
  int32_t trace_rows;     // 13 (p, q, nu) or 13 + A (and act)
  const uint32_t* ready;
  bool cmd_device;        // commands in device memory (not mapped host memory)
  HostOut out;            // mapped host rows for the result after the last step
};

template <typename R, int NT> struct RolloutArgs {
  StepArgs<R, NT> step;   // hulls, state view, cmd = slot 0, cmd_ld, K, dt
  int64_t slot_stride;    // elements between ring slots
  int32_t n_slots, start, steps;
  R* trace;               // (steps, trace_rows, trace_ld) or null
  int64_t trace_ld;
  int32_t trace_rows;     // 13, or 13 + A: act rows follow the pose rows
  int32_t prefetch;       // commands in device memory: L2-prefetch two steps ahead
  const uint32_t* ready;  // or null (every slot already written)
};

constexpr uint64_t kRolloutWaitNs = 10000000000ull;  // 10 s without a new command slot

UUV_D uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// LEAN: a lean batch (lean_batch: K = 1, no current, no reaction torques, no mount
// jitter) -- the branch-free substep<LEAN> every step-family kernel takes for it.
// PLAIN (implies LEAN): also no trace, no ready counter and commands in device memory
// -- the whole control step is one basic block (frozen rows computed and not
// committed; the next rows always loaded / prefetched: the ring slot is valid past
// the last step).
template <typename R, int NT, bool DR, int AC, bool DM, bool LEAN = false, bool PLAIN = false>
UUV_D void rollout_env(const RolloutArgs<R, NT>& ra, int64_t i, StepIn<R>& in) {
  const StepArgs<R, NT>& a = ra.step;
  const StateView<R>& sv = a.sv;
  const Hull<R>& H = a.hull[in.ty];
  const int A = AC > 0 ? AC : H.r.n_act;
  constexpr int NA = AC > 0 ? AC : UUV_MAX_ACT;
  const bool has_cur = !LEAN && sv.cur != nullptr;
  V3<R> cur{R(0), R(0), R(0)};
  if (has_cur) cur = V3<R>{sv.cur[i], sv.cur[sv.ld + i], sv.cur[2 * sv.ld + i]};
  const uint32_t* const ready = PLAIN ? nullptr : ra.ready;
  R* const trace = PLAIN ? nullptr : ra.trace;
  const int K = PLAIN ? 1 : a.K;
  uint32_t avail = 0;
  bool stalled = false;  // the producer never raised the counter: give up, never hang
  // ring slot of step t: the slot index advances with t (wrapping), no division per step
  const R* const ring0 = a.cmd + i * a.cmd_ld;
  int slot = (int)(ra.start % ra.n_slots), slot_t = 0;
  auto slot_row = [&](int t) {  // t advances by at most one per call
    if (slot_t < t) {
      ++slot_t;
      slot = slot + 1 == ra.n_slots ? 0 : slot + 1;
    }
    return ring0 + (int64_t)slot * ra.slot_stride;
  };
  auto wait_slot = [&](int t) {
    if (ready != nullptr && (uint32_t)t >= avail) {
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while ((avail = ld_acquire_gpu_u32(ready)) <= (uint32_t)t) {
        __nanosleep(100);
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if ((int64_t)(t1 - t0) > (int64_t)kRolloutWaitNs) {
          stalled = true;
          return;
        }
      }
    }
  };
  // the next step's command row is loaded during this step (PLAIN: the one after
  // next, see below); rows further ahead are pulled into L2 (prefetch, no register)
  // so those loads hit L2: a row from HBM takes longer than one step's compute
  // (measured on the first build: 0.66 us per step from a cold ring, 0.49 from L2)
  const bool pf = ra.prefetch && ready == nullptr;
  R un[UUV_MAX_ACT];
  auto load_row = [&](int t, R* dst) {
    const R* c = slot_row(t);
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) dst[j] = (j < NA && j < A) ? c[j] : R(0);
  };
  constexpr int kAhead = 8;  // L2 prefetch distance in steps
  int pslot = slot;           // ring slot of the last prefetched step
  auto prefetch_next = [&]() {
    pslot = pslot + 1 == ra.n_slots ? 0 : pslot + 1;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(ring0 + (int64_t)pslot * ra.slot_stride));
  };
  // the first command rows are requested before the per-env DR derivation, whose
  // float64 chain would otherwise delay their DRAM round trip to after it
  wait_slot(0);
  load_row(0, un);
  // PLAIN: two command rows in registers, used alternately by a two-step loop body
  // (no register copies): each row has two steps' compute to arrive from L2
  R ub[UUV_MAX_ACT];
  if (PLAIN) load_row(1, ub);
  if (pf)
    for (int t = 1; t < kAhead && t < ra.steps; ++t) prefetch_next();
  Sub<R> s;
  const double* jit = nullptr;
  if (DR) {
    EnvD e;
    derive_env(H.d, sv.ov, sv.ld, i, sv.slot, e);
    sub_from_env<R, DM, true, AC>(H.r, e, s);
    if (!LEAN && sv.slot[UUV_OV_JITTER] >= 0) jit = sv.ov + sv.slot[UUV_OV_JITTER] * sv.ld + i;
  }
  if constexpr (PLAIN) {
    auto one = [&](R* buf, int next) {
      R u[UUV_MAX_ACT];
#pragma unroll
      for (int j = 0; j < UUV_MAX_ACT; ++j) u[j] = clip_<R>(buf[j], R(-1), R(1));
      load_row(next, buf);  // unconditionally (the ring slot is valid): no branch
      prefetch_next();
      const bool ok = substep<R, DR, false, AC, DM, false, true, true>(
          H.r, s, nullptr, sv.ld, in.px, in.py, in.pz, in.q, in.nu, in.act, u, false, cur, a.dt,
          nullptr, in.div != 0);
      in.div = (in.div != 0 || !ok) ? 1 : 0;  // frozen from here on at its last finite state
      in.steps += 1;
    };
    int t = 0;
    for (; t + 1 < ra.steps; t += 2) {
      one(un, t + 2);
      one(ub, t + 3);
    }
    if (t < ra.steps) one(un, t + 2);
  }
  for (int t = 0; !PLAIN && t < ra.steps && !stalled; ++t) {
    R u[UUV_MAX_ACT];
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) u[j] = clip_<R>(un[j], R(-1), R(1));
    if (t + 1 < ra.steps) {  // the next step's command row, in flight during this step
      if (ready == nullptr || (uint32_t)(t + 1) < avail) load_row(t + 1, un);
      if (pf && t + kAhead < ra.steps) prefetch_next();  // step t + kAhead
    }
    if (LEAN && !in.div) {
      if (!substep<R, DR, false, AC, DM, false, true, true>(H.r, s, nullptr, sv.ld, in.px, in.py,
                                                           in.pz, in.q, in.nu, in.act, u, false,
                                                           cur, a.dt, nullptr))
        in.div = 1;
    } else if (!in.div) {
      bool ok = true;
      auto run = [&](auto with_jit) {
        for (int k = 0; k < K; ++k) {
          if (!substep<R, DR, false, AC, DM, decltype(with_jit)::value, true>(
                  H.r, s, jit, sv.ld, in.px, in.py, in.pz, in.q, in.nu, in.act, u, has_cur, cur,
                  a.dt, nullptr)) {
            ok = false;
            break;
          }
        }
      };
      if (DR && jit != nullptr) run(std::true_type{});
      else run(std::false_type{});
      if (!ok) in.div = 1;  // frozen from here on at its last finite state
    }
    in.steps += 1;
    if (trace != nullptr) {
      R* o = trace + (int64_t)t * ra.trace_rows * ra.trace_ld + i;
      const int64_t ld = ra.trace_ld;
      o[0] = in.px; o[ld] = in.py; o[2 * ld] = in.pz;
      o[3 * ld] = in.q.w; o[4 * ld] = in.q.x; o[5 * ld] = in.q.y; o[6 * ld] = in.q.z;
#pragma unroll
      for (int k = 0; k < 6; ++k) o[(7 + k) * ld] = in.nu[k];
      if (ra.trace_rows > 13) {  // the command width's act rows (zero past this env's A)
#pragma unroll
        for (int j = 0; j < UUV_MAX_ACT; ++j)
          if (j < ra.trace_rows - 13) o[(13 + j) * ld] = in.act[j];
      }
    }
    if (t + 1 < ra.steps && ready != nullptr && (uint32_t)(t + 1) >= avail) {
      wait_slot(t + 1);  // the producer had not filled slot t+1 when step t began
      load_row(t + 1, un);
    }
  }
  // the state after the last step: intermediate states live only in registers (and the
  // optional trace), as the substeps of one step do in k_step
  store_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
  sv.diverged[i] = in.div;
  sv.steps[i] = in.steps;
  put_host_out(a.out, i, sv.n, in, in.steps, in.div);
}

// Two builds: the latency-bound small batches get every register they want (one CTA
// per SM is all they fill); from 262,144 envs a 168-register build (3 CTAs/SM) hides
// more latency (bench at_scale: 1M envs 26.1 -> 21.9 us per step, 0.27 -> 0.32 of FP32;
// 128 registers spills and loses at 4096 envs: 1.08 -> 1.61 us)
constexpr int64_t kRolloutHiMinEnvs = 262144;
template <typename R, int NT, bool DR, int AC, bool DM, bool HI = false, bool LEAN = false,
          bool PLAIN = false>
__global__ void __launch_bounds__(kBlock, HI ? 3 : 1) k_rollout(const __grid_constant__ RolloutArgs<R, NT> ra) {
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  if (i >= ra.step.sv.n) return;
  const StateView<R>& sv = ra.step.sv;
  StepIn<R> in;
  in.ty = NT > 1 ? sv.type_id[i] : 0;
  const int A = AC > 0 ? AC : ra.step.hull[in.ty].r.n_act;
  in.steps = sv.steps[i];
  in.div = sv.diverged[i];
  load_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
  if constexpr (NT > 1 && sizeof(R) == 8) {
    if (diag_class(ra.step.cls[in.ty])) rollout_env<R, NT, DR, 0, true>(ra, i, in);
    else rollout_env<R, NT, DR, 0, false>(ra, i, in);
  } else if constexpr (NT > 1) {
    switch (ra.step.cls[in.ty]) {
      case 1: rollout_env<R, NT, DR, 6, true>(ra, i, in); return;
      case 2: rollout_env<R, NT, DR, 8, true>(ra, i, in); return;
      case 3: rollout_env<R, NT, DR, 6, false>(ra, i, in); return;
      case 4: rollout_env<R, NT, DR, 8, false>(ra, i, in); return;
      case 5: rollout_env<R, NT, DR, 0, true>(ra, i, in); return;
      case 6: rollout_env<R, NT, DR, kFinLayout, true>(ra, i, in); return;
      case 7: rollout_env<R, NT, DR, kFinLayout, false>(ra, i, in); return;
      default: rollout_env<R, NT, DR, 0, false>(ra, i, in); return;
    }
  } else {
    rollout_env<R, NT, DR, AC, DM, LEAN, PLAIN>(ra, i, in);
  }
}

// ------------------------------------------------------------------ step server
// A resident kernel that steps the batch whenever the host rings a doorbell in
// mapped pinned memory: no launch, no stream synchronisation per step.  Each CTA
// keeps its envs' state in registers, polls the doorbell (one thread, acquire at
// system scope), reads that step's command rows over the host link, runs the
// same physics as k_step, writes the state back to HBM and the pose rows to the
// caller's pinned buffer, fences at system scope and raises its done flag.  The
// host waits on all flags.  An idle timeout (%globaltimer) ends the kernel if
// the host goes away, so it can never hold the GPU.
struct alignas(16) ServeCtl {  // host-mapped, written by the host
  // {seq, cmd} share one 16-byte line read by a single load: the host stores cmd
  // before seq, so a read that sees the new seq sees that step's cmd.
  uint64_t seq;             // doorbell: step number (| kServeNewPose), or kServeQuit
  uint64_t cmd;             // device-visible address of the (n, cmd_ld) commands
  uint64_t pose;            // device-visible address of the (13, n) pose rows, or 0
  int64_t cmd_ld;           // {pose, cmd_ld, act, steps, div}: re-read only when
  uint64_t act;             //   kServeNewPose is set; act (n_act, n) rows, steps (n),
  uint64_t steps;           //   diverged (n) -- the rest of the step's result
  uint64_t div;
  uint64_t pad_;
  uint64_t stamp[8];        // phase times of the last step (ns; see uuv_server_stamps)
};
constexpr uint64_t kServeQuit = ~0ull;
constexpr uint64_t kServeNewPose = 1ull << 62;  // result addresses / cmd_ld changed this step

struct ServeSync {          // device memory: CTA 0 republishes the doorbell here
  uint64_t go;
  uint64_t cmd, pose;
  int64_t cmd_ld;
  uint64_t act, steps, div;
  uint32_t arrived;         // CTAs done with the current step
};

template <typename R, int NT> struct ServeArgs {
  StepArgs<R, NT> step;
  ServeCtl* ctl;
  uint64_t* done;           // host-mapped: last step the whole grid finished
  ServeSync* sync;
  uint64_t idle_ns;
  uint32_t sleep_ns;        // back-off between doorbell polls
  uint32_t stamps;          // write phase stamps (UUV_SERVE_STAMPS=1; profiling aid)
  int32_t n_act;            // act result rows
};

UUV_D uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
UUV_D uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
UUV_D void ld_relaxed_sys_v2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
UUV_D uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
UUV_D void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
UUV_D void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
UUV_D uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <typename R, int NT, bool DR, int AC, bool DM, bool LEAN = false>
UUV_D void serve_env(const StepArgs<R, NT>& a, int64_t i, StepIn<R>& in, const HostOut& out) {
  const StateView<R>& sv = a.sv;
  in.steps += 1;
  if (!in.div) {
    const Hull<R>& H = a.hull[in.ty];
    const int A = AC > 0 ? AC : H.r.n_act;
    const bool div = physics<R, DR, AC, DM, true, LEAN>(H, sv, i, a.K, a.dt, in.u, in.px, in.py,
                                                        in.pz, in.q, in.nu, in.act);
    store_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
    in.div = div ? 1 : 0;
    sv.diverged[i] = in.div;
  }
  sv.steps[i] = in.steps;
  put_host_out(out, i, sv.n, in, in.steps, in.div);
}

template <typename R, int NT, bool DR, int AC, bool DM, bool LEAN = false>
__global__ void __launch_bounds__(kBlock, (NT > 1 && sizeof(R) == 4) ? 3 : MinB<R>::value)
    k_serve(const __grid_constant__ ServeArgs<R, NT> sa) {
  __shared__ uint64_t s_seq, s_cmd;
  __shared__ HostOut s_out;
  __shared__ int64_t s_ld;
  const StepArgs<R, NT>& a = sa.step;
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool live = i < a.sv.n;
  StepIn<R> in;
  if (live) {
    const StateView<R>& sv = a.sv;
    in.ty = NT > 1 ? sv.type_id[i] : 0;
    const int A = AC > 0 ? AC : a.hull[in.ty].r.n_act;
    in.steps = sv.steps[i];
    in.div = sv.diverged[i];
    load_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
  }
  uint64_t seq = 0;
  // CTA 0: result-row addresses / command stride of the last step
  uint64_t cur_pose = 0, cur_act = 0, cur_steps = 0, cur_div = 0;
  int64_t cur_ld = 0;
  ServeSync* sy = sa.sync;
  if (sa.stamps && blockIdx.x == 0 && threadIdx.x == 0) {  // start marker + idle budget
    sa.ctl->stamp[4] = sa.idle_ns;
    sa.ctl->stamp[5] = global_ns();
  }
  for (;;) {
    if (threadIdx.x == 0) {
      uint64_t v;
      // CTA 0 alone polls the host doorbell and republishes it in L2: every CTA
      // polling over the link costs a system-scope acquire per CTA (measured
      // 190 us vs 20 us per step at 4096 envs)
      if (blockIdx.x == 0) {
        const uint64_t t0 = global_ns();
        uint64_t why = 0, word = 0, cmd = 0;
        for (;;) {
          ld_relaxed_sys_v2(&sa.ctl->seq, word, cmd);  // {seq, cmd} in one read
          v = word == kServeQuit ? kServeQuit : (word & ~kServeNewPose);
          if (v != seq) { why = 1; if (sa.stamps) sa.ctl->stamp[0] = global_ns(); break; }
          // signed: %globaltimer may step back slightly when it is re-synchronised
          if ((int64_t)(global_ns() - t0) > (int64_t)sa.idle_ns) { v = kServeQuit; why = 2; break; }
          __nanosleep(sa.sleep_ns);
        }
        if (v == kServeQuit && blockIdx.x == 0) {  // exit record (profiling aid)
          sa.ctl->stamp[0] = why;
          sa.ctl->stamp[1] = global_ns() - t0;
          sa.ctl->stamp[2] = seq;
        }
        s_cmd = cmd;
        if (v != kServeQuit && (word & kServeNewPose)) {
          uint64_t pose, ld, act, stp, div, pad;
          ld_relaxed_sys_v2(&sa.ctl->pose, pose, ld);
          ld_relaxed_sys_v2(&sa.ctl->act, act, stp);
          ld_relaxed_sys_v2(&sa.ctl->div, div, pad);
          cur_pose = pose;
          cur_ld = (int64_t)ld;
          cur_act = act;
          cur_steps = stp;
          cur_div = div;
        }
        s_ld = cur_ld;
        if (sa.stamps) sa.ctl->stamp[1] = global_ns();
        sy->cmd = s_cmd;
        sy->pose = cur_pose;
        sy->cmd_ld = s_ld;
        sy->act = cur_act;
        sy->steps = cur_steps;
        sy->div = cur_div;
        s_out.pose = (void*)cur_pose;
        s_out.act = (void*)cur_act;
        s_out.steps = (int32_t*)cur_steps;
        s_out.div = (uint8_t*)cur_div;
        st_release_gpu(&sy->go, v);
        // like every other CTA, acquire the republished word: a GPU-scope acquire
        // invalidates this SM's L1, so the command rows below are fetched fresh
        // from host memory (a system-scope acquire fence here cost 4.4 us/step)
        (void)ld_acquire_gpu(&sy->go);
      } else {
        while ((v = ld_acquire_gpu(&sy->go)) == seq) __nanosleep(64);
        s_cmd = *(volatile uint64_t*)&sy->cmd;
        s_ld = *(volatile int64_t*)&sy->cmd_ld;
        s_out.pose = (void*)*(volatile uint64_t*)&sy->pose;
        s_out.act = (void*)*(volatile uint64_t*)&sy->act;
        s_out.steps = (int32_t*)*(volatile uint64_t*)&sy->steps;
        s_out.div = (uint8_t*)*(volatile uint64_t*)&sy->div;
      }
      s_out.n_act = sa.n_act;
      s_out.any = s_out.pose != nullptr || s_out.act != nullptr || s_out.steps != nullptr ||
                  s_out.div != nullptr;
      s_seq = v;
    }
    __syncthreads();
    const uint64_t v = s_seq;
    if (v == kServeQuit) break;
    const bool stamp = sa.stamps && blockIdx.x == 0 && threadIdx.x == 0;
    if (live) {
      // plain coalesced loads over the link (after the GPU-scope acquire above;
      // L1-bypassing .cg/.cv loads of host memory were far slower at scale)
      const R* crow = (const R*)s_cmd + i * s_ld;
      const int A = AC > 0 ? AC : a.hull[in.ty].r.n_act;
#pragma unroll
      for (int j = 0; j < UUV_MAX_ACT; ++j)
        in.u[j] = (j < A) ? clip_<R>(crow[j], R(-1), R(1)) : R(0);
      if (stamp) sa.ctl->stamp[2] = global_ns() + (uint64_t)(in.u[0] > R(2));
      if constexpr (NT > 1 && sizeof(R) == 8) {
        if (diag_class(a.cls[in.ty])) serve_env<R, NT, DR, 0, true>(a, i, in, s_out);
        else serve_env<R, NT, DR, 0, false>(a, i, in, s_out);
      } else if constexpr (NT > 1) {
        switch (a.cls[in.ty]) {
          case 1: serve_env<R, NT, DR, 6, true>(a, i, in, s_out); break;
          case 2: serve_env<R, NT, DR, 8, true>(a, i, in, s_out); break;
          case 3: serve_env<R, NT, DR, 6, false>(a, i, in, s_out); break;
          case 4: serve_env<R, NT, DR, 8, false>(a, i, in, s_out); break;
          case 5: serve_env<R, NT, DR, 0, true>(a, i, in, s_out); break;
          case 6: serve_env<R, NT, DR, kFinLayout, true>(a, i, in, s_out); break;
          case 7: serve_env<R, NT, DR, kFinLayout, false>(a, i, in, s_out); break;
          default: serve_env<R, NT, DR, 0, false>(a, i, in, s_out); break;
        }
      } else {
        serve_env<R, NT, DR, AC, DM, LEAN>(a, i, in, s_out);
      }
    }
    if (stamp) sa.ctl->stamp[3] = global_ns() + (uint64_t)(in.px > R(1e30));
    // One system-scope fence per step: CTAs publish their stores at GPU scope
    // and count in; the last one fences at system scope (cumulative) and
    // releases the host's done flag.
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&sy->arrived, 1u) == gridDim.x - 1) {
        __threadfence();
        sy->arrived = 0;
        if (sa.stamps) sa.ctl->stamp[4] = global_ns();
        __threadfence_system();
        if (sa.stamps) sa.ctl->stamp[5] = global_ns();
        st_release_sys(sa.done, v);
      }
    }
    seq = v;
  }
}

// ------------------------------------------------------------------ task step
template <typename R> struct TaskArgs {
  Hull<R> hull[1];
  StateView<R> sv;
  TaskR<R> task;
  uuv_sampler smp;
  uint64_t seed;
  const R* cmd;
  int64_t cmd_ld;
  int32_t K;
  R dt_sub;
  R dt;  // control dt (time / tracking reference)
  double dt64;
  R* prev_u;
  R* dev_sum;
  R* obs;
  int64_t obs_ld;
  R* term_obs;
  R* rout;
  uint8_t* fout;
  double* stats;
  R* trace;
  int64_t trace_ld;
  // policy population + episode bookkeeping (uuv_policy_step only)
  const R* pol_theta;
  int64_t pol_ld;
  int32_t pol_members, pol_slot;
  double* ep_ret;
  R* ep_metric;
  uint8_t* ep_success;
  uint8_t* ep_pending;
  int32_t* ep_live;
  int32_t ep_t;
  const uint8_t* mask;  // task reset only
  int32_t mode;         // task reset kernel: 0 observe only, 1 reset masked then observe
  int32_t prefetch;     // batch beyond L2: hint the late-read rows into L2 at kernel entry
};

// Write the CTA's staged observation rows out with coalesced stores.
template <typename R>
UUV_D void flush_obs(const R* s_obs, R* obs, int64_t obs_ld, int obs_dim, int64_t row0, int64_t n) {
  const int rows = (int)min((int64_t)kBlock, n - row0);
  const int total = rows * obs_dim;
  if (obs_ld == obs_dim) {  // dense rows: the CTA's rows are one contiguous span
    R* dst = obs + row0 * obs_ld;
    const int bytes = total * (int)sizeof(R);
    if ((((uintptr_t)dst | (uintptr_t)s_obs) & 15) == 0) {  // 16-byte vector copies
      const int v = bytes >> 4;
      for (int e = threadIdx.x; e < v; e += kBlock)
        reinterpret_cast<uint4*>(dst)[e] = reinterpret_cast<const uint4*>(s_obs)[e];
      for (int e = (v << 4) / (int)sizeof(R) + threadIdx.x; e < total; e += kBlock) dst[e] = s_obs[e];
    } else {
      for (int e = threadIdx.x; e < total; e += kBlock) dst[e] = s_obs[e];
    }
    return;
  }
  for (int e = threadIdx.x; e < total; e += kBlock) {  // strided rows
    const int r = e / obs_dim, c = e - r * obs_dim;
    obs[(row0 + r) * obs_ld + c] = s_obs[e];
  }
}

// u = tanh(W_m obs + b_m) for the row's population member (baseline.py:62-64,
// 164-169): products summed in obs order without contraction, then + b.
template <typename R>
UUV_D void policy_command(const TaskArgs<R>& a, int A, int od, int64_t i, const R* obs, R* raw) {
  const int64_t m = i / a.pol_slot;
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j) raw[j] = R(0);
  if (m >= a.pol_members) return;  // rows past members * slot act with 0
  const R* th = a.pol_theta + m * a.pol_ld;
  // fully unrolled to the widest observation (predicated): every theta load is
  // issued up front and the A dot products interleave, instead of one
  // load-multiply-add chain of A * obs_dim steps
  R ob[kObsMax];
#pragma unroll
  for (int k = 0; k < kObsMax; ++k) ob[k] = k < od ? obs[k] : R(0);
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j) {
    if (j < A) {
      const R* w = th + j * od;
      R acc = R(0);
#pragma unroll
      for (int k = 0; k < kObsMax; ++k)
        if (k < od) acc = add_rn(acc, mul_rn(__ldg(w + k), ob[k]));
      raw[j] = tanh(add_rn(acc, __ldg(th + A * od + j)));
    }
  }
}

// Inputs of one env's task step (loaded from global memory, or carried in registers
// across the steps of the fused policy episode).
template <typename R> struct TaskIn {
  R raw[UUV_MAX_ACT];  // commands as given (unclipped; recorded in the trace)
  R pu[UUV_MAX_ACT];   // previous clipped command (tasks/core.py:333-335)
  R px, py, pz, nu[6], act[UUV_MAX_ACT];
  Q4<R> q;
  R dev;               // tracking deviation accumulator
  V3<R> cur;
  int32_t steps;
  bool div, has_cur;
};

template <typename R>
UUV_D void task_in_global(const TaskArgs<R>& a, int64_t i, bool load_cmd, TaskIn<R>& in) {
  const StateView<R>& sv = a.sv;
  const int A = a.hull[0].r.n_act;
  const int64_t ld = sv.ld;
  if (load_cmd) {  // command loads first: they are the longest-latency inputs
    const R* crow = a.cmd + i * a.cmd_ld;
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) in.raw[j] = j < A ? crow[j] : R(0);
  }
  in.steps = sv.steps[i];
  in.div = sv.diverged[i] != 0;
  load_state(sv, i, A, in.px, in.py, in.pz, in.q, in.nu, in.act);
  (void)ld;  // prev_u, dev_sum and the current are read where they are used (task_env)
}

// One env of VecTaskEnv.step (tasks/core.py:328-370): clip, physics (K substeps),
// reward / termination / info, auto-reset, next observation (staged at srow),
// state / prev_u / dev_sum stores, trace record, statistics into st.  The DR
// record is read at (ov, ov_ld, ov_i).  CARRY (the fused episode loop): previous
// command, current and deviation sum come from `in`, and the step's result is
// written back into `in` for the next step; otherwise they are loaded from global
// memory where they are used (shorter live ranges for the one-step kernel).
template <typename R, bool DR, int AC, bool DM, bool POL, bool CARRY = false, int LEAN = 0>
UUV_D void task_env(const TaskArgs<R>& a, int64_t i, TaskIn<R>& in, const double* ov,
                    int64_t ov_ld, int64_t ov_i, R* srow, double* st, bool& live) {
  const StateView<R>& sv = a.sv;
  const Hull<R>& H = a.hull[0];
  const TaskR<R>& T = a.task;
  const int A = H.r.n_act;
  const int64_t ld = sv.ld;
  if constexpr (POL) {
    // the observation the last step returned, recomputed from the stored state
    R pu[UUV_MAX_ACT];
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) pu[j] = j < A ? (CARRY ? in.pu[j] : a.prev_u[j * ld + i]) : R(0);
    observe_row<R>(T, A, in.px, in.py, in.pz, in.q, in.nu, pu, in.steps, a.dt, srow, nullptr);
    policy_command<R>(a, A, T.obs_dim, i, srow, in.raw);
  }
  // u = clip(commands); du = u - prev_u; prev_u = u  (tasks/core.py:329-335)
  R u[UUV_MAX_ACT], du[UUV_MAX_ACT];
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j) {
    if (j < A) {
      u[j] = clip_<R>(in.raw[j], R(-1), R(1));
      du[j] = u[j] - (CARRY ? in.pu[j] : a.prev_u[j * ld + i]);
    } else {
      u[j] = R(0);
      du[j] = R(0);
    }
  }
  R px = in.px, py = in.py, pz = in.pz;
  Q4<R> q = in.q;
  R* nu = in.nu;
  R* act = in.act;
  bool div = in.div;
  int32_t steps = in.steps;
  if (!div) {
    if (CARRY)
      div = physics_at<R, DR, AC, DM, false, LEAN>(H, sv, i, ov, ov_ld, ov_i, in.has_cur, in.cur, a.K,
                                      a.dt_sub, u, px, py, pz, q, nu, act);
    else
      div = physics<R, DR, AC, DM, false, LEAN>(H, sv, i, a.K, a.dt_sub, u, px, py, pz, q, nu, act);
  }
  steps += 1;
  R dev = CARRY ? in.dev : (a.dev_sum != nullptr ? a.dev_sum[i] : R(0));
  TaskOut<R> o;
  task_eval<R>(T, A, px, py, pz, q, nu, du, steps, div, a.dt, &dev, o);
  if (a.rout != nullptr) {
    a.rout[UUV_TR_REWARD * ld + i] = o.reward;
    a.rout[UUV_TR_POS_ERR * ld + i] = o.pos_err;
    a.rout[UUV_TR_ATT_ERR * ld + i] = o.att_err;
    a.rout[UUV_TR_METRIC * ld + i] = o.metric;
    a.rout[UUV_TR_TIME * ld + i] = o.time;
    if (T.kind == UUV_TASK_DOCKING) {
      a.rout[UUV_TR_CONTACT_DIST * ld + i] = o.c_dist;
      a.rout[UUV_TR_CONTACT_SPEED * ld + i] = o.c_speed;
      a.rout[UUV_TR_CONTACT_ATT * ld + i] = o.c_att;
    }
  }
  if (a.fout != nullptr) {
    a.fout[UUV_TF_TERMINATED * ld + i] = o.terminated;
    a.fout[UUV_TF_TRUNCATED * ld + i] = o.truncated;
    a.fout[UUV_TF_FINISHED * ld + i] = o.finished;
    a.fout[UUV_TF_FAILURE * ld + i] = o.failure;
    a.fout[UUV_TF_SUCCESS * ld + i] = o.success;
    a.fout[UUV_TF_DIVERGED * ld + i] = div;
    a.fout[UUV_TF_CONTACT * ld + i] = o.contact;
  }
  if constexpr (POL) {
    if (a.ep_ret != nullptr && a.ep_pending[i]) {  // _rollout_returns (baseline.py:116-123)
      a.ep_ret[i] += (double)o.reward;
      if (o.finished) {
        a.ep_metric[i] = o.metric;
        a.ep_success[i] = o.success;
        a.ep_pending[i] = 0;
      } else {
        live = true;
      }
    }
  }
  {  // statistics: one env per thread sets them, the fused episode loop sums its steps
    const double v[UUV_ST_COUNT] = {(double)o.reward, (double)o.finished, (double)o.success,
                                    (double)o.failure, (double)o.truncated,
                                    o.finished ? (double)o.metric : 0.0, (double)div, 1.0};
#pragma unroll
    for (int k = 0; k < UUV_ST_COUNT; ++k) st[k] = CARRY ? st[k] + v[k] : v[k];
  }
  if (o.finished) {
    if (a.term_obs != nullptr)  // final observation of the ended episode
      observe_row<R>(T, A, px, py, pz, q, nu, u, steps, a.dt, a.term_obs + i * a.obs_ld, nullptr);
    V3<R> cur;
    reset_env<R>(sv, i, a.smp, a.seed, px, py, pz, q, nu, cur);
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) { act[j] = R(0); u[j] = R(0); }
    steps = 0;
    div = false;
    dev = R(0);
    if (CARRY) in.cur = cur;
  }
  // (the policy episode loop passes no obs buffer: its next launch recomputes
  // the observation from the stored state)
  if (a.obs != nullptr) observe_row<R>(T, A, px, py, pz, q, nu, u, steps, a.dt, srow, nullptr);
  store_state(sv, i, A, px, py, pz, q, nu, act);
  sv.steps[i] = steps;
  sv.diverged[i] = div ? 1 : 0;
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j)
    if (j < A) a.prev_u[j * ld + i] = u[j];
  if (a.dev_sum != nullptr) a.dev_sum[i] = dev;
  if (a.trace != nullptr) {  // rollout record (cli.py:277-287), coalesced SoA rows
    R* tr = a.trace + i;
    const int64_t tl = a.trace_ld;
    tr[(UUV_TRACE_P + 0) * tl] = px;
    tr[(UUV_TRACE_P + 1) * tl] = py;
    tr[(UUV_TRACE_P + 2) * tl] = pz;
    tr[(UUV_TRACE_Q + 0) * tl] = q.w;
    tr[(UUV_TRACE_Q + 1) * tl] = q.x;
    tr[(UUV_TRACE_Q + 2) * tl] = q.y;
    tr[(UUV_TRACE_Q + 3) * tl] = q.z;
#pragma unroll
    for (int k = 0; k < 6; ++k) tr[(UUV_TRACE_NU + k) * tl] = nu[k];
    tr[UUV_TRACE_REWARD * tl] = o.reward;
    tr[UUV_TRACE_T * tl] = (R)(__dmul_rn((double)steps, a.dt64));
    for (int j = 0; j < A; ++j) tr[(UUV_TRACE_CMD + j) * tl] = in.raw[j];
  }
  if (CARRY) {  // the next step continues from registers (nu, act were updated in place)
    in.px = px; in.py = py; in.pz = pz;
    in.q = q;
    in.steps = steps;
    in.div = div;
    in.dev = dev;
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) in.pu[j] = u[j];
  }
}

// Deterministic CTA reduction of the per-thread statistics of one step (fixed shuffle
// tree, then warps in order) added to this CTA's slot.  The six counters are 0/1 per
// thread: a ballot and a popcount per warp (exact, as the float64 sums of 0/1 are)
// instead of five shuffle rounds of a double each.
UUV_D void cta_stats(const double* st, double (*s_red)[UUV_ST_COUNT], double* slot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < UUV_ST_COUNT; ++k) {
    if (k == UUV_ST_REWARD || k == UUV_ST_METRIC_FINISHED) {
      double v = st[k];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      if (lane == 0) s_red[warp][k] = v;
    } else {
      const int c = __popc(__ballot_sync(0xffffffffu, st[k] != 0.0));
      if (lane == 0) s_red[warp][k] = (double)c;
    }
  }
  __syncthreads();
  if (threadIdx.x < UUV_ST_COUNT) {
    double v = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) v += s_red[w][threadIdx.x];
    slot[threadIdx.x] += v;
  }
}

// HI: a 96-register build (5 CTAs per SM) of the lean eight-thruster task step for
// batches past L2, where more resident warps hide more HBM latency (config 5 at 1M
// envs 171.6 -> 163.5 us); the six-thruster K = 8 kernel is issue-bound and loses
// with it (202 -> 213 us), as does every class at small batches.
template <typename R, bool DR, int AC, bool DM, bool POL = false, int LEAN = 0, bool HI = false>
__global__ void __launch_bounds__(kBlock, HI ? 5 : MinBTask<R>::value)
    k_task_step(const __grid_constant__ TaskArgs<R> a) {
  __shared__ __align__(16) R s_obs[kBlock * kObsMax];
  __shared__ double s_red[kBlock / 32][UUV_ST_COUNT];
  if (POL && a.ep_live != nullptr && a.ep_live[a.ep_t - 1] == 0) return;  // the episode loop broke
  bool live = false;
  const int64_t row0 = (int64_t)blockIdx.x * kBlock;
  const int64_t i = row0 + threadIdx.x;
  const StateView<R>& sv = a.sv;
  const int od = a.task.obs_dim;
  double st[UUV_ST_COUNT];
#pragma unroll
  for (int k = 0; k < UUV_ST_COUNT; ++k) st[k] = 0.0;
  if (a.prefetch && i < sv.n) {
    // rows read only after the diverged-flag branch (DR record, current) or late
    // (previous command, deviation sum): start their DRAM reads into L2 now, so
    // those loads hit L2 instead of adding a second DRAM round trip per env
    prefetch_overlay_l2(sv, i);
    const int64_t ld = sv.ld;
    if (sv.cur != nullptr)
      for (int c = 0; c < 3; ++c) asm volatile("prefetch.global.L2 [%0];" ::"l"(sv.cur + c * ld + i));
    for (int j = 0; j < a.hull[0].r.n_act; ++j)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.prev_u + j * ld + i));
    if (a.dev_sum != nullptr) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.dev_sum + i));
  }
  if (i < sv.n) {
    TaskIn<R> in;
    task_in_global<R>(a, i, !POL, in);
    task_env<R, DR, AC, DM, POL, false, LEAN>(a, i, in, sv.ov, sv.ld, i, s_obs + threadIdx.x * od,
                                              st, live);
  }
  if constexpr (POL) {
    if (a.ep_live != nullptr) {
      const int cnt = __syncthreads_count(live);
      if (threadIdx.x == 0 && cnt != 0) atomicAdd(a.ep_live + a.ep_t, cnt);
    }
  }
  __syncthreads();
  if (a.obs != nullptr) flush_obs<R>(s_obs, a.obs, a.obs_ld, od, row0, sv.n);
  if (a.stats != nullptr) cta_stats(st, s_red, a.stats + blockIdx.x * UUV_ST_COUNT);
}

// ------------------------------------------------------------------ fused policy episode
// One whole episode loop of baseline._rollout_returns (baseline.py:109-127) in ONE
// launch: every thread keeps its env's state in registers across the steps
// (task_env<CARRY>) -- policy command, physics, reward / termination, auto-reset,
// return bookkeeping -- and the grid stops after the first step t at which no row
// of the WHOLE batch is pending, exactly where the reference loop breaks: per step,
// each CTA adds its pending count to live[t] and arrives on that step's counter
// (live[length + 1 + t]).  A CTA that still has pending rows knows the loop goes on
// and continues at once; only a CTA with none waits for every CTA's step-t arrival
// before reading live[t] (if all of them have none, all of them wait, read 0 and
// stop together).  The grid must be co-resident (checked on the host); same
// per-step results as `length` uuv_policy_step launches.
UUV_D uint32_t ld_acquire_gpu_i32(const int32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename R, bool DR, int AC, bool DM, int LEAN = 0>
__global__ void __launch_bounds__(kBlock, MinBTask<R>::value)
    k_policy_episode(const __grid_constant__ TaskArgs<R> a, int32_t length) {
  __shared__ __align__(16) R s_obs[kBlock * kObsMax];
  __shared__ int s_go;
  const StateView<R>& sv = a.sv;
  const int A = a.hull[0].r.n_act;
  const int od = a.task.obs_dim;
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool on = i < sv.n;
  const int64_t ld = sv.ld;
  int32_t* arrive = a.ep_live + length + 1;  // arrive[t]: CTAs done with step t
  TaskIn<R> in;
  if (on) {
    task_in_global<R>(a, i, false, in);
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) in.pu[j] = j < A ? a.prev_u[j * ld + i] : R(0);
    in.dev = a.dev_sum != nullptr ? a.dev_sum[i] : R(0);
    in.has_cur = sv.cur != nullptr;
    in.cur = V3<R>{R(0), R(0), R(0)};
    if (in.has_cur) in.cur = V3<R>{sv.cur[i], sv.cur[ld + i], sv.cur[2 * ld + i]};
  }
  double st[UUV_ST_COUNT];
#pragma unroll
  for (int k = 0; k < UUV_ST_COUNT; ++k) st[k] = 0.0;
  for (int t = 1; t <= length; ++t) {
    bool live = false;
    if (on)
      task_env<R, DR, AC, DM, true, true, LEAN>(a, i, in, sv.ov, sv.ld, i,
                                                s_obs + threadIdx.x * od, st, live);
    const int cnt = __syncthreads_count(live);
    if (threadIdx.x == 0) {
      if (cnt != 0) atomicAdd(a.ep_live + t, cnt);
      __threadfence();
      atomicAdd(arrive + t, 1);
      if (cnt != 0) {
        s_go = 1;  // this CTA's own rows keep the loop going
      } else {
        while (ld_acquire_gpu_i32(arrive + t) < gridDim.x) __nanosleep(20);
        s_go = ld_acquire_gpu_i32(a.ep_live + t) != 0;
      }
    }
    __syncthreads();
    if (!s_go) break;  // no row of the batch is pending: the reference loop's break
  }
}

// Task reset (mode 1: masked rows reset, prev_u / dev_sum cleared) + observe all rows.
template <typename R>
__global__ void __launch_bounds__(kBlock) k_task_reset(const __grid_constant__ TaskArgs<R> a) {
  __shared__ __align__(16) R s_obs[kBlock * kObsMax];
  const int64_t row0 = (int64_t)blockIdx.x * kBlock;
  const int64_t i = row0 + threadIdx.x;
  const StateView<R>& sv = a.sv;
  const TaskR<R>& T = a.task;
  const int A = a.hull[0].r.n_act;
  const int64_t ld = sv.ld;
  if (i < sv.n) {
    R px, py, pz, nu[6], act[UUV_MAX_ACT], pu[UUV_MAX_ACT];
    Q4<R> q;
    load_state(sv, i, A, px, py, pz, q, nu, act);
    int32_t steps = sv.steps[i];
    const bool do_reset = a.mode == 1 && (a.mask == nullptr || a.mask[i] != 0);
    if (do_reset) {
      V3<R> cur;
      reset_env<R>(sv, i, a.smp, a.seed, px, py, pz, q, nu, cur);
#pragma unroll
      for (int j = 0; j < UUV_MAX_ACT; ++j) act[j] = R(0);
      steps = 0;
      store_state(sv, i, A, px, py, pz, q, nu, act);
      sv.steps[i] = 0;
      sv.diverged[i] = 0;
      for (int j = 0; j < A; ++j) a.prev_u[j * ld + i] = R(0);
      if (a.dev_sum != nullptr) a.dev_sum[i] = R(0);
    }
#pragma unroll
    for (int j = 0; j < UUV_MAX_ACT; ++j) pu[j] = j < A ? a.prev_u[j * ld + i] : R(0);
    observe_row<R>(T, A, px, py, pz, q, nu, pu, steps, a.dt, s_obs + threadIdx.x * T.obs_dim,
                   nullptr);
  }
  __syncthreads();
  flush_obs<R>(s_obs, a.obs, a.obs_ld, T.obs_dim, row0, sv.n);
}

// ------------------------------------------------------------------ engine reset
template <typename R> struct ResetArgs {
  StateView<R> sv;
  uuv_sampler smp;
  uint64_t seed;
  const uint8_t* mask;
  int32_t a_max;
};

template <typename R>
__global__ void __launch_bounds__(kBlock) k_reset(const __grid_constant__ ResetArgs<R> a) {
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const StateView<R>& sv = a.sv;
  if (i >= sv.n) return;
  if (a.mask != nullptr && a.mask[i] == 0) return;
  R px, py, pz, nu[6];
  Q4<R> q;
  V3<R> cur;
  reset_env<R>(sv, i, a.smp, a.seed, px, py, pz, q, nu, cur);
  R act[UUV_MAX_ACT];
#pragma unroll
  for (int j = 0; j < UUV_MAX_ACT; ++j) act[j] = R(0);
  store_state(sv, i, a.a_max, px, py, pz, q, nu, act);
  sv.steps[i] = 0;
  sv.diverged[i] = 0;
}

// ------------------------------------------------------------------ statistics
#if UUV_TU_MAIN
static __global__ void k_stats(const double* stats, int64_t n_blocks, double* out, int32_t reset,
                        double* stats_rw) {
  // one CTA; thread k sums statistic k over blocks in index order (deterministic)
  const int k = threadIdx.x;
  if (k >= UUV_ST_COUNT) return;
  double v = 0.0;
  for (int64_t b = 0; b < n_blocks; ++b) v += stats[b * UUV_ST_COUNT + k];
  out[k] = v;
  if (reset)
    for (int64_t b = 0; b < n_blocks; ++b) stats_rw[b * UUV_ST_COUNT + k] = 0.0;
}
#endif

// ------------------------------------------------------------------ inspection kernels
template <typename R, int NT> struct DeriveArgs {
  Hull<R> hull[NT];
  StateView<R> sv;
  double* out12;
  double* minv;
  double* ct_tau;
  double* mounts;
};

template <typename R, int NT>
__global__ void __launch_bounds__(kBlock) k_derive(const __grid_constant__ DeriveArgs<R, NT> a) {
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const StateView<R>& sv = a.sv;
  if (i >= sv.n) return;
  const Hull<R>& H = a.hull[NT > 1 ? (int)sv.type_id[i] : 0];
  EnvD e;
  if (sv.ov != nullptr) {
    derive_env(H.d, sv.ov, sv.ld, i, sv.slot, e);
  } else {
    e.mass = H.d.mass; e.volume = H.d.volume; e.W = H.d.mass * H.d.g; e.B = H.d.rhog * H.d.volume;
    e.a = e.d = e.rt = e.rc = 1.0;
    for (int c = 0; c < 3; ++c) { e.r_g[c] = H.d.r_g[c]; e.r_b[c] = H.d.r_b[c]; }
    for (int k = 0; k < 9; ++k) e.I[k] = H.d.inertia[k];
  }
  if (a.out12 != nullptr) {
    double* o = a.out12 + i * 12;
    o[0] = e.mass; o[1] = e.volume;
    for (int c = 0; c < 3; ++c) { o[2 + c] = e.r_g[c]; o[5 + c] = e.r_b[c]; }
    o[8] = e.W; o[9] = e.B; o[10] = e.a; o[11] = e.d;
  }
  if (a.minv != nullptr) {  // M^-1 columns by LDL^T solves of unit vectors
    double M[21], L[15], Di[6];
    mass_matrix_d(H.d, e, M);
    ldl6_factor<double>(M, L, Di, Rcp<double>());
    for (int c = 0; c < 6; ++c) {
      double b[6] = {0, 0, 0, 0, 0, 0}, x[6];
      b[c] = 1.0;
      ldl6_apply<double>(L, Di, b, x);
      for (int r = 0; r < 6; ++r) a.minv[i * 36 + 6 * r + c] = x[r];
    }
  }
  const int am = sv.a_max;
  for (int j = 0; j < am; ++j) {
    if (a.ct_tau != nullptr) {
      a.ct_tau[i * 2 * am + j] = __dmul_rn(H.d.ct[j], e.rc);
      a.ct_tau[i * 2 * am + am + j] = __dmul_rn(H.d.tc[j], e.rt);
    }
    if (a.mounts != nullptr) {
      for (int c = 0; c < 3; ++c) {
        double m = H.d.mount[j][c];
        if (sv.ov != nullptr && sv.slot[UUV_OV_JITTER] >= 0)
          m = __dadd_rn(m, sv.ov[(sv.slot[UUV_OV_JITTER] + 3 * j + c) * sv.ld + i]);
        a.mounts[(i * am + j) * 3 + c] = m;
      }
    }
  }
}

template <typename R, int NT> struct TermsArgs {
  Hull<R> hull[NT];
  StateView<R> sv;
  const R* cmd;
  int64_t cmd_ld;
  R dt;
  double* out;
};

template <typename R, int NT, bool DR, int AC, bool DM>
__global__ void __launch_bounds__(kBlock) k_terms(const __grid_constant__ TermsArgs<R, NT> a) {
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const StateView<R>& sv = a.sv;
  if (i >= sv.n) return;
  const Hull<R>& H = a.hull[NT > 1 ? (int)sv.type_id[i] : 0];
  const int A = H.r.n_act;
  R u[UUV_MAX_ACT];
  for (int j = 0; j < UUV_MAX_ACT; ++j)
    u[j] = j < A ? clip_<R>(a.cmd[i * a.cmd_ld + j], R(-1), R(1)) : R(0);
  R px, py, pz, nu[6], act[UUV_MAX_ACT];
  Q4<R> q;
  load_state(sv, i, A, px, py, pz, q, nu, act);
  Sub<R> s;
  const double* jit = nullptr;
  if (DR) {
    EnvD e;
    derive_env(H.d, sv.ov, sv.ld, i, sv.slot, e);
    sub_from_env<R, DM>(H.r, e, s);
    if (sv.slot[UUV_OV_JITTER] >= 0) jit = sv.ov + sv.slot[UUV_OV_JITTER] * sv.ld + i;
  }
  const bool has_cur = sv.cur != nullptr;
  V3<R> cur{R(0), R(0), R(0)};
  if (has_cur) cur = V3<R>{sv.cur[i], sv.cur[sv.ld + i], sv.cur[2 * sv.ld + i]};
  Terms<R> tm;
  const bool ok = substep<R, DR, true, AC, DM>(H.r, s, jit, sv.ld, px, py, pz, q, nu, act, u, has_cur, cur,
                                       a.dt, &tm);
  double* o = a.out + i * 48;
  for (int k = 0; k < 6; ++k) {
    o[k] = tm.tau[k]; o[6 + k] = tm.hydro[k]; o[12 + k] = tm.c_rb[k]; o[18 + k] = tm.acc[k];
    o[24 + k] = nu[k];
  }
  o[30] = px; o[31] = py; o[32] = pz;
  o[33] = q.w; o[34] = q.x; o[35] = q.y; o[36] = q.z;
  for (int j = 0; j < UUV_MAX_ACT; ++j) o[37 + j] = act[j];
  o[45] = ok ? 1.0 : 0.0;
  o[46] = o[47] = 0.0;
}

// ================================================================== host dispatch
namespace {

int64_t grid_for(int64_t n) { return (n + kBlock - 1) / kBlock; }

uuv_status check_state(const uuv_ctx* ctx, const uuv_state* st) {
  if (ctx == nullptr || st == nullptr) return fail(UUV_ERR_ARG, "null ctx or state");
  if (st->dtype != UUV_F32 && st->dtype != UUV_F64)
    return fail(UUV_ERR_ARG, "state: unknown dtype %d", st->dtype);
  if (st->n_envs < 0 || st->ld < st->n_envs) return fail(UUV_ERR_SHAPE, "state: ld < n_envs");
  if (st->a_max < 1 || st->a_max > UUV_MAX_ACT)
    return fail(UUV_ERR_SHAPE, "state: a_max %d outside [1, %d]", st->a_max, UUV_MAX_ACT);
  if (!st->p || !st->q || !st->nu || !st->act || !st->steps || !st->episodes || !st->diverged)
    return fail(UUV_ERR_ARG, "state: null state array");
  if (ctx->hulls.empty()) return fail(UUV_ERR_ARG, "context has no hulls");
  if (ctx->hulls.size() > 1 && st->type_id == nullptr)
    return fail(UUV_ERR_ARG, "state: mixed fleet needs type_id");
  for (const auto& h : ctx->hulls)
    if (h.n_act > st->a_max) return fail(UUV_ERR_SHAPE, "state: a_max < hull actuators");
  if (st->overlay != nullptr)
    for (int k = 0; k < UUV_OV_COUNT; ++k)
      if (st->slot[k] >= st->n_slots) return fail(UUV_ERR_SHAPE, "state: slot beyond n_slots");
  if (st->n_runs < 0 || st->n_runs > UUV_MAX_RUNS)
    return fail(UUV_ERR_ARG, "state: n_runs %d outside [0, %d]", st->n_runs, UUV_MAX_RUNS);
  for (int r = 0; r < st->n_runs; ++r) {
    if (st->run_type[r] < 0 || st->run_type[r] >= (int)ctx->hulls.size())
      return fail(UUV_ERR_ARG, "state: run %d has no hull", r);
    if ((r == 0 && st->run_start[0] != 0) || (r > 0 && st->run_start[r] < st->run_start[r - 1]) ||
        st->run_start[r] > st->n_envs)
      return fail(UUV_ERR_ARG, "state: run starts must ascend from 0 within n_envs");
  }
  return UUV_OK;
}

// Actuator class of a hull (see substep): A first-order thrusters, else 0.
int hull_act_class(const uuv_hull& h) {
  for (int j = 0; j < h.n_act; ++j)
    if (h.model[j] != UUV_FIRST_ORDER) return 0;
  if (h.n_act == kFinLayout) {  // a propeller / tilt rotor, then four fins
    if (h.kind[0] == UUV_RUDDER) return 0;
    for (int j = 1; j < kFinLayout; ++j)
      if (h.kind[j] != UUV_RUDDER) return 0;
    return kFinLayout;
  }
  if (h.n_act != 6 && h.n_act != 8) return 0;
  for (int j = 0; j < h.n_act; ++j)
    if (h.kind[j] == UUV_RUDDER) return 0;
  return h.n_act;
}

int act_class(const uuv_ctx* ctx) {
  return ctx->hulls.size() == 1 ? hull_act_class(ctx->hulls[0]) : 0;
}

// Every env's composite mass matrix is diagonal: single diagonal hull with r_g = 0
// and diagonal inertia, and no payload placed off the origin.
bool hull_diag_mass(const uuv_hull& h, const uuv_state* st) {
  if (!(is_diag(h.M_A) && is_diag(h.D_lin) && is_diag(h.D_quad))) return false;
  if (h.r_g[0] != 0.0 || h.r_g[1] != 0.0 || h.r_g[2] != 0.0) return false;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      if (r != c && h.inertia[3 * r + c] != 0.0) return false;
  if (st->overlay != nullptr && st->slot[UUV_OV_PAYLOAD_POS] >= 0 &&
      !(st->flags & UUV_STATE_PAYLOAD_AT_ORIGIN))
    return false;
  return true;
}

bool diag_mass(const uuv_ctx* ctx, const uuv_state* st) {
  return ctx->hulls.size() == 1 && hull_diag_mass(ctx->hulls[0], st);
}

// Specialisation code of each type of a mixed fleet (step_any).
int8_t hull_class(const uuv_hull& h, const uuv_state* st) {
  const int ac = hull_act_class(h);
  const bool dm = hull_diag_mass(h, st);
  if (ac == 6) return dm ? 1 : 3;
  if (ac == 8) return dm ? 2 : 4;
  if (ac == kFinLayout) return dm ? 6 : 7;
  return dm ? 5 : 0;
}

template <typename R> const std::vector<Hull<R>>& hulls_of(const uuv_ctx* c);
template <> const std::vector<Hull<float>>& hulls_of<float>(const uuv_ctx* c) { return c->hf; }
template <> const std::vector<Hull<double>>& hulls_of<double>(const uuv_ctx* c) { return c->hd; }

template <typename R, int NT>
void fill_hulls(const uuv_ctx* ctx, Hull<R>* dst, double dt_sub, int first = 0) {
  const auto& hs = hulls_of<R>(ctx);
  for (int t = 0; t < NT; ++t) {
    dst[t] = hs[first + t < (int)hs.size() ? first + t : 0];
    for (int j = 0; j < UUV_MAX_ACT; ++j) dst[t].r.kdt0[j] = (R)(dt_sub / dst[t].d.tc[j]);
  }
}

// A lean batch: float32, K = 1, no current, no reaction torques on the hull, no mount
// jitter.  Every single-hull step-family kernel (k_step -- also each per-type run of a
// large fleet --, k_rollout, k_serve) takes the branch-free substep<LEAN> for it and
// the general one otherwise, so their results stay bit-identical to each other (the
// compiler contracts multiply-adds per basic block: one substep body with and one
// without branches round differently in the last bit).  Mixed-fleet kernels (one
// launch over every type) keep the general substep.
template <typename R>
bool lean_batch(const uuv_ctx* ctx, const uuv_state* st, int32_t K, int hull = 0) {
  if (sizeof(R) != 4 || K != 1) return false;
  if (st->current_ned != nullptr) return false;
  if (st->overlay != nullptr && st->slot[UUV_OV_JITTER] >= 0) return false;
  const uuv_hull& h = ctx->hulls[hull];
  for (int j = 0; j < h.n_act; ++j)
    if (h.reaction[j] != 0.0) return false;
  return true;
}

// A lean task batch (float32 task / policy launches): a six- or eight-thruster hull, no
// reaction torques, no mount jitter -- every task-family kernel (task step, policy
// step, fused episode) then takes the branch-free substep<LEAN>: 3 with the current
// compiled in, 2 without.  0: the general substep.
inline int lean_task(const uuv_ctx* ctx, const uuv_state* st) {
  const uuv_hull& h = ctx->hulls[0];
  const int ac = hull_act_class(h);
  if (ctx->hulls.size() != 1 || (ac != 6 && ac != 8)) return 0;
  if (st->overlay != nullptr && st->slot[UUV_OV_JITTER] >= 0) return 0;
  for (int j = 0; j < h.n_act; ++j)
    if (h.reaction[j] != 0.0) return 0;
  return st->current_ned != nullptr ? 3 : 2;
}

template <typename R, int NT, bool DR, int AC, bool DM = false>
uuv_status launch_step(const uuv_ctx* ctx, const uuv_state* st, const void* cmd, int64_t cmd_ld,
                       int32_t K, double dt, cudaStream_t s, const HostOut* out = nullptr,
                       int hull0 = 0) {
  StepArgs<R, NT> a;
  const double dt_sub = dt / K;
  fill_hulls<R, NT>(ctx, a.hull, dt_sub, hull0);
  for (int t = 0; t < NT; ++t)
    a.cls[t] = hull0 + t < (int)ctx->hulls.size() ? hull_class(ctx->hulls[hull0 + t], st) : 0;
  a.sv = make_view<R>(*st);
  a.cmd = (const R*)cmd;
  a.cmd_ld = cmd_ld;
  a.K = K;
  a.dt = (R)dt_sub;
  a.out = out != nullptr ? *out : HostOut{};
  a.prefetch_ov = st->n_envs >= (int64_t)1 << 19;  // >~100 MB of state + record: past L2
  const int64_t need = grid_for(st->n_envs);
  constexpr bool kHiOk = DR && NT == 1 && sizeof(R) == 4;
  static const int64_t hi_min = [] {
    const char* v = getenv("UUV_HI_OCC_MIN_ENVS");
    return v ? (int64_t)atoll(v) : (int64_t)UUV_HI_OCC_MIN_ENVS;
  }();
  // K = 1 only: with fused substeps the kernel is issue-bound and the uncapped
  // build is faster (cfg2 K = 8: 1M envs 129.4 -> 127.3 us, 4M 503.8 -> 495.1 us)
  const bool hi = kHiOk && st->n_envs >= hi_min && K == 1;
  auto kern = hi ? k_step<R, NT, DR, AC, DM, kHiOk> : k_step<R, NT, DR, AC, DM, false>;
  if constexpr (NT == 1 && sizeof(R) == 4) {
    UUV_REGISTER(k_step<R, NT, DR, AC, DM, false, true>);
    UUV_REGISTER(k_step<R, NT, DR, AC, DM, kHiOk, true>);
    if (lean_batch<R>(ctx, st, K, hull0))
      kern = hi ? k_step<R, NT, DR, AC, DM, kHiOk, true> : k_step<R, NT, DR, AC, DM, false, true>;
  }
  const int64_t wave = one_wave_ctas(kern);
  const int64_t grid = need;  // one thread per env
  // dependent-launch trigger: small grids (<= 64 CTAs) release the next step as
  // soon as their loads are issued (mode 3), larger grids after their stores
  // (mode 2).  Mode 3 overlaps the next step's command fetch with this step's
  // compute: 3.15 -> 2.35 us per step at 4096 envs when commands come from DRAM
  // (bench.py's ring), +3-6% when they are L2-hot (a fixed command tensor); at
  // 16k envs the L2-hot cost reached +12%, hence the cut-off.
  const int pm = pdl_mode();
  a.early_trigger = pm == 4 ? (grid <= 64 ? 3 : 2)
                            : (pm >= 2 ? pm : ((grid <= wave && pdl_enabled()) ? 1 : 0));
  UUV_REGISTER(k_step<R, NT, DR, AC, DM, false>);
  UUV_REGISTER(k_step<R, NT, DR, AC, DM, kHiOk>);
  cudaError_t e = launch_pdl(kern, (unsigned)grid, s, a);
  if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "uuv_step: %s", cudaGetErrorString(e));
  return check_launch("uuv_step");
}

// One specialised single-hull launch for rows of hull `type` (a run of a fleet).
template <typename R>
uuv_status dispatch_one(const uuv_ctx* ctx, const uuv_state* st, int type, const void* cmd,
                        int64_t cmd_ld, int32_t K, double dt, cudaStream_t s) {
  const bool dr = st->overlay != nullptr;
  const uuv_hull& h = ctx->hulls[type];
  const bool dm = hull_diag_mass(h, st);
  switch (hull_act_class(h)) {
    case 6:
      if (dm)
        return dr ? launch_step<R, 1, true, 6, true>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                  : launch_step<R, 1, false, 6, true>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
      return dr ? launch_step<R, 1, true, 6>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                : launch_step<R, 1, false, 6>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
    case 8:
      if (dm)
        return dr ? launch_step<R, 1, true, 8, true>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                  : launch_step<R, 1, false, 8, true>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
      return dr ? launch_step<R, 1, true, 8>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                : launch_step<R, 1, false, 8>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
    case kFinLayout:
      if (dm)
        return dr ? launch_step<R, 1, true, kFinLayout, true>(ctx, st, cmd, cmd_ld, K, dt, s,
                                                              nullptr, type)
                  : launch_step<R, 1, false, kFinLayout, true>(ctx, st, cmd, cmd_ld, K, dt, s,
                                                               nullptr, type);
      return dr ? launch_step<R, 1, true, kFinLayout>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                : launch_step<R, 1, false, kFinLayout>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
    default:
      if (dm)
        return dr ? launch_step<R, 1, true, 0, true>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                  : launch_step<R, 1, false, 0, true>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
      return dr ? launch_step<R, 1, true, 0>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type)
                : launch_step<R, 1, false, 0>(ctx, st, cmd, cmd_ld, K, dt, s, nullptr, type);
  }
}

// Mixed fleet in contiguous per-type runs: one specialised launch per run, the
// runs on forked streams (run 0 on the caller's) so they execute concurrently;
// the caller's stream then joins them.  Same source as the mixed-fleet kernel's
// per-type paths; the separate compilations may contract FMAs differently, so
// results agree to rounding (tests/test_gpu_parity.py::test_fleet_runs...).
static int64_t runs_min_envs() {
  static const int64_t v = [] {
    const char* e = getenv("UUV_RUNS_MIN_ENVS");
    return e ? (int64_t)atoll(e) : (int64_t)131072;
  }();
  return v;
}

template <typename R>
uuv_status dispatch_runs(const uuv_ctx* ctx, const uuv_state* st, const void* cmd, int64_t cmd_ld,
                         int32_t K, double dt, cudaStream_t s) {
  const int nr = st->n_runs;
  cudaError_t e = cudaSuccess;
  while ((int)ctx->fork.size() < nr - 1 && e == cudaSuccess) {
    cudaStream_t fs;
    cudaEvent_t ev;
    e = cudaStreamCreateWithFlags(&fs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) {
      ctx->fork.push_back(fs);
      ctx->done.push_back(ev);
    }
  }
  if (e == cudaSuccess && ctx->forked == nullptr)
    e = cudaEventCreateWithFlags(&ctx->forked, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->forked, s);
  if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "uuv_step (runs): %s", cudaGetErrorString(e));
  const size_t es = sizeof(R);
  for (int r = 0; r < nr; ++r) {
    const int64_t a = st->run_start[r], b = r + 1 < nr ? st->run_start[r + 1] : st->n_envs;
    if (b <= a) continue;
    uuv_state sub = *st;
    auto off = [&](void* p, size_t elem) { return p ? (void*)((char*)p + a * elem) : nullptr; };
    sub.p = off(st->p, es);
    sub.q = off(st->q, es);
    sub.nu = off(st->nu, es);
    sub.act = off(st->act, es);
    sub.current_ned = off(st->current_ned, es);
    sub.steps = (int32_t*)off(st->steps, sizeof(int32_t));
    sub.episodes = (int32_t*)off(st->episodes, sizeof(int32_t));
    sub.diverged = (uint8_t*)off(st->diverged, 1);
    sub.type_id = nullptr;
    sub.overlay = (double*)off(st->overlay, sizeof(double));
    sub.overlay_keys = (uint16_t*)off(st->overlay_keys, sizeof(uint16_t));
    sub.n_envs = b - a;
    sub.env_offset = st->env_offset + a;
    sub.n_runs = 0;
    cudaStream_t rs = r == 0 ? s : ctx->fork[r - 1];
    if (r > 0 && (e = cudaStreamWaitEvent(rs, ctx->forked, 0)) != cudaSuccess) break;
    const uuv_status us = dispatch_one<R>(ctx, &sub, st->run_type[r],
                                          (const char*)cmd + a * cmd_ld * es, cmd_ld, K, dt, rs);
    if (us != UUV_OK) return us;
    if (r > 0 && (e = cudaEventRecord(ctx->done[r - 1], rs)) != cudaSuccess) break;
  }
  for (int r = 1; r < nr && e == cudaSuccess; ++r) e = cudaStreamWaitEvent(s, ctx->done[r - 1], 0);
  if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "uuv_step (runs): %s", cudaGetErrorString(e));
  return UUV_OK;
}

template <typename R>
uuv_status dispatch_step(const uuv_ctx* ctx, const uuv_state* st, const void* cmd, int64_t cmd_ld,
                         int32_t K, double dt, cudaStream_t s, const HostOut* pose = nullptr) {
  if (ctx->hulls.size() > 1 && st->n_runs > 0 && pose == nullptr && st->n_envs >= runs_min_envs())
    return dispatch_runs<R>(ctx, st, cmd, cmd_ld, K, dt, s);
  const bool dr = st->overlay != nullptr;
  if (ctx->hulls.size() == 1) {
    const bool dm = diag_mass(ctx, st);
    switch (act_class(ctx)) {
      case 6:
        if (dm)
          return dr ? launch_step<R, 1, true, 6, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                    : launch_step<R, 1, false, 6, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
        return dr ? launch_step<R, 1, true, 6>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                  : launch_step<R, 1, false, 6>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
      case 8:
        if (dm)
          return dr ? launch_step<R, 1, true, 8, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                    : launch_step<R, 1, false, 8, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
        return dr ? launch_step<R, 1, true, 8>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                  : launch_step<R, 1, false, 8>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
      case kFinLayout:
        if (dm)
          return dr ? launch_step<R, 1, true, kFinLayout, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                    : launch_step<R, 1, false, kFinLayout, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
        return dr ? launch_step<R, 1, true, kFinLayout>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                  : launch_step<R, 1, false, kFinLayout>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
      default:
        if (dm)
          return dr ? launch_step<R, 1, true, 0, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                    : launch_step<R, 1, false, 0, true>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
        return dr ? launch_step<R, 1, true, 0>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
                  : launch_step<R, 1, false, 0>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
    }
  }
  return dr ? launch_step<R, UUV_MAX_TYPES, true, 0>(ctx, st, cmd, cmd_ld, K, dt, s, pose)
            : launch_step<R, UUV_MAX_TYPES, false, 0>(ctx, st, cmd, cmd_ld, K, dt, s, pose);
}

template <typename R, int NT, bool DR, int AC, bool DM = false>
uuv_status launch_rollout(const uuv_ctx* ctx, const uuv_state* st, const RolloutSpec& sp,
                          int32_t K, double dt, cudaStream_t s) {
  RolloutArgs<R, NT> ra;
  StepArgs<R, NT>& a = ra.step;
  fill_hulls<R, NT>(ctx, a.hull, dt / K);
  for (int t = 0; t < NT; ++t)
    a.cls[t] = t < (int)ctx->hulls.size() ? hull_class(ctx->hulls[t], st) : 0;
  a.sv = make_view<R>(*st);
  a.cmd = (const R*)sp.cmd;
  a.cmd_ld = sp.cmd_ld;
  a.K = K;
  a.dt = (R)(dt / K);
  a.early_trigger = 0;
  a.out = HostOut{};
  a.prefetch_ov = 0;
  ra.slot_stride = sp.slot_stride;
  ra.n_slots = sp.n_slots;
  ra.start = sp.start;
  ra.steps = sp.steps;
  ra.trace = (R*)sp.trace;
  ra.trace_ld = sp.trace_ld;
  ra.trace_rows = sp.trace_rows;
  ra.prefetch = sp.cmd_device && sp.steps > 2 ? 1 : 0;
  a.out = sp.out;
  ra.ready = sp.ready;
  UUV_REGISTER(k_rollout<R, NT, DR, AC, DM, false>);
  if constexpr (sizeof(R) == 4) UUV_REGISTER(k_rollout<R, NT, DR, AC, DM, true>);
  auto kern = k_rollout<R, NT, DR, AC, DM, false>;
  if constexpr (sizeof(R) == 4) {  // (the float64 validation build keeps every register)
    const bool hi = st->n_envs >= kRolloutHiMinEnvs;
    if (hi) kern = k_rollout<R, NT, DR, AC, DM, true>;
    if constexpr (NT == 1) {
      UUV_REGISTER(k_rollout<R, NT, DR, AC, DM, false, true>);
      UUV_REGISTER(k_rollout<R, NT, DR, AC, DM, true, true>);
      UUV_REGISTER(k_rollout<R, NT, DR, AC, DM, false, true, true>);
      UUV_REGISTER(k_rollout<R, NT, DR, AC, DM, true, true, true>);
      if (lean_batch<R>(ctx, st, K)) {
        if (sp.trace == nullptr && sp.ready == nullptr && sp.cmd_device)
          kern = hi ? k_rollout<R, NT, DR, AC, DM, true, true, true>
                    : k_rollout<R, NT, DR, AC, DM, false, true, true>;
        else
          kern = hi ? k_rollout<R, NT, DR, AC, DM, true, true> : k_rollout<R, NT, DR, AC, DM, false, true>;
      }
    }
  }
  kern<<<(unsigned)grid_for(st->n_envs), kBlock, 0, s>>>(ra);
  return check_launch("uuv_rollout");
}

template <typename R>
uuv_status dispatch_rollout(const uuv_ctx* ctx, const uuv_state* st, const RolloutSpec& sp,
                            int32_t K, double dt, cudaStream_t s) {
  const bool dr = st->overlay != nullptr;
  if (ctx->hulls.size() > 1)
    return dr ? launch_rollout<R, UUV_MAX_TYPES, true, 0>(ctx, st, sp, K, dt, s)
              : launch_rollout<R, UUV_MAX_TYPES, false, 0>(ctx, st, sp, K, dt, s);
  const bool dm = diag_mass(ctx, st);
  switch (act_class(ctx)) {
    case 6:
      if (dm)
        return dr ? launch_rollout<R, 1, true, 6, true>(ctx, st, sp, K, dt, s)
                  : launch_rollout<R, 1, false, 6, true>(ctx, st, sp, K, dt, s);
      return dr ? launch_rollout<R, 1, true, 6>(ctx, st, sp, K, dt, s)
                : launch_rollout<R, 1, false, 6>(ctx, st, sp, K, dt, s);
    case 8:
      if (dm)
        return dr ? launch_rollout<R, 1, true, 8, true>(ctx, st, sp, K, dt, s)
                  : launch_rollout<R, 1, false, 8, true>(ctx, st, sp, K, dt, s);
      return dr ? launch_rollout<R, 1, true, 8>(ctx, st, sp, K, dt, s)
                : launch_rollout<R, 1, false, 8>(ctx, st, sp, K, dt, s);
    case kFinLayout:
      if (dm)
        return dr ? launch_rollout<R, 1, true, kFinLayout, true>(ctx, st, sp, K, dt, s)
                  : launch_rollout<R, 1, false, kFinLayout, true>(ctx, st, sp, K, dt, s);
      return dr ? launch_rollout<R, 1, true, kFinLayout>(ctx, st, sp, K, dt, s)
                : launch_rollout<R, 1, false, kFinLayout>(ctx, st, sp, K, dt, s);
    default:
      if (dm)
        return dr ? launch_rollout<R, 1, true, 0, true>(ctx, st, sp, K, dt, s)
                  : launch_rollout<R, 1, false, 0, true>(ctx, st, sp, K, dt, s);
      return dr ? launch_rollout<R, 1, true, 0>(ctx, st, sp, K, dt, s)
                : launch_rollout<R, 1, false, 0>(ctx, st, sp, K, dt, s);
  }
}

uuv_status check_sampler(const uuv_sampler* smp) {
  if (smp == nullptr) return fail(UUV_ERR_ARG, "null sampler");
  if (smp->n_overlay < 0 || smp->n_overlay > UUV_MAX_DRAWS)
    return fail(UUV_ERR_ARG, "sampler: n_overlay %d", smp->n_overlay);
  for (int d = 0; d < smp->n_overlay; ++d) {
    const uuv_draw& dr = smp->overlay[d];
    if (dr.key < 0 || dr.key >= UUV_OV_COUNT) return fail(UUV_ERR_ARG, "sampler: bad key");
    if (dr.n_draws != 1 && dr.n_draws != 3) return fail(UUV_ERR_ARG, "sampler: bad n_draws");
    if (dr.dist < UUV_DIST_UNIFORM || dr.dist > UUV_DIST_GAUSSIAN)
      return fail(UUV_ERR_ARG, "sampler: bad distribution");
    if (dr.dist == UUV_DIST_GAUSSIAN && !(dr.sigma >= 0.0 && dr.lo <= dr.hi))
      return fail(UUV_ERR_ARG, "sampler: gaussian needs sigma >= 0 and lo <= hi");
    if (dr.dist == UUV_DIST_PIECEWISE &&
        (dr.pw_bins < 1 || dr.pw_offset < 0 || dr.pw_offset + 2 * dr.pw_bins + 1 > UUV_PW_MAX))
      return fail(UUV_ERR_ARG, "sampler: piecewise table out of range");
  }
  return UUV_OK;
}

template <typename R>
void fill_task_args(const uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                    const uuv_sampler* smp, uint64_t seed, double dt, int32_t K,
                    const uuv_task_io* io, TaskArgs<R>& a) {
  fill_hulls<R, 1>(ctx, a.hull, dt / K);
  a.sv = make_view<R>(*st);
  build_task<R>(*task, a.task);
  if (smp) a.smp = *smp;
  else memset(&a.smp, 0, sizeof a.smp);
  a.seed = seed;
  a.K = K;
  a.dt_sub = (R)(dt / K);
  a.dt = (R)dt;
  a.dt64 = dt;
  a.prev_u = (R*)io->prev_u;
  a.dev_sum = (R*)io->dev_sum;
  a.obs = (R*)io->obs;
  a.obs_ld = io->obs_ld;
  a.term_obs = (R*)io->term_obs;
  a.rout = (R*)io->real_out;
  a.fout = io->flag_out;
  a.stats = io->stats;
  a.trace = (R*)io->trace;
  a.trace_ld = io->trace_ld;
  a.pol_theta = nullptr;
  a.pol_ld = 0;
  a.pol_members = a.pol_slot = 0;
  a.ep_ret = nullptr;
  a.ep_metric = nullptr;
  a.ep_success = a.ep_pending = nullptr;
  a.ep_live = nullptr;
  a.ep_t = 0;
  a.mask = nullptr;
  a.mode = 0;
  a.cmd = nullptr;
  a.cmd_ld = 0;
  a.prefetch = st->n_envs >= ((int64_t)1 << 19);
}

template <typename R, int AC, bool DM, bool POL, int LEAN = 0>
void launch_task_dr(bool dr, unsigned g, cudaStream_t cs, const TaskArgs<R>& a) {
  UUV_REGISTER(k_task_step<R, true, AC, DM, POL, LEAN>);
  UUV_REGISTER(k_task_step<R, false, AC, DM, POL, LEAN>);
  if (dr) k_task_step<R, true, AC, DM, POL, LEAN><<<g, kBlock, 0, cs>>>(a);
  else k_task_step<R, false, AC, DM, POL, LEAN><<<g, kBlock, 0, cs>>>(a);
}

template <typename R, int AC, bool DM, bool POL, int LEAN>
void launch_task_hi(bool dr, unsigned g, cudaStream_t cs, const TaskArgs<R>& a) {
  UUV_REGISTER(k_task_step<R, true, AC, DM, POL, LEAN, true>);
  UUV_REGISTER(k_task_step<R, false, AC, DM, POL, LEAN, true>);
  if (dr) k_task_step<R, true, AC, DM, POL, LEAN, true><<<g, kBlock, 0, cs>>>(a);
  else k_task_step<R, false, AC, DM, POL, LEAN, true><<<g, kBlock, 0, cs>>>(a);
}

// lean (0, 2, 3; lean_task): the six- / eight-thruster classes only; the 96-register
// build for lean eight-thruster task steps from kTaskHiMinEnvs
constexpr int64_t kTaskHiMinEnvs = 262144;
template <typename R, int AC, bool DM, bool POL>
void launch_task_lean(int lean, bool dr, unsigned g, cudaStream_t cs, const TaskArgs<R>& a) {
  if constexpr (sizeof(R) == 4) {
    if constexpr (AC == 8 && !POL) {
      if (a.sv.n >= kTaskHiMinEnvs) {
        if (lean == 2) return launch_task_hi<R, AC, DM, POL, 2>(dr, g, cs, a);
        if (lean == 3) return launch_task_hi<R, AC, DM, POL, 3>(dr, g, cs, a);
      }
    }
    if (lean == 2) return launch_task_dr<R, AC, DM, POL, 2>(dr, g, cs, a);
    if (lean == 3) return launch_task_dr<R, AC, DM, POL, 3>(dr, g, cs, a);
  }
  launch_task_dr<R, AC, DM, POL>(dr, g, cs, a);
}

template <typename R, bool POL = false>
void launch_task_step(bool dr, int ac, bool dm, int lean, unsigned g, cudaStream_t cs,
                      const TaskArgs<R>& a) {
  if (ac == 6) {
    if (dm) launch_task_lean<R, 6, true, POL>(lean, dr, g, cs, a);
    else launch_task_lean<R, 6, false, POL>(lean, dr, g, cs, a);
  } else if (ac == 8) {
    if (dm) launch_task_lean<R, 8, true, POL>(lean, dr, g, cs, a);
    else launch_task_lean<R, 8, false, POL>(lean, dr, g, cs, a);
  } else if (ac == kFinLayout) {
    if (dm) launch_task_dr<R, kFinLayout, true, POL>(dr, g, cs, a);
    else launch_task_dr<R, kFinLayout, false, POL>(dr, g, cs, a);
  } else {
    if (dm) launch_task_dr<R, 0, true, POL>(dr, g, cs, a);
    else launch_task_dr<R, 0, false, POL>(dr, g, cs, a);
  }
}

// The fused episode loop (k_policy_episode): false when the grid cannot be co-resident
// (its per-step grid-wide wait needs every CTA running), so the caller falls back to
// one uuv_policy_step launch per step.
template <typename R, bool DR, int AC, bool DM, int LEAN = 0>
bool launch_episode_k(unsigned g, cudaStream_t cs, const TaskArgs<R>& a, int32_t length) {
  auto kern = k_policy_episode<R, DR, AC, DM, LEAN>;
  UUV_REGISTER(k_policy_episode<R, DR, AC, DM, LEAN>);
  if ((int64_t)g > one_wave_ctas(kern)) return false;
  kern<<<g, kBlock, 0, cs>>>(a, length);
  return true;
}

template <typename R, bool DR, int AC, bool DM>
bool launch_episode_lean(int lean, unsigned g, cudaStream_t cs, const TaskArgs<R>& a,
                         int32_t length) {
  if constexpr (sizeof(R) == 4) {
    if (lean == 2) return launch_episode_k<R, DR, AC, DM, 2>(g, cs, a, length);
    if (lean == 3) return launch_episode_k<R, DR, AC, DM, 3>(g, cs, a, length);
  }
  return launch_episode_k<R, DR, AC, DM>(g, cs, a, length);
}

template <typename R>
bool launch_episode(bool dr, int ac, bool dm, int lean, unsigned g, cudaStream_t cs,
                    const TaskArgs<R>& a, int32_t length) {
  auto pick = [&](auto dr_c) {
    constexpr bool D = decltype(dr_c)::value;
    if (ac == 6) return dm ? launch_episode_lean<R, D, 6, true>(lean, g, cs, a, length)
                           : launch_episode_lean<R, D, 6, false>(lean, g, cs, a, length);
    if (ac == 8) return dm ? launch_episode_lean<R, D, 8, true>(lean, g, cs, a, length)
                           : launch_episode_lean<R, D, 8, false>(lean, g, cs, a, length);
    if (ac == kFinLayout) return dm ? launch_episode_k<R, D, kFinLayout, true>(g, cs, a, length)
                                    : launch_episode_k<R, D, kFinLayout, false>(g, cs, a, length);
    return dm ? launch_episode_k<R, D, 0, true>(g, cs, a, length)
              : launch_episode_k<R, D, 0, false>(g, cs, a, length);
  };
  return dr ? pick(std::true_type{}) : pick(std::false_type{});
}

uuv_status check_task(const uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                      const uuv_task_io* io, bool obs_optional = false) {
  if (task == nullptr || io == nullptr) return fail(UUV_ERR_ARG, "null task or io");
  if (ctx->hulls.size() != 1) return fail(UUV_ERR_UNSUPPORTED, "tasks need a single-vehicle batch");
  const int A = ctx->hulls[0].n_act;
  const int extra = task->kind == UUV_TASK_TRACKING ? 3 : (task->kind == UUV_TASK_DOCKING ? 1 : 0);
  if (task->obs_dim != 12 + A + extra)
    return fail(UUV_ERR_SHAPE, "task: obs_dim %d != 12 + A + extra = %d", task->obs_dim,
                12 + A + extra);
  if ((io->obs == nullptr && !obs_optional) || io->prev_u == nullptr ||
      (io->obs != nullptr && io->obs_ld < task->obs_dim))
    return fail(UUV_ERR_ARG, "task io: obs / prev_u missing or obs_ld too small");
  if (task->kind == UUV_TASK_TRACKING && io->dev_sum == nullptr)
    return fail(UUV_ERR_ARG, "task io: tracking needs dev_sum");
  return UUV_OK;
}

}  // namespace

namespace uuv_tu {
template <typename R>
uuv_status step(const uuv_ctx* ctx, const uuv_state* st, const void* cmd, int64_t cmd_ld,
                int32_t K, double dt, cudaStream_t s, const HostOut* out);
template <typename R, bool POL>
void task(bool dr, int ac, bool dm, int lean, unsigned g, cudaStream_t cs, const TaskArgs<R>& a);
template <typename R>
bool episode(bool dr, int ac, bool dm, int lean, unsigned g, cudaStream_t cs, const TaskArgs<R>& a,
             int32_t length);
template <typename R>
uuv_status rollout(const uuv_ctx* ctx, const uuv_state* st, const RolloutSpec& sp, int32_t K,
                   double dt, cudaStream_t s);

#if UUV_TU_STEP
template <typename R>
uuv_status rollout(const uuv_ctx* ctx, const uuv_state* st, const RolloutSpec& sp, int32_t K,
                   double dt, cudaStream_t s) {
  return dispatch_rollout<R>(ctx, st, sp, K, dt, s);
}
template uuv_status rollout<float>(const uuv_ctx*, const uuv_state*, const RolloutSpec&, int32_t,
                                   double, cudaStream_t);
template uuv_status rollout<double>(const uuv_ctx*, const uuv_state*, const RolloutSpec&, int32_t,
                                    double, cudaStream_t);
template <typename R>
uuv_status step(const uuv_ctx* ctx, const uuv_state* st, const void* cmd, int64_t cmd_ld,
                int32_t K, double dt, cudaStream_t s, const HostOut* out) {
  return dispatch_step<R>(ctx, st, cmd, cmd_ld, K, dt, s, out);
}
template uuv_status step<float>(const uuv_ctx*, const uuv_state*, const void*, int64_t, int32_t,
                                double, cudaStream_t, const HostOut*);
template uuv_status step<double>(const uuv_ctx*, const uuv_state*, const void*, int64_t, int32_t,
                                 double, cudaStream_t, const HostOut*);
#endif
template <typename R>
uuv_status serve(const uuv_ctx* ctx, const uuv_state* st, int32_t K, double dt, cudaStream_t s,
                 ServeCtl* ctl, uint64_t* done, ServeSync* sync, uint64_t idle_ns,
                 int64_t* grid_out);

#if UUV_TU_SERVE
template <typename R, int NT, bool DR, int AC, bool DM = false>
uuv_status serve_kernel(const uuv_ctx* ctx, const uuv_state* st, int32_t K, double dt,
                        cudaStream_t s, ServeCtl* ctl, uint64_t* done, ServeSync* sync,
                        uint64_t idle_ns, int64_t* grid_out) {
  ServeArgs<R, NT> sa;
  StepArgs<R, NT>& a = sa.step;
  fill_hulls<R, NT>(ctx, a.hull, dt / K);
  for (int t = 0; t < NT; ++t)
    a.cls[t] = t < (int)ctx->hulls.size() ? hull_class(ctx->hulls[t], st) : 0;
  a.sv = make_view<R>(*st);
  a.cmd = nullptr;
  a.cmd_ld = 0;
  a.K = K;
  a.dt = (R)(dt / K);
  a.early_trigger = 0;
  a.out = HostOut{};
  a.prefetch_ov = 0;
  sa.ctl = ctl;
  sa.done = done;
  sa.sync = sync;
  sa.idle_ns = idle_ns;
  static const uint32_t sleep_ns = [] {
    const char* v = getenv("UUV_SERVE_SLEEP");
    return v ? (uint32_t)atoi(v) : 0u;
  }();
  sa.sleep_ns = sleep_ns;
  static const uint32_t stamps = [] {
    const char* v = getenv("UUV_SERVE_STAMPS");
    return v ? (uint32_t)atoi(v) : 0u;
  }();
  sa.stamps = stamps;
  sa.n_act = ctx->hulls.size() > 1 || st->type_id != nullptr ? st->a_max : ctx->hulls[0].n_act;

  const int64_t grid = grid_for(st->n_envs);
  auto kern = k_serve<R, NT, DR, AC, DM>;
  UUV_REGISTER(k_serve<R, NT, DR, AC, DM>);
  if constexpr (NT == 1 && sizeof(R) == 4) {
    UUV_REGISTER(k_serve<R, NT, DR, AC, DM, true>);
    if (lean_batch<R>(ctx, st, K)) kern = k_serve<R, NT, DR, AC, DM, true>;
  }
  if (grid > one_wave_ctas(kern))
    return fail(UUV_ERR_UNSUPPORTED, "step server: %lld CTAs do not fit one wave",
                (long long)grid);
  *grid_out = grid;
  kern<<<(unsigned)grid, kBlock, 0, s>>>(sa);
  return check_launch("uuv_server_start");
}

template <typename R>
uuv_status serve(const uuv_ctx* ctx, const uuv_state* st, int32_t K, double dt, cudaStream_t s,
                 ServeCtl* ctl, uint64_t* done, ServeSync* sy, uint64_t idle_ns, int64_t* g) {
  const bool dr = st->overlay != nullptr;
  if (ctx->hulls.size() > 1)
    return dr ? serve_kernel<R, UUV_MAX_TYPES, true, 0>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
              : serve_kernel<R, UUV_MAX_TYPES, false, 0>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
  const bool dm = diag_mass(ctx, st);
  switch (act_class(ctx)) {
    case 6:
      if (dm)
        return dr ? serve_kernel<R, 1, true, 6, true>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                  : serve_kernel<R, 1, false, 6, true>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
      return dr ? serve_kernel<R, 1, true, 6>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                : serve_kernel<R, 1, false, 6>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
    case 8:
      if (dm)
        return dr ? serve_kernel<R, 1, true, 8, true>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                  : serve_kernel<R, 1, false, 8, true>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
      return dr ? serve_kernel<R, 1, true, 8>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                : serve_kernel<R, 1, false, 8>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
    case kFinLayout:
      if (dm)
        return dr ? serve_kernel<R, 1, true, kFinLayout, true>(ctx, st, K, dt, s, ctl, done, sy,
                                                               idle_ns, g)
                  : serve_kernel<R, 1, false, kFinLayout, true>(ctx, st, K, dt, s, ctl, done, sy,
                                                                idle_ns, g);
      return dr ? serve_kernel<R, 1, true, kFinLayout>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                : serve_kernel<R, 1, false, kFinLayout>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
    default:
      if (dm)
        return dr ? serve_kernel<R, 1, true, 0, true>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                  : serve_kernel<R, 1, false, 0, true>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
      return dr ? serve_kernel<R, 1, true, 0>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g)
                : serve_kernel<R, 1, false, 0>(ctx, st, K, dt, s, ctl, done, sy, idle_ns, g);
  }
}
template uuv_status serve<float>(const uuv_ctx*, const uuv_state*, int32_t, double, cudaStream_t,
                                 ServeCtl*, uint64_t*, ServeSync*, uint64_t, int64_t*);
template uuv_status serve<double>(const uuv_ctx*, const uuv_state*, int32_t, double, cudaStream_t,
                                  ServeCtl*, uint64_t*, ServeSync*, uint64_t, int64_t*);
#endif

#if UUV_TU_TASK || UUV_TU_POLICY
template <typename R, bool POL>
void task(bool dr, int ac, bool dm, int lean, unsigned g, cudaStream_t cs, const TaskArgs<R>& a) {
  launch_task_step<R, POL>(dr, ac, dm, lean, g, cs, a);
}
#endif
#if UUV_TU_TASK
template void task<float, false>(bool, int, bool, int, unsigned, cudaStream_t, const TaskArgs<float>&);
template void task<double, false>(bool, int, bool, int, unsigned, cudaStream_t,
                                  const TaskArgs<double>&);
#endif
#if UUV_TU_POLICY
template void task<float, true>(bool, int, bool, int, unsigned, cudaStream_t, const TaskArgs<float>&);
template void task<double, true>(bool, int, bool, int, unsigned, cudaStream_t,
                                 const TaskArgs<double>&);
template <typename R>
bool episode(bool dr, int ac, bool dm, int lean, unsigned g, cudaStream_t cs, const TaskArgs<R>& a,
             int32_t length) {
  return launch_episode<R>(dr, ac, dm, lean, g, cs, a, length);
}
template bool episode<float>(bool, int, bool, int, unsigned, cudaStream_t, const TaskArgs<float>&,
                             int32_t);
template bool episode<double>(bool, int, bool, int, unsigned, cudaStream_t,
                              const TaskArgs<double>&, int32_t);
#endif
}  // namespace uuv_tu

#if UUV_TU_MAIN
namespace uuv_tu {
thread_local std::string g_err;

static std::vector<const void*>& kernel_registry() {
  static std::vector<const void*> r;
  return r;
}
void register_kernel(const void* fn) { kernel_registry().push_back(fn); }
}  // namespace uuv_tu

// Load every registered kernel now (cudaFuncGetAttributes forces a lazily
// loaded function resident).  Idempotent and cheap after the first call.
static uuv_status preload_kernels() {
  static std::vector<int> loaded_on;
  int dev = 0;
  cudaGetDevice(&dev);
  if (std::find(loaded_on.begin(), loaded_on.end(), dev) != loaded_on.end()) return UUV_OK;
  for (const void* fn : uuv_tu::kernel_registry()) {
    cudaFuncAttributes at;
    const cudaError_t e = cudaFuncGetAttributes(&at, fn);
    if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "preload: %s", cudaGetErrorString(e));
  }
  loaded_on.push_back(dev);
  return UUV_OK;
}

template <typename R, int NT>
static uuv_status derive_launch(const uuv_ctx* ctx, const uuv_state* st, double* o12, double* minv,
                                double* ct_tau, double* mounts, cudaStream_t cs) {
  DeriveArgs<R, NT> a;
  fill_hulls<R, NT>(ctx, a.hull, 1.0);
  a.sv = make_view<R>(*st);
  a.out12 = o12; a.minv = minv; a.ct_tau = ct_tau; a.mounts = mounts;
  UUV_REGISTER(k_derive<R, NT>);
  k_derive<R, NT><<<(unsigned)grid_for(st->n_envs), kBlock, 0, cs>>>(a);
  return check_launch("uuv_derive_params");
}

template <typename R, int NT, bool DR, int AC, bool DM = false>
static uuv_status terms_launch(const uuv_ctx* ctx, const uuv_state* st, const void* cmd,
                               int64_t cmd_ld, double dt_sub, double* out, cudaStream_t cs) {
  TermsArgs<R, NT> a;
  fill_hulls<R, NT>(ctx, a.hull, dt_sub);
  a.sv = make_view<R>(*st);
  a.cmd = (const R*)cmd;
  a.cmd_ld = cmd_ld;
  a.dt = (R)dt_sub;
  a.out = out;
  UUV_REGISTER(k_terms<R, NT, DR, AC, DM>);
  k_terms<R, NT, DR, AC, DM><<<(unsigned)grid_for(st->n_envs), kBlock, 0, cs>>>(a);
  return check_launch("uuv_substep_terms");
}

template <typename R>
static uuv_status terms_dispatch(const uuv_ctx* ctx, const uuv_state* st, const void* cmd,
                                 int64_t cmd_ld, double dt_sub, double* out, cudaStream_t cs) {
  const bool dr = st->overlay != nullptr, multi = ctx->hulls.size() > 1;
  if (multi)
    return dr ? terms_launch<R, UUV_MAX_TYPES, true, 0>(ctx, st, cmd, cmd_ld, dt_sub, out, cs)
              : terms_launch<R, UUV_MAX_TYPES, false, 0>(ctx, st, cmd, cmd_ld, dt_sub, out, cs);
  const bool dm = diag_mass(ctx, st);
  switch (act_class(ctx)) {
    case 6:
      if (dm)
        return dr ? terms_launch<R, 1, true, 6, true>(ctx, st, cmd, cmd_ld, dt_sub, out, cs)
                  : terms_launch<R, 1, false, 6, true>(ctx, st, cmd, cmd_ld, dt_sub, out, cs);
      return dr ? terms_launch<R, 1, true, 6>(ctx, st, cmd, cmd_ld, dt_sub, out, cs)
                : terms_launch<R, 1, false, 6>(ctx, st, cmd, cmd_ld, dt_sub, out, cs);
    case 8:
      if (dm)
        return dr ? terms_launch<R, 1, true, 8, true>(ctx, st, cmd, cmd_ld, dt_sub, out, cs)
                  : terms_launch<R, 1, false, 8, true>(ctx, st, cmd, cmd_ld, dt_sub, out, cs);
      return dr ? terms_launch<R, 1, true, 8>(ctx, st, cmd, cmd_ld, dt_sub, out, cs)
                : terms_launch<R, 1, false, 8>(ctx, st, cmd, cmd_ld, dt_sub, out, cs);
    default:
      return dr ? terms_launch<R, 1, true, 0>(ctx, st, cmd, cmd_ld, dt_sub, out, cs)
                : terms_launch<R, 1, false, 0>(ctx, st, cmd, cmd_ld, dt_sub, out, cs);
  }
}

static uuv_status task_reset_impl(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                                  const uuv_sampler* sampler, uint64_t seed, const uint8_t* mask,
                                  double dt, const uuv_task_io* io, int mode, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if ((s = check_task(ctx, st, task, io)) != UUV_OK) return s;
  if (mode == 1 && (s = check_sampler(sampler)) != UUV_OK) return s;
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const unsigned g = (unsigned)grid_for(st->n_envs);
  if (st->dtype == UUV_F32) {
    TaskArgs<float> a;
    fill_task_args<float>(ctx, st, task, sampler, seed, dt, 1, io, a);
    a.mask = mask;
    a.mode = mode;
    UUV_REGISTER(k_task_reset<float>);
    k_task_reset<float><<<g, kBlock, 0, cs>>>(a);
  } else {
    TaskArgs<double> a;
    fill_task_args<double>(ctx, st, task, sampler, seed, dt, 1, io, a);
    a.mask = mask;
    a.mode = mode;
    UUV_REGISTER(k_task_reset<double>);
    k_task_reset<double><<<g, kBlock, 0, cs>>>(a);
  }
  return check_launch(mode ? "uuv_task_reset" : "uuv_observe");
}

static uuv_status step_checked(uuv_ctx* ctx, const uuv_state* st, const void* commands,
                               int64_t cmd_ld, int32_t substeps, double dt, cudaStream_t cs,
                               const HostOut* out) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (commands == nullptr) return fail(UUV_ERR_ARG, "commands: null");
  if (cmd_ld < st->a_max && ctx->hulls.size() > 1)
    return fail(UUV_ERR_SHAPE, "commands: row stride %lld < a_max %d", (long long)cmd_ld, st->a_max);
  if (cmd_ld < ctx->hulls[0].n_act)
    return fail(UUV_ERR_SHAPE, "commands: row stride %lld < action_dim %d", (long long)cmd_ld,
                ctx->hulls[0].n_act);
  if (substeps < 1) return fail(UUV_ERR_ARG, "substeps must be >= 1, got %d", substeps);
  if (!(dt > 0)) return fail(UUV_ERR_ARG, "dt must be > 0");
  if (st->n_envs == 0) return UUV_OK;
  return st->dtype == UUV_F32
             ? uuv_tu::step<float>(ctx, st, commands, cmd_ld, substeps, dt, cs, out)
             : uuv_tu::step<double>(ctx, st, commands, cmd_ld, substeps, dt, cs, out);
}

// uuv_step_host transfer mode: 1 = mapped pinned memory (default), 0 = copy engines
// (UUV_HOST_STEP=copy).
static int host_step_mode() {
  static const int m = [] {
    const char* v = getenv("UUV_HOST_STEP");
    return (v != nullptr && strcmp(v, "copy") == 0) ? 0 : 1;
  }();
  return m;
}

// Device address of a pinned, mapped host buffer (the host address under UVA), or
// nullptr for pageable memory.  Looked up on every call: a cached answer could
// outlive the allocation (a freed pinned buffer whose address is reused by
// pageable memory would then be written through a stale mapping).
static void* host_mapped(const void* h) {
  if (h == nullptr) return nullptr;
  cudaPointerAttributes at;
  void* d = nullptr;
  if (cudaPointerGetAttributes(&at, h) == cudaSuccess && at.type == cudaMemoryTypeHost)
    d = at.devicePointer;
  cudaGetLastError();
  return d;
}

// Width of the act result rows: the command width (a_max for mixed fleets).
static int32_t out_act_rows(const uuv_ctx* ctx, const uuv_state* st) {
  return ctx->hulls.size() > 1 || st->type_id != nullptr ? st->a_max : ctx->hulls[0].n_act;
}

// Maps every non-null field of a uuv_host_out; false if one is not mapped pinned memory.
static bool map_host_out(const uuv_host_out* o, int32_t n_act, HostOut& m) {
  m = HostOut{};
  if (o == nullptr) return true;
  m.pose = host_mapped(o->pose);
  m.act = host_mapped(o->act);
  m.steps = (int32_t*)host_mapped(o->steps);
  m.div = (uint8_t*)host_mapped(o->diverged);
  m.n_act = n_act;
  m.any = o->pose != nullptr || o->act != nullptr || o->steps != nullptr || o->diverged != nullptr;
  return (o->pose == nullptr || m.pose) && (o->act == nullptr || m.act) &&
         (o->steps == nullptr || m.steps) && (o->diverged == nullptr || m.div);
}

struct uuv_server {
  ServeCtl* ctl = nullptr;   // host view of the doorbell (pinned, mapped)
  ServeCtl* ctl_dev = nullptr;
  uint64_t* done = nullptr;  // host view of the done flag
  uint64_t* done_dev = nullptr;
  ServeSync* sync = nullptr;  // device memory
  int64_t grid = 0;
  uint64_t seq = 0;
  cudaStream_t stream = nullptr;  // own non-blocking stream: legacy-stream work never waits on it
  cudaStream_t caller = nullptr;
  cudaEvent_t ev = nullptr;
  int32_t n_act = 0, dtype = 0;
  int64_t n = 0;
  uint64_t last_out[4] = {0, 0, 0, 0};  // result-row addresses of the last step
  int64_t last_ld = 0;
};

static void server_free(uuv_server* s) {
  if (s->ctl) cudaFreeHost(s->ctl);
  if (s->done) cudaFreeHost(s->done);
  if (s->sync) cudaFree(s->sync);
  if (s->ev) cudaEventDestroy(s->ev);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

// ================================================================== C ABI
extern "C" {

const char* uuv_last_error(void) { return uuv_tu::g_err.c_str(); }
int32_t uuv_abi_version(void) { return UUV_ABI_VERSION; }
void uuv_abi_sizes(int64_t out[6]) {
  out[0] = sizeof(uuv_hull);
  out[1] = sizeof(uuv_state);
  out[2] = sizeof(uuv_sampler);
  out[3] = sizeof(uuv_task);
  out[4] = sizeof(uuv_task_io);
  out[5] = sizeof(uuv_policy);
}

uuv_status uuv_ctx_set_hulls(uuv_ctx* ctx, const uuv_hull* hulls, int32_t n_types) {
  if (ctx == nullptr || hulls == nullptr) return fail(UUV_ERR_ARG, "null ctx or hulls");
  if (n_types < 1 || n_types > UUV_MAX_TYPES)
    return fail(UUV_ERR_UNSUPPORTED, "n_types %d outside [1, %d]", n_types, UUV_MAX_TYPES);
  for (int t = 0; t < n_types; ++t) {
    const uuv_hull& h = hulls[t];
    if (h.n_act < 1 || h.n_act > UUV_MAX_ACT)
      return fail(UUV_ERR_UNSUPPORTED, "hull %d: %d actuators outside [1, %d]", t, h.n_act,
                  UUV_MAX_ACT);
    if (h.mlp_layers < 0 || h.mlp_layers > UUV_MLP_MAX_LAYERS)
      return fail(UUV_ERR_UNSUPPORTED, "hull %d: rotor net depth %d", t, h.mlp_layers);
    int params = 0;
    for (int l = 0; l < h.mlp_layers; ++l) {
      if (h.mlp_sizes[l] < 1 || h.mlp_sizes[l] > UUV_MLP_MAX_WIDTH ||
          h.mlp_sizes[l + 1] < 1 || h.mlp_sizes[l + 1] > UUV_MLP_MAX_WIDTH)
        return fail(UUV_ERR_UNSUPPORTED, "hull %d: rotor net width", t);
      params += h.mlp_sizes[l] * h.mlp_sizes[l + 1] + h.mlp_sizes[l + 1];
    }
    if (params > UUV_MLP_MAX_PARAMS)
      return fail(UUV_ERR_UNSUPPORTED, "hull %d: rotor net has %d > %d parameters", t, params,
                  UUV_MLP_MAX_PARAMS);
    if (!(h.mass > 0)) return fail(UUV_ERR_ARG, "hull %d: mass must be > 0", t);
  }
  ctx->hulls.assign(hulls, hulls + n_types);
  ctx->hf.resize(n_types);
  ctx->hd.resize(n_types);
  for (int t = 0; t < n_types; ++t) {
    build_hull<float>(hulls[t], ctx->hf[t]);
    build_hull<double>(hulls[t], ctx->hd[t]);
    double dinv_min = 1e300;
    for (int k = 0; k < 6; ++k) dinv_min = ctx->hd[t].r.dinv[k] < dinv_min ? ctx->hd[t].r.dinv[k] : dinv_min;
    if (!(dinv_min > 0)) return fail(UUV_ERR_ARG, "hull %d: mass matrix not positive definite", t);
  }
  return UUV_OK;
}

uuv_status uuv_ctx_create(const uuv_hull* hulls, int32_t n_types, uuv_ctx** out) {
  if (out == nullptr) return fail(UUV_ERR_ARG, "null out");
  uuv_ctx* c = new uuv_ctx();
  uuv_status s = uuv_ctx_set_hulls(c, hulls, n_types);
  if (s != UUV_OK) {
    delete c;
    *out = nullptr;
    return s;
  }
  *out = c;
  return UUV_OK;
}

void uuv_ctx_destroy(uuv_ctx* ctx) { delete ctx; }

uuv_status uuv_step(uuv_ctx* ctx, const uuv_state* st, const void* commands, int64_t cmd_ld,
                    int32_t substeps, double dt, void* stream) {
  return step_checked(ctx, st, commands, cmd_ld, substeps, dt, (cudaStream_t)stream, nullptr);
}

uuv_status uuv_step_host(uuv_ctx* ctx, const uuv_state* st, const void* host_cmd, int64_t cmd_ld,
                         void* dev_cmd, const uuv_host_out* out, int32_t substeps, double dt,
                         void* stream, int32_t sync) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (host_cmd == nullptr || dev_cmd == nullptr) return fail(UUV_ERR_ARG, "commands: null");
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const size_t es = st->dtype == UUV_F32 ? sizeof(float) : sizeof(double);
  const int32_t n_act = out_act_rows(ctx, st);
  cudaError_t e = cudaSuccess;
  // Mapped pinned buffers: the step kernel reads the command rows and stores the
  // result rows over the host link itself -- no copy-engine round trips.
  const void* mcmd = host_mapped(host_cmd);
  HostOut mo;
  const bool out_mapped = map_host_out(out, n_act, mo);
  if (host_step_mode() == 1 && mcmd != nullptr && out_mapped) {
    if ((s = step_checked(ctx, st, mcmd, cmd_ld, substeps, dt, cs, mo.any ? &mo : nullptr)) !=
        UUV_OK)
      return s;
  } else {
    e = cudaMemcpyAsync(dev_cmd, host_cmd, (size_t)st->n_envs * cmd_ld * es,
                        cudaMemcpyHostToDevice, cs);
    if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "commands H2D: %s", cudaGetErrorString(e));
    if ((s = step_checked(ctx, st, dev_cmd, cmd_ld, substeps, dt, cs, nullptr)) != UUV_OK)
      return s;
    const int64_t n = st->n_envs;
    const size_t row = (size_t)n * es, pitch = (size_t)st->ld * es;
    if (out != nullptr && out->pose != nullptr) {
      char* hp = (char*)out->pose;
      const char* p = (const char*)st->p;
      if ((const char*)st->q == p + 3 * pitch && (const char*)st->nu == p + 7 * pitch) {
        e = cudaMemcpy2DAsync(hp, row, p, pitch, row, 13, cudaMemcpyDeviceToHost, cs);
      } else {
        e = cudaMemcpy2DAsync(hp, row, st->p, pitch, row, 3, cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess)
          e = cudaMemcpy2DAsync(hp + 3 * row, row, st->q, pitch, row, 4, cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess)
          e = cudaMemcpy2DAsync(hp + 7 * row, row, st->nu, pitch, row, 6, cudaMemcpyDeviceToHost, cs);
      }
    }
    if (e == cudaSuccess && out != nullptr && out->act != nullptr)
      e = cudaMemcpy2DAsync(out->act, row, st->act, pitch, row, n_act, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && out != nullptr && out->steps != nullptr)
      e = cudaMemcpyAsync(out->steps, st->steps, n * sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && out != nullptr && out->diverged != nullptr)
      e = cudaMemcpyAsync(out->diverged, st->diverged, n, cudaMemcpyDeviceToHost, cs);
    if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "result D2H: %s", cudaGetErrorString(e));
  }
  if (sync) {
    e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
  }
  return UUV_OK;
}

uuv_status uuv_server_start(uuv_ctx* ctx, const uuv_state* st, int32_t substeps, double dt,
                            void* stream, int32_t idle_timeout_ms, uuv_server** out) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (out == nullptr) return fail(UUV_ERR_ARG, "null server handle");
  if (substeps < 1 || !(dt > 0)) return fail(UUV_ERR_ARG, "substeps >= 1 and dt > 0 required");
  if (st->n_envs < 1) return fail(UUV_ERR_ARG, "step server needs n_envs >= 1");
  if (idle_timeout_ms < 1) return fail(UUV_ERR_ARG, "idle_timeout_ms must be >= 1");
  if ((s = preload_kernels()) != UUV_OK) return s;
  uuv_server* srv = new uuv_server();
  srv->caller = (cudaStream_t)stream;
  cudaError_t e = cudaStreamCreateWithFlags(&srv->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&srv->ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(srv->ev, srv->caller);  // after the caller's work
  if (e == cudaSuccess) e = cudaStreamWaitEvent(srv->stream, srv->ev, 0);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&srv->ctl, sizeof(ServeCtl), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&srv->done, sizeof(uint64_t), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaMalloc((void**)&srv->sync, sizeof(ServeSync));
  if (e == cudaSuccess) e = cudaMemsetAsync(srv->sync, 0, sizeof(ServeSync), srv->stream);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&srv->ctl_dev, srv->ctl, 0);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&srv->done_dev, srv->done, 0);
  if (e != cudaSuccess) {
    server_free(srv);
    return fail(UUV_ERR_CUDA, "step server buffers: %s", cudaGetErrorString(e));
  }
  memset(srv->ctl, 0, sizeof(ServeCtl));
  *srv->done = 0;
  srv->n_act = out_act_rows(ctx, st);
  srv->dtype = st->dtype;
  srv->n = st->n_envs;
  const uint64_t idle_ns = (uint64_t)idle_timeout_ms * 1000000ull;
  s = st->dtype == UUV_F32 ? uuv_tu::serve<float>(ctx, st, substeps, dt, srv->stream, srv->ctl_dev,
                                                  srv->done_dev, srv->sync, idle_ns, &srv->grid)
                           : uuv_tu::serve<double>(ctx, st, substeps, dt, srv->stream,
                                                   srv->ctl_dev, srv->done_dev, srv->sync,
                                                   idle_ns, &srv->grid);
  if (s != UUV_OK) {
    server_free(srv);
    return s;
  }
  *out = srv;
  return UUV_OK;
}

uuv_status uuv_server_step(uuv_server* srv, const void* host_cmd, int64_t cmd_ld,
                           const uuv_host_out* out) {
  if (srv == nullptr) return fail(UUV_ERR_ARG, "null server");
  if (cmd_ld < srv->n_act)
    return fail(UUV_ERR_SHAPE, "commands: row stride %lld < action_dim %d", (long long)cmd_ld,
                srv->n_act);
  const void* dc = host_mapped(host_cmd);
  HostOut mo;
  if (dc == nullptr || !map_host_out(out, srv->n_act, mo))
    return fail(UUV_ERR_ARG, "step server: commands and result rows must be pinned host memory");
  uint64_t flag = 0;
  if (srv->seq == 0 || (uint64_t)mo.pose != srv->last_out[0] ||
      (uint64_t)mo.act != srv->last_out[1] || (uint64_t)mo.steps != srv->last_out[2] ||
      (uint64_t)mo.div != srv->last_out[3] || cmd_ld != srv->last_ld) {
    srv->ctl->pose = (uint64_t)mo.pose;
    srv->ctl->cmd_ld = cmd_ld;
    srv->ctl->act = (uint64_t)mo.act;
    srv->ctl->steps = (uint64_t)mo.steps;
    srv->ctl->div = (uint64_t)mo.div;
    srv->last_out[0] = (uint64_t)mo.pose;
    srv->last_out[1] = (uint64_t)mo.act;
    srv->last_out[2] = (uint64_t)mo.steps;
    srv->last_out[3] = (uint64_t)mo.div;
    srv->last_ld = cmd_ld;
    flag = kServeNewPose;
  }
  srv->ctl->cmd = (uint64_t)dc;  // before seq (x86 stores are not reordered)
  const uint64_t seq = ++srv->seq;
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  srv->ctl->stamp[6] = (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
  __atomic_store_n(&srv->ctl->seq, seq | flag, __ATOMIC_RELEASE);
  {
    uint64_t spins = 0;
    while (__atomic_load_n(srv->done, __ATOMIC_ACQUIRE) != seq) {
      __builtin_ia32_pause();
      if ((++spins & 0xFFFF) == 0) {
        const cudaError_t q = cudaStreamQuery(srv->stream);
        if (q != cudaErrorNotReady) {
          cudaGetLastError();
          return fail(UUV_ERR_CUDA, "step server is not running (%s)",
                      q == cudaSuccess ? "idle timeout" : cudaGetErrorString(q));
        }
      }
    }
  }
  clock_gettime(CLOCK_REALTIME, &ts);
  srv->ctl->stamp[7] = (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
  return UUV_OK;
}

void uuv_server_stamps(const uuv_server* srv, uint64_t out[8]) {
  for (int k = 0; k < 8; ++k) out[k] = srv ? ((volatile uint64_t*)srv->ctl->stamp)[k] : 0;
}

uuv_status uuv_server_stop(uuv_server* srv) {
  if (srv == nullptr) return UUV_OK;
  __atomic_store_n(&srv->ctl->seq, kServeQuit, __ATOMIC_RELEASE);
  cudaError_t e = cudaStreamSynchronize(srv->stream);
  // later work on the caller's stream sees the served state
  if (e == cudaSuccess) e = cudaEventRecord(srv->ev, srv->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(srv->caller, srv->ev, 0);
  server_free(srv);
  if (e != cudaSuccess) return fail(UUV_ERR_CUDA, "step server: %s", cudaGetErrorString(e));
  return UUV_OK;
}

uuv_status uuv_reset(uuv_ctx* ctx, const uuv_state* st, const uint8_t* mask,
                     const uuv_sampler* sampler, uint64_t seed, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if ((s = check_sampler(sampler)) != UUV_OK) return s;
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const unsigned g = (unsigned)grid_for(st->n_envs);
  if (st->dtype == UUV_F32) {
    ResetArgs<float> a{make_view<float>(*st), *sampler, seed, mask, st->a_max};
    UUV_REGISTER(k_reset<float>);
    k_reset<float><<<g, kBlock, 0, cs>>>(a);
  } else {
    ResetArgs<double> a{make_view<double>(*st), *sampler, seed, mask, st->a_max};
    UUV_REGISTER(k_reset<double>);
    k_reset<double><<<g, kBlock, 0, cs>>>(a);
  }
  return check_launch("uuv_reset");
}

uuv_status uuv_task_step(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                         const uuv_sampler* sampler, uint64_t seed, const void* commands,
                         int64_t cmd_ld, int32_t substeps, double dt, const uuv_task_io* io,
                         void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if ((s = check_task(ctx, st, task, io)) != UUV_OK) return s;
  if ((s = check_sampler(sampler)) != UUV_OK) return s;
  if (commands == nullptr || cmd_ld < ctx->hulls[0].n_act)
    return fail(UUV_ERR_SHAPE, "commands: null or row stride < action_dim");
  if (substeps < 1 || !(dt > 0)) return fail(UUV_ERR_ARG, "substeps >= 1 and dt > 0 required");
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const unsigned g = (unsigned)grid_for(st->n_envs);
  const bool dr = st->overlay != nullptr;
  if (st->dtype == UUV_F32) {
    TaskArgs<float> a;
    fill_task_args<float>(ctx, st, task, sampler, seed, dt, substeps, io, a);
    a.cmd = (const float*)commands;
    a.cmd_ld = cmd_ld;
    uuv_tu::task<float, false>(dr, act_class(ctx), diag_mass(ctx, st), lean_task(ctx, st), g, cs, a);
  } else {
    TaskArgs<double> a;
    fill_task_args<double>(ctx, st, task, sampler, seed, dt, substeps, io, a);
    a.cmd = (const double*)commands;
    a.cmd_ld = cmd_ld;
    uuv_tu::task<double, false>(dr, act_class(ctx), diag_mass(ctx, st), 0, g, cs, a);
  }
  return check_launch("uuv_task_step");
}

static uuv_status policy_impl(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                              const uuv_sampler* sampler, uint64_t seed, const uuv_policy* pol,
                              int32_t substeps, double dt, const uuv_task_io* io,
                              int32_t length, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if ((s = check_task(ctx, st, task, io, true)) != UUV_OK) return s;
  if ((s = check_sampler(sampler)) != UUV_OK) return s;
  if (pol == nullptr || pol->theta == nullptr) return fail(UUV_ERR_ARG, "policy: null theta");
  const int A = ctx->hulls[0].n_act;
  if (pol->members < 1 || pol->slot < 1)
    return fail(UUV_ERR_ARG, "policy: members and slot must be >= 1");
  if (pol->theta_ld < (int64_t)A * task->obs_dim + A)
    return fail(UUV_ERR_SHAPE, "policy: theta row stride < action_dim * obs_dim + action_dim");
  if (pol->ret != nullptr &&
      (pol->metric == nullptr || pol->success == nullptr || pol->pending == nullptr ||
       pol->live == nullptr || (length == 0 && pol->t < 1)))
    return fail(UUV_ERR_ARG, "policy: episode buffers incomplete or t < 1");
  if (length > 0 && pol->ret == nullptr)
    return fail(UUV_ERR_ARG, "policy episode: needs the return / pending / live buffers");
  if (substeps < 1 || !(dt > 0)) return fail(UUV_ERR_ARG, "substeps >= 1 and dt > 0 required");
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const unsigned g = (unsigned)grid_for(st->n_envs);
  const bool dr = st->overlay != nullptr;
  auto fill_pol = [&](auto& a, auto* theta) {
    using RT = std::remove_const_t<std::remove_pointer_t<decltype(theta)>>;
    a.pol_theta = theta;
    a.pol_ld = pol->theta_ld;
    a.pol_members = pol->members;
    a.pol_slot = pol->slot;
    a.ep_ret = pol->ret;
    a.ep_metric = (RT*)pol->metric;
    a.ep_success = pol->success;
    a.ep_pending = pol->pending;
    a.ep_live = pol->ret != nullptr ? pol->live : nullptr;
    a.ep_t = pol->t;
  };
  bool launched = true;
  if (st->dtype == UUV_F32) {
    TaskArgs<float> a;
    fill_task_args<float>(ctx, st, task, sampler, seed, dt, substeps, io, a);
    fill_pol(a, (const float*)pol->theta);
    if (length > 0)
      launched = uuv_tu::episode<float>(dr, act_class(ctx), diag_mass(ctx, st), lean_task(ctx, st), g,
                                        cs, a, length);
    else
      uuv_tu::task<float, true>(dr, act_class(ctx), diag_mass(ctx, st), lean_task(ctx, st), g, cs, a);
  } else {
    TaskArgs<double> a;
    fill_task_args<double>(ctx, st, task, sampler, seed, dt, substeps, io, a);
    fill_pol(a, (const double*)pol->theta);
    if (length > 0)
      launched = uuv_tu::episode<double>(dr, act_class(ctx), diag_mass(ctx, st), 0, g, cs, a, length);
    else
      uuv_tu::task<double, true>(dr, act_class(ctx), diag_mass(ctx, st), 0, g, cs, a);
  }
  if (!launched)
    return fail(UUV_ERR_UNSUPPORTED, "policy episode: %u CTAs do not fit one wave (launch one "
                "uuv_policy_step per step instead)", g);
  return check_launch(length > 0 ? "uuv_policy_episode" : "uuv_policy_step");
}

uuv_status uuv_policy_step(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                           const uuv_sampler* sampler, uint64_t seed, const uuv_policy* pol,
                           int32_t substeps, double dt, const uuv_task_io* io, void* stream) {
  return policy_impl(ctx, st, task, sampler, seed, pol, substeps, dt, io, 0, stream);
}

uuv_status uuv_policy_episode(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                              const uuv_sampler* sampler, uint64_t seed, const uuv_policy* pol,
                              int32_t length, int32_t substeps, double dt,
                              const uuv_task_io* io, void* stream) {
  if (length < 1) return fail(UUV_ERR_ARG, "policy episode: length must be >= 1");
  return policy_impl(ctx, st, task, sampler, seed, pol, substeps, dt, io, length, stream);
}

uuv_status uuv_task_reset(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                          const uuv_sampler* sampler, uint64_t seed, const uint8_t* mask,
                          double dt, const uuv_task_io* io, void* stream) {
  return task_reset_impl(ctx, st, task, sampler, seed, mask, dt, io, 1, stream);
}

uuv_status uuv_observe(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task, double dt,
                       const uuv_task_io* io, void* stream) {
  return task_reset_impl(ctx, st, task, nullptr, 0, nullptr, dt, io, 0, stream);
}

int64_t uuv_stats_blocks(int64_t n_envs) { return grid_for(n_envs); }

uuv_status uuv_rollout_stats(const double* stats, int64_t n_blocks, double* out, int32_t reset,
                             void* stream) {
  if (stats == nullptr || out == nullptr || n_blocks < 0)
    return fail(UUV_ERR_ARG, "rollout_stats: bad arguments");
  UUV_REGISTER(k_stats);
  k_stats<<<1, 32, 0, (cudaStream_t)stream>>>(stats, n_blocks, out, reset, (double*)stats);
  return check_launch("uuv_rollout_stats");
}

uuv_status uuv_derive_params(uuv_ctx* ctx, const uuv_state* st, double* out12, double* minv,
                             double* ct_tau, double* mounts, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const bool multi = ctx->hulls.size() > 1;
  if (st->dtype == UUV_F32)
    return multi ? derive_launch<float, UUV_MAX_TYPES>(ctx, st, out12, minv, ct_tau, mounts, cs)
                 : derive_launch<float, 1>(ctx, st, out12, minv, ct_tau, mounts, cs);
  return multi ? derive_launch<double, UUV_MAX_TYPES>(ctx, st, out12, minv, ct_tau, mounts, cs)
               : derive_launch<double, 1>(ctx, st, out12, minv, ct_tau, mounts, cs);
}

uuv_status uuv_substep_terms(uuv_ctx* ctx, const uuv_state* st, const void* commands,
                             int64_t cmd_ld, double dt_sub, double* out, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (commands == nullptr || out == nullptr) return fail(UUV_ERR_ARG, "null commands/out");
  if (st->n_envs == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  return st->dtype == UUV_F32 ? terms_dispatch<float>(ctx, st, commands, cmd_ld, dt_sub, out, cs)
                              : terms_dispatch<double>(ctx, st, commands, cmd_ld, dt_sub, out, cs);
}


// ------------------------------------------------------------------ DLPack boundary
static const char* const kDlName[UUV_DL_COUNT] = {"p", "q", "nu", "act", "current_ned",
                                                  "steps", "episodes", "diverged"};

static bool dl_is_real(const DLDataType& t, int32_t* dtype) {
  if (t.code != kDLFloat || t.lanes != 1 || (t.bits != 32 && t.bits != 64)) return false;
  *dtype = t.bits == 32 ? UUV_F32 : UUV_F64;
  return true;
}

static uuv_status dl_device(const DLTensor* t, const char* what) {
  if (t->device.device_type != kDLCUDA)
    return fail(UUV_ERR_ARG, "%s: DLPack device type %d is not CUDA", what, (int)t->device.device_type);
  int dev = 0;
  cudaGetDevice(&dev);
  if (t->device.device_id != dev)
    return fail(UUV_ERR_ARG, "%s: on CUDA device %d, the current device is %d", what,
                (int)t->device.device_id, dev);
  if (t->data == nullptr) return fail(UUV_ERR_ARG, "%s: null data", what);
  return UUV_OK;
}

static int64_t dl_stride(const DLTensor* t, int d) {
  if (t->strides != nullptr) return t->strides[d];
  int64_t s = 1;
  for (int k = t->ndim - 1; k > d; --k) s *= t->shape[k];
  return s;
}

static void* dl_ptr(const DLTensor* t) { return (char*)t->data + t->byte_offset; }

// A row-major (n, >= width) Real matrix with unit column stride; returns the row stride.
static uuv_status dl_rows(const DLTensor* t, const char* what, int64_t n, int64_t width,
                          int32_t dtype, int64_t* ld) {
  if (t == nullptr) return fail(UUV_ERR_ARG, "%s: null tensor", what);
  uuv_status s = dl_device(t, what);
  if (s != UUV_OK) return s;
  int32_t dt = -1;
  if (!dl_is_real(t->dtype, &dt) || dt != dtype)
    return fail(UUV_ERR_ARG, "%s: dtype (code %d, %d bits) is not the state's float%d", what,
                (int)t->dtype.code, (int)t->dtype.bits, dtype == UUV_F32 ? 32 : 64);
  if (t->ndim != 2 || t->shape[0] != n || t->shape[1] != width)
    return fail(UUV_ERR_SHAPE, "%s: expected shape (%lld, %lld), got ndim %d (%lld, %lld)", what,
                (long long)n, (long long)width, (int)t->ndim,
                (long long)(t->ndim > 0 ? t->shape[0] : -1),
                (long long)(t->ndim > 1 ? t->shape[1] : -1));
  if (width > 1 && dl_stride(t, 1) != 1)
    return fail(UUV_ERR_SHAPE, "%s: column stride %lld, expected 1", what,
                (long long)dl_stride(t, 1));
  *ld = n > 1 ? dl_stride(t, 0) : width;
  if (*ld < width) return fail(UUV_ERR_SHAPE, "%s: row stride %lld < width %lld", what,
                               (long long)*ld, (long long)width);
  return UUV_OK;
}

// A (n,) vector with unit stride of one of the allowed element types.
static uuv_status dl_vec(const DLTensor* t, const char* what, int64_t n, bool flag) {
  uuv_status s = dl_device(t, what);
  if (s != UUV_OK) return s;
  const DLDataType& d = t->dtype;
  const bool ok = flag ? ((d.code == kDLBool || d.code == kDLUInt) && d.bits == 8 && d.lanes == 1)
                       : (d.code == kDLInt && d.bits == 32 && d.lanes == 1);
  if (!ok)
    return fail(UUV_ERR_ARG, "%s: dtype (code %d, %d bits), expected %s", what, (int)d.code,
                (int)d.bits, flag ? "bool or uint8" : "int32");
  if (t->ndim != 1 || t->shape[0] != n)
    return fail(UUV_ERR_SHAPE, "%s: expected shape (%lld,)", what, (long long)n);
  if (n > 1 && dl_stride(t, 0) != 1) return fail(UUV_ERR_SHAPE, "%s: stride must be 1", what);
  return UUV_OK;
}

static int32_t cmd_width(const uuv_ctx* ctx, const uuv_state* st) {
  return ctx->hulls.size() > 1 || st->type_id != nullptr ? st->a_max : ctx->hulls[0].n_act;
}

uuv_status uuv_state_from_dlpack(uuv_state* st, const DLTensor* const* f, int32_t n_fields) {
  if (st == nullptr || f == nullptr) return fail(UUV_ERR_ARG, "null state or fields");
  if (n_fields != UUV_DL_COUNT)
    return fail(UUV_ERR_ARG, "expected %d DLPack fields, got %d", UUV_DL_COUNT, n_fields);
  for (int k = 0; k < UUV_DL_COUNT; ++k)
    if (f[k] == nullptr && k != UUV_DL_CURRENT) return fail(UUV_ERR_ARG, "%s: null tensor", kDlName[k]);
  const DLTensor* p = f[UUV_DL_P];
  if (p->ndim != 2) return fail(UUV_ERR_SHAPE, "p: expected 2 dims, got %d", (int)p->ndim);
  const int64_t n = p->shape[0];
  int32_t dtype = -1;
  if (!dl_is_real(p->dtype, &dtype)) return fail(UUV_ERR_ARG, "p: dtype must be float32 or float64");
  const DLTensor* act = f[UUV_DL_ACT];
  if (act->ndim != 2 || act->shape[1] < 1 || act->shape[1] > UUV_MAX_ACT)
    return fail(UUV_ERR_SHAPE, "act: expected (N, 1..%d)", UUV_MAX_ACT);
  const int64_t widths[5] = {3, 4, 6, act->shape[1], 3};
  int64_t ld = -1;
  void* rows[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int k = UUV_DL_P; k <= UUV_DL_CURRENT; ++k) {
    const DLTensor* t = f[k];
    if (t == nullptr) continue;
    const char* what = kDlName[k];
    uuv_status s = dl_device(t, what);
    if (s != UUV_OK) return s;
    int32_t dt = -1;
    if (!dl_is_real(t->dtype, &dt) || dt != dtype)
      return fail(UUV_ERR_ARG, "%s: dtype differs from p's float%d", what, dtype == UUV_F32 ? 32 : 64);
    if (t->ndim != 2 || t->shape[0] != n || t->shape[1] != widths[k])
      return fail(UUV_ERR_SHAPE, "%s: expected shape (%lld, %lld)", what, (long long)n,
                  (long long)widths[k]);
    // struct-of-arrays: element i of component c at base[c * ld + i]
    const int64_t s0 = n > 1 ? dl_stride(t, 0) : 1, s1 = dl_stride(t, 1);
    if (s0 != 1)
      return fail(UUV_ERR_SHAPE, "%s: env stride %lld, the SoA layout needs 1 (a (C, ld) "
                  "component-major buffer viewed as (N, C))", what, (long long)s0);
    if (widths[k] > 1) {
      if (ld < 0) ld = s1;
      if (s1 != ld) return fail(UUV_ERR_SHAPE, "%s: component stride %lld != %lld of p", what,
                                (long long)s1, (long long)ld);
    }
    rows[k] = dl_ptr(t);
  }
  if (ld < n) return fail(UUV_ERR_SHAPE, "state: component stride %lld < n_envs %lld",
                          (long long)ld, (long long)n);
  uuv_status s;
  if ((s = dl_vec(f[UUV_DL_STEPS], "steps", n, false)) != UUV_OK) return s;
  if ((s = dl_vec(f[UUV_DL_EPISODES], "episodes", n, false)) != UUV_OK) return s;
  if ((s = dl_vec(f[UUV_DL_DIVERGED], "diverged", n, true)) != UUV_OK) return s;
  st->dtype = dtype;
  st->a_max = (int32_t)act->shape[1];
  st->n_envs = n;
  st->ld = ld;
  st->p = rows[UUV_DL_P];
  st->q = rows[UUV_DL_Q];
  st->nu = rows[UUV_DL_NU];
  st->act = rows[UUV_DL_ACT];
  st->current_ned = rows[UUV_DL_CURRENT];
  st->steps = (int32_t*)dl_ptr(f[UUV_DL_STEPS]);
  st->episodes = (int32_t*)dl_ptr(f[UUV_DL_EPISODES]);
  st->diverged = (uint8_t*)dl_ptr(f[UUV_DL_DIVERGED]);
  return UUV_OK;
}

uuv_status uuv_step_dl(uuv_ctx* ctx, const uuv_state* st, const DLTensor* commands,
                       int32_t substeps, double dt, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  int64_t ld = 0;
  if ((s = dl_rows(commands, "commands", st->n_envs, cmd_width(ctx, st), st->dtype, &ld)) != UUV_OK)
    return s;
  return step_checked(ctx, st, dl_ptr(commands), ld, substeps, dt, (cudaStream_t)stream, nullptr);
}

// Device address of a tensor the kernels may read / write: CUDA memory of the current
// device, or pinned (page-locked, mapped) host memory -- reached over the host link.
static uuv_status dl_kernel_ptr(const DLTensor* t, const char* what, void** p) {
  const int dt = t->device.device_type;
  if (dt == kDLCPU || dt == kDLCUDAHost) {
    if (t->data == nullptr) return fail(UUV_ERR_ARG, "%s: null data", what);
    *p = host_mapped(dl_ptr(t));
    if (*p == nullptr)
      return fail(UUV_ERR_ARG, "%s: host memory is not pinned (page-locked, mapped)", what);
    return UUV_OK;
  }
  uuv_status s = dl_device(t, what);
  if (s == UUV_OK) *p = dl_ptr(t);
  return s;
}

uuv_status uuv_rollout_dl(uuv_ctx* ctx, const uuv_state* st, const DLTensor* commands,
                          int32_t start, int32_t steps, int32_t substeps, double dt,
                          const DLTensor* trace, const DLTensor* ready,
                          const uuv_host_out* out, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (commands == nullptr) return fail(UUV_ERR_ARG, "commands: null tensor");
  void* cmd_p = nullptr;
  if ((s = dl_kernel_ptr(commands, "commands", &cmd_p)) != UUV_OK) return s;
  int32_t dt_code = -1;
  if (!dl_is_real(commands->dtype, &dt_code) || dt_code != st->dtype)
    return fail(UUV_ERR_ARG, "commands: dtype is not the state's float%d",
                st->dtype == UUV_F32 ? 32 : 64);
  const int64_t n = st->n_envs, w = cmd_width(ctx, st);
  if (commands->ndim != 3 || commands->shape[1] != n || commands->shape[2] != w)
    return fail(UUV_ERR_SHAPE, "commands: expected shape (slots, %lld, %lld)", (long long)n,
                (long long)w);
  const int64_t n_slots = commands->shape[0];
  if (n_slots < 1 || n_slots > INT32_MAX) return fail(UUV_ERR_SHAPE, "commands: no slots");
  if (w > 1 && dl_stride(commands, 2) != 1)
    return fail(UUV_ERR_SHAPE, "commands: column stride must be 1");
  const int64_t cmd_ld = n > 1 ? dl_stride(commands, 1) : w;
  const int64_t slot_stride = n_slots > 1 ? dl_stride(commands, 0) : 0;
  if (cmd_ld < w) return fail(UUV_ERR_SHAPE, "commands: row stride < width");
  if (steps < 0 || start < 0) return fail(UUV_ERR_ARG, "steps and start must be >= 0");
  if (substeps < 1 || !(dt > 0)) return fail(UUV_ERR_ARG, "substeps >= 1 and dt > 0 required");
  RolloutSpec sp{cmd_p, cmd_ld, slot_stride, (int32_t)n_slots, (int32_t)(start % n_slots),
                 steps, nullptr, 0, 13, nullptr, commands->device.device_type == kDLCUDA, HostOut{}};
  if (!map_host_out(out, out_act_rows(ctx, st), sp.out))
    return fail(UUV_ERR_ARG, "out: result buffers are not pinned (page-locked) host memory");
  if (trace != nullptr) {
    void* tp = nullptr;
    if ((s = dl_kernel_ptr(trace, "trace", &tp)) != UUV_OK) return s;
    int32_t tc = -1;
    if (!dl_is_real(trace->dtype, &tc) || tc != st->dtype)
      return fail(UUV_ERR_ARG, "trace: dtype is not the state's");
    const int64_t rows = trace->ndim == 3 ? trace->shape[1] : 0;
    if (trace->ndim != 3 || trace->shape[0] < steps || (rows != 13 && rows != 13 + w) ||
        trace->shape[2] != n)
      return fail(UUV_ERR_SHAPE, "trace: expected shape (>= %d, 13 or %lld, %lld)", steps,
                  (long long)(13 + w), (long long)n);
    if ((n > 1 && dl_stride(trace, 2) != 1) || dl_stride(trace, 0) != rows * dl_stride(trace, 1))
      return fail(UUV_ERR_SHAPE, "trace: expected contiguous (steps, rows, ld) rows");
    sp.trace = tp;
    sp.trace_ld = dl_stride(trace, 1);
    sp.trace_rows = (int32_t)rows;
  }
  if (ready != nullptr) {
    if ((s = dl_device(ready, "ready")) != UUV_OK) return s;
    if (ready->ndim < 1 || !((ready->dtype.code == kDLInt || ready->dtype.code == kDLUInt) &&
                             ready->dtype.bits == 32))
      return fail(UUV_ERR_ARG, "ready: expected a 32-bit integer counter");
    sp.ready = (const uint32_t*)dl_ptr(ready);
  }
  if (n == 0 || steps == 0) return UUV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  return st->dtype == UUV_F32 ? uuv_tu::rollout<float>(ctx, st, sp, substeps, dt, cs)
                              : uuv_tu::rollout<double>(ctx, st, sp, substeps, dt, cs);
}

uuv_status uuv_reset_dl(uuv_ctx* ctx, const uuv_state* st, const DLTensor* mask,
                        const uuv_sampler* sampler, uint64_t seed, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (mask != nullptr && (s = dl_vec(mask, "mask", st->n_envs, true)) != UUV_OK) return s;
  return uuv_reset(ctx, st, mask ? (const uint8_t*)dl_ptr(mask) : nullptr, sampler, seed, stream);
}

uuv_status uuv_task_step_dl(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                            const uuv_sampler* sampler, uint64_t seed, const DLTensor* commands,
                            int32_t substeps, double dt, const uuv_task_io* io,
                            const DLTensor* obs, void* stream) {
  uuv_status s = check_state(ctx, st);
  if (s != UUV_OK) return s;
  if (task == nullptr || io == nullptr) return fail(UUV_ERR_ARG, "null task or io");
  int64_t cld = 0, old = 0;
  if ((s = dl_rows(commands, "commands", st->n_envs, ctx->hulls[0].n_act, st->dtype, &cld)) != UUV_OK)
    return s;
  if ((s = dl_rows(obs, "obs", st->n_envs, task->obs_dim, st->dtype, &old)) != UUV_OK) return s;
  uuv_task_io io2 = *io;
  io2.obs = dl_ptr(obs);
  io2.obs_ld = old;
  return uuv_task_step(ctx, st, task, sampler, seed, dl_ptr(commands), cld, substeps, dt, &io2,
                       stream);
}

}  // extern "C"

#endif  // UUV_TU_MAIN
