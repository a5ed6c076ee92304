/*
 * uuv_b200.h — C ABI of the B200-native batched 6-DOF Fossen step.
 *
 * Drop-in boundary for the reference hot path (Python `uuvsim`, /root/reference):
 *
 *   uuv_state_from_dlpack  binds the BatchState fields (engine.py:269-295)
 *                   given as DLPack tensors (validated in C)
 *   uuv_step_dl / uuv_step  replace uuvsim/engine.py:465-484 step_batch
 *                   (and its callees _step_slice 405-418, _substeps 421-449,
 *                    _advance_rotors 335-352, _actuator_wrench_batch 355-402,
 *                    hydrodynamics.py:125-197, kinematics.py:245-266)
 *   uuv_rollout_dl  step_batch T times with known commands in one launch
 *                   (throughput_probe engine.py:541-564)
 *   uuv_step_host   step_batch on host arrays, whole result back (uuv_host_out)
 *   uuv_reset(_dl) replaces uuvsim/engine.py:487-512 reset_envs for declarative
 *                   samplers (default_sampler 265-266; the task samplers
 *                   tasks/core.py:282-289 + 402-407/454-460/503-507; DR draws
 *                   randomization.py:213-234; overlay math vehicles/__init__.py:418-505)
 *   uuv_task_step(_dl) replaces uuvsim/tasks/core.py:328-370 VecTaskEnv.step
 *                   (physics + observe 316-321 + rewards 170-214 + auto-reset)
 *   uuv_task_reset  replaces uuvsim/tasks/core.py:294-301 VecTaskEnv.reset
 *   uuv_observe     replaces uuvsim/tasks/core.py:316-321 VecTaskEnv.observe
 *   uuv_rollout_stats  (no reference analogue; reduces the per-block task
 *                   statistics accumulated by uuv_task_step, deterministic order)
 *
 * Conventions
 *  - Every array is DEVICE memory owned by the caller and borrowed for the
 *    call (plain pointers, or DLPack tensors in the *_dl entry points); nothing
 *    is retained and nothing is allocated inside uuv_step / uuv_task_step.
 *    All work is enqueued on `stream` (a cudaStream_t, NULL = legacy default
 *    stream); only the host-buffer entry points (sync != 0) synchronise.
 *  - Per-env state is struct-of-arrays: component c of env i lives at
 *    base[c * ld + i] (ld >= n_envs).  Commands and observations are
 *    row-major (n_envs, width) with an explicit row stride.
 *  - Real arrays are float32 or float64 as given by uuv_state.dtype; steps /
 *    episodes are int32; flags are uint8 (0/1).
 *  - Non-finite rows never raise: they freeze and set diverged (engine.py:414-449).
 *  - Return value is a uuv_status; uuv_last_error() holds a thread-local message.
 */
#ifndef UUV_B200_H
#define UUV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/*
 * DLPack (https://github.com/dmlc/dlpack, the v0.8/v1.0 ABI, unversioned
 * DLTensor) -- declared here only when the real dlpack.h has not been included,
 * so either header can come first.  The tensor-taking entry points below
 * (uuv_*_dl) borrow the DLTensor for the call: nothing is retained and the
 * caller's deleter is never invoked.
 */
#ifndef DLPACK_DLPACK_H_
#define DLPACK_DLPACK_H_
typedef enum { kDLCPU = 1, kDLCUDA = 2, kDLCUDAHost = 3, kDLCUDAManaged = 13 } DLDeviceType;
typedef struct {
  DLDeviceType device_type;
  int32_t device_id;
} DLDevice;
typedef enum { kDLInt = 0, kDLUInt = 1, kDLFloat = 2, kDLOpaqueHandle = 3, kDLBfloat = 4,
               kDLComplex = 5, kDLBool = 6 } DLDataTypeCode;
typedef struct {
  uint8_t code;
  uint8_t bits;
  uint16_t lanes;
} DLDataType;
typedef struct {
  void* data;
  DLDevice device;
  int32_t ndim;
  DLDataType dtype;
  int64_t* shape;
  int64_t* strides;        /* in elements; NULL = compact row-major */
  uint64_t byte_offset;
} DLTensor;
typedef struct DLManagedTensor {
  DLTensor dl_tensor;
  void* manager_ctx;
  void (*deleter)(struct DLManagedTensor* self);
} DLManagedTensor;
#endif

#define UUV_ABI_VERSION 7
#define UUV_MAX_RUNS 8
#define UUV_MAX_ACT 8        /* actuator columns per vehicle type             */
#define UUV_MAX_TYPES 6      /* vehicle types in one batch (mixed fleets)     */
#define UUV_MLP_MAX_PARAMS 128 /* packed weights+biases of one rotor network  */
#define UUV_MLP_MAX_WIDTH 16   /* widest layer of a rotor network             */
#define UUV_MLP_MAX_LAYERS 4
#define UUV_MAX_DRAWS 16     /* overlay keys per DR spec                      */
#define UUV_PW_MAX 64        /* piecewise breakpoint + cdf table entries     */

typedef enum {
  UUV_OK = 0,
  UUV_ERR_ARG = 1,         /* bad pointer / size / enum                     */
  UUV_ERR_SHAPE = 2,       /* inconsistent dimensions                        */
  UUV_ERR_CUDA = 3,        /* launch or runtime failure                      */
  UUV_ERR_UNSUPPORTED = 4  /* valid request outside this build's envelope   */
} uuv_status;

typedef enum { UUV_F32 = 0, UUV_F64 = 1 } uuv_dtype;

/* Actuator kinds / rotor families (engine.py:80-81). */
enum { UUV_PROPELLER = 0, UUV_RUDDER = 1, UUV_TILTROTOR = 2 };
enum { UUV_ZERO_ORDER = 0, UUV_FIRST_ORDER = 1, UUV_DATA_DRIVEN = 2 };

/* Hull flags. */
enum { UUV_HULL_DIAGONAL = 1 /* M_A, D_lin, D_quad all diagonal */ };

/*
 * One vehicle type, float64, as compiled from a VehicleConfig
 * (compile_layout engine.py:129-189 + BatchParams.write_row 220-234).
 * Matrices are row-major.  Tilt rotors carry their thrust axis already
 * rotated to the default tilt (engine.py:139-143).  For rudders `axis` is
 * the hinge and fin_xf/fin_yf its in-plane basis (engine.py:118-126).
 * The library factors the base composite mass matrix M_RB + M_A itself.
 */
typedef struct {
  int32_t n_act;
  int32_t flags;
  int32_t kind[UUV_MAX_ACT];
  int32_t model[UUV_MAX_ACT];
  int32_t mlp_layers;                      /* number of dense layers (0: none) */
  int32_t mlp_sizes[UUV_MLP_MAX_LAYERS + 1];
  int32_t mlp_relu;                        /* 0 tanh, 1 relu */
  int32_t pad_;
  double mass, volume, rho, g;
  double r_g[3], r_b[3];
  double inertia[9];
  double M_A[36], D_lin[36], D_quad[36];
  double limit[UUV_MAX_ACT], deadzone[UUV_MAX_ACT], reaction[UUV_MAX_ACT];
  double thrust_coeff[UUV_MAX_ACT], time_constant[UUV_MAX_ACT];
  double mount[UUV_MAX_ACT][3], axis[UUV_MAX_ACT][3];
  double fin_xf[UUV_MAX_ACT][3], fin_yf[UUV_MAX_ACT][3];
  double fin_area[UUV_MAX_ACT], fin_cla[UUV_MAX_ACT], fin_cd0[UUV_MAX_ACT];
  double fin_kd[UUV_MAX_ACT], fin_stall[UUV_MAX_ACT], fin_rho[UUV_MAX_ACT];
  double mlp[UUV_MLP_MAX_PARAMS];          /* W0 (out,in) row-major, b0, W1, b1, ... */
} uuv_hull;

/*
 * Per-env DR overlay record.  The record is a float64 array [n_slots][ld]
 * in both precisions (sampled values are kept bit-exact; derived parameters
 * are formed from it in float64 once per launch);
 * slot[k] gives the first slot of key k or -1 when the key is inactive in the
 * batch.  Inactive keys and rows without an overlay hold identity values
 * (ratios 1, cobm 0 = "absent", payload 0, positions/jitter 0) so that
 * overlay-free rows reproduce the base vehicle exactly (engine.py:497-502).
 */
enum {
  UUV_OV_MASS = 0,         /* mass*            */
  UUV_OV_VOLUME,           /* volume*          */
  UUV_OV_INERTIA,          /* inertia*         */
  UUV_OV_ADDED_MASS,       /* added_mass*      */
  UUV_OV_DAMPING,          /* damping*         */
  UUV_OV_TIME_CONSTANT,    /* time_constant*   */
  UUV_OV_THRUST_COEFF,     /* thrust_coeff*    */
  UUV_OV_COBM,             /* cobm (0 = absent)*/
  UUV_OV_PAYLOAD_MASS,     /* payload_mass*    */
  UUV_OV_PAYLOAD_POS,      /* payload_position, 3 slots */
  UUV_OV_JITTER,           /* mount_position_jitter, 3*UUV_MAX_ACT slots (actuator-major) */
  UUV_OV_COUNT
};

typedef struct {
  int32_t dtype;           /* uuv_dtype of every Real array below           */
  int32_t a_max;           /* actuator columns of act / commands            */
  int64_t n_envs;
  int64_t ld;              /* SoA leading dimension                          */
  int64_t env_offset;      /* global index of row 0 (RNG keys under sharding)*/
  void* p;                 /* [3][ld]  NED position                          */
  void* q;                 /* [4][ld]  body->NED quaternion (w,x,y,z)        */
  void* nu;                /* [6][ld]  body velocity                         */
  void* act;               /* [a_max][ld] rotor speeds / fin angles          */
  void* current_ned;       /* [3][ld]  or NULL: no current in this batch     */
  int32_t* steps;          /* [ld]                                           */
  int32_t* episodes;       /* [ld]                                           */
  uint8_t* diverged;       /* [ld]                                           */
  const uint8_t* type_id;  /* [ld] index into the hull list, or NULL (type 0)*/
  double* overlay;         /* [n_slots][ld] float64 (bit-exact draws) or NULL*/
  uint16_t* overlay_keys;  /* [ld] bit k set: key k present in the row's overlay, or NULL */
  int32_t n_slots;
  int32_t slot[UUV_OV_COUNT];
  int32_t flags;           /* UUV_STATE_* */
  /* Mixed fleets whose rows form contiguous per-type runs (make_fleet_batch):
   * run r covers rows [run_start[r], run_start[r+1]) (the last run to n_envs)
   * with hull run_type[r].  Large batches are then stepped by one specialised
   * single-hull launch per run on forked streams; n_runs = 0 means unknown
   * (one generic mixed-fleet launch). */
  int32_t n_runs;
  int32_t run_type[UUV_MAX_RUNS];
  int64_t run_start[UUV_MAX_RUNS];
} uuv_state;

/* uuv_state.flags */
enum { UUV_STATE_PAYLOAD_AT_ORIGIN = 1 /* every env's payload_position (if any) is 0 */ };

/* One draw of a DR key (randomization.py:48-117).  Gaussian draws are
 * clip(mu + sigma * z, lo, hi) with z from numpy's random_standard_normal
 * ziggurat, restated bit for bit (csrc/uuv_ziggurat.cuh). */
enum { UUV_DIST_UNIFORM = 0, UUV_DIST_PIECEWISE = 1, UUV_DIST_GAUSSIAN = 2 };
typedef struct {
  int32_t key;             /* UUV_OV_* (overlay draws) */
  int32_t dist;
  int32_t n_draws;         /* 1 scalar, 3 vector keys  */
  int32_t pw_bins;         /* piecewise: K bins        */
  int32_t pw_offset;       /* into pw_table: K+1 breakpoints then K cdf values */
  int32_t pad_;
  double lo, hi;           /* uniform bounds; gaussian clip interval */
  double mu, sigma;        /* gaussian                               */
} uuv_draw;

enum { UUV_START_IDENTITY = 0, UUV_START_BOX = 1 };
enum { UUV_CURRENT_NONE = 0, UUV_CURRENT_RANDOM_HEADING = 1, UUV_CURRENT_HEADING_DRAW = 2 };

/*
 * Declarative episode sampler.  Draw order per reset (Philox stream keyed
 * (seed, env_offset + i), counter word 1 = episode):
 *   overlay draws in the given (sorted-key) order,
 *   current speed [, heading],
 *   start box: p = p_base + U(p_lo, p_hi) (3), euler = U(eul_lo, eul_hi) (3),
 *              nu = U(nu_lo, nu_hi) (6).
 */
/* Per-(seed, env, episode) stream of a reset. */
enum { UUV_RNG_PHILOX = 0,  /* Philox4x64-10, key [seed, env], counter [0, episode, 0, 0] */
       UUV_RNG_PCG64 = 1 }; /* PCG64(SeedSequence(seed, spawn_key=(env, episode))): the
                               unmodified reference's BatchState.env_rng (engine.py:291-295) */

typedef struct {
  int32_t n_overlay;
  int32_t current_mode;
  int32_t start_mode;
  int32_t rng_mode;        /* UUV_RNG_* */
  uuv_draw overlay[UUV_MAX_DRAWS];
  uuv_draw current_speed, current_heading;
  double p_base[3], p_lo[3], p_hi[3];
  double eul_lo[3], eul_hi[3];
  double nu_lo[6], nu_hi[6];
  double pw_table[UUV_PW_MAX];
} uuv_sampler;

enum { UUV_TASK_STATION = 0, UUV_TASK_TRACKING = 1, UUV_TASK_DOCKING = 2 };
enum { UUV_TRAJ_HELIX = 0, UUV_TRAJ_LISSAJOUS = 1 };

/* Task constants (tasks/core.py:98-167, trajectories.py:23-53). */
typedef struct {
  int32_t kind;
  int32_t episode_length;
  int32_t traj_kind;
  int32_t obs_dim;
  double bounds, nu_max, fail_penalty;
  double w_p, w_a, w_v, w_u, w_b, r_tol, speed_cap;
  double dock_bonus, w_dock_dist, w_impact, w_level;
  double target_p[3], target_q[4];
  double success_tol;
  double dock_centre[3], dock_radius;
  double traj_radius, traj_rate, traj_climb, traj_z0, traj_phase;
  double traj_amp[3], traj_rates[3];
} uuv_task;

/* Real outputs of uuv_task_step: [UUV_TR_COUNT][ld]. */
enum { UUV_TR_REWARD = 0, UUV_TR_POS_ERR, UUV_TR_ATT_ERR, UUV_TR_METRIC, UUV_TR_TIME,
       UUV_TR_CONTACT_DIST, UUV_TR_CONTACT_SPEED, UUV_TR_CONTACT_ATT, UUV_TR_COUNT };
/* Flag outputs of uuv_task_step: uint8 [UUV_TF_COUNT][ld]. */
enum { UUV_TF_TERMINATED = 0, UUV_TF_TRUNCATED, UUV_TF_FINISHED, UUV_TF_FAILURE,
       UUV_TF_SUCCESS, UUV_TF_DIVERGED, UUV_TF_CONTACT, UUV_TF_COUNT };
/* Per-block rollout statistics accumulated by uuv_task_step (float64 sums). */
enum { UUV_ST_REWARD = 0, UUV_ST_FINISHED, UUV_ST_SUCCESS, UUV_ST_FAILURE, UUV_ST_TRUNCATED,
       UUV_ST_METRIC_FINISHED, UUV_ST_DIVERGED, UUV_ST_FRAMES, UUV_ST_COUNT };

typedef struct {
  void* prev_u;            /* [a_max][ld] previous (clipped) command          */
  void* dev_sum;           /* [ld] tracking deviation accumulator or NULL     */
  void* obs;               /* (n, obs_ld) row-major next observation          */
  int64_t obs_ld;
  void* term_obs;          /* (n, obs_ld) final obs of finished rows or NULL  */
  void* real_out;          /* [UUV_TR_COUNT][ld] or NULL (reset/observe)      */
  uint8_t* flag_out;       /* [UUV_TF_COUNT][ld] or NULL                      */
  double* stats;           /* [n_blocks][UUV_ST_COUNT] running sums or NULL   */
  void* trace;             /* [UUV_TRACE_COUNT + a_max][trace_ld] or NULL     */
  int64_t trace_ld;
} uuv_task_io;

/* Per-step trajectory record written by uuv_task_step when uuv_task_io.trace
 * is set (batch dtype, SoA rows): the post-step, post-auto-reset pose and
 * velocity, the reward, t = steps * dt and the raw (unclipped) command -- the
 * fields of the reference's rollout records (cli.py:261-303).  Rows
 * UUV_TRACE_CMD .. UUV_TRACE_CMD + a_max - 1 hold the command. */
enum { UUV_TRACE_P = 0, UUV_TRACE_Q = 3, UUV_TRACE_NU = 7, UUV_TRACE_REWARD = 13,
       UUV_TRACE_T = 14, UUV_TRACE_CMD = 15, UUV_TRACE_COUNT = 15 };

/*
 * Population of affine-tanh policies evaluated inside the task step
 * (baseline.py:37-84, 109-192): row i acts with member m = i / slot,
 *   u_i = tanh(W_m obs_i + b_m)  for m < members,  0 otherwise,
 * where obs_i is the observation the previous step (or reset) returned.
 * theta rows are [members][theta_ld] in the batch dtype: W (action_dim x
 * obs_dim, row-major) then b (action_dim) -- the reference's Policy.theta().
 * With `ret` set, the launch also runs one iteration of _rollout_returns
 * (baseline.py:109-127): pending rows accumulate the reward, a row's first
 * finish records metric/success and clears pending, and live[t] counts rows
 * still pending after step t.  Step t (1-based) is a no-op when live[t-1] is 0,
 * so a whole episode loop can be enqueued (or graph-captured) without host syncs
 * and stops exactly where the reference's `if not pending.any(): break` does.
 */
typedef struct {
  const void* theta;
  int64_t theta_ld;
  int32_t members;
  int32_t slot;
  double* ret;             /* [ld] or NULL (no episode bookkeeping) */
  void* metric;            /* [ld] batch dtype                      */
  uint8_t* success;        /* [ld]                                  */
  uint8_t* pending;        /* [ld] 1 until the row's first finish   */
  int32_t* live;           /* [>= t + 1], live[0] = initial pending */
  int32_t t;               /* this launch's step index, >= 1        */
  int32_t pad_;
} uuv_policy;

typedef struct uuv_ctx uuv_ctx;

const char* uuv_last_error(void);
int32_t uuv_abi_version(void);
/* sizeof of the ABI structs, for binding self-checks: hull, state, sampler, task, task_io. */
void uuv_abi_sizes(int64_t out[6]);  /* sizeof hull, state, sampler, task, task_io, policy */

/* Context: owns the hull list of one batch (host copy; travels by value in each launch).
 * Replaces compile_layout / VehicleLayout (engine.py:84-189) and the per-vehicle
 * part of make_batch (engine.py:298-326). */
uuv_status uuv_ctx_create(const uuv_hull* hulls, int32_t n_types, uuv_ctx** out);
uuv_status uuv_ctx_set_hulls(uuv_ctx* ctx, const uuv_hull* hulls, int32_t n_types);
void uuv_ctx_destroy(uuv_ctx* ctx);

/* Advance every env one control step of `substeps` fused physics substeps
 * (dt_sub = dt / substeps).  commands: (n_envs, cmd_ld) row-major Real,
 * clipped to [-1, 1] inside.  Replaces step_batch (engine.py:465-484) with
 * _step_slice / _substeps (engine.py:405-449); non-finite rows freeze and set
 * diverged (engine.py:435-449), never an error. */
uuv_status uuv_step(uuv_ctx* ctx, const uuv_state* st, const void* commands, int64_t cmd_ld,
                    int32_t substeps, double dt, void* stream);

/* Host-side result of one step: every field the reference's step_batch mutates
 * in place (engine.py:418, 444-449), as row-major host arrays (n = n_envs).  Any
 * field may be NULL (not returned). */
typedef struct {
  void* pose;              /* (13, n) Real: p (3), q (4), nu (6)                 */
  void* act;               /* (n_act, n) Real; n_act = command width             */
  int32_t* steps;          /* (n)                                                */
  uint8_t* diverged;       /* (n)                                                */
} uuv_host_out;

/* Host-buffer variant of uuv_step for callers whose commands and results live in
 * host memory: commands host_cmd (n_envs, cmd_ld) in, the step's result rows out
 * into `out` (may be NULL); sync != 0 waits.  When every buffer is pinned
 * (mapped) host memory the step kernel reads the commands and stores the result
 * rows over the host link itself (no copy-engine round trips; UUV_HOST_STEP=copy
 * forces the copy path); otherwise the commands are staged through dev_cmd and
 * the results copied back with async copies. */
uuv_status uuv_step_host(uuv_ctx* ctx, const uuv_state* st, const void* host_cmd, int64_t cmd_ld,
                         void* dev_cmd, const uuv_host_out* out, int32_t substeps, double dt,
                         void* stream, int32_t sync);

/*
 * Step server: a resident kernel that advances the batch one control step each
 * time the host rings a doorbell in mapped pinned memory -- no kernel launch and
 * no stream synchronisation per step (host-in-the-loop stepping, the reference's
 * numpy-in / numpy-out usage).  It runs on its own non-blocking stream, ordered
 * after the work already on `stream` at start; uuv_server_stop orders later work
 * on `stream` after it.  While it runs it owns the state, and a device-wide
 * synchronisation would wait for it.  The grid (one thread per env) must fit in
 * one wave.  The kernel ends by itself after idle_timeout_ms without a step.
 */
typedef struct uuv_server uuv_server;
uuv_status uuv_server_start(uuv_ctx* ctx, const uuv_state* state, int32_t substeps, double dt,
                            void* stream, int32_t idle_timeout_ms, uuv_server** out);
/* One step: host_cmd (n_envs, cmd_ld) and every non-NULL field of `out` must be
 * pinned host memory; returns when every env has stepped and its result rows
 * are in host memory.  Replaces step_batch (engine.py:465-484) called step after
 * step with host (numpy) arrays. */
uuv_status uuv_server_step(uuv_server* server, const void* host_cmd, int64_t cmd_ld,
                           const uuv_host_out* out);
/* Phase times of the last step, ns (profiling aid, written when the process
 * runs with UUV_SERVE_STAMPS=1; GPU %globaltimer and host CLOCK_REALTIME):
 * doorbell seen, doorbell fields read, commands read, physics done (CTA 0),
 * system fence begin / end (last CTA), host ring, host done. */
void uuv_server_stamps(const uuv_server* server, uint64_t out[8]);
/* Stop the kernel, wait for it and free the server. */
uuv_status uuv_server_stop(uuv_server* server);

/*
 * DLPack boundary.  The reference's BatchState fields (engine.py:270-295) as
 * borrowed DLPack tensors, validated in C (dtype, device, shape, strides):
 *   UUV_DL_P (N,3), UUV_DL_Q (N,4) wxyz, UUV_DL_NU (N,6), UUV_DL_ACT (N,a_max),
 *   UUV_DL_CURRENT (N,3) or NULL: float32 or float64 (all alike), strides
 *   (1, ld) -- the struct-of-arrays layout, one ld >= N for every field;
 *   UUV_DL_STEPS, UUV_DL_EPISODES (N,) int32; UUV_DL_DIVERGED (N,) bool or
 *   uint8; unit stride.  Every tensor lives on the current CUDA device.
 * uuv_state_from_dlpack fills dtype, a_max, n_envs, ld and the state pointers of
 * `st`; the batch-internal fields (type_id, overlay record, runs, env_offset,
 * flags) are left as the caller set them.
 */
enum { UUV_DL_P = 0, UUV_DL_Q, UUV_DL_NU, UUV_DL_ACT, UUV_DL_CURRENT, UUV_DL_STEPS,
       UUV_DL_EPISODES, UUV_DL_DIVERGED, UUV_DL_COUNT };
uuv_status uuv_state_from_dlpack(uuv_state* st, const DLTensor* const* fields, int32_t n_fields);

/* uuv_step with the commands as a DLPack tensor (n_envs, width), width = the
 * command width (action_dim; a_max for mixed fleets), the state's dtype and
 * device, unit column stride (any row stride >= width).  The entry point a
 * DLPack caller of step_batch (engine.py:465-484) binds. */
uuv_status uuv_step_dl(uuv_ctx* ctx, const uuv_state* st, const DLTensor* commands,
                       int32_t substeps, double dt, void* stream);

/* `steps` control steps in ONE launch with the state held in registers from the
 * first to the last (throughput_probe, engine.py:541-564, and open-loop
 * rollouts): step t applies slot (start + t) mod S of `commands`, a DLPack ring
 * (S, n_envs, width) of the state's dtype -- bit for bit `steps` calls of
 * uuv_step_dl(commands[slot]) (engine.py:465-484), state stored every step.
 * `trace` (>= steps, 13, n_envs) or NULL receives p, q, nu after every step;
 * (>= steps, 13 + width, n_envs) receives act too.  `commands` and `trace` may be
 * CUDA tensors of the current device or pinned (page-locked) host tensors
 * (kDLCPU / kDLCUDAHost): the kernel then reads each step's command rows over the
 * host link one step ahead and writes each step's trace rows as it produces them
 * -- a host-to-host rollout in one launch (wait on `stream` before reading).
 * `out` (or NULL): mapped pinned host rows receiving the result after the last
 * step (as uuv_step_host's: p, q, nu, act, steps, diverged; any field NULL),
 * written by the kernel itself.
 * `ready` (a uint32/int32 device counter) or NULL: step t waits until
 * *ready > t, so a producer on another stream can fill the ring while the
 * rollout runs (device-side command ring; fill slot, then raise the counter). */
uuv_status uuv_rollout_dl(uuv_ctx* ctx, const uuv_state* st, const DLTensor* commands,
                          int32_t start, int32_t steps, int32_t substeps, double dt,
                          const DLTensor* trace, const DLTensor* ready,
                          const uuv_host_out* out, void* stream);

/* uuv_reset with the mask as a DLPack tensor (n_envs,) bool/uint8, unit stride,
 * or NULL for every row (reset_envs, engine.py:487-512). */
uuv_status uuv_reset_dl(uuv_ctx* ctx, const uuv_state* st, const DLTensor* mask,
                        const uuv_sampler* sampler, uint64_t seed, void* stream);

/* uuv_task_step with DLPack commands (as uuv_step_dl) and the next observation
 * written into `obs` (n_envs, obs_dim) of the state's dtype, unit column stride;
 * io->obs is ignored (VecTaskEnv.step, tasks/core.py:328-370). */
uuv_status uuv_task_step_dl(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                            const uuv_sampler* sampler, uint64_t seed, const DLTensor* commands,
                            int32_t substeps, double dt, const uuv_task_io* io,
                            const DLTensor* obs, void* stream);

/* Reset rows with mask[i] != 0 (mask NULL = all rows) from the declarative
 * sampler: episodes += 1, per-(seed, env, episode) stream, overlay draws, start
 * state.  Replaces reset_envs (engine.py:487-512) with sample_overlay /
 * sample_current (randomization.py:213-234) and apply_overlay
 * (vehicles/__init__.py:443-505). */
uuv_status uuv_reset(uuv_ctx* ctx, const uuv_state* st, const uint8_t* mask,
                     const uuv_sampler* sampler, uint64_t seed, void* stream);

/* Fused task step: physics, reward/termination/info, auto-reset, next obs.
 * Replaces VecTaskEnv.step (tasks/core.py:328-370) with the per-task
 * _task_step / reward functions (tasks/core.py:170-214, 409-520). */
uuv_status uuv_task_step(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                         const uuv_sampler* sampler, uint64_t seed, const void* commands,
                         int64_t cmd_ld, int32_t substeps, double dt, const uuv_task_io* io,
                         void* stream);

/* uuv_task_step with the commands computed on the device by a policy
 * population (uuv_policy); io->obs may be NULL (the observation is recomputed
 * in-kernel from the state).  Replaces the act_fn(obs) -> env.step round trip
 * of baseline._rollout_returns / evaluate / cem_train (baseline.py:109-192). */
uuv_status uuv_policy_step(uuv_ctx* ctx, const uuv_state* state, const uuv_task* task,
                           const uuv_sampler* sampler, uint64_t seed, const uuv_policy* policy,
                           int32_t substeps, double dt, const uuv_task_io* io, void* stream);
/* A whole episode loop of uuv_policy_step (t = 1 .. length) in ONE launch, the state
 * held in registers across the steps; it stops after the first step at which no
 * row of the batch is pending -- exactly the reference loop's break
 * (baseline._rollout_returns, baseline.py:109-127).  Needs the episode buffers
 * (ret, metric, success, pending) and live[2 * (length + 1)]: live[0] = initial
 * pending count, live[1..length] zeroed (pending after step t), the second half
 * zeroed (the kernel's per-step arrival counters).  Returns UUV_ERR_UNSUPPORTED
 * when the grid cannot be co-resident (the per-step loop then applies). */
uuv_status uuv_policy_episode(uuv_ctx* ctx, const uuv_state* state, const uuv_task* task,
                              const uuv_sampler* sampler, uint64_t seed, const uuv_policy* policy,
                              int32_t length, int32_t substeps, double dt,
                              const uuv_task_io* io, void* stream);
/* Reset masked rows (prev_u and dev_sum zeroed too), then observe all rows.
 * Replaces VecTaskEnv.reset (tasks/core.py:294-301). */
uuv_status uuv_task_reset(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task,
                          const uuv_sampler* sampler, uint64_t seed, const uint8_t* mask,
                          double dt, const uuv_task_io* io, void* stream);

/* Observation of every row into io->obs.  Replaces VecTaskEnv.observe
 * (tasks/core.py:316-321). */
uuv_status uuv_observe(uuv_ctx* ctx, const uuv_state* st, const uuv_task* task, double dt,
                       const uuv_task_io* io, void* stream);

/* Number of stat blocks uuv_task_step uses for n_envs (size io->stats to this). */
int64_t uuv_stats_blocks(int64_t n_envs);

/* Reduce io->stats over blocks (fixed order) into out[UUV_ST_COUNT] (device float64);
 * reset != 0 zeroes the running sums afterwards.  Replaces the numpy return
 * reduction of baseline._rollout_returns (baseline.py:109-127). */
uuv_status uuv_rollout_stats(const double* stats, int64_t n_blocks, double* out, int32_t reset,
                             void* stream);

/* Materialise per-env derived parameters (the reference's BatchParams rows,
 * engine.py:193-234) into float64 device buffers, for inspection and tests:
 * out12 = [mass, volume, r_g(3), r_b(3), W, B, added_mass_scale, damping_scale] per env,
 * minv = M^-1 (36 per env), ct_tau = thrust_coeff (a_max) then time_constant (a_max),
 * mounts = (a_max*3) per env.  Any output may be NULL. */
uuv_status uuv_derive_params(uuv_ctx* ctx, const uuv_state* st, double* out12, double* minv,
                             double* ct_tau, double* mounts, void* stream);

/* Validation entry: the first substep's intermediates for every env, without
 * writing state (the quantities engine.py:425-433 forms), into out (n_envs, 48)
 * float64 rows: tau[6] hydro[6] c_rb[6] acc[6] nu_new[6] p_new[3] q_new[4]
 * act_new[8] ok[1] pad[2].  commands as in uuv_step; dt_sub = dt / substeps. */
uuv_status uuv_substep_terms(uuv_ctx* ctx, const uuv_state* st, const void* commands,
                             int64_t cmd_ld, double dt_sub, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UUV_B200_H */
