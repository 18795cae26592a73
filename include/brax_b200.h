/* brax_b200.h — C ABI of the B200-native batched Brax physics step.
 *
 * What it computes: the paper's physics step (arXiv 2106.13281, §3 and Alg. 1,
 * PAPER.md:60-75):  qp_{t+dt} = Brax_system.step(qp_t, actions),
 * i.e. `substeps` repetitions of
 *     kinematic integrator → Σ joints, Σ actuators, Σ colliders (all on the same qp)
 *     → potential integrator (dp_j + dp_a, dt) → collision integrator (dp_c),
 * for n independent environments (the paper's vmap over scenes),
 * with every formula as read in SURVEY.md §8(c) / DESIGN.md "Readings".
 *
 * Library: paper_2106_13281_b200/_lib/libbrax_b200.so (sm_100a only).
 * No CPU fallback exists: every compute entry point launches CUDA kernels.
 *
 * Conventions shared by all entry points
 *  - Return value: brax_status.  On error, brax_last_error_detail() returns a
 *    thread-local human-readable detail ("line:col: msg", "bodies[3].mass: must
 *    be > 0", or CUDA's error string).  Nothing is launched when an argument
 *    check fails.
 *  - Ownership: the library owns brax_config / brax_system objects until the
 *    matching *_destroy.  The caller owns every device buffer and the stream.
 *    brax_step allocates nothing; all scratch is on-chip.
 *  - Device pointers: every pointer in brax_qp, `action` and brax_step_extras is a
 *    CUDA device pointer on the system's device, fp32 / u8 / u32 as stated,
 *    C-contiguous, 16-byte aligned (else BRAX_E_MISALIGNED).
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are stream-ordered and never synchronise; BRAX_OK means
 *    "enqueued".  A failed launch returns BRAX_E_CUDA.
 *  - Thread safety: a brax_system is immutable after creation; concurrent
 *    brax_step calls on distinct streams are safe.
 *  - Device: entry points that launch work make the system's device current for
 *    the call and restore the caller's current device before returning.
 */
#ifndef BRAX_B200_H_
#define BRAX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BRAX_ABI_VERSION 1

typedef enum {
  BRAX_OK = 0,
  BRAX_E_INVALID_ARGUMENT = 1,   /* NULL pointer, negative size, partial aliasing, wrong shape */
  BRAX_E_PARSE = 2,              /* config text: syntax error (detail "line:col: msg") */
  BRAX_E_VALIDATION = 3,         /* config: semantic error (detail "path: msg") */
  BRAX_E_CYCLIC_JOINT_GRAPH = 4, /* joints do not form a forest */
  BRAX_E_UNSUPPORTED_PAIR = 5,   /* collider pair outside the supported set */
  BRAX_E_MISALIGNED = 6,         /* a device pointer is not 16-byte aligned */
  BRAX_E_CUDA = 7,               /* CUDA runtime error (no device, launch failure, ...) */
  BRAX_E_OUT_OF_MEMORY = 8
} brax_status;

/* Contact-slot types (integer contact indexing).  Part of the ABI:
 * brax_system_slot_table reports them and tests compare them bit-exactly. */
typedef enum {
  BRAX_SLOT_SPHERE_PLANE = 0,
  BRAX_SLOT_CAPSULE_PLANE = 1,   /* one slot per capsule end (point 0 = c + l·a, 1 = c − l·a) */
  BRAX_SLOT_BOX_PLANE = 2,       /* 8 corner slots, point k ↔ signs (k&1, k&2, k&4) of (hx, hy, hz) */
  BRAX_SLOT_SPHERE_SPHERE = 3,
  BRAX_SLOT_SPHERE_CAPSULE = 4,  /* sphere is A */
  BRAX_SLOT_CAPSULE_CAPSULE = 5  /* lower collider index is A */
} brax_slot_type;

/* ---------------------------------------------------------------- config
 * Text form: the ProtoBuf text subset of the paper's App. A:
 * top-level dt, substeps, gravity{x y z}, friction, elasticity, baumgarte_erp,
 * repeated bodies{name mass inertia{} frozen{position{} rotation{} all} colliders{
 * position{} rotation{} (sphere{radius} | capsule{radius length end} |
 * box{halfsize{}} | plane{})}}, joints{name parent child stiffness spring_damping
 * angular_damping limit_stiffness angular_stiffness parent_offset{} child_offset{}
 * rotation{} reference_rotation{} angle_limit{min max}×dof}, actuators{name joint
 * strength (torque{} | angle{})}, collide_include{first second},
 * defaults{qps{name pos{} rot{}}}.  Angles in degrees (Euler, intrinsic X-Y-Z). */
typedef struct brax_config brax_config;

/* Parse + validate `len` bytes of text (need not be NUL-terminated).
 * *out receives a new config on BRAX_OK (free with brax_config_destroy).
 * Errors: BRAX_E_PARSE, BRAX_E_VALIDATION, BRAX_E_CYCLIC_JOINT_GRAPH,
 * BRAX_E_UNSUPPORTED_PAIR, BRAX_E_INVALID_ARGUMENT. */
brax_status brax_config_parse(const char *text, size_t len, brax_config **out);
void brax_config_destroy(brax_config *cfg);

/* Programmatic form ("users can define systems in text, or they can
 * define systems programmatically"; the App. A Python listing).
 * Host structs, read only during the call (the caller keeps ownership; names are
 * copied).  Quaternions are (w, x, y, z) and must be unit (|q| = 1 ± 1e-6); joint
 * limits are in radians in [−π, π] (R9); frozen flags are 0 or 1 per axis (App. A
 * `frozen`).  Bodies, joints and actuators are referenced by index;
 * colliders are attached to bodies by index and take the text format's global order
 * (body order, then descriptor order within a body).  pairs == NULL selects the
 * all-pairs rule (R19: collider pairs on different, non-jointed, not-both-static
 * bodies), else the listed body pairs in order (the text `collide_include`).
 * The resulting config equals the text parse of the same scene (same integer
 * tables, same default_qp).  Errors: as brax_config_parse minus BRAX_E_PARSE; the
 * detail names the offending descriptor ("joints[2].stiffness: must be > 0"). */
typedef enum { BRAX_SHAPE_SPHERE = 0, BRAX_SHAPE_CAPSULE = 1, BRAX_SHAPE_BOX = 2, BRAX_SHAPE_PLANE = 3 } brax_shape;
typedef enum { BRAX_ACTUATOR_TORQUE = 0, BRAX_ACTUATOR_ANGLE = 1 } brax_actuator_kind;
typedef struct {
  const char *name;         /* may be NULL (then "body<i>"); names must be unique */
  double mass;              /* > 0 */
  double inertia[3];        /* body-frame diagonal, > 0 (App. A inertia{x y z}) */
  double frozen_pos[3], frozen_rot[3]; /* 1 = axis frozen */
  double init_pos[3], init_rot[4];     /* pose of a root body in default_qp (text: defaults.qps) */
} brax_body_desc;
typedef struct {
  const char *name;
  int32_t parent, child;    /* body indices */
  double parent_offset[3], child_offset[3];
  double rotation[4], reference_rotation[4]; /* joint frame J_p; reference frame (R7) */
  int32_t dof;              /* 0..3 free axes (the text form's number of angle_limit entries) */
  double limit_lo[3], limit_hi[3];           /* radians, first `dof` used */
  double stiffness;         /* > 0 */
  double spring_damping, angular_damping;    /* >= 0 */
  double limit_stiffness, angular_stiffness; /* >= 0; negative = stiffness (R8) */
} brax_joint_desc;
typedef struct {
  const char *name;
  int32_t joint;            /* joint index; at most one actuator per joint, dof >= 1 */
  int32_t kind;             /* brax_actuator_kind */
  double strength;
} brax_actuator_desc;
typedef struct {
  int32_t body;             /* body index */
  int32_t shape;            /* brax_shape */
  double pos[3], rot[4];    /* pose in the body frame */
  double radius, length;    /* sphere / capsule (length includes the caps, R17) */
  double halfsize[3];       /* box */
  int32_t capsule_end;      /* 0 both ends, +1 / −1 one end (R17) */
} brax_collider_desc;
typedef struct { int32_t first, second; } brax_body_pair;
typedef struct {
  double dt;                /* > 0 */
  int32_t substeps;         /* >= 1 */
  double gravity[3];
  double friction, elasticity, baumgarte_erp; /* μ >= 0, e in [0, 1], β in (0, 1] (R13) */
  int32_t n_bodies, n_joints, n_actuators, n_colliders, n_pairs;
  const brax_body_desc *bodies;
  const brax_joint_desc *joints;
  const brax_actuator_desc *actuators;
  const brax_collider_desc *colliders;
  const brax_body_pair *pairs;               /* NULL = all-pairs rule */
} brax_config_desc;
brax_status brax_config_from_desc(const brax_config_desc *desc, brax_config **out);

/* Host-only introspection of a parsed config (no GPU needed). */
brax_status brax_config_counts(const brax_config *cfg, int32_t *n_bodies, int32_t *n_joints, int32_t *act_dim,
                               int32_t *n_slots);          /* any output may be NULL */
/* Integer contact-slot table, host [C][7] int32 (see brax_system_slot_table). */
brax_status brax_config_slot_table(const brax_config *cfg, int32_t *out);
/* default_qp in fp64 (host): pos [B][3], rot [B][4] (velocities are zero). */
brax_status brax_config_default_qp(const brax_config *cfg, double *pos, double *rot);


/* ---------------------------------------------------------------- system
 * The paper's `system`: immutable device-resident static
 * tables (bodies, joints with their actuators, contact slots, per-body incidence
 * lists, warp work plan) built from a config.  `cuda_device` selects the GPU.
 * Errors: BRAX_E_INVALID_ARGUMENT, BRAX_E_CUDA, BRAX_E_OUT_OF_MEMORY. */
typedef struct brax_system brax_system;
brax_status brax_system_create(const brax_config *cfg, int cuda_device, brax_system **out);
void brax_system_destroy(brax_system *sys);

typedef struct {
  int32_t n_bodies;        /* B: rows per env in every QP array (incl. static bodies) */
  int32_t n_dynamic;       /* bodies with at least one unfrozen axis */
  int32_t n_joints;        /* J */
  int32_t act_dim;         /* A: action width (actuators in config order, dof-major) */
  int32_t n_contact_slots; /* C */
  int32_t substeps;        /* S */
  float dt;                /* step length; substep h = dt / S */
  int32_t warps_per_block; /* launch shape of the step kernel (32 envs per block) */
  int32_t n_lint_warnings; /* stability lint (R6) */
  int32_t smem_bytes;      /* dynamic shared memory per block of the step kernel */
} brax_system_info;
brax_status brax_system_get_info(const brax_system *sys, brax_system_info *out);

/* Integer contact-slot table, host buffer [C][7] int32 row-major:
 * (pair index, brax_slot_type, body A, body B, collider A, collider B, point). */
brax_status brax_system_slot_table(const brax_system *sys, int32_t *out);

/* Tracing: when enabled, every subsequent step launch adds, per block, the SM
 * cycles thread 0 spent in [0] the prologue (tables + QP staging), [1] joints,
 * actuators and contacts, [2] the body integrators, [3] the epilogue (write-back);
 * brax_system_phase_cycles reads the sums (synchronising) and resets them.
 * Not thread-safe with concurrent launches of the same system. */
brax_status brax_system_set_tracing(brax_system *sys, int enable);
brax_status brax_system_phase_cycles(brax_system *sys, uint64_t out[4]);

/* Launch configuration of the step kernel.  Every configuration
 * computes bit-identical results (explicit rounding of every operation), so the
 * choice only affects speed.  brax_step itself never tunes, allocates or
 * synchronises: it uses the configuration brax_system_tune measured for its n_envs,
 * else a size heuristic.  brax_system_tune(sys, in, action, n_envs, stream) times one
 * step of every configuration on the caller's state `in` (read only; outputs go to a
 * stream-ordered scratch allocation that is freed before return), synchronises
 * `stream`, and remembers the fastest for n_envs (thread-safe; call it once per batch
 * size, outside graph capture).  brax_system_set_autotune(sys, 0) makes
 * brax_system_tune a no-op.  Environment overrides for experiments:
 * BRAX_PLAN="G,V", BRAX_MAXREG=R.
 * brax_system_launch_config writes, for a launch of n_envs envs, out[6] =
 * {G lane groups per warp, V envs per lane, E envs per block, warps per block,
 * register budget, flags: bit 0 measured by the autotuner, bit 1 the fixed-shape
 * body-gather variant, bit 2 the lean kernel}; it does not tune.  BRAX_FIXED_GATHER=0/1
 * selects the gather variant together with BRAX_PLAN. */
brax_status brax_system_set_autotune(brax_system *sys, int enable);
brax_status brax_system_launch_config(const brax_system *sys, int64_t n_envs, int32_t out[6]);

/* Launch overlap (DESIGN.md §5 "Launch overlap").  The step launches of a system
 * (brax_step, brax_step_ex, brax_rollout*, brax_env_step*) register per group of 8 envs
 * on device counters the system owns (2 x 2^19 words, allocated by brax_system_create);
 * consecutive such launches on one stream, of the same system and n_envs, whose
 * buffers are identical array for array or disjoint, start each block as soon as the
 * earlier launches on its envs have finished instead of after the whole previous
 * grid.  Results are bit-identical either way.  The library tracks its own launches
 * per stream (and per stream capture); a kernel of OTHER code that uses programmatic
 * dependent launch and triggers early, placed between two step launches on the same
 * stream and writing their buffers, is not seen — separate such work with an event or
 * set BRAX_NO_OVERLAP=1 (every launch then waits for the previous grid). */

/* Lint warning i (0 <= i < n_lint_warnings) as text; NULL if out of range. */
const char *brax_system_lint_warning(const brax_system *sys, int32_t i);

/* default_qp: host fp32 buffers of B rows each:
 * pos [B][3], rot [B][4] (w,x,y,z), vel [B][3], ang [B][3]. */
brax_status brax_default_qp(const brax_system *sys, float *h_pos, float *h_rot, float *h_vel, float *h_ang);

/* ---------------------------------------------------------------- state
 * QP: structure of arrays, env-major: pos [n][B][3], rot [n][B][4]
 * (w,x,y,z), vel [n][B][3], ang [n][B][3]; fp32 device pointers. */
typedef struct {
  float *pos, *rot, *vel, *ang;
} brax_qp;

/* Launch-configuration tuning for n_envs (see "Launch configuration" above): reads `in`
 * and `action` (as brax_step would), allocates stream-ordered scratch, synchronises
 * `stream`.  Not capturable in a CUDA graph. */
brax_status brax_system_tune(brax_system *sys, brax_qp in, const float *action, int64_t n_envs, void *stream);

/* Broadcast default_qp to n_envs envs, then for every non-static body add
 * v += M_pos ⊙ vel_noise·u, ω += M_rot ⊙ ang_noise·u with u ∈ [−1, 1) from
 * Philox4x32-10(key = seed, counter = (env, body, field, 0)).
 * n_envs == 0 is a no-op.  Errors: INVALID_ARGUMENT, MISALIGNED, CUDA. */
brax_status brax_reset(const brax_system *sys, brax_qp out, int64_t n_envs, uint64_t seed, float vel_noise,
                       float ang_noise, void *stream);

/* One Brax step of n_envs envs: out = step(in, action).  action: [n][act_dim] fp32
 * device (may be NULL iff act_dim == 0), held for all substeps.  in == out (all four
 * pointers equal) is allowed; partial aliasing is BRAX_E_INVALID_ARGUMENT.
 * Static (fully frozen) bodies are copied through bit for bit. */
brax_status brax_step(const brax_system *sys, brax_qp in, const float *action, brax_qp out, int64_t n_envs,
                      void *stream);

typedef struct {
  uint32_t *status;        /* [n] bit0 non-finite value, bit1 |value| > 1e6; or NULL */
  uint8_t *contact_active; /* [n][C] number of substeps each slot was active; or NULL */
  float *contact_dp;       /* [n][B][6] Σ over the step's substeps of the collision integrator's
                              velocity change (Δv, Δω) per body (the input of Table 1's
                              contact observations); for brax_rollout, of its last
                              step; 16-byte aligned; or NULL */
} brax_step_extras;

/* brax_step plus optional per-env outputs (NULL extras or NULL members = skip). */
brax_status brax_step_ex(const brax_system *sys, brax_qp in, const float *action, brax_qp out, int64_t n_envs,
                         const brax_step_extras *extras, void *stream);

/* Run `n_steps` consecutive steps inside ONE kernel launch (the QP stays on-chip
 * between steps).  actions: [n_steps][n][act_dim].
 * Equivalent to n_steps brax_step calls (bitwise, same binary). */
brax_status brax_rollout(const brax_system *sys, brax_qp in, const float *actions, int64_t n_steps, brax_qp out,
                         int64_t n_envs, const brax_step_extras *extras, void *stream);

/* ---- NEXT-2: on-device random actions (no action buffer in HBM).  Step t of the
 * launch (global step step0 + t) of env i uses, for action component k,
 *   a_k = (x_(k mod 4) >> 8)·2⁻²³ − 1 ∈ [−1, 1),  x = Philox4x32-10(key = seed,
 *   counter = (env_offset + i, step0 + t, ⌊k/4⌋, 0x41435431)),
 * the same generator as the reset noise (separate counter space). */
typedef struct {
  uint64_t seed;
  int64_t env_offset;  /* global index of env 0 of this batch */
  int64_t step0;       /* global step index of the launch's first step */
} brax_random_actions;
/* brax_rollout with on-device random actions. */
brax_status brax_rollout_random(const brax_system *sys, brax_qp in, int64_t n_steps, brax_qp out, int64_t n_envs,
                                const brax_random_actions *ra, const brax_step_extras *extras, void *stream);

/* ---- NEXT-4: differentiable step, forward mode.  One step (as brax_step) that
 * also propagates a tangent: dout = ∂step/∂(qp, a) · (din, daction), computed with
 * (value, tangent) arithmetic through every operation of the kernel (exact
 * derivative of the fp32 step, not a finite difference).  Conventions at kinks
 * (R35): min / max / clamp follow the selected argument (the first on
 * ties), a contact's activity and the friction cone's regime are those of the
 * primal.  `out` is bit-identical to brax_step's output.  din members may be
 * NULL (zero tangent); daction may be NULL (zero).  Columns of the full Jacobian
 * ∂Q_out/∂(Q_in, a) are JVPs with unit tangents. */
brax_status brax_step_jvp(const brax_system *sys, brax_qp in, const float *action, brax_qp din,
                          const float *daction, brax_qp out, brax_qp dout, int64_t n_envs, void *stream);

/* Reverse mode (cotangent) of one step: g_in = (∂Q_out/∂Q_in)ᵀ·g_out and
 * g_action = (∂Q_out/∂a)ᵀ·g_out per env — the transpose of brax_step_jvp's
 * derivative (same conventions, R35), in one kernel launch (backwards
 * substep sweep).  Joints, plane contacts and the quaternion update
 * use hand-derived adjoints (equal to the transposed value+tangent derivative up to
 * fp32 rounding); with the environment variable BRAX_VJP_LOCAL_AD set they use local
 * value+tangent evaluations instead (cross-check).  g_out members may be NULL (zero); g_action may be
 * NULL (not written) and is [n][act_dim].  in is not modified.  With the
 * environment variable BRAX_VJP_COLUMNS set, the same result is assembled from
 * 13B + A JVP launches instead (cross-check; stream-ordered scratch). */
brax_status brax_step_vjp(const brax_system *sys, brax_qp in, const float *action, brax_qp g_out, brax_qp g_in,
                          float *g_action, int64_t n_envs, void *stream);

/* ---- NEXT-1: Gym-like env epilogue fused into the step (Table 1;
 * :505-509 rewards; R30-R35).  Needs a `task { ... }` block in the system
 * text.  Per step and env, after the last substep and while the bodies are still
 * in shared memory:
 *   reward = ((x'_torso − x_torso)·forward)/dt + survive_reward − ctrl_cost·Σ a²
 *   (goal tasks, R36 — grasp / fetch: the forward term is
 *   (|x_O − x_T| − |x'_O − x_T|)/dt + bonus·[|x'_O − x_T| < radius] for the object O and
 *   the frozen marker body T; a hit moves T to x̄_T + range ⊙ u(env, T, 2 + steps', episode),
 *   a reset of episode k to x̄_T + range ⊙ u(env, T, 2, k); obs gains x_T − x_O, x_O − x_torso,
 *   v_O before the contact terms)
 *   done   = torso z' outside healthy_z, or steps + 1 >= episode_length
 *   done envs auto-reset: default_qp + the task's reset noise with Philox counter
 *   (env_offset + env, body, field, episode + 1); steps = 0, episode += 1
 *   obs    = [z, quat | joint angles | v, ω | joint rates | clip(contact Δv, Δω, ±1)
 *            per body if contact_obs] of the returned (possibly reset) state.
 * All arrays are device arrays; steps and episode are updated in place. */
typedef struct brax_env_io {
  float *obs;          /* [n_steps][n][obs_dim] (brax_env_reset: [n][obs_dim]) or NULL */
  float *reward;       /* [n_steps][n] or NULL */
  uint8_t *done;       /* [n_steps][n] or NULL */
  int32_t *steps;      /* [n] in/out: steps since the env's last reset (required) */
  uint32_t *episode;   /* [n] in/out: resets so far = reset-noise counter (required) */
  uint64_t seed;       /* reset-noise key (as brax_reset's seed) */
  int64_t env_offset;  /* global index of env 0 of this batch (multi-GPU shards) */
} brax_env_io;
/* out = {has_task, obs_dim, episode_length, torso body index (or -1)}. */
brax_status brax_system_task_info(const brax_system *sys, int32_t out[4]);
/* n_steps steps with the epilogue after each (in may equal out; actions [n_steps][n][A]).
 * BRAX_E_INVALID_ARGUMENT if the system has no task or steps / episode are NULL. */
brax_status brax_env_step(const brax_system *sys, brax_qp in, const float *actions, int64_t n_steps, brax_qp out,
                          int64_t n_envs, const brax_env_io *io, void *stream);
/* brax_env_step with on-device random actions (NEXT-2; ctrl cost uses them). */
brax_status brax_env_step_random(const brax_system *sys, brax_qp in, int64_t n_steps, brax_qp out, int64_t n_envs,
                                 const brax_random_actions *ra, const brax_env_io *io, void *stream);
/* Episode-0 reset (the task's reset noise, Philox counter (env_offset + env, b, f, 0); goal tasks: the marker at x̄_T + range ⊙ u(env, T, 2, 0)),
 * steps = episode = 0, and io->obs (if not NULL). */
brax_status brax_env_reset(const brax_system *sys, brax_qp out, int64_t n_envs, const brax_env_io *io,
                           void *stream);
/* Observation rows [n][obs_dim] of a QP (contact terms zero); the QP is not modified. */
brax_status brax_env_observe(const brax_system *sys, brax_qp qp, int64_t n_envs, float *obs, void *stream);


const char *brax_status_string(brax_status s);
const char *brax_last_error_detail(void);
int brax_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BRAX_B200_H_ */
