// device_tables.h — layout of the system's static tables as seen by the step
// kernel.  Built on the host by system.cpp, uploaded once at brax_system_create
// as one 32-bit-word blob, staged into shared memory by every block.
//
// All per-item structs are plain 4-byte words so they can be read straight out
// of the shared-memory copy; a warp reads one item's struct with warp-uniform
// (broadcast) addresses.
#pragma once
#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <stdint.h>
#endif
#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define BRAX_HD __host__ __device__
#else
#define BRAX_HD
#endif

namespace brax {

constexpr int kEnvsPerBlock = 32;  // lane = env; warp = work item
// dynamic shared memory a block may request: 227 KB minus the kernel's static
// shared memory (the tracing sums)
constexpr int kMaxDynSmem = 227 * 1024 - 128;
constexpr int kMaxWarps = 16;      // 512 threads per block at most
// Cross-launch env-granule dependencies of the lean kernel (DESIGN.md §5 "Launch
// overlap"): per granule of kGranule envs, how many launches have started on it and
// how many have finished; kMaxGranules granules per system (2^22 envs).
constexpr int kGranule = 8;
constexpr int kMaxGranules = 1 << 19;

// Flag bits (precomputed on the host; warp-uniform tests in the kernel).  An
// exact-zero offset, identity frame, isotropic inertia or all-free mask makes the
// corresponding arithmetic an exact identity, which the kernel then skips.
enum : int32_t {
  kFlagIso = 1,       // body: isotropic inertia (I_w⁻¹ v = i·v)
  kFlagFreePos = 2,   // body: no frozen position axis
  kFlagFreeRot = 4,   // body: no frozen rotation axis
};
enum : int32_t {
  kJZeroOp = 1, kJZeroOc = 2, kJIdentP = 4, kJIdentC = 8, kJNoCl = 16, kJNoCa = 32,
};
enum : int32_t {
  kSZeroPa = 1, kSZeroPb = 2, kSIdentA = 4, kSIdentB = 8, kSIsoA = 16, kSIsoB = 32,
  kSZeroLa = 64,  // plane contacts: the A-side point in body A's frame (pa_local) is the origin
};

// Every struct is a whole number of 16-byte vectors so the kernel reads it with
// LDS.128 from the shared-memory copy (the blob offsets are 4-word aligned).
struct alignas(16) DBody {  // 16 words
  float inv_mass;
  float inv_inertia[3];     // 1 / body-frame diagonal inertia
  float mpos[3];            // 1 − frozen position (App. A `frozen`)
  int32_t is_static;        // all 6 axes frozen: never integrated (R21)
  float mrot[3];            // 1 − frozen rotation
  int32_t rot_frozen;       // all 3 rotation axes frozen: q untouched
  int32_t flags, pad0, pad1, pad2;
};
struct alignas(16) DJoint {  // 36 words
  int32_t parent, child, dof, act_kind;
  int32_t act_offset, flags, obs_off, pad1;  // obs_off: Σ dof of the joints before this one (R32)
  float o_p[3], k;          // parent anchor offset; stiffness
  float o_c[3], c_l;        // child anchor offset; linear (spring) damping
  float jp[4];              // J_p = rotation
  float jc[4];              // J_c = conj(reference_rotation) ⊗ rotation
  float lo[3], k_l;         // limits (rad) of the free axes; limit stiffness
  float hi[3], k_a;         // ... ; alignment stiffness
  float c_a, strength, pad2, pad3;  // angular damping; actuator strength (act_kind ≥ 0)
};
struct alignas(16) DSlot {  // 44 words
  int32_t type, a, b, point;
  int32_t a_static, b_static, flags, pad0;
  float ca_pos[3], ra;      // collider A offset in body A; radius A
  float ca_rot[4];          // collider A rotation in body A
  float cb_pos[3], rb;
  float cb_rot[4];
  float ell_a, ellb, inv_mass_a, inv_mass_b;  // ell_a: signed capsule-end offset (+ℓ end 0, −ℓ end 1)
  float corner[3], pad1;    // box: signed half-extent corner of slot `point`
  float inv_inertia_a[3], pad2;
  float inv_inertia_b[3], pad3;
  // plane contacts: the A-side point in body A's frame, ca_pos + rotate(ca_rot, v) with v = 0
  // (sphere), ±ℓ·ẑ (capsule end), the signed half-extent corner (box): its world position is
  // x_A + rotate(q_A, pa_local) — one rotation instead of the collider frame q_A ⊗ ca_rot
  float pa_local[3], pad4;
};

// Shared-memory layouts (words): per (item, lane) records, 16-byte aligned,
// strides chosen so a warp's LDS.128 / STS.128 are bank-conflict free (an odd
// number of 16-byte units).  One env per lane (V = 1):
constexpr int kQS = 20;   // QP record: pos 0-2 | rot 4-7 (w,x,y,z) | vel 8-10 | ang 12-14
constexpr int kJS = 12;   // joint record: F 0-2 | T_child 4-6 | T_parent 8-10
constexpr int kCS = 12;   // slot record: P 0-2, active 3 | r_A×P 4-6 | r_B×P 8-10
// Two envs per lane (V = 2): one record per lane holds both envs interleaved
// component by component — field f, component c, env half h at word
// 8f + 4(c >> 1) + 2(c & 1) + h — so an LDS.128 yields two (env0, env1) register
// pairs, the operands of the packed FP32 instructions (FFMA2 / FMUL2 / FADD2).
constexpr int kQS2 = 36;  // pos 0-7 | rot 8-15 | vel 16-23 | ang 24-31
constexpr int kJS2 = 28;  // F 0-7 | T_child 8-15 | T_parent 16-23
constexpr int kCS2 = 28;  // P 0-5, active 6-7 | r_A×P 8-15 | r_B×P 16-23
BRAX_HD inline int32_t rec_q(int32_t V) { return V == 2 ? kQS2 : kQS; }
BRAX_HD inline int32_t rec_j(int32_t V) { return V == 2 ? kJS2 : kJS; }
BRAX_HD inline int32_t rec_c(int32_t V) { return V == 2 ? kCS2 : kCS; }

// Incidence entries of the body gather (fixed order: joints by index, then slots
// by index, R29): (item index << 4) | torque-word offset in the record (4 for the
// child / A side, 8 for the parent / B side; the side also fixes the sign).
BRAX_HD inline int32_t inc_pack(int index, bool second_side) { return (index << 4) | (second_side ? 8 : 4); }

// Shared-memory layout of the step kernel (words; every region 16-byte aligned).
//   [2 mbarriers][tables][QP records B·L·rec_q][U][sA A·E][action staging E·A][counts C·E][status E]
//   [env epilogue, systems with a task: x0 3E | steps E | episode E | reset flag E | contact Δv 6·B·E]
//   (the contact Δv region also serves brax_step_extras.contact_dp of the physics-only kernel)
// with L = E/V lanes (records) per body or item.  U holds the joint and slot
// records during the substeps, the contiguous TMA staging chunks (pos|rot|vel|ang,
// E·B·13 words) while loading / storing, and the observation rows (E·obs_dim) in
// the env epilogue.
struct SmemLayout {
  int32_t blob, q, u, a, astg, cnt, stat, x0, steps, ep, rst, co, total_words;
};
BRAX_HD inline int32_t round4(int32_t w) { return (w + 3) & ~3; }
// E envs per block in LG lane slots; paired: two values per slot (V = 2 envs, or
// value + tangent of the JVP step); RW: words per row of a per-env array (actions,
// contact counts, contact Δv): LG·(paired ? 2 : 1).
BRAX_HD inline SmemLayout smem_layout(int32_t B, int32_t J, int32_t C, int32_t A, int32_t E, int32_t LG,
                                      int32_t paired, int32_t blob_words, int32_t obs_dim, int32_t contact_obs,
                                      int32_t contact_dp = 0) {
  SmemLayout L;
  const int32_t V = paired ? 2 : 1, RW = LG * V;
  L.blob = 4;
  L.q = L.blob + round4(blob_words);
  L.u = L.q + B * LG * rec_q(V);
  int32_t u = J * LG * rec_j(V) + C * LG * rec_c(V);
  if (u < E * B * 13) u = E * B * 13;
  if (u < E * obs_dim) u = E * obs_dim;
  L.a = L.u + round4(u);
  L.astg = L.a + round4(A * RW);
  L.cnt = L.astg + round4(A * E);
  L.stat = L.cnt + round4(C * RW);
  L.x0 = L.stat + round4(E);
  const int32_t env = obs_dim > 0 ? 1 : 0;
  L.steps = L.x0 + env * round4(3 * E);
  L.ep = L.steps + env * round4(E);
  L.rst = L.ep + env * round4(E);
  L.co = L.rst + env * round4(E);
  L.total_words = L.co + ((env && contact_obs) || contact_dp ? round4(6 * B * RW) : 0);
  return L;
}

// Env epilogue parameters (NEXT-1, R30-R35); present == 0: no task.
struct DTask {
  int32_t present, torso, episode_length, contact_obs;
  int32_t nq, obs_dim, has_healthy, has_goal;
  float fwd[3], dt;
  float survive, ctrl_cost, z_lo, z_hi;
  float noise_vel, noise_ang, radius, bonus;
  int32_t obj, target, pad0, pad1;  // goal task (R36): object body, frozen marker body
  float range[3], pad2;             // marker placement half-extents
};

// Arguments of one step launch (device pointers; see include/brax_b200.h).
struct StepArgs {
  const float *pos_in, *rot_in, *vel_in, *ang_in;
  float *pos_out, *rot_out, *vel_out, *ang_out;
  const float* actions;        // [n_steps][n][A] (NULL iff A == 0)
  uint32_t* status;            // [n] or NULL
  uint8_t* contact_active;     // [n][C] or NULL
  int64_t n_envs;
  int64_t n_steps;
  int32_t bulk_ok;             // all QP pointers 16-byte aligned: TMA bulk staging for full blocks
  int32_t act_bulk_ok;         // actions 16-byte aligned and n·A % 4 == 0: TMA bulk action staging
  unsigned long long* phase_cycles;  // [4] per-phase SM cycles summed over blocks (tracing), or NULL
  int32_t diag_block;          // diagnostics (BRAX_DIAG_BLOCK=b+1): block b prints per-warp clock stamps of one substep
  // env epilogue (NEXT-1): env == 0 -> physics only.  With env == 1 every step also
  // writes reward [t][n], done [t][n], obs [t][n][obs_dim] and auto-resets done envs;
  // n_steps == 0 with env == 1 only observes (obs [n][obs_dim], QP not written).
  int32_t env;
  float* obs;
  float* reward;
  uint8_t* done;
  int32_t* steps;              // [n] in/out
  uint32_t* episode;           // [n] in/out
  uint64_t seed;               // reset-noise key
  int64_t env_offset;          // global index of env 0 (Philox counter)
  const float* dqp;            // default_qp: pos [B][3] | rot [B][4]
  const float* masks;          // per body: mpos[3] mrot[3] static
  // NEXT-2 on-device random actions (actions == NULL): a_k = u(Philox(key = act_seed,
  // counter = (act_env_offset + env, act_step0 + step, k/4, kActTag)))_(k mod 4) ∈ [−1, 1)
  int32_t act_random;
  uint64_t act_seed;
  int64_t act_env_offset, act_step0;
  // NEXT-4 JVP (lane type D1): tangents of the inputs (NULL = zero) and of the outputs
  const float *dpos_in, *drot_in, *dvel_in, *dang_in, *dactions;
  float *dpos_out, *drot_out, *dvel_out, *dang_out;
  float* contact_dp;           // [n][B][6] Σ_substeps collision-integrator (Δv, Δω), or NULL (physics kernel only)
};
constexpr uint32_t kActTag = 0x41435431u;  // "ACT1": separates the action stream from the reset stream

// A work plan for one lane-group count G (E = 32/G envs per block): each warp's
// lanes form G groups of E lanes; group g runs item items[step*G + g] on the
// block's E envs (-1 = idle).  Items sharing a step have the same code class,
// so the groups do not diverge.
constexpr int kNumPlans = 6;       // (G, V) = (1,1) (2,1) (4,1) (1,2) (2,2) (4,2)
struct DPlan {
  int32_t G, V, E, W;  // lane groups per warp, envs per lane, envs per block E = 32·V/G, warps
  int32_t off_item_begin, off_items;          // per warp: item steps [begin, end); items[step*G + g]
  int32_t off_body_begin, off_bodies_of_warp;  // per warp: body steps; bodies[step*G + g]
  int32_t smem_bytes, smem_bytes_jvp, smem_bytes_env, smem_bytes_cdp;  // physics | JVP (V = 1) | env | + contact_dp
};

struct DHeader {            // passed by value as a kernel argument
  int32_t B, J, C, A, S;
  float h, beta_over_h, mu, e;
  float g[3];
  int32_t blob_words;       // total words (padded to a multiple of 4)
  int32_t off_bodies, off_joints, off_slots;
  int32_t off_jinc_begin, off_jinc;    // per body: joint incidence entries
  int32_t off_cinc_begin, off_cinc;    // per body: contact-slot incidence entries
  uint32_t row_magic[4];    // ⌈2³²/(B·K)⌉ for K = 3, 4 (index 0: K=3, 1: K=4), A (index 2)
  DTask task;
  DPlan plan[kNumPlans];
};

}  // namespace brax
