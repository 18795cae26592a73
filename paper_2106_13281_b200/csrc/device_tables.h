// device_tables.h — layout of the system's static tables as seen by the step
// kernel.  Built on the host by system.cpp, uploaded once at brax_system_create
// as one 32-bit-word blob, staged into shared memory by every block.
//
// All per-item structs are plain 4-byte words so they can be read straight out
// of the shared-memory copy; a warp reads one item's struct with warp-uniform
// (broadcast) addresses.
#pragma once
#include <stdint.h>

namespace brax {

constexpr int kEnvsPerBlock = 32;  // lane = env; warp = work item
constexpr int kMaxWarps = 16;      // 512 threads per block at most
constexpr int kQPFields = 13;      // pos 0-2, rot 3-6 (w,x,y,z), vel 7-9, ang 10-12
constexpr int kJointOut = 9;       // F (child), T child, T parent
constexpr int kSlotOut = 10;       // P, rA×P, rB×P, active

struct DBody {              // 12 words
  float inv_mass;
  float inv_inertia[3];     // 1 / body-frame diagonal inertia
  float mpos[3], mrot[3];   // 1 − frozen (App. A `frozen`)
  int32_t is_static;        // all 6 axes frozen: never integrated (R21)
  int32_t rot_frozen;       // all 3 rotation axes frozen: q untouched
};

struct DJoint {             // 32 words
  int32_t parent, child, dof, act_kind, act_offset, pad;
  float o_p[3], o_c[3];     // anchor offsets in the parent / child body frames
  float jp[4], jc[4];       // joint frames J_p = rotation, J_c = conj(reference_rotation) ⊗ rotation
  float k, c_l, c_a, k_l, k_a;
  float lo[3], hi[3];       // limits (rad) of the free axes
  float strength;           // actuator strength (act_kind ≥ 0)
};

struct DSlot {              // 36 words
  int32_t type, a, b, point, a_static, b_static;
  float ca_pos[3], ca_rot[4];  // collider A pose in body A
  float cb_pos[3], cb_rot[4];  // collider B pose in body B
  float ra, ella, rb, ellb;    // radii and capsule segment half-lengths ℓ = L/2 − r
  float hs[3];                 // box half-extents (A), signed by `point`
  float inv_mass_a, inv_mass_b;
  float inv_inertia_a[3], inv_inertia_b[3];
  float pad;
};

// Incidence entry kinds (body gather, fixed order: joints by index, then slots by index).
enum IncKind { kIncJointChild = 0, kIncJointParent = 1, kIncSlotA = 2, kIncSlotB = 3 };
__host__ __device__ inline int32_t inc_pack(int kind, int index) { return (kind << 16) | index; }

struct DHeader {            // passed by value as a kernel argument
  int32_t B, J, C, A, S, W;
  float h, beta_over_h, mu, e;
  float g[3];
  int32_t blob_words;       // total words (padded to a multiple of 4)
  int32_t off_bodies, off_joints, off_slots;
  int32_t off_item_begin, off_items;   // per warp: items (j < J: joint j; J + c: slot c)
  int32_t off_body_begin, off_bodies_of_warp;
  int32_t off_inc_begin, off_inc;      // per body: incidence list
  uint32_t row_magic[4];    // ⌈2³²/(B·K)⌉ for K = 3, 4 (index 0: K=3, 1: K=4), A (index 2)
};

}  // namespace brax
