// config.h — host-side scene description of the library (C++17).
//
// Parsed from the App. A text format by config.cpp; turned
// into device tables by system.cpp.  Independent of oracle/ (no shared code).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "brax_b200.h"

namespace brax {

// Error carrying a brax_status and a detail string; converted to a status at
// the C-ABI boundary (capi.cpp).
struct Error : std::runtime_error {
  brax_status status;
  Error(brax_status s, const std::string& detail) : std::runtime_error(detail), status(s) {}
};

enum ColliderKind { kSphere = 0, kCapsule = 1, kBox = 2, kPlane = 3 };
enum ActuatorKind { kNoActuator = -1, kTorque = 0, kAngle = 1 };

struct Collider {
  int body = 0;
  ColliderKind kind = kSphere;
  double pos[3] = {0, 0, 0};      // local offset in the body frame
  double rot[4] = {1, 0, 0, 0};   // local rotation (w, x, y, z)
  double radius = 0, length = 0;  // sphere / capsule (length includes the caps, R17)
  int end = 0;                    // capsule end selector: 0 both, +1, -1
  double halfsize[3] = {0, 0, 0}; // box
};

struct Body {
  std::string name;
  double mass = 1;
  double inertia[3] = {1, 1, 1};
  double frozen_pos[3] = {0, 0, 0}, frozen_rot[3] = {0, 0, 0};
  double init_pos[3] = {0, 0, 0}, init_rot[4] = {1, 0, 0, 0};
  bool is_static() const {
    for (int i = 0; i < 3; ++i)
      if (frozen_pos[i] != 1.0 || frozen_rot[i] != 1.0) return false;
    return true;
  }
  bool rot_frozen() const { return frozen_rot[0] == 1.0 && frozen_rot[1] == 1.0 && frozen_rot[2] == 1.0; }
};

struct Joint {
  std::string name;
  int parent = 0, child = 0;
  double stiffness = 0, spring_damping = 0, angular_damping = 0, limit_stiffness = 0, angular_stiffness = 0;
  double parent_offset[3] = {0, 0, 0}, child_offset[3] = {0, 0, 0};
  double rotation[4] = {1, 0, 0, 0}, reference_rotation[4] = {1, 0, 0, 0};
  int dof = 0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // radians
  // actuator folded into its joint (at most one per joint)
  ActuatorKind act_kind = kNoActuator;
  double act_strength = 0;
  int act_offset = 0;
};

struct Actuator {
  std::string name;
  int joint = 0;
  double strength = 0;
  ActuatorKind kind = kTorque;
  int act_offset = 0;
};

struct Pair { int col_a, col_b, type; };
struct Slot { int pair, type, a, b, col_a, col_b, point; };

// Locomotion env epilogue (NEXT-1; R30-R35): reward, done, auto-reset
// and observations computed by the step kernel while the bodies are resident.
struct Task {
  bool present = false;
  int torso = 0;
  double forward[3] = {1, 0, 0};
  double survive_reward = 1.0, ctrl_cost = 0.5;
  bool has_healthy = false;
  double z_lo = 0, z_hi = 0;
  int episode_length = 1000;
  bool contact_obs = false;
  double noise_vel = 0.1, noise_ang = 0.1;
  // goal-directed task (grasp / fetch, R36): bring `obj` within `radius` of the
  // frozen, collider-free marker body `target`, which is then placed again
  bool has_goal = false;
  int obj = 0, target = 0;
  double radius = 0, bonus = 0, range[3] = {0, 0, 0};
};

struct Config {
  double dt = 0.01;
  int substeps = 1;
  double gravity[3] = {0, 0, 0};
  double friction = 1.0, elasticity = 0.0, baumgarte = 0.2;
  std::vector<Body> bodies;
  std::vector<Collider> colliders;  // global collider order: body order, then in-body order
  std::vector<Joint> joints;
  std::vector<Actuator> actuators;
  std::vector<Pair> pairs;
  std::vector<Slot> slots;
  int act_dim = 0;
  Task task;
  int n_joint_dofs() const {
    int n = 0;
    for (const Joint& j : joints) n += j.dof;
    return n;
  }
  // z, quat | joint angles | v, ω | joint rates | goal (R36) | per-body contact Δv, Δω (R32)
  int obs_dim() const {
    if (!task.present) return 0;
    return 11 + 2 * n_joint_dofs() + (task.has_goal ? 9 : 0) + (task.contact_obs ? 6 * int(bodies.size()) : 0);
  }
};

// Parse + validate; throws brax::Error.
Config parse_config(const std::string& text);
// Programmatic form (brax_config_from_desc); throws brax::Error.
Config config_from_desc(const brax_config_desc& desc);

// Euler angles in degrees, intrinsic X-Y-Z: qx(a) ⊗ qy(b) ⊗ qz(c).
void euler_deg_to_quat(const double deg[3], double q[4]);

}  // namespace brax

struct brax_config {
  brax::Config cfg;
};
