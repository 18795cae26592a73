// system.cpp — builds the device tables, the warp work plan, default_qp and the
// stability lint for a parsed config (brax_system_create).
#include "system.h"

#include <algorithm>
#include <functional>
#include <tuple>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <sstream>

namespace brax {
// the kernel reads these records with 16-byte vector loads at fixed slots
static_assert(sizeof(DBody) == 64 && sizeof(DJoint) == 144 && sizeof(DSlot) == 176, "record sizes");
static_assert(offsetof(DJoint, o_p) == 32 && offsetof(DJoint, o_c) == 48 && offsetof(DJoint, jp) == 64 &&
                  offsetof(DJoint, jc) == 80 && offsetof(DJoint, lo) == 96 && offsetof(DJoint, hi) == 112 &&
                  offsetof(DJoint, c_a) == 128,
              "DJoint float4 slots");
namespace {

void qmul(const double a[4], const double b[4], double o[4]) {
  double r[4] = {a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                 a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                 a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                 a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]};
  std::memcpy(o, r, sizeof r);
}
void qconj(const double q[4], double o[4]) { o[0] = q[0]; o[1] = -q[1]; o[2] = -q[2]; o[3] = -q[3]; }
void qrot(const double q[4], const double v[3], double o[3]) {
  // v + w·t + u×t, t = 2 u×v
  double t[3] = {2 * (q[2] * v[2] - q[3] * v[1]), 2 * (q[3] * v[0] - q[1] * v[2]), 2 * (q[1] * v[1] - q[2] * v[0])};
  double r[3] = {v[0] + q[0] * t[0] + (q[2] * t[2] - q[3] * t[1]),
                 v[1] + q[0] * t[1] + (q[3] * t[0] - q[1] * t[2]),
                 v[2] + q[0] * t[2] + (q[1] * t[1] - q[2] * t[0])};
  std::memcpy(o, r, sizeof r);
}

template <class T>
int32_t push_struct(std::vector<uint32_t>& blob, const T& v) {
  static_assert(sizeof(T) % 4 == 0, "word struct");
  int32_t off = int32_t(blob.size());
  blob.resize(blob.size() + sizeof(T) / 4);
  std::memcpy(blob.data() + off, &v, sizeof(T));
  return off;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) throw Error(BRAX_E_OUT_OF_MEMORY, std::string(what) + ": out of memory");
  if (e != cudaSuccess) throw Error(BRAX_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

System::~System() {
  forget_system(this);
  if (d_blob) cudaFree(d_blob);
  if (d_default_qp) cudaFree(d_default_qp);
  if (d_masks) cudaFree(d_masks);
  if (d_phase_cycles) cudaFree(d_phase_cycles);
  if (d_gran) cudaFree(d_gran);
}

void default_qp(const Config& cfg, std::vector<double>& pos, std::vector<double>& rot) {
  // Roots at their defaults; children placed joint by joint (config order,
  // repeated until all are placed) so that the joint-frame relative rotation is
  // E(θ⁰), θ⁰_i = clamp(0, lo_i, hi_i), and the two anchors coincide.
  const size_t B = cfg.bodies.size();
  pos.assign(3 * B, 0.0);
  rot.assign(4 * B, 0.0);
  std::vector<char> placed(B, 0), is_child(B, 0);
  for (const Joint& j : cfg.joints) is_child[j.child] = 1;
  for (size_t b = 0; b < B; ++b)
    if (!is_child[b]) {
      std::memcpy(&pos[3 * b], cfg.bodies[b].init_pos, 3 * sizeof(double));
      std::memcpy(&rot[4 * b], cfg.bodies[b].init_rot, 4 * sizeof(double));
      placed[b] = 1;
    }
  for (bool progress = true; progress;) {
    progress = false;
    for (const Joint& j : cfg.joints) {
      if (!placed[j.parent] || placed[j.child]) continue;
      double th[3] = {0, 0, 0};
      for (int i = 0; i < j.dof; ++i) th[i] = std::min(std::max(0.0, j.lo[i]), j.hi[i]) * 180.0 / M_PI;
      double E[4], Jc[4], t1[4], t2[4], t3[4], qc[4];
      euler_deg_to_quat(th, E);
      qconj(j.rotation, Jc);
      const double* qp = &rot[4 * j.parent];
      qmul(qp, j.rotation, t1);
      qmul(t1, E, t2);
      qmul(t2, Jc, t3);
      qmul(t3, j.reference_rotation, qc);
      std::memcpy(&rot[4 * j.child], qc, sizeof qc);
      double rp[3], rc[3];
      qrot(qp, j.parent_offset, rp);
      qrot(qc, j.child_offset, rc);
      for (int k = 0; k < 3; ++k) pos[3 * j.child + k] = pos[3 * j.parent + k] + rp[k] - rc[k];
      placed[j.child] = 1;
      progress = true;
    }
  }
}

System* build_host(const Config& cfg) {
  std::unique_ptr<System> s(new System());
  s->cfg = cfg;
  const int B = int(cfg.bodies.size()), J = int(cfg.joints.size()), C = int(cfg.slots.size());
  const double h = cfg.dt / cfg.substeps;

  // ---- stability lint (R6) ----
  for (int ji = 0; ji < J; ++ji) {
    const Joint& j = cfg.joints[ji];
    double w = 0;
    const double* offs[2] = {j.parent_offset, j.child_offset};
    int bs[2] = {j.parent, j.child};
    for (int k = 0; k < 2; ++k) {
      const Body& b = cfg.bodies[bs[k]];
      if (b.is_static()) continue;
      double imin = std::min(b.inertia[0], std::min(b.inertia[1], b.inertia[2]));
      double o2 = offs[k][0] * offs[k][0] + offs[k][1] * offs[k][1] + offs[k][2] * offs[k][2];
      w += 1.0 / b.mass + o2 / imin;
    }
    std::ostringstream os;
    if (j.stiffness * w * h * h >= 3.6) {
      os << "joints[" << ji << "]: stiffness*w*h^2 = " << j.stiffness * w * h * h << " >= 3.6";
      s->lint.push_back(os.str());
    }
    if (j.spring_damping * w * h >= 1.8) {
      std::ostringstream o2s;
      o2s << "joints[" << ji << "]: spring_damping*w*h = " << j.spring_damping * w * h << " >= 1.8";
      s->lint.push_back(o2s.str());
    }
  }

  // ---- default_qp ----
  std::vector<double> dpos, drot;
  default_qp(cfg, dpos, drot);
  s->dqp_pos.assign(dpos.begin(), dpos.end());
  s->dqp_rot.assign(drot.begin(), drot.end());
  s->dqp_vel.assign(3 * B, 0.f);
  s->dqp_ang.assign(3 * B, 0.f);

  // ---- tables ----
  std::vector<uint32_t>& blob = s->blob;
  DHeader& hd = s->hd;
  hd.B = B;
  hd.J = J;
  hd.C = C;
  hd.A = cfg.act_dim;
  hd.S = cfg.substeps;
  hd.h = float(h);
  hd.beta_over_h = float(cfg.baumgarte / h);
  hd.mu = float(cfg.friction);
  hd.e = float(cfg.elasticity);
  for (int k = 0; k < 3; ++k) hd.g[k] = float(cfg.gravity[k]);
  {
    DTask& t = hd.task;
    const Task& src = cfg.task;
    t.present = src.present ? 1 : 0;
    t.torso = src.torso;
    t.episode_length = src.episode_length;
    t.contact_obs = src.contact_obs ? 1 : 0;
    t.nq = cfg.n_joint_dofs();
    t.obs_dim = cfg.obs_dim();
    t.has_healthy = src.has_healthy ? 1 : 0;
    for (int k = 0; k < 3; ++k) t.fwd[k] = float(src.forward[k]);
    t.dt = float(cfg.dt);
    t.survive = float(src.survive_reward);
    t.ctrl_cost = float(src.ctrl_cost);
    t.z_lo = float(src.z_lo);
    t.z_hi = float(src.z_hi);
    t.noise_vel = float(src.noise_vel);
    t.noise_ang = float(src.noise_ang);
    t.has_goal = src.has_goal ? 1 : 0;
    t.obj = src.has_goal ? src.obj : src.torso;  // the body whose start position the epilogue keeps
    t.target = src.target;
    t.radius = float(src.radius);
    t.bonus = float(src.bonus);
    for (int k = 0; k < 3; ++k) t.range[k] = float(src.range[k]);
  }

  std::vector<DBody> bodies(B);
  std::vector<int> dyn;
  for (int b = 0; b < B; ++b) {
    const Body& src = cfg.bodies[b];
    DBody d{};
    d.inv_mass = float(1.0 / src.mass);
    bool free_pos = true, free_rot = true;
    for (int k = 0; k < 3; ++k) {
      d.inv_inertia[k] = float(1.0 / src.inertia[k]);
      d.mpos[k] = float(1.0 - src.frozen_pos[k]);
      d.mrot[k] = float(1.0 - src.frozen_rot[k]);
      free_pos = free_pos && src.frozen_pos[k] == 0.0;
      free_rot = free_rot && src.frozen_rot[k] == 0.0;
    }
    d.is_static = src.is_static() ? 1 : 0;
    d.rot_frozen = src.rot_frozen() ? 1 : 0;
    bool iso = d.inv_inertia[0] == d.inv_inertia[1] && d.inv_inertia[1] == d.inv_inertia[2];
    d.flags = (iso ? kFlagIso : 0) | (free_pos ? kFlagFreePos : 0) | (free_rot ? kFlagFreeRot : 0);
    bodies[b] = d;
    if (!d.is_static) dyn.push_back(b);
  }
  s->n_dynamic = int(dyn.size());
  auto align4 = [&] { while (blob.size() % 4) blob.push_back(0); };
  hd.off_bodies = int32_t(blob.size());
  for (const DBody& d : bodies) push_struct(blob, d);

  auto zero3 = [](const float* p) { return p[0] == 0.f && p[1] == 0.f && p[2] == 0.f; };
  auto ident = [](const float* q) { return q[0] == 1.f && q[1] == 0.f && q[2] == 0.f && q[3] == 0.f; };
  hd.off_joints = int32_t(blob.size());
  int obs_off = 0;
  for (const Joint& j : cfg.joints) {
    DJoint d{};
    d.obs_off = obs_off;
    obs_off += j.dof;
    d.parent = j.parent;
    d.child = j.child;
    d.dof = j.dof;
    d.act_kind = j.act_kind;
    d.act_offset = j.act_offset;
    double jc[4], rc[4];
    qconj(j.reference_rotation, rc);
    qmul(rc, j.rotation, jc);
    for (int k = 0; k < 3; ++k) {
      d.o_p[k] = float(j.parent_offset[k]);
      d.o_c[k] = float(j.child_offset[k]);
      d.lo[k] = float(j.lo[k]);
      d.hi[k] = float(j.hi[k]);
    }
    for (int k = 0; k < 4; ++k) {
      d.jp[k] = float(j.rotation[k]);
      d.jc[k] = float(jc[k]);
    }
    d.k = float(j.stiffness);
    d.c_l = float(j.spring_damping);
    d.c_a = float(j.angular_damping);
    d.k_l = float(j.limit_stiffness);
    d.k_a = float(j.angular_stiffness);
    d.strength = float(j.act_strength);
    d.flags = (zero3(d.o_p) ? kJZeroOp : 0) | (zero3(d.o_c) ? kJZeroOc : 0) | (ident(d.jp) ? kJIdentP : 0) |
              (ident(d.jc) ? kJIdentC : 0) | (d.c_l == 0.f ? kJNoCl : 0) | (d.c_a == 0.f ? kJNoCa : 0);
    push_struct(blob, d);
  }

  hd.off_slots = int32_t(blob.size());
  for (const Slot& sl : cfg.slots) {
    DSlot d{};
    const Collider& A = cfg.colliders[sl.col_a];
    const Collider& Bc = cfg.colliders[sl.col_b];
    d.type = sl.type;
    d.a = sl.a;
    d.b = sl.b;
    d.point = sl.point;
    d.a_static = bodies[sl.a].is_static;
    d.b_static = bodies[sl.b].is_static;
    for (int k = 0; k < 3; ++k) {
      d.ca_pos[k] = float(A.pos[k]);
      d.cb_pos[k] = float(Bc.pos[k]);
      d.inv_inertia_a[k] = bodies[sl.a].inv_inertia[k];
      d.inv_inertia_b[k] = bodies[sl.b].inv_inertia[k];
    }
    if (sl.type == BRAX_SLOT_BOX_PLANE) {
      const int sg[3] = {(sl.point & 1) ? 1 : -1, (sl.point & 2) ? 1 : -1, (sl.point & 4) ? 1 : -1};
      for (int k = 0; k < 3; ++k) d.corner[k] = float(sg[k] * A.halfsize[k]);
    }
    for (int k = 0; k < 4; ++k) {
      d.ca_rot[k] = float(A.rot[k]);
      d.cb_rot[k] = float(Bc.rot[k]);
    }
    d.ra = float(A.radius);
    d.rb = float(Bc.radius);
    float ell_a = float(0.5 * A.length - A.radius);
    d.ell_a = (sl.type == BRAX_SLOT_CAPSULE_PLANE && sl.point == 1) ? -ell_a : ell_a;
    d.ellb = float(0.5 * Bc.length - Bc.radius);
    d.inv_mass_a = bodies[sl.a].inv_mass;
    d.inv_mass_b = bodies[sl.b].inv_mass;
    d.flags = (zero3(d.ca_pos) ? kSZeroPa : 0) | (zero3(d.cb_pos) ? kSZeroPb : 0) | (ident(d.ca_rot) ? kSIdentA : 0) |
              (ident(d.cb_rot) ? kSIdentB : 0) | ((bodies[sl.a].flags & kFlagIso) ? kSIsoA : 0) |
              ((bodies[sl.b].flags & kFlagIso) ? kSIsoB : 0);
    if (sl.type <= BRAX_SLOT_BOX_PLANE) {  // pa_local = ca_pos + rotate(ca_rot, v), in double
      double v[3] = {0, 0, 0};
      if (sl.type == BRAX_SLOT_CAPSULE_PLANE) v[2] = (sl.point == 1 ? -1.0 : 1.0) * (0.5 * A.length - A.radius);
      if (sl.type == BRAX_SLOT_BOX_PLANE) {
        const int sg[3] = {(sl.point & 1) ? 1 : -1, (sl.point & 2) ? 1 : -1, (sl.point & 4) ? 1 : -1};
        for (int k = 0; k < 3; ++k) v[k] = sg[k] * A.halfsize[k];
      }
      const double* q = A.rot;  // rotate(q, v) = v + w·t + u×t, t = 2 u×v
      const double t[3] = {2 * (q[2] * v[2] - q[3] * v[1]), 2 * (q[3] * v[0] - q[1] * v[2]),
                           2 * (q[1] * v[1] - q[2] * v[0])};
      const double r[3] = {v[0] + q[0] * t[0] + (q[2] * t[2] - q[3] * t[1]),
                           v[1] + q[0] * t[1] + (q[3] * t[0] - q[1] * t[2]),
                           v[2] + q[0] * t[2] + (q[1] * t[1] - q[2] * t[0])};
      for (int k = 0; k < 3; ++k) d.pa_local[k] = float(A.pos[k] + r[k]);
      if (zero3(d.pa_local)) d.flags |= kSZeroLa;
    }
    push_struct(blob, d);
  }

  align4();
  // ---- work plans: for G lane groups per warp (E = 32/G envs per block) ----
  // Items of one code class (joints with equal dof / actuator kind / flags;
  // contacts with equal type / flags / static sides) are packed G to a step so
  // a warp's groups never diverge on item kind; steps go to warps by
  // longest-processing-time-first over estimated costs (joint ≈ 5, contact ≈ 3).
  const DJoint* djoints = reinterpret_cast<const DJoint*>(blob.data() + hd.off_joints);
  const DSlot* dslots = reinterpret_cast<const DSlot*>(blob.data() + hd.off_slots);
  std::vector<std::vector<int>> classes;
  {
    std::vector<std::vector<int>> keys;
    auto add = [&](const std::vector<int>& key, int item) {
      for (size_t k = 0; k < keys.size(); ++k)
        if (keys[k] == key) { classes[k].push_back(item); return; }
      keys.push_back(key);
      classes.push_back({item});
    };
    for (int j = 0; j < J; ++j) add({0, djoints[j].dof, djoints[j].act_kind, djoints[j].flags}, j);
    for (int c = 0; c < C; ++c)
      add({1, dslots[c].type, dslots[c].flags, dslots[c].a_static, dslots[c].b_static}, J + c);
  }
  // dynamic bodies ordered by shape: (#joints, #contact slots incident, integrator flags)
  std::vector<int> dyn_shaped = dyn;
  std::function<std::tuple<int, int, int, int>(int)> body_key;
  {
    std::vector<int> nj(B, 0), nc(B, 0);
    for (const Joint& j : cfg.joints) {
      ++nj[j.parent];
      ++nj[j.child];
    }
    for (const Slot& sl : cfg.slots) {
      ++nc[sl.a];
      ++nc[sl.b];
    }
    body_key = [nj, nc, &bodies](int b) {
      return std::make_tuple(nj[b], nc[b], bodies[b].flags, bodies[b].rot_frozen);
    };
    std::stable_sort(dyn_shaped.begin(), dyn_shaped.end(), [&](int a, int b) { return body_key(a) < body_key(b); });
  }
  const int env_w = [] {
    const char* e = std::getenv("BRAX_WARPS_PER_BLOCK");
    int v = e ? std::atoi(e) : 0;
    return (v >= 1 && v <= kMaxWarps) ? v : 0;
  }();
  for (int pi = 0; pi < kNumPlans; ++pi) {
    DPlan& P = hd.plan[pi];
    const int G = 1 << (pi % 3), V = 1 + pi / 3, E = 32 * V / G;
    P.G = G;
    P.V = V;
    P.E = E;
    std::vector<std::vector<int>> steps;  // each: G items (-1 idle)
    std::vector<int> step_cost;
    for (const auto& cl : classes)
      for (size_t k = 0; k < cl.size(); k += G) {
        std::vector<int> st(G, -1);
        for (int g = 0; g < G && k + g < cl.size(); ++g) st[g] = cl[k + g];
        steps.push_back(st);
        step_cost.push_back(cl[k] < J ? 5 : 3);
      }
    // body steps: G bodies of one shape class each (idle slots pad a class to G)
    std::vector<std::vector<int>> bsteps;
    for (size_t k = 0; k < dyn_shaped.size();) {
      std::vector<int> st(G, -1);
      const auto cls = body_key(dyn_shaped[k]);
      for (int g = 0; g < G && k < dyn_shaped.size() && body_key(dyn_shaped[k]) == cls; ++g) st[g] = dyn_shaped[k++];
      bsteps.push_back(st);
    }
    const int n_body_steps = int(bsteps.size());
    // G = 1 (large batches, throughput-bound): ~2 item steps per warp; G > 1 (small
    // batches, latency-bound): one item step per warp (measured, profiles/)
    int W = G == 1 ? std::max(1, std::max(n_body_steps, (int(steps.size()) + 1) / 2))
                   : std::max(1, std::max(n_body_steps, int(steps.size())));
    W = std::min(W, kMaxWarps);
    if (env_w) W = env_w;
    P.W = W;
    std::vector<int> order(steps.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return step_cost[a] > step_cost[b]; });
    std::vector<std::vector<int>> per_warp(W);
    std::vector<int> load(W, 0);
    for (int k : order) {
      int w = int(std::min_element(load.begin(), load.end()) - load.begin());
      per_warp[w].push_back(k);
      load[w] += step_cost[k];
    }
    align4();
    P.off_item_begin = int32_t(blob.size());
    int acc = 0;
    for (int w = 0; w <= W; ++w) {
      blob.push_back(uint32_t(acc));
      if (w < W) acc += int(per_warp[w].size());
    }
    P.off_items = int32_t(blob.size());
    for (int w = 0; w < W; ++w) {
      std::sort(per_warp[w].begin(), per_warp[w].end());
      for (int k : per_warp[w])
        for (int g = 0; g < G; ++g) blob.push_back(uint32_t(steps[k][g]));
    }
    // dynamic bodies, G per step (bodies with the same gather / integrator shape share a
    // step, so a warp's lane groups do not diverge), steps round-robin over warps
    std::vector<std::vector<int>> wb(W);
    for (int k = 0; k < n_body_steps; ++k) wb[k % W].push_back(k);
    P.off_body_begin = int32_t(blob.size());
    acc = 0;
    for (int w = 0; w <= W; ++w) {
      blob.push_back(uint32_t(acc));
      if (w < W) acc += int(wb[w].size());
    }
    {
      size_t max_items = 0, max_bodies = 0;
      for (int w = 0; w < W; ++w) {
        max_items = std::max(max_items, per_warp[w].size());
        max_bodies = std::max(max_bodies, wb[w].size());
      }
      s->lean_items[pi] = max_bodies <= 1 && max_items <= 2 ? std::max<int>(1, int(max_items)) : 0;
    }
    P.off_bodies_of_warp = int32_t(blob.size());
    for (int w = 0; w < W; ++w)
      for (int k : wb[w])
        for (int g = 0; g < G; ++g) blob.push_back(uint32_t(bsteps[k][g]));
  }
  // incidence lists: joints by index (child / parent side), then slots by index (A / B side)
  std::vector<std::vector<int32_t>> jinc(B), cinc(B);
  for (int j = 0; j < J; ++j) {
    jinc[cfg.joints[j].child].push_back(inc_pack(j, false));
    jinc[cfg.joints[j].parent].push_back(inc_pack(j, true));
  }
  for (int c = 0; c < C; ++c) {
    cinc[cfg.slots[c].a].push_back(inc_pack(c, false));
    cinc[cfg.slots[c].b].push_back(inc_pack(c, true));
  }
  auto put_lists = [&](const std::vector<std::vector<int32_t>>& lists, int32_t* off_begin, int32_t* off_list) {
    *off_begin = int32_t(blob.size());
    int acc = 0;
    for (int b = 0; b <= B; ++b) {
      blob.push_back(uint32_t(acc));
      if (b < B) acc += int(lists[b].size());
    }
    *off_list = int32_t(blob.size());
    for (int b = 0; b < B; ++b)
      for (int32_t e : lists[b]) blob.push_back(uint32_t(e));
  };
  put_lists(jinc, &hd.off_jinc_begin, &hd.off_jinc);
  put_lists(cinc, &hd.off_cinc_begin, &hd.off_cinc);
  while (blob.size() % 4) blob.push_back(0);
  hd.blob_words = int32_t(blob.size());
  auto magic = [](uint32_t d) -> uint32_t { return d ? uint32_t(((uint64_t(1) << 32) + d - 1) / d) : 0; };
  hd.row_magic[0] = magic(uint32_t(3 * B));
  hd.row_magic[1] = magic(uint32_t(4 * B));
  hd.row_magic[2] = cfg.act_dim > 1 ? magic(uint32_t(cfg.act_dim)) : 0;  // A == 1 is special-cased
  hd.row_magic[3] = 0;

  for (int pi = 0; pi < kNumPlans; ++pi) {
    DPlan& P = hd.plan[pi];
    const int LG = P.E / P.V;
    P.smem_bytes = smem_layout(B, J, C, hd.A, P.E, LG, P.V == 2, hd.blob_words, 0, 0).total_words * 4;
    P.smem_bytes_env = smem_layout(B, J, C, hd.A, P.E, LG, P.V == 2, hd.blob_words, hd.task.obs_dim,
                                   hd.task.contact_obs).total_words * 4;
    P.smem_bytes_cdp = smem_layout(B, J, C, hd.A, P.E, LG, P.V == 2, hd.blob_words, 0, 0, 1).total_words * 4;
    P.smem_bytes_jvp = P.V == 1 ? smem_layout(B, J, C, hd.A, P.E, LG, 1, hd.blob_words, 0, 0).total_words * 4 : 0;
  }
  // smallest block (G = 4: 8 envs) must fit; larger blocks are used where they fit
  s->smem_bytes = size_t(hd.plan[0].smem_bytes);
  int smallest = hd.plan[0].smem_bytes;
  for (int pi = 0; pi < kNumPlans; ++pi) smallest = std::min(smallest, hd.plan[pi].smem_bytes);
  if (size_t(smallest) > kMaxDynSmem)
    throw Error(BRAX_E_VALIDATION, "config: system too large for one block's shared memory (" +
                                       std::to_string(smallest) + " bytes with 8 envs per block)");

  return s.release();
}

System* build_system(const Config& cfg, int device) {
  std::unique_ptr<System> s(build_host(cfg));
  s->device = device;
  std::vector<uint32_t>& blob = s->blob;
  const int B = s->hd.B;
  std::vector<DBody> bodies(B);
  std::memcpy(bodies.data(), blob.data() + s->hd.off_bodies, sizeof(DBody) * B);
  // ---- upload ----
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  {  // stream-ordered scratch (autotuner, reverse-mode checkpoints): keep freed blocks in the
     // device's default pool instead of returning them to the driver at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  cuda_check(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
  cuda_check(cudaMalloc(&s->d_blob, blob.size() * 4), "cudaMalloc(blob)");
  cuda_check(cudaMemcpy(s->d_blob, blob.data(), blob.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy(blob)");
  std::vector<float> dq(7 * size_t(B));
  for (int b = 0; b < B; ++b) {
    for (int k = 0; k < 3; ++k) dq[3 * b + k] = s->dqp_pos[3 * b + k];
    for (int k = 0; k < 4; ++k) dq[3 * B + 4 * b + k] = s->dqp_rot[4 * b + k];
  }
  cuda_check(cudaMalloc(&s->d_default_qp, dq.size() * 4), "cudaMalloc(default_qp)");
  cuda_check(cudaMemcpy(s->d_default_qp, dq.data(), dq.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
  s->d_masks_host.assign(7 * size_t(B), 0.f);
  for (int b = 0; b < B; ++b) {
    for (int k = 0; k < 3; ++k) {
      s->d_masks_host[7 * b + k] = bodies[b].mpos[k];
      s->d_masks_host[7 * b + 3 + k] = bodies[b].mrot[k];
    }
    s->d_masks_host[7 * b + 6] = float(bodies[b].is_static);
  }
  cuda_check(cudaMalloc(&s->d_phase_cycles, 4 * sizeof(unsigned long long)), "cudaMalloc(phase_cycles)");
  cuda_check(cudaMemset(s->d_phase_cycles, 0, 4 * sizeof(unsigned long long)), "cudaMemset");
  cuda_check(cudaMalloc(&s->d_gran, 2 * size_t(kMaxGranules) * 4), "cudaMalloc(granule counters)");
  cuda_check(cudaMemset(s->d_gran, 0, 2 * size_t(kMaxGranules) * 4), "cudaMemset(granule counters)");
  cuda_check(cudaMalloc(&s->d_masks, s->d_masks_host.size() * 4), "cudaMalloc(masks)");
  cuda_check(cudaMemcpy(s->d_masks, s->d_masks_host.data(), s->d_masks_host.size() * 4, cudaMemcpyHostToDevice),
             "cudaMemcpy(masks)");
  return s.release();
}

}  // namespace brax
