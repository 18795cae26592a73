// brax_oracle.cpp — plain fp64 CPU oracle of the Brax physics step.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code, header or table generator with the CUDA path
// (paper_2106_13281_b200/csrc); neither includes the other.
//
// What it computes: Alg. 1 of the paper (§3) — per substep
//   qp = kinematic_integrator.apply(qp, dt)
//   dp_j += joint.apply(qp); dp_a += actuator.apply(qp, action)
//   dp_c += collider.apply(qp)
//   qp = potential_integrator.apply(qp, dp_j + dp_a, dt)
//   qp = collision_integrator.apply(qp, dp_c)
// with every formula taken from SURVEY.md §8(c).1 and the readings R1-R29
// listed in DESIGN.md ("readings").  Scalar, one env at a time, one body /
// joint / slot at a time, in the paper's order; no blocking, fusion or
// reordering.  The scalar type is a template parameter so that the same code
// also runs with an op-counting type (SURVEY §8(d) counting convention:
// add/sub/mul = 1 flop, div/sqrt = 4 flops + 1 MUFU, atan2/asin/sin/cos = 20
// flops + 1 MUFU; comparisons, min/max and clamps are not counted).
//
// Parity pins: tests/test_oracle_pins.py (closed forms, invariants, brute force).
// Parity unpinned beyond invariants: whole-scene trajectories (ant, humanoid,
// halfcheetah, grasp, fetch) — no closed form exists.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// ----------------------------------------------------------------------------
// op-counting scalar
// ----------------------------------------------------------------------------
thread_local uint64_t g_flops = 0, g_mufu = 0;
// "lean" counting (second convention, reported beside the first): operations whose
// operand is an exactly neutral value fixed by the scene — a unit mask (no frozen
// axis), an isotropic inertia (I_w⁻¹ = 1/I, no rotation), a zero damping coefficient,
// a zero collider offset, an identity collider rotation — are not counted.  The
// values computed are identical; only the tally differs.
thread_local bool g_lean = false;
thread_local int g_mute = 0;  // > 0: inside a neutral operation in lean mode

struct Cnt {
  double v;
  Cnt() : v(0) {}
  Cnt(double x) : v(x) {}  // NOLINT: implicit from constants
};
inline void tally(uint64_t f, uint64_t m) {
  if (g_mute == 0) { g_flops += f; g_mufu += m; }
}
inline Cnt operator+(Cnt a, Cnt b) { tally(1, 0); return Cnt(a.v + b.v); }
inline Cnt operator-(Cnt a, Cnt b) { tally(1, 0); return Cnt(a.v - b.v); }
inline Cnt operator*(Cnt a, Cnt b) { tally(1, 0); return Cnt(a.v * b.v); }
inline Cnt operator/(Cnt a, Cnt b) { tally(4, 1); return Cnt(a.v / b.v); }
// Scope of an operation that is neutral for this scene: uncounted in lean mode (no
// effect on fp64 / fp32 runs, or on the default counting convention).
struct Neutral {
  bool on;
  explicit Neutral(bool neutral) : on(neutral && g_lean) { if (on) ++g_mute; }
  ~Neutral() { if (on) --g_mute; }
};
inline Cnt operator-(Cnt a) { return Cnt(-a.v); }
inline bool operator<(Cnt a, Cnt b) { return a.v < b.v; }
inline bool operator>(Cnt a, Cnt b) { return a.v > b.v; }
inline bool operator<=(Cnt a, Cnt b) { return a.v <= b.v; }
inline bool operator>=(Cnt a, Cnt b) { return a.v >= b.v; }
inline bool operator==(Cnt a, Cnt b) { return a.v == b.v; }
inline Cnt& operator+=(Cnt& a, Cnt b) { a = a + b; return a; }
inline Cnt& operator-=(Cnt& a, Cnt b) { a = a - b; return a; }

inline double val(double x) { return x; }
inline double val(Cnt x) { return x.v; }
inline double xsqrt(double x) { return std::sqrt(x); }
inline Cnt xsqrt(Cnt x) { tally(4, 1); return Cnt(std::sqrt(x.v)); }
inline double xatan2(double y, double x) { return std::atan2(y, x); }
inline Cnt xatan2(Cnt y, Cnt x) { tally(20, 1); return Cnt(std::atan2(y.v, x.v)); }
inline double xasin(double x) { return std::asin(x); }
inline double xsin(double x) { return std::sin(x); }
inline double xcos(double x) { return std::cos(x); }
inline Cnt xsin(Cnt x) { tally(20, 1); return Cnt(std::sin(x.v)); }
inline Cnt xcos(Cnt x) { tally(20, 1); return Cnt(std::cos(x.v)); }
inline Cnt xasin(Cnt x) { tally(20, 1); return Cnt(std::asin(x.v)); }
// fp32 instantiation (diagnostic only: measures the fp32 rounding floor of the
// same algorithm; never used as a parity reference)
inline double val(float x) { return x; }
inline float xsqrt(float x) { return std::sqrt(x); }
inline float xatan2(float y, float x) { return std::atan2(y, x); }
inline float xasin(float x) { return std::asin(x); }
inline float xsin(float x) { return std::sin(x); }
inline float xcos(float x) { return std::cos(x); }
template <class T> inline T xmax(T a, T b) { return (a < b) ? b : a; }
template <class T> inline T xmin(T a, T b) { return (b < a) ? b : a; }
template <class T> inline T xclamp(T x, T lo, T hi) { return xmin(xmax(x, lo), hi); }

// ----------------------------------------------------------------------------
// vectors and quaternions (w, x, y, z), Hamilton product — SURVEY §8(c).1
// ----------------------------------------------------------------------------
template <class T> struct V3 { T x, y, z; };
template <class T> struct Q4 { T w, x, y, z; };

template <class T> inline V3<T> v3(T x, T y, T z) { return V3<T>{x, y, z}; }
template <class T> inline V3<T> operator+(V3<T> a, V3<T> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class T> inline V3<T> operator-(V3<T> a, V3<T> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class T> inline V3<T> operator*(T s, V3<T> a) { return {s * a.x, s * a.y, s * a.z}; }
template <class T> inline V3<T> hadamard(V3<T> a, V3<T> b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
template <class T> inline V3<T> divide(V3<T> a, V3<T> b) { return {a.x / b.x, a.y / b.y, a.z / b.z}; }
template <class T> inline T dot(V3<T> a, V3<T> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class T> inline V3<T> cross(V3<T> a, V3<T> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class T> inline Q4<T> qmul(Q4<T> a, Q4<T> b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
          a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
          a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
template <class T> inline Q4<T> qconj(Q4<T> q) { return {q.w, -q.x, -q.y, -q.z}; }
// rotate(q, v) = v + w·t + u×t,  u = (x,y,z),  t = 2u×v
template <class T> inline V3<T> rotate(Q4<T> q, V3<T> v) {
  V3<T> u{q.x, q.y, q.z};
  V3<T> t = T(2.0) * cross(u, v);
  return v + q.w * t + cross(u, t);
}
template <class T> inline V3<T> inv_rotate(Q4<T> q, V3<T> v) { return rotate(qconj(q), v); }
// I_w⁻¹(q)·v = rotate(q, inv_rotate(q, v) ⊘ I_b)   (R4: world inverse inertia)
template <class T> inline V3<T> inv_inertia_world(Q4<T> q, V3<T> inertia, V3<T> v) {
  return rotate(q, divide(inv_rotate(q, v), inertia));
}
// lean count of an isotropic I_w⁻¹·v: three products v·(1/I) (1/I a scene constant)
template <class T> inline void lean_iso_count(V3<T> inertia) {
  if (g_lean && val(inertia.x) == val(inertia.y) && val(inertia.y) == val(inertia.z)) tally(3, 0);
}
template <class T> inline bool iso(V3<T> inertia) {
  return val(inertia.x) == val(inertia.y) && val(inertia.y) == val(inertia.z);
}
inline bool ones3(const double* m) { return m[0] == 1.0 && m[1] == 1.0 && m[2] == 1.0; }
inline bool zero3(const double* m) { return m[0] == 0.0 && m[1] == 0.0 && m[2] == 0.0; }
inline bool ident4(const double* q) { return q[0] == 1.0 && q[1] == 0.0 && q[2] == 0.0 && q[3] == 0.0; }
// mask ⊙ v, neutral (lean count) when no axis is frozen
template <class T> inline V3<T> mhad(const double* m, V3<T> v) {
  Neutral n(ones3(m));
  return hadamard(V3<T>{T(m[0]), T(m[1]), T(m[2])}, v);
}
// I_w⁻¹·v counted leanly: an isotropic body's rotate / divide / rotate is three products
template <class T> inline V3<T> iiw(Q4<T> q, V3<T> inertia, V3<T> v) {
  V3<T> r;
  {
    Neutral n(iso(inertia));
    r = inv_inertia_world(q, inertia, v);
  }
  lean_iso_count(inertia);
  return r;
}

// ----------------------------------------------------------------------------
// system description (mirrored by ctypes in oracle/__init__.py)
// ----------------------------------------------------------------------------
}  // namespace

extern "C" {
struct OBody {
  double mass, inertia[3], mpos[3], mrot[3];  // mpos/mrot = 1 − frozen (App. A `frozen`)
  int32_t is_static, rot_frozen;              // all 6 axes frozen; all 3 rotation axes frozen
};
struct OJoint {
  int32_t parent, child, dof, act_kind;  // act_kind: -1 none, 0 TORQUE, 1 ANGLE
  int32_t act_offset, pad_;
  double o_p[3], o_c[3], jp[4], jc[4];   // offsets; joint frames J_p = rotation, J_c = conj(Rf)⊗rotation
  double k, c_l, c_a, k_l, k_a;          // stiffness, spring/angular damping, limit/alignment stiffness
  double lo[3], hi[3], act_strength;     // limits (rad), actuator strength
};
struct OCollider {
  int32_t body, kind, end, pad_;         // kind: 0 sphere 1 capsule 2 box 3 plane
  double pos[3], rot[4], radius, length, halfsize[3];
};
struct OSlot { int32_t pair, type, a, b, col_a, col_b, point, pad_; };
struct OSys {
  int32_t nb, nj, ncol, ns, act_dim, substeps;
  double dt, gravity[3], mu, e, beta;
  const OBody* bodies;
  const OJoint* joints;
  const OCollider* colliders;
  const OSlot* slots;
};
struct OOpts {
  int32_t combine_sum, pad_;   // 1 = literal sum of contact impulses (test switch, R14); 0 = mean
  double amb_d, amb_jn, amb_par, amb_angle;  // R23 ambiguity thresholds
};
}

namespace {

enum { SPHERE_PLANE = 0, CAPSULE_PLANE, BOX_PLANE, SPHERE_SPHERE, SPHERE_CAPSULE, CAPSULE_CAPSULE };

template <class T> inline V3<T> V(const double* a) { return V3<T>{T(a[0]), T(a[1]), T(a[2])}; }
template <class T> inline Q4<T> Q(const double* a) { return Q4<T>{T(a[0]), T(a[1]), T(a[2]), T(a[3])}; }

template <class T> struct BodyState { V3<T> x; Q4<T> q; V3<T> v; V3<T> w; };

// Closest points between segments P1Q1 and P2Q2 (Ericson, Real-Time Collision
// Detection §5.1.9 ClosestPtSegmentSegment), including its degenerate and
// parallel cases.  Returns the two points.
template <class T>
void closest_segment_segment(V3<T> p1, V3<T> q1, V3<T> p2, V3<T> q2, V3<T>* c1, V3<T>* c2) {
  V3<T> d1 = q1 - p1, d2 = q2 - p2, r = p1 - p2;
  T a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r);
  T s(0.0), t(0.0);
  if (a <= T(0.0) && e <= T(0.0)) {
    s = T(0.0); t = T(0.0);
  } else if (a <= T(0.0)) {
    s = T(0.0); t = xclamp(f / e, T(0.0), T(1.0));
  } else {
    T c = dot(d1, r);
    if (e <= T(0.0)) {
      t = T(0.0); s = xclamp(-c / a, T(0.0), T(1.0));
    } else {
      T b = dot(d1, d2);
      T denom = a * e - b * b;
      s = (denom == T(0.0)) ? T(0.0) : xclamp((b * f - c * e) / denom, T(0.0), T(1.0));
      t = (b * s + f) / e;
      if (t < T(0.0)) {
        t = T(0.0); s = xclamp(-c / a, T(0.0), T(1.0));
      } else if (t > T(1.0)) {
        t = T(1.0); s = xclamp((b - c) / a, T(0.0), T(1.0));
      }
    }
  }
  *c1 = p1 + s * d1;
  *c2 = p2 + t * d2;
}

// Narrowphase of one contact slot: returns the normal n
// (from B into A), the contact point pt and the penetration d (> 0 penetrating).
// Sets *near_parallel for capsule–capsule pairs with |â×b̂|² < amb_par (R23).
template <class T>
void narrowphase(const OSys& S, const OSlot& sl, const BodyState<T>* st, double amb_par, V3<T>* n_out,
                 V3<T>* pt_out, T* d_out, bool* near_parallel) {
  const OCollider& CA = S.colliders[sl.col_a];
  const OCollider& CB = S.colliders[sl.col_b];
  const BodyState<T>& A = st[sl.a];
  const BodyState<T>& Bs = st[sl.b];
  V3<T> cA, cB;
  Q4<T> qA, qB;
  { Neutral n(zero3(CA.pos)); cA = A.x + rotate(A.q, V<T>(CA.pos)); }
  { Neutral n(zero3(CB.pos)); cB = Bs.x + rotate(Bs.q, V<T>(CB.pos)); }
  { Neutral n(ident4(CA.rot)); qA = qmul(A.q, Q<T>(CA.rot)); }
  { Neutral n(ident4(CB.rot)); qB = qmul(Bs.q, Q<T>(CB.rot)); }
  const V3<T> zhat = v3(T(0.0), T(0.0), T(1.0));
  V3<T> n, pt;
  T d;
  if (sl.type == SPHERE_PLANE || sl.type == CAPSULE_PLANE || sl.type == BOX_PLANE) {
    n = rotate(qB, zhat);
    V3<T> p0 = cB;
    if (sl.type == BOX_PLANE) {
      V3<T> hs = V<T>(CA.halfsize);
      V3<T> sgn = v3(T((sl.point & 1) ? 1.0 : -1.0), T((sl.point & 2) ? 1.0 : -1.0),
                     T((sl.point & 4) ? 1.0 : -1.0));
      V3<T> corner = cA + rotate(qA, hadamard(sgn, hs));
      d = -dot(corner - p0, n);
      pt = corner;
    } else {
      V3<T> c = cA;
      if (sl.type == CAPSULE_PLANE) {
        V3<T> ax = rotate(qA, zhat);
        T ell = T(0.5) * T(CA.length) - T(CA.radius);
        c = (sl.point == 0) ? cA + ell * ax : cA - ell * ax;
      }
      T r = T(CA.radius);
      d = r - dot(c - p0, n);
      pt = c - r * n;
    }
  } else {
    V3<T> pa = cA, pb = cB;
    T rA = T(CA.radius), rB = T(CB.radius);
    if (sl.type == SPHERE_CAPSULE) {
      V3<T> axB = rotate(qB, zhat);
      T ellB = T(0.5) * T(CB.length) - T(CB.radius);
      V3<T> e0 = cB + ellB * axB, e1 = cB - ellB * axB;
      V3<T> seg = e0 - e1;
      T L2 = dot(seg, seg);
      T t = (L2 > T(0.0)) ? xclamp(dot(cA - e1, seg) / L2, T(0.0), T(1.0)) : T(0.0);
      pb = e1 + t * seg;
    } else if (sl.type == CAPSULE_CAPSULE) {
      V3<T> axA = rotate(qA, zhat), axB = rotate(qB, zhat);
      T ellA = T(0.5) * T(CA.length) - T(CA.radius);
      T ellB = T(0.5) * T(CB.length) - T(CB.radius);
      closest_segment_segment(cA + ellA * axA, cA - ellA * axA, cB + ellB * axB, cB - ellB * axB, &pa, &pb);
      V3<T> cr = cross(axA, axB);
      if (val(dot(cr, cr)) < amb_par) *near_parallel = true;  // R23 near-parallel
    }
    V3<T> delta = pa - pb;
    T dist = xsqrt(dot(delta, delta));
    n = (dist > T(0.0)) ? (T(1.0) / dist) * delta : zhat;   // R16
    d = rA + rB - dist;
    pt = T(0.5) * ((pa - rA * n) + (pb + rB * n));
  }
  *n_out = n;
  *pt_out = pt;
  *d_out = d;
}

template <class T>
struct EnvOut {
  uint8_t* active;
  bool ambiguous;
  double* contact_dv;  // [B][6] or NULL: the collision integrator's Δv, Δω of this substep (NEXT-1 obs)
  double* contact_dp;  // [B][6] or NULL: the same summed over the step's substeps (brax_step_extras.contact_dp)
};

// One substep of Alg. 1 on one env.  `st` holds all B bodies.
template <class T>
void substep(const OSys& S, const OOpts& opt, BodyState<T>* st, const double* action, EnvOut<T>* out) {
  const int B = S.nb;
  const T h = T(S.dt / S.substeps);

  // ---- 1. kinematic integrator (R3) ----------------------------
  for (int b = 0; b < B; ++b) {
    const OBody& bd = S.bodies[b];
    if (bd.is_static) continue;  // R21: fully frozen body is bitwise unchanged
    BodyState<T>& s = st[b];
    s.x = s.x + h * mhad(bd.mpos, s.v);
    if (!bd.rot_frozen) {
      V3<T> wm = mhad(bd.mrot, s.w);
      Q4<T> dq = qmul(Q4<T>{T(0.0), wm.x, wm.y, wm.z}, s.q);
      T hh = T(0.5) * h;
      Q4<T> q{s.q.w + hh * dq.w, s.q.x + hh * dq.x, s.q.y + hh * dq.y, s.q.z + hh * dq.z};
      T n = xsqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
      s.q = Q4<T>{q.w / n, q.x / n, q.y / n, q.z / n};
    }
  }

  std::vector<V3<T>> F(B, v3(T(0.0), T(0.0), T(0.0))), Tq(B, v3(T(0.0), T(0.0), T(0.0)));
  std::vector<V3<T>> dV(B, v3(T(0.0), T(0.0), T(0.0))), dW(B, v3(T(0.0), T(0.0), T(0.0)));
  std::vector<int> cnt(B, 0);

  // ---- 2./3. joints with their actuators (R5, R7-R12) --
  for (int j = 0; j < S.nj; ++j) {
    const OJoint& J = S.joints[j];
    const BodyState<T>& P = st[J.parent];
    const BodyState<T>& C = st[J.child];
    V3<T> rp = rotate(P.q, V<T>(J.o_p));
    V3<T> rc = rotate(C.q, V<T>(J.o_c));
    V3<T> dx = (P.x - C.x) + (rp - rc);                                  // evaluated in this order
    const bool no_cl = J.c_l == 0.0, no_ca = J.c_a == 0.0;             // lean count: neutral damping terms
    V3<T> dv, cdv, f;
    {
      Neutral n(no_cl);
      dv = (P.v + cross(P.w, rp)) - (C.v + cross(C.w, rc));
      cdv = T(J.c_l) * dv;
    }
    const V3<T> kdx = T(J.k) * dx;
    { Neutral n(no_cl); f = kdx + cdv; }                               // F = k·Δx + c_l·Δv, force on child
    Q4<T> fp = qmul(P.q, Q<T>(J.jp));
    Q4<T> fc = qmul(C.q, Q<T>(J.jc));
    Q4<T> qr = qmul(qconj(fp), fc);
    if (qr.w < T(0.0)) qr = Q4<T>{-qr.w, -qr.x, -qr.y, -qr.z};
    // intrinsic X-Y-Z Euler angles of R(q_r)
    T R02 = T(2.0) * (qr.x * qr.z + qr.w * qr.y);
    T R12 = T(2.0) * (qr.y * qr.z - qr.w * qr.x);
    T R22 = T(1.0) - T(2.0) * (qr.x * qr.x + qr.y * qr.y);
    T R01 = T(2.0) * (qr.x * qr.y - qr.w * qr.z);
    T R00 = T(1.0) - T(2.0) * (qr.y * qr.y + qr.z * qr.z);
    T th[3];
    th[0] = xatan2(-R12, R22);
    th[1] = xasin(xclamp(R02, T(-1.0), T(1.0)));
    th[2] = xatan2(-R01, R00);
    if (std::fabs(val(R02)) > 1.0 - opt.amb_angle ||
        std::fabs(val(th[0])) > M_PI - opt.amb_angle || std::fabs(val(th[2])) > M_PI - opt.amb_angle)
      out->ambiguous = true;  // gimbal lock / ±π wrap (R7, R9)
    T tau[3];
    for (int i = 0; i < 3; ++i) {
      if (i < J.dof) tau[i] = T(J.k_l) * (xclamp(th[i], T(J.lo[i]), T(J.hi[i])) - th[i]);
      else tau[i] = -(T(J.k_a) * th[i]);
    }
    if (J.act_kind >= 0) {  // actuator on this joint (R11, R12)
      for (int i = 0; i < J.dof; ++i) {
        T a = T(action[J.act_offset + i]);
        if (J.act_kind == 0) tau[i] = tau[i] + T(J.act_strength) * xclamp(a, T(-1.0), T(1.0));
        else tau[i] = tau[i] + T(J.act_strength) * (xclamp(a, T(J.lo[i]), T(J.hi[i])) - th[i]);
      }
    }
    // τ_i is the generalised force conjugate to θ_i (R7 as amended in DESIGN.md): the
    // relative angular velocity is ω = Σ θ̇_i a_i with the rotation axes of R = Rx Ry Rz
    //   a0 = x,  a1 = Rx(θ0)·y = (0, cos θ0, sin θ0),  a2 = Rx(θ0)·Ry(θ1)·z,
    // so the torque whose power is Σ τ_i θ̇_i (the gradient of the spring potential) is
    // Σ τ_i b_i with b the dual basis (b_i·a_j = δ_ij), in the parent joint frame:
    //   b0 = (1, sin θ0 tan θ1, −cos θ0 tan θ1),  b1 = a1,  b2 = (0, −sin θ0, cos θ0)/cos θ1.
    // 1/cos θ1 is evaluated as cos θ1 / max(cos² θ1, 0.01) (gimbal-lock guard, R7).
    // The sines and cosines are read off R = Rx(θ0)Ry(θ1)Rz(θ2): R02 = sin θ1,
    // R12 = −sin θ0 cos θ1, R22 = cos θ0 cos θ1, so cos θ1 = √(R12² + R22²) ≥ 0.
    const T c1 = xsqrt(R12 * R12 + R22 * R22);
    const T s1 = xclamp(R02, T(-1.0), T(1.0));
    const T c0 = (val(c1) > 0.0) ? R22 / c1 : T(1.0);
    const T s0 = (val(c1) > 0.0) ? -(R12 / c1) : T(0.0);
    const T ic = c1 / xmax(c1 * c1, T(0.01));
    V3<T> b0 = v3(T(1.0), s0 * s1 * ic, -(c0 * s1 * ic));
    V3<T> b1 = v3(T(0.0), c0, s0);
    V3<T> b2 = v3(T(0.0), -(s0 * ic), c0 * ic);
    V3<T> tj = tau[0] * b0 + tau[1] * b1 + tau[2] * b2;
    V3<T> tw = rotate(fp, tj);
    V3<T> td, twd_c, twd_p;
    { Neutral n(no_ca); td = T(J.c_a) * (P.w - C.w); twd_c = tw + td; twd_p = tw + td; }
    F[J.child] = F[J.child] + f;
    Tq[J.child] = Tq[J.child] + (twd_c + cross(rc, f));
    F[J.parent] = F[J.parent] - f;
    Tq[J.parent] = Tq[J.parent] - (twd_p + cross(rp, f));
  }

  // ---- 4. contacts, velocity level + Baumgarte (R13-R19)
  for (int i = 0; i < S.ns; ++i) {
    const OSlot& sl = S.slots[i];
    const BodyState<T>& A = st[sl.a];
    const BodyState<T>& Bs = st[sl.b];
    const OBody& bA = S.bodies[sl.a];
    const OBody& bB = S.bodies[sl.b];
    V3<T> n, pt;
    T d;
    bool par = false;
    narrowphase<T>(S, sl, st, opt.amb_par, &n, &pt, &d, &par);
    // R23: a near-parallel capsule pair only matters if it can be in contact
    // (the segment distance is unique; only the contact point is not)
    if (par && val(d) > -opt.amb_d) out->ambiguous = true;
    if (std::fabs(val(d)) < opt.amb_d) out->ambiguous = true;  // R23 onset band
    if (!(d > T(0.0))) continue;                                 // R16: strict d > 0

    V3<T> rA = pt - A.x, rB = pt - Bs.x;
    V3<T> u = (A.v + cross(A.w, rA)) - (Bs.v + cross(Bs.w, rB));
    T un = dot(u, n);
    auto eff = [&](V3<T> dir) {  // k(dir) = Σ_X not static [1/m_X + (r_X×dir)·I_w⁻¹(r_X×dir)]
      T k(0.0);
      if (!bA.is_static) {
        V3<T> rn = cross(rA, dir);
        k = k + T(1.0) / T(bA.mass) + dot(rn, iiw(A.q, V<T>(bA.inertia), rn));
      }
      if (!bB.is_static) {
        V3<T> rn = cross(rB, dir);
        k = k + T(1.0) / T(bB.mass) + dot(rn, iiw(Bs.q, V<T>(bB.inertia), rn));
      }
      return k;
    };
    T kn = eff(n);
    T jn = xmax(T(0.0), (-(T(1.0) + T(S.e)) * un + (T(S.beta) / h) * d) / kn);
    if (!(jn > T(0.0))) continue;                                // R15
    if (val(jn) * val(kn) < opt.amb_jn) out->ambiguous = true;   // R23 weak impulse (diagnostic: not counted)
    V3<T> ut = u - un * n;
    T st_ = xsqrt(dot(ut, ut));
    V3<T> P = jn * n;
    if (st_ > T(0.0)) {
      V3<T> that = (T(1.0) / st_) * ut;
      T jt = xmin(st_ / eff(that), T(S.mu) * jn);
      P = P - jt * that;
    }
    if (!bA.is_static) {
      dV[sl.a] = dV[sl.a] + (T(1.0) / T(bA.mass)) * P;
      dW[sl.a] = dW[sl.a] + iiw(A.q, V<T>(bA.inertia), cross(rA, P));
      cnt[sl.a] += 1;
    }
    if (!bB.is_static) {
      dV[sl.b] = dV[sl.b] - (T(1.0) / T(bB.mass)) * P;
      dW[sl.b] = dW[sl.b] - iiw(Bs.q, V<T>(bB.inertia), cross(rB, P));
      cnt[sl.b] += 1;
    }
    if (out->active) out->active[i] += 1;
  }

  // ---- 5. potential integrator (R2, R21) ------------------
  const V3<T> g = V<T>(S.gravity);
  for (int b = 0; b < B; ++b) {
    const OBody& bd = S.bodies[b];
    if (bd.is_static) continue;
    BodyState<T>& s = st[b];
    s.v = mhad(bd.mpos, s.v + h * ((T(1.0) / T(bd.mass)) * F[b] + g));
    s.w = mhad(bd.mrot, s.w + h * iiw(s.q, V<T>(bd.inertia), Tq[b]));
  }
  // ---- 6. collision integrator (R14 mean over active contacts) -
  for (int b = 0; b < B; ++b) {
    if (out->contact_dv)
      for (int k = 0; k < 6; ++k) out->contact_dv[6 * b + k] = 0.0;
    const OBody& bd = S.bodies[b];
    if (bd.is_static || cnt[b] == 0) continue;
    BodyState<T>& s = st[b];
    const V3<T> v0 = s.v, w0 = s.w;
    T scale = opt.combine_sum ? T(1.0) : T(1.0) / T(double(cnt[b]));
    s.v = mhad(bd.mpos, s.v + scale * dV[b]);
    s.w = mhad(bd.mrot, s.w + scale * dW[b]);
    if (out->contact_dv || out->contact_dp) {  // velocity change of the collision integrator: after − before
      const V3<T> dv = s.v - v0, dw = s.w - w0;
      const double d6[6] = {val(dv.x), val(dv.y), val(dv.z), val(dw.x), val(dw.y), val(dw.z)};
      if (out->contact_dv)
        for (int k = 0; k < 6; ++k) out->contact_dv[6 * b + k] = d6[k];
      if (out->contact_dp)
        for (int k = 0; k < 6; ++k) out->contact_dp[6 * b + k] += d6[k];
    }
  }
}

template <class T>
void step_range(const OSys& S, const OOpts& opt, int64_t e0, int64_t e1, double* pos, double* rot,
                double* vel, double* ang, const double* action, uint8_t* contact_active,
                uint32_t* status, uint8_t* ambiguous, double* contact_dv, double* contact_dp) {
  const int B = S.nb;
  std::vector<BodyState<T>> st(B);
  for (int64_t e = e0; e < e1; ++e) {
    double* p = pos + e * B * 3;
    double* r = rot + e * B * 4;
    double* v = vel + e * B * 3;
    double* w = ang + e * B * 3;
    for (int b = 0; b < B; ++b) {
      st[b].x = V<T>(p + 3 * b);
      st[b].q = Q<T>(r + 4 * b);
      st[b].v = V<T>(v + 3 * b);
      st[b].w = V<T>(w + 3 * b);
    }
    EnvOut<T> out{contact_active ? contact_active + e * S.ns : nullptr, false,
                  contact_dv ? contact_dv + e * B * 6 : nullptr, contact_dp ? contact_dp + e * B * 6 : nullptr};
    if (out.active) std::memset(out.active, 0, S.ns);
    if (out.contact_dp) std::memset(out.contact_dp, 0, sizeof(double) * 6 * B);
    const double* a = action ? action + e * S.act_dim : nullptr;
    for (int s = 0; s < S.substeps; ++s) substep<T>(S, opt, st.data(), a, &out);
    uint32_t stat = 0;
    for (int b = 0; b < B; ++b) {
      double vals[13] = {val(st[b].x.x), val(st[b].x.y), val(st[b].x.z), val(st[b].q.w), val(st[b].q.x),
                         val(st[b].q.y), val(st[b].q.z), val(st[b].v.x), val(st[b].v.y), val(st[b].v.z),
                         val(st[b].w.x), val(st[b].w.y), val(st[b].w.z)};
      for (double x : vals) {
        if (!std::isfinite(x)) stat |= 1u;                       // SPEC.md:231 NumericalBlowup
        else if (std::fabs(x) > 1e6) stat |= 2u;
      }
      p[3 * b + 0] = vals[0]; p[3 * b + 1] = vals[1]; p[3 * b + 2] = vals[2];
      r[4 * b + 0] = vals[3]; r[4 * b + 1] = vals[4]; r[4 * b + 2] = vals[5]; r[4 * b + 3] = vals[6];
      v[3 * b + 0] = vals[7]; v[3 * b + 1] = vals[8]; v[3 * b + 2] = vals[9];
      w[3 * b + 0] = vals[10]; w[3 * b + 1] = vals[11]; w[3 * b + 2] = vals[12];
    }
    if (status) status[e] = stat;
    if (ambiguous) ambiguous[e] = out.ambiguous ? 1 : 0;
  }
}

}  // namespace

extern "C" {

// In-place: advances envs [e0, e1) of the batch by one step (S.substeps substeps).
// pos/rot/vel/ang: [n][B][3|4|3|3] fp64; action: [n][act_dim] fp64 (may be NULL iff act_dim == 0).
// contact_active: [n][ns] u8 number of substeps each slot was active (or NULL).
// status: [n] bit0 non-finite, bit1 |x| > 1e6 (or NULL).  ambiguous: [n] R23 flag (or NULL).
// contact_dv: [n][B][6] the last substep's collision-integrator Δv, Δω per body (or NULL).
// contact_dp: [n][B][6] the same summed over the step's substeps (or NULL).
int oracle_step(const OSys* S, const OOpts* opt, int64_t e0, int64_t e1, double* pos, double* rot,
                double* vel, double* ang, const double* action, uint8_t* contact_active,
                uint32_t* status, uint8_t* ambiguous, double* contact_dv, double* contact_dp) {
  if (!S || !opt || e1 < e0) return 1;
  step_range<double>(*S, *opt, e0, e1, pos, rot, vel, ang, action, contact_active, status, ambiguous,
                     contact_dv, contact_dp);
  return 0;
}

// Diagnostic: the same step in fp32 arithmetic (inputs/outputs fp64 arrays).
int oracle_step_f32(const OSys* S, const OOpts* opt, int64_t e0, int64_t e1, double* pos, double* rot,
                    double* vel, double* ang, const double* action, uint8_t* contact_active,
                    uint32_t* status, uint8_t* ambiguous, double* contact_dv, double* contact_dp) {
  if (!S || !opt || e1 < e0) return 1;
  step_range<float>(*S, *opt, e0, e1, pos, rot, vel, ang, action, contact_active, status, ambiguous,
                    contact_dv, contact_dp);
  return 0;
}

// Same step run with the op-counting scalar; returns the algorithmic counts
// (SURVEY §8(d) convention) summed over envs [e0, e1).  Not thread-safe
// across concurrent calls on the same thread (counters are thread_local).
int oracle_count_ops(const OSys* S, const OOpts* opt, int64_t e0, int64_t e1, double* pos, double* rot,
                     double* vel, double* ang, const double* action, uint64_t* flops, uint64_t* mufu) {
  if (!S || !opt || e1 < e0) return 1;
  g_flops = 0;
  g_mufu = 0;
  g_mute = 0;
  step_range<Cnt>(*S, *opt, e0, e1, pos, rot, vel, ang, action, nullptr, nullptr, nullptr, nullptr, nullptr);
  *flops = g_flops;
  *mufu = g_mufu;
  return 0;
}

// Narrowphase of slot `slot` for one env's post-kinematic state (test entry):
// pos [B][3], rot [B][4] fp64 -> d, n[3], pt[3]; returns 1 if near-parallel (R23).
int oracle_slot_geometry(const OSys* S, int32_t slot, const double* pos, const double* rot, double* d,
                         double* n, double* pt) {
  std::vector<BodyState<double>> st(S->nb);
  for (int b = 0; b < S->nb; ++b) {
    st[b].x = V<double>(pos + 3 * b);
    st[b].q = Q<double>(rot + 4 * b);
    st[b].v = v3(0.0, 0.0, 0.0);
    st[b].w = v3(0.0, 0.0, 0.0);
  }
  V3<double> nn, pp;
  double dd;
  bool par = false;
  narrowphase<double>(*S, S->slots[slot], st.data(), 1e-6, &nn, &pp, &dd, &par);
  *d = dd;
  n[0] = nn.x; n[1] = nn.y; n[2] = nn.z;
  pt[0] = pp.x; pt[1] = pp.y; pt[2] = pp.z;
  return par ? 1 : 0;
}

// The same count in the "lean" convention (see g_lean): scene-neutral operations uncounted.
int oracle_count_ops_lean(const OSys* S, const OOpts* opt, int64_t e0, int64_t e1, double* pos, double* rot,
                          double* vel, double* ang, const double* action, uint64_t* flops, uint64_t* mufu) {
  g_lean = true;
  const int rc = oracle_count_ops(S, opt, e0, e1, pos, rot, vel, ang, action, flops, mufu);
  g_lean = false;
  return rc;
}

int oracle_abi_version(void) { return 1; }
}
