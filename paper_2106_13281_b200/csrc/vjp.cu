// vjp.cu — reverse mode of one step in ONE launch (NEXT-4).
//
// For every env: g_in = (∂Q_out/∂Q_in)ᵀ g_out and g_action = (∂Q_out/∂a)ᵀ g_out,
// the exact transpose of brax_step_jvp's derivative (same conventions, R35).  A
// block keeps E envs' states in shared memory and sweeps the substeps backwards:
//   for s = S−1 … 0:
//     the state at the start of substep s from a checkpoint (one forward sweep
//     wrote all S of them to HBM), then S2(s) and the items of substep s (their
//     contact counts and summed forces);
//     integrator adjoint (S7, S8: linear in v, ω, F, T, dV, dW; I_w⁻¹(q) by local
//       forward derivatives for anisotropic bodies)        — one thread per (body, env)
//     item adjoints: each joint / contact slot's local Jacobian-transpose product,
//       from value+tangent (D1) evaluations of the same item code along each of its
//       26 (+dof) inputs                                    — warp (lane group) per item
//     gather of the item input adjoints onto the bodies (fixed incidence order)
//     S2 adjoint (kinematic integrator; the rotation update by local D1 derivatives)
// Costs O(26) item evaluations per item and substep instead of the column method's
// O(13B + A) whole steps.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "dual_k.cuh"
#include "step_device.cuh"
#include "system.h"

namespace brax {

int choose_regs(const System& sys, const DPlan& P, int64_t grid);

namespace {

using namespace dev;

struct VjpIO {
  const float *pos, *rot, *vel, *ang, *actions;  // primal inputs [n][B][w], [n][A]
  const float *gpos, *grot, *gvel, *gang;        // output cotangents (NULL = zero)
  float *opos, *orot, *ovel, *oang, *oact;       // input cotangents (oact NULL = skip)
  int64_t n_envs;
  float4* ckpt;  // [blocks][S][B·E·kQS/4]: the state at the start of every substep (one forward sweep)
  int32_t local_ad;  // 1: joint adjoints from value+tangent evaluations too (cross-check)
};

struct VjpArgs {
  VjpIO io;
  const uint32_t* blob;
  DHeader hd;
  int32_t plan;
};

// shared-memory layout (words) for E envs per block, one per lane.  Per-(body, env)
// force / adjoint rows and per-(item, env) input-adjoint rows use odd strides, so a
// warp's scalar accesses (lane = env) hit 32 different banks.
constexpr int kFS = 17;  // FW / FA rows: 16 used words
constexpr int kIS = 27;  // IA rows: 26 item inputs
struct VjpLayout {
  int32_t blob, q, q0, qk, gq, fw, fa, rec, a, ga, cnt, total;
};
__host__ __device__ inline VjpLayout vjp_layout(int B, int J, int C, int A, int E, int blob_words) {
  VjpLayout L;
  const int rq = B * E * kQS;
  L.blob = 0;
  L.q = L.blob + round4(blob_words);
  L.q0 = L.q + rq;
  L.qk = L.q0 + rq;
  L.gq = L.qk + rq;
  L.fw = L.gq + rq;
  L.fa = L.fw + B * E * kFS;
  L.rec = L.fa + B * E * kFS;
  int recs = (J + C) * E * 12, ia = (J + C) * E * kIS;
  L.a = L.rec + round4(recs > ia ? recs : ia);
  L.ga = L.a + round4(A * E);
  L.cnt = L.ga + round4(A * E);
  L.total = L.cnt + round4(C * E);
  return L;
}

// a body state in registers with a unit tangent on coordinate j (0-2 pos, 3-6 rot,
// 7-9 vel, 10-12 ang; j < 0: no tangent), read from an F1 record
template <class S> struct RegRow {
  V3T<S> p;
  Q4T<S> q;
  V3T<S> v, w;
  __device__ __forceinline__ V3T<S> pos() const { return p; }
  __device__ __forceinline__ Q4T<S> rot() const { return q; }
  __device__ __forceinline__ V3T<S> vel() const { return v; }
  __device__ __forceinline__ V3T<S> ang() const { return w; }
};
__device__ __forceinline__ RegRow<D1> load_d1(const float* rec, int j) {
  auto t = [&](int k) { return k == j ? 1.f : 0.f; };
  RegRow<D1> r;
  r.p = {{rec[0], t(0)}, {rec[1], t(1)}, {rec[2], t(2)}};
  r.q = {{rec[4], t(3)}, {rec[5], t(4)}, {rec[6], t(5)}, {rec[7], t(6)}};
  r.v = {{rec[8], t(7)}, {rec[9], t(8)}, {rec[10], t(9)}};
  r.w = {{rec[12], t(10)}, {rec[13], t(11)}, {rec[14], t(12)}};
  return r;
}
__device__ __forceinline__ float dot_t(V3T<D1> a, const float* g) {
  return __fmaf_rn(a.x.t, g[0], __fmaf_rn(a.y.t, g[1], __fmul_rn(a.z.t, g[2])));
}
// K tangents at once: tangent k on item input j0 + k; this row's inputs are base..base+12
constexpr int KT = 2;  // tangents per local evaluation
using DT = DK<KT>;
__device__ __forceinline__ DT mk_dt(float v, int j, int j0) {
  DT d;
  d.v = v;
#pragma unroll
  for (int k = 0; k < KT; ++k) d.t[k] = (j == j0 + k) ? 1.f : 0.f;
  return d;
}
__device__ __forceinline__ RegRow<DT> load_dt(const float* rec, int base, int j0) {
  RegRow<DT> r;
  r.p = {mk_dt(rec[0], base, j0), mk_dt(rec[1], base + 1, j0), mk_dt(rec[2], base + 2, j0)};
  r.q = {mk_dt(rec[4], base + 3, j0), mk_dt(rec[5], base + 4, j0), mk_dt(rec[6], base + 5, j0),
         mk_dt(rec[7], base + 6, j0)};
  r.v = {mk_dt(rec[8], base + 7, j0), mk_dt(rec[9], base + 8, j0), mk_dt(rec[10], base + 9, j0)};
  r.w = {mk_dt(rec[12], base + 10, j0), mk_dt(rec[13], base + 11, j0), mk_dt(rec[14], base + 12, j0)};
  return r;
}
__device__ __forceinline__ float dot_tk(const V3T<DT>& a, const float* g, int k) {
  return __fmaf_rn(a.x.t[k], g[0], __fmaf_rn(a.y.t[k], g[1], __fmul_rn(a.z.t[k], g[2])));
}

// ---- hand-derived adjoint of joint_f (step_device.cuh) for one env, plain fp32:
// given the cotangents of (F, T_child, T_parent-as-stored) returns those of the
// parent's and the child's (pos, rot, vel, ang) and of the joint's actions.  Same
// conventions as the value+tangent path (R35): clamps pass the derivative where the
// argument is selected (ties included), the joint angles' derivatives are the
// analytic ones of atan2 / asin (the kernel's polynomials agree to ~1e-6).
struct V3f { float x, y, z; };
__device__ __forceinline__ V3f v3(float x, float y, float z) { return {x, y, z}; }
__device__ __forceinline__ V3f operator+(V3f a, V3f b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3f operator-(V3f a, V3f b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3f operator*(float s, V3f a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ float dot3(V3f a, V3f b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3f cross3(V3f a, V3f b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
struct Qf { float w, x, y, z; };
__device__ __forceinline__ Qf qmulf(Qf a, Qf b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
__device__ __forceinline__ Qf qconjf(Qf q) { return {q.w, -q.x, -q.y, -q.z}; }
__device__ __forceinline__ V3f rotf(Qf q, V3f v) {
  const V3f u{q.x, q.y, q.z};
  return v + (2.f * q.w) * cross3(u, v) + 2.f * cross3(u, cross3(u, v));
}
// cotangent of q for r = rotate(q, v) (any q, not only unit ones)
__device__ __forceinline__ Qf rot_adj_q(Qf q, V3f v, V3f g) {
  const V3f u{q.x, q.y, q.z};
  const V3f gu = (2.f * q.w) * cross3(v, g) + 2.f * (dot3(u, v) * g + dot3(u, g) * v - (2.f * dot3(v, g)) * u);
  return {2.f * dot3(g, cross3(u, v)), gu.x, gu.y, gu.z};
}
__device__ __forceinline__ void joint_adj(const DJoint& Jm, const float* recP, const float* recC, const float* act,
                                          int act_stride, const float* gF, const float* gTc, const float* gTp,
                                          float* ia, float* g_act) {
  const float4* J4 = reinterpret_cast<const float4*>(&Jm);
  const int4 h0 = *reinterpret_cast<const int4*>(&Jm), h1 = reinterpret_cast<const int4*>(&Jm)[1];
  const int dof = h0.z, act_kind = h0.w, act_offset = h1.x, flags = h1.y;
  const float4 op_k = J4[2], oc_cl = J4[3], jpv = J4[4], jcv = J4[5], lo_kl = J4[6], hi_ka = J4[7], ca_s = J4[8];
  const float lo[3] = {lo_kl.x, lo_kl.y, lo_kl.z}, hi[3] = {hi_ka.x, hi_ka.y, hi_ka.z};
  const V3f xp{recP[0], recP[1], recP[2]}, vp{recP[8], recP[9], recP[10]}, wp{recP[12], recP[13], recP[14]};
  const V3f xc{recC[0], recC[1], recC[2]}, vc{recC[8], recC[9], recC[10]}, wc{recC[12], recC[13], recC[14]};
  const Qf qp{recP[4], recP[5], recP[6], recP[7]}, qc{recC[4], recC[5], recC[6], recC[7]};
  const Qf jp{jpv.x, jpv.y, jpv.z, jpv.w}, jc{jcv.x, jcv.y, jcv.z, jcv.w};
  const V3f op{op_k.x, op_k.y, op_k.z}, oc{oc_cl.x, oc_cl.y, oc_cl.z};
  // ---- forward intermediates
  const V3f rp = rotf(qp, op), rc = rotf(qc, oc);
  const V3f dx = (xp - xc) + (rp - rc);
  V3f f = op_k.w * dx;
  const bool cl = !(flags & kJNoCl), ca = !(flags & kJNoCa);
  if (cl) f = f + oc_cl.w * ((cross3(wp, rp) + vp) - (cross3(wc, rc) + vc));
  const Qf fp = qmulf(qp, jp), fc = qmulf(qc, jc);
  const Qf qr0 = qmulf(qconjf(fp), fc);
  const float sg = qr0.w < 0.f ? -1.f : 1.f;
  const Qf qr{sg * qr0.w, sg * qr0.x, sg * qr0.y, sg * qr0.z};
  const float R02 = 2.f * (qr.x * qr.z + qr.w * qr.y), R12 = 2.f * (qr.y * qr.z - qr.w * qr.x);
  const float R22 = 1.f - 2.f * (qr.x * qr.x + qr.y * qr.y), R01 = 2.f * (qr.x * qr.y - qr.w * qr.z);
  const float R00 = 1.f - 2.f * (qr.y * qr.y + qr.z * qr.z);
  const float s1 = fminf(fmaxf(R02, -1.f), 1.f);
  const float th[3] = {atan2_f(F1{-R12}, F1{R22}).x, asin_f(F1{s1}).x, atan2_f(F1{-R01}, F1{R00}).x};
  float tau[3];
  for (int i = 0; i < 3; ++i) tau[i] = i < dof ? lo_kl.w * (fminf(fmaxf(th[i], lo[i]), hi[i]) - th[i]) : -(hi_ka.w * th[i]);
  if (act_kind >= 0)
    for (int i = 0; i < dof; ++i) {
      const float a = act[(act_offset + i) * act_stride];
      tau[i] += act_kind == 0 ? ca_s.y * fminf(fmaxf(a, -1.f), 1.f) : ca_s.y * (fminf(fmaxf(a, lo[i]), hi[i]) - th[i]);
    }
  const float c2 = R12 * R12 + R22 * R22;
  const float ic = c2 > 0.f ? rsqrt_mufu(c2) : 0.f;
  const float t1 = tau[1] * ic, m = fminf(ic * ic, 100.f), u = (tau[2] - tau[0] * R02) * m;
  const V3f tj{tau[0], u * R12 + t1 * R22, u * R22 - t1 * R12};
  // ---- reverse
  const V3f gTcv{gTc[0], gTc[1], gTc[2]}, gtp{-gTp[0], -gTp[1], -gTp[2]};  // tp_pos = −T_parent
  V3f gf = v3(gF[0], gF[1], gF[2]) + cross3(gTcv, rc) + cross3(gtp, rp);
  V3f grc = cross3(f, gTcv), grp = cross3(f, gtp);
  const V3f gtwd = gTcv + gtp;
  V3f gwp{0.f, 0.f, 0.f}, gwc{0.f, 0.f, 0.f}, gvp{0.f, 0.f, 0.f}, gvc{0.f, 0.f, 0.f};
  if (ca) {
    gwp = ca_s.x * gtwd;
    gwc = (-ca_s.x) * gtwd;
  }
  Qf gfp = rot_adj_q(fp, tj, gtwd);
  const V3f gtj = rotf(qconjf(fp), gtwd);
  float gtau[3] = {gtj.x, 0.f, 0.f}, gR02 = 0.f, gR12 = 0.f, gR22 = 0.f, gR01 = 0.f, gR00 = 0.f;
  const float gu = gtj.y * R12 + gtj.z * R22, gt1 = gtj.y * R22 - gtj.z * R12;
  gR12 += gtj.y * u - gtj.z * t1;
  gR22 += gtj.y * t1 + gtj.z * u;
  gtau[2] += gu * m;
  gtau[0] -= gu * m * R02;
  gR02 -= gu * m * tau[0];
  float gic = 0.f;
  if (ic * ic <= 100.f) gic += gu * (tau[2] - tau[0] * R02) * 2.f * ic;
  gtau[1] += gt1 * ic;
  gic += gt1 * tau[1];
  if (c2 > 0.f) {
    const float gc2 = gic * (-0.5f * ic * ic * ic);
    gR12 += 2.f * R12 * gc2;
    gR22 += 2.f * R22 * gc2;
  }
  float gth[3] = {0.f, 0.f, 0.f};
  if (act_kind >= 0)
    for (int i = 0; i < dof; ++i) {
      const float a = act[(act_offset + i) * act_stride];
      const float l = act_kind == 0 ? -1.f : lo[i], h = act_kind == 0 ? 1.f : hi[i];
      const float ga = (a >= l && a <= h) ? ca_s.y * gtau[i] : 0.f;
      g_act[i] += ga;
      if (act_kind == 1) gth[i] -= ca_s.y * gtau[i];
    }
  for (int i = 0; i < 3; ++i) {
    if (i < dof) gth[i] += (th[i] >= lo[i] && th[i] <= hi[i]) ? 0.f : -lo_kl.w * gtau[i];
    else gth[i] -= hi_ka.w * gtau[i];
  }
  {  // th0 = atan2(−R12, R22), th1 = asin(clamp R02), th2 = atan2(−R01, R00)
    const float n0 = R12 * R12 + R22 * R22, n2 = R01 * R01 + R00 * R00;
    if (n0 > 0.f) {
      const float g0 = div_mufu(gth[0], n0);
      gR12 -= g0 * R22;
      gR22 += g0 * R12;
    }
    if (R02 > -1.f && R02 < 1.f) gR02 += gth[1] * rsqrt_mufu((1.f - s1) * (1.f + s1));
    if (n2 > 0.f) {
      const float g2 = div_mufu(gth[2], n2);
      gR01 -= g2 * R00;
      gR00 += g2 * R01;
    }
  }
  Qf gqr{2.f * qr.y * gR02 - 2.f * qr.x * gR12 - 2.f * qr.z * gR01,
         2.f * qr.z * gR02 - 2.f * qr.w * gR12 - 4.f * qr.x * gR22 + 2.f * qr.y * gR01,
         2.f * qr.w * gR02 + 2.f * qr.z * gR12 - 4.f * qr.y * gR22 + 2.f * qr.x * gR01 - 4.f * qr.y * gR00,
         2.f * qr.x * gR02 + 2.f * qr.y * gR12 - 2.f * qr.w * gR01 - 4.f * qr.z * gR00};
  const Qf gqr0{sg * gqr.w, sg * gqr.x, sg * gqr.y, sg * gqr.z};
  // qr0 = conj(fp) ⊗ fc
  const Qf gcf = qmulf(gqr0, qconjf(fc));
  const Qf gfc = qmulf(fp, gqr0);
  gfp = {gfp.w + gcf.w, gfp.x - gcf.x, gfp.y - gcf.y, gfp.z - gcf.z};
  Qf gqp = qmulf(gfp, qconjf(jp)), gqc = qmulf(gfc, qconjf(jc));
  if (cl) {
    const V3f gd = oc_cl.w * gf;
    gvp = gvp + gd;
    gvc = gvc - gd;
    gwp = gwp + cross3(rp, gd);
    grp = grp + cross3(gd, wp);
    gwc = gwc - cross3(rc, gd);
    grc = grc - cross3(gd, wc);
  }
  const V3f gdx = op_k.w * gf;
  grp = grp + gdx;
  grc = grc - gdx;
  const Qf a1 = rot_adj_q(qp, op, grp), a2 = rot_adj_q(qc, oc, grc);
  gqp = {gqp.w + a1.w, gqp.x + a1.x, gqp.y + a1.y, gqp.z + a1.z};
  gqc = {gqc.w + a2.w, gqc.x + a2.x, gqc.y + a2.y, gqc.z + a2.z};
  const float outP[13] = {gdx.x, gdx.y, gdx.z, gqp.w, gqp.x, gqp.y, gqp.z, gvp.x, gvp.y, gvp.z, gwp.x, gwp.y, gwp.z};
  const float outC[13] = {-gdx.x, -gdx.y, -gdx.z, gqc.w, gqc.x, gqc.y, gqc.z, gvc.x, gvc.y, gvc.z, gwc.x, gwc.y, gwc.z};
  for (int j = 0; j < 13; ++j) {
    ia[j] = outP[j];
    ia[13 + j] = outC[j];
  }
}

// ---- hand-derived adjoint of contact_f (step_device.cuh) for the plane contacts
// (types 0-2: sphere, capsule end, box corner vs a plane), one env, plain fp32 reverse
// after a forward pass that repeats contact_f<F1>'s operations (so every decision —
// penetration, activity, the friction clamp — is taken on the same values).  Given the
// cotangents of (P, r_A×P, r_B×P) returns those of body A's and body B's (pos, rot,
// vel, ang).  Conventions as in the value+tangent path (R35): max / min pass the
// derivative to the selected argument (the first on ties), an inactive slot has zero
// derivative.  Returns false for the shape–shape types (the caller then uses the
// local value+tangent evaluations).
__device__ __forceinline__ V3f v3of(V3T<F1> a) { return {a.x.x, a.y.x, a.z.x}; }
__device__ __forceinline__ V3T<F1> v3t(V3f a) { return {{a.x}, {a.y}, {a.z}}; }
// cotangent of q for n = rotate(q, ẑ) (contact_f's rotate_z)
__device__ __forceinline__ Qf rotz_adj_q(Qf q, V3f g) {
  return {2.f * (q.y * g.x - q.x * g.y), 2.f * (q.z * g.x - q.w * g.y) - 4.f * q.x * g.z,
          2.f * (q.w * g.x + q.z * g.y) - 4.f * q.y * g.z, 2.f * (q.x * g.x + q.y * g.y)};
}
__device__ __forceinline__ Qf qaddf(Qf a, Qf b) { return {a.w + b.w, a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ bool contact_adj(const DSlot& SLm, const float* recA, const float* recB, float opl_e,
                                            float beta_over_h, float mu, const float* gPv, const float* gtav,
                                            const float* gtbv, float* ia) {
  const float4* S4 = reinterpret_cast<const float4*>(&SLm);
  const int4 h0 = *reinterpret_cast<const int4*>(&SLm), h1 = reinterpret_cast<const int4*>(&SLm)[1];
  const int type = h0.x, a_static = h1.x, b_static = h1.y, fl = h1.z;
  if (type > 2) return false;
  for (int j = 0; j < 26; ++j) ia[j] = 0.f;
  const float4 ca = S4[2], cb = S4[4], ells = S4[6], ra4 = S4[3], rb4 = S4[5], k4 = S4[7];
  const float ra = ca.w;
  const float4 iia4 = S4[8], iib4 = S4[9];
  const float iia[3] = {iia4.x, iia4.y, iia4.z}, iib[3] = {iib4.x, iib4.y, iib4.z};
  const bool isa = fl & kSIsoA, isb = fl & kSIsoB;
  const Row<F1> A{const_cast<float*>(recA)}, B{const_cast<float*>(recB)};
  // ---- forward, as contact_f<F1>
  const Q4T<F1> qa = A.rot(), qb = B.rot();
  const V3T<F1> xa = A.pos(), xb = B.pos();
  const V3T<F1> cA = (fl & kSZeroPa) ? xa : xa + rotate(qa, V3T<F1>{{ca.x}, {ca.y}, {ca.z}});
  const V3T<F1> cB = (fl & kSZeroPb) ? xb : xb + rotate(qb, V3T<F1>{{cb.x}, {cb.y}, {cb.z}});
  Q4T<F1> qA = qa, qB = qb;
  if (!(fl & kSIdentA)) qA = qmul(qa, Q4T<F1>{{ra4.x}, {ra4.y}, {ra4.z}, {ra4.w}});
  if (!(fl & kSIdentB)) qB = qmul(qb, Q4T<F1>{{rb4.x}, {rb4.y}, {rb4.z}, {rb4.w}});
  const V3T<F1> n = rotate_z(qB);
  V3T<F1> c, pt;
  F1 d;
  if (type == 2) {
    c = cA + rotate(qA, V3T<F1>{{k4.x}, {k4.y}, {k4.z}});
    d = -dot(c - cB, n);
    pt = c;
  } else {
    c = (type == 1) ? axpy(ells.x, rotate_z(qA), cA) : cA;
    d = ra - dot(c - cB, n);
    pt = axpy(-ra, n, c);
  }
  if (!(d.x > 0.f)) return true;  // R16: not penetrating, zero derivative
  const V3T<F1> rA = pt - xa, rB = pt - xb;
  const V3T<F1> u = cross_add(A.ang(), rA, A.vel()) - cross_add(B.ang(), rB, B.vel());
  const F1 un = dot(u, n);
  auto eff = [&](V3T<F1> dir) {
    F1 k = {0.f};
    if (!a_static) {
      V3T<F1> rn = cross(rA, dir);
      k = k + ells.z + dot(rn, iw(qa, iia, isa, rn));
    }
    if (!b_static) {
      V3T<F1> rn = cross(rB, dir);
      k = k + ells.w + dot(rn, iw(qb, iib, isb, rn));
    }
    return k;
  };
  const F1 kn = eff(n);
  const F1 num = -opl_e * un + beta_over_h * d;
  const F1 raw = vdiv(num, kn);
  if (!(raw.x > 0.f)) return true;  // R15: inactive (jn = 0), zero derivative
  const F1 jn = raw;
  const V3T<F1> ut = u - un * n;
  const F1 st2 = dot(ut, ut);
  const bool sl = st2.x > 0.f;
  const F1 ist = sl ? vrsqrt(st2) : F1{0.f};
  const F1 st = st2 * ist;
  const V3T<F1> th = ist * ut;
  const F1 kt = sl ? eff(th) : F1{1.f};
  const F1 q = vdiv(st, kt), mjn = mu * jn;
  const bool fric_q = !(mjn.x < q.x);  // jt = min(q, μ·jn): q selected (first on ties)
  const F1 jt = fric_q ? q : mjn;
  const V3T<F1> Pv = jn * n - jt * th;
  // ---- reverse (plain fp32)
  const V3f P = v3of(Pv), vn = v3of(n), vrA = v3of(rA), vrB = v3of(rB), vu = v3of(u), vth = v3of(th), vut = v3of(ut);
  const V3f gta{gtav[0], gtav[1], gtav[2]}, gtb{gtbv[0], gtbv[1], gtbv[2]};
  V3f gP = v3(gPv[0], gPv[1], gPv[2]) + cross3(gta, vrA) + cross3(gtb, vrB);  // t = r×P: ḡP += ḡt×r
  V3f grA = cross3(P, gta), grB = cross3(P, gtb);                               // ḡr += P×ḡt
  // P = jn·n − jt·th
  float gjn = dot3(gP, vn), gjt = -dot3(gP, vth);
  V3f gn = jn.x * gP, gth = (-jt.x) * gP;
  float gst = 0.f, gkt = 0.f;
  if (fric_q) {  // q = st / kt
    const float ikt = div_mufu(1.f, kt.x);
    gst += gjt * ikt;
    gkt -= gjt * q.x * ikt;
  } else {
    gjn += mu * gjt;
  }
  float gst2 = 0.f, gist = 0.f;
  V3f gut{0.f, 0.f, 0.f};
  // eff(dir): Σ_X not static (1/m_X + w·M_X w), w = r_X × dir, M_X = I_w⁻¹(q_X) (symmetric)
  float gq_a[4] = {0.f, 0.f, 0.f, 0.f}, gq_b[4] = {0.f, 0.f, 0.f, 0.f};
  auto eff_adj = [&](V3f dir, float g, V3f& gdir) {
    auto side = [&](bool st_, const Q4T<F1>& qx, const float* ii, bool iso, V3f r, V3f& gr, float* gq) {
      if (st_) return;
      const V3f w = cross3(r, dir);
      const V3f Mw = v3of(iw(qx, ii, iso, v3t(w)));
      const V3f gw = (2.f * g) * Mw;
      gr = gr + cross3(dir, gw);   // w = r×dir: ḡr += dir×ḡw
      gdir = gdir + cross3(gw, r); // ḡdir += ḡw×r
      if (!iso) {  // ∂(w·M(q)w)/∂q by local forward derivatives
        for (int k = 0; k < 4; ++k) {
          Q4T<D1> qd{{qx.w.x, k == 0 ? 1.f : 0.f}, {qx.x.x, k == 1 ? 1.f : 0.f}, {qx.y.x, k == 2 ? 1.f : 0.f},
                     {qx.z.x, k == 3 ? 1.f : 0.f}};
          const V3T<D1> wd{{w.x, 0.f}, {w.y, 0.f}, {w.z, 0.f}};
          const V3T<D1> m = iw(qd, ii, false, wd);
          gq[k] += g * (w.x * m.x.t + w.y * m.y.t + w.z * m.z.t);
        }
      }
    };
    side(a_static, qa, iia, isa, vrA, grA, gq_a);
    side(b_static, qb, iib, isb, vrB, grB, gq_b);
  };
  if (sl) {
    eff_adj(vth, gkt, gth);  // kt = eff(th)
    // th = ist·ut, st = st2·ist, ist = rsqrt(st2), st2 = ut·ut
    gut = gut + ist.x * gth;
    gist += dot3(gth, vut) + st2.x * gst;
    gst2 += ist.x * gst;
    gst2 += gist * (-0.5f * ist.x * ist.x * ist.x);
    gut = gut + (2.f * gst2) * vut;
  }
  // ut = u − un·n
  V3f gu = gut;
  float gun = -dot3(gut, vn);
  gn = gn - un.x * gut;
  // jn = num / kn (active)
  const float ikn = div_mufu(1.f, kn.x);
  const float gnum = gjn * ikn, gkn = -gjn * raw.x * ikn;
  gun += -opl_e * gnum;
  float gd = beta_over_h * gnum;
  eff_adj(vn, gkn, gn);  // kn = eff(n)
  // un = u·n
  gu = gu + gun * vn;
  gn = gn + gun * vu;
  // u = (v_A + ω_A×r_A) − (v_B + ω_B×r_B)
  const V3f wa{recA[12], recA[13], recA[14]}, wb{recB[12], recB[13], recB[14]};
  const V3f gva = gu, gwa = cross3(vrA, gu), gvb = (-1.f) * gu, gwb = (-1.f) * cross3(vrB, gu);
  grA = grA + cross3(gu, wa);
  grB = grB - cross3(gu, wb);
  // r_A = pt − x_A, r_B = pt − x_B
  V3f gpt = grA + grB, gxa = (-1.f) * grA, gxb = (-1.f) * grB;
  // narrowphase
  V3f gc = gpt, gcA{0.f, 0.f, 0.f}, gcB{0.f, 0.f, 0.f};
  Qf gqA{0.f, 0.f, 0.f, 0.f};
  const V3f vc = v3of(c), vcB = v3of(cB);
  if (type == 2) {  // pt = c, d = −(c − cB)·n
    gc = gc - gd * vn;
    gcB = gcB + gd * vn;
    gn = gn - gd * (vc - vcB);
    gcA = gc;
    gqA = rot_adj_q(Qf{qA.w.x, qA.x.x, qA.y.x, qA.z.x}, v3(k4.x, k4.y, k4.z), gc);
  } else {  // pt = c − r·n, d = r − (c − cB)·n
    gn = gn - ra * gpt;
    gc = gc - gd * vn;
    gcB = gcB + gd * vn;
    gn = gn - gd * (vc - vcB);
    gcA = gc;
    if (type == 1) gqA = rotz_adj_q(Qf{qA.w.x, qA.x.x, qA.y.x, qA.z.x}, ells.x * gc);  // c = cA + ℓ·rotate_z(qA)
  }
  Qf gqB = rotz_adj_q(Qf{qB.w.x, qB.x.x, qB.y.x, qB.z.x}, gn);  // n = rotate_z(qB)
  // qA = qa ⊗ r_colA, qB = qb ⊗ r_colB
  Qf gqa = (fl & kSIdentA) ? gqA : qmulf(gqA, qconjf(Qf{ra4.x, ra4.y, ra4.z, ra4.w}));
  Qf gqb = (fl & kSIdentB) ? gqB : qmulf(gqB, qconjf(Qf{rb4.x, rb4.y, rb4.z, rb4.w}));
  // cA = xa + rotate(qa, ca), cB = xb + rotate(qb, cb)
  gxa = gxa + gcA;
  gxb = gxb + gcB;
  if (!(fl & kSZeroPa)) gqa = qaddf(gqa, rot_adj_q(Qf{qa.w.x, qa.x.x, qa.y.x, qa.z.x}, v3(ca.x, ca.y, ca.z), gcA));
  if (!(fl & kSZeroPb)) gqb = qaddf(gqb, rot_adj_q(Qf{qb.w.x, qb.x.x, qb.y.x, qb.z.x}, v3(cb.x, cb.y, cb.z), gcB));
  gqa = qaddf(gqa, Qf{gq_a[0], gq_a[1], gq_a[2], gq_a[3]});
  gqb = qaddf(gqb, Qf{gq_b[0], gq_b[1], gq_b[2], gq_b[3]});
  const float outA[13] = {gxa.x, gxa.y, gxa.z, gqa.w, gqa.x, gqa.y, gqa.z, gva.x, gva.y, gva.z, gwa.x, gwa.y, gwa.z};
  const float outB[13] = {gxb.x, gxb.y, gxb.z, gqb.w, gqb.x, gqb.y, gqb.z, gvb.x, gvb.y, gvb.z, gwb.x, gwb.y, gwb.z};
  for (int j = 0; j < 13; ++j) {
    ia[j] = outA[j];
    ia[13 + j] = outB[j];
  }
  return true;
}

template <int R>
__global__ void __maxnreg__(R) brax_vjp_kernel(const __grid_constant__ VjpArgs ka) {
  extern __shared__ __align__(16) uint32_t smem[];
  const DHeader& H = ka.hd;
  const DPlan& P = H.plan[ka.plan];
  const VjpIO& io = ka.io;
  const int B = H.B, J = H.J, C = H.C, A = H.A, E = P.E, G = P.G;
  const VjpLayout L = vjp_layout(B, J, C, A, E, H.blob_words);
  uint32_t* sBlob = smem + L.blob;
  float* Q = reinterpret_cast<float*>(smem + L.q);
  float* Q0 = reinterpret_cast<float*>(smem + L.q0);
  float* QK = reinterpret_cast<float*>(smem + L.qk);
  float* GQ = reinterpret_cast<float*>(smem + L.gq);
  float* FW = reinterpret_cast<float*>(smem + L.fw);
  float* FA = reinterpret_cast<float*>(smem + L.fa);
  float* REC = reinterpret_cast<float*>(smem + L.rec);  // item records, then item input adjoints
  float* IA = REC;
  float* sA = reinterpret_cast<float*>(smem + L.a);
  float* GA = reinterpret_cast<float*>(smem + L.ga);
  float* sCnt = reinterpret_cast<float*>(smem + L.cnt);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  const int LG = 32 / G, grp = lane / LG, el = lane - grp * LG;
  const int64_t e0 = int64_t(blockIdx.x) * E;
  const int nvalid = (io.n_envs - e0 < E) ? int(io.n_envs - e0) : E;
  const float h = H.h;
  const bool hand_adj = !io.local_ad;

  // ---- tables, primal state (identity in padded slots), cotangents, actions
  for (int i = tid; i < H.blob_words / 4; i += nt)
    reinterpret_cast<uint4*>(sBlob)[i] = reinterpret_cast<const uint4*>(ka.blob)[i];
  for (int i = tid; i < B * E; i += nt) {
    const int b = i / E, env = i - b * E;
    float* q0 = Q0 + i * kQS;
    float* gq = GQ + i * kQS;
    for (int k = 0; k < kQS; ++k) q0[k] = gq[k] = 0.f;
    q0[4] = 1.f;
    if (env < nvalid) {
      const int64_t g = e0 + env;
      for (int k = 0; k < 3; ++k) {
        q0[k] = io.pos[(g * B + b) * 3 + k];
        q0[8 + k] = io.vel[(g * B + b) * 3 + k];
        q0[12 + k] = io.ang[(g * B + b) * 3 + k];
        gq[k] = io.gpos ? io.gpos[(g * B + b) * 3 + k] : 0.f;
        gq[8 + k] = io.gvel ? io.gvel[(g * B + b) * 3 + k] : 0.f;
        gq[12 + k] = io.gang ? io.gang[(g * B + b) * 3 + k] : 0.f;
      }
      for (int k = 0; k < 4; ++k) {
        q0[4 + k] = io.rot[(g * B + b) * 4 + k];
        gq[4 + k] = io.grot ? io.grot[(g * B + b) * 4 + k] : 0.f;
      }
    }
  }
  for (int i = tid; i < A * E; i += nt) {
    const int k = i / E, env = i - k * E;
    sA[i] = env < nvalid ? io.actions[(e0 + env) * A + k] : 0.f;
    GA[i] = 0.f;
  }
  __syncthreads();

  const DBody* bodies = reinterpret_cast<const DBody*>(sBlob + H.off_bodies);
  const DJoint* joints = reinterpret_cast<const DJoint*>(sBlob + H.off_joints);
  const DSlot* slots = reinterpret_cast<const DSlot*>(sBlob + H.off_slots);
  const int32_t* item_begin = reinterpret_cast<const int32_t*>(sBlob + P.off_item_begin);
  const int32_t* items = reinterpret_cast<const int32_t*>(sBlob + P.off_items) + grp;
  const int32_t* body_begin = reinterpret_cast<const int32_t*>(sBlob + P.off_body_begin);
  const int32_t* bodies_of_warp = reinterpret_cast<const int32_t*>(sBlob + P.off_bodies_of_warp) + grp;
  const int32_t* jinc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_jinc_begin);
  const int32_t* jinc = reinterpret_cast<const int32_t*>(sBlob + H.off_jinc);
  const int32_t* cinc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_cinc_begin);
  const int32_t* cinc = reinterpret_cast<const int32_t*>(sBlob + H.off_cinc);
  const int it0 = item_begin[warp], it1 = item_begin[warp + 1];
  const int bw0 = body_begin[warp], bw1 = body_begin[warp + 1];
  float* sJ = REC;
  float* sC = REC + J * E * kJS;

  // ---- forward pieces on the F1 records (the step kernel's arithmetic, unfused S2)
  auto fwd_kin = [&]() {
    for (int i = bw0; i < bw1; ++i) {
      const int b = bodies_of_warp[i * G];
      if (b >= 0) kinematic<F1>(bodies[b], Row<F1>{Q + (b * LG + el) * kQS}, h);
    }
  };
  auto fwd_items = [&]() {
    for (int it = it0; it < it1; ++it) {
      const int item = items[it * G];
      if (item < 0) continue;
      if (item < J) {
        const DJoint& jt = joints[item];
        joint<F1>(jt, Row<F1>{Q + (jt.parent * LG + el) * kQS}, Row<F1>{Q + (jt.child * LG + el) * kQS}, sA + el,
                  E, sJ + (item * LG + el) * kJS);
      } else {
        const int c = item - J;
        const DSlot& sl = slots[c];
        F1 cnt = {0.f};
        contact<F1>(sl, Row<F1>{Q + (sl.a * LG + el) * kQS}, Row<F1>{Q + (sl.b * LG + el) * kQS}, 1.f + H.e,
                    H.beta_over_h, H.mu, sC + (c * LG + el) * kCS, cnt);
      }
    }
  };
  auto gather = [&](int b) {
    Acc<F1> acc;
    for (int k = jinc_begin[b]; k < jinc_begin[b + 1]; ++k) {
      const int e = jinc[k];
      acc.joint(sJ + el * kJS + (e >> 4) * (LG * kJS), e);
    }
    for (int k = cinc_begin[b]; k < cinc_begin[b + 1]; ++k) {
      const int e = cinc[k];
      acc.slot(sC + el * kCS + (e >> 4) * (LG * kCS), e);
    }
    return acc;
  };
  auto fwd_integrate = [&]() {
    for (int i = bw0; i < bw1; ++i) {
      const int b = bodies_of_warp[i * G];
      if (b < 0) continue;
      Acc<F1> acc = gather(b);
      integrate<F1>(bodies[b], Row<F1>{Q + (b * LG + el) * kQS}, acc, h, H.g, false, nullptr, E);
    }
  };

  // ---- one forward sweep: the state at the start of every substep -> checkpoints (HBM)
  const int nq4 = B * E * kQS / 4;
  float4* ck = io.ckpt + int64_t(blockIdx.x) * H.S * nq4;
  for (int i = tid; i < nq4; i += nt) reinterpret_cast<float4*>(Q)[i] = reinterpret_cast<const float4*>(Q0)[i];
  __syncthreads();
  for (int k = 0; k < H.S; ++k) {
    for (int i = tid; i < nq4; i += nt) ck[int64_t(k) * nq4 + i] = reinterpret_cast<const float4*>(Q)[i];
    if (k + 1 == H.S) break;
    fwd_kin();
    __syncthreads();
    fwd_items();
    __syncthreads();
    fwd_integrate();
    __syncthreads();
  }
  __syncthreads();

  for (int s = H.S - 1; s >= 0; --s) {
    // ---- the state at the start of substep s (checkpoint), S2(s), the items of s
    for (int i = tid; i < nq4; i += nt) {
      const float4 v = ck[int64_t(s) * nq4 + i];
      reinterpret_cast<float4*>(QK)[i] = v;
      reinterpret_cast<float4*>(Q)[i] = v;
    }
    __syncthreads();
    fwd_kin();
    __syncthreads();
    fwd_items();
    __syncthreads();
    for (int i = bw0; i < bw1; ++i) {  // the summed forces / impulses and contact counts of s
      const int b = bodies_of_warp[i * G];
      if (b < 0) continue;
      const Acc<F1> acc = gather(b);
      float* fw = FW + (b * E + el) * kFS;
      fw[0] = acc.F.x.x; fw[1] = acc.F.y.x; fw[2] = acc.F.z.x; fw[3] = acc.cnt.x;
      fw[4] = acc.T.x.x; fw[5] = acc.T.y.x; fw[6] = acc.T.z.x;
      fw[8] = acc.dV.x.x; fw[9] = acc.dV.y.x; fw[10] = acc.dV.z.x;
      fw[12] = acc.dW.x.x; fw[13] = acc.dW.y.x; fw[14] = acc.dW.z.x;
    }
    __syncthreads();

    // ---- S7 + S8 adjoint (one thread per (body, env)): GQ holds ḡ(x', q', v'', ω'')
    for (int i = tid; i < B * E; i += nt) {
      const int b = i / E;
      const DBody& bd = bodies[b];
      float* fa = FA + i * kFS;
      for (int k = 0; k < 16; ++k) fa[k] = 0.f;
      if (bd.is_static) continue;
      const float* fw = FW + i * kFS;
      float* gq = GQ + i * kQS;
      const float* q = Q + i * kQS + 4;
      const bool iso = bd.flags & kFlagIso;
      const float cnt = fw[3];
      const bool hit = cnt > 0.f;
      const float ic = hit ? div_mufu(1.f, cnt) : 0.f;
      const float mic = __fmul_rn(bd.inv_mass, ic);
      float av[3], aw[3], bv[3], bw[3];
      for (int k = 0; k < 3; ++k) {
        av[k] = hit ? bd.mpos[k] * gq[8 + k] : gq[8 + k];
        aw[k] = hit ? bd.mrot[k] * gq[12 + k] : gq[12 + k];
        bv[k] = bd.mpos[k] * av[k];
        bw[k] = bd.mrot[k] * aw[k];
      }
      const Q4T<F1> qf{{q[0]}, {q[1]}, {q[2]}, {q[3]}};
      const V3T<F1> gt = iw(qf, bd.inv_inertia, iso, V3T<F1>{{bw[0]}, {bw[1]}, {bw[2]}});
      const V3T<F1> gw = iw(qf, bd.inv_inertia, iso, V3T<F1>{{aw[0]}, {aw[1]}, {aw[2]}});
      const float gtv[3] = {gt.x.x, gt.y.x, gt.z.x}, gwv[3] = {gw.x.x, gw.y.x, gw.z.x};
      for (int k = 0; k < 3; ++k) {
        fa[k] = h * bd.inv_mass * bv[k];           // ḡF
        fa[4 + k] = h * gtv[k];                    // ḡT
        fa[8 + k] = hit ? mic * av[k] : 0.f;       // ḡdV
        fa[12 + k] = hit ? ic * gwv[k] : 0.f;      // ḡdW
        gq[8 + k] = bv[k];                         // ḡv (before S7)
        gq[12 + k] = bw[k];                        // ḡω
      }
      if (!iso) {  // ∂(I_w⁻¹(q)·T)/∂q and ∂(I_w⁻¹(q)·dW)/∂q by local forward derivatives
        const V3T<D1> T{{fw[4], 0.f}, {fw[5], 0.f}, {fw[6], 0.f}}, dW{{fw[12], 0.f}, {fw[13], 0.f}, {fw[14], 0.f}};
        for (int k = 0; k < 4; ++k) {
          Q4T<D1> qd{{q[0], k == 0 ? 1.f : 0.f}, {q[1], k == 1 ? 1.f : 0.f}, {q[2], k == 2 ? 1.f : 0.f},
                     {q[3], k == 3 ? 1.f : 0.f}};
          const V3T<D1> r1 = iw(qd, bd.inv_inertia, false, T);
          float g = h * (r1.x.t * bw[0] + r1.y.t * bw[1] + r1.z.t * bw[2]);
          if (hit) {
            const V3T<D1> r2 = iw(qd, bd.inv_inertia, false, dW);
            g += ic * (r2.x.t * aw[0] + r2.y.t * aw[1] + r2.z.t * aw[2]);
          }
          gq[4 + k] += g;
        }
      }
    }
    __syncthreads();

    // ---- item adjoints (warp lane group per item, lane = env): IA[item][env][26]
    for (int it = it0; it < it1; ++it) {
      const int item = items[it * G];
      if (item < 0) continue;
      float* ia = IA + (item * E + el) * kIS;
      if (item < J) {
        const DJoint& jt = joints[item];
        const float* fc = FA + (jt.child * E + el) * kFS;
        const float* fp = FA + (jt.parent * E + el) * kFS;
        const float gF[3] = {fc[0] - fp[0], fc[1] - fp[1], fc[2] - fp[2]};
        const float* recP = Q + (jt.parent * LG + el) * kQS;
        const float* recC = Q + (jt.child * LG + el) * kQS;
        const int4 h0 = *reinterpret_cast<const int4*>(&jt), h1 = reinterpret_cast<const int4*>(&jt)[1];
        const int n_act = h0.w >= 0 ? h0.z : 0, act_off = h1.x;
        const int n_in = 26 + n_act;  // parent row 0-12, child row 13-25, the joint's actions 26-
        if (hand_adj) {
          float ga[3] = {0.f, 0.f, 0.f};
          joint_adj(jt, recP, recC, sA + el, E, gF, fc + 4, fp + 4, ia, ga);
          for (int k = 0; k < n_act; ++k) GA[(act_off + k) * E + el] += ga[k];
          continue;
        }
        for (int j0 = 0; j0 < n_in; j0 += KT) {
          const JointOut<DT> o =
              joint_f<DT>(jt, load_dt(recP, 0, j0), load_dt(recC, 13, j0),
                          [&](int k) { return mk_dt(sA[k * E + el], 26 + (k - act_off), j0); });
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            const int j = j0 + k;
            if (j >= n_in) break;
            const float g = dot_tk(o.f, gF, k) + dot_tk(o.tc, fc + 4, k) + dot_tk(o.tp, fp + 4, k);
            if (j < 26) ia[j] = g;
            else GA[(act_off + j - 26) * E + el] += g;
          }
        }
      } else {
        const DSlot& sl = slots[item - J];
        const float* fa_ = FA + (sl.a * E + el) * kFS;
        const float* fb_ = FA + (sl.b * E + el) * kFS;
        const float gP[3] = {fa_[8] - fb_[8], fa_[9] - fb_[9], fa_[10] - fb_[10]};
        const float gtb[3] = {-fb_[12], -fb_[13], -fb_[14]};
        const float* recA = Q + (sl.a * LG + el) * kQS;
        const float* recB = Q + (sl.b * LG + el) * kQS;
        if (hand_adj && contact_adj(sl, recA, recB, 1.f + H.e, H.beta_over_h, H.mu, gP, fa_ + 12, gtb, ia)) continue;
        for (int j0 = 0; j0 < 26; j0 += KT) {
          const ContactOut<DT> o =
              contact_f<DT>(sl, load_dt(recA, 0, j0), load_dt(recB, 13, j0), 1.f + H.e, H.beta_over_h, H.mu);
#pragma unroll
          for (int k = 0; k < KT; ++k)
            if (j0 + k < 26) ia[j0 + k] = dot_tk(o.P, gP, k) + dot_tk(o.ta, fa_ + 12, k) + dot_tk(o.tb, gtb, k);
        }
      }
    }
    __syncthreads();

    // ---- gather the item input adjoints onto the bodies (all bodies, fixed order)
    for (int i = tid; i < B * E; i += nt) {
      const int b = i / E, env = i - b * E;
      float* gq = GQ + i * kQS;
      auto add = [&](const float* src) {
        for (int m = 0; m < 3; ++m) gq[m] += src[m];
        for (int m = 0; m < 4; ++m) gq[4 + m] += src[3 + m];
        for (int m = 0; m < 3; ++m) gq[8 + m] += src[7 + m];
        for (int m = 0; m < 3; ++m) gq[12 + m] += src[10 + m];
      };
      for (int k = jinc_begin[b]; k < jinc_begin[b + 1]; ++k) {  // child side 4: inputs 13-25; parent 8: 0-12
        const int e = jinc[k];
        add(IA + ((e >> 4) * E + env) * kIS + ((e & 8) ? 0 : 13));
      }
      for (int k = cinc_begin[b]; k < cinc_begin[b + 1]; ++k) {  // A side 4: inputs 0-12; B side 8: 13-25
        const int e = cinc[k];
        add(IA + ((J + (e >> 4)) * E + env) * kIS + ((e & 8) ? 13 : 0));
      }
    }
    __syncthreads();

    // ---- S2 adjoint: (x', q') = K(x, q, v, ω) with the pre-S2 state in QK
    for (int i = tid; i < B * E; i += nt) {
      const int b = i / E;
      const DBody& bd = bodies[b];
      if (bd.is_static) continue;
      float* gq = GQ + i * kQS;
      const float* pre = QK + i * kQS;
      for (int k = 0; k < 3; ++k) gq[8 + k] += h * bd.mpos[k] * gq[k];  // x' = x + h·m⊙v
      if (!bd.rot_frozen && io.local_ad) {  // cross-check path: local value+tangent derivatives
        float gr[4], gw[3] = {0.f, 0.f, 0.f};
        for (int j = 0; j < 7; ++j) {
          auto t = [&](int k) { return k == j ? 1.f : 0.f; };
          Q4T<D1> qd{{pre[4], t(0)}, {pre[5], t(1)}, {pre[6], t(2)}, {pre[7], t(3)}};
          V3T<D1> wd{{pre[12], t(4)}, {pre[13], t(5)}, {pre[14], t(6)}};
          if (!(bd.flags & kFlagFreeRot)) wd = had(bd.mrot, wd);
          const Q4T<D1> qn = kin_rot(qd, wd, h);
          const float g = qn.w.t * gq[4] + qn.x.t * gq[5] + qn.y.t * gq[6] + qn.z.t * gq[7];
          if (j < 4) gr[j] = g;
          else gw[j - 4] = g;
        }
        for (int k = 0; k < 4; ++k) gq[4 + k] = gr[k];
        for (int k = 0; k < 3; ++k) gq[12 + k] += gw[k];
      } else if (!bd.rot_frozen) {
        // hand-derived adjoint of q' = normalize(p), p = q + (h/2)·(0, ω̃)⊗q, ω̃ = m⊙ω:
        // ḡp = (ḡ − q'(q'·ḡ))/|p|; p.w = q.w − (h/2) ω̃·u, p.u = u + (h/2)(q.w ω̃ + ω̃×u)
        const float hh = 0.5f * h;
        const V3f u{pre[5], pre[6], pre[7]};
        const float qw = pre[4];
        V3f w{pre[12], pre[13], pre[14]};
        if (!(bd.flags & kFlagFreeRot)) w = v3(bd.mrot[0] * w.x, bd.mrot[1] * w.y, bd.mrot[2] * w.z);
        const float pw = qw - hh * dot3(w, u);
        const V3f pu = u + hh * (qw * w + cross3(w, u));
        const float n2 = pw * pw + dot3(pu, pu);
        float inv = rsqrt_mufu(n2);
        inv = inv * (1.5f - 0.5f * n2 * inv * inv);
        const float qnw = pw * inv;
        const V3f qnu = inv * pu;
        const V3f gu_{gq[5], gq[6], gq[7]};
        const float dg = qnw * gq[4] + dot3(qnu, gu_);
        const float gpw = inv * (gq[4] - dg * qnw);
        const V3f gpu = inv * (gu_ - dg * qnu);
        const float gqw = gpw + hh * dot3(w, gpu);
        const V3f gqu = gpu - (hh * gpw) * w + hh * cross3(gpu, w);
        V3f gw = (-hh * gpw) * u + hh * (qw * gpu + cross3(u, gpu));
        if (!(bd.flags & kFlagFreeRot)) gw = v3(bd.mrot[0] * gw.x, bd.mrot[1] * gw.y, bd.mrot[2] * gw.z);
        gq[4] = gqw;
        gq[5] = gqu.x;
        gq[6] = gqu.y;
        gq[7] = gqu.z;
        gq[12] += gw.x;
        gq[13] += gw.y;
        gq[14] += gw.z;
      }
    }
    __syncthreads();
  }

  // ---- write the input cotangents
  for (int i = tid; i < B * E; i += nt) {
    const int b = i / E, env = i - b * E;
    if (env >= nvalid) continue;
    const int64_t g = e0 + env;
    const float* gq = GQ + i * kQS;
    for (int k = 0; k < 3; ++k) {
      io.opos[(g * B + b) * 3 + k] = gq[k];
      io.ovel[(g * B + b) * 3 + k] = gq[8 + k];
      io.oang[(g * B + b) * 3 + k] = gq[12 + k];
    }
    for (int k = 0; k < 4; ++k) io.orot[(g * B + b) * 4 + k] = gq[4 + k];
  }
  if (io.oact)
    for (int i = tid; i < A * E; i += nt) {
      const int k = i / E, env = i - k * E;
      if (env < nvalid) io.oact[(e0 + env) * A + k] = GA[i];
    }
}

template <int R>
cudaError_t launch_vjp_variant(const VjpArgs& ka, dim3 grid, dim3 block, size_t smem, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(brax_vjp_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  brax_vjp_kernel<R><<<grid, block, smem, stream>>>(ka);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_step_vjp_fused(const System& sys, const StepArgs& primal, const float* const g_out[4],
                                  float* const g_in[4], float* g_action, cudaStream_t stream) {
  const int64_t n = primal.n_envs;
  if (n <= 0) return cudaSuccess;
  note_other_launch(sys, stream);
  const DHeader& H = sys.hd;
  int p = -1;  // the largest one-env-per-lane block whose layout fits
  for (int q : {0, 1, 2}) {
    const VjpLayout L = vjp_layout(H.B, H.J, H.C, H.A, H.plan[q].E, H.blob_words);
    if (L.total * 4 <= kMaxDynSmem) {
      p = q;
      break;
    }
  }
  if (p < 0) return cudaErrorInvalidValue;
  const DPlan& P = H.plan[p];
  const VjpLayout L = vjp_layout(H.B, H.J, H.C, H.A, P.E, H.blob_words);
  dim3 grid(unsigned((n + P.E - 1) / P.E)), block(unsigned(P.W * 32));
  float4* ckpt = nullptr;
  const size_t ck_bytes = size_t(grid.x) * H.S * H.B * P.E * kQS * 4;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ckpt), ck_bytes, stream);
  if (e != cudaSuccess) return e;
  VjpArgs ka{{primal.pos_in, primal.rot_in, primal.vel_in, primal.ang_in, primal.actions, g_out[0], g_out[1],
              g_out[2], g_out[3], g_in[0], g_in[1], g_in[2], g_in[3], g_action, n, ckpt,
              std::getenv("BRAX_VJP_LOCAL_AD") ? 1 : 0},
             sys.d_blob, H, p};
  DPlan Pv = P;
  Pv.smem_bytes = L.total * 4;
  const int regs = choose_regs(sys, Pv, int64_t(grid.x));
  if (regs >= 255) e = launch_vjp_variant<255>(ka, grid, block, size_t(L.total) * 4, stream);
  else if (regs >= 168) e = launch_vjp_variant<168>(ka, grid, block, size_t(L.total) * 4, stream);
  else e = launch_vjp_variant<128>(ka, grid, block, size_t(L.total) * 4, stream);
  cudaError_t f = cudaFreeAsync(ckpt, stream);
  return e != cudaSuccess ? e : f;
}

}  // namespace brax
