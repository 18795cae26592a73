// config.cpp — ProtoBuf-text scene parser, schema mapping and validation.
//
// Grammar: the text subset the paper exhibits in App. A:
//   file := field* ;  field := NAME ':' scalar | NAME ':'? '{' field* '}'
// '#' comments, ',' and ';' separators are ignored.  Semantic rules (defaults,
// pair enumeration R19, forest check) follow SPEC.md:290-298 and SURVEY §8(c).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>

#include "config.h"

namespace brax {
namespace {

struct Node {
  enum Kind { kNum, kStr, kIdent, kMsg } kind = kNum;
  std::string name;
  double num = 0;
  std::string str;
  std::vector<Node> children;
  int line = 1, col = 1;
};

struct Token {
  enum Kind { kName, kNumber, kString, kPunct, kEof } kind;
  std::string text;
  int line, col;
};

[[noreturn]] void parse_error(int line, int col, const std::string& msg) {
  std::ostringstream os;
  os << line << ":" << col << ": " << msg;
  throw Error(BRAX_E_PARSE, os.str());
}

std::vector<Token> tokenize(const std::string& s) {
  std::vector<Token> out;
  size_t i = 0;
  int line = 1;
  size_t line_start = 0;
  auto isdig = [](char c) { return c >= '0' && c <= '9'; };
  while (i < s.size()) {
    char c = s[i];
    int col = int(i - line_start) + 1;
    if (c == '\n') { ++i; ++line; line_start = i; continue; }
    if (c == ' ' || c == '\t' || c == '\r' || c == ',' || c == ';') { ++i; continue; }
    if (c == '#') { while (i < s.size() && s[i] != '\n') ++i; continue; }
    if (c == '{' || c == '}' || c == ':') { out.push_back({Token::kPunct, std::string(1, c), line, col}); ++i; continue; }
    if (c == '"') {
      size_t j = i + 1;
      std::string val;
      while (j < s.size() && s[j] != '"') {
        if (s[j] == '\n') parse_error(line, col, "unterminated string");
        if (s[j] == '\\' && j + 1 < s.size()) {
          char e = s[j + 1];
          val += (e == 'n') ? '\n' : (e == 't') ? '\t' : e;
          j += 2;
        } else {
          val += s[j++];
        }
      }
      if (j >= s.size()) parse_error(line, col, "unterminated string");
      out.push_back({Token::kString, val, line, col});
      i = j + 1;
      continue;
    }
    if (isdig(c) || c == '.' || c == '-' || c == '+') {
      size_t j = i;
      if (s[j] == '-' || s[j] == '+') ++j;
      size_t digits = 0;
      while (j < s.size() && isdig(s[j])) { ++j; ++digits; }
      if (j < s.size() && s[j] == '.') {
        ++j;
        while (j < s.size() && isdig(s[j])) { ++j; ++digits; }
      }
      if (digits == 0) parse_error(line, col, std::string("unexpected character '") + c + "'");
      if (j < s.size() && (s[j] == 'e' || s[j] == 'E')) {
        size_t k = j + 1;
        if (k < s.size() && (s[k] == '-' || s[k] == '+')) ++k;
        if (k < s.size() && isdig(s[k])) {
          while (k < s.size() && isdig(s[k])) ++k;
          j = k;
        }
      }
      out.push_back({Token::kNumber, s.substr(i, j - i), line, col});
      i = j;
      continue;
    }
    if ((c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_') {
      size_t j = i;
      while (j < s.size() && ((s[j] >= 'a' && s[j] <= 'z') || (s[j] >= 'A' && s[j] <= 'Z') || s[j] == '_' ||
                              isdig(s[j])))
        ++j;
      out.push_back({Token::kName, s.substr(i, j - i), line, col});
      i = j;
      continue;
    }
    parse_error(line, col, std::string("unexpected character '") + c + "'");
  }
  out.push_back({Token::kEof, "", line, int(s.size() - line_start) + 1});
  return out;
}

struct Parser {
  std::vector<Token> t;
  size_t i = 0;
  std::vector<Node> block(bool top) {
    std::vector<Node> out;
    for (;;) {
      const Token& k = t[i];
      if (k.kind == Token::kEof) {
        if (!top) parse_error(k.line, k.col, "unexpected end of input: missing '}'");
        return out;
      }
      if (k.kind == Token::kPunct && k.text == "}") {
        if (top) parse_error(k.line, k.col, "unbalanced '}'");
        ++i;
        return out;
      }
      if (k.kind != Token::kName) parse_error(k.line, k.col, "expected field name, got '" + k.text + "'");
      Node n;
      n.name = k.text;
      n.line = k.line;
      n.col = k.col;
      ++i;
      const Token* v = &t[i];
      bool colon = v->kind == Token::kPunct && v->text == ":";
      if (colon) v = &t[++i];
      if (v->kind == Token::kPunct && v->text == "{") {
        ++i;
        n.kind = Node::kMsg;
        n.children = block(false);
      } else if (!colon) {
        parse_error(v->line, v->col, "expected ':' or '{' after '" + n.name + "'");
      } else if (v->kind == Token::kNumber) {
        n.kind = Node::kNum;
        n.num = std::strtod(v->text.c_str(), nullptr);
        ++i;
      } else if (v->kind == Token::kString) {
        n.kind = Node::kStr;
        n.str = v->text;
        ++i;
      } else if (v->kind == Token::kName) {
        n.kind = Node::kIdent;
        n.str = v->text;
        ++i;
      } else {
        parse_error(v->line, v->col, "expected value after ':', got '" + v->text + "'");
      }
      out.push_back(std::move(n));
    }
  }
};

[[noreturn]] void invalid(const std::string& path, const std::string& msg, brax_status st = BRAX_E_VALIDATION) {
  throw Error(st, path + ": " + msg);
}

// Field access with schema checking.
struct Fields {
  std::map<std::string, std::vector<const Node*>> by;
  std::string path;
  Fields(const std::vector<Node>& nodes, const std::string& p, std::initializer_list<const char*> allowed)
      : path(p) {
    std::set<std::string> ok(allowed.begin(), allowed.end());
    for (const Node& n : nodes) {
      if (!ok.count(n.name)) invalid(path + "." + n.name, "unknown field");
      by[n.name].push_back(&n);
    }
  }
  const Node* one(const std::string& key) const {
    auto it = by.find(key);
    if (it == by.end()) return nullptr;
    if (it->second.size() > 1) invalid(path + "." + key, "field given more than once");
    return it->second[0];
  }
  double num(const std::string& key, double dflt) const {
    const Node* n = one(key);
    if (!n) return dflt;
    if (n->kind != Node::kNum) invalid(path + "." + key, "expected a number");
    return n->num;
  }
  std::string str(const std::string& key, bool* present = nullptr) const {
    const Node* n = one(key);
    if (present) *present = n != nullptr;
    if (!n) return "";
    if (n->kind != Node::kStr) invalid(path + "." + key, "expected a string");
    return n->str;
  }
  const std::vector<Node>* msg(const std::string& key) const {
    const Node* n = one(key);
    if (!n) return nullptr;
    if (n->kind != Node::kMsg) invalid(path + "." + key, "expected a { } block");
    return &n->children;
  }
  std::vector<const Node*> all(const std::string& key) const {
    auto it = by.find(key);
    return it == by.end() ? std::vector<const Node*>{} : it->second;
  }
  bool has(const std::string& key) const { return by.count(key) > 0; }
};

void vec3(const std::vector<Node>* node, const std::string& path, double out[3]) {
  if (!node) return;
  for (const Node& n : *node) {
    if ((n.name != "x" && n.name != "y" && n.name != "z") || n.kind != Node::kNum)
      invalid(path + "." + n.name, "expected x/y/z numbers");
    out[n.name[0] - 'x'] = n.num;
  }
}

void qmul(const double a[4], const double b[4], double out[4]) {
  double r[4] = {a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                 a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                 a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                 a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]};
  for (int i = 0; i < 4; ++i) out[i] = r[i];
}

void euler_field(const std::vector<Node>* node, const std::string& path, double q[4]) {
  double deg[3] = {0, 0, 0};
  vec3(node, path, deg);
  euler_deg_to_quat(deg, q);
}

std::string idx(const char* what, size_t i) { return std::string(what) + "[" + std::to_string(i) + "]"; }

struct ActuatorSpec { std::string name; int joint = 0; double strength = 0; ActuatorKind kind = kTorque; std::string path; };
struct IncludeSpec { int first, second; std::string path; };

// Checks and derived tables shared by the text parser and the programmatic
// descriptors (brax_config_from_desc): the joint forest, actuators folded into
// their joints (action offsets in actuator order, dof-major), and the contact
// pair list + slot table (naive pairwise collision; rule R19).
void finalize_config(Config& c, const std::vector<ActuatorSpec>& acts, const std::vector<IncludeSpec>* include) {
  // forest: every body is the child of at most one joint, no cycles
  std::vector<int> parent_of(c.bodies.size(), -1);
  for (size_t ji = 0; ji < c.joints.size(); ++ji) {
    int ch = c.joints[ji].child;
    if (parent_of[ch] >= 0) invalid(idx("joints", ji) + ".child", "body is already the child of another joint");
    parent_of[ch] = c.joints[ji].parent;
  }
  for (size_t b = 0; b < c.bodies.size(); ++b) {
    size_t steps = 0;
    for (int x = int(b); parent_of[x] >= 0; x = parent_of[x])
      if (++steps > c.bodies.size()) invalid(idx("bodies", b), "cyclic joint graph", BRAX_E_CYCLIC_JOINT_GRAPH);
  }

  std::set<int> actuated;
  for (const ActuatorSpec& s : acts) {
    if (s.joint < 0 || s.joint >= int(c.joints.size())) invalid(s.path + ".joint", "unknown joint");
    if (actuated.count(s.joint)) invalid(s.path + ".joint", "joint already has an actuator");
    if (c.joints[s.joint].dof == 0) invalid(s.path + ".joint", "actuated joint must have dof >= 1");
    actuated.insert(s.joint);
    Actuator a;
    a.name = s.name;
    a.joint = s.joint;
    a.strength = s.strength;
    a.kind = s.kind;
    a.act_offset = c.act_dim;
    c.act_dim += c.joints[a.joint].dof;
    Joint& j = c.joints[a.joint];
    j.act_kind = a.kind;
    j.act_strength = a.strength;
    j.act_offset = a.act_offset;
    c.actuators.push_back(a);
  }

  // ---- pairs (naive pairwise collision; enumeration rule R19) ----
  struct Cand { int i, j; std::string path; };
  std::vector<Cand> cand;
  if (include) {
    for (const IncludeSpec& in : *include) {
      const int ba = in.first, bb = in.second;
      if (ba < 0 || bb < 0 || ba >= int(c.bodies.size()) || bb >= int(c.bodies.size()))
        invalid(in.path, "unknown body");
      if (ba == bb) invalid(in.path, "a body cannot collide with itself");
      if (c.bodies[ba].is_static() && c.bodies[bb].is_static()) invalid(in.path, "static-static pair");
      for (size_t i = 0; i < c.colliders.size(); ++i)
        if (c.colliders[i].body == ba)
          for (size_t j = 0; j < c.colliders.size(); ++j)
            if (c.colliders[j].body == bb) cand.push_back({int(i), int(j), in.path});
    }
  } else {
    std::set<std::pair<int, int>> jointed;
    for (const Joint& j : c.joints) {
      jointed.insert({j.parent, j.child});
      jointed.insert({j.child, j.parent});
    }
    for (size_t i = 0; i < c.colliders.size(); ++i)
      for (size_t j = i + 1; j < c.colliders.size(); ++j) {
        int bi = c.colliders[i].body, bj = c.colliders[j].body;
        if (bi == bj || jointed.count({bi, bj})) continue;
        if (c.bodies[bi].is_static() && c.bodies[bj].is_static()) continue;
        cand.push_back({int(i), int(j), "colliders[" + std::to_string(i) + "]x[" + std::to_string(j) + "]"});
      }
  }
  static const char* kind_name[] = {"sphere", "capsule", "box", "plane"};
  for (const Cand& cd : cand) {
    int a = cd.i, b = cd.j;
    int ka = c.colliders[a].kind, kb = c.colliders[b].kind;  // enum order = orientation rank
    if (ka > kb || (ka == kb && a > b)) { std::swap(a, b); std::swap(ka, kb); }
    int type = -1;
    if (kb == kPlane) type = (ka == kSphere) ? BRAX_SLOT_SPHERE_PLANE : (ka == kCapsule) ? BRAX_SLOT_CAPSULE_PLANE
                                            : (ka == kBox) ? BRAX_SLOT_BOX_PLANE : -1;
    else if (ka == kSphere && kb == kSphere) type = BRAX_SLOT_SPHERE_SPHERE;
    else if (ka == kSphere && kb == kCapsule) type = BRAX_SLOT_SPHERE_CAPSULE;
    else if (ka == kCapsule && kb == kCapsule) type = BRAX_SLOT_CAPSULE_CAPSULE;
    if (type < 0)
      invalid(cd.path, std::string("unsupported collider pair ") + kind_name[ka] + "-" + kind_name[kb],
              BRAX_E_UNSUPPORTED_PAIR);
    c.pairs.push_back({a, b, type});
  }
  for (size_t pi = 0; pi < c.pairs.size(); ++pi) {
    const Pair& pr = c.pairs[pi];
    const Collider& A = c.colliders[pr.col_a];
    int first = 0, count = 1;
    if (pr.type == BRAX_SLOT_CAPSULE_PLANE) {
      if (A.end == 0) count = 2;
      else first = (A.end == 1) ? 0 : 1;
    } else if (pr.type == BRAX_SLOT_BOX_PLANE) {
      count = 8;
    }
    for (int k = 0; k < count; ++k)
      c.slots.push_back({int(pi), pr.type, A.body, c.colliders[pr.col_b].body, pr.col_a, pr.col_b, first + k});
  }
  if (c.slots.size() > 255) invalid("config", "more than 255 contact slots");
}

}  // namespace

void euler_deg_to_quat(const double deg[3], double q[4]) {
  const double k = M_PI / 180.0;
  double qx[4] = {std::cos(deg[0] * k / 2), std::sin(deg[0] * k / 2), 0, 0};
  double qy[4] = {std::cos(deg[1] * k / 2), 0, std::sin(deg[1] * k / 2), 0};
  double qz[4] = {std::cos(deg[2] * k / 2), 0, 0, std::sin(deg[2] * k / 2)};
  double t[4];
  qmul(qx, qy, t);
  qmul(t, qz, q);
}

Config parse_config(const std::string& text) {
  Parser p{tokenize(text)};
  std::vector<Node> root = p.block(true);
  Fields top(root, "config", {"dt", "substeps", "gravity", "friction", "elasticity", "baumgarte_erp", "bodies",
                              "joints", "actuators", "collide_include", "defaults", "task"});
  Config c;
  c.dt = top.num("dt", 0.01);
  double sub = top.num("substeps", 1.0);
  if (!(c.dt > 0)) invalid("config.dt", "must be > 0");
  if (sub != std::floor(sub) || sub < 1) invalid("config.substeps", "must be a positive integer");
  c.substeps = int(sub);
  vec3(top.msg("gravity"), "config.gravity", c.gravity);
  c.friction = top.num("friction", 1.0);
  c.elasticity = top.num("elasticity", 0.0);
  c.baumgarte = top.num("baumgarte_erp", 0.2);
  if (c.friction < 0) invalid("config.friction", "must be >= 0");
  if (!(c.elasticity >= 0 && c.elasticity <= 1)) invalid("config.elasticity", "must be in [0, 1]");
  if (!(c.baumgarte > 0 && c.baumgarte <= 1)) invalid("config.baumgarte_erp", "must be in (0, 1]");

  std::map<std::string, int> body_ix;
  auto bnodes = top.all("bodies");
  for (size_t bi = 0; bi < bnodes.size(); ++bi) {
    std::string path = idx("bodies", bi);
    if (bnodes[bi]->kind != Node::kMsg) invalid(path, "expected a { } block");
    Fields bf(bnodes[bi]->children, path, {"name", "mass", "inertia", "frozen", "colliders"});
    Body b;
    bool has_name = false;
    b.name = bf.str("name", &has_name);
    if (!has_name) invalid(path + ".name", "required");
    if (body_ix.count(b.name)) invalid(path + ".name", "duplicate body name '" + b.name + "'");
    body_ix[b.name] = int(bi);
    b.mass = bf.num("mass", 1.0);
    if (!(b.mass > 0)) invalid(path + ".mass", "must be > 0");
    vec3(bf.msg("inertia"), path + ".inertia", b.inertia);
    for (double v : b.inertia)
      if (!(v > 0)) invalid(path + ".inertia", "must be > 0");
    if (const std::vector<Node>* fz = bf.msg("frozen")) {
      Fields ff(*fz, path + ".frozen", {"position", "rotation", "all"});
      if (const Node* a = ff.one("all")) {
        if (a->kind == Node::kIdent && a->str == "true")
          for (int k = 0; k < 3; ++k) b.frozen_pos[k] = b.frozen_rot[k] = 1;
      }
      double fp[3] = {0, 0, 0}, fr[3] = {0, 0, 0};
      vec3(ff.msg("position"), path + ".frozen.position", fp);
      vec3(ff.msg("rotation"), path + ".frozen.rotation", fr);
      for (int k = 0; k < 3; ++k) {
        if ((fp[k] != 0 && fp[k] != 1) || (fr[k] != 0 && fr[k] != 1))
          invalid(path + ".frozen", "axis flags must be 0 or 1");
        b.frozen_pos[k] = std::max(b.frozen_pos[k], fp[k]);
        b.frozen_rot[k] = std::max(b.frozen_rot[k], fr[k]);
      }
    }
    auto cnodes = bf.all("colliders");
    for (size_t ci = 0; ci < cnodes.size(); ++ci) {
      std::string cpath = path + "." + idx("colliders", ci);
      if (cnodes[ci]->kind != Node::kMsg) invalid(cpath, "expected a { } block");
      Fields cf(cnodes[ci]->children, cpath, {"position", "rotation", "sphere", "capsule", "box", "plane"});
      int nshape = cf.has("sphere") + cf.has("capsule") + cf.has("box") + cf.has("plane");
      if (nshape != 1) invalid(cpath, "exactly one of sphere/capsule/box/plane required");
      Collider col;
      col.body = int(bi);
      vec3(cf.msg("position"), cpath + ".position", col.pos);
      euler_field(cf.msg("rotation"), cpath + ".rotation", col.rot);
      if (cf.has("sphere")) {
        Fields sf(*cf.msg("sphere"), cpath + ".sphere", {"radius"});
        col.kind = kSphere;
        col.radius = sf.num("radius", 0);
        if (!(col.radius > 0)) invalid(cpath + ".sphere.radius", "must be > 0");
      } else if (cf.has("capsule")) {
        Fields sf(*cf.msg("capsule"), cpath + ".capsule", {"radius", "length", "end"});
        col.kind = kCapsule;
        col.radius = sf.num("radius", 0);
        col.length = sf.num("length", 0);
        double end = sf.num("end", 0);
        if (!(col.radius > 0)) invalid(cpath + ".capsule.radius", "must be > 0");
        if (!(col.length >= 2 * col.radius)) invalid(cpath + ".capsule.length", "must be >= 2*radius");
        if (end != 0 && end != 1 && end != -1) invalid(cpath + ".capsule.end", "must be -1, 0 or 1");
        col.end = int(end);
      } else if (cf.has("box")) {
        Fields sf(*cf.msg("box"), cpath + ".box", {"halfsize"});
        col.kind = kBox;
        vec3(sf.msg("halfsize"), cpath + ".box.halfsize", col.halfsize);
        for (double v : col.halfsize)
          if (!(v > 0)) invalid(cpath + ".box.halfsize", "must be > 0");
      } else {
        Fields sf(*cf.msg("plane"), cpath + ".plane", {});
        col.kind = kPlane;
      }
      c.colliders.push_back(col);
    }
    c.bodies.push_back(b);
  }
  if (c.bodies.empty()) invalid("config.bodies", "no bodies");

  auto dnodes = top.all("defaults");
  for (size_t di = 0; di < dnodes.size(); ++di) {
    std::string dpath = idx("defaults", di);
    Fields df(dnodes[di]->children, dpath, {"qps"});
    auto qn = df.all("qps");
    for (size_t qi = 0; qi < qn.size(); ++qi) {
      std::string qpath = dpath + "." + idx("qps", qi);
      Fields qf(qn[qi]->children, qpath, {"name", "pos", "rot"});
      std::string nm = qf.str("name");
      if (!body_ix.count(nm)) invalid(qpath + ".name", "unknown body '" + nm + "'");
      Body& b = c.bodies[body_ix[nm]];
      b.init_pos[0] = b.init_pos[1] = b.init_pos[2] = 0;
      vec3(qf.msg("pos"), qpath + ".pos", b.init_pos);
      euler_field(qf.msg("rot"), qpath + ".rot", b.init_rot);
    }
  }

  std::map<std::string, int> joint_ix;
  auto jnodes = top.all("joints");
  for (size_t ji = 0; ji < jnodes.size(); ++ji) {
    std::string path = idx("joints", ji);
    Fields jf(jnodes[ji]->children, path,
              {"name", "parent", "child", "stiffness", "spring_damping", "angular_damping", "limit_stiffness",
               "angular_stiffness", "parent_offset", "child_offset", "rotation", "reference_rotation",
               "angle_limit"});
    Joint j;
    bool has_name = false;
    j.name = jf.str("name", &has_name);
    if (!has_name) invalid(path + ".name", "required");
    if (joint_ix.count(j.name)) invalid(path + ".name", "duplicate joint name '" + j.name + "'");
    joint_ix[j.name] = int(ji);
    std::string pn = jf.str("parent"), cn = jf.str("child");
    if (!body_ix.count(pn)) invalid(path + ".parent", "unknown body '" + pn + "'");
    if (!body_ix.count(cn)) invalid(path + ".child", "unknown body '" + cn + "'");
    if (pn == cn) invalid(path + ".child", "parent and child must differ");
    j.parent = body_ix[pn];
    j.child = body_ix[cn];
    j.stiffness = jf.num("stiffness", 0);
    if (!(j.stiffness > 0)) invalid(path + ".stiffness", "must be > 0");
    j.spring_damping = jf.num("spring_damping", 0);
    j.angular_damping = jf.num("angular_damping", 0);
    j.limit_stiffness = jf.num("limit_stiffness", j.stiffness);    // R8
    j.angular_stiffness = jf.num("angular_stiffness", j.stiffness);
    vec3(jf.msg("parent_offset"), path + ".parent_offset", j.parent_offset);
    vec3(jf.msg("child_offset"), path + ".child_offset", j.child_offset);
    euler_field(jf.msg("rotation"), path + ".rotation", j.rotation);
    euler_field(jf.msg("reference_rotation"), path + ".reference_rotation", j.reference_rotation);
    auto lnodes = jf.all("angle_limit");
    for (size_t li = 0; li < lnodes.size(); ++li) {
      std::string lpath = path + "." + idx("angle_limit", li);
      Fields lf(lnodes[li]->children, lpath, {"min", "max"});
      double lo = lf.num("min", 0), hi = lf.num("max", 0);
      if (lo > hi) invalid(lpath, "min > max");
      if (lo < -180 || hi > 180) invalid(lpath, "limits must lie in [-180, 180] degrees (R9)");
      if (li < 3) {
        j.lo[li] = lo * M_PI / 180.0;
        j.hi[li] = hi * M_PI / 180.0;
      }
    }
    if (lnodes.size() > 3) invalid(path + ".angle_limit", "at most 3 (dof <= 3)");
    j.dof = int(lnodes.size());
    const char* nonneg[] = {"spring_damping", "angular_damping", "limit_stiffness", "angular_stiffness"};
    double vals[] = {j.spring_damping, j.angular_damping, j.limit_stiffness, j.angular_stiffness};
    for (int k = 0; k < 4; ++k)
      if (vals[k] < 0) invalid(path + "." + nonneg[k], "must be >= 0");
    c.joints.push_back(j);
  }

  // actuators and collide_include pairs (resolved by name), then the shared checks
  std::vector<ActuatorSpec> acts;
  auto anodes = top.all("actuators");
  for (size_t ai = 0; ai < anodes.size(); ++ai) {
    std::string path = idx("actuators", ai);
    Fields af(anodes[ai]->children, path, {"name", "joint", "strength", "torque", "angle"});
    ActuatorSpec a;
    a.name = af.str("name");
    std::string jn = af.str("joint");
    if (!joint_ix.count(jn)) invalid(path + ".joint", "unknown joint '" + jn + "'");
    if (af.has("torque") + af.has("angle") != 1) invalid(path, "exactly one of torque/angle required");
    a.joint = joint_ix[jn];
    a.strength = af.num("strength", 0);
    a.kind = af.has("torque") ? kTorque : kAngle;
    a.path = path;
    acts.push_back(a);
  }
  std::vector<IncludeSpec> inc;
  auto inodes = top.all("collide_include");
  for (size_t ii = 0; ii < inodes.size(); ++ii) {
    std::string path = idx("collide_include", ii);
    Fields f(inodes[ii]->children, path, {"first", "second"});
    std::string a = f.str("first"), b = f.str("second");
    if (!body_ix.count(a)) invalid(path + ".first", "unknown body '" + a + "'");
    if (!body_ix.count(b)) invalid(path + ".second", "unknown body '" + b + "'");
    inc.push_back({body_ix[a], body_ix[b], path});
  }
  finalize_config(c, acts, inodes.empty() ? nullptr : &inc);
  if (const std::vector<Node>* tn = top.msg("task")) {
    const std::string path = "config.task";
    Fields tf(*tn, path, {"torso", "forward", "survive_reward", "ctrl_cost", "healthy_z", "episode_length",
                          "contact_obs", "reset_noise", "goal"});
    Task& t = c.task;
    t.present = true;
    bool has = false;
    const std::string torso = tf.str("torso", &has);
    if (!has) invalid(path + ".torso", "required");
    if (!body_ix.count(torso)) invalid(path + ".torso", "unknown body '" + torso + "'");
    t.torso = body_ix[torso];
    if (c.bodies[t.torso].is_static()) invalid(path + ".torso", "must not be a static body");
    if (const std::vector<Node>* f = tf.msg("forward")) {
      t.forward[0] = t.forward[1] = t.forward[2] = 0;
      vec3(f, path + ".forward", t.forward);
    }
    if (t.forward[0] == 0 && t.forward[1] == 0 && t.forward[2] == 0) invalid(path + ".forward", "must be nonzero");
    t.survive_reward = tf.num("survive_reward", 1.0);
    t.ctrl_cost = tf.num("ctrl_cost", 0.5);
    if (t.ctrl_cost < 0) invalid(path + ".ctrl_cost", "must be >= 0");
    if (const std::vector<Node>* hz = tf.msg("healthy_z")) {
      Fields hf(*hz, path + ".healthy_z", {"min", "max"});
      if (!hf.has("min") || !hf.has("max")) invalid(path + ".healthy_z", "needs min < max");
      t.z_lo = hf.num("min", 0);
      t.z_hi = hf.num("max", 0);
      if (!(t.z_lo < t.z_hi)) invalid(path + ".healthy_z", "needs min < max");
      t.has_healthy = true;
    }
    const double L = tf.num("episode_length", 1000.0);
    if (L != std::floor(L) || L < 1 || L > 2147483647.0) invalid(path + ".episode_length", "must be a positive integer");
    t.episode_length = int(L);
    if (const Node* co = tf.one("contact_obs")) {
      if (co->kind != Node::kIdent || (co->str != "true" && co->str != "false"))
        invalid(path + ".contact_obs", "expected true or false");
      t.contact_obs = co->str == "true";
    }
    if (const std::vector<Node>* rn = tf.msg("reset_noise")) {
      Fields rf(*rn, path + ".reset_noise", {"vel", "ang"});
      t.noise_vel = rf.num("vel", 0.1);
      t.noise_ang = rf.num("ang", 0.1);
    }
    if (t.noise_vel < 0 || t.noise_ang < 0) invalid(path + ".reset_noise", "must be >= 0");
    if (const std::vector<Node>* gn = tf.msg("goal")) {  // R36
      const std::string gp = path + ".goal";
      Fields gf(*gn, gp, {"object", "target", "radius", "bonus", "range"});
      int ix[2];
      const char* keys[2] = {"object", "target"};
      for (int k = 0; k < 2; ++k) {
        bool has_k = false;
        const std::string nm = gf.str(keys[k], &has_k);
        if (!has_k) invalid(gp + "." + keys[k], "required");
        if (!body_ix.count(nm)) invalid(gp + "." + keys[k], "unknown body '" + nm + "'");
        ix[k] = body_ix[nm];
      }
      t.has_goal = true;
      t.obj = ix[0];
      t.target = ix[1];
      if (c.bodies[t.obj].is_static()) invalid(gp + ".object", "must not be a static body");
      if (!c.bodies[t.target].is_static()) invalid(gp + ".target", "must be a frozen { all: true } marker body");
      for (const Collider& col : c.colliders)
        if (col.body == t.target) invalid(gp + ".target", "must have no colliders");
      if (!gf.has("radius")) invalid(gp + ".radius", "must be > 0");
      t.radius = gf.num("radius", 0);
      if (!(t.radius > 0)) invalid(gp + ".radius", "must be > 0");
      t.bonus = gf.num("bonus", 0);
      if (const std::vector<Node>* rg = gf.msg("range")) vec3(rg, gp + ".range", t.range);
      if (t.range[0] < 0 || t.range[1] < 0 || t.range[2] < 0) invalid(gp + ".range", "must be >= 0");
    }
  }
  return c;
}

// Programmatic construction ("define systems programmatically"; the
// App. A listing at): the same Config the text parser yields, from
// plain C descriptors.  Quaternions (w, x, y, z) instead of Euler degrees, limits in
// radians; the numeric checks are the text parser's, the structural ones shared.
Config config_from_desc(const brax_config_desc& d) {
  auto finite = [](const double* v, int n) {
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(v[i])) return false;
    return true;
  };
  auto unit_quat = [&](const double* q, const std::string& path, double out[4]) {
    if (!finite(q, 4)) invalid(path, "must be finite");
    const double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(std::fabs(n - 1.0) <= 1e-6)) invalid(path, "must be a unit quaternion (w, x, y, z)");
    for (int k = 0; k < 4; ++k) out[k] = q[k];
  };
  Config c;
  c.dt = d.dt;
  if (!(c.dt > 0)) invalid("config.dt", "must be > 0");
  if (d.substeps < 1) invalid("config.substeps", "must be a positive integer");
  c.substeps = d.substeps;
  if (!finite(d.gravity, 3)) invalid("config.gravity", "must be finite");
  for (int k = 0; k < 3; ++k) c.gravity[k] = d.gravity[k];
  c.friction = d.friction;
  c.elasticity = d.elasticity;
  c.baumgarte = d.baumgarte_erp;
  if (!(c.friction >= 0)) invalid("config.friction", "must be >= 0");
  if (!(c.elasticity >= 0 && c.elasticity <= 1)) invalid("config.elasticity", "must be in [0, 1]");
  if (!(c.baumgarte > 0 && c.baumgarte <= 1)) invalid("config.baumgarte_erp", "must be in (0, 1]");
  if (d.n_bodies <= 0 || !d.bodies) invalid("config.bodies", "no bodies");
  if (d.n_joints < 0 || d.n_actuators < 0 || d.n_colliders < 0 || d.n_pairs < 0)
    invalid("config", "negative count");
  if ((d.n_joints && !d.joints) || (d.n_actuators && !d.actuators) || (d.n_colliders && !d.colliders))
    invalid("config", "NULL array with a nonzero count");
  std::set<std::string> names;
  for (int bi = 0; bi < d.n_bodies; ++bi) {
    const brax_body_desc& bd = d.bodies[bi];
    const std::string path = idx("bodies", size_t(bi));
    Body b;
    b.name = bd.name ? bd.name : ("body" + std::to_string(bi));
    if (bd.name && !names.insert(b.name).second) invalid(path + ".name", "duplicate body name '" + b.name + "'");
    b.mass = bd.mass;
    if (!(b.mass > 0)) invalid(path + ".mass", "must be > 0");
    for (int k = 0; k < 3; ++k) {
      b.inertia[k] = bd.inertia[k];
      if (!(b.inertia[k] > 0)) invalid(path + ".inertia", "must be > 0");
      if ((bd.frozen_pos[k] != 0 && bd.frozen_pos[k] != 1) || (bd.frozen_rot[k] != 0 && bd.frozen_rot[k] != 1))
        invalid(path + ".frozen", "axis flags must be 0 or 1");
      b.frozen_pos[k] = bd.frozen_pos[k];
      b.frozen_rot[k] = bd.frozen_rot[k];
    }
    if (!finite(bd.init_pos, 3)) invalid(path + ".init_pos", "must be finite");
    for (int k = 0; k < 3; ++k) b.init_pos[k] = bd.init_pos[k];
    unit_quat(bd.init_rot, path + ".init_rot", b.init_rot);
    c.bodies.push_back(b);
  }
  // colliders: global order = body order, then the descriptor order within a body
  // (the text format's order, so both forms enumerate the same slots)
  std::vector<int> corder(size_t(d.n_colliders));
  for (int i = 0; i < d.n_colliders; ++i) corder[size_t(i)] = i;
  for (int i = 0; i < d.n_colliders; ++i)
    if (d.colliders[i].body < 0 || d.colliders[i].body >= d.n_bodies)
      invalid(idx("colliders", size_t(i)) + ".body", "out of range");
  std::stable_sort(corder.begin(), corder.end(),
                   [&](int x, int y) { return d.colliders[x].body < d.colliders[y].body; });
  for (int i : corder) {
    const brax_collider_desc& cd = d.colliders[i];
    const std::string path = idx("colliders", size_t(i));
    Collider col;
    col.body = cd.body;
    if (!finite(cd.pos, 3)) invalid(path + ".pos", "must be finite");
    for (int k = 0; k < 3; ++k) col.pos[k] = cd.pos[k];
    unit_quat(cd.rot, path + ".rot", col.rot);
    switch (cd.shape) {
      case BRAX_SHAPE_SPHERE:
        col.kind = kSphere;
        col.radius = cd.radius;
        if (!(col.radius > 0)) invalid(path + ".radius", "must be > 0");
        break;
      case BRAX_SHAPE_CAPSULE:
        col.kind = kCapsule;
        col.radius = cd.radius;
        col.length = cd.length;
        if (!(col.radius > 0)) invalid(path + ".radius", "must be > 0");
        if (!(col.length >= 2 * col.radius)) invalid(path + ".length", "must be >= 2*radius");
        if (cd.capsule_end != 0 && cd.capsule_end != 1 && cd.capsule_end != -1)
          invalid(path + ".capsule_end", "must be -1, 0 or 1");
        col.end = cd.capsule_end;
        break;
      case BRAX_SHAPE_BOX:
        col.kind = kBox;
        for (int k = 0; k < 3; ++k) {
          col.halfsize[k] = cd.halfsize[k];
          if (!(col.halfsize[k] > 0)) invalid(path + ".halfsize", "must be > 0");
        }
        break;
      case BRAX_SHAPE_PLANE:
        col.kind = kPlane;
        break;
      default:
        invalid(path + ".shape", "unknown shape");
    }
    c.colliders.push_back(col);
  }
  std::set<std::string> jnames;
  for (int ji = 0; ji < d.n_joints; ++ji) {
    const brax_joint_desc& jd = d.joints[ji];
    const std::string path = idx("joints", size_t(ji));
    Joint j;
    j.name = jd.name ? jd.name : ("joint" + std::to_string(ji));
    if (jd.name && !jnames.insert(j.name).second) invalid(path + ".name", "duplicate joint name '" + j.name + "'");
    if (jd.parent < 0 || jd.parent >= d.n_bodies) invalid(path + ".parent", "out of range");
    if (jd.child < 0 || jd.child >= d.n_bodies) invalid(path + ".child", "out of range");
    if (jd.parent == jd.child) invalid(path + ".child", "parent and child must differ");
    j.parent = jd.parent;
    j.child = jd.child;
    j.stiffness = jd.stiffness;
    if (!(j.stiffness > 0)) invalid(path + ".stiffness", "must be > 0");
    j.spring_damping = jd.spring_damping;
    j.angular_damping = jd.angular_damping;
    j.limit_stiffness = jd.limit_stiffness < 0 ? j.stiffness : jd.limit_stiffness;  // R8 (negative = default)
    j.angular_stiffness = jd.angular_stiffness < 0 ? j.stiffness : jd.angular_stiffness;
    if (!(j.spring_damping >= 0)) invalid(path + ".spring_damping", "must be >= 0");
    if (!(j.angular_damping >= 0)) invalid(path + ".angular_damping", "must be >= 0");
    if (!finite(jd.parent_offset, 3) || !finite(jd.child_offset, 3)) invalid(path, "offsets must be finite");
    for (int k = 0; k < 3; ++k) {
      j.parent_offset[k] = jd.parent_offset[k];
      j.child_offset[k] = jd.child_offset[k];
    }
    unit_quat(jd.rotation, path + ".rotation", j.rotation);
    unit_quat(jd.reference_rotation, path + ".reference_rotation", j.reference_rotation);
    if (jd.dof < 0 || jd.dof > 3) invalid(path + ".dof", "must be 0..3");
    j.dof = jd.dof;
    for (int k = 0; k < j.dof; ++k) {
      if (!(jd.limit_lo[k] <= jd.limit_hi[k])) invalid(path + ".limit", "min > max");
      if (jd.limit_lo[k] < -M_PI - 1e-12 || jd.limit_hi[k] > M_PI + 1e-12)
        invalid(path + ".limit", "limits must lie in [-pi, pi] (R9)");
      j.lo[k] = jd.limit_lo[k];
      j.hi[k] = jd.limit_hi[k];
    }
    c.joints.push_back(j);
  }
  std::vector<ActuatorSpec> acts;
  for (int ai = 0; ai < d.n_actuators; ++ai) {
    const brax_actuator_desc& ad = d.actuators[ai];
    ActuatorSpec a;
    a.path = idx("actuators", size_t(ai));
    a.name = ad.name ? ad.name : ("actuator" + std::to_string(ai));
    a.joint = ad.joint;
    if (ad.kind != BRAX_ACTUATOR_TORQUE && ad.kind != BRAX_ACTUATOR_ANGLE) invalid(a.path + ".kind", "unknown kind");
    a.kind = ad.kind == BRAX_ACTUATOR_TORQUE ? kTorque : kAngle;
    a.strength = ad.strength;
    acts.push_back(a);
  }
  std::vector<IncludeSpec> inc;
  if (d.pairs)
    for (int pi = 0; pi < d.n_pairs; ++pi) inc.push_back({d.pairs[pi].first, d.pairs[pi].second, idx("pairs", size_t(pi))});
  finalize_config(c, acts, d.pairs ? &inc : nullptr);
  return c;
}

}  // namespace brax
