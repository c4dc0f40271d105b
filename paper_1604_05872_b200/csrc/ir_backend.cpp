// ir_backend.cpp -- femopt kernel IR -> sm_100a kernel, behind the C ABI
// (the GPU counterpart of the reference's only backend,
// emit_c, /root/reference/proj/src/emit_c.cpp:108-174).
//
// femgpu_ir_create parses a femopt kernel IR (the JSON of proj/README.md:68-100:
// flat statements with levels, or the nested body femopt's to_json writes),
// generates CUDA C for it and compiles it with NVRTC for sm_100a; launches go
// through the CUDA runtime's library API.  The generated code:
//
//   * maps the order-free element loop onto the grid -- one thread per cell, or
//     one warp per cell with the output rows spread over the lanes and
//     accumulated in registers (warp whenever the row loop has >= 8 rows; both exact);
//   * prints every expression exactly as emit_c prints it (precedence-driven,
//     nested sums and products flattened, emit_c.cpp:47-80) and is compiled
//     with --fmad=false, so it performs femopt's emitted arithmetic operation
//     for operation: results are bit-identical to femopt's emitted C compiled
//     with -ffp-contract=off (tests/test_emit_cuda.py, golden IRs made by the
//     reference itself);
//   * keeps emit_c's calling convention: outputs, input tables, constants,
//     each group sorted by name (emit_c.cpp:137-140); pre-evaluated tables are
//     baked into the module; outputs are accumulated with += (:91-92,129).
//
// NVRTC is loaded with dlopen on first use, so libfemgpu does not depend on it
// unless this backend is used.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/femgpu.h"
#include "femgpu_internal.h"

namespace irgen {

struct IRError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ----------------------------------------------------------------------------
// minimal JSON
// ----------------------------------------------------------------------------
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& k) const {
    const Json* j = get(k);
    if (!j) throw IRError("IR: missing key '" + k + "'");
    return *j;
  }
};

struct Parser {
  const char* p;
  const char* end;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
  }
  [[noreturn]] void fail(const char* what) { throw IRError(std::string("IR JSON: ") + what); }
  Json value() {
    ws();
    if (p >= end) fail("unexpected end");
    Json j;
    const char c = *p;
    if (c == '{') {
      ++p;
      j.kind = Json::Obj;
      ws();
      if (p < end && *p == '}') { ++p; return j; }
      for (;;) {
        ws();
        Json k = value();
        if (k.kind != Json::Str) fail("object key");
        ws();
        if (p >= end || *p != ':') fail("':'");
        ++p;
        j.obj.emplace_back(k.str, value());
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == '}') { ++p; return j; }
        fail("',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      j.kind = Json::Arr;
      ws();
      if (p < end && *p == ']') { ++p; return j; }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == ']') { ++p; return j; }
        fail("',' or ']'");
      }
    }
    if (c == '"') {
      ++p;
      j.kind = Json::Str;
      while (p < end && *p != '"') {
        if (*p == '\\') {
          ++p;
          if (p >= end) fail("escape");
          const char e = *p;
          j.str += e == 'n' ? '\n' : e == 't' ? '\t' : e;
        } else {
          j.str += *p;
        }
        ++p;
      }
      if (p >= end) fail("unterminated string");
      ++p;
      return j;
    }
    if (!strncmp(p, "true", 4)) { p += 4; j.kind = Json::Bool; j.b = true; return j; }
    if (!strncmp(p, "false", 5)) { p += 5; j.kind = Json::Bool; return j; }
    if (!strncmp(p, "null", 4)) { p += 4; return j; }
    char* q = nullptr;
    j.num = strtod(p, &q);
    if (q == p) fail("value");
    p = q;
    j.kind = Json::Num;
    return j;
  }
};

Json parse(const char* text) {
  Parser ps{text, text + strlen(text)};
  Json j = ps.value();
  ps.ws();
  if (ps.p != ps.end) ps.fail("trailing characters");
  return j;
}

// ----------------------------------------------------------------------------
// IR tree
// ----------------------------------------------------------------------------
struct Node {
  bool loop = false;
  std::string index, cls, name, op;  // loop: index/cls; stmt: name/op
  long begin = 0, end = 0;
  std::vector<Node> body;
  std::vector<std::string> idx;  // stmt lhs subscripts
  const Json* rhs = nullptr;
};

[[noreturn]] void irfail(const std::string& m) { throw IRError("IR: " + m); }

Node stmt_node(const Json& st) {
  Node n;
  const Json& lhs = st.at("lhs");
  if (lhs.kind == Json::Str) {
    n.name = lhs.str;
  } else {
    if (lhs.kind != Json::Arr || lhs.arr.empty()) irfail("bad lhs");
    n.name = lhs.arr[0].str;
    for (size_t i = 1; i < lhs.arr.size(); ++i) n.idx.push_back(lhs.arr[i].str);
  }
  const Json* op = st.get("op");
  n.op = op ? op->str : "=";
  n.rhs = &st.at("rhs");
  return n;
}

std::vector<Node> from_nested(const Json& nodes, const std::map<std::string, long>& ext) {
  std::vector<Node> out;
  for (const Json& n : nodes.arr) {
    const Json* L = n.get("loop");
    if (!L && n.get("body") && n.get("index")) L = &n;
    if (L) {
      Node x;
      x.loop = true;
      x.index = L->at("index").str;
      const Json* c = L->get("class");
      if (c && c->kind == Json::Str) x.cls = c->str;
      const Json* b = L->get("begin");
      const Json* e = L->get("end");
      x.begin = b ? (long)b->num : 0;
      x.end = e ? (long)e->num : ext.at(x.index);
      x.body = from_nested(L->at("body"), ext);
      out.push_back(std::move(x));
    } else {
      out.push_back(stmt_node(n));
    }
  }
  return out;
}

std::vector<Node> build_tree(const Json& ir, const std::map<std::string, long>& ext) {
  if (ir.get("body")) return from_nested(ir.at("body"), ext);
  std::vector<std::string> loops;
  std::map<std::string, std::string> classes;
  for (const Json& L : ir.at("loops").arr) {
    loops.push_back(L.at("index").str);
    const Json* c = L.get("class");
    if (c && c->kind == Json::Str) classes[loops.back()] = c->str;
  }
  std::vector<Node> root;
  std::vector<std::vector<Node>*> stack{&root};
  for (const Json& st : ir.at("statements").arr) {
    if (st.get("body") && st.get("index")) {
      Json wrap;
      wrap.kind = Json::Arr;
      wrap.arr.push_back(st);
      auto v = from_nested(wrap, ext);
      stack.back()->push_back(std::move(v[0]));
      continue;
    }
    const long level = (long)st.at("level").num;
    if (level > (long)loops.size()) irfail("statement level exceeds the loop nest");
    while ((long)stack.size() - 1 > level) stack.pop_back();
    while ((long)stack.size() - 1 < level) {
      Node x;
      x.loop = true;
      x.index = loops[stack.size() - 1];
      x.cls = classes.count(x.index) ? classes[x.index] : "";
      x.begin = 0;
      x.end = ext.at(x.index);
      stack.back()->push_back(std::move(x));
      stack.push_back(&stack.back()->back().body);
    }
    stack.back()->push_back(stmt_node(st));
  }
  return root;
}

// ----------------------------------------------------------------------------
// code generation
// ----------------------------------------------------------------------------
std::string lit(double x) {
  char buf[64];
  if (x == 0.0) return "0.0";
  if (std::isfinite(x) && x == std::floor(x) && std::fabs(x) < 4503599627370496.0) {
    snprintf(buf, sizeof buf, "%.1f", x);
    return buf;
  }
  snprintf(buf, sizeof buf, "%a", x);
  return buf;
}

bool ident_ok(const std::string& s) {
  if (s.empty() || !(isalpha((unsigned char)s[0]) || s[0] == '_')) return false;
  for (char c : s)
    if (!(isalnum((unsigned char)c) || c == '_')) return false;
  return true;
}
const std::string& ident(const std::string& s) {
  if (!ident_ok(s)) irfail("bad name '" + s + "'");
  return s;
}

const std::map<std::string, std::string>& calls() {
  static const std::map<std::string, std::string> m = {
      {"fabs", "fabs"}, {"sqrt", "sqrt"}, {"exp", "exp"},   {"log", "log"},   {"pow", "pow"},
      {"sin", "sin"},   {"cos", "cos"},   {"tan", "tan"},   {"atan", "atan"}, {"atan2", "atan2"},
      {"cbrt", "cbrt"}, {"fmin", "fmin"}, {"fmax", "fmax"}, {"abs", "fabs"}};
  return m;
}

long ops(const Json& x) {
  if (x.kind == Json::Arr && !x.arr.empty() && x.arr[0].kind == Json::Str) {
    const std::string& op = x.arr[0].str;
    if (op == "+" || op == "*" || op == "/" || op == "call") {
      long s = std::max<long>(1, (long)x.arr.size() - 2);
      for (size_t i = 1; i < x.arr.size(); ++i) s += ops(x.arr[i]);
      return s;
    }
  }
  return 0;
}

void op_counts(const std::vector<Node>& nodes, double mult, bool inJ, const std::string& J,
               double tot[2]) {
  for (const Node& n : nodes) {
    if (n.loop) {
      if (n.cls == "orderfree")
        op_counts(n.body, mult, inJ, J, tot);
      else
        op_counts(n.body, mult * std::max<long>(0, n.end - n.begin), inJ || n.index == J, J, tot);
    } else {
      tot[inJ ? 1 : 0] += mult * (1 + ops(*n.rhs));
    }
  }
}

void names_in(const Json& x, std::set<std::string>& acc) {
  if (x.kind == Json::Str) {
    acc.insert(x.str);
  } else if (x.kind == Json::Arr && !x.arr.empty()) {
    if (x.arr[0].kind == Json::Str && x.arr[0].str == "sym" && x.arr.size() > 1)
      acc.insert(x.arr[1].str);
    for (size_t i = 1; i < x.arr.size(); ++i) names_in(x.arr[i], acc);
  }
}

struct Emitter {
  std::map<std::string, long> ext;
  std::map<std::string, std::vector<std::string>> dims;   // tables and outputs
  std::map<std::string, std::vector<std::string>> temps;
  std::set<std::string> outs, tabs, consts;
  std::string e_index, J;
  bool warp = false;
  long R = 0;
  std::map<std::string, long> rest;
  std::set<std::string> acc_dims;
  std::vector<std::string> lines;
  // warp mapping: loops outside the row loop whose iterations fill per-index
  // array temporaries are spread over the lanes; those arrays live in shared
  // memory (one row per warp) and are read by every lane
  std::set<const Node*> dist;
  std::set<std::string> shared;
  bool in_J = false;
  // warp mapping: baked (pre-evaluated) tables with a dimension named J are stored
  // with that dimension innermost, so the lanes' reads T[..][j=lane][..] are
  // consecutive addresses (femopt's row-major [j][k] layout strides them by n_k)
  std::map<std::string, std::vector<size_t>> perm;  // stored position -> IR position

  std::string temp_ref(const std::string& name, const std::string& flat) const {
    if (shared.count(name)) return "s_" + ident(name) + "[w_][" + flat + "]";
    return "v_" + ident(name) + "[" + flat + "]";
  }

  std::string ext_of(const std::string& d) const {
    return d == e_index ? std::string("E") : std::to_string(ext.at(d));
  }
  std::string offset(const std::string& name, const std::vector<std::string>& idx) const {
    const auto& dd = dims.at(name);
    if (idx.size() != dd.size()) irfail(name + " subscripted with the wrong rank");
    if (idx.empty()) return "0";
    auto it = perm.find(name);
    auto at = [&](size_t i) { return it == perm.end() ? i : it->second[i]; };
    std::string e = "(long)i_" + idx[at(0)];
    for (size_t i = 1; i < dd.size(); ++i)
      e = "(" + e + " * " + ext_of(dd[at(i)]) + " + i_" + idx[at(i)] + ")";
    return e;
  }
  std::string temp_flat(const std::string& name, const std::vector<std::string>& idx) const {
    const auto& td = temps.at(name);
    if (idx.size() != td.size()) irfail("temporary " + name + " subscript count");
    std::string f = "0";
    for (size_t i = 0; i < td.size(); ++i)
      f = "(" + f + " * " + std::to_string(ext.at(td[i])) + " + i_" + idx[i] + ")";
    return f;
  }
  std::string expr(const Json& x, int prec) const {
    if (x.kind == Json::Num) {
      std::string s = lit(x.num);
      return (x.num < 0 && prec >= 1) ? "(" + s + ")" : s;
    }
    if (x.kind == Json::Str) {
      if (temps.count(x.str)) {
        if (!temps.at(x.str).empty()) irfail("array temporary " + x.str + " read without subscripts");
        return "v_" + ident(x.str);
      }
      if (consts.count(x.str)) return "c_" + ident(x.str);
      irfail("unknown scalar '" + x.str + "'");
    }
    if (x.kind != Json::Arr || x.arr.empty() || x.arr[0].kind != Json::Str) irfail("bad expression");
    const std::string& op = x.arr[0].str;
    if (op == "sym") {
      const std::string& name = x.arr.at(1).str;
      std::vector<std::string> idx;
      for (size_t i = 2; i < x.arr.size(); ++i) idx.push_back(x.arr[i].str);
      if (tabs.count(name)) return "t_" + ident(name) + "[" + offset(name, idx) + "]";
      if (temps.count(name)) return temp_ref(name, temp_flat(name, idx));
      if (outs.count(name)) return "o_" + ident(name) + "[" + offset(name, idx) + "]";
      irfail("unknown array '" + name + "'");
    }
    if (op == "+" || op == "*") {
      std::string s;
      for (size_t i = 1; i < x.arr.size(); ++i) {
        if (i > 1) s += op == "+" ? " + " : " * ";
        s += expr(x.arr[i], op == "+" ? 0 : 1);
      }
      const int wrap_at = op == "+" ? 1 : 2;
      return prec >= wrap_at ? "(" + s + ")" : s;
    }
    if (op == "/") {
      if (x.arr.size() != 3) irfail("'/' takes two operands");
      std::string s = expr(x.arr[1], 1) + " / " + expr(x.arr[2], 2);
      return prec >= 2 ? "(" + s + ")" : s;
    }
    if (op == "call") {
      const std::string& fn = x.arr.at(1).str;
      auto it = calls().find(fn);
      if (it == calls().end()) irfail("unsupported call '" + fn + "'");
      std::string s = it->second + "(";
      for (size_t i = 2; i < x.arr.size(); ++i) {
        if (i > 2) s += ", ";
        s += expr(x.arr[i], 0);
      }
      return s + ")";
    }
    irfail("unknown operator '" + op + "'");
  }
  void emit_nodes(const std::vector<Node>& nodes, int ind) {
    const std::string pad(2 * ind, ' ');
    for (const Node& n : nodes) {
      if (n.loop) {
        if (n.index == e_index) irfail("nested element loop");
        if (warp && n.index == J) {
          lines.push_back(pad + "#pragma unroll");
          lines.push_back(pad + "for (int r_ = 0; r_ < " + std::to_string(R) + "; ++r_) {");
          lines.push_back(pad + "  const int i_" + ident(J) + " = lane_ + 32 * r_;");
          lines.push_back(pad + "  if (i_" + J + " < " + std::to_string(n.end) + ") {");
          in_J = true;
          emit_nodes(n.body, ind + 2);
          in_J = false;
          lines.push_back(pad + "  }");
          lines.push_back(pad + "}");
          continue;
        }
        if (warp && !in_J && dist.count(&n)) {
          const long cnt = std::max<long>(0, n.end - n.begin);
          lines.push_back(pad + "__syncwarp();");
          lines.push_back(pad + "for (int d_ = 0; d_ < " + std::to_string((cnt + 31) / 32) + "; ++d_) {");
          lines.push_back(pad + "  const int i_" + ident(n.index) + " = " + std::to_string(n.begin) +
                          " + lane_ + 32 * d_;");
          lines.push_back(pad + "  if (i_" + n.index + " < " + std::to_string(n.end) + ") {");
          emit_nodes(n.body, ind + 2);
          lines.push_back(pad + "  }");
          lines.push_back(pad + "}");
          lines.push_back(pad + "__syncwarp();");
          continue;
        }
        if (warp && n.end - n.begin <= 64 && acc_dims.count(n.index)) {
          double t[2] = {0, 0};
          op_counts(n.body, 1, false, "", t);
          if ((n.end - n.begin) * t[0] <= 4096) lines.push_back(pad + "#pragma unroll");
        }
        lines.push_back(pad + "for (int i_" + ident(n.index) + " = " + std::to_string(n.begin) + "; i_" +
                        n.index + " < " + std::to_string(n.end) + "; ++i_" + n.index + ") {");
        emit_nodes(n.body, ind + 1);
        lines.push_back(pad + "}");
      } else {
        std::string target;
        if (outs.count(n.name) && warp) {
          std::string f = "0";
          const auto& dd = dims.at(n.name);
          for (size_t i = 2; i < dd.size(); ++i)
            f = "(" + f + " * " + std::to_string(ext.at(dd[i])) + " + i_" + n.idx[i] + ")";
          target = "a_" + n.name + "[r_ * " + std::to_string(rest.at(n.name)) + " + " + f + "]";
        } else if (outs.count(n.name)) {
          target = "o_" + n.name + "[" + offset(n.name, n.idx) + "]";
        } else if (!temps.at(n.name).empty()) {
          target = temp_ref(n.name, temp_flat(n.name, n.idx));
        } else {
          target = "v_" + n.name;
        }
        if (n.op == "+=")
          lines.push_back(pad + target + " += " + expr(*n.rhs, 0) + ";");
        else if (n.op == "=")
          lines.push_back(pad + target + " = " + expr(*n.rhs, 0) + ";");
        else
          irfail("unknown assignment '" + n.op + "'");
      }
    }
  }
};

struct Kernel {
  std::string source, fn = "femopt_kernel", cls_strategy;
  std::vector<std::string> outputs, inputs, constants, preevaluated;
  std::map<std::string, std::vector<std::string>> dims;
  std::map<std::string, long> ext;
  std::string e_index;
  bool warp = false;
  // GEMM mapping (femopt's pre-evaluated nests): the generated kernel writes
  // P[e][t] (ldp = Kp), then C[e][n] += P[e][:] . Bm[:][n] on DMMA
  bool gemm = false;
  int gK = 0, gKp = 0, gN = 0, gldb = 0;
  std::vector<double> gB;                    // [Kp][ldb], zero-padded
  std::map<int, double*> gB_dev;             // per device
  struct Scratch {
    double* p = nullptr;
    size_t n = 0;
    cudaEvent_t done = nullptr;  // recorded after the last GEMM that read it
  };
  std::map<int, Scratch> gP_dev;             // P buffer per device, reused across launches
  std::vector<char> cubin;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;

  long size_of(const std::string& name, long ncells) const {
    long s = 1;
    for (const auto& d : dims.at(name)) s *= d == e_index ? ncells : ext.at(d);
    return s;
  }
};

bool warp_plan(const std::vector<Node>& tree, Emitter& em) {
  if (em.e_index.empty()) return false;
  std::set<std::pair<std::string, std::string>> rows;
  for (const auto& o : em.outs) {
    const auto& d = em.dims.at(o);
    if (d.size() < 2) return false;
    rows.insert({d[0], d[1]});
  }
  if (rows.size() != 1 || rows.begin()->first != em.e_index) return false;
  const std::string J = rows.begin()->second;
  bool ok = true;
  std::set<std::string> written_in_J, read_outside_J;
  std::function<void(const std::vector<Node>&, bool)> walk = [&](const std::vector<Node>& ns,
                                                                 bool inJ) {
    for (const Node& n : ns) {
      if (n.loop) {
        if (n.index == J) {
          if (inJ || n.begin != 0 || n.end != em.ext.at(J)) ok = false;
          walk(n.body, true);
        } else {
          walk(n.body, inJ);
        }
      } else {
        std::set<std::string> used;
        names_in(*n.rhs, used);
        for (const auto& o : em.outs)
          if (used.count(o)) ok = false;
        if (em.outs.count(n.name)) {
          if (!inJ || n.op != "+=" || n.idx.size() < 2 || n.idx[0] != em.e_index || n.idx[1] != J)
            ok = false;
        } else if (inJ) {
          written_in_J.insert(n.name);
        }
        if (!inJ) read_outside_J.insert(used.begin(), used.end());
      }
    }
  };
  walk(tree, false);
  for (const auto& w : written_in_J)
    if (read_outside_J.count(w)) ok = false;
  if (ok) em.J = J;
  return ok;
}

void refs(const std::vector<Node>& ns, const Node* skip, std::set<std::string>& acc) {
  for (const Node& n : ns) {
    if (&n == skip) continue;
    if (n.loop) {
      refs(n.body, skip, acc);
    } else {
      acc.insert(n.name);
      names_in(*n.rhs, acc);
    }
  }
}

// Loops of the element body, outside the row loop J, that can run lane-parallel
// in the warp mapping: statements only (no nested loops), each writing either an
// array temporary subscripted by exactly the loop index, or a scalar temporary
// used nowhere else; no outputs.  Such an array is shared (one copy per warp)
// when every write of it is in such a loop.
void plan_distribution(const std::vector<Node>& body, Emitter& em) {
  std::vector<const Node*> cand;
  std::function<void(const std::vector<Node>&)> find = [&](const std::vector<Node>& ns) {
    for (const Node& n : ns) {
      if (!n.loop || n.index == em.J) continue;
      bool flat = true;
      for (const Node& c : n.body) flat = flat && !c.loop;
      if (!flat) {
        find(n.body);
        continue;
      }
      std::set<std::string> outside;
      refs(body, &n, outside);
      bool ok = n.end > n.begin;
      for (const Node& c : n.body) {
        std::set<std::string> used;
        names_in(*c.rhs, used);
        for (const auto& o : em.outs)
          if (used.count(o)) ok = false;
        if (em.outs.count(c.name) || !em.temps.count(c.name)) {
          ok = false;
        } else if (em.temps.at(c.name).empty()) {
          if (outside.count(c.name)) ok = false;
        } else if (em.temps.at(c.name) != std::vector<std::string>{n.index} ||
                   c.idx != std::vector<std::string>{n.index}) {
          ok = false;
        }
      }
      if (ok) cand.push_back(&n);
    }
  };
  find(body);
  // writes of each array temporary: all of them / inside candidate loops
  std::map<std::string, int> all_w;
  std::function<void(const std::vector<Node>&)> count = [&](const std::vector<Node>& ns) {
    for (const Node& n : ns) {
      if (n.loop) count(n.body);
      else if (em.temps.count(n.name) && !em.temps.at(n.name).empty()) ++all_w[n.name];
    }
  };
  count(body);
  for (bool changed = true; changed;) {
    changed = false;
    std::map<std::string, int> in_w;
    for (const Node* L : cand)
      for (const Node& c : L->body)
        if (!em.temps.at(c.name).empty()) ++in_w[c.name];
    for (auto it = cand.begin(); it != cand.end();) {
      bool keep = true;
      for (const Node& c : (*it)->body)
        if (!em.temps.at(c.name).empty() && in_w[c.name] != all_w[c.name]) keep = false;
      if (keep) {
        ++it;
      } else {
        it = cand.erase(it);
        changed = true;
      }
    }
  }
  for (const Node* L : cand) {
    em.dist.insert(L);
    for (const Node& c : L->body)
      if (!em.temps.at(c.name).empty()) em.shared.insert(c.name);
  }
}

// femopt's pre-evaluated (tensor) nest as a GEMM (preeval.cpp:279-451): the element
// body is scalar statements then ONE nest j { k { OUT[e][j][k] += sum_t T_t[j][k] * p_t } }
// with T_t pre-evaluated [j][k] (or [k][j]) tables and p_t products of scalars.
struct GemmTerm {
  std::string table;
  bool transposed = false;
  std::vector<const Json*> factors;  // scalar factors (names, numbers), in order
};
struct GemmPlan {
  std::string out, J, K;
  long nj = 0, nk = 0;
  const Node* nest = nullptr;
  std::vector<GemmTerm> terms;
};

bool gemm_plan(const std::vector<Node>& tree, const Emitter& em,
               const std::map<std::string, const Json*>& tables, GemmPlan& gp) {
  if (em.e_index.empty() || em.outs.size() != 1 || tree.size() != 1 || !tree[0].loop) return false;
  const std::vector<Node>& body = tree[0].body;
  if (body.empty() || !body.back().loop) return false;
  for (size_t i = 0; i + 1 < body.size(); ++i)
    if (body[i].loop || em.outs.count(body[i].name) || !em.temps.count(body[i].name) ||
        !em.temps.at(body[i].name).empty())
      return false;  // the preheader: scalar temporaries only
  const Node& Lj = body.back();
  if (Lj.body.size() != 1 || !Lj.body[0].loop) return false;
  const Node& Lk = Lj.body[0];
  if (Lk.body.size() != 1 || Lk.body[0].loop) return false;
  const Node& st = Lk.body[0];
  if (Lj.begin != 0 || Lj.end != em.ext.at(Lj.index) || Lk.begin != 0 ||
      Lk.end != em.ext.at(Lk.index))
    return false;
  if (!em.outs.count(st.name) || st.op != "+=" ||
      st.idx != std::vector<std::string>{em.e_index, Lj.index, Lk.index})
    return false;
  gp.out = st.name;
  gp.J = Lj.index;
  gp.K = Lk.index;
  gp.nj = Lj.end;
  gp.nk = Lk.end;
  gp.nest = &Lj;
  auto is_pre = [&](const std::string& n) {
    auto it = tables.find(n);
    if (it == tables.end()) return false;
    const Json* pv = it->second->get("provenance");
    return pv && pv->kind == Json::Str && pv->str == "preevaluated";
  };
  auto scalar = [&](const Json& x) {
    return x.kind == Json::Num ||
           (x.kind == Json::Str && (em.consts.count(x.str) ||
                                    (em.temps.count(x.str) && em.temps.at(x.str).empty())));
  };
  auto add_term = [&](const Json& x) {
    GemmTerm t;
    auto take = [&](const Json& f) {
      if (f.kind == Json::Arr && f.arr.size() == 4 && f.arr[0].kind == Json::Str &&
          f.arr[0].str == "sym" && t.table.empty() && is_pre(f.arr[1].str)) {
        // subscripts name the table's dims in order: [j][k] or (stored transposed) [k][j]
        const std::vector<std::string> sub{f.arr[2].str, f.arr[3].str};
        const auto& dd = em.dims.at(f.arr[1].str);
        if (sub != dd) return false;
        if (sub != std::vector<std::string>{gp.J, gp.K} && sub != std::vector<std::string>{gp.K, gp.J})
          return false;
        t.table = f.arr[1].str;
        return true;
      }
      if (scalar(f)) {
        t.factors.push_back(&f);
        return true;
      }
      return false;
    };
    if (x.kind == Json::Arr && !x.arr.empty() && x.arr[0].kind == Json::Str && x.arr[0].str == "*") {
      for (size_t i = 1; i < x.arr.size(); ++i)
        if (!take(x.arr[i])) return false;
    } else if (!take(x)) {
      return false;
    }
    if (t.table.empty()) return false;
    gp.terms.push_back(std::move(t));
    return true;
  };
  const Json& r = *st.rhs;
  if (r.kind == Json::Arr && !r.arr.empty() && r.arr[0].kind == Json::Str && r.arr[0].str == "+") {
    for (size_t i = 1; i < r.arr.size(); ++i)
      if (!add_term(r.arr[i])) return false;
  } else if (!add_term(r)) {
    return false;
  }
  return !gp.terms.empty();
}

void scan(const std::vector<Node>& nodes, Emitter& em) {
  for (const Node& n : nodes) {
    if (n.loop) {
      scan(n.body, em);
      continue;
    }
    if (em.outs.count(n.name)) {
      auto it = em.dims.find(n.name);
      if (it != em.dims.end() && it->second != n.idx) irfail("output " + n.name + " written with different subscripts");
      em.dims[n.name] = n.idx;
    } else if (em.tabs.count(n.name)) {
      irfail("statement writes table " + n.name);
    } else {
      auto it = em.temps.find(n.name);
      if (it != em.temps.end() && it->second != n.idx) irfail("temporary " + n.name + " used with different subscripts");
      em.temps[n.name] = n.idx;
    }
  }
}

// The GEMM mapping: a thread-per-cell kernel evaluates the element preheader and
// writes the term products P[e][t]; the contraction runs in gemm_f64.cu.
std::unique_ptr<Kernel> generate_gemm(const Json& ir, Emitter& em,
                                      const std::map<std::string, const Json*>& tables,
                                      const GemmPlan& gp, std::unique_ptr<Kernel> K,
                                      const std::vector<Node>& tree) {
  (void)ir;
  const int KT = femgpu::gemm_f64_tile_k(), NT = femgpu::gemm_f64_tile_n();
  K->gemm = true;
  K->gK = (int)gp.terms.size();
  K->gKp = (K->gK + KT - 1) / KT * KT;
  K->gN = (int)(gp.nj * gp.nk);
  K->gldb = (K->gN + NT - 1) / NT * NT;
  K->gB.assign((size_t)K->gKp * K->gldb, 0.0);
  for (int t = 0; t < K->gK; ++t) {
    const auto& vals = tables.at(gp.terms[t].table)->at("values").arr;
    const bool kj = em.dims.at(gp.terms[t].table) == std::vector<std::string>{gp.K, gp.J};
    for (long j = 0; j < gp.nj; ++j)
      for (long k = 0; k < gp.nk; ++k)
        K->gB[(size_t)t * K->gldb + j * gp.nk + k] = vals.at(kj ? k * gp.nj + j : j * gp.nk + k).num;
  }
  for (const auto& kv : tables) {
    const Json* pv = kv.second->get("provenance");
    const bool pre = pv && pv->kind == Json::Str && pv->str == "preevaluated";
    (pre ? K->preevaluated : K->inputs).push_back(kv.first);
  }
  K->outputs.assign(em.outs.begin(), em.outs.end());
  K->constants.assign(em.consts.begin(), em.consts.end());
  std::sort(K->inputs.begin(), K->inputs.end());
  std::sort(K->preevaluated.begin(), K->preevaluated.end());
  std::vector<Node> pre(tree[0].body.begin(), tree[0].body.end() - 1);  // scalar statements
  em.lines.push_back("  const long i_" + em.e_index + " = e0_ + (long)blockIdx.x * blockDim.x + threadIdx.x;");
  em.lines.push_back("  if (i_" + em.e_index + " >= E) return;");
  em.emit_nodes(pre, 1);
  // P stored transposed, [Kp][ldp] (ldp = cells per chunk): each term's stores are
  // consecutive across the threads of a warp
  auto row = [&](int t) {
    return "o_P_[(long)" + std::to_string(t) + " * ldp_ + (i_" + em.e_index + " - e0_)";
  };
  for (int t = 0; t < K->gK; ++t) {
    Json prod;
    prod.kind = Json::Arr;
    Json op;
    op.kind = Json::Str;
    op.str = "*";
    prod.arr.push_back(op);
    for (const Json* f : gp.terms[t].factors) prod.arr.push_back(*f);
    std::string e;
    if (prod.arr.size() == 1) e = "1.0";
    else if (prod.arr.size() == 2) e = em.expr(prod.arr[1], 0);
    else e = em.expr(prod, 0);
    em.lines.push_back("  " + row(t) + "] = " + e + ";");
  }
  for (int t = K->gK; t < K->gKp; ++t) em.lines.push_back("  " + row(t) + "] = 0.0;");
  std::string src = "// generated by libfemgpu (femgpu_ir_create, GEMM mapping) from a femopt kernel IR\n";
  src += "extern \"C\" __global__ void __launch_bounds__(128) " + K->fn + "(double* __restrict__ o_P_";
  for (const auto& t : K->inputs) src += ", const double* __restrict__ t_" + ident(t);
  for (const auto& c : K->constants) src += ", const double c_" + ident(c);
  src += ", const long e0_, const long E, const long ldp_) {\n";
  for (const auto& kv : em.temps) {
    if (!kv.second.empty()) irfail("array temporary in a GEMM preheader");
    src += "  double v_" + ident(kv.first) + ";\n";
  }
  for (const auto& l : em.lines) src += l + "\n";
  src += "}\n";
  K->source = src;
  K->dims = em.dims;
  K->ext = em.ext;
  K->e_index = em.e_index;
  return K;
}

std::unique_ptr<Kernel> generate(const char* json, int strategy) {
  Json ir = parse(json);
  auto K = std::make_unique<Kernel>();
  Emitter em;
  for (const auto& kv : ir.at("indices").obj) em.ext[kv.first] = (long)kv.second.num;
  const Json* T = ir.get("tables");
  std::map<std::string, const Json*> tables;
  if (T)
    for (const auto& kv : T->obj) {
      tables[kv.first] = &kv.second;
      em.tabs.insert(kv.first);
      std::vector<std::string> dd;
      for (const auto& d : kv.second.at("dims").arr) dd.push_back(d.str);
      em.dims[kv.first] = dd;
    }
  const Json* C = ir.get("constants");
  std::map<std::string, double> cvals;
  if (C && C->kind == Json::Obj)
    for (const auto& kv : C->obj) {
      em.consts.insert(kv.first);
      cvals[kv.first] = kv.second.num;
    }
  for (const auto& o : ir.at("outputs").arr) em.outs.insert(o.str);
  std::vector<Node> tree = build_tree(ir, em.ext);

  std::vector<const Node*> top;
  for (const Node& n : tree)
    if (n.loop) top.push_back(&n);
  if (top.size() == 1 && (top[0]->cls == "orderfree" || (top[0]->cls.empty() && top[0]->index == "e")))
    em.e_index = top[0]->index;
  scan(tree, em);
  for (const auto& o : em.outs)
    if (!em.dims.count(o)) irfail("output " + o + " is never written");
  // An output without the element index is a sum over the cells (the reference's
  // corpus kernels, proj/tests/kernels.hpp, accumulate A[j][k] over e): the element
  // loop is then a reduction, run in order inside one thread like emit_c's loop
  // (bit-identical), not spread over the grid.
  if (!em.e_index.empty())
    for (const auto& o : em.outs) {
      const auto& dd = em.dims.at(o);
      if (std::find(dd.begin(), dd.end(), em.e_index) == dd.end()) {
        em.e_index.clear();
        break;
      }
    }

  GemmPlan gp;
  const bool can_gemm = gemm_plan(tree, em, tables, gp);
  if (strategy == 3 && !can_gemm) irfail("the gemm mapping does not apply to this nest");
  if (strategy == 3 || (strategy == 0 && can_gemm && (long)gp.terms.size() * gp.nj * gp.nk >= 2048))
    return generate_gemm(ir, em, tables, gp, std::move(K), tree);
  const bool can_warp = warp_plan(tree, em);
  bool warp = false;
  if (strategy == 0) {
    // warp per cell whenever a row loop of >= 8 rows exists: its register
    // accumulators replace the thread mapping's per-statement global += (which
    // femopt's optimized nests put inside the quadrature loop) and spread the
    // j-loop over lanes.  Measured on the BASELINE forms (profiles/
    // bench_generic_r01.jsonl): warp 1.1-42x faster for n >= 20, raw and
    // optimized alike; thread 2-12x faster for n = 4 (P1), where 28 lanes idle.
    warp = can_warp && em.ext.at(em.J) >= 8;
  } else if (strategy == 2) {
    if (!can_warp) irfail("the warp mapping does not apply to this nest");
    warp = true;
  } else if (strategy != 1 && strategy != 3) {
    irfail("unknown strategy");
  }
  em.warp = warp;
  if (warp) {
    em.R = (em.ext.at(em.J) + 31) / 32;
    for (const auto& o : em.outs) {
      long r = 1;
      const auto& dd = em.dims.at(o);
      for (size_t i = 2; i < dd.size(); ++i) r *= em.ext.at(dd[i]), em.acc_dims.insert(dd[i]);
      em.rest[o] = r;
    }
  }

  for (const auto& kv : tables) {
    const Json* pv = kv.second->get("provenance");
    const bool pre = pv && pv->kind == Json::Str && pv->str == "preevaluated";
    (pre ? K->preevaluated : K->inputs).push_back(kv.first);
    if (pre && warp) {
      const auto& dd = em.dims.at(kv.first);
      auto j = std::find(dd.begin(), dd.end(), em.J);
      if (j != dd.end() && j + 1 != dd.end()) {
        std::vector<size_t> order;
        for (size_t i = 0; i < dd.size(); ++i)
          if (i != (size_t)(j - dd.begin())) order.push_back(i);
        order.push_back(j - dd.begin());
        em.perm[kv.first] = order;
      }
    }
  }
  K->outputs.assign(em.outs.begin(), em.outs.end());
  K->constants.assign(em.consts.begin(), em.consts.end());
  std::sort(K->inputs.begin(), K->inputs.end());
  std::sort(K->preevaluated.begin(), K->preevaluated.end());

  // body
  std::vector<Node> pre, body;
  if (!em.e_index.empty()) {
    for (const Node& n : tree)
      if (&n != top[0]) pre.push_back(n);
    body = top[0]->body;
  } else {
    body = tree;
  }
  for (const Node& n : pre)
    if (!n.loop && em.outs.count(n.name)) irfail("output written outside the element loop");
  em.emit_nodes(pre, 1);
  if (warp) {
    plan_distribution(body, em);
    em.lines.push_back("  const long i_" + em.e_index + " = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;");
    em.lines.push_back("  const int lane_ = threadIdx.x & 31;");
    if (!em.shared.empty()) em.lines.push_back("  const int w_ = threadIdx.x >> 5;");
    em.lines.push_back("  if (i_" + em.e_index + " >= E) return;");
    for (const auto& o : em.outs) {
      const std::string n = std::to_string(em.R * em.rest[o]);
      em.lines.push_back("  double a_" + o + "[" + n + "];");
      em.lines.push_back("  #pragma unroll");
      em.lines.push_back("  for (int x_ = 0; x_ < " + n + "; ++x_) a_" + o + "[x_] = 0.0;");
    }
  } else if (!em.e_index.empty()) {
    em.lines.push_back("  const long i_" + em.e_index + " = (long)blockIdx.x * blockDim.x + threadIdx.x;");
    em.lines.push_back("  if (i_" + em.e_index + " >= E) return;");
  } else {
    em.lines.push_back("  if (blockIdx.x != 0 || threadIdx.x != 0) return;");
  }
  em.emit_nodes(body, 1);
  if (warp) {
    const std::string nJ = std::to_string(em.ext.at(em.J)), R = std::to_string(em.R);
    for (const auto& o : em.outs) {
      const std::string rs = std::to_string(em.rest[o]);
      em.lines.push_back("  #pragma unroll");
      em.lines.push_back("  for (int r_ = 0; r_ < " + R + "; ++r_) {");
      em.lines.push_back("    const long row_ = lane_ + 32 * r_;");
      em.lines.push_back("    if (row_ < " + nJ + ") {");
      em.lines.push_back("      double* dst_ = o_" + o + " + (i_" + em.e_index + " * " + nJ + " + row_) * " + rs + ";");
      em.lines.push_back("      for (int x_ = 0; x_ < " + rs + "; ++x_) dst_[x_] += a_" + o + "[r_ * " + rs + " + x_];");
      em.lines.push_back("    }");
      em.lines.push_back("  }");
    }
  }

  std::string src = "// generated by libfemgpu (femgpu_ir_create) from a femopt kernel IR\n";
  for (const auto& name : K->preevaluated) {
    const Json& vals = tables[name]->at("values");
    src += "__device__ const double t_" + ident(name) + "[" + std::to_string(std::max<size_t>(1, vals.arr.size())) + "] = {";
    auto pit = em.perm.find(name);
    std::vector<long> ex, stride;  // IR (row-major) extents and strides
    if (pit != em.perm.end()) {
      for (const auto& d : em.dims.at(name)) ex.push_back(em.ext.at(d));
      stride.assign(ex.size(), 1);
      for (size_t i = ex.size() - 1; i > 0; --i) stride[i - 1] = stride[i] * ex[i];
    }
    for (size_t i = 0; i < vals.arr.size(); ++i) {
      if (i) src += ",";
      size_t src_i = i;
      if (pit != em.perm.end()) {  // stored flat index i -> IR flat index
        const auto& ord = pit->second;
        size_t rem = i, k = 0;
        for (size_t a = ord.size(); a-- > 0;) {
          const long c = (long)(rem % ex[ord[a]]);
          rem /= ex[ord[a]];
          k += c * stride[ord[a]];
        }
        src_i = k;
      }
      src += lit(vals.arr[src_i].num);
    }
    src += "};\n";
  }
  src += "extern \"C\" __global__ void __launch_bounds__(128) " + K->fn + "(";
  std::vector<std::string> params;
  for (const auto& o : K->outputs) params.push_back("double* __restrict__ o_" + ident(o));
  for (const auto& t : K->inputs) params.push_back("const double* __restrict__ t_" + ident(t));
  for (const auto& c : K->constants) params.push_back("const double c_" + ident(c));
  params.push_back("const long E");
  for (size_t i = 0; i < params.size(); ++i) src += (i ? ", " : "") + params[i];
  src += ") {\n";
  for (const auto& kv : em.temps) {
    if (!kv.second.empty()) {
      long n = 1;
      for (const auto& d : kv.second) {
        if (d == em.e_index) irfail("temporary " + kv.first + " indexed by the element loop");
        n *= em.ext.at(d);
      }
      if (em.shared.count(kv.first))
        src += "  __shared__ double s_" + ident(kv.first) + "[4][" + std::to_string(n) + "];\n";
      else
        src += "  double v_" + ident(kv.first) + "[" + std::to_string(n) + "];\n";
    } else {
      src += "  double v_" + ident(kv.first) + ";\n";
    }
  }
  for (const auto& l : em.lines) src += l + "\n";
  src += "}\n";
  K->source = src;
  K->dims = em.dims;
  K->ext = em.ext;
  K->e_index = em.e_index;
  K->warp = warp;
  return K;
}

// ----------------------------------------------------------------------------
// NVRTC (dlopen) and module load
// ----------------------------------------------------------------------------
struct Nvrtc {
  void* h = nullptr;
  int (*create)(void**, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  int (*compile)(void*, int, const char* const*) = nullptr;
  int (*logsize)(void*, size_t*) = nullptr;
  int (*log)(void*, char*) = nullptr;
  int (*cubinsize)(void*, size_t*) = nullptr;
  int (*cubin)(void*, char*) = nullptr;
  int (*destroy)(void**) = nullptr;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.create = (decltype(n.create))dlsym(n.h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(n.h, "nvrtcCompileProgram");
    n.logsize = (decltype(n.logsize))dlsym(n.h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(n.h, "nvrtcGetProgramLog");
    n.cubinsize = (decltype(n.cubinsize))dlsym(n.h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(n.h, "nvrtcGetCUBIN");
    n.destroy = (decltype(n.destroy))dlsym(n.h, "nvrtcDestroyProgram");
  });
  if (!n.h || !n.create || !n.compile || !n.cubin)
    throw CudaError("CUDA: NVRTC (libnvrtc.so.12) is not available");
  return n;
}

void compile(Kernel& K) {
  const Nvrtc& nv = nvrtc();
  void* prog = nullptr;
  if (nv.create(&prog, K.source.c_str(), "femopt_kernel.cu", 0, nullptr, nullptr) != 0)
    throw CudaError("CUDA: nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--prec-div=true",
                        "--prec-sqrt=true", "-std=c++17", "-default-device"};
  const int rc = nv.compile(prog, 6, opts);
  if (rc != 0) {
    size_t n = 0;
    nv.logsize(prog, &n);
    std::string log(n, '\0');
    nv.log(prog, log.data());
    nv.destroy(&prog);
    throw CudaError("CUDA: NVRTC compile failed:\n" + log);
  }
  size_t n = 0;
  nv.cubinsize(prog, &n);
  K.cubin.resize(n);
  nv.cubin(prog, K.cubin.data());
  nv.destroy(&prog);
}

}  // namespace irgen

// ============================================================================
// C ABI
// ============================================================================
struct femgpu_ir {
  std::unique_ptr<irgen::Kernel> k;
  std::mutex mu;
};

namespace {
template <class Fn>
int ir_guard(Fn&& fn) {
  try {
    fn();
    femgpu::set_last_error("");
    return FEMGPU_OK;
  } catch (const irgen::IRError& e) {
    femgpu::set_last_error(e.what());
    return FEMGPU_ERR_NOT_FEM_NEST;
  } catch (const irgen::CudaError& e) {
    femgpu::set_last_error(e.what());
    return FEMGPU_ERR_CUDA;
  } catch (const std::exception& e) {
    femgpu::set_last_error(e.what());
    return FEMGPU_ERR_INTERNAL;
  }
}

int bad_arg(const char* m) {
  femgpu::set_last_error(m);
  return FEMGPU_ERR_INVALID_ARG;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw irgen::CudaError(std::string("CUDA ") + what + ": " + cudaGetErrorString(e));
}

cudaKernel_t loaded(femgpu_ir* f) {
  std::lock_guard<std::mutex> lock(f->mu);
  auto& K = *f->k;
  // a cudaLibrary is context-independent: one load serves every device (the module
  // is loaded into a device's context on that device's first launch)
  if (!K.kern) {
    cuda_ok(cudaLibraryLoadData(&K.lib, K.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
            "cudaLibraryLoadData");
    cuda_ok(cudaLibraryGetKernel(&K.kern, K.lib, K.fn.c_str()), "cudaLibraryGetKernel");
  }
  return K.kern;
}
}  // namespace

extern "C" {

int femgpu_ir_create(const char* json, int strategy, femgpu_ir** out) {
  if (!json || !out) return bad_arg("null argument");
  *out = nullptr;
  return ir_guard([&] {
    auto f = std::make_unique<femgpu_ir>();
    f->k = irgen::generate(json, strategy);
    irgen::compile(*f->k);
    *out = f.release();
  });
}

void femgpu_ir_free(femgpu_ir* f) {
  if (f && f->k) {
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : f->k->gB_dev) {
      cudaSetDevice(kv.first);
      cudaFree(kv.second);
    }
    for (auto& kv : f->k->gP_dev) {
      cudaSetDevice(kv.first);
      if (kv.second.done) cudaEventSynchronize(kv.second.done);
      cudaFree(kv.second.p);
      if (kv.second.done) cudaEventDestroy(kv.second.done);
    }
    cudaSetDevice(cur);
    if (f->k->lib) cudaLibraryUnload(f->k->lib);
  }
  delete f;
}

int femgpu_ir_get_info(const femgpu_ir* f, femgpu_ir_info* info) {
  if (!f || !info) return bad_arg("null argument");
  const auto& K = *f->k;
  info->noutputs = (int)K.outputs.size();
  info->ninputs = (int)K.inputs.size();
  info->nconstants = (int)K.constants.size();
  info->per_cell = K.e_index.empty() ? 0 : 1;
  info->strategy = K.gemm ? 3 : K.warp ? 2 : 1;
  return FEMGPU_OK;
}

int femgpu_ir_argname(const femgpu_ir* f, int group, int index, char* buf, size_t len) {
  if (!f || !buf || group < 0 || group > 2) return bad_arg("bad argument");
  const auto& v = group == 0 ? f->k->outputs : group == 1 ? f->k->inputs : f->k->constants;
  if (index < 0 || index >= (int)v.size()) return bad_arg("argument index out of range");
  std::snprintf(buf, len, "%s", v[index].c_str());
  return FEMGPU_OK;
}

int femgpu_ir_arg_size(const femgpu_ir* f, int group, int index, long ncells, long* size) {
  if (!f || !size || group < 0 || group > 1) return bad_arg("bad argument");
  const auto& v = group == 0 ? f->k->outputs : f->k->inputs;
  if (index < 0 || index >= (int)v.size()) return bad_arg("argument index out of range");
  *size = f->k->size_of(v[index], ncells);
  return FEMGPU_OK;
}

const char* femgpu_ir_source(const femgpu_ir* f) { return f ? f->k->source.c_str() : ""; }

int femgpu_ir_launch(femgpu_ir* f, long ncells, double* const* outputs, const double* const* inputs,
                     const double* constants, void* stream) {
  if (!f || ncells < 0 || (!f->k->outputs.empty() && !outputs) ||
      (!f->k->inputs.empty() && !inputs) || (!f->k->constants.empty() && !constants))
    return bad_arg("bad argument");
  return ir_guard([&] {
    auto& K = *f->k;
    if (!K.e_index.empty() && ncells == 0) return;
    cudaKernel_t kern = loaded(f);
    if (K.gemm) {
      cudaStream_t s = static_cast<cudaStream_t>(stream);
      int dev = 0;
      cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
      double* dB = nullptr;
      // one P scratch per (kernel, device), handed between launches (any stream) by
      // an event: this launch's stream waits for the previous launch's last GEMM
      std::lock_guard<std::mutex> lock(f->mu);
      auto it = K.gB_dev.find(dev);
      if (it == K.gB_dev.end()) {
        cuda_ok(cudaMalloc(&dB, K.gB.size() * sizeof(double)), "cudaMalloc(tables)");
        cuda_ok(cudaMemcpy(dB, K.gB.data(), K.gB.size() * sizeof(double), cudaMemcpyHostToDevice),
                "H2D(tables)");
        K.gB_dev[dev] = dB;
      } else {
        dB = it->second;
      }
      // P[chunk][Kp], chunks of <= 2^17 cells
      const long chunk = std::min<long>(ncells, 1L << 17);
      auto& sc = K.gP_dev[dev];
      if (!sc.done) cuda_ok(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming), "cudaEventCreate");
      const size_t need = (size_t)((chunk + 1) / 2 * 2) * K.gKp;
      if (sc.n < need) {
        cuda_ok(cudaEventSynchronize(sc.done), "cudaEventSynchronize");
        cudaFree(sc.p);
        sc.p = nullptr;
        sc.n = 0;
        cuda_ok(cudaMalloc(&sc.p, need * sizeof(double)), "cudaMalloc(P)");
        sc.n = need;
      }
      cuda_ok(cudaStreamWaitEvent(s, sc.done, 0), "cudaStreamWaitEvent");
      double* dP = sc.p;
      long e0 = 0, Eend = 0;
      std::vector<void*> args;
      void* pP = dP;
      std::vector<const void*> ptrs(K.inputs.size());
      for (size_t i = 0; i < K.inputs.size(); ++i) ptrs[i] = inputs[i];
      args.push_back(&pP);
      for (auto& p : ptrs) args.push_back(&p);
      std::vector<double> cv(K.constants.size());
      for (size_t i = 0; i < cv.size(); ++i) {
        cv[i] = constants[i];
        args.push_back(&cv[i]);
      }
      long ldp = (chunk + 1) / 2 * 2;
      args.push_back(&e0);
      args.push_back(&Eend);
      args.push_back(&ldp);
      cudaError_t err = cudaSuccess;
      for (long c0 = 0; c0 < ncells && err == cudaSuccess; c0 += chunk) {
        e0 = c0;
        Eend = std::min(ncells, c0 + chunk);
        const unsigned grid = (unsigned)((Eend - c0 + 127) / 128);
        err = cudaLaunchKernel((const void*)kern, dim3(grid), dim3(128), args.data(), 0, s);
        if (err == cudaSuccess)
          err = femgpu::launch_gemm_f64_acc(Eend - c0, K.gN, K.gK, (int)ldp, dP, dB, K.gldb,
                                            outputs[0] + c0 * (long)K.gN, s, true);
      }
      if (err == cudaSuccess) err = cudaEventRecord(sc.done, s);
      cuda_ok(err, "GEMM mapping");
      return;
    }
    std::vector<void*> args;
    std::vector<const void*> ptrs(K.outputs.size() + K.inputs.size());
    for (size_t i = 0; i < K.outputs.size(); ++i) ptrs[i] = outputs[i];
    for (size_t i = 0; i < K.inputs.size(); ++i) ptrs[K.outputs.size() + i] = inputs[i];
    for (auto& p : ptrs) args.push_back(&p);
    std::vector<double> cv(K.constants.size());
    for (size_t i = 0; i < cv.size(); ++i) {
      cv[i] = constants[i];
      args.push_back(&cv[i]);
    }
    long E = ncells;
    args.push_back(&E);
    const long threads = K.e_index.empty() ? 1 : ncells * (K.warp ? 32 : 1);
    const unsigned grid = (unsigned)std::max<long>(1, (threads + 127) / 128);
    cuda_ok(cudaLaunchKernel((const void*)kern, dim3(grid), dim3(128), args.data(), 0,
                             static_cast<cudaStream_t>(stream)),
            "cudaLaunchKernel");
  });
}

int femgpu_ir_argv(femgpu_ir* f, long ncells, double* const* o, const double* const* t,
                   const double* c) {
  if (!f || ncells < 0) return bad_arg("bad argument");
  return ir_guard([&] {
    const auto& K = *f->k;
    std::vector<double*> d_o(K.outputs.size()), d_t(K.inputs.size());
    std::vector<long> so(K.outputs.size());
    auto cleanup = [&] {
      for (auto p : d_o) cudaFree(p);
      for (auto p : d_t) cudaFree(p);
    };
    try {
      for (size_t i = 0; i < K.outputs.size(); ++i) {
        so[i] = K.size_of(K.outputs[i], ncells);
        cuda_ok(cudaMalloc(&d_o[i], std::max<long>(1, so[i]) * sizeof(double)), "cudaMalloc");
        cuda_ok(cudaMemcpy(d_o[i], o[i], so[i] * sizeof(double), cudaMemcpyHostToDevice), "H2D");
      }
      for (size_t i = 0; i < K.inputs.size(); ++i) {
        const long s = K.size_of(K.inputs[i], ncells);
        cuda_ok(cudaMalloc(&d_t[i], std::max<long>(1, s) * sizeof(double)), "cudaMalloc");
        cuda_ok(cudaMemcpy(d_t[i], t[i], s * sizeof(double), cudaMemcpyHostToDevice), "H2D");
      }
      std::vector<const double*> ct(d_t.begin(), d_t.end());
      const int rc = femgpu_ir_launch(f, ncells, d_o.data(), ct.data(), c, nullptr);
      if (rc != FEMGPU_OK) throw irgen::CudaError(femgpu_last_error());
      cuda_ok(cudaDeviceSynchronize(), "kernel");
      for (size_t i = 0; i < K.outputs.size(); ++i)
        cuda_ok(cudaMemcpy(o[i], d_o[i], so[i] * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

}  // extern "C"
