// K1 -- batched mapping evaluation.
//
// A pm_program (the lowered per-point suffix of a Mapple mapping function,
// see paper_2507_17087_b200/dsl/lower.py) is turned into CUDA C++ with every
// processor-space extent, stride and divisor baked in as an immediate, JIT
// compiled by NVRTC for sm_100a and launched over the points of an index
// launch.  Replaces the reference's interpreted per-point loop
// (dsl/interp.py:401-418 + spaces.py:185-213, driven by cli.py:155-161).
//
// The kernel is HBM-bound: each thread maps 4 consecutive points, loads their
// coordinates with 16-byte vector loads (explicit mode) or derives them from
// the linear index (implicit row-major mode, 0 input bytes), evaluates the
// integer program in registers and writes 4 processor ids with one 16-byte
// store.  Register widths come from the host's interval analysis, so most
// programs run in 32-bit integer arithmetic with constant divisors.

#include <nvrtc.h>

#include <climits>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "plan.h"
#include "pm_common.h"

namespace pm {

namespace {

const char* kSigned[3] = {"int", "long long", "__int128"};
const char* kUnsigned[3] = {"unsigned", "unsigned long long", "unsigned __int128"};

const char* kPrelude = R"CUDA(
template <typename T> __device__ __forceinline__ T pm_fdiv(T a, T b) {
  T q = a / b; T r = a - q * b;
  return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}
template <typename T> __device__ __forceinline__ T pm_fmod(T a, T b) {
  T r = a % b;
  return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}
#define PM_FAIL(s) do { *site_out = (s); return -1; } while (0)
template <typename T> __device__ __forceinline__ T pm_min2(T a, T b) { return a < b ? a : b; }
template <typename T> __device__ __forceinline__ T pm_max2(T a, T b) { return a > b ? a : b; }
)CUDA";

struct Gen {
  const pm_program* p;
  std::ostringstream o;
  int max_w = 0;

  int w(int r) const { return p->reg_width[r]; }

  std::string cst(int width, long long lo, long long hi) {
    std::ostringstream s;
    if (width == 2) {
      s << "((__int128)(((unsigned __int128)(unsigned long long)" << (unsigned long long)hi
        << "ULL << 64) | (unsigned __int128)(unsigned long long)" << (unsigned long long)lo
        << "ULL))";
    } else {
      s << "((" << kSigned[width] << ")(long long)" << (unsigned long long)lo << "ULL)";
    }
    return s.str();
  }

  int check() {
    for (int i = 0; i < p->n_regs; ++i) {
      if (p->reg_width[i] > 2) return set_error("register %d has bad width", i), PM_ERR_INVALID;
      if (p->reg_width[i] > max_w) max_w = p->reg_width[i];
    }
    int depth = 0;
    bool ret = false;
    for (int i = 0; i < p->n_insns; ++i) {
      const pm_insn& in = p->insns[i];
      auto bad = [&](int r) { return r < 0 || r >= p->n_regs; };
      switch (in.op) {
        case PM_OP_CONST: case PM_OP_COORD:
          if (bad(in.dst)) return set_error("insn %d: bad dst", i), PM_ERR_INVALID;
          if (in.op == PM_OP_COORD && (in.lo < 0 || in.lo >= p->n_coords))
            return set_error("insn %d: bad coordinate", i), PM_ERR_INVALID;
          break;
        case PM_OP_ADD: case PM_OP_SUB: case PM_OP_MUL: case PM_OP_DIV: case PM_OP_MOD:
        case PM_OP_GT: case PM_OP_LT: case PM_OP_EQ:
          if (bad(in.dst) || bad(in.a) || bad(in.b))
            return set_error("insn %d: bad operand", i), PM_ERR_INVALID;
          break;
        case PM_OP_SELECT:
          if (bad(in.dst) || bad(in.a) || bad(in.b) || bad(in.c))
            return set_error("insn %d: bad operand", i), PM_ERR_INVALID;
          break;
        case PM_OP_MOV:
          if (bad(in.dst) || bad(in.a)) return set_error("insn %d: bad operand", i), PM_ERR_INVALID;
          break;
        case PM_OP_CHECK: case PM_OP_IF: case PM_OP_RET:
          if (bad(in.a)) return set_error("insn %d: bad operand", i), PM_ERR_INVALID;
          if (in.op == PM_OP_IF) ++depth;
          if (in.op == PM_OP_RET) ret = true;
          break;
        case PM_OP_FAIL: break;
        case PM_OP_ELSE: if (depth <= 0) return set_error("insn %d: stray else", i), PM_ERR_INVALID; break;
        case PM_OP_ENDIF:
          if (--depth < 0) return set_error("insn %d: stray endif", i), PM_ERR_INVALID;
          break;
        default: return set_error("insn %d: unknown opcode %d", i, in.op), PM_ERR_INVALID;
      }
      if ((in.op == PM_OP_CHECK || in.op == PM_OP_FAIL ||
           ((in.op == PM_OP_DIV || in.op == PM_OP_MOD) && in.site >= 0)) &&
          (in.site < 0 || in.site > 0xFFFF))
        return set_error("insn %d: bad site %d", i, in.site), PM_ERR_INVALID;
    }
    if (depth != 0) return set_error("unbalanced if/endif"), PM_ERR_INVALID;
    (void)ret;
    if (p->n_coords < 0 || p->n_coords > 16) return set_error("bad rank"), PM_ERR_INVALID;
    return PM_OK;
  }

  void reg(int r) { o << "r" << r; }

  void body() {
    int ind = 1;
    auto pad = [&]() { for (int i = 0; i < ind; ++i) o << "  "; };
    for (int i = 0; i < p->n_insns; ++i) {
      const pm_insn& in = p->insns[i];
      if (in.op == PM_OP_ELSE || in.op == PM_OP_ENDIF) --ind;
      pad();
      const int d = in.dst;
      switch (in.op) {
        case PM_OP_CONST: o << "r" << d << " = " << cst(w(d), in.lo, in.hi) << ";\n"; break;
        case PM_OP_COORD: o << "r" << d << " = (" << kSigned[w(d)] << ")c" << in.lo << ";\n"; break;
        case PM_OP_ADD: case PM_OP_SUB: case PM_OP_MUL: {
          const char* op = in.op == PM_OP_ADD ? "+" : in.op == PM_OP_SUB ? "-" : "*";
          const char* u = kUnsigned[w(d)];
          o << "r" << d << " = (" << kSigned[w(d)] << ")((" << u << ")r" << in.a << " " << op
            << " (" << u << ")r" << in.b << ");\n";
          break;
        }
        case PM_OP_DIV: case PM_OP_MOD: {
          int cw = std::max(w(d), std::max(w(in.a), w(in.b)));
          const char* ct = kSigned[cw];
          const char* ut = kUnsigned[cw];
          o << "{ " << ct << " x = (" << ct << ")r" << in.a << ", y = (" << ct << ")r" << in.b
            << "; ";
          if (in.site >= 0) o << "if (y == 0) PM_FAIL(" << in.site << "); ";
          if (in.c & 1) {
            o << "r" << d << " = (" << kSigned[w(d)] << ")((" << ut << ")x "
              << (in.op == PM_OP_DIV ? "/" : "%") << " (" << ut << ")y); }\n";
          } else {
            o << "r" << d << " = (" << kSigned[w(d)] << ")"
              << (in.op == PM_OP_DIV ? "pm_fdiv" : "pm_fmod") << "(x, y); }\n";
          }
          break;
        }
        case PM_OP_GT: case PM_OP_LT: case PM_OP_EQ: {
          int cw = std::max(w(in.a), w(in.b));
          const char* op = in.op == PM_OP_GT ? ">" : in.op == PM_OP_LT ? "<" : "==";
          o << "r" << d << " = ((" << kSigned[cw] << ")r" << in.a << " " << op << " ("
            << kSigned[cw] << ")r" << in.b << ") ? 1 : 0;\n";
          break;
        }
        case PM_OP_SELECT:
          o << "r" << d << " = r" << in.a << " ? (" << kSigned[w(d)] << ")r" << in.b << " : ("
            << kSigned[w(d)] << ")r" << in.c << ";\n";
          break;
        case PM_OP_MOV: o << "r" << d << " = (" << kSigned[w(d)] << ")r" << in.a << ";\n"; break;
        case PM_OP_CHECK: {
          int cw = std::max(w(in.a), (in.lo < INT_MIN || in.hi > INT_MAX) ? 1 : 0);
          const char* ct = kSigned[cw];
          o << "if ((" << ct << ")r" << in.a << " < (" << ct << ")" << in.lo << "LL || ("
            << ct << ")r" << in.a << " >= (" << ct << ")" << in.hi << "LL) PM_FAIL(" << in.site
            << ");\n";
          break;
        }
        case PM_OP_FAIL: o << "PM_FAIL(" << in.site << ");\n"; break;
        case PM_OP_IF: o << "if (r" << in.a << " != 0) {\n"; ++ind; break;
        case PM_OP_ELSE: o << "} else {\n"; ++ind; break;
        case PM_OP_ENDIF: o << "}\n"; break;
        case PM_OP_RET: o << "return (int)r" << in.a << ";\n"; break;
      }
    }
  }

  // Interval version of the point program over a box of coordinates [bl_i, bh_i]
  // (registers l<r> / h<r>): returns the bin if every point of the box provably
  // maps to it without failure, else -1 ("not proven").  Each register's tile
  // interval lies inside the host's static interval for it, so the endpoint
  // arithmetic never leaves the register widths the host chose.  Floor division
  // is monotone in each argument while the divisor keeps its sign, so its
  // extremes sit at the corners; a condition that is not decided over the box,
  // a check that may fail, a reachable failure or a possibly-zero divisor gives
  // up.
  void ibody() {
    for (int i = 0; i < p->n_insns; ++i) {
      const pm_insn& in = p->insns[i];
      const int d = in.dst;
      const char* T = kSigned[in.op == PM_OP_CHECK || in.op == PM_OP_IF || in.op == PM_OP_RET ||
                                      in.op == PM_OP_FAIL || in.op == PM_OP_ELSE ||
                                      in.op == PM_OP_ENDIF ? 0 : w(d)];
      const char* U = kUnsigned[in.op == PM_OP_CHECK || in.op == PM_OP_IF || in.op == PM_OP_RET ||
                                        in.op == PM_OP_FAIL || in.op == PM_OP_ELSE ||
                                        in.op == PM_OP_ENDIF ? 0 : w(d)];
      auto L = [&](int r) { return "l" + std::to_string(r); };
      auto H = [&](int r) { return "h" + std::to_string(r); };
      auto cast = [&](const std::string& x) { return std::string("(") + T + ")(" + x + ")"; };
      auto ucast = [&](const std::string& x) { return std::string("(") + U + ")(" + x + ")"; };
      switch (in.op) {
        case PM_OP_CONST: {
          const std::string c = cst(w(d), in.lo, in.hi);
          o << "  " << L(d) << " = " << c << "; " << H(d) << " = " << c << ";\n";
          break;
        }
        case PM_OP_COORD:
          o << "  " << L(d) << " = (" << T << ")bl" << in.lo << "; " << H(d) << " = (" << T
            << ")bh" << in.lo << ";\n";
          break;
        case PM_OP_ADD:
          o << "  " << L(d) << " = " << cast(ucast(L(in.a)) + " + " + ucast(L(in.b))) << "; "
            << H(d) << " = " << cast(ucast(H(in.a)) + " + " + ucast(H(in.b))) << ";\n";
          break;
        case PM_OP_SUB:
          o << "  " << L(d) << " = " << cast(ucast(L(in.a)) + " - " + ucast(H(in.b))) << "; "
            << H(d) << " = " << cast(ucast(H(in.a)) + " - " + ucast(L(in.b))) << ";\n";
          break;
        case PM_OP_MUL: {
          o << "  { const " << T << " p0 = " << cast(ucast(L(in.a)) + " * " + ucast(L(in.b)))
            << ", p1 = " << cast(ucast(L(in.a)) + " * " + ucast(H(in.b)))
            << ", p2 = " << cast(ucast(H(in.a)) + " * " + ucast(L(in.b)))
            << ", p3 = " << cast(ucast(H(in.a)) + " * " + ucast(H(in.b))) << "; "
            << L(d) << " = pm_min2(pm_min2(p0, p1), pm_min2(p2, p3)); " << H(d)
            << " = pm_max2(pm_max2(p0, p1), pm_max2(p2, p3)); }\n";
          break;
        }
        case PM_OP_DIV: case PM_OP_MOD: {
          const int cw = std::max(w(d), std::max(w(in.a), w(in.b)));
          const char* ct = kSigned[cw];
          o << "  { const " << ct << " xa = (" << ct << ")" << L(in.a) << ", xb = (" << ct << ")"
            << H(in.a) << ", ya = (" << ct << ")" << L(in.b) << ", yb = (" << ct << ")"
            << H(in.b) << "; if (ya <= 0 && yb >= 0) return -1; ";
          if (in.op == PM_OP_DIV) {
            o << "const " << ct << " q0 = pm_fdiv(xa, ya), q1 = pm_fdiv(xa, yb), q2 = "
              << "pm_fdiv(xb, ya), q3 = pm_fdiv(xb, yb); " << L(d) << " = (" << T
              << ")pm_min2(pm_min2(q0, q1), pm_min2(q2, q3)); " << H(d) << " = (" << T
              << ")pm_max2(pm_max2(q0, q1), pm_max2(q2, q3)); }\n";
          } else {
            o << "if (ya == yb && pm_fdiv(xa, ya) == pm_fdiv(xb, ya)) { " << L(d) << " = (" << T
              << ")pm_fmod(xa, ya); " << H(d) << " = (" << T << ")pm_fmod(xb, ya); } "
              << "else if (ya > 0) { " << L(d) << " = 0; " << H(d) << " = (" << T
              << ")(yb - 1); } else { " << L(d) << " = (" << T << ")(ya + 1); " << H(d)
              << " = 0; } }\n";
          }
          break;
        }
        case PM_OP_GT: case PM_OP_LT: case PM_OP_EQ: {
          const int cw = std::max(w(in.a), w(in.b));
          const char* ct = kSigned[cw];
          const std::string la = std::string("(") + ct + ")" + L(in.a), ha = std::string("(") + ct + ")" + H(in.a);
          const std::string lb = std::string("(") + ct + ")" + L(in.b), hb = std::string("(") + ct + ")" + H(in.b);
          std::string yes, no;
          if (in.op == PM_OP_GT) { yes = la + " > " + hb; no = ha + " <= " + lb; }
          else if (in.op == PM_OP_LT) { yes = ha + " < " + lb; no = la + " >= " + hb; }
          else { yes = "(" + la + " == " + ha + " && " + lb + " == " + hb + " && " + la + " == " + lb + ")";
                 no = "(" + ha + " < " + lb + " || " + hb + " < " + la + ")"; }
          o << "  if (" << yes << ") { " << L(d) << " = 1; " << H(d) << " = 1; } else if (" << no
            << ") { " << L(d) << " = 0; " << H(d) << " = 0; } else { " << L(d) << " = 0; "
            << H(d) << " = 1; }\n";
          break;
        }
        case PM_OP_SELECT:
          o << "  if (" << L(in.a) << " > 0 || " << H(in.a) << " < 0) { " << L(d) << " = (" << T
            << ")" << L(in.b) << "; " << H(d) << " = (" << T << ")" << H(in.b) << "; } else if ("
            << L(in.a) << " == 0 && " << H(in.a) << " == 0) { " << L(d) << " = (" << T << ")"
            << L(in.c) << "; " << H(d) << " = (" << T << ")" << H(in.c) << "; } else { " << L(d)
            << " = pm_min2((" << T << ")" << L(in.b) << ", (" << T << ")" << L(in.c) << "); "
            << H(d) << " = pm_max2((" << T << ")" << H(in.b) << ", (" << T << ")" << H(in.c)
            << "); }\n";
          break;
        case PM_OP_MOV:
          o << "  " << L(d) << " = (" << T << ")" << L(in.a) << "; " << H(d) << " = (" << T
            << ")" << H(in.a) << ";\n";
          break;
        case PM_OP_CHECK: {
          const int cw = std::max(w(in.a), (in.lo < INT_MIN || in.hi > INT_MAX) ? 1 : 0);
          const char* ct = kSigned[cw];
          o << "  if ((" << ct << ")" << L(in.a) << " < (" << ct << ")" << in.lo << "LL || ("
            << ct << ")" << H(in.a) << " >= (" << ct << ")" << in.hi << "LL) return -1;\n";
          break;
        }
        case PM_OP_FAIL: o << "  return -1;\n"; break;
        case PM_OP_IF:
          o << "  { const int t_ = (" << L(in.a) << " > 0 || " << H(in.a) << " < 0) ? 1 : ("
            << L(in.a) << " == 0 && " << H(in.a) << " == 0) ? 0 : -1; if (t_ < 0) return -1; "
            << "if (t_) {\n";
          break;
        case PM_OP_ELSE: o << "  } else {\n"; break;
        case PM_OP_ENDIF: o << "  } }\n"; break;
        case PM_OP_RET:
          o << "  return (" << L(in.a) << " == " << H(in.a) << " && " << L(in.a) << " >= 0 && "
            << L(in.a) << " <= 0x7FFFFFFF) ? (int)" << L(in.a) << " : -1;\n";
          break;
      }
    }
  }

  // Width (0/1) of the implicit row-major index and coordinate types.
  bool implicit_wide() const {
    unsigned long long total = 1;
    for (int i = 0; i < p->n_coords; ++i) {
      unsigned long long e = (unsigned long long)std::max<long long>(p->extents[i], 1);
      if (e > 0 && total > ULLONG_MAX / e) return true;
      total *= e;
    }
    return total > 0xFFFFFFFFull;
  }

  // Diagnostic twin of pm_point for one failing point (pm_map_probe): on a
  // failure it stores the whole register file (each register as two 64-bit
  // words, sign-extended) so the host can format the reference's message with
  // the operand values of the failing site, e.g. "index (3, 8) out of range
  // for shape (2, 2)" (spaces.py:215-221, dsl/interp.py:207-214,245-258).
  std::string emit_probe() {
    const int k = p->n_coords;
    std::ostringstream q;
    o.str("");
    o << "// generated by libmapple_b200 (K1 failure probe)\n" << kPrelude;
    o << "#undef PM_FAIL\n#define PM_FAIL(s) do { *site_out = (s); goto pm_fail_; } while (0)\n";
    o << "__device__ __noinline__ int pm_point_probe(";
    for (int i = 0; i < k; ++i) o << "long long c" << i << ", ";
    o << "int* __restrict__ site_out, long long* __restrict__ dump) {\n";
    for (int r = 0; r < p->n_regs; ++r) o << "  " << kSigned[w(r)] << " r" << r << " = 0;\n";
    body();
    o << "  PM_FAIL(0xFFFF);\npm_fail_:\n";
    for (int r = 0; r < p->n_regs; ++r)
      o << "  dump[" << 2 * r << "] = (long long)r" << r << "; dump[" << 2 * r + 1
        << "] = (long long)((__int128)r" << r << " >> 64);\n";
    o << "  return -1;\n}\n\n";
    o << "extern \"C\" __global__ void pm_map_probe(const int* pts, long long idx, "
         "long long* dump, int* site) {\n  if (threadIdx.x | blockIdx.x) return;\n";
    if (p->implicit) {
      o << "  unsigned long long t = (unsigned long long)idx;\n";
      for (int i = k - 1; i >= 0; --i) {
        if (i == 0) o << "  long long c0 = (long long)t;\n";
        else
          o << "  long long c" << i << " = (long long)(t % " << p->extents[i] << "ULL); t /= "
            << p->extents[i] << "ULL;\n";
      }
      o << "  (void)pts;\n";
    } else {
      for (int i = 0; i < k; ++i) o << "  long long c" << i << " = pts[idx * " << k << " + " << i << "];\n";
    }
    o << "  int s = -1;\n  const int r = pm_point_probe(";
    for (int i = 0; i < k; ++i) o << "c" << i << ", ";
    o << "&s, dump);\n  site[0] = r < 0 ? s : -1;\n  site[1] = r;\n}\n";
    std::string out = o.str();
    o.str("");
    return out;
  }

  std::string emit() {
    const int k = p->n_coords;
    const bool impl = p->implicit != 0;
    o << "// generated by libmapple_b200 (K1 point program)\n" << kPrelude;
    o << "__device__ __forceinline__ int pm_point(";
    for (int i = 0; i < k; ++i) o << "long long c" << i << ", ";
    o << "int* __restrict__ site_out) {\n";
    if (max_w == 2 || p->n_regs > 0) {
      for (int r = 0; r < p->n_regs; ++r)
        o << "  " << kSigned[w(r)] << " r" << r << " = 0;\n";
    }
    body();
    o << "  PM_FAIL(0xFFFF);\n}\n\n";

    const bool wide = impl && implicit_wide();
    const char* it = wide ? "unsigned long long" : "unsigned";
    o << "__device__ __forceinline__ int pm_eval(long long lin, const int* __restrict__ pv, "
         "int* site) {\n";
    if (impl) {
      o << "  " << it << " t = (" << it << ")lin;\n";
      for (int i = k - 1; i >= 0; --i) {
        if (i == 0) {
          o << "  long long c0 = (long long)t;\n";
        } else {
          o << "  long long c" << i << " = (long long)(t % (" << it << ")" << p->extents[i]
            << "ULL); t /= (" << it << ")" << p->extents[i] << "ULL;\n";
        }
      }
      o << "  (void)pv;\n";
    } else {
      for (int i = 0; i < k; ++i) o << "  long long c" << i << " = pv[" << i << "];\n";
      o << "  (void)lin;\n";
    }
    o << "  return pm_point(";
    for (int i = 0; i < k; ++i) o << "c" << i << ", ";
    o << "site);\n}\n\n";

    // pm_tile_bin(lin0, cnt): the bin shared by every point of [lin0, lin0 + cnt),
    // proven over the row-major coordinate box of that range, or -1
    o << "__device__ __noinline__ int pm_tile_box(";
    for (int i = 0; i < k; ++i) o << "long long bl" << i << ", long long bh" << i << ", ";
    o << "int unused_) {\n";
    for (int r = 0; r < p->n_regs; ++r)
      o << "  " << kSigned[w(r)] << " l" << r << " = 0, h" << r << " = 0;\n";
    ibody();
    o << "  return -1;\n}\n\n";
    o << "__device__ __forceinline__ int pm_tile_bin(long long lin0, long long cnt) {\n";
    if (!impl) {
      o << "  (void)lin0; (void)cnt; return -1;\n}\n\n";
    } else {
      for (int i = 0; i < k; ++i) o << "  long long cf" << i << ", cl" << i << ";\n";
      for (int e = 0; e < 2 && k > 0; ++e) {
        const char* nm = e ? "cl" : "cf";
        o << "  { " << it << " t = (" << it << ")(lin0" << (e ? " + cnt - 1" : "") << ");\n";
        for (int i = k - 1; i >= 0; --i) {
          if (i == 0) {
            o << "    " << nm << "0 = (long long)t;\n";
          } else {
            o << "    " << nm << i << " = (long long)(t % (" << it << ")" << p->extents[i]
              << "ULL); t /= (" << it << ")" << p->extents[i] << "ULL;\n";
          }
        }
        o << "  }\n";
      }
      o << "  int diff_ = 0;\n";
      for (int i = 0; i < k; ++i) {
        o << "  long long bl" << i << ", bh" << i << ";\n";
        o << "  if (diff_) { bl" << i << " = 0; bh" << i << " = " << (p->extents[i] - 1)
          << "LL; } else { bl" << i << " = cf" << i << "; bh" << i << " = cl" << i
          << "; diff_ = cf" << i << " != cl" << i << "; }\n";
      }
      o << "  return pm_tile_box(";
      for (int i = 0; i < k; ++i) o << "bl" << i << ", bh" << i << ", ";
      o << "0);\n}\n\n";
    }

    const int K = impl ? 0 : k;
    o << "#define PM_K " << K << "\n";
    o << R"CUDA(
__device__ __forceinline__ void pm_report(unsigned long long* status, long long idx, int site) {
  atomicMin(status, ((unsigned long long)idx << 16) | (unsigned long long)(site & 0xFFFF));
}

extern "C" __global__ void __launch_bounds__(256)
pm_map_points(const int* __restrict__ pts, long long n, long long first,
              int* __restrict__ out, unsigned long long* __restrict__ status, int vec_ok) {
  const long long ngroups = (n + 3) >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += stride) {
    const long long i0 = g << 2;
    long long bad_idx = -1;
    int bad_site = 0;
    if (vec_ok && i0 + 4 <= n) {
#if PM_K > 0
      int buf[4 * PM_K];
      const int4* src = reinterpret_cast<const int4*>(pts + i0 * PM_K);
#pragma unroll
      for (int j = 0; j < PM_K; ++j) {
        int4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + j));
        buf[4 * j] = v.x; buf[4 * j + 1] = v.y; buf[4 * j + 2] = v.z; buf[4 * j + 3] = v.w;
      }
#else
      const int* buf = nullptr;
#endif
      int res[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        int site = 0;
        const int r = pm_eval(first + i0 + v, buf + v * PM_K, &site);
        if (r < 0 && bad_idx < 0) { bad_idx = i0 + v; bad_site = site; }
        res[v] = r;
      }
      asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};"
                   :: "l"(out + i0), "r"(res[0]), "r"(res[1]), "r"(res[2]), "r"(res[3]) : "memory");
    } else {
      for (int v = 0; v < 4; ++v) {
        const long long i = i0 + v;
        if (i >= n) break;
        int site = 0;
        const int r = pm_eval(first + i, pts + i * PM_K, &site);
        if (r < 0 && bad_idx < 0) { bad_idx = i; bad_site = site; }
        out[i] = r;
      }
    }
    if (bad_idx >= 0) pm_report(status, first + bad_idx, bad_site);
  }
}
)CUDA";
    return o.str();
  }
};

// Fused map + partition kernels: the key of a point is its processor id,
// computed in registers by pm_eval -- the id array of K1 is never read back.
const char* kFused = R"CUDA(
#include "partition_device.cuh"

struct PmMapKey {
  const int* pts;
  long long first;
  unsigned long long* status;
  int* out;  // optional processor-id output (scatter pass)
  int nbins;
  static constexpr bool kVec4 = false;
  static constexpr bool kPeek = true;
  __device__ __forceinline__ int tile_bin(long long base, long long count) const {
    return pm_tile_bin(first + base, count);
  }
  __device__ __forceinline__ int peek(long long i) const {
    int site = 0;
    return pm_eval(first + i, pts + i * PM_K, &site);
  }
  __device__ __forceinline__ void uniform(long long base, int count, int b) const {
    if (out)
      for (int k = threadIdx.x; k < count; k += blockDim.x) out[base + k] = b;
  }
  __device__ __forceinline__ int operator()(long long i) const {
    int site = 0;
    int r = pm_eval(first + i, pts + i * PM_K, &site);
    if (r >= nbins) { site = 0xFFFE; r = -1; }
    if (r < 0) pm_report(status, first + i, site);
    if (out) out[i] = r;
    return r;
  }
};

struct PmPermSink {
  int* __restrict__ perm;
  long long base;
  __device__ __forceinline__ void put(int, long long pos, long long i) const {
    perm[pos] = (int)(base + i);
  }
  __device__ __forceinline__ void put_run(int, long long pos, long long i, int count) const {
    pmdev::store_iota(perm + pos, (int)(base + i), count);
  }
};

// per-bin destination: tab[2 b] = int32 pointer (possibly a peer GPU's), tab[2 b + 1] =
// element shift applied to the local grouped position
struct PmPeerSink {
  const long long* __restrict__ tab;
  long long base;
  __device__ __forceinline__ void put(int b, long long pos, long long i) const {
    int* p = reinterpret_cast<int*>(__ldg(tab + 2 * b));
    p[pos + __ldg(tab + 2 * b + 1)] = (int)(base + i);
  }
  __device__ __forceinline__ void put_run(int b, long long pos, long long i, int count) const {
    int* p = reinterpret_cast<int*>(__ldg(tab + 2 * b));
    pmdev::store_iota(p + pos + __ldg(tab + 2 * b + 1), (int)(base + i), count);
  }
};

extern "C" __global__ void __launch_bounds__(256)
pm_map_hist(const int* pts, long long n, long long first, int nbins, long long ntiles,
            long long* __restrict__ hist, unsigned long long* status) {
  extern __shared__ __align__(16) int smem_words[];
  const PmMapKey key{pts, first, status, nullptr, nbins};
  pmdev::small_hist_proof(key, n, nbins, ntiles, hist, smem_words);
}

extern "C" __global__ void __launch_bounds__(256, 6)
pm_map_scatter(const int* pts, long long n, long long first, int nbins, long long ntiles,
               const long long* __restrict__ pos0, unsigned long long* status, int* out,
               int* perm, long long base) {
  extern __shared__ __align__(16) int smem_words[];
  const PmMapKey key{pts, first, status, out, nbins};
  pmdev::small_scatter_tiles<pmdev::kScatterTiles>(key, PmPermSink{perm, base}, n, nbins, ntiles, pos0,
                                                   smem_words,
                                                   (long long)blockIdx.x * pmdev::kScatterTiles);
}

extern "C" __global__ void __launch_bounds__(256, 6)
pm_map_scatter_peer(const int* pts, long long n, long long first, int nbins, long long ntiles,
                    const long long* __restrict__ pos0, unsigned long long* status, int* out,
                    const long long* tab, long long base) {
  extern __shared__ __align__(16) int smem_words[];
  const PmMapKey key{pts, first, status, out, nbins};
  pmdev::small_scatter_tiles<pmdev::kScatterTiles>(key, PmPeerSink{tab, base}, n, nbins, ntiles, pos0,
                                                   smem_words,
                                                   (long long)blockIdx.x * pmdev::kScatterTiles);
}
)CUDA";

std::mutex g_cache_mu;
std::unordered_map<std::string, std::vector<char>> g_cubins;

// Device half of the small-bin stable partition (partition_device.cuh), as text
// for NVRTC; build/partition_device_src.inc is generated by the Makefile.
const char kPartitionDevice[] =
#include "partition_device_src.inc"
    ;

int nvrtc_compile(const std::string& src, std::vector<char>* cubin, bool with_partition = false) {
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cubins.find(with_partition ? "P" + src : src);
    if (it != g_cubins.end()) {
      *cubin = it->second;
      return PM_OK;
    }
  }
  nvrtcProgram prog;
  const char* hdr_src[] = {kPartitionDevice};
  const char* hdr_name[] = {"partition_device.cuh"};
  if (nvrtcCreateProgram(&prog, src.c_str(), "pm_point_program.cu", with_partition ? 1 : 0,
                         with_partition ? hdr_src : nullptr,
                         with_partition ? hdr_name : nullptr) != NVRTC_SUCCESS)
    return set_error("nvrtcCreateProgram failed"), PM_ERR_NVRTC;
#define PM_STR2(x) #x
#define PM_STR(x) PM_STR2(x)
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-device-int128", "-lineinfo",
                        "-default-device", "-w", "-DPM_SCATTER_TILES=" PM_STR(PM_SCATTER_TILES)};
  nvrtcResult rc = nvrtcCompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    set_error("NVRTC compile failed: %s\n%.4000s", nvrtcGetErrorString(rc), log.c_str());
    return PM_ERR_NVRTC;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  if (const char* dump = getenv("PM_DUMP_CUBIN")) {  // debugging: inspect with cuobjdump
    if (FILE* f = fopen(dump, "wb")) {
      fwrite(cubin->data(), 1, cubin->size(), f);
      fclose(f);
    }
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cubins.emplace(with_partition ? "P" + src : src, *cubin);
  return PM_OK;
}

int generate(const pm_program* prog, std::string* out, std::string* probe = nullptr) {
  if (!prog || (prog->n_insns > 0 && !prog->insns) || (prog->n_regs > 0 && !prog->reg_width))
    return set_error("null program"), PM_ERR_INVALID;
  if (prog->implicit && prog->n_coords > 0 && !prog->extents)
    return set_error("implicit program without extents"), PM_ERR_INVALID;
  Gen g;
  g.p = prog;
  int rc = g.check();
  if (rc) return rc;
  if (probe) *probe = g.emit_probe();
  *out = g.emit();
  return PM_OK;
}

}  // namespace

int plan_fused(pm_plan* p) {
  std::lock_guard<std::mutex> lk(p->fused_mu);
  if (p->fused_ready) return PM_OK;
  std::vector<char> cubin;
  int rc = nvrtc_compile(p->src + kFused, &cubin, true);
  if (rc) return rc;
  const Driver* d = driver();
  if (!d) return PM_ERR_CUDA;
  PM_CU_TRY(d->moduleLoadData(&p->fused_mod, cubin.data()));
  PM_CU_TRY(d->moduleGetFunction(&p->fn_hist, p->fused_mod, "pm_map_hist"));
  PM_CU_TRY(d->moduleGetFunction(&p->fn_scatter, p->fused_mod, "pm_map_scatter"));
  PM_CU_TRY(d->moduleGetFunction(&p->fn_scatter_peer, p->fused_mod, "pm_map_scatter_peer"));
  p->fused_ready = true;
  return PM_OK;
}

}  // namespace pm

extern "C" {

int pm_codegen(const pm_program* prog, char* buf, size_t cap, size_t* len) {
  std::string src;
  int rc = pm::generate(prog, &src);
  if (rc) return rc;
  if (len) *len = src.size();
  if (buf && cap) {
    size_t n = std::min(cap - 1, src.size());
    std::memcpy(buf, src.data(), n);
    buf[n] = '\0';
  }
  return PM_OK;
}

int pm_compile_check(const pm_program* prog) {
  std::string src;
  int rc = pm::generate(prog, &src);
  if (rc) return rc;
  std::vector<char> cubin;
  return pm::nvrtc_compile(src, &cubin);
}

int pm_compile_check_probe(const pm_program* prog) {
  std::string src, probe;
  int rc = pm::generate(prog, &src, &probe);
  if (rc) return rc;
  std::vector<char> cubin;
  return pm::nvrtc_compile(probe, &cubin);
}

int pm_compile_check_fused(const pm_program* prog) {
  std::string src;
  int rc = pm::generate(prog, &src);
  if (rc) return rc;
  std::vector<char> cubin;
  return pm::nvrtc_compile(src + pm::kFused, &cubin, true);
}

int pm_plan_create(const pm_program* prog, pm_plan** out) {
  if (!out) return pm::set_error("null out"), PM_ERR_INVALID;
  *out = nullptr;
  std::string src, probe;
  int rc = pm::generate(prog, &src, &probe);
  if (rc) return rc;
  std::vector<char> cubin;
  rc = pm::nvrtc_compile(src, &cubin);
  if (rc) return rc;
  const pm::Driver* d = pm::driver();
  if (!d) return PM_ERR_CUDA;
  PM_CUDA_TRY(cudaFree(nullptr));  // make sure the primary context exists
  pm_plan* p = new pm_plan();
  PM_CUDA_TRY(cudaGetDevice(&p->device));
  CUresult r = d->moduleLoadData(&p->mod, cubin.data());
  if (r != CUDA_SUCCESS) {
    delete p;
    pm::set_error("cuModuleLoadData failed: CUresult %d", (int)r);
    return PM_ERR_CUDA;
  }
  r = d->moduleGetFunction(&p->fn, p->mod, "pm_map_points");
  if (r != CUDA_SUCCESS) {
    d->moduleUnload(p->mod);
    delete p;
    pm::set_error("cuModuleGetFunction failed: CUresult %d", (int)r);
    return PM_ERR_CUDA;
  }
  p->n_coords = prog->n_coords;
  p->implicit = prog->implicit;
  p->n_regs = prog->n_regs;
  p->src = src;
  p->probe_src = probe;
  *out = p;
  return PM_OK;
}

void pm_plan_destroy(pm_plan* plan) {
  if (!plan) return;
  const pm::Driver* d = pm::driver();
  if (d && plan->mod) d->moduleUnload(plan->mod);
  if (d && plan->fused_mod) d->moduleUnload(plan->fused_mod);
  if (d && plan->probe_mod) d->moduleUnload(plan->probe_mod);
  delete plan;
}

int pm_map_batch(const pm_plan* plan, const int32_t* points, int64_t n, int64_t first,
                 int32_t* out_proc, uint64_t* status, void* stream) {
  if (!plan || !out_proc || !status || n < 0 || first < 0)
    return pm::set_error("pm_map_batch: bad arguments"), PM_ERR_INVALID;
  if (!plan->implicit && plan->n_coords > 0 && !points)
    return pm::set_error("pm_map_batch: explicit plan needs points"), PM_ERR_INVALID;
  if (first + n >= (1LL << 47)) return pm::set_error("pm_map_batch: index too large"), PM_ERR_UNSUPPORTED;
  if (n == 0) return PM_OK;
  const pm::Driver* d = pm::driver();
  if (!d) return PM_ERR_CUDA;
  const int threads = 256;
  const long long groups = (n + 3) / 4;
  long long blocks = (groups + threads - 1) / threads;
  // 4 grid-stride iterations (16 points) per thread: a pure store stream runs best with
  // short-lived CTAs that still write more than one group each -- 32768^2 block launch:
  // 0.71 ms persistent (8 CTAs / SM), 0.96 ms one group per thread, 0.585 ms here = 7.3 TB/s,
  // the fill_ ceiling (tools/k1_ab.sh)
  const long long iters = 4;
  blocks = (groups + threads * iters - 1) / (threads * iters);
  if (blocks > (1LL << 30)) blocks = 1LL << 30;  // the kernel's grid-stride loop covers the rest
  int vec_ok = ((uintptr_t)out_proc % 16 == 0) &&
               (plan->implicit || plan->n_coords == 0 || (uintptr_t)points % 16 == 0);
  const int32_t* pts = points;
  long long nn = n, ff = first;
  void* args[] = {(void*)&pts, (void*)&nn, (void*)&ff, (void*)&out_proc, (void*)&status,
                  (void*)&vec_ok};
  PM_CU_TRY(d->launchKernel(plan->fn, (unsigned)blocks, 1, 1, threads, 1, 1, 0,
                            (CUstream)stream, args, nullptr));
  return PM_OK;
}

int pm_plan_regs(const pm_plan* plan) { return plan ? plan->n_regs : -1; }

int pm_map_probe(pm_plan* plan, const int32_t* points, int64_t index, int64_t* dump,
                 int32_t* site, void* stream) {
  if (!plan || !dump || !site || index < 0 || (!plan->implicit && plan->n_coords > 0 && !points))
    return pm::set_error("pm_map_probe: bad arguments"), PM_ERR_INVALID;
  const pm::Driver* d = pm::driver();
  if (!d) return PM_ERR_CUDA;
  {
    std::lock_guard<std::mutex> lk(plan->fused_mu);
    if (!plan->probe_fn) {  // compiled on the first failure only
      std::vector<char> cubin;
      int rc = pm::nvrtc_compile(plan->probe_src, &cubin);
      if (rc) return rc;
      PM_CU_TRY(d->moduleLoadData(&plan->probe_mod, cubin.data()));
      PM_CU_TRY(d->moduleGetFunction(&plan->probe_fn, plan->probe_mod, "pm_map_probe"));
    }
  }
  const int32_t* pts = points;
  long long idx = index;
  void* args[] = {(void*)&pts, (void*)&idx, (void*)&dump, (void*)&site};
  PM_CU_TRY(d->launchKernel(plan->probe_fn, 1, 1, 1, 32, 1, 1, 0, (CUstream)stream, args,
                            nullptr));
  return PM_OK;
}

}  // extern "C"
