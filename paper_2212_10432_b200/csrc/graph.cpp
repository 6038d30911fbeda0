// Operator Graph IR: DSL parser, canonical printer, dependency validator.
//
// Operators: converting / mapping / implementing stages (§IV-A; draft P:11-31).
// Dependencies: "operators prefixed with BMW and BMT cannot be followed by operators
// prefixed with BMTB" plus the stage rules "COMPRESS, the last operator in
// converting stage" and "mapping stage always begins after the COMPRESS operator"
// (P:279).  The full rule table R1..R11 is reading A16.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>

#include "internal.h"

namespace as {

namespace {

enum PType { P_INT, P_FLOAT, P_LIST, P_SCOPE };
struct PSpec {
  const char* key;
  PType t;
  bool has_default;
  double def;
  const char* sdef;
};
struct OpSpec {
  const char* name;
  int stage;  // 0 converting, 1 COMPRESS, 2 mapping, 3 implementing, 4 terminal (DIA/DENSE)
  std::vector<PSpec> ps;
};

const std::vector<OpSpec>& specs() {
  static const std::vector<OpSpec> S = {
      {"ROW_DIV", 0, {{"cuts", P_LIST, false, 0, nullptr}}},
      {"COL_DIV", 0, {{"cuts", P_LIST, false, 0, nullptr}}},
      {"SORT", 0, {}},
      {"SORT_SUB", 0, {{"g", P_INT, false, 0, nullptr}}},
      {"BIN", 0, {{"t", P_LIST, false, 0, nullptr}}},
      {"DIA_DECOM", 0, {{"theta", P_FLOAT, false, 0, nullptr}, {"max", P_INT, true, 8, nullptr}}},
      {"DENSE_DECOM", 0, {{"b", P_INT, false, 0, nullptr}, {"theta", P_FLOAT, false, 0, nullptr}}},
      {"HYB_DECOM", 0, {{"w", P_INT, false, 0, nullptr}}},
      {"COMPRESS", 1, {}},
      {"DIA", 4, {}},
      {"DENSE", 4, {}},
      {"BMTB_ROW_BLOCK", 2, {{"rows", P_INT, false, 0, nullptr}}},
      {"BMTB_NNZ_BLOCK", 2, {{"nnz", P_INT, false, 0, nullptr}}},
      {"BMW_ROW_BLOCK", 2, {{"rows", P_INT, false, 0, nullptr}}},
      {"BMW_NNZ_BLOCK", 2, {{"nnz", P_INT, false, 0, nullptr}}},
      {"BMT_ROW_BLOCK", 2, {{"rows", P_INT, false, 0, nullptr}}},
      {"BMT_NNZ_BLOCK", 2, {{"nnz", P_INT, false, 0, nullptr}}},
      {"BMT_PAD", 2, {{"scope", P_SCOPE, true, 0, "GLOBAL"}, {"vec", P_INT, true, 0, nullptr}}},
      {"SORT_BMTB", 2, {}},
      {"SET_RESOURCE", 3,
       {{"tpb", P_INT, true, 256, nullptr}, {"grid", P_INT, true, 0, nullptr}, {"stages", P_INT, true, 2, nullptr},
        {"xcache", P_INT, true, 0, nullptr}, {"stream", P_INT, true, 0, nullptr}}},
      {"THREAD_TOTAL_RED", 3, {}},
      {"THREAD_BITMAP_RED_G", 3, {}},
      {"WARP_TOTAL_RED", 3, {}},
      {"WARP_BITMAP_RED", 3, {}},
      {"WARP_SEG_ADD_RED", 3, {}},
      {"SHMEM_TOTAL_RED", 3, {}},
      {"SHMEM_OFFSET_RED", 3, {}},
      {"GMEM_ATOM_RED", 3, {}},
  };
  return S;
}

const OpSpec* find_spec(const std::string& n) {
  for (auto& s : specs())
    if (n == s.name) return &s;
  return nullptr;
}

// Draft / typo aliases, reading A37 (P:29 footnote).
std::string canonical_name(const std::string& n) {
  static const std::map<std::string, std::string> A = {
      {"WARP_SEG_RED", "WARP_SEG_ADD_RED"},     {"THREAD_BITMAP_RED", "THREAD_BITMAP_RED_G"},
      {"SET_RESOURCES", "SET_RESOURCE"},        {"BMTB_ROW_DIV", "BMTB_ROW_BLOCK"},
      {"THREAD_TOTOAL_RED", "THREAD_TOTAL_RED"}};
  auto it = A.find(n);
  return it == A.end() ? n : it->second;
}

// level of a blocking op / reduction: 0 BMTB, 1 BMW, 2 BMT, 3 GMEM
int red_level(const std::string& n) {
  if (n.rfind("THREAD_", 0) == 0) return 2;
  if (n.rfind("WARP_", 0) == 0) return 1;
  if (n.rfind("SHMEM_", 0) == 0) return 0;
  if (n == "GMEM_ATOM_RED") return 3;
  return -1;
}
int block_level(const std::string& n) {
  if (n.rfind("BMTB_", 0) == 0) return 0;
  if (n.rfind("BMW_", 0) == 0) return 1;
  if (n.rfind("BMT_", 0) == 0) return 2;
  return -1;
}
// reduction order THREAD(0) -> WARP(1) -> SHMEM(2) -> GMEM(3)
int red_rank(int lvl) { return lvl == 2 ? 0 : lvl == 1 ? 1 : lvl == 0 ? 2 : 3; }

// ------------------------------------------------------------------ tokenizer / parser
struct Tok {
  enum K { NUM, ID, P, END } k;
  std::string s;
};

std::vector<Tok> tokenize(const std::string& t) {
  std::vector<Tok> out;
  size_t i = 0;
  while (i < t.size()) {
    char c = t[i];
    if (std::isspace((unsigned char)c)) {
      ++i;
      continue;
    }
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < t.size() && (std::isalnum((unsigned char)t[j]) || t[j] == '_')) ++j;
      out.push_back({Tok::ID, t.substr(i, j - i)});
      i = j;
      continue;
    }
    if (std::isdigit((unsigned char)c) || c == '-' || c == '+' || c == '.') {
      size_t j = i;
      if (t[j] == '-' || t[j] == '+') ++j;
      size_t d0 = j;
      while (j < t.size() && std::isdigit((unsigned char)t[j])) ++j;
      if (j < t.size() && t[j] == '.') {
        ++j;
        while (j < t.size() && std::isdigit((unsigned char)t[j])) ++j;
      }
      if (j == d0 || (j == d0 + 1 && t[d0] == '.')) fail(AS_ERR_GRAPH_PARSE, "bad number at " + std::to_string(i));
      if (j < t.size() && (t[j] == 'e' || t[j] == 'E')) {
        size_t k = j + 1;
        if (k < t.size() && (t[k] == '-' || t[k] == '+')) ++k;
        size_t k0 = k;
        while (k < t.size() && std::isdigit((unsigned char)t[k])) ++k;
        if (k > k0) j = k;
      }
      out.push_back({Tok::NUM, t.substr(i, j - i)});
      i = j;
      continue;
    }
    if (std::strchr("();{}|,=[]", c)) {
      out.push_back({Tok::P, std::string(1, c)});
      ++i;
      continue;
    }
    fail(AS_ERR_GRAPH_PARSE, std::string("bad character '") + c + "' at " + std::to_string(i));
  }
  out.push_back({Tok::END, ""});
  return out;
}

bool is_int_text(const std::string& s) {
  size_t i = (s[0] == '-' || s[0] == '+') ? 1 : 0;
  if (i >= s.size()) return false;
  for (; i < s.size(); ++i)
    if (!std::isdigit((unsigned char)s[i])) return false;
  return true;
}

struct RawVal {
  int kind;  // 0 num, 1 list, 2 ident
  std::string num;
  std::vector<std::string> list;
  std::string id;
};

struct Parser {
  std::vector<Tok> t;
  size_t i = 0;
  const Tok& peek(size_t d = 0) { return t[std::min(i + d, t.size() - 1)]; }
  bool isp(const char* p, size_t d = 0) { return peek(d).k == Tok::P && peek(d).s == p; }
  void expect(const char* p) {
    if (!isp(p)) fail(AS_ERR_GRAPH_PARSE, std::string("expected '") + p + "', got '" + peek().s + "'");
    ++i;
  }
  Seq seq() {
    Seq s;
    s.push_back(op());
    while (isp(";")) {
      ++i;
      s.push_back(op());
    }
    return s;
  }
  RawVal value() {
    RawVal v;
    if (isp("[")) {
      ++i;
      v.kind = 1;
      if (!isp("]")) {
        while (true) {
          if (peek().k != Tok::NUM) fail(AS_ERR_GRAPH_PARSE, "number expected in list");
          v.list.push_back(peek().s);
          ++i;
          if (isp(",")) {
            ++i;
            continue;
          }
          break;
        }
      }
      expect("]");
      return v;
    }
    if (peek().k == Tok::NUM) {
      v.kind = 0;
      v.num = peek().s;
      ++i;
      return v;
    }
    if (peek().k == Tok::ID) {
      v.kind = 2;
      v.id = peek().s;
      ++i;
      return v;
    }
    fail(AS_ERR_GRAPH_PARSE, "bad value '" + peek().s + "'");
  }
  Op op() {
    if (peek().k != Tok::ID) fail(AS_ERR_GRAPH_PARSE, "operator name expected, got '" + peek().s + "'");
    Op o;
    o.name = canonical_name(peek().s);
    ++i;
    const OpSpec* sp = find_spec(o.name);
    if (!sp) fail(AS_ERR_GRAPH_PARSE, "unknown operator " + o.name);
    std::vector<RawVal> pos;
    std::vector<std::pair<std::string, RawVal>> kw;
    if (isp("(")) {
      ++i;
      if (!isp(")")) {
        while (true) {
          if (peek().k == Tok::ID && isp("=", 1)) {
            std::string key = peek().s;
            i += 2;
            for (auto& p : kw)
              if (p.first == key) fail(AS_ERR_GRAPH_PARSE, "duplicate key " + key);
            kw.push_back({key, value()});
          } else {
            if (!kw.empty()) fail(AS_ERR_GRAPH_PARSE, "positional after keyword");
            pos.push_back(value());
          }
          if (isp(",")) {
            ++i;
            continue;
          }
          break;
        }
      }
      expect(")");
    }
    if (pos.size() > sp->ps.size()) fail(AS_ERR_GRAPH_PARSE, o.name + ": too many arguments");
    std::vector<const RawVal*> got(sp->ps.size(), nullptr);
    for (size_t a = 0; a < pos.size(); ++a) got[a] = &pos[a];
    for (auto& p : kw) {
      size_t j = 0;
      for (; j < sp->ps.size(); ++j)
        if (p.first == sp->ps[j].key) break;
      if (j == sp->ps.size()) fail(AS_ERR_GRAPH_PARSE, o.name + ": unknown parameter " + p.first);
      if (got[j]) fail(AS_ERR_GRAPH_PARSE, o.name + ": " + p.first + " given twice");
      got[j] = &p.second;
    }
    for (size_t j = 0; j < sp->ps.size(); ++j) {
      const PSpec& ps = sp->ps[j];
      Value v;
      if (!got[j]) {
        if (!ps.has_default) fail(AS_ERR_GRAPH_PARSE, o.name + ": missing parameter " + ps.key);
        if (ps.t == P_SCOPE) {
          v.k = Value::IDENT;
          v.s = ps.sdef;
        } else if (ps.t == P_FLOAT) {
          v.k = Value::FLOAT;
          v.f = ps.def;
        } else {
          v.k = Value::INT;
          v.i = (int64_t)ps.def;
        }
      } else {
        const RawVal& r = *got[j];
        auto as_int = [&](const std::string& s) -> int64_t {
          if (is_int_text(s)) return std::stoll(s);
          double d = std::stod(s);
          if (d != std::floor(d)) fail(AS_ERR_GRAPH_PARSE, o.name + "." + ps.key + ": integer expected");
          return (int64_t)d;
        };
        if (ps.t == P_INT) {
          if (r.kind != 0) fail(AS_ERR_GRAPH_PARSE, o.name + "." + ps.key + ": integer expected");
          v.k = Value::INT;
          v.i = as_int(r.num);
        } else if (ps.t == P_FLOAT) {
          if (r.kind != 0) fail(AS_ERR_GRAPH_PARSE, o.name + "." + ps.key + ": number expected");
          v.k = Value::FLOAT;
          v.f = std::stod(r.num);
        } else if (ps.t == P_LIST) {
          v.k = Value::LIST;
          if (r.kind == 0)
            v.l.push_back(as_int(r.num));
          else if (r.kind == 1)
            for (auto& s : r.list) v.l.push_back(as_int(s));
          else
            fail(AS_ERR_GRAPH_PARSE, o.name + "." + ps.key + ": integer list expected");
        } else {
          if (r.kind != 2 || (r.id != "GLOBAL" && r.id != "BMTB" && r.id != "BMW"))
            fail(AS_ERR_GRAPH_PARSE, o.name + "." + ps.key + ": GLOBAL|BMTB|BMW expected");
          v.k = Value::IDENT;
          v.s = r.id;
        }
      }
      o.params.push_back({ps.key, v});
    }
    if (isp("{")) {
      ++i;
      o.br.push_back(seq());
      while (isp("|")) {
        ++i;
        o.br.push_back(seq());
      }
      expect("}");
    }
    return o;
  }
};

int64_t n_branches(const Op& o) {
  if (o.name == "ROW_DIV" || o.name == "COL_DIV") return (int64_t)o.getl("cuts").size() + 1;
  if (o.name == "BIN") return (int64_t)o.getl("t").size() + 1;
  if (o.name == "DIA_DECOM" || o.name == "DENSE_DECOM" || o.name == "HYB_DECOM") return 2;
  return 0;
}

void expand(Seq& s) {
  for (auto& o : s) {
    for (auto& b : o.br) expand(b);
    if ((o.name == "ROW_DIV" || o.name == "COL_DIV" || o.name == "BIN" || o.name == "HYB_DECOM") && o.br.size() == 1) {
      int64_t k = n_branches(o);
      Seq one = o.br[0];
      o.br.assign((size_t)k, one);
    }
  }
}

void number(Seq& s, int& c) {
  for (auto& o : s) {
    o.id = c++;
    for (auto& b : o.br) number(b, c);
  }
}

[[noreturn]] void illegal(const char* rule, int node, const std::string& msg) {
  fail(AS_ERR_GRAPH_ILLEGAL, std::string(rule) + " at node " + std::to_string(node) + ": " + msg);
}

void check_params(const Op& o) {
  auto bad = [&](const std::string& m) { illegal("PARAM", o.id, o.name + ": " + m); };
  if (o.name == "ROW_DIV" || o.name == "COL_DIV") {
    auto& c = o.getl("cuts");
    if (c.empty() || c[0] <= 0) bad("cuts must be non-empty, positive, strictly increasing");
    for (size_t i = 1; i < c.size(); ++i)
      if (c[i] <= c[i - 1]) bad("cuts must be non-empty, positive, strictly increasing");
  } else if (o.name == "BIN") {
    auto& t = o.getl("t");
    if (t.empty() || t[0] < 1) bad("thresholds must be non-empty, >= 1, strictly ascending");
    for (size_t i = 1; i < t.size(); ++i)
      if (t[i] <= t[i - 1]) bad("thresholds must be non-empty, >= 1, strictly ascending");
  } else if (o.name == "SORT_SUB") {
    if (o.geti("g") < 2) bad("g >= 2");
  } else if (o.name == "DIA_DECOM") {
    double th = o.getf("theta");
    if (!(th > 0.0 && th <= 1.0) || o.geti("max") < 1) bad("0 < theta <= 1, max >= 1");
  } else if (o.name == "DENSE_DECOM") {
    double th = o.getf("theta");
    if (!(th > 0.0 && th <= 1.0) || o.geti("b") < 1) bad("0 < theta <= 1, b >= 1");
  } else if (o.name == "HYB_DECOM") {
    if (o.geti("w") < 1) bad("w >= 1");
  } else if (block_level(o.name) >= 0 && o.name.size() > 6 && o.name.substr(o.name.size() - 6) == "_BLOCK") {
    int64_t v = o.params[0].second.i;
    if (v < 1) bad("block size >= 1");
  } else if (o.name == "BMT_PAD") {
    int64_t v = o.geti("vec");
    if (v != 0 && v != 1 && v != 2 && v != 4) bad("vec in {0,1,2,4}");
  } else if (o.name == "SET_RESOURCE") {
    int64_t tpb = o.geti("tpb");
    int64_t st = o.geti("stages");
    const int64_t xc = o.geti("xcache");
    const int64_t sq = o.geti("stream");
    if (tpb < 32 || tpb > 1024 || tpb % 32 || o.geti("grid") < 0 || (st != 0 && st != 2) || xc < 0 || xc > 65536 ||
        sq < 0 || sq > 3)
      bad("tpb multiple of 32 in [32,1024], grid >= 0, stages in {0,2}, xcache in [0,65536], stream in [0,3]");
  }
}

bool is_sort_family(const std::string& n) { return n == "SORT" || n == "SORT_SUB" || n == "BIN"; }

// Validate one root-to-leaf path (or a prefix ending in a branching op when partial).
void check_path(const std::vector<const Op*>& path, bool partial) {
  int stage = 0, n_compress = 0, n_set = 0;
  std::set<std::string> conv;
  bool sorted = false, pad = false, sort_bmtb = false;
  std::vector<int> levels;
  int lkind[3] = {-1, -1, -1};  // 0 ROW, 1 NNZ
  std::vector<int> reds;
  for (const Op* op : path) {
    const OpSpec* sp = find_spec(op->name);
    int st = sp->stage;
    if (st >= 2 && n_compress == 0) illegal("R1", op->id, op->name + " before COMPRESS");
    if (st < stage || (st == 1 && stage >= 1)) illegal("R1", op->id, op->name + " out of stage order");
    stage = st;
    if (st == 0) {
      if (conv.count(op->name)) illegal("R11", op->id, op->name + " twice on a path");
      if (is_sort_family(op->name)) {
        for (auto& c : conv)
          if (is_sort_family(c)) illegal("R11", op->id, "SORT/SORT_SUB/BIN are mutually exclusive");
      }
      if ((op->name == "DIA_DECOM" || op->name == "DENSE_DECOM") && sorted)
        illegal("R10", op->id, op->name + " after a row permutation");
      if (is_sort_family(op->name)) sorted = true;
      conv.insert(op->name);
    } else if (st == 1) {
      ++n_compress;
    } else if (st == 2) {
      int bl = block_level(op->name);
      bool is_block = op->name.size() > 6 && op->name.substr(op->name.size() - 6) == "_BLOCK";
      if (is_block) {
        if (lkind[bl] >= 0) illegal("R4", op->id, std::string("second blocking at the same level"));
        if (!levels.empty() && levels.back() > bl) illegal("R3", op->id, op->name + " after a finer level");
        if (pad) illegal("R5", op->id, "blocking after BMT_PAD");
        levels.push_back(bl);
        lkind[bl] = op->name.find("_NNZ_") != std::string::npos ? 1 : 0;
      } else if (op->name == "BMT_PAD") {
        if (pad) illegal("R5", op->id, "BMT_PAD twice");
        if (lkind[2] < 0) illegal("R5", op->id, "BMT_PAD needs BMT blocking");
        const std::string& sc = op->gets("scope");
        if (sc == "BMTB" && lkind[0] < 0) illegal("R5", op->id, "BMT_PAD scope BMTB needs BMTB blocking");
        if (sc == "BMW" && lkind[1] < 0) illegal("R5", op->id, "BMT_PAD scope BMW needs BMW blocking");
        pad = true;
      } else if (op->name == "SORT_BMTB") {
        if (sort_bmtb) illegal("R5", op->id, "SORT_BMTB twice");
        if (lkind[0] != 0 || lkind[1] >= 0 || lkind[2] >= 0)
          illegal("R5", op->id, "SORT_BMTB needs BMTB_ROW_BLOCK and precedes BMW/BMT");
        sort_bmtb = true;
      }
    } else if (st == 3) {
      if (op->name == "SET_RESOURCE") {
        if (++n_set > 1) illegal("R9", op->id, "SET_RESOURCE twice");
        continue;
      }
      int rl = red_level(op->name);
      if (rl < 3 && lkind[rl] < 0) illegal("R6", op->id, op->name + " needs blocking at its level");
      if (!reds.empty() && red_rank(reds.back()) >= red_rank(rl)) illegal("R6", op->id, op->name + " out of reduction order");
      reds.push_back(rl);
    }
  }
  if (partial) {
    if (n_compress) illegal("R1", path.back()->id, "branching after COMPRESS");
    return;
  }
  int nid = path.empty() ? 0 : path.back()->id;
  if (n_compress != 1) illegal("R2", nid, "path needs exactly one COMPRESS");
  if (reds.empty() || reds.back() != 3) illegal("R7", nid, "path must end with GMEM_ATOM_RED");
  if (path.back()->name != "GMEM_ATOM_RED") illegal("R7", nid, "GMEM_ATOM_RED must be the last operator");
}

void check_terminal(const Op& dec, const Seq& b) {
  const char* want = dec.name == "DIA_DECOM" ? "DIA" : "DENSE";
  if (b.empty() || b[0].name != want) illegal("R8", dec.id, std::string("first branch must start with ") + want);
  for (size_t i = 1; i < b.size(); ++i) {
    if (b[i].name != "SET_RESOURCE" || !b[i].br.empty())
      illegal("R8", b[i].id, std::string(want) + " branch admits only SET_RESOURCE");
    check_params(b[i]);
  }
  if (b.size() > 2) illegal("R9", b[2].id, "at most one SET_RESOURCE");
}

void walk(const Seq& s, std::vector<const Op*> prefix) {
  for (size_t k = 0; k < s.size(); ++k) {
    const Op& op = s[k];
    check_params(op);
    if (is_branching(op.name)) {
      if (k != s.size() - 1) illegal("R8", op.id, "a branching operator must end its sequence");
      if (op.name == "DIA_DECOM" || op.name == "DENSE_DECOM") {
        if (op.br.size() != 1 && op.br.size() != 2) illegal("R8", op.id, "DIA/DENSE_DECOM take 1 or 2 branches");
      } else if ((int64_t)op.br.size() != n_branches(op)) {
        illegal("R8", op.id, "expected " + std::to_string(n_branches(op)) + " branches, got " + std::to_string(op.br.size()));
      }
      std::vector<const Op*> path = prefix;
      for (size_t j = 0; j <= k; ++j) path.push_back(&s[j]);
      check_path(path, true);
      for (size_t bi = 0; bi < op.br.size(); ++bi) {
        const Seq& b = op.br[bi];
        if ((op.name == "DIA_DECOM" || op.name == "DENSE_DECOM") && bi == 0) {
          check_terminal(op, b);
        } else {
          if (!b.empty() && (b[0].name == "DIA" || b[0].name == "DENSE"))
            illegal("R8", b[0].id, "DIA/DENSE only open the first decomposition branch");
          walk(b, path);
        }
      }
      return;
    }
    if (!op.br.empty()) illegal("R8", op.id, op.name + " does not branch");
    if (op.name == "DIA" || op.name == "DENSE") illegal("R8", op.id, "DIA/DENSE only open the first decomposition branch");
  }
  std::vector<const Op*> path = prefix;
  for (auto& o : s) path.push_back(&o);
  check_path(path, false);
}

// shortest round-trip decimal for a double (matches Python repr for the values we print)
std::string fmt_double(double d) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*g", p, d);
    if (std::strtod(buf, nullptr) == d) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  // Python repr uses e-05 style; %g gives e-05 too.  Python prints 1e+16 as '1e+16'.
  return s;
}

void print_seq(const Seq& s, std::string& out) {
  for (size_t k = 0; k < s.size(); ++k) {
    if (k) out += "; ";
    const Op& o = s[k];
    out += o.name;
    if (!o.params.empty()) {
      out += "(";
      for (size_t j = 0; j < o.params.size(); ++j) {
        // SET_RESOURCE stream (R-conc) is printed only when it names a side stream, so the
        // canonical text of every single-stream graph is unchanged
        if (o.params[j].first == "stream" && o.params[j].second.i == 0) continue;
        if (j) out += ",";
        out += o.params[j].first;
        out += "=";
        const Value& v = o.params[j].second;
        if (v.k == Value::INT)
          out += std::to_string(v.i);
        else if (v.k == Value::FLOAT)
          out += fmt_double(v.f);
        else if (v.k == Value::IDENT)
          out += v.s;
        else {
          out += "[";
          for (size_t a = 0; a < v.l.size(); ++a) {
            if (a) out += ",";
            out += std::to_string(v.l[a]);
          }
          out += "]";
        }
      }
      out += ")";
    }
    if (!o.br.empty()) {
      out += " { ";
      for (size_t b = 0; b < o.br.size(); ++b) {
        if (b) out += " | ";
        print_seq(o.br[b], out);
      }
      out += " }";
    }
  }
}

}  // namespace

bool is_branching(const std::string& n) {
  return n == "ROW_DIV" || n == "COL_DIV" || n == "BIN" || n == "DIA_DECOM" || n == "DENSE_DECOM" || n == "HYB_DECOM";
}

int64_t Op::geti(const char* k) const {
  for (auto& p : params)
    if (p.first == k) return p.second.i;
  fail(AS_ERR_INVALID_ARG, name + ": no parameter " + k);
}
double Op::getf(const char* k) const {
  for (auto& p : params)
    if (p.first == k) return p.second.f;
  fail(AS_ERR_INVALID_ARG, name + ": no parameter " + k);
}
const std::vector<int64_t>& Op::getl(const char* k) const {
  for (auto& p : params)
    if (p.first == k) return p.second.l;
  fail(AS_ERR_INVALID_ARG, name + ": no parameter " + k);
}
const std::string& Op::gets(const char* k) const {
  for (auto& p : params)
    if (p.first == k) return p.second.s;
  fail(AS_ERR_INVALID_ARG, name + ": no parameter " + k);
}

Seq parse_graph(const std::string& text) {
  Parser p;
  p.t = tokenize(text);
  Seq g = p.seq();
  if (p.peek().k != Tok::END) fail(AS_ERR_GRAPH_PARSE, "unexpected '" + p.peek().s + "'");
  expand(g);
  int c = 0;
  number(g, c);
  walk(g, {});
  return g;
}

std::string print_graph(const Seq& g) {
  std::string out;
  print_seq(g, out);
  return out;
}

}  // namespace as
