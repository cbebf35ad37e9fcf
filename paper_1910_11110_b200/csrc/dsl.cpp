// DSL front end and CLI reporting: the reference command line
// (tools/cohere_main.cpp) over program text, with `run` executed by the device interpreter
// of general block programs (sweep.cu).  Host restatements, each following the reference:
//
//   lexer / parser        parse.hpp:34-353 (tokens, '/*shadow*/', declarations, blocks,
//                         statements, error texts and positions)
//   declarations          program.hpp:47-130 (ConstructionError texts)
//   normal form           ast.hpp:207-240 (flat statement lists, Noop only as empty)
//   printers              pretty.hpp:10-148 (to_string, one-line core form, pretty)
//   overlap closure       overlap.hpp:17-20, 86-108, 177-244 (query, infer, rewrite)
//   translation           modes.hpp:14-66 (translate_mode / _block / _program)
//   checker               checker.hpp:16-318 (rules, messages, positions, notes)
//   reporting             tools/cohere_main.cpp:38-230 (text and JSON records, exit codes)
//
// There is no CPU evaluator here: `run` compiles the translated program to the bytecode of
// sweep.hpp and launches k_sweep_run for one (program, schedule) item.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "internal.hpp"
#include "sweep.hpp"

namespace cohb {
namespace dsl {

struct Pos {
  int line = 0, col = 0;
};
struct ParseError : std::runtime_error {
  ParseError(Pos p, const std::string& m)
      : std::runtime_error(std::to_string(p.line) + ":" + std::to_string(p.col) + ": " + m) {}
};
struct ConstructionError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OverlapError : std::runtime_error {
  explicit OverlapError(const std::string& v)
      : std::runtime_error("inferred modes put '" + v + "' on both sites in one block") {}
};

enum Site : uint8_t { LOCAL = 0, REMOTE = 1 };
enum Kind : uint8_t { R = 0, W = 1, RW = 2 };

// ---- declarations (program.hpp:47-130) ------------------------------------------------
struct ScalarDecl { std::string name; Pos pos; };
struct BufferDecl { std::string id; int length; Pos pos; };
struct ViewDecl {
  std::string name, buffer;
  int lo, hi;
  Pos pos;
  int length() const { return hi - lo + 1; }
};
struct Decls {
  std::vector<ScalarDecl> scalars;
  std::vector<BufferDecl> buffers;
  std::vector<ViewDecl> views;
  const ScalarDecl* scalar(const std::string& n) const {
    for (const auto& s : scalars) if (s.name == n) return &s;
    return nullptr;
  }
  const BufferDecl* buffer(const std::string& n) const {
    for (const auto& b : buffers) if (b.id == n) return &b;
    return nullptr;
  }
  const ViewDecl* view(const std::string& n) const {
    for (const auto& v : views) if (v.name == n) return &v;
    return nullptr;
  }
  void fresh(const std::string& n) const {
    if (scalar(n) || view(n)) throw ConstructionError("duplicate declaration of '" + n + "'");
  }
  void add_scalar(ScalarDecl d) {
    fresh(d.name);
    scalars.push_back(std::move(d));
  }
  void add_buffer(BufferDecl d) {
    if (d.length < 1) throw ConstructionError("buffer '" + d.id + "' needs length >= 1");
    if (buffer(d.id)) throw ConstructionError("duplicate buffer '" + d.id + "'");
    buffers.push_back(std::move(d));
  }
  void add_view(ViewDecl d) {
    fresh(d.name);
    const BufferDecl* b = buffer(d.buffer);
    if (!b) throw ConstructionError("view '" + d.name + "' names unknown buffer '" + d.buffer + "'");
    if (d.lo < 0 || d.hi >= b->length || d.lo > d.hi)
      throw ConstructionError("view '" + d.name + "' range [" + std::to_string(d.lo) + ":" + std::to_string(d.hi) +
                              "] does not fit buffer '" + b->id + "[" + std::to_string(b->length) + "]'");
    views.push_back(std::move(d));
  }
};

// ---- statements in normal form --------------------------------------------------------
// VarKey (ast.hpp:30-46): kind order Scalar < Element < Abstract in the store map.
struct Key {
  uint8_t kind = 0;  // 0 scalar, 1 element, 2 abstract
  std::string name;
  int index = -1;
  bool operator<(const Key& o) const {
    if (name != o.name) return name < o.name;
    if (kind != o.kind) return kind < o.kind;
    return index < o.index;
  }
  bool operator==(const Key& o) const { return kind == o.kind && name == o.name && index == o.index; }
};
std::string key_str(const Key& k) {
  if (k.kind == 1) return k.name + "[" + std::to_string(k.index) + "]";
  return k.kind == 2 ? k.name + "^" : k.name;
}

struct Target {
  uint8_t kind = 0;  // 0 scalar, 1 abstract, 2 element, 3 whole view
  std::string name, buffer;
  int offset = -1, abs = -1, lo = -1, hi = -1;
};
struct Cond {
  uint8_t kind = 2;  // 0 valid, 1 gvalid, 2 opaque
  Key key;
};
struct Stmt;
using List = std::vector<Stmt>;
struct Stmt {
  uint8_t op = 0;  // 0 effect, 1 if, 2 while
  uint8_t eff = 0, site = 0;
  Target t;
  Cond c;
  List a, b;  // then | body, else
  Pos pos;
};
struct Mode {
  Kind kind;
  Site site;
  std::string view;
  bool shadow = false;
  Pos pos;
};
struct Block {
  std::vector<Mode> modes;
  List body;
  Pos pos;
};
struct Program {
  Decls decls;
  std::vector<Block> blocks;
  List raw;  // --raw: the bare statement list
};

// ---- lexer (parse.hpp:34-106) -----------------------------------------------------------
enum Tk { IDENT, INT, LPAREN, RPAREN, LBRACE, RBRACE, LBRACKET, RBRACKET, SEMI, COMMA, EQ, COLON, CARET, SHADOW, END };
struct Token {
  Tk kind;
  std::string text;
  long value = 0;
  Pos pos;
};

std::vector<Token> lex(const std::string& src) {
  std::vector<Token> out;
  int line = 1, col = 1;
  size_t i = 0;
  auto step = [&](size_t n = 1) {
    while (n-- && i < src.size()) {
      if (src[i] == '\n') { ++line; col = 1; } else { ++col; }
      ++i;
    }
  };
  while (i < src.size()) {
    const char c = src[i];
    if (c == ' ' || c == '\t' || c == '\r' || c == '\n') { step(); continue; }
    if (c == '/' && i + 1 < src.size() && src[i + 1] == '/') {
      while (i < src.size() && src[i] != '\n') step();
      continue;
    }
    if (c == '/' && i + 1 < src.size() && src[i + 1] == '*') {
      const Pos pos{line, col};
      const size_t start = i + 2, end = src.find("*/", start);
      if (end == std::string::npos) throw ParseError(pos, "unterminated comment");
      const std::string body = src.substr(start, end - start);
      step(end + 2 - i);
      const size_t b = body.find_first_not_of(" \t"), e = body.find_last_not_of(" \t");
      if (b != std::string::npos && body.substr(b, e - b + 1) == "shadow") out.push_back({SHADOW, "shadow", 0, pos});
      continue;
    }
    const Pos pos{line, col};
    if (std::isalpha((unsigned char)c) || c == '_') {
      const size_t start = i;
      while (i < src.size() && (std::isalnum((unsigned char)src[i]) || src[i] == '_')) step();
      out.push_back({IDENT, src.substr(start, i - start), 0, pos});
      continue;
    }
    if (std::isdigit((unsigned char)c)) {
      const size_t start = i;
      while (i < src.size() && std::isdigit((unsigned char)src[i])) step();
      const std::string text = src.substr(start, i - start);
      long v = 0;
      try {
        v = std::stol(text);
      } catch (const std::exception&) {
        throw std::runtime_error("stol");  // std::stol's out_of_range in the reference
      }
      out.push_back({INT, text, v, pos});
      continue;
    }
    Tk k;
    switch (c) {
      case '(': k = LPAREN; break;
      case ')': k = RPAREN; break;
      case '{': k = LBRACE; break;
      case '}': k = RBRACE; break;
      case '[': k = LBRACKET; break;
      case ']': k = RBRACKET; break;
      case ';': k = SEMI; break;
      case ',': k = COMMA; break;
      case '=': k = EQ; break;
      case ':': k = COLON; break;
      case '^': k = CARET; break;
      default: throw ParseError(pos, std::string("unexpected character '") + c + "'");
    }
    out.push_back({k, std::string(1, c), 0, pos});
    step();
  }
  out.push_back({END, "", 0, {line, col}});
  return out;
}

// ---- parser (parse.hpp:108-353) -------------------------------------------------------
class Parser {
 public:
  explicit Parser(const std::string& src) : t_(lex(src)) {}

  Program annotated() {
    Program p;
    p.decls = decls();
    while (!at(END)) p.blocks.push_back(block(p.decls));
    return p;
  }
  Program raw() {
    Program p;
    p.decls = decls();
    while (!at(END)) p.raw.push_back(stmt(p.decls));
    return p;
  }

 private:
  static bool keyword(const std::string& s) {
    static const char* w[] = {"scalar", "buffer", "view", "if", "else", "while", "valid", "gvalid", "opaque", "push", "pull",
                              "r", "w", "gr", "gw", "R", "W", "RW", "GR", "GW", "GRW"};
    for (const char* k : w)
      if (s == k) return true;
    return false;
  }
  const Token& peek() const { return t_[std::min(p_, t_.size() - 1)]; }
  bool at(Tk k) const { return peek().kind == k; }
  bool at_word(const char* w) const { return peek().kind == IDENT && peek().text == w; }
  const Token& take() { return t_[p_ < t_.size() - 1 ? p_++ : p_]; }
  const Token& expect(Tk k, const char* what) {
    if (!at(k)) throw ParseError(peek().pos, std::string("expected ") + what);
    return take();
  }
  std::string name(const char* what) {
    const Token& t = expect(IDENT, what);
    if (keyword(t.text)) throw ParseError(t.pos, "'" + t.text + "' is reserved and cannot name a variable");
    return t.text;
  }
  int integer(const char* what) { return (int)expect(INT, what).value; }
  template <class F>
  static void here(Pos pos, F&& f) {
    try {
      f();
    } catch (const ConstructionError& e) {
      throw ParseError(pos, e.what());
    }
  }

  Decls decls() {
    Decls out;
    for (;;) {
      if (at_word("scalar")) {
        const Pos pos = take().pos;
        const std::string n = name("scalar name");
        here(pos, [&] { out.add_scalar({n, pos}); });
      } else if (at_word("buffer")) {
        const Pos pos = take().pos;
        const std::string id = name("buffer name");
        expect(LBRACKET, "'['");
        const int len = integer("buffer length");
        expect(RBRACKET, "']'");
        here(pos, [&] { out.add_buffer({id, len, pos}); });
      } else if (at_word("view")) {
        const Pos pos = take().pos;
        const std::string vn = name("view name");
        expect(EQ, "'='");
        const std::string buf = name("buffer name");
        expect(LBRACKET, "'['");
        const int lo = integer("range start");
        expect(COLON, "':'");
        const int hi = integer("range end");
        expect(RBRACKET, "']'");
        here(pos, [&] { out.add_view({vn, buf, lo, hi, pos}); });
      } else {
        return out;
      }
    }
  }

  static bool mode_word(const std::string& s, Kind& k, Site& site) {
    std::string base = s;
    site = LOCAL;
    if (!base.empty() && base[0] == 'G') {
      site = REMOTE;
      base = base.substr(1);
    }
    if (base == "R") k = R;
    else if (base == "W") k = W;
    else if (base == "RW") k = RW;
    else return false;
    return true;
  }

  Block block(const Decls& d) {
    Block b;
    b.pos = peek().pos;
    auto one_mode = [&] {
      Kind k;
      Site site;
      if (peek().kind != IDENT || !mode_word(peek().text, k, site)) throw ParseError(peek().pos, "expected an access mode");
      const Pos pos = take().pos;
      expect(LPAREN, "'('");
      const std::string v = name("variable name");
      expect(RPAREN, "')'");
      if (!d.scalar(v) && !d.view(v)) throw ParseError(pos, "mode names undeclared variable '" + v + "'");
      Mode m{k, site, v, false, pos};
      if (at(SHADOW)) {
        take();
        m.shadow = true;
      }
      for (const auto& seen : b.modes)
        if (seen.view == v) throw ParseError(pos, "variable '" + v + "' declared twice in one block");
      b.modes.push_back(m);
    };
    Kind k;
    Site site;
    if (peek().kind == IDENT && mode_word(peek().text, k, site)) {
      one_mode();
      while (at(COMMA)) {
        take();
        one_mode();
      }
    }
    if (at_word("scalar") || at_word("buffer") || at_word("view"))
      throw ParseError(peek().pos, "declarations must precede all blocks");
    expect(LBRACE, "mode list or '{'");
    while (!at(RBRACE)) b.body.push_back(stmt(d));
    take();
    return b;
  }

  Cond cond(const Decls& d) {
    Cond c;
    if (at_word("opaque")) {
      take();
      return c;
    }
    bool remote;
    if (at_word("valid")) remote = false;
    else if (at_word("gvalid")) remote = true;
    else throw ParseError(peek().pos, "expected valid(...), gvalid(...) or opaque");
    take();
    expect(LPAREN, "'('");
    const Pos pos = peek().pos;
    const std::string n = name("variable name");
    const bool hat = at(CARET);
    if (hat) take();
    expect(RPAREN, "')'");
    if (!d.scalar(n) && !d.view(n)) throw ParseError(pos, "condition names undeclared variable '" + n + "'");
    c.kind = remote ? 1 : 0;
    c.key.kind = (hat || d.view(n)) ? 2 : 0;
    c.key.name = n;
    return c;
  }

  Stmt stmt(const Decls& d) {
    const Token& t = peek();
    if (t.kind != IDENT) throw ParseError(t.pos, "expected a statement");
    if (t.text == "if" || t.text == "while") {
      Stmt s;
      s.op = t.text == "if" ? 1 : 2;
      s.pos = take().pos;
      expect(LPAREN, "'('");
      s.c = cond(d);
      expect(RPAREN, "')'");
      s.a = braced(d);
      if (s.op == 1 && at_word("else")) {
        take();
        s.b = braced(d);
      }
      return s;
    }
    Stmt s;
    bool sync = false;
    if (t.text == "r") s.eff = COH_READ;
    else if (t.text == "w") s.eff = COH_WRITE;
    else if (t.text == "gr") { s.eff = COH_READ; s.site = REMOTE; }
    else if (t.text == "gw") { s.eff = COH_WRITE; s.site = REMOTE; }
    else if (t.text == "push") { s.eff = COH_PUSH; sync = true; }
    else if (t.text == "pull") { s.eff = COH_PULL; sync = true; }
    else throw ParseError(t.pos, "expected a statement");
    s.pos = take().pos;
    const Pos np = peek().pos;
    const std::string n = name("variable name");
    if (at(LBRACKET)) {
      take();
      const int off = integer("element index");
      expect(RBRACKET, "']'");
      if (sync) throw ParseError(np, "push/pull take a whole variable, not an element");
      if (d.scalar(n)) throw ParseError(np, "scalar '" + n + "' takes no index");
      here(np, [&] {
        const ViewDecl* v = d.view(n);
        if (!v) throw ConstructionError("unknown view '" + n + "'");
        if (off < 0 || off >= v->length())
          throw ConstructionError("index " + std::to_string(off) + " outside view '" + n + "' of length " +
                                  std::to_string(v->length()));
        s.t.kind = 2;
        s.t.name = n;
        s.t.offset = off;
        s.t.buffer = v->buffer;
        s.t.abs = v->lo + off;
      });
    } else if (d.scalar(n)) {
      s.t.kind = 0;
      s.t.name = n;
    } else if (const ViewDecl* v = d.view(n)) {
      if (!sync) throw ParseError(np, "view '" + n + "' needs an element index here");
      s.t.kind = 3;
      s.t.name = n;
      s.t.buffer = v->buffer;
      s.t.lo = v->lo;
      s.t.hi = v->hi;
    } else {
      throw ParseError(np, "undeclared variable '" + n + "'");
    }
    expect(SEMI, "';'");
    return s;
  }

  List braced(const Decls& d) {
    expect(LBRACE, "'{'");
    List out;
    while (!at(RBRACE)) out.push_back(stmt(d));
    take();
    return out;
  }

  std::vector<Token> t_;
  size_t p_ = 0;
};

// ---- printers (pretty.hpp) ----------------------------------------------------------------
const char* eff_name(uint32_t e) {
  static const char* n[] = {"push", "pull", "r", "w", "noop"};
  return n[e];
}
std::string target_str(const Target& t) {
  switch (t.kind) {
    case 1: return t.name + "^";
    case 2: return t.name + "[" + std::to_string(t.offset) + "]";
    default: return t.name;
  }
}
std::string cond_str(const Cond& c) {
  if (c.kind == 2) return "opaque";
  return std::string(c.kind == 0 ? "valid(" : "gvalid(") + key_str(c.key) + ")";
}
std::string mode_name(Kind k, Site s) { return std::string(s == REMOTE ? "G" : "") + (k == R ? "R" : k == W ? "W" : "RW"); }
std::string mode_str(const Mode& m) {
  std::string out = mode_name(m.kind, m.site) + "(" + m.view + ")";
  if (m.shadow) out += " /*shadow*/";
  return out;
}
std::string effect_word(const Stmt& s) { return std::string(s.site == REMOTE ? "g" : "") + eff_name(s.eff); }

void one_line(const List& l, std::string& out) {  // stmt_one_line (pretty.hpp:41-79)
  for (const auto& s : l) {
    if (s.op == 0) {
      if (!out.empty()) out += ' ';
      out += effect_word(s) + " " + target_str(s.t) + ";";
      continue;
    }
    std::string a, b;
    one_line(s.a, a);
    if (!out.empty()) out += ' ';
    if (s.op == 1) {
      one_line(s.b, b);
      out += "if (" + cond_str(s.c) + ") { " + a + (a.empty() ? "}" : " }");
      if (!s.b.empty()) out += " else { " + b + " }";
    } else {
      out += "while (" + cond_str(s.c) + ") { " + a + (a.empty() ? "}" : " }");
    }
  }
}

void lines(const List& l, int indent, std::string& out) {  // stmt_lines (pretty.hpp:81-111)
  const std::string pad(2 * (size_t)indent, ' ');
  for (const auto& s : l) {
    if (s.op == 0) {
      out += pad + effect_word(s) + " " + target_str(s.t) + ";\n";
      continue;
    }
    out += pad + (s.op == 1 ? "if (" : "while (") + cond_str(s.c) + ") {\n";
    lines(s.a, indent + 1, out);
    if (s.op == 1 && !s.b.empty()) {
      out += pad + "} else {\n";
      lines(s.b, indent + 1, out);
    }
    out += pad + "}\n";
  }
}

std::string pretty(const Program& p) {  // pretty.hpp:113-148
  std::string out;
  for (const auto& s : p.decls.scalars) out += "scalar " + s.name + "\n";
  for (const auto& b : p.decls.buffers) out += "buffer " + b.id + "[" + std::to_string(b.length) + "]\n";
  for (const auto& v : p.decls.views)
    out += "view " + v.name + " = " + v.buffer + "[" + std::to_string(v.lo) + ":" + std::to_string(v.hi) + "]\n";
  for (const auto& b : p.blocks) {
    if (!out.empty()) out += "\n";
    std::string header;
    for (const auto& m : b.modes) {
      if (!header.empty()) header += ", ";
      header += mode_str(m);
    }
    out += header + (header.empty() ? "{\n" : " {\n");
    lines(b.body, 1, out);
    out += "}\n";
  }
  return out;
}

// ---- overlap closure (overlap.hpp) ------------------------------------------------------
std::vector<std::string> query(const Decls& d, const ViewDecl& probe) {  // name-sorted, probe excluded
  std::set<std::string> hits;
  for (const auto& v : d.views)
    if (v.buffer == probe.buffer && v.lo <= probe.hi && v.hi >= probe.lo) hits.insert(v.name);
  hits.erase(probe.name);
  return {hits.begin(), hits.end()};
}

std::vector<Mode> infer_closure(const std::vector<Mode>& modes, const Decls& d) {  // overlap.hpp:177-230
  std::vector<Mode> out = modes;
  std::map<std::string, Site> needed;
  for (const auto& m : modes) {
    if (m.kind == R || m.shadow) continue;
    const ViewDecl* view = d.view(m.view);
    if (!view) continue;
    for (const auto& y : query(d, *view)) {
      if (m.kind == W) {
        bool same = false;
        for (const auto& o : modes)
          if (o.view == y && o.kind == W && o.site == m.site) same = true;
        if (same) continue;
      }
      auto [it, fresh] = needed.emplace(y, m.site);
      if (!fresh && it->second != m.site) throw OverlapError(y);
    }
  }
  std::vector<std::pair<std::string, Site>> shadows;
  for (const auto& [y, site] : needed) {
    Mode* existing = nullptr;
    for (auto& m : out)
      if (m.view == y) existing = &m;
    if (existing) {
      if (existing->site != site) throw OverlapError(y);
      if (existing->kind == R) existing->kind = RW;
    } else {
      shadows.emplace_back(y, site);
    }
  }
  for (const auto& v : d.views)
    for (const auto& [y, site] : shadows)
      if (y == v.name) out.push_back(Mode{RW, site, y, true, Pos{}});
  return out;
}

void rewrite(Program& p) {  // rewrite_program (overlap.hpp:234-244)
  for (auto& b : p.blocks) b.modes = infer_closure(b.modes, p.decls);
}

// ---- translation (modes.hpp:14-66) ---------------------------------------------------------
List translate_block(const Block& b, const Decls& d) {
  List out;
  for (const auto& m : b.modes) {
    const Site sync_site = LOCAL;
    const uint8_t sync = m.site == REMOTE ? COH_PUSH : COH_PULL;
    Target abs;
    abs.kind = 1;
    abs.name = m.view;
    if (m.kind == R || m.kind == RW) {
      Stmt guard;
      guard.op = 1;
      guard.c.kind = m.site == REMOTE ? 1 : 0;
      guard.c.key = Key{2, m.view, -1};
      Stmt conc;
      conc.eff = sync;
      conc.site = sync_site;
      if (d.scalar(m.view)) {
        conc.t.kind = 0;
        conc.t.name = m.view;
      } else {
        const ViewDecl* v = d.view(m.view);
        conc.t.kind = 3;
        conc.t.name = m.view;
        conc.t.buffer = v->buffer;
        conc.t.lo = v->lo;
        conc.t.hi = v->hi;
      }
      Stmt a;
      a.eff = sync;
      a.site = sync_site;
      a.t = abs;
      guard.b = {conc, a};
      out.push_back(guard);
    }
    if (m.kind == W || m.kind == RW) {
      Stmt w;
      w.eff = COH_WRITE;
      w.site = m.site;
      w.t = abs;
      out.push_back(w);
    }
  }
  for (const auto& s : b.body) out.push_back(s);
  return out;
}

// ---- checker (checker.hpp) -----------------------------------------------------------------
struct Diag {
  std::string rule, view;
  Pos pos;
  std::string message;
};
struct Access {
  bool reads = false, writes = false, touched = false;
  std::set<int> cells;
  Pos first_read, first_write, first_touch;
};
struct Summary {
  std::map<std::pair<std::string, int>, Access> per_site;
  bool sync = false, abstract_effect = false;
  std::string sync_view, abstract_name;
  Pos sync_pos, abstract_pos;
};

void collect(const List& l, Summary& out) {  // collect_accesses (checker.hpp:60-115)
  for (const auto& s : l) {
    if (s.op != 0) {
      collect(s.a, out);
      collect(s.b, out);
      continue;
    }
    if (s.t.kind == 1) {
      if (!out.abstract_effect) {
        out.abstract_effect = true;
        out.abstract_name = s.t.name;
        out.abstract_pos = s.pos;
      }
      continue;
    }
    Access& a = out.per_site[{s.t.name, (int)s.site}];
    if (!a.touched) {
      a.touched = true;
      a.first_touch = s.pos;
    }
    if (s.eff == COH_READ) {
      if (!a.reads) a.first_read = s.pos;
      a.reads = true;
    } else if (s.eff == COH_WRITE) {
      if (!a.writes) a.first_write = s.pos;
      a.writes = true;
      if (s.t.kind == 2) a.cells.insert(s.t.abs);
    } else if (s.eff == COH_PUSH || s.eff == COH_PULL) {
      if (!out.sync) {
        out.sync = true;
        out.sync_view = s.t.name;
        out.sync_pos = s.pos;
      }
    }
  }
}

bool must_write_scalar(const List& l, const std::string& n, int site) {  // checker.hpp:127-143
  for (const auto& s : l) {
    if (s.op == 0 && s.eff == COH_WRITE && s.site == site && s.t.kind == 0 && s.t.name == n) return true;
    if (s.op == 1 && must_write_scalar(s.a, n, site) && must_write_scalar(s.b, n, site)) return true;
  }
  return false;
}
std::set<int> must_cells(const List& l, const std::string& v, int site) {  // checker.hpp:145-170
  std::set<int> out;
  for (const auto& s : l) {
    if (s.op == 0 && s.eff == COH_WRITE && s.site == site && s.t.kind == 2 && s.t.name == v) out.insert(s.t.abs);
    if (s.op == 1) {
      const std::set<int> a = must_cells(s.a, v, site), b = must_cells(s.b, v, site);
      for (int i : a)
        if (b.count(i)) out.insert(i);
    }
  }
  return out;
}

std::vector<Diag> check_localised(const Block& b) {  // checker.hpp:191-208
  std::vector<Diag> out;
  Summary sm;
  collect(b.body, sm);
  std::set<std::string> reported;
  for (const auto& [key, acc] : sm.per_site) {
    const auto& [name, site] = key;
    if (!acc.touched || site != LOCAL) continue;
    auto it = sm.per_site.find({name, (int)REMOTE});
    if (it != sm.per_site.end() && it->second.touched && !reported.count(name)) {
      reported.insert(name);
      out.push_back({"P3-MIXED-SITE", name, acc.first_touch, "'" + name + "' is accessed from both sites in one body"});
    }
  }
  return out;
}

std::vector<Diag> check_block(const Block& b, const Decls& d) {  // checker.hpp:213-288
  std::vector<Diag> out;
  Summary sm;
  collect(b.body, sm);
  auto mode_for = [&](const std::string& n) -> const Mode* {
    for (const auto& m : b.modes)
      if (m.view == n) return &m;
    return nullptr;
  };
  if (sm.sync)
    out.push_back({"D2-NO-SYNC", sm.sync_view, sm.sync_pos, "declared blocks may not push or pull; declare a mode instead"});
  if (sm.abstract_effect)
    out.push_back({"BODY-ABSTRACT-EFFECT", sm.abstract_name, sm.abstract_pos,
                   "abstract key '" + sm.abstract_name + "^' cannot be addressed from a body"});
  for (const auto& [key, acc] : sm.per_site) {
    const auto& [name, site] = key;
    const Mode* m = mode_for(name);
    const bool here = m && (int)m->site == site;
    const char* sn = site == LOCAL ? "local" : "remote";
    if (acc.reads && !(here && (m->kind == R || m->kind == RW)))
      out.push_back({"D2-UNDECLARED-READ", name, acc.first_read,
                     "'" + name + "' is read " + sn + "ly but has no R or RW declaration there"});
    if (acc.writes && !(here && (m->kind == W || m->kind == RW)))
      out.push_back({"D2-UNDECLARED-WRITE", name, acc.first_write,
                     "'" + name + "' is written " + sn + "ly but has no W or RW declaration there"});
  }
  for (const auto& m : b.modes) {
    if (m.kind != W) continue;
    bool all;
    if (d.scalar(m.view)) {
      all = must_write_scalar(b.body, m.view, m.site);
    } else {
      const ViewDecl* v = d.view(m.view);
      const std::set<int> cells = must_cells(b.body, m.view, m.site);
      all = true;
      for (int i = v->lo; i <= v->hi; ++i)
        if (!cells.count(i)) all = false;
    }
    if (all) continue;
    if (d.scalar(m.view))
      out.push_back({"D2-W-NOT-ALL-PATHS", m.view, m.pos, "'" + m.view + "' is declared W but not written on every path"});
    else
      out.push_back({"D4-W-NOT-ALL-ELEMENTS", m.view, m.pos,
                     "'" + m.view + "' is declared W but some cells are not written on every path"});
  }
  for (const auto& [key, acc] : sm.per_site) {
    const auto& [name, site] = key;
    if (!acc.writes) continue;
    const ViewDecl* view = d.view(name);
    if (!view) continue;
    for (const auto& on : query(d, *view)) {
      const ViewDecl* other = d.view(on);
      const int slo = std::max(view->lo, other->lo), shi = std::min(view->hi, other->hi);
      bool hits = false;
      for (int c : acc.cells)
        if (c >= slo && c <= shi) hits = true;
      if (!hits) continue;
      const Mode* om = mode_for(on);
      if (om && (int)om->site == site && (om->kind == W || om->kind == RW)) continue;
      out.push_back({"OVL-MISSING-RW", on, acc.first_write,
                     "writes through '" + name + "' reach cells shared with '" + on +
                         "', which needs W or RW at the same site"});
    }
  }
  return out;
}

std::vector<Diag> check_program(const Program& p) {
  std::vector<Diag> out;
  for (const auto& b : p.blocks) {
    auto x = check_block(b, p.decls);
    out.insert(out.end(), x.begin(), x.end());
    auto y = check_localised(b);
    out.insert(out.end(), y.begin(), y.end());
  }
  return out;
}

std::vector<Diag> check_notes(const Program& p) {  // checker.hpp:302-318
  std::vector<Diag> out;
  for (const auto& b : p.blocks) {
    Summary sm;
    collect(b.body, sm);
    for (const auto& m : b.modes) {
      if (m.kind != R || m.shadow) continue;
      auto it = sm.per_site.find({m.view, (int)m.site});
      if (it == sm.per_site.end() || !it->second.reads)
        out.push_back({"NOTE-UNUSED-MODE", m.view, m.pos,
                       "'" + m.view + "' is declared " + mode_name(m.kind, m.site) + " but never read"});
    }
  }
  return out;
}

// ---- JSON (nlohmann::json dump of std::map-ordered objects) ---------------------------
std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

// ---- GPU run ---------------------------------------------------------------------------------
struct KeyMap {
  std::vector<Key> keys;  // index -> key
  std::map<std::string, uint32_t> scalar, abs;
  std::map<std::string, uint32_t> buf_base;
  uint32_t id(const Key& k) const {
    if (k.kind == 0) return scalar.at(k.name);
    if (k.kind == 2) return abs.at(k.name);
    return buf_base.at(k.name) + (uint32_t)k.index;
  }
};

KeyMap key_map(const Decls& d) {  // initial_store (program.hpp:174-184): every key (V,I)
  KeyMap km;
  for (const auto& s : d.scalars) {
    km.scalar[s.name] = (uint32_t)km.keys.size();
    km.keys.push_back(Key{0, s.name, -1});
    km.abs[s.name] = (uint32_t)km.keys.size();
    km.keys.push_back(Key{2, s.name, -1});
  }
  for (const auto& b : d.buffers) {
    km.buf_base[b.id] = (uint32_t)km.keys.size();
    for (int i = 0; i < b.length; ++i) km.keys.push_back(Key{1, b.id, i});
  }
  for (const auto& v : d.views) {
    km.abs[v.name] = (uint32_t)km.keys.size();
    km.keys.push_back(Key{2, v.name, -1});
  }
  return km;
}

struct Emit {
  const KeyMap& km;
  std::vector<uint32_t> code;
  std::vector<std::string> head;  // per instruction: to_string of the statement it starts
  void note(const Stmt& s) {
    std::string h;
    one_line(List{s}, h);
    head.resize(code.size() + 1);
    head[code.size()] = h;
  }
  uint32_t key(const Target& t) const {
    switch (t.kind) {
      case 0: return km.scalar.at(t.name);
      case 1: return km.abs.at(t.name);
      default: return km.buf_base.at(t.buffer) + (uint32_t)t.abs;
    }
  }
  void list(const List& l) {
    for (const auto& s : l) {
      note(s);
      if (s.op == 0) {
        if (s.t.kind == 3) {
          const uint32_t base = km.buf_base.at(s.t.buffer);
          code.push_back(BC_WHOLE | ((uint32_t)s.eff << 4) | ((uint32_t)s.site << 7) | ((base + s.t.lo) << 8) |
                         ((base + s.t.hi) << 16));
        } else {
          code.push_back(BC_EFF | ((uint32_t)s.eff << 4) | ((uint32_t)s.site << 7) | (key(s.t) << 8));
        }
        continue;
      }
      const uint32_t ck = s.c.kind == 2 ? 0 : km.id(s.c.key);
      const uint32_t head = (uint32_t)code.size();
      code.push_back((s.op == 1 ? BC_IF : BC_WHILE) | ((uint32_t)s.c.kind << 4) | (ck << 8));
      list(s.a);
      if (s.op == 1) {
        if (!s.b.empty()) {
          const uint32_t j = (uint32_t)code.size();
          code.push_back(BC_JMP);
          code[head] |= (uint32_t)code.size() << 16;
          list(s.b);
          code[j] |= (uint32_t)code.size() << 16;
        } else {
          code[head] |= (uint32_t)code.size() << 16;
        }
      } else {
        code.push_back(BC_JMP | (head << 16));
        code[head] |= (uint32_t)code.size() << 16;
      }
    }
  }
};

struct RunOut {
  uint32_t status, steps, consumed, overflowed;
  uint64_t store;
  bool stuck;
  uint32_t stuck_key, stuck_eff, stuck_site, stuck_actual;
};

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
};

int device_run(coh_ctx* ctx, const std::vector<uint32_t>& code, uint32_t n_keys, int32_t fuel, uint64_t bits,
               uint32_t len, RunOut* r, std::string* err, std::vector<SweepTrace>* trace = nullptr) {
  if (!ctx) {
    *err = "run needs a device context";
    return COH_E_ARG;
  }
  if (cudaSetDevice(ctx->device) != cudaSuccess) {
    *err = "cudaSetDevice failed";
    return COH_E_CUDA;
  }
  DevBuf d_code, d_meta, d_checks, d_item, d_out, d_trace;
  SweepMeta meta{0, n_keys, 0, 0};
  SweepItem item{0, (uint32_t)bits, len, (uint32_t)(bits >> 32)};
  SweepOut out{};
  cudaStream_t s = nullptr;
  cudaError_t e;
#define COH_D(x)                                              \
  if ((e = (x)) != cudaSuccess) {                             \
    *err = std::string(#x ": ") + cudaGetErrorString(e);      \
    return COH_E_CUDA;                                        \
  }
  COH_D(cudaMalloc(&d_code.p, code.size() * 4));
  COH_D(cudaMalloc(&d_meta.p, sizeof meta));
  COH_D(cudaMalloc(&d_checks.p, 16));
  COH_D(cudaMalloc(&d_item.p, sizeof item));
  COH_D(cudaMalloc(&d_out.p, sizeof out));
  COH_D(cudaMemcpy(d_code.p, code.data(), code.size() * 4, cudaMemcpyHostToDevice));
  COH_D(cudaMemcpy(d_meta.p, &meta, sizeof meta, cudaMemcpyHostToDevice));
  COH_D(cudaMemcpy(d_item.p, &item, sizeof item, cudaMemcpyHostToDevice));
  if (trace) COH_D(cudaMalloc(&d_trace.p, (size_t)fuel * sizeof(SweepTrace)));
  const int rc = launch_sweep_run(static_cast<uint32_t*>(d_code.p), static_cast<SweepMeta*>(d_meta.p),
                                  static_cast<uint16_t*>(d_checks.p), static_cast<SweepItem*>(d_item.p), 1u, fuel,
                                  static_cast<SweepOut*>(d_out.p), s, err, static_cast<SweepTrace*>(d_trace.p));
  if (rc) return rc;
  COH_D(cudaMemcpy(&out, d_out.p, sizeof out, cudaMemcpyDeviceToHost));
  if (trace) {
    trace->resize(out.steps);
    if (out.steps) COH_D(cudaMemcpy(trace->data(), d_trace.p, out.steps * sizeof(SweepTrace), cudaMemcpyDeviceToHost));
  }
#undef COH_D
  ctx->launches++;
  r->status = out.status_consumed & 3u;
  r->consumed = (out.status_consumed >> 2) & 0xFFu;
  r->overflowed = (out.status_consumed >> 10) & 1u;
  r->steps = out.steps;
  r->store = out.store;
  r->stuck = r->status == COH_RUN_STUCK;
  r->stuck_key = out.status_consumed >> 24;
  r->stuck_eff = out.stuck & 7u;
  r->stuck_site = (out.stuck >> 3) & 1u;
  r->stuck_actual = (out.stuck >> 5) & 3u;
  return COH_OK;
}

std::string pair_str(uint32_t bits) {
  return std::string("(") + ((bits & 1u) ? "V" : "I") + "," + ((bits & 2u) ? "V" : "I") + ")";
}
const char* pre_str(uint32_t eff) {  // pre_to_string(effect_signature(e)) (validity.hpp:79-99)
  static const char* p[] = {"(V,*)", "(*,V)", "(V,*)", "(*,*)", "(*,*)"};
  return p[eff];
}

struct Cli {
  std::string out, err;
  int exit = 0;
};

// report_run (tools/cohere_main.cpp:96-158), text and JSON
std::string store_record(const KeyMap& km, uint32_t k, uint32_t bits) {
  return "{\"key\":" + jstr(key_str(km.keys[k])) + ",\"local\":" + jstr((bits & 1u) ? "V" : "I") +
         ",\"remote\":" + jstr((bits & 2u) ? "V" : "I") + "}";
}

// the --trace listing (tools/cohere_main.cpp:97-120): step, rule, head, changed keys in
// application order (a whole-view sync changes its cells ascending = key order)
void report_trace(const KeyMap& km, const std::vector<std::string>& head, const std::vector<SweepTrace>& tr,
                  const coh_cli_opts& o, Cli& c) {
  static const char* rule[] = {"effect", "remote-effect", "while-true", "while-false", "if-true", "if-false"};
  unsigned long long before = 0;
  for (uint32_t k = 0; k < km.keys.size(); ++k) before |= 1ull << (2 * k);  // initial_store: (V,I)
  for (size_t i = 0; i < tr.size(); ++i) {
    const unsigned long long after = tr[i].store;
    std::string delta;
    for (uint32_t k = 0; k < km.keys.size(); ++k) {
      const uint32_t a = (uint32_t)(after >> (2 * k)) & 3u;
      if (a == ((uint32_t)(before >> (2 * k)) & 3u)) continue;
      if (o.json) delta += (delta.empty() ? "" : ",") + store_record(km, k, a);
      else delta += (delta.empty() ? " => " : " ") + key_str(km.keys[k]) + "=" + pair_str(a);
    }
    const std::string& h = head[tr[i].pc];
    if (o.json) {
      c.out += "{\"delta\":[" + delta + "],\"head\":" + jstr(h) + ",\"rule\":" + jstr(rule[tr[i].rule]) +
               ",\"step\":" + std::to_string(i + 1) + "}\n";
    } else {
      std::string line = std::to_string(i + 1) + " " + rule[tr[i].rule];
      if (line.size() < 16) line.append(16 - line.size(), ' ');
      c.out += line + h + delta + "\n";
    }
    before = after;
  }
}

void report(const KeyMap& km, const RunOut& r, const coh_cli_opts& o, bool schedule_given, Cli& c) {
  static const char* st[] = {"done", "stuck", "fuel-exhausted", "defect"};
  if (o.json) {
    std::string rec = "{\"outcome\":" + jstr(st[r.status]) + ",\"schedule_consumed\":" + std::to_string(r.consumed) +
                      ",\"steps\":" + std::to_string(r.steps);
    if (r.stuck)
      rec += ",\"stuck\":{\"effect\":" + jstr(eff_name(r.stuck_eff)) + ",\"have\":" + jstr(pair_str(r.stuck_actual)) +
             ",\"key\":" + jstr(key_str(km.keys[r.stuck_key])) + ",\"site\":" +
             jstr(r.stuck_site ? "remote" : "local") + "}";
    c.out += rec + "}\n";
  } else {
    c.out += std::string("outcome: ") + st[r.status] + "\n";
    c.out += "steps: " + std::to_string(r.steps) + "\n";
    if (r.stuck) {
      std::string d = std::string(r.stuck_site ? "g" : "") + eff_name(r.stuck_eff) + " " + key_str(km.keys[r.stuck_key]) +
                      ": have " + pair_str(r.stuck_actual) + ", need " + pre_str(r.stuck_eff);
      if (r.stuck_site) d += " against the swapped pair";
      c.out += "stuck at: " + d + "\n";
    }
  }
  std::vector<uint32_t> order(km.keys.size());
  for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return km.keys[a] < km.keys[b]; });
  for (uint32_t k : order) {
    const uint32_t bits = (uint32_t)(r.store >> (2 * k)) & 3u;
    if (o.json)
      c.out += store_record(km, k, bits) + "\n";
    else
      c.out += key_str(km.keys[k]) + " " + pair_str(bits) + "\n";
  }
  if (r.overflowed && schedule_given) c.err += "note: schedule exhausted; later opaque conditions answered false\n";
  c.exit = r.status == COH_RUN_DONE ? 0 : r.status == COH_RUN_STUCK ? 3 : 4;
}

std::string diag_text(const Diag& d) {
  return std::to_string(d.pos.line) + ":" + std::to_string(d.pos.col) + ": " + d.rule + " [" + d.view + "] " + d.message;
}

int cli(coh_ctx* ctx, const std::string& cmd, const std::string& src, const coh_cli_opts& o, Cli& c,
        std::string* fatal) {
  const std::string schedule = o.schedule ? o.schedule : "";
  if (cmd == "check") {
    std::vector<Diag> diags, notes;
    if (o.raw) {
      Program p = Parser(src).raw();
      Block pseudo;
      pseudo.body = p.raw;
      diags = check_localised(pseudo);
    } else {
      Program p = Parser(src).annotated();
      diags = check_program(p);  // the registry is only consulted (no rewrite) here
      if (o.no_overlap) {
        // an empty registry: OVL-MISSING-RW cannot fire
        diags.erase(std::remove_if(diags.begin(), diags.end(), [](const Diag& d) { return d.rule == "OVL-MISSING-RW"; }),
                    diags.end());
      }
      notes = check_notes(p);
    }
    for (const auto& d : diags) {
      if (o.json)
        c.out += "{\"col\":" + std::to_string(d.pos.col) + ",\"line\":" + std::to_string(d.pos.line) +
                 ",\"message\":" + jstr(d.message) + ",\"rule\":" + jstr(d.rule) + ",\"view\":" + jstr(d.view) + "}\n";
      else
        c.out += diag_text(d) + "\n";
    }
    if (!o.json)
      for (const auto& n : notes) c.out += "note: " + diag_text(n) + "\n";
    c.exit = diags.empty() ? 0 : 1;
    return COH_OK;
  }
  if (cmd == "run" || cmd == "trace") {
    const bool tracing = cmd == "trace" || o.trace;
    for (char ch : schedule)
      if (ch != '0' && ch != '1') throw ConstructionError("schedule must be a string of 0s and 1s");
    if (schedule.size() > 64) throw ConstructionError("schedules longer than 64 answers are not supported");
    uint64_t bits = 0;
    for (size_t i = 0; i < schedule.size(); ++i)
      if (schedule[i] == '1') bits |= 1ull << i;
    Program p = o.raw ? Parser(src).raw() : Parser(src).annotated();
    List prog;
    if (o.raw) {
      prog = p.raw;
    } else {
      if (!o.no_overlap) rewrite(p);
      std::vector<Diag> diags = check_program(p);
      if (o.no_overlap)
        diags.erase(std::remove_if(diags.begin(), diags.end(), [](const Diag& d) { return d.rule == "OVL-MISSING-RW"; }),
                    diags.end());
      if (!diags.empty()) {
        for (const auto& d : diags) c.err += diag_text(d) + "\n";
        c.exit = 1;
        return COH_OK;
      }
      for (const auto& b : p.blocks) {  // translate_program (modes.hpp:61-66)
        List t = translate_block(b, p.decls);
        prog.insert(prog.end(), t.begin(), t.end());
      }
    }
    const KeyMap km = key_map(p.decls);
    if (km.keys.size() > 32) {
      *fatal = "program has " + std::to_string(km.keys.size()) + " store keys; the device interpreter holds 32";
      return COH_E_CONSTRUCTION;
    }
    Emit e{km, {}, {}};
    e.list(prog);
    e.code.push_back(BC_END);
    if (e.code.size() > 65535) {
      *fatal = "program exceeds 64K interpreter instructions";
      return COH_E_CONSTRUCTION;
    }
    if (tracing && o.fuel > (1 << 22)) {
      *fatal = "--trace records at most 4M steps (lower --fuel)";
      return COH_E_ARG;
    }
    RunOut r{};
    std::vector<SweepTrace> tr;
    const int rc = device_run(ctx, e.code, (uint32_t)km.keys.size(), o.fuel, bits, (uint32_t)schedule.size(), &r, fatal,
                              tracing ? &tr : nullptr);
    if (rc) return rc;
    if (tracing) {
      e.head.resize(e.code.size());
      report_trace(km, e.head, tr, o, c);
    }
    report(km, r, o, !schedule.empty(), c);
    return COH_OK;
  }
  if (cmd == "infer" || cmd == "translate") {
    if (o.raw) throw std::runtime_error(cmd + " needs an annotated program");
    Program p = Parser(src).annotated();
    if (!o.no_overlap) rewrite(p);
    if (cmd == "infer") {
      if (o.json) {
        for (size_t i = 0; i < p.blocks.size(); ++i) {
          std::string modes;
          for (const auto& m : p.blocks[i].modes) {
            if (!modes.empty()) modes += ",";
            modes += "{\"kind\":" + jstr(mode_name(m.kind, LOCAL)) + ",\"shadow\":" + (m.shadow ? "true" : "false") +
                     ",\"site\":" + jstr(m.site == REMOTE ? "remote" : "local") + ",\"view\":" + jstr(m.view) + "}";
          }
          c.out += "{\"block\":" + std::to_string(i) + ",\"modes\":[" + modes + "]}\n";
        }
      } else {
        c.out += pretty(p);
      }
    } else {
      for (size_t i = 0; i < p.blocks.size(); ++i) {
        std::string core;
        one_line(translate_block(p.blocks[i], p.decls), core);
        if (o.json) c.out += "{\"block\":" + std::to_string(i) + ",\"core\":" + jstr(core) + "}\n";
        else c.out += "block " + std::to_string(i) + ": " + core + "\n";
      }
    }
    c.exit = 0;
    return COH_OK;
  }
  *fatal = "unknown command '" + cmd + "'";
  return COH_E_ARG;
}

}  // namespace dsl
}  // namespace cohb

namespace {
void put(const std::string& s, char* buf, size_t cap) {
  if (!buf || !cap) return;
  const size_t n = std::min(s.size(), cap - 1);
  std::memcpy(buf, s.data(), n);
  buf[n] = '\0';
}
}  // namespace

extern "C" int coh_cli(coh_ctx* ctx, const char* command, const char* src, const coh_cli_opts* opts, char* out,
                       size_t out_cap, char* err, size_t err_cap, int* exit_code) {
  using namespace cohb::dsl;
  if (!command || !src || !exit_code) return COH_E_ARG;
  coh_cli_opts o = opts ? *opts : coh_cli_opts{0, 0, 0, 10000, nullptr, 0};
  Cli c;
  std::string fatal;
  int rc = COH_OK;
  // exception classes -> CLI exit codes (tools/cohere_main.cpp:262-274)
  try {
    if (o.fuel < 1) throw ConstructionError("--fuel: value must be positive");
    rc = cli(ctx, command, src, o, c, &fatal);
  } catch (const ParseError& e) {
    c.err += std::string("error: ") + e.what() + "\n";
    c.exit = 2;
  } catch (const OverlapError& e) {
    c.err += std::string("error: ") + e.what() + "\n";
    c.exit = 1;
  } catch (const std::exception& e) {
    c.err += std::string("error: ") + e.what() + "\n";
    c.exit = 2;
  }
  if (rc != COH_OK) {
    if (ctx) ctx->err = fatal;
    put(fatal, err, err_cap);
    return rc;
  }
  put(c.out, out, out_cap);
  put(c.err, err, err_cap);
  *exit_code = c.exit;
  return (c.out.size() >= out_cap || c.err.size() >= err_cap) ? -(int)std::max(c.out.size(), c.err.size()) - 1 : COH_OK;
}
