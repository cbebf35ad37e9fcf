// Program-text front end and CLI reporting: the commands of the
// reference tool (tools/cohere_main.cpp:152-276: check / run / trace / infer / translate)
// over program text, with `run` executed on the GPU by the bit-plane interpreter of
// progrun.cu.  The observable behaviour (texts, positions, orders, exit codes) is the
// reference's; the organisation is this file's own:
//
//   * a character-class table drives the scanner; positions are derived from byte
//     offsets through a line-start index (parse.hpp:34-106 defines the token language);
//   * declarations are matched against a table of token patterns (program.hpp:47-130
//     defines their meaning and ConstructionError texts);
//   * statements are parsed without recursion, by a frame stack, into a flat node arena
//     whose targets name declaration symbols (ast.hpp:60-247, parse.hpp:206-340);
//   * the overlap closure works on per-view overlap lists in name order
//     (overlap.hpp:17-20, 86-108, 177-244); translation follows modes.hpp:14-66;
//   * the checker gathers one fact table per block and evaluates its rules over it, with a
//     single must-write set analysis for scalars and cells (checker.hpp:16-318);
//   * printers share one traversal for the one-line and the indented form (pretty.hpp).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <utility>
#include <vector>

#include "internal.hpp"
#include "progrun.hpp"

namespace cohb {
namespace front {

struct Pos {
  int line = 0, col = 0;
};

// Error classes, by the exit code the CLI gives them (tools/cohere_main.cpp:262-274).
struct SyntaxError : std::runtime_error {  // ParseError: "L:C: message", exit 2
  SyntaxError(Pos p, const std::string& m)
      : std::runtime_error(std::to_string(p.line) + ":" + std::to_string(p.col) + ": " + m) {}
};
struct DeclError : std::runtime_error {  // ConstructionError, exit 2
  using std::runtime_error::runtime_error;
};
struct ConflictError : std::runtime_error {  // OverlapInferenceError, exit 1
  explicit ConflictError(const std::string& v)
      : std::runtime_error("inferred modes put '" + v + "' on both sites in one block") {}
};

// ---- source text and scanner --------------------------------------------------------------
class Text {
 public:
  explicit Text(std::string_view s) : s_(s) {
    starts_.push_back(0);
    for (size_t i = 0; i < s_.size(); ++i)
      if (s_[i] == '\n') starts_.push_back(i + 1);
  }
  Pos at(size_t off) const {
    const size_t k = (size_t)(std::upper_bound(starts_.begin(), starts_.end(), off) - starts_.begin());
    return Pos{(int)k, (int)(off - starts_[k - 1] + 1)};
  }
  std::string_view str() const { return s_; }

 private:
  std::string_view s_;
  std::vector<size_t> starts_;
};

enum Tok : uint8_t {
  T_WORD, T_NUM, T_LPAREN, T_RPAREN, T_LBRACE, T_RBRACE, T_LBRACK, T_RBRACK,
  T_SEMI, T_COMMA, T_EQ, T_COLON, T_HAT, T_SHADOW, T_EOF
};
struct Lexeme {
  Tok tok;
  uint32_t off, len;
  long num;
};

enum CharClass : uint8_t { K_BAD = 0, K_SPACE, K_ALPHA, K_DIGIT, K_PUNCT, K_SLASH };
struct ClassTable {
  CharClass cls[256];
  Tok punct[256];
};
constexpr ClassTable make_class_table() {
  ClassTable t{};
  for (int c = 'a'; c <= 'z'; ++c) t.cls[c] = K_ALPHA;
  for (int c = 'A'; c <= 'Z'; ++c) t.cls[c] = K_ALPHA;
  for (int c = '0'; c <= '9'; ++c) t.cls[c] = K_DIGIT;
  t.cls[(int)'_'] = K_ALPHA;
  for (char c : {' ', '\t', '\r', '\n'}) t.cls[(unsigned char)c] = K_SPACE;
  t.cls[(int)'/'] = K_SLASH;
  const char p[] = "(){}[];,=:^";
  const Tok k[] = {T_LPAREN, T_RPAREN, T_LBRACE, T_RBRACE, T_LBRACK, T_RBRACK, T_SEMI, T_COMMA, T_EQ, T_COLON, T_HAT};
  for (int i = 0; i < 11; ++i) {
    t.cls[(unsigned char)p[i]] = K_PUNCT;
    t.punct[(unsigned char)p[i]] = k[i];
  }
  return t;
}
constexpr ClassTable kChars = make_class_table();

std::vector<Lexeme> scan(const Text& text) {
  const std::string_view s = text.str();
  const size_t n = s.size();
  std::vector<Lexeme> out;
  size_t i = 0;
  while (i < n) {
    const unsigned char c = (unsigned char)s[i];
    switch (kChars.cls[c]) {
      case K_SPACE:
        ++i;
        break;
      case K_ALPHA: {
        size_t j = i + 1;
        while (j < n && (kChars.cls[(unsigned char)s[j]] == K_ALPHA || kChars.cls[(unsigned char)s[j]] == K_DIGIT)) ++j;
        out.push_back(Lexeme{T_WORD, (uint32_t)i, (uint32_t)(j - i), 0});
        i = j;
        break;
      }
      case K_DIGIT: {
        long v = 0;
        bool big = false;
        size_t j = i;
        for (; j < n && kChars.cls[(unsigned char)s[j]] == K_DIGIT; ++j) {
          const long d = s[j] - '0';
          if (v > (__LONG_MAX__ - d) / 10) big = true;
          else v = v * 10 + d;
        }
        if (big) throw std::out_of_range("stol");  // the reference converts with std::stol
        out.push_back(Lexeme{T_NUM, (uint32_t)i, (uint32_t)(j - i), v});
        i = j;
        break;
      }
      case K_PUNCT:
        out.push_back(Lexeme{kChars.punct[c], (uint32_t)i, 1, 0});
        ++i;
        break;
      case K_SLASH:
        if (i + 1 < n && s[i + 1] == '/') {
          const size_t e = s.find('\n', i);
          i = e == std::string_view::npos ? n : e;
          break;
        }
        if (i + 1 < n && s[i + 1] == '*') {
          const size_t e = s.find("*/", i + 2);
          if (e == std::string_view::npos) throw SyntaxError(text.at(i), "unterminated comment");
          std::string_view body = s.substr(i + 2, e - i - 2);
          while (!body.empty() && (body.front() == ' ' || body.front() == '\t')) body.remove_prefix(1);
          while (!body.empty() && (body.back() == ' ' || body.back() == '\t')) body.remove_suffix(1);
          if (body == "shadow") out.push_back(Lexeme{T_SHADOW, (uint32_t)i, 0, 0});
          i = e + 2;
          break;
        }
        [[fallthrough]];
      default:
        throw SyntaxError(text.at(i), std::string("unexpected character '") + (char)c + "'");
    }
  }
  out.push_back(Lexeme{T_EOF, (uint32_t)n, 0, 0});
  return out;
}

// ---- declarations, symbols, IR ------------------------------------------------------------
enum Kind : uint8_t { M_R = 0, M_W = 1, M_RW = 2 };
enum Site : uint8_t { LOCAL = 0, REMOTE = 1 };

struct Buffer {
  std::string name;
  int length;
};
struct View {
  std::string name;
  int buffer;
  int lo, hi;
  int length() const { return hi - lo + 1; }
};
struct Symbol {  // a scalar or a view: the names modes, conditions and effects refer to
  bool is_view;
  int index;
};

struct Decls {
  std::vector<std::string> scalars;
  std::vector<Buffer> buffers;
  std::vector<View> views;
  std::vector<Symbol> syms;
  std::unordered_map<std::string, int> sym_by_name, buffer_by_name;

  int sym(const std::string& n) const {
    auto it = sym_by_name.find(n);
    return it == sym_by_name.end() ? -1 : it->second;
  }
  const std::string& name(int s) const { return syms[s].is_view ? views[syms[s].index].name : scalars[syms[s].index]; }
  const View* view_of(int s) const { return s >= 0 && syms[s].is_view ? &views[syms[s].index] : nullptr; }
  bool is_scalar(int s) const { return s >= 0 && !syms[s].is_view; }

  void declare(const std::string& n, bool is_view, int index) {
    sym_by_name.emplace(n, (int)syms.size());
    syms.push_back(Symbol{is_view, index});
  }
  void fresh(const std::string& n) const {
    if (sym(n) >= 0) throw DeclError("duplicate declaration of '" + n + "'");
  }
  void add_scalar(const std::string& n) {
    fresh(n);
    declare(n, false, (int)scalars.size());
    scalars.push_back(n);
  }
  void add_buffer(const std::string& n, int length) {
    if (length < 1) throw DeclError("buffer '" + n + "' needs length >= 1");
    if (buffer_by_name.count(n)) throw DeclError("duplicate buffer '" + n + "'");
    buffer_by_name.emplace(n, (int)buffers.size());
    buffers.push_back(Buffer{n, length});
  }
  void add_view(const std::string& n, const std::string& buf, int lo, int hi) {
    fresh(n);
    auto it = buffer_by_name.find(buf);
    if (it == buffer_by_name.end()) throw DeclError("view '" + n + "' names unknown buffer '" + buf + "'");
    const Buffer& b = buffers[it->second];
    if (lo < 0 || hi >= b.length || lo > hi)
      throw DeclError("view '" + n + "' range [" + std::to_string(lo) + ":" + std::to_string(hi) +
                      "] does not fit buffer '" + b.name + "[" + std::to_string(b.length) + "]'");
    declare(n, true, (int)views.size());
    views.push_back(View{n, it->second, lo, hi});
  }
};

enum TargetKind : uint8_t { G_SCALAR, G_ABSTRACT, G_ELEMENT, G_WHOLE };
struct Target {
  TargetKind kind = G_SCALAR;
  int sym = -1;
  int offset = 0;  // G_ELEMENT: view-relative index
};
enum CondKind : uint8_t { C_VALID = 0, C_GVALID = 1, C_OPAQUE = 2 };
struct Cond {
  CondKind kind = C_OPAQUE;
  bool abstract = false;
  int sym = -1;
};
enum NodeOp : uint8_t { N_EFFECT, N_IF, N_WHILE };
struct Node {
  NodeOp op = N_EFFECT;
  uint8_t eff = 0, site = LOCAL;
  Target t;
  Cond c;
  int kids[2] = {-1, -1};  // lists: then / loop body, else
  Pos pos;
};
struct Mode {
  Kind kind;
  Site site;
  int sym;
  bool shadow;
  Pos pos;
};
struct Block {
  std::vector<Mode> modes;
  int body = -1;
  Pos pos;
};

struct Unit {
  Decls d;
  std::vector<Node> nodes;
  std::vector<std::vector<int>> lists;
  std::vector<Block> blocks;
  int raw = -1;  // --raw: the bare statement list

  int new_list() {
    lists.emplace_back();
    return (int)lists.size() - 1;
  }
  int add(const Node& n) {
    nodes.push_back(n);
    return (int)nodes.size() - 1;
  }
  int cell_of(const Target& t) const { return d.view_of(t.sym)->lo + t.offset; }
};

// ---- parser -------------------------------------------------------------------------------
bool reserved(std::string_view w) {
  static const std::set<std::string_view> words = {"scalar", "buffer", "view", "if", "else", "while", "valid",
                                                   "gvalid", "opaque", "push", "pull", "r", "w", "gr", "gw",
                                                   "R", "W", "RW", "GR", "GW", "GRW"};
  return words.count(w) != 0;
}

struct EffectWord {
  const char* word;
  uint8_t eff, site;
  bool sync;
};
constexpr EffectWord kEffects[] = {{"r", COH_READ, LOCAL, false},  {"w", COH_WRITE, LOCAL, false},
                                   {"gr", COH_READ, REMOTE, false}, {"gw", COH_WRITE, REMOTE, false},
                                   {"push", COH_PUSH, LOCAL, true}, {"pull", COH_PULL, LOCAL, true}};

// Declaration forms as token patterns (parse.hpp:162-204 grammar): a field is a token
// kind plus the phrase its "expected ..." error uses.
struct Field {
  Tok tok;
  const char* what;
};
struct DeclForm {
  const char* keyword;
  int n;
  Field f[8];
};
constexpr DeclForm kDeclForms[] = {
    {"scalar", 1, {{T_WORD, "scalar name"}}},
    {"buffer", 4, {{T_WORD, "buffer name"}, {T_LBRACK, "'['"}, {T_NUM, "buffer length"}, {T_RBRACK, "']'"}}},
    {"view", 8,
     {{T_WORD, "view name"}, {T_EQ, "'='"}, {T_WORD, "buffer name"}, {T_LBRACK, "'['"}, {T_NUM, "range start"},
      {T_COLON, "':'"}, {T_NUM, "range end"}, {T_RBRACK, "']'"}}},
};

bool mode_word(std::string_view w, Kind* k, Site* s) {
  *s = LOCAL;
  if (!w.empty() && w[0] == 'G') {
    *s = REMOTE;
    w.remove_prefix(1);
  }
  if (w == "R") *k = M_R;
  else if (w == "W") *k = M_W;
  else if (w == "RW") *k = M_RW;
  else return false;
  return true;
}

class Reader {
 public:
  explicit Reader(std::string_view src) : text_(src), lx_(scan(text_)) {}

  Unit annotated() {
    Unit u;
    declarations(u.d);
    while (!is(T_EOF)) read_block(u);
    return u;
  }
  Unit raw() {
    Unit u;
    declarations(u.d);
    u.raw = u.new_list();
    read_statements(u, u.raw, /*top_level=*/true);
    return u;
  }

 private:
  const Lexeme& cur() const { return lx_[std::min(k_, lx_.size() - 1)]; }
  Pos where() const { return text_.at(cur().off); }
  std::string_view word() const { return text_.str().substr(cur().off, cur().len); }
  bool is(Tok t) const { return cur().tok == t; }
  bool is_word(std::string_view w) const { return is(T_WORD) && word() == w; }
  const Lexeme& advance() {
    const Lexeme& l = cur();
    if (k_ + 1 < lx_.size()) ++k_;
    return l;
  }
  const Lexeme& need(Tok t, const char* what) {
    if (!is(t)) throw SyntaxError(where(), std::string("expected ") + what);
    return advance();
  }
  std::string ident(const char* what) {
    const Lexeme& l = need(T_WORD, what);
    std::string s(text_.str().substr(l.off, l.len));
    if (reserved(s)) throw SyntaxError(text_.at(l.off), "'" + s + "' is reserved and cannot name a variable");
    return s;
  }
  template <class F>
  void at_pos(Pos p, F&& f) {  // a ConstructionError reported at the declaration / name
    try {
      f();
    } catch (const DeclError& e) {
      throw SyntaxError(p, e.what());
    }
  }

  void declarations(Decls& d) {
    for (;;) {
      const DeclForm* form = nullptr;
      for (const DeclForm& f : kDeclForms)
        if (is_word(f.keyword)) form = &f;
      if (!form) return;
      const Pos pos = where();
      advance();
      std::vector<std::string> names;
      std::vector<int> nums;
      for (int i = 0; i < form->n; ++i) {
        const Field& f = form->f[i];
        if (f.tok == T_WORD) names.push_back(ident(f.what));
        else if (f.tok == T_NUM) nums.push_back((int)need(T_NUM, f.what).num);
        else need(f.tok, f.what);
      }
      at_pos(pos, [&] {
        if (form == &kDeclForms[0]) d.add_scalar(names[0]);
        else if (form == &kDeclForms[1]) d.add_buffer(names[0], nums[0]);
        else d.add_view(names[0], names[1], nums[0], nums[1]);
      });
    }
  }

  Mode read_mode(const Decls& d, const Block& b) {
    Kind k;
    Site s;
    if (!is(T_WORD) || !mode_word(word(), &k, &s)) throw SyntaxError(where(), "expected an access mode");
    const Pos pos = where();
    advance();
    need(T_LPAREN, "'('");
    const std::string v = ident("variable name");
    need(T_RPAREN, "')'");
    const int sym = d.sym(v);
    if (sym < 0) throw SyntaxError(pos, "mode names undeclared variable '" + v + "'");
    Mode m{k, s, sym, false, pos};
    if (is(T_SHADOW)) {
      advance();
      m.shadow = true;
    }
    for (const Mode& o : b.modes)
      if (o.sym == sym) throw SyntaxError(pos, "variable '" + v + "' declared twice in one block");
    return m;
  }

  void read_block(Unit& u) {
    Block b;
    b.pos = where();
    Kind k;
    Site s;
    if (is(T_WORD) && mode_word(word(), &k, &s)) {
      b.modes.push_back(read_mode(u.d, b));
      while (is(T_COMMA)) {
        advance();
        b.modes.push_back(read_mode(u.d, b));
      }
    }
    if (is_word("scalar") || is_word("buffer") || is_word("view"))
      throw SyntaxError(where(), "declarations must precede all blocks");
    need(T_LBRACE, "mode list or '{'");
    b.body = u.new_list();
    read_statements(u, b.body, false);
    u.blocks.push_back(std::move(b));
  }

  Cond read_cond(const Decls& d) {
    Cond c;
    if (is_word("opaque")) {
      advance();
      return c;
    }
    if (is_word("valid")) c.kind = C_VALID;
    else if (is_word("gvalid")) c.kind = C_GVALID;
    else throw SyntaxError(where(), "expected valid(...), gvalid(...) or opaque");
    advance();
    need(T_LPAREN, "'('");
    const Pos pos = where();
    const std::string n = ident("variable name");
    const bool hat = is(T_HAT);
    if (hat) advance();
    need(T_RPAREN, "')'");
    c.sym = d.sym(n);
    if (c.sym < 0) throw SyntaxError(pos, "condition names undeclared variable '" + n + "'");
    c.abstract = hat || d.view_of(c.sym);  // a bare view name is its flag pair
    return c;
  }

  Node read_effect(const Decls& d) {
    const EffectWord* ew = nullptr;
    for (const EffectWord& e : kEffects)
      if (word() == e.word) ew = &e;
    if (!ew) throw SyntaxError(where(), "expected a statement");
    Node n;
    n.eff = ew->eff;
    n.site = ew->site;
    n.pos = where();
    advance();
    const Pos np = where();
    const std::string v = ident("variable name");
    const int sym = d.sym(v);
    if (is(T_LBRACK)) {
      advance();
      const int off = (int)need(T_NUM, "element index").num;
      need(T_RBRACK, "']'");
      if (ew->sync) throw SyntaxError(np, "push/pull take a whole variable, not an element");
      if (d.is_scalar(sym)) throw SyntaxError(np, "scalar '" + v + "' takes no index");
      at_pos(np, [&] {
        const View* view = d.view_of(sym);
        if (!view) throw DeclError("unknown view '" + v + "'");
        if (off < 0 || off >= view->length())
          throw DeclError("index " + std::to_string(off) + " outside view '" + v + "' of length " +
                          std::to_string(view->length()));
      });
      n.t = Target{G_ELEMENT, sym, off};
    } else if (d.is_scalar(sym)) {
      n.t = Target{G_SCALAR, sym, 0};
    } else if (d.view_of(sym)) {
      if (!ew->sync) throw SyntaxError(np, "view '" + v + "' needs an element index here");
      n.t = Target{G_WHOLE, sym, 0};
    } else {
      throw SyntaxError(np, "undeclared variable '" + v + "'");
    }
    need(T_SEMI, "';'");
    return n;
  }

  // Statement lists without recursion: a frame per open list.  A frame closes at its '}'
  // (the top level of a raw program at the end of input); closing an if's then-list may
  // open its else-list.
  void read_statements(Unit& u, int list, bool top_level) {
    struct Frame {
      int list, node;
      bool then_part;
    };
    std::vector<Frame> open{{list, -1, false}};
    while (!open.empty()) {
      const Frame f = open.back();
      const bool outer = top_level && open.size() == 1;
      if (outer ? is(T_EOF) : is(T_RBRACE)) {
        if (!outer) advance();
        open.pop_back();
        if (f.then_part && is_word("else")) {
          advance();
          need(T_LBRACE, "'{'");
          open.push_back(Frame{u.nodes[f.node].kids[1], f.node, false});
        }
        continue;
      }
      if (!is(T_WORD)) throw SyntaxError(where(), "expected a statement");
      if (is_word("if") || is_word("while")) {
        Node n;
        n.op = is_word("if") ? N_IF : N_WHILE;
        n.pos = where();
        advance();
        need(T_LPAREN, "'('");
        n.c = read_cond(u.d);
        need(T_RPAREN, "')'");
        need(T_LBRACE, "'{'");
        n.kids[0] = u.new_list();
        n.kids[1] = u.new_list();
        const int id = u.add(n);
        u.lists[f.list].push_back(id);
        open.push_back(Frame{n.kids[0], id, n.op == N_IF});
        continue;
      }
      u.lists[f.list].push_back(u.add(read_effect(u.d)));
    }
  }

  Text text_;
  std::vector<Lexeme> lx_;
  size_t k_ = 0;
};

// ---- printing -------------------------------------------------------------------------------
const char* effect_name(uint32_t e) {
  static const char* n[] = {"push", "pull", "r", "w", "noop"};
  return n[e];
}
std::string mode_name(Kind k, Site s) { return std::string(s == REMOTE ? "G" : "") + (k == M_R ? "R" : k == M_W ? "W" : "RW"); }

class Printer {
 public:
  Printer(const Unit& u, bool indented) : u_(u), indented_(indented) {}

  std::string target(const Target& t) const {
    const std::string& n = u_.d.name(t.sym);
    if (t.kind == G_ABSTRACT) return n + "^";
    if (t.kind == G_ELEMENT) return n + "[" + std::to_string(t.offset) + "]";
    return n;
  }
  std::string cond(const Cond& c) const {
    if (c.kind == C_OPAQUE) return "opaque";
    return std::string(c.kind == C_VALID ? "valid(" : "gvalid(") + u_.d.name(c.sym) + (c.abstract ? "^" : "") + ")";
  }
  std::string effect(const Node& n) const {
    return std::string(n.site == REMOTE ? "g" : "") + effect_name(n.eff) + " " + target(n.t) + ";";
  }
  // A statement list (by node ids), one-line (stmt_one_line) or indented (stmt_lines).
  std::string list(const std::vector<int>& ids, int depth = 0) const {
    std::string out;
    for (int id : ids) piece(u_.nodes[id], depth, out);
    return out;
  }
  std::string node(const Node& n) const {
    std::string out;
    piece(n, 0, out);
    return out;
  }

 private:
  void piece(const Node& n, int depth, std::string& out) const {
    const std::string pad = indented_ ? std::string(2 * (size_t)depth, ' ') : std::string();
    const char* gap = indented_ ? "\n" : "";
    if (!indented_ && !out.empty()) out += ' ';
    if (n.op == N_EFFECT) {
      out += pad + effect(n) + gap;
      return;
    }
    const std::string head = std::string(n.op == N_IF ? "if (" : "while (") + cond(n.c) + ")";
    const std::vector<int>& a = u_.lists[n.kids[0]];
    const std::vector<int>& b = u_.lists[n.kids[1]];
    if (indented_) {
      out += pad + head + " {\n" + list(a, depth + 1);
      if (n.op == N_IF && !b.empty()) out += pad + "} else {\n" + list(b, depth + 1);
      out += pad + "}\n";
      return;
    }
    const std::string ta = list(a);
    out += head + " { " + ta + (ta.empty() ? "}" : " }");
    if (n.op == N_IF && !b.empty()) out += " else { " + list(b) + " }";
  }

  const Unit& u_;
  bool indented_;
};

std::string mode_text(const Unit& u, const Mode& m) {
  return mode_name(m.kind, m.site) + "(" + u.d.name(m.sym) + ")" + (m.shadow ? " /*shadow*/" : "");
}

std::string pretty(const Unit& u) {  // pretty.hpp:113-148
  std::string out;
  for (const auto& s : u.d.scalars) out += "scalar " + s + "\n";
  for (const auto& b : u.d.buffers) out += "buffer " + b.name + "[" + std::to_string(b.length) + "]\n";
  for (const auto& v : u.d.views)
    out += "view " + v.name + " = " + u.d.buffers[v.buffer].name + "[" + std::to_string(v.lo) + ":" +
           std::to_string(v.hi) + "]\n";
  const Printer pr(u, true);
  for (const Block& b : u.blocks) {
    if (!out.empty()) out += "\n";
    std::string header;
    for (size_t i = 0; i < b.modes.size(); ++i) header += (i ? ", " : "") + mode_text(u, b.modes[i]);
    out += header + (header.empty() ? "{\n" : " {\n") + pr.list(u.lists[b.body], 1) + "}\n";
  }
  return out;
}

// ---- overlaps and the mode closure ----------------------------------------------------------
// Per view, the other views on its buffer whose ranges intersect it, in name order (the
// order registry queries return, overlap.hpp:86-108).
std::vector<std::vector<int>> overlap_lists(const Decls& d) {
  std::vector<int> by_name(d.views.size());
  for (size_t i = 0; i < by_name.size(); ++i) by_name[i] = (int)i;
  std::sort(by_name.begin(), by_name.end(), [&](int a, int b) { return d.views[a].name < d.views[b].name; });
  std::vector<std::vector<int>> out(d.views.size());
  for (size_t v = 0; v < d.views.size(); ++v)
    for (int y : by_name) {
      const View &p = d.views[v], &q = d.views[y];
      if ((size_t)y != v && q.buffer == p.buffer && q.lo <= p.hi && q.hi >= p.lo) out[v].push_back(y);
    }
  return out;
}

// infer_overlap_closure (overlap.hpp:177-230): a W / RW mode on a view requires RW at the
// same site on every view sharing cells with it (a W already declared at that site on the
// other view satisfies a W); such a view already in the block is upgraded from R, the rest
// are appended as shadow modes in declaration order; two sites for one view conflict.
std::vector<Mode> close_modes(const std::vector<Mode>& modes, const Decls& d,
                              const std::vector<std::vector<int>>& ovl) {
  std::vector<int> need(d.views.size(), -1), mode_of(d.views.size(), -1);
  for (size_t i = 0; i < modes.size(); ++i)
    if (const View* v = d.view_of(modes[i].sym)) mode_of[v - d.views.data()] = (int)i;
  std::vector<int> order;  // views needing a mode, recorded in name order below
  for (const Mode& m : modes) {
    const View* v = d.view_of(m.sym);
    if (m.kind == M_R || m.shadow || !v) continue;
    for (int y : ovl[v - d.views.data()]) {
      const int o = mode_of[y];
      if (m.kind == M_W && o >= 0 && modes[o].kind == M_W && modes[o].site == m.site) continue;
      if (need[y] < 0) need[y] = m.site;
      else if (need[y] != m.site) throw ConflictError(d.views[y].name);
    }
  }
  for (size_t y = 0; y < need.size(); ++y)
    if (need[y] >= 0) order.push_back((int)y);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return d.views[a].name < d.views[b].name; });
  std::vector<Mode> out = modes;
  std::vector<char> shadow(d.views.size(), 0);
  for (int y : order) {
    if (mode_of[y] >= 0) {
      Mode& e = out[mode_of[y]];
      if (e.site != need[y]) throw ConflictError(d.views[y].name);
      if (e.kind == M_R) e.kind = M_RW;
    } else {
      shadow[y] = 1;
    }
  }
  for (size_t y = 0; y < d.views.size(); ++y)
    if (shadow[y]) out.push_back(Mode{M_RW, (Site)need[y], d.sym(d.views[y].name), true, Pos{}});
  return out;
}

void close_program(Unit& u) {  // rewrite_program (overlap.hpp:234-244)
  const auto ovl = overlap_lists(u.d);
  for (Block& b : u.blocks) b.modes = close_modes(b.modes, u.d, ovl);
}

// ---- translation (modes.hpp:14-66) ----------------------------------------------------------
// R / GR:  if (valid(x^)) { } else { pull x; pull x^; }  (push for the remote form; the
// syncs are local-site statements); W: w x^ at the mode's site; RW: both; then the body.
int translate(Unit& u, const Block& b) {
  const int out = u.new_list();
  for (const Mode& m : b.modes) {
    if (m.kind != M_W) {
      const uint8_t sync = m.site == REMOTE ? COH_PUSH : COH_PULL;
      Node g;
      g.op = N_IF;
      g.c = Cond{m.site == REMOTE ? C_GVALID : C_VALID, true, m.sym};
      g.kids[0] = u.new_list();
      g.kids[1] = u.new_list();
      Node conc;
      conc.eff = sync;
      conc.t = Target{u.d.view_of(m.sym) ? G_WHOLE : G_SCALAR, m.sym, 0};
      Node abs = conc;
      abs.t = Target{G_ABSTRACT, m.sym, 0};
      const int c_id = u.add(conc), a_id = u.add(abs);
      u.lists[g.kids[1]] = {c_id, a_id};
      const int g_id = u.add(g);
      u.lists[out].push_back(g_id);
    }
    if (m.kind != M_R) {
      Node w;
      w.eff = COH_WRITE;
      w.site = m.site;
      w.t = Target{G_ABSTRACT, m.sym, 0};
      const int w_id = u.add(w);
      u.lists[out].push_back(w_id);
    }
  }
  const std::vector<int> body = u.lists[b.body];
  for (int id : body) u.lists[out].push_back(id);
  return out;
}

// ---- checker --------------------------------------------------------------------------------
struct Diag {
  std::string rule, subject;
  Pos pos;
  std::string message;
};

// What one block's body does, gathered in one pre-order walk (then before else).
struct Facts {
  struct Use {
    std::string name;
    int site;
    bool reads = false, writes = false;
    Pos first_touch, first_read, first_write;
    std::set<int> cells;  // absolute cells written through element targets
  };
  std::vector<Use> uses;  // sorted by (name, site) after the walk
  int sync_sym = -1, abs_sym = -1;
  Pos sync_pos, abs_pos;

  const Use* find(const std::string& n, int site) const {
    for (const Use& x : uses)
      if (x.name == n && x.site == site) return &x;
    return nullptr;
  }
};

Facts gather(const Unit& u, int list) {
  Facts f;
  std::map<std::pair<std::string, int>, size_t> slot;
  std::vector<std::pair<int, size_t>> stack{{list, 0}};
  while (!stack.empty()) {
    auto& [l, i] = stack.back();
    if (i >= u.lists[l].size()) {
      stack.pop_back();
      continue;
    }
    const Node& n = u.nodes[u.lists[l][i++]];
    if (n.op != N_EFFECT) {
      if (n.op == N_IF) stack.push_back({n.kids[1], 0});  // visited after the then-list
      stack.push_back({n.kids[0], 0});
      continue;
    }
    if (n.t.kind == G_ABSTRACT) {
      if (f.abs_sym < 0) f.abs_sym = n.t.sym, f.abs_pos = n.pos;
      continue;
    }
    const auto key = std::make_pair(u.d.name(n.t.sym), (int)n.site);
    auto it = slot.find(key);
    if (it == slot.end()) {
      it = slot.emplace(key, f.uses.size()).first;
      Facts::Use x;
      x.name = key.first;
      x.site = key.second;
      x.first_touch = n.pos;
      f.uses.push_back(x);
    }
    Facts::Use& x = f.uses[it->second];
    if (n.eff == COH_READ) {
      if (!x.reads) x.first_read = n.pos;
      x.reads = true;
    } else if (n.eff == COH_WRITE) {
      if (!x.writes) x.first_write = n.pos;
      x.writes = true;
      if (n.t.kind == G_ELEMENT) x.cells.insert(u.cell_of(n.t));
    } else if (f.sync_sym < 0) {
      f.sync_sym = n.t.sym, f.sync_pos = n.pos;
    }
  }
  std::sort(f.uses.begin(), f.uses.end(),
            [](const Facts::Use& a, const Facts::Use& b) { return std::tie(a.name, a.site) < std::tie(b.name, b.site); });
  return f;
}

// Writes that happen on every path through a list (checker.hpp:125-170): (symbol, site,
// cell or -1 for a scalar).  An if contributes what both branches do; a loop nothing.
using WriteKey = std::tuple<int, int, int>;
std::set<WriteKey> certain_writes(const Unit& u, int list) {
  std::set<WriteKey> out;
  for (int id : u.lists[list]) {
    const Node& n = u.nodes[id];
    if (n.op == N_EFFECT) {
      if (n.eff == COH_WRITE && n.t.kind == G_SCALAR) out.emplace(n.t.sym, n.site, -1);
      if (n.eff == COH_WRITE && n.t.kind == G_ELEMENT) out.emplace(n.t.sym, n.site, u.cell_of(n.t));
    } else if (n.op == N_IF) {
      const std::set<WriteKey> a = certain_writes(u, n.kids[0]), b = certain_writes(u, n.kids[1]);
      for (const WriteKey& k : a)
        if (b.count(k)) out.insert(k);
    }
  }
  return out;
}

const char* site_word(int s) { return s == LOCAL ? "local" : "remote"; }

void rule_sync_and_abstract(const Unit& u, const Block&, const Facts& f, std::vector<Diag>& out) {
  if (f.sync_sym >= 0)
    out.push_back({"D2-NO-SYNC", u.d.name(f.sync_sym), f.sync_pos,
                   "declared blocks may not push or pull; declare a mode instead"});
  if (f.abs_sym >= 0) {
    const std::string& n = u.d.name(f.abs_sym);
    out.push_back({"BODY-ABSTRACT-EFFECT", n, f.abs_pos, "abstract key '" + n + "^' cannot be addressed from a body"});
  }
}

const Mode* mode_for(const Unit& u, const Block& b, const std::string& name) {
  for (const Mode& m : b.modes)
    if (u.d.name(m.sym) == name) return &m;
  return nullptr;
}

void rule_undeclared(const Unit& u, const Block& b, const Facts& f, std::vector<Diag>& out) {
  for (const Facts::Use& x : f.uses) {
    const Mode* m = mode_for(u, b, x.name);
    const bool here = m && (int)m->site == x.site;
    if (x.reads && !(here && m->kind != M_W))
      out.push_back({"D2-UNDECLARED-READ", x.name, x.first_read,
                     "'" + x.name + "' is read " + site_word(x.site) + "ly but has no R or RW declaration there"});
    if (x.writes && !(here && m->kind != M_R))
      out.push_back({"D2-UNDECLARED-WRITE", x.name, x.first_write,
                     "'" + x.name + "' is written " + site_word(x.site) + "ly but has no W or RW declaration there"});
  }
}

void rule_write_coverage(const Unit& u, const Block& b, const Facts&, std::vector<Diag>& out) {
  std::set<WriteKey> sure;
  bool have = false;
  for (const Mode& m : b.modes) {
    if (m.kind != M_W) continue;
    if (!have) sure = certain_writes(u, b.body), have = true;
    const std::string& n = u.d.name(m.sym);
    if (const View* v = u.d.view_of(m.sym)) {
      bool all = true;
      for (int c = v->lo; c <= v->hi && all; ++c) all = sure.count(WriteKey{m.sym, m.site, c}) != 0;
      if (!all)
        out.push_back({"D4-W-NOT-ALL-ELEMENTS", n, m.pos, "'" + n + "' is declared W but some cells are not written on every path"});
    } else if (!sure.count(WriteKey{m.sym, m.site, -1})) {
      out.push_back({"D2-W-NOT-ALL-PATHS", n, m.pos, "'" + n + "' is declared W but not written on every path"});
    }
  }
}

void rule_overlap(const Unit& u, const Block& b, const Facts& f, const std::vector<std::vector<int>>& ovl,
                  std::vector<Diag>& out) {
  for (const Facts::Use& x : f.uses) {
    const View* v = x.writes ? u.d.view_of(u.d.sym(x.name)) : nullptr;
    if (!v) continue;
    for (int y : ovl[v - u.d.views.data()]) {
      const View& o = u.d.views[y];
      const int lo = std::max(v->lo, o.lo), hi = std::min(v->hi, o.hi);
      auto it = x.cells.lower_bound(lo);
      if (it == x.cells.end() || *it > hi) continue;
      const Mode* om = mode_for(u, b, o.name);
      if (om && (int)om->site == x.site && om->kind != M_R) continue;
      out.push_back({"OVL-MISSING-RW", o.name, x.first_write,
                     "writes through '" + x.name + "' reach cells shared with '" + o.name +
                         "', which needs W or RW at the same site"});
    }
  }
}

void rule_mixed_site(const Facts& f, std::vector<Diag>& out) {  // check_localised (checker.hpp:191-208)
  for (const Facts::Use& x : f.uses)
    if (x.site == LOCAL && f.find(x.name, REMOTE))
      out.push_back({"P3-MIXED-SITE", x.name, x.first_touch, "'" + x.name + "' is accessed from both sites in one body"});
}

std::vector<Diag> check_unit(const Unit& u, bool with_overlaps) {
  std::vector<Diag> out;
  std::vector<std::vector<int>> ovl = overlap_lists(u.d);
  if (!with_overlaps) ovl.assign(u.d.views.size(), {});  // an empty registry (tools/cohere_main.cpp:67-68)
  for (const Block& b : u.blocks) {
    const Facts f = gather(u, b.body);
    rule_sync_and_abstract(u, b, f, out);
    rule_undeclared(u, b, f, out);
    rule_write_coverage(u, b, f, out);
    rule_overlap(u, b, f, ovl, out);
    rule_mixed_site(f, out);
  }
  return out;
}

std::vector<Diag> unused_modes(const Unit& u) {  // check_notes (checker.hpp:302-318)
  std::vector<Diag> out;
  for (const Block& b : u.blocks) {
    const Facts f = gather(u, b.body);
    for (const Mode& m : b.modes) {
      if (m.kind != M_R || m.shadow) continue;
      const std::string& n = u.d.name(m.sym);
      const Facts::Use* x = f.find(n, m.site);
      if (!x || !x->reads)
        out.push_back({"NOTE-UNUSED-MODE", n, m.pos, "'" + n + "' is declared " + mode_name(m.kind, m.site) + " but never read"});
    }
  }
  return out;
}

// ---- the store's keys and the device program ---------------------------------------------------
// initial_store (program.hpp:174-184) keys, numbered: per scalar its concrete and abstract
// key, every buffer cell, every view's abstract key.  VarKey order (ast.hpp:30-46) sorts
// by name, then kind Scalar < Element < Abstract, then index.
struct KeySpace {
  struct Key {
    std::string name;
    uint8_t kind;  // 0 scalar, 1 element, 2 abstract
    int index;
  };
  std::vector<Key> keys;
  std::vector<uint32_t> scalar_key, scalar_abs, buffer_base, view_abs;

  explicit KeySpace(const Decls& d) {
    for (const auto& s : d.scalars) {
      scalar_key.push_back((uint32_t)keys.size());
      keys.push_back({s, 0, -1});
      scalar_abs.push_back((uint32_t)keys.size());
      keys.push_back({s, 2, -1});
    }
    for (const auto& b : d.buffers) {
      buffer_base.push_back((uint32_t)keys.size());
      for (int i = 0; i < b.length; ++i) keys.push_back({b.name, 1, i});
    }
    for (const auto& v : d.views) {
      view_abs.push_back((uint32_t)keys.size());
      keys.push_back({v.name, 2, -1});
    }
  }
  std::string text(uint32_t k) const {
    const Key& x = keys[k];
    if (x.kind == 1) return x.name + "[" + std::to_string(x.index) + "]";
    return x.kind == 2 ? x.name + "^" : x.name;
  }
  std::vector<uint32_t> sorted() const {
    std::vector<uint32_t> o(keys.size());
    for (uint32_t i = 0; i < o.size(); ++i) o[i] = i;
    std::sort(o.begin(), o.end(), [&](uint32_t a, uint32_t b) {
      return std::tie(keys[a].name, keys[a].kind, keys[a].index) < std::tie(keys[b].name, keys[b].kind, keys[b].index);
    });
    return o;
  }
};

class Lowering {  // node lists -> ProgIns, with the one-line text of each statement
 public:
  Lowering(const Unit& u, const KeySpace& ks) : u_(u), ks_(ks), pr_(u, false) {}

  uint32_t key(const Target& t) const {
    const Symbol& s = u_.d.syms[t.sym];
    if (t.kind == G_ABSTRACT) return s.is_view ? ks_.view_abs[s.index] : ks_.scalar_abs[s.index];
    if (t.kind == G_ELEMENT) return ks_.buffer_base[u_.d.views[s.index].buffer] + (uint32_t)u_.cell_of(t);
    return ks_.scalar_key[s.index];
  }
  uint32_t cond_key(const Cond& c) const {
    if (c.kind == C_OPAQUE) return 0;
    return key(Target{c.abstract ? G_ABSTRACT : G_SCALAR, c.sym, 0});
  }
  void lower(int list) {
    for (int id : u_.lists[list]) {
      const Node& n = u_.nodes[id];
      heads.resize(code.size() + 1);
      heads[code.size()] = pr_.node(n);
      if (n.op == N_EFFECT) {
        const uint32_t op = (n.eff << 4) | ((uint32_t)n.site << 7);
        if (n.t.kind == G_WHOLE) {
          const View& v = *u_.d.view_of(n.t.sym);
          const uint32_t base = ks_.buffer_base[v.buffer];
          code.push_back(ProgIns{PI_WHOLE | op, base + (uint32_t)v.lo, base + (uint32_t)v.hi, 0});
        } else {
          code.push_back(ProgIns{PI_EFF | op, key(n.t), 0, 0});
        }
        continue;
      }
      const size_t head = code.size();
      code.push_back(ProgIns{(n.op == N_IF ? PI_IF : PI_WHILE) | ((uint32_t)n.c.kind << 8), cond_key(n.c), 0, 0});
      lower(n.kids[0]);
      if (n.op == N_WHILE) {
        code.push_back(ProgIns{PI_JMP, 0, 0, (uint32_t)head});
        code[head].target = (uint32_t)code.size();
      } else if (u_.lists[n.kids[1]].empty()) {
        code[head].target = (uint32_t)code.size();
      } else {
        const size_t jump = code.size();
        code.push_back(ProgIns{PI_JMP, 0, 0, 0});
        code[head].target = (uint32_t)code.size();
        lower(n.kids[1]);
        code[jump].target = (uint32_t)code.size();
      }
    }
  }

  std::vector<ProgIns> code;
  std::vector<std::string> heads;

 private:
  const Unit& u_;
  const KeySpace& ks_;
  Printer pr_;
};

// ---- reporting (tools/cohere_main.cpp:38-158) -----------------------------------------------------
std::string quoted(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}
std::string pair_text(uint32_t p) {
  return std::string("(") + ((p & 1u) ? "V" : "I") + "," + ((p & 2u) ? "V" : "I") + ")";
}
std::string store_json(const std::string& key, uint32_t p) {
  return "{\"key\":" + quoted(key) + ",\"local\":" + quoted((p & 1u) ? "V" : "I") + ",\"remote\":" +
         quoted((p & 2u) ? "V" : "I") + "}";
}
const char* needs_text(uint32_t eff) {  // pre_to_string(effect_signature(e)) (validity.hpp:79-99)
  static const char* p[] = {"(V,*)", "(*,V)", "(V,*)", "(*,*)", "(*,*)"};
  return p[eff];
}

struct Outcome {
  std::string out, err;
  int exit = 0;
};

void report_run(const KeySpace& ks, const std::vector<std::string>& heads, const ProgRunResult& r, bool json,
                bool trace, bool schedule_given, Outcome& o) {
  static const char* status_name[] = {"done", "stuck", "fuel-exhausted", "defect"};
  static const char* rule_name[] = {"effect", "remote-effect", "while-true", "while-false", "if-true", "if-false"};
  if (trace) {
    uint32_t d0 = 0;
    for (size_t i = 0; i < r.trace.size(); ++i) {
      const ProgStep& st = r.trace[i];
      std::string delta;
      for (uint32_t k = d0; k < st.delta_end; ++k) {
        const ProgDelta& x = r.deltas[k];
        if (json) delta += (delta.empty() ? "" : ",") + store_json(ks.text(x.key), x.pair);
        else delta += (delta.empty() ? " => " : " ") + ks.text(x.key) + "=" + pair_text(x.pair);
      }
      d0 = st.delta_end;
      if (json) {
        o.out += "{\"delta\":[" + delta + "],\"head\":" + quoted(heads[st.pc]) + ",\"rule\":" + quoted(rule_name[st.rule]) +
                 ",\"step\":" + std::to_string(i + 1) + "}\n";
      } else {
        std::string line = std::to_string(i + 1) + " " + rule_name[st.rule];
        if (line.size() < 16) line.append(16 - line.size(), ' ');
        o.out += line + heads[st.pc] + delta + "\n";
      }
    }
  }
  const bool stuck = r.status == COH_RUN_STUCK;
  if (json) {
    o.out += "{\"outcome\":" + quoted(status_name[r.status]) + ",\"schedule_consumed\":" + std::to_string(r.consumed) +
             ",\"steps\":" + std::to_string(r.steps);
    if (stuck)
      o.out += ",\"stuck\":{\"effect\":" + quoted(effect_name(r.stuck_eff)) + ",\"have\":" + quoted(pair_text(r.stuck_actual)) +
               ",\"key\":" + quoted(ks.text(r.stuck_key)) + ",\"site\":" + quoted(r.stuck_site ? "remote" : "local") + "}";
    o.out += "}\n";
  } else {
    o.out += std::string("outcome: ") + status_name[r.status] + "\nsteps: " + std::to_string(r.steps) + "\n";
    if (stuck)  // StuckInfo::describe (semantics.hpp:68-74)
      o.out += std::string("stuck at: ") + (r.stuck_site ? "g" : "") + effect_name(r.stuck_eff) + " " +
               ks.text(r.stuck_key) + ": have " + pair_text(r.stuck_actual) + ", need " + needs_text(r.stuck_eff) +
               (r.stuck_site ? " against the swapped pair" : "") + "\n";
  }
  for (uint32_t k : ks.sorted()) {
    const uint32_t p = ((r.L[k >> 5] >> (k & 31u)) & 1u) | (((r.R[k >> 5] >> (k & 31u)) & 1u) << 1);
    o.out += json ? store_json(ks.text(k), p) + "\n" : ks.text(k) + " " + pair_text(p) + "\n";
  }
  if (r.overflowed && schedule_given) o.err += "note: schedule exhausted; later opaque conditions answered false\n";
  o.exit = r.status == COH_RUN_DONE ? 0 : r.status == COH_RUN_STUCK ? 3 : 4;
}

std::string diag_line(const Diag& d) {
  return std::to_string(d.pos.line) + ":" + std::to_string(d.pos.col) + ": " + d.rule + " [" + d.subject + "] " + d.message;
}

// ---- commands ---------------------------------------------------------------------------------------
int command(coh_ctx* ctx, const std::string& cmd, std::string_view src, const coh_cli_opts& opt, Outcome& o,
            std::string* fatal) {
  if (cmd == "check") {  // cmd_check (tools/cohere_main.cpp:58-90)
    std::vector<Diag> diags, notes;
    if (opt.raw) {
      Unit u = Reader(src).raw();
      const Facts f = gather(u, u.raw);
      rule_mixed_site(f, diags);
    } else {
      Unit u = Reader(src).annotated();
      diags = check_unit(u, !opt.no_overlap);
      notes = unused_modes(u);
    }
    for (const Diag& d : diags)
      o.out += opt.json ? "{\"col\":" + std::to_string(d.pos.col) + ",\"line\":" + std::to_string(d.pos.line) +
                              ",\"message\":" + quoted(d.message) + ",\"rule\":" + quoted(d.rule) + ",\"view\":" +
                              quoted(d.subject) + "}\n"
                        : diag_line(d) + "\n";
    if (!opt.json)
      for (const Diag& n : notes) o.out += "note: " + diag_line(n) + "\n";
    o.exit = diags.empty() ? 0 : 1;
    return COH_OK;
  }
  if (cmd == "run" || cmd == "trace") {  // cmd_run (tools/cohere_main.cpp:152-179)
    const bool tracing = cmd == "trace" || opt.trace;
    const std::string schedule = opt.schedule ? opt.schedule : "";
    uint64_t bits = 0;
    for (size_t i = 0; i < schedule.size(); ++i) {
      if (schedule[i] != '0' && schedule[i] != '1') throw DeclError("schedule must be a string of 0s and 1s");
      if (schedule[i] == '1' && i < 64) bits |= 1ull << i;
    }
    if (schedule.size() > 64) throw DeclError("schedules longer than 64 answers are not supported");
    Unit u = opt.raw ? Reader(src).raw() : Reader(src).annotated();
    int prog = u.raw;
    if (!opt.raw) {
      if (!opt.no_overlap) close_program(u);
      const std::vector<Diag> diags = check_unit(u, !opt.no_overlap);
      if (!diags.empty()) {
        for (const Diag& d : diags) o.err += diag_line(d) + "\n";
        o.exit = 1;
        return COH_OK;
      }
      prog = u.new_list();  // translate_program: the blocks' core forms in sequence
      const size_t nb = u.blocks.size();
      for (size_t i = 0; i < nb; ++i) {
        const int t = translate(u, u.blocks[i]);
        const std::vector<int> part = u.lists[t];
        u.lists[prog].insert(u.lists[prog].end(), part.begin(), part.end());
      }
    }
    if (tracing && opt.fuel > (1 << 22)) {
      *fatal = "--trace records at most 4M steps (lower --fuel)";
      return COH_E_ARG;
    }
    if (!ctx) {
      *fatal = "run needs a device context";
      return COH_E_ARG;
    }
    const KeySpace ks(u.d);
    if (ks.keys.size() >= (1ull << 32) - 64) {
      *fatal = "program has too many store keys";
      return COH_E_CONSTRUCTION;
    }
    Lowering low(u, ks);
    low.lower(prog);
    low.code.push_back(ProgIns{PI_END, 0, 0, 0});
    if (cudaSetDevice(ctx->device) != cudaSuccess) {
      *fatal = "cudaSetDevice failed";
      return COH_E_CUDA;
    }
    ProgRunResult r;
    const int rc = prog_run(low.code, (uint32_t)ks.keys.size(), opt.fuel, bits,
                            (uint32_t)std::min<size_t>(schedule.size(), 64), tracing, &r, fatal);
    if (rc) return rc;
    ctx->launches++;
    report_run(ks, low.heads, r, opt.json, tracing, !schedule.empty(), o);
    return COH_OK;
  }
  if (cmd == "infer" || cmd == "translate") {  // cmd_infer / cmd_translate (tools/cohere_main.cpp:181-222)
    if (opt.raw) throw std::runtime_error(cmd + " needs an annotated program");
    Unit u = Reader(src).annotated();
    if (!opt.no_overlap) close_program(u);
    if (cmd == "infer" && !opt.json) {
      o.out += pretty(u);
    } else {
      const Printer one_line(u, false);
      for (size_t i = 0; i < u.blocks.size(); ++i) {
        std::string rec = "{\"block\":" + std::to_string(i) + ",";
        if (cmd == "infer") {
          std::string modes;
          for (const Mode& m : u.blocks[i].modes)
            modes += std::string(modes.empty() ? "" : ",") + "{\"kind\":" + quoted(mode_name(m.kind, LOCAL)) +
                     ",\"shadow\":" + (m.shadow ? "true" : "false") + ",\"site\":" +
                     quoted(m.site == REMOTE ? "remote" : "local") + ",\"view\":" + quoted(u.d.name(m.sym)) + "}";
          o.out += rec + "\"modes\":[" + modes + "]}\n";
        } else {
          const std::string core = one_line.list(u.lists[translate(u, u.blocks[i])]);
          o.out += opt.json ? rec + "\"core\":" + quoted(core) + "}\n" : "block " + std::to_string(i) + ": " + core + "\n";
        }
      }
    }
    o.exit = 0;
    return COH_OK;
  }
  *fatal = "unknown command '" + cmd + "'";
  return COH_E_ARG;
}

void copy_out(const std::string& s, char* buf, size_t cap) {
  if (!buf || !cap) return;
  const size_t n = std::min(s.size(), cap - 1);
  std::memcpy(buf, s.data(), n);
  buf[n] = '\0';
}

// One command on one program text, every exception class mapped to its exit code
// (tools/cohere_main.cpp:262-274).  Returns COH_OK or a COH_E_* with *fatal set.
int one_command(coh_ctx* ctx, const std::string& cmd, std::string_view src, const coh_cli_opts& opt, Outcome& o,
                std::string* fatal) {
  int rc = COH_OK;
  try {
    if (opt.fuel < 1) throw DeclError("--fuel: value must be positive");
    rc = command(ctx, cmd, src, opt, o, fatal);
  } catch (const ConflictError& e) {
    o.err += std::string("error: ") + e.what() + "\n";
    o.exit = 1;
  } catch (const std::exception& e) {  // SyntaxError, DeclError, std::out_of_range, ...
    o.err += std::string("error: ") + e.what() + "\n";
    o.exit = 2;
  }
  return rc;
}

}  // namespace front
}  // namespace cohb

extern "C" int coh_cli(coh_ctx* ctx, const char* cmd, const char* src, const coh_cli_opts* opts, char* out,
                       size_t out_cap, char* err, size_t err_cap, int* exit_code) {
  using namespace cohb::front;
  if (!cmd || !src || !exit_code) return COH_E_ARG;
  const coh_cli_opts opt = opts ? *opts : coh_cli_opts{0, 0, 0, 10000, nullptr, 0};
  Outcome o;
  std::string fatal;
  const int rc = one_command(ctx, cmd, src, opt, o, &fatal);
  if (rc != COH_OK) {
    if (ctx) ctx->err = fatal;
    copy_out(fatal, err, err_cap);
    return rc;
  }
  copy_out(o.out, out, out_cap);
  copy_out(o.err, err, err_cap);
  *exit_code = o.exit;
  return (o.out.size() >= out_cap || o.err.size() >= err_cap) ? -(int)std::max(o.out.size(), o.err.size()) - 1 : COH_OK;
}

// Batched host passes: check / infer / translate over many program
// texts on the host threads -- the reference's checker is a per-program syntactic pass
// (checker.hpp:217-300), so the batch is its data-parallel unit.  Per program the same
// stdout / stderr text and exit code as coh_cli, concatenated into out / err with offsets
// (n + 1 entries each).  Returns COH_OK, COH_E_ARG (run / trace need coh_cli), or
// -(needed bytes of the larger buffer) - 1 when out or err is too small.
extern "C" int coh_cli_batch(const char* cmd, const char* const* srcs, uint32_t n, const coh_cli_opts* opts,
                             int n_threads, char* out, size_t out_cap, uint64_t* out_off, char* err, size_t err_cap,
                             uint64_t* err_off, int* exit_codes) {
  using namespace cohb::front;
  if (!cmd || (n && (!srcs || !out_off || !err_off || !exit_codes))) return COH_E_ARG;
  const std::string command_name = cmd;
  if (command_name != "check" && command_name != "infer" && command_name != "translate") return COH_E_ARG;
  const coh_cli_opts opt = opts ? *opts : coh_cli_opts{0, 0, 0, 10000, nullptr, 0};
  std::vector<Outcome> res(n);
  std::vector<int> rcs(n, COH_OK);
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nth = std::max(1u, std::min<unsigned>(n_threads > 0 ? (unsigned)n_threads : hw, n ? n : 1u));
  std::atomic<uint32_t> next{0};
  auto worker = [&] {
    for (uint32_t i; (i = next.fetch_add(1)) < n;) {
      std::string fatal;
      rcs[i] = one_command(nullptr, command_name, srcs[i] ? srcs[i] : "", opt, res[i], &fatal);
      if (rcs[i] != COH_OK) res[i].err = fatal;
    }
  };
  std::vector<std::thread> pool;
  for (unsigned k = 1; k < nth; ++k) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  size_t need_out = 0, need_err = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (rcs[i] != COH_OK) return rcs[i];
    out_off[i] = need_out;
    err_off[i] = need_err;
    need_out += res[i].out.size();
    need_err += res[i].err.size();
    exit_codes[i] = res[i].exit;
  }
  if (n) out_off[n] = need_out, err_off[n] = need_err;
  if (need_out > out_cap || need_err > err_cap) return -(int)std::min<size_t>(std::max(need_out, need_err), 0x7FFFFFFE) - 1;
  for (uint32_t i = 0; i < n; ++i) {
    if (!res[i].out.empty()) std::memcpy(out + out_off[i], res[i].out.data(), res[i].out.size());
    if (!res[i].err.empty()) std::memcpy(err + err_off[i], res[i].err.data(), res[i].err.size());
  }
  return COH_OK;
}
