// Interchange IO of the placer API, host C++:
//
//   parse_comm_model / load_comm_model / save_comm_model  cost_model.cpp:71-134
//   parse_graph / load_graph / graph_to_json               graph.cpp:196-309
//   placement_to_json / placement_from_json                placers.cpp:367-432
//   a binary CSR sidecar of a meta graph (bx_graph), for sweeps that place
//   the same graphs many times without re-parsing JSON.
//
// The reference reads JSON through nlohmann::json into a DOM and then walks
// it. Here one schema-directed pass reads the text straight into the node /
// edge arrays (no DOM), with the reference's validation order and texts:
// check_keys reports the smallest unknown key (nlohmann objects iterate
// keys in std::map order) and then the first missing key of the sorted
// allowed set, a duplicated key keeps its last value (nlohmann's operator[]),
// integers are "number_integer" only without fraction or exponent, and a
// value beyond uint64 becomes a float. Emission reproduces nlohmann's
// dump(2): two-space indentation, ": " separators, "[]" for empty arrays,
// the same string escapes, and doubles as the shortest round-trip digits in
// nlohmann's fixed/exponent layout.
//
// Malformed JSON (a syntax error) is a ValidationError with a "parse error: "
// prefix as in the reference; the rest of that text (nlohmann's lexer
// message) is not reproduced byte for byte.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/baechi_b200.h"

namespace {

struct JErr {
  std::string msg;
};

[[noreturn]] void fail(const std::string &m) { throw JErr{m}; }

// ---- lexer ------------------------------------------------------------------
enum Kind { K_NULL, K_BOOL, K_INT, K_UINT, K_FLOAT, K_STRING, K_ARRAY, K_OBJECT };

struct Lexer {
  const char *p, *b, *e;
  Lexer(const char *text, size_t len) : p(text), b(text), e(text + len) {}

  [[noreturn]] void syntax(const char *what) {
    int line = 1, col = 1;
    for (const char *q = b; q < p && q < e; ++q) {
      if (*q == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    fail(std::string("parse error: [json.exception.parse_error.101] parse error at line ") + std::to_string(line) +
         ", column " + std::to_string(col) + ": syntax error while parsing value - " + what);
  }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  char peek() {
    ws();
    return p < e ? *p : '\0';
  }
  void expect(char c) {
    ws();
    if (p >= e || *p != c) syntax("unexpected token");
    ++p;
  }
  static void put_utf8(std::string &s, uint32_t cp) {
    if (cp < 0x80) {
      s += static_cast<char>(cp);
    } else if (cp < 0x800) {
      s += static_cast<char>(0xc0 | (cp >> 6));
      s += static_cast<char>(0x80 | (cp & 0x3f));
    } else if (cp < 0x10000) {
      s += static_cast<char>(0xe0 | (cp >> 12));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3f));
      s += static_cast<char>(0x80 | (cp & 0x3f));
    } else {
      s += static_cast<char>(0xf0 | (cp >> 18));
      s += static_cast<char>(0x80 | ((cp >> 12) & 0x3f));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3f));
      s += static_cast<char>(0x80 | (cp & 0x3f));
    }
  }
  uint32_t hex4() {
    if (e - p < 4) syntax("invalid string: '\\u' must be followed by 4 hex digits");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else syntax("invalid string: '\\u' must be followed by 4 hex digits");
    }
    return v;
  }
  // A string with escapes resolved; raw bytes must be valid UTF-8.
  std::string str() {
    expect('"');
    std::string s;
    for (;;) {
      if (p >= e) syntax("invalid string: missing closing quote");
      const unsigned char c = static_cast<unsigned char>(*p);
      if (c == '"') {
        ++p;
        return s;
      }
      if (c < 0x20) syntax("invalid string: control character must be escaped");
      if (c == '\\') {
        ++p;
        if (p >= e) syntax("invalid string: missing closing quote");
        const char x = *p++;
        switch (x) {
          case '"': s += '"'; break;
          case '\\': s += '\\'; break;
          case '/': s += '/'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'n': s += '\n'; break;
          case 'r': s += '\r'; break;
          case 't': s += '\t'; break;
          case 'u': {
            uint32_t cp = hex4();
            if (cp >= 0xd800 && cp <= 0xdbff) {
              if (e - p < 6 || p[0] != '\\' || p[1] != 'u') syntax("invalid string: surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
              p += 2;
              const uint32_t lo = hex4();
              if (lo < 0xdc00 || lo > 0xdfff) syntax("invalid string: surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
              cp = 0x10000 + ((cp - 0xd800) << 10) + (lo - 0xdc00);
            } else if (cp >= 0xdc00 && cp <= 0xdfff) {
              syntax("invalid string: surrogate U+DC00..U+DFFF must follow U+D800..U+DBFF");
            }
            put_utf8(s, cp);
            break;
          }
          default: syntax("invalid string: forbidden character after backslash");
        }
        continue;
      }
      // raw UTF-8 sequence
      int len = c < 0x80 ? 1 : (c >> 5) == 6 ? 2 : (c >> 4) == 14 ? 3 : (c >> 3) == 30 ? 4 : 0;
      if (len == 0 || e - p < len) syntax("invalid string: ill-formed UTF-8 byte");
      uint32_t cp = len == 1 ? c : len == 2 ? (c & 0x1f) : len == 3 ? (c & 0x0f) : (c & 0x07);
      for (int i = 1; i < len; ++i) {
        const unsigned char d = static_cast<unsigned char>(p[i]);
        if ((d & 0xc0) != 0x80) syntax("invalid string: ill-formed UTF-8 byte");
        cp = (cp << 6) | (d & 0x3f);
      }
      const uint32_t lo = len == 2 ? 0x80 : len == 3 ? 0x800 : len == 4 ? 0x10000 : 0;
      if (cp < lo || cp > 0x10ffff || (cp >= 0xd800 && cp <= 0xdfff)) syntax("invalid string: ill-formed UTF-8 byte");
      s.append(p, p + len);
      p += len;
    }
  }
  // A scalar value of any JSON kind; arrays and objects are skipped.
  struct Scalar {
    Kind kind = K_NULL;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0;
    bool bval = false;
    std::string s;
  };
  void literal(const char *word) {
    const size_t n = std::strlen(word);
    if (static_cast<size_t>(e - p) < n || std::strncmp(p, word, n) != 0) syntax("invalid literal");
    p += n;
  }
  Scalar number() {
    Scalar v;
    const char *s0 = p;
    bool neg = false;
    if (*p == '-') {
      neg = true;
      ++p;
    }
    if (p >= e || !(*p >= '0' && *p <= '9')) syntax("invalid number; expected digit after '-'");
    if (*p == '0') {
      ++p;
    } else {
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    bool is_float = false;
    if (p < e && *p == '.') {
      is_float = true;
      ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) syntax("invalid number; expected digit after '.'");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) syntax("invalid number; expected digit after exponent sign");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (!is_float) {
      if (neg) {
        int64_t x = 0;
        auto r = std::from_chars(s0, p, x);
        if (r.ec == std::errc()) {
          v.kind = K_INT;
          v.i = x;
          return v;
        }
      } else {
        uint64_t x = 0;
        auto r = std::from_chars(s0, p, x);
        if (r.ec == std::errc()) {
          v.kind = K_UINT;
          v.u = x;
          return v;
        }
      }
    }
    v.kind = K_FLOAT;  // out-of-range integers fall back to a float, as nlohmann's lexer does
    v.d = std::strtod(std::string(s0, p).c_str(), nullptr);
    return v;
  }
  void skip_value() {
    const char c = peek();
    if (c == '{') {
      ++p;
      if (peek() == '}') {
        ++p;
        return;
      }
      for (;;) {
        str();
        expect(':');
        skip_value();
        const char d = peek();
        if (d == ',') {
          ++p;
          continue;
        }
        if (d == '}') {
          ++p;
          return;
        }
        syntax("unexpected token; expected '}'");
      }
    }
    if (c == '[') {
      ++p;
      if (peek() == ']') {
        ++p;
        return;
      }
      for (;;) {
        skip_value();
        const char d = peek();
        if (d == ',') {
          ++p;
          continue;
        }
        if (d == ']') {
          ++p;
          return;
        }
        syntax("unexpected token; expected ']'");
      }
    }
    (void)scalar();
  }
  Scalar scalar() {
    Scalar v;
    const char c = peek();
    if (c == '"') {
      v.kind = K_STRING;
      v.s = str();
    } else if (c == 't') {
      literal("true");
      v.kind = K_BOOL;
      v.bval = true;
    } else if (c == 'f') {
      literal("false");
      v.kind = K_BOOL;
    } else if (c == 'n') {
      literal("null");
      v.kind = K_NULL;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      v = number();
    } else if (c == '[') {
      skip_value();
      v.kind = K_ARRAY;
    } else if (c == '{') {
      skip_value();
      v.kind = K_OBJECT;
    } else {
      syntax("unexpected token");
    }
    return v;
  }
  void end() {
    ws();
    if (p != e) syntax("unexpected token; expected end of input");
  }
};

bool is_int(const Lexer::Scalar &v) { return v.kind == K_INT || v.kind == K_UINT; }

// nlohmann's basic_json::type_name() of a value kind (type_error texts).
const char *type_name(Kind k) {
  switch (k) {
    case K_NULL: return "null";
    case K_BOOL: return "boolean";
    case K_STRING: return "string";
    case K_ARRAY: return "array";
    case K_OBJECT: return "object";
    default: return "number";
  }
}
int64_t as_i64(const Lexer::Scalar &v) { return v.kind == K_INT ? v.i : static_cast<int64_t>(v.u); }

// An object of scalar fields read in one pass: per allowed key its last
// value; `unknown` the smallest unknown key (std::map order), if any.
struct Fields {
  std::vector<Lexer::Scalar> val;
  std::vector<char> has;
  std::string unknown;
  bool any_unknown = false;
};

// Reads an object whose allowed keys are `keys` (already sorted, as the
// reference's std::set is). `nested(key_index)` returns true when that key's
// value is consumed by a caller-provided reader (arrays of the graph doc).
template <typename Nested>
void read_object(Lexer &L, const std::vector<std::string> &keys, Fields &f, Nested nested) {
  f.val.assign(keys.size(), Lexer::Scalar());
  f.has.assign(keys.size(), 0);
  f.any_unknown = false;
  L.expect('{');
  if (L.peek() == '}') {
    ++L.p;
    return;
  }
  for (;;) {
    std::string k = L.str();
    L.expect(':');
    int idx = -1;
    for (size_t i = 0; i < keys.size(); ++i)
      if (keys[i] == k) idx = static_cast<int>(i);
    if (idx < 0) {
      if (!f.any_unknown || k < f.unknown) f.unknown = k;
      f.any_unknown = true;
      L.skip_value();
    } else {
      f.has[idx] = 1;
      if (!nested(idx)) f.val[idx] = L.scalar();
    }
    const char d = L.peek();
    if (d == ',') {
      ++L.p;
      continue;
    }
    if (d == '}') {
      ++L.p;
      return;
    }
    L.syntax("unexpected token; expected '}'");
  }
}

// check_keys (graph.cpp:19-37) on a read object.
void check_keys(const Fields &f, const std::vector<std::string> &keys, const char *what) {
  if (f.any_unknown) fail(std::string("parse error: unknown key \"") + f.unknown + "\" in " + what);
  for (size_t i = 0; i < keys.size(); ++i)
    if (!f.has[i]) fail(std::string("parse error: missing key \"") + keys[i] + "\" in " + what);
}

int64_t require_count(const Lexer::Scalar &v, const char *what, const char *key) {
  if (!is_int(v)) fail(std::string("parse error: ") + what + "." + key + " must be an integer");
  const int64_t n = as_i64(v);
  if (n < 0) fail(std::string("parse error: ") + what + "." + key + " must be non-negative");
  return n;
}

// ---- emission (nlohmann dump(2)) -------------------------------------------
void esc(std::string &o, const std::string &s) {
  o += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  o += '"';
}

// nlohmann's to_chars layout (format_buffer, min_exp -4, max_exp 15) of the
// shortest round-trip digits.
void dbl(std::string &o, double x) {
  if (!std::isfinite(x)) {
    o += "null";
    return;
  }
  if (x == 0) {
    o += std::signbit(x) ? "-0.0" : "0.0";
    return;
  }
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  std::string s(buf, r.ptr);  // d[.ddd]e±XX
  std::string sign;
  if (s[0] == '-') {
    sign = "-";
    s.erase(0, 1);
  }
  const size_t epos = s.find('e');
  std::string digits = s.substr(0, epos);
  const int exp10 = std::stoi(s.substr(epos + 1));
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // position of the decimal point after the first n digits
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int ex = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  o += sign + out;
}

int emit(const std::string &s, char *buf, int64_t buflen, int64_t *needed) {
  if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
  if (!buf || buflen < static_cast<int64_t>(s.size()) + 1) return BX_VALIDATION;
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  return BX_OK;
}

void put(char *msg, int len, const std::string &s) {
  if (msg && len > 0) std::snprintf(msg, static_cast<size_t>(len), "%s", s.c_str());
}

bool read_file(const char *path, std::string &out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  std::ostringstream b;
  b << in.rdbuf();
  out = b.str();
  return true;
}

}  // namespace

// A parsed graph file (parse_graph before make_graph): node and edge arrays
// in file order, names and colocation group strings kept for emission.
struct bx_json_graph {
  std::vector<int64_t> id, k, temp, perm, out, peer;
  std::vector<int32_t> label;
  std::vector<uint8_t> has_pair;
  std::vector<std::string> name, groups;  // groups[label] (sorted distinct strings)
  std::vector<const char *> name_c, group_c;
  std::vector<int64_t> src, dst, bytes;
};

extern "C" {

int bx_comm_model_parse(const char *text, int64_t len, bx_comm *out, char *msg, int msglen) {
  put(msg, msglen, "");
  static const std::vector<std::string> keys = {"intercept_us", "mode", "us_per_byte"};
  try {
    Lexer L(text, static_cast<size_t>(len));
    if (L.peek() != '{') {
      Lexer::Scalar v = L.scalar();
      (void)v;
      L.end();
      fail("parse error: comm model must be a JSON object");
    }
    Fields f;
    read_object(L, keys, f, [](int) { return false; });
    L.end();
    if (f.any_unknown) fail("parse error: unknown key \"" + f.unknown + "\" in comm model");
    // missing keys in the reference's listing order (cost_model.cpp:87-92)
    for (int i : {0, 2, 1})
      if (!f.has[i]) fail("parse error: missing key \"" + keys[i] + "\" in comm model");
    auto num = [](const Lexer::Scalar &v) {
      return v.kind == K_INT || v.kind == K_UINT || v.kind == K_FLOAT;
    };
    auto dv = [](const Lexer::Scalar &v) {
      return v.kind == K_INT ? static_cast<double>(v.i) : v.kind == K_UINT ? static_cast<double>(v.u) : v.d;
    };
    if (!num(f.val[0]) || !num(f.val[2])) fail("parse error: comm model fields must be numbers");
    const double ic = dv(f.val[0]), pb = dv(f.val[2]);
    if (ic < 0 || pb < 0) fail("comm model coefficients must be non-negative");
    if (f.val[1].kind != K_STRING)  // nlohmann get<std::string> on a non-string
      fail(std::string("[json.exception.type_error.302] type must be string, but is ") + type_name(f.val[1].kind));
    int mode;
    if (f.val[1].s == "sequential") mode = BX_COMM_SEQUENTIAL;
    else if (f.val[1].s == "parallel") mode = BX_COMM_PARALLEL;
    else fail("comm model mode must be sequential or parallel");
    out->intercept_us = ic;
    out->us_per_byte = pb;
    out->mode = mode;
    return BX_OK;
  } catch (const JErr &e) {
    put(msg, msglen, e.msg);
    return BX_VALIDATION;
  }
}

int bx_comm_model_load(const char *path, bx_comm *out, char *msg, int msglen) {
  std::string text;
  if (!read_file(path, text)) {
    put(msg, msglen, std::string("cannot open comm model file: ") + path);
    return BX_VALIDATION;
  }
  return bx_comm_model_parse(text.data(), static_cast<int64_t>(text.size()), out, msg, msglen);
}

int bx_comm_model_to_json(const bx_comm *cm, char *buf, int64_t buflen, int64_t *needed) {
  std::string o = "{\n  \"intercept_us\": ";
  dbl(o, cm->intercept_us);
  o += ",\n  \"us_per_byte\": ";
  dbl(o, cm->us_per_byte);
  o += ",\n  \"mode\": ";
  esc(o, cm->mode == BX_COMM_SEQUENTIAL ? "sequential" : "parallel");
  o += "\n}\n";
  return emit(o, buf, buflen, needed);
}

int bx_graph_parse(const char *text, int64_t len, bx_json_graph **out, char *msg, int msglen) {
  *out = nullptr;
  put(msg, msglen, "");
  static const std::vector<std::string> top = {"edges", "nodes"};
  static const std::vector<std::string> nkeys = {"colocation_group", "compute_time_us", "coplace_pair", "id",
                                                 "name",             "out_mem_bytes",   "perm_mem_bytes",
                                                 "temp_mem_bytes"};
  static const std::vector<std::string> ekeys = {"dst", "src", "tensor_bytes"};
  enum { N_GROUP, N_K, N_PAIR, N_ID, N_NAME, N_OUT, N_PERM, N_TEMP };
  enum { E_DST, E_SRC, E_BYTES };
  try {
    Lexer L(text, static_cast<size_t>(len));
    // nodes / edges raw records (validated after the whole document parsed,
    // in the reference's order: doc keys, array kinds, nodes, then edges)
    std::vector<Fields> nodes, edges;
    bool nodes_arr = false, edges_arr = false;
    auto read_array = [&](std::vector<Fields> &rows, const std::vector<std::string> &keys, bool &is_arr) {
      rows.clear();
      if (L.peek() != '[') {
        (void)L.scalar();
        is_arr = false;
        return;
      }
      is_arr = true;
      ++L.p;
      if (L.peek() == ']') {
        ++L.p;
        return;
      }
      for (;;) {
        rows.emplace_back();
        if (L.peek() == '{') {
          read_object(L, keys, rows.back(), [](int) { return false; });
        } else {
          (void)L.scalar();
          rows.back().val.clear();  // marks "not an object"
          rows.back().has.clear();
        }
        const char d = L.peek();
        if (d == ',') {
          ++L.p;
          continue;
        }
        if (d == ']') {
          ++L.p;
          return;
        }
        L.syntax("unexpected token; expected ']'");
      }
    };
    Fields doc;
    bool doc_obj = L.peek() == '{';
    if (doc_obj) {
      read_object(L, top, doc, [&](int idx) {
        if (idx == 0) read_array(edges, ekeys, edges_arr);
        else read_array(nodes, nkeys, nodes_arr);
        return true;
      });
    } else {
      (void)L.scalar();
    }
    L.end();
    if (!doc_obj) fail("parse error: graph is not a JSON object");
    check_keys(doc, top, "graph");
    if (!nodes_arr || !edges_arr) fail("parse error: nodes and edges must be arrays");
    auto G = std::make_unique<bx_json_graph>();
    std::map<std::string, int> group_ix;
    std::vector<std::string> node_group;
    std::vector<char> node_has_group;
    for (const Fields &f : nodes) {
      if (f.val.empty()) fail("parse error: node is not a JSON object");
      check_keys(f, nkeys, "node");
      if (!is_int(f.val[N_ID])) fail("parse error: node.id must be an integer");
      G->id.push_back(as_i64(f.val[N_ID]));
      if (f.val[N_NAME].kind != K_STRING) fail("parse error: node.name must be a string");
      G->name.push_back(f.val[N_NAME].s);
      G->k.push_back(require_count(f.val[N_K], "node", "compute_time_us"));
      G->temp.push_back(require_count(f.val[N_TEMP], "node", "temp_mem_bytes"));
      G->perm.push_back(require_count(f.val[N_PERM], "node", "perm_mem_bytes"));
      G->out.push_back(require_count(f.val[N_OUT], "node", "out_mem_bytes"));
      if (f.val[N_GROUP].kind == K_STRING) {
        node_group.push_back(f.val[N_GROUP].s);
        node_has_group.push_back(1);
        group_ix.emplace(f.val[N_GROUP].s, 0);
      } else if (f.val[N_GROUP].kind == K_NULL) {
        node_group.emplace_back();
        node_has_group.push_back(0);
      } else {
        fail("parse error: node.colocation_group must be a string or null");
      }
      if (is_int(f.val[N_PAIR])) {
        G->has_pair.push_back(1);
        G->peer.push_back(as_i64(f.val[N_PAIR]));
      } else if (f.val[N_PAIR].kind == K_NULL) {
        G->has_pair.push_back(0);
        G->peer.push_back(0);
      } else {
        fail("parse error: node.coplace_pair must be an integer or null");
      }
    }
    for (const Fields &f : edges) {
      if (f.val.empty()) fail("parse error: edge is not a JSON object");
      check_keys(f, ekeys, "edge");
      if (!is_int(f.val[E_SRC]) || !is_int(f.val[E_DST])) fail("parse error: edge endpoints must be integers");
      G->src.push_back(as_i64(f.val[E_SRC]));
      G->dst.push_back(as_i64(f.val[E_DST]));
      G->bytes.push_back(require_count(f.val[E_BYTES], "edge", "tensor_bytes"));
    }
    int gi = 0;
    for (auto &kv : group_ix) {
      kv.second = gi++;
      G->groups.push_back(kv.first);
    }
    for (size_t i = 0; i < G->id.size(); ++i) G->label.push_back(node_has_group[i] ? group_ix[node_group[i]] : -1);
    for (auto &s : G->name) G->name_c.push_back(s.c_str());
    for (auto &s : G->groups) G->group_c.push_back(s.c_str());
    // make_graph's own validation runs where the graph is used
    // (bx_grouped_create), as parse_graph ends in make_graph (graph.cpp:260)
    *out = G.release();
    return BX_OK;
  } catch (const JErr &e) {
    put(msg, msglen, e.msg);
    return BX_VALIDATION;
  }
}

int bx_graph_load(const char *path, bx_json_graph **out, char *msg, int msglen) {
  std::string text;
  if (!read_file(path, text)) {
    *out = nullptr;
    put(msg, msglen, std::string("cannot open graph file: ") + path);
    return BX_VALIDATION;
  }
  return bx_graph_parse(text.data(), static_cast<int64_t>(text.size()), out, msg, msglen);
}

int bx_json_graph_view(const bx_json_graph *g, bx_base_graph *base, const char *const **names,
                       const char *const **groups, int32_t *ngroups) {
  base->nodes = static_cast<int32_t>(g->id.size());
  base->id = g->id.data();
  base->compute_us = g->k.data();
  base->temp_bytes = g->temp.data();
  base->perm_bytes = g->perm.data();
  base->out_bytes = g->out.data();
  base->coloc_label = g->label.data();
  base->has_pair = g->has_pair.data();
  base->coplace_peer = g->peer.data();
  base->edges = static_cast<int32_t>(g->src.size());
  base->src = g->src.data();
  base->dst = g->dst.data();
  base->tensor_bytes = g->bytes.data();
  if (names) *names = g->name_c.data();
  if (groups) *groups = g->group_c.data();
  if (ngroups) *ngroups = static_cast<int32_t>(g->groups.size());
  return BX_OK;
}

void bx_json_graph_destroy(bx_json_graph *g) { delete g; }

int bx_graph_to_json(const bx_base_graph *g, const char *const *names, const char *const *groups, char *buf,
                     int64_t buflen, int64_t *needed) {
  // graph_to_json (graph.cpp:283-309) emits a ProfiledGraph, i.e. after
  // make_graph: nodes by ascending id, edges by ascending (src, dst)
  std::vector<int> no(static_cast<size_t>(g->nodes)), eo(static_cast<size_t>(g->edges));
  std::iota(no.begin(), no.end(), 0);
  std::iota(eo.begin(), eo.end(), 0);
  std::stable_sort(no.begin(), no.end(), [&](int a, int b) { return g->id[a] < g->id[b]; });
  std::stable_sort(eo.begin(), eo.end(), [&](int a, int b) {
    return g->src[a] != g->src[b] ? g->src[a] < g->src[b] : g->dst[a] < g->dst[b];
  });
  std::string o;
  o.reserve(static_cast<size_t>(g->nodes) * 260 + static_cast<size_t>(g->edges) * 80 + 64);
  auto num = [&](int64_t v) { o += std::to_string(v); };
  o += "{\n  \"nodes\": ";
  if (g->nodes == 0) {
    o += "[]";
  } else {
    o += "[\n";
    for (size_t r = 0; r < no.size(); ++r) {
      const int i = no[r];
      o += "    {\n      \"id\": ";
      num(g->id[i]);
      o += ",\n      \"name\": ";
      esc(o, names && names[i] ? names[i] : "");
      o += ",\n      \"compute_time_us\": ";
      num(g->compute_us[i]);
      o += ",\n      \"temp_mem_bytes\": ";
      num(g->temp_bytes[i]);
      o += ",\n      \"perm_mem_bytes\": ";
      num(g->perm_bytes[i]);
      o += ",\n      \"out_mem_bytes\": ";
      num(g->out_bytes[i]);
      o += ",\n      \"colocation_group\": ";
      const int32_t lab = g->coloc_label ? g->coloc_label[i] : -1;
      if (lab >= 0) {
        esc(o, groups ? std::string(groups[lab]) : "g" + std::to_string(lab));
      } else {
        o += "null";
      }
      o += ",\n      \"coplace_pair\": ";
      if (g->has_pair && g->has_pair[i]) num(g->coplace_peer[i]);
      else o += "null";
      o += r + 1 < no.size() ? "\n    },\n" : "\n    }\n";
    }
    o += "  ]";
  }
  o += ",\n  \"edges\": ";
  if (g->edges == 0) {
    o += "[]";
  } else {
    o += "[\n";
    for (size_t r = 0; r < eo.size(); ++r) {
      const int e = eo[r];
      o += "    {\n      \"src\": ";
      num(g->src[e]);
      o += ",\n      \"dst\": ";
      num(g->dst[e]);
      o += ",\n      \"tensor_bytes\": ";
      num(g->tensor_bytes[e]);
      o += r + 1 < eo.size() ? "\n    },\n" : "\n    }\n";
    }
    o += "  ]";
  }
  o += "\n}\n";
  return emit(o, buf, buflen, needed);
}

int bx_placement_to_json(const bx_grouping *gp, const char *algorithm, int32_t n, const int32_t *exec_order,
                         const int32_t *exec_off, const int64_t *sim_start_us, int64_t makespan_us,
                         const int64_t *peak_bytes, char *buf, int64_t buflen, int64_t *needed) {
  std::string o;
  o.reserve(static_cast<size_t>(gp->base_nodes) * 80 + 256);
  o += "{\n  \"algorithm\": ";
  esc(o, algorithm ? algorithm : "");
  o += ",\n  \"assignments\": ";
  const int32_t total = n > 0 ? exec_off[n] : 0;
  if (total == 0) {
    o += "[]";
  } else {
    o += "[\n";
    bool first = true;
    for (int d = 0; d < n; ++d) {
      for (int x = exec_off[d]; x < exec_off[d + 1]; ++x) {
        const int meta = exec_order[x];
        for (int y = gp->member_off[meta]; y < gp->member_off[meta + 1]; ++y) {
          if (!first) o += ",\n";
          first = false;
          o += "    {\n      \"node\": ";
          o += std::to_string(gp->base_ids[gp->members[y]]);
          o += ",\n      \"device\": ";
          o += std::to_string(d);
          o += ",\n      \"start_us\": ";
          o += std::to_string(sim_start_us[meta]);
          o += "\n    }";
        }
      }
    }
    o += "\n  ]";
  }
  o += ",\n  \"makespan_us\": ";
  o += std::to_string(makespan_us);
  o += ",\n  \"per_device_peak_bytes\": ";
  if (n <= 0) {
    o += "[]";
  } else {
    o += "[\n";
    for (int d = 0; d < n; ++d) {
      o += "    " + std::to_string(peak_bytes[d]);
      o += d + 1 < n ? ",\n" : "\n";
    }
    o += "  ]";
  }
  o += "\n}\n";
  return emit(o, buf, buflen, needed);
}

int bx_placement_from_json(const bx_grouping *gp, int32_t V, const char *text, int64_t len, int32_t n,
                           char *algorithm, int algolen, int32_t *device_of, int64_t *start_us, int32_t *exec_order,
                           int32_t *exec_off, char *msg, int msglen) {
  put(msg, msglen, "");
  static const std::vector<std::string> top = {"algorithm", "assignments"};
  static const std::vector<std::string> rkeys = {"device", "node", "start_us"};
  try {
    Lexer L(text, static_cast<size_t>(len));
    struct Row {
      Fields f;
      Kind kind;
    };
    std::vector<Row> rows;
    char rows_kind = 'n';
    Fields doc;
    const bool doc_obj = L.peek() == '{';
    if (doc_obj) {
      // keep every key (unknown ones are allowed here); only the two used are read
      doc.val.assign(2, Lexer::Scalar());
      doc.has.assign(2, 0);
      L.expect('{');
      if (L.peek() != '}') {
        for (;;) {
          std::string k = L.str();
          L.expect(':');
          if (k == "assignments") {
            // nlohmann iterates an array's elements, an object's values, a
            // primitive as itself and null as nothing
            doc.has[1] = 1;
            rows.clear();
            rows_kind = L.peek();
            auto one_row = [&]() {
              rows.emplace_back();
              rows.back().kind = K_OBJECT;
              if (L.peek() == '{') {
                read_object(L, rkeys, rows.back().f, [](int) { return false; });
              } else {
                rows.back().kind = L.scalar().kind;
              }
            };
            if (rows_kind == '[' || rows_kind == '{') {
              const bool arr = rows_kind == '[';
              ++L.p;
              if (L.peek() == (arr ? ']' : '}')) {
                ++L.p;
              } else {
                for (;;) {
                  if (!arr) {
                    L.str();
                    L.expect(':');
                  }
                  one_row();
                  const char d = L.peek();
                  if (d == ',') {
                    ++L.p;
                    continue;
                  }
                  if (d == (arr ? ']' : '}')) {
                    ++L.p;
                    break;
                  }
                  L.syntax(arr ? "unexpected token; expected ']'" : "unexpected token; expected '}'");
                }
              }
            } else if (rows_kind == 'n') {
              L.skip_value();
            } else {
              one_row();
            }
          } else if (k == "algorithm") {
            doc.has[0] = 1;
            doc.val[0] = L.scalar();
          } else {
            L.skip_value();
          }
          const char d = L.peek();
          if (d == ',') {
            ++L.p;
            continue;
          }
          if (d == '}') {
            ++L.p;
            break;
          }
          L.syntax("unexpected token; expected '}'");
        }
      } else {
        ++L.p;
      }
    } else {
      L.skip_value();
    }
    L.end();
    if (!doc_obj || !doc.has[0] || !doc.has[1]) fail("placement file must carry algorithm/assignments");
    if (doc.val[0].kind != K_STRING)
      fail(std::string("[json.exception.type_error.302] type must be string, but is ") + type_name(doc.val[0].kind));
    put(algorithm, algolen, doc.val[0].s);
    for (int j = 0; j < V; ++j) {
      device_of[j] = -1;
      start_us[j] = 0;
    }
    std::vector<std::vector<int>> lists(static_cast<size_t>(std::max(n, 0)));
    auto get = [&](const Row &r, int idx, const char *key) -> int64_t {
      if (r.kind != K_OBJECT)
        fail(std::string("[json.exception.type_error.304] cannot use at() with ") + type_name(r.kind));
      if (!r.f.has[idx]) fail(std::string("[json.exception.out_of_range.403] key '") + key + "' not found");
      const Lexer::Scalar &v = r.f.val[idx];
      if (v.kind == K_FLOAT) return static_cast<int64_t>(v.d);
      if (v.kind == K_BOOL) return v.bval ? 1 : 0;
      if (!is_int(v)) fail(std::string("[json.exception.type_error.302] type must be number, but is ") + type_name(v.kind));
      return as_i64(v);
    };
    for (const Row &r : rows) {
      const int64_t id = get(r, 1, "node");
      const int dev = static_cast<int>(get(r, 0, "device"));
      const int64_t start = get(r, 2, "start_us");
      if (dev < 0 || dev >= n) fail("assignment device " + std::to_string(dev) + " outside the roster");
      auto it = std::lower_bound(gp->base_ids, gp->base_ids + gp->base_nodes, id);
      if (it == gp->base_ids + gp->base_nodes || *it != id)
        fail("dangling reference: unknown node id " + std::to_string(id));
      const int meta = gp->group_of[it - gp->base_ids];
      if (device_of[meta] >= 0 && device_of[meta] != dev)
        fail("grouped nodes assigned to different devices around base node " + std::to_string(id));
      if (device_of[meta] < 0) {
        device_of[meta] = dev;
        start_us[meta] = start;
        lists[dev].push_back(meta);  // file order is execution order
      }
    }
    for (int j = 0; j < V; ++j)
      if (device_of[j] < 0) fail("placement misses meta node " + std::to_string(j));
    int x = 0;
    for (int d = 0; d < n; ++d) {
      exec_off[d] = x;
      for (int m : lists[d]) exec_order[x++] = m;
    }
    if (n >= 0) exec_off[n] = x;
    return BX_OK;
  } catch (const JErr &e) {
    put(msg, msglen, e.msg);
    return BX_VALIDATION;
  }
}

// trace_to_csv (simulator.cpp:311-324)
int bx_trace_to_csv(const bx_trace_event *trace, int64_t count, char *buf, int64_t buflen, int64_t *needed) {
  static const char *kNames[4] = {"start", "finish", "xfer_begin", "xfer_end"};
  std::vector<int64_t> order(static_cast<size_t>(std::max<int64_t>(count, 0)));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return trace[a].time_us < trace[b].time_us; });
  std::string o = "time_us,device,event,node\n";
  o.reserve(o.size() + order.size() * 32);
  for (int64_t i : order) {
    const bx_trace_event &ev = trace[i];
    o += std::to_string(ev.time_us);
    o += ',';
    o += std::to_string(ev.device);
    o += ',';
    o += ev.event >= 0 && ev.event < 4 ? kNames[ev.event] : "?";
    o += ',';
    o += std::to_string(ev.node);
    o += '\n';
  }
  return emit(o, buf, buflen, needed);
}

// ---- binary CSR sidecar ----------------------------------------------------
// Layout (native little-endian): "BXG1", int32 V, int32 E, int32 has_first_id,
// int32 0, then k, temp, perm, out [V] int64, esrc, edst [E] int32,
// tensor_bytes [E] int64, in_off [V+1], in_edge [E], out_off [V+1] int32,
// first_id [V] int64 when present.
int bx_graph_save_bin(const bx_graph *g, const char *path, char *msg, int msglen) {
  std::ofstream f(path, std::ios::binary);
  if (!f) {
    put(msg, msglen, std::string("cannot write graph file: ") + path);
    return BX_VALIDATION;
  }
  const int32_t hdr[4] = {g->V, g->E, g->first_id ? 1 : 0, 0};
  f.write("BXG1", 4);
  f.write(reinterpret_cast<const char *>(hdr), sizeof hdr);
  auto w = [&](const void *p, size_t bytes) {
    if (bytes) f.write(static_cast<const char *>(p), static_cast<std::streamsize>(bytes));
  };
  const size_t V = static_cast<size_t>(g->V), E = static_cast<size_t>(g->E);
  w(g->compute_us, 8 * V);
  w(g->temp_bytes, 8 * V);
  w(g->perm_bytes, 8 * V);
  w(g->out_bytes, 8 * V);
  w(g->esrc, 4 * E);
  w(g->edst, 4 * E);
  w(g->tensor_bytes, 8 * E);
  w(g->in_off, 4 * (V + 1));
  w(g->in_edge, 4 * E);
  w(g->out_off, 4 * (V + 1));
  if (g->first_id) w(g->first_id, 8 * V);
  if (!f) {
    put(msg, msglen, std::string("cannot write graph file: ") + path);
    return BX_VALIDATION;
  }
  put(msg, msglen, "");
  return BX_OK;
}

}  // extern "C"

struct bx_bin_graph {
  std::vector<int64_t> k, temp, perm, out, ebytes, first_id;
  std::vector<int32_t> esrc, edst, in_off, in_edge, out_off;
  bx_graph view{};
};

extern "C" {

int bx_graph_load_bin(const char *path, bx_bin_graph **out, bx_graph *view, char *msg, int msglen) {
  *out = nullptr;
  std::ifstream f(path, std::ios::binary);
  char magic[4];
  int32_t hdr[4];
  if (!f || !f.read(magic, 4) || std::memcmp(magic, "BXG1", 4) != 0 ||
      !f.read(reinterpret_cast<char *>(hdr), sizeof hdr) || hdr[0] < 0 || hdr[1] < 0) {
    put(msg, msglen, std::string("not a graph sidecar file: ") + path);
    return BX_VALIDATION;
  }
  auto G = std::make_unique<bx_bin_graph>();
  const size_t V = static_cast<size_t>(hdr[0]), E = static_cast<size_t>(hdr[1]);
  auto rd = [&](auto &vec, size_t count) {
    vec.resize(count);
    if (count) f.read(reinterpret_cast<char *>(vec.data()), static_cast<std::streamsize>(count * sizeof(vec[0])));
  };
  rd(G->k, V);
  rd(G->temp, V);
  rd(G->perm, V);
  rd(G->out, V);
  rd(G->esrc, E);
  rd(G->edst, E);
  rd(G->ebytes, E);
  rd(G->in_off, V + 1);
  rd(G->in_edge, E);
  rd(G->out_off, V + 1);
  if (hdr[2]) rd(G->first_id, V);
  if (!f) {
    put(msg, msglen, std::string("truncated graph sidecar file: ") + path);
    return BX_VALIDATION;
  }
  bx_graph &v = G->view;
  v.V = hdr[0];
  v.E = hdr[1];
  v.compute_us = G->k.data();
  v.temp_bytes = G->temp.data();
  v.perm_bytes = G->perm.data();
  v.out_bytes = G->out.data();
  v.esrc = G->esrc.data();
  v.edst = G->edst.data();
  v.tensor_bytes = G->ebytes.data();
  v.in_off = G->in_off.data();
  v.in_edge = G->in_edge.data();
  v.out_off = G->out_off.data();
  v.first_id = hdr[2] ? G->first_id.data() : nullptr;
  // the adjacency must be the one bx_build_adjacency derives from the edges
  std::vector<int32_t> io(V + 1), ie(std::max<size_t>(E, 1)), oo(V + 1);
  char m2[256];
  if (bx_build_adjacency(v.V, v.E, v.esrc, v.edst, io.data(), ie.data(), oo.data(), m2, sizeof m2) != BX_OK) {
    put(msg, msglen, m2);
    return BX_VALIDATION;
  }
  if (!std::equal(io.begin(), io.end(), G->in_off.begin()) || !std::equal(oo.begin(), oo.end(), G->out_off.begin()) ||
      !std::equal(G->in_edge.begin(), G->in_edge.end(), ie.begin())) {
    put(msg, msglen, std::string("graph sidecar adjacency disagrees with its edges: ") + path);
    return BX_VALIDATION;
  }
  if (view) *view = v;
  *out = G.release();
  put(msg, msglen, "");
  return BX_OK;
}

void bx_bin_graph_destroy(bx_bin_graph *g) { delete g; }

}  // extern "C"
