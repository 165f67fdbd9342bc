// Wire formats (see ce_io.hpp): tensor JSON / binary (tensor.cpp:132-186) and layer
// descriptor JSON (layers.cpp:425-467), with a small recursive-descent JSON reader.
#include "ce_io.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <system_error>

namespace ce {

// ------------------------------------------------------------------ numbers
// The reference serialises with nlohmann::json, whose dump() prints a double with Grisu2
// (Loitsch, "Printing Floating-Point Numbers Quickly and Accurately with Integers", PLDI
// 2010): a 64-bit "do-it-yourself" float w = f * 2^e is scaled by a cached power of ten so
// its exponent lands in [alpha, gamma] = [-60, -32], and digits are generated until the
// remainder falls inside the rounding interval [M-, M+] of the input's neighbours.  The
// result round-trips but is not always the shortest (or the nearest shortest) string, so
// byte-identical output needs this exact procedure rather than std::to_chars.
namespace {

struct Dfp {  // f * 2^e
  uint64_t f;
  int e;
};

Dfp dfp_mul(Dfp x, Dfp y) {  // upper 64 bits of the 128-bit product, rounded half up
  const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f;
  const uint64_t hi = static_cast<uint64_t>(p >> 64), lo = static_cast<uint64_t>(p);
  return {hi + (lo >> 63), x.e + y.e + 64};
}

Dfp dfp_normalize(Dfp x) {
  const int s = __builtin_clzll(x.f);
  return {x.f << s, x.e - s};
}

// 10^k ~= f * 2^e for k = -300, -292, ..., 324: the significand rounded to nearest
// (generated with exact rational arithmetic).
struct Pow10 {
  uint64_t f;
  int e, k;
};
constexpr Pow10 kPow10[79] = {
    {0xAB70FE17C79AC6CAULL, -1060, -300},
    {0xFF77B1FCBEBCDC4FULL, -1034, -292},
    {0xBE5691EF416BD60CULL, -1007, -284},
    {0x8DD01FAD907FFC3CULL, -980, -276},
    {0xD3515C2831559A83ULL, -954, -268},
    {0x9D71AC8FADA6C9B5ULL, -927, -260},
    {0xEA9C227723EE8BCBULL, -901, -252},
    {0xAECC49914078536DULL, -874, -244},
    {0x823C12795DB6CE57ULL, -847, -236},
    {0xC21094364DFB5637ULL, -821, -228},
    {0x9096EA6F3848984FULL, -794, -220},
    {0xD77485CB25823AC7ULL, -768, -212},
    {0xA086CFCD97BF97F4ULL, -741, -204},
    {0xEF340A98172AACE5ULL, -715, -196},
    {0xB23867FB2A35B28EULL, -688, -188},
    {0x84C8D4DFD2C63F3BULL, -661, -180},
    {0xC5DD44271AD3CDBAULL, -635, -172},
    {0x936B9FCEBB25C996ULL, -608, -164},
    {0xDBAC6C247D62A584ULL, -582, -156},
    {0xA3AB66580D5FDAF6ULL, -555, -148},
    {0xF3E2F893DEC3F126ULL, -529, -140},
    {0xB5B5ADA8AAFF80B8ULL, -502, -132},
    {0x87625F056C7C4A8BULL, -475, -124},
    {0xC9BCFF6034C13053ULL, -449, -116},
    {0x964E858C91BA2655ULL, -422, -108},
    {0xDFF9772470297EBDULL, -396, -100},
    {0xA6DFBD9FB8E5B88FULL, -369, -92},
    {0xF8A95FCF88747D94ULL, -343, -84},
    {0xB94470938FA89BCFULL, -316, -76},
    {0x8A08F0F8BF0F156BULL, -289, -68},
    {0xCDB02555653131B6ULL, -263, -60},
    {0x993FE2C6D07B7FACULL, -236, -52},
    {0xE45C10C42A2B3B06ULL, -210, -44},
    {0xAA242499697392D3ULL, -183, -36},
    {0xFD87B5F28300CA0EULL, -157, -28},
    {0xBCE5086492111AEBULL, -130, -20},
    {0x8CBCCC096F5088CCULL, -103, -12},
    {0xD1B71758E219652CULL, -77, -4},
    {0x9C40000000000000ULL, -50, 4},
    {0xE8D4A51000000000ULL, -24, 12},
    {0xAD78EBC5AC620000ULL, 3, 20},
    {0x813F3978F8940984ULL, 30, 28},
    {0xC097CE7BC90715B3ULL, 56, 36},
    {0x8F7E32CE7BEA5C70ULL, 83, 44},
    {0xD5D238A4ABE98068ULL, 109, 52},
    {0x9F4F2726179A2245ULL, 136, 60},
    {0xED63A231D4C4FB27ULL, 162, 68},
    {0xB0DE65388CC8ADA8ULL, 189, 76},
    {0x83C7088E1AAB65DBULL, 216, 84},
    {0xC45D1DF942711D9AULL, 242, 92},
    {0x924D692CA61BE758ULL, 269, 100},
    {0xDA01EE641A708DEAULL, 295, 108},
    {0xA26DA3999AEF774AULL, 322, 116},
    {0xF209787BB47D6B85ULL, 348, 124},
    {0xB454E4A179DD1877ULL, 375, 132},
    {0x865B86925B9BC5C2ULL, 402, 140},
    {0xC83553C5C8965D3DULL, 428, 148},
    {0x952AB45CFA97A0B3ULL, 455, 156},
    {0xDE469FBD99A05FE3ULL, 481, 164},
    {0xA59BC234DB398C25ULL, 508, 172},
    {0xF6C69A72A3989F5CULL, 534, 180},
    {0xB7DCBF5354E9BECEULL, 561, 188},
    {0x88FCF317F22241E2ULL, 588, 196},
    {0xCC20CE9BD35C78A5ULL, 614, 204},
    {0x98165AF37B2153DFULL, 641, 212},
    {0xE2A0B5DC971F303AULL, 667, 220},
    {0xA8D9D1535CE3B396ULL, 694, 228},
    {0xFB9B7CD9A4A7443CULL, 720, 236},
    {0xBB764C4CA7A44410ULL, 747, 244},
    {0x8BAB8EEFB6409C1AULL, 774, 252},
    {0xD01FEF10A657842CULL, 800, 260},
    {0x9B10A4E5E9913129ULL, 827, 268},
    {0xE7109BFBA19C0C9DULL, 853, 276},
    {0xAC2820D9623BF429ULL, 880, 284},
    {0x80444B5E7AA7CF85ULL, 907, 292},
    {0xBF21E44003ACDD2DULL, 933, 300},
    {0x8E679C2F5E44FF8FULL, 960, 308},
    {0xD433179D9C8CB841ULL, 986, 316},
    {0x9E19DB92B4E31BA9ULL, 1013, 324}
};

void round_last(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  // move the last digit towards w while it stays inside the interval and gets closer
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}

// digits of v > 0 (finite) into buf, value = buf * 10^dec_exp
void grisu2(double v, char* buf, int& len, int& dec_exp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t E = bits >> 52, F = bits & ((1ull << 52) - 1);
  const Dfp w = E == 0 ? Dfp{F, 1 - 1075} : Dfp{F | (1ull << 52), static_cast<int>(E) - 1075};
  // neighbours' midpoints m- / m+ (the lower gap is half as wide at a power of two)
  const Dfp mp = dfp_normalize({2 * w.f + 1, w.e - 1});
  Dfp mm = (F == 0 && E > 1) ? Dfp{4 * w.f - 1, w.e - 2} : Dfp{2 * w.f - 1, w.e - 1};
  mm = {mm.f << (mm.e - mp.e), mp.e};
  const Dfp wn = dfp_normalize(w);
  // cached power c = 10^-k with alpha <= e_c + e + 64 <= gamma
  const int f = -60 - mp.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
  const Pow10& c = kPow10[(300 + k + 7) / 8];
  const Dfp cw = dfp_mul(wn, {c.f, c.e}), cm = dfp_mul(mm, {c.f, c.e}), cp = dfp_mul(mp, {c.f, c.e});
  const Dfp Mm{cm.f + 1, cm.e}, Mp{cp.f - 1, cp.e};
  dec_exp = -c.k;
  uint64_t delta = Mp.f - Mm.f, dist = Mp.f - cw.f;
  const int sh = -Mp.e;
  const uint64_t one = 1ull << sh;
  uint32_t p1 = static_cast<uint32_t>(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  uint32_t pow10 = 1;
  int n = 1;
  while (n < 10 && p1 >= pow10 * 10u) {
    pow10 *= 10;
    ++n;
  }
  len = 0;
  // integral part
  while (n > 0) {
    buf[len++] = static_cast<char>('0' + p1 / pow10);
    p1 %= pow10;
    --n;
    const uint64_t rest = (static_cast<uint64_t>(p1) << sh) + p2;
    if (rest <= delta) {
      dec_exp += n;
      round_last(buf, len, dist, delta, rest, static_cast<uint64_t>(pow10) << sh);
      return;
    }
    pow10 /= 10;
  }
  // fractional part
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[len++] = static_cast<char>('0' + (p2 >> sh));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dec_exp -= m;
  round_last(buf, len, dist, delta, p2, one);
}

}  // namespace

std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";  // nlohmann dumps NaN / inf as null
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  std::string out;
  if (v < 0) {
    out = "-";
    v = -v;
  }
  char dg[32];
  int k = 0, dec = 0;
  grisu2(v, dg, k, dec);
  const std::string digits(dg, static_cast<std::size_t>(k));
  const int n = k + dec;  // position of the decimal point relative to the digits
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out += digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= kMaxExp) {
    out += digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
  } else if (kMinExp < n && n <= 0) {
    out += "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return out;
}

// ------------------------------------------------------------------ JSON reader
namespace {

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0;
  bool is_int = false;
  int64_t inum = 0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct Reader {
  const std::string& t;
  std::size_t i = 0;
  [[noreturn]] void fail(const std::string& what) const {
    throw ParseError("JSON: " + what, i);
  }
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\t' || t[i] == '\r')) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < t.size() && t[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  std::string string_lit() {
    expect('"');
    std::string s;
    while (i < t.size() && t[i] != '"') {
      if (t[i] == '\\') {
        if (++i >= t.size()) fail("bad escape");
        const char e = t[i];
        s += e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e;
      } else {
        s += t[i];
      }
      ++i;
    }
    if (i >= t.size()) fail("unterminated string");
    ++i;
    return s;
  }
  JVal value() {
    ws();
    if (i >= t.size()) fail("unexpected end");
    JVal v;
    const char c = t[i];
    if (c == '{') {
      ++i;
      v.kind = JVal::Obj;
      if (eat('}')) return v;
      do {
        ws();
        std::string k = string_lit();
        expect(':');
        v.obj[k] = value();
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i;
      v.kind = JVal::Arr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.str = string_lit();
    } else if (t.compare(i, 4, "true") == 0) {
      i += 4;
      v.kind = JVal::Bool;
      v.b = true;
    } else if (t.compare(i, 5, "false") == 0) {
      i += 5;
      v.kind = JVal::Bool;
    } else if (t.compare(i, 4, "null") == 0) {
      i += 4;
    } else {
      const std::size_t st = i;
      if (t[i] == '-') ++i;
      bool frac = false;
      while (i < t.size() && (std::isdigit(static_cast<unsigned char>(t[i])) || t[i] == '.' || t[i] == 'e' ||
                              t[i] == 'E' || t[i] == '+' || t[i] == '-')) {
        frac |= t[i] == '.' || t[i] == 'e' || t[i] == 'E';
        ++i;
      }
      if (i == st) fail("unexpected character");
      v.kind = JVal::Num;
      const char* b = t.data() + st;
      const char* e = t.data() + i;
      auto rd = std::from_chars(b, e, v.num);
      if (rd.ec != std::errc() || rd.ptr != e) fail("bad number");
      if (!frac) {
        auto ri = std::from_chars(b, e, v.inum);
        v.is_int = ri.ec == std::errc() && ri.ptr == e;
      }
    }
    return v;
  }
};

JVal parse_json(const std::string& text) {
  Reader r{text};
  JVal v = r.value();
  r.ws();
  if (r.i != text.size()) r.fail("trailing characters");
  return v;
}

const JVal& at(const JVal& o, const char* key) {
  if (o.kind != JVal::Obj) throw ParseError("JSON: expected an object", 0);
  auto it = o.obj.find(key);
  if (it == o.obj.end()) throw ParseError(std::string("JSON: missing key '") + key + "'", 0);
  return it->second;
}

int64_t as_int(const JVal& v, const char* what) {
  if (v.kind != JVal::Num || !v.is_int) throw ParseError(std::string("JSON: '") + what + "' must be an integer", 0);
  return v.inum;
}

std::vector<int64_t> int_list(const JVal& v, const char* what) {
  std::vector<int64_t> out;
  if (v.kind == JVal::Arr) {
    for (const JVal& x : v.arr) out.push_back(as_int(x, what));
  } else {
    out.push_back(as_int(v, what));
  }
  return out;
}

int64_t count_of(const std::vector<int64_t>& shape) {
  int64_t n = 1;
  for (int64_t d : shape) {
    if (d < 0) throw ShapeError("tensor: negative dimension");
    n *= d;
  }
  return n;
}

}  // namespace

// ------------------------------------------------------------------ tensors
std::string tensor_to_json(const std::vector<int64_t>& shape, const double* data) {
  // nlohmann objects are key-sorted: "data" before "shape"
  std::string s = "{\"data\":[";
  const int64_t n = count_of(shape);
  for (int64_t i = 0; i < n; ++i) {
    if (i) s += ',';
    s += json_number(data[i]);
  }
  s += "],\"shape\":[";
  for (std::size_t i = 0; i < shape.size(); ++i) s += (i ? "," : "") + std::to_string(shape[i]);
  return s + "]}";
}

void tensor_from_json(const std::string& text, std::vector<int64_t>* shape, std::vector<double>* data) {
  const JVal j = parse_json(text);
  *shape = int_list(at(j, "shape"), "shape");
  if (at(j, "shape").kind != JVal::Arr) throw ParseError("JSON: 'shape' must be an array", 0);
  const JVal& d = at(j, "data");
  if (d.kind != JVal::Arr) throw ParseError("JSON: 'data' must be an array", 0);
  data->clear();
  for (const JVal& x : d.arr) {
    if (x.kind != JVal::Num) throw ParseError("JSON: tensor data must be numbers", 0);
    data->push_back(x.num);
  }
  if (static_cast<int64_t>(data->size()) != count_of(*shape))
    throw ShapeError("tensor JSON: data length does not match shape");
}

namespace {
void put_u64(std::string& s, uint64_t v) {
  for (int i = 0; i < 8; ++i) s += static_cast<char>((v >> (8 * i)) & 0xff);
}
uint64_t get_u64(const std::string& s, std::size_t& pos) {
  if (pos + 8 > s.size()) throw ShapeError("tensor binary: truncated stream");
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | static_cast<unsigned char>(s[pos + static_cast<std::size_t>(i)]);
  pos += 8;
  return v;
}
}  // namespace

std::string tensor_to_binary(const std::vector<int64_t>& shape, const double* data) {
  std::string s;
  put_u64(s, shape.size());
  for (int64_t d : shape) put_u64(s, static_cast<uint64_t>(d));
  const int64_t n = count_of(shape);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits;
    std::memcpy(&bits, &data[i], 8);
    put_u64(s, bits);
  }
  return s;
}

void tensor_from_binary(const std::string& bytes, std::vector<int64_t>* shape, std::vector<double>* data) {
  std::size_t pos = 0;
  const uint64_t rank = get_u64(bytes, pos);
  if (rank > 64) throw ShapeError("tensor binary: rank " + std::to_string(rank) + " out of range");
  shape->assign(rank, 0);
  for (auto& d : *shape) d = static_cast<int64_t>(get_u64(bytes, pos));
  const int64_t n = count_of(*shape);
  if (static_cast<uint64_t>(n) > (bytes.size() - pos) / 8) throw ShapeError("tensor binary: truncated stream");
  data->resize(static_cast<std::size_t>(n));
  for (auto& v : *data) {
    const uint64_t bits = get_u64(bytes, pos);
    std::memcpy(&v, &bits, 8);
  }
}

// ------------------------------------------------------------------ layers
LayerSpec layer_from_json(const std::string& text) {
  const JVal j = parse_json(text);
  LayerSpec l;
  const JVal& k = at(j, "kind");
  if (k.kind != JVal::Str) throw ParseError("JSON: 'kind' must be a string", 0);
  l.kind = layer_kind_from_string(k.str);
  l.t_factors = int_list(at(j, "T"), "T");
  l.s_factors = int_list(at(j, "S"), "S");
  l.filter_h = as_int(at(j, "H"), "H");
  l.filter_w = as_int(at(j, "W"), "W");
  l.feature_h = as_int(at(j, "Hp"), "Hp");
  l.feature_w = as_int(at(j, "Wp"), "Wp");
  l.batch = j.obj.count("B") ? as_int(j.obj.at("B"), "B") : 1;  // j.value("B", 1)
  const std::size_t slots = rank_slot_count(l.kind, l.order());
  if (j.obj.count("rank")) {
    auto ranks = int_list(j.obj.at("rank"), "rank");
    if (ranks.size() == 1 && slots > 1) ranks.assign(slots, ranks[0]);
    l.ranks = std::move(ranks);
  }
  validate(l);
  return l;
}

}  // namespace ce
