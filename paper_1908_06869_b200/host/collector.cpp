// libstrata_b200: collector drop-in (reference: collector.hpp / collector.cpp).
//
// The JSONL codec is self-contained: a strict RFC 8259 reader for one record
// per line and a writer that emits the reference's wire form byte for byte
// (keys in lexicographic order, no whitespace, integers in decimal, doubles as
// the reference's JSON library prints them: Grisu2 digits laid out as
// "15700000000000.0", "0.5", "1e-05"). Number typing follows the
// reference: an integer literal is unsigned when it fits u64 and has no sign,
// signed when negative and it fits i64, otherwise a double.
//
// Ordering and validation of an ingested or merged bundle run on the GPU
// (sort_timeline / validate_bundle in span.cpp go through the C ABI).
#include "strata/collector.hpp"

#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <memory>
#include <sstream>
#include <unordered_set>
#include <utility>

namespace strata {

namespace {

// ---------------------------------------------------------------------------
// JSON values

struct JVal {
  enum Type { Null, Bool, Int, UInt, Float, Str, Arr, Obj } t = Null;
  bool b = false;
  std::int64_t i = 0;
  std::uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;  // later duplicate keys win (find searches backwards)

  bool is_number() const { return t == Int || t == UInt || t == Float; }
  const JVal* find(const char* key) const {
    for (auto it = obj.rbegin(); it != obj.rend(); ++it)
      if (it->first == key) return &it->second;
    return nullptr;
  }
  double as_double() const { return t == Float ? d : t == UInt ? static_cast<double>(u) : static_cast<double>(i); }
  std::int64_t as_i64() const {
    return t == Int ? i : t == UInt ? static_cast<std::int64_t>(u) : static_cast<std::int64_t>(d);
  }
  std::uint64_t as_u64() const {
    return t == UInt ? u : t == Int ? static_cast<std::uint64_t>(i) : static_cast<std::uint64_t>(d);
  }
};

class Parser {
 public:
  Parser(const char* p, const char* e) : p_(p), e_(e) {}

  // Whole-input parse; false on any syntax error or trailing content.
  bool parse(JVal& out) {
    ws();
    if (!value(out, 0)) return false;
    ws();
    return p_ == e_;
  }

 private:
  const char* p_;
  const char* e_;

  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::strlen(w);
    if (static_cast<std::size_t>(e_ - p_) < n || std::memcmp(p_, w, n) != 0) return false;
    p_ += n;
    return true;
  }
  bool value(JVal& v, int depth) {
    if (depth > 512 || p_ >= e_) return false;
    switch (*p_) {
      case '{': return object(v, depth);
      case '[': return array(v, depth);
      case '"': v.t = JVal::Str; return string(v.s);
      case 't': v.t = JVal::Bool; v.b = true; return lit("true");
      case 'f': v.t = JVal::Bool; v.b = false; return lit("false");
      case 'n': v.t = JVal::Null; return lit("null");
      default: return number(v);
    }
  }
  bool object(JVal& v, int depth) {
    v.t = JVal::Obj;
    ++p_;
    ws();
    if (p_ < e_ && *p_ == '}') { ++p_; return true; }
    for (;;) {
      ws();
      if (p_ >= e_ || *p_ != '"') return false;
      std::string key;
      if (!string(key)) return false;
      ws();
      if (p_ >= e_ || *p_ != ':') return false;
      ++p_;
      ws();
      JVal item;
      if (!value(item, depth + 1)) return false;
      v.obj.emplace_back(std::move(key), std::move(item));
      ws();
      if (p_ < e_ && *p_ == ',') { ++p_; continue; }
      if (p_ < e_ && *p_ == '}') { ++p_; return true; }
      return false;
    }
  }
  bool array(JVal& v, int depth) {
    v.t = JVal::Arr;
    ++p_;
    ws();
    if (p_ < e_ && *p_ == ']') { ++p_; return true; }
    for (;;) {
      ws();
      JVal item;
      if (!value(item, depth + 1)) return false;
      v.arr.push_back(std::move(item));
      ws();
      if (p_ < e_ && *p_ == ',') { ++p_; continue; }
      if (p_ < e_ && *p_ == ']') { ++p_; return true; }
      return false;
    }
  }
  static void put_utf8(std::string& s, std::uint32_t cp) {
    if (cp < 0x80) {
      s += static_cast<char>(cp);
    } else if (cp < 0x800) {
      s += static_cast<char>(0xC0 | (cp >> 6));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      s += static_cast<char>(0xE0 | (cp >> 12));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      s += static_cast<char>(0xF0 | (cp >> 18));
      s += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  bool hex4(std::uint32_t& cp) {
    if (e_ - p_ < 4) return false;
    cp = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p_++;
      cp <<= 4;
      if (c >= '0' && c <= '9') cp |= c - '0';
      else if (c >= 'a' && c <= 'f') cp |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') cp |= c - 'A' + 10;
      else return false;
    }
    return true;
  }
  // one well-formed UTF-8 sequence (no overlongs, no surrogates, <= U+10FFFF)
  bool utf8(std::string& s) {
    const auto c0 = static_cast<unsigned char>(*p_);
    int n = c0 >= 0xF0 ? 3 : c0 >= 0xE0 ? 2 : c0 >= 0xC2 ? 1 : -1;
    if (n < 0 || c0 > 0xF4 || e_ - p_ < n + 1) return false;
    std::uint32_t cp = c0 & (0x3F >> n);
    for (int k = 1; k <= n; ++k) {
      const auto c = static_cast<unsigned char>(p_[k]);
      if ((c & 0xC0) != 0x80) return false;
      cp = (cp << 6) | (c & 0x3F);
    }
    if ((n == 2 && (cp < 0x800 || (cp >= 0xD800 && cp <= 0xDFFF))) || (n == 3 && (cp < 0x10000 || cp > 0x10FFFF)))
      return false;
    s.append(p_, n + 1);
    p_ += n + 1;
    return true;
  }
  bool string(std::string& s) {
    ++p_;  // opening quote
    for (;;) {
      if (p_ >= e_) return false;
      const auto c = static_cast<unsigned char>(*p_);
      if (c == '"') { ++p_; return true; }
      if (c < 0x20) return false;
      if (c >= 0x80) {
        if (!utf8(s)) return false;
        continue;
      }
      if (c != '\\') { s += static_cast<char>(c); ++p_; continue; }
      ++p_;
      if (p_ >= e_) return false;
      const char esc = *p_++;
      switch (esc) {
        case '"': s += '"'; break;
        case '\\': s += '\\'; break;
        case '/': s += '/'; break;
        case 'b': s += '\b'; break;
        case 'f': s += '\f'; break;
        case 'n': s += '\n'; break;
        case 'r': s += '\r'; break;
        case 't': s += '\t'; break;
        case 'u': {
          std::uint32_t cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp <= 0xDBFF) {  // high surrogate: a low one must follow
            std::uint32_t lo;
            if (!(lit("\\u") && hex4(lo) && lo >= 0xDC00 && lo <= 0xDFFF)) return false;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            return false;
          }
          put_utf8(s, cp);
          break;
        }
        default: return false;
      }
    }
  }
  bool number(JVal& v) {
    const char* b = p_;
    bool neg = false, frac = false;
    if (p_ < e_ && *p_ == '-') { neg = true; ++p_; }
    if (p_ >= e_) return false;
    if (*p_ == '0') {
      ++p_;
    } else if (*p_ >= '1' && *p_ <= '9') {
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    } else {
      return false;
    }
    if (p_ < e_ && *p_ == '.') {
      frac = true;
      ++p_;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
      frac = true;
      ++p_;
      if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (!frac) {
      if (neg) {
        std::int64_t x;
        auto r = std::from_chars(b, p_, x);
        if (r.ec == std::errc() && r.ptr == p_) { v.t = JVal::Int; v.i = x; return true; }
      } else {
        std::uint64_t x;
        auto r = std::from_chars(b, p_, x);
        if (r.ec == std::errc() && r.ptr == p_) { v.t = JVal::UInt; v.u = x; return true; }
      }
    }
    // fraction, exponent or integer overflow: a double (correctly rounded)
    v.t = JVal::Float;
    const std::string text(b, p_);
    v.d = std::strtod(text.c_str(), nullptr);
    return std::isfinite(v.d);  // out of double range: not a number the reference accepts
  }
};

// ---------------------------------------------------------------------------
// writer

void put_string(std::string& out, const std::string& s) {
  static const char* hex = "0123456789abcdef";
  out += '"';
  for (const char ch : s) {
    const auto c = static_cast<unsigned char>(ch);
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          out += "\\u00";
          out += hex[c >> 4];
          out += hex[c & 15];
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

void put_u64(std::string& out, std::uint64_t v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, r.ptr);
}

void put_i64(std::string& out, std::int64_t v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, r.ptr);
}

// ---------------------------------------------------------------------------
// Grisu2 (F. Loitsch, "Printing floating-point numbers quickly and accurately
// with integers", PLDI 2010) as the reference's JSON library (nlohmann/json
// 3.11.3, a dependency the reference does not vendor) uses it to print doubles:
// digits within the rounding interval of the value, NOT always the shortest
// (5.81e21 prints as 5.809999999999999e+21), so the wire bytes can only match
// by running the same algorithm. Cached powers 10^k (k = -300, -292, ..., 324):
// the 64-bit significand of 10^k rounded to nearest, with its binary exponent
// (generated exactly with rational arithmetic).

struct DiyFp {
  std::uint64_t f;
  int e;
};

DiyFp diy_sub(DiyFp x, DiyFp y) { return {x.f - y.f, x.e}; }

DiyFp diy_mul(DiyFp x, DiyFp y) {  // upper 64 bits of the 128-bit product, rounded half up
  const std::uint64_t ul = x.f & 0xFFFFFFFFu, uh = x.f >> 32, vl = y.f & 0xFFFFFFFFu, vh = y.f >> 32;
  const std::uint64_t p0 = ul * vl, p1 = ul * vh, p2 = uh * vl, p3 = uh * vh;
  std::uint64_t q = (p0 >> 32) + (p1 & 0xFFFFFFFFu) + (p2 & 0xFFFFFFFFu);
  q += std::uint64_t{1} << 31;
  return {p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}

DiyFp diy_normalize(DiyFp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

struct CachedPow {
  std::uint64_t f;
  int e;
  int k;
};

constexpr CachedPow kCachedPow[] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324},
};

void grisu2_round(char* buf, int len, std::uint64_t dist, std::uint64_t delta, std::uint64_t rest,
                  std::uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}

// digits of v (finite, > 0) into buf; value = digits * 10^dec_exp
int grisu2(char* buf, int& dec_exp, double value) {
  std::uint64_t bits;
  std::memcpy(&bits, &value, 8);
  const std::uint64_t F = bits & ((std::uint64_t{1} << 52) - 1);
  const int E = static_cast<int>(bits >> 52);
  const DiyFp v = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F + (std::uint64_t{1} << 52), E - 1075};
  const bool lower_closer = F == 0 && E > 1;
  const DiyFp m_plus{2 * v.f + 1, v.e - 1};
  const DiyFp m_minus = lower_closer ? DiyFp{4 * v.f - 1, v.e - 2} : DiyFp{2 * v.f - 1, v.e - 1};
  const DiyFp w_plus = diy_normalize(m_plus);
  const DiyFp w_minus{m_minus.f << (m_minus.e - w_plus.e), w_plus.e};
  const DiyFp w = diy_normalize(v);
  // cached power c = 10^-k with the product's exponent in [-60, -32]
  const int fexp = -60 - w_plus.e - 1;
  const int kk = (fexp * 78913) / (1 << 18) + static_cast<int>(fexp > 0);
  const CachedPow& c = kCachedPow[(300 + kk + 7) / 8];
  const DiyFp cm{c.f, c.e};
  const DiyFp W = diy_mul(w, cm), Wm = diy_mul(w_minus, cm), Wp = diy_mul(w_plus, cm);
  const DiyFp M_minus{Wm.f + 1, Wm.e}, M_plus{Wp.f - 1, Wp.e};
  dec_exp = -c.k;
  // digit generation
  std::uint64_t delta = diy_sub(M_plus, M_minus).f;
  std::uint64_t dist = diy_sub(M_plus, W).f;
  const int sh = -M_plus.e;
  const std::uint64_t one = std::uint64_t{1} << sh;
  auto p1 = static_cast<std::uint32_t>(M_plus.f >> sh);
  std::uint64_t p2 = M_plus.f & (one - 1);
  std::uint32_t pow10 = 1;
  int n = 1;
  for (std::uint32_t t = 1000000000u, d = 10; d > 1; t /= 10, --d)
    if (p1 >= t) {
      pow10 = t;
      n = static_cast<int>(d);
      break;
    }
  int len = 0;
  while (n > 0) {
    const std::uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[len++] = static_cast<char>('0' + d);
    p1 = r;
    --n;
    const std::uint64_t rest = (std::uint64_t{p1} << sh) + p2;
    if (rest <= delta) {
      dec_exp += n;
      grisu2_round(buf, len, dist, delta, rest, std::uint64_t{pow10} << sh);
      return len;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const std::uint64_t d = p2 >> sh, r = p2 & (one - 1);
    buf[len++] = static_cast<char>('0' + d);
    p2 = r;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dec_exp -= m;
  grisu2_round(buf, len, dist, delta, p2, one);
  return len;
}

// The reference's layout of those digits: fixed notation for decimal
// exponents in (-4, 15], with ".0" on integral values; otherwise
// d[.ddd]e(+|-)XX with at least two exponent digits.
void put_double(std::string& out, double x) {
  if (!std::isfinite(x)) {
    out += "null";
    return;
  }
  if (std::signbit(x)) {
    out += '-';
    x = -x;
  }
  if (x == 0.0) {
    out += "0.0";
    return;
  }
  char buf[32];
  int dec_exp = 0;
  const int k = grisu2(buf, dec_exp, x);
  const std::string digits(buf, k);
  const int n = k + dec_exp;  // decimal point position relative to the digit string
  if (k <= n && n <= 15) {
    out += digits;
    out.append(n - k, '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out.append(digits, 0, n);
    out += '.';
    out.append(digits, n, std::string::npos);
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append(-n, '0');
    out += digits;
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out.append(digits, 1, std::string::npos);
    }
    const int ex = n - 1;
    out += 'e';
    out += ex < 0 ? '-' : '+';
    const int a = ex < 0 ? -ex : ex;
    if (a < 10) out += '0';
    put_i64(out, a);
  }
}

struct Obj {  // keys are written in lexicographic order by construction at each call site
  std::string& out;
  bool first = true;
  explicit Obj(std::string& o) : out(o) { out += '{'; }
  ~Obj() { out += '}'; }
  std::string& key(const char* k) {
    if (!first) out += ',';
    first = false;
    put_string(out, k);
    out += ':';
    return out;
  }
};

void put_system(std::string& out, const SystemSpec& s) {
  Obj o(out);
  put_double(o.key("mem_bw"), s.memory_bandwidth_bytes_per_s);
  put_string(o.key("name"), s.name);
  put_double(o.key("peak_flops"), s.peak_flops);
}

void put_tag(std::string& out, const TagValue& v) {
  if (const auto* s = std::get_if<std::string>(&v)) put_string(out, *s);
  else if (const auto* i = std::get_if<std::int64_t>(&v)) put_i64(out, *i);
  else put_double(out, std::get<double>(v));
}

// ---------------------------------------------------------------------------
// record decoding (collector.cpp:23-186)

std::uint64_t require_u64(const JVal& rec, const char* field) {
  const JVal* v = rec.find(field);
  if (!v || !v->is_number())
    throw IngestError(std::string("missing or non-numeric field '") + field + "'");
  if (v->t == JVal::Float) throw IngestError(std::string("field '") + field + "' must be an integer");
  if (v->t == JVal::Int && v->i < 0) throw IngestError(std::string("field '") + field + "' must be non-negative");
  return v->as_u64();
}

std::string require_string(const JVal& rec, const char* field) {
  const JVal* v = rec.find(field);
  if (!v || v->t != JVal::Str) throw IngestError(std::string("missing or non-string field '") + field + "'");
  return v->s;
}

TagValue tag_value(const JVal& v) {
  switch (v.t) {
    case JVal::Str: return v.s;
    case JVal::Float: return v.d;
    case JVal::Int:
    case JVal::UInt: return v.as_i64();
    case JVal::Bool: return static_cast<std::int64_t>(v.b);
    default: throw IngestError("tag value must be a string or number");
  }
}

SystemSpec system_from(const JVal& v) {
  if (v.t != JVal::Obj) throw IngestError("'system' must be an object");
  SystemSpec spec;
  spec.name = require_string(v, "name");
  const JVal* peak = v.find("peak_flops");
  const JVal* bw = v.find("mem_bw");
  if (!peak || !peak->is_number()) throw IngestError("missing or non-numeric field 'peak_flops'");
  if (!bw || !bw->is_number()) throw IngestError("missing or non-numeric field 'mem_bw'");
  spec.peak_flops = peak->as_double();
  spec.memory_bandwidth_bytes_per_s = bw->as_double();
  return spec;
}

RunMeta meta_from(const JVal& rec) {
  RunMeta meta;
  meta.trace_id = require_u64(rec, "trace_id");
  meta.batch_size = static_cast<std::uint32_t>(require_u64(rec, "batch_size"));
  meta.run_index = static_cast<std::uint32_t>(require_u64(rec, "run_index"));
  const JVal* levels = rec.find("levels");
  if (!levels || levels->t != JVal::Arr) throw IngestError("missing or non-array field 'levels'");
  for (const JVal& e : levels->arr) {
    if (e.t != JVal::Str) throw IngestError("level names must be strings");
    auto level = level_from_name(e.s);
    if (!level) throw IngestError("unknown level '" + e.s + "'");
    meta.profiling_levels.insert(*level);
  }
  if (const JVal* ser = rec.find("serialized")) {
    if (ser->t != JVal::Bool) throw IngestError("field 'serialized' must be a boolean");
    meta.serialized = ser->b;
  }
  const JVal* system = rec.find("system");
  if (!system) throw IngestError("missing field 'system'");
  meta.system = system_from(*system);
  return meta;
}

Span span_from(const JVal& rec) {
  Span span;
  span.trace_id = require_u64(rec, "trace_id");
  span.span_id = require_u64(rec, "span_id");
  span.name = require_string(rec, "name");
  auto level = level_from_name(require_string(rec, "level"));
  if (!level) throw IngestError("unknown level name");
  span.level = *level;
  auto kind = kind_from_name(require_string(rec, "kind"));
  if (!kind) throw IngestError("unknown kind name");
  span.kind = *kind;
  span.begin_ns = require_u64(rec, "begin_ns");
  span.end_ns = require_u64(rec, "end_ns");
  if (const JVal* p = rec.find("parent_id"); p && p->t != JVal::Null) span.parent_id = require_u64(rec, "parent_id");
  if (const JVal* c = rec.find("correlation_id"); c && c->t != JVal::Null)
    span.correlation_id = require_u64(rec, "correlation_id");
  if (const JVal* tags = rec.find("tags"); tags && tags->t != JVal::Null) {
    if (tags->t != JVal::Obj) throw IngestError("'tags' must be an object");
    // duplicate keys: the later value is the object's value; the tag map keeps one entry per key
    for (std::size_t k = 0; k < tags->obj.size(); ++k) {
      const std::string& key = tags->obj[k].first;
      if (span.tags.count(key)) continue;
      span.tags.emplace(key, tag_value(*tags->find(key.c_str())));
    }
  }
  return span;
}

bool parse_line(const std::string& line, JVal& out) {
  Parser p(line.data(), line.data() + line.size());
  return p.parse(out);
}

}  // namespace

// ---------------------------------------------------------------------------
// public API

std::string encode_meta_record(const RunMeta& meta) {
  std::string out;
  {
    Obj o(out);
    put_u64(o.key("batch_size"), meta.batch_size);
    std::string& lv = o.key("levels");
    lv += '[';
    bool first = true;
    for (Level level : meta.profiling_levels) {
      if (!first) lv += ',';
      first = false;
      put_string(lv, level_name(level));
    }
    lv += ']';
    put_string(o.key("rec"), "meta");
    put_u64(o.key("run_index"), meta.run_index);
    o.key("serialized") += meta.serialized ? "true" : "false";
    put_system(o.key("system"), meta.system);
    put_u64(o.key("trace_id"), meta.trace_id);
  }
  return out;
}

std::string encode_span_record(const Span& span) {
  std::string out;
  {
    Obj o(out);
    put_u64(o.key("begin_ns"), span.begin_ns);
    if (span.correlation_id) put_u64(o.key("correlation_id"), *span.correlation_id);
    else o.key("correlation_id") += "null";
    put_u64(o.key("end_ns"), span.end_ns);
    put_string(o.key("kind"), kind_name(span.kind));
    put_string(o.key("level"), level_name(span.level));
    put_string(o.key("name"), span.name);
    if (span.parent_id) put_u64(o.key("parent_id"), *span.parent_id);
    else o.key("parent_id") += "null";
    put_string(o.key("rec"), "span");
    put_u64(o.key("span_id"), span.span_id);
    {
      std::string& t = o.key("tags");
      Obj to(t);
      for (const auto& [key, value] : span.tags) put_tag(to.key(key.c_str()), value);
    }
    put_u64(o.key("trace_id"), span.trace_id);
  }
  return out;
}

SystemSpec parse_system_spec(const std::string& json_text) {
  JVal v;
  if (!parse_line(json_text, v)) throw IngestError("system spec is not valid JSON");
  return system_from(v);
}

std::string encode_system_spec(const SystemSpec& spec) {
  std::string out;
  put_system(out, spec);
  return out;
}

SystemSpec load_system_spec(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open system spec '" + path + "'");
  std::ostringstream text;
  text << in.rdbuf();
  return parse_system_spec(text.str());
}

TraceBundle ingest(std::istream& stream) {
  TraceBundle bundle;
  bool have_meta = false;
  std::string line;
  std::size_t line_no = 0;
  while (std::getline(stream, line)) {
    ++line_no;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;  // blank lines are allowed
    JVal rec;
    if (!parse_line(line, rec) || rec.t != JVal::Obj)
      throw IngestError("line " + std::to_string(line_no) + ": not a JSON object");
    const JVal* kind = rec.find("rec");
    const std::string r = kind && kind->t == JVal::Str ? kind->s : std::string{};
    try {
      if (r == "meta") {
        if (have_meta) throw IngestError("duplicate meta record");
        bundle.meta = meta_from(rec);
        have_meta = true;
      } else if (r == "span") {
        bundle.spans.push_back(span_from(rec));
      }
      // other record kinds are skipped (forward compatibility)
    } catch (const IngestError& e) {
      throw IngestError("line " + std::to_string(line_no) + ": " + e.what());
    }
  }
  if (!have_meta) throw IngestError("stream holds no meta record");
  for (const Span& span : bundle.spans) {
    if (span.trace_id != bundle.meta.trace_id)
      throw IngestError("span " + std::to_string(span.span_id) + " carries trace_id " +
                        std::to_string(span.trace_id) + " but the meta record declares " +
                        std::to_string(bundle.meta.trace_id));
  }
  sort_timeline(bundle.spans);                          // GPU
  const ValidationReport report = validate_bundle(bundle);  // GPU
  if (!report.empty()) {
    std::ostringstream msg;
    msg << "bundle fails validation (" << report.size() << " violation" << (report.size() == 1 ? "" : "s") << "):";
    for (const Violation& v : report) {
      msg << "\n  span " << v.span_id << ": " << v.rule;
      if (!v.detail.empty()) msg << " (" << v.detail << ")";
    }
    throw IngestError(msg.str());
  }
  return bundle;
}

TraceBundle ingest_string(const std::string& text) {
  std::istringstream stream(text);
  return ingest(stream);
}

TraceBundle merge(const std::vector<TraceBundle>& bundles) {
  if (bundles.empty()) throw MergeError("nothing to merge");
  TraceBundle merged;
  merged.meta = bundles.front().meta;
  std::unordered_set<std::uint64_t> seen;
  std::size_t total = 0;
  for (const TraceBundle& b : bundles) total += b.spans.size();
  merged.spans.reserve(total);
  seen.reserve(total);
  for (const TraceBundle& bundle : bundles) {
    if (bundle.meta.trace_id != merged.meta.trace_id)
      throw MergeError("trace_id mismatch: " + std::to_string(bundle.meta.trace_id) + " vs " +
                       std::to_string(merged.meta.trace_id));
    if (!(bundle.meta == merged.meta))
      throw MergeError("run metadata disagrees across bundles of trace " + std::to_string(merged.meta.trace_id));
    for (const Span& span : bundle.spans) {
      if (!seen.insert(span.span_id).second)
        throw MergeError("duplicate span_id " + std::to_string(span.span_id) + " across merged bundles");
      merged.spans.push_back(span);
    }
  }
  sort_timeline(merged.spans);  // GPU
  return merged;
}

std::string to_jsonl(const TraceBundle& bundle) {
  std::string out = encode_meta_record(bundle.meta);
  out += '\n';
  for (const Span& span : bundle.spans) {
    out += encode_span_record(span);
    out += '\n';
  }
  return out;
}

void persist(const TraceBundle& bundle, const std::string& path) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  out << to_jsonl(bundle);
  if (!out) throw IoError("write to '" + path + "' failed");
}

TraceBundle load(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open '" + path + "'");
  return ingest(in);
}

void RunSet::add(TraceBundle bundle) {
  if (groups.empty()) {
    system = bundle.meta.system;
  } else if (!(bundle.meta.system == system)) {
    throw MergeError("system spec disagrees across runs of one experiment");
  }
  GroupKey key{bundle.meta.batch_size, bundle.meta.profiling_levels};
  auto& group = groups[key];
  for (const TraceBundle& existing : group) {
    if (existing.meta.trace_id == bundle.meta.trace_id && existing.meta.run_index == bundle.meta.run_index)
      throw MergeError("duplicate run (trace " + std::to_string(bundle.meta.trace_id) + ", run_index " +
                       std::to_string(bundle.meta.run_index) + ")");
  }
  group.push_back(std::move(bundle));
}

RunSet RunSet::from_bundles(std::vector<TraceBundle> bundles) {
  RunSet set;
  for (TraceBundle& bundle : bundles) set.add(std::move(bundle));
  return set;
}

}  // namespace strata
