// Model geometry: small pages, the LCM large page, config parsing.
// Semantics follow reference proj/src/model_config.cpp (cited per function);
// the JSON reader is a small self-contained recursive-descent parser so the
// runtime has no third-party dependency.
#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <map>
#include <numeric>
#include <set>

#include "jenga_host.hpp"

namespace jenga {

uint64_t checked_mul(uint64_t a, uint64_t b, const char* what) {
  uint64_t out = 0;
  if (__builtin_mul_overflow(a, b, &out))
    throw ConfigError(std::string("byte arithmetic overflow in ") + what);
  return out;
}

uint64_t checked_add(uint64_t a, uint64_t b, const char* what) {
  uint64_t out = 0;
  if (__builtin_add_overflow(a, b, &out))
    throw ConfigError(std::string("byte arithmetic overflow in ") + what);
  return out;
}

uint64_t hash_str(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

const char* layer_kind_name(LayerKind k) {
  switch (k) {
    case LayerKind::kFullAttention: return "full";
    case LayerKind::kSlidingWindow: return "sliding_window";
    case LayerKind::kMamba: return "mamba";
    case LayerKind::kCrossAttention: return "cross_attention";
    case LayerKind::kVisionEmbedding: return "vision_embedding";
  }
  return "?";
}

LayerKind layer_kind_from_name(const std::string& s) {
  static const std::map<std::string, LayerKind> kinds = {
      {"full", LayerKind::kFullAttention},
      {"sliding_window", LayerKind::kSlidingWindow},
      {"mamba", LayerKind::kMamba},
      {"cross_attention", LayerKind::kCrossAttention},
      {"vision_embedding", LayerKind::kVisionEmbedding}};
  auto it = kinds.find(s);
  if (it == kinds.end()) throw ConfigError("unknown layer kind '" + s + "'");
  return it->second;
}

// reference model_config.cpp:85-89
uint64_t small_page_size(const LayerGroupSpec& g) {
  const uint64_t per_token =
      checked_mul(g.bytes_per_token_per_layer, g.num_layers, "small_page_size");
  return checked_mul(per_token, g.tokens_per_page, "small_page_size");
}

// reference model_config.cpp:41-70
void ModelSpec::validate() const {
  if (groups.empty()) throw ConfigError("model '" + name + "' has no layer groups");
  std::set<std::string> names;
  for (const auto& g : groups) {
    if (g.name.empty()) throw ConfigError("layer group with empty name");
    if (!names.insert(g.name).second)
      throw ConfigError("duplicate layer group name '" + g.name + "'");
    if (g.num_layers == 0) throw ConfigError("group '" + g.name + "': num_layers must be > 0");
    if (g.bytes_per_token_per_layer == 0)
      throw ConfigError("group '" + g.name + "': bytes_per_token_per_layer must be > 0");
    if (g.tokens_per_page == 0)
      throw ConfigError("group '" + g.name + "': tokens_per_page must be >= 1");
    if (g.kind == LayerKind::kSlidingWindow && g.window_tokens == 0)
      throw ConfigError("group '" + g.name + "': window_tokens must be >= 1");
    if (g.kind == LayerKind::kMamba && g.checkpoint_interval_tokens == 0)
      throw ConfigError("group '" + g.name + "': checkpoint_interval_tokens must be >= 1");
    (void)small_page_size(g);
  }
}

bool ModelSpec::has_cross_attention() const {
  for (const auto& g : groups)
    if (g.kind == LayerKind::kCrossAttention) return true;
  return false;
}

// reference model_config.cpp:93-107 (checked_lcm folded over the groups)
uint64_t lcm_page_size(const ModelSpec& spec) {
  spec.validate();
  uint64_t l = 1;
  for (const auto& g : spec.groups) {
    const uint64_t s = small_page_size(g);
    l = checked_mul(l / std::gcd(l, s), s, "compatible_page_size (lcm)");
  }
  return l;
}

// reference model_config.cpp:129-142
double lcm_blowup_ratio(const ModelSpec& spec) {
  const uint64_t lcm = lcm_page_size(spec);
  uint64_t mn = UINT64_MAX;
  for (const auto& g : spec.groups) mn = std::min(mn, small_page_size(g));
  return static_cast<double>(lcm) / static_cast<double>(mn);
}

// ------------------------------------------------------------ mini JSON
namespace {

struct JValue {
  enum Type { kNull, kBool, kNum, kStr, kArr, kObj } type = kNull;
  bool b = false;
  double num = 0;
  bool is_uint = false;
  uint64_t u = 0;
  std::string s;
  std::vector<JValue> arr;
  std::vector<std::pair<std::string, JValue>> obj;
  const JValue* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JParser {
 public:
  explicit JParser(const std::string& t) : t_(t) {}
  JValue parse() {
    JValue v = value();
    ws();
    if (i_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) {
    throw ConfigError(std::string("model config parse error: ") + what + " at offset " +
                      std::to_string(i_));
  }
  void ws() {
    while (i_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[i_]))) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < t_.size() && t_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  JValue value() {
    ws();
    if (i_ >= t_.size()) fail("unexpected end");
    const char c = t_[i_];
    JValue v;
    if (c == '{') {
      ++i_;
      v.type = JValue::kObj;
      if (eat('}')) return v;
      do {
        ws();
        std::string k = str();
        if (!eat(':')) fail("expected ':'");
        v.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      if (!eat('}')) fail("expected '}'");
    } else if (c == '[') {
      ++i_;
      v.type = JValue::kArr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) fail("expected ']'");
    } else if (c == '"') {
      v.type = JValue::kStr;
      v.s = str();
    } else if (t_.compare(i_, 4, "true") == 0) {
      i_ += 4;
      v.type = JValue::kBool;
      v.b = true;
    } else if (t_.compare(i_, 5, "false") == 0) {
      i_ += 5;
      v.type = JValue::kBool;
    } else if (t_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
      const size_t b = i_;
      bool integral = true;
      if (t_[i_] == '-') { ++i_; integral = false; }
      while (i_ < t_.size() && (std::isdigit(static_cast<unsigned char>(t_[i_])) ||
                                t_[i_] == '.' || t_[i_] == 'e' || t_[i_] == 'E' ||
                                t_[i_] == '+' || t_[i_] == '-')) {
        if (!std::isdigit(static_cast<unsigned char>(t_[i_]))) integral = false;
        ++i_;
      }
      const std::string n = t_.substr(b, i_ - b);
      v.type = JValue::kNum;
      v.num = std::strtod(n.c_str(), nullptr);
      if (integral) {
        v.is_uint = true;
        v.u = std::strtoull(n.c_str(), nullptr, 10);
      }
    } else {
      fail("unexpected character");
    }
    return v;
  }
  std::string str() {
    if (i_ >= t_.size() || t_[i_] != '"') fail("expected string");
    ++i_;
    std::string out;
    while (i_ < t_.size() && t_[i_] != '"') {
      char c = t_[i_++];
      if (c == '\\') {
        if (i_ >= t_.size()) fail("bad escape");
        const char e = t_[i_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i_ + 4 > t_.size()) fail("bad unicode escape");
            const unsigned cp = std::strtoul(t_.substr(i_, 4).c_str(), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (i_ >= t_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  const std::string& t_;
  size_t i_ = 0;
};

uint64_t get_uint(const JValue& o, const char* key, uint64_t dflt, const std::string& grp) {
  const JValue* v = o.get(key);
  if (v == nullptr || v->type == JValue::kNull) return dflt;
  if (v->type != JValue::kNum || !v->is_uint)
    throw ConfigError("group '" + grp + "': '" + key + "' must be a non-negative integer");
  return v->u;
}

}  // namespace

// reference model_config.cpp:196-235
ModelSpec parse_model_spec_json(const std::string& text) {
  const JValue j = JParser(text).parse();
  if (j.type != JValue::kObj) throw ConfigError("model config must be a JSON object");
  ModelSpec spec;
  const JValue* name = j.get("name");
  spec.name = (name && name->type == JValue::kStr) ? name->s : "unnamed";
  const JValue* groups = j.get("groups");
  if (groups == nullptr || groups->type != JValue::kArr)
    throw ConfigError("model config missing 'groups' list");
  for (const JValue& gj : groups->arr) {
    if (gj.type != JValue::kObj) throw ConfigError("group must be an object");
    LayerGroupSpec g;
    const JValue* gn = gj.get("name");
    if (gn == nullptr || gn->type != JValue::kStr) throw ConfigError("group missing 'name'");
    g.name = gn->s;
    const JValue* kind = gj.get("kind");
    if (kind == nullptr || kind->type != JValue::kStr)
      throw ConfigError("group '" + g.name + "' missing 'kind'");
    g.kind = layer_kind_from_name(kind->s);
    g.num_layers = static_cast<uint32_t>(get_uint(gj, "num_layers", 0, g.name));
    g.bytes_per_token_per_layer = get_uint(gj, "bytes_per_token_per_layer", 0, g.name);
    g.tokens_per_page = static_cast<uint32_t>(get_uint(gj, "tokens_per_page", 1, g.name));
    g.window_tokens = get_uint(gj, "window_tokens", 0, g.name);
    g.checkpoint_interval_tokens = get_uint(gj, "checkpoint_interval_tokens",
                                            g.kind == LayerKind::kMamba ? 512 : 0, g.name);
    spec.groups.push_back(std::move(g));
  }
  spec.validate();
  return spec;
}

}  // namespace jenga
