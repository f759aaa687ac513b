// C ABI for the host-side pieces: errors, adapter model, page pool and the
// synthetic workload generator.  Each function cites the reference code it
// restates (paths under /root/reference/proj).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include <fstream>
#include <cctype>
#include <iterator>
#include "common.hpp"
#include "pagepool.hpp"
#include "store.hpp"

namespace plora {
namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// adapter.cpp:12-20
static void validate_dims(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp) {
  if (r < 1) throw ValidationError("rank must be >= 1");
  if (r >= std::min(d, k))
    throw ValidationError("rank must be < min(d, k), got r=" + std::to_string(r));
  if (adapted < 1) throw ValidationError("adapted_matrices must be >= 1");
  if (bpp != 1 && bpp != 2 && bpp != 4)
    throw ValidationError("bytes_per_param must be 1, 2 or 4");
}

// adapter.cpp:22-26
static uint64_t param_count(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp) {
  validate_dims(d, k, r, adapted, bpp);
  return static_cast<uint64_t>(adapted) * r * (static_cast<uint64_t>(d) + k);
}

}  // namespace plora

using namespace plora;

// AdapterSizeTable (adapter.hpp:32-47)
struct plora_size_table {
  std::map<uint32_t, uint64_t> table;
  uint32_t anchor_rank = 8;
  uint64_t anchor_bytes = 13ull << 20;
  bool linear_fallback = true;

  uint64_t bytes_for(uint32_t rank) const {  // adapter.cpp:43-50
    auto it = table.find(rank);
    if (it != table.end()) return it->second;
    if (!linear_fallback)
      throw ConfigError("no size configured for rank " + std::to_string(rank) +
                        " and linear fallback is disabled");
    return anchor_bytes * rank / anchor_rank;
  }
};

// ---- catalog JSON (load_catalog_json, adapter.cpp:81-108): a minimal JSON
// reader for the catalog's grammar — an array of objects whose "id" is a
// string and "rank" / "size_bytes" unsigned integers; every other value of
// any JSON type is skipped.  Malformed input is a ParseError, as the
// reference's nlohmann parse failure is.
namespace {

struct CatalogEntry {
  std::string id;
  bool has_id = false, has_rank = false, has_size = false;
  uint64_t rank = 0, size = 0;
};

class JsonReader {
 public:
  JsonReader(const std::string& text, const std::string& path) : s_(text), path_(path) {}
  std::vector<CatalogEntry> catalog() {
    ws();
    if (peek() != '[') throw ParseError("adapter catalog must be a JSON array");
    ++i_;
    std::vector<CatalogEntry> out;
    ws();
    if (peek() == ']') {
      ++i_;
    } else {
      while (true) {
        out.push_back(entry());
        ws();
        const char c = next();
        if (c == ']') break;
        if (c != ',') fail("expected ',' or ']'");
      }
    }
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return out;
  }

 private:
  CatalogEntry entry() {
    ws();
    if (peek() != '{') {  // a non-object entry has no 'id' / 'rank'
      skip_value();
      return CatalogEntry{};
    }
    ++i_;
    CatalogEntry e;
    ws();
    if (peek() == '}') {
      ++i_;
      return e;
    }
    while (true) {
      ws();
      const std::string key = string();
      ws();
      if (next() != ':') fail("expected ':'");
      ws();
      if (key == "id" && peek() == '"') {
        e.id = string();
        e.has_id = true;
      } else if (key == "id") {  // nlohmann's get<std::string> on a non-string
        skip_value();
        throw ParseError("adapter catalog " + path_ + ": catalog entry 'id' must be a string");
      } else if (key == "rank" || key == "size_bytes") {
        const uint64_t v = unsigned_int(key);
        if (key == "rank") {
          if (v > 0xffffffffull) throw ParseError("adapter catalog " + path_ + ": rank out of range");
          e.rank = v;
          e.has_rank = true;
        } else {
          e.size = v;
          e.has_size = true;
        }
      } else {
        skip_value();
      }
      ws();
      const char c = next();
      if (c == '}') break;
      if (c != ',') fail("expected ',' or '}'");
    }
    return e;
  }
  uint64_t unsigned_int(const std::string& key) {
    const std::size_t b = i_;
    if (peek() == '-' || !std::isdigit(static_cast<unsigned char>(peek()))) {
      skip_value();
      throw ParseError("adapter catalog " + path_ + ": '" + key + "' must be an unsigned integer");
    }
    uint64_t v = 0;
    while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) {
      const uint64_t d = static_cast<uint64_t>(s_[i_++] - '0');
      if (v > (~0ull - d) / 10) fail("integer overflow");
      v = v * 10 + d;
    }
    if (i_ < s_.size() && (s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E')) {
      i_ = b;
      skip_value();
      throw ParseError("adapter catalog " + path_ + ": '" + key + "' must be an unsigned integer");
    }
    return v;
  }
  std::string string() {
    if (next() != '"') fail("expected a string");
    std::string out;
    while (true) {
      if (i_ >= s_.size()) fail("unterminated string");
      const char c = s_[i_++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (i_ >= s_.size()) fail("unterminated escape");
      const char e = s_[i_++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {  // BMP code point -> UTF-8 (surrogate pairs combined)
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (i_ + 1 >= s_.size() || s_[i_] != '\\' || s_[i_ + 1] != 'u') fail("lone surrogate");
            i_ += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
          } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          } else if (cp < 0x10000) {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          } else {
            out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  uint32_t hex4() {
    if (i_ + 4 > s_.size()) fail("short \\u escape");
    uint32_t v = 0;
    for (int q = 0; q < 4; ++q) {
      const char c = s_[i_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }
  void skip_value(int depth = 0) {
    if (depth > 512) fail("nesting too deep");
    ws();
    const char c = peek();
    if (c == '"') {
      string();
    } else if (c == '{' || c == '[') {
      const char close = c == '{' ? '}' : ']';
      ++i_;
      ws();
      if (peek() == close) {
        ++i_;
        return;
      }
      while (true) {
        ws();
        if (c == '{') {
          string();
          ws();
          if (next() != ':') fail("expected ':'");
        }
        skip_value(depth + 1);
        ws();
        const char d = next();
        if (d == close) break;
        if (d != ',') fail("expected ','");
      }
    } else if (s_.compare(i_, 4, "true") == 0 || s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else if (s_.compare(i_, 5, "false") == 0) {
      i_ += 5;
    } else if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
      if (c == '-') ++i_;
      if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("bad number");
      while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
      if (peek() == '.') {
        ++i_;
        if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("bad number");
        while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
      }
      if (peek() == 'e' || peek() == 'E') {
        ++i_;
        if (peek() == '+' || peek() == '-') ++i_;
        if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("bad number");
        while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
      }
    } else {
      fail("unexpected character");
    }
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
  }
  char peek() const { return i_ < s_.size() ? s_[i_] : '\0'; }
  char next() {
    if (i_ >= s_.size()) fail("unexpected end of input");
    return s_[i_++];
  }
  [[noreturn]] void fail(const std::string& what) const {
    throw ParseError("adapter catalog " + path_ + ": " + what + " at byte " + std::to_string(i_));
  }
  const std::string& s_;
  std::string path_;
  std::size_t i_ = 0;
};

}  // namespace


extern "C" {

const char* plora_last_error(void) { return plora::g_last_error.c_str(); }
const char* plora_version(void) { return "plora-b200 0.1.0 (sm_100a)"; }
uint64_t plora_kernel_launch_count(void) { return plora::g_launches.load(); }

// ---------------------------------------------------------------- adapter model
int plora_lora_dims_validate(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted,
                             uint32_t bpp) {
  return guard([&] {
    validate_dims(d, k, r, adapted, bpp);
    return 0;
  });
}

int plora_param_count(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp,
                      uint64_t* out) {
  return guard([&] {
    *out = param_count(d, k, r, adapted, bpp);
    return 0;
  });
}

int plora_size_table_create(uint32_t anchor_rank, uint64_t anchor_bytes, int linear_fallback,
                            plora_size_table** out) {
  return guard([&] {
    // adapter.cpp:28-35
    if (anchor_rank == 0 || anchor_bytes == 0)
      throw ConfigError("size table anchor must be positive");
    auto* t = new plora_size_table();
    t->anchor_rank = anchor_rank;
    t->anchor_bytes = anchor_bytes;
    t->linear_fallback = linear_fallback != 0;
    *out = t;
    return 0;
  });
}

void plora_size_table_destroy(plora_size_table* t) { delete t; }

int plora_size_table_set(plora_size_table* t, uint32_t rank, uint64_t bytes) {
  return guard([&] {
    // adapter.cpp:37-40
    if (bytes == 0) throw ConfigError("adapter size must be positive");
    t->table[rank] = bytes;
    return 0;
  });
}

int plora_size_table_bytes_for(const plora_size_table* t, uint32_t rank, uint64_t* out) {
  return guard([&] {
    *out = t->bytes_for(rank);
    return 0;
  });
}

int64_t plora_load_catalog_json(const char* path, const plora_size_table* sizes, uint32_t d,
                                uint32_t k, uint32_t adapted, uint32_t bpp, uint32_t* ranks_out,
                                uint64_t* bytes_out, char* ids_out, uint64_t id_stride,
                                uint64_t cap) {
  int64_t n = 0;
  const int rc = guard([&] {  // load_catalog_json, adapter.cpp:81-108
    if (!path) throw ValidationError("null path");
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ConfigError(std::string("cannot open adapter catalog: ") + path);
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const std::vector<CatalogEntry> cat = JsonReader(text, path).catalog();
    plora_size_table def;
    const plora_size_table& st = sizes ? *sizes : def;
    std::vector<std::pair<uint32_t, uint64_t>> out;
    for (const CatalogEntry& e : cat) {
      if (!e.has_id || !e.has_rank) throw ParseError("catalog entry needs 'id' and 'rank'");
      const uint32_t r = static_cast<uint32_t>(e.rank);
      const uint64_t bytes = e.has_size ? e.size : st.bytes_for(r);
      // AdapterSpec::sized -> validate (adapter.cpp:61-79)
      validate_dims(d, k, r, adapted, bpp);
      if (bytes == 0) throw ValidationError("adapter weight_bytes must be > 0");
      out.emplace_back(r, bytes);
    }
    if (out.empty()) throw ValidationError("adapter catalog is empty");
    for (uint64_t i = 0; i < out.size() && i < cap; ++i) {
      if (ranks_out) ranks_out[i] = out[i].first;
      if (bytes_out) bytes_out[i] = out[i].second;
      if (ids_out && id_stride) {
        const std::string& id = cat[i].id;
        const uint64_t m = std::min<uint64_t>(id.size(), id_stride - 1);
        std::memcpy(ids_out + i * id_stride, id.data(), m);
        ids_out[i * id_stride + m] = '\0';
      }
    }
    n = static_cast<int64_t>(out.size());
    return 0;
  });
  return rc < 0 ? rc : n;
}

int plora_generate_catalog(uint32_t count, const uint32_t* mix_ranks, const double* mix_weights,
                           uint64_t n_mix, uint64_t seed, const plora_size_table* sizes,
                           uint32_t d, uint32_t k, uint32_t adapted, uint32_t bpp,
                           uint32_t* ranks_out, uint64_t* bytes_out) {
  return guard([&] {
    // adapter.cpp:110-144 (ids are the dense index; the zero-padded string id
    // "a%0*u" is derivable by the caller)
    if (count == 0) throw ValidationError("catalog count must be >= 1");
    if (n_mix == 0) throw ConfigError("rank mix is empty");
    std::vector<double> weights;
    for (uint64_t i = 0; i < n_mix; ++i) {
      if (mix_weights[i] < 0) throw ConfigError("rank mix weights must be nonnegative");
      weights.push_back(mix_weights[i]);
    }
    plora_size_table def;
    const plora_size_table& st = sizes ? *sizes : def;
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
    std::discrete_distribution<std::size_t> pick(weights.begin(), weights.end());
    for (uint32_t i = 0; i < count; ++i) {
      uint32_t r = mix_ranks[pick(rng)];
      validate_dims(d, k, r, adapted, bpp);  // AdapterSpec::sized -> validate
      uint64_t b = st.bytes_for(r);
      if (b == 0) throw ValidationError("adapter weight_bytes must be > 0");
      ranks_out[i] = r;
      bytes_out[i] = b;
    }
    return 0;
  });
}

// ------------------------------------------------------------------- page pool
int plora_pool_create(uint64_t page_bytes, uint32_t total_pages, plora_pool** out) {
  return guard([&] {
    *out = new plora_pool{PagePool(page_bytes, total_pages), {}};
    return 0;
  });
}

void plora_pool_destroy(plora_pool* p) { delete p; }

uint32_t plora_pool_pages_needed(const plora_pool* p, uint64_t bytes) {
  return p->pool.pages_needed(bytes);
}

int plora_pool_alloc(plora_pool* p, uint32_t adapter, uint64_t weight_bytes) {
  return guard([&] { return static_cast<int>(p->pool.alloc(adapter, weight_bytes)); });
}

int plora_pool_free(plora_pool* p, uint32_t adapter) {
  return guard([&] {
    p->pool.free(adapter);
    return 0;
  });
}

int plora_pool_translate(const plora_pool* p, uint32_t adapter, uint32_t logical,
                         uint32_t* phys) {
  return guard([&] {
    *phys = p->pool.translate(adapter, logical);
    return 0;
  });
}

int plora_pool_table(const plora_pool* p, uint32_t adapter, const uint32_t** entries,
                     uint32_t* n_entries, uint64_t* weight_bytes) {
  return guard([&] {
    const PageTable& t = p->pool.table(adapter);
    if (entries) *entries = t.entries.data();
    if (n_entries) *n_entries = static_cast<uint32_t>(t.entries.size());
    if (weight_bytes) *weight_bytes = t.weight_bytes;
    return 0;
  });
}

int plora_pool_has(const plora_pool* p, uint32_t adapter) { return p->pool.has(adapter) ? 1 : 0; }

int plora_pool_compact(plora_pool* p, uint64_t* moved) {
  return guard([&] {
    uint64_t m = p->pool.compact();
    if (moved) *moved = m;
    return 0;
  });
}

int plora_pool_last_relocations(const plora_pool* p, const plora_reloc** relocs, uint64_t* n) {
  const auto& r = p->pool.last_relocations();
  if (relocs) *relocs = r.data();
  if (n) *n = r.size();
  return 0;
}

void plora_pool_report(const plora_pool* p, plora_frag_report* out) {
  FragmentationReport r = p->pool.report();
  out->external_frag = r.external_frag;
  out->internal_frag = r.internal_frag;
  out->utilization = r.utilization;
}

uint32_t plora_pool_free_pages(const plora_pool* p) { return p->pool.free_pages(); }
uint32_t plora_pool_total_pages(const plora_pool* p) { return p->pool.total_pages(); }
uint64_t plora_pool_page_bytes(const plora_pool* p) { return p->pool.page_bytes(); }
uint64_t plora_pool_used_bytes(const plora_pool* p) { return p->pool.used_bytes(); }
uint64_t plora_pool_allocated_bytes(const plora_pool* p) { return p->pool.allocated_bytes(); }
uint64_t plora_pool_total_bytes(const plora_pool* p) { return p->pool.total_bytes(); }

uint64_t plora_pool_resident(const plora_pool* p, uint32_t* out, uint64_t cap) {
  auto r = p->pool.resident();
  for (uint64_t i = 0; i < r.size() && i < cap; ++i) out[i] = r[i];
  return r.size();
}

int plora_pool_check_invariants(const plora_pool* p) {
  return guard([&] {
    p->pool.check_invariants();
    return 0;
  });
}

int plora_pool_dump(const plora_pool* p, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    std::string s = p->pool.dump();
    if (len) *len = s.size();
    if (buf && cap) {
      uint64_t n = std::min<uint64_t>(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
    return 0;
  });
}

// ------------------------------------------------------------ synthetic workload
void plora_synthetic_profile_default(plora_synthetic_profile* p) {
  // workload.hpp:19-50 member initializers
  p->num_adapters = 20;
  p->base_rate = 50.0;
  p->diurnal_amplitude = 0.0;
  p->period_s = 3600.0;
  p->hot_set_size = 5;
  p->hot_rotation_s = 7.0;
  p->hot_share = 0.9;
  p->rotation_jitter = 0.0;
  p->burstiness_cv = 1.0;
  p->input_median = 256.0;
  p->input_sigma = 0.6;
  p->output_median = 128.0;
  p->output_sigma = 0.6;
  p->max_tokens = 8192;
}

namespace {
// workload.cpp:26-31
uint32_t clamp_tokens(double v, uint32_t max_tokens) {
  if (!(v >= 1.0)) return 1;
  if (v > max_tokens) return max_tokens;
  return static_cast<uint32_t>(std::llround(v));
}
}  // namespace

int64_t plora_generate_synthetic(const plora_synthetic_profile* pp, double duration_s,
                                 uint64_t seed, double* arrival_ms, uint32_t* adapter,
                                 uint32_t* input_tokens, uint32_t* output_tokens, uint64_t cap) {
  int64_t count = 0;
  int rc = guard([&] {
    const plora_synthetic_profile& p = *pp;
    // SyntheticProfile::validate (workload.cpp:45-57)
    if (p.num_adapters < 1) throw ValidationError("num_adapters must be >= 1");
    if (p.base_rate <= 0) throw ValidationError("base_rate must be positive");
    if (p.diurnal_amplitude < 0 || p.diurnal_amplitude > 1)
      throw ValidationError("diurnal_amplitude must be in [0, 1]");
    if (p.period_s <= 0) throw ValidationError("period must be positive");
    if (p.hot_set_size < 1 || p.hot_set_size > p.num_adapters)
      throw ValidationError("hot_set_size must be in [1, num_adapters]");
    if (p.hot_rotation_s <= 0) throw ValidationError("hot_rotation_s must be positive");
    if (p.hot_share < 0 || p.hot_share > 1) throw ValidationError("hot_share must be in [0, 1]");
    if (p.rotation_jitter < 0 || p.rotation_jitter >= 1)
      throw ValidationError("rotation_jitter must be in [0, 1)");
    if (p.burstiness_cv <= 0) throw ValidationError("burstiness_cv must be positive");
    if (duration_s <= 0) throw ValidationError("duration must be positive");

    // workload.cpp:59-144
    constexpr double kPi = 3.14159265358979323846;
    std::mt19937_64 rng(seed);
    const uint32_t num_groups = (p.num_adapters + p.hot_set_size - 1) / p.hot_set_size;
    std::vector<double> rotation_ends;
    {
      std::uniform_real_distribution<double> u(-1.0, 1.0);
      double t = 0.0;
      while (t < duration_s) {
        double len = p.hot_rotation_s;
        if (p.rotation_jitter > 0) len *= 1.0 + p.rotation_jitter * u(rng);
        t += std::max(len, 1e-3);
        rotation_ends.push_back(t);
      }
    }
    auto group_at = [&](double t_s) -> uint32_t {
      auto it = std::upper_bound(rotation_ends.begin(), rotation_ends.end(), t_s);
      return static_cast<uint32_t>(it - rotation_ends.begin()) % num_groups;
    };
    const double rate_max = p.base_rate * (1.0 + p.diurnal_amplitude);
    auto rate_at = [&](double t_s) {
      return p.base_rate * (1.0 + p.diurnal_amplitude * std::sin(2.0 * kPi * t_s / p.period_s));
    };
    const double shape = 1.0 / (p.burstiness_cv * p.burstiness_cv);
    std::gamma_distribution<double> gap(shape, 1.0 / (rate_max * shape));
    std::uniform_real_distribution<double> accept(0.0, 1.0);
    std::uniform_int_distribution<uint32_t> hot_pick(0, p.hot_set_size - 1);
    auto sample_len = [&](double median, double sigma) {  // workload.cpp:33-43
      std::normal_distribution<double> n(std::log(median), sigma);
      return clamp_tokens(std::exp(n(rng)), p.max_tokens);
    };
    double t = 0.0;
    while (true) {
      t += gap(rng);
      if (t >= duration_s) break;
      if (accept(rng) > rate_at(t) / rate_max) continue;
      uint32_t g = group_at(t);
      uint32_t idx;
      if (accept(rng) < p.hot_share) {
        idx = (g * p.hot_set_size + hot_pick(rng)) % p.num_adapters;
      } else {
        uint32_t cold = p.num_adapters - p.hot_set_size;
        if (cold == 0) {
          idx = (g * p.hot_set_size + hot_pick(rng)) % p.num_adapters;
        } else {
          std::uniform_int_distribution<uint32_t> cold_pick(0, cold - 1);
          uint32_t o = cold_pick(rng);
          uint32_t hot_base = (g * p.hot_set_size) % p.num_adapters;
          idx = (hot_base + p.hot_set_size + o) % p.num_adapters;
        }
      }
      uint32_t in = sample_len(p.input_median, p.input_sigma);
      uint32_t out = sample_len(p.output_median, p.output_sigma);
      if (static_cast<uint64_t>(count) < cap) {
        arrival_ms[count] = t * 1000.0;
        adapter[count] = idx;
        input_tokens[count] = in;
        output_tokens[count] = out;
      }
      ++count;
    }
    return 0;
  });
  return rc ? rc : count;
}

}  // extern "C"
