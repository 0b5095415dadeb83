// The reference's host-side run surface above the device step, in C++:
//
//   deck format      parse_deck / serialize_deck / apply_override / make_grid
//                    (proj/src/deck.cpp:20-395, proj/include/minipic/sim.hpp:23-88)
//   SimState         initialize / step / run / emit_diagnostics
//                    (proj/src/sim.cpp:25-47, 74-134, 143-183, 217-306)
//   particle load    Rng = std::mt19937_64 + the reference's uniform and
//                    Box-Muller mappings (proj/include/minipic/rng.hpp:17-51),
//                    so the initial state is bit-identical to the reference's
//   field dumps      dump_fields, binary form (proj/src/fields.cpp:315-344)
//
// The device work goes through the same launchers the C-ABI exposes; this
// file only sequences them the way SimState does.  Keys that select CPU
// strategies (run.workers, layout, scatter_backend, chunk_size, kernel) are
// parsed and validated like the reference and have no device effect.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "pic_internal.hpp"

namespace picb {

// ---- deck -----------------------------------------------------------------
struct DeckSpecies {
  std::string name;
  float q = 0, m = 1;
  int ppc = 0;
  float u_th = 0;
  float drift[3] = {0, 0, 0};
  int sort_interval = 20;
  int sort_order = PIC_SORT_BLOCKED;
  float perturb_ux = 0;
  int perturb_kmode = 1;
};

struct Deck {
  // [grid]
  int nx = 0, ny = 0, nz = 0;
  float lx = 0, ly = 0, lz = 0;
  std::optional<float> dt;
  float cfl_fraction = 0.95f;
  long steps = 0;
  std::vector<DeckSpecies> species;
  // [run]
  uint64_t seed = 1;
  std::string layout = "field_major", scatter_backend = "replicated", kernel = "auto";
  int workers = 1;
  size_t chunk_size = 2048;
  bool deterministic = false, exact_gyration = false;
  long diag_interval = 10, field_dump_interval = 0;
  std::string out_dir = "out";
};

namespace {

[[noreturn]] void bad_key(const std::string& key, int line, const std::string& why) {
  throw DeckParseError("deck: key '" + key + "' (line " + std::to_string(line) + "): " + why);
}

std::string strip(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && (s[b] == ' ' || s[b] == '\t' || s[b] == '\r')) ++b;
  while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\t' || s[e - 1] == '\r')) --e;
  return s.substr(b, e - b);
}

// number conversions with the reference's acceptance rules (whole token
// consumed, std::stod / std::stol semantics)
double as_real(const std::string& key, int line, const std::string& v) {
  size_t used = 0;
  double d = 0;
  try {
    d = std::stod(v, &used);
  } catch (...) {
    bad_key(key, line, "not a number: '" + v + "'");
  }
  if (used != v.size()) bad_key(key, line, "trailing characters in '" + v + "'");
  return d;
}
long as_int(const std::string& key, int line, const std::string& v) {
  size_t used = 0;
  long d = 0;
  try {
    d = std::stol(v, &used);
  } catch (...) {
    bad_key(key, line, "not an integer: '" + v + "'");
  }
  if (used != v.size()) bad_key(key, line, "trailing characters in '" + v + "'");
  return d;
}
bool as_bool(const std::string& key, int line, const std::string& v) {
  for (const char* t : {"true", "1", "on"})
    if (v == t) return true;
  for (const char* f : {"false", "0", "off"})
    if (v == f) return false;
  bad_key(key, line, "not a boolean: '" + v + "'");
}
std::string as_choice(const std::string& key, int line, const std::string& v,
                      std::initializer_list<const char*> allowed) {
  std::string msg = "expected ";
  bool first = true;
  for (const char* a : allowed) {
    if (v == a) return v;
    msg += (first ? "" : "|") + std::string(a);
    first = false;
  }
  bad_key(key, line, msg);
}

using Setter = std::function<void(const std::string& full, int line, const std::string& v)>;

void set_grid(Deck& d, const std::string& key, const std::string& v, int line) {
  const std::map<std::string, Setter> keys = {
      {"nx", [&](auto& k, int l, auto& x) { d.nx = (int)as_int(k, l, x); }},
      {"ny", [&](auto& k, int l, auto& x) { d.ny = (int)as_int(k, l, x); }},
      {"nz", [&](auto& k, int l, auto& x) { d.nz = (int)as_int(k, l, x); }},
      {"lx", [&](auto& k, int l, auto& x) { d.lx = (float)as_real(k, l, x); }},
      {"ly", [&](auto& k, int l, auto& x) { d.ly = (float)as_real(k, l, x); }},
      {"lz", [&](auto& k, int l, auto& x) { d.lz = (float)as_real(k, l, x); }},
      {"dt", [&](auto& k, int l, auto& x) { d.dt = (float)as_real(k, l, x); }},
      {"cfl_fraction", [&](auto& k, int l, auto& x) { d.cfl_fraction = (float)as_real(k, l, x); }},
      {"steps", [&](auto& k, int l, auto& x) { d.steps = as_int(k, l, x); }},
  };
  const auto it = keys.find(key);
  if (it == keys.end()) bad_key("grid." + key, line, "unknown key");
  it->second(key, line, v);
}

void set_species(DeckSpecies& s, const std::string& key, const std::string& v, int line) {
  const std::string full = "species." + s.name + "." + key;
  const std::map<std::string, Setter> keys = {
      {"q", [&](auto& k, int l, auto& x) { s.q = (float)as_real(k, l, x); }},
      {"m", [&](auto& k, int l, auto& x) { s.m = (float)as_real(k, l, x); }},
      {"ppc", [&](auto& k, int l, auto& x) { s.ppc = (int)as_int(k, l, x); }},
      {"u_th", [&](auto& k, int l, auto& x) { s.u_th = (float)as_real(k, l, x); }},
      {"drift",
       [&](auto& k, int l, auto& x) {
         std::istringstream in(x);
         std::string a[3], extra;
         if (!(in >> a[0] >> a[1] >> a[2]) || (in >> extra)) bad_key(k, l, "expected three numbers, got '" + x + "'");
         for (int i = 0; i < 3; ++i) s.drift[i] = (float)as_real(k, l, a[i]);
       }},
      {"sort_interval", [&](auto& k, int l, auto& x) { s.sort_interval = (int)as_int(k, l, x); }},
      {"sort_order",
       [&](auto& k, int l, auto& x) {
         s.sort_order = as_choice(k, l, x, {"blocked", "interleaved"}) == "blocked" ? PIC_SORT_BLOCKED
                                                                                   : PIC_SORT_INTERLEAVED;
       }},
      {"perturb_ux", [&](auto& k, int l, auto& x) { s.perturb_ux = (float)as_real(k, l, x); }},
      {"perturb_kmode", [&](auto& k, int l, auto& x) { s.perturb_kmode = (int)as_int(k, l, x); }},
  };
  const auto it = keys.find(key);
  if (it == keys.end()) bad_key(full, line, "unknown key");
  it->second(full, line, v);
}

void set_run(Deck& d, const std::string& key, const std::string& v, int line) {
  const std::string full = "run." + key;
  const std::map<std::string, Setter> keys = {
      {"seed", [&](auto& k, int l, auto& x) { d.seed = (uint64_t)as_int(k, l, x); }},
      {"layout", [&](auto& k, int l, auto& x) { d.layout = as_choice(k, l, x, {"record_major", "field_major"}); }},
      {"scatter_backend",
       [&](auto& k, int l, auto& x) {
         d.scatter_backend = as_choice(k, l, x, {"replicated", "shared_update", "sequential"});
       }},
      {"workers", [&](auto& k, int l, auto& x) { d.workers = (int)as_int(k, l, x); }},
      {"chunk_size", [&](auto& k, int l, auto& x) { d.chunk_size = (size_t)as_int(k, l, x); }},
      {"deterministic", [&](auto& k, int l, auto& x) { d.deterministic = as_bool(k, l, x); }},
      {"diag_interval", [&](auto& k, int l, auto& x) { d.diag_interval = as_int(k, l, x); }},
      {"field_dump_interval", [&](auto& k, int l, auto& x) { d.field_dump_interval = as_int(k, l, x); }},
      {"out_dir", [&](auto&, int, auto& x) { d.out_dir = x; }},
      {"exact_gyration", [&](auto& k, int l, auto& x) { d.exact_gyration = as_bool(k, l, x); }},
      {"kernel", [&](auto& k, int l, auto& x) { d.kernel = as_choice(k, l, x, {"auto", "scalar", "simd"}); }},
  };
  const auto it = keys.find(key);
  if (it == keys.end()) bad_key(full, line, "unknown key");
  it->second(full, line, v);
}

// validate_grid / cfl_limit (proj/src/grid.cpp:7-20) on the resolved grid
float cfl_limit(float hx, float hy, float hz) {
  const float s = 1.0f / (hx * hx) + 1.0f / (hy * hy) + 1.0f / (hz * hz);
  return 1.0f / std::sqrt(s);
}

}  // namespace

pic_grid deck_grid(const Deck& d) {
  pic_grid g{};
  g.nx = d.nx;
  g.ny = d.ny;
  g.nz = d.nz;
  g.hx = d.lx / (float)d.nx;
  g.hy = d.ly / (float)d.ny;
  g.hz = d.lz / (float)d.nz;
  g.dt = d.dt ? *d.dt : d.cfl_fraction * cfl_limit(g.hx, g.hy, g.hz);
  return g;
}

static void deck_check(const Deck& d) {
  auto fail = [](const std::string& m) { throw DeckParseError("deck: " + m); };
  if (d.nx < 2 || d.ny < 2 || d.nz < 2) fail("grid.nx/ny/nz must be >= 2");
  if (!(d.lx > 0) || !(d.ly > 0) || !(d.lz > 0)) fail("grid.lx/ly/lz must be positive");
  if (d.steps < 0) fail("grid.steps must be >= 0");
  if (!(d.cfl_fraction > 0) || d.cfl_fraction > 0.99f) fail("grid.cfl_fraction must be in (0, 0.99]");
  if (d.species.empty()) fail("at least one [species.NAME] block required");
  for (const auto& s : d.species) {
    const std::string p = "species." + s.name + ".";
    if (!(s.m > 0)) fail(p + "m must be positive");
    if (s.ppc < 0) fail(p + "ppc must be >= 0");
    if (s.u_th < 0) fail(p + "u_th must be >= 0");
    if (s.sort_interval < 0) fail(p + "sort_interval must be >= 0");
    if (s.perturb_kmode < 1) fail(p + "perturb_kmode must be >= 1");
  }
  if (d.workers < 1) fail("run.workers must be >= 1");
  if (d.chunk_size < 1) fail("run.chunk_size must be >= 1");
  if (d.diag_interval < 1) fail("run.diag_interval must be >= 1");
  if (d.field_dump_interval < 0) fail("run.field_dump_interval must be >= 0");
  const pic_grid g = deck_grid(d);
  std::string why;
  if (!(g.hx > 0) || !(g.hy > 0) || !(g.hz > 0))
    why = "grid: spacings must be positive";
  else if (!(g.dt > 0) || g.dt > 0.99f * cfl_limit(g.hx, g.hy, g.hz))
    why = "grid: dt must satisfy 0 < dt <= 0.99 * cfl_limit";
  if (!why.empty()) fail("grid.dt: " + why);
}

Deck parse_deck(const std::string& text) {
  Deck d;
  enum { kNone, kGrid, kSpecies, kRun } where = kNone;
  bool have_grid = false, have_run = false;
  std::vector<std::string> grid_keys;
  std::vector<std::vector<std::string>> species_keys;
  std::istringstream in(text);
  std::string raw;
  for (int line = 1; std::getline(in, raw); ++line) {
    const std::string s = strip(raw.substr(0, raw.find('#')));
    if (s.empty()) continue;
    const std::string at = " (line " + std::to_string(line) + ")";
    if (s[0] == '[') {
      if (s.back() != ']') throw DeckParseError("deck: malformed section header" + at);
      const std::string name = strip(s.substr(1, s.size() - 2));
      if (name == "grid" || name == "run") {
        bool& seen = name == "grid" ? have_grid : have_run;
        if (seen) throw DeckParseError("deck: duplicate [" + name + "] section" + at);
        seen = true;
        where = name == "grid" ? kGrid : kRun;
      } else if (name.compare(0, 8, "species.") == 0) {
        DeckSpecies sp;
        sp.name = name.substr(8);
        if (sp.name.empty()) throw DeckParseError("deck: species section needs a name" + at);
        for (const auto& o : d.species)
          if (o.name == sp.name) throw DeckParseError("deck: duplicate species '" + sp.name + "'" + at);
        d.species.push_back(sp);
        species_keys.emplace_back();
        where = kSpecies;
      } else {
        throw DeckParseError("deck: unknown section '" + name + "'" + at);
      }
      continue;
    }
    const size_t eq = s.find('=');
    if (eq == std::string::npos) throw DeckParseError("deck: expected key = value" + at);
    const std::string key = strip(s.substr(0, eq)), value = strip(s.substr(eq + 1));
    if (key.empty()) bad_key("?", line, "empty key");
    if (value.empty()) bad_key(key, line, "empty value");
    switch (where) {
      case kNone:
        throw DeckParseError("deck: key '" + key + "' outside any section" + at);
      case kGrid:
        set_grid(d, key, value, line);
        grid_keys.push_back(key);
        break;
      case kSpecies:
        set_species(d.species.back(), key, value, line);
        species_keys.back().push_back(key);
        break;
      case kRun:
        set_run(d, key, value, line);
        break;
    }
  }
  auto has = [](const std::vector<std::string>& v, const char* k) {
    for (const auto& x : v)
      if (x == k) return true;
    return false;
  };
  if (!have_grid) throw DeckParseError("deck: missing [grid] section");
  for (const char* k : {"nx", "ny", "nz", "lx", "ly", "lz", "steps"})
    if (!has(grid_keys, k)) throw DeckParseError(std::string("deck: missing required key grid.") + k);
  for (size_t i = 0; i < d.species.size(); ++i)
    for (const char* k : {"q", "m", "ppc"})
      if (!has(species_keys[i], k))
        throw DeckParseError("deck: missing required key species." + d.species[i].name + "." + k);
  deck_check(d);
  return d;
}

static std::string real_text(float v) {  // fmt_real: %.9g for fp32 (proj/src/sim.cpp:27-32)
  char b[48];
  std::snprintf(b, sizeof b, "%.9g", (double)v);
  return b;
}
static std::string double_text(double v) {
  char b[48];
  std::snprintf(b, sizeof b, "%.9g", v);
  return b;
}

std::string serialize_deck(const Deck& d) {
  std::ostringstream o;
  o << "[grid]\nnx = " << d.nx << "\nny = " << d.ny << "\nnz = " << d.nz << "\n";
  o << "lx = " << real_text(d.lx) << "\nly = " << real_text(d.ly) << "\nlz = " << real_text(d.lz) << "\n";
  if (d.dt)
    o << "dt = " << real_text(*d.dt) << "\n";
  else
    o << "cfl_fraction = " << real_text(d.cfl_fraction) << "\n";
  o << "steps = " << d.steps << "\n";
  for (const auto& s : d.species) {
    o << "\n[species." << s.name << "]\nq = " << real_text(s.q) << "\nm = " << real_text(s.m)
      << "\nppc = " << s.ppc << "\nu_th = " << real_text(s.u_th) << "\ndrift = " << real_text(s.drift[0]) << ' '
      << real_text(s.drift[1]) << ' ' << real_text(s.drift[2]) << "\nsort_interval = " << s.sort_interval
      << "\nsort_order = " << (s.sort_order == PIC_SORT_BLOCKED ? "blocked" : "interleaved") << "\n";
    if (s.perturb_ux != 0)
      o << "perturb_ux = " << real_text(s.perturb_ux) << "\nperturb_kmode = " << s.perturb_kmode << "\n";
  }
  o << "\n[run]\nseed = " << d.seed << "\nlayout = " << d.layout << "\nscatter_backend = " << d.scatter_backend
    << "\nworkers = " << d.workers << "\nchunk_size = " << d.chunk_size
    << "\ndeterministic = " << (d.deterministic ? "true" : "false") << "\ndiag_interval = " << d.diag_interval
    << "\nfield_dump_interval = " << d.field_dump_interval << "\nout_dir = " << d.out_dir
    << "\nexact_gyration = " << (d.exact_gyration ? "true" : "false") << "\nkernel = " << d.kernel << "\n";
  return o.str();
}

void apply_override(Deck& d, const std::string& kv) {
  const size_t eq = kv.find('=');
  if (eq == std::string::npos) throw DeckParseError("override: expected key=value, got '" + kv + "'");
  const std::string path = strip(kv.substr(0, eq)), value = strip(kv.substr(eq + 1));
  const size_t dot = path.find('.');
  if (dot == std::string::npos) throw DeckParseError("override: key '" + path + "' must be section.key");
  const std::string section = path.substr(0, dot), rest = path.substr(dot + 1);
  if (section == "grid") {
    set_grid(d, rest, value, 0);
  } else if (section == "run") {
    set_run(d, rest, value, 0);
  } else if (section == "species") {
    const size_t dot2 = rest.find('.');
    if (dot2 == std::string::npos) throw DeckParseError("override: species key must be species.NAME.key");
    const std::string name = rest.substr(0, dot2);
    DeckSpecies* sp = nullptr;
    for (auto& s : d.species)
      if (s.name == name) sp = &s;
    if (!sp) throw DeckParseError("override: no species named '" + name + "'");
    set_species(*sp, rest.substr(dot2 + 1), value, 0);
  } else {
    throw DeckParseError("override: unknown section '" + section + "'");
  }
  deck_check(d);
}

// ---- SimState --------------------------------------------------------------
namespace {

// Rng (proj/include/minipic/rng.hpp:17-51): the standard-fixed engine and
// the reference's own mappings.
class LoadRng {
 public:
  explicit LoadRng(uint64_t seed) : e_(seed) {}
  double uniform() { return (double)(e_() >> 11) * 0x1.0p-53; }
  double uniform_pm1() { return 2.0 * uniform() - 1.0; }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double a = uniform(), b = uniform();
    while (a == 0.0) a = uniform();
    const double r = std::sqrt(-2.0 * std::log(a)), t = 2.0 * 3.14159265358979323846 * b;
    spare_ = r * std::sin(t);
    spare_ok_ = true;
    return r * std::cos(t);
  }

 private:
  std::mt19937_64 e_;
  double spare_ = 0.0;
  bool spare_ok_ = false;
};

}  // namespace

struct Sim {
  Deck deck;
  pic_grid grid{};
  Context* ctx = nullptr;
  long step_count = 0;
  std::vector<std::string> warnings;
  // hooks (sim.hpp:102-127) and their host mirrors (allocated on first use)
  struct Hook {
    std::string name;
    long interval;
    pic_hook_flags flags;
    pic_hook_fn fn;
    void* user;
  };
  std::vector<Hook> hooks;
  std::vector<float> host_fields;
  std::vector<std::vector<float>> host_lanes;
  std::vector<std::vector<int32_t>> host_ids;
  uint64_t copies = 0;
  pic_sim* handle = nullptr;
  bool header_done = false;
  std::chrono::steady_clock::time_point last_wall;
  long last_step = 0;

  unsigned flags() const {
    return (deck.deterministic ? PIC_DETERMINISTIC : 0u) | (deck.exact_gyration ? PIC_EXACT_GYRATION : 0u);
  }
  std::string kept_row;  // pic_sim_emit_diagnostics: computed by a size query, returned by the fill
  bool row_kept = false;

  size_t total_particles() const {
    size_t n = 0;
    for (const auto& s : ctx->species) n += s.n;
    return n;
  }

  // SimState::initialize (proj/src/sim.cpp:74-134)
  Sim(int device, const Deck& d) : deck(d), grid(deck_grid(d)) {
    ctx = make_context(device, grid);
    // deterministic decks: energies in the reference's fp32 summation order,
    // so the diagnostics CSV is the reference's byte for byte
    ctx->reference_order_sums = deck.deterministic;
    try {
      const size_t interior = (size_t)grid.nx * grid.ny * grid.nz;
      const float hx = grid.hx, lx = grid.hx * (float)grid.nx;
      for (size_t si = 0; si < deck.species.size(); ++si) {
        const DeckSpecies& ds = deck.species[si];
        const size_t n = (size_t)ds.ppc * interior;
        Species sp;
        sp.name = ds.name;
        sp.q = ds.q;
        sp.m = ds.m;
        sp.cap = n;
        const size_t cap = n ? n : 1;
        CUDA_OK(cudaMalloc(&sp.pos, cap * sizeof(float4)));
        CUDA_OK(cudaMalloc(&sp.mom, cap * sizeof(float4)));
        ctx->species.push_back(sp);
        // host load in the reference's order (iz, iy, ix, k), one engine per species
        std::vector<float> lanes(7 * n);
        std::vector<int32_t> ids(n);
        LoadRng rng(deck.seed + 0x9e3779b9u * (si + 1));
        const float kx = (float)(2.0 * 3.14159265358979323846 * ds.perturb_kmode);
        size_t p = 0;
        for (int iz = 1; iz <= grid.nz; ++iz)
          for (int iy = 1; iy <= grid.ny; ++iy)
            for (int ix = 1; ix <= grid.nx; ++ix) {
              const int v = ix + (grid.nx + 2) * (iy + (grid.ny + 2) * iz);
              for (int k = 0; k < ds.ppc; ++k, ++p) {
                const float dx = (float)rng.uniform_pm1(), dy = (float)rng.uniform_pm1(),
                            dz = (float)rng.uniform_pm1();
                float ux = ds.drift[0] + ds.u_th * (float)rng.normal();
                const float uy = ds.drift[1] + ds.u_th * (float)rng.normal();
                const float uz = ds.drift[2] + ds.u_th * (float)rng.normal();
                if (ds.perturb_ux != 0) {
                  const float xg = ((float)(ix - 1) + (dx + 1) * 0.5f) * hx;
                  ux += ds.perturb_ux * std::sin(kx * xg / lx);
                }
                const float rec[7] = {dx, dy, dz, ux, uy, uz, 1.0f};
                for (int l = 0; l < 7; ++l) lanes[(size_t)l * n + p] = rec[l];
                ids[p] = v;
              }
            }
        Species& s = ctx->species.back();
        s.n = n;
        if (n) {
          char* stg = static_cast<char*>(ctx->scratch_bytes(Context::kScrStaging, n * 32));
          CUDA_OK(cudaMemcpyAsync(stg, lanes.data(), n * 28, cudaMemcpyHostToDevice, ctx->stream));
          CUDA_OK(cudaMemcpyAsync(stg + n * 28, ids.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
          launch_pack_species(*ctx, s, reinterpret_cast<float*>(stg), reinterpret_cast<int32_t*>(stg + n * 28), n);
          CUDA_OK(cudaStreamSynchronize(ctx->stream));
        }
      }
      // zero-E start is Gauss-consistent only for neutral decks (sim.cpp:114-126)
      float total = 0, absq = 0;
      for (const auto& s : ctx->species) {
        total += s.q * (float)s.n;
        absq += std::fabs(s.q) * (float)s.n;
      }
      if (std::fabs(total) > 1e-12f * (absq + 1.0f))
        warnings.push_back(
            "non-neutral deck with zero-E initialization: the Gauss residual starts nonzero and should stay "
            "constant");
      launch_ghost_sync(*ctx);
      refresh_charge();
      quiesce(*ctx);
    } catch (...) {
      destroy_context(ctx);
      throw;
    }
    last_wall = std::chrono::steady_clock::now();
  }
  ~Sim() { destroy_context(ctx); }

  void refresh_charge() {  // SimState::refresh_charge_diagnostics (sim.cpp:230-234)
    launch_clear_rho(*ctx);
    materialize_for_sums(*ctx);
    for (auto& s : ctx->species) launch_deposit_rho(*ctx, s);
    launch_compute_div_errors(*ctx);
  }

  void do_step() {  // SimState::step (sim.cpp:143-183), replayed as CUDA graphs where it can be
    step_graphed(*ctx, flags());
    ++step_count;
  }

  void sort_due() {  // SimState::sort_due_species (sim.cpp:217-222)
    for (size_t i = 0; i < ctx->species.size(); ++i) {
      const DeckSpecies& ds = deck.species[i];
      if (ds.sort_interval > 0 && step_count % ds.sort_interval == 0) sort_species(*ctx, ctx->species[i], ds.sort_order);
    }
  }

  // SimState::emit_diagnostics (sim.cpp:267-283) with current_diagnostics
  // (sim.cpp:236-266): header on first use, one row.
  std::string diagnostics_row() {
    quiesce(*ctx);
    std::string out;
    if (!header_done) {
      out += "step,time,e_energy,b_energy";
      for (const auto& s : deck.species) out += ",kinetic_" + s.name;
      out += ",total_energy,max_div_e_err,max_div_b_err,particle_count,wall_seconds_this_interval,push_rate\n";
      header_done = true;
    }
    float eb[2], mdiv[2];
    std::vector<float> kin(ctx->species.size());
    diagnostics_batch(*ctx, eb, kin.data(), mdiv);
    float total = eb[0] + eb[1];
    for (float k : kin) total += k;
    const float mde = mdiv[0], mdb = mdiv[1];
    const auto now = std::chrono::steady_clock::now();
    double wall = std::chrono::duration<double>(now - last_wall).count();
    const long dsteps = step_count - last_step;
    double rate = wall > 0 ? (double)total_particles() * (double)dsteps / wall : 0;
    if (deck.deterministic) wall = rate = 0;  // byte-identical reruns (sim.cpp:254-257)
    last_wall = now;
    last_step = step_count;
    out += std::to_string(step_count) + "," + real_text((float)step_count * grid.dt) + "," + real_text(eb[0]) + "," +
           real_text(eb[1]);
    for (float k : kin) out += "," + real_text(k);
    out += "," + real_text(total) + "," + real_text(mde) + "," + real_text(mdb) + "," +
           std::to_string(total_particles()) + "," + double_text(wall) + "," + double_text(rate) + "\n";
    return out;
  }

  // dump_fields, binary (proj/src/fields.cpp:315-344): "nx ny nz float32\n"
  // then 16 fp32 lanes per interior voxel in (z, y, x) order
  void dump_fields(const std::string& path) {
    quiesce(*ctx);
    const size_t V = (size_t)ctx->gc.V;
    std::vector<float> f(F_COUNT * V);
    CUDA_OK(cudaMemcpyAsync(f.data(), ctx->f, f.size() * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    std::ofstream out(path, std::ios::binary);
    if (!out) throw RunAbort("dump_fields: cannot open " + path);
    out << grid.nx << ' ' << grid.ny << ' ' << grid.nz << " float32\n";
    float rec[F_COUNT];
    for (int iz = 1; iz <= grid.nz; ++iz)
      for (int iy = 1; iy <= grid.ny; ++iy)
        for (int ix = 1; ix <= grid.nx; ++ix) {
          const size_t v = (size_t)ix + (size_t)(grid.nx + 2) * ((size_t)iy + (size_t)(grid.ny + 2) * iz);
          for (int l = 0; l < F_COUNT; ++l) rec[l] = f[(size_t)l * V + v];
          out.write(reinterpret_cast<const char*>(rec), sizeof rec);
        }
    if (!out) throw RunAbort("dump_fields: write failed for " + path);
  }

  // SimState::run_hooks (sim.cpp:190-215): mirrors refreshed / copied back
  // per the hook's flags, one counted copy per species or field array
  void run_hooks() {
    for (auto& h : hooks) {
      if (step_count == 0 || step_count % h.interval != 0) continue;
      const size_t ns = ctx->species.size();
      host_lanes.resize(ns);
      host_ids.resize(ns);
      const size_t V = (size_t)ctx->gc.V;
      if (host_fields.size() != F_COUNT * V) host_fields.assign(F_COUNT * V, 0.f);
      std::vector<size_t> counts(ns);
      for (size_t i = 0; i < ns; ++i) {
        counts[i] = ctx->species[i].n;
        if (host_lanes[i].size() != 7 * counts[i]) host_lanes[i].assign(7 * counts[i], 0.f);
        if (host_ids[i].size() != counts[i]) host_ids[i].assign(counts[i], 0);
      }
      pic_context view_ctx{ctx, true};
      if (h.flags.particles_to_host)
        for (size_t i = 0; i < ns; ++i) {
          if (int rc = pic_species_download(&view_ctx, (int)i, host_lanes[i].data(), host_ids[i].data()))
            throw RunAbort(std::string("run_hooks: particle mirror: ") + pic_last_error() + " (" +
                           std::to_string(rc) + ")");
          ++copies;
        }
      if (h.flags.fields_to_host) {
        if (pic_fields_download(&view_ctx, host_fields.data())) throw RunAbort(pic_last_error());
        ++copies;
      }
      if (h.fn) {
        std::vector<float*> lp(ns);
        std::vector<int32_t*> ip(ns);
        for (size_t i = 0; i < ns; ++i) {
          lp[i] = host_lanes[i].data();
          ip[i] = host_ids[i].data();
        }
        pic_hook_view v{handle, step_count, host_fields.data(), ns, lp.data(), ip.data(), counts.data()};
        const int rc = h.fn(&v, h.user);
        if (rc != 0)
          throw RunAbort("hook '" + h.name + "' failed at step " + std::to_string(step_count) +
                         ": callback returned " + std::to_string(rc));
      }
      if (h.flags.particles_back)
        for (size_t i = 0; i < ns; ++i) {
          if (int rc = pic_species_upload(&view_ctx, (int)i, counts[i], host_lanes[i].data(), host_ids[i].data()))
            throw RunAbort(std::string("run_hooks: particle copy-back: ") + pic_last_error() + " (" +
                           std::to_string(rc) + ")");
          ++copies;
        }
      if (h.flags.fields_back) {
        if (pic_fields_upload(&view_ctx, host_fields.data())) throw RunAbort(pic_last_error());
        ++copies;
      }
    }
  }

  // SimState::run (sim.cpp:285-306)
  void run(std::ostream* csv) {
    namespace fs = std::filesystem;
    if (deck.field_dump_interval > 0) fs::create_directories(deck.out_dir);
    if (csv) *csv << diagnostics_row();
    // every species sorted (blocked) on one cadence: the graphs of the run's
    // steps captured ahead (pic_prepare_step_graphs), so every step replays
    long si = -1;
    bool one_cadence = !deck.deterministic && !deck.species.empty();
    for (const auto& ds : deck.species) {
      if (si < 0) si = ds.sort_interval;
      one_cadence = one_cadence && ds.sort_interval == si && ds.sort_order == PIC_SORT_BLOCKED;
    }
    if (one_cadence && si > 0 && deck.steps > 2)
      prepare_step_graphs(*ctx, flags(), (int)std::min<long>(deck.steps, 1 << 16), (int)si, step_count);
    for (long i = 0; i < deck.steps; ++i) {
      do_step();
      sort_due();
      const bool due = step_count % deck.diag_interval == 0;
      if (due) refresh_charge();
      run_hooks();
      if (due && csv) *csv << diagnostics_row();
      if (deck.field_dump_interval > 0 && step_count % deck.field_dump_interval == 0)
        dump_fields((fs::path(deck.out_dir) / ("fields_" + std::to_string(step_count) + ".bin")).string());
      if (csv && !*csv) throw RunAbort("emit_diagnostics: sink write failed");
    }
    quiesce(*ctx);
  }
};

}  // namespace picb

// ===========================================================================
// C-ABI (declared in include/pic_b200.h)
using namespace picb;

struct pic_deck {
  Deck d;
};
struct pic_sim {
  Sim* s;
  pic_context* h;  // borrowed view of the sim's device state
};

static size_t copy_out(const std::string& s, char* buf, size_t cap) {
  if (buf && cap) {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size();
}

// the sim's device is current for every call (several GPUs, one host thread)
static Sim& S_(pic_sim* s) {
  if (!s || !s->s) throw UsageError("null pic_sim");
  CUDA_OK(cudaSetDevice(s->s->ctx->device));
  return *s->s;
}

extern "C" {

int pic_deck_parse(const char* text, pic_deck** out) {
  return capi_guard([&] {
    if (!text || !out) throw UsageError("pic_deck_parse: null argument");
    *out = nullptr;
    *out = new pic_deck{parse_deck(text)};
  });
}
int pic_deck_destroy(pic_deck* d) {
  delete d;
  return PIC_OK;
}
int pic_deck_override(pic_deck* d, const char* key_eq_value) {
  return capi_guard([&] {
    if (!d || !key_eq_value) throw UsageError("pic_deck_override: null argument");
    Deck copy = d->d;  // a failed override leaves the deck unchanged
    apply_override(copy, key_eq_value);
    d->d = copy;
  });
}
int pic_deck_serialize(const pic_deck* d, char* buf, size_t cap, size_t* len) {
  return capi_guard([&] {
    if (!d) throw UsageError("pic_deck_serialize: null deck");
    const size_t n = copy_out(serialize_deck(d->d), buf, cap);
    if (len) *len = n;
  });
}
int pic_deck_grid(const pic_deck* d, pic_grid* out) {
  return capi_guard([&] {
    if (!d || !out) throw UsageError("pic_deck_grid: null argument");
    *out = deck_grid(d->d);
  });
}
int pic_deck_steps(const pic_deck* d, long* out) {
  return capi_guard([&] {
    if (!d || !out) throw UsageError("pic_deck_steps: null argument");
    *out = d->d.steps;
  });
}

int pic_sim_create(int device, const pic_deck* d, pic_sim** out) {
  return capi_guard([&] {
    if (!d || !out) throw UsageError("pic_sim_create: null argument");
    *out = nullptr;
    Sim* s = new Sim(device, d->d);
    *out = new pic_sim{s, new pic_context{s->ctx, true}};
    s->handle = *out;
  });
}
int pic_sim_destroy(pic_sim* s) {
  if (!s) return PIC_OK;
  return capi_guard([&] {
    delete s->h;
    delete s->s;
    delete s;
  });
}
int pic_sim_context(pic_sim* s, pic_context** out) {
  return capi_guard([&] {
    if (!s || !out) throw UsageError("pic_sim_context: null argument");
    *out = s->h;
  });
}
int pic_sim_step(pic_sim* s) {
  return capi_guard([&] {
    Sim& m = S_(s);
    m.do_step();
    m.sort_due();
    quiesce(*m.ctx);
  });
}
int pic_sim_step_count(pic_sim* s, long* out) {
  return capi_guard([&] { *out = S_(s).step_count; });
}
int pic_sim_refresh_charge_diagnostics(pic_sim* s) {
  return capi_guard([&] { S_(s).refresh_charge(); });
}
int pic_sim_emit_diagnostics(pic_sim* s, char* buf, size_t cap, size_t* len) {
  return capi_guard([&] {
    // a size query (or a short buffer) computes the row and keeps it: the
    // next call returns the same row, not a second one
    Sim& m = S_(s);
    if (!m.row_kept) {
      m.kept_row = m.diagnostics_row();
      m.row_kept = true;
    }
    const size_t n = copy_out(m.kept_row, buf, cap);
    if (buf && cap > n) m.row_kept = false;
    if (len) *len = n;
  });
}
int pic_sim_run(pic_sim* s, const char* csv_path) {
  return capi_guard([&] {
    Sim& m = S_(s);
    if (csv_path) {
      std::ofstream f(csv_path);
      if (!f) throw RunAbort(std::string("pic_sim_run: cannot open ") + csv_path);
      m.run(&f);
    } else {
      m.run(nullptr);
    }
  });
}
int pic_sim_dump_fields(pic_sim* s, const char* path) {
  return capi_guard([&] { S_(s).dump_fields(path); });
}
int pic_sim_register_hook(pic_sim* s, const char* name, long interval, const pic_hook_flags* flags,
                          pic_hook_fn fn, void* user) {
  return capi_guard([&] {
    Sim& m = S_(s);
    if (interval < 1) throw UsageError("register_hook: interval must be >= 1");
    const pic_hook_flags legacy{1, 1, 1, 1};
    m.hooks.push_back({name ? name : "hook", interval, flags ? *flags : legacy, fn, user});
  });
}
int pic_sim_copies_performed(pic_sim* s, uint64_t* out) {
  return capi_guard([&] { *out = S_(s).copies; });
}
int pic_sim_warnings(pic_sim* s, char* buf, size_t cap, size_t* len) {
  return capi_guard([&] {
    std::string all;
    for (const auto& w : s->s->warnings) all += w + "\n";
    const size_t n = copy_out(all, buf, cap);
    if (len) *len = n;
  });
}

}  // extern "C"
