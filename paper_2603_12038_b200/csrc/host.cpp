// host.cpp — the C++ operator API (include/sfi/*.hpp, namespace sfi) over the
// C ABI. Host code validates arguments (the reference's error codes, in the
// reference's order), stages host vectors to / from HBM and launches the
// device path; the Selector stages, top-k, attention, appends, gathers and
// the normalisation all run in the sm_100a kernels. Host arithmetic is
// limited to bookkeeping: u(j) of make_cache_stats (an integer ratio), the
// distribution predicates and the two reductions callers use for checks
// (dot, squared_norm), config I/O and the scheduler's integer logic.
#include "sfi_b200.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <map>
#include <numeric>
#include <ostream>
#include <sstream>

namespace sfi {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorCode::kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaStream_t st(void* s) { return static_cast<cudaStream_t>(s); }

// Grow-only device scratch owned by the calling thread.
struct Scratch {
  void* p = nullptr;
  size_t n = 0;
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      cuda_check(cudaMalloc(&p, bytes), "scratch alloc");
      n = bytes;
    }
    return p;
  }
  ~Scratch() {
    if (p) cudaFree(p);
  }
};
thread_local Scratch t_scratch;

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

uint16_t to_bf16(float x) {
  const __nv_bfloat16 b = __float2bfloat16_rn(x);
  uint16_t u;
  std::memcpy(&u, &b, 2);
  return u;
}
float from_bf16(uint16_t u) {
  uint32_t w = static_cast<uint32_t>(u) << 16;
  float f;
  std::memcpy(&f, &w, 4);
  return f;
}

void require(bool ok, const std::string& what) {
  if (!ok) fail(ErrorCode::kConfig, "config: " + what);
}

}  // namespace

// ---------------------------------------------------------------------------
// errors

void check(int status) {
  if (status == SFI_OK) return;
  const std::string msg = sfi_last_error();
  if (status >= 1 && status <= 10) fail(static_cast<ErrorCode>(status - 1), msg);
  if (status == SFI_ERR_UNSUPPORTED) fail(ErrorCode::kUnsupported, msg);
  if (status == SFI_ERR_INVALID_ARGUMENT) fail(ErrorCode::kOutOfRange, msg);
  fail(ErrorCode::kCuda, msg);
}

// ---------------------------------------------------------------------------
// config (config.cpp:68-200)

void SelectorConfig::validate() const {
  require(alpha > 0.0 && alpha <= 1.0, "alpha must be in (0, 1]");
  require(gamma >= 0.0, "gamma must be >= 0");
  require(beta >= 0.0, "beta must be >= 0");
  require(p_curve >= 1.0, "p_curve must be >= 1");
  require(eta >= 0.0, "eta must be >= 0");
  require(lambda_clip >= 0.0 && lambda_clip <= 1.0, "lambda_clip must be in [0, 1]");
  require(alpha_soft >= 0.0, "alpha_soft must be >= 0");
  require(alpha_cross >= 0.0, "alpha_cross must be >= 0");
  require(temperature > 0.0, "temperature must be > 0");
  require(nms_radius >= 0, "nms_radius must be >= 0");
  require(epsilon > 0.0, "epsilon must be > 0");
  require(k_budget >= 0, "k_budget must be >= 0");
  for (double v : {alpha, gamma, beta, p_curve, eta, lambda_clip, alpha_soft, alpha_cross,
                   temperature, epsilon})
    require(std::isfinite(v), "selector values must be finite");
}

sfi_selector_params to_params(const SelectorConfig& c) {
  sfi_selector_params p;
  p.alpha = c.alpha;
  p.gamma = c.gamma;
  p.beta = c.beta;
  p.p_curve = c.p_curve;
  p.eta = c.eta;
  p.lambda_clip = c.lambda_clip;
  p.alpha_soft = c.alpha_soft;
  p.alpha_cross = c.alpha_cross;
  p.temperature = c.temperature;
  p.epsilon = c.epsilon;
  p.nms_radius = c.nms_radius;
  p.pool = c.pool == PoolMode::kMax ? SFI_POOL_MAX : SFI_POOL_MEAN;
  return p;
}

void TriggerConfig::validate() const {
  require(t_max >= 1, "t_max must be >= 1");
  require(window_decode >= 1, "window_decode must be >= 1");
  require(window_prefill >= 1, "window_prefill must be >= 1");
}

bool TriggerConfig::is_trigger(TokenId id) const {
  return std::find(trigger_tokens.begin(), trigger_tokens.end(), id) != trigger_tokens.end();
}

void CacheLimits::validate() const {
  require(n_sink >= 0, "n_sink must be >= 0");
  require(n_recent >= 1, "n_recent must be >= 1");
  require(k_budget >= 0, "k_budget must be >= 0");
}

void Config::validate() const {
  selector.validate();
  trigger.validate();
  limits.validate();
}

Config default_config() { return Config{}; }

namespace {

std::string strip(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

template <typename T>
T parse_num(const std::string& key, const std::string& s) {
  T v{};
  const auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc() || end != s.data() + s.size())
    fail(ErrorCode::kConfig, std::string("config: bad ") + (std::is_integral_v<T> ? "integer" : "numeric") +
                                 " value for " + key + ": '" + s + "'");
  return v;
}

std::string shortest(double v) {  // round-trips exactly
  char buf[64];
  const auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  (void)ec;
  return std::string(buf, end);
}

}  // namespace

void save_config(const Config& cfg, std::ostream& out) {
  const SelectorConfig& s = cfg.selector;
  const std::pair<const char*, double> doubles[] = {
      {"alpha", s.alpha}, {"gamma", s.gamma}, {"beta", s.beta}, {"p_curve", s.p_curve}, {"eta", s.eta},
      {"lambda_clip", s.lambda_clip}, {"alpha_soft", s.alpha_soft}, {"alpha_cross", s.alpha_cross},
      {"temperature", s.temperature}};
  for (const auto& [k, v] : doubles) out << k << '=' << shortest(v) << '\n';
  out << "nms_radius=" << s.nms_radius << '\n' << "epsilon=" << shortest(s.epsilon) << '\n'
      << "k_budget=" << s.k_budget << '\n' << "logit_pool=" << (s.pool == PoolMode::kMax ? "max" : "mean") << '\n';
  out << "trigger_tokens=";
  for (size_t i = 0; i < cfg.trigger.trigger_tokens.size(); ++i)
    out << (i ? "," : "") << cfg.trigger.trigger_tokens[i];
  out << '\n' << "t_max=" << cfg.trigger.t_max << '\n' << "window_decode=" << cfg.trigger.window_decode << '\n'
      << "window_prefill=" << cfg.trigger.window_prefill << '\n' << "n_sink=" << cfg.limits.n_sink << '\n'
      << "n_recent=" << cfg.limits.n_recent << '\n';
}

void save_config_file(const Config& cfg, const std::string& path) {
  std::ofstream out(path);
  if (!out) fail(ErrorCode::kIo, "cannot open config file for writing: " + path);
  save_config(cfg, out);
}

Config load_config(std::istream& in) {
  Config cfg;
  SelectorConfig& s = cfg.selector;
  const std::map<std::string, double*> doubles = {
      {"alpha", &s.alpha}, {"gamma", &s.gamma}, {"beta", &s.beta}, {"p_curve", &s.p_curve}, {"eta", &s.eta},
      {"lambda_clip", &s.lambda_clip}, {"alpha_soft", &s.alpha_soft}, {"alpha_cross", &s.alpha_cross},
      {"temperature", &s.temperature}, {"epsilon", &s.epsilon}};
  const std::map<std::string, int*> ints = {
      {"nms_radius", &s.nms_radius}, {"t_max", &cfg.trigger.t_max},
      {"window_decode", &cfg.trigger.window_decode}, {"window_prefill", &cfg.trigger.window_prefill},
      {"n_sink", &cfg.limits.n_sink}, {"n_recent", &cfg.limits.n_recent}};
  std::string line;
  for (int lineno = 1; std::getline(in, line); ++lineno) {
    const std::string t = strip(line);
    if (t.empty() || t[0] == '#') continue;
    const size_t eq = t.find('=');
    if (eq == std::string::npos)
      fail(ErrorCode::kConfig, "config: line " + std::to_string(lineno) + " is not key=value: '" + t + "'");
    const std::string key = strip(t.substr(0, eq)), val = strip(t.substr(eq + 1));
    if (auto d = doubles.find(key); d != doubles.end()) {
      *d->second = parse_num<double>(key, val);
    } else if (auto i = ints.find(key); i != ints.end()) {
      *i->second = parse_num<int>(key, val);
    } else if (key == "k_budget") {  // one knob for both structs (config.cpp:173-176)
      s.k_budget = parse_num<int>(key, val);
      cfg.limits.k_budget = s.k_budget;
    } else if (key == "logit_pool") {
      if (val == "mean") s.pool = PoolMode::kMean;
      else if (val == "max") s.pool = PoolMode::kMax;
      else fail(ErrorCode::kConfig, "config: logit_pool must be mean or max");
    } else if (key == "trigger_tokens") {
      cfg.trigger.trigger_tokens.clear();
      std::stringstream ss(val);
      std::string tok;
      while (!val.empty() && std::getline(ss, tok, ','))
        cfg.trigger.trigger_tokens.push_back(parse_num<int>(key, strip(tok)));
    } else {
      fail(ErrorCode::kConfig, "config: unknown key '" + key + "' (line " + std::to_string(lineno) + ")");
    }
  }
  cfg.validate();
  return cfg;
}

Config load_config_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ErrorCode::kIo, "cannot open config file: " + path);
  return load_config(in);
}

void ModelSpec::validate() const {
  auto bad = [](const std::string& what) { fail(ErrorCode::kConfig, "model spec: " + what); };
  if (n_layers < 1) bad("n_layers must be >= 1");
  if (n_query_heads < 1 || n_kv_heads < 1) bad("head counts must be >= 1");
  if (n_query_heads % n_kv_heads != 0) bad("n_query_heads must be a multiple of n_kv_heads");
  if (head_dim < 2 || head_dim % 2 != 0) bad("head_dim must be even and >= 2");
  if (vocab_size < 2) bad("vocab_size must be >= 2");
  if (max_positions < 1) bad("max_positions must be >= 1");
  if (!(rope_base > 0.0)) bad("rope_base must be > 0");
}

// ---------------------------------------------------------------------------
// distributions (distribution.cpp)

bool validate_distribution(const ScoreDistribution& d) {
  if (d.support.size() != d.mass.size() || d.support.empty()) return false;
  Pos prev = 0;
  double sum = 0.0;
  for (size_t i = 0; i < d.support.size(); ++i) {
    if (d.support[i] <= prev) return false;
    prev = d.support[i];
    if (!std::isfinite(d.mass[i]) || d.mass[i] < 0.0) return false;
    sum += d.mass[i];
  }
  return std::abs(sum - 1.0) <= 1e-9;
}

bool same_support(const ScoreDistribution& a, const ScoreDistribution& b) { return a.support == b.support; }

double dot(const ScoreDistribution& a, const ScoreDistribution& b) {
  if (!same_support(a, b)) fail(ErrorCode::kSupportMismatch, "dot: distributions on different supports");
  double acc = 0.0;
  for (size_t i = 0; i < a.mass.size(); ++i) acc += a.mass[i] * b.mass[i];
  return acc;
}

double squared_norm(const ScoreDistribution& d) {
  double acc = 0.0;
  for (double m : d.mass) acc += m * m;
  return acc;
}

// ---------------------------------------------------------------------------
// Selector stages on the device (sfi_selector_stage)

namespace {

struct StageIO {
  double* a;
  double* b;
  double* out;
  double* out2;
  int32_t* err;
};

// Device buffers for one stage call: a [na], b [nb], out [nout], out2 [nout2], err [H]
StageIO stage_buffers(size_t na, size_t nb, size_t nout, size_t nout2, int H) {
  uint8_t* p = static_cast<uint8_t*>(
      t_scratch.get(al(na * 8) + al(nb * 8) + al(nout * 8) + al(nout2 * 8) + al(std::max(H, 1) * 4)));
  StageIO io;
  io.a = reinterpret_cast<double*>(p);
  p += al(na * 8);
  io.b = reinterpret_cast<double*>(p);
  p += al(nb * 8);
  io.out = reinterpret_cast<double*>(p);
  p += al(nout * 8);
  io.out2 = reinterpret_cast<double*>(p);
  p += al(nout2 * 8);
  io.err = reinterpret_cast<int32_t*>(p);
  return io;
}

void up(double* dst, const double* src, size_t n, const char* what) {
  if (n) cuda_check(cudaMemcpy(dst, src, n * 8, cudaMemcpyHostToDevice), what);
}

std::vector<double> down(const double* src, size_t n, const char* what) {
  std::vector<double> v(n);
  if (n) cuda_check(cudaMemcpy(v.data(), src, n * 8, cudaMemcpyDeviceToHost), what);
  return v;
}

// Throws the first per-head error (heads in order) with the reference's message.
void head_errors(const int32_t* d_err, int H, const char* stage) {
  if (H <= 0) return;
  std::vector<int32_t> e(static_cast<size_t>(H));
  cuda_check(cudaMemcpy(e.data(), d_err, H * 4, cudaMemcpyDeviceToHost), stage);
  for (int h = 0; h < H; ++h) {
    if (e[h] == SFI_ERR_NON_FINITE_INPUT) {
      if (std::strcmp(stage, "evidence") == 0)
        fail(ErrorCode::kNonFiniteInput, "evidence_from_window: non-finite logit");
      if (std::strcmp(stage, "prior") == 0) fail(ErrorCode::kNonFiniteInput, "prior_from_stats: bad key norm");
      fail(ErrorCode::kNonFiniteInput, "normalize: weights must be finite and >= 0");
    }
    if (e[h] == SFI_ERR_EMPTY_SUPPORT) {
      if (std::strcmp(stage, "evidence") == 0)
        fail(ErrorCode::kEmptySupport, "evidence_from_window: fully masked row");
      fail(ErrorCode::kEmptySupport, "normalize: all weights are zero");
    }
    if (e[h]) fail(ErrorCode::kCuda, std::string(stage) + ": device stage error");
  }
}

void run_stage(int stage, int H, int W, int n, const StageIO& io, const SelectorConfig& cfg) {
  const sfi_selector_params prm = to_params(cfg);
  if (stage <= SFI_STAGE_NORMALIZE) cuda_check(cudaMemset(io.err, 0, std::max(H, 1) * 4), "stage");
  check(sfi_selector_stage(stage, H, W, n, io.a, io.b, &prm, io.out, io.out2, io.err, nullptr));
  cuda_check(cudaDeviceSynchronize(), "stage");
}

void count_ops(SelectorTrace* trace, std::uint64_t n) {
  if (trace) trace->elementary_ops += n;
}

void dump_scores(SelectorTrace* trace, const char* stage, int head, const std::vector<Pos>& support,
                 const std::vector<double>& scores) {
  if (!trace || !trace->capture_debug) return;
  std::ostringstream os;
  os << "{\"stage\":\"" << stage << "\",\"head\":" << head << ",\"support\":[";
  for (size_t i = 0; i < support.size(); ++i) os << (i ? "," : "") << support[i];
  os << "],\"scores\":[";
  os.precision(17);
  for (size_t i = 0; i < scores.size(); ++i) os << (i ? "," : "") << scores[i];
  os << "]}";
  trace->debug_lines.push_back(os.str());
}

std::uint64_t nms_ops(int n, int R) {
  std::uint64_t ops = 0;
  for (int j = 0; j < n; ++j) ops += static_cast<std::uint64_t>(std::min(n - 1, j + R) - std::max(0, j - R) + 1) + 2;
  return ops;
}

}  // namespace

ScoreDistribution normalize(std::span<const Pos> support, std::span<const double> weights) {
  if (support.empty() || weights.empty()) fail(ErrorCode::kEmptySupport, "normalize: empty support");
  if (support.size() != weights.size())
    fail(ErrorCode::kSupportMismatch, "normalize: support/weight length mismatch");
  const size_t n = weights.size();
  StageIO io = stage_buffers(n, 0, n, 0, 1);
  up(io.a, weights.data(), n, "normalize");
  run_stage(SFI_STAGE_NORMALIZE, 1, 1, static_cast<int>(n), io, SelectorConfig{});
  head_errors(io.err, 1, "normalize");
  ScoreDistribution d;
  d.support.assign(support.begin(), support.end());
  d.mass = down(io.out, n, "normalize");
  return d;
}

CacheStats make_cache_stats(std::vector<std::vector<double>> key_norms, const std::vector<Pos>& allowed,
                            double epsilon) {
  if (allowed.empty()) fail(ErrorCode::kEmptySupport, "make_cache_stats: empty allowed set");
  for (const auto& per_head : key_norms)
    if (per_head.size() != allowed.size())
      fail(ErrorCode::kSupportMismatch, "make_cache_stats: key_norms misaligned with J");
  CacheStats stats;
  stats.key_norms = std::move(key_norms);
  stats.j_min = allowed.front();
  stats.j_max = allowed.back();
  stats.normalized_pos.resize(allowed.size());
  const double denom = static_cast<double>(stats.j_max - stats.j_min) + epsilon;
  for (size_t i = 0; i < allowed.size(); ++i)
    stats.normalized_pos[i] = static_cast<double>(allowed[i] - stats.j_min) / denom;
  return stats;
}

std::vector<ScoreDistribution> evidence_from_window(const LogitWindow& w, const SelectorConfig& cfg,
                                                    SelectorTrace* trace) {
  if (w.allowed.empty()) fail(ErrorCode::kEmptySupport, "evidence_from_window: empty support");
  if (w.width < 1) fail(ErrorCode::kOutOfRange, "evidence_from_window: window width must be >= 1");
  const int n = static_cast<int>(w.allowed.size()), W = w.width;
  int H = w.heads();
  int bad_shape = H;  // the reference validates head h's shape just before computing it
  for (int h = 0; h < H; ++h)
    if (w.values[h].size() != static_cast<size_t>(W) * n) {
      bad_shape = h;
      break;
    }
  const int Hc = bad_shape;
  std::vector<double> f;
  if (Hc > 0) {
    StageIO io = stage_buffers(static_cast<size_t>(Hc) * W * n, 0, static_cast<size_t>(Hc) * n, 0, Hc);
    for (int h = 0; h < Hc; ++h) up(io.a + static_cast<size_t>(h) * W * n, w.values[h].data(), W * n, "evidence");
    run_stage(SFI_STAGE_EVIDENCE, Hc, W, n, io, cfg);
    head_errors(io.err, Hc, "evidence");
    f = down(io.out, static_cast<size_t>(Hc) * n, "evidence");
  }
  if (bad_shape < H) fail(ErrorCode::kSupportMismatch, "evidence_from_window: bad window shape");
  std::vector<ScoreDistribution> out(static_cast<size_t>(H));
  for (int h = 0; h < H; ++h) {
    out[h].support = w.allowed;
    out[h].mass.assign(f.begin() + static_cast<size_t>(h) * n, f.begin() + static_cast<size_t>(h + 1) * n);
    count_ops(trace, static_cast<std::uint64_t>(3) * n * W + 2ull * n);
    dump_scores(trace, "evidence", h, w.allowed, out[h].mass);
  }
  return out;
}

std::vector<ScoreDistribution> prior_from_stats(const CacheStats& stats, const std::vector<Pos>& allowed,
                                                const SelectorConfig& cfg, SelectorTrace* trace) {
  if (allowed.empty()) fail(ErrorCode::kEmptySupport, "prior_from_stats: empty allowed set");
  if (stats.normalized_pos.size() != allowed.size())
    fail(ErrorCode::kSupportMismatch, "prior_from_stats: stats misaligned with J");
  const int n = static_cast<int>(allowed.size());
  const int H = static_cast<int>(stats.key_norms.size());
  int Hc = H;
  for (int h = 0; h < H; ++h)
    if (stats.key_norms[h].size() != static_cast<size_t>(n)) {
      Hc = h;
      break;
    }
  std::vector<double> r;
  if (Hc > 0) {
    StageIO io = stage_buffers(static_cast<size_t>(Hc) * n, n, static_cast<size_t>(Hc) * n, 0, Hc);
    for (int h = 0; h < Hc; ++h) up(io.a + static_cast<size_t>(h) * n, stats.key_norms[h].data(), n, "prior");
    up(io.b, stats.normalized_pos.data(), n, "prior");
    run_stage(SFI_STAGE_PRIOR, Hc, 1, n, io, cfg);
    head_errors(io.err, Hc, "prior");
    r = down(io.out, static_cast<size_t>(Hc) * n, "prior");
  }
  if (Hc < H) fail(ErrorCode::kSupportMismatch, "prior_from_stats: key_norms misaligned with J");
  std::vector<ScoreDistribution> out(static_cast<size_t>(H));
  for (int h = 0; h < H; ++h) {
    out[h].support = allowed;
    out[h].mass.assign(r.begin() + static_cast<size_t>(h) * n, r.begin() + static_cast<size_t>(h + 1) * n);
    count_ops(trace, 5ull * n);
    dump_scores(trace, "prior", h, allowed, out[h].mass);
  }
  return out;
}

FusedScore fuse(const ScoreDistribution& f, const ScoreDistribution& r, const SelectorConfig& cfg,
                SelectorTrace* trace) {
  if (!same_support(f, r)) fail(ErrorCode::kSupportMismatch, "fuse: evidence and prior on different supports");
  if (f.mass.size() != r.mass.size()) fail(ErrorCode::kSupportMismatch, "fuse: mass length mismatch");
  const size_t n = f.mass.size();
  FusedScore res;
  res.evidence = f;
  res.prior = r;
  res.fused.support = f.support;
  if (n > 0) {
    StageIO io = stage_buffers(n, n, n, 1, 1);
    up(io.a, f.mass.data(), n, "fuse");
    up(io.b, r.mass.data(), n, "fuse");
    run_stage(SFI_STAGE_FUSE, 1, 1, static_cast<int>(n), io, cfg);
    res.fused.mass = down(io.out, n, "fuse");
    res.lambda_star = down(io.out2, 1, "fuse")[0];
  }
  count_ops(trace, 5ull * n);
  return res;
}

std::vector<double> refine_soft_nms(const std::vector<double>& z, const SelectorConfig& cfg,
                                    SelectorTrace* trace) {
  const size_t n = z.size();
  std::vector<double> out;
  if (n > 0) {
    StageIO io = stage_buffers(n, 0, n, 0, 1);
    up(io.a, z.data(), n, "refine_soft_nms");
    run_stage(SFI_STAGE_SOFT_NMS, 1, 1, static_cast<int>(n), io, cfg);
    out = down(io.out, n, "refine_soft_nms");
  }
  count_ops(trace, nms_ops(static_cast<int>(n), cfg.nms_radius));
  return out;
}

std::vector<std::vector<double>> refine_cross_head(const std::vector<std::vector<double>>& z,
                                                   const SelectorConfig& cfg, SelectorTrace* trace) {
  const size_t H = z.size();
  if (H == 0) return {};
  const size_t n = z[0].size();
  for (const auto& zh : z)
    if (zh.size() != n) fail(ErrorCode::kSupportMismatch, "refine_cross_head: ragged score matrix");
  std::vector<std::vector<double>> out(H, std::vector<double>(n));
  if (n > 0) {
    StageIO io = stage_buffers(H * n, 0, H * n, 0, static_cast<int>(H));
    for (size_t h = 0; h < H; ++h) up(io.a + h * n, z[h].data(), n, "refine_cross_head");
    run_stage(SFI_STAGE_CROSS_HEAD, static_cast<int>(H), 1, static_cast<int>(n), io, cfg);
    const std::vector<double> v = down(io.out, H * n, "refine_cross_head");
    for (size_t h = 0; h < H; ++h) std::copy(v.begin() + h * n, v.begin() + (h + 1) * n, out[h].begin());
  }
  count_ops(trace, 6ull * H * n);
  return out;
}

std::vector<Pos> select_top_k(const std::vector<double>& scores, const std::vector<Pos>& allowed, int k) {
  if (scores.size() != allowed.size()) fail(ErrorCode::kSupportMismatch, "select_top_k: score/support mismatch");
  if (k < 0) fail(ErrorCode::kOutOfRange, "select_top_k: negative budget");
  const int n = static_cast<int>(scores.size());
  const size_t kk = static_cast<size_t>(std::max(1, std::min(k, std::max(n, 1))));
  const size_t nn = static_cast<size_t>(std::max(n, 1));
  uint8_t* base = static_cast<uint8_t*>(t_scratch.get(al(nn * 8) + al(nn * 4) + al(kk * 4) + al(4)));
  double* d_scores = reinterpret_cast<double*>(base);
  int32_t* d_allowed = reinterpret_cast<int32_t*>(base + al(nn * 8));
  int32_t* d_sel = reinterpret_cast<int32_t*>(base + al(nn * 8) + al(nn * 4));
  int32_t* d_cnt = reinterpret_cast<int32_t*>(base + al(nn * 8) + al(nn * 4) + al(kk * 4));
  if (n > 0) {
    cuda_check(cudaMemcpy(d_scores, scores.data(), n * 8, cudaMemcpyHostToDevice), "select_top_k");
    cuda_check(cudaMemcpy(d_allowed, allowed.data(), n * 4, cudaMemcpyHostToDevice), "select_top_k");
  }
  check(sfi_select_top_k(1, n, k, d_scores, d_allowed, d_sel, d_cnt, nullptr));
  int32_t cnt = 0;
  cuda_check(cudaMemcpy(&cnt, d_cnt, 4, cudaMemcpyDeviceToHost), "select_top_k");
  std::vector<Pos> out(static_cast<size_t>(cnt));
  if (cnt) cuda_check(cudaMemcpy(out.data(), d_sel, cnt * 4, cudaMemcpyDeviceToHost), "select_top_k");
  return out;
}

namespace {

// run_selector with a trace that asks for the stage arrays / debug lines: the
// stage kernels in the reference's order (selector.cpp:254-299).
std::vector<std::vector<Pos>> run_selector_staged(const LogitWindow& w, const CacheStats& stats,
                                                  const SelectorConfig& cfg, SelectorTrace* trace) {
  const std::vector<ScoreDistribution> evidence = evidence_from_window(w, cfg, trace);
  const std::vector<ScoreDistribution> prior = prior_from_stats(stats, w.allowed, cfg, trace);
  const size_t H = evidence.size(), n = w.allowed.size();
  std::vector<FusedScore> fusion(H);
  std::vector<std::vector<double>> z_base(H);
  for (size_t h = 0; h < H; ++h) {
    fusion[h] = fuse(evidence[h], prior[h], cfg, trace);
    StageIO io = stage_buffers(n, 0, n, 0, 1);
    up(io.a, fusion[h].fused.mass.data(), n, "z_base");
    run_stage(SFI_STAGE_Z_BASE, 1, 1, static_cast<int>(n), io, cfg);
    z_base[h] = down(io.out, n, "z_base");
    count_ops(trace, 2ull * n);
    dump_scores(trace, "z_base", static_cast<int>(h), w.allowed, z_base[h]);
  }
  std::vector<std::vector<double>> z_nms(H);
  for (size_t h = 0; h < H; ++h) {
    z_nms[h] = refine_soft_nms(z_base[h], cfg, trace);
    dump_scores(trace, "soft_nms", static_cast<int>(h), w.allowed, z_nms[h]);
  }
  std::vector<std::vector<double>> z_adj = refine_cross_head(z_nms, cfg, trace);
  for (size_t h = 0; h < H; ++h) dump_scores(trace, "cross_head", static_cast<int>(h), w.allowed, z_adj[h]);
  if (trace->capture_stages) {
    trace->stages.base = z_base;
    trace->stages.after_nms = z_nms;
    trace->stages.after_cross = z_adj;
    trace->fusion = fusion;
  }
  std::vector<std::vector<Pos>> selected(H);
  for (size_t h = 0; h < H; ++h) selected[h] = select_top_k(z_adj[h], w.allowed, cfg.k_budget);
  return selected;
}

}  // namespace

std::vector<std::vector<Pos>> run_selector(const LogitWindow& w, const CacheStats& stats,
                                           const SelectorConfig& cfg, SelectorTrace* trace) {
  if (w.heads() != static_cast<int>(stats.key_norms.size()))
    fail(ErrorCode::kSupportMismatch, "run_selector: window/stats head count mismatch");
  if (trace && (trace->capture_stages || trace->capture_debug)) return run_selector_staged(w, stats, cfg, trace);
  // argument checks in the reference's order (selector.cpp:99-108, 133-143)
  if (w.allowed.empty()) fail(ErrorCode::kEmptySupport, "evidence_from_window: empty support");
  if (w.width < 1) fail(ErrorCode::kOutOfRange, "evidence_from_window: window width must be >= 1");
  const int H = w.heads();
  const int W = w.width;
  const int n = static_cast<int>(w.allowed.size());
  for (int h = 0; h < H; ++h)
    if (w.values[h].size() != static_cast<size_t>(W) * n)
      fail(ErrorCode::kSupportMismatch, "evidence_from_window: bad window shape");
  if (stats.normalized_pos.size() != w.allowed.size())
    fail(ErrorCode::kSupportMismatch, "prior_from_stats: stats misaligned with J");
  for (int h = 0; h < H; ++h)
    if (stats.key_norms[h].size() != static_cast<size_t>(n))
      fail(ErrorCode::kSupportMismatch, "prior_from_stats: key_norms misaligned with J");
  if (H == 0) return {};
  const int K = cfg.k_budget;
  if (K < 0) fail(ErrorCode::kOutOfRange, "select_top_k: negative budget");
  if (trace) {  // elementary-operation count of the reference pipeline (top-k excluded)
    const std::uint64_t nn = static_cast<std::uint64_t>(n);
    trace->elementary_ops += static_cast<std::uint64_t>(H) *
                                 (3 * nn * W + 2 * nn + 5 * nn + 5 * nn + 2 * nn + nms_ops(n, cfg.nms_radius)) +
                             6ull * H * nn;
  }
  const size_t hn = static_cast<size_t>(H) * n;
  const size_t kk = static_cast<size_t>(std::max(K, 1));
  const size_t b_logits = al(hn * W * 8), b_norms = al(hn * 8), b_allowed = al(n * 4);
  const size_t b_scr = al(sfi_selector_explicit_scratch_bytes(H, n));
  const size_t b_sel = al(H * kk * 4), b_cnt = al(H * 4), b_err = al(4);
  uint8_t* base =
      static_cast<uint8_t*>(t_scratch.get(b_logits + b_norms + b_allowed + b_scr + b_sel + b_cnt + b_err));
  double* d_logits = reinterpret_cast<double*>(base);
  double* d_norms = reinterpret_cast<double*>(base + b_logits);
  int32_t* d_allowed = reinterpret_cast<int32_t*>(base + b_logits + b_norms);
  void* d_scr = base + b_logits + b_norms + b_allowed;
  int32_t* d_sel = reinterpret_cast<int32_t*>(base + b_logits + b_norms + b_allowed + b_scr);
  int32_t* d_cnt = reinterpret_cast<int32_t*>(base + b_logits + b_norms + b_allowed + b_scr + b_sel);
  uint32_t* d_err = reinterpret_cast<uint32_t*>(base + b_logits + b_norms + b_allowed + b_scr + b_sel + b_cnt);
  std::vector<double> flat(hn * W);
  std::vector<double> nflat(hn);
  for (int h = 0; h < H; ++h) {
    std::copy(w.values[h].begin(), w.values[h].end(), flat.begin() + static_cast<size_t>(h) * W * n);
    std::copy(stats.key_norms[h].begin(), stats.key_norms[h].end(), nflat.begin() + static_cast<size_t>(h) * n);
  }
  cuda_check(cudaMemcpy(d_logits, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice), "run_selector");
  cuda_check(cudaMemcpy(d_norms, nflat.data(), nflat.size() * 8, cudaMemcpyHostToDevice), "run_selector");
  cuda_check(cudaMemcpy(d_allowed, w.allowed.data(), n * 4, cudaMemcpyHostToDevice), "run_selector");
  cuda_check(cudaMemset(d_err, 0, 4), "run_selector");
  const sfi_selector_params prm = to_params(cfg);
  check(sfi_selector_explicit(H, W, n, K, d_logits, d_norms, d_allowed, &prm, d_scr, d_sel, d_cnt, d_err, nullptr));
  uint32_t err = 0;
  cuda_check(cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost), "run_selector");
  if (err & (1u << SFI_ERR_NON_FINITE_INPUT))
    fail(ErrorCode::kNonFiniteInput, "run_selector: non-finite logit or bad key norm");
  if (err & (1u << SFI_ERR_EMPTY_SUPPORT))
    fail(ErrorCode::kEmptySupport, "run_selector: fully masked row or all-zero weights");
  std::vector<int32_t> cnt(H);
  std::vector<int32_t> sel(static_cast<size_t>(H) * kk);
  cuda_check(cudaMemcpy(cnt.data(), d_cnt, H * 4, cudaMemcpyDeviceToHost), "run_selector");
  if (K > 0) cuda_check(cudaMemcpy(sel.data(), d_sel, sel.size() * 4, cudaMemcpyDeviceToHost), "run_selector");
  std::vector<std::vector<Pos>> out(static_cast<size_t>(H));
  for (int h = 0; h < H; ++h)
    out[h].assign(sel.begin() + static_cast<size_t>(h) * kk, sel.begin() + static_cast<size_t>(h) * kk + cnt[h]);
  return out;
}

// ---------------------------------------------------------------------------
// device cache

namespace {

struct Allocator {
  std::vector<void*>& owned;
  void* operator()(size_t bytes) const {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "DeviceCache alloc");
    cuda_check(cudaMemset(p, 0, std::max<size_t>(bytes, 256)), "DeviceCache memset");
    owned.push_back(p);
    return p;
  }
};

}  // namespace

DeviceCache::DeviceCache(const sfi_shape& shape) : shape_(shape) {
  check(sfi_buffer_sizes(&shape_, &sizes_));
  Allocator alloc{allocs_};
  cache_.k_cache = alloc(sizes_.kv_cache);
  cache_.v_cache = alloc(sizes_.kv_cache);
  cache_.key_norms = static_cast<double*>(alloc(sizes_.key_norms));
  cache_.ck = alloc(sizes_.compact);
  cache_.cv = alloc(sizes_.compact);
  cache_.sel = static_cast<int32_t*>(alloc(sizes_.sel));
  cache_.n_sel = static_cast<int32_t*>(alloc(sizes_.n_sel));
  cache_.prefix_len = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.n_sink_b = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.recent_len = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.error_flags = static_cast<uint32_t*>(alloc(4));
  cache_.workspace = alloc(sizes_.workspace);
  cache_.workspace_bytes = sizes_.workspace;
  logits_ = static_cast<float*>(alloc(sizes_.pooled_logits));
}

DeviceCache::DeviceCache(const sfi_shape& shape, void* k_cache, void* v_cache, double* key_norms) : shape_(shape) {
  if (shape.n_layers != 1) fail(ErrorCode::kConfig, "DeviceCache view: one layer");
  check(sfi_buffer_sizes(&shape_, &sizes_));
  Allocator alloc{allocs_};
  cache_.k_cache = k_cache;
  cache_.v_cache = v_cache;
  cache_.key_norms = key_norms;
  cache_.ck = alloc(sizes_.compact);
  cache_.cv = alloc(sizes_.compact);
  cache_.sel = static_cast<int32_t*>(alloc(sizes_.sel));
  cache_.n_sel = static_cast<int32_t*>(alloc(sizes_.n_sel));
  cache_.prefix_len = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.n_sink_b = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.recent_len = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.error_flags = static_cast<uint32_t*>(alloc(4));
  cache_.workspace = alloc(sizes_.workspace);
  cache_.workspace_bytes = sizes_.workspace;
  logits_ = nullptr;
}

DeviceCache::~DeviceCache() {
  for (void* p : allocs_) cudaFree(p);
}

// ---------------------------------------------------------------------------
// KvStore (attention.cpp:120-244)

namespace {

sfi_shape store_shape(const ModelSpec& spec, const CacheLimits& limits) {
  sfi_shape s{};
  s.n_layers = spec.n_layers;
  s.batch = 1;
  s.n_kv_heads = spec.n_kv_heads;
  s.n_q_heads = spec.n_query_heads;
  s.head_dim = spec.head_dim;
  s.max_positions = spec.max_positions;
  s.n_sink = limits.n_sink;
  s.k_budget = limits.k_budget;
  s.n_recent = limits.n_recent;
  return s;
}

// A one-layer view of `layer` of the store's paged KV with room for `rows`
// gathered rows per head (n_sink 0, ring of one unused row).
std::unique_ptr<DeviceCache> layer_view(const DeviceCache& dev, int layer, int rows) {
  sfi_shape s = dev.shape();
  const size_t slice = static_cast<size_t>(s.n_kv_heads) * s.max_positions;
  s.n_layers = 1;
  s.n_sink = 0;
  s.k_budget = std::max(rows, 1);
  s.n_recent = 1;
  const size_t kv_off = static_cast<size_t>(layer) * slice * s.head_dim * 2;  // bf16 bytes
  return std::make_unique<DeviceCache>(s, static_cast<uint8_t*>(dev.cache().k_cache) + kv_off,
                                       static_cast<uint8_t*>(dev.cache().v_cache) + kv_off,
                                       dev.cache().key_norms + static_cast<size_t>(layer) * slice);
}

// Gathers per-head position lists (ascending, 1-based, <= L) into a view's compact rows.
void gather_into(const DeviceCache& view, const std::vector<std::vector<Pos>>& rows, Pos L, void* stream) {
  const sfi_shape& s = view.shape();
  const int H = s.n_kv_heads, K = s.k_budget;
  const int32_t Lh = L, zero = 0;
  check(sfi_set_lengths(&s, &view.cache(), &Lh, &zero, &zero, stream));
  std::vector<int32_t> sel(static_cast<size_t>(H) * K, 0), cnt(H);
  for (int h = 0; h < H; ++h) {
    std::copy(rows[h].begin(), rows[h].end(), sel.begin() + static_cast<size_t>(h) * K);
    cnt[h] = static_cast<int32_t>(rows[h].size());
  }
  check(sfi_set_selection(&s, &view.cache(), 0, sel.data(), cnt.data(), stream));
  uint32_t flags = 0;
  check(sfi_read_errors(&view.cache(), &flags, stream));
}

}  // namespace

KvStore::KvStore(const ModelSpec& spec) : KvStore(spec, CacheLimits{}, nullptr) {}

KvStore::KvStore(const ModelSpec& spec, const CacheLimits& limits, void* stream)
    : spec_(spec), limits_(limits), stream_(stream), layers_(spec.n_layers), mirror_(spec.n_layers) {
  spec.validate();
  limits.validate();
  const sfi_shape s = store_shape(spec, limits);
  check(sfi_shape_validate(&s));
  dev_ = std::make_unique<DeviceCache>(s);
  for (auto& m : mirror_) {
    m.compact.resize(spec.n_kv_heads);
    m.compact_fresh.assign(spec.n_kv_heads, false);
  }
}

KvStore::~KvStore() = default;

void KvStore::set_window(int n_sink_b, int recent_len, Pos len) const {
  if (len < 0) len = len_;
  if (n_sink_b == cur_nsb_ && recent_len == cur_rl_ && len == cur_len_) return;
  const int32_t L = len, nsb = n_sink_b, rl = recent_len;
  check(sfi_set_lengths(&dev_->shape(), &dev_->cache(), &L, &nsb, &rl, stream_));
  cur_nsb_ = n_sink_b;
  cur_rl_ = recent_len;
  cur_len_ = len;
}

std::vector<double> KvStore::key_norms(int layer, int head, Pos first, int count) const {
  std::vector<double> out(static_cast<size_t>(std::max(count, 0)));
  if (count <= 0) return out;
  const Pos visible = len_ + (pending_layers_ > layer ? 1 : 0);
  if (first < 1 || first + count - 1 > visible) fail(ErrorCode::kOutOfRange, "KvStore: key norm range not written");
  const size_t off = (static_cast<size_t>(layer) * spec_.n_kv_heads + head) * spec_.max_positions + (first - 1);
  cuda_check(cudaStreamSynchronize(st(stream_)), "key_norms");
  cuda_check(cudaMemcpy(out.data(), dev_->cache().key_norms + off, out.size() * 8, cudaMemcpyDeviceToHost),
             "key_norms");
  return out;
}

void KvStore::begin_token() {
  if (pending_layers_ != -1) fail(ErrorCode::kOutOfRange, "KvStore: token already open");
  if (len_ >= spec_.max_positions) fail(ErrorCode::kContextOverflow, "KvStore: max_positions exceeded");
  pending_layers_ = 0;
}

void KvStore::append_layer(int layer, const float* k, const float* v) {
  if (pending_layers_ != layer) fail(ErrorCode::kOutOfRange, "KvStore: layers must be appended in order");
  const int hd = spec_.n_kv_heads * spec_.head_dim;
  std::vector<uint16_t> hk(hd), hv(hd);
  for (int i = 0; i < hd; ++i) {
    hk[i] = to_bf16(k[i]);
    hv[i] = to_bf16(v[i]);
  }
  set_window(std::max(cur_nsb_, 0), 0);
  uint16_t* d = static_cast<uint16_t*>(t_scratch.get(al(hd * 2) * 2));
  cuda_check(cudaMemcpyAsync(d, hk.data(), hd * 2, cudaMemcpyHostToDevice, st(stream_)), "append_layer");
  cuda_check(cudaMemcpyAsync(d + al(hd * 2) / 2, hv.data(), hd * 2, cudaMemcpyHostToDevice, st(stream_)),
             "append_layer");
  check(sfi_append_block(&dev_->shape(), &dev_->cache(), layer, 1, d, d + al(hd * 2) / 2, stream_));
  cuda_check(cudaStreamSynchronize(st(stream_)), "append_layer");
  ++pending_layers_;
}

void KvStore::end_token() {
  if (pending_layers_ != spec_.n_layers)
    fail(ErrorCode::kOutOfRange, "KvStore: token closed before all layers were appended");
  pending_layers_ = -1;
  ++len_;
}

void KvStore::append_tokens(int count, const float* k, const float* v) {
  if (pending_layers_ != -1) fail(ErrorCode::kOutOfRange, "KvStore: token already open");
  if (count < 0) fail(ErrorCode::kOutOfRange, "KvStore: negative token count");
  if (len_ + count > spec_.max_positions) fail(ErrorCode::kContextOverflow, "KvStore: max_positions exceeded");
  if (count == 0) return;
  const int H = spec_.n_kv_heads, d = spec_.head_dim;
  const size_t per = static_cast<size_t>(count) * H * d;
  std::vector<uint16_t> hk(per), hv(per);
  set_window(std::max(cur_nsb_, 0), 0);
  uint16_t* dk = static_cast<uint16_t*>(t_scratch.get(al(per * 2) * 2));
  uint16_t* dv = dk + al(per * 2) / 2;
  for (int l = 0; l < spec_.n_layers; ++l) {
    // [count][H][d] -> [H][count][d]
    const float* kl = k + static_cast<size_t>(l) * per;
    const float* vl = v + static_cast<size_t>(l) * per;
    for (int t = 0; t < count; ++t)
      for (int h = 0; h < H; ++h)
        for (int c = 0; c < d; ++c) {
          const size_t src = (static_cast<size_t>(t) * H + h) * d + c;
          const size_t dst = (static_cast<size_t>(h) * count + t) * d + c;
          hk[dst] = to_bf16(kl[src]);
          hv[dst] = to_bf16(vl[src]);
        }
    cuda_check(cudaMemcpyAsync(dk, hk.data(), per * 2, cudaMemcpyHostToDevice, st(stream_)), "append_tokens");
    cuda_check(cudaMemcpyAsync(dv, hv.data(), per * 2, cudaMemcpyHostToDevice, st(stream_)), "append_tokens");
    check(sfi_append_block(&dev_->shape(), &dev_->cache(), l, count, dk, dv, stream_));
    cuda_check(cudaStreamSynchronize(st(stream_)), "append_tokens");
  }
  len_ += count;
}

// Host fp32 mirror of the written rows of `layer` ([pos][H][d], the reference's
// paged layout), extended incrementally: rows are immutable once written.
void KvStore::sync_host_rows(int layer) const {
  HostMirror& m = mirror_[layer];
  const Pos rows = len_ + (pending_layers_ > layer ? 1 : 0);
  if (rows <= m.rows) return;
  const int H = spec_.n_kv_heads, d = spec_.head_dim;
  const int count = rows - m.rows;
  const size_t hd = static_cast<size_t>(H) * d;
  std::vector<uint16_t> raw(static_cast<size_t>(count) * d);
  m.k.resize(static_cast<size_t>(rows) * hd);
  m.v.resize(static_cast<size_t>(rows) * hd);
  cuda_check(cudaStreamSynchronize(st(stream_)), "key_at");
  for (int which = 0; which < 2; ++which) {
    const uint16_t* base = static_cast<const uint16_t*>(which ? dev_->cache().v_cache : dev_->cache().k_cache);
    std::vector<float>& dst = which ? m.v : m.k;
    for (int h = 0; h < H; ++h) {
      const size_t off = ((static_cast<size_t>(layer) * H + h) * spec_.max_positions + m.rows) * d;
      cuda_check(cudaMemcpy(raw.data(), base + off, raw.size() * 2, cudaMemcpyDeviceToHost), "key_at");
      for (int t = 0; t < count; ++t)
        for (int c = 0; c < d; ++c)
          dst[(static_cast<size_t>(m.rows) + t) * hd + static_cast<size_t>(h) * d + c] =
              from_bf16(raw[static_cast<size_t>(t) * d + c]);
    }
  }
  m.rows = rows;
}

const float* KvStore::key_at(int layer, Pos pos) const {
  const Pos rows = len_ + (pending_layers_ > layer ? 1 : 0);
  if (pos < 1 || pos > rows) fail(ErrorCode::kOutOfRange, "KvStore: position " + std::to_string(pos) + " not written");
  sync_host_rows(layer);
  return mirror_[layer].k.data() + static_cast<size_t>(pos - 1) * spec_.n_kv_heads * spec_.head_dim;
}

const float* KvStore::value_at(int layer, Pos pos) const {
  const Pos rows = len_ + (pending_layers_ > layer ? 1 : 0);
  if (pos < 1 || pos > rows) fail(ErrorCode::kOutOfRange, "KvStore: position " + std::to_string(pos) + " not written");
  sync_host_rows(layer);
  return mirror_[layer].v.data() + static_cast<size_t>(pos - 1) * spec_.n_kv_heads * spec_.head_dim;
}

std::vector<float> KvStore::key_row(int layer, Pos pos) const {
  const float* p = key_at(layer, pos);
  return std::vector<float>(p, p + static_cast<size_t>(spec_.n_kv_heads) * spec_.head_dim);
}

std::vector<float> KvStore::value_row(int layer, Pos pos) const {
  const float* p = value_at(layer, pos);
  return std::vector<float>(p, p + static_cast<size_t>(spec_.n_kv_heads) * spec_.head_dim);
}

double KvStore::key_norm(int layer, int head, Pos pos) const {
  const Pos rows = len_ + (pending_layers_ > layer ? 1 : 0);
  if (pos < 1 || pos > rows)
    fail(ErrorCode::kOutOfRange, "KvStore: no key norm for position " + std::to_string(pos));
  double v = 0.0;
  const size_t off = (static_cast<size_t>(layer) * spec_.n_kv_heads + head) * spec_.max_positions + (pos - 1);
  cuda_check(cudaStreamSynchronize(st(stream_)), "key_norm");
  cuda_check(cudaMemcpy(&v, dev_->cache().key_norms + off, 8, cudaMemcpyDeviceToHost), "key_norm");
  return v;
}

void KvStore::reorganize(int layer, const std::vector<Pos>& sink, const std::vector<std::vector<Pos>>& selected) {
  // attention.cpp:186-217: per head, merge, strictly increasing, written range
  const int H = spec_.n_kv_heads;
  if (static_cast<int>(selected.size()) != H)
    fail(ErrorCode::kSupportMismatch, "reorganize: selected sets must cover every KV head");
  std::vector<std::vector<Pos>> merged(H);
  size_t widest = 0;
  for (int h = 0; h < H; ++h) {
    std::merge(sink.begin(), sink.end(), selected[h].begin(), selected[h].end(), std::back_inserter(merged[h]));
    for (size_t i = 0; i + 1 < merged[h].size(); ++i)
      if (merged[h][i] >= merged[h][i + 1])
        fail(ErrorCode::kOverlapViolation, "reorganize: sink and selected sets overlap or are unsorted");
    for (Pos p : merged[h])
      if (p < 1 || p > len_) fail(ErrorCode::kOutOfRange, "reorganize: position " + std::to_string(p) + " not written");
    widest = std::max(widest, merged[h].size());
  }
  LayerState& ls = layers_[layer];
  const int m = static_cast<int>(sink.size());
  bool standard = m <= limits_.n_sink;
  for (int i = 0; standard && i < m; ++i) standard = sink[i] == i + 1;
  for (int h = 0; standard && h < H; ++h) standard = static_cast<int>(selected[h].size()) <= limits_.k_budget;
  if (standard) {
    // the production layout: sink rows {1..m} ahead of the selected rows (K3 compact_kernel)
    const int K = limits_.k_budget;
    std::vector<int32_t> sel(static_cast<size_t>(H) * std::max(K, 1), 0), cnt(H);
    for (int h = 0; h < H; ++h) {
      std::copy(selected[h].begin(), selected[h].end(), sel.begin() + static_cast<size_t>(h) * std::max(K, 1));
      cnt[h] = static_cast<int32_t>(selected[h].size());
    }
    set_window(m, 0);
    check(sfi_set_selection(&dev_->shape(), &dev_->cache(), layer, sel.data(), cnt.data(), stream_));
    uint32_t flags = 0;
    check(sfi_read_errors(&dev_->cache(), &flags, stream_));
    ls.view.reset();
  } else {
    // any other sink / size: the merged rows gathered into this layer's own view
    if (!ls.view || ls.view->shape().k_budget < static_cast<int>(widest))
      ls.view = layer_view(*dev_, layer, static_cast<int>(widest));
    gather_into(*ls.view, merged, len_, stream_);
  }
  ls.positions = std::move(merged);
  ls.valid = true;
  mirror_[layer].compact_fresh.assign(H, false);
}

bool KvStore::compact_matches(int layer, const std::vector<Pos>& sink,
                              const std::vector<std::vector<Pos>>& selected) const {
  const LayerState& l = layers_[layer];
  if (!l.valid) return false;
  if (static_cast<int>(selected.size()) != spec_.n_kv_heads) return false;
  for (int h = 0; h < spec_.n_kv_heads; ++h) {
    std::vector<Pos> merged;
    std::merge(sink.begin(), sink.end(), selected[h].begin(), selected[h].end(), std::back_inserter(merged));
    if (merged != l.positions[h]) return false;
  }
  return true;
}

int KvStore::compact_rows(int layer, int head) const {
  return layers_[layer].valid ? static_cast<int>(layers_[layer].positions[head].size()) : 0;
}

const KvStore::CompactSegment& KvStore::compact(int layer, int head) const {
  HostMirror& mm = mirror_[layer];
  CompactSegment& seg = mm.compact[head];
  const LayerState& l = layers_[layer];
  if (!l.valid) {
    seg = CompactSegment{};
    return seg;
  }
  if (mm.compact_fresh[head]) return seg;
  seg.positions = l.positions[head];
  const int d = spec_.head_dim;
  const size_t n = seg.positions.size();
  const DeviceCache& src = l.view ? *l.view : *dev_;
  const sfi_shape& s = src.shape();
  const int crows = s.n_recent + s.n_sink + s.k_budget;
  const int lay = l.view ? 0 : layer;
  const size_t row0 = (static_cast<size_t>(lay) * spec_.n_kv_heads + head) * crows + s.n_recent;
  std::vector<uint16_t> rk(n * d), rv(n * d);
  cuda_check(cudaStreamSynchronize(st(stream_)), "compact");
  if (n) {
    cuda_check(cudaMemcpy(rk.data(), static_cast<const uint16_t*>(src.cache().ck) + row0 * d, n * d * 2,
                          cudaMemcpyDeviceToHost), "compact");
    cuda_check(cudaMemcpy(rv.data(), static_cast<const uint16_t*>(src.cache().cv) + row0 * d, n * d * 2,
                          cudaMemcpyDeviceToHost), "compact");
  }
  seg.k.resize(n * d);
  seg.v.resize(n * d);
  for (size_t i = 0; i < n * d; ++i) {
    seg.k[i] = from_bf16(rk[i]);
    seg.v[i] = from_bf16(rv[i]);
  }
  mm.compact_fresh[head] = true;
  return seg;
}

std::pair<Pos, int> KvStore::recent_tail(int n_recent) const {
  const int len = std::min<int>(n_recent, len_);
  return {len_ - len + 1, len};
}

void KvStore::record_compact_access(int layer, int head, int slot) const {
  if (trace_on_) trace_.push_back({layer, head, slot});
}

// ---------------------------------------------------------------------------
// attention kernels (attention.cpp:502-550)

namespace {

struct DecodeIO {
  float* q;
  float* out;
};

DecodeIO stage_q(const KvStore& store, const std::vector<double>& q) {
  const ModelSpec& spec = store.spec();
  const size_t n = static_cast<size_t>(spec.n_query_heads) * spec.head_dim;
  if (q.size() != n) fail(ErrorCode::kSupportMismatch, "attention: q must hold n_query_heads * head_dim values");
  float* base = static_cast<float*>(t_scratch.get(al(n * 4) * 2));
  std::vector<float> qf(q.begin(), q.end());
  cuda_check(cudaMemcpyAsync(base, qf.data(), n * 4, cudaMemcpyHostToDevice, st(store.stream())), "attention");
  return {base, base + al(n * 4) / 4};
}

std::vector<double> fetch_out(const KvStore& store, const DeviceCache& dev, const DecodeIO& io) {
  const ModelSpec& spec = store.spec();
  const size_t n = static_cast<size_t>(spec.n_query_heads) * spec.head_dim;
  std::vector<float> o(n);
  cuda_check(cudaMemcpyAsync(o.data(), io.out, n * 4, cudaMemcpyDeviceToHost, st(store.stream())), "attention");
  cuda_check(cudaStreamSynchronize(st(store.stream())), "attention");
  uint32_t flags = 0;
  check(sfi_read_errors(&dev.cache(), &flags, store.stream()));
  return std::vector<double>(o.begin(), o.end());
}

}  // namespace

std::vector<double> attention_kernel_dense(const KvStore& store, int layer, const std::vector<double>& q,
                                           KernelStats* stats) {
  const ModelSpec& spec = store.spec();
  if (store.size() < 1) fail(ErrorCode::kOutOfRange, "KvStore: position 1 not written");
  store.set_window(0, 0);
  DecodeIO io = stage_q(store, q);
  check(sfi_dense_decode(&store.device().shape(), &store.device().cache(), layer, io.q, io.out, nullptr,
                         SFI_POOL_MEAN, store.stream()));
  std::vector<double> out = fetch_out(store, store.device(), io);
  if (stats) {
    stats->reads += static_cast<std::uint64_t>(spec.n_kv_heads) * store.size();
    stats->flops += 2ull * store.size() * spec.head_dim * spec.n_query_heads;
  }
  return out;
}

std::vector<double> attention_kernel_sparse(const KvStore& store, int layer, const std::vector<double>& q,
                                            const SupportSet& support, KernelStats* stats) {
  const ModelSpec& spec = store.spec();
  const int H = spec.n_kv_heads;
  if (!store.compact_matches(layer, support.sink, support.selected))
    fail(ErrorCode::kStaleCompact, "attention_kernel_sparse: compact buffer does not match the support");
  if (support.recent_len > 0 &&
      (support.recent_start < 1 || support.recent_start + support.recent_len - 1 > store.size()))
    fail(ErrorCode::kOutOfRange, "KvStore: position " + std::to_string(support.recent_start) + " not written");
  std::uint64_t reads = 0;
  for (int h = 0; h < H; ++h) {
    const int total = support.size_for_head(h);
    if (total == 0) fail(ErrorCode::kEmptySupport, "sparse_attention_step: empty support");
    reads += static_cast<std::uint64_t>(total);
  }
  const auto& ls = store.layers_[layer];
  const int R = store.device().shape().n_recent;
  const bool tail = support.recent_len == 0 || support.recent_start + support.recent_len - 1 == store.size();
  DecodeIO io = stage_q(store, q);
  std::vector<double> out;
  if (!ls.view && tail && support.recent_len <= R) {
    // production layout: compact rows + the recent ring, one K4 launch
    store.set_window(static_cast<int>(support.sink.size()), support.recent_len);
    check(sfi_sparse_decode(&store.device().shape(), &store.device().cache(), layer, io.q, io.out, store.stream()));
    out = fetch_out(store, store.device(), io);
  } else {
    // general support: sink + selected + the recent range gathered into one view
    std::vector<std::vector<Pos>> rows(H);
    size_t widest = 0;
    for (int h = 0; h < H; ++h) {
      rows[h] = ls.positions[h];
      for (int i = 0; i < support.recent_len; ++i) rows[h].push_back(support.recent_start + i);
      std::sort(rows[h].begin(), rows[h].end());
      if (std::adjacent_find(rows[h].begin(), rows[h].end()) != rows[h].end())
        fail(ErrorCode::kUnsupported, "attention_kernel_sparse: the recent range overlaps the compact segment");
      widest = std::max(widest, rows[h].size());
    }
    auto& view = store.support_view_;
    if (!view || view->shape().k_budget < static_cast<int>(widest) ||
        view->cache().k_cache != static_cast<const uint8_t*>(store.device().cache().k_cache) +
                                     static_cast<size_t>(layer) * H * spec.max_positions * spec.head_dim * 2)
      view = layer_view(store.device(), layer, static_cast<int>(widest));
    gather_into(*view, rows, store.size(), store.stream());
    check(sfi_sparse_decode(&view->shape(), &view->cache(), 0, io.q, io.out, store.stream()));
    out = fetch_out(store, *view, io);
  }
  if (store.trace_on())  // compact reads in the reference's order (attend per q head, attention.cpp:88-96)
    for (int h = 0; h < H; ++h)
      for (int g = 0; g < spec.group_size(); ++g)
        for (int slot = 0; slot < static_cast<int>(ls.positions[h].size()); ++slot)
          store.record_compact_access(layer, h, slot);
  if (stats) {
    stats->reads += reads;
    for (int h = 0; h < H; ++h) stats->flops += 2ull * support.size_for_head(h) * spec.head_dim * spec.group_size();
  }
  return out;
}

DenseCapture dense_capture(const KvStore& store, int layer, const std::vector<double>& q,
                           const std::vector<Pos>& allowed, PoolMode pool) {
  const ModelSpec& spec = store.spec();
  const Pos L = store.size();
  if (L < 1) fail(ErrorCode::kOutOfRange, "KvStore: position 1 not written");
  for (size_t i = 0; i < allowed.size(); ++i) {
    if (allowed[i] < 1 || allowed[i] > L)
      fail(ErrorCode::kOutOfRange,
           "dense_attention_step: allowed position " + std::to_string(allowed[i]) + " out of range");
    if (i && allowed[i] <= allowed[i - 1]) fail(ErrorCode::kOutOfRange, "dense_capture: allowed must be ascending");
  }
  const int nJ = static_cast<int>(allowed.size());
  // pooled logits over the hull [allowed.front(), allowed.back()] = the device's
  // J = [n_sink_b + 1, L - recent_len]; the allowed columns are picked from it
  const int nsb = nJ ? allowed.front() - 1 : 0;
  const int rl = nJ ? L - allowed.back() : 0;
  const int hull = nJ ? allowed.back() - allowed.front() + 1 : 0;
  DenseCapture cap;
  cap.window.width = 1;
  cap.window.allowed = allowed;
  cap.window.values.assign(spec.n_kv_heads, std::vector<double>(nJ));
  store.set_window(nsb, rl);
  DecodeIO io = stage_q(store, q);
  float* logits = store.device().logits();
  check(sfi_dense_decode(&store.device().shape(), &store.device().cache(), layer, io.q, io.out,
                         nJ ? logits : nullptr, pool == PoolMode::kMax ? SFI_POOL_MAX : SFI_POOL_MEAN, store.stream()));
  cap.context = fetch_out(store, store.device(), io);
  if (nJ) {
    std::vector<float> lg(static_cast<size_t>(hull));
    for (int h = 0; h < spec.n_kv_heads; ++h) {
      cuda_check(cudaMemcpy(lg.data(), logits + static_cast<size_t>(h) * spec.max_positions, hull * 4,
                            cudaMemcpyDeviceToHost), "dense_capture");
      for (int c = 0; c < nJ; ++c) cap.window.values[h][c] = lg[allowed[c] - allowed.front()];
    }
  }
  return cap;
}

// ---------------------------------------------------------------------------
// scheduler (scheduler.cpp:28-145): host-side integer bookkeeping

std::string step_record_to_json(const StepRecord& rec) {
  std::ostringstream os;
  os << "{\"t\":" << rec.t << ",\"type\":\"" << (rec.slow ? "slow" : "fast") << '"';
  if (rec.cause == StepCause::kInitial) os << ",\"cause\":\"initial\"";
  if (rec.cause == StepCause::kTrigger) os << ",\"cause\":\"trigger\"";
  if (rec.cause == StepCause::kForced) os << ",\"cause\":\"forced\"";
  os << ",\"support_size\":" << rec.support_size << ",\"allowed_size\":" << rec.allowed_size << "}";
  return os.str();
}

std::vector<Pos> SparseState::recent() const {
  std::vector<Pos> out(static_cast<size_t>(recent_len));
  std::iota(out.begin(), out.end(), recent_start);
  return out;
}

SupportSet SparseState::support() const {
  SupportSet s;
  s.sink = sink;
  s.selected = selected;
  s.recent_start = recent_start;
  s.recent_len = recent_len;
  return s;
}

namespace {

void slide(SparseState& s, Pos prefix_len, const CacheLimits& limits) {
  int32_t rs = 0, rl = 0;
  sfi_recent_window(prefix_len, static_cast<int32_t>(s.sink.size()), limits.n_recent, &rs, &rl);
  s.recent_len = rl;
  s.recent_start = rs;
}

bool in_recent(const SparseState& s, Pos p) { return p >= s.recent_start && p < s.recent_start + s.recent_len; }

}  // namespace

DecodeState init_decode_state(Pos prompt_len, int n_layers, int n_kv_heads, const CacheLimits& limits) {
  limits.validate();
  if (prompt_len < 1) fail(ErrorCode::kOutOfRange, "init_decode_state: empty prompt");
  DecodeState state;
  state.prefix_len = prompt_len;
  state.g = 1;
  state.per_layer.resize(static_cast<size_t>(n_layers));
  const int n_sink = std::min<int>(limits.n_sink, prompt_len);
  for (int l = 0; l < n_layers; ++l) {
    SparseState& s = state.per_layer[l];
    s.layer = l;
    s.sink.resize(static_cast<size_t>(n_sink));
    std::iota(s.sink.begin(), s.sink.end(), Pos{1});
    s.selected.assign(static_cast<size_t>(n_kv_heads), {});
    slide(s, prompt_len, limits);
  }
  return state;
}

std::vector<Pos> compute_allowed(const SparseState& state, Pos prefix_len) {
  if (prefix_len < 1) fail(ErrorCode::kOutOfRange, "compute_allowed: prefix_len must be >= 1");
  std::vector<Pos> out;
  for (Pos p = 1; p <= prefix_len; ++p) {
    if (std::binary_search(state.sink.begin(), state.sink.end(), p)) continue;
    if (in_recent(state, p)) continue;
    out.push_back(p);
  }
  return out;
}

int next_step_type(const DecodeState& state, const TriggerConfig& trig) {
  if (trig.is_trigger(state.last_token)) return 1;
  if (state.steps_since_slow + 1 >= trig.t_max) return 1;
  return 0;
}

void fast_step_update(DecodeState& state, const CacheLimits& limits) {
  state.t += 1;
  state.prefix_len += 1;
  state.steps_since_slow += 1;
  for (SparseState& s : state.per_layer) slide(s, state.prefix_len, limits);
}

void slow_step_update(DecodeState& state, const std::vector<std::vector<std::vector<Pos>>>& selected_per_layer,
                      const CacheLimits& limits) {
  if (selected_per_layer.size() != state.per_layer.size())
    fail(ErrorCode::kSupportMismatch, "slow_step_update: one selected set per layer required");
  for (size_t l = 0; l < state.per_layer.size(); ++l) {
    SparseState& s = state.per_layer[l];
    for (const std::vector<Pos>& head_sel : selected_per_layer[l]) {
      if (static_cast<int>(head_sel.size()) > limits.k_budget)
        fail(ErrorCode::kOutOfRange, "slow_step_update: selected set exceeds k_budget");
      for (Pos p : head_sel)
        if (std::binary_search(s.sink.begin(), s.sink.end(), p) || in_recent(s, p))
          fail(ErrorCode::kOverlapViolation,
               "slow_step_update: selected position " + std::to_string(p) + " overlaps sink or recent");
    }
    s.selected = selected_per_layer[l];
  }
  state.t += 1;
  state.prefix_len += 1;
  state.steps_since_slow = 0;
  for (SparseState& s : state.per_layer) slide(s, state.prefix_len, limits);
}

double flop_model(double prefix_len, double support, double slow_fraction) {
  if (!(support > 0.0) || support > prefix_len)
    fail(ErrorCode::kOutOfRange, "flop_model: support must be in (0, L]");
  if (slow_fraction < 0.0 || slow_fraction > 1.0)
    fail(ErrorCode::kOutOfRange, "flop_model: slow_fraction must be in [0, 1]");
  const double mixed = slow_fraction * prefix_len + (1.0 - slow_fraction) * support;
  return prefix_len / mixed;
}

}  // namespace sfi
