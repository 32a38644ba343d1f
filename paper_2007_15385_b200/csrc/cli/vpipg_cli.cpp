// vpipg_cli.cpp -- `vpipg`, the B200 drop-in for the reference CLI's data
// path (proj/tools/vpip.cpp:114-152 `vpip test`, :105-112 `convert`,
// :154-164 `validate`), SURVEY.md §8(f)3.
//
//   vpipg test     --polygon P --points F --engine voronoi|offset|crossing
//                  [--format csv|binary] [--out O] [--dtype f64|f32]
//   vpipg convert  --polygon P [--out O]
//   vpipg validate --polygon P [--points F] [--count N] [--seed S] [--band B]
//   vpipg bench    [--edges 3..15] [--batch N] [--reps R] [--seed S]
//                  [--engines voronoi,sign_of_offset,ray_crossing] [--threads T] [--out O]
//
// `bench` is run_benchmark (bench.cpp:115-222) over the drop-in: the same
// regular n-gons, batches, discarded warm-ups, seeded shuffled repetition
// order and CSV schema (bench.cpp:224-234), with every batch call going
// through the vpip:: API to the B200 (host f64 batch in, byte mask out);
// `--threads` is accepted and ignored, as in the C++ shim.
//
// File formats are the reference's (io.hpp:24-40): polygon JSON
// {"vertices": [[x, y], ...]} or headerless "x,y" CSV (sniffed); points "x,y"
// CSV or PIPB (16-byte header "PIPB", u32 version 1, u64 count, interleaved
// f64 pairs); masks one 0/1 per CSV row or PIPM (same header convention, bits
// LSB-first). The binary mask payload is written straight from the engine's
// ballot words: bit j of the payload is point j in both. Exit codes match the
// reference: 0 ok, 2 on any input / usage / device error. The default dtype is
// f64, the reference-exact kernels, so masks equal `vpip test` bit for bit.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "vpip/engines.hpp"
#include "vpip/sampling.hpp"
#include "vpip/voronoi.hpp"
#include "vpipg.h"

namespace {

struct Fail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Fail("parse error: cannot read '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

double number(std::string_view s) {
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
  double v = 0;
  const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc{} || p != s.data() + s.size()) throw Fail("parse error: bad number '" + std::string(s) + "'");
  if (!std::isfinite(v)) throw Fail("non-finite value");
  return v;
}

void parse_csv(const std::string& text, std::vector<double>& xs, std::vector<double>& ys) {
  size_t pos = 0;
  while (pos < text.size()) {
    size_t eol = text.find('\n', pos);
    if (eol == std::string::npos) eol = text.size();
    std::string_view line(text.data() + pos, eol - pos);
    pos = eol + 1;
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.remove_suffix(1);
    if (line.empty()) continue;
    const size_t c = line.find(',');
    if (c == std::string_view::npos) throw Fail("parse error: expected 'x,y'");
    xs.push_back(number(line.substr(0, c)));
    ys.push_back(number(line.substr(c + 1)));
  }
}

// {"vertices": [[x, y], ...]}: the numbers of the "vertices" array, in pairs.
void parse_polygon_json(const std::string& text, std::vector<double>& xs, std::vector<double>& ys) {
  const size_t key = text.find("\"vertices\"");
  if (key == std::string::npos) throw Fail("parse error: polygon JSON needs \"vertices\"");
  size_t p = text.find('[', key);
  if (p == std::string::npos) throw Fail("parse error: invalid JSON");
  int depth = 0;
  std::vector<double> nums;
  for (; p < text.size(); ++p) {
    const char ch = text[p];
    if (ch == '[') ++depth;
    else if (ch == ']') {
      if (--depth == 0) break;
    } else if (ch == '-' || ch == '+' || ch == '.' || (ch >= '0' && ch <= '9')) {
      size_t e = p;
      while (e < text.size() && std::strchr("+-.0123456789eE", text[e])) ++e;
      nums.push_back(number(std::string_view(text).substr(p, e - p)));
      p = e - 1;
    } else if (!std::strchr(" \t\r\n,", ch)) {
      throw Fail("parse error: invalid JSON");
    }
  }
  if (depth != 0 || nums.size() % 2) throw Fail("parse error: expected [x, y] pairs");
  for (size_t i = 0; i < nums.size(); i += 2) {
    xs.push_back(nums[i]);
    ys.push_back(nums[i + 1]);
  }
}

void read_polygon(const std::string& path, std::vector<double>& xs, std::vector<double>& ys) {
  const std::string text = read_file(path);
  const size_t first = text.find_first_not_of(" \t\r\n");
  if (first != std::string::npos && text[first] == '{') parse_polygon_json(text, xs, ys);
  else parse_csv(text, xs, ys);
}

struct Header {
  char magic[4];
  uint32_t version;
  uint64_t count;
};
static_assert(sizeof(Header) == 16);

void read_points(const std::string& path, std::vector<double>& xs, std::vector<double>& ys) {
  const std::string text = read_file(path);
  if (text.size() >= 4 && std::memcmp(text.data(), "PIPB", 4) == 0) {
    if (text.size() < sizeof(Header)) throw Fail("parse error: truncated point stream");
    Header h;
    std::memcpy(&h, text.data(), sizeof h);
    if (h.version != 1) throw Fail("parse error: unsupported point stream version");
    if (text.size() != sizeof(Header) + 16 * h.count) throw Fail("parse error: truncated point stream");
    xs.resize(h.count);
    ys.resize(h.count);
    const char* p = text.data() + sizeof(Header);
    for (uint64_t j = 0; j < h.count; ++j) {  // interleaved f64 (x, y)
      std::memcpy(&xs[j], p + 16 * j, 8);
      std::memcpy(&ys[j], p + 16 * j + 8, 8);
      if (!std::isfinite(xs[j]) || !std::isfinite(ys[j])) throw Fail("non-finite value");
    }
    return;
  }
  parse_csv(text, xs, ys);
}

void check(int rc) {
  if (rc) throw Fail(vpipg_strerror(rc));
}

struct Handle {
  vpipg_poly* p = nullptr;
  ~Handle() { vpipg_destroy(p); }
};

std::ostream& output(const std::string& path, std::ofstream& file) {
  if (path.empty()) return std::cout;
  file.open(path, std::ios::binary);
  if (!file) throw Fail("parse error: cannot write '" + path + "'");
  return file;
}

int cmd_test(std::map<std::string, std::string>& o) {
  const std::string engine = o["--engine"], format = o.count("--format") ? o["--format"] : "csv";
  const int e = engine == "voronoi" ? VPIPG_ENGINE_VORONOI
                : engine == "offset" ? VPIPG_ENGINE_OFFSET
                : engine == "crossing" ? VPIPG_ENGINE_CROSSING
                                       : -1;
  if (e < 0 || (format != "csv" && format != "binary") || !o.count("--polygon") || !o.count("--points"))
    throw Fail("usage: vpipg test --polygon P --points F --engine voronoi|offset|crossing");
  std::vector<double> vx, vy, xs, ys;
  read_polygon(o["--polygon"], vx, vy);
  read_points(o["--points"], xs, ys);
  const uint32_t kind = e == VPIPG_ENGINE_VORONOI ? VPIPG_KIND_VORONOI
                        : e == VPIPG_ENGINE_OFFSET ? VPIPG_KIND_OFFSET
                                                   : VPIPG_KIND_CROSSING;
  if (e == VPIPG_ENGINE_CROSSING && vx.size() < 3) check(1);  // vpip.cpp:121-123
  Handle h;
  check(vpipg_prepare(vx.data(), vy.data(), static_cast<uint32_t>(vx.size()), kind, 0, nullptr, &h.p));
  const uint64_t m = xs.size();
  std::vector<uint32_t> words((m + 31) / 32);
  uint64_t inside = 0;
  if (o.count("--dtype") && o["--dtype"] == "f32") {
    std::vector<float> fx(xs.begin(), xs.end()), fy(ys.begin(), ys.end());
    check(vpipg_test_host(h.p, e, VPIPG_F32, fx.data(), fy.data(), m, words.data(), nullptr, &inside));
  } else {
    check(vpipg_test_host(h.p, e, VPIPG_F64, xs.data(), ys.data(), m, words.data(), nullptr, &inside));
  }
  std::ofstream file;
  std::ostream& out = output(o.count("--out") ? o["--out"] : "", file);
  if (format == "binary") {  // PIPM: the ballot words are the payload (io.cpp:272-279)
    Header hd{{'P', 'I', 'P', 'M'}, 1, m};
    out.write(reinterpret_cast<const char*>(&hd), sizeof hd);
    out.write(reinterpret_cast<const char*>(words.data()), static_cast<std::streamsize>((m + 7) / 8));
  } else {
    std::string s;
    s.reserve(2 * m);
    for (uint64_t j = 0; j < m; ++j) {
      s.push_back(((words[j >> 5] >> (j & 31)) & 1u) ? '1' : '0');
      s.push_back('\n');
    }
    out << s;
  }
  std::cerr << inside << " of " << m << " points inside\n";
  return 0;
}

int cmd_convert(std::map<std::string, std::string>& o) {
  if (!o.count("--polygon")) throw Fail("usage: vpipg convert --polygon P [--out O]");
  std::vector<double> vx, vy;
  read_polygon(o["--polygon"], vx, vy);
  Handle h;
  check(vpipg_prepare(vx.data(), vy.data(), static_cast<uint32_t>(vx.size()), VPIPG_KIND_VORONOI, 0,
                      nullptr, &h.p));
  int reversed = 0;
  vpipg_poly_info(h.p, nullptr, nullptr, &reversed);
  if (reversed) std::cerr << "note: input was clockwise, reversed to counter-clockwise\n";
  std::vector<double> outer(2 * vx.size());
  double inner[2];
  check(vpipg_poly_generators(h.p, inner, outer.data()));
  char buf[96];
  std::string s = "{\"inner\": [";
  std::snprintf(buf, sizeof buf, "%.17g, %.17g], \"outer\": [", inner[0], inner[1]);
  s += buf;
  for (size_t k = 0; k < vx.size(); ++k) {
    std::snprintf(buf, sizeof buf, "%s[%.17g, %.17g]", k ? ", " : "", outer[2 * k], outer[2 * k + 1]);
    s += buf;
  }
  s += "]}\n";
  std::ofstream file;
  output(o.count("--out") ? o["--out"] : "", file) << s;
  return 0;
}

int cmd_validate(std::map<std::string, std::string>& o) {
  if (!o.count("--polygon")) throw Fail("usage: vpipg validate --polygon P [--points F]");
  std::vector<double> vx, vy, xs, ys;
  read_polygon(o["--polygon"], vx, vy);
  std::vector<vpip::Point2> v;
  for (size_t i = 0; i < vx.size(); ++i) v.push_back({vx[i], vy[i]});
  const vpip::ConvexPolygon poly = vpip::validate_polygon(v);  // throws vpip::Error
  std::vector<double> cvx, cvy;
  for (const vpip::Point2& p : poly.vertices()) {
    cvx.push_back(p.x);
    cvy.push_back(p.y);
  }
  if (o.count("--points")) {
    read_points(o["--points"], xs, ys);
  } else {
    const size_t count = o.count("--count") ? std::stoull(o["--count"]) : 100000;
    const uint64_t seed = o.count("--seed") ? std::stoull(o["--seed"]) : 42;
    const vpip::PointBatch b = vpip::sample_points(count, vpip::bounding_box(poly.vertices()).scaled(2.0), seed);
    xs = b.xs;
    ys = b.ys;
  }
  const double band = o.count("--band") ? number(o["--band"]) : 1e-9;
  Handle h;
  check(vpipg_prepare(cvx.data(), cvy.data(), static_cast<uint32_t>(cvx.size()), VPIPG_KIND_ALL, 0,
                      nullptr, &h.p));
  const uint64_t m = xs.size();
  // device copies of the batch, then run_validation on the device
  void* dx = nullptr;
  void* dy = nullptr;
  if (cudaMalloc(&dx, std::max<uint64_t>(m, 1) * 8) || cudaMalloc(&dy, std::max<uint64_t>(m, 1) * 8))
    throw Fail("device allocation failed");
  cudaMemcpy(dx, xs.data(), m * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, ys.data(), m * 8, cudaMemcpyHostToDevice);
  vpipg_report rep;
  const int rc = vpipg_validate(h.p, VPIPG_F64, dx, dy, m, band, 0, &rep, nullptr);
  cudaFree(dx);
  cudaFree(dy);
  check(rc);
  // print_validation_report (bench.cpp:310-338)
  std::cout << "points tested:        " << rep.point_count << "\n";
  const char* names[3] = {"voronoi vs offset:    ", "voronoi vs crossing:  ", "offset vs crossing:   "};
  for (int i = 0; i < 3; ++i)
    std::cout << names[i] << rep.point_count - rep.pair_disagreements[i] << " agree, "
              << rep.pair_disagreements[i] << " differ\n";
  std::cout << "disagreeing points:   " << rep.disagreeing_points << "\n";
  if (rep.n_samples) {
    std::cout << "first " << rep.n_samples
              << " disagreements (v/o/c, distance to nearest edge line):\n";
    for (uint32_t i = 0; i < rep.n_samples; ++i) {
      const uint64_t j = rep.sample_index[i];
      const uint32_t b = rep.sample_engines[i];
      char line[160];
      std::snprintf(line, sizeof line, "  #%llu (%.17g, %.17g) %u/%u/%u dist=%.3g\n",
                    static_cast<unsigned long long>(j), xs[j], ys[j], b & 1u, (b >> 1) & 1u,
                    (b >> 2) & 1u, rep.sample_dist[i]);
      std::cout << line;
    }
  }
  std::cout << "verdict:              " << (rep.pass ? "PASS" : "FAIL");
  if (rep.pass && rep.disagreeing_points > 0) std::cout << " (all disagreements within the boundary band)";
  std::cout << "\n";
  return rep.pass ? 0 : 1;
}

// "3..15", "7" or "3,5,9" (vpip.cpp:46-77)
std::vector<int> parse_edge_spec(const std::string& spec) {
  std::vector<int> counts;
  std::stringstream ss(spec);
  std::string tok;
  auto to_int = [](const std::string& t) {
    int v = 0;
    const auto [ptr, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    if (ec != std::errc{} || ptr != t.data() + t.size()) throw Fail("bad edge count '" + t + "'");
    return v;
  };
  while (std::getline(ss, tok, ',')) {
    if (tok.empty()) continue;
    const size_t dots = tok.find("..");
    if (dots == std::string::npos) {
      counts.push_back(to_int(tok));
    } else {
      const int lo = to_int(tok.substr(0, dots)), hi = to_int(tok.substr(dots + 2));
      if (hi < lo) throw Fail("empty edge range '" + tok + "'");
      for (int n = lo; n <= hi; ++n) counts.push_back(n);
    }
  }
  return counts;
}

int cmd_bench(std::map<std::string, std::string>& o) {
  const std::vector<int> edges = parse_edge_spec(o.count("--edges") ? o["--edges"] : "3..15");
  const size_t batch = o.count("--batch") ? std::stoull(o["--batch"]) : 1000000;
  const int reps = o.count("--reps") ? std::stoi(o["--reps"]) : 10;
  const uint64_t seed = o.count("--seed") ? std::stoull(o["--seed"]) : 42;
  const int threads = o.count("--threads") ? std::stoi(o["--threads"]) : 1;
  std::vector<vpip::EngineKind> engines;
  {
    std::stringstream ss(o.count("--engines") ? o["--engines"]
                                              : "voronoi,sign_of_offset,ray_crossing");
    std::string tok;
    while (std::getline(ss, tok, ',')) {
      if (tok.empty()) continue;
      const std::optional<vpip::EngineKind> k = vpip::parse_engine(tok);
      if (!k) throw Fail("unknown engine '" + tok + "'");
      engines.push_back(*k);
    }
  }
  // check_config (bench.cpp:48-67)
  if (edges.empty()) throw Fail("no edge counts configured");
  for (int n : edges)
    if (n < 3) throw Fail("edge count " + std::to_string(n) + " is below 3");
  if (batch < 1 || reps < 1 || threads < 1 || engines.empty()) throw Fail("bad bench configuration");

  using Clock = std::chrono::steady_clock;
  auto ns_since = [](Clock::time_point t0) {
    return std::max<uint64_t>(1, std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
  };
  struct Work {
    vpip::ConvexPolygon polygon;
    vpip::PointBatch batch;
  };
  std::vector<Work> work;
  for (int n : edges) {
    vpip::ConvexPolygon poly = vpip::regular_polygon(static_cast<size_t>(n), 1.0);
    const vpip::Box box = vpip::bounding_box(poly.vertices()).scaled(2.0);
    vpip::PointBatch b = vpip::sample_points(batch, box, vpip::mix_seed(seed, static_cast<uint64_t>(n)));
    work.push_back({std::move(poly), std::move(b)});
  }
  struct Rec {
    vpip::EngineKind engine;
    int n;
    size_t batch;
    int rep;
    bool convert;
    uint64_t ns;
  };
  struct Pair {
    std::optional<Rec> convert;
    std::vector<Rec> queries;
    vpip::GeneratorSet gen;
  };
  std::vector<std::vector<Pair>> res(engines.size(), std::vector<Pair>(edges.size()));
  uint64_t sink = 0;
  auto run_once = [&](vpip::EngineKind e, const Work& w, const vpip::GeneratorSet& g) {
    switch (e) {
      case vpip::EngineKind::Voronoi: return vpip::voronoi_contains_batch(g, w.batch, threads);
      case vpip::EngineKind::SignOfOffset:
        return vpip::sign_of_offset_contains_batch(w.polygon, w.batch, threads);
      default: return vpip::ray_crossing_contains_batch(w.polygon.vertices(), w.batch, threads);
    }
  };
  for (size_t e = 0; e < engines.size(); ++e)
    for (size_t i = 0; i < edges.size(); ++i) {
      Pair& pr = res[e][i];
      if (engines[e] == vpip::EngineKind::Voronoi) {
        const auto t0 = Clock::now();
        pr.gen = vpip::to_voronoi(work[i].polygon);
        pr.convert = Rec{engines[e], edges[i], 0, 0, true, ns_since(t0)};
      }
      sink += vpip::count_inside(run_once(engines[e], work[i], pr.gen));  // discarded warm-up
    }
  std::vector<std::pair<size_t, size_t>> order;
  for (size_t e = 0; e < engines.size(); ++e)
    for (size_t i = 0; i < edges.size(); ++i) order.emplace_back(e, i);
  for (int rep = 0; rep < reps; ++rep) {
    std::mt19937_64 rng(vpip::mix_seed(seed, 0x0bef0000u + static_cast<unsigned>(rep)));
    std::shuffle(order.begin(), order.end(), rng);
    for (const auto& [e, i] : order) {
      const auto t0 = Clock::now();
      const vpip::InclusionMask mask = run_once(engines[e], work[i], res[e][i].gen);
      res[e][i].queries.push_back(Rec{engines[e], edges[i], batch, rep, false, ns_since(t0)});
      sink += vpip::count_inside(mask);
    }
  }
  std::ostringstream csv;
  csv << "engine,n_edges,batch_size,repetition,phase,wall_time_ns,throughput_pts_per_s\n";
  std::map<std::pair<int, int>, std::vector<double>> med;
  for (size_t e = 0; e < engines.size(); ++e)
    for (size_t i = 0; i < edges.size(); ++i) {
      std::vector<Rec> rs;
      if (res[e][i].convert) rs.push_back(*res[e][i].convert);
      rs.insert(rs.end(), res[e][i].queries.begin(), res[e][i].queries.end());
      for (const Rec& r : rs) {
        const double tp = r.batch ? static_cast<double>(r.batch) / (static_cast<double>(r.ns) * 1e-9) : 0.0;
        char buf[64];
        std::snprintf(buf, sizeof buf, "%.17g", tp);
        csv << vpip::engine_name(r.engine) << ',' << r.n << ',' << r.batch << ',' << r.rep << ','
            << (r.convert ? "convert" : "query") << ',' << r.ns << ',' << buf << '\n';
        if (!r.convert) med[{static_cast<int>(e), r.n}].push_back(static_cast<double>(r.ns));
      }
    }
  std::ofstream file;
  output(o.count("--out") ? o["--out"] : "", file) << csv.str();
  std::cerr << "engine          n   median ms   median pts/s\n";
  for (auto& [key, v] : med) {
    std::sort(v.begin(), v.end());
    const size_t k = v.size();
    const double ns = k % 2 ? v[k / 2] : 0.5 * (v[k / 2 - 1] + v[k / 2]);
    char line[128];
    std::snprintf(line, sizeof line, "%-14s %3d   %9.3f   %.4g\n",
                  std::string(vpip::engine_name(engines[key.first])).c_str(), key.second, ns * 1e-6,
                  static_cast<double>(batch) / (ns * 1e-9));
    std::cerr << line;
  }
  (void)sink;
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: vpipg test|convert|validate|bench [options]\n";
    return 2;
  }
  const std::string cmd = argv[1];
  std::map<std::string, std::string> opts;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--", 0) != 0 || i + 1 >= argc) {
      std::cerr << "error: bad argument '" << a << "'\n";
      return 2;
    }
    opts[a] = argv[++i];
  }
  try {
    if (cmd == "test") return cmd_test(opts);
    if (cmd == "convert") return cmd_convert(opts);
    if (cmd == "validate") return cmd_validate(opts);
    if (cmd == "bench") return cmd_bench(opts);
    std::cerr << "error: unknown subcommand '" << cmd << "'\n";
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
  }
  return 2;
}
