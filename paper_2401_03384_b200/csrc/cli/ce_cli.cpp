// ce_cli: the SPEC command-line interface (the reference ships only a
// placeholder for it, proj/tools/CMakeLists.txt) over libce's C-ABI (include/ce/ce.h).
//
//   ce_cli analyze --expr STR --shapes JSON | --layer JSON [--cr X]  [--mode M] [--cost C] [--json]
//   ce_cli eval    --expr STR --shapes JSON --seed N [--plan optimal|ltr|both] [--out FILE]
//                  [--mode M] [--math fp32|auto] [--device D] [--tol T]
//   ce_cli layer   --kind K --desc JSON [--cr X] [--json]
//   ce_cli bench   --suite resnet34-cp --batch B --cr X [--json]
//
// Exit codes: 0 ok, 2 parse error, 3 shape error, 4 numerical mismatch, 1 other.
// Output to stdout, diagnostics to stderr.  Tensors on the wire (--out) use the reference's
// formats: JSON when FILE ends in .json, else the little-endian binary (tensor.hpp:63-68).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/ce/ce.h"

namespace {

struct Fail {
  int code;
  std::string msg;
};

int exit_code(ce_status st) {
  switch (st) {
    case CE_OK: return 0;
    case CE_ERR_PARSE: return 2;
    case CE_ERR_SHAPE: return 3;
    case CE_ERR_NUMERIC: return 4;
    default: return 1;
  }
}

void chk(ce_status st) {
  if (st != CE_OK) throw Fail{exit_code(st), ce_last_error()};
}

std::map<std::string, std::string> flags(int argc, char** argv, int from) {
  std::map<std::string, std::string> f;
  for (int i = from; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw Fail{1, "unexpected argument '" + k + "'"};
    k = k.substr(2);
    if (k == "json") {
      f[k] = "1";
    } else {
      if (i + 1 >= argc) throw Fail{1, "missing value for --" + k};
      f[k] = argv[++i];
    }
  }
  return f;
}

std::string get(const std::map<std::string, std::string>& f, const char* k, const char* def = nullptr) {
  auto it = f.find(k);
  if (it != f.end()) return it->second;
  if (def) return def;
  throw Fail{1, std::string("missing --") + k};
}

// shapes JSON {"dims": [[..], [..]]} (or a bare list of lists)
std::vector<std::vector<int64_t>> parse_shapes(const std::string& s) {
  std::vector<std::vector<int64_t>> out;
  std::size_t i = s.find('[');
  if (i == std::string::npos) throw Fail{3, "shapes: expected {\"dims\": [[...], ...]}"};
  int depth = 0;
  std::vector<int64_t> cur;
  for (; i < s.size(); ++i) {
    const char c = s[i];
    if (c == '[') {
      ++depth;
      if (depth == 2) cur.clear();
      if (depth > 2) throw Fail{3, "shapes: nesting too deep"};
    } else if (c == ']') {
      if (depth == 2) out.push_back(cur);
      if (--depth == 0) break;
    } else if ((c >= '0' && c <= '9') || c == '-') {
      if (depth != 2) throw Fail{3, "shapes: dims must be lists of integers"};
      char* end = nullptr;
      const long long v = std::strtoll(s.c_str() + i, &end, 10);
      if (v < 1) throw Fail{3, "shapes: dims must be >= 1"};
      cur.push_back(v);
      i = static_cast<std::size_t>(end - s.c_str()) - 1;
    } else if (c != ',' && c != ' ' && c != '\n' && c != '\t') {
      throw Fail{3, std::string("shapes: unexpected '") + c + "'"};
    }
  }
  if (depth != 0) throw Fail{3, "shapes: unbalanced brackets"};
  return out;
}

std::string shapes_json(const std::vector<std::vector<int64_t>>& d) {
  std::string s = "[";
  for (std::size_t i = 0; i < d.size(); ++i) {
    s += i ? ",[" : "[";
    for (std::size_t j = 0; j < d[i].size(); ++j) s += (j ? "," : "") + std::to_string(d[i][j]);
    s += "]";
  }
  return s + "]";
}

struct Flat {
  std::vector<int64_t> dims;
  std::vector<int> ranks;
};
Flat flatten(const std::vector<std::vector<int64_t>>& d) {
  Flat f;
  for (const auto& x : d) {
    f.ranks.push_back(static_cast<int>(x.size()));
    f.dims.insert(f.dims.end(), x.begin(), x.end());
  }
  return f;
}

std::string u128s(uint64_t lo, uint64_t hi) {
  if (hi == 0) return std::to_string(lo);
  unsigned __int128 v = (static_cast<unsigned __int128>(hi) << 64) | lo;
  std::string s;
  while (v) {
    s.insert(s.begin(), static_cast<char>('0' + static_cast<int>(v % 10)));
    v /= 10;
  }
  return s;
}
double u128d(uint64_t lo, uint64_t hi) { return static_cast<double>(hi) * 18446744073709551616.0 + static_cast<double>(lo); }

std::string eng(double v) {
  char b[32];
  std::snprintf(b, sizeof b, "%.3g", v);
  return b;
}

struct PlanH {
  ce_plan* p = nullptr;
  ~PlanH() {
    if (p) ce_plan_destroy(p);
  }
};

// expression + shapes from --expr/--shapes or a --layer descriptor (with --cr)
void resolve_input(const std::map<std::string, std::string>& f, std::string* expr,
                   std::vector<std::vector<int64_t>>* dims) {
  if (f.count("layer")) {
    char kind[64];
    int64_t t[CE_MAX_LAYER_RANKS], s[CE_MAX_LAYER_RANKS], hw[5], r[CE_MAX_LAYER_RANKS];
    int nt = 0, ns = 0, nr = 0;
    chk(ce_layer_from_json(f.at("layer").c_str(), kind, sizeof kind, t, &nt, s, &ns, hw, r, &nr));
    const double cr = f.count("cr") ? std::atof(f.at("cr").c_str()) : 0.0;
    char ebuf[4096];
    int64_t d[512];
    int rofi[CE_MAX_LAYER_INPUTS], nin = 0, nro = 0;
    int64_t rout[CE_MAX_LAYER_RANKS];
    uint64_t pc = 0;
    chk(ce_layer_expression(kind, t, nt, s, ns, hw[0], hw[1], hw[2], hw[3], hw[4], r, nr, cr, ebuf, sizeof ebuf, d,
                            512, rofi, &nin, rout, &nro, &pc));
    *expr = ebuf;
    dims->clear();
    int pos = 0;
    for (int i = 0; i < nin; ++i) {
      dims->emplace_back(d + pos, d + pos + rofi[i]);
      pos += rofi[i];
    }
    return;
  }
  *expr = get(f, "expr");
  *dims = parse_shapes(get(f, "shapes"));
}

int cmd_analyze(const std::map<std::string, std::string>& f) {
  std::string expr;
  std::vector<std::vector<int64_t>> dims;
  resolve_input(f, &expr, &dims);
  const std::string mode = get(f, "mode", "same"), cost = get(f, "cost", "inference");
  char rendered[4096], classes[4096];
  chk(ce_parse(expr.c_str(), rendered, sizeof rendered, classes, sizeof classes));
  const Flat fl = flatten(dims);
  PlanH opt, ltr;
  chk(ce_plan_create(expr.c_str(), fl.dims.data(), fl.ranks.data(), static_cast<int>(dims.size()), mode.c_str(),
                     cost.c_str(), CE_PLAN_OPTIMAL, &opt.p));
  chk(ce_plan_create(expr.c_str(), fl.dims.data(), fl.ranks.data(), static_cast<int>(dims.size()), mode.c_str(),
                     cost.c_str(), CE_PLAN_LEFT_TO_RIGHT, &ltr.p));
  ce_plan_info io{}, il{};
  chk(ce_plan_get_info(opt.p, &io));
  chk(ce_plan_get_info(ltr.p, &il));
  static char js_o[1 << 16], js_l[1 << 16], tr_o[4096], tr_l[4096];
  chk(ce_plan_json(opt.p, js_o, sizeof js_o));
  chk(ce_plan_json(ltr.p, js_l, sizeof js_l));
  chk(ce_plan_tree_encoding(opt.p, tr_o, sizeof tr_o));
  chk(ce_plan_tree_encoding(ltr.p, tr_l, sizeof tr_l));
  const double su_inf = u128d(il.inference_cost_lo, il.inference_cost_hi) / u128d(io.inference_cost_lo, io.inference_cost_hi);
  const double su_tr = u128d(il.training_cost_lo, il.training_cost_hi) / u128d(io.training_cost_lo, io.training_cost_hi);
  if (f.count("json")) {
    auto side = [&](const char* js, const char* tr, const ce_plan_info& i) {
      return std::string("{\"plan\":") + js + ",\"tree\":\"" + tr + "\",\"inference_cost\":\"" +
             u128s(i.inference_cost_lo, i.inference_cost_hi) + "\",\"training_cost\":\"" +
             u128s(i.training_cost_lo, i.training_cost_hi) + "\",\"multiplications\":\"" +
             u128s(i.flops_actual_lo, i.flops_actual_hi) + "\",\"peak_elems\":" +
             std::to_string(i.peak_intermediate_elements) + "}";
    };
    char sp[128];
    std::snprintf(sp, sizeof sp, "{\"inference\":%.17g,\"training\":%.17g}", su_inf, su_tr);
    std::printf("{\"expression\":\"%s\",\"dims\":%s,\"mode\":\"%s\",\"cost_mode\":\"%s\",\"optimal\":%s,"
                "\"left_to_right\":%s,\"speedup\":%s}\n",
                rendered, shapes_json(dims).c_str(), mode.c_str(), cost.c_str(), side(js_o, tr_o, io).c_str(),
                side(js_l, tr_l, il).c_str(), sp);
    return 0;
  }
  std::printf("expression   %s\n", rendered);
  for (std::size_t i = 0; i < dims.size(); ++i) {
    std::printf("  input %zu    [", i);
    for (std::size_t j = 0; j < dims[i].size(); ++j) std::printf("%s%lld", j ? ", " : "", static_cast<long long>(dims[i][j]));
    std::printf("]\n");
  }
  std::printf("%-14s %-24s %24s %24s %14s\n", "plan", "tree", "inference cost", "training cost", "peak elems");
  auto row = [&](const char* name, const char* tr, const ce_plan_info& i) {
    const std::string a = u128s(i.inference_cost_lo, i.inference_cost_hi), b = u128s(i.training_cost_lo, i.training_cost_hi);
    std::printf("%-14s %-24s %15s (%7s) %15s (%7s) %14llu\n", name, tr, a.c_str(),
                eng(u128d(i.inference_cost_lo, i.inference_cost_hi)).c_str(), b.c_str(),
                eng(u128d(i.training_cost_lo, i.training_cost_hi)).c_str(),
                static_cast<unsigned long long>(i.peak_intermediate_elements));
  };
  row("optimal", tr_o, io);
  row("left-to-right", tr_l, il);
  std::printf("speedup        inference %.4g   training %.4g\n", su_inf, su_tr);
  return 0;
}

struct DevBuf {  // device memory through the C-ABI (the CLI links no CUDA runtime of its own)
  ce_ctx* ctx = nullptr;
  float* p = nullptr;
  void alloc(ce_ctx* c, int64_t n) {
    ctx = c;
    void* q = nullptr;
    chk(ce_ctx_alloc(c, static_cast<size_t>(std::max<int64_t>(n, 1)) * 4, &q));
    p = static_cast<float*>(q);
  }
  ~DevBuf() {
    if (p) ce_ctx_free(ctx, p);
  }
};

int cmd_eval(const std::map<std::string, std::string>& f) {
  std::string expr;
  std::vector<std::vector<int64_t>> dims;
  resolve_input(f, &expr, &dims);
  const std::string mode = get(f, "mode", "same"), which = get(f, "plan", "optimal"), math = get(f, "math", "fp32");
  const uint64_t seed = std::strtoull(get(f, "seed", "1").c_str(), nullptr, 10);
  const int device = std::atoi(get(f, "device", "0").c_str());
  // the SPEC's 1e-8 is for the FP64 reference; the device computes in FP32 (or TF32)
  const double tol = std::atof(get(f, "tol", math == "fp32" ? "1e-5" : "5e-3").c_str());
  const Flat fl = flatten(dims);
  ce_options o{};
  o.math = math == "fp32" ? CE_MATH_FP32_SIMT : CE_MATH_AUTO;
  ce_ctx* ctx = nullptr;
  chk(ce_ctx_create(device, &o, &ctx));
  std::vector<DevBuf> in(dims.size());
  std::vector<const float*> ptrs;
  for (std::size_t i = 0; i < dims.size(); ++i) {
    int64_t n = 1;
    for (int64_t d : dims[i]) n *= d;
    in[i].alloc(ctx, n);
    chk(ce_fill_random(ctx, in[i].p, n, seed + i));  // fill_random(dims[i], seed + i), rounded to FP32
    ptrs.push_back(in[i].p);
  }
  struct Res {
    std::string name;
    std::vector<float> out;
    std::vector<int64_t> shape;
    std::string mults;
  };
  std::vector<Res> res;
  for (const char* w : {"optimal", "ltr"}) {
    if (which != "both" && which != w) continue;
    PlanH p;
    chk(ce_plan_create(expr.c_str(), fl.dims.data(), fl.ranks.data(), static_cast<int>(dims.size()), mode.c_str(),
                       "inference", std::strcmp(w, "ltr") == 0 ? CE_PLAN_LEFT_TO_RIGHT : CE_PLAN_OPTIMAL, &p.p));
    ce_plan_info info{};
    chk(ce_plan_get_info(p.p, &info));
    int64_t n = 1;
    Res r;
    r.name = w;
    for (int i = 0; i < info.out_rank; ++i) {
      r.shape.push_back(info.out_dims[i]);
      n *= info.out_dims[i];
    }
    DevBuf out;
    out.alloc(ctx, n);
    ce_executor* ex = nullptr;
    chk(ce_executor_create(ctx, p.p, 0, &ex));
    ce_exec_stats st{};
    const ce_status s1 = ce_execute(ex, ptrs.data(), out.p, &st);
    const ce_status s2 = s1 == CE_OK ? ce_ctx_synchronize(ctx) : s1;
    ce_executor_destroy(ex);
    chk(s2);
    r.out.resize(static_cast<std::size_t>(n));
    chk(ce_ctx_memcpy(ctx, r.out.data(), out.p, static_cast<size_t>(n) * 4));
    r.mults = u128s(info.flops_actual_lo, info.flops_actual_hi);
    res.push_back(std::move(r));
  }
  int rc = 0;
  for (const Res& r : res) {
    double sum = 0, amax = 0;
    for (float v : r.out) {
      sum += v;
      amax = std::max(amax, std::fabs(static_cast<double>(v)));
    }
    std::printf("%-8s multiplications %s  sum %.9g  max|y| %.9g\n", r.name.c_str(), r.mults.c_str(), sum, amax);
  }
  if (res.size() == 2) {
    double dev = 0, scale = 0;
    for (std::size_t i = 0; i < res[0].out.size(); ++i) {
      dev = std::max(dev, std::fabs(static_cast<double>(res[0].out[i]) - res[1].out[i]));
      scale = std::max(scale, std::fabs(static_cast<double>(res[1].out[i])));
    }
    const double rel = scale > 0 ? dev / scale : dev;
    std::printf("max relative deviation %.3e (tolerance %.1e)\n", rel, tol);
    if (!(rel <= tol)) rc = 4;
  }
  in.clear();  // device inputs freed while the context is alive
  ce_ctx_destroy(ctx);
  if (f.count("out") && !res.empty()) {
    const Res& r = res[0];
    const std::vector<double> d(r.out.begin(), r.out.end());
    const std::string path = f.at("out");
    const bool js = path.size() > 5 && path.compare(path.size() - 5, 5, ".json") == 0;
    std::string blob;
    if (js) {
      size_t len = 0;
      ce_tensor_to_json(r.shape.data(), static_cast<int>(r.shape.size()), d.data(), nullptr, 0, &len);
      blob.resize(len);
      chk(ce_tensor_to_json(r.shape.data(), static_cast<int>(r.shape.size()), d.data(), blob.data(), len, &len));
      blob.resize(len - 1);
    } else {
      size_t len = 8 * (1 + r.shape.size() + d.size());
      blob.resize(len);
      chk(ce_tensor_to_binary(r.shape.data(), static_cast<int>(r.shape.size()), d.data(),
                              reinterpret_cast<unsigned char*>(blob.data()), len, &len));
      blob.resize(len);
    }
    std::ofstream os(path, std::ios::binary);
    os.write(blob.data(), static_cast<std::streamsize>(blob.size()));
    if (!os) throw Fail{1, "cannot write " + path};
  }
  return rc;
}

int cmd_layer(const std::map<std::string, std::string>& f) {
  // --desc is the layer descriptor JSON; --kind overrides its "kind"
  std::string desc = get(f, "desc");
  char kind[64];
  int64_t t[CE_MAX_LAYER_RANKS], s[CE_MAX_LAYER_RANKS], hw[5], r[CE_MAX_LAYER_RANKS];
  int nt = 0, ns = 0, nr = 0;
  if (desc.find("\"kind\"") == std::string::npos) {
    const std::size_t b = desc.find('{');
    if (b == std::string::npos) throw Fail{1, "--desc must be a JSON object"};
    desc.insert(b + 1, "\"kind\":\"" + get(f, "kind") + "\",");
  }
  ce_status st = ce_layer_from_json(desc.c_str(), kind, sizeof kind, t, &nt, s, &ns, hw, r, &nr);
  if (st != CE_OK && desc.find("\"rank\"") == std::string::npos) {
    // no ranks given (--cr solves them): validate() needs a placeholder for rank-carrying kinds
    desc.insert(desc.find('{') + 1, "\"rank\":1,");
    st = ce_layer_from_json(desc.c_str(), kind, sizeof kind, t, &nt, s, &ns, hw, r, &nr);
  }
  chk(st);
  if (f.count("kind")) std::snprintf(kind, sizeof kind, "%s", f.at("kind").c_str());
  const double cr = f.count("cr") ? std::atof(f.at("cr").c_str()) : 0.0;
  char ebuf[4096];
  int64_t d[512];
  int rofi[CE_MAX_LAYER_INPUTS], nin = 0, nro = 0;
  int64_t rout[CE_MAX_LAYER_RANKS];
  uint64_t pc = 0;
  chk(ce_layer_expression(kind, t, nt, s, ns, hw[0], hw[1], hw[2], hw[3], hw[4], r, nr, cr, ebuf, sizeof ebuf, d, 512,
                          rofi, &nin, rout, &nro, &pc));
  std::vector<std::vector<int64_t>> dims;
  int pos = 0;
  for (int i = 0; i < nin; ++i) {
    dims.emplace_back(d + pos, d + pos + rofi[i]);
    pos += rofi[i];
  }
  std::string ranks = "[";
  for (int i = 0; i < nro; ++i) ranks += (i ? "," : "") + std::to_string(rout[i]);
  ranks += "]";
  if (f.count("json")) {
    std::printf("{\"expression\":\"%s\",\"dims\":%s,\"params\":%llu,\"ranks\":%s}\n", ebuf, shapes_json(dims).c_str(),
                static_cast<unsigned long long>(pc), ranks.c_str());
  } else {
    std::printf("expression  %s\nshapes      %s\nparams      %llu\nranks       %s\n", ebuf, shapes_json(dims).c_str(),
                static_cast<unsigned long long>(pc), ranks.c_str());
  }
  return 0;
}

int cmd_bench(const std::map<std::string, std::string>& f) {
  const std::string suite = get(f, "suite", "resnet34-cp");
  if (suite != "resnet34-cp") throw Fail{1, "unknown suite '" + suite + "'"};
  const int64_t batch = std::atoll(get(f, "batch", "128").c_str());
  const double cr = std::atof(get(f, "cr", "1.0").c_str());
  // resnet34_cp_blocks (layers.cpp:400-423)
  struct Blk {
    const char* name;
    int64_t s, t, k, hp;
  };
  const Blk blocks[] = {{"conv1", 3, 64, 7, 112}, {"conv2_x", 64, 64, 3, 56}, {"conv3_x", 128, 128, 3, 28},
                        {"conv4_x", 256, 256, 3, 14}, {"conv5_x", 512, 512, 3, 7}};
  std::string js = "[";
  if (!f.count("json")) std::printf("%-8s %6s %26s %26s %10s\n", "layer", "rank", "left-to-right mults", "optimal mults", "speedup");
  for (const Blk& b : blocks) {
    const int64_t one = 1;
    char ebuf[4096];
    int64_t d[512];
    int rofi[CE_MAX_LAYER_INPUTS], nin = 0, nro = 0;
    int64_t rout[CE_MAX_LAYER_RANKS];
    uint64_t pc = 0;
    chk(ce_layer_expression("cp", &b.t, 1, &b.s, 1, b.k, b.k, b.hp, b.hp, batch, &one, 1, cr, ebuf, sizeof ebuf, d, 512,
                            rofi, &nin, rout, &nro, &pc));
    PlanH opt, ltr;
    chk(ce_plan_create(ebuf, d, rofi, nin, "same", "inference", CE_PLAN_OPTIMAL, &opt.p));
    chk(ce_plan_create(ebuf, d, rofi, nin, "same", "inference", CE_PLAN_LEFT_TO_RIGHT, &ltr.p));
    ce_plan_info io{}, il{};
    chk(ce_plan_get_info(opt.p, &io));
    chk(ce_plan_get_info(ltr.p, &il));
    const std::string a = u128s(il.total_cost_lo, il.total_cost_hi), o = u128s(io.total_cost_lo, io.total_cost_hi);
    const double sp = u128d(il.total_cost_lo, il.total_cost_hi) / u128d(io.total_cost_lo, io.total_cost_hi);
    if (f.count("json")) {
      char row[512];
      std::snprintf(row, sizeof row, "%s{\"layer\":\"%s\",\"rank\":%lld,\"left_to_right\":\"%s\",\"optimal\":\"%s\",\"speedup\":%.17g}",
                    js.size() > 1 ? "," : "", b.name, static_cast<long long>(rout[0]), a.c_str(), o.c_str(), sp);
      js += row;
    } else {
      std::printf("%-8s %6lld %16s (%7s) %16s (%7s) %10.4g\n", b.name, static_cast<long long>(rout[0]), a.c_str(),
                  eng(u128d(il.total_cost_lo, il.total_cost_hi)).c_str(), o.c_str(),
                  eng(u128d(io.total_cost_lo, io.total_cost_hi)).c_str(), sp);
    }
  }
  if (f.count("json")) std::printf("%s]\n", js.c_str());
  return 0;
}

void usage() {
  std::fprintf(stderr,
               "usage: ce_cli analyze --expr STR --shapes JSON | --layer JSON [--cr X] [--mode M] [--cost C] [--json]\n"
               "       ce_cli eval --expr STR --shapes JSON --seed N [--plan optimal|ltr|both] [--out FILE]\n"
               "                   [--mode M] [--math fp32|auto] [--device D] [--tol T]\n"
               "       ce_cli layer --kind K --desc JSON [--cr X] [--json]\n"
               "       ce_cli bench --suite resnet34-cp --batch B --cr X [--json]\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    const auto f = flags(argc, argv, 2);
    if (cmd == "analyze") return cmd_analyze(f);
    if (cmd == "eval") return cmd_eval(f);
    if (cmd == "layer") return cmd_layer(f);
    if (cmd == "bench") return cmd_bench(f);
    usage();
    return 1;
  } catch (const Fail& e) {
    std::fprintf(stderr, "error: %s\n", e.msg.c_str());
    return e.code;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
