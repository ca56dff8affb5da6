// Reference DevicePrograms for the vocabulary-pass executor: parser and the
// vocabulary-pass subset of the dependency validator.  See vocab_program.h.
#include "vocab_program.h"

#include <map>
#include <sstream>
#include <tuple>
#include <utility>

namespace vp {

bool is_collective(PKind k) { return k == PKind::C0 || k == PKind::C1 || k == PKind::C2; }
bool is_vocab_pass(PKind k) { return k == PKind::S || k == PKind::T || is_collective(k); }

const char* kind_name(PKind k) {
  switch (k) {
    case PKind::F: return "F";
    case PKind::B: return "B";
    case PKind::S: return "S";
    case PKind::T: return "T";
    case PKind::C0: return "C0";
    case PKind::C1: return "C1";
    case PKind::C2: return "C2";
    case PKind::IF: return "IF";
    case PKind::IB: return "IB";
  }
  return "?";
}

namespace {

PKind kind_from_name(const std::string& s) {
  static const std::pair<const char*, PKind> names[] = {{"F", PKind::F},   {"B", PKind::B},   {"S", PKind::S},
                                                        {"T", PKind::T},   {"C0", PKind::C0}, {"C1", PKind::C1},
                                                        {"C2", PKind::C2}, {"IF", PKind::IF}, {"IB", PKind::IB}};
  for (const auto& [nm, k] : names)
    if (s == nm) return k;
  throw std::invalid_argument("unknown pass kind: " + s);
}

// method name -> (has vocabulary passes, barriers); P/src/schedule.cpp:57-88
void set_method(Program& p, const std::string& name) {
  static const std::tuple<const char*, bool, int> methods[] = {
      {"baseline", false, 0}, {"redis", false, 0},     {"vocab1", true, 2},      {"vocab2", true, 1},
      {"interlaced", true, 2}, {"vhalf", false, 0}, {"vhalf-vocab1", true, 2}};
  for (const auto& [nm, vocab, bar] : methods) {
    if (name == nm) {
      p.method = name;
      p.vocab = vocab;
      p.barriers = bar;
      return;
    }
  }
  throw std::invalid_argument("unknown method: " + name);
}

[[noreturn]] void fail(const std::string& what) { throw ProgramParseError("parse_program: " + what); }

std::string label(PKind k, int dev, int mb, int chunk, bool collective) {
  std::string s = std::string(kind_name(k)) + " microbatch " + std::to_string(mb);
  if (!collective) {
    s += " device " + std::to_string(dev);
    if (chunk != 0) s += " chunk " + std::to_string(chunk);
  }
  return s;
}

}  // namespace

Program parse_program(const std::string& text) {
  std::istringstream in(text);
  Program prog;
  set_method(prog, "baseline");
  std::string magic;
  int version = 0;
  if (!(in >> magic >> version) || magic != "vpipe-program" || version != 1) fail("bad header");
  std::size_t total = 0;
  for (;;) {
    std::string key;
    if (!(in >> key)) fail("truncated header");
    if (key == "passes") {
      if (!(in >> total)) fail("bad pass count");
      break;
    }
    if (key == "method") {
      std::string value;
      in >> value;
      set_method(prog, value);
      continue;
    }
    int64_t value = 0;
    if (!(in >> value)) fail("bad header value for " + key);
    int64_t* field = key == "b" ? &prog.b
                     : key == "s" ? &prog.s
                     : key == "h" ? &prog.h
                     : key == "V" ? &prog.V
                     : key == "L" ? &prog.L
                     : key == "p" ? &prog.p
                     : key == "n" ? &prog.n
                                  : nullptr;
    if (!field) fail("unknown header key " + key);
    *field = value;
  }
  // ModelConfig::validate (P/src/cost_model.cpp:8-22)
  for (const auto& [v, nm] : {std::pair{prog.b, "b"}, {prog.s, "s"}, {prog.h, "h"}, {prog.V, "V"}, {prog.L, "L"},
                              {prog.p, "p"}, {prog.n, "n"}})
    if (v < 1) throw std::invalid_argument(std::string("ModelConfig: ") + nm + " must be >= 1");
  prog.order.resize(size_t(prog.p));
  for (std::size_t line = 0; line < total; ++line) {
    int device = 0, mb = 0, chunk = 0;
    std::string kind;
    if (!(in >> device >> mb >> kind >> chunk)) fail("truncated pass list");
    if (device < 0 || device >= prog.p) fail("pass device out of range");
    prog.order[size_t(device)].push_back(PPass{kind_from_name(kind), device, mb, chunk});
  }
  return prog;
}

std::vector<std::string> validate_vocab(const Program& prog) {
  const int p = int(prog.p), n = int(prog.n);
  struct Node {
    PKind kind;
    int dev, mb, chunk;
    bool collective;
    std::vector<std::pair<int, int>> loc;  // (device, index in that device's order)
  };
  std::vector<Node> nodes;
  std::vector<std::vector<int>> at(static_cast<size_t>(p));  // [device][index] -> node
  std::map<std::tuple<int, int, int, int>, int> pass_id;
  std::map<std::pair<int, int>, int> coll_id;
  try {
    // structural pass (every pass, so duplicates and ranges are caught as in
    // build_pass_graph, P/src/schedule.cpp:248-300)
    if (int(prog.order.size()) != p) throw std::invalid_argument("program: device list count != p");
    for (int d = 0; d < p; ++d) {
      for (int j = 0; j < int(prog.order[size_t(d)].size()); ++j) {
        const PPass& ps = prog.order[size_t(d)][size_t(j)];
        if (ps.device != d) throw std::invalid_argument("program: pass device field mismatch");
        if (ps.microbatch < 0 || ps.microbatch >= n) throw std::invalid_argument("program: microbatch out of range");
        int id;
        if (is_collective(ps.kind)) {
          const auto key = std::make_pair(int(ps.kind), ps.microbatch);
          auto it = coll_id.find(key);
          if (it == coll_id.end()) {
            id = int(nodes.size());
            coll_id.emplace(key, id);
            nodes.push_back({ps.kind, -1, ps.microbatch, 0, true, {}});
          } else {
            id = it->second;
          }
          for (const auto& l : nodes[size_t(id)].loc)
            if (l.first == d) throw std::invalid_argument("program: duplicate collective participation");
        } else {
          const auto key = std::make_tuple(int(ps.kind), d, ps.microbatch, ps.chunk);
          if (pass_id.count(key)) throw std::invalid_argument("program: duplicate pass");
          id = int(nodes.size());
          pass_id.emplace(key, id);
          nodes.push_back({ps.kind, d, ps.microbatch, ps.chunk, false, {}});
        }
        nodes[size_t(id)].loc.emplace_back(d, j);
        at[size_t(d)].push_back(id);
      }
    }
  } catch (const std::invalid_argument& e) {
    return {e.what()};
  }
  // vocabulary dependencies per microbatch (P/src/schedule.cpp:339-366):
  //   C0_i -> S(d,i) -> C1_i;  2 barriers: C1_i -> T(d,i) -> C2_i;  1 barrier: C1_i -> T(d,i)
  std::vector<std::vector<int>> preds(nodes.size());
  if (prog.vocab) {
    auto find = [&](PKind k, int d, int mb) {
      auto it = pass_id.find(std::make_tuple(int(k), d, mb, 0));
      if (it == pass_id.end())
        throw std::invalid_argument(std::string("program: missing required pass ") + kind_name(k) + " device " +
                                    std::to_string(d) + " microbatch " + std::to_string(mb));
      return it->second;
    };
    auto find_coll = [&](PKind k, int mb) {
      auto it = coll_id.find(std::make_pair(int(k), mb));
      if (it == coll_id.end())
        throw std::invalid_argument(std::string("program: missing collective ") + kind_name(k) + " microbatch " +
                                    std::to_string(mb));
      return it->second;
    };
    try {
      for (int i = 0; i < n; ++i) {
        const int c0 = find_coll(PKind::C0, i), c1 = find_coll(PKind::C1, i);
        for (int d = 0; d < p; ++d) {
          const int sn = find(PKind::S, d, i);
          preds[size_t(sn)].push_back(c0);
          preds[size_t(c1)].push_back(sn);
        }
        if (prog.barriers == 2) {
          const int c2 = find_coll(PKind::C2, i);
          for (int d = 0; d < p; ++d) {
            const int tn = find(PKind::T, d, i);
            preds[size_t(tn)].push_back(c1);
            preds[size_t(c2)].push_back(tn);
          }
        } else {
          for (int d = 0; d < p; ++d) preds[size_t(find(PKind::T, d, i))].push_back(c1);
        }
      }
    } catch (const std::invalid_argument& e) {
      return {e.what()};
    }
  }
  std::vector<std::string> out;
  // same-device order against every dependency (P/src/schedule.cpp:400-416)
  for (std::size_t v = 0; v < nodes.size(); ++v) {
    for (int u : preds[v]) {
      for (const auto& [du, iu] : nodes[size_t(u)].loc) {
        for (const auto& [dv, iv] : nodes[v].loc) {
          if (du == dv && iu >= iv) {
            const Node& a = nodes[v];
            const Node& b = nodes[size_t(u)];
            out.push_back("device " + std::to_string(dv) + ": " + label(a.kind, a.dev, a.mb, a.chunk, a.collective) +
                          " scheduled before its dependency " + label(b.kind, b.dev, b.mb, b.chunk, b.collective));
          }
        }
      }
    }
  }
  // acyclicity over the dependencies plus each device's order (:418-446)
  std::vector<std::vector<int>> succ(nodes.size());
  std::vector<int> indeg(nodes.size(), 0);
  for (std::size_t v = 0; v < nodes.size(); ++v)
    for (int u : preds[v]) {
      succ[size_t(u)].push_back(int(v));
      ++indeg[v];
    }
  for (const auto& list : at)
    for (std::size_t j = 1; j < list.size(); ++j) {
      succ[size_t(list[j - 1])].push_back(list[j]);
      ++indeg[size_t(list[j])];
    }
  std::vector<int> ready;
  for (std::size_t v = 0; v < nodes.size(); ++v)
    if (indeg[v] == 0) ready.push_back(int(v));
  std::size_t seen = 0;
  while (!ready.empty()) {
    const int u = ready.back();
    ready.pop_back();
    ++seen;
    for (int v : succ[size_t(u)])
      if (--indeg[size_t(v)] == 0) ready.push_back(v);
  }
  if (seen != nodes.size())
    out.push_back("cyclic dependency among " + std::to_string(nodes.size() - seen) + " passes");
  return out;
}

}  // namespace vp
