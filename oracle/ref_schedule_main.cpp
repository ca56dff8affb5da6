// Test infrastructure only: a driver around the REFERENCE's own schedule
// builder and validator (compiled from /root/reference/proj/src/schedule.cpp
// and cost_model.cpp by oracle/Makefile into oracle/_ref/vpipe_sched; never
// shipped, never on the product path).  Used by tests/golden/make_programs.py
// to pin the vocabulary-pass executor's program parser and validator
// (paper_2411_05288_b200 vp_program_*) against the reference itself.
//
//   vpipe_sched build <method> <p> <n>   -> serialize_program(build_program(method, cfg))
//                                           with the reference tests' make_cfg(p, n)
//                                           (P/tests/test_schedule.cpp:14-24)
//   vpipe_sched simulate <method> <b> <s> <h> <V> <L> <p> <n> <unit_rate> [<s> <t> <collective>]
//                                        -> JSON: the reference machine model (build_machine,
//                                           P/src/simulator.cpp:26-101) and its simulated
//                                           makespan / MFU / bubble; with the optional
//                                           measured S, T and collective durations, the same
//                                           simulation with those overriding the model's
//                                           (tools/calibrate.py)
//   vpipe_sched validate                 <- program text on stdin
//                                        -> one violation per line (validate_dependencies,
//                                           P/src/schedule.cpp:390-447); "error: ..." when
//                                           parse_program throws
#include <algorithm>
#include <iostream>
#include <iterator>
#include <sstream>
#include <string>

#include "vpipe/schedule.hpp"
#include "vpipe/simulator.hpp"

int main(int argc, char** argv) {
  using namespace vpipe;
  if (argc < 2) {
    std::cerr << "usage: vpipe_sched build <method> <p> <n> | validate\n";
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "build" && argc == 5) {
      ModelConfig cfg;
      const int p = std::stoi(argv[3]), n = std::stoi(argv[4]);
      cfg.b = 1;
      cfg.s = 8;
      cfg.h = 16;
      cfg.V = 16 * p;
      cfg.L = 2 * p;
      cfg.p = p;
      cfg.n = n;
      std::cout << serialize_program(build_program(method_from_name(argv[2]), cfg));
      return 0;
    }
    if (cmd == "simulate" && (argc == 11 || argc == 14)) {
      ModelConfig cfg;
      cfg.b = std::stoll(argv[3]);
      cfg.s = std::stoll(argv[4]);
      cfg.h = std::stoll(argv[5]);
      cfg.V = std::stoll(argv[6]);
      cfg.L = std::stoll(argv[7]);
      cfg.p = std::stoll(argv[8]);
      cfg.n = std::stoll(argv[9]);
      const DeviceProgram program = build_program(method_from_name(argv[2]), cfg);
      MachineOptions mo;
      mo.unit_rate = std::stod(argv[10]);
      MachineModel m = build_machine(program, mo);
      auto run = [&](const MachineModel& mm) {
        const Timeline tl = simulate(program, mm);
        const Metrics mt = metrics(tl, cfg);
        double bubble = 0.0;
        for (const auto& d : mt.devices) bubble = std::max(bubble, d.bubble_ratio);
        std::ostringstream os;
        os << "{\"f\": " << mm.f[0][0] << ", \"b\": " << mm.b[0][0] << ", \"s\": " << mm.s << ", \"t\": " << mm.t
           << ", \"collective\": " << mm.collective << ", \"makespan\": " << tl.makespan << ", \"mfu\": " << mt.mfu
           << ", \"max_bubble_ratio\": " << bubble << "}";
        return os.str();
      };
      std::cout << "{\"model\": " << run(m);
      if (argc == 14) {
        m.s = std::stod(argv[11]);
        m.t = std::stod(argv[12]);
        m.collective = std::stod(argv[13]);
        std::cout << ", \"measured\": " << run(m);
      }
      std::cout << "}\n";
      return 0;
    }
    if (cmd == "validate") {
      const std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
      for (const auto& v : validate_dependencies(parse_program(text))) std::cout << v << "\n";
      return 0;
    }
  } catch (const std::exception& e) {
    std::cout << "error: " << e.what() << "\n";
    return 1;
  }
  std::cerr << "bad arguments\n";
  return 2;
}
