// Reference DevicePrograms (P/include/vpipe/schedule.hpp:95-100) for the
// vocabulary-pass executor: the text form written by the
// reference's serialize_program (P/src/schedule.cpp:512-529), its parser's
// rules and messages (:531-577), and validate_dependencies (:390-447)
// restricted to the vocabulary passes C0 -> S -> C1 -> T [-> C2].
// Host-only; internal to libvpipe_b200.so (C ABI: vp_program_* in vpipe_b200.h).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace vp {

// P/include/vpipe/schedule.hpp:9-19, names as pass_kind_name (P/src/schedule.cpp:16-29)
enum class PKind { F, B, S, T, C0, C1, C2, IF, IB };

struct PPass {
  PKind kind;
  int device, microbatch, chunk;
};

struct Program {
  std::string method;  // reference method name (method_name, P/src/schedule.cpp:44-55)
  bool vocab = false;  // method_has_vocab_passes (:68-71)
  int barriers = 0;    // method_barriers (:80-88): 1 = Algorithm 2 (vocab2), 2 = Algorithm 1
  int64_t b = 1, s = 1, h = 1, V = 1, L = 1, p = 1, n = 1;
  std::vector<std::vector<PPass>> order;  // [device] -> passes in program order
};

// parse errors: the reference's parse_program throws std::runtime_error
// ("parse_program: ..."); unknown names / bad config std::invalid_argument.
struct ProgramParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

Program parse_program(const std::string& text);
bool is_collective(PKind k);
bool is_vocab_pass(PKind k);
const char* kind_name(PKind k);

// Violations of the vocabulary-pass dependencies, in the reference
// validator's order and wording; structural errors (missing / duplicate
// passes) come back as a single message, as in the reference.
std::vector<std::string> validate_vocab(const Program& prog);

}  // namespace vp
