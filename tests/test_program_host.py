"""Reference DevicePrograms for the vocabulary-pass executor (host side, no GPU):
the library's parser and vocabulary-pass validator against the REFERENCE's own
builder/validator output (tests/golden/programs.json, made by
tests/golden/make_programs.py from oracle/_ref/vpipe_sched)."""
import json
import os

import pytest

from paper_2411_05288_b200 import vocab_math as vm

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "programs.json")))


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_validator_matches_the_reference_validator(name):
    # P/tests/test_schedule.cpp:94-144: clean programs for every vocabulary
    # method, injected reorderings and deletions -> identical violation lists
    case = GOLDEN[name]
    assert vm.Program(case["text"]).validate() == case["violations"]


def test_program_info():
    pr = vm.Program(GOLDEN["vocab2_p4_n8"]["text"])
    assert (pr.barriers, pr.p, pr.n) == (1, 4, 8)
    pr = vm.Program(GOLDEN["vocab1_p2_n4"]["text"])
    assert (pr.barriers, pr.p, pr.n) == (2, 2, 4)
    assert vm.Program(GOLDEN["baseline_p2_n4"]["text"]).barriers == 0


def test_parser_rejects_malformed_input():
    # P/tests/test_schedule.cpp:247-255 and the parser's messages (schedule.cpp:531-577)
    with pytest.raises(ValueError, match="parse_program: bad header"):
        vm.Program("garbage")
    with pytest.raises(ValueError, match="parse_program: bad header"):
        vm.Program("vpipe-program 2\n")
    good = GOLDEN["baseline_p2_n4"]["text"]
    with pytest.raises(ValueError, match="parse_program: truncated pass list"):
        vm.Program(good[:-4])
    with pytest.raises(ValueError, match="unknown method: nope"):
        vm.Program(good.replace("method baseline", "method nope"))
    with pytest.raises(ValueError, match="unknown pass kind: Q"):
        vm.Program(good.replace(" F 0\n", " Q 0\n", 1))
    with pytest.raises(ValueError, match="parse_program: pass device out of range"):
        vm.Program(good.replace("\n1 0 F 0\n", "\n7 0 F 0\n", 1))
    with pytest.raises(ValueError, match="ModelConfig: n must be >= 1"):
        vm.Program(good.replace("\nn 4\n", "\nn 0\n"))


def test_program_texts_round_trip_through_the_reference_format():
    # every golden program parses; pass counts agree with the header
    for case in GOLDEN.values():
        text = case["text"]
        total = int(next(ln for ln in text.splitlines() if ln.startswith("passes ")).split()[1])
        assert total == len([ln for ln in text.splitlines()[10:] if ln.strip()])
        vm.Program(text)
