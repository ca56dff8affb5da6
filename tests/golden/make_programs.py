#!/usr/bin/env python3
"""Generates tests/golden/programs.json: reference DevicePrograms (the text form of
P/src/schedule.cpp serialize_program) and the reference validator's verdicts on them,
produced by the REFERENCE's own builder/validator compiled from its sources
(oracle/_ref/vpipe_sched, see oracle/Makefile).  Pins the vocabulary-pass program
parser/validator of the executor (vp_program_*).

Cases: clean programs for every vocabulary method, and programs with one vocabulary
pass moved (the fault injection of P/tests/test_schedule.cpp:111-132 and variants)
or deleted (:134-144).
"""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SCHED = os.path.join(ROOT, "oracle", "_ref", "vpipe_sched")


def build(method, p, n):
    return subprocess.run([SCHED, "build", method, str(p), str(n)], check=True, capture_output=True,
                          text=True).stdout


def validate(text):
    r = subprocess.run([SCHED, "validate"], input=text, capture_output=True, text=True)
    return [ln for ln in r.stdout.splitlines() if ln]


def split(text):
    lines = text.splitlines()
    k = next(i for i, ln in enumerate(lines) if ln.startswith("passes "))
    return lines[:k + 1], [ln.split() for ln in lines[k + 1:]]


def join(head, passes):
    head = [ln if not ln.startswith("passes ") else f"passes {len(passes)}" for ln in head]
    return "\n".join(head + [" ".join(p) for p in passes]) + "\n"


def find(passes, dev, mb, kind):
    return next(i for i, p in enumerate(passes) if p[0] == str(dev) and p[1] == str(mb) and p[2] == kind)


def move_before(text, dev, mb, kind, dev2, mb2, kind2):
    """Move pass (dev, mb, kind) to just before (dev2, mb2, kind2) in the device list."""
    head, passes = split(text)
    a = passes.pop(find(passes, dev, mb, kind))
    passes.insert(find(passes, dev2, mb2, kind2), a)
    return join(head, passes)


def swap(text, dev, mb, kind, mb2, kind2):
    head, passes = split(text)
    i, j = find(passes, dev, mb, kind), find(passes, dev, mb2, kind2)
    passes[i], passes[j] = passes[j], passes[i]
    return join(head, passes)


def delete(text, dev, mb, kind):
    head, passes = split(text)
    passes.pop(find(passes, dev, mb, kind))
    return join(head, passes)


def main():
    cases = {}
    for method, p, n in [("vocab2", 1, 3), ("vocab2", 2, 4), ("vocab2", 4, 8), ("vocab1", 2, 4), ("vocab1", 4, 8),
                         ("interlaced", 4, 8), ("vhalf-vocab1", 2, 4), ("baseline", 2, 4)]:
        cases[f"{method}_p{p}_n{n}"] = build(method, p, n)
    v1 = cases["vocab1_p4_n8"]
    v2 = cases["vocab2_p2_n4"]
    cases["vocab1_p4_n8_T3_before_C1"] = swap(v1, 2, 3, "C1", 3, "T")          # test_schedule.cpp:111-132
    cases["vocab2_p2_n4_S1_after_C1"] = swap(v2, 1, 1, "S", 1, "C1")
    cases["vocab1_p2_n4_C2_before_T1"] = swap(cases["vocab1_p2_n4"], 1, 1, "T", 1, "C2")
    cases["vocab2_p4_n8_C1_before_C0"] = move_before(cases["vocab2_p4_n8"], 3, 5, "C1", 3, 5, "C0")
    cases["vocab2_p2_n4_missing_T2"] = delete(v2, 0, 2, "T")
    cases["vocab2_p2_n4_missing_C1"] = delete(v2, 1, 3, "C1")
    out = {name: {"text": text, "violations": validate(text)} for name, text in cases.items()}
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "programs.json"), "w"), indent=1)
    for name, c in out.items():
        print(f"{name}: {len(c['violations'])} violations", c["violations"][:3])


if __name__ == "__main__":
    main()
