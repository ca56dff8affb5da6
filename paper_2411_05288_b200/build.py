"""Builds every native artefact in-tree (sm_100a cross-compiles without a GPU):

  paper_2411_05288_b200/lib/libvpipe_b200.so   product: kernels + C ABI + C++ API
  oracle/liboracle.so                          test infrastructure (CPU oracle)
  tools/vpipe_verify                           parity CLI (C++ API, mirrors `vpipe verify`)
"""
from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _make(path: str, *targets: str) -> None:
    subprocess.run(["make", "-s", "-j4", "-C", path, *targets], check=True)


def build() -> None:
    _make(os.path.join(ROOT, "paper_2411_05288_b200", "csrc"))
    _make(os.path.join(ROOT, "oracle"))
    if os.path.exists(os.path.join(ROOT, "tools", "Makefile")):
        _make(os.path.join(ROOT, "tools"))


if __name__ == "__main__":
    build()
