"""cortex:: gate (proj/include/cortex/gate.hpp:9-31, proj/src/gate.cpp:12-61): the
cosine between the main model's hidden state and a side agent's thought, computed
on the GPU in fp64 with the reference's sequential sums (bitwise-equal scores).
The batched device form is ``device.gate_decide``.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import errors
from ._lib import c_f32p, check, lib, ptr


@dataclass
class GateDecision:
    """gate.hpp:9-19."""
    score: float = 0.0  # NaN when degenerate
    threshold: float = 0.5
    accepted: bool = False
    degenerate: bool = False
    thought_id: int = -1

    @staticmethod
    def csv_header() -> str:
        return "thought_id,score,theta,accepted"

    def csv_row(self) -> str:
        """gate.cpp:14-25: 17 significant digits, "nan" when degenerate."""
        score = "nan" if self.degenerate else f"{self.score:.17g}"
        return f"{self.thought_id},{score},{self.threshold:.17g},{1 if self.accepted else 0}"


def gate_score(h_main, t_side) -> float:
    """gate.cpp:27-43: cosine in fp64, clamped to [-1, 1]; degenerate_input_error on a zero norm."""
    h = np.ascontiguousarray(h_main, np.float32).reshape(-1)
    t = np.ascontiguousarray(t_side, np.float32).reshape(-1)
    if h.size != t.size:
        raise errors.precondition_error("gate_score: width mismatch")
    out = C.c_double(0.0)
    check(lib.cx_gate_score(ptr(h, c_f32p), ptr(t, c_f32p), h.size, C.byref(out)), "gate_score")
    return out.value


def decide(h_main, t_side, theta: float, thought_id: int = -1) -> GateDecision:
    """gate.cpp:45-61: accepted iff score >= theta; zero norms -> rejected, degenerate."""
    if theta < -1.0 or theta > 1.0:
        raise errors.precondition_error("decide: theta must be in [-1,1]")
    d = GateDecision(threshold=theta, thought_id=thought_id)
    try:
        d.score = gate_score(h_main, t_side)
        d.accepted = d.score >= theta
    except errors.degenerate_input_error:
        d.score, d.degenerate, d.accepted = math.nan, True, False
    return d


