"""CPU: DeepSpeed's step-counter semantics (cpu_adam.h IncrementStep, the
running product of beta^t across consecutive adam_update calls) in the
product's C ABI (fy_adam_counter_next) and in the oracle
(oracle_counter_increment), both pinned to the golden sequences of an
independent transcription (tests/golden/make_step_counter_golden.py)."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = json.loads((Path(__file__).parent / "golden" / "deepspeed_step_counter.json").read_text())


def _bits(x: float) -> int:
    return int(np.array([x], dtype=np.float32).view(np.uint32)[0])


@pytest.mark.parametrize("case", sorted(GOLDEN))
def test_library_counter_matches_golden(case):
    from paper_2403_06504_b200._lib import LIB, AdamCounter, AdamHparams, check
    seq = GOLDEN[case]
    first = seq[0]
    # the optimizer's constructor betas = the first call's unless the case changes them
    ctor = (0.9, 0.999) if case in ("betas_change", "adam_defaults_2000") else (first["beta1"], first["beta2"])
    c = AdamCounter()
    check(LIB.fy_adam_counter_init(C.byref(c), *ctor))
    for i, e in enumerate(seq):
        hp = AdamHparams(1e-4, e["beta1"], e["beta2"], 1e-8, 0.1, e["step"], 1, 1, 1.0, 0, 0.0, 0.0)
        check(LIB.fy_adam_counter_next(C.byref(c), C.byref(hp)))
        assert hp.beta_t_given == 1
        assert _bits(hp.beta1_t) == e["b1t"], f"{case} call {i} beta1^t"
        assert _bits(hp.beta2_t) == e["b2t"], f"{case} call {i} beta2^t"


@pytest.mark.parametrize("case", sorted(GOLDEN))
def test_oracle_counter_matches_golden(case):
    from oracle import oracle as O
    seq = GOLDEN[case]
    ctor = (0.9, 0.999) if case in ("betas_change", "adam_defaults_2000") else (seq[0]["beta1"], seq[0]["beta2"])
    k = O.StepCounter(*ctor)
    for i, e in enumerate(seq):
        b1t, b2t = k.next(e["step"], e["beta1"], e["beta2"])
        assert (_bits(b1t), _bits(b2t)) == (e["b1t"], e["b2t"]), f"{case} call {i}"
        s = O.scalars_bt(b1t, b2t, beta1=e["beta1"], beta2=e["beta2"])
        assert _bits(s.bias_correction1) == e["bc1"] and _bits(s.bias_correction2) == e["bc2"]


def test_lazy_counter_equals_constructed():
    """A counter constructed lazily (first call's betas) behaves like one
    constructed with the same betas — the pipeline / shard's own counters."""
    from paper_2403_06504_b200 import optim as F
    a, b = F.StepCounter(), F.StepCounter(0.9, 0.95)
    for t in range(1, 30):
        for _ in range(3):
            ha, hb = a.next(F.Hparams(step=t)), b.next(F.Hparams(step=t))
            assert ha.beta_t == hb.beta_t


def test_golden_has_teeth():
    """The running product really differs from pow in the fixtures (else the
    test would not distinguish the two semantics)."""
    assert sum(e["differs_from_pow"] for e in GOLDEN["one_chunk_300_steps"]) > 100
    assert sum(e["differs_from_pow"] for e in GOLDEN["twelve_chunks_40_steps"]) > 0
    # chunks 1..K-1 of a step always take pow
    tw = GOLDEN["twelve_chunks_40_steps"]
    assert all(e["path"] == "pow" for i, e in enumerate(tw) if i % 12 and i >= 12)
    assert all(e["path"] == "product" for i, e in enumerate(tw) if i % 12 == 0)


def test_counter_rejects_step_zero():
    from paper_2403_06504_b200._lib import LIB, AdamCounter, AdamHparams, FY_ERR_CONFIG
    c = AdamCounter()
    hp = AdamHparams(1e-4, 0.9, 0.95, 1e-8, 0.1, 0, 1, 1, 1.0, 0, 0.0, 0.0)
    assert LIB.fy_adam_counter_next(C.byref(c), C.byref(hp)) == FY_ERR_CONFIG
