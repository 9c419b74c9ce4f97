"""Generates tests/golden/deepspeed_step_counter.json: the beta1^t / beta2^t
DeepSpeed 0.9.3's CPU Adam hands its kernel over call sequences, from an
independent pure-Python transcription of Adam_Optimizer::IncrementStep
(deepspeed csrc/includes/cpu_adam.h; DeepSpeed is not vendored under
/root/reference and not installed here — PAPER.md:275,471 name it):

    members: float _betta1, _betta2, _betta1_t = 1.0, _betta2_t = 1.0;
             size_t _step = 0   (constructor, betas of the optimizer)
    IncrementStep(size_t step, float beta1, float beta2):
        if (beta1 != _betta1 || beta2 != _betta2) {
            _step = step; _betta1 = beta1; _betta2 = beta2;
            _betta1_t = std::pow(_betta1, step);   // pow(double, double) -> float
            _betta2_t = std::pow(_betta2, step);
        } else {
            _step++;
            if (_step != step) { _betta1_t = std::pow(_betta1, step); ...; _step = step; }
            else { _betta1_t *= _betta1; _betta2_t *= _betta2; }   // float running product
        }

DeepSpeedCPUAdam.step() calls adam_update (-> IncrementStep) once per
parameter tensor; under ZeRO-Infinity once per sub-group, i.e. once per
chunk, with state['step'] already incremented for the current step.
Float32 arithmetic is numpy float32 (IEEE single, round to nearest).
Run: python tests/golden/make_step_counter_golden.py
"""
import json
import math
from pathlib import Path

import numpy as np

f32 = np.float32


class IncrementStep:
    def __init__(self, beta1, beta2):
        self.b1, self.b2 = f32(beta1), f32(beta2)
        self.b1t, self.b2t = f32(1.0), f32(1.0)
        self.step = 0

    def __call__(self, step, beta1, beta2):
        beta1, beta2 = f32(beta1), f32(beta2)
        path = "pow"
        if beta1 != self.b1 or beta2 != self.b2:
            self.step, self.b1, self.b2 = step, beta1, beta2
            self.b1t = f32(math.pow(float(self.b1), float(step)))
            self.b2t = f32(math.pow(float(self.b2), float(step)))
        else:
            self.step += 1
            if self.step != step:
                self.b1t = f32(math.pow(float(self.b1), float(step)))
                self.b2t = f32(math.pow(float(self.b2), float(step)))
                self.step = step
            else:
                self.b1t = f32(self.b1t * self.b1)
                self.b2t = f32(self.b2t * self.b2)
                path = "product"
        return self.b1t, self.b2t, path


def bits(x):
    return int(np.array([x], dtype=np.float32).view(np.uint32)[0])


def sequence(ctor, calls):
    k = IncrementStep(*ctor)
    out = []
    for step, b1, b2 in calls:
        b1t, b2t, path = k(step, b1, b2)
        bc1 = f32(f32(1.0) - b1t)
        bc2 = f32(f32(1.0) / np.sqrt(f32(f32(1.0) - b2t)))
        pow1 = f32(math.pow(float(f32(b1)), float(step)))
        out.append(dict(step=step, beta1=float(f32(b1)), beta2=float(f32(b2)), b1t=bits(b1t),
                        b2t=bits(b2t), bc1=bits(bc1), bc2=bits(bc2), path=path,
                        differs_from_pow=bits(b1t) != bits(pow1)))
    return out


def main():
    g = (0.9, 0.95)
    cases = {
        # one chunk per step: the running product over 300 steps
        "one_chunk_300_steps": sequence(g, [(t, *g) for t in range(1, 301)]),
        # C1-like: 12 chunks per step, 40 steps (chunk 0 on the product, 1..11 on pow)
        "twelve_chunks_40_steps": sequence(g, [(t, *g) for t in range(1, 41) for _ in range(12)]),
        # resumed from a checkpoint at step 1000 (fresh optimizer), 3 chunks, 20 steps
        "resume_at_1000": sequence(g, [(t, *g) for t in range(1000, 1020) for _ in range(3)]),
        # betas changed at step 11 (warm-up schedule), 2 chunks per step
        "betas_change": sequence((0.9, 0.999), [(t, 0.9, 0.999 if t <= 10 else 0.95)
                                                for t in range(1, 21) for _ in range(2)]),
        # torch defaults, 1 chunk, 2000 steps: the product drifts from pow
        "adam_defaults_2000": sequence((0.9, 0.999), [(t, 0.9, 0.999) for t in range(1, 2001)]),
    }
    out = Path(__file__).with_name("deepspeed_step_counter.json")
    out.write_text(json.dumps(cases, separators=(",", ":")))
    for k, v in cases.items():
        print(k, len(v), "calls,", sum(e["differs_from_pow"] for e in v), "differ from pow")


if __name__ == "__main__":
    main()
