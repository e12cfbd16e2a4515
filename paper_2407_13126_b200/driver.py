"""Per-window planning loop around the hot path.

The reference describes the loop (the CLI at proj/tools/main.cpp is
a placeholder) and ships its pieces; this module chains them around the GPU
planner:

  for each window w:
      forecast = predict_arrivals(predictor, history = trace[:w*S], S, S,
                                  actual_next = trace window w)   predictor.hpp:53-91
      plan     = solve_dp(PlanContext{w, initial}, forecast)      solvers.hpp:242  (GPU)
      initial  = final_ranges(plan)                               evaluate.hpp:213-226
      realized = evaluate_plan(plan, actual window-w counts)      evaluate.hpp:153 (GPU)

Windows of one scenario are sequential (each needs the previous plan's final
ranges); independent scenarios advance together, one batched GPU launch per
window index (mgs_solve_batch lanes). The predictor is O(M*S) host arithmetic
(an upstream input). The first window has no history; with a
non-oracle predictor it is planned from its actual counts (what the reference's
predict_arrivals would refuse with predictor.history).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import scenario as SC


class PredictorError(ValueError):
    def __init__(self, code, message):
        super().__init__("%s: %s" % (code, message))
        self.code = code


def parse_predictor(text: str):
    """parse_predictor_spec (predictor.hpp:39-48): oracle | persistence | ewma:<alpha>."""
    if text in ("oracle", "persistence"):
        return (text, 0.0)
    if text.startswith("ewma:"):
        try:
            a = float(text[5:])
        except ValueError:
            raise PredictorError("input.number", "predictor alpha: '%s' is not a number" % text[5:])
        if not (0.0 < a <= 1.0):
            raise PredictorError("input.predictor", "ewma alpha must lie in (0,1], got %.9g" % a)
        return ("ewma", a)
    raise PredictorError("input.predictor", "unknown predictor '%s' (want oracle|persistence|ewma:<alpha>)" % text)


def _llround(e: float) -> int:
    """std::llround for the non-negative values the EWMA produces (half away from zero)."""
    r = math.floor(e)
    return r + 1 if e - r >= 0.5 else r


def predict_arrivals(spec, history, window_size, horizon, actual_next=None):
    """predict_arrivals (predictor.hpp:53-91). history: int64 [M][k*window_size]."""
    kind, alpha = spec
    if window_size < 1 or horizon < 1:
        raise PredictorError("input.predictor", "window size and horizon must be positive")
    if kind == "oracle":
        if actual_next is None:
            raise PredictorError("predictor.history", "oracle predictor needs the actual next-window counts")
        return np.asarray(actual_next, np.int64)
    out = []
    for per_model in np.asarray(history, np.int64):
        full = len(per_model) // window_size
        if full < 1:
            raise PredictorError("predictor.history", "%s needs at least one full prior window of history" % kind)
        fc = np.zeros(horizon, np.int64)
        if kind == "persistence":
            base = (full - 1) * window_size
            for ofs in range(horizon):
                fc[ofs] = per_model[base + ofs % window_size]
        else:
            for ofs in range(horizon):
                o = ofs % window_size
                e = float(per_model[o])
                for w in range(1, full):  # e = a*x + (1-a)*e, two roundings each (no FMA)
                    e = alpha * float(per_model[w * window_size + o]) + (1.0 - alpha) * e
                fc[ofs] = _llround(e)
        if (fc < 0).any():
            raise PredictorError("predictor.negative", "forecast produced a negative count")
        out.append(fc)
    return np.stack(out)


def final_ranges(sc, config, labels):
    """final_ranges (evaluate.hpp:213-226) of a plan given per-step configuration
    indices and labels: the last step's slot ranges per task, as
    [(model, 'i'|'r', start, size)]."""
    c = int(config[-1])
    out = []
    for k, (size, start) in enumerate(sc.catalog.configs[c].slots):
        lab = int(labels[-1][k])
        if lab == 0:
            continue
        m, retrain = (lab - 1) // 2, (lab - 1) % 2 == 1
        out.append((sc.models[m].name, "r" if retrain else "i", start, size))
    return sorted(out)


@dataclass
class WindowPlan:
    window: int
    options: np.ndarray
    config: np.ndarray
    labels: np.ndarray
    forecast: np.ndarray
    objective: float          # evaluate_plan on the forecast (the planner's objective)
    realized: float           # evaluate_plan on the window's actual counts
    initial: list | None      # the carried-over ranges this window was planned with


def plan_scenarios(planner, scenarios, predictor="oracle", max_windows=None):
    """Plans every window (or the first max_windows) of every scenario; returns
    [[WindowPlan per window] per scenario]. Scenarios must share window_count;
    each window index is one batched solve."""
    spec = parse_predictor(predictor)
    W = scenarios[0].window_count
    if any(sc.window_count != W for sc in scenarios):
        raise ValueError("batched scenarios must have the same window count")
    out = [[] for _ in scenarios]
    initial = [None] * len(scenarios)
    for w in range(W if max_windows is None else min(W, max_windows)):
        probs, fcs = [], []
        for i, sc in enumerate(scenarios):
            S = sc.window_size
            actual = np.stack([sc.window_arrivals(m, w) for m in range(len(sc.models))])
            if spec[0] == "oracle" or w == 0:
                fc = predict_arrivals(("oracle", 0.0), None, S, S, actual)
            else:
                fc = predict_arrivals(spec, sc.counts[:, :w * S], S, S)
            fcs.append(fc)
            probs.append(SC.Problem(sc, w, forecast=fc, initial=initial[i]))
        opts, obj, status, stats, errs = planner.solve_batch(probs)
        for i, sc in enumerate(scenarios):
            if status[i] != 0:
                from .capi import PlannerError
                raise PlannerError(int(status[i]), errs[i])
            p = probs[i]
            o = opts[i, :p.S].copy()
            en = planner.enumerate(p)
            cfg, lab = en["config"][o], en["labels"][o]
            actual = np.stack([sc.window_arrivals(m, w) for m in range(len(sc.models))])
            realized = float(planner.evaluate_batch(p, o[None], actual[None])[0, 0])
            out[i].append(WindowPlan(w, o, cfg, lab, fcs[i], float(obj[i]), realized, initial[i]))
            initial[i] = final_ranges(sc, cfg, lab)
    return out
