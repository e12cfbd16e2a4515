"""Host-side scenario model: the reference's catalog / scenario / trace grammar
loaded into flat C-ABI problems (mgs_problem).

Mirrors, in meaning and error codes, the reference loaders:
  load_catalog          proj/include/migsim/catalog.hpp:93-154
  parse_scenario_doc    proj/include/migsim/workload.hpp:164-228
  parse_trace_csv       workload.hpp:99-137
  finalize_scenario     workload.hpp:255-330 (RT derivation :80-88, accuracy carry-over :314-315)
  engine::Tables::build space.hpp:47-86 (universe, cap/rt tables)
  initial_masks         space.hpp:305-323
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import capi


class ScenarioError(ValueError):
    def __init__(self, code, message):
        self.code = code
        super().__init__("%s: %s" % (code, message))


@dataclass
class Config:
    id: str
    slots: list  # [(size, start)] sorted by start


@dataclass
class Catalog:
    gpc_count: int = 7
    mem_slices: int = 8
    configs: list = field(default_factory=list)

    def find(self, cid):
        for i, c in enumerate(self.configs):
            if c.id == cid:
                return i
        return -1


@dataclass
class Model:
    name: str
    gflops: float
    floor: int
    latency_full: float
    psi: float
    capability: dict  # size -> req/step
    data_volume: int
    rt_table: dict     # size -> steps
    acc_pre: list
    acc_post: list


@dataclass
class Scenario:
    catalog: Catalog
    models: list
    counts: np.ndarray  # int64 [M][S*W]
    window_size: int
    window_count: int

    def window_arrivals(self, m, w):
        return self.counts[m, w * self.window_size:(w + 1) * self.window_size]


def _strip(line):
    return line.split("#", 1)[0].strip(" \t\r\n")


def _int(tok, what):
    try:
        if tok.strip() != tok or not tok:
            raise ValueError
        return int(tok)
    except ValueError:
        raise ScenarioError("input.number", "%s: '%s' is not an integer" % (what, tok))


def _real(tok, what):
    try:
        return float(tok)
    except ValueError:
        raise ScenarioError("input.number", "%s: '%s' is not a number" % (what, tok))


def parse_catalog(text, source="<inline>"):
    cat = Catalog()
    saw_entry = False
    for lineno, raw in enumerate(text.splitlines(), 1):
        body = _strip(raw)
        if not body:
            continue
        toks = body.split()
        where = "%s:%d" % (source, lineno)
        if toks[0] in ("gpc_count", "mem_slices"):
            if saw_entry:
                raise ScenarioError("input.catalog", where + ": %s must precede rule/config entries" % toks[0])
            if len(toks) != 2:
                raise ScenarioError("input.catalog", where + ": expected one value")
            v = _int(toks[1], where)
            if v < 1:
                raise ScenarioError("input.catalog", where + ": value must be positive")
            setattr(cat, toks[0] if toks[0] == "mem_slices" else "gpc_count", v)
        elif toks[0] == "rule":
            saw_entry = True  # placement rules are not consumed by the planner (catalog.hpp:48-52)
        elif toks[0] == "config":
            saw_entry = True
            if len(toks) < 3:
                raise ScenarioError("input.catalog", where + ": expected 'config <id> <size>@<start>...'")
            cid = toks[1]
            if cat.find(cid) >= 0:
                raise ScenarioError("input.catalog", where + ": duplicate configuration id '%s'" % cid)
            slots = []
            for tok in toks[2:]:
                parts = tok.split("@")
                if len(parts) != 2:
                    raise ScenarioError("input.catalog", where + ": configuration '%s': malformed slot '%s'" % (cid, tok))
                size, start = _int(parts[0], where), _int(parts[1], where)
                if size < 1 or size > cat.gpc_count:
                    raise ScenarioError("input.catalog", "configuration '%s': slot size %d out of range" % (cid, size))
                if start < 0 or start + size > cat.gpc_count:
                    raise ScenarioError("input.catalog", "configuration '%s': slot exceeds the axis" % cid)
                slots.append((size, start))
            slots.sort(key=lambda x: x[1])  # stable, like std::sort on distinct starts
            for a, b in zip(slots, slots[1:]):
                if a[1] + a[0] > b[1]:
                    raise ScenarioError("input.catalog", "configuration '%s': overlapping slices" % cid)
            cat.configs.append(Config(cid, slots))
        else:
            raise ScenarioError("input.catalog", where + ": unknown key '%s'" % toks[0])
    if not cat.configs:
        raise ScenarioError("input.catalog", source + ": no configurations declared")
    if cat.gpc_count > capi.MAX_SLOTS:
        raise ScenarioError("input.catalog", "gpc_count above %d is not supported by the ABI" % capi.MAX_SLOTS)
    return cat


def load_catalog(path):
    with open(path) as f:
        return parse_catalog(f.read(), path)


def derive_rt_table(capability, volume, name):
    """RT[k] = ceil(3*volume/cap[k]) (workload.hpp:80-88)."""
    if volume <= 0:
        raise ScenarioError("input.scenario", "model '%s': data_volume must be positive" % name)
    rt = {}
    for k, cap in sorted(capability.items()):
        if cap <= 0:
            raise ScenarioError("input.scenario", "model '%s': capability[%d] must be positive" % (name, k))
        rt[k] = int(math.ceil(3.0 * float(volume) / cap))
    return rt


def _size_map(text, path):
    out = {}
    for tok in text.split():
        parts = tok.split(":")
        if len(parts) != 2:
            raise ScenarioError("input.scenario", path + ": expected '<size>:<value>' pairs")
        k = _int(parts[0], path)
        if k in out:
            raise ScenarioError("input.scenario", path + ": duplicate size %d" % k)
        out[k] = _real(parts[1], path)
    if not out:
        raise ScenarioError("input.scenario", path + ": empty map")
    return out


def finalize(catalog, models, counts, window_size, window_count):
    """finalize_scenario (workload.hpp:255-330)."""
    if window_size < 2:
        raise ScenarioError("input.scenario", "windows.size: must be >= 2")
    if window_count < 1:
        raise ScenarioError("input.scenario", "windows.count: must be >= 1")
    sizes = sorted({s for c in catalog.configs for (s, _) in c.slots})
    for m in models:
        path = "models[%s]" % m.name
        if m.gflops <= 0:
            raise ScenarioError("input.scenario", path + ".gflops: must be positive")
        if m.floor < 1 or m.floor > catalog.gpc_count:
            raise ScenarioError("input.scenario", path + ".min_deploy_gpcs: out of range")
        if m.latency_full <= 0:
            raise ScenarioError("input.scenario", path + ".latency_full: must be positive")
        if m.psi < 0:
            raise ScenarioError("input.scenario", path + ".reconfig_overhead: must be >= 0")
        prev = 0.0
        for k, v in sorted(m.capability.items()):
            if k < 1 or k > catalog.gpc_count:
                raise ScenarioError("input.scenario", path + ".capability: size %d out of range" % k)
            if v < prev:
                raise ScenarioError("input.scenario", path + ".capability: not nondecreasing at size %d" % k)
            prev = v
            if k >= m.floor and v <= 0:
                raise ScenarioError("input.scenario", path + ".capability[%d]: must be positive" % k)
        for k in sizes:
            if k >= m.floor and k not in m.capability:
                raise ScenarioError("input.scenario", path + ".capability: missing catalog size %d" % k)
        if not m.rt_table:
            m.rt_table = derive_rt_table(m.capability, m.data_volume, m.name)
        prev_rt = -1
        for k, v in sorted(m.rt_table.items()):
            if k < 1 or k > catalog.gpc_count:
                raise ScenarioError("input.scenario", path + ".rt_table: size %d out of range" % k)
            if v < 1:
                raise ScenarioError("input.scenario", path + ".rt_table[%d]: must be >= 1 second" % k)
            if prev_rt >= 0 and v > prev_rt:
                raise ScenarioError("input.scenario", path + ".rt_table: not nonincreasing at size %d" % k)
            prev_rt = v
        if not m.acc_pre or not m.acc_post:
            raise ScenarioError("input.scenario", path + ".accuracy: required")
        if len(m.acc_post) == 1:
            m.acc_post = m.acc_post * window_count
        if len(m.acc_post) != window_count:
            raise ScenarioError("input.scenario", path + ".accuracy_post: want 1 or %d values" % window_count)
        if len(m.acc_pre) > window_count:
            raise ScenarioError("input.scenario", path + ".accuracy_pre: more values than windows")
        for x in m.acc_pre + m.acc_post:
            if x < 0.0 or x > 1.0:
                raise ScenarioError("input.scenario", path + ".accuracy: values must lie in [0,1]")
        while len(m.acc_pre) < window_count:  # carry-over (workload.hpp:314-315)
            m.acc_pre.append(m.acc_post[len(m.acc_pre) - 1])
    counts = np.asarray(counts, dtype=np.int64)
    if counts.shape[0] != len(models):
        raise ScenarioError("input.trace-length-mismatch", "trace: model count mismatch")
    if counts.shape[1] != window_size * window_count:
        raise ScenarioError("input.trace-length-mismatch", "trace-length-mismatch")
    if (counts < 0).any():
        raise ScenarioError("input.trace", "trace: negative count")
    return Scenario(catalog, models, counts, window_size, window_count)


def load_scenario(path):
    """load_scenario (workload.hpp:337-385), granularity 1 only."""
    sec, cur = None, None
    size = count = None
    gran = 1.0
    cat_file = trace_file = None
    order, keys = [], {}
    with open(path) as f:
        lines = f.read().splitlines()
    for lineno, raw in enumerate(lines, 1):
        body = _strip(raw)
        if not body:
            continue
        where = "%s:%d" % (path, lineno)
        if body[0] == "[":
            if body[-1] != "]":
                raise ScenarioError("input.scenario", where + ": malformed section header")
            sec = body[1:-1]
            cur = None
            if sec not in ("windows", "catalog", "models", "trace"):
                raise ScenarioError("input.scenario", where + ": unknown section '%s'" % sec)
            continue
        toks = body.split()
        key = toks[0]
        if sec == "windows":
            if len(toks) != 2:
                raise ScenarioError("input.scenario", where + ": expected one value")
            if key == "size":
                size = _int(toks[1], "windows.size")
            elif key == "count":
                count = _int(toks[1], "windows.count")
            elif key == "granularity":
                gran = _real(toks[1], "windows.granularity")
            else:
                raise ScenarioError("input.scenario", where + ": windows: unknown key '%s'" % key)
        elif sec in ("catalog", "trace"):
            if key == "file" and len(toks) == 2:
                if sec == "catalog":
                    cat_file = toks[1]
                else:
                    trace_file = toks[1]
            else:
                raise ScenarioError("input.scenario", where + ": %s: unknown key '%s'" % (sec, key))
        elif sec == "models":
            if key == "model":
                if len(toks) != 2:
                    raise ScenarioError("input.scenario", where + ": model declaration needs a name")
                cur = toks[1]
                if cur in keys:
                    raise ScenarioError("input.scenario", where + ": duplicate model '%s'" % cur)
                order.append(cur)
                keys[cur] = {}
            else:
                if cur is None:
                    raise ScenarioError("input.scenario", where + ": model key before any 'model' line")
                if key in keys[cur]:
                    raise ScenarioError("input.scenario", where + ": duplicate key '%s'" % key)
                keys[cur][key] = " ".join(toks[1:])
        else:
            raise ScenarioError("input.scenario", where + ": key outside any section")
    if size is None or count is None:
        raise ScenarioError("input.scenario", path + ": windows.size and windows.count are required")
    if gran != 1.0:
        raise ScenarioError("input.granularity", "granularity rescale is outside the planner hot path")
    d = os.path.dirname(path)
    res = lambda p: p if os.path.isabs(p) else os.path.join(d, p)
    catalog = load_catalog(res(cat_file))
    models = []
    for name in order:
        k = keys[name]
        mp = "models[%s]" % name

        def need(key):
            if key not in k:
                raise ScenarioError("input.scenario", "%s.%s: required key missing" % (mp, key))
            return k[key]
        rt = {}
        if "rt_table" in k:
            rt = {kk: int(v) for kk, v in _size_map(k["rt_table"], mp + ".rt_table").items()}
        elif "data_volume" not in k:
            raise ScenarioError("input.scenario", mp + ": either rt_table or data_volume is required")
        models.append(Model(name, _real(need("gflops"), mp), _int(need("min_deploy_gpcs"), mp),
                            _real(need("latency_full"), mp), _real(need("reconfig_overhead"), mp),
                            _size_map(need("capability"), mp + ".capability"),
                            _int(k["data_volume"], mp) if "data_volume" in k else 0, rt,
                            [_real(x, mp) for x in need("accuracy_pre").split()],
                            [_real(x, mp) for x in need("accuracy_post").split()]))
    horizon = size * count
    counts = np.full((len(order), horizon), -1, dtype=np.int64)
    idx = {n: i for i, n in enumerate(order)}
    with open(res(trace_file)) as f:
        tl = f.read().splitlines()
    if not tl or tl[0].strip() != "second,model,count":
        raise ScenarioError("input.trace", "expected header 'second,model,count'")
    for raw in tl[1:]:
        b = raw.strip()
        if not b:
            continue
        parts = [x.strip() for x in b.split(",")]
        if len(parts) != 3:
            raise ScenarioError("input.trace", "expected 'second,model,count'")
        s, m, c = int(parts[0]), parts[1], int(parts[2])
        if m not in idx:
            raise ScenarioError("input.trace", "unknown model '%s'" % m)
        if c < 0:
            raise ScenarioError("input.trace", "negative count")
        if s < 0 or s >= horizon:
            raise ScenarioError("input.trace-length-mismatch", "second outside horizon")
        if counts[idx[m], s] >= 0:
            raise ScenarioError("input.trace", "duplicate row")
        counts[idx[m], s] = c
    if (counts < 0).any():
        raise ScenarioError("input.trace-length-mismatch", "trace-length-mismatch")
    return finalize(catalog, models, counts, size, count)


def universe(catalog):
    """Distinct (start, size) instances in first-appearance order (space.hpp:56-64)."""
    uid = {}
    for c in catalog.configs:
        for size, start in c.slots:
            uid.setdefault((start, size), len(uid))
    return uid


def initial_masks(sc, initial):
    """initial_masks (space.hpp:305-323). `initial`: iterable of (model_name, kind,
    start, size) with kind 'i' or 'r'."""
    uid = universe(sc.catalog)
    names = [m.name for m in sc.models]
    masks = [0] * capi.MAX_MODELS
    per = {}
    for name, kind, start, size in initial:
        if kind != "i" or name not in names:
            continue
        per.setdefault(names.index(name), []).append((start, size))
    for m, ranges in per.items():
        mask, foreign = 0, False
        for r in ranges:
            if r in uid:
                mask |= 1 << uid[r]
            else:
                foreign = True
        masks[m] = capi.FOREIGN_MASK if foreign else mask
    return masks


class Problem:
    """An mgs_problem plus the numpy buffers it points into (kept alive here)."""

    def __init__(self, sc: Scenario, window: int = 0, forecast=None, initial=None, state_budget=4_000_000,
                 workers=1):
        self.scenario = sc
        self.window = window
        cat = sc.catalog
        offs, sizes, starts = [0], [], []
        for c in cat.configs:
            for size, start in c.slots:
                sizes.append(size)
                starts.append(start)
            offs.append(len(sizes))
        self.slot_offset = np.asarray(offs, dtype=np.int32)
        self.slot_size = np.asarray(sizes, dtype=np.int32)
        self.slot_start = np.asarray(starts, dtype=np.int32)
        M = len(sc.models)
        S = sc.window_size
        if forecast is None:
            forecast = np.stack([sc.window_arrivals(m, window) for m in range(M)])
        self.forecast = np.ascontiguousarray(np.asarray(forecast, dtype=np.int64))
        p = capi.mgs_problem()
        lat = p.lattice
        lat.n_configs = len(cat.configs)
        lat.gpc_count = cat.gpc_count
        lat.slot_offset = capi.ptr(self.slot_offset, C.c_int32)
        lat.slot_size = capi.ptr(self.slot_size, C.c_int32)
        lat.slot_start = capi.ptr(self.slot_start, C.c_int32)
        t = p.tables
        t.models = M
        t.steps = S
        for m, mod in enumerate(sc.models[:capi.MAX_MODELS]):
            for k in range(capi.SIZES):
                t.cap_by_size[m][k] = 0.0
                t.rt_by_size[m][k] = -1
            for k, v in mod.capability.items():
                if 1 <= k <= 7:
                    t.cap_by_size[m][k] = v
            for k, v in mod.rt_table.items():
                if 1 <= k <= 7:
                    t.rt_by_size[m][k] = v
            t.floor_gpcs[m] = mod.floor
            t.psi[m] = mod.psi
            t.acc_pre[m] = mod.acc_pre[window]
            t.acc_post[m] = mod.acc_post[window]
        p.forecast = capi.ptr(self.forecast, C.c_int64)
        p.forecast_len = self.forecast.shape[1]
        p.has_initial = 0
        if initial is not None:
            p.has_initial = 1
            for m, v in enumerate(initial_masks(sc, initial)):
                p.init_mask[m] = v
        p.state_budget = int(state_budget)
        p.workers = workers
        self.c = p
        self.M, self.S = M, S

    def byref(self):
        return C.byref(self.c)
