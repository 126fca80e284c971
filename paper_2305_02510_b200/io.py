"""Wire formats of the reference (proj/src/io.cpp:107-373, io.hpp:16-60), so
files produced by the spikeforge CLI load here and rasters written here are
byte-identical to ``write_raster``:

* network JSON v1 (serialize_network / parse_network, io.cpp:107-210):
  fixed key order, 2-space indent, shortest round-trip numbers, "inf" for the
  infinite leak;
* raster CSV ``step,neuron_id`` (io.cpp:212-248);
* stimulus CSV ``step,neuron_id,amplitude`` (io.cpp:250-280);
* STDP JSON (io.cpp:282-315);
* bench CSV (io.cpp:317-373).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from decimal import Decimal
from typing import List, Optional

import numpy as np

from .model import (NetworkDef, NeuronParams, SpikeRaster, StdpConfig, StimulusEntry,
                    StimulusSchedule, SynapseDef, validate_network, validate_stdp)


class FormatError(RuntimeError):
    """Malformed document or schema violation (spikeforge::FormatError)."""


def _num(v: float) -> str:
    """Shortest round-trip rendering; integral doubles as '1.0' like nlohmann."""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    r = repr(float(v))
    if r == "inf" or r == "nan":
        raise FormatError("non-finite number")
    return r


def _shortest(v: float) -> str:
    """std::to_chars(double) with no format (io.cpp:17-21): the shortest
    round-trip digits (those of repr), written in fixed or scientific notation,
    whichever has fewer characters, fixed on a tie -- so 2 (not 2.0), 0.001,
    1e-04, 1e+05, 1.5e-07, 123456; a fixed integral value prints all its exact
    digits (531527556293501632, not ...630)."""
    f = float(v)
    if not math.isfinite(f):
        raise FormatError("non-finite number")
    if f == 0.0:
        return "-0" if math.copysign(1.0, f) < 0 else "0"
    sign, digs, exp = Decimal(repr(f)).as_tuple()
    full = "".join(map(str, digs))
    d = full.rstrip("0")            # value = d * 10**e, d without trailing zeros
    e = exp + len(full) - len(d)
    k = len(d)
    if e >= 0:   # integral: printf("%.0f")'s exact digits, same width as d + "0" * e
        fixed = str(int(abs(f)))
    else:
        point = k + e
        fixed = d[:point] + "." + d[point:] if point > 0 else "0." + "0" * (-point) + d
    x = k - 1 + e
    sci = d[0] + ("." + d[1:] if k > 1 else "") + "e" + ("-" if x < 0 else "+") + str(abs(x)).zfill(2)
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + out


def serialize_network(net: NetworkDef) -> str:
    a = net.to_arrays()
    beh = a.get("behavior") or ["lif"] * len(a["threshold"])
    lines = ["{", '  "version": 1,', '  "neurons": [']
    nn = len(a["threshold"])
    for i in range(nn):
        leak = a["leak"][i]
        leak_s = '"inf"' if math.isinf(leak) else _num(leak)
        body = (f'      "threshold": {_num(a["threshold"][i])},\n'
                f'      "leak": {leak_s},\n'
                f'      "reset": {_num(a["reset"][i])},\n'
                f'      "refractory": {int(a["refractory"][i])},\n'
                f'      "axonal_delay": {int(a["axonal"][i])},\n'
                f'      "behavior": {json.dumps(beh[i])}')
        lines.append("    {\n" + body + "\n    }" + ("," if i + 1 < nn else ""))
    lines.append("  ],")
    m = len(a["pre"])
    if m == 0:
        lines[-1] = "  ],"
        lines.append('  "synapses": [],')
    else:
        lines.append('  "synapses": [')
        for s in range(m):
            body = (f'      "pre": {int(a["pre"][s])},\n'
                    f'      "post": {int(a["post"][s])},\n'
                    f'      "weight": {_num(a["weight"][s])},\n'
                    f'      "delay": {int(a["delay"][s])},\n'
                    f'      "stdp": {"true" if a["stdp"][s] else "false"}')
            lines.append("    {\n" + body + "\n    }" + ("," if s + 1 < m else ""))
        lines.append("  ],")
    if net.metadata:
        lines.append('  "metadata": {')
        items = sorted(net.metadata.items())
        for k, (key, val) in enumerate(items):
            lines.append(f"    {json.dumps(key)}: {json.dumps(val)}" + ("," if k + 1 < len(items) else ""))
        lines.append("  }")
    else:
        lines.append('  "metadata": {}')
    if nn == 0:
        lines[2] = '  "neurons": [],'
        del lines[3]
    lines.append("}")
    return "\n".join(lines) + "\n"


def _require(obj, where, required, optional=()):
    for k in required:
        if k not in obj:
            raise FormatError(f'{where}: missing required key "{k}"')
    for k in obj:
        if k not in required and k not in optional:
            raise FormatError(f'{where}: unknown key "{k}"')


def _int(obj, where, key):
    v = obj[key]
    if isinstance(v, bool) or not isinstance(v, int):
        raise FormatError(f"{where}.{key}: expected an integer")
    return v


def _number(obj, where, key):
    v = obj[key]
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise FormatError(f"{where}.{key}: expected a number")
    return float(v)


def _parse_json(text: str, what: str):
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise FormatError(f"{what}: malformed JSON at byte {e.pos}: {e.msg}") from None


def parse_network(text: str) -> NetworkDef:
    doc = _parse_json(text, "network")
    if not isinstance(doc, dict):
        raise FormatError("network: top-level value must be an object")
    _require(doc, "network", ("version", "neurons", "synapses"), ("metadata",))
    if isinstance(doc["version"], bool) or doc["version"] != 1:
        raise FormatError("network.version: unsupported version (expected 1)")
    if not isinstance(doc["neurons"], list):
        raise FormatError("network.neurons: expected an array")
    if not isinstance(doc["synapses"], list):
        raise FormatError("network.synapses: expected an array")
    net = NetworkDef()
    for i, q in enumerate(doc["neurons"]):
        where = f"neurons[{i}]"
        if not isinstance(q, dict):
            raise FormatError(f"{where}: expected an object")
        _require(q, where, ("threshold", "leak", "reset", "refractory"), ("axonal_delay", "behavior"))
        p = NeuronParams()
        p.threshold = _number(q, where, "threshold")
        leak = q["leak"]
        if isinstance(leak, str):
            if leak != "inf":
                raise FormatError(f'{where}.leak: expected a number or "inf"')
            p.leak = math.inf
        elif isinstance(leak, (int, float)) and not isinstance(leak, bool):
            p.leak = float(leak)
        else:
            raise FormatError(f'{where}.leak: expected a number or "inf"')
        p.reset = _number(q, where, "reset")
        p.refractory = _int(q, where, "refractory")
        p.axonal_delay = _int(q, where, "axonal_delay") if "axonal_delay" in q else 0
        if "behavior" in q:
            if not isinstance(q["behavior"], str):
                raise FormatError(f"{where}.behavior: expected a string")
            p.behavior = q["behavior"]
        net.neurons.append(p)
    for i, q in enumerate(doc["synapses"]):
        where = f"synapses[{i}]"
        if not isinstance(q, dict):
            raise FormatError(f"{where}: expected an object")
        _require(q, where, ("pre", "post", "weight", "delay"), ("stdp",))
        s = SynapseDef(_int(q, where, "pre"), _int(q, where, "post"), _number(q, where, "weight"),
                       _int(q, where, "delay"))
        if "stdp" in q:
            if not isinstance(q["stdp"], bool):
                raise FormatError(f"{where}.stdp: expected a boolean")
            s.stdp_enabled = q["stdp"]
        net.synapses.append(s)
    if "metadata" in doc:
        if not isinstance(doc["metadata"], dict):
            raise FormatError("network.metadata: expected an object")
        for k, v in doc["metadata"].items():
            if not isinstance(v, str):
                raise FormatError(f"network.metadata.{k}: expected a string value")
            net.metadata[k] = v
    bad = validate_network(net)
    if bad:
        raise FormatError(f"network: {bad[0]}")
    return net


def write_raster(r: SpikeRaster) -> str:
    """io.cpp:212-225 -- byte-identical."""
    st = np.asarray(r.steps_array, dtype=np.int64)
    nr = np.asarray(r.neurons_array, dtype=np.int64)
    if st.size == 0:
        return "step,neuron_id\n"
    body = "\n".join(f"{a},{b}" for a, b in zip(st.tolist(), nr.tolist()))
    return "step,neuron_id\n" + body + "\n"


def _csv_lines(text: str, what: str) -> List[str]:
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise FormatError(f"{what}: empty input")
    return lines


def _ll(field: str, where: str) -> int:
    f = field.strip() if False else field
    if not f or not (f.lstrip("-").isdigit()):
        raise FormatError(f'{where}: expected an integer, got "{field}"')
    return int(f)


def parse_raster(text: str) -> SpikeRaster:
    lines = _csv_lines(text, "raster")
    if lines[0] != "step,neuron_id":
        raise FormatError('raster: line 1: expected header "step,neuron_id"')
    steps, neurons = [], []
    last = None
    for i, line in enumerate(lines[1:], start=2):
        where = f"raster: line {i}"
        fields = line.split(",")
        if len(fields) != 2:
            raise FormatError(f"{where}: expected 2 fields")
        s, n = _ll(fields[0], where), _ll(fields[1], where)
        if s < 0 or n < 0:
            raise FormatError(f"{where}: negative value")
        if last is not None and not (last < (s, n)):
            raise FormatError(f"{where}: rows must be strictly increasing by (step, neuron_id)")
        last = (s, n)
        steps.append(s)
        neurons.append(n)
    st = np.array(steps, dtype=np.int32)
    nr = np.array(neurons, dtype=np.int32)
    return SpikeRaster(neuron_count=int(nr.max()) + 1 if nr.size else 0,
                       step_count=int(st.max()) + 1 if st.size else 0, steps_array=st, neurons_array=nr)


def write_stimulus(stim: StimulusSchedule) -> str:
    out = ["step,neuron_id,amplitude"]
    for e in stim.entries:
        out.append(f"{e.step},{e.neuron},{_shortest(e.amplitude)}")
    return "\n".join(out) + "\n"


def parse_stimulus(text: str) -> StimulusSchedule:
    lines = _csv_lines(text, "stimulus")
    if lines[0] != "step,neuron_id,amplitude":
        raise FormatError('stimulus: line 1: expected header "step,neuron_id,amplitude"')
    stim = StimulusSchedule()
    for i, line in enumerate(lines[1:], start=2):
        where = f"stimulus: line {i}"
        fields = line.split(",")
        if len(fields) != 3:
            raise FormatError(f"{where}: expected 3 fields")
        try:
            amp = float(fields[2])
        except ValueError:
            raise FormatError(f'{where}: expected a number, got "{fields[2]}"') from None
        stim.entries.append(StimulusEntry(_ll(fields[0], where), _ll(fields[1], where), amp))
    return stim


def serialize_stdp(cfg: StdpConfig) -> str:
    def arr(v):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(f"    {_num(x)}" for x in v) + "\n  ]"
    return ("{\n"
            f'  "window": {int(cfg.window)},\n'
            f'  "a_plus": {arr(cfg.a_plus)},\n'
            f'  "a_minus": {arr(cfg.a_minus)},\n'
            f'  "w_min": {_num(cfg.w_min)},\n'
            f'  "w_max": {_num(cfg.w_max)}\n'
            "}\n")


def parse_stdp(text: str) -> StdpConfig:
    doc = _parse_json(text, "stdp")
    if not isinstance(doc, dict):
        raise FormatError("stdp: top-level value must be an object")
    _require(doc, "stdp", ("window", "a_plus", "a_minus", "w_min", "w_max"))
    cfg = StdpConfig(window=_int(doc, "stdp", "window"), a_plus=[], a_minus=[])
    if not isinstance(doc["a_plus"], list) or not isinstance(doc["a_minus"], list):
        raise FormatError("stdp: a_plus and a_minus must be arrays")
    for key, dst in (("a_plus", cfg.a_plus), ("a_minus", cfg.a_minus)):
        for v in doc[key]:
            if isinstance(v, bool) or not isinstance(v, (int, float)):
                raise FormatError(f"stdp.{key}: expected numbers")
            dst.append(float(v))
    cfg.w_min = _number(doc, "stdp", "w_min")
    cfg.w_max = _number(doc, "stdp", "w_max")
    bad = validate_stdp(cfg)
    if bad:
        raise FormatError(bad[0])
    return cfg


BENCH_HEADER = "backend,neurons,connection_probability,steps,wall_time_seconds,spike_count,seed"


@dataclass
class BenchRow:  # io.hpp:40-50
    backend: str = ""
    neurons: int = 0
    connection_probability: float = 0.0
    steps: int = 0
    wall_time_seconds: Optional[float] = None
    spike_count: int = 0
    seed: int = 0


def format_bench_row(row: BenchRow) -> str:
    wall = "timeout" if row.wall_time_seconds is None else "%.6f" % row.wall_time_seconds
    return (f"{row.backend},{row.neurons},{_shortest(row.connection_probability)},{row.steps},"
            f"{wall},{row.spike_count},{row.seed}\n")


def write_bench(rows: List[BenchRow]) -> str:
    return BENCH_HEADER + "\n" + "".join(format_bench_row(r) for r in rows)


def parse_bench(text: str) -> List[BenchRow]:
    lines = _csv_lines(text, "bench")
    if lines[0] != BENCH_HEADER:
        raise FormatError("bench: line 1: unexpected header")
    rows = []
    for i, line in enumerate(lines[1:], start=2):
        where = f"bench: line {i}"
        f = line.split(",")
        if len(f) != 7:
            raise FormatError(f"{where}: expected 7 fields")
        rows.append(BenchRow(f[0], _ll(f[1], where), float(f[2]), _ll(f[3], where),
                             None if f[4] == "timeout" else float(f[4]), _ll(f[5], where),
                             _ll(f[6], where)))
    return rows


def read_file(path: str) -> str:
    try:
        with open(path, "r", newline="") as fh:
            return fh.read()
    except OSError:
        raise FormatError(f"cannot open file: {path}") from None


def write_file(path: str, contents: str) -> None:
    try:
        with open(path, "w", newline="") as fh:
            fh.write(contents)
    except OSError:
        raise FormatError(f"cannot write file: {path}") from None
