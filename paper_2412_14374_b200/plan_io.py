"""Plan artifacts in the reference CLI's wire format.

``pipecraft plan`` (pkg/src/pipecraft/cli.py:194-204) compiles one JSON run
config into ``schedule.json``, ``taskgraph.json`` and ``commplan.json``.  This
module reads the same config document (version 1: ``model.*``, ``parallel.*``,
``output.dir``; cli.py:75-126) and writes the same three files byte for byte,
so plans interchange both ways: a schedule written by the reference loads here
(``parallel.schedule_file``, cli.py:129-137) and a commplan written here
loads into the reference (its ``CommPlan`` JSON, comms.py:103-118).

Errors keep the reference's contract: a bad field raises ``ConfigError`` whose
message starts with the dotted field path.
"""
from __future__ import annotations

import json
from pathlib import Path

from . import comms as C
from . import ir as I
from . import schedules as S
from . import taskgraph as T

SCHEDULE_NAMES = ("gpipe", "1f1b", "interleaved")


class ConfigError(ValueError):
    """Invalid run configuration; message cites the offending field."""


def _field(doc: dict, path: str, default=None, required=False):
    cur = doc
    for part in path.split("."):
        if not isinstance(cur, dict) or part not in cur:
            if required:
                raise ConfigError(f"{path}: missing required field")
            return default
        cur = cur[part]
    return cur


class PlanConfig:
    """The planning half of the reference's RunConfig (cli.py:75-126); the
    cost model / sweep fields belong to the simulator and are ignored."""

    def __init__(self, doc: dict, base_dir: Path | str = "."):
        self.doc, self.base_dir = doc, Path(base_dir)
        if _field(doc, "version", default=1) != 1:
            raise ConfigError("version: only config version 1 is supported")
        try:
            self.model = I.ModelConfig(
                layers=int(_field(doc, "model.layers", required=True)),
                width=int(_field(doc, "model.width", required=True)),
                microbatch_size=int(_field(doc, "model.microbatch_size", required=True)),
                yield_every=int(_field(doc, "model.yield_every", default=1)),
                tied_weights=bool(_field(doc, "model.tied_weights", default=False)))
        except I.GraphError as e:
            raise ConfigError(f"model: {e}") from e
        self.learning_rate = float(_field(doc, "model.learning_rate", default=0.1))
        self.P = int(_field(doc, "parallel.num_actors", required=True))
        self.M = int(_field(doc, "parallel.num_microbatches", required=True))
        self.V = int(_field(doc, "parallel.circular_repeat", default=1))
        for name, v in (("num_actors", self.P), ("num_microbatches", self.M),
                        ("circular_repeat", self.V)):
            if v < 1:
                raise ConfigError(f"parallel.{name}: must be >= 1")
        self.schedule_name = _field(doc, "parallel.schedule", default="1f1b")
        self.schedule_file = _field(doc, "parallel.schedule_file")
        if self.schedule_file is None and self.schedule_name not in SCHEDULE_NAMES:
            raise ConfigError(f"parallel.schedule: {self.schedule_name!r} not in {SCHEDULE_NAMES}")
        if self.V > 1 and self.M % self.P != 0:
            raise ConfigError("parallel.num_microbatches: M must be divisible by P when "
                              "parallel.circular_repeat > 1")
        self.commute = bool(_field(doc, "parallel.commute_shared_grads", default=True))
        self.seed = int(_field(doc, "seed", default=0))
        self.out_dir = Path(_field(doc, "output.dir", default="out"))

    @classmethod
    def load(cls, path) -> "PlanConfig":
        p = Path(path)
        try:
            doc = json.loads(p.read_text())
        except OSError as e:
            raise ConfigError(f"config: cannot read {path} ({e})") from e
        except json.JSONDecodeError as e:
            raise ConfigError(f"config: invalid JSON in {path} ({e})") from e
        return cls(doc, p.parent)

    def schedule(self) -> S.Schedule:
        if self.schedule_file:
            path = Path(self.schedule_file)
            if not path.is_absolute() and not path.exists():
                path = self.base_dir / path
            try:
                s = S.load_schedule(path)
            except (OSError, S.ScheduleError) as e:
                raise ConfigError(f"parallel.schedule_file: {e}") from e
        else:
            s = {"gpipe": lambda: S.gpipe(self.P, self.M),
                 "1f1b": lambda: S.one_f_one_b(self.P, self.M),
                 "interleaved": lambda: S.interleaved_1f1b(self.P, self.M, self.V)
                 }[self.schedule_name]()
        if s.num_actors != self.P or s.num_microbatches != self.M:
            raise ConfigError(
                f"parallel.schedule_file: schedule is for P={s.num_actors}, "
                f"M={s.num_microbatches}, config says P={self.P}, M={self.M}")
        return s

    def partition(self) -> I.StagePartition:
        p = I.derive_backward(I.partition_stages(I.build_model(self.model)))
        want = None if self.schedule_file else self.P * self.V
        if want is not None and p.num_stages != want:
            raise ConfigError(
                f"model.yield_every: model has {p.num_stages} stages but parallel config "
                f"needs num_actors x circular_repeat = {want}")
        return p


def compile_plan(cfg: PlanConfig):
    """(partition, schedule, TaskGraph, fused CommPlan), as cli.py:167-186."""
    p, s = cfg.partition(), cfg.schedule()
    if p.num_stages != s.num_stages:
        raise ConfigError(f"model.yield_every: model has {p.num_stages} stages but the "
                          f"schedule has {s.num_stages}")
    tg = T.unroll(p, s)
    if cfg.commute:
        tg = T.commute_grad_accumulation(tg)
    tg = T.infer_outer_placement(tg, p)
    return p, s, tg, C.plan_pipeline(tg)


def _write_json(path: Path, doc: dict):
    path.write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def write_plan(out_dir, s: S.Schedule, tg: T.TaskGraph, cp: C.CommPlan) -> dict:
    """schedule.json / taskgraph.json / commplan.json as ``pipecraft plan``
    writes them; returns {file name: path}."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    S.dump_schedule(s, out / "schedule.json")
    _write_json(out / "taskgraph.json", tg.to_json())
    _write_json(out / "commplan.json", cp.to_json())
    return {n: out / n for n in ("schedule.json", "taskgraph.json", "commplan.json")}


def load_commplan(path) -> C.CommPlan:
    return C.CommPlan.from_json(json.loads(Path(path).read_text()))
