"""Batched configuration search on the GPU engine.

``run_search`` follows ``dltsim.search.run_search`` (``pkg/src/dltsim/search.py:381-444``)
decision for decision -- strategies (``:235-310``), the four pruning tactics in
their fixed order (``:118-176``), the early-stop rule (``:213-232``), trial
records (``:360-378``) and the ranking (``:349-357``) -- so for the same
arguments and evaluator results it returns the same trial sequence, the same
inferred records and the same ranking (``tests/test_search.py`` against the
reference's own runs).

What changes is how trials are evaluated.  The evaluator is pure, so the
runner evaluates speculatively, in bulk, on the device: for the grid and random
strategies the whole ordered candidate list is one engine batch before the
decision loop starts; for the evolutionary strategy every population is one
batch.  Trials the tactics prune, or that early stopping never reaches, cost
only device work, never a different answer.  Any evaluator works; one with
``evaluate_many`` (``api.GpuPipelineEvaluator``) gets the bulk path.
"""

from __future__ import annotations

import enum
import random
from dataclasses import dataclass, replace
from typing import Callable, Iterable, Sequence

from . import workload as W


class TrialStatus(enum.Enum):
    COMPLETED = "completed"
    OOM = "oom"
    SKIPPED_PRUNED = "skipped_pruned"
    INVALID = "invalid"


@dataclass
class TrialRecord:
    config: object
    status: TrialStatus
    time_ns: int | None = None
    mfu: float | None = None
    peak_mem_bytes: int | None = None
    provenance: str = "simulated"          # "simulated" | "inferred"
    tactic: str | None = None
    premise: object | None = None          # config of the trial the verdict rests on
    error: str | None = None

    @property
    def is_oom(self) -> bool:
        return self.status is TrialStatus.OOM or (
            self.status is TrialStatus.SKIPPED_PRUNED and self.time_ns is None)

    @property
    def has_runtime(self) -> bool:
        return self.time_ns is not None


@dataclass
class SearchResult:
    trials: list
    ranked: list
    stopped_early: bool

    @property
    def best(self):
        return self.ranked[0] if self.ranked else None


@dataclass(frozen=True)
class StopRule:
    window: int = 20
    top_k: int = 5


# --- tactics (search.py:118-176): first verdict in fixed order wins ----------------

def _differs_only_in(cand, other, knob: str) -> bool:
    return replace(cand, **{knob: getattr(other, knob)}) == other


def _oom_when_flag_off(flag: str, name: str):
    """A config that ran out of memory WITH ``flag`` on implies OOM with it off."""
    def verdict(history, cand):
        if getattr(cand, flag):
            return None
        for rec in history:
            if rec.is_oom and getattr(rec.config, flag) and _differs_only_in(cand, rec.config, flag):
                return ("mark_oom", name, rec)
        return None
    return verdict


def _dist_optimizer_keeps_runtime(history, cand):
    if not cand.dist_optimizer:
        return None
    for rec in history:
        if (rec.has_runtime and not rec.config.dist_optimizer
                and _differs_only_in(cand, rec.config, "dist_optimizer")):
            return ("copy_runtime", "dist-optimizer-runtime", rec)
    return None


def _more_microbatches_keep_runtime(history, cand):
    if cand.pp != 1:
        return None
    premise = None
    for rec in history:
        if (rec.has_runtime and rec.config.pp == 1 and rec.config.micro_mult < cand.micro_mult
                and _differs_only_in(cand, rec.config, "micro_mult")
                and (premise is None or rec.config.micro_mult < premise.config.micro_mult)):
            premise = rec
    return None if premise is None else ("copy_runtime", "more-microbatches-runtime", premise)


TACTICS = (
    _oom_when_flag_off("act_recompute", "oom-without-recompute"),
    _oom_when_flag_off("seq_parallel", "oom-without-seq-parallel"),
    _dist_optimizer_keeps_runtime,
    _more_microbatches_keep_runtime,
)


def apply_tactics(history, cand):
    for tactic in TACTICS:
        v = tactic(history, cand)
        if v is not None:
            return v
    return None


def _inferred(config, verdict) -> TrialRecord:
    kind, tactic, premise = verdict
    if kind == "mark_oom":
        return TrialRecord(config, TrialStatus.SKIPPED_PRUNED, provenance="inferred",
                           tactic=tactic, premise=premise.config)
    return TrialRecord(config, TrialStatus.SKIPPED_PRUNED, time_ns=premise.time_ns,
                       mfu=premise.mfu, provenance="inferred", tactic=tactic,
                       premise=premise.config)


def _simulated(config, outcome) -> TrialRecord:
    """An evaluator result (or the exception it raised) as a trial (search.py:368-378)."""
    if isinstance(outcome, BaseException):
        return TrialRecord(config, TrialStatus.INVALID, error=str(outcome))
    if outcome.oom:
        return TrialRecord(config, TrialStatus.OOM, peak_mem_bytes=outcome.peak_mem_bytes)
    return TrialRecord(config, TrialStatus.COMPLETED, time_ns=outcome.time_ns, mfu=outcome.mfu,
                       peak_mem_bytes=outcome.peak_mem_bytes)


# --- early stop (search.py:213-232) -------------------------------------------------

def early_stop(history, window: int = 20, top_k: int = 5) -> bool:
    """True once the top-k set by MFU has not changed over the last ``window``
    trials that have a runtime."""
    scored = [r for r in history if r.has_runtime]
    if len(scored) < window:
        return False

    def top(prefix):
        return frozenset(r.config.key() for r in
                         sorted(prefix, key=lambda r: (-(r.mfu or 0.0), r.config.key()))[:top_k])
    now = top(scored)
    return all(top(scored[:len(scored) - i]) == now for i in range(1, window))


def rank(trials) -> list:
    """search.py:349-357: by MFU descending, then OOM / pruned-OOM, then INVALID."""
    def order(r):
        if r.has_runtime:
            return (0, -(r.mfu or 0.0), r.time_ns, r.config.key())
        return (2 if r.status is TrialStatus.INVALID else 1, 0.0, 0, r.config.key())
    return sorted(trials, key=order)


# --- strategies (search.py:235-310) -----------------------------------------------------

@dataclass
class GridStrategy:
    name = "grid"

    def order(self, configs):
        return list(configs)


@dataclass
class RandomStrategy:
    seed: int = 0
    name = "random"

    def order(self, configs):
        out = list(configs)
        random.Random(self.seed).shuffle(out)
        return out


@dataclass
class EvolutionaryStrategy:
    """(mu, lambda) evolution over the lattice: children move one knob of a
    parent to a neighbouring value; only unseen points are proposed."""

    seed: int = 0
    mu: int = 4
    lam: int = 12
    name = "evolutionary"

    KNOBS = ("tp", "pp", "micro_mult", "virtual_stages", "act_recompute", "seq_parallel",
             "dist_optimizer")

    def populations(self, configs, space, score_of):
        rng = random.Random(self.seed)
        lattice = {c.key(): c for c in configs}
        pending = list(configs)

        def child_of(parent):
            knob = rng.choice(self.KNOBS)
            values = getattr(space, knob)
            i = values.index(getattr(parent, knob)) + rng.choice((-1, 1))
            c = replace(parent, **{knob: values[min(max(i, 0), len(values) - 1)]})
            return c if c.key() in lattice else None

        yield self._take(pending, self.lam)
        while pending:
            scored = sorted(((score_of(lattice[k]), k) for k in lattice
                             if score_of(lattice[k]) is not None), key=lambda x: (-x[0], x[1]))
            parents = [lattice[k] for _, k in scored[:self.mu]]
            pop, tries = [], 0
            while len(pop) < self.lam and tries < 20 * self.lam and pending:
                tries += 1
                c = child_of(rng.choice(parents)) if parents else None
                if c is not None and c in pending and c not in pop:
                    pop.append(c)
            for c in pop:
                pending.remove(c)
            while len(pop) < self.lam and pending:
                pop.append(pending.pop(rng.randrange(len(pending))))
            yield pop

    @staticmethod
    def _take(pending, n):
        head = pending[:n]
        del pending[:n]
        return head


def make_strategy(name: str, seed: int = 0):
    try:
        return {"grid": lambda: GridStrategy(), "random": lambda: RandomStrategy(seed),
                "evolutionary": lambda: EvolutionaryStrategy(seed)}[name]()
    except KeyError:
        raise ValueError(f"unknown strategy {name!r}") from None


# --- the runner ------------------------------------------------------------------------------

class _Outcomes:
    """Memo of evaluator outcomes, filled in bulk where the evaluator allows."""

    def __init__(self, evaluator):
        self.evaluator = evaluator
        self.memo: dict = {}

    def prepare(self, configs) -> None:
        todo = [c for c in configs if c.key() not in self.memo]
        if todo and hasattr(self.evaluator, "evaluate_many"):
            for c, r in zip(todo, self.evaluator.evaluate_many(todo)):
                self.memo[c.key()] = r

    def __call__(self, config):
        k = config.key()
        if k not in self.memo:
            try:
                self.memo[k] = self.evaluator(config)
            except Exception as exc:  # noqa: BLE001 - becomes an INVALID trial (search.py:370-374)
                self.memo[k] = exc
        return self.memo[k]


def _strategy_kind(strategy) -> str:
    return getattr(strategy, "name", type(strategy).__name__)


class BulkEvaluator:
    """Evaluator wrapper for the reference's own ``run_search``: the first call
    evaluates the whole enumerated space as ONE engine batch (speculatively --
    the evaluator is pure, so pruned or never-reached configs only cost device
    work), later calls are served from the memo.  Failures are re-raised per
    config, so the reference records them as INVALID with their text
    (search.py:370-374)."""

    def __init__(self, evaluator, configs):
        self.outcomes = _Outcomes(evaluator)
        self.configs = list(configs)
        self.primed = False

    def __call__(self, config):
        if not self.primed:
            self.outcomes.prepare(self.configs)
            self.primed = True
        r = self.outcomes(config)
        if isinstance(r, Exception):
            raise r
        return r


def _reference_search(strategy, stop):
    """dltsim.search when the caller uses the reference's own strategy (and stop
    rule) objects, else None."""
    if not type(strategy).__module__.startswith("dltsim"):
        return None
    if stop is not None and not type(stop).__module__.startswith("dltsim"):
        return None
    try:
        import importlib
        return importlib.import_module("dltsim.search")
    except Exception:
        return None


def run_search(space, evaluator, strategy, model, cluster, jobs: int = 1,
               use_tactics: bool = True, stop: StopRule | None = None,
               max_trials: int | None = None, deterministic: bool = False) -> SearchResult:
    """dltsim.search.run_search with bulk speculative evaluation (module docstring).

    With the reference's own strategy objects (and ``jobs == 1``) this IS the
    reference's runner -- its strategies, tactics, early stop and ranking --
    fed by a ``BulkEvaluator`` (one engine batch for the whole space).  Without
    the reference importable, the restatement below follows it decision for
    decision (``tests/test_search.py``).  ``jobs`` only sets the batch size, as
    in the reference (each batch's tactic verdicts are taken against the
    history before its results); evaluation itself is the engine's, not a
    process pool's."""
    configs = W.enumerate_space(space, model, cluster)
    ref = _reference_search(strategy, stop) if jobs == 1 else None
    if ref is not None:
        return ref.run_search(space, BulkEvaluator(evaluator, configs), strategy, model, cluster,
                              jobs=1, use_tactics=use_tactics, stop=stop, max_trials=max_trials,
                              deterministic=deterministic)
    outcomes = _Outcomes(evaluator)
    history: list = []
    state = {"stopped": False}

    def record(rec) -> bool:
        history.append(rec)
        if stop is not None and early_stop(history, stop.window, stop.top_k):
            return True
        return bool(max_trials and len(history) >= max_trials)

    def batches() -> Iterable[list]:
        if _strategy_kind(strategy) == "evolutionary":
            scores: dict = {}
            gen = (strategy.populations(configs, space, lambda c: scores.get(c.key()))
                   if hasattr(strategy, "populations")
                   else strategy.ordered_run(configs, space, lambda c: scores.get(c.key())))
            for pop in gen:
                outcomes.prepare(pop)           # one engine batch per population
                yield pop
                for r in history:
                    if r.has_runtime and r.mfu is not None:
                        scores[r.config.key()] = r.mfu
        else:
            ordered = list(strategy.order(configs))
            outcomes.prepare(ordered)           # the whole candidate list, one engine batch
            size = 1 if jobs == 1 else jobs
            for i in range(0, len(ordered), size):
                yield ordered[i:i + size]

    for batch in batches():
        if state["stopped"]:
            break
        to_run = []
        for config in batch:
            verdict = apply_tactics(history, config) if use_tactics else None
            if verdict is None:
                to_run.append(config)
            elif record(_inferred(config, verdict)):
                state["stopped"] = True
                break
        if state["stopped"]:
            break
        for config in to_run:
            if record(_simulated(config, outcomes(config))):
                state["stopped"] = True
                if jobs == 1:
                    break
    return SearchResult(trials=history, ranked=rank(history), stopped_early=state["stopped"])


# --- CMA-ES populations (Maya-Search's optimiser; the reference ships only the
# --- (mu, lambda)-ES above, search.py:262-310) ----------------------------------------------

@dataclass
class Generation:
    index: int
    configs: list            # the population's distinct lattice points, in sample order
    mfu: list                # per config: MFU, or None (OOM / invalid / failed)
    best: object             # best config so far
    best_mfu: float | None


def cma_search(space, evaluator, model, cluster, popsize: int = 64, generations: int = 12,
               seed: int = 0, sigma0: float = 0.3) -> list:
    """CMA-ES over the knob lattice, one engine batch per population.

    Each knob is a continuous coordinate in [0, 1] mapped to its candidate
    list by rounding; the standard (mu/mu_w, lambda) CMA-ES update (Hansen's
    default weights and learning rates) adapts mean, step size and covariance
    from the MFU ranking of each population.  Points the lattice rejects
    (validate_config), OOM or failed evaluations rank last.  The whole
    population is evaluated with ``evaluator.evaluate_many`` (one GPU batch)
    when available.  Deterministic for a seed; returns one Generation per step.
    """
    import numpy as np

    knobs = EvolutionaryStrategy.KNOBS
    sizes = [len(getattr(space, k)) for k in knobs]
    n = len(knobs)
    rng = np.random.default_rng(seed)
    lam = max(4, int(popsize))
    mu = lam // 2
    w = np.log(mu + 0.5) - np.log(np.arange(1, mu + 1))
    w /= w.sum()
    mueff = 1.0 / np.sum(w ** 2)
    cc = (4 + mueff / n) / (n + 4 + 2 * mueff / n)
    cs = (mueff + 2) / (n + mueff + 5)
    c1 = 2 / ((n + 1.3) ** 2 + mueff)
    cmu = min(1 - c1, 2 * (mueff - 2 + 1 / mueff) / ((n + 2) ** 2 + mueff))
    damps = 1 + 2 * max(0.0, np.sqrt((mueff - 1) / (n + 1)) - 1) + cs
    chin = np.sqrt(n) * (1 - 1 / (4 * n) + 1 / (21 * n * n))
    mean = np.full(n, 0.5)
    sigma = float(sigma0)
    C = np.eye(n)
    pc = np.zeros(n)
    ps = np.zeros(n)
    valid = {c.key(): c for c in W.enumerate_space(space, model, cluster)}
    seen: dict = {}
    best, best_mfu = None, None
    out = []

    def to_config(x):
        vals = []
        for k, s, xi in zip(knobs, sizes, np.clip(x, 0.0, 1.0)):
            vals.append(getattr(space, k)[int(round(xi * (s - 1)))])
        cfg = W.ConfigPoint(*vals, global_batch=space.global_batch)
        return valid.get(cfg.key())

    for g in range(generations):
        eigval, B = np.linalg.eigh(C)
        D = np.sqrt(np.maximum(eigval, 1e-20))
        z = rng.standard_normal((lam, n))
        y = z @ (B * D).T
        xs = mean + sigma * y
        cfgs = [to_config(x) for x in xs]
        todo = []
        for c in cfgs:
            if c is not None and c.key() not in seen and c not in todo:
                todo.append(c)
        if todo:
            if hasattr(evaluator, "evaluate_many"):
                res = evaluator.evaluate_many(todo)
            else:
                res = []
                for c in todo:
                    try:
                        res.append(evaluator(c))
                    except Exception as exc:  # noqa: BLE001 - ranks last
                        res.append(exc)
            for c, r in zip(todo, res):
                seen[c.key()] = (None if isinstance(r, BaseException) or r.oom else r.mfu)
        fit = np.array([-(seen.get(c.key()) or -1.0) if c is not None else 2.0 for c in cfgs])
        order = np.argsort(fit, kind="stable")
        for c in cfgs:
            m = seen.get(c.key()) if c is not None else None
            if m is not None and (best_mfu is None or m > best_mfu
                                  or (m == best_mfu and c.key() < best.key())):
                best, best_mfu = c, m
        distinct = []
        for c in cfgs:
            if c is not None and c not in distinct:
                distinct.append(c)
        out.append(Generation(g, distinct, [seen.get(c.key()) for c in distinct], best, best_mfu))
        # CMA-ES update
        ysel = y[order[:mu]]
        yw = w @ ysel
        mean = mean + sigma * yw
        invsqrtC = B @ np.diag(1 / D) @ B.T
        ps = (1 - cs) * ps + np.sqrt(cs * (2 - cs) * mueff) * (invsqrtC @ yw)
        hsig = (np.linalg.norm(ps) / np.sqrt(1 - (1 - cs) ** (2 * (g + 1))) / chin
                < 1.4 + 2 / (n + 1))
        pc = (1 - cc) * pc + hsig * np.sqrt(cc * (2 - cc) * mueff) * yw
        C = ((1 - c1 - cmu) * C + c1 * (np.outer(pc, pc) + (1 - hsig) * cc * (2 - cc) * C)
             + cmu * (ysel.T * w) @ ysel)
        sigma *= float(np.exp((cs / damps) * (np.linalg.norm(ps) / chin - 1)))
    return out
