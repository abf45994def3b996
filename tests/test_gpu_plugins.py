"""Miss-handler and watchdog plug-ins with the reference's signatures
(miss.py:66-140, prefetch.py:163-221), restating the reference's own unit
tests (tests/test_miss.py, tests/test_prefetch.py:168-252). The miss
decision and every victim choice run on the device (esim_miss_decide,
esim_policy_apply); cache / channel here are minimal engine stand-ins."""
import pytest

pytestmark = pytest.mark.gpu

from paper_2602_03921_b200.eviction import AccessContext, LRUPolicy, LSPolicy
from paper_2602_03921_b200.miss import (DROP, DROPPED, FETCH, FETCH_LOW, FETCH_PRIORITY, FETCHED, SUBST,
                                        SUBSTITUTED, MissConfig, find_substitute, resolve_miss)
from paper_2602_03921_b200.models import ModelSpec
from paper_2602_03921_b200.prefetch import PrefetchQueue, PrefetchRequest, watchdog_step

TINY = ModelSpec("tiny", num_layers=2, experts_per_layer=4, top_k=1, expert_bytes_fp16=1_000_000)


class FetchRecorder:
    def __init__(self, plan=None, blocked=600):
        self.calls, self.plan, self.blocked = [], list(plan) if plan is not None else None, blocked

    def __call__(self, precision, final):
        self.calls.append((precision, final))
        return self.plan.pop(0) if self.plan is not None else self.blocked


def resolve(cfg, *, rank=1, gate=0.5, weight=0.5, layer_scores=(), residents=(), fetch=None):
    fetch = fetch if fetch is not None else FetchRecorder()
    return resolve_miss(cfg, TINY, "int4", rank, gate, weight, list(layer_scores), list(residents), fetch), fetch


def test_find_substitute_prefers_nearest_then_lower_index():
    residents = [(3, 0.30), (1, 0.52), (2, 0.48)]
    assert find_substitute(residents, 0.50, 0.05) == 1
    assert find_substitute(residents, 0.50, 0.2) == 1
    assert find_substitute(residents, 0.31, 0.05) == 3
    assert find_substitute(residents, 0.9, 0.05) is None
    assert find_substitute([], 0.5, 1.0) is None
    many = [(e, 0.5 + (e % 7) * 0.001) for e in range(100, 0, -1)]        # > one warp of residents
    assert find_substitute(many, 0.5, 0.01) == 7


def test_fetch_drop_subst_decisions():
    out, f = resolve(MissConfig(FETCH))
    assert (out.kind, out.precision, out.blocked_us, f.calls) == (FETCHED, "int4", 600, [("int4", True)])
    out, f = resolve(MissConfig(DROP, drop_rank_threshold=2), rank=3, weight=0.12)
    assert out.kind == DROPPED and out.weight_delta == pytest.approx(-0.12) and f.calls == []
    out, f = resolve(MissConfig(DROP, drop_rank_threshold=2), rank=2)
    assert out.kind == FETCHED and f.calls == [("int4", True)]
    out, f = resolve(MissConfig(SUBST, subst_tolerance=0.05), gate=0.50, weight=0.5, residents=[(2, 0.47), (0, 0.10)])
    assert (out.kind, out.substitute, f.calls) == (SUBSTITUTED, 2, []) and out.weight_delta == pytest.approx(-0.5)
    out, f = resolve(MissConfig(SUBST, subst_tolerance=0.01), gate=0.50, residents=[(2, 0.10)])
    assert (out.kind, out.precision, f.calls) == (FETCHED, "int4", [("int4", True)])
    out, f = resolve(MissConfig(FETCH_LOW))
    assert (out.precision, f.calls) == ("int2", [("int2", True)])


def test_fetch_priority_cascade():
    out, f = resolve(MissConfig(FETCH_PRIORITY), gate=0.4, layer_scores=[0.4, 0.3, 0.15, 0.1, 0.05],
                     fetch=FetchRecorder(plan=[None, None, None, 150]))
    assert (out.precision, out.blocked_us) == ("int2", 150)
    assert f.calls == [("fp16", False), ("int8", False), ("int4", False), ("int2", True)]
    out, f = resolve(MissConfig(FETCH_PRIORITY), gate=0.4, layer_scores=[0.4, 0.1], fetch=FetchRecorder(plan=[900]))
    assert out.precision == "fp16" and f.calls == [("fp16", False)]
    # p60 by nearest rank of these five is 0.15: a 0.1 gate starts one rung down, 0.15 does not
    out, f = resolve(MissConfig(FETCH_PRIORITY, degrade_percentile=60.0), gate=0.1,
                     layer_scores=[0.4, 0.3, 0.15, 0.1, 0.05], fetch=FetchRecorder(plan=[700]))
    assert out.precision == "int8" and f.calls[0] == ("int8", False)
    out, f = resolve(MissConfig(FETCH_PRIORITY, degrade_percentile=60.0), gate=0.15,
                     layer_scores=[0.4, 0.3, 0.15, 0.1, 0.05], fetch=FetchRecorder(plan=[700]))
    assert out.precision == "fp16"
    out, f = resolve(MissConfig(FETCH_PRIORITY), layer_scores=[], fetch=FetchRecorder(plan=[500]))
    assert out.precision == "fp16"
    flat = ModelSpec("flat", 2, 4, 1, 1_000_000, precisions=("fp16",))
    f = FetchRecorder(plan=[300])
    out = resolve_miss(MissConfig(FETCH_PRIORITY), flat, "fp16", 1, 0.1, 0.1, [0.9, 0.1], [], f)
    assert out.precision == "fp16" and f.calls == [("fp16", True)]
    with pytest.raises(RuntimeError, match="cascade"):
        resolve(MissConfig(FETCH_PRIORITY), layer_scores=[], fetch=FetchRecorder(plan=[None] * 4))


# ---- watchdog (prefetch.py:163-221) with engine stand-ins -------------------
class Cache:
    def __init__(self, capacity):
        self.capacity, self.resident, self.reserved = capacity, {}, 0

    @property
    def free_bytes(self):
        return self.capacity - sum(self.resident.values()) - self.reserved

    def admit(self, ident, precision, nbytes, score):
        self.resident[ident] = nbytes

    def evict(self, ident):
        del self.resident[ident]

    def reserve(self, nbytes):
        self.reserved += nbytes

    def is_resident(self, ident):
        return ident in self.resident


class Channel:
    def __init__(self):
        self.q = {}

    def append(self, ident, nbytes, kind, now, score, precision):
        self.q[ident] = (nbytes, kind, now, score, precision)

    def in_flight(self, ident):
        return self.q.get(ident)


class Callbacks:
    def __init__(self):
        self.started, self.skipped, self.dropped, self.evicted = [], [], [], []

    def on_start(self, req):
        self.started.append((req.target_layer, req.expert))

    def on_skip(self, req, reason):
        self.skipped.append(((req.target_layer, req.expert), reason))

    def on_drop(self, req, reason):
        self.dropped.append(((req.target_layer, req.expert), reason))

    def evict_fn(self, cache):
        def inner(victim, cause, forced):
            cache.evict(victim)
            self.evicted.append((victim, cause, forced))
        return inner


def run_watchdog(q, cache, policy, channel, cb):
    return watchdog_step(q, cache, policy, channel, 0, AccessContext(layer=0, pass_id=1), 10, "fp16",
                         cb.evict_fn(cache), cb.on_start, cb.on_skip, cb.on_drop)


def test_watchdog_skips_residents_and_in_flight():
    cache, policy, channel = Cache(30), LRUPolicy(), Channel()
    cache.admit((1, 0), "fp16", 10, 0.9)
    policy.note_admit((1, 0), AccessContext(0, 0))
    channel.append((1, 1), 10, "prefetch", 0, 0.5, "fp16")
    cache.reserve(10)
    q = PrefetchQueue()
    for e, s in ((0, 0.9), (1, 0.5), (2, 0.4)):
        q.submit(PrefetchRequest(1, e, s, 0))
    cb = Callbacks()
    assert run_watchdog(q, cache, policy, channel, cb) == 1
    assert cb.skipped == [((1, 0), "resident"), ((1, 1), "in_flight")] and cb.started == [(1, 2)]
    assert cache.free_bytes == 0 and channel.in_flight((1, 2)) is not None


def test_watchdog_marks_residents_before_making_space():
    cache, policy, channel = Cache(10), LSPolicy(), Channel()
    policy.begin_pass(0)
    cache.admit((1, 0), "fp16", 10, 0.9)
    policy.note_admit((1, 0), AccessContext(0, 0))
    policy.begin_pass(1)
    q = PrefetchQueue()
    q.submit(PrefetchRequest(1, 7, 0.8, 0))
    q.submit(PrefetchRequest(1, 0, 0.9, 0))
    cb = Callbacks()
    assert run_watchdog(q, cache, policy, channel, cb) == 0
    assert cache.is_resident((1, 0)) and cb.skipped == [((1, 0), "resident")]
    assert cb.dropped == [((1, 7), "no_space")] and cb.evicted == []
    assert policy.refusals == 1 and policy.unforced_current_evictions == 0


def test_watchdog_evicts_unforced_and_ls_keeps_current():
    cache, policy, channel = Cache(10), LRUPolicy(), Channel()
    cache.admit((1, 0), "fp16", 10, 0.9)
    policy.note_admit((1, 0), AccessContext(0, 0))
    q = PrefetchQueue()
    q.submit(PrefetchRequest(2, 3, 0.7, 0))
    cb = Callbacks()
    assert run_watchdog(q, cache, policy, channel, cb) == 1
    assert cb.evicted == [((1, 0), "prefetch", False)] and channel.in_flight((2, 3)) is not None
    cache, policy, channel = Cache(20), LSPolicy(), Channel()
    policy.begin_pass(0)
    for e in (0, 1):
        cache.admit((1, e), "fp16", 10, 0.5)
        policy.note_admit((1, e), AccessContext(0, 0))
    policy.begin_pass(1)
    policy.note_access((1, 1), AccessContext(1, 1))
    q = PrefetchQueue()
    q.submit(PrefetchRequest(2, 0, 0.9, 0))
    q.submit(PrefetchRequest(2, 1, 0.8, 0))
    cb = Callbacks()
    assert run_watchdog(q, cache, policy, channel, cb) == 1
    assert cb.evicted == [((1, 0), "prefetch", False)] and cb.dropped == [((2, 1), "no_space")]
    assert cache.is_resident((1, 1))
