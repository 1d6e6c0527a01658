"""Measurement policy (reference ``timing.py:1-59``) for device work.

``TimingPolicy`` and ``measure`` keep the reference's contract: warm-up
runs, ``measured_runs`` samples aggregated by median/min/mean, an injectable
clock, ``setup`` outside the timed region, and ``MeasurementError`` on a
non-positive elapsed time.

The difference is the default clock.  Device work is asynchronous, so the
default ``device_clock`` synchronises the current CUDA device before
reading the host's monotonic clock; ``measure`` then brackets exactly the
device work ``fn`` enqueued.  ``EventTimer`` gives the CUDA-event timings
(on the launching stream) used by the predictor and by ``bench.py``.
"""

import statistics
import time
from dataclasses import dataclass, field

from .errors import MeasurementError

def _reduce(samples, how):
    if how == "median":
        return statistics.median(samples)
    return min(samples) if how == "min" else statistics.fmean(samples)


_AGGREGATORS = ("median", "min", "mean")


def device_clock():
    """Monotonic seconds after all queued work on the current device."""
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize()
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    return time.perf_counter()


@dataclass
class TimingPolicy:
    """The reference's fields and defaults (timing.py:22-35); only the
    default clock differs (device_clock)."""
    warmup_runs: int = 0
    measured_runs: int = 1
    aggregator: str = "median"
    clock: object = field(default=device_clock, repr=False)

    def __post_init__(self):
        problems = {
            "measured_runs must be >= 1": self.measured_runs < 1,
            "warmup_runs must be >= 0": self.warmup_runs < 0,
            f"unknown aggregator {self.aggregator!r}": self.aggregator not in _AGGREGATORS,
        }
        for message, wrong in problems.items():
            if wrong:
                raise ValueError(message)


def _collect(fn, policy, setup, interval):
    """Warm-up runs, then ``measured_runs`` samples of ``interval(fn)`` --
    one timed call each, ``setup`` before every call and never timed --
    aggregated as the policy says."""
    def one(timed):
        if setup is not None:
            setup()
        if not timed:
            fn()
            return None
        elapsed = interval(fn)
        if elapsed <= 0.0:
            raise MeasurementError(f"non-positive elapsed time {elapsed!r}")
        return elapsed

    for _ in range(policy.warmup_runs):
        one(False)
    return _reduce([one(True) for _ in range(policy.measured_runs)], policy.aggregator)


def measure(fn, policy, setup=None):
    """Elapsed seconds for ``fn()`` under ``policy`` by the policy's clock
    (reference timing.py:38-59); ``setup`` runs before every sample, untimed."""
    clock = policy.clock

    def interval(f):
        t0 = clock()
        f()
        return clock() - t0
    return _collect(fn, policy, setup, interval)


class EventTimer:
    """CUDA-event timing on a given stream (default: the current stream).

    ``with EventTimer() as t: enqueue(...)`` then ``t.seconds`` (syncs).
    """

    def __init__(self, stream=None):
        import torch
        self._torch = torch
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.start = torch.cuda.Event(enable_timing=True)
        self.end = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.start.record(self.stream)
        return self

    def __exit__(self, *exc):
        self.end.record(self.stream)
        return False

    @property
    def seconds(self):
        self.end.synchronize()
        return self.start.elapsed_time(self.end) / 1e3


def measure_events(fn, policy, setup=None, stream=None):
    """Like :func:`measure` but each sample is a CUDA-event interval on
    ``stream`` around the device work ``fn`` enqueues."""
    def interval(f):
        with EventTimer(stream) as t:
            f()
        return t.seconds
    return _collect(fn, policy, setup, interval)
