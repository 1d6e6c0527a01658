"""Block-algorithm time prediction (reference ``predict.py:1-104``), refit
for the GPU.

The reference times the leading ``2 * n_min`` rows of A against all of B
and scales by the row ratio (``predict.py:37-50,62-75``).  Those functions
keep their exact arithmetic here (``slice_rows_for``, ``predict_full_time``,
``choose_best``) because the tuner tables and the paper's Table 1 values
depend on it.

On a B200 a 2*n_min-row slice launches a few dozen CTAs against 148 SMs,
so time does not scale with rows: it scales with *waves* of CTAs
(SURVEY.md s7 hard part 4).  ``select_block_size`` therefore predicts on
the device with a wave model: the slice is grown to at least one full wave
of resident CTAs (``gpu_slice_rows``), and the full time is
``t_slice * waves(m) / waves(slice_rows)`` with
``waves(r) = ceil(ctas(r) / (SMs * ctas_per_SM))`` from the kernel's real
tile and occupancy (``mpmm_gemm_geometry``).
"""

import math
from dataclasses import dataclass

from . import _cuda, backend
from .matrix import DenseMatrix, leading_rows
from .multiply import _block_into
from .timing import TimingPolicy, measure, measure_events

DEFAULT_SLICE_MULTIPLIER = 2


@dataclass(frozen=True)
class PredictionRecord:
    """One block-size candidate: measured slice time and extrapolation."""
    n_min: int
    slice_rows: int
    full_rows: int
    slice_time_s: float
    predicted_full_s: float

    @property
    def scale_factor(self):
        return self.full_rows / self.slice_rows


def slice_rows_for(n_min, m, slice_multiplier=DEFAULT_SLICE_MULTIPLIER):
    """Rows of A in the reference's timed slice: min(k * n_min, m)."""
    if n_min < 1 or m < 1:
        raise ValueError("block size and row count must be positive")
    if slice_multiplier < 1:
        raise ValueError("slice multiplier must be positive")
    return min(slice_multiplier * n_min, m)


def predict_full_time(slice_time_s, m, n_min, slice_multiplier=DEFAULT_SLICE_MULTIPLIER):
    """Reference row-ratio extrapolation (predict.py:46-50)."""
    if slice_time_s <= 0.0:
        raise ValueError("slice time must be positive")
    return slice_time_s * (m / slice_rows_for(n_min, m, slice_multiplier))


# ---------------------------------------------------------------------------
# wave model
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class WaveModel:
    tile_m: int
    tile_n: int
    concurrent_ctas: int

    def ctas(self, rows, cols):
        return math.ceil(rows / self.tile_m) * math.ceil(cols / self.tile_n)

    def waves(self, rows, cols):
        return max(1, math.ceil(self.ctas(rows, cols) / self.concurrent_ctas))


def wave_model(comps, n_min):
    g = _cuda.gemm_geometry(comps, _cuda.ALGO_BLOCK, n_min)
    return WaveModel(g["tile_m"], g["tile_n"], max(1, g["ctas_per_sm"] * g["sm_count"]))


def gpu_slice_rows(model, n_min, m, n, slice_multiplier=DEFAULT_SLICE_MULTIPLIER):
    """Smallest row count >= the reference's slice that fills a whole wave
    (rounded to the tile height), clamped to m."""
    rows = max(slice_rows_for(n_min, m, slice_multiplier), model.tile_m)
    tiles_n = math.ceil(n / model.tile_n)
    rows_per_wave = math.ceil(model.concurrent_ctas / tiles_n) * model.tile_m
    rows = max(rows, rows_per_wave)
    rows = math.ceil(rows / model.tile_m) * model.tile_m
    return min(rows, m)


def predict_full_time_waves(slice_time_s, model, slice_rows, m, n):
    if slice_time_s <= 0.0:
        raise ValueError("slice time must be positive")
    return slice_time_s * model.waves(m, n) / model.waves(slice_rows, n)


# ---------------------------------------------------------------------------
# timing and selection
# ---------------------------------------------------------------------------

def _zero(mat):
    if mat.is_device:
        mat.data.zero_()
    else:
        mat.data.fill(0.0)


def time_slice(a, b, n_min, threads=1, policy=None,
               slice_multiplier=DEFAULT_SLICE_MULTIPLIER, rows=None):
    """Seconds for the leading-rows slice of ``a`` times all of ``b``
    (reference predict.py:62-75).  ``rows`` overrides the slice height.
    On the device the sample is a CUDA-event interval."""
    policy = policy or TimingPolicy()
    if rows is None:
        rows = slice_rows_for(n_min, a.rows, slice_multiplier)
    on_dev = backend.is_cuda()
    if on_dev:
        a, b = a.to_device(), b.to_device(a.device if a.is_device else None)
    a_slice = leading_rows(a, rows)
    out = DenseMatrix.zeros(rows, b.cols, a.prec, a.device if on_dev else None)
    run = lambda: _block_into(a_slice, b, out, n_min, threads)  # noqa: E731
    if on_dev and policy.clock is TimingPolicy().clock:
        elapsed = measure_events(run, policy, setup=lambda: _zero(out))
    else:
        elapsed = measure(run, policy, setup=lambda: _zero(out))
    return elapsed, rows


def choose_best(records):
    """Smallest predicted time; ties go to the smaller block size."""
    return min(records, key=lambda r: (r.predicted_full_s, r.n_min)).n_min


def select_block_size(a, b, candidates, threads=1, policy=None,
                      slice_multiplier=DEFAULT_SLICE_MULTIPLIER, wave_aware=None):
    """Predict the full-size time of each candidate; returns
    ``(best_n_min, records)`` (reference predict.py:83-104).

    ``wave_aware`` (default: on for the cuda backend) switches from the
    reference's row ratio to the wave model above."""
    if not candidates:
        raise ValueError("need at least one block-size candidate")
    if list(candidates) != sorted(candidates):
        raise ValueError("candidates must be sorted ascending")
    if wave_aware is None:
        wave_aware = backend.is_cuda()
    records = []
    for n_min in candidates:
        if wave_aware:
            model = wave_model(a.prec.comps, n_min)
            rows = gpu_slice_rows(model, n_min, a.rows, b.cols, slice_multiplier)
            elapsed, rows = time_slice(a, b, n_min, threads, policy, slice_multiplier, rows)
            predicted = predict_full_time_waves(elapsed, model, rows, a.rows, b.cols)
        else:
            elapsed, rows = time_slice(a, b, n_min, threads, policy, slice_multiplier)
            predicted = elapsed * (a.rows / rows)
        records.append(PredictionRecord(n_min=n_min, slice_rows=rows, full_rows=a.rows,
                                        slice_time_s=elapsed, predicted_full_s=predicted))
    return choose_best(records), records
