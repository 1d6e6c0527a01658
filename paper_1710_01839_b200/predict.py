"""Block-algorithm time prediction (reference ``predict.py:1-104``), refit
for the GPU.

The reference times the leading ``2 * n_min`` rows of A against all of B
and scales by the row ratio (``predict.py:37-50,62-75``).  Those functions
keep their exact arithmetic here (``slice_rows_for``, ``predict_full_time``,
``choose_best``) because the tuner tables and the paper's Table 1 values
depend on it.

On a B200 a 2*n_min-row slice launches a few dozen CTAs against 148 SMs,
so time does not scale with rows: it scales with the per-SM load of CTAs
(SURVEY.md s7 hard part 4).  ``select_block_size`` therefore predicts on
the device with a load model built from the kernel's real tile and
occupancy (``mpmm_gemm_geometry``): two slices, each at least one full
complement of resident CTAs per SM (``gpu_slice_rows``), fix
``t = alpha + beta * load(rows)`` and the fit is evaluated at the full row
count (``fit_two_slices``).  When the slices would cover the whole
product the product itself is timed.
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
    slice2_rows: int = 0          # wave-aware mode: the second (smaller) slice
    slice2_time_s: float = 0.0
    extra_time_s: float = 0.0     # slices timed and then superseded by a refinement

    @property
    def phase_time_s(self):
        """Everything timed for this candidate (what the prediction cost)."""
        return self.slice_time_s + (self.slice2_time_s or 0.0) + self.extra_time_s

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
    """Per-SM load of a launch: the kernels are FP64-pipe bound, so an SM
    holding k CTAs of one product takes ~k times one CTA's pipe time, and
    the launch takes as long as its most loaded SM."""
    tile_m: int
    tile_n: int
    ctas_per_sm: int
    sm_count: int
    balanced: bool = False   # persistent largest-first kernel (TILE_LPT)

    @property
    def concurrent_ctas(self):
        return max(1, self.ctas_per_sm * self.sm_count)

    def ctas(self, rows, cols):
        return math.ceil(rows / self.tile_m) * math.ceil(cols / self.tile_n)

    def load(self, rows, cols):
        c = self.ctas(rows, cols)
        if self.balanced:
            return c / self.concurrent_ctas
        return math.ceil(c / self.sm_count) / self.ctas_per_sm

    def waves(self, rows, cols):
        return max(1, math.ceil(self.ctas(rows, cols) / self.concurrent_ctas))


def wave_model(comps, n_min):
    g = _cuda.gemm_geometry(comps, _cuda.ALGO_BLOCK, n_min)
    tile, _ = _cuda.tile_for_nmin(n_min)
    # only the DD tile set has a persistent largest-first kernel (the QD
    # configurations are all plain grids, csrc/gemm_qd.cu)
    return WaveModel(g["tile_m"], g["tile_n"], max(1, g["ctas_per_sm"]), g["sm_count"],
                     balanced=(tile == TILE_LPT and comps == 2))


TILE_LPT = 4   # csrc/kernels.h enum Tile


def gpu_slice_rows(model, n_min, m, n, slice_multiplier=DEFAULT_SLICE_MULTIPLIER):
    """Smallest row count >= the reference's slice that gives every SM a
    full complement of resident CTAs (rounded to the tile height), clamped
    to m."""
    rows = max(slice_rows_for(n_min, m, slice_multiplier), model.tile_m)
    tiles_n = math.ceil(n / model.tile_n)
    rows_per_wave = math.ceil(model.concurrent_ctas / tiles_n) * model.tile_m
    rows = max(rows, rows_per_wave)
    rows = math.ceil(rows / model.tile_m) * model.tile_m
    return min(rows, m)


def predict_full_time_waves(slice_time_s, model, slice_rows, m, n):
    """One-point extrapolation by per-SM load."""
    if slice_time_s <= 0.0:
        raise ValueError("slice time must be positive")
    return slice_time_s * model.load(m, n) / model.load(slice_rows, n)


def fit_two_slices(model, r1, t1, r2, t2, m, n):
    """t = alpha + beta * load(rows) through two slices; the launch and
    ramp costs (alpha) are what make one-point scaling miss on a GPU."""
    l1, l2, lf = model.load(r1, n), model.load(r2, n), model.load(m, n)
    if l2 <= l1 or t2 <= 0.0 or t1 <= 0.0:
        return predict_full_time_waves(t2 if t2 > 0 else t1, model, r2, m, n)
    beta = (t2 - t1) / (l2 - l1)
    if beta <= 0.0:
        return predict_full_time_waves(t2, model, r2, m, n)
    alpha = max(0.0, t1 - beta * l1)
    return alpha + beta * lf


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
                      slice_multiplier=DEFAULT_SLICE_MULTIPLIER, wave_aware=None, refine=True):
    """Predict the full-size time of each candidate; returns
    ``(best_n_min, records)`` (reference predict.py:83-104).

    ``wave_aware`` (default: on for the cuda backend) switches from the
    reference's row ratio to the wave model above; ``refine`` re-measures
    candidates predicted within 1 % of the best on a larger slice."""
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
            r1 = gpu_slice_rows(model, n_min, a.rows, b.cols, slice_multiplier)
            r2 = min(a.rows, math.ceil(2 * r1 / model.tile_m) * model.tile_m)
            if r2 >= a.rows:
                # the slice would be the whole product: measure it (exact)
                elapsed, rows = time_slice(a, b, n_min, threads, policy, slice_multiplier,
                                           a.rows)
                records.append(PredictionRecord(n_min, rows, a.rows, elapsed, elapsed))
                continue
            t1, _ = time_slice(a, b, n_min, threads, policy, slice_multiplier, r1)
            t2, _ = time_slice(a, b, n_min, threads, policy, slice_multiplier, r2)
            predicted = fit_two_slices(model, r1, t1, r2, t2, a.rows, b.cols)
            records.append(PredictionRecord(n_min, r2, a.rows, t2, predicted,
                                            slice2_rows=r1, slice2_time_s=t1))
        else:
            elapsed, rows = time_slice(a, b, n_min, threads, policy, slice_multiplier)
            records.append(PredictionRecord(n_min=n_min, slice_rows=rows, full_rows=a.rows,
                                            slice_time_s=elapsed,
                                            predicted_full_s=elapsed * (a.rows / rows)))
    if wave_aware and refine:
        records = _refine_close_candidates(a, b, records, threads, policy, slice_multiplier)
    return choose_best(records), records


def _refine_close_candidates(a, b, records, threads, policy, slice_multiplier,
                             within=0.01, growth=4):
    """A second look at candidates whose predictions are within ``within`` of
    the best: the two-slice fit extrapolates from ~1-3 waves of CTAs to
    hundreds and is good to a few tenths of a percent, which is also how far
    apart the best tile configurations are at large sizes.  Each close
    candidate gets one ``growth`` times larger slice (at most half the
    product), and the fit is redone through its two largest slices; the
    superseded slice's time stays charged (``extra_time_s``)."""
    best = min(r.predicted_full_s for r in records)
    close = [i for i, r in enumerate(records)
             if r.predicted_full_s <= best * (1.0 + within) and r.slice2_rows
             and r.slice_rows < a.rows]
    if len(close) < 2:
        return records
    out = list(records)
    for i in close:
        r = records[i]
        model = wave_model(a.prec.comps, r.n_min)
        r3 = min(a.rows // 2, growth * r.slice_rows)
        r3 = (r3 // model.tile_m) * model.tile_m
        if r3 <= r.slice_rows:
            continue
        t3, _ = time_slice(a, b, r.n_min, threads, policy, slice_multiplier, r3)
        predicted = fit_two_slices(model, r.slice_rows, r.slice_time_s, r3, t3, a.rows, b.cols)
        out[i] = PredictionRecord(r.n_min, r3, a.rows, t3, predicted,
                                  slice2_rows=r.slice_rows, slice2_time_s=r.slice_time_s,
                                  extra_time_s=r.extra_time_s + (r.slice2_time_s or 0.0))
    return out
