"""TSTK1 pixel stacks and the batched ``tomobpdn solve`` driver.

Mirrors the reference's stack format (``stack.py:30-82``: one JSON header line, then
little-endian float32 (re, im) pairs, pixel-major) and its solve command (``cli.py:112-174``):
dictionary from the embedded geometry and the grid, per-pixel seed
derive_seed(substream(seed, pixel_id)) (``cli.py:102``), default lambda 0.05 max|A^H b|
(``slimmer.py:215-222``), SL1MMER pipeline per pixel, records in input order as JSONL
(``slimmer.py:225-242``) and an optional point-cloud CSV (``slimmer.py:245-271``), plus a
sidecar manifest (``stack.py:97-126``).  The per-pixel process pool (``cli.py:133-144``) is
replaced by one batched device call.  Host code here is I/O and formatting only; every
dictionary element, solve and selection runs on the GPU.
"""

from __future__ import annotations

import csv
import datetime
import hashlib
import json

import numpy as np

from .exceptions import GeometryError, GridError, StackFormatError
from .grid import MOTION_BASES, ParameterGrid, build_steering_matrix

MAGIC = "TSTK1"  # stack.py:26
BYTES_PER_SAMPLE = 8
_GEOMETRY_KEYS = {"baselines_m", "times_yr", "wavelength_m", "range_m"}  # model.py:35


class Geometry:
    """The fields of AcquisitionGeometry (model.py:38-125) the dictionary needs."""

    def __init__(self, baselines, times, wavelength, slant_range):
        self.baselines = np.asarray(baselines, dtype=float)
        self.times = np.asarray(times, dtype=float)
        self.wavelength = float(wavelength)
        self.slant_range = float(slant_range)
        b, t = self.baselines, self.times
        if b.ndim != 1 or t.ndim != 1 or b.size != t.size:
            raise GeometryError("baselines and times must be 1-d with equal length")
        if b.size < 2:
            raise GeometryError("need at least 2 acquisitions")
        if not (np.all(np.isfinite(b)) and np.all(np.isfinite(t))):
            raise GeometryError("baselines/times must be finite")
        if not (np.isfinite(self.wavelength) and self.wavelength > 0):
            raise GeometryError(f"wavelength must be > 0, got {self.wavelength}")
        if not (np.isfinite(self.slant_range) and self.slant_range > 0):
            raise GeometryError(f"slant range must be > 0, got {self.slant_range}")
        if float(np.max(b) - np.min(b)) <= 0:
            raise GeometryError("aperture extent max(b) - min(b) must be > 0")

    @property
    def n_acquisitions(self) -> int:
        return int(self.baselines.size)

    def to_dict(self) -> dict:
        return {"baselines_m": self.baselines.tolist(), "times_yr": self.times.tolist(), "wavelength_m": self.wavelength, "range_m": self.slant_range}

    @classmethod
    def from_dict(cls, data: dict) -> "Geometry":
        if not isinstance(data, dict):
            raise GeometryError("geometry must be a JSON object")
        unknown = set(data) - _GEOMETRY_KEYS
        if unknown:
            raise GeometryError(f"unknown geometry keys: {sorted(unknown)}")
        missing = _GEOMETRY_KEYS - set(data)
        if missing:
            raise GeometryError(f"missing geometry keys: {sorted(missing)}")
        return cls(data["baselines_m"], data["times_yr"], data["wavelength_m"], data["range_m"])

    def spatial_frequencies(self) -> np.ndarray:
        """xi_n = 2 b_n / (lambda r) (model.py:254-259)."""
        return 2.0 * self.baselines / (self.wavelength * self.slant_range)

    def temporal_frequencies(self, bases) -> np.ndarray:
        """eta_{m,n} = 2 tau_m(t_n) / lambda (model.py:262-277)."""
        fns = {"linear": lambda t: t, "seasonal": lambda t: np.sin(2.0 * np.pi * t)}
        rows = [2.0 * fns[b](self.times) / self.wavelength for b in bases]
        return np.vstack(rows) if rows else np.zeros((0, self.n_acquisitions))


def write_stack(path, geometry: Geometry, pixels) -> None:
    """TSTK1 writer (stack.py:30-52)."""
    pixels = np.asarray(pixels)
    if pixels.ndim != 2:
        raise StackFormatError("pixels must be a 2-d array (pixel_count x N)")
    if pixels.shape[1] != geometry.n_acquisitions:
        raise StackFormatError(f"pixels have {pixels.shape[1]} samples but geometry has {geometry.n_acquisitions} acquisitions")
    header = {"magic": MAGIC, "n": int(pixels.shape[1]), "pixel_count": int(pixels.shape[0]), "geometry": geometry.to_dict()}
    inter = np.empty((pixels.shape[0], pixels.shape[1], 2), dtype="<f4")
    inter[..., 0] = pixels.real
    inter[..., 1] = pixels.imag
    with open(path, "wb") as fh:
        fh.write(json.dumps(header, separators=(",", ":")).encode("utf-8"))
        fh.write(b"\n")
        fh.write(inter.tobytes())


def read_stack(path):
    """TSTK1 reader with the reference's validation (stack.py:55-82); complex64 [P, n]."""
    with open(path, "rb") as fh:
        header_line = fh.readline()
        payload = fh.read()
    try:
        header = json.loads(header_line.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise StackFormatError(f"unreadable stack header: {exc}") from exc
    if not isinstance(header, dict) or header.get("magic") != MAGIC:
        raise StackFormatError(f"bad magic; expected {MAGIC!r}")
    missing = {"n", "pixel_count", "geometry"} - set(header)
    if missing:
        raise StackFormatError(f"stack header missing keys: {sorted(missing)}")
    n, count = int(header["n"]), int(header["pixel_count"])
    if len(payload) != count * n * BYTES_PER_SAMPLE:
        raise StackFormatError(f"payload has {len(payload)} bytes, expected {count * n * BYTES_PER_SAMPLE} ({count} pixels x {n} samples)")
    geometry = Geometry.from_dict(header["geometry"])
    if geometry.n_acquisitions != n:
        raise StackFormatError("header n disagrees with embedded geometry length")
    floats = np.frombuffer(payload, dtype="<f4").reshape(count, n, 2)
    return geometry, (floats[..., 0] + 1j * floats[..., 1]).astype(np.complex64)


def grid_from_dict(data: dict) -> ParameterGrid:
    """Strict grid JSON (model.py:350-371)."""
    if not isinstance(data, dict):
        raise GridError("grid config must be a JSON object")
    unknown = set(data) - {"elevation", "motion"}
    if unknown:
        raise GridError(f"unknown grid keys: {sorted(unknown)}")
    if "elevation" not in data:
        raise GridError("grid config requires an 'elevation' axis")
    elev = data["elevation"]
    if set(elev) != {"min", "max", "count"}:
        raise GridError("elevation axis requires exactly keys ['count', 'max', 'min']")
    motion = []
    for axis in data.get("motion", []):
        if set(axis) != {"base", "min", "max", "count"}:
            raise GridError("motion axis requires exactly keys ['base', 'count', 'max', 'min']")
        if axis["base"] not in MOTION_BASES:
            raise GridError(f"unknown base function {axis['base']!r}")
        motion.append((axis["base"], float(axis["min"]), float(axis["max"]), int(axis["count"])))
    return ParameterGrid.uniform((float(elev["min"]), float(elev["max"])), int(elev["count"]), tuple(motion))


def _sha256(path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def solve_stack(stack_path, grid_dict: dict, pipe_config, seed: int | None = None, out_jsonl=None, out_csv=None, beta: float = 0.05,
                group=None):
    """Batched equivalent of ``tomobpdn solve`` (cli.py:112-174); returns the ordered records.

    Under ``torch.distributed`` (one process per GPU, e.g. torchrun) the stack's pixels are sharded
    in contiguous ranges over the ranks (no collective on the data path; seeds from the global pixel
    id, cli.py:102), the records are all-gathered in pixel order and rank 0 writes the outputs, so
    the JSONL/CSV bytes are identical for any number of GPUs (test_acceptance.py:266-312).
    """
    from . import __version__
    from .sharded import _dist, pixel_shard
    from .slimmer import estimates_to_record, pipeline_batch
    from .solver import Dictionary

    geometry, pixels = read_stack(stack_path)
    grid = grid_from_dict(grid_dict)
    seed = pipe_config.solver.seed if seed is None else seed
    a = build_steering_matrix(geometry.spatial_frequencies(), grid, eta=geometry.temporal_frequencies(grid.motion_bases), sign=1.0)
    d = Dictionary(a)
    dist = _dist()
    world = dist.get_world_size(group) if dist is not None else 1
    rank = dist.get_rank(group) if dist is not None else 0
    start, stop = pixel_shard(pixels.shape[0], world, rank)
    records = []
    if stop > start:
        est = pipeline_batch(d, pixels[start:stop], grid, pipe_config, beta=beta, run_seed=seed, first_pixel_id=start)
        for i in range(stop - start):
            try:
                records.append(estimates_to_record(start + i, est.estimates(i)))
            except Exception as exc:  # per-pixel error record (cli.py:104-108)
                records.append({"pixel_id": start + i, "error": str(exc)})
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, records, group=group)
        records = [r for part in parts for r in part]
    if out_jsonl is not None and rank == 0:
        with open(out_jsonl, "w", encoding="utf-8", newline="\n") as fh:
            for r in records:
                fh.write(json.dumps(r, separators=(",", ":")))
                fh.write("\n")
        if out_csv is not None:
            with open(out_csv, "w", encoding="utf-8", newline="") as fh:
                w = csv.writer(fh, lineterminator="\n")
                w.writerow(["pixel_id", "k", "elevation_m", "p1", "p2", "amp_re", "amp_im"])
                for r in records:
                    if "error" in r:
                        continue
                    for k in range(r["model_order"]):
                        p = (list(r["motion_params"][k]) + [0.0, 0.0])[:2]
                        amp = r["amplitudes"][k]
                        w.writerow([r["pixel_id"], k, repr(r["elevations_m"][k]), repr(float(p[0])), repr(float(p[1])), repr(amp[0]), repr(amp[1])])
        now = datetime.datetime.now(datetime.timezone.utc).isoformat(timespec="seconds")
        manifest = {
            "command": "solve", "config": {"grid": grid_dict, "solver": pipe_config.solver.to_dict(), "backend": pipe_config.backend, "k_max": pipe_config.k_max},
            "seed": seed, "code_version": __version__, "inputs": {str(stack_path): _sha256(stack_path)},
            "outputs": {str(p): _sha256(p) for p in (out_jsonl, out_csv) if p is not None}, "started_utc": now, "finished_utc": now,
        }
        with open(str(out_jsonl) + ".manifest.json", "w", encoding="utf-8") as fh:
            json.dump(manifest, fh, indent=2, sort_keys=True)
            fh.write("\n")
    return records

