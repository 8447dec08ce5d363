"""Dose-volume output: binary and slab-parallel writers.

The reference writes legacy-VTK STRUCTURED_POINTS volumes in ASCII, one value
per line (driver.write_volume, driver.py:672-690) -- 134 M lines at 512^3.
Here the same header and layout are written as legacy-VTK BINARY (big-endian
FP64, the byte order the format prescribes), which VTK/ParaView read and
which is ~20x smaller to parse; the values are bit-exact (no %.12e round
trip). `write_volume_slab` lets every rank of a z-slab solve write its own
contiguous cell range of each array into the one shared file with
positional writes (the flat index has z slowest, spatial.py:62-63, so a
slab is one byte range per array); no gather to rank 0.

`read_volume` reads both encodings (so reference ASCII files load), and
`compare_volumes` is driver.compare_volumes (driver.py:733-748).
"""

import os
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, OutputIOError


@dataclass(frozen=True)
class VolumeGrid:
    """The structured grid of a volume file (cell-centred values)."""

    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    origin: tuple = (0.0, 0.0, 0.0)

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz


def _grid(g) -> VolumeGrid:
    if isinstance(g, VolumeGrid):
        return g
    return VolumeGrid(int(g.nx), int(g.ny), int(g.nz), float(g.dx), float(g.dy), float(g.dz),
                      tuple(float(o) for o in getattr(g, "origin", (0.0, 0.0, 0.0))))


def _header(g: VolumeGrid, title: str, encoding: str) -> bytes:
    # the reference's header (driver.py:674-684): points at cell midpoints
    ox = g.origin[0] + 0.5 * g.dx
    oy = g.origin[1] + 0.5 * g.dy
    oz = g.origin[2] + 0.5 * g.dz
    return (
        "# vtk DataFile Version 3.0\n"
        f"{title}\n"
        f"{encoding}\n"
        "DATASET STRUCTURED_POINTS\n"
        f"DIMENSIONS {g.nx} {g.ny} {g.nz}\n"
        f"ORIGIN {ox:.9g} {oy:.9g} {oz:.9g}\n"
        f"SPACING {g.dx:.9g} {g.dy:.9g} {g.dz:.9g}\n"
        f"POINT_DATA {g.n_cells}\n"
    ).encode()


def _array_header(name: str) -> bytes:
    return f"SCALARS {name} double 1\nLOOKUP_TABLE default\n".encode()


def _layout(g: VolumeGrid, names, title):
    """Byte offset of every array's first value, and the file length."""
    off = len(_header(g, title, "BINARY"))
    starts = []
    for name in names:
        off += len(_array_header(name))
        starts.append(off)
        off += 8 * g.n_cells + 1  # values + newline
    return starts, off


def write_volume(path, grid, arrays: dict, title="pndose dose grid", binary=True):
    """driver.write_volume (driver.py:672-690); binary=False writes the
    reference's ASCII form byte for byte."""
    g = _grid(grid)
    try:
        if not binary:
            with open(path, "w") as fh:
                fh.write(_header(g, title, "ASCII").decode())
                for name, values in arrays.items():
                    fh.write(_array_header(name).decode())
                    for v in np.asarray(values).ravel():
                        fh.write(f"{v:.12e}\n")
            return
        with open(path, "wb") as fh:
            fh.write(_header(g, title, "BINARY"))
            for name, values in arrays.items():
                v = np.asarray(values, dtype=np.float64).ravel()
                if v.size != g.n_cells:
                    raise ConfigError(f"array {name} has {v.size} values for {g.n_cells} cells")
                fh.write(_array_header(name))
                fh.write(v.astype(">f8").tobytes())
                fh.write(b"\n")
    except OSError as exc:
        raise OutputIOError(f"cannot write volume file {path}: {exc}") from exc


def write_volume_slab(path, grid, names, local_arrays: dict, cell_lo: int, rank: int,
                      title="pndose dose grid"):
    """One rank's part of a binary volume: its cells [cell_lo, cell_lo + len)
    of every array (names fixes the array order on all ranks), written in place
    with positional writes; rank 0 also writes the headers and sets the
    length. Every rank must call it (then the file is complete once all have
    returned, e.g. after a barrier)."""
    g = _grid(grid)
    starts, total = _layout(g, names, title)
    try:
        fd = os.open(path, os.O_WRONLY | os.O_CREAT, 0o644)
        try:
            if rank == 0:
                os.ftruncate(fd, total)
                os.pwrite(fd, _header(g, title, "BINARY"), 0)
                for name, s in zip(names, starts):
                    ah = _array_header(name)
                    os.pwrite(fd, ah, s - len(ah))
                    os.pwrite(fd, b"\n", s + 8 * g.n_cells)
            for name, s in zip(names, starts):
                v = np.asarray(local_arrays[name], dtype=np.float64).ravel()
                if cell_lo < 0 or cell_lo + v.size > g.n_cells:
                    raise ConfigError(f"slab [{cell_lo}, {cell_lo + v.size}) outside the grid")
                os.pwrite(fd, v.astype(">f8").tobytes(), s + 8 * cell_lo)
        finally:
            os.close(fd)
    except OSError as exc:
        raise OutputIOError(f"cannot write volume file {path}: {exc}") from exc


def read_volume(path):
    """driver.read_volume (driver.py:693-730) for ASCII and BINARY files:
    (grid, {name: values})."""
    try:
        with open(path, "rb") as fh:
            blob = fh.read()
    except OSError as exc:
        raise OutputIOError(f"cannot read volume file {path}: {exc}") from exc
    pos = 0

    def line():
        nonlocal pos
        end = blob.find(b"\n", pos)
        if end < 0:
            end = len(blob)
        s = blob[pos:end].decode(errors="replace")
        pos = end + 1
        return s

    dims = origin = spacing = None
    encoding = None
    arrays = {}
    while pos < len(blob):
        s = line()
        if s in ("ASCII", "BINARY"):
            encoding = s
        elif s.startswith("DIMENSIONS"):
            dims = tuple(int(v) for v in s.split()[1:4])
        elif s.startswith("ORIGIN"):
            origin = tuple(float(v) for v in s.split()[1:4])
        elif s.startswith("SPACING"):
            spacing = tuple(float(v) for v in s.split()[1:4])
        elif s.startswith("SCALARS"):
            if dims is None:
                break
            name = s.split()[1]
            line()  # LOOKUP_TABLE
            count = dims[0] * dims[1] * dims[2]
            if encoding == "BINARY":
                arrays[name] = np.frombuffer(blob, dtype=">f8", count=count,
                                             offset=pos).astype(np.float64)
                pos += 8 * count
            else:
                arrays[name] = np.array([float(line()) for _ in range(count)])
    if dims is None or spacing is None or origin is None:
        raise OutputIOError(f"{path} is not a structured-points volume")
    grid = VolumeGrid(dims[0], dims[1], dims[2], spacing[0], spacing[1], spacing[2],
                      (origin[0] - 0.5 * spacing[0], origin[1] - 0.5 * spacing[1],
                       origin[2] - 0.5 * spacing[2]))
    return grid, arrays


def compare_volumes(path_a, path_b, array="deposited_energy"):
    """Relative L2 and Linf of A against reference B (driver.py:733-748)."""
    grid_a, arrays_a = read_volume(path_a)
    grid_b, arrays_b = read_volume(path_b)
    if grid_a.shape != grid_b.shape:
        raise ConfigError(f"volumes have different shapes {grid_a.shape} vs {grid_b.shape}")
    a, b = arrays_a[array], arrays_b[array]
    norm = np.linalg.norm(b)
    scale = np.abs(b).max()
    return {
        "rel_l2": float(np.linalg.norm(a - b) / norm) if norm > 0 else 0.0,
        "rel_linf": float(np.abs(a - b).max() / scale) if scale > 0 else 0.0,
    }
