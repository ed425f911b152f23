"""XYZ trajectory frames for large systems.

Same text format as the reference's write_xyz / read_xyz / state_from_xyz
(pkg/src/tersoffmd/system.py:233-307): a count line, a comment line carrying
`box Lx Ly Lz periodic ppp time t` (%.10g), then `symbol x y z` rows with
%.10f coordinates -- files are interchangeable with the reference's.  The
implementation is built for millions of atoms: positions may be a CUDA tensor
(one device-to-host copy per frame), rows are formatted in one vectorised
pass (no per-atom Python loop) and frames are parsed with numpy.
"""

import numpy as np

from .errors import InputError
from .state import MASSES, SimulationBox, SimulationState


def _host(a):
    return a if isinstance(a, np.ndarray) else a.detach().cpu().numpy()


def box_comment(state):
    L = state.box.lengths
    flags = "".join("1" if p else "0" for p in state.box.periodic)
    return (f"box {L[0]:.10g} {L[1]:.10g} {L[2]:.10g} periodic {flags} "
            f"time {getattr(state, 'time', 0.0):.10g}")


def format_frame(symbols, species, positions, comment):
    """The text of one frame (vectorised %.10f formatting)."""
    pos = np.ascontiguousarray(_host(positions), dtype=np.float64)
    names = np.asarray(symbols, dtype=object)[np.asarray(_host(species), dtype=np.int64)]
    n = pos.shape[0]
    body = ("%s %.10f %.10f %.10f\n" * n) % tuple(
        np.column_stack([names, pos]).ravel()) if n else ""
    return f"{n}\n{comment}\n{body}"


def write_xyz(path, state, comment=None, append=False):
    """Append (or write) one frame of `state` to `path`."""
    text = format_frame(state.symbols, state.species, state.positions,
                        box_comment(state) if comment is None else comment)
    with open(path, "a" if append else "w") as fh:
        fh.write(text)


def read_xyz(path):
    """Every frame as (symbols list, positions (n,3), comment)."""
    lines = open(path).read().split("\n")
    frames, at = [], 0
    while at < len(lines) and lines[at].strip():
        try:
            n = int(lines[at])
        except ValueError as exc:
            raise InputError(f"bad XYZ atom-count line {lines[at]!r}") from exc
        comment = lines[at + 1] if at + 1 < len(lines) else ""
        rows = [r.split() for r in lines[at + 2:at + 2 + n]]
        if len(rows) < n or any(len(r) < 4 for r in rows):
            bad = next((k for k, r in enumerate(rows) if len(r) < 4), len(rows))
            raise InputError(f"truncated XYZ row {bad}")
        tab = np.array([r[:4] for r in rows], dtype=object).reshape(n, 4)
        frames.append((list(tab[:, 0]), tab[:, 1:].astype(np.float64), comment))
        at += 2 + n
    return frames


def parse_box(comment):
    toks = comment.split()
    try:
        i, j = toks.index("box"), toks.index("periodic")
        return SimulationBox([float(t) for t in toks[i + 1:i + 4]],
                             tuple(ch == "1" for ch in toks[j + 1]))
    except (ValueError, IndexError):
        return None


def state_from_xyz(path, frame=-1, box=None):
    """A SimulationState from one frame; without a box comment the atoms are
    placed in a free box with 6 A margins (as the reference)."""
    frames = read_xyz(path)
    if not frames:
        raise InputError(f"no frames in {path}")
    symbols, pos, comment = frames[frame]
    box = box or parse_box(comment)
    if box is None:
        lo = pos.min(axis=0)
        box = SimulationBox(pos.max(axis=0) - lo + 12.0)
        pos = pos - lo + 6.0
    kinds = sorted(set(symbols))
    index = {k: q for q, k in enumerate(kinds)}
    species = np.fromiter((index[s] for s in symbols), dtype=np.int64, count=len(symbols))
    return SimulationState(pos, box, species=species,
                           masses=np.array([MASSES.get(k, MASSES["C"]) for k in kinds]),
                           symbols=tuple(kinds))
