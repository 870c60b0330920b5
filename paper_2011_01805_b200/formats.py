"""Host file formats either side of pack / unpack.

  dense tensor text   dense.hpp:200-242 (read_tensor / write_tensor):
                      "shape: n1 ... nk", then row-major values, %.17g
  packed tile file    tools/tiletensor_main.cpp:76-128 (write_tiles_file /
                      read_tiles_file): "shape: <shape>", optional
                      "relaxed: true", "slots: s", then one "tile: v ..." line
                      per tile in row-major external order

Both are plain text; values print with 17 significant digits, so a write ->
read round trip is bit exact.  '#' lines are comments.
"""
from __future__ import annotations

from typing import Union

import numpy as np

from .nn import read_tensor, write_tensor  # noqa: F401  (dense text format)
from .tiletensor import Session, TileTensor, TileTensorShape, format_shape, parse_shape


def write_tiles(t: TileTensor) -> str:
    """Text of write_tiles_file for a tile tensor (tiles read back from the GPU)."""
    out = [f"shape: {format_shape(t.shape())}\n"]
    if t.shape().relaxed():
        out.append("relaxed: true\n")
    out.append(f"slots: {t.session().slot_count()}\n")
    for row in t.tiles():
        out.append("tile:" + "".join(" " + format(float(v), ".17g") for v in row) + "\n")
    return "".join(out)


def read_tiles(text: Union[str, bytes], session: Session) -> TileTensor:
    """read_tiles_file: the tile tensor (uploaded to the session's GPU)."""
    if isinstance(text, bytes):
        text = text.decode()
    shape = None
    slots = 0
    rows = []
    for line in text.splitlines():
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        tag = parts[0] if parts else ""
        if tag == "shape:":
            shape = parse_shape(parts[1])
        elif tag == "relaxed:":
            if shape is not None:
                shape = TileTensorShape(shape.dims(), True)
        elif tag == "slots:":
            slots = int(parts[1])
            if slots != session.slot_count():
                raise RuntimeError(f"tile file was packed with {slots} slots; rerun with --slots "
                                   f"{slots}")
        elif tag == "tile:":
            vals = [float(x) for x in parts[1:]]
            if len(vals) != session.slot_count():
                raise ValueError("tile width does not match the slot count")
            rows.append(vals)
        else:
            raise RuntimeError("unrecognized line in tile file: " + line)
    if shape is None:
        raise RuntimeError("tile file has no shape line")
    tiles = np.array(rows, dtype=np.float64).reshape(len(rows), session.slot_count())
    return TileTensor(shape, tiles, session)
