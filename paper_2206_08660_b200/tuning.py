"""Explicit library switches (no environment variables are read by the
library). Every switch is exact: results are bit-identical either way; only
speed and memory change. Set attributes on `TUNING` (tests and tools do), or
pass the per-call arguments where a function offers them."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class Tuning:
    # corner records (vdi_volume_cells) for generation / DVR sampling:
    # None = automatic (u8 volumes whose records fit in a quarter of HBM)
    cells: bool | None = None
    # the largest band-sharded world whose ranks still build the corner
    # records (each rank builds them for the whole volume)
    cells_max_world: int = 2
    # empty-tile skipping in the render DDA (VdiRenderArgs.list_tiles)
    list_tiles: bool = False
    # per-list depth ranges for the render's search-first path
    # (VdiRenderArgs.list_range)
    list_ranges: bool = True
    # render as one resident grid taking 8x4 tiles from a counter
    # (VdiRenderArgs.tile_counter)
    dyn_tiles: bool = False
    # multi-GPU VDI exchange as packed VDI1 shards (False: plain all-gather)
    packed_exchange: bool = True


TUNING = Tuning()
