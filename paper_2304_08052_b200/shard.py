"""Room sharding across GPUs (one process per GPU, no collective on the data path).

Rooms are independent (the reference farms them out to worker processes,
mixture.py:385-391).  Each rank takes a contiguous range of GLOBAL room
indices; because every room draws from Philox(SeedSequence((config, room)))
(workloads.py) the content is identical for any number of ranks.
"""

from __future__ import annotations


def shard_ranges(cfg: int, rank: int, world: int, rooms: int | None = None, chunk: int = 4096):
    """(start, count) room ranges rank `rank` of `world` renders, and the
    scaling kind.  Config 5 splits its fixed total (strong scaling) and streams
    it in `chunk`-room launches; configs 2-4 give every rank its own `rooms`
    (weak scaling); config 1 is the single fixed room."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if cfg == 1:
        return [(0, 1)], "weak"
    if cfg == 5:
        total = rooms or 65536
        lo, hi = rank * total // world, (rank + 1) * total // world
        return [(s, min(chunk, hi - s)) for s in range(lo, hi, chunk)], "strong"
    per = rooms or {2: 1024, 3: 4096, 4: 512}[cfg]
    return [(rank * per, per)], "weak"
