"""Sample sharding of a logical batch across ranks: rank r owns the contiguous
slice [r*B/W, (r+1)*B/W). Params are replicated; each rank clips and sums its own samples; one
all-reduce of the flat clipped sum; noise once from the shared seed on every rank."""


def shard_range(batch: int, world: int, rank: int):
    lo = batch * rank // world
    hi = batch * (rank + 1) // world
    return lo, hi
