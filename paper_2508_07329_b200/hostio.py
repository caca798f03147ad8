"""Host-buffer serving loop shared by the single-GPU layer, the stack and
the expert-parallel runtime: a list of pinned host batches goes through
``forward(x_dev, out=...)`` with the H2D of batch b+1 and the D2H of batch
b-1 overlapping the forward of batch b (three streams, a ring of device
staging buffers so the caching allocator never frees across streams)."""

from __future__ import annotations

import torch


def _split_ends(batches: list, d: int, out_dtype, split_ends: int, quantum: int):
    """Allocate missing outputs; cut the first and the last batch into
    ``split_ends`` chunks (multiples of ``quantum`` rows) so the pipeline's
    fill (first H2D) and drain (last D2H) expose one chunk's copy, not a
    whole batch's. Returns (work items, the callers' output tensors)."""
    outs, items = [], []
    last = len(batches) - 1
    for i, (xh, oh) in enumerate(batches):
        n = xh.shape[0]
        if oh is None:
            oh = torch.empty((n, d), dtype=out_dtype, pin_memory=True)
        outs.append(oh)
        per = (n // split_ends) // quantum * quantum
        if split_ends > 1 and (i == 0 or i == last) and per > 0:
            cuts = [k * per for k in range(split_ends)] + [n]
            items += [(xh[a:b], oh[a:b]) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        else:
            items.append((xh, oh))
    return items, outs


def stream_batches(owner, forward, d: int, out_dtype, batches: list, depth: int = 2, split_ends: int = 1,
                   quantum: int = 1) -> list:
    """batches = [(x_host, out_host | None), ...] -> the out_host tensors
    after the last D2H. ``forward(x_dev, out=o)`` must write its [n, d]
    result into ``o`` on the current stream (and be row-parallel in chunks
    of ``quantum`` rows when ``split_ends`` > 1 cuts the end batches). The
    staging ring and copy streams are cached on ``owner`` (``_stream_io``)."""
    if not batches:
        return []
    batches, final = _split_ends(batches, d, out_dtype, split_ends, quantum)
    T = max(x.shape[0] for x, _ in batches)
    cur = torch.cuda.current_stream()
    io = getattr(owner, "_stream_io", None)
    if io is None or io["bufs"][0].shape[0] < T or len(io["bufs"]) < depth or io["bufs"][0].dtype != batches[0][0].dtype:
        io = {"h2d": torch.cuda.Stream(), "d2h": torch.cuda.Stream(),
              "bufs": [torch.empty((T, d), dtype=batches[0][0].dtype, device="cuda") for _ in range(depth)],
              "outs": [torch.empty((T, d), dtype=out_dtype, device="cuda") for _ in range(depth)]}
        owner._stream_io = io
    h2d, d2h, bufs, obufs = io["h2d"], io["d2h"], io["bufs"], io["outs"]
    h2d.wait_stream(cur)
    done = [None] * len(batches)          # forward of batch i finished (its input slot is free)
    copied = [None] * len(batches)        # D2H of batch i finished (its output slot is free)
    outs = []
    for i, (xh, oh) in enumerate(batches):
        slot, oslot = bufs[i % depth], obufs[i % depth]
        n = xh.shape[0]
        if oh is None:
            oh = torch.empty((n, d), dtype=out_dtype, pin_memory=True)
        with torch.cuda.stream(h2d):
            if i >= depth:
                h2d.wait_event(done[i - depth])
            slot[:n].copy_(xh, non_blocking=True)
            loaded = torch.cuda.Event()
            loaded.record(h2d)
        cur.wait_event(loaded)
        if i >= depth:
            cur.wait_event(copied[i - depth])
        forward(slot[:n], out=oslot[:n])
        done[i] = torch.cuda.Event()
        done[i].record(cur)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done[i])
            oh.copy_(oslot[:n], non_blocking=True)
            copied[i] = torch.cuda.Event()
            copied[i].record(d2h)
        outs.append(oh)
    d2h.synchronize()
    return final
