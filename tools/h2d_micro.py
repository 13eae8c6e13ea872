"""Host-link microbenchmark: H2D GB/s for query-sized copies (~7 MB, the int64
indices of a 300-item cfg3 RMC2 query) from regular vs write-combined pinned
memory (rs_alloc_pinned_flags), back to back on one stream.

  python tools/h2d_micro.py
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2001_02772_b200 as rs
    out = {}
    for wc in (False, True):
        for mb in (1, 7, 32):
            nbytes = mb << 20
            bufs = [rs.PinnedBuffer(nbytes, write_combined=wc) for _ in range(4)]
            srcs = []
            for b in bufs:
                b.view(np.uint8, (nbytes,))[...] = 1
                t = torch.frombuffer((ctypes.c_char * nbytes).from_address(b.ptr), dtype=torch.uint8)
                srcs.append(t)
            dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            reps = max(8, (1 << 30) // nbytes)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for i in range(4):
                    dst.copy_(srcs[i], non_blocking=True)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for i in range(reps):
                    dst.copy_(srcs[i % 4], non_blocking=True)
                e1.record(s)
            torch.cuda.synchronize()
            gbs = reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
            out[f"{'wc' if wc else 'pinned'}_{mb}MB"] = round(gbs, 1)
            out["src_is_pinned"] = bool(srcs[0].is_pinned())
    # two copy streams alternating 7 MB copies (two DMA engines on the link)
    nbytes = 7 << 20
    bufs = [rs.PinnedBuffer(nbytes) for _ in range(4)]
    srcs = [torch.frombuffer((ctypes.c_char * nbytes).from_address(b.ptr), dtype=torch.uint8)
            for b in bufs]
    dsts = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    reps = 256
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)
    for i in range(reps):
        with torch.cuda.stream(streams[i % 2]):
            dsts[i % 2].copy_(srcs[i % 4], non_blocking=True)
    streams[0].wait_stream(streams[1])
    e1.record(streams[0])
    torch.cuda.synchronize()
    out["pinned_7MB_two_streams"] = round(reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    # many distinct source buffers (a pool of queries, 1.8 GB) vs the 4 above:
    # host-side translation of a large pinned footprint
    many = [rs.PinnedBuffer(nbytes) for _ in range(256)]
    msrc = [torch.frombuffer((ctypes.c_char * nbytes).from_address(b.ptr), dtype=torch.uint8)
            for b in many]
    for b in many:
        b.view(np.uint8, (nbytes,))[...] = 1
    torch.cuda.synchronize()
    e0.record(streams[0])
    streams[1].wait_event(e0)
    for i in range(reps):
        with torch.cuda.stream(streams[i % 2]):
            dsts[i % 2].copy_(msrc[i % 256], non_blocking=True)
    streams[0].wait_stream(streams[1])
    e1.record(streams[0])
    torch.cuda.synchronize()
    out["pinned_7MB_256_buffers"] = round(reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
