"""Host-link microbenchmark: H2D GB/s for query-sized copies (~7 MB, the int64
indices of a 300-item cfg3 RMC2 query) from regular vs write-combined pinned
memory (rs_alloc_pinned_flags), back to back on one stream; two alternating
streams; 256 distinct source buffers; D2H alone and duplex (H2D and D2H on
separate streams at once: ~45 GB/s each way on the B200 box).

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
    # duplex: H2D on one stream while D2H runs on another (is the link's
    # other direction free for outputs?)
    hdst = [rs.PinnedBuffer(nbytes) for _ in range(2)]
    hd = [torch.frombuffer((ctypes.c_char * nbytes).from_address(b.ptr), dtype=torch.uint8)
          for b in hdst]
    d2h_stream = torch.cuda.Stream()
    for mode in ("d2h_only", "duplex"):
        torch.cuda.synchronize()
        e0.record(streams[0])
        d2h_stream.wait_event(e0)
        for i in range(reps):
            if mode == "duplex":
                with torch.cuda.stream(streams[0]):
                    dsts[0].copy_(srcs[i % 4], non_blocking=True)
            with torch.cuda.stream(d2h_stream):
                hd[i % 2].copy_(dsts[1], non_blocking=True)
        streams[0].wait_stream(d2h_stream)
        e1.record(streams[0])
        torch.cuda.synchronize()
        gbs = reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
        out[f"pinned_7MB_{mode}_gbs_per_direction"] = round(gbs, 1)
    # duplex with two H2D streams alternating (the library's host queue)
    torch.cuda.synchronize()
    e0.record(streams[0])
    streams[1].wait_event(e0)
    d2h_stream.wait_event(e0)
    for i in range(reps):
        with torch.cuda.stream(streams[i % 2]):
            dsts[i % 2].copy_(srcs[i % 4], non_blocking=True)
        with torch.cuda.stream(d2h_stream):
            hd[i % 2].copy_(dsts[(i + 1) % 2], non_blocking=True)
    streams[0].wait_stream(streams[1])
    streams[0].wait_stream(d2h_stream)
    e1.record(streams[0])
    torch.cuda.synchronize()
    out["pinned_7MB_duplex_two_h2d_streams_gbs_per_direction"] = round(
        reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
