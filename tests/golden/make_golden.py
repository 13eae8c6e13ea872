"""Generates tests/golden/forward_golden.npz: tiny models of every pooling kind,
their seeded parameters (re-implemented here in numpy), inputs,
and fp64 outputs computed with torch CPU ops (F.linear, nn.GRUCell,
tril_indices) — an implementation independent of both oracle/forward.c and
the CUDA kernels. The oracle is pinned against these fixtures
(tests/test_oracle.py); the reference itself has no numeric forward pass.

Run:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.nn.functional as F

M64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tid: int) -> int:
    v = (seed ^ ((tid * 0xD1B54A32D192ED03) & M64)) & M64
    return int(splitmix64(np.array([v], dtype=np.uint64))[0])


def lattice(h: np.ndarray) -> np.ndarray:
    q = (h >> np.uint64(40)).astype(np.int64) - 8388608
    return q.astype(np.float32) * np.float32(1.0 / 8388608.0)


def param(seed: int, tid: int, n: int, bound: np.float32) -> np.ndarray:
    k = stream_key(seed, tid)
    with np.errstate(over="ignore"):
        e = np.uint64(k) + np.arange(n, dtype=np.uint64)
    return (lattice(splitmix64(e)) * np.float32(bound)).astype(np.float32)


def fan(n: int) -> np.float32:
    return np.float32(1.0) / np.sqrt(np.float32(n))


def table(seed, t, rows, D):
    return param(seed, 0x1000 + t, rows * D, np.float32(0.05)).reshape(rows, D)


MODELS = {
    "tiny-dlrm": dict(dense_fc=[8, 8], predict_fc=[6, 2], stacks=1, T=3, L=4, D=8,
                      pooling="Sum", dense_in=6, hidden=0),
    "tiny-sum-nodense": dict(dense_fc=None, predict_fc=[5, 1], stacks=1, T=2, L=3, D=8,
                             pooling="Sum", dense_in=3, hidden=0),
    "tiny-concat": dict(dense_fc=None, predict_fc=[7, 3], stacks=2, T=2, L=2, D=8,
                        pooling="Concat", dense_in=5, hidden=0),
    "tiny-din": dict(dense_fc=None, predict_fc=[16, 2], stacks=1, T=2, L=5, D=8,
                     pooling="AttentionFC", dense_in=0, hidden=0),
    "tiny-dien": dict(dense_fc=None, predict_fc=[16, 2], stacks=1, T=2, L=4, D=8,
                      pooling="AttentionRNN", dense_in=0, hidden=6),
}
ROWS, SEED, S = 50, 5, 3


def forward(name, cfg, augru, dense, idx):
    T, L, D, H = cfg["T"], cfg["L"], cfg["D"], cfg["hidden"]
    t64 = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64))  # noqa: E731
    tabs = [t64(table(SEED, t, ROWS, D)) for t in range(T)]
    x = t64(dense)
    feats = []
    if cfg["dense_fc"]:
        fan_in = cfg["dense_in"]
        for l, o in enumerate(cfg["dense_fc"]):
            W = t64(param(SEED, 0x2000 + 2 * l, o * fan_in, fan(fan_in)).reshape(o, fan_in))
            b = t64(param(SEED, 0x2001 + 2 * l, o, fan(fan_in)))
            x = F.relu(F.linear(x, W, b))
            fan_in = o
    feats.append(x)
    gathered = torch.stack([torch.stack([tabs[t][torch.from_numpy(idx[:, t, l])]
                                         for l in range(L)], 1) for t in range(T)], 1)
    # gathered: [S, T, L, D]
    pool = cfg["pooling"]
    if pool == "Sum":
        pooled = gathered.sum(2)                                     # [S,T,D]
        feats.append(pooled.sum(1))
        if cfg["dense_fc"]:
            Z = torch.cat([x.unsqueeze(1), pooled], 1)               # [S,T+1,D]
            G = torch.bmm(Z, Z.transpose(1, 2))
            li, lj = torch.tril_indices(T + 1, T + 1, offset=-1)
            feats.append(G[:, li, lj])
        pooled_out = pooled.reshape(S, -1)
    elif pool == "Concat":
        pooled_out = gathered.reshape(S, -1)
        feats.append(pooled_out)
    elif pool == "AttentionFC":
        outs = []
        for t in range(T):
            W = t64(param(SEED, 0x4000 + t, D * D, fan(D)).reshape(D, D))
            q = gathered[:, t, 0, :]                                 # [S,D]
            e = gathered[:, t]                                       # [S,L,D]
            s = torch.sigmoid(torch.einsum("si,ij,slj->sl", q, W, e))
            outs.append(torch.einsum("sl,sld->sd", s, e))
        pooled_out = torch.cat(outs, 1)
        feats.append(pooled_out)
    else:
        outs = []
        for t in range(T):
            base = 0x5000 + 8 * t
            cell = torch.nn.GRUCell(D, H).double()
            with torch.no_grad():
                cell.weight_ih.copy_(t64(param(SEED, base + 0, 3 * H * D, fan(H)).reshape(3 * H, D)))
                cell.weight_hh.copy_(t64(param(SEED, base + 1, 3 * H * H, fan(H)).reshape(3 * H, H)))
                cell.bias_ih.copy_(t64(param(SEED, base + 2, 3 * H, fan(H))))
                cell.bias_hh.copy_(t64(param(SEED, base + 3, 3 * H, fan(H))))
            Wa = t64(param(SEED, base + 4, D * D, fan(D)).reshape(D, D))
            h = torch.zeros(S, H, dtype=torch.float64)
            ua = gathered[:, t, 0, :] @ Wa                           # [S,D]
            with torch.no_grad():
                for l in range(L):
                    xl = gathered[:, t, l, :]
                    if not augru:
                        h = cell(xl, h)
                    else:
                        gi = F.linear(xl, cell.weight_ih, cell.bias_ih)
                        gh = F.linear(h, cell.weight_hh, cell.bias_hh)
                        ir, iz, inn = gi.chunk(3, 1)
                        hr, hz, hn = gh.chunk(3, 1)
                        r = torch.sigmoid(ir + hr)
                        z = torch.sigmoid(iz + hz)
                        n = torch.tanh(inn + r * hn)
                        a = torch.sigmoid((ua * xl).sum(1, keepdim=True))
                        u = a * (1 - z)
                        h = (1 - u) * h + u * n
            outs.append(h)
        pooled_out = torch.cat(outs, 1)
        feats.append(pooled_out)
    X = torch.cat([f for f in feats if f.shape[1] > 0], 1)
    outs = []
    for z in range(cfg["stacks"]):
        y = X
        fan_in = X.shape[1]
        dims = cfg["predict_fc"]
        for l, o in enumerate(dims):
            wid = 0x3000 + 64 * z + 2 * l
            W = t64(param(SEED, wid, o * fan_in, fan(fan_in)).reshape(o, fan_in))
            b = t64(param(SEED, wid + 1, o, fan(fan_in)))
            y = F.linear(y, W, b)
            if l + 1 < len(dims):
                y = F.relu(y)
            fan_in = o
        outs.append(y)
    return torch.cat(outs, 1).detach().numpy(), pooled_out.detach().numpy()


def main():
    rng = np.random.default_rng(20010277)
    data = {}
    for name, cfg in MODELS.items():
        for augru in ([False, True] if cfg["pooling"] == "AttentionRNN" else [False]):
            key = name + ("-augru" if augru else "")
            dense = rng.uniform(-1, 1, size=(S, cfg["dense_in"])).astype(np.float32)
            idx = rng.integers(0, ROWS, size=(S, cfg["T"], cfg["L"]), dtype=np.int64)
            out, pooled = forward(name, cfg, augru, dense, idx)
            data[key + "/dense"] = dense
            data[key + "/idx"] = idx
            data[key + "/out"] = out
            data[key + "/pooled"] = pooled
    # a spec pin: the first elements of table 0 and of a query's index stream
    data["spec/table0_row7"] = table(SEED, 0, ROWS, 8)[7]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "forward_golden.npz")
    np.savez_compressed(path, **data)
    print("wrote", path, len(data), "arrays")


if __name__ == "__main__":
    main()
