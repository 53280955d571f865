"""Test-side order-independent digest of a composed graph, computed from the
graph's arrays in numpy -- independent of both the CUDA path and the oracle's C implementation of the
same definition (oracle/compose.c, orc_digest):

    D_f = sum over states s of hS_f(key(s), start, accept, out-degree)
        + sum over arcs   of hA_f(key(src), key(dst), ilabel, olabel, weight bits)   (mod 2^64), f = 0, 1
    key(a, b) = a * V_B + b;  fin = splitmix64 finalizer;
    hS_f = fin(fin(fin(key ^ seed_f) ^ (start | accept << 1 | 4)) ^ deg)
    hA_f = fin(fin(fin(fin(ksrc ^ seed_f ^ 0x5555...) ^ kdst) ^ (uint32(il) << 32 | uint32(ol))) ^ wbits)

Sums of per-state and per-arc hashes do not depend on state numbering or arc order, so two graphs
that are equal in canonical form (reading 24) have equal digests."""
import numpy as np

SEEDS = (np.uint64(0x9E3779B97F4A7C15), np.uint64(0xD1B54A32D192ED03))
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
FIVES = np.uint64(0x5555555555555555)


def fin(z):
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def digest_arrays(row_ptr, dst, ilabel, olabel, weight, is_start, is_accept, pair_a, pair_b, VB, chunk=1 << 24):
    """Digest of a composed graph given as host arrays (row_ptr int64 [V+1], arc arrays [E], state
    arrays [V]); chunked over arcs so graphs with billions of arcs fit in memory."""
    VB = np.uint64(VB)
    with np.errstate(over="ignore"):
        key = pair_a.astype(np.uint64) * VB + pair_b.astype(np.uint64)
        deg = np.diff(np.asarray(row_ptr, np.int64)).astype(np.uint64)
        fl = (is_start.astype(np.uint64) | (is_accept.astype(np.uint64) << np.uint64(1)) | np.uint64(4))
        d = []
        for f in range(2):
            d.append(int(np.sum(fin(fin(fin(key ^ SEEDS[f]) ^ fl) ^ deg), dtype=np.uint64)))
        E = int(row_ptr[-1])
        src_state = None
        for e0 in range(0, E, chunk):
            e1 = min(E, e0 + chunk)
            # source state of every arc of the chunk (row_ptr is monotone)
            src_state = np.searchsorted(np.asarray(row_ptr), np.arange(e0, e1, dtype=np.int64), side="right") - 1
            ks = key[src_state]
            kd = key[np.asarray(dst[e0:e1], np.int64)]
            lab = (np.asarray(ilabel[e0:e1]).astype(np.uint32).astype(np.uint64) << np.uint64(32)) | \
                np.asarray(olabel[e0:e1]).astype(np.uint32).astype(np.uint64)
            wb = np.ascontiguousarray(weight[e0:e1], dtype=np.float32).view(np.uint32).astype(np.uint64)
            for f in range(2):
                h = fin(fin(fin(fin(ks ^ SEEDS[f] ^ FIVES) ^ kd) ^ lab) ^ wb)
                d[f] = (d[f] + int(np.sum(h, dtype=np.uint64))) % (1 << 64)
        d = [x % (1 << 64) for x in d]
    return {"num_states": int(len(key)), "num_arcs": int(row_ptr[-1]), "d0": d[0], "d1": d[1]}


def digest_graph(g, VB):
    """Digest of a dict of host arrays as returned by fst.compose / Fst.to_host / oracle.compose."""
    return digest_arrays(g["row_ptr"], g["dst"], g["ilabel"], g["olabel"], g["weight"], g["is_start"],
                         g["is_accept"], g["pair_a"], g["pair_b"], VB)


# ------------------------------------------------------------------ the same definition in torch (GPU)
def _s64(x: int) -> int:
    x %= 1 << 64
    return x - (1 << 64) if x >= 1 << 63 else x


def digest_device(t, VB, chunk=1 << 26):
    """The digest of a composed graph from its DEVICE arrays (Fst.device_tensors(): zero-copy torch
    views), in int64 torch arithmetic (wrapping multiply; logical shifts emulated by masking) -- for
    graphs too large to copy to the host in test time.  Cross-checked against digest_arrays."""
    import torch

    def lsr(z, s):
        return (z >> s) & ((1 << (64 - s)) - 1)

    def fin_t(z):
        z = (z ^ lsr(z, 30)) * _s64(0xBF58476D1CE4E5B9)
        z = (z ^ lsr(z, 27)) * _s64(0x94D049BB133111EB)
        return z ^ lsr(z, 31)

    seeds = [_s64(int(x)) for x in SEEDS]
    fives = _s64(0x5555555555555555)
    rp = t["row_ptr"]
    key = t["pair_a"].to(torch.int64) * int(VB) + t["pair_b"].to(torch.int64)
    deg = rp[1:] - rp[:-1]
    fl = t["is_start"].to(torch.int64) | (t["is_accept"].to(torch.int64) << 1) | 4
    d = [int(fin_t(fin_t(fin_t(key ^ seeds[f]) ^ fl) ^ deg).sum().item()) for f in range(2)]
    E = int(rp[-1].item())
    for e0 in range(0, E, chunk):
        e1 = min(E, e0 + chunk)
        idx = torch.arange(e0, e1, device=rp.device, dtype=torch.int64)
        src = torch.searchsorted(rp, idx, right=True) - 1
        ks = key[src]
        kd = key[t["dst"][e0:e1].to(torch.int64)]
        lab = ((t["ilabel"][e0:e1].to(torch.int64) & 0xFFFFFFFF) << 32) | (t["olabel"][e0:e1].to(torch.int64) & 0xFFFFFFFF)
        wb = t["weight"][e0:e1].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        for f in range(2):
            d[f] += int(fin_t(fin_t(fin_t(fin_t(ks ^ (seeds[f] ^ fives)) ^ kd) ^ lab) ^ wb).sum().item())
    return {"num_states": int(key.numel()), "num_arcs": E, "d0": d[0] % (1 << 64), "d1": d[1] % (1 << 64)}
