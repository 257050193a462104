"""Multi-GPU assembly: one process per GPU (torch.distributed, NCCL over NVLink).

Outer elements are independent units.  Each rank
  1. builds the element pairs of its contiguous range of outer elements only,
     all-gathers the 4-byte partner lists and per-element pair counts, and
     builds the node pattern from the gathered list (identical on every rank:
     the list is the single-GPU one, concatenated in outer order),
  2. integrates its range of outer elements (z-slabs on lattice
     meshes, whose element ids are z-major) into the fixed-point partial sums
     of the pattern (integer words),
  3. all-reduces the partials (int64 words; per-element rhs partials are written
     by one rank only) -- integer addition is exact and order-free, so the sum is
     bit-identical to a single-GPU run for any number of ranks,
  4. finalizes its own block of output rows,
  5. all-gathers the CSR row blocks, row pointers and rhs.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous split of n items."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_by_weight(offsets: np.ndarray, rank: int, world: int) -> tuple[int, int]:
    """Contiguous split of items whose prefix weights are `offsets` (len n+1)
    into `world` ranges of about equal weight (e.g. outer elements by pairs)."""
    n = len(offsets) - 1
    total = offsets[-1]
    cut = [0] + [int(np.searchsorted(offsets, total * k / world, side="left")) for k in
                 range(1, world)] + [n]
    cut = np.maximum.accumulate(np.clip(cut, 0, n))
    return int(cut[rank]), int(cut[rank + 1])


def concat_csr(blocks: list[dict]) -> dict:
    """Stack CSR row blocks (row_ptr relative to each block) into one system."""
    rp = [np.zeros(1, np.int64)]
    base = 0
    for b in blocks:
        r = b["row_ptr"].astype(np.int64)
        rp.append(r[1:] + base)
        base += int(r[-1])
    return {"row_ptr": np.concatenate(rp).astype(np.int32),
            "col_idx": np.concatenate([b["col_idx"] for b in blocks]).astype(np.int32),
            "values": np.concatenate([b["values"] for b in blocks]).astype(np.float64),
            "rhs": np.concatenate([b["rhs"] for b in blocks]).astype(np.float64)}


def allgather_csr(block: dict, group=None, device=None) -> dict:
    """All-gather variable-size CSR row blocks (NCCL for CUDA tensors, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")

    def gather(arr: np.ndarray, dtype) -> list[np.ndarray]:
        t = torch.as_tensor(np.ascontiguousarray(arr), dtype=dtype, device=dev)
        n = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
        sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        m = int(max(int(s.item()) for s in sizes))
        pad = torch.zeros(max(m, 1), dtype=dtype, device=dev)
        pad[: t.numel()] = t
        outs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        return [o[: int(s.item())].cpu().numpy() for o, s in zip(outs, sizes)]

    rps = gather(block["row_ptr"], torch.int32)
    cis = gather(block["col_idx"], torch.int32)
    vas = gather(block["values"], torch.float64)
    rhs = gather(block["rhs"], torch.float64)
    return concat_csr([{"row_ptr": a, "col_idx": b, "values": c, "rhs": d}
                       for a, b, c, d in zip(rps, cis, vas, rhs)])


def _comm_device(group=None):
    """Where the collectives' buffers live: HBM for NCCL, host memory for gloo
    (the CPU test backend; it also drives several ranks on one GPU)."""
    import torch
    import torch.distributed as dist
    return torch.device("cpu") if dist.get_backend(group) == "gloo" else torch.device("cuda")


def allreduce_partials(V, rhsT, group=None) -> None:
    """In-place integer sum of the fixed-point partials across ranks."""
    import torch.distributed as dist
    if V.device.type == "cuda" and _comm_device(group).type == "cpu":
        for t in (V, rhsT):
            h = t.cpu()
            dist.all_reduce(h, group=group)
            t.copy_(h)
        return
    dist.all_reduce(V, group=group)
    dist.all_reduce(rhsT, group=group)


def gather_pairs(session, lo: int, hi: int, group=None, device=None) -> int:
    """Build this rank's element pairs (outer elements [lo, hi)), all-gather the
    pair counts and partner ids of every rank (NCCL, padded device tensors) and
    install the concatenation -- the unsharded pair list -- for the next
    run_shard.  Returns the total number of element pairs."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    npairs = session.pairs_shard(lo, hi)
    cview, pview = session.pairs_shard_out()
    dev = torch.device("cuda") if device is None else torch.device(device)
    src = "cuda" if torch.cuda.is_available() else dev  # the session's arrays live in HBM
    counts = (torch.as_tensor(cview, device=src).to(dev) if hi > lo
              else torch.zeros(0, dtype=torch.int32, device=dev))
    partners = (torch.as_tensor(pview, device=src).to(dev) if npairs > 0
                else torch.zeros(0, dtype=torch.int32, device=dev))
    counts, partners = counts.to(torch.int32), partners.to(torch.int32)
    # the install reads device arrays, after torch's current stream
    stream = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    if world == 1:
        if counts.device.type != "cuda" and torch.cuda.is_available():
            counts, partners = counts.cuda(), partners.cuda()
        session.pairs_install(counts, partners, npairs, stream=stream)
        return npairs
    # flat outputs viewed as (world, n): accepted by NCCL and gloo alike
    meta = torch.tensor([hi - lo, npairs], dtype=torch.int64, device=dev)
    metas = torch.empty(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(metas, meta, group=group)
    m = metas.view(world, 2).cpu().numpy()

    def gather(t, n_max):
        pad = torch.zeros(max(int(n_max), 1), dtype=t.dtype, device=dev)
        pad[: t.numel()] = torch.as_tensor(t, device=dev)
        out = torch.empty(world * pad.numel(), dtype=t.dtype, device=dev)
        dist.all_gather_into_tensor(out, pad, group=group)
        return out.view(world, pad.numel())

    gc = gather(counts, m[:, 0].max())
    gp = gather(partners, m[:, 1].max())
    all_counts = torch.cat([gc[r, : int(m[r, 0])] for r in range(world)])
    all_partners = torch.cat([gp[r, : int(m[r, 1])] for r in range(world)])
    total = int(m[:, 1].sum())
    if all_counts.device.type != "cuda" and torch.cuda.is_available():
        all_counts, all_partners = all_counts.cuda(), all_partners.cuda()
    session.pairs_install(all_counts, all_partners, total, stream=stream)
    return total


def assemble_distributed(session, group=None, stream: int | None = None) -> tuple[dict, dict]:
    """Sharded assembly on this rank's GPU; every rank returns the full system
    on the host: device_step (partials all-reduced and row blocks all-gathered
    in HBM over NCCL), then one device-to-host copy of the gathered CSR."""
    import torch
    (va, ci, rh), st = device_step(session, group, stream)
    ro = torch.as_tensor(session.outputs()[0], device="cuda")
    full = {"row_ptr": ro.to(torch.int32).cpu().numpy(), "col_idx": ci.cpu().numpy(),
            "values": va.cpu().numpy(), "rhs": rh.cpu().numpy()}
    return full, st.as_dict()


def device_step(session, group=None, stream: int | None = None):
    """One sharded assembly with every array staying in HBM: integrate this
    rank's outer elements, all-reduce the exact partials (NCCL), finalize this
    rank's row block, all-gather the row blocks' values, columns and rhs
    (NCCL all_gather on padded device tensors).  Returns the gathered device
    tensors (values, col_idx, rhs) and the run statistics."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cdev = _comm_device(group)
    lo, hi = shard_range(session.interior_count, rank, world)
    gather_pairs(session, lo, hi, group, device=cdev)
    st = session.run_shard(lo, hi, finalize=False, stream=stream)
    vv, rv = session.partials()
    V = torch.as_tensor(vv, device="cuda")
    R = torch.as_tensor(rv, device="cuda")
    allreduce_partials(V, R, group)
    r0, r1 = shard_range(session.unknowns, rank, world)
    # the reduced partials are ready on torch's current stream (NCCL enqueues
    # there): the session's finalize waits on it
    session.finalize(r0, r1, stream=torch.cuda.current_stream().cuda_stream)
    ro, ci, va, rh = (torch.as_tensor(x, device="cuda") for x in session.outputs())
    # row-block extents on every rank (row offsets are identical everywhere)
    bounds = [shard_range(session.unknowns, r, world) for r in range(world)]
    offs = ro.cpu().numpy() if world > 1 else None
    out = []
    for arr, per_row in ((va, False), (ci, False), (rh, True)):
        if world == 1:
            out.append(arr)
            continue
        ext = [((a, b) if per_row else (int(offs[a]), int(offs[b]))) for a, b in bounds]
        m = max(b - a for a, b in ext)
        a, b = ext[rank]
        pad = torch.zeros(max(m, 1), dtype=arr.dtype, device=cdev)
        pad[: b - a] = arr[a:b].to(cdev)
        gathered = torch.empty(world * max(m, 1), dtype=arr.dtype, device=cdev)
        dist.all_gather_into_tensor(gathered, pad, group=group)
        gathered = gathered.view(world, max(m, 1))
        out.append(torch.cat([gathered[r, : e[1] - e[0]] for r, e in enumerate(ext)]).to("cuda"))
    return out, st
