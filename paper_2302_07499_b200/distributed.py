"""Multi-GPU assembly: one process per GPU (torch.distributed, NCCL over NVLink),
owner-computes (north star: "each rank assembles its own row
block").

Outer elements are independent units.  Rank r
  1. builds the element pairs of its contiguous range of outer elements only
     (z-slabs on lattice meshes, whose element ids are z-major), its LOCAL node
     pattern (the rows its pairs touch) and integrates the range into it as
     exact fixed-point partial sums (Session.run_local) -- no rank holds the
     global pair list or the global pattern;
  2. owns the unknown rows [b[r], b[r+1]) (row_bounds) and sends every local
     slot of another rank's rows to that rank as a record (row, col, 4 int64
     words), and the load-vector partials of its outer elements to the owners
     of their nodes (all-to-all of the halo only: exchange_records);
  3. sorts the records it received, sums equal keys as integers (exact and
     order-free: the merged row of node i is the global pattern row, its sums
     are the one-GPU sums) and finalizes its row block (finalize_merged);
  4. all-gathers the row blocks' row lengths (-> row pointers), columns,
     values and rhs.
The result is bit-identical to a one-GPU run for any number of ranks.
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


def row_bounds(unknowns: int, world: int) -> list[int]:
    """Row-block boundaries: rank r owns unknowns [b[r], b[r+1]) (dofs follow
    node ids, so on lattice meshes a block is a z-slab, like the outer-element
    shards)."""
    return [shard_range(unknowns, r, world)[0] for r in range(world)] + [unknowns]


def alltoallv(send, send_counts, recv_counts, group=None, device=None):
    """Variable-size all-to-all of a flat tensor whose entries are grouped by
    destination rank (send_counts[r] entries for rank r); returns the entries
    received from every rank, concatenated in rank order.  NCCL on device
    tensors; gloo stages through host memory."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else _comm_device(group)
    src = torch.as_tensor(send, device="cuda" if torch.cuda.is_available() else "cpu")
    src = src.to(dev)
    out = torch.empty(int(sum(recv_counts)), dtype=src.dtype, device=dev)
    dist.all_to_all_single(out, src, [int(c) for c in recv_counts],
                           [int(c) for c in send_counts], group=group)
    return out


def exchange_records(send: dict, counts: dict, group=None, device=None) -> dict:
    """Ship each rank's records to their owners.  send: name -> (flat tensor,
    words per record); counts: name -> per-destination record counts (numpy).
    Returns name -> flat tensor of the records this rank received."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else _comm_device(group)
    names = sorted(send)
    sc = torch.tensor(np.stack([np.asarray(counts[n], np.int64) for n in names], 1).reshape(-1),
                      dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)  # the record counts themselves
    rc = rc.view(world, len(names)).cpu().numpy()
    out = {}
    for k, n in enumerate(names):
        t, w = send[n]
        out[n] = alltoallv(t, np.asarray(counts[n], np.int64) * w, rc[:, k] * w, group, dev)
    return out


def assemble_distributed(session, group=None, stream: int | None = None) -> tuple[dict, dict]:
    """Sharded assembly on this rank's GPU; every rank returns the full system
    on the host: device_step (owner-computes, halo records exchanged, row
    blocks all-gathered in HBM over NCCL), then one device-to-host copy of the
    gathered CSR."""
    (va, ci, rh, rp), st = device_step(session, group, stream)
    rp = rp.cpu().numpy()
    if rp[-1] > 2**31 - 1:
        raise OverflowError(f"{int(rp[-1])} nonzeros exceed the int32 row pointers of the CSR")
    full = {"row_ptr": rp.astype(np.int32), "col_idx": ci.cpu().numpy(),
            "values": va.cpu().numpy(), "rhs": rh.cpu().numpy()}
    return full, st.as_dict()


def device_step(session, group=None, stream: int | None = None):
    """One owner-computes sharded assembly with every array in HBM (NCCL):

    1. run_local: this rank's outer elements [lo, hi) -- their pairs, the local
       node pattern and the integration (no other rank's pairs or pattern);
    2. halo exchange: every local slot of an unknown row goes to the rank that
       owns the row as a (row, col, 4 int64 words) record, and the load-vector
       partials of the outer elements at a rank's nodes go to it
       (all-to-all; NCCL send/recv over NVLink);
    3. finalize_merged: the owner sorts what it received, sums equal keys as
       integers and finalizes its row block -- bit for bit the one-GPU rows;
    4. the row blocks' values, columns and rhs are all-gathered.

    Returns the gathered device tensors (values, col_idx, rhs) and this rank's
    run statistics (its own outer elements)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cdev = _comm_device(group)
    KI, U = session.interior_count, session.unknowns
    lo, hi = shard_range(KI, rank, world)
    st = session.run_local(lo, hi, stream=stream)
    bounds = row_bounds(U, world)
    keys, words, kc = session.halo_records(bounds)
    ridx, rvals, rcnt = session.rhs_records(bounds)
    got = exchange_records({"keys": (keys, 1), "words": (words, 4), "ridx": (ridx, 1),
                            "rvals": (rvals, 32)},
                           {"keys": kc, "words": kc, "ridx": rcnt, "rvals": rcnt}, group, cdev)
    got = {k: v.to("cuda") for k, v in got.items()}
    r0, r1 = bounds[rank], bounds[rank + 1]
    # the received records are ready on torch's current stream
    session.finalize_merged(r0, r1, got["keys"], got["words"], got["ridx"], got["rvals"],
                            stream=torch.cuda.current_stream().cuda_stream)
    ro, ci, va, rh = (torch.as_tensor(x, device="cuda") for x in session.outputs())
    if world == 1:
        return [va, ci, rh, ro], st
    # all-gather the row blocks: row lengths (-> row pointers), columns,
    # values and rhs of every block, in rank order
    a, b = int(ro[r0].item()), int(ro[r1].item())
    parts = {"len": (ro[r0 + 1:r1 + 1] - ro[r0:r1]), "ci": ci[a:b], "va": va[a:b],
             "rh": rh[r0:r1]}
    full = {}
    for name, arr in parts.items():
        full[name] = allgather_var(arr, group, cdev).to("cuda")
    rp = torch.zeros(U + 1, dtype=torch.int64, device="cuda")
    rp[1:] = torch.cumsum(full["len"], 0)
    return [full["va"], full["ci"], full["rh"], rp], st


def allgather_var(arr, group=None, device=None):
    """All-gather variable-length flat tensors (padded to the longest), result
    concatenated in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else _comm_device(group)
    n = torch.tensor([arr.numel()], dtype=torch.int64, device=dev)
    sizes = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, n, group=group)
    sizes = sizes.cpu().numpy()
    m = int(max(sizes.max(), 1))
    pad = torch.zeros(m, dtype=arr.dtype, device=dev)
    pad[: arr.numel()] = arr.to(dev)
    g = torch.empty(world * m, dtype=arr.dtype, device=dev)
    dist.all_gather_into_tensor(g, pad, group=group)
    g = g.view(world, m)
    return torch.cat([g[r, : int(sizes[r])] for r in range(world)])
