"""Process bodies for the one-process-per-rank tests (imported by spawned children).

Each child joins a gloo group on 127.0.0.1 (the exchange used by
L.RankSession at setup and on errors), builds the cloud from arrays and runs
its RCB piece; results go back to the parent through a queue.
"""
import os
import socket
import traceback

import numpy as np


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def run_rank(rank, world, port, arrays, prim0, cfg, splits, device, out):
    """Runs `sum(splits)` iterations in the given slices; puts (rank, result)."""
    dist = _init(rank, world, port)
    try:
        from paper_2403_13287_b200 import lskum as L

        pc = L.Cloud.from_arrays(*arrays)
        pc.reset_store(0)
        pc.set_primitives(prim0)
        conf = L.Config(**cfg)
        try:
            with L.RankSession(pc, conf, rank, world, device, capacity=sum(splits), from_state=True) as s:
                for n in splits:
                    s.iterate(n)
                res = s.residues()
                info = s.info()
                s.download()
            out.put((rank, ("ok", res, pc.fields(), info)))
        except L.LskumError as e:
            out.put((rank, ("err", e.status, e.message)))
    except Exception:  # surfaced by the parent
        out.put((rank, ("crash", traceback.format_exc())))
    finally:
        dist.destroy_process_group()


def host_maps(rank, world, port, arrays, n_parts, out):
    """Every rank derives the RCB owner map on its own; ranks must agree bit for bit."""
    dist = _init(rank, world, port)
    try:
        from paper_2403_13287_b200 import lskum as L

        pc = L.Cloud.from_arrays(*arrays)
        owned, ghosts = L.partition(pc, n_parts)
        mine = ([o.tobytes() for o in owned], [g.tobytes() for g in ghosts])
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
        out.put((rank, ("ok", all(e == everyone[0] for e in everyone), owned)))
    except Exception:
        out.put((rank, ("crash", traceback.format_exc())))
    finally:
        dist.destroy_process_group()


def create_without_device(rank, world, port, arrays, out):
    """RankSession creation on a host with no usable device fails on every rank
    with the same collectively agreed error (no rank hangs in the exchange)."""
    dist = _init(rank, world, port)
    try:
        from paper_2403_13287_b200 import lskum as L

        pc = L.Cloud.from_arrays(*arrays)
        try:
            L.RankSession(pc, L.Config(iters=2), rank, world, device=0, capacity=2)
            out.put((rank, ("ok",)))
        except L.LskumError as e:
            out.put((rank, ("err", e.status, e.message)))
    except Exception:
        out.put((rank, ("crash", traceback.format_exc())))
    finally:
        dist.destroy_process_group()


def launch(target, world, *args, timeout=240):
    """Spawns `world` ranks of target(rank, world, port, *args, queue)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(world):
            r, v = q.get(timeout=timeout)
            got[r] = v
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, v in got.items():
        assert v[0] != "crash", f"rank {r}:\n{v[1]}"
    return [got[r] for r in range(world)]
