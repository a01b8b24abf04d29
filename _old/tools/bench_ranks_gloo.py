"""Two ranks sharing one GPU (gloo, host-staged comm) through bench.pint_leg: checks the
sharded MGRIT legs' collective logic (max-over-ranks timing, summed fine-step
accounting) outside NCCL.  python tools/bench_ranks_gloo.py"""
import json, os, socket, sys
import multiprocessing as mp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import bench
    from paper_2306_09497_b200 import pint
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = {n: bench.pint_leg(torch, n, pint.Comm(), iters=3) for n in ("cfg1", "cfg2")}
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    ps = [ctx.Process(target=main, args=(r, 2, port, out)) for r in range(2)]
    for p in ps: p.start()
    for p in ps: p.join()
    assert all(p.exitcode == 0 for p in ps)
    for n in ("cfg1", "cfg2"):
        a, b = out[0][n], out[1][n]
        assert a["fine_steps_per_iteration"] == a["fine_steps_per_iteration_expected"], a
        assert a["value"] == b["value"] and a["ranks"] == 2
        print(json.dumps({k: a[k] for k in ("value", "ranks", "slices_per_rank", "iterations",
                                             "fine_steps_per_iteration", "ms_per_iteration",
                                             "collectives")}))
