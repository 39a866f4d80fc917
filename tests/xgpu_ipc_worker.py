"""Worker of tests/test_gpu_xgpu.py::test_distributed_ipc_two_processes (launched by torchrun,
two ranks on cuda:0, gloo).  Each rank holds a block of the strips of every stripe in its own
IPC arena; encode and recovery go through xgpu.Distributed (partial -> barrier -> combine),
and each rank checks the strips it holds against the oracle / the generator."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from paper_cs_0611109_b200 import xgpu  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    p, N, nbytes, S, cfg = 13, 12, 2 * 12288 + 333, 3, 15
    stream = torch.cuda.Stream()
    plan = R.Plan(p, N, nbytes, 0, stream)
    X = xgpu.Distributed(plan, S, 0, backend="gloo")
    k_lo, k_hi = X.blocks[rank]
    pb = plan.pbytes
    for k in range(k_lo, k_hi):
        if k < N:
            R.fill(X.strip_addr(k), 0, X.ss, nbytes, 1, S, 0, cfg, 0, k, 0, stream)
        else:  # parity is an output: start from garbage
            R.fill(X.strip_addr(k), 0, X.ps, pb, 1, S, 99, cfg, 0, k, 0, stream)
    refs = []
    for s in range(S):
        data = synthetic.stripe_strips(0, cfg, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        refs.append(data + [P, Q])
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")

    def check(tag):
        stream.synchronize()
        dist.barrier()
        cnt.zero_()
        torch.cuda.synchronize()
        for k in range(k_lo, k_hi):
            ln = nbytes if k < N else pb
            for s in range(S):
                ref = torch.from_numpy(refs[s][k]).cuda()
                R.count_mismatch(X.strip_addr(k) + s * X.stride(k), int(ref.data_ptr()), ln, cnt, stream)
                stream.synchronize()
        assert int(cnt.item()) == 0, f"rank {rank} {tag}: {int(cnt.item())} bytes differ"

    X.step(stream, None)  # encode
    check("encode")
    for pairs in ([(1, 10), (3, N), (N, N + 1)], [(5, N + 1), (8, 9), (0, 11)]):
        for s, (x, y) in enumerate(pairs):  # owners poison their lost strips
            for k in (x, y):
                if k_lo <= k < k_hi:
                    R.fill(X.strip_addr(k) + s * X.stride(k), 0, 0, nbytes if k < N else pb, 1, 1, 77, cfg, 0, k, 0,
                           stream)
        stream.synchronize()
        dist.barrier()
        X.step(stream, pairs)
        check(f"recover {pairs}")
    X.close()
    plan.close()
    print(f"xgpu-ipc ok rank {rank}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
