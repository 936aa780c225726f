"""One slab rank per GPU (run by tests/test_gpu_dist_spawn.py under torchrun):
fm_ctx_create_dist over a real NCCL communicator, the projection and the
matrix-free matvec on this rank's x-slab with the fused peer-store transposes
and with the staged ncclSend/ncclRecv all-to-all (FM_TRANSPOSE=nccl), each
against the single-device result of the same global input, bit for bit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402


def main():
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    pts = tuple(int(x) for x in sys.argv[1].split("x"))
    ng = int(np.prod(pts))
    A = M.uniform_field(pts, 9, seed=3)
    lam_g, mu_g, _, _ = M.bind_parameters(M.bernoulli(pts, 0.3, 2),
                                          [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
    F_g = abi.identity_field(pts, 3) + 0.05 * M.uniform_field(pts, 9, 41)
    with abi.Context(pts, 3, device=local) as c1:
        g_ref = c1.projection(c1.field(9, A)).download()
        m1 = abi.Model(c1, "hyper", lam_g, mu_g, matrix_free=True)
        F1, P1, d1, o1 = c1.field(9, F_g), c1.field(9), c1.field(9, A), c1.field(9)
        m1.evaluate(F1, P1)
        m1.apply(d1, o1)
        mv_ref = o1.download()
        m1.close()
    ok = True
    for arm in ("peer", "nccl"):
        if arm == "nccl":
            os.environ["FM_TRANSPOSE"] = "nccl"
        uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(abi.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        with abi.Context(pts, 3, device=local, dist=(world, rank, bytes(uid.cpu().numpy()))) as ctx:
            n = ctx.n
            sl = lambda a: np.concatenate([a[c * ng + rank * n:c * ng + (rank + 1) * n] for c in range(9)])
            assert ctx.ranks() == (world, rank, False)
            g = ctx.projection(ctx.field(9, sl(A))).download()
            m = abi.Model(ctx, "hyper", lam_g[rank * n:(rank + 1) * n], mu_g[rank * n:(rank + 1) * n],
                          matrix_free=True)
            F, P, dF, out = ctx.field(9, sl(F_g)), ctx.field(9), ctx.field(9, sl(A)), ctx.field(9)
            m.evaluate(F, P)
            m.apply(dF, out)
            mv = out.download()
            nA = ctx.norm(ctx.field(9, sl(A)))  # a cross-rank reduction (ordered sum over ranks)
            m.close()
        good = np.array_equal(g, sl(g_ref)) and np.array_equal(mv, sl(mv_ref)) and \
            abs(nA - np.linalg.norm(A)) <= 1e-12 * np.linalg.norm(A)
        print(f"rank {rank} arm {arm}: {'OK' if good else 'MISMATCH'}", flush=True)
        ok = ok and good
        os.environ.pop("FM_TRANSPOSE", None)
    t = torch.tensor([1.0 if ok else 0.0], device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 1.0 else 1)


if __name__ == "__main__":
    main()
