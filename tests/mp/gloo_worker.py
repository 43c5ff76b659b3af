"""One rank of the world-size-2 CPU test of bench.py's multi-GPU host logic
(tests/test_multi_rank.py launches it with torch.distributed.run, gloo)."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as dist

    import bench
    from oracle import acoustic as O
    from paper_1608_03984_b200.synthetic import config1

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    # max over ranks: rank r "took" 3 + 2r ms
    ms = bench.max_over_ranks(3.0 + 2.0 * rank, dist, "cpu")
    rate = bench.whole_job_rate(world, 1.0e9, ms)
    # replicas only: each rank runs the same independent simulation; no
    # data-path collective, and every replica's result is identical
    st = O.simulate(config1(n_t=4))
    digest = hashlib.sha256(st.latest().tobytes()).hexdigest()
    digests = [None] * world
    dist.all_gather_object(digests, digest)
    # the reference arm does its work on rank 0 only: other ranks exit 0 at once
    ref_rc, ref_s = None, None
    if rank != 0:
        sys.argv = ["bench.py", "--impl", "reference"]
        t0 = time.perf_counter()
        ref_rc = bench.reference_arm(bench.parse())
        ref_s = time.perf_counter() - t0
    others = [None] * world
    dist.all_gather_object(others, {"ms": ms, "rate": rate, "ref_rc": ref_rc, "ref_s": ref_s})
    if rank == 0:
        with open(os.environ["FDR_MP_OUT"], "w", encoding="utf-8") as fh:
            json.dump({"world": world, "ranks": others, "digests": digests}, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
