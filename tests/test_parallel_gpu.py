"""The multi-rank paths with the real CUDA op: two ranks
(gloo, both on the one leased GPU -- NCCL needs one GPU per rank) run
  * head-sharded attention (no collective on the data path), and
  * the Ulysses path on sequence-sharded input (per-head all-to-all straight
    into the preallocated head buffer, head groups of 1 and 2),
and every rank's output must equal the single-process call BITWISE: heads
are independent problems and K1-K3 are deterministic, so the
reshuffle may not change a single bit."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

WORLD = 2
H, T_V, T_T, D, BLK = 4, 128 * 24, 256, 128, 128


def _inputs():
    g = torch.Generator().manual_seed(11)
    q, k, v = (torch.randn(1, H, T_V + T_T, D, generator=g).to(torch.bfloat16) for _ in range(3))
    return q, k, v


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out_dir, q_):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import paper_2511_19835_b200 as rsa
        from paper_2511_19835_b200.parallel import head_parallel_attention, ulysses_attention
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        q, k, v = (x.cuda() for x in _inputs())
        kw = dict(block=BLK, top_k_fraction=0.1)
        hp_out = head_parallel_attention(q, k, v, num_text_tokens=T_T, gather=True, **kw)
        s_loc = T_V // WORLD
        sl = slice(rank * s_loc, (rank + 1) * s_loc)
        res = {"head_parallel": hp_out.cpu()}
        for hpg in (1, 2):
            ov, ot = ulysses_attention(q[:, :, sl].contiguous(), k[:, :, sl].contiguous(), v[:, :, sl].contiguous(),
                                       q[:, :, T_V:].contiguous(), k[:, :, T_V:].contiguous(),
                                       v[:, :, T_V:].contiguous(), heads_per_group=hpg, check_status=False, **kw)
            res[f"ulysses{hpg}_video"] = ov.cpu()
            res[f"ulysses{hpg}_text"] = ot.cpu()
        torch.save(res, os.path.join(out_dir, f"rank{rank}.pt"))
        dist.destroy_process_group()
        q_.put((rank, "ok"))
        del rsa
    except Exception as exc:  # report to the parent
        q_.put((rank, repr(exc)))
        raise


def test_two_rank_paths_bitwise_equal_single_process(tmp_path):
    import paper_2511_19835_b200 as rsa
    q, k, v = (x.cuda() for x in _inputs())
    want = rsa.rectified_sparse_attention(q, k, v, num_text_tokens=T_T, block=BLK, top_k_fraction=0.1).cpu()
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, str(tmp_path), qq)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = [qq.get(timeout=5) for _ in range(WORLD)]
    assert all(msg == "ok" for _, msg in results), results
    s_loc = T_V // WORLD
    for r in range(WORLD):
        got = torch.load(tmp_path / f"rank{r}.pt")
        assert torch.equal(got["head_parallel"], want)
        for hpg in (1, 2):
            assert torch.equal(got[f"ulysses{hpg}_video"], want[:, :, r * s_loc:(r + 1) * s_loc])
            assert torch.equal(got[f"ulysses{hpg}_text"], want[:, :, T_V:])
