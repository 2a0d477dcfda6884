"""RSAT files (reference rsat.py) and their GPU ingest."""

from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def files():
    return np.load(GOLDEN / "rsat_files.npz")


def test_writer_bytes_match_reference(files, tmp_path):
    from paper_2511_19835_b200.rsat import read_rsat, write_rsat
    for name in ("f32_2d", "f64_3d", "f32_1d"):
        p = tmp_path / f"{name}.rsat"
        write_rsat(p, files[name])
        assert p.read_bytes() == files[name + "_bytes"].tobytes(), name
        back = read_rsat(p)
        assert back.dtype == files[name].dtype and np.array_equal(back, files[name])


def test_reader_errors(tmp_path, files):
    from paper_2511_19835_b200 import IoError
    from paper_2511_19835_b200.rsat import read_rsat, write_rsat
    good = files["f32_2d_bytes"].tobytes()
    cases = {"magic": b"XSAT" + good[4:], "version": good[:4] + b"\x02" + good[5:],
             "dtype": good[:5] + b"\x07" + good[6:], "short": good[:-3], "tiny": good[:5]}
    for name, raw in cases.items():
        p = tmp_path / f"{name}.rsat"
        p.write_bytes(raw)
        with pytest.raises(IoError):
            read_rsat(p)
    with pytest.raises(IoError):
        read_rsat(tmp_path / "missing.rsat")
    with pytest.raises(IoError):
        write_rsat(tmp_path / "x.rsat", np.zeros(3, dtype=np.int32))


@pytest.mark.gpu
def test_device_ingest_and_problem_manifest(tmp_path):
    import torch

    import paper_2511_19835_b200 as rsa
    from oracle import rsa_oracle as O
    from paper_2511_19835_b200.rsat import load_problem, read_rsat_to_device, write_rsat
    qv, qt, k, v = O.random_problem(3, t_v=64, t_t=10, d=16, dtype=np.float32)
    paths = {"block": 16, "grid_dims": [1, 8, 8]}
    for name, a in (("q_video", qv), ("q_text", qt), ("k", k), ("v", v)):
        paths[name] = str(tmp_path / f"{name}.rsat")
        write_rsat(paths[name], a)
    t = read_rsat_to_device(paths["k"])
    assert t.is_cuda and t.dtype == torch.float32 and np.array_equal(t.cpu().numpy(), k)
    b = read_rsat_to_device(paths["k"], dtype=torch.bfloat16)
    assert torch.equal(b.cpu(), torch.from_numpy(k).to(torch.bfloat16))
    prob = load_problem(paths)
    assert prob.q_video.is_cuda and prob.grid_dims == (1, 8, 8) and prob.d == 16
    res = rsa.rectified_attention_pipeline(prob, rsa.SparsityConfig(0.25, 0.0, 0, False))
    ref = O.pipeline(qv, qt, k, v, 16, 0.25, 0.0, 0, False, "sparse-rectified")
    np.testing.assert_allclose(res.output.o_video.cpu().numpy(), ref["o_video"], atol=1e-5)
