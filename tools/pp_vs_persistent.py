"""HV-size consistency of the ping-pong kernel against the persistent kernel:
    RSA_TC_PP=0 python tools/pp_vs_persistent.py save /tmp/ref.pt
    RSA_TC_PP=1 python tools/pp_vs_persistent.py cmp /tmp/ref.pt     (repeat)"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402
cfg = bench.CONFIGS["hv"]
heads = 8
q, k, v = bench.synth_inputs(torch, cfg, heads, 1234, torch.device("cuda"))
shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16")
conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
ws = workspace_for(shape, "cuda")
out = torch.empty_like(q)
nat.check(nat.lib().rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out), None,
                                _ptr(ws), _stream()))
nat.check(nat.lib().rsa_check_device_status(_ptr(ws), _stream()))
torch.cuda.synchronize()
if sys.argv[1] == "save":
    torch.save(out.cpu(), sys.argv[2])
    print("saved")
else:
    ref = torch.load(sys.argv[2])
    d = (out.cpu().float() - ref.float()).abs().amax(-1)
    print("max |pp - persistent| %.4g, rows > 2e-2: %d of %d" % (d.max().item(), int((d > 2e-2).sum()), d.numel()))
