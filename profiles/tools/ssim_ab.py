"""loss_image_grad through the library named by UBS_B200_LIB: saves g and the
loss parts for a few image sizes, and times the 1080p call."""
import sys, os, json
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_2510_03312_b200 import _lib
lib = _lib.load()
out = {}
for (H, W) in [(1080, 1920), (37, 53), (16, 12), (100, 140)]:
    g = torch.Generator(device="cpu").manual_seed(H * 7 + W)
    a = torch.rand(H, W, 3, generator=g).cuda()
    b = torch.rand(H, W, 3, generator=g).cuda()
    gi = torch.empty_like(a)
    parts = torch.zeros(2, dtype=torch.float64, device="cuda")
    scr = torch.empty(int(lib.ubs_loss_scratch_bytes(H, W, 0)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    call = lambda: lib.ubs_loss_image_grad(a.data_ptr(), b.data_ptr(), H, W, 0, 0.2, 1.0, gi.data_ptr(),
                                           parts.data_ptr(), scr.data_ptr(), s)
    assert call() == 0
    torch.cuda.synchronize()
    np.save(f"/tmp/ssim_{H}x{W}.npy", gi.cpu().numpy())
    out[f"{H}x{W}"] = parts.cpu().tolist()
    if H == 1080:
        for _ in range(5): call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): call()
        e1.record(); torch.cuda.synchronize()
        out["ms"] = e0.elapsed_time(e1) / 50
print(json.dumps(out))
