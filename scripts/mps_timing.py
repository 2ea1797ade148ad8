"""write_mps on the device (mps_device.cu) against the host writer
(XE_MPS_HOST=1): wall time of xe_write_mps (size call + copy-out) for
VGG-16 / ResNet-50 / U-Net, text bytes and equality."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402
import ctypes as C  # noqa: E402
C.pythonapi.PyBytes_FromStringAndSize.restype = C.py_object
C.pythonapi.PyBytes_FromStringAndSize.argtypes = [C.c_void_p, C.c_ssize_t]
from paper_2212_09290_b200._lib import LIB, check  # noqa: E402

print("THP", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
out = {}
for name in ("vgg16", "resnet50", "unet"):
    prob = xe.Problem.from_json(configs.CONFIGS[name]())
    row = {}
    texts = {}
    for mode in ("device", "host"):
        if mode == "host":
            os.environ["XE_MPS_HOST"] = "1"
        else:
            os.environ.pop("XE_MPS_HOST", None)
        best = None
        for _ in range(5):
            m = xe.build_model(prob, xe.ModelOptions(strict_free=False))
            m.csc()  # CSC build (shared with K3) outside the emission timing
            torch.cuda.synchronize()
            n = C.c_size_t()
            t0 = time.perf_counter()
            check(LIB.xe_write_mps(m._h, None, C.byref(n)))
            t1 = time.perf_counter()
            text = C.pythonapi.PyBytes_FromStringAndSize(None, n.value)
            t2 = time.perf_counter()
            check(LIB.xe_write_mps(m._h, C.c_char_p(text), C.byref(n)))
            t3 = time.perf_counter()
            dt = t3 - t0
            row.setdefault(mode + "_split_ms", []).append([round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2), round((t3 - t2) * 1e3, 2)])
            best = dt if best is None else min(best, dt)
        texts[mode] = text
        row[mode + "_ms"] = round(best * 1e3, 2)
    row["bytes"] = len(texts["device"])
    row["equal"] = texts["device"] == texts["host"]
    row["device_GB_per_s"] = round(row["bytes"] / (row["device_ms"] * 1e-3) / 1e9, 2)
    out[name] = row
    print(name, row, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/mps_timing.json", "w"), indent=1)
