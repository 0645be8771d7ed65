"""Zero-copy random-row gather rate vs row stride/alignment of the pinned host
store: does padding 400-B rows to 448 / 512 B (64- / 128-B aligned) cut the
PCIe read-request overhead? Rows/s and useful (400-B) GB/s per layout."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_08541_b200 import _lib  # noqa: E402

n_rows, m = 2_400_000, 80_000
ids = torch.randint(0, n_rows, (m,), dtype=torch.int32, device="cuda").sort().values
pos = torch.arange(m, dtype=torch.int32, device="cuda")
cnt = torch.tensor([m], dtype=torch.int64, device="cuda")
for stride in (400, 416, 448, 512):
    host = torch.zeros(n_rows * stride, dtype=torch.uint8).pin_memory()
    tab = _lib.host_device_pointer(host)
    out = torch.empty((m, stride), dtype=torch.uint8, device="cuda")
    for rif in (2, 4):
        ts = []
        for it in range(6):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            _lib.call("bgl_gather_list", pos.data_ptr(), cnt.data_ptr(), m, ids.data_ptr(), tab, stride,
                      out.data_ptr(), None, None, rif, 74, _lib.stream_ptr())
            e.record()
            e.synchronize()
            if it:
                ts.append(s.elapsed_time(e))
        t = min(ts) * 1e-3
        print(f"stride {stride} rows_in_flight {rif}: {m / t / 1e6:.2f} M rows/s, useful 400-B GB/s "
              f"{m * 400 / t / 1e9:.2f}, bytes read GB/s {m * stride / t / 1e9:.2f}", flush=True)
    del host
