"""Host-buffer pipeline: the end-to-end replacement of run_apply's read -> transform -> write loop
(tools/hygt_main.cpp:130-172) for data that lives in host memory.

Rows are processed in chunks on two CUDA streams so that the H2D copy of chunk i+1, the
transforms of chunk i and the D2H copy of chunk i-1 overlap (copy engines run both directions
concurrently with the SMs). Host buffers should be pinned.
"""
from __future__ import annotations

import torch

from .plan import HyGTPlan


class HostPipeline:
    def __init__(self, plan: HyGTPlan, rows_per_chunk: int = 1 << 20, device=None, streams: int = 2):
        self.plan = plan
        self.rows = rows_per_chunk
        self.device = device or torch.device("cuda")
        n = plan.n
        self.slots = []
        for _ in range(streams):
            self.slots.append({
                "stream": torch.cuda.Stream(device=self.device),
                "x": torch.empty((rows_per_chunk, n), dtype=torch.float32, device=self.device),
                "y": torch.empty((rows_per_chunk, n), dtype=torch.float32, device=self.device),
                "r": torch.empty((rows_per_chunk, n), dtype=torch.float32, device=self.device),
                "c": torch.empty(rows_per_chunk, dtype=torch.uint16, device=self.device),
                "ws": torch.zeros(plan.workspace_bytes(rows_per_chunk), dtype=torch.uint8,
                                  device=self.device),
            })

    def _chunks(self, total):
        for k, a in enumerate(range(0, total, self.rows)):
            yield k, a, min(total, a + self.rows)

    def forward(self, xh: torch.Tensor, ch, yh: torch.Tensor):
        """Host rows -> host coefficients (one direction)."""
        return self._run(xh, ch, yh, None, inverse=False)

    def inverse(self, yh: torch.Tensor, ch, xh: torch.Tensor):
        return self._run(yh, ch, xh, None, inverse=True)

    def roundtrip(self, xh: torch.Tensor, ch, yh: torch.Tensor, rh: torch.Tensor):
        """Encoder + decoder: host x -> host coefficients y and reconstruction r."""
        return self._run(xh, ch, yh, rh, inverse=False)

    def _run(self, src, ch, dst, rec, inverse):
        main = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(main)
        for k, a, b in self._chunks(src.shape[0]):
            s = self.slots[k % len(self.slots)]
            st = s["stream"]
            st.wait_event(start)
            m = b - a
            with torch.cuda.stream(st):
                x, y = s["x"][:m], s["y"][:m]
                x.copy_(src[a:b], non_blocking=True)
                c = None
                if ch is not None:
                    c = s["c"][:m]
                    c.copy_(ch[a:b], non_blocking=True)
                fn = self.plan.inverse if inverse else self.plan.forward
                fn(x, c, out=y, stream=st, workspace=s["ws"])
                dst[a:b].copy_(y, non_blocking=True)
                if rec is not None:
                    r = s["r"][:m]
                    self.plan.inverse(y, c, out=r, stream=st, workspace=s["ws"], reuse_buckets=True)
                    rec[a:b].copy_(r, non_blocking=True)
        for s in self.slots:
            ev = torch.cuda.Event()
            ev.record(s["stream"])
            main.wait_event(ev)
        return dst
