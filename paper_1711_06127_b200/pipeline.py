"""Host-buffer pipeline over the C ABI: the end-to-end public API.

``HostPipeline.run(raw_host, img_host)`` takes frames in pinned host memory,
and for every chunk of frames overlaps, on two CUDA streams, the host->device
copy of chunk i+1 with ``supra_bf_beamform`` + ``supra_bf_scanconvert`` of
chunk i and the device->host copy of chunk i-1's B-mode images.  Argument
marshalling and stream ordering only -- every computation is a library
kernel.  (The paper's nodes hand data containers that "may reside either on
the CPU or the GPU" to each other; this is that hand-off.)
"""
from __future__ import annotations

import torch

from .binding import SupraBF


class HostPipeline:
    def __init__(self, bf: SupraBF, chunk: int, device: int = 0):
        self.bf = bf
        self.chunk = chunk
        w = bf.w
        self.dev = torch.device(f"cuda:{device}")
        self.streams = [torch.cuda.Stream(self.dev), torch.cuda.Stream(self.dev)]
        shape = (chunk, w.num_events, w.C, w.S)
        self.raw = [torch.empty(shape, dtype=torch.int16, device=self.dev) for _ in range(2)]
        self.li = [bf.empty_line_img(chunk) for _ in range(2)]
        self.img = [bf.empty_img(chunk) for _ in range(2)]
        # one handle must not be used from two streams concurrently: the
        # kernels of chunk i and i+1 are ordered through `done` events
        self.done = [torch.cuda.Event() for _ in range(2)]

    def run(self, raw_host: torch.Tensor, img_host: torch.Tensor) -> None:
        """raw_host: pinned int16 [F][E][C][S]; img_host: pinned [F][nz][ny][nx]."""
        F = raw_host.shape[0]
        prev = None
        for i, f0 in enumerate(range(0, F, self.chunk)):
            n = min(self.chunk, F - f0)
            b = i % 2
            st = self.streams[b]
            with torch.cuda.stream(st):
                self.raw[b][:n].copy_(raw_host[f0:f0 + n], non_blocking=True)
                if prev is not None:
                    st.wait_event(prev)          # serialise handle use across streams
                self.bf.beamform(self.raw[b], n, line_img=self.li[b], stream=st)
                self.bf.scanconvert(self.li[b], n, self.img[b], stream=st)
                self.done[b].record(st)
                prev = self.done[b]
                img_host[f0:f0 + n].copy_(self.img[b][:n], non_blocking=True)
        for st in self.streams:
            st.synchronize()
