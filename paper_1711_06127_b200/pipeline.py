"""Host-buffer pipeline over the C ABI: the end-to-end public API.

``HostPipeline.run(raw_host, img_host)`` takes frames in pinned host memory,
and for every chunk of frames overlaps, on two CUDA streams, the host->device
transfer of chunk i+1 with ``supra_bf_beamform`` + ``supra_bf_scanconvert`` of
chunk i and the device->host copy of chunk i-1's B-mode images.  The
transfer is ``supra_bf_stage_raw``: the device reads only the sample ranges
the beamformer uses from the pinned buffer (C2: 41 % of each frame);
``referenced_only=False`` copies whole frames instead.  Argument
marshalling and stream ordering only -- every computation is a library
kernel.  (The paper's nodes hand data containers that "may reside either on
the CPU or the GPU" to each other; this is that hand-off.)
"""
from __future__ import annotations

import torch

from .binding import SupraBF


class HostPipeline:
    def __init__(self, bf: SupraBF, chunk: int, device: int = 0, referenced_only: bool = True):
        self.bf = bf
        self.chunk = chunk
        self.referenced_only = referenced_only
        self.h2d_bytes = 0  # host->device bytes of the last run()
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
        self.h2d_bytes = 0
        for i, f0 in enumerate(range(0, F, self.chunk)):
            n = min(self.chunk, F - f0)
            b = i % 2
            st = self.streams[b]
            with torch.cuda.stream(st):
                if self.referenced_only:
                    self.h2d_bytes += n * self.bf.stage_raw(raw_host[f0:f0 + n], self.raw[b], n, stream=st)
                else:
                    self.raw[b][:n].copy_(raw_host[f0:f0 + n], non_blocking=True)
                    self.h2d_bytes += raw_host[f0:f0 + n].numel() * raw_host.element_size()
                if prev is not None:
                    st.wait_event(prev)          # serialise handle use across streams
                self.bf.beamform(self.raw[b], n, line_img=self.li[b], stream=st)
                self.bf.scanconvert(self.li[b], n, self.img[b], stream=st)
                self.done[b].record(st)
                prev = self.done[b]
                img_host[f0:f0 + n].copy_(self.img[b][:n], non_blocking=True)
        for st in self.streams:
            st.synchronize()
