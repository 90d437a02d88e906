"""CUDA-graph execution of a fixed bi-network forward (latency path).

A single-image forward (BASELINE config 1) issues ~800 reference-level HE
ops -> thousands of small kernel launches plus Python dispatch.  For a fixed
(network, weights, context, input shape) that sequence never changes, so it
is captured once into a CUDA graph and replayed per request: encryption
(fresh Philox ids from a device-side counter), plaintext branch, every HE
op, decryption of the logits -- one graph launch.  The OpRecorder counts of
the captured forward are kept so each replay still reports the reference's
op counts.  This replaces a tracing compiler: the capture is of the real
library launches, nothing is re-implemented.

The graph replays raw device pointers: into the context's scratch arenas and
pointer tables, and into the HBM plaintext cache.  So after capture the
context is frozen (`bcn_ctx_freeze`: a later call that would grow or free an
arena raises UsageError instead of moving memory under the graph) and the
cache entries the forward used are pinned by strong references here (an LRU
eviction then only drops the cache's own reference).  `close()` releases both.
"""

from __future__ import annotations

import numpy as np
import torch

from .network import forward_bicrypto
from .errors import UsageError
from .sim import HeContext


class GraphedForward:
    def __init__(self, net, weights, ctx: HeContext, sens_shape, full_shape, *, strategy: str = "hw",
                 group_size: int | None = None, warmup: int = 2):
        self._frozen = False
        eng = ctx.engine
        self.ctx, self.eng = ctx, eng
        dev = eng.device
        self.sens = torch.zeros(sens_shape, dtype=torch.float64, device=dev)
        self.full = torch.zeros(full_shape, dtype=torch.float64, device=dev)
        self.counter = torch.zeros(1, dtype=torch.int64, device=dev)
        n_img = sens_shape[0]
        # >= ciphertexts encrypted per forward: every input channel, plus the first
        # conv's pre-rotated copies (network._encrypt_channels)
        first = net.cipher_layers[0] if getattr(net, "cipher_layers", None) else None
        taps = first.kernel[0] * first.kernel[1] if first is not None and first.kind == "conv" else 1
        self._ids_per_call = n_img * sens_shape[1] * taps + 1
        eng.graph_counter = self.counter
        try:
            kw = dict(strategy=strategy, group_size=group_size)
            for _ in range(warmup):          # keys, level tables, plaintext cache, scratch size
                self._next_counter()
                r = forward_bicrypto(net, (self.sens, self.full), weights, ctx, **kw)
                eng.decrypt(r.logits_ct.data, r.logits_ct.level, r.logits_ct.scale)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(self.graph, stream=s):
                    res = forward_bicrypto(net, (self.sens, self.full), weights, ctx, **kw)
                    ct = res.logits_ct
                    self.slots = eng.decrypt(ct.data, ct.level, ct.scale)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            eng.freeze(+1)
            self._frozen = True
        finally:
            eng.graph_counter = None
        self._pinned = list(ctx._pt_cache.values())      # every plaintext / plane / key the graph reads
        self.result = res
        idx = np.arange(res.tiles)[:, None] * res.tile_step + np.arange(res.n_outputs)[None, :]
        self._idx = torch.as_tensor(idx.ravel(), device=dev)
        self.n_images = n_img
        self.recorder = res.recorder

    def close(self) -> None:
        """Drop the graph and release the context (arenas may move again)."""
        if getattr(self, "_frozen", False):
            self._frozen = False
            self.graph = None
            self._pinned = []
            self.eng.freeze(-1)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _next_counter(self):
        self.counter.fill_(self.eng.next_counter(self._ids_per_call))

    def __call__(self, sens, full) -> np.ndarray:
        """Run one request: host (or device) inputs -> decrypted logits on the host."""
        self.sens.copy_(torch.as_tensor(sens), non_blocking=True)
        self.full.copy_(torch.as_tensor(full), non_blocking=True)
        if not self._frozen:
            raise UsageError("GraphedForward was closed")
        self._next_counter()
        self.graph.replay()
        return self.slots[:, self._idx].reshape(-1, self.result.n_outputs)[:self.n_images].cpu().numpy()
