"""Host-resident fields through the device engine with the transfers hidden.

A caller holding many fields in host memory (a batch of trial states of a line
search or a multi-start minimisation, an ensemble of load cases) evaluates
J and grad J (gradients.py:124-149 + assembly.py:94-106) for each of them.
Serially, one evaluation is H2D(v) -> kernel -> D2H(g): at config 4 that is
103 MB in, 1.5 ms of kernel, 103 MB out, with the PCIe copies dominating.
``FieldStream`` keeps ``depth`` device slots and puts the three phases on
three streams, so that field i+1's upload, field i's kernel and field i-1's
download run at the same time (PCIe is full duplex; the copy engines do not
compete with the kernel for SMs).  Every field is still copied in full and
every result is copied back: this is a throughput schedule, not a cache.

Ordering per slot k (events, no host synchronisation):
    upload   waits  kernel(k) of the previous round   (v slot free)
    kernel   waits  upload(k), download(k) of the previous round (g slot free)
    download waits  kernel(k)
With an ``exchange`` (parallel.SlabExchange) the slab reduction runs on the
compute stream right after the kernel, as in the serial path.

Host buffers must be pinned (``torch.empty(..., pin_memory=True)``) for the
copies to be asynchronous; a result buffer may be read after ``wait(ticket)``.
Inadmissible states latch in the context exactly as in the serial path and
raise at ``wait`` / ``synchronize`` (models.py:107-110).
"""

from __future__ import annotations

import torch


class FieldStream:
    def __init__(self, dm, model, b=None, depth: int = 2, exchange=None, with_J: bool = True):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.dm, self.model, self.b, self.exchange = dm, model, b, exchange
        self.depth = int(depth)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.compute = torch.cuda.current_stream(dev)
        self.up = torch.cuda.Stream(dev)
        self.down = torch.cuda.Stream(dev)
        nv = dm.nn * dm.d
        self.v = [torch.empty(nv, dtype=torch.float64, device=dev) for _ in range(depth)]
        self.g = [torch.empty(dm.nfree_dofs, dtype=torch.float64, device=dev)
                  for _ in range(depth)]
        self.J = [torch.empty(3, dtype=torch.float64, device=dev) if with_J else None
                  for _ in range(depth)]
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]  # noqa: E731
        self.uploaded, self.computed, self.downloaded = ev(), ev(), ev()
        self.used = [False] * depth
        self.n = 0

    def submit(self, v_host: torch.Tensor, g_host: torch.Tensor, J_host=None) -> int:
        """Queue one evaluation; returns a ticket for ``wait``."""
        if v_host.numel() != self.v[0].numel() or g_host.numel() != self.g[0].numel():
            raise ValueError("field / gradient buffer sizes do not match the mesh")
        k = self.n % self.depth
        first = not self.used[k]
        with torch.cuda.stream(self.up):
            if not first:
                self.up.wait_event(self.computed[k])
            self.v[k].copy_(v_host.reshape(-1), non_blocking=True)
            self.uploaded[k].record(self.up)
        self.compute.wait_event(self.uploaded[k])
        if not first:
            self.compute.wait_event(self.downloaded[k])
        self.dm.exact_gradient(self.v[k], self.model, self.b, g=self.g[k], J=self.J[k])
        if self.exchange is not None:
            self.exchange.reduce(self.g[k], self.J[k])
        self.computed[k].record(self.compute)
        with torch.cuda.stream(self.down):
            self.down.wait_event(self.computed[k])
            g_host.reshape(-1).copy_(self.g[k], non_blocking=True)
            if J_host is not None and self.J[k] is not None:
                J_host.reshape(-1).copy_(self.J[k], non_blocking=True)
            self.downloaded[k].record(self.down)
        self.used[k] = True
        ticket = self.n
        self.n += 1
        return ticket

    def wait(self, ticket: int):
        """Block until field ``ticket``'s results are in its host buffers."""
        # the slot's event is this ticket's download or a later one on the same
        # (in-order) download stream
        self.downloaded[ticket % self.depth].synchronize()

    def synchronize(self):
        """Wait for everything queued; raise for latched inadmissible states."""
        for k in range(self.depth):
            if self.used[k]:
                self.downloaded[k].synchronize()
        self.dm.check()

    def map(self, fields, grads, Js=None):
        """Evaluate every field of ``fields`` into ``grads`` (and ``Js``)."""
        for i, (v, g) in enumerate(zip(fields, grads)):
            self.submit(v, g, None if Js is None else Js[i])
        self.synchronize()
