"""Discrete-event model of the transfer engine and memory pool — TEST INFRASTRUCTURE.

Restatement of ``swapgraph/sim.py:139-476`` used as the modelled side when
the GPU executor's *measured* report is compared with the schedule model,
and pinned against the reference's own reports (tests/golden/sim_cases).
Model (sim.py:3-27):

* one compute engine per device (one engine overall in serial mode); ready
  ops start in (order, id) order;
* outputs are allocated when an op starts; inputs are released when it
  finishes; a residency is dropped when its refcount reaches zero after it
  completed (consumers, outbound transfers and update commits all hold refs);
* a read of a tensor produced on another device enqueues a transfer when the
  tensor completes at home; per-direction channels or one shared channel;
  the destination is allocated when the transfer starts;
* variables are permanently resident and excluded from peaks; peaks are
  sampled once per instant after it settles;
* transfer_wait_total = sum over ops of (time ready) - (time its origin
  producers / control predecessors finished).
"""

from __future__ import annotations

import heapq
import math


def _val(x):
    return x.value if hasattr(x, "value") else x


class _Res:
    __slots__ = ("refs", "done", "fixed", "nbytes")

    def __init__(self, refs, nbytes, fixed=False):
        self.refs, self.nbytes, self.fixed, self.done = refs, nbytes, fixed, False


class Model:
    """One simulation run; ``run()`` returns the report fields as a dict."""

    def __init__(self, g, order, *, capacity=16 * 2**30, h2d_bw=float(80 * 2**30),
                 d2h_bw=float(80 * 2**30), overlap=True, serial=False):
        self.g, self.order = g, order
        self.capacity, self.h2d_bw, self.d2h_bw = capacity, h2d_bw, d2h_bw
        self.overlap, self.serial = overlap, serial
        self.trace = []
        nbi = g.node_by_id
        live = {n.id for n in g.nodes if n.parameterized}
        stack = list(live)
        while stack:
            for e in g.out_edges(stack.pop()):
                if _val(e.action) != "update" and e.dst not in live:
                    live.add(e.dst)
                    stack.append(e.dst)
        self.ex = {nid for nid in live if not nbi[nid].parameterized}
        for t in g.tensors:
            p = nbi[t.producer]
            if (p.parameterized or t.producer in self.ex) and t.size_bytes <= 0:
                raise ValueError(f"tensor {t.id} participates in simulation but has "
                                 f"size_bytes={t.size_bytes}")
        # consumer counts per tensor and device
        self.reads = {t.id: {} for t in g.tensors}
        self.updates = {t.id: {} for t in g.tensors}
        for e in g.edges:
            if e.tensor is None or e.dst not in nbi:
                continue
            dev = nbi[e.dst].device
            if _val(e.action) == "read" and e.dst in self.ex:
                self.reads[e.tensor][dev] = self.reads[e.tensor].get(dev, 0) + 1
            elif _val(e.action) == "update":
                self.updates[e.tensor][dev] = self.updates[e.tensor].get(dev, 0) + 1

    # -- helpers -------------------------------------------------------------
    def home(self, tid):
        return self.g.node_by_id[self.g.tensor_by_id[tid].producer].device

    def remotes(self, tid):
        h = self.home(tid)
        return sorted((set(self.reads[tid]) | set(self.updates[tid])) - {h})

    def emit(self, time, ev, node=None, tensor=None, nbytes=0, device=None):
        self.trace.append((time, ev, node, tensor, nbytes, device))

    def alloc(self, tid, dev, refs, fixed=False):
        r = _Res(refs, self.g.tensor_by_id[tid].size_bytes, fixed)
        self.res[(tid, dev)] = r
        if not fixed:
            self.used[dev] = self.used.get(dev, 0) + r.nbytes
        return r

    def maybe_free(self, time, tid, dev, trigger):
        r = self.res.get((tid, dev))
        if r is None or r.fixed or r.refs > 0 or not r.done:
            return
        del self.res[(tid, dev)]
        self.used[dev] -= r.nbytes
        self.emit(time, "free", trigger, tid, r.nbytes, dev)

    def origin(self, tid):
        g = self.g
        for _ in range(len(g.nodes) + 1):
            p = g.tensor_by_id[tid].producer
            if _val(g.node_by_id[p].kind) not in ("swap_out", "swap_in"):
                return p
            ins = [e for e in g.in_edges(p) if _val(e.action) == "read"]
            if len(ins) != 1:
                return p
            tid = ins[0].tensor
        return g.tensor_by_id[tid].producer

    def ready_since(self, nid):
        t = 0.0
        for e in self.g.in_edges(nid):
            a = _val(e.action)
            if a == "read":
                t = max(t, self.fin.get(self.origin(e.tensor), 0.0))
            elif a == "control" and e.src in self.ex:
                t = max(t, self.fin.get(e.src, 0.0))
        return t

    def dec(self, time, nid):
        self.pending[nid] -= 1
        if self.pending[nid] == 0:
            self.wait_total += max(0.0, time - self.ready_since(nid))
            heapq.heappush(self.ready, (self.order[nid], nid))

    def push(self, time, kind, payload):
        heapq.heappush(self.events, (time, self.seq, kind, payload))
        self.seq += 1

    def bandwidth(self, dst_dev):
        if self.serial:
            return math.inf
        return self.d2h_bw if dst_dev == "host" else self.h2d_bw

    def enqueue(self, time, tid, src, dst):
        key = "xfer" if not self.overlap else f"{src}->{dst}"
        heapq.heappush(self.chan.setdefault(key, []), (time, tid, dst, self.seq, src))
        self.seq += 1

    def complete_local(self, time, tid, dev):
        g = self.g
        r = self.res[(tid, dev)]
        r.done = True
        for e in g.consumer_edges(tid):
            d = g.node_by_id.get(e.dst)
            if d is None:
                continue
            a = _val(e.action)
            if a == "read" and e.dst in self.ex and d.device == dev:
                if e.dst not in self.done and e.dst not in self.running:
                    self.dec(time, e.dst)
            elif a == "update" and d.device == dev:
                r.refs -= 1
        home = self.home(tid)
        self.maybe_free(time, tid, dev, g.tensor_by_id[tid].producer if dev == home else None)
        if dev == home:
            for rd in self.remotes(tid):
                self.enqueue(time, tid, home, rd)

    def complete_remote(self, time, tid, dev):
        g = self.g
        r = self.res[(tid, dev)]
        r.done = True
        for e in g.consumer_edges(tid):
            d = g.node_by_id.get(e.dst)
            if d is None or d.device != dev:
                continue
            a = _val(e.action)
            if a == "read" and e.dst in self.ex:
                if e.dst not in self.done and e.dst not in self.running:
                    self.dec(time, e.dst)
            elif a == "update":
                r.refs -= 1
        self.maybe_free(time, tid, dev, None)

    def start_transfers(self, time):
        moved = False
        for key in sorted(self.chan):
            q = self.chan[key]
            while q and self.chan_free.get(key, 0.0) <= time:
                _, tid, dst, _, src = heapq.heappop(q)
                size = self.g.tensor_by_id[tid].size_bytes
                bw = self.bandwidth(dst)
                dur = 0.0 if math.isinf(bw) else size / bw
                self.alloc(tid, dst, self.reads[tid].get(dst, 0) + self.updates[tid].get(dst, 0))
                self.emit(time, "alloc", None, tid, size, dst)
                self.emit(time, "xfer_start", None, tid, size, dst)
                self.chan_free[key] = time + dur
                self.xfer_total += dur
                self.push(time + dur, "x", (tid, src, dst))
                moved = True
        return moved

    def start_nodes(self, time):
        g = self.g
        moved = False
        later = []
        while self.ready:
            item = heapq.heappop(self.ready)
            nid = item[1]
            eng = "serial" if self.serial else g.node_by_id[nid].device
            if self.engine_free.get(eng, 0.0) > time:
                later.append(item)
                continue
            n = g.node_by_id[nid]
            self.running.add(nid)
            self.emit(time, "start", nid, None, 0, n.device)
            for t in g.produced_tensors(nid):
                refs = (self.reads[t.id].get(n.device, 0) + self.updates[t.id].get(n.device, 0)
                        + len(self.remotes(t.id)))
                self.alloc(t.id, n.device, refs)
                self.emit(time, "alloc", nid, t.id, t.size_bytes, n.device)
            self.engine_free[eng] = time + n.cost_hint
            self.push(time + n.cost_hint, "n", nid)
            moved = True
        for item in later:
            heapq.heappush(self.ready, item)
        return moved

    def finish_node(self, time, nid):
        g = self.g
        n = g.node_by_id[nid]
        self.running.discard(nid)
        self.done.add(nid)
        self.fin[nid] = time
        self.emit(time, "finish", nid, None, 0, n.device)
        for e in g.in_edges(nid):
            if _val(e.action) != "read":
                continue
            p = g.node_by_id[g.tensor_by_id[e.tensor].producer]
            if p.parameterized and p.device == n.device:
                continue
            r = self.res.get((e.tensor, n.device))
            if r is not None and not r.fixed:
                r.refs -= 1
                self.maybe_free(time, e.tensor, n.device, nid)
        for e in g.out_edges(nid):
            if _val(e.action) == "control" and e.dst in self.ex:
                if e.dst not in self.done and e.dst not in self.running:
                    self.dec(time, e.dst)
        for t in g.produced_tensors(nid):
            self.complete_local(time, t.id, n.device)

    def finish_xfer(self, time, tid, src, dst):
        self.emit(time, "xfer_finish", None, tid, self.g.tensor_by_id[tid].size_bytes, dst)
        r = self.res.get((tid, src))
        if r is not None and not r.fixed:
            r.refs -= 1
            self.maybe_free(time, tid, src, None)
        self.complete_remote(time, tid, dst)

    def run(self):
        g = self.g
        self.res, self.used, self.peak = {}, {}, {}
        self.events, self.seq = [], 0
        self.chan, self.chan_free, self.engine_free = {}, {}, {}
        self.xfer_total = self.wait_total = 0.0
        self.fin, self.done, self.running = {}, set(), set()
        self.pending = {}
        for nid in self.ex:
            n = g.node_by_id[nid]
            c = 0
            for e in g.in_edges(nid):
                a = _val(e.action)
                if a == "read":
                    p = g.node_by_id[g.tensor_by_id[e.tensor].producer]
                    if not (p.parameterized and p.device == n.device):
                        c += 1
                elif a == "control" and e.src in self.ex:
                    c += 1
            self.pending[nid] = c
        self.ready = []
        for n in g.nodes:
            if not n.parameterized:
                continue
            for t in g.produced_tensors(n.id):
                self.alloc(t.id, n.device, 0, fixed=True).done = True
                for rd in self.remotes(t.id):
                    self.enqueue(0.0, t.id, n.device, rd)
        for nid in sorted(self.ex):
            if self.pending[nid] == 0:
                heapq.heappush(self.ready, (self.order[nid], nid))
        time = makespan = 0.0
        while True:
            while True:
                moved = False
                while self.events and self.events[0][0] <= time:
                    _, _, kind, payload = heapq.heappop(self.events)
                    if kind == "n":
                        self.finish_node(time, payload)
                    else:
                        self.finish_xfer(time, *payload)
                    moved = True
                moved |= self.start_nodes(time)
                moved |= self.start_transfers(time)
                if not moved:
                    break
            for dev, used in self.used.items():
                if used > self.peak.get(dev, 0):
                    self.peak[dev] = used
            makespan = max(makespan, time)
            if not self.events:
                break
            time = self.events[0][0]
        if self.done != self.ex:
            raise RuntimeError("simulation stalled; blocked: " + str(sorted(self.ex - self.done)[:8]))
        dev_peak = max((v for d, v in self.peak.items() if d.startswith("acc:")), default=0)
        return {
            "peak_device_bytes": dev_peak,
            "peak_host_bytes": self.peak.get("host", 0),
            "makespan": makespan,
            "transfer_time_total": self.xfer_total,
            "transfer_wait_total": self.wait_total,
            "oom": dev_peak > self.capacity,
            "event_trace": [dict(time=t, event=ev, node=nd, tensor=tn, bytes=b, device=dv)
                            for t, ev, nd, tn, b, dv in self.trace],
        }


def simulate(g, order, *, capacity=16 * 2**30, h2d_bw=float(80 * 2**30), d2h_bw=float(80 * 2**30),
             overlap=True, serial=False):
    return Model(g, order, capacity=capacity, h2d_bw=h2d_bw, d2h_bw=d2h_bw, overlap=overlap,
                 serial=serial).run()
