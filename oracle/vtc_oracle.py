"""ORACLE — Virtual Token Counter (VTC) fair scheduling, restated on the CPU.

Test infrastructure only: imported by tests/ and oracle/gen_golden.py, never
by the product (paper_2411_18424_b200/) or bench.py's measured legs.

The reference has no fairness policy: priorities are offline trace inputs
(/root/reference/pkg/src/kvswitch/scheduler.py:47-90) and VTC is listed as
related work only.  BASELINE
config 3 names "fairness-aware (VTC priority) preemption", so this module
restates the published algorithm — Sheng et al., "Fairness in Serving Large
Language Models", OSDI'24, Algorithm 2 — from the paper (no code of it is
vendored in /root/reference; no third-party dependency is involved):

  monitoring stream — request r of client u arrives:
      if u is not backlogged:
          if nobody is backlogged:  c_u <- max(c_u, l)      l = counter of the
          else:                     c_u <- max(c_u, min_{i backlogged} c_i)
                                                             last client to leave
  execution stream — while a request can be added:
      k <- argmin_{i with queued requests} c_i
      admit k's earliest queued request r;  c_k <- c_k + w_p * r.n_input
  after each decode step:  c_i <- c_i + w_q * (tokens generated for client i)

with the weighted-token cost h(n_p, n_q) = w_p n_p + w_q n_q, w_p = 1, w_q = 2.
The paper's fairness bound: for backlogged clients the counters stay within
U = max(w_p * L_input, w_q * M) of each other (M = batch token capacity), so
two continuously backlogged clients' service differs by at most 2U.

Two uses:

  * `paper_server` — the paper's own setting (a continuous-batching server
    with a token-capacity batch, no preemption), for the bound property and a
    call-for-call check of the product's counter primitives;
  * `vtc_reference_engine` — the UNMODIFIED reference Engine
    (kvswitch/engine.py) with VTC supplying its priorities at the engine's
    own hook points: turn arrival (engine.py:285-307, the mid-epoch
    insertion), the priority epoch (engine.py:386-393, via the module-level
    apply_priority_update), scheduling (engine.py:558), token emission
    (engine.py:740-762) and turn end (engine.py:765).  Everything else —
    allocation, planning, swapping, the clock — is the reference's, so the
    golden reports it records pin config 3's preemption / resume decisions.
"""

from __future__ import annotations

from typing import Iterable

W_PROMPT = 1
W_OUTPUT = 2


class VTC:
    """Algorithm 2's counter state; integer arithmetic."""

    def __init__(self, wp: int = W_PROMPT, wq: int = W_OUTPUT) -> None:
        self.wp = wp
        self.wq = wq
        self.c: dict = {}
        self.l = 0

    def counter(self, u) -> int:
        return self.c[u] if u in self.c else 0

    def arrive(self, u, backlog: Iterable) -> None:
        """u becomes backlogged while `backlog` (excluding u) already is."""
        others = [self.counter(i) for i in backlog if i != u]
        lift = min(others) if others else self.l
        self.c[u] = max(self.counter(u), lift)

    def depart(self, u) -> None:
        self.l = self.counter(u)

    def serve(self, u, prompt: int = 0, output: int = 0) -> None:
        self.c[u] = self.counter(u) + self.wp * prompt + self.wq * output

    def pick(self, candidates: Iterable):
        """argmin counter, ties to the smallest id."""
        best = None
        for u in candidates:
            if best is None or (self.counter(u), u) < (self.counter(best), best):
                best = u
        return best

    def order(self, clients: Iterable) -> list:
        pool = list(clients)
        out = []
        while pool:
            u = self.pick(pool)
            out.append(u)
            pool.remove(u)
        return out


# --------------------------------------------------------------- paper setting

def paper_server(requests, capacity: int, steps: int, wp: int = W_PROMPT,
                 wq: int = W_OUTPUT, vtc_factory=None):
    """Continuous batching under VTC (Alg. 2), no preemption.

    requests: iterable of (arrival_step, client, n_input, n_output).  A batch
    holds requests whose KV tokens (input + generated so far, + the token
    being generated) fit in `capacity`.  Returns (trace, vtc) where trace has
    one entry per step: (step, {client: counter} over backlogged clients,
    admitted [(client, request index)], served {client: output tokens}).
    `vtc_factory(wp, wq)` substitutes another counter implementation with
    VTC's interface (tests drive the product's primitives through it).
    """
    vtc = (vtc_factory or VTC)(wp, wq)
    pending = sorted((a, i, u, n_in, n_out) for i, (a, u, n_in, n_out) in enumerate(requests))
    queue: dict = {}  # client -> [request index] in arrival order
    reqs = {}
    running: dict = {}  # request index -> generated
    trace = []
    p = 0
    for step in range(steps):
        while p < len(pending) and pending[p][0] <= step:
            _, i, u, n_in, n_out = pending[p]
            p += 1
            reqs[i] = (u, n_in, n_out)
            if u not in queue:
                vtc.arrive(u, list(queue))
                queue[u] = []
            queue[u].append(i)
        used = sum(reqs[i][1] + g + 1 for i, g in running.items())
        admitted = []
        while queue:
            k = vtc.pick(queue)
            i = queue[k][0]
            need = reqs[i][1] + 1
            if used + need > capacity:
                break
            queue[k].pop(0)
            if not queue[k]:
                del queue[k]
                vtc.depart(k)
            running[i] = 0
            used += need
            vtc.serve(k, prompt=reqs[i][1])
            admitted.append((k, i))
        served: dict = {}
        for i in sorted(running):
            running[i] += 1
            u = reqs[i][0]
            served[u] = served.get(u, 0) + 1
        for u in sorted(served):
            vtc.serve(u, output=served[u])
        for i in [i for i, g in running.items() if g >= reqs[i][2]]:
            del running[i]
        trace.append((step, {u: vtc.counter(u) for u in queue}, admitted, served))
    return trace, vtc


def fairness_bound(wp: int, wq: int, max_input: int, capacity: int) -> int:
    """U = max(w_p * L_input, w_q * M) (Sheng et al., Thm. on VTC's bound)."""
    return max(wp * max_input, wq * capacity)


# --------------------------------------------------------------- reference hook

LIVE = ("waiting", "running", "swapped", "ongoing_swap_in")
QUEUED = ("waiting", "swapped")


def vtc_reference_engine(engine_module, wp: int = W_PROMPT, wq: int = W_OUTPUT):
    """Subclass of the reference Engine whose priorities come from VTC.

    Build its config with a priority pattern the reference accepts ("markov"):
    only the trace's epoch period is used; the pattern's own permutation is
    never drawn (apply_priority_update is replaced for the run)."""
    Ref = engine_module.Engine

    class VtcReferenceEngine(Ref):
        def __init__(self, config, conversations, **kw) -> None:
            super().__init__(config, conversations, **kw)
            self.vtc = VTC(wp, wq)

        def run(self):
            saved = engine_module.apply_priority_update

            def epoch_update(epoch, trace, live, running):
                return {u: k for k, u in enumerate(self.vtc.order(sorted(live)))}

            engine_module.apply_priority_update = epoch_update
            try:
                return super().run()
            finally:
                engine_module.apply_priority_update = saved

        def _begin_turn(self, req, arrival) -> None:
            before = dict(self.ranks)
            super()._begin_turn(req, arrival)  # its seeded slot is per-turn; no shared RNG
            backlog = [r for r, st in self.states.items() if st.phase in LIVE and r != req]
            self.vtc.arrive(req, backlog)
            self.ranks.clear()
            self.ranks.update(before)
            self.ranks[req] = 1 + max(before.values()) if before else 0
            self.store.update_ranks(self.ranks)

        def _schedule(self):
            queued = [r for r, st in self.states.items() if st.phase in QUEUED and r in self.ranks]
            slots = sorted(self.ranks[r] for r in queued)
            for slot, r in zip(slots, self.vtc.order(queued)):
                self.ranks[r] = slot
            self.store.update_ranks(self.ranks)
            return super()._schedule()

        def _emit_tokens(self, prefillers, decoders, end):
            before = {r: (self.states[r].pending_input, self.states[r].remaining_output)
                      for r in list(prefillers) + list(decoders)}
            n = super()._emit_tokens(prefillers, decoders, end)
            pset = set(prefillers)
            for r, (pin, rem) in before.items():
                self.vtc.serve(r, prompt=pin if r in pset else 0,
                               output=rem - self.states[r].remaining_output)
            return n

        def _finish_turn(self, req) -> None:
            self.vtc.depart(req)
            super()._finish_turn(req)

    return VtcReferenceEngine


def reference_doc(doc: dict) -> tuple[dict, int, int]:
    """A config document the reference accepts, plus the VTC weights."""
    import copy

    ref = copy.deepcopy(doc)
    tr = ref.setdefault("trace", {})
    wp = tr.pop("vtc_wp", W_PROMPT)
    wq = tr.pop("vtc_wq", W_OUTPUT)
    if tr.get("pattern") == "vtc":
        tr["pattern"] = "markov"
    return ref, wp, wq


__all__ = ["VTC", "paper_server", "fairness_bound", "vtc_reference_engine", "reference_doc",
           "W_PROMPT", "W_OUTPUT"]
