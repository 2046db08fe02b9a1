"""CUDA-graph execution of a whole hot-path step (host plumbing only; every node is a libencf launch).

A BERT-layer step is ~3000 launches from the batched evaluator; enqueuing them eagerly costs ~100 ms of
host time, as much as the device time.  The C ABI is stream-capturable once a warm-up call has filled the
mask cache (include/encf.h, encf_profile_peek), so the step is captured ONCE into a CUDA graph and
replayed: static device inputs, static outputs, one graph launch per step.
"""
import torch


class GraphedStep:
    """Capture ``fn(inputs)`` into a CUDA graph; ``__call__`` replays it.

    ``inputs`` is a dict of lists of device Ciphertexts (their tensors are the graph's static input
    buffers); ``fn`` must have been run eagerly once on inputs of the same shapes (mask-cache warm-up).
    ``outputs`` holds the objects ``fn`` returned during capture; every replay rewrites their tensors.
    """

    def __init__(self, fn, inputs, pool=None):
        self.inputs = inputs
        self.graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(self.graph, pool=pool):
            self.outputs = fn(inputs)
        torch.cuda.synchronize()

    def load(self, host_inputs):
        """Asynchronous H2D copy of a step's inputs (pinned host words, same layout) into the static buffers."""
        for k, hs in host_inputs.items():
            for dst, h in zip(self.inputs[k], hs):
                dst.data.copy_(h, non_blocking=True)

    def __call__(self, host_inputs=None):
        if host_inputs is not None:
            self.load(host_inputs)
        self.graph.replay()
        return self.outputs


class PipelinedStep:
    """Two CUDA graphs of the same step on two static input sets (A, B), replayed alternately, so the H2D copy of
    step i+1's inputs (one side stream) and the D2H copy of step i's exports (another side stream) overlap step i's
    device work.  Ordering by events: a set's inputs are rewritten only after the graph that last read them has
    finished, a graph starts only after its inputs have landed and after its previous exports have been copied out.
    The exports' mask state is one device buffer advanced inside both graphs (every replay draws fresh pads)."""

    def __init__(self, fn, step_a, inputs_b):
        """``step_a``: an existing GraphedStep of ``fn`` (set A); set B is captured here on ``inputs_b``, sharing A's
        memory pool: the two graphs replay one after the other on one stream, and each one's outputs (read by the
        D2H stream while the other runs) stay live tensors, so only intermediates are shared."""
        self.g = [step_a, GraphedStep(fn, inputs_b, pool=step_a.graph.pool())]
        self.s_in = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()

    def run(self, host_inputs, host_outs, steps):
        """``steps`` steps on the current stream; every step copies ``host_inputs`` (pinned, same layout as the
        static inputs) in and its exports out to ``host_outs[set]`` = list of (pinned words, pinned share or None)."""
        comp = torch.cuda.current_stream()
        done = [None, None]      # graph of set b finished (its inputs may be rewritten)
        copied = [None, None]    # exports of set b copied out (its outputs may be rewritten)
        landed = [None, None]

        def load(b):
            self.s_in.wait_stream(comp) if done[b] is None else self.s_in.wait_event(done[b])
            with torch.cuda.stream(self.s_in):
                self.g[b].load(host_inputs)
                landed[b] = torch.cuda.Event()
                landed[b].record(self.s_in)

        load(0)
        for i in range(steps):
            b = i % 2
            comp.wait_event(landed[b])
            if copied[b] is not None:
                comp.wait_event(copied[b])
            self.g[b].graph.replay()
            done[b] = torch.cuda.Event()
            done[b].record(comp)
            if i + 1 < steps:
                load(1 - b)
            self.s_out.wait_event(done[b])
            with torch.cuda.stream(self.s_out):
                for (m, sh), (hm, hs) in zip(self.g[b].outputs, host_outs[b]):
                    hm.copy_(m.data, non_blocking=True)
                    if sh is not None:
                        hs.copy_(sh, non_blocking=True)
                copied[b] = torch.cuda.Event()
                copied[b].record(self.s_out)
        comp.wait_stream(self.s_out)
        comp.wait_stream(self.s_in)
