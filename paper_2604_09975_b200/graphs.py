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

    def __init__(self, fn, inputs):
        self.inputs = inputs
        self.graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(self.graph):
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
