"""vLLM weight loading through this loader (the paper's own application:
model-server startup).

vLLM's ``--load-format fastsafetensors`` iterates over the checkpoint with
upstream fastsafetensors (vllm/model_executor/model_loader/weight_utils.py,
``fastsafetensors_weights_iterator``): groups of files, one per rank,
``get_tensor`` per key, yielding ``(name, tensor)`` pairs that the model's
weight loaders copy into their parameters. :func:`weights_iterator` is the
same contract over the B200 path: every file of the rank lands in HBM through
the C++ engine in one plan, each key is a zero-copy CUDA view (``auto_release``
off: vLLM copies the tensor before asking for the next), and the landed
buffers are released when the iteration ends. :func:`install` points vLLM's
fastsafetensors load format at it (run the engine in-process:
``VLLM_ENABLE_V1_MULTIPROCESSING=0``, or call it in the worker).
"""

from __future__ import annotations

from collections.abc import Iterator

import torch

from .collective import DistGroup, SingleGroup
from .loader import LoaderConfig, SafeTensorsFileLoader

__all__ = ["weights_iterator", "install"]


def weights_iterator(hf_weights_files: list[str], use_tqdm_on_load: bool = False) -> Iterator[tuple[str, torch.Tensor]]:
    """``(name, tensor)`` for every tensor of the checkpoint, tensors on the
    current CUDA device. Under torch.distributed the files are spread over the
    ranks (file i -> rank i mod W) and every rank receives every tensor."""
    import re

    def natural(s: str):
        return [int(t) if t.isdigit() else t for t in re.split(r"(\d+)", s)]

    files = sorted(hf_weights_files, key=natural)
    dist = torch.distributed.is_available() and torch.distributed.is_initialized()
    device = torch.device("cuda", torch.cuda.current_device())
    group = DistGroup(device=device) if dist else SingleGroup()
    world = group.world_size
    loader = SafeTensorsFileLoader(group, device, config=LoaderConfig(auto_release=False))
    try:
        loader.add_filenames({r: [f for i, f in enumerate(files) if i % world == r] for r in range(world)})
        fb = loader.copy_files_to_device()
        try:
            for key in fb.keys():
                yield key, fb.get_tensor(key).torch
        finally:
            torch.cuda.current_stream(device).synchronize()  # consumers' copies are done
            fb.close()
    finally:
        loader.close()


def install() -> None:
    """Route vLLM's ``load_format="fastsafetensors"`` through :func:`weights_iterator`."""
    from vllm.model_executor.model_loader import default_loader, weight_utils

    weight_utils.fastsafetensors_weights_iterator = weights_iterator
    default_loader.fastsafetensors_weights_iterator = weights_iterator
