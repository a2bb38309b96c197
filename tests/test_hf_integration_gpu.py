"""Drop-in use: a HuggingFace Llama model filled from this loader's tensors
gives bit-identical logits to the same model filled by safetensors' own
loader (a 2-block Llama-2-7B-shaped checkpoint, bf16)."""

from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup, synth  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ckpt(tmp_path_factory):
    d = tmp_path_factory.mktemp("hf")
    return synth.generate("llama2-7b", d, layers=2, device="cuda", max_bytes=600_000_000)


def _model():
    cfg = transformers.LlamaConfig(hidden_size=4096, intermediate_size=11008, num_hidden_layers=2,
                                   num_attention_heads=32, num_key_value_heads=32, vocab_size=32000,
                                   max_position_embeddings=256, tie_word_embeddings=False)
    torch.manual_seed(0)
    with torch.device("cuda"):
        m = transformers.LlamaForCausalLM(cfg).to(torch.bfloat16)
    return m.eval()


@pytest.mark.parametrize("batched", [False, True])
def test_llama_logits_match_safetensors(ckpt, batched):
    from safetensors.torch import load_file

    assert len(ckpt) > 1  # several files: keys gathered across them
    loader = SafeTensorsFileLoader(SingleGroup(), "cuda:0", config=LoaderConfig(auto_release=True))
    loader.add_filenames({0: [str(p) for p in ckpt]})
    fb = loader.copy_files_to_device()
    keys = fb.keys()
    views = fb.get_tensors(keys) if batched else {k: fb.get_tensor(k) for k in keys}
    ours = {k: v.torch for k, v in views.items()}
    fb.close()  # auto-release outputs outlive the file buffers
    loader.close()

    ref = {}
    for p in ckpt:
        ref.update(load_file(str(p), device="cuda:0"))
    assert set(ours) == set(ref)
    for k in ref:
        assert ours[k].dtype == ref[k].dtype and ours[k].shape == ref[k].shape
        assert torch.equal(ours[k].view(torch.int16), ref[k].view(torch.int16)), k

    tokens = torch.randint(0, 32000, (2, 16), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    with torch.no_grad():
        m = _model()
        m.load_state_dict(ours, strict=True)
        a = m(tokens).logits
        m.load_state_dict(ref, strict=True)
        b = m(tokens).logits
    assert torch.isfinite(a).all()
    assert torch.equal(a, b)


def test_vllm_weights_iterator_matches_safetensors(ckpt):
    """The vLLM load-format hook yields every (name, tensor) of the
    checkpoint on the GPU, bit-identical to safetensors."""
    from safetensors.torch import load_file

    from paper_2505_23072_b200.vllm_loader import weights_iterator

    ref = {}
    for p in ckpt:
        ref.update(load_file(str(p), device="cuda:0"))
    seen = {}
    for name, t in weights_iterator([str(p) for p in ckpt]):
        assert t.is_cuda and t.dtype == ref[name].dtype and t.shape == ref[name].shape
        seen[name] = torch.equal(t.view(torch.int16), ref[name].view(torch.int16))
    assert set(seen) == set(ref) and all(seen.values())
