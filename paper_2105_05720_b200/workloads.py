"""Synthetic workloads named by BASELINE.json's configs (shapes only; values
are generated on the device, see collectives.gen_values)."""
from __future__ import annotations


def bert_large_param_shapes(vocab: int = 30528, hidden: int = 1024, ffn: int = 4096,
                            layers: int = 24, max_pos: int = 512, types: int = 2):
    """BERT-large (336M) parameter tensors in the usual order: 398 tensors,
    336,232,258 elements. Decoder weight tied to the word
    embedding, so only its bias appears."""
    H = hidden
    shapes = [("embeddings.word", (vocab, H)), ("embeddings.position", (max_pos, H)),
              ("embeddings.token_type", (types, H)), ("embeddings.ln.weight", (H,)),
              ("embeddings.ln.bias", (H,))]
    for i in range(layers):
        p = f"layer{i}."
        shapes += [(p + "attn.q.weight", (H, H)), (p + "attn.q.bias", (H,)),
                   (p + "attn.k.weight", (H, H)), (p + "attn.k.bias", (H,)),
                   (p + "attn.v.weight", (H, H)), (p + "attn.v.bias", (H,)),
                   (p + "attn.out.weight", (H, H)), (p + "attn.out.bias", (H,)),
                   (p + "attn.ln.weight", (H,)), (p + "attn.ln.bias", (H,)),
                   (p + "ffn.in.weight", (ffn, H)), (p + "ffn.in.bias", (ffn,)),
                   (p + "ffn.out.weight", (H, ffn)), (p + "ffn.out.bias", (H,)),
                   (p + "ffn.ln.weight", (H,)), (p + "ffn.ln.bias", (H,))]
    shapes += [("pooler.weight", (H, H)), ("pooler.bias", (H,)),
               ("mlm.transform.weight", (H, H)), ("mlm.transform.bias", (H,)),
               ("mlm.ln.weight", (H,)), ("mlm.ln.bias", (H,)), ("mlm.decoder.bias", (vocab,)),
               ("nsp.weight", (2, H)), ("nsp.bias", (2,))]
    return shapes


def numel(shape) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n


def bert_large_counts():
    return [numel(s) for _, s in bert_large_param_shapes()]


BERT_LARGE_TENSORS = 398
BERT_LARGE_PARAMS = 336_232_258
