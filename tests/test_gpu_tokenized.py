"""§8f-4: client tokenized mode on the device vs the reference's
``ChunkStreamer.tokenized`` (client.py:451-506) on the same files and chunks.

The reference registers JSON-lines files, builds the index and generates
chunks; for every chunk its ChunkStreamer reads the records and packs
tokens with the reference tokenizers. The device path tokenizes every record
once (TokenStore) and packs each chunk in one kernel: the sequences (tokens
and per-token key tags) must be identical, and the tags must feed
per_domain_loss (stage 3) with the same per-key sums as the reference's
per_domain_loss over the TokenBatchItems."""

from __future__ import annotations

import json
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def mp():
    if not (REF / "mixplane").exists():
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, str(REF))
    import mixplane

    return mixplane


WORDS = ["alpha", "beta", "γάμμα", "δ", "日本", "naïve", "x", "quote\"d", "back\\slash", "tab\tbed", "nl\nx",
         "emoji😀", "nbsp sep", "ideo　sep", "fs\x1csep", "", "  lead", "trail  "]


def _text(rng):
    k = int(rng.integers(0, 12))
    return " ".join(str(rng.choice(WORDS)) for _ in range(k))


def _corpus(tmp_path, seed=4, files=5):
    rng = np.random.default_rng(seed)
    paths = []
    for f in range(files):
        lines, cur = [], None
        for i in range(int(rng.integers(200, 500))):
            if cur is None or rng.random() < 0.1:
                cur = {"language": str(rng.choice(["py", "go", "rs"])), "src": str(rng.choice(["web", "book"]))}
            rec = dict(cur)
            r = rng.random()
            if r < 0.05:
                pass                                   # no text field: ""
            elif r < 0.1:
                rec["text"] = ""                       # empty: skipped
            else:
                rec["text"] = _text(rng)
            if rng.random() < 0.05:
                rec["text2"] = {"text": "nested, not top level"}
            lines.append(json.dumps(rec, ensure_ascii=bool(rng.random() < 0.5)))
        path = tmp_path / f"t{f}.jsonl"
        path.write_text("\n".join(lines) + "\n", encoding="utf-8")
        paths.append(path)
    return paths


@pytest.mark.parametrize("tok", ["byte", "whitespace"])
def test_tokenized_mode_matches_the_reference(mp, tmp_path, tok):
    import torch

    from paper_2502_19790_b200 import per_domain_loss
    from paper_2502_19790_b200.chunks import Chunk
    from paper_2502_19790_b200.tokenized import TokenStore, tokenized
    from mixplane.client import ChunkStreamer, ResultStreamingArgs, StreamStats
    from mixplane.client import per_domain_loss as ref_pdl

    paths = _corpus(tmp_path)
    props = ["language", "src"]
    cat = mp.MetadataCatalog()
    cat.register_dataset("d", paths, mp.JsonFieldParser.for_properties(props),
                         mp.PropertySchema([mp.PropertyDef(p) for p in props]))
    fids = sorted(cat._files)
    files = {f: cat._files[f].path for f in fids}
    store = TokenStore.build([files[f] for f in fids], file_ids=fids, text_field="text", tokenizer=tok)
    spec = mp.MixtureSpec({mp.MixtureKey.of({"language": "py"}): 0.5, mp.MixtureKey.of({"src": "book"}): 0.3,
                           mp.MixtureKey.of({"language": ["go", "rs"], "src": "web"}): 0.2}, 96)
    gen = mp.ChunkGenerator(mp.build_index(cat.filter_intervals([])), 42)
    tokenizer = mp.get_tokenizer(tok)
    n_seq = 0
    for L in ((7, 16) if tok == "byte" else (2, 3)):  # whitespace: ~5 tokens per sample
        for c in range(6):
            chunk = gen.generate(spec)
            if chunk is None:
                break
            args = ResultStreamingArgs(job_id="j", mode="tokenized", sequence_length=L, text_field="text",
                                       tokenizer=tok)
            want = list(ChunkStreamer(chunk, files, args, StreamStats(), tokenizer=tokenizer).tokenized())
            ours = Chunk.deserialize(chunk.serialize())
            toks, tags, keys = tokenized(ours, store, L)
            assert toks.shape == (len(want), L)
            assert toks.cpu().numpy().tolist() == [w.tokens for w in want]
            ks = [k.canonical_string() for k in keys]
            assert [[ks[t] for t in row] for row in tags.cpu().numpy().tolist()] == \
                [[k.canonical_string() for k in w.tags] for w in want]
            n_seq += len(want)
            if want:  # stage 3: the packed tags are per_domain_loss's domain ids
                rng = np.random.default_rng(c)
                losses = rng.gamma(5.0, 0.2, size=len(want) * L).astype(np.float32)
                ref = ref_pdl(losses.tolist(), [k for w in want for k in w.tags])
                got = per_domain_loss(torch.from_numpy(losses).cuda(), tags.flatten(), keys)
                for k, (s, n) in ref.items():
                    gs, gn = got[keys[ks.index(k.canonical_string())]]
                    assert gn == n and abs(gs - s) <= 1e-9 * max(1.0, abs(s))
    assert n_seq > 20
    assert store.n_records == sum(cat._files[f].n_samples for f in fids)
