"""Metadata registration on the GPU.

``DeviceMetadataCatalog.register_dataset(name, files, parser, schema)`` has
the reference's signature, checks and errors
(``MetadataCatalog.register_dataset``, ``catalog.py:323-435``) and produces
the stage-1 input directly in HBM: one int32 code column per property over
all samples of all files (``ColumnarCatalog`` layout), without parsing the
records in Python.

Pipeline per dataset:

1. the files' bytes are read into one pinned buffer (each file newline-
   terminated, padded to 16 bytes), hashed for re-registration checks
   (``_hash_file``) and copied to the device;
2. ``mx_jsonl_records`` (``csrc/register.cu``) finds the records -- the
   non-empty lines, in file order, as ``iter_records`` yields them;
3. ``mx_jsonl_extract`` validates every record as JSON on the device and
   returns, per requested field, the NORMALISED value
   (``_normalize_values``) as a 128-bit hash, its distinct element count and
   its byte span; records outside the device fast path are flagged;
4. interning: per property the distinct hashes (``torch.unique`` on the
   device), the value strings of each from ONE representative record's span,
   codes in first-appearance order, the code column by a gather;
5. errors: every record that may raise (flagged records, a missing
   non-nullable property, several values for a single-valued property, a
   value outside a categorical property's categories, a parser field that is
   not in the schema) is evaluated with the reference semantics in record
   order -- ``json.loads``, ``parser.parse``, ``_normalize_values`` -- so the
   first failure raises exactly the reference's exception and message; the
   flagged records that pass contribute their values.

Scope: JSON-lines files read with the reference's ``JsonFieldParser`` (a
parser exposing ``fields``); zstd-compressed files are not decoded on the
device (``NotImplementedError``).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
from pathlib import Path
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from .catalog import ColumnarCatalog
from .errors import DataReadError, RegistrationError, SchemaError

JSONL_SUFFIX = ".jsonl"
ZST_SUFFIX = ".jsonl.zst"


def normalize_values(prop, raw: object, where: str) -> tuple[str, ...]:
    """``_normalize_values`` (``catalog.py:186-232``): parser output -> tuple of
    strings (() = null), with the reference's SchemaErrors."""
    if raw is None:
        values: tuple[str, ...] = ()
    elif isinstance(raw, str):
        values = (raw,)
    elif isinstance(raw, (list, tuple, set)):
        values = tuple(sorted(str(v) for v in raw))
    elif isinstance(raw, (int, float, bool)):
        values = (str(raw),)
    else:
        raise SchemaError(f"{where}: property {prop.name!r} got unsupported value {raw!r}")
    if not values:
        if not prop.nullable:
            raise SchemaError(f"{where}: non-nullable property {prop.name!r} is missing")
        return ()
    if len(values) > 1 and not prop.multiple:
        raise SchemaError(f"{where}: property {prop.name!r} is single-valued but got {len(values)} values")
    if len(set(values)) != len(values):
        values = tuple(sorted(set(values)))
    if prop.kind == "categorical":
        bad = [v for v in values if v not in prop.categories]
        if bad:
            raise SchemaError(f"{where}: value {bad[0]!r} not in categories of {prop.name!r}")
    return values


_STAGE = None


class LoadedJsonl:
    """JSON-lines files resident in HBM with their record spans."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def load_jsonl(paths, device) -> LoadedJsonl:
    """Every file into its own slot of one pinned buffer (+1 byte: a newline
    where the file lacks a final one, else an empty line that iter_records
    skips), read and BLAKE2b-hashed (_hash_file) by a thread pool, copied to
    the device; the records (non-empty lines, iter_records order) found by
    mx_jsonl_records."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import torch

    sizes = [os.stat(p).st_size for p in paths]
    starts = np.zeros(len(paths) + 1, np.int64)
    np.cumsum([n + 1 for n in sizes], out=starts[1:])
    total = int(starts[-1])
    padded = max(16, (total + 15) // 16 * 16)
    host = _staging(padded)
    hv = host.numpy()
    hv[total:] = 0x20
    mv = memoryview(hv)

    def load(i):
        s0, n = int(starts[i]), sizes[i]
        with open(paths[i], "rb", buffering=0) as fh:
            got = fh.readinto(mv[s0:s0 + n])
        if got != n:
            raise DataReadError(f"{paths[i]}: short read ({got} of {n} bytes)")
        hv[s0 + n] = 0x0A
        digest = hashlib.blake2b(mv[s0:s0 + n], digest_size=16).hexdigest()
        return digest, int(np.count_nonzero(hv[s0:s0 + n + 1] == 0x0A))

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1, max(1, len(paths)))) as pool:
        done = list(pool.map(load, range(len(paths))))
    buf = host.to(device, non_blocking=True)
    L = _lib.lib()
    stream = C.c_void_p(_lib.stream_ptr())
    n_rec, n_lines = C.c_int64(), C.c_int64()
    _lib.check(L.mx_jsonl_records(buf.data_ptr(), padded, None, None, None, 0, C.byref(n_rec), C.byref(n_lines),
                                  stream))
    R = n_rec.value
    rs = torch.empty(max(R, 1), dtype=torch.int64, device=device)
    re = torch.empty_like(rs)
    rl = torch.empty_like(rs)
    _lib.check(L.mx_jsonl_records(buf.data_ptr(), padded, rs.data_ptr(), re.data_ptr(), rl.data_ptr(), R,
                                  C.byref(n_rec), C.byref(n_lines), stream))
    return LoadedJsonl(buf=buf, host=hv, starts=starts, digests=[d for d, _ in done],
                       nl_counts=[c for _, c in done], n_records=R, rs=rs[:R], re=re[:R], rl=rl[:R], padded=padded)


def _staging(n: int):
    """Grow-only pinned staging buffer shared by registrations (pinning a few
    hundred MB costs more than reading them from the page cache)."""
    import torch

    global _STAGE
    if _STAGE is None or _STAGE.numel() < n:
        _STAGE = torch.empty(max(n, 1 << 20), dtype=torch.uint8, pin_memory=True)
    return _STAGE[:n]


class DeviceMetadataCatalog:
    """Registered datasets with their code columns in HBM.

    Mirrors the registration half of the reference ``MetadataCatalog``
    (``register_dataset``, dataset / file ids, property merging, vocabularies)
    and hands the result to the hot path as a ``ColumnarCatalog`` /
    ``DeviceCatalog``."""

    def __init__(self, device=None):
        import torch

        self.device = torch.device(device or "cuda")
        self._props: dict[str, object] = {}
        self._vocab: dict[str, list] = {}        # prop -> code -> str | tuple (multi)
        self._vocab_idx: dict[str, dict] = {}
        self._dataset_names: list[str] = []
        self._dataset_schemas: dict[int, object] = {}
        self._dataset_files: dict[int, list[int]] = {}
        self._files: dict[int, dict] = {}       # fid -> path, dataset_id, n_samples, content_hash
        self._columns: dict[str, list] = {}      # prop -> per-dataset device int32 columns (None = all null)
        self._sizes: list[int] = []              # samples per dataset, registration order
        self.timings: dict[str, float] = {}

    # ------------------------------------------------------------ registration
    def register_dataset(self, name: str, files: Sequence, parser, schema, workers: int = 1) -> int:
        """``register_dataset`` (``catalog.py:323-435``); ``workers`` is
        accepted for signature parity (the device pass does not depend on it)."""
        paths = [str(Path(p)) for p in files]
        if not paths:
            raise RegistrationError(f"dataset {name!r}: no files given")
        for p in paths:
            if not Path(p).is_file():
                raise RegistrationError(f"dataset {name!r}: file not found: {p}")
            if not (p.endswith(JSONL_SUFFIX) or p.endswith(ZST_SUFFIX)):
                raise RegistrationError(f"dataset {name!r}: unsupported file type: {p}")
        for p in paths:
            if p.endswith(ZST_SUFFIX):
                raise NotImplementedError(f"{p}: zstd-compressed metadata is not decoded on the device")
        fields = getattr(parser, "fields", None)
        if fields is None:
            raise NotImplementedError("device registration reads JSON fields (JsonFieldParser-like parsers)")
        import time

        t0 = time.perf_counter()
        parsed = self._parse(paths, parser, tuple(fields), schema)
        self._validate(parsed, schema)  # the first failing record raises, as the reference's parse does
        t1 = time.perf_counter()
        if name in self._dataset_names:
            return self._check_reregistration(name, paths, parsed["digests"], schema)
        props = dict(self._props)
        for prop in schema.properties:
            held = props.get(prop.name)
            if held is None:
                props[prop.name] = prop
            elif (held.kind, held.multiple, held.categories) != (prop.kind, prop.multiple, prop.categories):
                raise SchemaError(f"property {prop.name!r} conflicts with an earlier dataset's definition")
        # commit: vocab (values in first-appearance order), columns, ids
        vocab = {p: list(v) for p, v in self._vocab.items()}
        vocab_idx = {p: dict(v) for p, v in self._vocab_idx.items()}
        for prop in schema.properties:
            if prop.name not in vocab:
                if prop.kind == "categorical" and not prop.multiple:
                    vocab[prop.name] = list(prop.categories)
                else:
                    vocab[prop.name] = []
                vocab_idx[prop.name] = {v: i for i, v in enumerate(vocab[prop.name])}
        cols = self._intern(parsed, schema, vocab, vocab_idx)
        dataset_id = len(self._dataset_names)
        n_new = int(parsed["n_records"])
        for p in props:
            self._columns.setdefault(p, [None] * len(self._sizes))
        for p, col in self._columns.items():
            col.append(cols.get(p))
        self._sizes.append(n_new)
        self._props = props
        self._vocab, self._vocab_idx = vocab, vocab_idx
        self._dataset_names.append(name)
        self._dataset_schemas[dataset_id] = schema
        next_fid = 1 + max(self._files, default=0)
        ids = []
        for path, digest, n in zip(paths, parsed["digests"], parsed["per_file"]):
            self._files[next_fid] = dict(path=path, dataset_id=dataset_id, n_samples=int(n), content_hash=digest)
            ids.append(next_fid)
            next_fid += 1
        self._dataset_files[dataset_id] = ids
        self.timings.update(parse_validate_s=t1 - t0, intern_commit_s=time.perf_counter() - t1)
        return dataset_id

    def _check_reregistration(self, name, paths, digests, schema) -> int:
        dataset_id = self._dataset_names.index(name)
        if schema != self._dataset_schemas[dataset_id]:
            raise RegistrationError(f"dataset {name!r} already registered with a different schema")
        held = sorted((self._files[f]["path"], self._files[f]["content_hash"]) for f in self._dataset_files[dataset_id])
        if held != sorted(zip(paths, digests)):
            raise RegistrationError(f"dataset {name!r} already registered with different content")
        return dataset_id

    # ------------------------------------------------------------ device pass
    def _parse(self, paths, parser, fields, schema) -> dict:
        import time

        import torch

        t0 = time.perf_counter()
        lf = load_jsonl(paths, self.device)
        t1 = time.perf_counter()
        dev = self.device
        L = _lib.lib()
        stream = C.c_void_p(_lib.stream_ptr())
        buf, starts, digests, nl_counts, hv = lf.buf, lf.starts, lf.digests, lf.nl_counts, lf.host
        R, rs, re, rl = lf.n_records, lf.rs, lf.re, lf.rl
        # files of the records; each file's first global line index
        fstart = torch.from_numpy(starts[:-1]).to(dev)
        rec_file = torch.searchsorted(fstart, rs[:R], right=True) - 1
        per_file = torch.bincount(rec_file, minlength=len(paths)).cpu().numpy()
        first_line = np.zeros(len(paths), np.int64)
        if len(paths) > 1:
            np.cumsum(nl_counts[:-1], out=first_line[1:])
        # requested fields: every parser field (a field mapped to a property
        # outside the schema must be absent: the reference raises otherwise)
        fld_names = sorted({f for _, f in fields})
        fpos = {f: i for i, f in enumerate(fld_names)}
        enc = [f.encode("utf-8") for f in fld_names]
        foff = np.zeros(len(enc) + 1, np.int64)
        np.cumsum([len(x) for x in enc], out=foff[1:])
        fblob = torch.from_numpy(np.frombuffer(b"".join(enc) or b"\0", np.uint8).copy()).to(dev)
        foff_d = torch.from_numpy(foff).to(dev)
        F = len(enc)
        kind = torch.zeros((max(R, 1), max(F, 1)), dtype=torch.uint8, device=dev)
        nelem = torch.zeros_like(kind)
        ha = torch.zeros((max(R, 1), max(F, 1)), dtype=torch.int64, device=dev)
        hb = torch.zeros_like(ha)
        vs = torch.zeros_like(ha)
        vl = torch.zeros((max(R, 1), max(F, 1)), dtype=torch.int32, device=dev)
        flag = torch.zeros(max(R, 1), dtype=torch.uint8, device=dev)
        _lib.check(L.mx_jsonl_extract(buf.data_ptr(), rs.data_ptr(), re.data_ptr(), R, fblob.data_ptr(),
                                      foff_d.data_ptr(), F, kind.data_ptr(), nelem.data_ptr(), ha.data_ptr(),
                                      hb.data_ptr(), vs.data_ptr(), vl.data_ptr(), flag.data_ptr(), stream))
        self.timings["read_s"] = t1 - t0
        return dict(paths=paths, parser=parser, fields=fields, fpos=fpos, starts=starts, host=hv,
                    digests=digests, n_records=R, per_file=per_file, first_line=first_line, rs=rs, re=re,
                    rl=rl, rec_file=rec_file, kind=kind[:R], nelem=nelem[:R], ha=ha[:R], hb=hb[:R],
                    vs=vs[:R], vl=vl[:R], flag=flag[:R], schema=schema)

    def _where(self, ps, r: int) -> tuple[str, int, int]:
        """(path, sample id within the file, physical line number) of record r."""
        f = int(ps["rec_file_h"][r])
        sample = r - int(ps["file_rec0"][f])
        line = int(ps["rl_h"][r]) - int(ps["first_line"][f])
        return ps["paths"][f], sample, line

    def _record(self, ps, r: int) -> dict:
        """Reference semantics for one record: json.loads + parser.parse +
        _normalize_values; raises the reference's error for this record."""
        path, sample, line = self._where(ps, r)
        s, e = int(ps["rs_h"][r]), int(ps["re_h"][r])
        raw = bytes(ps["host"][s:e])
        try:
            record = json.loads(raw)
        except (ValueError, UnicodeDecodeError) as exc:
            raise DataReadError(f"{path}: malformed JSON on line {line + 1}: {exc}") from exc
        out = ps["parser"].parse(sample, record)
        where = f"{path} sample {sample}"
        schema = ps["schema"]
        unknown = set(out) - set(schema.names())
        if unknown:
            raise SchemaError(f"{where}: unknown property {sorted(unknown)[0]!r}")
        values = {}
        for prop in schema.properties:
            norm = normalize_values(prop, out.get(prop.name), where)
            if norm:
                values[prop.name] = norm
        return values

    def _validate(self, ps, schema) -> None:
        import torch

        R = ps["n_records"]
        dev = self.device
        ps["rec_file_h"] = ps["rec_file"].cpu().numpy()
        ps["file_rec0"] = np.concatenate([[0], np.cumsum(ps["per_file"])[:-1]]).astype(np.int64)
        ps["rl_h"] = ps["rl"].cpu().numpy()
        ps["rs_h"] = ps["rs"].cpu().numpy()
        ps["re_h"] = ps["re"].cpu().numpy()
        prop_field = {}
        for prop, fld in ps["fields"]:
            prop_field.setdefault(prop, fld)  # JsonFieldParser: the first mapping of a property
        # records that may raise or that the device did not cover
        cand = ps["flag"].bool().clone() if R else torch.zeros(0, dtype=torch.bool, device=dev)
        names = set(schema.names())
        for prop, fld in ps["fields"]:
            if prop not in names:  # present at all -> "unknown property"
                cand |= ps["kind"][:, ps["fpos"][fld]] != 0
        uniq = {}
        for prop in schema.properties:
            fld = prop_field.get(prop.name)
            if fld is None:
                if not prop.nullable:  # never produced by the parser: every record fails
                    cand[:] = True
                continue
            k = ps["kind"][:, ps["fpos"][fld]]
            if not prop.nullable:
                cand |= (k == 0) | (k == 3)
            if not prop.multiple:
                cand |= (k == 1) & (ps["nelem"][:, ps["fpos"][fld]] > 1)
            ok = (k == 1) & ~ps["flag"].bool()
            idx = torch.nonzero(ok).flatten()
            a = ps["ha"][idx, ps["fpos"][fld]]
            b = ps["hb"][idx, ps["fpos"][fld]]
            ua, inv = torch.unique(a, return_inverse=True)
            ub = torch.zeros_like(ua).scatter_(0, inv, b)
            if not torch.equal(ub[inv], b):
                raise RuntimeError(f"property {prop.name!r}: 64-bit hash collision between distinct values")
            first = torch.full((ua.numel(),), R, dtype=torch.int64, device=dev).scatter_reduce_(
                0, inv, idx, reduce="amin")
            # value strings of each distinct hash from its first record's span
            fh = first.cpu().numpy()
            st = ps["vs"][first, ps["fpos"][fld]].cpu().numpy()
            ln = ps["vl"][first, ps["fpos"][fld]].cpu().numpy()
            hv = ps["host"]
            vals = []
            for s0, n0 in zip(st.tolist(), ln.tolist()):
                if s0 >= 0:
                    vals.append((bytes(hv[s0:s0 + n0]).decode("utf-8", "surrogatepass"),))
                else:
                    s1 = ~s0
                    vals.append(tuple(sorted(set(json.loads(bytes(hv[s1:s1 + n0]))))))
            bad_first = []
            if prop.kind == "categorical":
                cats = set(prop.categories)
                bad_first = [int(r) for r, v in zip(fh.tolist(), vals) if any(x not in cats for x in v)]
            uniq[prop.name] = (idx, inv, fh, vals, fld)
            if bad_first:
                cand[torch.tensor(bad_first, device=dev)] = True
        # evaluate the candidate records in order: the first failure raises
        host_vals = {}
        flag_h = ps["flag"].cpu().numpy()
        for r in torch.nonzero(cand).flatten().cpu().numpy().tolist():
            values = self._record(ps, r)
            if flag_h[r]:
                host_vals[r] = values
        ps["uniq"], ps["host_vals"] = uniq, host_vals

    def _intern(self, ps, schema, vocab, vocab_idx) -> dict:
        import torch

        R, dev = ps["n_records"], self.device
        uniq, host_vals = ps["uniq"], ps["host_vals"]
        # codes in first-appearance order (device uniques and host records)
        cols = {}
        for prop in schema.properties:
            col = torch.full((R,), -1, dtype=torch.int32, device=dev)
            u = uniq.get(prop.name)
            items = []
            if u is not None:
                idx, inv, fh, vals, _ = u
                items += [(int(r), v, j) for j, (r, v) in enumerate(zip(fh.tolist(), vals))]
            items += [(r, v[prop.name], None) for r, v in host_vals.items() if prop.name in v]
            items.sort(key=lambda x: x[0])
            code_of_unique = np.zeros(len(u[3]) if u is not None else 0, np.int32)
            host_codes = []
            for r, v, j in items:
                key = v if prop.multiple else v[0]
                c = vocab_idx[prop.name].get(key)
                if c is None:
                    c = len(vocab[prop.name])
                    vocab[prop.name].append(key)
                    vocab_idx[prop.name][key] = c
                if j is not None:
                    code_of_unique[j] = c
                else:
                    host_codes.append((r, c))
            if u is not None and u[0].numel():
                col[u[0]] = torch.from_numpy(code_of_unique).to(dev)[u[1]]
            if host_codes:
                rr = torch.tensor([r for r, _ in host_codes], device=dev)
                col[rr] = torch.tensor([c for _, c in host_codes], dtype=torch.int32, device=dev)
            cols[prop.name] = col
        return cols

    # ------------------------------------------------------------ hot-path views
    def file_table(self):
        fids = sorted(self._files)
        return (np.array(fids, np.int64), np.array([self._files[f]["dataset_id"] for f in fids], np.int32),
                np.array([self._files[f]["n_samples"] for f in fids], np.int64))

    def device_columns(self) -> dict:
        """prop -> device int32[N] over all registered samples (file-id order)."""
        import torch

        out = {}
        for p, parts in self._columns.items():
            segs = [c if c is not None else torch.full((n,), -1, dtype=torch.int32, device=self.device)
                    for c, n in zip(parts, self._sizes)]
            out[p] = torch.cat(segs) if segs else torch.zeros(0, dtype=torch.int32, device=self.device)
        return out

    def columnar(self, with_columns: bool = True) -> ColumnarCatalog:
        fids, ds, sizes = self.file_table()
        multiple = {p: bool(d.multiple) for p, d in self._props.items()}
        if not with_columns:
            return ColumnarCatalog.meta_only(self._vocab, sizes, ds, fids, multiple)
        cols = {p: c.cpu().numpy() for p, c in self.device_columns().items()}
        offsets = np.zeros(len(sizes) + 1, np.int64)
        np.cumsum(sizes, out=offsets[1:])
        return ColumnarCatalog(columns=cols, vocab={p: list(v) for p, v in self._vocab.items()}, multiple=multiple,
                               file_ids=fids, file_ds=ds, file_offsets=offsets,
                               dataset_names=list(self._dataset_names),
                               file_paths={f: self._files[f]["path"] for f in fids})

    def device_catalog(self):
        """The registered catalog as the hot path's ``DeviceCatalog`` (columns
        stay in HBM)."""
        from .index import DeviceCatalog

        cols = self.device_columns()
        return DeviceCatalog(self.columnar(with_columns=False), columns=cols)
