"""A minimal in-process model hub for running the hot path without the
reference installed (e.g. on the GPU box, in bench.py).

The reference's registry (pkg/src/modelci/registry/) is out of scope for the
B200 rebuild: with the reference present, the profiler
here takes its ``ModelRegistry`` unchanged (tests/test_dropin.py).  This hub
implements only the methods the hot path calls — ``register``, ``get``,
``get_blob``/``put_blob``, ``append_variant``, ``append_result``,
``advance_status`` — with the reference's record/variant documents and
lifecycle order (registry/types.py:13-28, 46-64, 75-244), plus a dict-backed
document store for ``JobStore``.
"""

from __future__ import annotations

import hashlib
import threading
import uuid
from dataclasses import dataclass, field
from datetime import datetime, timezone
from typing import Optional

from .errors import InvalidManifest, NotFound

LIFECYCLE = ["registered", "converting", "converted", "profiling", "profiled", "serving"]


def legal_transition(cur: str, new: str) -> bool:
    if new == cur:
        return False
    if cur == "failed":
        return new == "converting"
    if new == "failed":
        return cur != "serving"
    return new in LIFECYCLE and LIFECYCLE.index(new) == LIFECYCLE.index(cur) + 1


def _now() -> str:
    return datetime.now(timezone.utc).isoformat()


@dataclass
class TensorSpec:
    name: str
    shape: list
    dtype: str = "float32"

    def sample_size(self) -> int:
        n = 1
        for d in self.shape:
            if d != -1:
                n *= d
        return n


@dataclass
class ModelVariant:
    id: str
    parent_id: str
    format: str
    blob_digest: str
    serving_backends: list
    created_at: str = field(default_factory=_now)


@dataclass
class ModelRecord:
    id: str
    name: str
    framework: str
    version: int
    inputs: list
    weight_digest: str
    status: str = "registered"
    variants: list = field(default_factory=list)
    profiling_results: list = field(default_factory=list)

    def variant_by_id(self, vid: str) -> Optional[ModelVariant]:
        return next((v for v in self.variants if v.id == vid), None)


class MemoryStore:
    """Document + blob store (the StoreBackend subset JobStore needs)."""

    def __init__(self):
        self._docs: dict = {}
        self._blobs: dict = {}
        self._lock = threading.Lock()

    def put_doc(self, coll: str, doc_id: str, doc: dict) -> None:
        with self._lock:
            self._docs.setdefault(coll, {})[doc_id] = doc

    def get_doc(self, coll: str, doc_id: str):
        return self._docs.get(coll, {}).get(doc_id)

    def list_docs(self, coll: str):
        return list(self._docs.get(coll, {}).values())

    def put_blob(self, data: bytes) -> str:
        d = hashlib.sha256(data).hexdigest()
        with self._lock:
            self._blobs[d] = data
        return d

    def get_blob(self, digest: str) -> bytes:
        try:
            return self._blobs[digest]
        except KeyError:
            raise NotFound(f"no blob {digest}") from None


class Hub:
    def __init__(self, store: Optional[MemoryStore] = None):
        self.store = store or MemoryStore()
        self._records: dict[str, ModelRecord] = {}
        self._lock = threading.Lock()

    def register(self, name: str, framework: str, weights: bytes, inputs: list) -> ModelRecord:
        if not weights:
            raise InvalidManifest("weights must be non-empty")
        digest = self.store.put_blob(weights)
        with self._lock:
            version = 1 + max((r.version for r in self._records.values()
                               if r.name == name and r.framework == framework), default=0)
            rec = ModelRecord(uuid.uuid4().hex[:12], name, framework, version, list(inputs),
                              digest)
            self._records[rec.id] = rec
        return rec

    def get(self, record_id: str) -> ModelRecord:
        try:
            return self._records[record_id]
        except KeyError:
            raise NotFound(f"no model with id {record_id}") from None

    def put_blob(self, data: bytes) -> str:
        return self.store.put_blob(data)

    def get_blob(self, digest: str) -> bytes:
        return self.store.get_blob(digest)

    def append_variant(self, record_id: str, variant: ModelVariant) -> ModelRecord:
        rec = self.get(record_id)
        with self._lock:
            rec.variants.append(variant)
        return rec

    def append_result(self, record_id: str, result) -> ModelRecord:
        rec = self.get(record_id)
        with self._lock:
            rec.profiling_results.append(result)
        return rec

    def advance_status(self, record_id: str, status: str) -> ModelRecord:
        rec = self.get(record_id)
        with self._lock:
            if legal_transition(rec.status, status):
                rec.status = status
        return rec

    def convert(self, record: ModelRecord, plugin) -> ModelVariant:
        """Run one converter plugin and attach its variant (what the
        reference's Converter._convert_one does, converter.py:84-97)."""
        self.advance_status(record.id, "converting")
        out = plugin.run(self.get_blob(record.weight_digest))
        v = ModelVariant(uuid.uuid4().hex[:12], record.id, plugin.target_format,
                         self.put_blob(out), list(plugin.produces_backends))
        self.append_variant(record.id, v)
        self.advance_status(record.id, "converted")
        return v
