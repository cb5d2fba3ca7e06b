"""TemplateLibrary persistence (templates.py:364-401): the saved
JSONL is byte-identical to the reference's own save for the same templates."""

import hashlib
import os
import tempfile

import pytest

from paper_2605_04357_b200.library import TemplateLibrary, library_meta
from paper_2605_04357_b200.specs import NodeComboKey, Placement, ServingTemplate
from tests.helpers import golden, workload


def library_from_lines(name, lines):
    configs, models, slos, caps, ctx, regions, prices = workload(name)
    cfg = {c.name: c for c in configs}
    entries = []
    for ln in lines:
        model, phase, combo, S, layers, son, T = ln.split("|")
        items = tuple((cfg[t.rsplit("*", 1)[0]], int(t.rsplit("*", 1)[1])) for t in combo.split("+"))
        entries.append(ServingTemplate(model, phase, slos[model], NodeComboKey(items),
                                       Placement(int(S), tuple(int(x) for x in layers.split(",")),
                                                 tuple(int(x) for x in son.split(","))), float(T)))
    meta = library_meta(sorted(configs, key=lambda c: c.name), models, slos, caps, ctx)
    return TemplateLibrary(entries=entries, meta=meta)


@pytest.mark.parametrize("name", ["c1", "core"])
def test_python_save_is_byte_identical_to_reference(name):
    lib = library_from_lines(name, golden(f"library_{name}.json.gz")["records"])
    ref = golden("saved_libraries.json.gz")[name]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "lib.jsonl")
        lib.save(path)
        data = open(path, "rb").read()
        assert data.split(b"\n", 1)[0].decode() == ref["header"]
        assert len(data) == ref["bytes"]
        assert hashlib.sha256(data).hexdigest() == ref["sha256"]
        back = TemplateLibrary.load(path)
        assert [t.template_id for t in back.entries] == [t.template_id for t in lib.entries]
        assert [t.throughput_tps for t in back.entries] == [t.throughput_tps for t in lib.entries]


def test_load_rejects_duplicate_templates(tmp_path):
    """A saved file with the same template twice: load raises the reference's
    DomainError('duplicate template ...') (templates.py:339-347), even though the
    duplicate lines are adjacent (in order)."""
    from paper_2605_04357_b200.specs import DomainError
    lib = library_from_lines("c1", golden("library_c1.json.gz")["records"])
    path = str(tmp_path / "lib.jsonl")
    lib.save(path)
    lines = open(path).read().splitlines(keepends=True)
    dup = str(tmp_path / "dup.jsonl")
    with open(dup, "w") as fh:
        fh.writelines(lines[:3] + [lines[2]] + lines[3:])
    with pytest.raises(DomainError, match="duplicate template"):
        TemplateLibrary.load(dup)
