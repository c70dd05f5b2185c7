"""CPU: the drop-in CLI's parser mirrors specdraft's (ref cli.py:160-227) and
the host-side boundary helpers reject ids the device cannot represent."""

import subprocess
import sys

import numpy as np
import pytest

from paper_2411_05894_b200 import cli, kvconfig
from paper_2411_05894_b200.datastore import as_u32


def test_parser_has_the_reference_subcommands():
    p = cli.build_parser()
    sub = next(a for a in p._actions if a.dest == "command")
    assert set(sub.choices) == {"build-datastore", "simulate", "calibrate", "plan", "bench-retrieval"}
    a = p.parse_args(["build-datastore", "--in", "a.tok", "b.txt", "--out", "x.bin", "--separator", "7"])
    assert a.inputs == ["a.tok", "b.txt"] and a.separator == 7 and a.vocab_size is None
    a = p.parse_args(["simulate", "--datastore", "d", "--data", "x.jsonl", "--sweep", "1,4,16"])
    assert a.sweep == [1, 4, 16] and a.sources == "both" and a.threads == 1
    a = p.parse_args(["bench-retrieval", "--datastore", "d", "--data", "x"])
    assert a.batch_sizes == [1, 8] and a.threads == [1, 2, 8] and a.repeats == 3


def test_missing_subcommand_exits():
    with pytest.raises(SystemExit):
        cli.main([])


def test_module_entry_point_help():
    r = subprocess.run([sys.executable, "-m", "paper_2411_05894_b200", "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "build-datastore" in r.stdout


def test_bad_input_file_is_an_error(tmp_path, capsys):
    bad = tmp_path / "bad.txt"
    bad.write_text("1 frog 3")
    assert cli.main(["build-datastore", "--in", str(bad), "--out", str(tmp_path / "x.bin")]) == 1
    assert "error:" in capsys.readouterr().err


def test_format_kv_round_trip(tmp_path):
    items = {"P": 4, "alpha": 0.8, "dec_len": 30}
    assert kvconfig.format_kv(items) == "P = 4\nalpha = 0.8\ndec_len = 30\n"
    path = tmp_path / "c.txt"
    kvconfig.write_kv(path, items)
    assert kvconfig.read_kv(path) == {"P": "4", "alpha": "0.8", "dec_len": "30"}


def test_as_u32_range():
    assert as_u32([0, 5, 2**32 - 1]).tolist() == [0, 5, 2**32 - 1]
    assert as_u32(np.array([3], dtype=np.uint64)).dtype == np.dtype("<u4")
    for bad in ([-1], [2**32], [2**70]):
        with pytest.raises(ValueError, match="out of range"):
            as_u32(bad)
