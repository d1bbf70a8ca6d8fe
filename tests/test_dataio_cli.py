"""File formats and the command-line front end (reference test_dataio.py /
test_cli.py), pinned to the reference CLI's own outputs (tests/golden/cli_8.npz,
recorded by oracle/make_golden.py from /root/reference's cli.main).

CPU: formats, error paths, ``generate`` byte-identical to the reference.
GPU: ``solve`` / ``bench`` end to end against the reference's reports.
"""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_2502_04217_b200 import GridShape, Mask
from paper_2502_04217_b200.cli import EXIT_INPUT_ERROR, EXIT_MAX_ITERS, EXIT_OK, main
from paper_2502_04217_b200.dataio import read_mask, read_volume, sidecar_path, write_mask, write_volume


def read_report(path):
    with open(path, encoding="utf-8") as fh:
        return [json.loads(line) for line in fh if line.strip()]


def strip(rows, *keys):
    drop = {"wall_time", *keys}
    return [{k: v for k, v in r.items() if k not in drop} for r in rows]


@pytest.fixture(scope="module")
def gold():
    return load_golden("cli_8")


@pytest.fixture
def ref_files(gold, tmp_path):
    """The reference CLI's generated 8^3 problem, written back to disk."""
    paths = {}
    for key, name in (("signal", "signal.f64"), ("mask_idx", "mask.idx"), ("mask_byte", "mask.byte")):
        p = tmp_path / name
        p.write_bytes(gold[key].tobytes())
        (tmp_path / (name + ".json")).write_text(str(gold[key + "_json"]))
        paths[key] = str(p)
    return paths, tmp_path


# ---------------------------------------------------------------- file formats

class TestVolumeFile:
    def test_round_trip_bit_exact(self, tmp_path, rng):
        values = rng.standard_normal(4 * 6 * 2)
        path = str(tmp_path / "vol.f64")
        write_volume(path, values, (4, 6, 2))
        back, dims = read_volume(path)
        assert dims == (4, 6, 2)
        assert back.tobytes() == values.tobytes()

    def test_payload_length_checked_on_write(self, tmp_path):
        with pytest.raises(ValueError):
            write_volume(str(tmp_path / "v"), np.zeros(5), (4,))

    def test_missing_sidecar(self, tmp_path):
        path = tmp_path / "orphan.f64"
        np.zeros(4).tofile(path)
        with pytest.raises(ValueError, match="sidecar"):
            read_volume(str(path))

    def test_malformed_sidecar(self, tmp_path):
        path = tmp_path / "bad.f64"
        np.zeros(4).tofile(path)
        (tmp_path / "bad.f64.json").write_text("{not json")
        with pytest.raises(ValueError, match="malformed"):
            read_volume(str(path))

    def test_sidecar_without_dims(self, tmp_path):
        path = tmp_path / "nodims.f64"
        np.zeros(4).tofile(path)
        (tmp_path / "nodims.f64.json").write_text("[4]")
        with pytest.raises(ValueError, match="dims"):
            read_volume(str(path))

    def test_size_mismatch(self, tmp_path):
        path = tmp_path / "short.f64"
        np.zeros(3).tofile(path)
        (tmp_path / "short.f64.json").write_text(
            json.dumps({"dims": [4], "order": "row-major", "dtype": "f64-le"}))
        with pytest.raises(ValueError, match="samples"):
            read_volume(str(path))

    def test_trailing_partial_sample_ignored_like_fromfile(self, tmp_path):
        path = tmp_path / "tail.f64"
        path.write_bytes(np.arange(4.0).tobytes() + b"\x01\x02")
        (tmp_path / "tail.f64.json").write_text(json.dumps({"dims": [4]}))
        back, _ = read_volume(str(path))
        assert back.tolist() == [0.0, 1.0, 2.0, 3.0]

    @pytest.mark.parametrize("key,val", [("dtype", "f32-le"), ("order", "column-major")])
    def test_unknown_dtype_or_order(self, tmp_path, key, val):
        path = tmp_path / "odd.f64"
        np.zeros(4).tofile(path)
        meta = {"dims": [4], "order": "row-major", "dtype": "f64-le"}
        meta[key] = val
        (tmp_path / "odd.f64.json").write_text(json.dumps(meta))
        with pytest.raises(ValueError, match=key):
            read_volume(str(path))

    def test_reads_reference_written_volume(self, gold, ref_files):
        paths, _ = ref_files
        values, dims = read_volume(paths["signal"])
        assert dims == (8, 8, 8)
        assert values.tobytes() == gold["signal"].tobytes()


class TestMaskFile:
    @pytest.mark.parametrize("fmt", ["indices", "bytemask"])
    def test_round_trip(self, tmp_path, fmt):
        mask = Mask(np.array([1, 5, 6]), GridShape((4, 2)))
        path = str(tmp_path / f"mask.{fmt}")
        write_mask(path, mask, fmt=fmt)
        back = read_mask(path)
        np.testing.assert_array_equal(back.missing, mask.missing)
        assert back.shape.dims == mask.shape.dims

    def test_sidecar_contents(self, tmp_path):
        path = str(tmp_path / "m")
        write_mask(path, Mask(np.array([0]), GridShape((4,))))
        assert json.loads(open(sidecar_path(path)).read()) == {"format": "indices", "dims": [4]}

    def test_unknown_format(self, tmp_path):
        path = tmp_path / "m"
        np.zeros(1, dtype="<u8").tofile(path)
        (tmp_path / "m.json").write_text(json.dumps({"format": "bitmap", "dims": [4]}))
        with pytest.raises(ValueError, match="format"):
            read_mask(str(path))

    def test_unknown_format_on_write(self, tmp_path):
        with pytest.raises(ValueError, match="format"):
            write_mask(str(tmp_path / "m"), Mask(np.array([0]), GridShape((4,))), fmt="bitmap")

    def test_bytemask_size_checked(self, tmp_path):
        path = tmp_path / "m"
        np.zeros(3, dtype=np.uint8).tofile(path)
        (tmp_path / "m.json").write_text(json.dumps({"format": "bytemask", "dims": [4]}))
        with pytest.raises(ValueError):
            read_mask(str(path))

    def test_reference_formats_agree(self, ref_files):
        paths, _ = ref_files
        a, b = read_mask(paths["mask_idx"]), read_mask(paths["mask_byte"])
        np.testing.assert_array_equal(a.missing, b.missing)
        assert a.shape.dims == (8, 8, 8) and a.n_missing > 0


# ---------------------------------------------------------------- CLI (host side)

class TestGenerate:
    @pytest.mark.parametrize("fmt,key", [("indices", "mask_idx"), ("bytemask", "mask_byte")])
    def test_byte_identical_to_reference(self, gold, tmp_path, fmt, key):
        sig, msk = str(tmp_path / "s.f64"), str(tmp_path / "m")
        assert main(["generate", "--dims", "8,8,8", "--noise-seed", "3", "--missing-seed", "4",
                     "--signal", sig, "--mask", msk, "--mask-format", fmt]) == EXIT_OK
        assert open(sig, "rb").read() == gold["signal"].tobytes()
        assert open(msk, "rb").read() == gold[key].tobytes()
        assert json.loads(open(sig + ".json").read()) == json.loads(str(gold["signal_json"]))
        assert json.loads(open(msk + ".json").read()) == json.loads(str(gold[key + "_json"]))

    def test_truth_output(self, tmp_path):
        truth = str(tmp_path / "truth.f64")
        assert main(["generate", "--dims", "4x4", "--signal", str(tmp_path / "s.f64"),
                     "--mask", str(tmp_path / "m"), "--truth", truth]) == EXIT_OK
        values, dims = read_volume(truth)
        assert dims == (4, 4) and values[0] == pytest.approx(1.0)

    def test_bad_dims(self, tmp_path, capsys):
        code = main(["generate", "--dims", "banana", "--signal", str(tmp_path / "s"),
                     "--mask", str(tmp_path / "m")])
        assert code == EXIT_INPUT_ERROR
        assert "error" in capsys.readouterr().err


class TestSolveInputErrors:
    def test_missing_input(self, tmp_path, capsys):
        code = main(["solve", "--input", str(tmp_path / "nope.f64"), "--mask", str(tmp_path / "nope.m"),
                     "--output", str(tmp_path / "out.f64")])
        assert code == EXIT_INPUT_ERROR
        assert "error" in capsys.readouterr().err

    def test_malformed_header(self, tmp_path, capsys):
        bad = tmp_path / "bad.f64"
        np.zeros(4).tofile(bad)
        (tmp_path / "bad.f64.json").write_text("{oops")
        code = main(["solve", "--input", str(bad), "--mask", str(bad), "--output", str(tmp_path / "o")])
        assert code == EXIT_INPUT_ERROR
        assert "error" in capsys.readouterr().err

    def test_odd_dims_rejected(self, tmp_path, capsys):
        vol = tmp_path / "odd.f64"
        np.zeros(5).tofile(vol)
        (tmp_path / "odd.f64.json").write_text(json.dumps({"dims": [5], "order": "row-major",
                                                           "dtype": "f64-le"}))
        msk = tmp_path / "odd.mask"
        np.array([1], dtype="<u8").tofile(msk)
        (tmp_path / "odd.mask.json").write_text(json.dumps({"format": "indices", "dims": [5]}))
        code = main(["solve", "--input", str(vol), "--mask", str(msk), "--output", str(tmp_path / "b")])
        assert code == EXIT_INPUT_ERROR
        assert "even" in capsys.readouterr().err

    def test_dims_mismatch(self, ref_files, tmp_path, capsys):
        paths, _ = ref_files
        other = str(tmp_path / "other.mask")
        assert main(["generate", "--dims", "4,4", "--signal", str(tmp_path / "s2.f64"),
                     "--mask", other]) == EXIT_OK
        code = main(["solve", "--input", paths["signal"], "--mask", other,
                     "--output", str(tmp_path / "b.f64")])
        assert code == EXIT_INPUT_ERROR
        assert "dims" in capsys.readouterr().err


# ---------------------------------------------------------------- CLI on the GPU

def _compare_reports(ours, ref):
    """Same records, keys and decisions; floats to the parity tolerance."""
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert a.keys() == b.keys()
        for k in a:
            if k == "input":
                continue
            va, vb = a[k], b[k]
            if isinstance(vb, float) and isinstance(va, float):
                if k in ("lambda", "tol", "cg_tol", "final_objective", "objective"):
                    assert va == pytest.approx(vb, rel=1e-9, abs=0.0), k
                # residual-type floats (mu, infeasibilities, pcg residuals) are
                # rounding-level at convergence; checked by order of magnitude
                elif abs(vb) > 1e-6:
                    assert va == pytest.approx(vb, rel=1e-4), k
            else:
                assert va == vb, k


@pytest.mark.gpu
class TestSolveGpu:
    def test_end_to_end_matches_reference(self, gold, ref_files):
        paths, tmp = ref_files
        out, rep, imp = str(tmp / "beta.f64"), str(tmp / "r.jsonl"), str(tmp / "imp.f64")
        code = main(["solve", "--input", paths["signal"], "--mask", paths["mask_idx"],
                     "--output", out, "--report", rep, "--impute", imp])
        assert code == int(gold["code"]) == EXIT_OK
        ours, ref = strip(read_report(rep)), json.loads(str(gold["records_json"]))
        _compare_reports(ours, ref)
        iters = [r for r in ours if r["record"] == "iteration"]
        assert [r["iteration"] for r in iters] == list(range(1, ours[-1]["iterations"] + 1))
        beta, dims = read_volume(out)
        ref_beta = np.frombuffer(gold["beta"].tobytes(), dtype="<f8")
        assert dims == (8, 8, 8)
        assert np.linalg.norm(beta - ref_beta) <= 1e-6 * np.linalg.norm(ref_beta)
        imputed, _ = read_volume(imp)
        ref_imp = np.frombuffer(gold["imputed"].tobytes(), dtype="<f8")
        assert np.linalg.norm(imputed - ref_imp) <= 1e-6 * np.linalg.norm(ref_imp)

    def test_bytemask_input_same_result(self, ref_files):
        paths, tmp = ref_files
        outs = []
        for key in ("mask_idx", "mask_byte"):
            out = str(tmp / f"b_{key}.f64")
            assert main(["solve", "--input", paths["signal"], "--mask", paths[key], "--output", out]) == EXIT_OK
            outs.append(open(out, "rb").read())
        assert outs[0] == outs[1]

    def test_max_iters_exit_code(self, gold, ref_files):
        paths, tmp = ref_files
        rep = str(tmp / "r2.jsonl")
        code = main(["solve", "--input", paths["signal"], "--mask", paths["mask_idx"], "--max-iters", "2",
                     "--output", str(tmp / "b2.f64"), "--report", rep])
        assert code == int(gold["code_max"]) == EXIT_MAX_ITERS
        _compare_reports(strip(read_report(rep)), json.loads(str(gold["records_max_json"])))

    def test_explicit_lambda_recorded(self, ref_files):
        paths, tmp = ref_files
        rep = str(tmp / "r.jsonl")
        assert main(["solve", "--input", paths["signal"], "--mask", paths["mask_idx"], "--lambda", "5.0",
                     "--output", str(tmp / "b.f64"), "--report", rep]) == EXIT_OK
        meta = read_report(rep)[0]
        assert meta["lambda"] == 5.0 and meta["lambda_source"] == "flag"

    def test_deterministic_reports(self, ref_files):
        paths, tmp = ref_files
        outs = []
        for tag in ("a", "b"):
            rep = str(tmp / f"rep_{tag}.jsonl")
            assert main(["solve", "--input", paths["signal"], "--mask", paths["mask_idx"],
                         "--output", str(tmp / f"beta_{tag}.f64"), "--report", rep]) == EXIT_OK
            outs.append(json.dumps(strip(read_report(rep)), sort_keys=True))
        assert outs[0] == outs[1]


@pytest.mark.gpu
def test_bench_rows_match_reference(gold, tmp_path):
    path = str(tmp_path / "bench.jsonl")
    assert main(["bench", "--sizes", "4,8", "--seed", "7", "--report", path]) == int(gold["code_bench"])
    ours, ref = strip(read_report(path)), json.loads(str(gold["bench_json"]))
    assert [r["unknowns"] for r in ours] == [64, 512]
    assert [r["ipm_variables"] for r in ours] == [128, 1024]
    _compare_reports(ours, ref)
