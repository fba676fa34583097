"""Model / image files and the CLI: files written by
the REFERENCE (tests/golden/io_*) load bit-exactly here and our writer
reproduces them byte for byte; the CLI's despeckle equals run_diffusion."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import io as tio
from paper_1702_07482_b200 import synth
from paper_1702_07482_b200.cli import main


def test_reference_model_file_loads_bit_exact():
    m = tio.load_model(os.path.join(GOLDEN, "io_model_v1.txt"))
    g = load_golden("io_arrays")
    assert m.filter_size == int(g["m"]) and m.num_stages == 2 and m.looks == 1
    for t, st in enumerate(m.stages):
        assert st.beta == float(g["betas"][t])
        np.testing.assert_array_equal(st.coeffs, g["coeffs"][t])
        np.testing.assert_array_equal(st.weights, g["weights"][t])
    assert m.rbf.count == int(g["rbf_count"]) and m.rbf.radius == float(g["rbf_radius"])
    assert m.metadata == {"note": "golden"}


def test_model_writer_reproduces_reference_bytes(tmp_path):
    src = os.path.join(GOLDEN, "io_model_v1.txt")
    out = tmp_path / "m.txt"
    tio.save_model(tio.load_model(src), out)
    assert out.read_bytes() == open(src, "rb").read()


def test_model_round_trip_and_errors(tmp_path):
    model = synth.make_model(7, 4, 3, 63, seed=5, beta=0.3)
    p = tmp_path / "m.txt"
    tio.save_model(model, p)
    back = tio.load_model(p)
    for a, b in zip(model.stages, back.stages):
        assert a.beta == b.beta
        np.testing.assert_array_equal(a.coeffs, b.coeffs)
        np.testing.assert_array_equal(a.weights, b.weights)
    text = p.read_text()
    (tmp_path / "v2.txt").write_text(text.replace("specklediff-model 1", "specklediff-model 2", 1))
    with pytest.raises(ValueError, match="version"):
        tio.load_model(tmp_path / "v2.txt")
    (tmp_path / "noend.txt").write_text(text.replace("\nend\n", "\n"))
    with pytest.raises(ValueError, match="end marker"):
        tio.load_model(tmp_path / "noend.txt")
    (tmp_path / "junk.txt").write_text("hello\n")
    with pytest.raises(ValueError, match="not a model file"):
        tio.load_model(tmp_path / "junk.txt")


def test_reference_images_load():
    g = load_golden("io_arrays")
    np.testing.assert_array_equal(tio.load_image(os.path.join(GOLDEN, "io_image.fgrid")), g["img"])
    np.testing.assert_array_equal(tio.load_image(os.path.join(GOLDEN, "io_image8.pgm")), g["pgm8"])
    np.testing.assert_array_equal(tio.load_image(os.path.join(GOLDEN, "io_image16.pgm")), g["pgm16"])


def test_image_writers_match_reference_bytes(tmp_path):
    g = load_golden("io_arrays")
    for name, peak in (("io_image.fgrid", 255.0), ("io_image8.pgm", 255.0), ("io_image16.pgm", 1000.0)):
        out = tmp_path / name
        tio.save_image(g["img"], out, peak=peak)
        assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read(), name


def test_image_errors(tmp_path):
    (tmp_path / "bad.fgrid").write_text("FGRID 2 2\n1 2 3\n")
    with pytest.raises(ValueError, match="expected 4 values"):
        tio.load_image(tmp_path / "bad.fgrid")
    (tmp_path / "x.txt").write_text("nope")
    with pytest.raises(ValueError, match="unsupported image format"):
        tio.load_image(tmp_path / "x.txt")
    with pytest.raises(ValueError, match="suffix"):
        tio.save_image(np.ones((2, 2)), tmp_path / "a.png")


def test_cli_errors_exit_1(tmp_path, capsys):
    rc = main(["simulate", "--input", str(tmp_path / "nope.fgrid"), "--output", str(tmp_path / "o.fgrid")])
    assert rc == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_despeckle_matches_api(cuda, tmp_path):
    model = synth.make_model(7, 8, 3, 63, seed=2)
    mp = tmp_path / "m.txt"
    tio.save_model(model, mp)
    _, f = synth.noisy_image(synth.CONFIGS["c2"], 0, 48, 40)
    ip, op = tmp_path / "in.fgrid", tmp_path / "out.fgrid"
    tio.save_image(f.astype(np.float64), ip)
    assert main(["despeckle", "--model", str(mp), "--input", str(ip), "--output", str(op)]) == 0
    u, _ = tn.run_diffusion(f, tio.load_model(mp))
    np.testing.assert_array_equal(tio.load_image(op), u)


@pytest.mark.gpu
def test_reference_model_file_runs_on_gpu(cuda, oracle):
    m = tio.load_model(os.path.join(GOLDEN, "io_model_v1.txt"))
    f = np.random.default_rng(0).uniform(1, 255, (30, 26))
    u, _ = tn.run_diffusion(f, m)
    ref = oracle.run_diffusion(f.astype(np.float32).astype(np.float64), m)
    assert np.max(np.abs(u - ref) / ref) <= 1e-4
