"""PGM I/O and the CLI on the GPU engine (reference pkg/src/fsrkit/pgm.py,
cli.py; their tests pkg/tests/test_pgm.py, test_cli.py).  The CPU-only
subcommands and error paths run here; reconstruct runs on the GPU."""

import numpy as np
import pytest

from paper_2202_13926_b200 import cli, pgm
from paper_2202_13926_b200.frames import GrayImage
from oracle import port as oracle


def test_pgm_roundtrip_and_bytes(tmp_path):
    a = np.array([[0.0, 1.49, 1.5, 254.5], [255.7, -3.0, 128.0, 7.5]])
    p = tmp_path / "a.pgm"
    pgm.write_pgm(p, a)
    data = p.read_bytes()
    assert data[:11] == b"P5\n4 2\n255\n"
    assert list(data[11:]) == [0, 1, 2, 255, 255, 0, 128, 8]  # clamp, round half away from zero
    back = pgm.read_pgm(p)
    assert back.pixels.tolist() == [[0, 1, 2, 255], [255, 0, 128, 8]]
    pgm.write_pgm(tmp_path / "b.pgm", back)
    assert (tmp_path / "b.pgm").read_bytes() == data  # byte-stable


def test_pgm_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5 # comment\n3 # w\n 1\n255\n\x01\x02\x03")
    assert pgm.read_pgm(p).pixels.tolist() == [[1, 2, 3]]
    p.write_bytes(b"P2\n1 1\n255\n0")
    with pytest.raises(pgm.PgmError):
        pgm.read_pgm(p)
    p.write_bytes(b"P5\n4 4\n255\n\x00")
    with pytest.raises(pgm.PgmError, match="truncated"):
        pgm.read_pgm(p)
    p.write_bytes(b"P5\n1 1\n65535\n\x00\x00")
    with pytest.raises(pgm.PgmError, match="8-bit"):
        pgm.read_pgm(p)


def test_cli_sample_matches_reference_sampler(tmp_path):
    img = np.round(oracle.synthetic_frame(21, 30, 4))
    pgm.write_pgm(tmp_path / "x.pgm", img)
    rc = cli.main(["sample", "--input", str(tmp_path / "x.pgm"), "--output", str(tmp_path / "s.pgm"),
                   "--mask", str(tmp_path / "m.pgm"), "--seed", "42"])
    assert rc == 0
    mask = pgm.read_pgm(tmp_path / "m.pgm").pixels != 0
    assert np.array_equal(mask, oracle.quarter_sample_mask(img.shape, 42))
    s = pgm.read_pgm(tmp_path / "s.pgm").pixels
    assert np.array_equal(s, np.where(mask, img, 0.0))


def test_cli_evaluate_and_errors(tmp_path, capsys):
    a = np.full((4, 5), 100.0)
    pgm.write_pgm(tmp_path / "r.pgm", a)
    pgm.write_pgm(tmp_path / "t.pgm", a + 1)
    assert cli.main(["evaluate", "--reference", str(tmp_path / "r.pgm"), "--input", str(tmp_path / "t.pgm"),
                     "--csv", str(tmp_path / "e.csv")]) == 0
    out = capsys.readouterr().out
    assert "psnr_db=48.130804" in out and "mse=1.000000" in out
    assert (tmp_path / "e.csv").read_text().startswith("input,psnr_db,mse,elapsed_s")
    assert cli.main(["evaluate", "--reference", str(tmp_path / "nope.pgm"),
                     "--input", str(tmp_path / "t.pgm")]) == 2
    assert cli.main(["bench"]) == 2
    assert cli.main(["bench", "--list-only", "--support-list", "7"]) == 2


def test_cli_paper_grid_listing(capsys):
    assert cli.main(["bench", "--list-only", "--paper-grid"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert out[-1] == "points=640" and len(out) == 641


@pytest.mark.gpu
def test_cli_reconstruct_on_gpu(tmp_path, capsys):
    import paper_2202_13926_b200 as fsr
    img = np.round(oracle.synthetic_frame(40, 36, 6))
    pgm.write_pgm(tmp_path / "x.pgm", img)
    assert cli.main(["sample", "--input", str(tmp_path / "x.pgm"), "--output", str(tmp_path / "s.pgm"),
                     "--mask", str(tmp_path / "m.pgm"), "--seed", "3"]) == 0
    assert cli.main(["reconstruct", "--input", str(tmp_path / "s.pgm"), "--mask", str(tmp_path / "m.pgm"),
                     "--output", str(tmp_path / "r.pgm"), "--iterations", "60"]) == 0
    out = capsys.readouterr().out
    assert "blocks=90" in out
    s, m = oracle.quarter_sample(img, 3)
    ref = oracle.reconstruct_image(s, m, 4, 6, 60)
    got = pgm.read_pgm(tmp_path / "r.pgm").pixels
    assert np.abs(got - np.floor(np.clip(ref, 0, 255) + 0.5)).max() <= 1.0
    assert cli.main(["bench", "--input", str(tmp_path / "x.pgm"), "--iterations-list", "20",
                     "--argmax", "both", "--csv", str(tmp_path / "b.csv")]) == 0
    rows = (tmp_path / "b.csv").read_text().splitlines()
    assert rows[0] == ",".join(cli.CSV_HEADER) and len(rows) == 3
