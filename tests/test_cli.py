"""CLI: the reference's subcommands and exit contract (cli.py)."""

import numpy as np
import pytest

from paper_1609_01567_b200 import cli, configs, parse_alist, serialize_alist


def test_gen(tmp_path):
    out = tmp_path / "h.alist"
    assert cli.main(["gen", "--n", "96", "--wc", "3", "--wr", "6", "--seed", "1", "--out", str(out)]) == 0
    H = parse_alist(out.read_text())
    assert (H.n, H.m, H.total_edges) == (96, 48, 288)
    assert all(len(c) == 3 for c in H.col_rows()) and all(len(r) == 6 for r in H.row_cols())


@pytest.mark.gpu
def test_tables(tmp_path, capsys, cuda):   # tables are built on the GPU (no CPU fallback)
    out = tmp_path / "h.alist"
    assert cli.main(["gen", "--n", "96", "--wc", "3", "--wr", "6", "--seed", "1", "--out", str(out)]) == 0
    assert cli.main(["tables", "--code", str(out)]) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "code: n=96 m=48 edges=288" in text and text.count("e | ") == 2


def test_usage_errors(tmp_path, capsys):
    assert cli.main(["tables", "--code", str(tmp_path / "missing.alist")]) == cli.EXIT_USAGE
    bad = tmp_path / "bad.alist"
    bad.write_text("3 x\n")
    assert cli.main(["tables", "--code", str(bad)]) == cli.EXIT_USAGE
    assert "error:" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        cli.main(["frobnicate"])


@pytest.mark.gpu
def test_decode_and_ber(tmp_path, capsys, cuda):
    H = configs.code("C1")
    code = tmp_path / "c1.alist"
    code.write_text(serialize_alist(H))
    obs = tmp_path / "y.txt"
    obs.write_text("\n".join(["-1.0"] * H.n) + "\n")
    assert cli.main(["decode", "--code", str(code), "--ebno", "2", str(obs)]) == cli.EXIT_OK
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "0" * H.n and lines[1] == "success: True" and lines[2] == "iterations: 0"
    csv = tmp_path / "ber.csv"
    assert cli.main(["ber", "--code", str(code), "--ebno", "1,2", "--frames", "40", "--max-iter", "20",
                     "--batch", "16", "--out", str(csv)]) == cli.EXIT_OK
    rows = csv.read_text().splitlines()
    assert rows[0].startswith("ebno_db,sigma2,frames") and len(rows) == 3
    assert cli.main(["bench", "--code", str(code), "--frames", "8", "--max-iter", "20"]) == cli.EXIT_OK


def test_dense_format_round_trip_and_errors():
    from paper_1609_01567_b200 import CodeFormatError, parse_dense, serialize_dense

    H = configs.code("C1")
    assert parse_dense(serialize_dense(H)) == H
    with pytest.raises(CodeFormatError, match="line 2: illegal character 'x'"):
        parse_dense("0 1 1\n1 x 0\n")
    with pytest.raises(CodeFormatError, match="line 3: ragged row"):
        parse_dense("011\n\n10\n")
    with pytest.raises(CodeFormatError, match="line 1: empty matrix"):
        parse_dense("\n \n")


def test_gallager_generator_matches_reference_golden():
    # codes.py:241-294 + rng.py:84-96, against fixtures made by running the reference
    import pathlib

    from paper_1609_01567_b200 import generate_gallager_code
    from paper_1609_01567_b200.channel import derive_state, randrange, shuffle

    g = np.load(pathlib.Path(__file__).with_name("golden") / "gallager.npz")
    for k in range(int(g["cases"])):
        n, wc, wr, seed = (int(x) for x in g[f"g{k}/params"])
        H = generate_gallager_code(n, wc, wr, seed)
        assert np.array_equal(np.array(H.ones, dtype=np.int64).reshape(-1, 2), g[f"g{k}/ones"]), (n, wc, wr, seed)
    st = derive_state(5, 6, 7)
    items = list(range(50))
    st2 = shuffle(items, st)
    st3, draws = st2, []
    for b in (1, 2, 7, 1000, 2**40 + 3):
        st3, v = randrange(st3, b)
        draws.append(v)
    assert [st.s0, st.s1, st2.s0, st2.s1, st3.s0, st3.s1] == [int(x) for x in g["rng/state"]]
    assert items == [int(x) for x in g["rng/shuffled"]] and draws == [int(x) for x in g["rng/draws"]]
    with pytest.raises(ValueError):
        generate_gallager_code(10, 1, 2)
    with pytest.raises(ValueError):
        generate_gallager_code(10, 3, 7)


@pytest.mark.gpu
def test_ber_precision_and_fixed_iterations(tmp_path, cuda):
    H = configs.code("C1")
    code = tmp_path / "c1.alist"
    code.write_text(serialize_alist(H))
    for extra in (["--fixed-iters"], ["--precision", "fp32"], ["--channel", "device", "--fixed-iters"]):
        csv = tmp_path / "ber.csv"
        assert cli.main(["ber", "--code", str(code), "--ebno", "1.5", "--frames", "32", "--max-iter", "8",
                         "--batch", "32", "--out", str(csv)] + extra) == cli.EXIT_OK
        row = csv.read_text().splitlines()[1].split(",")
        if "--fixed-iters" in extra:
            assert float(row[5]) == 8.0   # mean_iterations: every frame ran the full budget
