"""Command line (paper_2601_11437_b200/cli.py) host logic: dataset formats, parse errors and
exit codes (cli.py:15-16, 83-117), RunRecord std errors (cli.py:120-151) and the benchmark
summary (cli.py:336-390) against the reference's own functions where the reference is
importable.  The GPU-backed commands are in tests/test_gpu_cli.py."""

import json

import numpy as np
import pytest

from paper_2601_11437_b200 import cli


def test_csv_round_trip_17_digits(tmp_path):
    rng = np.random.default_rng(0)
    loc, z = rng.uniform(size=(37, 2)), rng.standard_normal(37)
    path = tmp_path / "d.csv"
    cli.write_dataset(path, loc, z)
    text = path.read_bytes()
    assert text.startswith(b"x,y,z\n") and b"\r" not in text
    data = cli.read_dataset(path)
    assert np.array_equal(data.locations, loc) and np.array_equal(data.values, z)
    npz = tmp_path / "d.npz"
    cli.write_dataset(npz, loc, z)
    d2 = cli.read_dataset(npz)
    assert np.array_equal(d2.locations, loc) and np.array_equal(d2.values, z)


def test_csv_matches_reference_writer(tmp_path, reference):
    from maternmle import cli as ref_cli

    rng = np.random.default_rng(1)
    loc, z = rng.uniform(size=(11, 2)), rng.standard_normal(11)
    ours, theirs = tmp_path / "a.csv", tmp_path / "b.csv"
    cli.write_dataset(ours, loc, z)
    ref_cli.write_dataset(theirs, loc, z)
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.parametrize("body,line", [
    ("x,y\n1,2\n", 1),
    ("x,y,z\n1,2,3\n1,2\n", 3),
    ("x,y,z\n1,2,abc\n", 2),
    ("x,y,z\n", 2),
    ("x,y,z\n0,0,1\n1,1,inf\n", 2),
])
def test_dataset_format_errors(tmp_path, body, line):
    path = tmp_path / "bad.csv"
    path.write_text(body)
    with pytest.raises(cli.DatasetFormatError) as info:
        cli.read_dataset(path)
    assert info.value.line == line
    assert cli.main(["loglik", str(path), "--theta", "1,0.1,0.5"]) == 2


def test_parse_errors_exit_2(tmp_path, capsys):
    path = tmp_path / "d.csv"
    cli.write_dataset(path, np.array([[0.0, 0.0], [1.0, 0.0]]), np.array([0.1, -0.2]))
    assert cli.main(["loglik", str(path), "--theta", "1,0.1"]) == 2
    assert cli.main(["loglik", str(path), "--theta", "1,-0.1,0.5"]) == 2
    assert cli.main(["estimate", str(path), "--lower", "1,1,1", "--upper", "0.5,1,1"]) == 2
    assert cli.main(["simulate", str(tmp_path / "s.csv"), "--n", "10", "--theta", "1,0.1,0.5"]) == 2
    assert cli.main(["benchmark", "--theta", "1,0.1,0.5", "--n", "10", "--m", "1",
                     "--out-dir", str(tmp_path / "b")]) == 2
    assert "error:" in capsys.readouterr().err


def test_std_errors_match_reference(reference):
    from maternmle import cli as ref_cli

    rng = np.random.default_rng(2)
    a = rng.standard_normal((3, 3))
    for info in (a @ a.T + 0.1 * np.eye(3), -np.eye(3), np.diag([1.0, 2.0, 0.0])):
        assert cli._std_errors(info) == ref_cli._std_errors(info)


def test_summary_matches_reference(reference):
    """Same per-replicate records -> the same summary rows as the reference's _summarize."""
    from maternmle import cli as ref_cli

    rng = np.random.default_rng(3)
    thetas = [reference.MaternParams(1.0, 0.1, 0.5), reference.MaternParams(0.7, 0.2, 1.3)]
    sizes = [16, 25]
    results = []
    for ti in range(2):
        for ni in range(2):
            for rep in range(3):
                recs = []
                for method in ("fisher-bt", "nelder-mead"):
                    if rep == 2 and method == "nelder-mead":
                        recs.append({"method": method, "seed": rep, "error": "failed"})
                        continue
                    th = rng.uniform(0.05, 2.0, 3)
                    recs.append({"method": method,
                                 "theta_hat": {"sigma2": th[0], "alpha": th[1], "nu": th[2]},
                                 "loglik": float(rng.normal(-100, 5)),
                                 "loglik_calls": int(rng.integers(9, 40)),
                                 "grad_calls": int(rng.integers(1, 12)),
                                 "wall_time": float(rng.uniform(0.1, 2.0))})
                results.append({"theta_index": ti, "n_index": ni, "replicate": rep,
                                "records": recs})
    methods = ["fisher-bt", "nelder-mead"]
    ours = cli._summarize(results, thetas, sizes, methods)
    theirs = ref_cli._summarize(json.loads(json.dumps(results)), thetas, sizes, methods)
    assert ours == theirs


def test_parser_surface_matches_reference(reference):
    """Every subcommand and option of the reference CLI exists here with the same default."""
    from maternmle import cli as ref_cli

    def table(parser):
        sub = next(a for a in parser._actions if a.__class__.__name__ == "_SubParsersAction")
        return {name: {a.dest: a.default for a in p._actions if a.dest != "help"}
                for name, p in sub.choices.items()}

    ours, theirs = table(cli.build_parser()), table(ref_cli.build_parser())
    assert set(ours) == set(theirs)
    for cmd, opts in theirs.items():
        for dest, default in opts.items():
            if dest == "func":
                continue
            assert dest in ours[cmd], (cmd, dest)
            assert ours[cmd][dest] == default, (cmd, dest)
