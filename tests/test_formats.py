"""Text formats (rules.hpp:87-103): round trips and errors."""
import io

import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from oracle import binding as ob
from paper_2205_04401_b200 import formats


def test_mesh_round_trip_is_bit_exact(tmp_path):
    pr = vp.load_config(1, with_rules=False)
    p = tmp_path / "m.txt"
    formats.write_mesh(p, pr.vxy, pr.tri)
    v, t, b = formats.read_mesh(p)
    assert np.array_equal(v, pr.vxy) and np.array_equal(t, pr.tri)


def test_mesh_errors(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("3\n")
    with pytest.raises(ValueError, match="header"):
        formats.read_mesh(p)
    p.write_text("1 1\nv 0 0 0\ne 0 1 2 0\n")
    with pytest.raises(ValueError, match="out of range"):
        formats.read_mesh(p)


def test_rule_table_round_trip_and_validation():
    x, y, w = vp.simplex_rule(12)
    buf = io.StringIO()
    formats.write_rule(buf, "X-G", 12, x, y, w)
    buf.seek(0)
    kind, order, x2, y2, w2 = formats.read_rule(buf)
    assert kind == "X-G" and order == 12
    assert np.array_equal(x, x2) and np.array_equal(w, w2)
    ob.validate_rule(order, x2, y2, w2)
    with pytest.raises(ValueError, match="truncated"):
        formats.read_rule(io.StringIO("X-G 12 49\n0.1 0.1 0.1\n"))
    with pytest.raises(ValueError, match="unknown kind"):
        formats.read_rule(io.StringIO("ABC 12 1\n0.1 0.1 0.5\n"))


def test_csv_writers(tmp_path):
    formats.write_nodes_csv(tmp_path / "n.csv", np.array([[0.5, 0.25]]), [1.5])
    assert (tmp_path / "n.csv").read_text().splitlines() == ["x,y,u", "0.5,0.25,1.5"]
    formats.write_sweep_csv(tmp_path / "s.csv", [dict(Nf=16, TF=1.0, TN=2.0, TS=3.0, Ttot=6.0, c=2.5, sn=20.0)])
    assert (tmp_path / "s.csv").read_text().splitlines()[0] == "Nf,TF,TN,TS,Ttot,c,sn"
