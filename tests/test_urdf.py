"""Host front end: our URDF parser reproduces the reference parser's models
(golden fixtures) and its error taxonomy (reference urdf.py:22-39)."""
import numpy as np
import pytest

from conftest import MODELS, golden
from paper_2109_06976_b200 import models, schedule, urdf


@pytest.mark.parametrize("name", MODELS)
def test_parser_matches_reference_model(name):
    g = golden(name)
    m = models.load(name)
    assert list(g["parent"]) == m.parent
    assert [str(k) for k in g["kind"]] == [j.kind for j in m.joints]
    for key, get in (("axis", lambda j, i: j.axis), ("origin_rotation", lambda j, i: j.origin_rotation),
                     ("origin_translation", lambda j, i: j.origin_translation)):
        assert np.allclose(g[key], [get(j, i) for i, j in enumerate(m.joints)], rtol=0, atol=1e-15)
    assert np.allclose(g["mass"], [i.mass for i in m.inertias], rtol=0, atol=1e-15)
    assert np.allclose(g["com"], [i.com for i in m.inertias], rtol=0, atol=1e-15)
    assert np.allclose(g["icom"], [i.inertia_about_com for i in m.inertias], rtol=0, atol=1e-15)
    assert np.allclose(g["gravity"], m.gravity)


def _robot(body):
    return f'<robot name="t"><link name="base"/>{body}</robot>'


def _link(name, mass=1.0, xyz="0 0 0"):
    return (f'<link name="{name}"><inertial><origin xyz="{xyz}"/><mass value="{mass}"/>'
            '<inertia ixx="0.01" iyy="0.01" izz="0.01" ixy="0" ixz="0" iyz="0"/></inertial></link>')


def _joint(name, kind, parent, child, xyz="0 0 0"):
    return (f'<joint name="{name}" type="{kind}"><parent link="{parent}"/><child link="{child}"/>'
            f'<origin xyz="{xyz}"/><axis xyz="0 0 1"/></joint>')


def test_errors():
    with pytest.raises(urdf.UrdfParseError, match="line"):
        urdf.parse_urdf("<robot><link name='a'></robot>")
    with pytest.raises(urdf.UnsupportedFeatureError):
        urdf.parse_urdf(_robot(_link("a") + _joint("j", "floating", "base", "a")))
    with pytest.raises(urdf.TopologyError):
        urdf.parse_urdf(_robot(_link("a") + _joint("j", "revolute", "base", "zz")))
    with pytest.raises(urdf.TopologyError):
        urdf.parse_urdf(_robot(_link("a") + _link("b") + _joint("j", "revolute", "base", "a")))
    with pytest.raises(urdf.ModelValidationError):
        urdf.parse_urdf(_robot(_link("a") + _link("a")))
    with pytest.raises(urdf.UrdfError):
        urdf.parse_urdf(_robot(_link("a") + _joint("j", "revolute", "base", "a")
                               + _joint("j", "revolute", "base", "a")))


def test_fixed_fusion_and_continuous():
    # fused masses add; a massless parent takes the child's com
    body = (_link("a", 1.0) + _link("b", 2.0) + _link("c", 1.0) + _link("d", 0.0)
            + _joint("j0", "continuous", "base", "a") + _joint("j1", "fixed", "a", "b")
            + _joint("j2", "revolute", "b", "d", "0 0 1") + _joint("j3", "fixed", "d", "c", "1 0 0"))
    m = urdf.parse_urdf(_robot(body))
    assert m.n_frames == 2 and m.parent == [-1, 0]
    assert m.joints[0].kind == "revolute"
    assert m.inertias[0].mass == pytest.approx(3.0)
    assert m.inertias[1].mass == pytest.approx(1.0)
    assert np.allclose(m.inertias[1].com, [1, 0, 0])


def test_topology_and_levels():
    assert urdf.classify_topology(models.load("chain7")) == "serial_chain"
    assert urdf.classify_topology(models.load("quad12")) == "branched_tree"
    # SPEC.md:560 (paper Fig. 2)
    assert schedule.build_levels(models.load("tree7")).levels == [[0], [1, 5], [2, 4, 6], [3]]
    # quad12 retains <= 40% of the dense gradient temporaries
    assert schedule.analyze_sparsity(models.load("quad12"), "gradFD").retained_fraction() <= 0.4
    m = models.load("humanoid30")
    assert [len(m.subtree(r)) for r in m.roots()] == [16, 7, 7]
