"""The drop-in on the reference's OWN classes: hefir (installed unmodified in
baseline/_ref, gmpy2 shimmed) builds the parameters, keys, ciphertexts and
model; the GPU engine evaluates them through the reference's layer API
(engine.eval_network, engine.py:400-423; bfv.hsquare / relinearize /
hmult_raw, bfv.py:368-443) and must return hefir's own CipherTensor /
Ciphertext / RingElem objects holding exactly the residues hefir itself
computes."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from conftest import import_installed_reference  # noqa: E402

from paper_1811_00778_b200 import engine as E  # noqa: E402
from paper_1811_00778_b200 import ops  # noqa: E402

SET1_PRIMES = [1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641,
               1071513601, 1071415297, 1071087617, 1070727169, 1070432257]
MNIST_T = 5522259017729


@pytest.fixture(scope="module")
def ref_world():
    hefir = import_installed_reference()
    from hefir import bfv, engine, nn_oracle, ring
    from hefir.batching import SlotEncoder

    n = 1024
    params = bfv.BfvParams(ring.RnsContext(n, SET1_PRIMES), MNIST_T)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(2101))
    images = [np.random.default_rng(2102 + i).integers(0, 5, (8, 8, 1)) for i in range(6)]
    enc = SlotEncoder(MNIST_T, n)
    tin = engine.pack_images(images, engine.PackingLayout(6, n), enc, pk, params,
                             np.random.default_rng(2110), delta=4)
    spec = nn_oracle.toy_hcnn()
    wrng = np.random.default_rng(2111)
    weights = []
    shapes = {"conv1": (spec.layers[0].filters, 3, 3, 1)}
    for layer in spec.layers:
        if layer.kind is nn_oracle.LayerKind.CONV:
            weights.append(wrng.integers(-15, 16, shapes[layer.name]))
        elif layer.kind is nn_oracle.LayerKind.FC:
            weights.append(wrng.integers(-15, 16, (layer.filters, 3 * 3 * spec.layers[0].filters)))
        else:
            weights.append(None)
    model = nn_oracle.QuantizedModel(spec=spec, bit_width=4, weights=weights)
    return dict(hefir=hefir, bfv=bfv, engine=engine, ring=ring, params=params, sk=sk, rlk=rlk,
                tin=tin, model=model, enc=enc, images=images)


def _res(ct):
    return np.stack([p.residues for p in ct.parts])


def test_eval_network_on_hefir_objects_returns_hefir_objects(ref_world):
    w = ref_world
    engine = w["engine"]
    ref_counter = engine.OpCounter()
    seen_ref = {}
    exp = engine.eval_network(w["tin"], w["model"], w["rlk"], w["params"], ref_counter,
                              layer_hook=lambda name, t: seen_ref.__setitem__(name, [_res(c) for c in t.cts]))
    counter = engine.OpCounter()  # the caller's own counter class
    seen = {}
    got = E.eval_network(w["tin"], w["model"], w["rlk"], w["params"], counter,
                         layer_hook=lambda name, t: seen.__setitem__(name, t.residues().astype(np.int64)))
    assert type(got) is engine.CipherTensor
    assert type(got.cts[0]) is w["bfv"].Ciphertext
    assert type(got.cts[0].parts[0]) is w["ring"].RingElem
    assert got.shape == exp.shape and got.delta == exp.delta and got.channel_modulus == exp.channel_modulus
    for a, b in zip(got.cts, exp.cts):
        assert np.array_equal(_res(a), _res(b))
    for name, cts in seen_ref.items():
        assert np.array_equal(seen[name], np.stack(cts)), name
    assert counter.__dict__ == ref_counter.__dict__
    vals = engine.unpack_tensor(got, w["sk"], w["enc"], w["params"], len(w["images"]))
    assert np.array_equal(vals, engine.unpack_tensor(exp, w["sk"], w["enc"], w["params"], len(w["images"])))


def test_per_ciphertext_ops_on_hefir_objects(ref_world):
    w = ref_world
    bfv, params, rlk = w["bfv"], w["params"], w["rlk"]
    c0, c1 = w["tin"].cts[0], w["tin"].cts[5]
    raw = ops.hmult_raw(c0, c1, params)
    raw_ref = bfv.hmult_raw(c0, c1, params)
    assert type(raw) is bfv.Ciphertext and np.array_equal(_res(raw), _res(raw_ref))
    rel = ops.relinearize(raw_ref.parts, rlk, params)
    rel_ref = bfv.relinearize(raw_ref.parts, rlk, params)
    assert type(rel) is bfv.Ciphertext and type(rel.parts[0]) is w["ring"].RingElem
    assert np.array_equal(_res(rel), _res(rel_ref))
    sq = ops.hsquare(c1, rlk, params)
    assert type(sq) is bfv.Ciphertext and np.array_equal(_res(sq), _res(bfv.hsquare(c1, rlk, params)))
    sq3 = ops.hsquare(raw_ref, rlk, params)  # 3-part input: relinearised first, caller's class out
    assert type(sq3) is bfv.Ciphertext
    assert np.array_equal(_res(sq3), _res(bfv.hsquare(rel_ref, rlk, params)))
