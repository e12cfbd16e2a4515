"""CPU: the per-window driver's predictor (predictor.hpp:39-91 restated in
paper_2407_13126_b200/driver.py) against the forecasts the unmodified
reference produced in the same loop (tests/golden/drive/), plus its error codes."""
import json
import os

import numpy as np
import pytest

from paper_2407_13126_b200 import driver
from paper_2407_13126_b200 import scenario as SC

D = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "drive")


def test_forecasts_match_reference():
    gold = json.load(open(os.path.join(D, "drive_golden.json")))
    n = 0
    for stem in ("d_c1_40", "d_c1_40v"):
        sc = SC.load_scenario(os.path.join(D, stem + ".scn"))
        S = sc.window_size
        for pred in ("oracle", "persistence", "ewma:0.3"):
            spec = driver.parse_predictor(pred)
            for w, want in enumerate(gold[stem][pred]["windows"]):
                actual = np.stack([sc.window_arrivals(m, w) for m in range(len(sc.models))])
                if spec[0] == "oracle" or w == 0:
                    fc = driver.predict_arrivals(("oracle", 0.0), None, S, S, actual)
                else:
                    fc = driver.predict_arrivals(spec, sc.counts[:, :w * S], S, S)
                assert fc.tolist() == want["forecast"], (stem, pred, w)
                n += 1
    assert n == 18


def test_predictor_errors_and_rounding():
    with pytest.raises(driver.PredictorError) as e:
        driver.parse_predictor("ewma:0")
    assert e.value.code == "input.predictor"
    with pytest.raises(driver.PredictorError) as e:
        driver.parse_predictor("lstm")
    assert e.value.code == "input.predictor"
    with pytest.raises(driver.PredictorError) as e:
        driver.predict_arrivals(("persistence", 0.0), np.zeros((1, 3), np.int64), 4, 4)
    assert e.value.code == "predictor.history"
    # ewma over two windows, alpha 0.5: (1 + 2)/2 = 1.5 rounds half up
    fc = driver.predict_arrivals(("ewma", 0.5), np.array([[1, 4, 2, 4]]), 2, 2)
    assert fc.tolist() == [[2, 4]]
    assert driver._llround(2.4999999999999996) == 2 and driver._llround(0.5) == 1
