"""Writes the regression fixtures under tests/golden/ by calling ONLY oracle/.

ico_ref0_faces.json: the base icosahedron's face table under the orientation
rule of DESIGN.md reading R1 (faces = lexicographic vertex triples, stored
counter-clockwise seen from outside).  Its independent pins are
test_faces_counter_clockwise_from_outside and test_ref0_faces_lexicographic.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

h = oracle.Hierarchy(0, 0, 1, 0.01, 1e-4, np.ones((1, 20)))
faces = h.level(0)["faces"].tolist()
with open(os.path.join(HERE, "ico_ref0_faces.json"), "w") as fh:
    json.dump({"source": "oracle/hmg_oracle.c base_mesh(); reading R1 (SURVEY 8(c).2 O1)",
               "faces": faces}, fh, indent=1)
