"""The reference-side adapter (dropin/minikv_reference_adapter.cpp) compiles against the
reference's own unchanged headers and defines the reference's hot-path symbols
(namespace minikv, exact signatures) on top of the B200 C++ API.  CPU only; skipped
where the reference headers are absent (the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFINC = "/root/reference/proj/core/include"


@pytest.mark.skipif(not os.path.exists(os.path.join(REFINC, "minikv", "attention.hpp")),
                    reason="reference headers not present")
def test_adapter_compiles_against_reference_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "dropin")], check=True)
    obj = os.path.join(ROOT, "dropin", "build", "minikv_reference_adapter.o")
    syms = subprocess.run(["nm", "-C", "--defined-only", obj], capture_output=True, text=True).stdout
    for sig in ["minikv::selective_flash_attn(minikv::Matrix const&, minikv::Matrix const&, minikv::Matrix const&, "
                "float, bool, minikv::TileConfig)",
                "minikv::select_token_counts(std::vector<float, std::allocator<float> > const&, unsigned long, "
                "unsigned long)",
                "minikv::allocate_pyramid(unsigned long, unsigned long, unsigned long, minikv::PyramidOrientation)",
                "minikv::allocate_variance(", "minikv::layer_score_variance(", "minikv::prefill(",
                "minikv::select_tokens("]:
        assert sig in syms, sig
