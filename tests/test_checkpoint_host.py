"""cache_load's file checks run before any device work (no GPU needed): a missing file, a
foreign file and a truncated header are refused with CACHE_E_INVALID_ARG and no handle."""
import pytest


@pytest.mark.parametrize("content", [None, b"hello world" * 100, b"NVCACHE1"])
def test_load_refuses_bad_files(tmp_path, content):
    from paper_2312_04429_b200 import binding as B
    p = tmp_path / "x.snap"
    if content is not None:
        p.write_bytes(content)
    with pytest.raises(B.CacheError) as ei:
        B.NirvanaCache.load(str(p), device=0)
    assert ei.value.code == B.E_INVALID_ARG
