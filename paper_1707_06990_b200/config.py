"""Named presets and the flat key=value config text.

Restates densenet.hpp:86-115 (`preset_config`) and densenet.hpp:276-377
(`config_to_text`, `parse_key_values`, `parse_int_list`,
`config_from_key_values`, `config_from_file`), with the reference's error
classes and messages.  Numbers parse the way std::stoi / std::stod do:
leading whitespace skipped, the longest numeric prefix taken, trailing text
ignored.  Missing keys take the reference's DenseNetConfig defaults (growth
12, no bottleneck, compression 1, 24 initial channels, pre-activation, 10
classes).  tests/test_config.py pins every function against the reference's
own output (tests/golden/config_kats.json, oracle/gen_golden.py).
"""
from __future__ import annotations

import math
import re

from .errors import ConfigError, FormatError
from .model import DenseNetConfig

# std::isspace in the "C" locale
_SPACE = " \t\n\v\f\r"


def build_config(blocks, growth_rate: int, bottleneck: bool, compression: float, activation: str,
                 num_classes: int, initial_channels: int = -1) -> DenseNetConfig:
    """densenet.hpp:71-85: initial channels default to 2k; validated."""
    cfg = DenseNetConfig(tuple(blocks), growth_rate, bottleneck, compression, num_classes,
                         initial_channels if initial_channels > 0 else 2 * growth_rate, activation=activation)
    validate(cfg)
    return cfg


def validate(cfg: DenseNetConfig) -> None:
    """DenseNetConfig::validate (densenet.hpp:55-66)."""
    if not cfg.block_sizes:
        raise ConfigError("no dense blocks configured")
    for m in cfg.block_sizes:
        if m < 1:
            raise ConfigError("block size must be >= 1")
    if cfg.growth_rate < 1:
        raise ConfigError("growth rate must be >= 1")
    if cfg.initial_channels < 1:
        raise ConfigError("initial channels must be >= 1")
    if not (cfg.compression > 0.0) or cfg.compression > 1.0:
        raise ConfigError("compression must be in (0, 1]")
    if cfg.num_classes < 1:
        raise ConfigError("num_classes must be >= 1")


_PRESETS = {
    "desk": (([2, 2, 2], 4, False, 1.0, "pre", 4), {}),
    "tiny": (([2], 4, False, 1.0, "pre", 4), {"initial_channels": 8}),
    "paper-264-k48": (([6, 32, 64, 48], 48, True, 0.5, "pre", 1000), {}),
    "paper-264-k32": (([6, 32, 64, 48], 32, True, 0.5, "pre", 1000), {}),
    "paper-232-k48": (([6, 32, 48, 48], 48, True, 0.5, "pre", 1000), {}),
    "bc-160-k12": (([26, 26, 26], 12, True, 0.5, "pre", 10), {}),
}


def preset_config(name: str) -> DenseNetConfig:
    """preset_config (densenet.hpp:89-115)."""
    if name not in _PRESETS:
        raise ConfigError(f"unknown preset '{name}'")
    args, kw = _PRESETS[name]
    return build_config(*args, **kw)


def _fmt_double(x: float) -> str:
    """std::ostream << double with the default format (%g, precision 6)."""
    if math.isnan(x):
        return "-nan" if math.copysign(1.0, x) < 0 else "nan"
    if math.isinf(x):
        return "-inf" if x < 0 else "inf"
    return "%g" % x


def config_to_text(cfg: DenseNetConfig) -> str:
    """config_to_text (densenet.hpp:279-297)."""
    return ("blocks=" + ",".join(str(m) for m in cfg.block_sizes) + "\n"
            f"growth_rate={cfg.growth_rate}\n"
            f"bottleneck={1 if cfg.bottleneck else 0}\n"
            f"compression={_fmt_double(cfg.compression)}\n"
            f"initial_channels={cfg.initial_channels}\n"
            f"activation={'pre' if cfg.activation == 'pre' else 'post'}\n"
            f"num_classes={cfg.num_classes}\n")


def parse_key_values(text: str) -> dict:
    """parse_key_values (densenet.hpp:300-323): '#' starts a comment, lines are
    trimmed, blank lines skipped, the first '=' splits key and value (neither
    trimmed further), a later duplicate key wins."""
    kv = {}
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline yields no line after a final newline
    for lineno, line in enumerate(lines, start=1):
        hash_ = line.find("#")
        if hash_ >= 0:
            line = line[:hash_]
        line = line.strip(_SPACE)
        if not line:
            continue
        eq = line.find("=")
        if eq < 0:
            raise FormatError(f"config line {lineno} is not key=value: '{line}'")
        kv[line[:eq]] = line[eq + 1:]
    return kv


class _StdError(Exception):
    """std::invalid_argument / std::out_of_range from std::stoi / std::stod."""


_INT = re.compile(r"[ \t\n\v\f\r]*([+-]?\d+)")
_DEC = r"(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?"
_HEX = r"0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?"
_FLOAT = re.compile(r"[ \t\n\v\f\r]*([+-]?)(" + _HEX + r"|" + _DEC +
                    r"|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)", re.IGNORECASE)


def _stoi(s: str) -> int:
    m = _INT.match(s)
    if not m:
        raise _StdError("stoi")
    v = int(m.group(1))
    if not -2 ** 31 <= v < 2 ** 31:
        raise _StdError("stoi")
    return v


def _stod(s: str) -> float:
    m = _FLOAT.match(s)
    if not m:
        raise _StdError("stod")
    sign, body = m.group(1), m.group(2)
    low = body.lower()
    if low.startswith("inf"):
        v = math.inf
    elif low.startswith("nan"):
        v = math.nan
    elif low.startswith("0x"):
        v = float.fromhex(body)
    else:
        v = float(body)
        mant = re.sub(r"[eE].*", "", body)
        if math.isinf(v) or (v == 0.0 and re.search(r"[1-9]", mant)):
            raise _StdError("stod")  # ERANGE: overflow / underflow to zero
    return -v if sign == "-" else v


def parse_int_list(s: str) -> list:
    """parse_int_list (densenet.hpp:325-336): comma items as std::getline splits them."""
    items = s.split(",")
    if items and items[-1] == "":
        items.pop()  # no item after a trailing comma (or for an empty string)
    out = []
    for item in items:
        try:
            out.append(_stoi(item))
        except _StdError:
            raise FormatError(f"bad integer '{item}' in list '{s}'") from None
    return out


def config_from_key_values(kv: dict) -> DenseNetConfig:
    """config_from_key_values (densenet.hpp:338-370), then validate()."""
    f = {"block_sizes": [], "growth_rate": 12, "bottleneck": False, "compression": 1.0,
         "initial_channels": 24, "activation": "pre", "num_classes": 10}
    try:
        if "blocks" in kv:
            f["block_sizes"] = parse_int_list(kv["blocks"])
        if "growth_rate" in kv:
            f["growth_rate"] = _stoi(kv["growth_rate"])
        if "bottleneck" in kv:
            f["bottleneck"] = _stoi(kv["bottleneck"]) != 0
        if "compression" in kv:
            f["compression"] = _stod(kv["compression"])
        if "initial_channels" in kv:
            f["initial_channels"] = _stoi(kv["initial_channels"])
        if "activation" in kv:
            if kv["activation"] not in ("pre", "post"):
                raise FormatError("activation must be 'pre' or 'post'")
            f["activation"] = kv["activation"]
        if "num_classes" in kv:
            f["num_classes"] = _stoi(kv["num_classes"])
    except _StdError as e:
        raise FormatError(f"bad config value: {e}") from None
    cfg = DenseNetConfig(tuple(f["block_sizes"]), f["growth_rate"], f["bottleneck"], f["compression"],
                         f["num_classes"], f["initial_channels"], activation=f["activation"])
    validate(cfg)
    return cfg


def config_from_text(text: str) -> DenseNetConfig:
    return config_from_key_values(parse_key_values(text))


def config_from_file(path: str) -> DenseNetConfig:
    """config_from_file (densenet.hpp:372-376)."""
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise FormatError(f"cannot open config file '{path}'") from None
    return config_from_text(text)
