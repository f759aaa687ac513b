"""Exception types of the drop-in surface.

Mirror lorasim's errors (include/lorasim/errors.hpp:9-24) as the reference's
Python bindings expose them: ValidationError / ConfigError / ParseError are
ValueError subclasses (bindings/module.cpp:48-50); std::logic_error surfaces
as RuntimeError (pybind11's default translation), here ``LogicError``.
"""


class ValidationError(ValueError):
    """Invalid domain values (lorasim::ValidationError)."""


class ConfigError(ValueError):
    """Bad or inconsistent configuration (lorasim::ConfigError)."""


class ParseError(ValueError):
    """Malformed input data (lorasim::ParseError)."""


class LogicError(RuntimeError):
    """Programming error / corruption (std::logic_error), e.g. double free."""
