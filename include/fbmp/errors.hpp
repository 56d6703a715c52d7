// fbmp/errors.hpp -- exception taxonomy of the fbmp:: API (reference: include/fbmp/errors.hpp).
// Status codes of the C ABI (fbmp_gpu.h) map 1:1 onto these types via throw_status().
#pragma once

#include <stdexcept>
#include <string>

namespace fbmp {

// Base of everything the pipeline throws. CLI exit-code convention of the reference:
// parameter/dimension -> 1, file -> 2, numerical -> 3.
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class DimensionError : public Error {
public:
    explicit DimensionError(const std::string& what) : Error(what) {}
};
class ParamError : public Error {
public:
    explicit ParamError(const std::string& what) : Error(what) {}
};
class NumericalError : public Error {
public:
    explicit NumericalError(const std::string& what) : Error(what) {}
};
class FormatError : public Error {
public:
    explicit FormatError(const std::string& what) : Error(what) {}
};
class IoError : public Error {
public:
    explicit IoError(const std::string& what) : Error(what) {}
};

// Device / driver failure (status 4 of the C ABI); not part of the reference taxonomy.
class DeviceError : public Error {
public:
    explicit DeviceError(const std::string& what) : Error(what) {}
};

}  // namespace fbmp
