// Precondition checks of the host library.  The exception classes are the
// reference's contract (std::invalid_argument, domain_error, length_error,
// out_of_range, overflow_error, runtime_error, logic_error: SURVEY.md
// section 8(b)); the messages are this library's.  The message expression is
// evaluated only when the check fails.
#pragma once

#include <stdexcept>
#include <string>

#define QPK_REQUIRE(cond, Exception, message)    \
    do {                                          \
        if (!(cond)) throw Exception(message);    \
    } while (0)

#include <sstream>

#include "qpack/common.hpp"

namespace qpack::detail {

// a message from its parts: text and numbers (u128 in decimal)
inline void put_part(std::ostringstream& os, u128 v) { os << to_string(v); }
template <class T>
void put_part(std::ostringstream& os, const T& v) {
    os << v;
}

template <class... Parts>
std::string cat(const Parts&... parts) {
    std::ostringstream os;
    (put_part(os, parts), ...);
    return os.str();
}

}  // namespace qpack::detail
