// A minimal GoogleTest-compatible shim (GoogleTest is absent from this image,
// SURVEY.md section 4): TEST, EXPECT_* / ASSERT_* with streamed messages,
// EXPECT_THROW. Enough to compile the reference's unmodified
// proj/tests/test_ple.cpp against the B200 binding (tests/cpp/b200_redirect.hpp).
// ASSERT_* returns from the enclosing void function, as in GoogleTest.
#pragma once

#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gtshim {

struct TestCase {
    std::string name;
    void (*body)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

inline int& current_failures() {
    static int n = 0;
    return n;
}

struct Reg {
    Reg(const char* name, void (*body)()) { registry().push_back({name, body}); }
};

class Message {
public:
    template <class T>
    Message& operator<<(const T& v) {
        ss_ << v;
        return *this;
    }
    std::string str() const { return ss_.str(); }

private:
    std::ostringstream ss_;
};

struct Helper {
    const char* file;
    int line;
    const char* what;
    void operator=(const Message& m) const {
        ++current_failures();
        std::printf("%s:%d: Failure: %s %s\n", file, line, what, m.str().c_str());
    }
};

template <class E>
bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

}  // namespace gtshim

namespace testing {
inline void InitGoogleTest(int*, char**) {}
}  // namespace testing

#define GTS_NONFATAL(cond, text) \
    if (cond)                    \
        ;                        \
    else                         \
        ::gtshim::Helper{__FILE__, __LINE__, text} = ::gtshim::Message()
#define GTS_FATAL(cond, text) \
    if (cond)                 \
        ;                     \
    else                      \
        return ::gtshim::Helper{__FILE__, __LINE__, text} = ::gtshim::Message()

#define EXPECT_TRUE(c) GTS_NONFATAL(bool(c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GTS_NONFATAL(!bool(c), "EXPECT_FALSE(" #c ")")
#define EXPECT_EQ(a, b) GTS_NONFATAL((a) == (b), "EXPECT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GTS_NONFATAL((a) != (b), "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GTS_NONFATAL((a) < (b), "EXPECT_LT(" #a ", " #b ")")
#define EXPECT_LE(a, b) GTS_NONFATAL((a) <= (b), "EXPECT_LE(" #a ", " #b ")")
#define EXPECT_GT(a, b) GTS_NONFATAL((a) > (b), "EXPECT_GT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GTS_NONFATAL((a) >= (b), "EXPECT_GE(" #a ", " #b ")")
#define ASSERT_TRUE(c) GTS_FATAL(bool(c), "ASSERT_TRUE(" #c ")")
#define ASSERT_FALSE(c) GTS_FATAL(!bool(c), "ASSERT_FALSE(" #c ")")
#define ASSERT_EQ(a, b) GTS_FATAL((a) == (b), "ASSERT_EQ(" #a ", " #b ")")
#define ASSERT_NE(a, b) GTS_FATAL((a) != (b), "ASSERT_NE(" #a ", " #b ")")
#define ASSERT_LT(a, b) GTS_FATAL((a) < (b), "ASSERT_LT(" #a ", " #b ")")
#define ASSERT_LE(a, b) GTS_FATAL((a) <= (b), "ASSERT_LE(" #a ", " #b ")")
#define ASSERT_GT(a, b) GTS_FATAL((a) > (b), "ASSERT_GT(" #a ", " #b ")")
#define ASSERT_GE(a, b) GTS_FATAL((a) >= (b), "ASSERT_GE(" #a ", " #b ")")
#define EXPECT_THROW(stmt, exc) \
    GTS_NONFATAL(::gtshim::throws<exc>([&] { stmt; }), "EXPECT_THROW(" #stmt ", " #exc ")")
#define ASSERT_THROW(stmt, exc) \
    GTS_FATAL(::gtshim::throws<exc>([&] { stmt; }), "ASSERT_THROW(" #stmt ", " #exc ")")

#define GTS_CAT2(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT2(a, b)
#define TEST(suite, name)                                                                   \
    static void GTS_CAT(gts_body_, GTS_CAT(suite, GTS_CAT(_, name)))();                    \
    static ::gtshim::Reg GTS_CAT(gts_reg_, GTS_CAT(suite, GTS_CAT(_, name)))(              \
        #suite "." #name, &GTS_CAT(gts_body_, GTS_CAT(suite, GTS_CAT(_, name))));          \
    static void GTS_CAT(gts_body_, GTS_CAT(suite, GTS_CAT(_, name)))()
